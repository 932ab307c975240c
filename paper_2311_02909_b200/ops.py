"""Device implementations of the reference's sparse/sampling operators."""

from __future__ import annotations

import numpy as np

from . import _lib


def uniforms(seed, epoch, depth, rows, t):
    """u(seed, epoch, depth, row, t) on the device (gb_uniforms)."""
    import torch

    rows = torch.as_tensor(np.asarray(rows, dtype=np.int64)).cuda()
    t = torch.as_tensor(np.asarray(t, dtype=np.int64)).cuda()
    out = torch.empty(rows.numel(), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().gb_uniforms(int(seed), int(epoch), int(depth), _lib.ptr(rows),
                                      _lib.ptr(t), rows.numel(), _lib.ptr(out),
                                      _lib.stream_ptr()), "gb_uniforms")
    return out.cpu().numpy()
