"""Row-reuse statistics of one SAGE bulk (products shape, k=64): per layer
the gathered entries over all rows vs over distinct vertices."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2311_02909_b200 import graphgen
    from paper_2311_02909_b200.engine import SageBulk
    from paper_2311_02909_b200.pipeline import make_batches

    n, m, sym = graphgen.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "products"]
    dg = graphgen.rmat_device_graph(n, m, symmetric=sym, seed=0)
    batches = make_batches(np.arange(n), 1024, 0, 0)[:64]
    off = np.zeros(65, np.int64)
    off[1:] = np.cumsum([len(b) for b in batches])
    d_off = torch.as_tensor(off).cuda()
    d_cat = torch.as_tensor(np.concatenate(batches).astype(np.int32)).cuda()
    bulk = SageBulk(dg, 64, int(off[-1]), 1024, (15, 10, 5), mode="pfree")
    bulk.launch(d_off, d_cat, 0, 0, 0)
    sizes = bulk.sizes.cpu().numpy()
    deg = dg.rowptr[1:] - dg.rowptr[:-1]
    rv = d_cat
    for l in range(3):
        R = int(sizes[3 * l])
        v = rv[:R].long()
        G = int(deg[v].sum())
        u = torch.unique(v)
        Gd = int(deg[u].sum())
        print(f"layer {l + 1}: rows {R} distinct {u.numel()} G_rows {G} G_distinct {Gd} "
              f"ratio {G / max(Gd, 1):.2f}")
        rv = bulk.out[l]["fcol"]


if __name__ == "__main__":
    main()
