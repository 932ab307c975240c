"""Minimal driver for ncu: build the products-shape graph, run `--warm`
eager bulks then `--iters` more (same stream).

SAGE kernel order per layer: prep, scans, k_sage_pick, [k_sage_stream],
extraction.  LADIES (--sampler ladies, b = s = 512, race mode): count,
compaction, race keys + select, emit, extraction."""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--sampler", default="sage")
    p.add_argument("--mode", default=None)
    p.add_argument("--workload", default="products")
    p.add_argument("--k", type=int, default=64)
    p.add_argument("--warm", type=int, default=2)
    p.add_argument("--iters", type=int, default=1)
    a = p.parse_args()
    import torch

    from paper_2311_02909_b200 import graphgen
    from paper_2311_02909_b200.engine import LadiesBulk, SageBulk
    from paper_2311_02909_b200.pipeline import make_batches

    n, m, sym = graphgen.SHAPES[a.workload]
    dg = graphgen.rmat_device_graph(n, m, symmetric=sym, seed=0)
    b = 1024 if a.sampler == "sage" else 512
    batches = make_batches(np.arange(n), b, 0, 0)[:a.k]
    if a.sampler == "ladies":
        batches = [np.sort(x) for x in batches]
    off = np.zeros(a.k + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in batches])
    d_off = torch.as_tensor(off).cuda()
    d_cat = torch.as_tensor(np.concatenate(batches).astype(np.int32)).cuda()
    if a.sampler == "sage":
        bulk = SageBulk(dg, a.k, int(off[-1]), 1024, (15, 10, 5), mode=a.mode or "stream")
    else:
        bulk = LadiesBulk(dg, a.k, int(off[-1]), (512,) * 3, mode=a.mode or "race")
    for _ in range(a.warm + a.iters):
        bulk.launch(d_off, d_cat, 0, 0, 0)
    torch.cuda.synchronize()
    print("sizes", bulk.sizes.cpu().numpy().tolist())


if __name__ == "__main__":
    main()
