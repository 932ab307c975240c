"""Debug: reference test_acceptance test_09 configurations through the package."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def d_regular_graph(gb, n, d, seed):
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for v in range(n):
        nb = rng.choice(np.delete(np.arange(n), v), size=d, replace=False)
        src += [v] * d
        dst += nb.tolist()
    return gb.Graph.from_edges(n, src, dst)


def main():
    import paper_2311_02909_b200 as gb
    from oracle import oracle as O

    n, b = 230, 7
    G = d_regular_graph(gb, n, 5, 9)
    A = G.adjacency
    for k in (0, 1, 2, 4, 5, 8, 33):
        for mode in ("dedup", "pfree", "stream"):
            rng = np.random.default_rng(k)
            batches = [rng.permutation(n)[:b] for _ in range(k)]
            cfg = gb.SamplerConfig.sage(2, b, (3, 2), bulk_count=max(k, 1), seed=19)
            print("k", k, mode, flush=True)
            ep = gb.sample_epoch_bulk(G, cfg, batches, mode=mode)
            if k:
                want = O.sage_bulk(n, A.row_offsets, A.col_indices, batches, b, (3, 2), 19)
                print(" ", O.compare_epochs(want, ep.to_arrays())[:2], flush=True)


if __name__ == "__main__":
    main()
