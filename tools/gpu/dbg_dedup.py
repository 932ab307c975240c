"""Debug driver: every SAGE golden through the dedup mode, one by one."""
import glob
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import paper_2311_02909_b200 as gb
    from oracle import oracle as O

    for path in sorted(glob.glob("tests/golden/epoch_*sage*.npz")):
        g, want = O.load_golden(path)
        G = gb.Graph(gb.SparseMatrix(g["n"], g["n"], g["rowptr"], g["col"],
                                     np.ones(len(g["col"])), validate=False))
        cfg = gb.SamplerConfig.sage(g["layers_cfg"], g["batch_size"], tuple(g["fanouts"]),
                                    bulk_count=len(g["batches"]), seed=g["seed"])
        print("run", path, flush=True)
        ep = gb.sample_epoch_bulk(G, cfg, g["batches"], epoch=g["epoch"],
                                  batch_offset=g["batch_offset"], mode=sys.argv[1])
        print(path, O.compare_epochs(want, ep.to_arrays())[:3], flush=True)


if __name__ == "__main__":
    main()
