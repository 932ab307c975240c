"""torch.profiler breakdown of one 1.5D SAGE bulk (rank 0), launched with
torchrun: python -m torch.distributed.run --nproc-per-node P tools/profile_15d.py --c C"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c", type=int, default=2)
    ap.add_argument("--workload", default="products")
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--fetch", default="owner")
    ap.add_argument("--sampler", default="sage", choices=["sage", "ladies"])
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    from paper_2311_02909_b200 import graphgen
    from paper_2311_02909_b200.dist import ProcessGrid
    from paper_2311_02909_b200.dist_exec import Ladies15D, Sage15D
    from paper_2311_02909_b200.pipeline import make_batches

    grid = ProcessGrid(world, a.c)
    n, m, sym = graphgen.SHAPES[a.workload]
    dg = graphgen.rmat_device_graph(n, m, symmetric=sym, seed=0)
    if a.sampler == "sage":
        allb = make_batches(np.arange(n), 1024, 0, 0)[:a.k * grid.rows]
        s = Sage15D(dg, grid, (15, 10, 5), 1024, mode="pfree", fetch=a.fetch)
        mine = [np.asarray(x) for x in allb[s.i * a.k:(s.i + 1) * a.k]]
    else:
        allb = make_batches(np.arange(n), 512, 0, 0)[:a.k * grid.rows]
        s = Ladies15D(dg, grid, (512,) * 3, 512)
        mine = [np.sort(np.asarray(x)) for x in allb[s.i * a.k:(s.i + 1) * a.k]]
    for _ in range(3):
        s.sample(mine, 0, s.i * a.k, 0)
    torch.cuda.synchronize()
    dist.barrier()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        s.sample(mine, 0, s.i * a.k, 0)
        torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
        print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
