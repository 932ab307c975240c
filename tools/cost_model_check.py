"""α–β cost model against real NCCL traffic (reference
dist.py:82-138 ledger, 580-596 predict_costs).

Runs the 1.5D SAGE executor in its Alg. 2 variant (sparsity-aware row fetch,
fetch="rows") with a CommLedger in reference semantics (words and messages at
the sender), for several bulk sizes k, and records per rank the ledger
charges, the bytes NCCL actually moved and the wall time of the fetch and
reduce phases.  Fits α (per message) and β (per word) of the fetch phase by
least squares over the runs and prints measured vs fitted vs predict_costs'
T_rowdata.  Launch: python -m torch.distributed.run --nproc-per-node P
tools/cost_model_check.py --c C [--out file.json]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c", type=int, default=1)
    ap.add_argument("--workload", default="products")
    ap.add_argument("--ks", default="8,16,32,64")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    from paper_2311_02909_b200 import graphgen
    from paper_2311_02909_b200.dist import CommLedger, CostModelParams, ProcessGrid, predict_costs
    from paper_2311_02909_b200.dist_exec import Sage15D
    from paper_2311_02909_b200.pipeline import make_batches

    grid = ProcessGrid(world, a.c)
    n, m, sym = graphgen.SHAPES[a.workload]
    dg = graphgen.rmat_device_graph(n, m, symmetric=sym, seed=0)
    runs = []
    for k in (int(x) for x in a.ks.split(",")):
        allb = make_batches(np.arange(n), 1024, 0, 0)[:k * grid.rows]
        led = CommLedger(world)
        smp = Sage15D(dg, grid, (15, 10, 5), 1024, mode="pfree", fetch="rows", ledger=None)
        mine = [np.asarray(x) for x in allb[smp.i * k:(smp.i + 1) * k]]
        smp.sample(mine, 0, smp.i * k, 0)  # warm-up
        smp.ledger, smp.profile = led, True
        smp.stats = {key: 0 for key in smp.stats}
        smp.phase_ms = {"fetch": 0.0, "reduce": 0.0}
        for _ in range(a.reps):
            dist.barrier()
            smp.sample(mine, 0, smp.i * k, 0)
        row = torch.tensor([led.messages("gather-cols", rank) + led.messages("row-data", rank),
                            led.words("gather-cols", rank) + led.words("row-data", rank),
                            4 * (smp.stats["fetch_ids"] + smp.stats["fetch_words"]),
                            smp.phase_ms["fetch"], smp.phase_ms["reduce"],
                            led.words("all-reduce", rank)], dtype=torch.float64, device="cuda")
        allr = [torch.zeros_like(row) for _ in range(world)]
        dist.all_gather(allr, row)
        if rank == 0:
            R = torch.stack(allr).cpu().numpy() / a.reps
            U = sum(len(x) for x in mine)
            runs.append({"k": k, "rows_per_group": U,
                         "per_rank": {"messages": R[:, 0].tolist(), "words": R[:, 1].tolist(),
                                      "nccl_bytes": R[:, 2].tolist(), "fetch_ms": R[:, 3].tolist(),
                                      "reduce_ms": R[:, 4].tolist(),
                                      "allreduce_words": R[:, 5].tolist()}})
    if rank == 0:
        # fit T_fetch(max over ranks) = α·msgs + β·words (max over ranks)
        X = np.array([[max(r["per_rank"]["messages"]), max(r["per_rank"]["words"])] for r in runs])
        y = np.array([max(r["per_rank"]["fetch_ms"]) for r in runs])
        coef, *_ = np.linalg.lstsq(X, y, rcond=None)
        alpha, beta = (float(x) for x in coef)
        out = {"grid": [world, a.c], "workload": a.workload, "alpha_ms_per_msg": alpha,
               "beta_ms_per_word": beta, "runs": runs}
        print(f"grid p={world} c={a.c}: alpha={alpha:.4f} ms/message, "
              f"beta={beta * 1e6:.3f} ms per 1e6 words")
        print("| k | ledger words (max rank) | ledger words (all ranks) | NCCL bytes moved "
              "(all ranks) | fetch ms (max rank) | α–β fit ms | predict_costs T_rowdata ms | "
              "our all-reduce words | model P all-reduce words |")
        print("|---|---|---|---|---|---|---|---|---|")
        for r in runs:
            w = max(r["per_rank"]["words"])
            msg = max(r["per_rank"]["messages"])
            fit = alpha * msg + beta * w
            d = w / max(1, r["rows_per_group"]) * grid.c  # words per row fetched
            pred = predict_costs(CostModelParams(world, a.c, r["k"], 1024, 15, max(d, 1e-9),
                                                 alpha=max(alpha, 0), beta=max(beta, 0)))
            kbd = r["k"] * 1024 * d
            print(f"| {r['k']} | {w:.0f} | {sum(r['per_rank']['words']):.0f} | "
                  f"{sum(r['per_rank']['nccl_bytes']):.0f} | "
                  f"{max(r['per_rank']['fetch_ms']):.2f} | {fit:.2f} | "
                  f"{pred.t_rowdata:.2f} | {max(r['per_rank']['allreduce_words']):.0f} | "
                  f"{a.c * kbd / world:.0f} |")
        if a.out:
            json.dump(out, open(a.out, "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
