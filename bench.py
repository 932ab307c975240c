"""Benchmark: sampled minibatches/s of the 3-layer GraphSAGE (15,10,5) bulk
sampler (BASELINE.json metric; workload = configs[1]: ogbn-products-shape
synthetic R-MAT, b=1024, k=64 per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload products|cfg1|papers] [--mode stream|pfree]

One step = one bulk: all 3 layers (P = Q^l A formed on chip, norm, exact
keyed ITS, extraction) for the k minibatches of this rank, inputs resident in
HBM.  Multi-GPU (torchrun): replicated graph, disjoint contiguous batch
ranges per rank (dist.py:417-429 replicated mode), no data-path collective
-> weak scaling; time = max over ranks of the per-rank device time.

Timing: W warm-up bulks, then K bulks each bracketed by CUDA events on the
launching stream (one CUDA-graph replay per bulk); between bulks a 256 MiB
buffer is written to flush L2 (outside the events).  nvidia-smi clocks are
sampled during the timed region.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "sampled minibatches/sec (3-layer SAGE, k-batch bulk)"
UNIT = "minibatches/s"
FANOUTS = (15, 10, 5)
BATCH = 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="products", choices=["products", "cfg1", "papers"])
    p.add_argument("--k", type=int, default=None, help="minibatches per bulk per GPU")
    p.add_argument("--mode", default="dedup", choices=["dedup", "stream", "pfree"])
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-pfree", action="store_true")
    p.add_argument("--no-ladies", action="store_true")
    p.add_argument("--no-aggregation", action="store_true")
    p.add_argument("--dist", default="replicated", choices=["replicated", "15d"],
                   help="multi-GPU mode: replicated graph (cfg4) or 1.5D partitioned (cfg5)")
    p.add_argument("--c", type=int, default=2, help="1.5D replication factor")
    p.add_argument("--fetch", default="auto", choices=["auto", "rows", "owner", "p2p", "split"],
                   help="1.5D SAGE: Alg. 2 row fetch / owner-computes over NCCL, owner "
                        "sampling over peer memory (p2p), replicas splitting the batches "
                        "with rows read from peer memory (split); auto = split")
    return p.parse_args()


def default_k(workload):
    return 8 if workload == "cfg1" else 64


# ------------------------------------------------------------------ clocks

class ClockSampler:
    def __init__(self):
        self.proc = None
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self, index):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # nvidia-smi takes a while to come up: start timing only once it
        # writes, so the timed region is covered by samples
        import time as _t

        t0 = _t.time()
        while _t.time() - t0 < 5.0:
            self.fh.flush()
            if os.path.getsize(self.path) > 0:
                break
            _t.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ helpers

def make_batches_for(n, k_total):
    from paper_2311_02909_b200.pipeline import make_batches

    return make_batches(np.arange(n), BATCH, seed=0, epoch=0)[:k_total]


def layer_stats(bulk, dg, sizes):
    """R, G (gathered entries = sum of row degrees), F, U per layer."""
    import torch

    out = []
    rowv = None
    for l in range(len(FANOUTS)):
        R, F, U = (int(x) for x in sizes[3 * l:3 * l + 3])
        if l == 0:
            rv = bulk._bverts[:R].long()
        else:
            rv = bulk.out[l - 1]["fcol"][:R].long()
        G = int((dg.rowptr[rv + 1] - dg.rowptr[rv]).sum().item()) if R else 0
        uv = torch.unique(rv) if R else rv
        Gd = int((dg.rowptr[uv + 1] - dg.rowptr[uv]).sum().item()) if R else 0
        out.append({"R": R, "G": G, "F": F, "U": U, "D": int(uv.numel()), "G_distinct": Gd})
        del rv, uv
    del rowv
    torch.cuda.synchronize()
    return out


def sage_bytes(st):
    """SURVEY.md §8(d) SAGE algorithmic bytes per bulk: sum_l 28R + 4G + 12F + 4U + 8."""
    return sum(28 * s["R"] + 4 * s["G"] + 12 * s["F"] + 4 * s["U"] + 8 for s in st)


def kernel_bytes(s, kernel):
    """Algorithmic bytes of one launch: every byte the
    kernel must move by design, no re-reads, per layer statistics s.
      stream (k_sage_stream): deg 4 + fptr 8 + vertex 4 + row_ptr 8 + gstart 8
                              per row, 4 per gathered entry, pick idx 4 + col 4;
      pick   (k_sage_pick<false>): deg 4 + fptr 8 per row, 4 per pick idx;
      pfree  (k_sage_pick<true>):  deg 4 + fptr 8 + vertex 4 + row_ptr 8 per
                                   row, col read 4 + write 4 per pick."""
    if kernel == "stream":
        return 32 * s["R"] + 4 * s["G"] + 8 * s["F"]
    if kernel == "dedup":
        # the sampling core of a dedup layer (k_dd_pick + k_dd_serve): per
        # grouped row its 16-B record + 16-B row_ptr pair, per pick the
        # picked column read 4 + frontier write 4 + batch bit 4.  (Rows of
        # the few vertices staged whole add their 4 B per entry, not counted.)
        return 32 * s["R"] + 12 * s["F"]
    if kernel == "dedup_first":
        # the first layer of a dedup bulk is sampled P-free (k_sage_pick<1>)
        return 24 * s["R"] + 12 * s["F"]
    if kernel == "pick":
        return 12 * s["R"] + 4 * s["F"]
    return 24 * s["R"] + 8 * s["F"]


def dedup_bytes(st):
    """Compulsory bytes of the dedup bulk: SURVEY.md §8(d)'s per-layer terms
    with the gathered entries of the DISTINCT rows only."""
    return sum(28 * s["R"] + 4 * s["G_distinct"] + 12 * s["F"] + 4 * s["U"] + 8 for s in st)


def oracle_prefix(layers, kc):
    """Restrict per-layer arrays of a k-batch bulk to its first kc batches."""
    out = []
    for a in layers:
        R = int(a["rowv_off"][kc])
        F = int(a["sampv_off"][kc])
        U = int(a["colv_off"][kc])
        out.append({
            "frontier_shape": np.array([R, a["frontier_shape"][1]]),
            "frontier_ptr": a["frontier_ptr"][:R + 1], "frontier_col": a["frontier_col"][:F],
            "adj_shape": np.array([R, U]), "adj_ptr": a["adj_ptr"][:R + 1],
            "adj_col": a["adj_col"][:F],
            "rowv_off": a["rowv_off"][:kc + 1], "rowv_cat": a["rowv_cat"][:R],
            "colv_off": a["colv_off"][:kc + 1], "colv_cat": a["colv_cat"][:U],
            "sampv_off": a["sampv_off"][:kc + 1], "sampv_cat": a["sampv_cat"][:F],
        })
    return out


def cpu_baseline(host_graph, batches, seconds, gpu_layers=None):
    """Oracle port (oracle/, C + OpenMP, all host threads) on a bounded sample
    of the same workload: the first kc batches (batch_offset 0).  Also checks
    the GPU bulk's first kc batches against it bit for bit."""
    from oracle import oracle as O

    n, rowptr, col = host_graph
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.sage_bulk(n, rowptr, col, batches[:1], BATCH, FANOUTS, 0, 0, 0, threads=threads)
    t1 = time.perf_counter() - t0
    kc = int(max(1, min(len(batches), seconds / max(t1, 1e-3))))
    t0 = time.perf_counter()
    want = O.sage_bulk(n, rowptr, col, batches[:kc], BATCH, FANOUTS, 0, 0, 0, threads=threads)
    dt = time.perf_counter() - t0
    parity = None
    if gpu_layers is not None:
        errs = O.compare_epochs(want, oracle_prefix(gpu_layers, kc))
        parity = "bit-exact" if not errs else f"MISMATCH: {errs[:3]}"
    return {"value": kc / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {kc} of the bulk's minibatches (batch_offset 0), same graph; "
                      f"{dt:.1f} s"}, kc, parity


def ladies_bytes(st, k):
    """SURVEY.md §8(d) LADIES algorithmic bytes per bulk:
    sum_l 44 nnz(Q) + 8 G + 16 N + 4 |S| + 4 E + 8 k + 16."""
    return sum(44 * s["Q"] + 8 * s["G"] + 16 * s["N"] + 4 * s["S"] + 4 * s["E"] + 8 * k + 16
               for s in st)


def measure_aggregation(bulk, d_off, d_cat, sizes, st, n, k, peak, f=128):
    """feature fetch of the deepest col_vertices and the
    aggregation chain of the whole bulk (pipeline.propagate_bulk: Y = A^l X
    per layer + first-occurrence carry), fp32 features of width f, random
    H in HBM.  Algorithmic bytes: every gathered X row read once, every Y /
    X row written once."""
    import torch

    from paper_2311_02909_b200.pipeline import _gather_rows, propagate_bulk
    from paper_2311_02909_b200.sampler import SampledEpoch, SamplerKind

    layers = bulk.layers(d_off, d_cat, sizes)
    ep = SampledEpoch(SamplerKind.SAGE, 0, list(range(k)), layers, len(layers))
    H = torch.rand((n, f), device="cuda")
    colv = layers[-1].device["colv_cat"]

    def run():
        return propagate_bulk(ep, _gather_rows(colv, H))

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    reps = 5
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    row = 4 * f
    byt = 2 * st[-1]["U"] * row  # fetch: read + write
    for li, s_ in enumerate(st):
        byt += s_["F"] * row + s_["R"] * row  # gathered X rows + Y rows
        if li > 0:
            byt += 2 * st[li - 1]["U"] * row  # carry to the shallower layer
    del H
    return {"ms_per_bulk": ms, "f": f, "dtype": "f32", "bytes_per_bulk": byt,
            "gb_s": byt / (ms / 1e3) / 1e9, "frac_of_peak": byt / (ms / 1e3) / 1e9 / peak,
            "api": "pipeline.propagate_bulk after the device fetch of layers[-1].col_vertices"}


def measure_ladies(args, dg, rank, world, flush, peak):
    """LADIES b=s=512, L=3, k=64 per GPU on the products-shape graph
    (exponential-race sampling; exact replay is the small-graph parity mode)."""
    import torch

    from paper_2311_02909_b200.engine import LadiesBulk
    from paper_2311_02909_b200.pipeline import make_batches

    k, b, s, L = 64, 512, 512, 3
    allb = make_batches(np.arange(dg.n), b, seed=0, epoch=0)[:k * world]
    batches = [np.sort(x) for x in allb[rank * k:(rank + 1) * k]]
    off = np.zeros(k + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in batches])
    d_off = torch.as_tensor(off).cuda()
    d_cat = torch.as_tensor(np.concatenate(batches).astype(np.int32)).cuda()
    bulk = LadiesBulk(dg, k, int(off[-1]), (s,) * L, mode="race")
    for _ in range(3):
        bulk.launch(d_off, d_cat, 0, 0, rank * k)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        bulk.launch(d_off, d_cat, 0, 0, rank * k)
        with torch.cuda.graph(graph, stream=cs):
            bulk.launch(d_off, d_cat, 0, 0, rank * k)
    torch.cuda.current_stream().wait_stream(cs)
    torch.cuda.synchronize()
    steps = max(5, min(args.steps, 20))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i)
        evs[i][0].record()
        graph.replay()
        evs[i][1].record()
    torch.cuda.synchronize()
    T = float(sum(a.elapsed_time(bb) for a, bb in evs))
    if world > 1:
        t = torch.tensor([T], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        T = float(t.item())
    sizes = bulk.sizes.cpu().numpy()
    st = []
    qoff, qcol = d_off, d_cat
    for li in range(L):
        QN, F, E, C, N = (int(x) for x in sizes[5 * li:5 * li + 5])
        rv = qcol[:QN].long()
        G = int((dg.rowptr[rv + 1] - dg.rowptr[rv]).sum().item())
        st.append({"Q": QN, "G": G, "N": N, "S": F, "E": E, "cols": C})
        qoff, qcol = bulk.out[li]["fptr"], bulk.out[li]["fcol"]
    B = ladies_bytes(st, k)
    ms = T / steps
    return {"metric": "sampled minibatches/sec (LADIES 512/layer, 3 layers, k-batch bulk)",
            "value": world * k * steps / (T / 1e3), "unit": UNIT, "ms_per_step": ms,
            "config": "products-shape R-MAT, b=s=512, L=3, k=64 per GPU, exponential-race "
                      "sampling", "layers": st, "bulk_bytes": B,
            "bulk_gbs": B / (ms / 1e3) / 1e9, "frac_of_peak": B / (ms / 1e3) / 1e9 / peak}


# ------------------------------------------------------------------ arms

def run_reference(args, rank, world):
    """--impl reference: the oracle port of the reference CPU sampler on the
    host cores, rank 0 only, same graph/batches/metric."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2311_02909_b200.graphgen import SHAPES

    # the same graph the GPU arm builds (gb_rmat_graph), restated on the host
    # (oracle/csrc/gen.c): the reference arm never loads the product library
    n, m, sym = SHAPES[args.workload]
    t0 = time.perf_counter()
    rowptr, col = O.rmat_graph(n, m, symmetric=sym, seed=0)
    t_graph = time.perf_counter() - t0
    host = (n, rowptr, col)
    k = args.k or default_k(args.workload)
    batches = make_batches_for(n, k)

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.sage_bulk(n, host[1], host[2], batches[:1], BATCH, FANOUTS, 0, 0, 0, threads=threads)
    t1 = time.perf_counter() - t0
    per_step = max(10.0, min(60.0, 150.0 / max(1, args.steps + args.warmup)))
    kc = int(max(1, min(k, per_step / max(t1, 1e-3))))
    times = []
    for i in range(args.warmup + args.steps):
        lo = (i * kc) % max(1, k - kc + 1)
        t0 = time.perf_counter()
        O.sage_bulk(n, host[1], host[2], batches[lo:lo + kc], BATCH, FANOUTS, 0, 0, lo,
                    threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    T = float(np.sum(times))
    value = kc * len(times) / T
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}-shape R-MAT, GraphSAGE (15,10,5), b=1024",
                   "k_per_step": kc, "n": n, "nnz": int(len(host[2])),
                   "graph": f"oracle/csrc/gen.c host build, {t_graph:.1f} s (no product library)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{kc} minibatches per step of the {k}-minibatch bulk"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2311_02909_b200 as gb
    from paper_2311_02909_b200 import _lib, graphgen
    from paper_2311_02909_b200.engine import BulkSampler, SageBulk

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n, m, sym = graphgen.SHAPES[args.workload]
    t0 = time.perf_counter()
    dg = graphgen.rmat_device_graph(n, m, symmetric=sym, seed=0)
    t_graph = time.perf_counter() - t0
    k = args.k or default_k(args.workload)
    all_batches = make_batches_for(n, k * world)
    batches = all_batches[rank * k:(rank + 1) * k]
    boff = rank * k
    off = np.zeros(k + 1, np.int64)
    off[1:] = np.cumsum([len(b) for b in batches])
    d_off = torch.as_tensor(off).cuda()
    d_cat = torch.as_tensor(np.concatenate(batches).astype(np.int32)).cuda()
    lib = _lib.lib()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    def measure(mode):
        bulk = SageBulk(dg, k, int(off[-1]), BATCH, FANOUTS, mode=mode)
        bulk._bverts = d_cat
        for _ in range(max(args.warmup, 3)):
            bulk.launch(d_off, d_cat, 0, 0, boff)
        torch.cuda.synchronize()
        lib.gb_launch_counter(1)
        bulk.launch(d_off, d_cat, 0, 0, boff)
        launches_per_bulk = int(lib.gb_launch_counter(1))
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            bulk.launch(d_off, d_cat, 0, 0, boff)  # warm the capture stream
            with torch.cuda.graph(graph, stream=s):
                bulk.launch(d_off, d_cat, 0, 0, boff)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        for _ in range(2):
            graph.replay()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        clk = ClockSampler()
        clk.start(local_rank)
        for i in range(args.steps):
            flush.fill_(i)
            evs[i][0].record()
            graph.replay()
            evs[i][1].record()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        clocks = clk.stop()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        # sample-kernel durations (events around each launch, same stream)
        ppl = 1 if mode == "pfree" else 2
        cap = ppl * len(FANOUTS) * 4
        lib.gb_profile_begin(2 * cap)
        for i in range(4):
            flush.fill_(i)
            bulk.launch(d_off, d_cat, 0, 0, boff)
        ms = (ctypes.c_float * cap)()
        npairs = ctypes.c_int32()
        lib.gb_profile_end(ms, cap, ctypes.byref(npairs))
        kern_ms = np.array(ms[:npairs.value]).reshape(4, len(FANOUTS), ppl)
        sizes = bulk.sizes.cpu().numpy()
        return bulk, step_ms, clocks, kern_ms, sizes, launches_per_bulk, graph

    bulk, step_ms, clocks, kern_ms, sizes, lpb, graph = measure(args.mode)
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * k * args.steps / (total_ms / 1e3)
    st = layer_stats(bulk, dg, sizes)
    peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    agg = measure_aggregation(bulk, d_off, d_cat, sizes, st, n, k, peak) \
        if not args.no_aggregation else None
    KERNEL = {"stream": "k_sage_stream", "pfree": "k_sage_pick<true>",
              "dedup": "k_dd_pick + k_dd_serve (layer 1: k_sage_pick<true>)"}
    if args.mode == "dedup":
        # which layers the library grouped (gb_sage.cu group_pays: the layer's
        # row bound >= 0.25 n, and never the first layer); the others ran
        # the P-free pick
        rcap = [k * BATCH * int(np.prod(FANOUTS[:i])) for i in range(len(FANOUTS))]
        kb = [kernel_bytes(s_, "dedup" if i >= 1 and rcap[i] >= 0.25 * n else "dedup_first")
              for i, s_ in enumerate(st)]
        kern_avg = kern_ms.mean(axis=0).sum(axis=1)  # pick + serve intervals, per layer
    else:
        kb = [kernel_bytes(s_, args.mode) for s_ in st]
        kern_avg = kern_ms.mean(axis=0)[:, -1]  # dominant kernel, per layer
    pick_avg = kern_ms.mean(axis=0)[:, 0]
    achieved4 = sum(kb) / (kern_avg.sum() / 1e3) / 1e9
    # a path that reads only the picked entries is held to
    # its own sector-granular byte count — every random 4-B pick moves one
    # 32-B sector — which is how the dedup bulk reads the picks of its direct
    # rows (and of its P-free first layer); the 4-B count stays beside it
    sector = [b + 28 * s_["F"] for b, s_ in zip(kb, st)] if args.mode in ("dedup", "pfree") \
        else kb
    achieved = sum(sector) / (kern_avg.sum() / 1e3) / 1e9
    bulk_bytes = sage_bytes(st)
    traffic = None
    tpath = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and args.workload == "products" and k == 64:
        tk = json.load(open(tpath)).get({"dedup": "dedup_sampling"}.get(args.mode,
                                                                        KERNEL[args.mode]))
        traffic = tk["bulk_bytes"] if tk else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": f"{args.workload}-shape R-MAT (n={n}, nnz={dg.nnz}), GraphSAGE "
                        f"(15,10,5), b=1024, k={k} per GPU, replicated graph",
            "mode": args.mode, "l2": "flushed between steps (256 MiB write, untimed)",
            "parallelism": f"replicated x{world}", "graph_build_s": round(t_graph, 2),
        },
        "gpu_launches": lpb * args.steps,
        **({"aggregation": agg} if agg else {}),
        "clocks": clocks,
        "layers": st,
        "edges_per_s": world * sum(s["G"] for s in st) * args.steps / (total_ms / 1e3),
        "bulk_bytes": bulk_bytes,
        "bulk_gbs": bulk_bytes / (total_ms / args.steps / 1e3) / 1e9,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_note": "dram__bytes_read+write of the dominant kernel's launches of one "
                            "bulk (ncu, profiles/ncu_traffic.json); achieved/per_layer_bytes "
                            "aggregate the same launches",
            "kernel": KERNEL[args.mode],
            "pick_kernel_ms": [round(x, 4) for x in pick_avg.tolist()],
            "per_layer_ms": [round(x, 4) for x in kern_avg.tolist()],
            "per_layer_bytes": sector, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
            **({"bytes_note": "per_layer_bytes: 32R + 12F per grouped layer (24R + 12F for the "
                              "P-free first layer) with every in-place pick charged its 32-B "
                              "sector (SURVEY.md 8(f)1: a picked-entries-only path is held to "
                              "its sector-granular byte count); staged rows' entries not counted",
                "per_layer_bytes_4b": kb, "achieved_4b": achieved4, "frac_4b": achieved4 / peak}
               if args.mode in ("dedup", "pfree") else {}),
            "kernel_share_of_step": float(kern_avg.sum() / (total_ms / args.steps)),
            # the whole step against the bytes Alg. 1 with duplicate-row
            # elimination must move (28R + 4G_distinct + 12F + 4U + 8)
            "step_bytes_dedup": dedup_bytes(st),
            "step_frac_dedup": dedup_bytes(st) / (total_ms / args.steps / 1e3) / 1e9 / peak,
        },
    }
    # the other SAGE kernel modes on the same workload (identical outputs)
    for other in ("stream", "pfree") if not args.no_pfree else ():
        if other == args.mode:
            continue
        b2, sm2, _, km2, sz2, lpb2, g2 = measure(other)
        t2 = float(np.sum(sm2))
        if world > 1:
            t = torch.tensor([t2], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            t2 = float(t.item())
        kb2 = [kernel_bytes(s, other) for s in st]
        km = km2.mean(axis=0)[:, -1]
        a2 = sum(kb2) / (km.sum() / 1e3) / 1e9
        line[other] = {"value": world * k * args.steps / (t2 / 1e3), "unit": UNIT,
                       "ms_per_step": t2 / args.steps,
                       "same_sizes": bool(np.array_equal(sz2, sizes)),
                       "roofline": {"achieved": a2, "peak": peak, "unit": "GB/s",
                                    "frac": a2 / peak, "kernel": KERNEL[other],
                                    "per_layer_ms": km.tolist(), "per_layer_bytes": kb2}}
        if other == "pfree":
            # the P-free path's roofline is against its own
            # sector-granular byte count (every random 4-B pick moves 32 B)
            sec = sum(kb2) + 28 * sum(s["F"] for s in st)
            line[other]["roofline"]["achieved_sector_floor"] = sec / (km.sum() / 1e3) / 1e9
            line[other]["roofline"]["frac_sector_floor"] = sec / (km.sum() / 1e3) / 1e9 / peak
        if other == "stream":
            line[other]["roofline"]["note"] = (
                "algorithmic bytes stream every frontier row's A row, duplicates included; "
                "repeated hub rows are served by the 126 MB L2, so achieved can exceed the "
                "HBM peak (DRAM traffic: profiles/ncu_traffic.json k_sage_stream)")
        del b2, g2
    # LADIES, BASELINE configs[2]: same graph, 512 nodes/layer, 3 layers, k=64
    if not args.no_ladies:
        line["ladies_cfg3"] = measure_ladies(args, dg, rank, world, flush, peak)
    # end-to-end through the public API (host batches in, host arrays out)
    G = gb.Graph.from_device(dg)
    cfg = gb.SamplerConfig.sage(3, BATCH, FANOUTS, bulk_count=k, seed=0)
    bs = BulkSampler(G, cfg, mode=args.mode)
    ep = None
    for _ in range(3):  # steady state: the held epoch's block + one pooled block
        ep = bs.sample(batches, 0, boff)
    torch.cuda.synchronize()
    nst = max(3, min(args.steps, 10))
    # one synchronous call per bulk (latency)
    e2e_t = []
    for _ in range(nst):
        t0 = time.perf_counter()
        ep = bs.sample(batches, 0, boff)
        e2e_t.append(time.perf_counter() - t0)
    e2e_sync = float(np.mean(e2e_t))
    # the epoch loop: sample_stream overlaps bulk j's device->host copy with
    # bulk j + 1's sampling (every bulk still uploads its batches and reads
    # back all its arrays)
    def consume(ep):
        # the reference's output types, as a trainer reads them
        # (LayerSample fields, sampler.py:240-261): zero-copy views here
        for layer in ep.layers:
            layer.frontier, layer.adjacency
            layer.row_vertices, layer.col_vertices, layer.sampled_vertices

    for ep in bs.sample_stream([(batches, boff)] * 2):
        consume(ep)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for ep in bs.sample_stream([(batches, boff)] * nst):
        consume(ep)
    e2e_s = (time.perf_counter() - t0) / nst
    if world > 1:
        t = torch.tensor([e2e_s, e2e_sync], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s, e2e_sync = (float(x) for x in t.tolist())
    line["e2e"] = {"value": world * k / e2e_s, "unit": UNIT, "h2d_bytes_per_step": bs.h2d_bytes,
                   "d2h_bytes_per_step": bs.d2h_bytes,
                   "api": "paper_2311_02909_b200.BulkSampler.sample_stream (host batches -> "
                          "host SampledEpoch with every LayerSample field read as the reference "
                          "types; copy of bulk j overlapping bulk j+1)",
                   "sync_call": {"value": world * k / e2e_sync, "unit": UNIT,
                                 "api": "BulkSampler.sample, one blocking call per bulk"}}
    # CPU baseline (oracle port) on rank 0 at N=1, with a full-size parity check
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gpu_layers = ep.to_arrays()
        host = (n, dg.rowptr.cpu().numpy(), dg.col[:dg.nnz].cpu().numpy())
        cb, kc, parity = cpu_baseline(host, batches, args.cpu_seconds, gpu_layers)
        line["cpu_baseline"] = cb
        line["parity_full_size"] = f"{parity} on the first {kc} of {k} minibatches vs oracle"
    if rank == 0:
        emit(line)


def run_15d(args, rank, world, local_rank):
    """cfg5: GraphSAGE (15,10,5) with the graph 1.5D-partitioned over a
    (p/c) x c grid: sparsity-aware row fetch inside grid columns (NCCL p2p),
    sample-then-reduce inside grid rows, k=64 minibatches per grid row."""
    import torch
    import torch.distributed as dist

    from paper_2311_02909_b200 import graphgen
    from paper_2311_02909_b200.dist import ProcessGrid
    from paper_2311_02909_b200.dist_exec import BlockGraph, Sage15D

    c = args.c if (world % args.c == 0 and args.c ** 2 <= world and
                   world % (args.c ** 2) == 0) else 1
    grid = ProcessGrid(world, c)
    torch.cuda.set_device(local_rank)
    n, m, sym = graphgen.SHAPES[args.workload]
    # only this rank's block row is built and kept (gb_rmat_block); the
    # global degrees are all-gathered (partition_block_rows, dist.py:200-214)
    t0 = time.perf_counter()
    dg = BlockGraph.rmat(n, m, sym, grid, seed=0)
    t_part = time.perf_counter() - t0
    torch.cuda.empty_cache()
    resident = dg.resident_bytes()
    full_bytes = 8 * (n + 1) + 4 * (2 * m if sym else m)
    k = args.k or default_k(args.workload)
    allb = make_batches_for(n, k * grid.rows)
    # the grid samples row by row at the owner: stream or P-free kernels
    # auto: the grid row's replicas split its batches and run the dedup bulk
    # with rows staged from the owners' peer memory (round 2, split vs owner
    # sampling over peer memory: products 2x2 88.7K vs -, 4x1 104.0K vs
    # 56.5K, 2x1 67.5K vs 50.0K; papers 2x2 32.2K vs 14.3K, 2x1 23.2K vs
    # 15.2K)
    fetch = args.fetch if args.fetch != "auto" else "split"
    args.fetch = fetch
    m15 = "dedup" if fetch == "split" else ("stream" if args.mode == "stream" else "pfree")
    s = Sage15D(dg, grid, FANOUTS, BATCH, mode=m15, fetch=args.fetch)
    i = s.i
    mine = [np.asarray(x) for x in allb[i * k:(i + 1) * k]]
    for _ in range(max(args.warmup, 3)):
        s.sample(mine, 0, i * k, 0)
    torch.cuda.synchronize()
    dist.barrier()
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.sample(mine, 0, i * k, 0)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    T = float(np.sum(times))
    t = torch.tensor([T], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    T = float(t.item())
    value = k * grid.rows * args.steps / (T / 1e3)
    # feature fetch of the bulk's deepest col_vertices (f = 128, fp32): the
    # NCCL all-to-allv against the gather fused over peer memory
    from paper_2311_02909_b200.dist_exec import (PeerFeatures, fetch_features_nccl,
                                                 fetch_features_p2p)

    lay = s.sample(mine, 0, i * k, 0)[-1]
    verts = lay["colv_cat"].cpu().numpy()
    rs = np.linspace(0, n, grid.rows + 1).astype(np.int64)
    fdim = 128
    Hb = torch.rand((int(rs[s.i + 1] - rs[s.i]), fdim), device="cuda")
    peer = PeerFeatures(Hb, rs, grid)
    ftimes = {}
    for name, fn in (("nccl", lambda: fetch_features_nccl(verts, Hb, rs, grid,
                                                           grid.col_group(s.j))),
                     ("p2p", lambda: fetch_features_p2p(verts, peer))):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        tt = torch.tensor([a.elapsed_time(b) / 5], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ftimes[name] = float(tt.item())
    fetch_line = {"rows": int(verts.size), "f": fdim, "dtype": "f32",
                  "ms_nccl": ftimes["nccl"], "ms_p2p": ftimes["p2p"],
                  "gb_s_p2p": verts.size * fdim * 4 / (ftimes["p2p"] / 1e3) / 1e9,
                  "api": "dist_exec.fetch_features_p2p vs fetch_features_nccl"}
    peer.handle.barrier(channel=0)
    del peer, Hb
    # LADIES (b = s = 512, L = 3) on the same grid, race sampling
    from paper_2311_02909_b200.dist_exec import Ladies15D
    from paper_2311_02909_b200.pipeline import make_batches

    lb = make_batches(np.arange(n), 512, seed=0, epoch=0)[:k * grid.rows]
    lmine = [np.sort(np.asarray(x)) for x in lb[i * k:(i + 1) * k]]
    ls = Ladies15D(dg, grid, (512,) * 3, 512,
                   fetch="p2p" if args.fetch in ("p2p", "split") else "rows")
    for _ in range(2):
        ls.sample(lmine, 0, i * k, 0)
    lt = []
    for _ in range(max(3, min(args.steps, 10))):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ls.sample(lmine, 0, i * k, 0)
        b.record()
        torch.cuda.synchronize()
        lt.append(a.elapsed_time(b))
    LT = torch.tensor([float(np.sum(lt))], device="cuda", dtype=torch.float64)
    dist.all_reduce(LT, op=dist.ReduceOp.MAX)
    ladies_value = k * grid.rows * len(lt) / (float(LT.item()) / 1e3)
    if rank == 0:
        emit({
            "metric": METRIC + " [1.5D partitioned graph]", "value": value, "unit": UNIT,
            "ladies_15d": {"value": ladies_value, "unit": UNIT,
                           "ms_per_step": float(LT.item()) / len(lt),
                           "config": "LADIES b=s=512, L=3, k per grid row, race sampling"},
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": T / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}-shape R-MAT, GraphSAGE (15,10,5), "
                                   f"b=1024, k={k} per grid row",
                       "parallelism": f"1.5D grid {grid.rows}x{grid.c} (p={world}, c={grid.c})",
                       "mode": m15, "fetch": args.fetch},
            "graph_per_rank": {"resident_bytes_rank0": resident,
                               "replicated_graph_bytes": full_bytes,
                               "fraction": resident / full_bytes,
                               "build_s": t_part,
                               "how": "BlockGraph.rmat: block row only (gb_rmat_block) + "
                                      "all-gathered global degrees"},
            "traffic_rank0": {k2: int(v) for k2, v in s.stats.items()},
            "feature_fetch_rank0_group": fetch_line,
        })


_JSON_FD = None  # the process's real stdout; fd 1 itself is pointed at stderr


def emit(obj):
    """Write the one JSON line to the real stdout (everything else a library
    prints to stdout -- e.g. the NCCL version banner under torchrun -- has
    been sent to stderr by main())."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(obj) + "\n").encode())


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        elif args.dist == "15d":
            run_15d(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
