"""Multi-GPU parity check of the 1.5D executor (run under torchrun, one
process per GPU; not collected by pytest):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tests/dist_exec_check.py

For every valid grid (p = N, c with c | p, c^2 <= p, c^2 | p) and both SAGE
kernel modes: the gathered distributed epoch must equal the serial bulk
epoch bit for bit; fetch_features over NCCL must equal direct indexing."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    # GB_DIST_BACKEND=gloo: every rank shares cuda:0 and the exchanges travel
    # through host copies — the executors' partitioning, keys and message
    # logic checked on a one-GPU box (the peer-memory modes need NCCL)
    gloo = os.environ.get("GB_DIST_BACKEND", "nccl") == "gloo"
    torch.cuda.set_device(0 if gloo else int(os.environ.get("LOCAL_RANK", rank)))
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl",
                                device_id=torch.device("cuda", torch.cuda.current_device()))
    import paper_2311_02909_b200 as gb
    from paper_2311_02909_b200 import graphgen
    from paper_2311_02909_b200.dist import CommLedger, ProcessGrid, _bounds
    from paper_2311_02909_b200.dist_exec import (BlockGraph, Ladies15D, PeerFeatures, Sage15D,
                                                 fetch_features_nccl, fetch_features_p2p,
                                                 ladies_epoch_15d, sage_epoch_15d)

    shape = (1 << 14, 200_000, True)
    dg = graphgen.rmat_device_graph(*shape, seed=3)
    G = gb.Graph.from_device(dg)
    rng = np.random.default_rng(0)
    batches = [rng.permutation(dg.n)[:64] for _ in range(8)]
    cfg = gb.SamplerConfig.sage(3, 64, (15, 10, 5), bulk_count=8, seed=4)
    serial = gb.sample_epoch_bulk(G, cfg, batches, epoch=1, batch_offset=5)
    ok = True
    grids = [(world, c) for c in (1, 2) if world % c == 0 and c * c <= world and world % (c * c) == 0]
    modes = (("pfree", "rows"), ("stream", "rows"), ("pfree", "owner"))
    if not gloo:
        modes += (("pfree", "p2p"), ("dedup", "split"))
    for p, c in grids:
        grid = ProcessGrid(p, c)
        # block-only partition (gb_rmat_block): this rank's block equals the
        # replicated graph's rows, the global degree metadata is exact, and
        # only the block's columns are resident
        part = BlockGraph.rmat(*shape, grid, seed=3)
        full = BlockGraph.from_full(dg, grid)
        same = (torch.equal(part.brp, full.brp) and
                torch.equal(part.bcol[:part.nnz], full.bcol[:full.nnz]) and
                torch.equal(part.tables.rowptr, dg.rowptr) and
                part.tables.max_degree == dg.max_degree and
                part.tables.table_slots == dg.table_slots)
        ok &= same
        if rank == 0:
            print(f"grid ({p},{c}) block partition: {'PASS' if same else 'FAIL'} "
                  f"resident {part.resident_bytes()} B vs replicated "
                  f"{dg.rowptr.numel() * 8 + dg.nnz * 4} B", flush=True)
        for mode, fetch in modes:
            led = CommLedger(p)
            src = part if fetch != "rows" else dg
            s = Sage15D(src, grid, cfg.fanouts, cfg.batch_size, mode=mode, ledger=led, fetch=fetch)
            ep = sage_epoch_15d(s, cfg, batches, epoch=1, batch_offset=5)
            same = serial.equals(ep)
            ok &= same
            if rank == 0:
                print(f"grid ({p},{c}) {mode}/{fetch}: {'PASS' if same else 'FAIL'} "
                      f"stats={s.stats}", flush=True)
        # LADIES (race) on the grid == single-GPU race sampler
        lcfg = gb.SamplerConfig.ladies(3, 64, 48, bulk_count=8, seed=4)
        lser = gb.sample_epoch_bulk(G, lcfg, batches, epoch=1, batch_offset=5, mode="race")
        for lf in (("rows",) if gloo else ("rows", "p2p")):
            ls = Ladies15D(part, grid, lcfg.fanouts, lcfg.batch_size, fetch=lf)
            lep = ladies_epoch_15d(ls, lcfg, batches, epoch=1, batch_offset=5)
            same = lser.equals(lep)
            ok &= same
            if rank == 0:
                print(f"grid ({p},{c}) ladies race/{lf}: {'PASS' if same else 'FAIL'} "
                      f"stats={ls.stats}", flush=True)
        # features: replicas of the block rows in every grid column
        f = 16
        H = torch.arange(dg.n * f, dtype=torch.float32, device="cuda").view(dg.n, f)
        rs = _bounds(dg.n, grid.rows)
        i, j = grid.coords(rank)
        Hb = H[int(rs[i]):int(rs[i + 1])].contiguous()
        want = rng.integers(0, dg.n, size=500)
        got = fetch_features_nccl(want, Hb, rs, grid, grid.col_group(j))
        same = bool(torch.equal(got, H[torch.as_tensor(want).cuda()]))
        ok &= same
        if rank == 0:
            print(f"grid ({p},{c}) fetch_features: {'PASS' if same else 'FAIL'}", flush=True)
        if not gloo:
            peer = PeerFeatures(Hb, rs, grid)
            got = fetch_features_p2p(want, peer)
            torch.cuda.synchronize()
            same = bool(torch.equal(got, H[torch.as_tensor(want).cuda()]))
            ok &= same
            if rank == 0:
                print(f"grid ({p},{c}) fetch_features p2p: {'PASS' if same else 'FAIL'}",
                      flush=True)
            peer.handle.barrier(channel=0)
    ok &= cost_model_band(gb, world, rank, gloo)
    t = torch.tensor([1 if ok else 0], device="cpu" if gloo else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("ALL PASS" if int(t.item()) else "SOME FAILED", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(t.item()) else 1)


def cost_model_band(gb, world, rank, gloo):
    """Reference test_acceptance.py:193-240 over the real transport: the
    Alg. 2 row fetch (fetch="rows") on a d-out-regular graph, one layer
    (Q = the seed matrix), k = 4 batches of b = 128.  Checks (a) the bytes
    the executor handed to NCCL / gloo equal 4 x the ledger's words (the
    reference's accounting describes the wire), (b) each grid column's
    row-data words equal the sparsity-aware volume (d per distinct remote
    row, dist.py:308-378) and (c) lie in [0.5, 2] x the model's kbd/c scaled
    by the remote fraction of the rows (the model ignores locality)."""
    import torch
    import torch.distributed as dist

    from paper_2311_02909_b200 import dist_exec
    from paper_2311_02909_b200.dist import CommLedger, ProcessGrid, _bounds
    from paper_2311_02909_b200.dist_exec import Sage15D, sage_epoch_15d

    n, d, k, b = 1 << 13, 8, 4, 128
    rng = np.random.default_rng(77)
    offs = rng.choice(np.arange(1, n), size=d, replace=False)
    src = np.repeat(np.arange(n), d)
    dst = (src + np.tile(offs, n)) % n
    G = gb.Graph.from_edges(n, src, dst)
    batches = list(rng.permutation(n)[: k * b].reshape(k, b))
    cfg = gb.SamplerConfig.sage(1, b, (d,), bulk_count=k, seed=1)
    serial = gb.sample_epoch_bulk(G, cfg, batches)
    ok = True
    for c in (1, 2):
        if world % c or c * c > world or world % (c * c):
            continue
        grid = ProcessGrid(world, c)
        led = CommLedger(world)
        dist_exec.WIRE["bytes"] = 0
        smp = Sage15D(G.device(), grid, (d,), b, mode="pfree", ledger=led, fetch="rows")
        same = serial.equals(sage_epoch_15d(smp, cfg, batches))
        wire = torch.tensor([dist_exec.WIRE["bytes"]], dtype=torch.int64,
                            device="cpu" if gloo else "cuda")
        dist.all_reduce(wire)
        words = sum(led.words(phase=ph) for ph in ("gather-cols", "row-data"))
        wsum = torch.tensor([words], dtype=torch.int64, device=wire.device)
        dist.all_reduce(wsum)
        ledger_eq = int(wire.item()) == 4 * int(wsum.item())
        # exact sparsity-aware volume per grid column
        bounds = _bounds(n, grid.rows)
        gb_ = _bounds(len(batches), grid.rows)
        st = grid.stages
        band = True
        for j in range(c):
            col_words = torch.tensor([led.words(phase="row-data", process=rank)
                                      if grid.coords(rank)[1] == j else 0],
                                     dtype=torch.int64, device=wire.device)
            dist.all_reduce(col_words)
            expect, remote, total = 0, 0, 0
            for i in range(grid.rows):
                U = np.unique(np.concatenate(batches[int(gb_[i]):int(gb_[i + 1])]))
                for q in range(st):
                    kb = j * st + q
                    cnt = int(np.sum((U >= bounds[kb]) & (U < bounds[kb + 1])))
                    total += cnt
                    if kb != i:
                        expect += d * cnt
                        remote += cnt
            model = k * b * d / c * (remote / max(total, 1))
            cw = int(col_words.item())
            band &= cw == expect and 0.5 * model <= cw <= 2.0 * model
            if rank == 0:
                print(f"  column {j}: row-data words {cw} (sparsity-aware volume {expect}, "
                      f"model kbd/c x remote {model:.0f})", flush=True)
        good = same and ledger_eq and band
        ok &= good
        if rank == 0:
            print(f"grid ({world},{c}) cost-model band: {'PASS' if good else 'FAIL'} "
                  f"(epoch {same}, wire bytes {int(wire.item())} = 4 x ledger words "
                  f"{int(wsum.item())}: {ledger_eq})", flush=True)
    return ok


if __name__ == "__main__":
    main()
