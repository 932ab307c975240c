python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
GB_SYNC_DEBUG=1 timeout 120 python tools/gpu/dbg_dedup.py dedup 2>&1 | grep -v "^  " | tail -4
timeout 600 python -m pytest tests/test_sage_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/profile_bulk.py --mode dedup > gpurun_out/pb.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dedup.csv \
    python tools/profile_bulk.py --mode dedup --warm 1 > gpurun_out/ncu_a.log 2>&1
python tools/bulk_launches.py gpurun_out/launches_dedup.csv k_ws_clear 2>&1 | tail -40
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench7.log 2>&1
grep -o '"value": [0-9.]*, "unit": "minibatches/s", "n_gpus": 1, "steps": 20, "warmup": 5, "ms_per_step": [0-9.]*' gpurun_out/bench7.log
