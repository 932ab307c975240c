python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
GB_SYNC_DEBUG=1 timeout 900 python -m pytest tests/test_ladies_gpu.py -x -q -k "not inclusion_law" 2>&1 | tail -3
timeout 300 python tools/profile_bulk.py --sampler ladies > gpurun_out/pbl.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ladies.csv \
    python tools/profile_bulk.py --sampler ladies --warm 1 > gpurun_out/ncu_l.log 2>&1
python tools/bulk_launches.py gpurun_out/launches_ladies.csv k_lad_tiles 2>&1 | tail -45
timeout 600 python bench.py --steps 10 --warmup 3 --no-pfree --no-cpu-baseline --no-aggregation > gpurun_out/bench13.log 2>&1
grep -o '"ladies_cfg3": {[^}]*' gpurun_out/bench13.log
