# Build, SAGE parity tests, dedup-only bench (ms_per_step) and per-layer kernel times.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest ${TESTS:-tests/test_sage_gpu.py} -m gpu -x -q > gpurun_out/quick_pytest.log 2>&1; tail -2 gpurun_out/quick_pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 5 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['pick_kernel_ms'], d['roofline']['per_layer_ms'], d['clocks']['sm_mhz'])"
done
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/quick_launches.csv python bench.py --steps 2 --warmup 3 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/quick_launches.csv k_ws_clear 2
fi
if [ -n "$FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:${FULLK:-k_dd_serve|k_dd_pick|k_sage_rank128|k_grp_rows|k_grp_items|k_grp_count}" \
    --launch-skip ${FULLS:-40} --launch-count ${FULLC:-8} \
    -o gpurun_out/quick_full -f python tools/profile_bulk.py --mode dedup --warm 1 > gpurun_out/quick_full.log 2>&1
tail -2 gpurun_out/quick_full.log
fi
