# papers-shape SAGE (cfg4 per GPU): bench value and launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload papers --steps 20 --warmup 3 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/ps_bench.json 2> gpurun_out/ps_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/ps_bench.json').read().strip().splitlines()[-1])
print('sage', d['value'], d['ms_per_step'], d['roofline']['per_layer_ms'], d['layers'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ps_launches.csv python tools/profile_bulk.py --workload papers --mode dedup --warm 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/ps_launches.csv k_ws_clear 2 2>/dev/null | head -24
