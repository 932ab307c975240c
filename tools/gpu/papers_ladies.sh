# papers-shape LADIES: bench value and launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload papers --steps 5 --warmup 3 --no-pfree --no-cpu-baseline --no-aggregation > gpurun_out/pl_bench.json 2> gpurun_out/pl_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/pl_bench.json').read().strip().splitlines()[-1])
l=d['ladies_cfg3']; print('ladies', l['value'], l['ms_per_step'], l['layers']); print('sage', d['value'], d['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pl_launches.csv python tools/profile_bulk.py --workload papers --sampler ladies --warm 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/pl_launches.csv k_lad_tiles 2 2>/dev/null | head -14
