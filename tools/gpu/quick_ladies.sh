# Build, LADIES parity tests, LADIES cfg3 bench value.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
[ -z "$NOTEST" ] && { timeout 900 python -m pytest tests/test_ladies_gpu.py -m gpu -x -q > gpurun_out/ql_pytest.log 2>&1; tail -2 gpurun_out/ql_pytest.log; }
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-pfree --no-cpu-baseline --no-aggregation > gpurun_out/ql_bench.json 2> gpurun_out/ql_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/ql_bench.json').read().strip().splitlines()[-1])
l=d['ladies_cfg3']; print('ladies', l['value'], l['ms_per_step'], 'sage', d['value'])"
done
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ql_launches.csv python tools/profile_bulk.py --sampler ladies --warm 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/ql_launches.csv k_lad_tiles 2 | head -12
fi
if [ -n "$PAPERS" ]; then
timeout 900 python bench.py --workload papers --steps 5 --warmup 3 --no-pfree --no-cpu-baseline --no-aggregation > gpurun_out/pl_bench.json 2> gpurun_out/pl_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/pl_bench.json').read().strip().splitlines()[-1])
l=d['ladies_cfg3']; print('papers ladies', l['value'], l['ms_per_step'])"
fi
