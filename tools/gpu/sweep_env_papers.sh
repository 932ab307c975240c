# papers-shape SAGE under VAR=value for each value in VALS
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for rep in 1 2; do
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --workload papers --steps 30 --warmup 3 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/sweep_ep.log 2>&1
  echo "$rep $VAR=$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_ep.log | head -1)"
done
done
