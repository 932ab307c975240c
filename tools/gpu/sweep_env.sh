# Bench (dedup only) under VAR=value for each value in VALS: VAR=GB_SERVE_BULKMIN VALS="64 128" bash tools/gpu/sweep_env.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
[ -n "$TESTS" ] && { timeout 900 python -m pytest $TESTS -m gpu -x -q > gpurun_out/sweep_pytest.log 2>&1; tail -2 gpurun_out/sweep_pytest.log; }
for rep in 1 2; do
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/sweep_env.log 2>&1
  echo "$rep $VAR=$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_env.log | head -1)"
done
done
