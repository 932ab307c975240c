# Serve-tier sweep: bench (dedup only) under GB_SERVE_TIERS=hi0,hi1, twice each.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for rep in 1 2; do
for t in ${TIERS:-"1024,8192" "1024,4096" "2048,4096" "2048,8192" "1536,4096" "2048,3072" "1024,3072"}; do
  GB_SERVE_TIERS=$t timeout 300 python bench.py --steps 100 --warmup 5 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/sweep_$t.log 2>&1
  echo "$rep $t $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_$t.log | head -1)"
done
done
