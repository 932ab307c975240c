python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for t in "1024,8192" "512,8192" "2048,8192" "1024,4096" "1024,16384" "256,4096" "4096,16384"; do
  GB_SERVE_TIERS=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/sweep_$t.log 2>&1
  echo "$t $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_$t.log | head -1)"
done
