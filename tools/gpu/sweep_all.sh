# Rebuild the whole library with each EXTRA flag set in $FLAGS (";"-separated); SAGE ms/bulk (+ LADIES if LAD=1).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
IFS=';' read -ra FS <<< "$FLAGS"
for f in "${FS[@]}"; do
  touch paper_2311_02909_b200/csrc/*.cu
  make -s -C paper_2311_02909_b200/csrc EXTRA="$f" > gpurun_out/sweep_build.log 2>&1 || { echo "build failed: $f"; continue; }
  for rep in 1 2; do
    timeout 300 python bench.py --steps 100 --warmup 5 --no-pfree --no-cpu-baseline --no-aggregation $([ -z "$LAD" ] && echo --no-ladies) > gpurun_out/sweep_b.log 2>&1
    echo "$rep [$f] $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_b.log | head -1) $(grep -o '"ladies_cfg3": {[^}]*"ms_per_step": [0-9.]*' gpurun_out/sweep_b.log | grep -o '"ms_per_step": [0-9.]*$')"
  done
done
