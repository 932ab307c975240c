# Rebuild gb_sage.o with each EXTRA flag set in $FLAGS (";"-separated); papers-shape SAGE ms/bulk.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
IFS=';' read -ra FS <<< "$FLAGS"
for f in "${FS[@]}"; do
  touch paper_2311_02909_b200/csrc/gb_sage.cu
  make -s -C paper_2311_02909_b200/csrc EXTRA="$f" > gpurun_out/sweep_build.log 2>&1 || { echo "build failed: $f"; continue; }
  for rep in 1 2; do
    timeout 600 python bench.py --workload papers --steps 30 --warmup 3 --no-pfree --no-ladies --no-cpu-baseline --no-aggregation > gpurun_out/sweep_p.log 2>&1
    echo "$rep [$f] $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_p.log | head -1)"
  done
done
