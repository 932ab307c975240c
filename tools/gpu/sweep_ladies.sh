# Rebuild gb_ladies.o with each EXTRA flag set in $FLAGS (";"-separated); LADIES cfg3 and papers values.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
IFS=';' read -ra FS <<< "$FLAGS"
for f in "${FS[@]}"; do
  touch paper_2311_02909_b200/csrc/gb_ladies.cu
  make -s -C paper_2311_02909_b200/csrc EXTRA="$f" > gpurun_out/sweep_build.log 2>&1 || { echo "build failed: $f"; continue; }
  echo "[$f]"
  NOTEST=1 PAPERS=${PAPERS:-} bash tools/gpu/quick_ladies.sh 2>&1 | grep ladies
done
