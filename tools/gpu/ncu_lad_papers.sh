python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python tools/profile_bulk.py --workload papers --sampler ladies --warm 0 > gpurun_out/plp.log 2>&1 || { tail -5 gpurun_out/plp.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_lad_tile$" --launch-skip 14 --launch-count 1 \
  -o gpurun_out/lad_papers_full -f python tools/profile_bulk.py --workload papers --sampler ladies --warm 0 > gpurun_out/plp_ncu.log 2>&1
tail -2 gpurun_out/plp_ncu.log
