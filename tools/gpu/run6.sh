python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python tools/profile_bulk.py --mode dedup > gpurun_out/pb.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_dd_serve_a|k_dd_pick|k_grp_items|k_grp_rows|k_sage_rank8" \
   --launch-skip 25 --launch-count 5 -o gpurun_out/r2_dedup_full -f python tools/profile_bulk.py --mode dedup --warm 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/*.ncu-rep
