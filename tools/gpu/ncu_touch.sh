python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_rec_scan_touch|k_enum_touch|k_touch" --launch-skip 6 --launch-count 3 \
  -o gpurun_out/touch_full -f python tools/profile_bulk.py --workload papers --mode dedup --warm 0 > gpurun_out/touch_ncu.log 2>&1
tail -2 gpurun_out/touch_ncu.log
