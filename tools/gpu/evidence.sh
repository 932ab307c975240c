# Round evidence: build, SASS listing, bench line, launch lists and ncu captures (tools/capture_evidence.sh).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
cuobjdump -sass paper_2311_02909_b200/libgnnbulk_b200.so > gpurun_out/sass_all.txt 2>&1
timeout 2400 bash tools/capture_evidence.sh > gpurun_out/evidence.log 2>&1
tail -3 gpurun_out/evidence.log
ls -la gpurun_out/ev_*
