python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all8.log 2>&1
tail -15 gpurun_out/pytest_all8.log
