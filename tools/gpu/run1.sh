set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "ingest or ladies" > gpurun_out/pytest_new.log 2>&1
tail -5 gpurun_out/pytest_new.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1
tail -5 gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.log 2>&1
tail -c 3000 gpurun_out/bench1.log
