python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi -L
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q > gpurun_out/pytest_mg.log 2>&1
tail -3 gpurun_out/pytest_mg.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tests/dist_exec_check.py > gpurun_out/mg_check.log 2>&1
grep -E "PASS|FAIL|column" gpurun_out/mg_check.log | head -30
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --dist 15d --c 1 > gpurun_out/bench_15d_p2.json 2> gpurun_out/bench_15d_p2.err
tail -c 1500 gpurun_out/bench_15d_p2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
grep -o '"value": [0-9.]*, "unit": "minibatches/s", "n_gpus": 2[^}]*' gpurun_out/bench_n2.json | head -2
