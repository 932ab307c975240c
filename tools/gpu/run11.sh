python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_all11.log 2>&1
tail -8 gpurun_out/pytest_all11.log
cd .reftests && timeout 600 env PYTHONPATH=.:.. python -m pytest tests -q -p no:cacheprovider --ignore=tests/test_cli.py > ../gpurun_out/reftests.log 2>&1; cd ..
tail -25 gpurun_out/reftests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench11.log 2>&1
grep -o '"value": [0-9.]*, "unit": "minibatches/s", "n_gpus": 1, "steps": 20, "warmup": 5, "ms_per_step": [0-9.]*' gpurun_out/bench11.log
grep -o '"e2e": {[^}]*' gpurun_out/bench11.log
