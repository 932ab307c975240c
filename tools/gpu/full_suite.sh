# Full GPU suite (pytest -m gpu) and the reference pkg/tests run unmodified against the package
# (tools/reftests/prepare.sh must have populated .reftests/ in the snapshot).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1
tail -8 gpurun_out/pytest_all.log
cd .reftests && timeout 600 env PYTHONPATH=.:.. python -m pytest tests -q -p no:cacheprovider --ignore=tests/test_cli.py > ../gpurun_out/reftests.log 2>&1; cd ..
tail -25 gpurun_out/reftests.log
