# 1.5D split with / without direct peer rows: parity job, then products and papers benches
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_multigpu_gpu.py -m gpu -x -q > gpurun_out/pd_pytest.log 2>&1; tail -1 gpurun_out/pd_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for pd in 1 0; do
  for w in products papers; do
    for pc in "$N 2" "$N 1"; do
      set -- $pc
      GB_PEER_DIRECT=$pd timeout 900 $TR $1 --master-addr 127.0.0.1 --master-port 2954$1 bench.py --gpus $1 --workload $w --dist 15d --c $2 --steps 20 --warmup 3 --no-cpu-baseline --no-aggregation --no-pfree --no-ladies > gpurun_out/pd_${w}_p$1_c$2_$pd.json 2> gpurun_out/pd.err
      echo "peer_direct=$pd $w p=$1 c=$2 $(grep -o '"value": [0-9.]*' gpurun_out/pd_${w}_p$1_c$2_$pd.json | head -1)"
    done
  done
done
