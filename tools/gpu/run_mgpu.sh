# Multi-GPU evidence (run under gpurun --gpus N): NCCL parity of the
# distributed executors, replicated and 1.5D bench lines.
set -u
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 900 python -m pytest tests/test_multigpu_gpu.py -m gpu -x -q > gpurun_out/mg_pytest.log 2>&1; tail -2 gpurun_out/mg_pytest.log
for n in 2 $N; do
  timeout 600 $TR $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 50 --warmup 5 --no-cpu-baseline --no-aggregation > gpurun_out/mg_bench_n$n.json 2> gpurun_out/mg_bench_n$n.err
  echo "replicated n=$n $(grep -o '"value": [0-9.]*' gpurun_out/mg_bench_n$n.json | head -1) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mg_bench_n$n.json | head -1)"
done
for pc in "$N 2" "$N 1" "2 1"; do
  set -- $pc
  timeout 900 $TR $1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $1 --dist 15d --c $2 --steps 20 --warmup 3 --no-cpu-baseline --no-aggregation --no-pfree > gpurun_out/mg_15d_p$1_c$2.json 2> gpurun_out/mg_15d_p$1_c$2.err
  echo "15d p=$1 c=$2 $(grep -o '"value": [0-9.]*' gpurun_out/mg_15d_p$1_c$2.json | head -1) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mg_15d_p$1_c$2.json | head -1)"
done
if [ "${PAPERS:-0}" = 1 ]; then
  timeout 1500 $TR $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --workload papers --steps 20 --warmup 3 --no-cpu-baseline --no-aggregation --no-pfree --no-ladies > gpurun_out/mg_papers_n$N.json 2> gpurun_out/mg_papers_n$N.err
  echo "papers replicated n=$N $(grep -o '"value": [0-9.]*' gpurun_out/mg_papers_n$N.json | head -1)"
fi
