# papers-shape replicated SAGE at 1, 2 and N GPUs (cfg4)
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for n in 1 2 $N; do
  timeout 1200 $TR $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --workload papers --steps 20 --warmup 3 --no-cpu-baseline --no-aggregation --no-pfree > gpurun_out/mg_papers_n$n.json 2> gpurun_out/mg_papers_n$n.err
  echo "papers replicated n=$n $(grep -o '"value": [0-9.]*' gpurun_out/mg_papers_n$n.json | head -1) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mg_papers_n$n.json | head -1)"
done
