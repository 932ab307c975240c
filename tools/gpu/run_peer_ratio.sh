N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for r in 1 2 4; do
  for w in products papers; do
    GB_DIRECT_RATIO=$r timeout 900 $TR $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --workload $w --dist 15d --c 2 --steps 20 --warmup 3 --no-cpu-baseline --no-aggregation --no-pfree --no-ladies > gpurun_out/pr.json 2> gpurun_out/pr.err
    echo "ratio=$r $w p=$N c=2 $(grep -o '"value": [0-9.]*' gpurun_out/pr.json | head -1)"
  done
done
