# papers-shape 1.5D (cfg5): SAGE + LADIES at p = N, c = 2 and p = 2, c = 1
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for pc in "$N 2" "2 1"; do
  set -- $pc
  timeout 1500 $TR $1 --master-addr 127.0.0.1 --master-port 2952$1 bench.py --gpus $1 --workload papers --dist 15d --c $2 --fetch ${FETCH:-auto} --steps 10 --warmup 3 --no-cpu-baseline --no-aggregation --no-pfree > gpurun_out/mg_15d_papers_p$1_c$2.json 2> gpurun_out/mg_15d_papers_p$1_c$2.err
  echo "papers 15d p=$1 c=$2 $(grep -o '"value": [0-9.]*' gpurun_out/mg_15d_papers_p$1_c$2.json | head -2 | tr '\n' ' ') $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mg_15d_papers_p$1_c$2.json | head -2 | tr '\n' ' ')"
  tail -2 gpurun_out/mg_15d_papers_p$1_c$2.err
done
