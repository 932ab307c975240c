python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench15.json 2> gpurun_out/bench15.err; tail -c 600 gpurun_out/bench15.err
python - <<'P'
import json; d=json.loads(open("gpurun_out/bench15.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d["gpu_launches"], d["clocks"])
print("cpu", d["cpu_baseline"]); print("lad", d.get("ladies_cfg3",{}).get("value"), "pfree", d["pfree"]["value"])
P
