python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_sage_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/profile_bulk.py --mode dedup > gpurun_out/pb.log 2>&1 && \
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dedup_warm.csv \
    python tools/profile_bulk.py --mode dedup --warm 1 > gpurun_out/ncu_a.log 2>&1
python tools/bulk_launches.py gpurun_out/launches_dedup_warm.csv k_set_i64 2>&1 | tail -40
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench5.log 2>&1
python - <<'PY'
import json
s=open("gpurun_out/bench5.log").read()
i=s.rfind('{"metric"')
d=json.loads(s[i:])
print({k:d.get(k) for k in ("value","ms_per_step","gpu_launches")})
print("roofline", d.get("roofline"))
print("pfree", d.get("pfree",{}).get("value"), "ladies", d.get("ladies_cfg3",{}).get("value"), "e2e", d.get("e2e",{}).get("value"))
print("parity", d.get("parity_full_size"))
PY
