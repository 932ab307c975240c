#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root): bench
# line, launch lists and ncu captures of the headline SAGE dedup bulk and the
# LADIES bulk.  Each ncu command runs only after the same program exited 0
# without ncu.  Outputs land in gpurun_out/ (summarised into profiles/ by
# tools/evidence_summary.sh and tools/traffic_json.py).
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/ev_bench.json 2> $O/ev_bench.err || exit 1
python tools/profile_bulk.py --mode dedup > $O/ev_pb_dedup.log 2>&1 || exit 1
python tools/profile_bulk.py --sampler ladies > $O/ev_pb_ladies.log 2>&1 || exit 1
# launch lists (one warm bulk + one measured bulk)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev_launches_dedup.csv \
    python tools/profile_bulk.py --mode dedup --warm 1 > $O/ev_ncu_a.log 2>&1
ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/ev_launches_dedup_warm.csv python tools/profile_bulk.py --mode dedup --warm 1 \
    > $O/ev_ncu_a2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev_launches_ladies.csv \
    python tools/profile_bulk.py --sampler ladies --warm 1 > $O/ev_ncu_b.log 2>&1
# DRAM traffic of every sampling launch of the second bulk (layer 1: the
# P-free pick; layers 2-3: pick + 3 serve tiers)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv -k "regex:k_dd_serve|k_dd_pick|k_sage_pick" --launch-skip 9 --launch-count 9 \
    --log-file $O/ev_traffic_dedup.csv python tools/profile_bulk.py --mode dedup --warm 1 > $O/ev_ncu_c.log 2>&1
# full captures: layer 3 of the dedup bulk (grouping, pick, serve tiers,
# rank), layer 2 of LADIES.  Per bulk the regex matches 3 rank launches and
# count/items/rows/pick/serve x3 of layers 2 and 3: 17; the second bulk's
# layer 3 starts at 17 + 1 + 7 + 1 (layer 1 rank, layer 2, its rank) = 26
ncu --set full --clock-control none --import-source on \
    -k "regex:k_dd_serve|k_dd_pick|k_sage_rank128|k_grp_rows|k_grp_items|k_grp_count" \
    --launch-skip 26 --launch-count 8 \
    -o $O/ev_dedup_full -f python tools/profile_bulk.py --mode dedup --warm 1 > $O/ev_ncu_d.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_lad_tile$|k_lad_extract" \
    --launch-skip 8 --launch-count 2 -o $O/ev_ladies_full -f \
    python tools/profile_bulk.py --sampler ladies --warm 1 > $O/ev_ncu_e.log 2>&1
echo done
