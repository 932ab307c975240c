#!/bin/bash
# Summaries of a tools/capture_evidence.sh run (gpurun_out/ev_*) for
# profiles/r2_ncu_summary.md: launch lists, full-capture tables and the
# source lines with the most warp-stall samples.  Prints markdown to stdout.
set -u
O=${1:-gpurun_out}
echo "## Launch list, dedup bulk (cold-cache, serialised)"; echo
python tools/launch_summary.py $O/ev_launches_dedup.csv k_ws_clear 2; echo
echo -n "Warm-cache list (--cache-control none): "
python tools/launch_summary.py $O/ev_launches_dedup_warm.csv k_ws_clear 2 2>/dev/null | head -1 | sed "s/cold-cache/warm-cache/"; echo
echo "## Launch list, LADIES bulk (cold-cache, serialised)"; echo
python tools/launch_summary.py $O/ev_launches_ladies.csv k_lad_tiles 2; echo
echo "## Full captures (layer 3 of the dedup bulk; layer 2 of the LADIES bulk)"; echo
python tools/ncu_summary.py $O/ev_dedup_full.ncu-rep | sed 's|## gpurun_out/|### |'; echo
python tools/ncu_summary.py $O/ev_ladies_full.ncu-rep | sed 's|## gpurun_out/|### |'; echo
echo "## Where the time goes (source lines, warp-stall samples)"; echo
for f in "k_dd_pick<(int)5" "k_sage_rank128" "k_grp_rows" "k_grp_count"; do
  timeout 300 python tools/ncu_lines.py $O/ev_dedup_full.ncu-rep "$f" 10; echo
done
for f in "k_lad_tile" "k_lad_extract"; do
  timeout 300 python tools/ncu_lines.py $O/ev_ladies_full.ncu-rep "$f" 10; echo
done
