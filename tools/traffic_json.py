"""Refresh profiles/ncu_traffic.json from an ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum CSV of one dedup bulk's sampling
launches (tools/capture_evidence.sh): layer 1 k_sage_pick<1> (P-free), then
per layer one k_dd_pick and the three k_dd_serve tiers.  Writes
"dedup_sampling" (all of them, per layer: the bench's roofline kernel),
"k_dd_pick" and "k_dd_serve".

usage: traffic_json.py TRAFFIC.csv [SOURCE_NOTE]"""
import collections
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path = sys.argv[1]
    note = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(path)
    rows = [r for r in csv.reader(open(path)) if r]
    i = [k for k, r in enumerate(rows) if r[0] == "ID"][0]
    h = rows[i]
    kn, mn, mv, idc = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                       h.index("ID"))
    per = collections.OrderedDict()  # launch id -> (name, bytes)
    for r in rows[i + 1:]:
        if r[mn] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        name = r[kn].split("(")[0].replace("void ", "").replace("gb::", "")
        b = float(r[mv].replace(",", ""))
        nm, acc = per.get(r[idc], (name, 0.0))
        per[r[idc]] = (nm, acc + b)
    serve, pick, core = [], [], []
    for name, b in per.values():
        if name.startswith("k_dd_pick") or name.startswith("k_sage_pick"):
            pick.append(b)  # one pick launch opens each layer
            serve.append(0.0)
            core.append(b)
        elif name.startswith("k_dd_serve") and serve:
            serve[-1] += b
            core[-1] += b
    out_path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    d = json.load(open(out_path))
    d["k_dd_serve"] = {"per_layer_bytes": serve, "bulk_bytes": sum(serve),
                       "source": note + " (ncu --metrics dram__bytes_read.sum,"
                       "dram__bytes_write.sum; per layer the 3 serve tier launches)"}
    d["k_dd_pick"] = {"per_layer_bytes": pick, "bulk_bytes": sum(pick), "source": "same capture"}
    d["dedup_sampling"] = {"per_layer_bytes": core, "bulk_bytes": sum(core),
                           "source": "same capture: per layer the pick launch (layer 1 "
                                     "k_sage_pick<1>, then k_dd_pick) and the serve tiers"}
    json.dump(d, open(out_path, "w"), indent=1)
    print(json.dumps({k: d[k] for k in ("dedup_sampling", "k_dd_serve", "k_dd_pick")}, indent=1))


if __name__ == "__main__":
    main()
