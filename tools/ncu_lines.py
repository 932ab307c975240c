"""Per-source-line warp-stall samples and executed instructions of one kernel
from an ncu report (cuda,sass source page).

usage: ncu_lines.py REPORT.ncu-rep FUNCTION_SUBSTR [TOP]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, fn = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    path = func = None
    hdr = None
    samp, inst, src = collections.Counter(), collections.Counter(), {}
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or fn not in (func or "") or not r[0].isdigit() or r[2] != "-":
            continue
        key = (path, int(r[0]))
        samp[key] += int(r[4])
        inst[key] += int(r[7])
        src[key] = r[1].strip()[:70]
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    print(f"{fn}: {ts} stall samples, {ti} warp instructions")
    print("| file:line | samples % | inst % | source |\n|---|---|---|---|")
    for key, v in samp.most_common(top):
        print(f"| {key[0]}:{key[1]} | {100 * v / ts:.1f} | {100 * inst[key] / ti:.1f} | `{src[key]}` |")


if __name__ == "__main__":
    main()
