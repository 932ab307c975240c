"""Per-kernel totals of the last bulk in an ncu --metrics gpu__time_duration.sum
CSV launch list.  usage: launch_summary.py launches.csv FIRST_KERNEL_SUBSTR BULKS"""
import collections
import csv
import sys


def main():
    path, first, nb = sys.argv[1], sys.argv[2], int(sys.argv[3])
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    kn, val, unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    seq = [(r[kn].split("(")[0].replace("void ", ""),
            float(r[val].replace(",", "")) * scale.get(r[unit], 1.0)) for r in data]
    # the last bulk starts at the last run of consecutive FIRST_KERNEL launches
    hits = [k for k, (n, _) in enumerate(seq) if first in n]
    starts = [k for i, k in enumerate(hits) if i == 0 or hits[i - 1] != k - 1]
    if len(starts) >= nb:
        last = seq[starts[-1]:]
    else:  # markers absent per bulk: split evenly
        bulk = seq[hits[0]:]
        last = bulk[-(len(bulk) // nb):]
    per = len(last)
    agg = collections.OrderedDict()
    cnt = collections.Counter()
    for n, v in last:
        agg[n] = agg.get(n, 0.0) + v
        cnt[n] += 1
    T = sum(agg.values())
    print(f"one bulk: {per} launches, {T / 1e3:.3f} ms (cold-cache, serialised)")
    print("| kernel | launches | time | share |\n|---|---|---|---|")
    for n, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"| {n} | {cnt[n]} | {v / 1e3:.3f} ms | {100 * v / T:.1f}% |")


if __name__ == "__main__":
    main()
