"""Per-launch durations of the last bulk in an ncu --metrics
gpu__time_duration.sum CSV launch list (the bulk starts at the last launch of
the marker kernel).  usage: bulk_launches.py launches.csv MARKER"""
import csv
import sys


def main():
    path, marker = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    kn, val, unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    seq = [(r[kn].split("(")[0].replace("void ", ""),
            float(r[val].replace(",", "")) * scale.get(r[unit], 1.0)) for r in data]
    idx = [k for k, (n, _) in enumerate(seq) if marker in n]
    last = seq[idx[-1]:]
    tot = 0.0
    for n, v in last:
        print(f"{v:9.1f} us  {n}")
        tot += v
    print(f"one bulk: {len(last)} launches, {tot / 1e3:.3f} ms (cold-cache, serialised)")


if __name__ == "__main__":
    main()
