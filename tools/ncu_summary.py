"""Summarise an ncu report (raw page) into a small table for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [more...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_sector_hit_rate.pct", "L2_hit%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
]


def main():
    for path in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        print(f"## {path}")
        cols = [(m, n) for m, n in METRICS if m in hdr]
        print("| kernel | " + " | ".join(n for _, n in cols) + " |")
        print("|---" * (len(cols) + 1) + "|")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0]
            vals = []
            for m, _ in cols:
                i = hdr.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            print(f"| {name} | " + " | ".join(vals) + " |")
        print()


if __name__ == "__main__":
    main()
