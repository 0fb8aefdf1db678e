"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/r1a/launches.csv > profiles/r1/launches_summary.txt
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]   # skip the program's own output
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    mi = hdr.index("Metric Name")
    rows = [rows[0]] + [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {sum(a[0] for a in agg.values())} launches, {tot / 1e3:.1f} us total (cold-cache, serialised)")
    print(f"{'kernel':50s} {'n':>5s} {'total_us':>10s} {'us/launch':>10s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:50s} {n:5d} {t / 1e3:10.1f} {t / n / 1e3:10.2f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
