"""Median warm duration per kernel from an `ncu --metrics gpu__time_duration.sum --csv` log.

    python tools/launch_median.py FILE.csv
"""
import collections
import csv
import io
import sys


def main(path):
    lines = [l for l in open(path).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        d[r[ki][:48]].append(v * (1e-3 if r[ui] == "nsecond" else 1.0))
    for k, v in d.items():
        print(f"{k:50s} n={len(v):4d} median_us={sorted(v)[len(v) // 2]:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
