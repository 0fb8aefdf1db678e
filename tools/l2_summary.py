"""Per-kernel medians of an ncu --metrics CSV (tools/gpu_l2_metrics.sh): duration,
L2 (lts) bytes and DRAM bytes per launch, and the implied GB/s.

    python tools/l2_summary.py c1.csv c2.csv ...
"""
import collections
import csv
import os
import statistics
import sys


def main(paths):
    for path in paths:
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        if not rows:
            print(os.path.basename(path), "no data")
            continue
        hdr = rows[0]
        ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
        per = collections.defaultdict(lambda: collections.defaultdict(dict))
        for r in rows[1:]:
            try:
                per[r[ki].split("(")[0]][r[ii]][r[mi]] = float(r[vi].replace(",", ""))
            except (ValueError, IndexError):
                continue
        for k, launches in per.items():
            ls = [v for v in launches.values() if "gpu__time_duration.sum" in v]
            if not ls:
                continue
            med = {m: statistics.median(v[m] for v in ls if m in v) for m in ls[0]}
            t = med["gpu__time_duration.sum"] * 1e-9
            l2 = med.get("lts__t_bytes.sum", 0.0)
            dram = med.get("dram__bytes_read.sum", 0.0) + med.get("dram__bytes_write.sum", 0.0)
            print(f"{os.path.basename(path)[:-4]:4s} {k[:40]:40s} n={len(ls):2d} {t * 1e6:8.1f} us  "
                  f"L2 {l2 / 1e6:8.1f} MB ({l2 / t / 1e9:7.0f} GB/s)  DRAM {dram / 1e6:8.1f} MB ({dram / t / 1e9:6.0f} GB/s)")


if __name__ == "__main__":
    main(sys.argv[1:])
