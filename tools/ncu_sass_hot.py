"""Hottest SASS instructions (warp-stall samples) of the first kernel in an ncu report.

    python tools/ncu_sass_hot.py REPORT [N]
"""
import csv
import io
import subprocess
import sys


def main(path, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    data = []
    tot = 0
    for r in rows[1:]:
        try:
            smp = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        tot += smp
        data.append((smp, r))
    data.sort(key=lambda t: -t[0])
    print(f"total samples {tot}")
    for smp, r in data[:n]:
        st = sorted(((int(r[ci[c]] or 0), c[6:]) for c in stall_cols if (r[ci[c]] or "0").isdigit()), reverse=True)[:3]
        print(f"{smp:6d} {100*smp/tot:5.1f}% {r[ci['Address']]:>6s} {r[ci['Source']][:60]:60s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
