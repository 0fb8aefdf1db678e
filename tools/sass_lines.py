"""Attribute ncu SASS stall samples of one kernel to CUDA source lines.

    python tools/sass_lines.py REPORT KERNEL_SUBSTR [N]

Needs the same libtomesh.so that was profiled (nvdisasm -g line info).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_line_map(mangled_substr):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1009_4975_b200", "libtomesh.so")],
                   cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.startswith("tomesh") and f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    funcs = {}
    cur, line, idx = None, None, 0
    for l in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m:
            line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m and cur is not None:
            funcs[cur].append((int(m.group(1), 16), line, m.group(2)))
    keys = [k for k in funcs if mangled_substr in k]
    return funcs[keys[0]] if keys else None


def main(rep, kname, n=30, which=-1):
    """which: index among the report's launches whose demangled name contains
    the kernel's short name (default: the last one)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    short = re.sub(r"I.*", "", re.sub(r"^_ZN\d+tomesh\d+", "", kname))
    cand = [b for b in blocks if short in b["name"]]
    blk = cand[which]
    hdr = blk["rows"][0]
    ci = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    body = blk["rows"][1:]
    base = int(body[0][ci["Address"]], 16)
    fmap = sass_line_map(kname)
    bymap = {off: ln for off, ln, _ in fmap} if fmap else {}
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = 0
    for r in body:
        try:
            smp = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError):
            continue
        off = int(r[ci["Address"]], 16) - base
        ln = bymap.get(off, "?")
        tot += smp
        agg[ln]["_all"] += smp
        for c in stall_cols:
            v = r[ci[c]]
            if v and v.isdigit():
                agg[ln][c[6:]] += int(v)
    print(f"total samples {tot}")
    for ln, c in sorted(agg.items(), key=lambda t: -t[1]["_all"])[:n]:
        top = [(k, v) for k, v in c.most_common(4) if k != "_all"][:3]
        print(f"{c['_all']:7d} {100 * c['_all'] / tot:5.1f}%  {ln:32s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30,
         int(sys.argv[4]) if len(sys.argv) > 4 else -1)


def top_instructions(rep, kname, line_suffix, n=10, which=-1):
    """The SASS instructions of one source line with the most samples."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    short = re.sub(r"I.*", "", re.sub(r"^_ZN\d+tomesh\d+", "", kname))
    blk = [b for b in blocks if short in b["name"]][which]
    hdr = blk["rows"][0]
    ci = {h: i for i, h in enumerate(hdr)}
    body = blk["rows"][1:]
    base = int(body[0][ci["Address"]], 16)
    fmap = sass_line_map(kname)
    bymap = {off: (ln, ins) for off, ln, ins in fmap}
    res = []
    for r in body:
        off = int(r[ci["Address"]], 16) - base
        ln, ins = bymap.get(off, ("?", "?"))
        if ln.endswith(line_suffix):
            res.append((int(r[ci["Warp Stall Sampling (All Samples)"]] or 0), hex(off), ins))
    for t in sorted(res, reverse=True)[:n]:
        print(t)


def inst_by_line(rep, kname, n=40, which=-1):
    """Executed warp instructions per source line and opcode (one launch)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    short = re.sub(r"I.*", "", re.sub(r"^_ZN\d+tomesh\d+", "", kname))
    blk = [b for b in blocks if short in b["name"]][which]
    hdr = blk["rows"][0]
    ci = {h: i for i, h in enumerate(hdr)}
    body = blk["rows"][1:]
    base = int(body[0][ci["Address"]], 16)
    fmap = sass_line_map(kname)
    bymap = {off: (ln, ins) for off, ln, ins in fmap}
    agg = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for r in body:
        off = int(r[ci["Address"]], 16) - base
        ln, ins = bymap.get(off, ("?", "?"))
        ex = int(r[ci["Instructions Executed"]] or 0)
        op = re.sub(r"^@!?U?P\w+\s+", "", ins.strip()).split()[0].split(".")[0] if ins.strip() else "?"
        agg[ln][op] += ex
        tot[op] += ex
    allx = sum(tot.values())
    print(f"total executed {allx}")
    for ln, c in sorted(agg.items(), key=lambda t: -sum(t[1].values()))[:n]:
        sm = sum(c.values())
        print(f"{sm:10d} {100 * sm / allx:5.1f}%  {ln:30s} {c.most_common(4)}")
