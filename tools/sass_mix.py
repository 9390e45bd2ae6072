#!/usr/bin/env python
"""Instruction mix + hot instructions of an ncu source-page SASS CSV (gz).
    python tools/sass_mix.py gpurun_out/sass_c2_h1.csv.gz [--hot 0.002] [--list A:B]"""
import argparse, collections, csv, gzip
ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--hot", type=float, default=0.0)
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
rows = list(csv.reader(gzip.open(a.csv, "rt")))
i0 = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[i0]; data = [r for r in rows[i0 + 1:] if len(r) == len(hdr)]
ie = hdr.index("Instructions Executed"); src = hdr.index("Source")
tot = sum(int(r[ie] or 0) for r in data)
print("total warp instructions", tot)
mn = collections.Counter()
for r in data:
    t = r[src].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    mn[op.split(".")[0]] += int(r[ie] or 0)
for k, v in mn.most_common(a.top):
    print(f"  {k:10s} {v / tot * 100:5.1f}%")
if a.hot:
    for i, r in enumerate(data):
        c = int(r[ie] or 0)
        if c > tot * a.hot:
            print(i, f"{c / 1e6:7.3f}M", r[src].strip()[:100])
