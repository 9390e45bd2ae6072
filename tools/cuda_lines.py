#!/usr/bin/env python
"""Aggregate an `ncu --page source --print-source cuda,sass --csv` export by CUDA source line.
    python tools/cuda_lines.py export.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file, hdr = None, None
agg = collections.Counter(); text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        n = int(r[ie] or 0)
    except ValueError:
        continue
    if r[0] and r[0].isdigit():
        key = (cur_file, int(r[0])); text[key] = r[1].strip()[:80]
        agg[key] += n
tot = sum(agg.values()) or 1
print("total", tot)
for (f, l), n in agg.most_common(top):
    print(f"{n / tot * 100:5.1f}% {f}:{l} {text.get((f, l), '')}")
