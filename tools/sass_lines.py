#!/usr/bin/env python
"""Attribute an ncu SASS source export (`--page source --csv --print-source sass`,
gzipped or not) to CUDA source lines, using the line table of the cubin the
profiled library was built from (nvdisasm -g).

    python tools/sass_lines.py EXPORT.csv[.gz] OBJ.o KERNEL_SUBSTRING [top]

The export's addresses are absolute; offsets are taken from the kernel's first
instruction, which nvdisasm numbers 0."""
import collections
import csv
import gzip
import io
import os
import re
import subprocess
import sys
import tempfile

exp, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

opener = gzip.open if exp.endswith(".gz") else open
rows = list(csv.reader(io.TextIOWrapper(opener(exp, "rb"))))
hdr = rows[1]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
prof = [(int(r[ia], 16), int(r[ie] or 0), int(r[iss] or 0), r[isrc].strip()) for r in rows[2:] if len(r) > ie]
base = prof[0][0]

with tempfile.TemporaryDirectory() as td:
    subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, stdout=subprocess.DEVNULL)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.check_output(["nvdisasm", "-g", "-c", os.path.join(td, cub)], text=True)

# pick the function whose text contains the kernel name substring and whose
# instruction sequence matches the export's first opcodes
funcs = re.split(r"\n//-+ \.text\.", sass)
line_of = None
for f in funcs:
    name = f.split(" ", 1)[0]
    if kname not in name:
        continue
    cur = None
    m = {}
    ops = {}
    for ln in f.splitlines():
        mm = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if mm:
            cur = (os.path.basename(mm.group(1)), int(mm.group(2)))
            continue
        mi = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if mi:
            off = int(mi.group(1), 16)
            m[off] = cur
            ops[off] = mi.group(2).split()[0] if mi.group(2).split() else ""
    first = prof[0][3].split()[0]
    if ops.get(0, "").lstrip("@!P0123456789 ") == first.lstrip("@!P0123456789 ") and len(m) >= len(prof) * 0.9:
        line_of = m
        print("function", name[:100], "instructions", len(m))
        break
if line_of is None:
    sys.exit("kernel not found / no match")

agg = collections.Counter()
st = collections.Counter()
for a, n, s, _ in prof:
    key = line_of.get(a - base)
    agg[key] += n
    st[key] += s
tot = sum(agg.values()) or 1
stot = sum(st.values()) or 1
print(f"total instructions {tot:.4g}")
src_cache = {}


def text(key):
    if key is None:
        return ""
    f, l = key
    if f not in src_cache:
        path = None
        for root, _, files in os.walk("paper_2501_17168_b200"):
            if f in files:
                path = os.path.join(root, f)
        src_cache[f] = open(path).read().splitlines() if path else []
    lines = src_cache[f]
    return lines[l - 1].strip()[:90] if 0 < l <= len(lines) else ""


for key, n in agg.most_common(top):
    print(f"{n / tot * 100:5.1f}% instr {st[key] / stot * 100:5.1f}% stall  {key[0] if key else '?'}:{key[1] if key else ''}  {text(key)}")
