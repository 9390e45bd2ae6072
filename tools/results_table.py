#!/usr/bin/env python
"""Markdown results table from bench JSON lines: python tools/results_table.py DIR_OR_TAG"""
import json, os, sys
src = sys.argv[1]
rows = ["| Config | value (GPops/s) | strategy | kernel (GPops/s) | roof frac | e2e (GPops/s) | oracle (GPops/s, cores) | notes |",
        "|---|---|---|---|---|---|---|---|"]
for c in ("c3", "c2", "c4", "c5", "c5b", "c1", "g1", "n2"):
    p = os.path.join(src, f"bench_{c}.json") if os.path.isdir(src) else f"gpurun_out/bench_{c}_{src}.json"
    if os.path.isdir(src) and not os.path.exists(p):
        p = os.path.join(src, f"{c}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    r = d["roofline"]
    e = (d.get("e2e") or {}).get("value")
    cb = d.get("cpu_baseline") or {}
    notes = []
    if r.get("unit") == "GB/s":
        notes.append(f"{r['achieved']:.0f} GB/s = {r['frac']:.3f} of HBM")
    if r.get("hbm_view"):
        notes.append(f"output store {r['hbm_view']['achieved']:.0f} GB/s = {r['hbm_view']['frac']:.3f} of HBM")
    if d.get("graph_replay"):
        notes.append(f"CUDA-graph replay {d['graph_replay']['value']:.3g} GPops/s")
    if c == "g1":
        notes.append("fitness kernel share %.2f" % r.get("step_share", {}).get("fitness", 0))
    kern = r["achieved"] if r.get("unit") != "GB/s" else r.get("alu_view", {}).get("achieved", 0)
    frac = r["frac"] if r.get("unit") != "GB/s" else r.get("alu_view", {}).get("frac", 0)
    rows.append(f"| {c} | {d['value']:.3g} | {d['config'].get('strategy')} | {kern:.3g} | {frac:.3f} | "
                + (f"{e:.3g}" if e else "–") + " | "
                + (f"{cb['value']:.2g} ({cb['cores']})" if cb else "–") + " | " + "; ".join(notes) + " |")
print("\n".join(rows))
