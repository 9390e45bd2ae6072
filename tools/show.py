#!/usr/bin/env python
"""Print value / kernel / frac of bench JSON lines: python tools/show.py TAG [configs]"""
import json, sys
tag = sys.argv[1]
for c in (sys.argv[2:] or ["c1", "c2", "c3", "c4", "c5", "g1", "n2"]):
    try:
        d = json.load(open(f"gpurun_out/bench_{c}_{tag}.json"))
    except Exception:
        continue
    r = d["roofline"]
    e = (d.get("e2e") or {}).get("value")
    print(f"{c}: value {d['value']:.3e} kernel {r['achieved']:.3e} frac {r['frac']:.3f} ms/step {d['ms_per_step']:.3f}"
          + (f" e2e {e:.3e}" if e else "") + f" cold {d['config'].get('cold_rerun_chunks_last_step')}")
