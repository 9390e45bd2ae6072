#!/usr/bin/env python
"""Copy a gpu_profile_all.sh refresh (gpurun_out/) into profiles/: the ncu
summaries under the names bench.py reads (ncu_<config>_<kernel>_summary.json,
with the launch-list shares merged in), the launch lists, the SASS source
CSVs and the bench result lines.   python tools/install_profiles.py TAG"""
import collections
import csv
import json
import os
import shutil
import sys

TAG = sys.argv[1]
R = f"gpurun_out/summaries_{TAG}"


def launch_stats(path):
    per = collections.defaultdict(list)
    hdr = None
    for r in csv.reader(open(path)):
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"])
                u = d.get("Metric Unit", "ns")
                per[d["Kernel Name"]].append(v * {"us": 1e3, "ms": 1e6}.get(u, 1.0))
    allt = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share_of_listed_time": sum(v) / allt}
            for k, v in per.items() if "evogp" in k}


names = {}
for c in ["c2", "c3", "c4", "c5", "c5b", "n2"]:
    # named after the kernel the capture holds (the selector's choice), as bench.py looks it up
    d = json.load(open(f"{R}/prof_{c}_{TAG}.json"))
    kind = "paired" if "k_paired" in d["kernel"] else ("intra" if "k_intra" in d["kernel"] else "inter")
    out = names[c] = f"ncu_{c}_{kind}_summary.json"
    d["note"] = f"refresh {TAG}: bench.py --config {c}"
    d["launch_list"] = launch_stats(f"gpurun_out/launches_{c}_{TAG}.csv")
    json.dump(d, open("profiles/" + out, "w"), indent=1)
    shutil.copy(f"gpurun_out/launches_{c}_{TAG}.csv", f"profiles/launches_{c}_{TAG}.csv")
    shutil.copy(f"{R}/prof_{c}_{TAG}.sass.csv.gz", f"profiles/sass_{c}_{TAG}.csv.gz")
for k in ["k_eval", "k_prepare", "k_reproduce"]:
    d = json.load(open(f"{R}/prof_g1_{k}_{TAG}.json"))
    d["note"] = f"refresh {TAG}: bench.py --config g1 --warmup 20 (populations grown by 20 generations)"
    d["launch_list"] = launch_stats(f"gpurun_out/launches_g1_{TAG}.csv")
    json.dump(d, open(f"profiles/ncu_g1_{k}_summary.json", "w"), indent=1)
shutil.copy(f"gpurun_out/launches_g1_{TAG}.csv", f"profiles/launches_g1_{TAG}.csv")
os.makedirs(f"profiles/results_{TAG}", exist_ok=True)
for c in ["c1", "c2", "c3", "c4", "c5", "c5b", "n2", "g1"]:
    shutil.copy(f"gpurun_out/results_{TAG}/{c}.json", f"profiles/results_{TAG}/{c}.json")
for c in names:
    d = json.load(open("profiles/" + names[c]))
    print(c, d["kernel"][:30], "ipc", d["ipc_active"]["value"], "issue", d["issue_slots_busy_pct"]["value"],
          {k[:28]: round(v["share_of_listed_time"], 3) for k, v in d["launch_list"].items()})
