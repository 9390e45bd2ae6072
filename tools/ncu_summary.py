#!/usr/bin/env python
"""Summarise an ncu --set full report (+ optional launch list) into the JSON
kept under profiles/ (bench.py reads `dram_bytes_per_launch` as `traffic`).

    python tools/ncu_summary.py REPORT.ncu-rep [--launches LAUNCHES.csv] --out profiles/X.json
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess

WANT = {
    "Duration": "duration",
    "Elapsed Cycles": "elapsed_cycles",
    "SM Frequency": "sm_frequency",
    "Executed Ipc Active": "ipc_active",
    "Issue Slots Busy": "issue_slots_busy_pct",
    "Compute (SM) Throughput": "sm_throughput_pct",
    "DRAM Throughput": "dram_throughput_pct",
    "Memory Throughput": "memory_throughput",
    "L1/TEX Hit Rate": "l1_hit_rate_pct",
    "L2 Hit Rate": "l2_hit_rate_pct",
    "Registers Per Thread": "registers_per_thread",
    "Dynamic Shared Memory Per Block": "dyn_smem_per_block",
    "Theoretical Active Warps per SM": "theoretical_warps_per_sm",
    "Achieved Active Warps Per SM": "achieved_warps_per_sm",
    "Eligible Warps Per Scheduler": "eligible_warps_per_scheduler",
    "Warp Cycles Per Issued Instruction": "warp_cycles_per_issued_instruction",
    "Executed Instructions": "executed_instructions",
    "Grid Size": "grid_size",
    "Block Size": "block_size",
    "Branch Efficiency": "branch_efficiency_pct",
}

RAW = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
    "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout
    start = out.find('"')
    return list(csv.reader(io.StringIO(out[start:])))


def num(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"report": a.report, "note": a.note}
    rows = ncu_csv(["-i", a.report, "--page", "details", "--csv"])
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        res.setdefault("kernel", d.get("Kernel Name"))
        k = WANT.get(d.get("Metric Name"))
        if k and k not in res:
            res[k] = {"value": num(d["Metric Value"]), "unit": d.get("Metric Unit")}
    raw = ncu_csv(["-i", a.report, "--page", "raw", "--csv"])
    rh, ru, rv = raw[0], raw[1], raw[2]
    for name in RAW:
        if name in rh:
            i = rh.index(name)
            res[name] = {"value": num(rv[i]), "unit": ru[i]}
    rb = res.get("dram__bytes_read.sum", {}).get("value")
    wb = res.get("dram__bytes_write.sum", {}).get("value")
    unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if isinstance(rb, float) and isinstance(wb, float):
        s1 = unit_scale.get(res["dram__bytes_read.sum"]["unit"], 1)
        s2 = unit_scale.get(res["dram__bytes_write.sum"]["unit"], 1)
        res["dram_bytes_per_launch"] = rb * s1 + wb * s2
    # warp-state sampling: share of samples per stall reason
    stalls = {}
    for i, name in enumerate(rh):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
            v = num(rv[i])
            if isinstance(v, float):
                stalls[name[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
    tot = sum(stalls.values())
    if tot > 0:
        res["stall_reasons_pct"] = {k: round(100.0 * v / tot, 1)
                                    for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]}
    # stall reasons from the source page (sampling)
    src = ncu_csv(["-i", a.report, "--page", "source", "--csv", "--print-source", "sass"])
    sh = src[1]
    data = [dict(zip(sh, r)) for r in src[2:] if len(r) == len(sh)]
    hist = collections.Counter()
    tot = 0
    for d in data:
        n = int(float(d.get("Instructions Executed") or 0))
        tot += n
        op = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip()).split(" ")[0].split(".")[0]
        hist[op] += n
    res["sass_instructions_executed"] = tot
    res["sass_opcode_mix_pct"] = {k: round(100.0 * v / max(tot, 1), 2) for k, v in hist.most_common(25)}
    if a.launches:
        lr = ncu_csv(["--version"])  # noqa: F841 (ensure ncu exists)
        with open(a.launches) as f:
            txt = f.read()
        lines = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
        lh = lines[0]
        per = collections.defaultdict(list)
        for r in lines[1:]:
            d = dict(zip(lh, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                per[d["Kernel Name"]].append(float(d["Metric Value"]))
        totals = {k: sum(v) for k, v in per.items()}
        allt = sum(totals.values())
        res["launch_list"] = {
            k: {"launches": len(per[k]), "mean_ns": sum(per[k]) / len(per[k]), "share_of_listed_time": totals[k] / allt}
            for k in sorted(totals, key=lambda x: -totals[x])}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in res if k in ("kernel", "duration", "dram_bytes_per_launch",
                                                    "issue_slots_busy_pct", "ipc_active")}, indent=None))


if __name__ == "__main__":
    main()
