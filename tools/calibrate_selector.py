#!/usr/bin/env python
"""Selector (c) calibration (PAPER §V-B "Threshold Analysis for Adaptive
Parallelism", re-measured on B200): time forced kernel (a) and
forced kernel (b) of evogp_sr_fitness over a D x P x L grid (M-paper mix,
Pagie-n targets) and record, per (P, L), the smallest D from which (b) is
faster. Writes selector_table.json and the compiled-in table
paper_2501_17168_b200/csrc/selector_table.inc.

    python tools/calibrate_selector.py [--quick]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2501_17168_b200 as evogp  # noqa: E402
import synth  # noqa: E402

WORK_CAP = 6e10  # node x datapoint steps per timed call (keeps each call < ~40 ms)


def time_call(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "selector_table.json"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    Ps = [100, 1000, 10_000, 100_000] if not a.quick else [1000, 10_000]
    Ls = [15, 63, 127] if not a.quick else [63]
    Ds = [1 << k for k in range(5, 23)]
    rows = []
    table = []
    for L in Ls:
        for P in Ps:
            pt = synth.trees(2501017168 + 17, 0, P, L, synth.M_PAPER, 8)
            t, v, s = (torch.from_numpy(x).to(dev) for x in evogp.tensorize(pt.offsets, pt.types, pt.values, L, 8))
            nodes = int(np.diff(pt.offsets).sum())
            crossover = None
            for D in Ds:
                if nodes * D > WORK_CAP:
                    break
                X, y = synth.config_data(synth.Config("cal", P, L, 8, 1, D, "uniform", -1.0, 1.0, 0.0, 17), 0, D)
                Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
                out = torch.empty(P, dtype=torch.float64, device=dev)
                ms = {}
                for strat in ("inter", "intra"):
                    ms[strat] = time_call(lambda: evogp.sr_fitness(t, v, s, Xd, yd, strategy=strat, out=out))
                auto = evogp.select_strategy(P, D, L)
                rows.append({"L": L, "P": P, "D": D, "ms_inter": ms["inter"], "ms_intra": ms["intra"],
                             "gpops_inter": nodes * D / ms["inter"] * 1e3, "gpops_intra": nodes * D / ms["intra"] * 1e3,
                             "auto_before": auto})
                print(json.dumps(rows[-1]), flush=True)
                if crossover is None and ms["intra"] < ms["inter"]:
                    crossover = D
            table.append({"L": L, "P": P, "crossover_D": crossover})
    res = {"when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "device": torch.cuda.get_device_name(0),
           "sms": torch.cuda.get_device_properties(0).multi_processor_count, "mix": "paper", "n_in": 8,
           "method": "median of 5 CUDA-event timings of evogp_sr_fitness, forced inter vs forced intra",
           "rows": rows}
    finish(res, a.out)


def finish(res, path):
    res["table"] = robust_table(res["rows"])
    res["regret_max"], res["regret_mean"] = regret(res["rows"], res["table"])
    res["regret_max_ge_0.5ms"], res["regret_mean_ge_0.5ms"] = regret(res["rows"], res["table"], 0.5)
    paper = [{"L": e["L"], "P": e["P"], "crossover_D": res["sms"] * 128} for e in res["table"]]
    res["paper_rule_regret_max"], res["paper_rule_regret_mean"] = regret(res["rows"], paper)
    res["paper_rule_regret_max_ge_0.5ms"], _ = regret(res["rows"], paper, 0.5)
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    write_inc(res)
    print("table:", res["table"])
    print({k: round(v, 4) for k, v in res.items() if "regret" in k})


def robust_table(rows):
    """Per (L, P): the smallest swept D at which (b) is faster and stays at
    least 0.97x as fast as (a) for every larger swept D (noise-robust); None if
    there is no such D."""
    from collections import defaultdict
    g = defaultdict(list)
    for r in rows:
        g[(r["L"], r["P"])].append(r)
    out = []
    for (L, P), rs in sorted(g.items()):
        rs.sort(key=lambda r: r["D"])
        ratio = [r["ms_inter"] / r["ms_intra"] for r in rs]
        cross = None
        for i, r in enumerate(rs):
            if ratio[i] >= 1.0 and all(x >= 0.97 for x in ratio[i:]):
                cross = r["D"]
                break
        truncated = rs[-1]["D"] < (1 << 20)  # the work cap stopped the sweep early
        if cross is None and truncated and out and out[-1]["L"] == L and out[-1]["crossover_D"]:
            cross = out[-1]["crossover_D"]  # inherit from the next smaller P
        out.append({"L": L, "P": P, "crossover_D": cross})
    return out


def regret(rows, table, min_ms=0.0):
    """Fraction by which the table's choice is slower than the best kernel
    (over rows whose best time is >= min_ms)."""
    worst, tot = 0.0, []
    for r in rows:
        if min(r["ms_intra"], r["ms_inter"]) < min_ms:
            continue
        e = min((e for e in table), key=lambda e: (abs(np.log(e["L"] / r["L"])), abs(np.log(e["P"] / r["P"]))))
        intra = e["crossover_D"] is not None and r["D"] >= e["crossover_D"]
        t = r["ms_intra"] if intra else r["ms_inter"]
        best = min(r["ms_intra"], r["ms_inter"])
        worst = max(worst, t / best - 1)
        tot.append(t / best - 1)
    return worst, float(np.mean(tot))


def write_inc(res):
    """Compiled-in crossover table: {L, P, crossover D} (0 = intra never won)."""
    lines = ["// generated by tools/calibrate_selector.py from selector_table.json — do not edit",
             f"// {res['device']} ({res['sms']} SMs), {res['when']}, {res['method']}",
             "static const SelectorEntry kSelectorTable[] = {"]
    for e in res["table"]:
        lines.append(f"    {{{e['L']}, {e['P']}, {e['crossover_D'] or 0}}},")
    lines.append("};")
    with open(os.path.join(ROOT, "paper_2501_17168_b200", "csrc", "selector_table.inc"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
