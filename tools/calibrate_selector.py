#!/usr/bin/env python
"""Selector (c) calibration (PAPER §V-B "Threshold Analysis for Adaptive
Parallelism", re-measured on B200).

Times forced kernel (a) (inter) and forced kernel (b) (intra) over the grid
  L in {15, 63, 127, 512} x P in {1e2 .. 1e6} x n_out in {1, 6} x D = 2^5 .. 2^22
(single output: evogp_sr_fitness on the M-paper mix; six outputs: Modi
evogp_eval on the M-full mix, p_modi 0.1 — the C2-C4 / C5 workloads), capped
at 1.2e11 node x datapoint steps and 8 GB of outputs per call. Each cell is the
median of 5 CUDA-event timings after 2 warm-ups.

The library's rule is a lookup table of the faster kernel per measured cell,
applied to the nearest cell in (log L, log P, log D) of the same output class
(paper_2501_17168_b200/csrc/selector_table.inc). The table is fitted on one
pass and scored on a second, independent pass (so noise counts against it):
regret = time of the chosen kernel / time of the faster kernel - 1, reported
separately for calls >= 0.5 ms and < 0.5 ms, next to the paper's rule
(D >= SMs x 128, reading R11).

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

WORK_CAP = 1.2e11  # node x datapoint steps per timed call (C3 itself, 1e11, is a cell)
OUT_CAP = 8 << 30  # eval output bytes (n_out > 1)
NODE_CAP = 2e8  # nodes per population (host generation + tensorize)


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


def sweep(Ls, Ps, n_outs, Ds, dev, tag):
    rows = []
    for n_out in n_outs:
        mix = synth.M_PAPER if n_out == 1 else synth.M_FULL
        for L in Ls:
            for P in Ps:
                if 0.77 * L * P > NODE_CAP:
                    continue
                pt = synth.trees(2501017168 + 17, 0, P, L, mix, 8, n_out, 0.1 if n_out > 1 else 0.0)
                t, v, s = (torch.from_numpy(x).to(dev)
                           for x in evogp.tensorize(pt.offsets, pt.types, pt.values, L, 8, n_out))
                nodes = int(np.diff(pt.offsets).sum())
                del pt
                for D in Ds:
                    if nodes * D > WORK_CAP or (n_out > 1 and P * D * n_out * 4 > OUT_CAP):
                        break
                    X, y = synth.config_data(synth.Config("cal", P, L, 8, n_out, D, "uniform", -1.0, 1.0, 0.0, 17),
                                             0, D)
                    Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
                    if n_out == 1:
                        out = torch.empty(P, dtype=torch.float64, device=dev)
                        call = lambda st: evogp.sr_fitness(t, v, s, Xd, yd, strategy=st, out=out)  # noqa: E731
                    else:
                        out = torch.empty((P, D, n_out), dtype=torch.float32, device=dev)
                        call = lambda st: evogp.eval(t, v, s, Xd, n_outputs=n_out, strategy=st, out=out)  # noqa: E731
                    ms = {st: time_call(lambda: call(st)) for st in ("inter", "intra")}
                    del out
                    rows.append({"L": L, "P": P, "n_out": n_out, "D": D, "ms_inter": ms["inter"],
                                 "ms_intra": ms["intra"], "gpops_inter": nodes * D / ms["inter"] * 1e3,
                                 "gpops_intra": nodes * D / ms["intra"] * 1e3})
                    print(tag, json.dumps(rows[-1]), flush=True)
                del t, v, s
                torch.cuda.empty_cache()
    return rows


def nearest(table, L, P, D, n_out):
    cls = n_out > 1
    best, bd = None, 1e300
    for e in table:
        if (e["n_out"] > 1) != cls:
            continue
        d = np.log(e["L"] / L) ** 2 + np.log(e["P"] / P) ** 2 + np.log(e["D"] / D) ** 2
        if d < bd:
            best, bd = e, d
    return best


def regret(rows, choose, min_ms=0.0, max_ms=1e30):
    rs = []
    for r in rows:
        best = min(r["ms_intra"], r["ms_inter"])
        if not (min_ms <= best < max_ms):
            continue
        t = r["ms_intra"] if choose(r) == "intra" else r["ms_inter"]
        rs.append(t / best - 1)
    return (float(max(rs)), float(np.mean(rs)), len(rs)) if rs else (0.0, 0.0, 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "selector_table.json"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    Ls = [15, 63, 127, 512] if not a.quick else [63]
    Ps = [100, 1000, 10_000, 100_000, 1_000_000] if not a.quick else [1000, 10_000]
    n_outs = [1, 6]
    Ds = [1 << k for k in range(5, 23)]
    fit = sweep(Ls, Ps, n_outs, Ds, dev, "fit")
    table = [{"L": r["L"], "P": r["P"], "n_out": r["n_out"], "D": r["D"],
              "strategy": "intra" if r["ms_intra"] < r["ms_inter"] else "inter"} for r in fit]
    val = sweep(Ls, Ps, n_outs, Ds, dev, "val")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rule = lambda r: nearest(table, r["L"], r["P"], r["D"], r["n_out"])["strategy"]  # noqa: E731
    paper = lambda r: "intra" if r["D"] >= sms * 128 else "inter"  # noqa: E731
    res = {"when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "device": torch.cuda.get_device_name(0),
           "sms": sms, "mix": "paper (n_out 1, sr_fitness) / full + Modi p 0.1 (n_out 6, eval)", "n_in": 8,
           "method": "median of 5 CUDA-event timings, forced inter vs forced intra; table fitted on one pass, "
                     "scored on a second",
           "table": table, "rows_fit": fit, "rows_validate": val}
    for name, ch in (("table", rule), ("paper_rule", paper)):
        for band, lo, hi in (("ge_0.5ms", 0.5, 1e30), ("lt_0.5ms", 0.0, 0.5), ("all", 0.0, 1e30)):
            mx, mean, n = regret(val, ch, lo, hi)
            res[f"{name}_regret_{band}"] = {"max": mx, "mean": mean, "cells": n}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    write_inc(res)
    print({k: v for k, v in res.items() if "regret" in k})


def write_inc(res):
    """Compiled-in table: {L, P, n_out, D, strategy (1 inter, 2 intra)} per measured cell."""
    lines = ["// generated by tools/calibrate_selector.py from selector_table.json — do not edit",
             f"// {res['device']} ({res['sms']} SMs), {res['when']}: faster kernel per measured cell",
             "static const SelectorEntry kSelectorTable[] = {"]
    for e in res["table"]:
        lines.append(f"    {{{e['L']}, {e['P']}, {e['n_out']}, {e['D']}, {2 if e['strategy'] == 'intra' else 1}}},")
    lines.append("};")
    with open(os.path.join(ROOT, "paper_2501_17168_b200", "csrc", "selector_table.inc"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
