#!/usr/bin/env python
"""Host-side cost of one API call at C1's shape (the launch-bound config):
wall time per call of sr_fitness through the binding, of the selector and
of the plan alone, with the GPU kept busy enough that launches queue.
    python tools/host_overhead.py"""
import time

import numpy as np
import torch

import paper_2501_17168_b200 as evogp
import synth

cfg = synth.CONFIGS["c1"]
pt = synth.trees(cfg.seed, 0, cfg.P, cfg.max_len, synth.MIXES["paper"], cfg.n_in)
t, v, s = (torch.from_numpy(a).cuda() for a in evogp.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in))
X, y = synth.config_data(cfg)
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
out = torch.empty(cfg.P, dtype=torch.float64, device="cuda")
ws = evogp.Workspace(cfg.P, cfg.D, cfg.max_len, cfg.n_in, 1, device="cuda:0")
for _ in range(50):
    evogp.sr_fitness(t, v, s, Xd, yd, out=out, workspace=ws)
torch.cuda.synchronize()


def per_call(fn, n=2000):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    return dt * 1e6


print("sr_fitness (binding, out + workspace given) us/call", per_call(lambda: evogp.sr_fitness(t, v, s, Xd, yd, out=out, workspace=ws)))
print("sr_fitness (binding, defaults) us/call", per_call(lambda: evogp.sr_fitness(t, v, s, Xd, yd)))
print("select_strategy us/call", per_call(lambda: evogp.select_strategy(cfg.P, cfg.D, cfg.max_len)))
print("workspace_size us/call", per_call(lambda: evogp.workspace_size(cfg.P, cfg.D, cfg.max_len, cfg.n_in, 1)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(1000):
    evogp.sr_fitness(t, v, s, Xd, yd, out=out, workspace=ws)
e1.record()
torch.cuda.synchronize()
print("device-timed us/call (1000 back to back)", e0.elapsed_time(e1))
