#!/usr/bin/env python
"""Row-length distribution of the g1 population over generations (sizes the
compile pass's per-warp scratch).   python tools/g1_lengths.py [generations]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_17168_b200 as evogp  # noqa: E402
import synth  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = synth.CONFIGS["g1"]
X, y = synth.config_data(cfg)
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
gp = bench.loop_gp_config(cfg)
ev = evogp.Evolution(cfg.P, gp, Xd, yd, seed=cfg.seed)
for g in range(gens + 1):
    if g % 5 == 0:
        s = ev.population[2][:, 0].cpu().numpy().astype(np.int64)
        q = np.percentile(s, [50, 90, 99, 99.9])
        print(g, "mean %.1f" % s.mean(), "p50/90/99/99.9", q, "max", s.max(), ">128: %.4f" % (s > 128).mean(),
              ">192: %.4f" % (s > 192).mean(), ">256: %.4f" % (s > 256).mean(), flush=True)
    ev.step()
