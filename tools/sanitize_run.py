#!/usr/bin/env python
"""Small calls of every kernel of libevogp.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; tools/sanitize.sh):

  k_prepare + k_inter      (C1-shaped SR fitness and eval, paper mix -> the
                            inline-PTX hot loop; full mix -> the packed C++ copy)
  k_prepare + k_intra      (TMA bulk-copy staging of program rows, mbarrier)
  k_combine                (trees split over several units)
  deep-stack paths         (left combs with reordering off: multi-pass split,
                            per-warp global stacks, locked pool)
  Modi / classification   (multi-output store, argmax epilogue)
  k_paired, tensorize_device, generate / reproduce / exchange / tournament
  full-set kernel variants  (tuning full_set: the packed multi loop on
                            single-output rows, exp / tanh / pow in the loop)
  fused compile             (tuning fused_compile: kernel (a) compiling its
                            own rows into shared memory)
  two-tier compile          (max_len 512: k_prepare_long)

Sizes are tiny (sanitizers replay every access); the values are checked
loosely against the oracle so a sanitizer-induced misbehaviour shows too.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2501_17168_b200 as evogp  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def dev_trees(pt, L, n_in, n_out=1):
    t, v, s = evogp.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
    return [torch.from_numpy(a).to(dev) for a in (t, v, s)], (t, v, s)


def check_close(g, r, what):
    g = np.asarray(g, np.float64)
    ok = oracle.within_tol(g, r)
    assert ok.mean() > 0.8, (what, ok.mean())


def main():
    # single-output SR: both kernels, paper mix (PTX loop) and full mix (C++ packed copy)
    for mix in ("paper", "full"):
        P, L, n_in, D = 64, 15, 2, 300
        pt = synth.trees(11, 0, P, L, synth.MIXES[mix], n_in)
        X = synth.dataset_X(11, 0, D, n_in, "uniform", -5.0, 5.0)
        y = synth.pagie_y(X)
        (t, v, s), host = dev_trees(pt, L, n_in)
        Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
        r64 = oracle.evaluate(*host, X, mode=0)[:, :, 0]
        for strat in ("inter", "intra"):
            g = evogp.eval(t, v, s, Xd, strategy=strat)[:, :, 0].cpu().numpy()
            check_close(g, r64, (mix, strat))
            m = evogp.sr_fitness(t, v, s, Xd, yd, strategy=strat).cpu().numpy()
            assert np.isfinite(m).mean() > 0.5
    # full-set kernel variants and the fused compile, single output (K = 8 / 4)
    P, L, n_in, D = 64, 63, 3, 600
    pt = synth.trees(21, 0, P, L, synth.M_FULL, n_in)
    X = synth.dataset_X(21, 0, D, n_in, "normal")
    y = synth.pagie_y(X)
    (t, v, s), host = dev_trees(pt, L, n_in)
    Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
    base = evogp.eval(t, v, s, Xd, strategy="intra").cpu().numpy()
    for kw in (dict(full_set=True), dict(full_set=True, K=4), dict(fused_compile=True)):
        evogp.set_tuning(**kw)
        Dk = 256 if "fused_compile" in kw else D  # one work unit per tree
        for strat in ("inter", "intra"):
            g = evogp.eval(t, v, s, Xd[:Dk].contiguous(), strategy=strat).cpu().numpy()
            assert np.array_equal(g.view(np.uint32), base[:, :Dk].view(np.uint32)), (kw, strat)
            evogp.sr_fitness(t, v, s, Xd[:Dk].contiguous(), yd[:Dk].contiguous(), strategy=strat)
    evogp.set_tuning()
    # two-tier compile: max_len 512 with rows beyond the first tier's 192 nodes
    gc = evogp.GPConfig(max_len=512, n_inputs=3, n_outputs=1, funcs=tuple(synth.M_PAPER), depth_min=6,
                        depth_max=9)
    pop = evogp.generate(48, gc, 5, device=dev)
    Xd = torch.from_numpy(synth.dataset_X(22, 0, 300, 3)).to(dev)
    for strat in ("inter", "intra"):
        evogp.sr_fitness(*pop, Xd, Xd[:, 0].contiguous(), strategy=strat)
    # deep rows (left combs), reordering off: multi-pass / per-warp global / locked pool
    L, n_in, P, D = 127, 2, 12, 700
    offs, tys, vas = [0], [], []
    for _ in range(P):
        tys += [3] * 63 + [1] * 64
        vas += [0.0] * 63 + [float(i % 2) for i in range(64)]
        offs.append(len(tys))
    pt = synth.PrefixTrees(np.array(offs, np.int64), np.array(tys, np.int16), np.array(vas, np.float32))
    X = synth.dataset_X(12, 0, D, n_in, lo=0.5, hi=1.5)
    (t, v, s), host = dev_trees(pt, L, n_in)
    r32 = oracle.evaluate(*host, X, mode=1)[:, :, 0]
    for tw in (0, 64):
        evogp.set_tuning(target_warps=tw, no_reorder=True)
        for strat in ("inter", "intra"):
            g = evogp.eval(t, v, s, torch.from_numpy(X).to(dev), strategy=strat)[:, :, 0].cpu().numpy()
            assert np.array_equal(g, r32.astype(np.float32)), strat
    evogp.set_tuning()
    # multi-output Modi + classification (K = 4 kernels, store_outn, lane_correct)
    P, L, n_in, n_out, D = 40, 31, 5, 3, 260
    pt = synth.trees(13, 0, P, L, synth.M_FULL, n_in, n_out, 0.2)
    X = synth.dataset_X(13, 0, D, n_in, "normal")
    (t, v, s), host = dev_trees(pt, L, n_in, n_out)
    Xd = torch.from_numpy(X).to(dev)
    lab = torch.from_numpy((np.arange(D) % n_out).astype(np.int32)).to(dev)
    for strat in ("inter", "intra"):
        evogp.eval(t, v, s, Xd, n_outputs=n_out, strategy=strat)
        evogp.classification_accuracy(t, v, s, Xd, lab, n_out, strategy=strat)
    # paired inference
    obs = torch.from_numpy(synth.dataset_X(14, 0, P * 2, n_in, "normal").reshape(P, 2, n_in)).to(dev)
    evogp.eval_paired(t, v, s, obs, n_outputs=n_out)
    # device tensorize
    pt = synth.trees(15, 0, 50, 31, synth.M_PAPER, 3)
    d = [torch.from_numpy(a).to(dev) for a in (pt.offsets, pt.types, pt.values)]
    evogp.tensorize_device(*d, 31, 3)
    # genetic operators
    gc = evogp.GPConfig(max_len=63, n_inputs=3, n_outputs=1, funcs=tuple(synth.M_PAPER), tournament_size=5,
                        p_crossover=0.9, p_mutation=0.5, depth_min=2, depth_max=5,
                        mutation_weights=(1, 1, 1, 1, 1, 1, 1, 1))
    pop = evogp.generate(64, gc, 3, device=dev)
    fit = torch.rand(64, dtype=torch.float64, device=dev)
    evogp.reproduce(pop, fit, 64, gc, 4)
    evogp.tournament(fit, 5, 64, 7)
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
