#!/usr/bin/env python
"""bench.py — GPops/s of the EvoGP hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--mix paper]
    python bench.py --impl reference ...        # the oracle on the host cores

A step is one pass of the whole hot path over one batch: dataset staging
(a2), strategy selection (a3), tree staging (a4), stack interpretation (a5),
the fused FP64 SSE/MSE (a7) — or the multi-output store (a6) for c5 — and,
for N > 1, the NCCL combine (a8). GPops/s = sum_p len_p * D / t (PAPER.md
P:600-605 with the factor D the tables need, reading R10). Tensorizing
(a1) is timed in the `e2e` leg only: the prefix lists are copied from pinned
host memory, tensorized on the device (evogp_tensorize_device), then the
hot path runs and its result is read back. `--config g1` times the whole
generational loop instead (NEXT-4).

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
launching stream; L2 is flushed (256 MiB write) before every timed step,
outside the events; the K-step region is bracketed by barrier + synchronize;
the reported time is the max over ranks. For N > 1 launch with torchrun.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded inputs; no method arithmetic)

METRIC = "GPops/s (nodes × datapoints / s) at 1/2/4/8 B200, % of FP32/SFU roofline"
UNIT = "GPops/s"
SFU_FUNCS = (3, 4, 5, 6, 9, 10, 11, 12, 15, 16)  # DIV SIN COS TAN POW LOG EXP TANH SQRT INV (R3)
FP32_LANES = 128  # per SM per clock
SFU_LANES = 16  # per SM per clock (measured 15.9, profiles/microbench_pipes_r01.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(synth.CONFIGS), default="c3")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="population axis: strong = one population of P trees sharded over the ranks "
                         "(SURVEY §8(e)); weak = P trees per rank")
    ap.add_argument("--mix", choices=sorted(synth.MIXES), default=None)
    ap.add_argument("--strategy", choices=["auto", "inter", "intra"], default="auto")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sustain-seconds", type=float, default=1.0)
    ap.add_argument("--tune", default="", help="evogp_set_tuning overrides, e.g. target_warps=48,no_reorder=1 "
                                                "(calibration sweeps; results never depend on them)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0}, "fallback"


def default_mix(cfg):
    return "full" if (cfg.n_out > 1 or cfg.eval_only) else "paper"


def workload_desc(cfg, mix):
    return (f"{cfg.name}: P={cfg.P} trees, max_len={cfg.max_len}, n_inputs={cfg.n_in}, n_outputs={cfg.n_out}, "
            f"D={cfg.D}, mix={mix}")


def tree_stats(pt):
    lens = np.diff(pt.offsets)
    kinds = pt.types & 7
    fn = kinds >= 2
    sfu = np.isin(pt.values[fn].astype(np.int64), SFU_FUNCS).sum()
    return int(lens.sum()), float(sfu) / max(1, len(pt.types))


def local_shards(cfg, rank, world, scaling="strong"):
    """c3: datapoint-sharded (strong scaling: fixed total D). Others:
    population-sharded; strong = one population of cfg.P trees, rank r owns
    rows shard_rows(P, world, r); weak = cfg.P trees per rank."""
    from paper_2501_17168_b200.dist import shard_rows

    if cfg.index == 3:
        d0, d1 = shard_rows(cfg.D, world, rank)
        return "data", (0, cfg.P), (d0, d1)
    if scaling == "weak":
        return "pop", (rank * cfg.P, (rank + 1) * cfg.P), (0, cfg.D)
    return "pop", shard_rows(cfg.P, world, rank), (0, cfg.D)


def relaunch_distributed(n):
    """`bench.py --gpus N` run as a plain command: re-exec under torchrun with
    N ranks (one per GPU, NCCL) and pass its exit status through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm = []
        reasons = set()
        smax = None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except ValueError:
                continue
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [x for x in sm if x > 600] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- oracle (cpu_baseline / reference arm)
def oracle_pass(pt, cfg, X, y, threads):
    import oracle

    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in, cfg.n_out)
    if cfg.paired:
        oracle.evaluate_paired(t, v, s, X.reshape(t.shape[0], cfg.D, cfg.n_in), n_out=cfg.n_out, mode=0)
        return
    out = oracle.evaluate(t, v, s, X, n_out=cfg.n_out, mode=0, threads=threads)
    if cfg.n_out == 1 and not cfg.eval_only:
        oracle.mse(out[:, :, 0], y)


def oracle_sample(cfg, mix, target_work=4e8):
    """A bounded sample of the workload: the first n trees (all trees if small)
    and at most 2^16 datapoints, about `target_work` node x datapoint steps."""
    D = min(cfg.D, 1 << 16)
    per_tree = 0.75 * cfg.max_len * D
    n = int(max(1, min(cfg.P, target_work // per_tree)))
    if cfg.paired:  # the oracle walks one individual at a time: a smaller sample
        n = min(n, 20_000)
    pt = synth.trees(cfg.seed, 0, n, cfg.max_len, synth.MIXES[mix], cfg.n_in, cfg.n_out, cfg.modi_prob)
    X, y = synth.config_data(cfg, 0, n * cfg.D if cfg.paired else D)
    nodes = int(np.diff(pt.offsets).sum())
    desc = f"first {n} of {cfg.P} trees x first {D} of {cfg.D} datapoints ({nodes * D:.3e} node*dp per pass)"
    if cfg.paired:
        desc = f"first {n} of {cfg.P} individuals, each on its own {cfg.D} observation(s) ({nodes * D:.3e} node*obs)"
    return pt, X, y, nodes * D, desc


def time_oracle(cfg, mix, seconds, threads):
    pt, X, y, work, desc = oracle_sample(cfg, mix)
    oracle_pass(pt, cfg, X, y, threads)  # warm (builds/loads the library)
    t0 = time.perf_counter()
    passes = 0
    while True:
        oracle_pass(pt, cfg, X, y, threads)
        passes += 1
        el = time.perf_counter() - t0
        if el >= seconds or passes >= 1000:
            break
    return work * passes / el, desc + f", {passes} passes in {el:.1f} s"


def run_reference(args, cfg, mix):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    pt, X, y, work, desc = oracle_sample(cfg, mix)
    for _ in range(args.warmup):
        oracle_pass(pt, cfg, X, y, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_pass(pt, cfg, X, y, threads)
    el = time.perf_counter() - t0
    value = work * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.scaling == "weak" and cfg.index != 3 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg, mix), "parallelism": "host threads (oracle)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": "each step: " + desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0



# ---------------------------------------------------------------- NEXT-4: the whole generational loop
def loop_gp_config(cfg):
    """tab:sr_params: max size 512, tournament 20, p_c 0.9, p_m 0.1,
    {+,-,x,/,sin,cos,tan}; subtree mutation (Algorithm 1's classic loop, R18)."""
    from paper_2501_17168_b200.gp import GPConfig

    return GPConfig(max_len=cfg.max_len, n_inputs=cfg.n_in, n_outputs=1, funcs=tuple(synth.M_PAPER),
                    tournament_size=20, p_crossover=0.9, p_mutation=0.1, depth_min=2, depth_max=6,
                    subtree_depth=4, mutation_weights=(1, 0, 0, 0, 0, 0, 0, 0))


def loop_oracle_sample(cfg, seconds, warm_gens=0):
    """The oracle's Algorithm 1 on a bounded sample: a 2,000-tree population of
    the same configuration, generations of (evaluate + MSE + reproduce) for
    about `seconds`. Returns (GPops/s, description)."""
    import oracle

    gp = loop_gp_config(cfg)
    d = {k: getattr(gp, k) for k in ("max_len", "n_inputs", "n_outputs", "const_lo", "const_hi", "p_const",
                                     "p_leaf", "p_modi", "depth_min", "depth_max", "tournament_size",
                                     "p_crossover", "p_mutation", "crossover_kind", "leaf_bias", "point_rate",
                                     "const_sigma", "subtree_depth")}
    d["funcs"] = list(gp.funcs)
    d["mutation_weights"] = list(gp.mutation_weights)
    n = 2000
    X, y = synth.config_data(cfg)
    t, v, s = oracle.generate(n, d, cfg.seed)
    threads = os.cpu_count() or 1
    work, gens = 0.0, 0
    t0 = time.perf_counter()
    while True:
        work += float(s[:, 0].astype(np.int64).sum()) * cfg.D
        fit = oracle.mse(oracle.evaluate(t, v, s, X, mode=0, threads=threads)[:, :, 0], y)
        t, v, s, _, _ = oracle.reproduce(t, v, s, fit, n, d, cfg.seed + 1 + gens)
        gens += 1
        el = time.perf_counter() - t0
        if el >= seconds or gens >= 100:
            break
    desc = (f"Algorithm 1 on a {n}-tree population of {cfg.name} (D={cfg.D}), {gens} generations from the "
            f"initial population in {el:.1f} s")
    return work / el, desc, threads


def run_loop(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2501_17168_b200 as evogp

    rank, world, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        value, desc, threads = loop_oracle_sample(cfg, args.cpu_seconds)
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{cfg.name}: Algorithm 1, P={cfg.P}, max_len={cfg.max_len}, "
                                       f"n_inputs={cfg.n_in}, D={cfg.D}", "parallelism": "host threads (oracle)"},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    if args.tune:
        evogp.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tune.split(","))})
    gp = loop_gp_config(cfg)
    X, y = synth.config_data(cfg)
    Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
    P = cfg.P
    # island model across ranks: rank r evolves its own P trees
    seed = cfg.seed + 1_000_003 * rank
    ws = evogp.Workspace(P, cfg.D, cfg.max_len, cfg.n_in, 1, device=dev)
    # selector (c) keyed on the population's own tree lengths (gp.selector_strategy)
    strategy = evogp.Evolution(P, gp, Xd, yd, seed=seed).strategy

    launches = [0]

    def make_run():
        ev = evogp.Evolution(P, gp, Xd, yd, seed=seed, strategy=strategy)
        ev.ws = ws
        return ev

    def gen_step(ev, kev=None, rev=None):
        """One generation of Algorithm 1: fused SR fitness, then reproduction."""
        t, v, s = ev.population
        if kev is not None:
            evogp.set_kernel_timing(*kev)
        evogp.sr_fitness(t, v, s, Xd, yd, strategy=strategy, out=ev.fitness, workspace=ws)
        launches[0] += evogp.last_launch_count() + 1  # + the reproduce kernel
        if kev is not None:
            evogp.set_kernel_timing(None, None)
        if rev is not None:
            rev[0].record()
        nxt = 1 - ev.cur
        evogp.reproduce(ev.population, ev.fitness, P, gp, ev.seed + 1 + ev.generation, out=ev.bufs[nxt],
                        record=False)
        if rev is not None:
            rev[1].record()
        ev.cur = nxt
        ev.generation += 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local])
                           if "CUDA_VISIBLE_DEVICES" in os.environ else local)
    sampler.start()
    # sustain the load for the clock sampler (untimed, a throwaway run)
    warm = make_run()
    t_end = time.perf_counter() + args.sustain_seconds
    while True:
        gen_step(warm)
        torch.cuda.synchronize()
        if time.perf_counter() >= t_end:
            break
    del warm
    run = make_run()
    for _ in range(args.warmup):
        gen_step(run)
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    rev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in kev:
        a.record()
        b.record()
    lens = torch.zeros(K, dtype=torch.int64, device=dev)
    barrier()
    launches[0] = 0
    for i in range(K):
        ev[i][0].record()
        gen_step(run, kev[i], rev[i])
        ev[i][1].record()
        # bookkeeping outside the events: nodes of the population just evaluated
        t_prev, v_prev, s_prev = run.bufs[1 - run.cur]
        lens[i] = s_prev[:, 0].to(torch.int64).sum()
    barrier()
    timed_launches = launches[0]
    clocks = sampler.stop()
    step_ms = sum(a.elapsed_time(b) for a, b in ev)
    kern_ms = sum(a.elapsed_time(b) for a, b in kev)
    rep_ms = sum(a.elapsed_time(b) for a, b in rev)
    nodes_per_gen = lens.to(torch.float64)
    work_local = float(nodes_per_gen.sum().item()) * cfg.D
    tt = torch.tensor([step_ms, kern_ms, rep_ms], dtype=torch.float64, device=dev)
    work = torch.tensor([work_local], dtype=torch.float64, device=dev)
    best = torch.nan_to_num(run.evaluate(), nan=float("inf")).min().reshape(1)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(work, op=dist.ReduceOp.SUM)
        dist.all_reduce(best, op=dist.ReduceOp.MIN)
    step_ms, kern_ms, rep_ms = tt.tolist()
    value = work.item() / (step_ms * 1e-3)
    mean_len = float(nodes_per_gen.mean().item()) / P

    # ---- e2e: Algorithm 1 through the public API from host data: X, y copied
    # from pinned host memory, the population generated on the device, and the
    # best fitness read back every generation (Algorithm 1's target check)
    e2e = None
    if not args.no_e2e:
        h_X, h_y = torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()
        h_best = torch.empty(1, dtype=torch.float64).pin_memory()
        barrier()
        t0 = time.perf_counter()
        Xd.copy_(h_X, non_blocking=True)
        yd.copy_(h_y, non_blocking=True)
        r2 = make_run()
        for _ in range(args.warmup + K):
            gen_step(r2)
            h_best.copy_(torch.nan_to_num(r2.fitness, nan=float("inf")).min().reshape(1), non_blocking=True)
            torch.cuda.current_stream().synchronize()
        barrier()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        # same seeds -> the same populations as the timed run: its node counts apply
        # (warm-up generations counted at the first timed generation's size, a lower bound)
        e2e_nodes = float(nodes_per_gen.sum().item()) + args.warmup * float(nodes_per_gen[0].item())
        e2e = {"value": e2e_nodes * cfg.D * world / el.item(), "unit": UNIT,
               "h2d_bytes_per_step": int((X.nbytes + y.nbytes) / (args.warmup + K)),
               "d2h_bytes_per_step": 8,
               "includes": "H2D of X, y + on-device generation + (fitness + reproduce + best-fitness D2H) "
                           f"x {args.warmup + K} generations, wall clock"}

    if rank == 0:
        peaks, peak_src = measured_peaks()
        f = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        # SFU-node fraction (/, sin, cos, tan of the paper set), measured on the
        # last population evaluated
        t, v, s = run.bufs[1 - run.cur]
        tl = t.to(torch.int32) & 7
        fn = tl >= 2
        vals = v[fn].to(torch.int64)
        n_sfu = torch.isin(vals, torch.tensor(SFU_FUNCS, device=dev)).sum().item()
        n_nodes = (s[:, 0].to(torch.int64)).sum().item()
        sfu_frac = n_sfu / max(1, n_nodes)
        SMS = torch.cuda.get_device_properties(dev).multi_processor_count
        roof = 1.0 / max(1.0 / (SMS * FP32_LANES * f), sfu_frac / (SMS * SFU_LANES * f))
        achieved = work_local / (kern_ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": step_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: Algorithm 1 (fitness + tournament + crossover + mutation per "
                                   f"generation), P={P} per rank, max_len={cfg.max_len}, n_inputs={cfg.n_in}, "
                                   f"D={cfg.D}, mix=paper, tab:sr_params",
                       "P_per_rank": P, "D": cfg.D, "max_len": cfg.max_len, "mean_len": mean_len,
                       "generations_timed": K, "generation_of_first_timed": args.warmup,
                       "strategy": strategy, "parallelism": f"islands x{world}",
                       "best_mse_final": float(best.item()),
                       "l2": "inputs larger than L2 (population rows 2 x P x max_len x 8 B)",
                       "step": "one generation: evogp_sr_fitness + evogp_reproduce",
                       "paper_context": "1.00e11 GPops/s, RTX 4090, P=1e5, D=392, S=482 (P:592)"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": roof, "unit": UNIT, "frac": achieved / roof,
                         "traffic": None, "kernel": f"k_{strategy} (fitness)",
                         "peak_basis": f"{SMS} SMs x min({FP32_LANES} FP32, {SFU_LANES}/s MUFU) lanes/clk at "
                                       f"sm_max_mhz={f / 1e6:.0f} ({peak_src}), s={sfu_frac:.3f}",
                         "step_share": {"fitness": kern_ms / step_ms, "reproduce": rep_ms / step_ms}},
            "gpu_launches": timed_launches,
            "clocks": clocks,
            "e2e": e2e,
        }
        if world == 1 and not args.no_cpu_baseline:
            cv, desc, threads = loop_oracle_sample(cfg, args.cpu_seconds)
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)
    cfg = synth.CONFIGS[args.config]
    mix = args.mix or default_mix(cfg)
    if cfg.loop:
        return run_loop(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg, mix)

    import torch
    import torch.distributed as dist

    import paper_2501_17168_b200 as evogp
    from paper_2501_17168_b200 import dist as edist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (even one rank) the sharded path + NCCL combine runs
    use_dist = world > 1 or "WORLD_SIZE" in os.environ
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    tune = {k: int(v) for k, v in (kv.split("=") for kv in args.tune.split(","))} if args.tune else {}
    if mix != "paper" and cfg.n_out == 1 and not cfg.paired:
        # full-set single-output population: the full-set kernel variants
        # (evogp_tuning.full_set, include/evogp.h), unless --tune says otherwise
        tune.setdefault("full_set", 1)
    if tune:
        evogp.set_tuning(**tune)
    axis, (p0, p1), (d0, d1) = local_shards(cfg, rank, world, args.scaling)
    pt = synth.trees(cfg.seed, p0, p1 - p0, cfg.max_len, synth.MIXES[mix], cfg.n_in, cfg.n_out, cfg.modi_prob)
    if cfg.paired:  # NEXT-2: every individual's own B observations, rows p0*B ...
        X, y = synth.config_data(cfg, p0 * cfg.D, (p1 - p0) * cfg.D)
        X = X.reshape(p1 - p0, cfg.D, cfg.n_in) if cfg.D > 1 else X
    else:
        X, y = synth.config_data(cfg, d0, d1 - d0)
    nodes, sfu_frac = tree_stats(pt)
    t, v, s = evogp.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in, cfg.n_out)
    td, vd, sd = (torch.from_numpy(a).to(dev) for a in (t, v, s))
    Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
    P_local, D_local = p1 - p0, d1 - d0
    strategy = args.strategy
    if cfg.paired:
        chosen = "paired"
    else:
        chosen = (evogp.select_strategy(P_local, D_local, cfg.max_len, cfg.n_out, local) if strategy == "auto"
                  else strategy)
    ws = evogp.Workspace(P_local, D_local, cfg.max_len, cfg.n_in, cfg.n_out, device=dev)
    evalcfg = cfg.n_out > 1 or cfg.eval_only  # outputs only (evogp_eval), no fitness
    out_eval = torch.empty((P_local, D_local, cfg.n_out), dtype=torch.float32, device=dev) if evalcfg else None
    if cfg.paired:
        out_eval = torch.empty(((P_local, cfg.n_out) if cfg.D == 1 else (P_local, cfg.D, cfg.n_out)),
                               dtype=torch.float32, device=dev)
    P_total = cfg.P * world if (axis == "pop" and args.scaling == "weak") else cfg.P
    # population axis: the rank's MSEs go into its equal-size all-gather slot
    slot = edist.padded_shard(P_total, world) if (axis == "pop" and use_dist) else P_local
    mse_slot = torch.full((slot,), float("nan"), dtype=torch.float64, device=dev)
    mse_local = mse_slot[:P_local]

    def step():
        if cfg.paired:
            evogp.eval_paired(td, vd, sd, Xd, n_outputs=cfg.n_out, out=out_eval, workspace=ws)
            return out_eval
        if evalcfg:
            evogp.eval(td, vd, sd, Xd, n_outputs=cfg.n_out, strategy=strategy, out=out_eval, workspace=ws)
            return out_eval
        if axis == "data":
            if not use_dist:
                return evogp.sr_fitness(td, vd, sd, Xd, yd, strategy=strategy, out=mse_local, workspace=ws)
            return edist.sr_fitness_data_sharded(
                td, vd, sd, Xd, yd, cfg.D, out=mse_local,
                sse_fn=lambda a, b, c, x, yy, o: evogp.sr_sse(a, b, c, x, yy, strategy=strategy, out=o, workspace=ws))
        if not use_dist:
            return evogp.sr_fitness(td, vd, sd, Xd, yd, strategy=strategy, out=mse_local, workspace=ws)
        return edist.sr_fitness_population_sharded(
            td, vd, sd, Xd, yd, P_total, local_out=mse_slot,
            fitness_fn=lambda a, b, c, x, yy, o: evogp.sr_fitness(a, b, c, x, yy, strategy=strategy, out=o,
                                                                  workspace=ws))

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local])
                           if "CUDA_VISIBLE_DEVICES" in os.environ else local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    barrier()
    # sustain the load for the clock sampler (untimed)
    t_end = time.perf_counter() + args.sustain_seconds
    while time.perf_counter() < t_end:
        for _ in range(20):
            step()
        torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:  # materialise the CUDA events before handing them to the library
        a.record()
        b.record()
    launches = 0
    barrier()
    for i in range(args.steps):
        flush.zero_()
        evogp.set_kernel_timing(*kev[i])
        ev[i][0].record()
        step()
        ev[i][1].record()
        evogp.set_kernel_timing(None, None)
        launches += evogp.last_launch_count()
    barrier()
    clocks = sampler.stop()
    step_ms = sum(a.elapsed_time(b) for a, b in ev)
    kern_ms = sum(a.elapsed_time(b) for a, b in kev)
    # diagnostic: chunks of the last step that were re-run on the cold interpreter copy
    off = ws.ptr - ws.buf.data_ptr()
    cold_chunks = int(ws.buf[off + 4: off + 8].view(torch.int32).item())
    tt = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dev)
    work = torch.tensor([float(nodes) * D_local], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(work, op=dist.ReduceOp.SUM)
    step_ms, kern_ms = tt.tolist()
    total_work = work.item()  # node x datapoint evaluations per step, all ranks
    # config 5: the fraction of (tree, output slot) pairs some
    # Modi node wrote (slots no Modi node targets stay 0, reading R4)
    modi_nonzero = None
    if cfg.n_out > 1 and out_eval is not None:
        modi_nonzero = float((out_eval != 0).flatten(0, -3).any(dim=-2).float().mean().item()) if out_eval.dim() == 3 else None
    value = total_work * args.steps / (step_ms * 1e-3)

    # ---- e2e: host prefix lists -> tensorize -> H2D -> device call -> D2H
    e2e = None
    if not args.no_e2e:
        # the caller's prefix lists (CSR) in pinned memory -> H2D -> tensorized
        # on the device (evogp_tensorize_device, row a1) -> hot path -> D2H
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        h_off, h_ty, h_va = pin(pt.offsets.astype(np.int64)), pin(pt.types), pin(pt.values)
        d_off, d_ty, d_va = (torch.empty_like(x, device=dev) for x in (h_off, h_ty, h_va))
        h_X, h_y = pin(X), pin(y)
        res_len = P_total if not evalcfg else P_local * D_local * cfg.n_out
        h_res = torch.empty(res_len, dtype=torch.float32 if evalcfg else torch.float64).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in (h_off, h_ty, h_va, h_X, h_y))
        d2h = h_res.numel() * h_res.element_size()

        def e2e_step():
            for dst, src in ((d_off, h_off), (d_ty, h_ty), (d_va, h_va), (Xd, h_X), (yd, h_y)):
                dst.copy_(src, non_blocking=True)
            evogp.tensorize_device(d_off, d_ty, d_va, cfg.max_len, cfg.n_in, cfg.n_out, out=(td, vd, sd),
                                   status=False)
            r = step()
            h_res.copy_(r.reshape(-1), non_blocking=True)
            torch.cuda.current_stream().synchronize()

        e2e_mode = "one pass"
        n_chunks = int(os.environ.get("EVOGP_E2E_CHUNKS", "1"))  # with 2 steps in flight, chunking measured no gain (c4) or a loss (c2)
        depth = min(2, int(os.environ.get("EVOGP_E2E_DEPTH", "2")))  # two host result buffers
        if not evalcfg and not use_dist and not cfg.paired and (n_chunks > 1 or depth > 1):
            # single-output populations: the streaming public path. Copies of
            # chunk c+1 overlap the device work of chunk c; with depth 2 the
            # next step's copies (its trees AND its dataset) also overlap this
            # step's device work, and the host waits for step i-1's MSEs after
            # enqueuing step i.
            from paper_2501_17168_b200.stream import HostSRFitness

            pipe = HostSRFitness(P_local, int(h_ty.numel()), cfg.max_len, cfg.n_in, Xd, yd, chunks=n_chunks,
                                 strategy=strategy)
            h_res2 = [h_res, torch.empty_like(h_res).pin_memory()]
            pending, n_sub = [], [0]
            e2e_mode = (f"HostSRFitness, {n_chunks} chunk(s) on 2 streams, {depth} step(s) in flight "
                        "(X and y copied every step)")

            def e2e_step():  # noqa: F811
                pending.append(pipe.submit(h_off, h_ty, h_va, h_res2[n_sub[0] & 1], X=h_X, y=h_y))
                n_sub[0] += 1
                while len(pending) >= max(1, depth):
                    pending.pop(0).synchronize()  # the oldest step's MSEs are on the host

        # a wall-clock region of a few milliseconds (K short steps) is at the
        # mercy of host jitter: the e2e leg runs at least ~0.3 s of steps
        e2e_steps = max(args.steps, min(2000, int(300.0 / max(step_ms / args.steps, 0.01))))
        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        barrier()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if use_dist:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e = {"value": total_work * e2e_steps / el.item(), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "includes": "H2D of the prefix lists (CSR) + X + y from pinned memory, device tensorize (a1), "
                           "hot path, D2H of the result", "path": e2e_mode}

    # ---- launch-bound configs (c1; c2's 0.1 ms step): the same step replayed
    # (after the e2e leg: a captured graph left alive slowed the host-bound
    # e2e pipeline that followed it, c2 2.0 -> 1.6e12)
    # from a CUDA graph: G steps captured once, the
    # graph replayed K times; value = G * K * work / device time of the replays
    graph = None
    if cfg.index in (1, 2) and world == 1 and not cfg.paired and not evalcfg:
        G = 100 if cfg.index == 1 else 20
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(gs):
            for _ in range(3):
                step()  # plan caches, occupancy queries, function attributes
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(G):
                step()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        gms = a.elapsed_time(b)
        graph = {"value": total_work * G * args.steps / (gms * 1e-3), "unit": UNIT, "steps_per_graph": G,
                 "replays": args.steps, "us_per_step": gms * 1e3 / (G * args.steps),
                 "note": "CUDA-graph-batched replay of the same step (launch-bound config); the graph's kernels "
                         "are the same launches per step, no L2 flush between graph steps"}

    if rank == 0:
        peaks, peak_src = measured_peaks()
        f = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        SMS = torch.cuda.get_device_properties(dev).multi_processor_count
        r_fp32 = SMS * FP32_LANES * f
        r_sfu = SMS * SFU_LANES * f
        roof = 1.0 / max(1.0 / r_fp32, sfu_frac / r_sfu)  # per GPU
        per_launch_work = float(nodes) * D_local  # rank 0's units per launch
        achieved = per_launch_work * args.steps / (kern_ms * 1e-3)
        if cfg.paired:
            # NEXT-2 is a single streaming pass: bound by HBM. Algorithmic bytes
            # per launch: type+value of every node (6 B), size[0] per row, the
            # observations and the outputs
            alg_bytes = 6.0 * nodes + 2.0 * P_local + 4.0 * P_local * cfg.D * (cfg.n_in + cfg.n_out)
            hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
            gbs = alg_bytes * args.steps / (kern_ms * 1e-3) / 1e9
        # DRAM traffic of the dominant kernel from the committed `ncu --set
        # full` capture of this config (a profiler number: never taken here)
        traffic, traffic_src = None, None
        prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}_{chosen}_summary.json")
        if os.path.exists(prof):
            with open(prof) as fh:
                pj = json.load(fh)
            traffic, traffic_src = pj.get("dram_bytes_per_launch"), f"profiles/{os.path.basename(prof)} ({pj.get('note', '')})"
        hbm_view = None
        if evalcfg and not cfg.paired:
            # multi-output eval: the P x D x n_out FP32 output store is the one
            # HBM-relevant stream: report it against HBM
            out_bytes = 4.0 * P_local * D_local * cfg.n_out
            alg_bytes_n = out_bytes + 8.0 * nodes + 4.0 * D_local * cfg.n_in
            hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
            gbs_n = alg_bytes_n * args.steps / (kern_ms * 1e-3) / 1e9
            hbm_view = {"achieved": gbs_n, "peak": hbm_peak, "unit": "GB/s", "frac": gbs_n / hbm_peak,
                        "algorithmic_bytes_per_launch": alg_bytes_n, "output_bytes_per_launch": out_bytes,
                        "peak_basis": f"hbm_gbs ({peak_src})"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (axis == "data" or args.scaling == "strong") else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": workload_desc(cfg, mix), "P_total": P_total, "P_per_rank": P_local,
                       "D_per_rank": D_local,
                       "max_len": cfg.max_len, "n_inputs": cfg.n_in, "n_outputs": cfg.n_out,
                       "mean_len": nodes / max(1, P_local), "sfu_node_fraction": sfu_frac,
                       "strategy": chosen, **({"tuning": tune} if tune else {}),
                       "parallelism": f"{axis}-shard x{world}" + (" (NCCL)" if use_dist else " (no collective)"),
                       "cold_rerun_chunks_last_step": cold_chunks,
                       **({"modi_nonzero_slot_fraction": modi_nonzero} if modi_nonzero is not None else {}),
                       "l2": "flushed (256 MiB write) before every timed step",
                       "step": ("evogp_eval_paired" if cfg.paired else
                                "evogp_eval" if evalcfg else "evogp_sr_fitness") +
                               (" + NCCL combine" if use_dist and not evalcfg and not cfg.paired else "")},
            "roofline": ({"bound": "alu", "achieved": achieved, "peak": roof, "unit": UNIT, "frac": achieved / roof,
                          "traffic": traffic, "traffic_source": traffic_src, "kernel": f"k_{chosen}",
                          "peak_basis": f"{SMS} SMs x min({FP32_LANES} FP32, {SFU_LANES}/s MUFU) lanes/clk at "
                                        f"sm_max_mhz={f / 1e6:.0f} ({peak_src}), s={sfu_frac:.3f}",
                          **({"hbm_view": hbm_view} if hbm_view else {})}
                         if not cfg.paired else
                         {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                          "traffic": traffic, "traffic_source": traffic_src, "kernel": "k_paired",
                          "algorithmic_bytes_per_launch": alg_bytes,
                          "alu_view": {"achieved": achieved, "unit": UNIT, "fp32_sfu_roof": roof,
                                       "frac": achieved / roof},
                          "peak_basis": f"hbm_gbs ({peak_src})"}),
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
        }
        if graph is not None:
            line["graph_replay"] = graph
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            cv, desc = time_oracle(cfg, mix, args.cpu_seconds, threads)
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc}
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
