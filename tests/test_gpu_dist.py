"""Multi-GPU combine with the CUDA evaluator on the
B200: the sharded drivers of paper_2501_17168_b200.dist run through a real
process group whose per-shard evaluator is the C-ABI (evogp_sr_fitness /
evogp_sr_sse).

* world_size 1 over NCCL in this process: all_gather_into_tensor of the FP64
  MSEs (population axis) and the FP64 all-reduce with PREMUL_SUM(1/D)
  (datapoint axis) — the exact NCCL calls the N-GPU bench makes;
* world_size 2 over gloo, both ranks on cuda:0 (NCCL refuses two ranks on one
  GPU): the padded all-gather of uneven population shards and the 2-way SSE
  all-reduce, each rank evaluating its shard with the CUDA kernels;
* bench.py under torchrun with one rank: the NCCL-combined step end to end.

Reference values: the oracle's FP32-faithful outputs (IEEE-exact mix, where
the GPU outputs are bit-identical, DESIGN.md §3 Tier A) reduced to the MSE by
the oracle. Population sharding only moves whole per-tree results, so
it must equal the single-call GPU fitness bit for bit; datapoint sharding
re-associates the FP64 sum, so it agrees to 1e-12 relative.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
dist = torch.distributed

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(seed, P=2000, L=63, n_in=4, D=3001):
    pt = synth.trees(seed, 0, P, L, synth.M_IEEE, n_in, 1, 0.0)
    X = synth.dataset_X(seed, 0, D, n_in, "uniform", -2.0, 2.0)
    y = synth.pagie_y(X)
    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in, 1)
    r32 = oracle.evaluate(t, v, s, X, mode=1)[:, :, 0]
    return (t, v, s), X, y, oracle.mse(r32, y)


def _rel(a, b):
    fin = np.isfinite(b)
    assert (np.isfinite(a) == fin).all() and (np.isnan(a) == np.isnan(b)).all()
    return np.abs(a[fin] - b[fin]) / np.maximum(np.abs(b[fin]), 1e-300)


def test_nccl_world1_population_and_data_sharded():
    import paper_2501_17168_b200 as evogp
    from paper_2501_17168_b200 import dist as edist

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    (t, v, s), X, y, m_ref = _case(31)
    P, D = t.shape[0], X.shape[0]
    td, vd, sd = (torch.from_numpy(a).to(dev) for a in (t, v, s))
    Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    try:
        assert dist.get_backend() == "nccl"
        single = evogp.sr_fitness(td, vd, sd, Xd, yd).cpu().numpy()
        # population axis: every rank's rows, all-gathered (NCCL all_gather_into_tensor)
        pop = edist.sr_fitness_population_sharded(td, vd, sd, Xd, yd, P).cpu().numpy()
        assert pop.view(np.uint64).tolist() == single.view(np.uint64).tolist()
        assert _rel(pop, m_ref).max() <= 1e-12
        # datapoint axis: sse of the rank's rows, NCCL all-reduce with PREMUL_SUM(1/D)
        ds = edist.sr_fitness_data_sharded(td, vd, sd, Xd, yd, D).cpu().numpy()
        assert _rel(ds, m_ref).max() <= 1e-12
        assert _rel(ds, single).max() <= 1e-14
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def _gloo_worker(rank, world, port, case, q):
    import paper_2501_17168_b200 as evogp
    from paper_2501_17168_b200 import dist as edist

    try:
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        (t, v, s), X, y = case
        P, D = t.shape[0], X.shape[0]
        # population axis: this rank's rows only (uneven shards -> padded gather)
        p0, p1 = edist.shard_rows(P, world, rank)
        rows = [torch.from_numpy(np.ascontiguousarray(a[p0:p1])).to(dev) for a in (t, v, s)]
        Xd, yd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
        pop = edist.sr_fitness_population_sharded(*rows, Xd, yd, P).cpu().numpy()
        # datapoint axis: all trees, this rank's rows of X / y
        d0, d1 = edist.shard_rows(D, world, rank)
        full = [torch.from_numpy(a).to(dev) for a in (t, v, s)]
        ds = edist.sr_fitness_data_sharded(*full, Xd[d0:d1].contiguous(), yd[d0:d1].contiguous(), D).cpu().numpy()
        single = evogp.sr_fitness(*full, Xd, yd).cpu().numpy()
        q.put((rank, pop, ds, single, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, None, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_gloo_world2_cuda_evaluator():
    import torch.multiprocessing as mp

    (t, v, s), X, y, m_ref = _case(32, P=1001, D=2049)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, ((t, v, s), X, y), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, pop, ds, single, err in res:
        assert err is None, err
        # the gathered population equals one GPU's fitness bit for bit, on every rank
        assert pop.view(np.uint64).tolist() == single.view(np.uint64).tolist()
        assert _rel(pop, m_ref).max() <= 1e-12
        assert _rel(ds, m_ref).max() <= 1e-12


def test_bench_one_rank_torchrun_nccl():
    """bench.py under torchrun (one rank): the step is the NCCL-combined,
    population-sharded fitness (strong scaling of one population)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
           "--sustain-seconds", "0.2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["config"]["parallelism"] == "pop-shard x1 (NCCL)"
    assert line["scaling"] == "strong" and line["n_gpus"] == 1
    assert line["config"]["step"] == "evogp_sr_fitness + NCCL combine"
    assert line["value"] > 0
