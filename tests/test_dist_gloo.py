"""Multi-process host logic of the sharded path,
world_size 2 over gloo on CPU. The per-shard evaluator is the oracle here
(test infrastructure); on GPUs it is the CUDA C-ABI with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2501_17168_b200.dist import gather_fitness, padded_shard, shard_rows, sr_fitness_data_sharded, \
    sr_fitness_population_sharded


def test_shard_rows_partition():
    for n in (0, 1, 7, 100, 10_001):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
            assert max(sizes) <= padded_shard(n, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_fitness(L, n_in):
    def fn(t, v, s, X, y, out):
        r = oracle.evaluate(t.numpy(), v.numpy(), s.numpy(), X.numpy())[:, :, 0]
        out.copy_(torch.from_numpy(oracle.mse(r, y.numpy())))
        return out
    return fn


def _oracle_sse(L, n_in):
    def fn(t, v, s, X, y, out):
        r = oracle.evaluate(t.numpy(), v.numpy(), s.numpy(), X.numpy())[:, :, 0]
        m = oracle.mse(r, y.numpy()) * X.shape[0]
        out.copy_(torch.from_numpy(m))
        return out
    return fn


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P, L, n_in, D = 37, 31, 3, 101
        pt = synth.trees(77, 0, P, L, synth.M_PAPER, n_in)
        X, y = synth.dataset_X(77, 0, D, n_in), None
        y = synth.pagie_y(X)
        t, v, s = (torch.from_numpy(a) for a in oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in))
        # population axis: rows shard_rows(P, world, rank), all-gathered fitness
        b, e = shard_rows(P, world, rank)
        full = sr_fitness_population_sharded(t[b:e].contiguous(), v[b:e].contiguous(), s[b:e].contiguous(),
                                             torch.from_numpy(X), torch.from_numpy(y), P,
                                             fitness_fn=_oracle_fitness(L, n_in))
        # datapoint axis: rows shard_rows(D, world, rank) of X / y, all-reduced SSE / D
        db, de = shard_rows(D, world, rank)
        mse_d = sr_fitness_data_sharded(t, v, s, torch.from_numpy(X[db:de].copy()), torch.from_numpy(y[db:de].copy()),
                                        D, sse_fn=_oracle_sse(L, n_in))
        # gather_fitness handles a ragged last shard
        slot = padded_shard(10, world)
        mine = torch.full((slot,), float("nan"), dtype=torch.float64)
        rb, re_ = shard_rows(10, world, rank)
        mine[: re_ - rb] = torch.arange(rb, re_, dtype=torch.float64)
        g = gather_fitness(mine, 10, world)
        q.put((rank, full.numpy(), mse_d.numpy(), g.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_fitness_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P, L, n_in, D = 37, 31, 3, 101
    pt = synth.trees(77, 0, P, L, synth.M_PAPER, n_in)
    X = synth.dataset_X(77, 0, D, n_in)
    y = synth.pagie_y(X)
    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in)
    ref = oracle.mse(oracle.evaluate(t, v, s, X)[:, :, 0], y)
    fin = np.isfinite(ref)
    for rank, full, mse_d, g in res:
        # population sharding: bit-identical to the unsharded evaluation
        assert np.array_equal(full[fin], ref[fin]) and (np.isfinite(full) == fin).all()
        # datapoint sharding: equal up to FP64 re-association
        assert np.allclose(mse_d[fin], ref[fin], rtol=1e-12, atol=0)
        assert np.array_equal(g, np.arange(10, dtype=np.float64))
