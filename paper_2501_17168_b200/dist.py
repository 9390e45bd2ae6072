"""Multi-GPU sharding of the hot path.

One process per GPU (torchrun), ``torch.distributed`` with NCCL over
NVLink/NVSwitch for the two exchange steps the path has:

* population axis: trees are independent, so rank r evaluates rows
  ``shard_rows(P, world, r)`` and the per-tree MSEs are all-gathered
  (``all_gather_into_tensor``, P x 8 bytes in total);
* datapoint axis: rank r evaluates every tree on its rows of X / y
  (``shard_rows(D, world, r)``) with ``evogp_sr_sse`` and the per-tree SSEs
  are all-reduced in FP64, then scaled by 1/D (NCCL PREMUL_SUM, so the
  division happens inside the collective, no extra kernel).

The paper is single-GPU (§V); these combines are the
only collectives on the path. The per-shard evaluator defaults to the CUDA
C-ABI; tests inject another evaluator to cover the host logic with gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal split: rank r owns [begin, end); shard sizes differ by <= 1."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    end = begin + base + (1 if rank < extra else 0)
    return begin, end


def padded_shard(n: int, world: int) -> int:
    """Per-rank slot count for equal-size all-gathers (ceil(n / world))."""
    return -(-n // world)


def _default_fitness(type_, value, size, X, y, out):
    from . import sr_fitness

    return sr_fitness(type_, value, size, X, y, out=out)


def _default_sse(type_, value, size, X, y, out):
    from . import sr_sse

    return sr_sse(type_, value, size, X, y, out=out)


def gather_fitness(local_mse: torch.Tensor, n_total: int, world: int, group=None) -> torch.Tensor:
    """all-gather per-rank MSE slots (each padded_shard(n_total, world) long)
    and return the n_total-long population vector in global row order."""
    slot = local_mse.numel()
    full = torch.empty(slot * world, dtype=local_mse.dtype, device=local_mse.device)
    dist.all_gather_into_tensor(full, local_mse, group=group)
    if slot * world == n_total:
        return full
    idx = []
    for r in range(world):
        b, e = shard_rows(n_total, world, r)
        idx.append((r * slot, r * slot + (e - b)))
    return torch.cat([full[a:b] for a, b in idx])


def sr_fitness_population_sharded(type_shard, value_shard, size_shard, X, y, n_total: int, group=None,
                                  fitness_fn=None, local_out: torch.Tensor | None = None) -> torch.Tensor:
    """Rank-local rows -> fitness of the whole population (replicated on every rank).

    type/value/size_shard: this rank's rows, i.e. rows shard_rows(n_total, world, rank).
    """
    world = dist.get_world_size(group)
    fn = fitness_fn or _default_fitness
    slot = padded_shard(n_total, world)
    if local_out is None or local_out.numel() != slot:
        local_out = torch.full((slot,), float("nan"), dtype=torch.float64, device=X.device)
    n_local = type_shard.shape[0]
    if n_local:
        fn(type_shard, value_shard, size_shard, X, y, local_out[:n_local])
    return gather_fitness(local_out, n_total, world, group)


def sr_fitness_data_sharded(type_, value, size, X_shard, y_shard, D_total: int, group=None, sse_fn=None,
                            out: torch.Tensor | None = None) -> torch.Tensor:
    """Every rank holds all trees and rows shard_rows(D_total, world, rank) of X/y;
    returns mse = (sum over ranks of sse) / D_total on every rank."""
    fn = sse_fn or _default_sse
    P = type_.shape[0]
    if out is None:
        out = torch.empty(P, dtype=torch.float64, device=X_shard.device)
    if X_shard.shape[0] > 0:
        fn(type_, value, size, X_shard, y_shard, out)
    else:
        out.zero_()
    backend = dist.get_backend(group)
    if backend == "nccl":
        op = dist._make_nccl_premul_sum(1.0 / D_total)
        dist.all_reduce(out, op=op, group=group)
    else:  # gloo has no PREMUL_SUM (host tests only)
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
        out.div_(D_total)
    return out
