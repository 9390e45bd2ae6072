"""Genetic operators and the generational loop on the device (SURVEY §8(f)
NEXT-3 / NEXT-4). Argument marshalling over the C-ABI of include/evogp.h:
``generate`` (Algorithm 1 "Randomly generate N trees"),
``subtree_exchange`` (§III-B exchange(T_old, k, T_new)),
``tournament`` (Algorithm 1 "Select parents"; size P:477),
``reproduce`` (Algorithm 1 loop body, operators of Table I)
and ``evolve`` (Algorithm 1 for SR: evaluate -> select -> crossover ->
mutate, every step in the library's kernels; tab:sr_params P:470-483 are the
defaults). All randomness is the counter-based draw of DESIGN.md R16.
"""
from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass, field

from ._lib import OK

MUTATIONS = ("subtree", "hoist", "point", "multi_point", "insert", "delete", "const", "multi_const")
PAPER_FUNCS = (0, 1, 2, 3, 4, 5, 6)  # tab:sr_params P:480: {+, -, x, /, sin, cos, tan}


class _CCfg(ctypes.Structure):
    """Mirror of evogp_gp_config (include/evogp.h)."""
    _fields_ = [("max_len", ctypes.c_int32), ("n_inputs", ctypes.c_int32), ("n_outputs", ctypes.c_int32),
                ("func_mask", ctypes.c_uint32), ("const_lo", ctypes.c_float), ("const_hi", ctypes.c_float),
                ("p_const", ctypes.c_float), ("p_leaf", ctypes.c_float), ("p_modi", ctypes.c_float),
                ("depth_min", ctypes.c_int32), ("depth_max", ctypes.c_int32),
                ("tournament_size", ctypes.c_int32), ("p_crossover", ctypes.c_float),
                ("p_mutation", ctypes.c_float), ("crossover_kind", ctypes.c_int32),
                ("leaf_bias", ctypes.c_float), ("mutation_weights", ctypes.c_float * 8),
                ("point_rate", ctypes.c_float), ("const_sigma", ctypes.c_float),
                ("subtree_depth", ctypes.c_int32)]


@dataclass
class GPConfig:
    """Generation + variation settings; defaults follow tab:sr_params
    where the paper fixes them and DESIGN.md R18-R21 elsewhere."""
    max_len: int = 512
    n_inputs: int = 1
    n_outputs: int = 1
    funcs: tuple = PAPER_FUNCS
    const_lo: float = -1.0
    const_hi: float = 1.0
    p_const: float = 0.5
    p_leaf: float = 0.1
    p_modi: float = 0.1
    depth_min: int = 2
    depth_max: int = 6
    tournament_size: int = 20
    p_crossover: float = 0.9
    p_mutation: float = 0.1
    crossover_kind: int = 0  # 0 one-point, 1 leaf-biased
    leaf_bias: float = 0.1
    mutation_weights: tuple = field(default=(1.0, 0, 0, 0, 0, 0, 0, 0))
    point_rate: float = 0.1
    const_sigma: float = 0.1
    subtree_depth: int = 4

    def c(self) -> _CCfg:
        c = _CCfg()
        for name, _ in _CCfg._fields_:
            if name == "func_mask":
                c.func_mask = sum(1 << int(f) for f in self.funcs)
            elif name == "mutation_weights":
                c.mutation_weights = (ctypes.c_float * 8)(*[float(w) for w in self.mutation_weights])
            else:
                setattr(c, name, getattr(self, name))
        return c

    @classmethod
    def from_dict(cls, d: dict) -> "GPConfig":
        return cls(**d)


def _api():
    from . import _LIB, EvogpError, _stream_ptr, _vp
    return _LIB, EvogpError, _stream_ptr, _vp


def _rows(P, L, device):
    import torch

    return (torch.empty((P, L), dtype=torch.int16, device=device),
            torch.empty((P, L), dtype=torch.float32, device=device),
            torch.empty((P, L), dtype=torch.int16, device=device))


def generate(P: int, cfg: GPConfig, seed: int, device="cuda", out=None, stream=None):
    """Device: ramped half-and-half population (type, value, size), each [P, max_len]."""
    import torch

    lib, Err, sp, vp = _api()
    device = torch.device(device)
    t, v, s = out if out is not None else _rows(P, cfg.max_len, device)
    cc = cfg.c()
    st = lib.evogp_generate(P, ctypes.byref(cc), seed, vp(t), vp(v), vp(s), sp(stream, device))
    if st != OK:
        raise Err(st, "evogp_generate")
    return t, v, s


def subtree_exchange(old, parent, k, donors, donor, j, max_len: int, out=None, rejected=True, stream=None):
    """Device: child c = exchange(old[parent[c]], k[c], donors[donor[c]] at j[c])
    (§III-B). old / donors: (type, value, size) tuples; index
    arrays int32 CUDA tensors. Returns (type, value, size, rejected uint8)."""
    import torch

    lib, Err, sp, vp = _api()
    ot, ov, os_ = old
    dt, dv, ds = donors
    n = int(parent.numel())
    dev = ot.device
    t, v, s = out if out is not None else _rows(n, max_len, dev)
    rej = torch.empty(n, dtype=torch.uint8, device=dev) if rejected else None
    st = lib.evogp_subtree_exchange(n, vp(ot), vp(ov), vp(os_), int(ot.shape[1]), vp(parent), vp(k), vp(dt),
                                    vp(dv), vp(ds), int(dt.shape[1]), vp(donor), vp(j), max_len, vp(t), vp(v),
                                    vp(s), vp(rej), sp(stream, dev))
    if st != OK:
        raise Err(st, "evogp_subtree_exchange")
    return t, v, s, rej


def tournament(fitness, T: int, n_winners: int, seed: int, purpose: int = 1, out=None, stream=None):
    """Device: int32 winners [n_winners] (Algorithm 1 "Select parents"; lower fitness wins)."""
    import torch

    lib, Err, sp, vp = _api()
    w = out if out is not None else torch.empty(n_winners, dtype=torch.int32, device=fitness.device)
    st = lib.evogp_tournament(vp(fitness), int(fitness.numel()), T, n_winners, seed, purpose, vp(w),
                              sp(stream, fitness.device))
    if st != OK:
        raise Err(st, "evogp_tournament")
    return w


def reproduce(pop, fitness, n_children: int, cfg: GPConfig, seed: int, child0: int = 0, out=None,
              record: bool = True, stream=None):
    """Device: the next population (Algorithm 1 loop body).
    Returns (type, value, size, parents int32 [n,2] | None, ops int32 [n] | None)."""
    import torch

    lib, Err, sp, vp = _api()
    t0, v0, s0 = pop
    dev = t0.device
    t, v, s = out if out is not None else _rows(n_children, cfg.max_len, dev)
    par = torch.empty((n_children, 2), dtype=torch.int32, device=dev) if record else None
    ops = torch.empty(n_children, dtype=torch.int32, device=dev) if record else None
    cc = cfg.c()
    st = lib.evogp_reproduce(vp(t0), vp(v0), vp(s0), int(t0.shape[0]), int(t0.shape[1]), vp(fitness), n_children,
                             child0, ctypes.byref(cc), seed, vp(t), vp(v), vp(s), vp(par), vp(ops), sp(stream, dev))
    if st != OK:
        raise Err(st, "evogp_reproduce")
    return t, v, s, par, ops


def selector_strategy(pop, D: int) -> str:
    """Selector (c) for a population whose trees may be much shorter than its
    row length: the calibration (tools/calibrate_selector.py) draws tree
    lengths uniformly in [L/2, L] (mean 0.75 L), so the table is keyed on the
    row length a population of this mean length would have. One device
    reduction + sync (call it outside timed loops)."""
    from . import select_strategy

    t, v, s = pop
    P, L = int(s.shape[0]), int(s.shape[1])
    mean = float(s[:, 0].float().mean().item()) if P else float(L)
    L_eff = max(1, min(L, int(round(mean / 0.75))))
    return select_strategy(P, D, L_eff)


class Evolution:
    """Algorithm 1 for symbolic regression, device-resident:
    generation -> [fitness (fused SR MSE) -> reproduce] x G. Two population
    buffers are swapped each generation; nothing leaves the device except
    what the caller reads. ``step()`` is one generation."""

    def __init__(self, P: int, cfg: GPConfig, X, y, seed: int = 0, strategy="auto"):
        import torch

        from . import sr_fitness

        self._sr = sr_fitness
        self.P, self.cfg, self.X, self.y, self.seed, self.strategy = P, cfg, X, y, seed, strategy
        dev = X.device
        self.bufs = [_rows(P, cfg.max_len, dev), _rows(P, cfg.max_len, dev)]
        self.cur = 0
        generate(P, cfg, seed, device=dev, out=self.bufs[0])
        self.fitness = torch.empty(P, dtype=torch.float64, device=dev)
        self.generation = 0
        # a function set beyond the paper's: the full-set kernel variants
        # (evogp_tuning.full_set, include/evogp.h)
        self._full_set = bool(set(cfg.funcs) - set(PAPER_FUNCS))
        if strategy == "auto":
            with self._hint():
                self.strategy = selector_strategy(self.bufs[0], int(X.shape[0]))

    def _hint(self):
        from . import tuning_hint

        return tuning_hint(full_set=True) if self._full_set else contextlib.nullcontext()

    @property
    def population(self):
        return self.bufs[self.cur]

    def evaluate(self):
        t, v, s = self.population
        with self._hint():
            self._sr(t, v, s, self.X, self.y, strategy=self.strategy, out=self.fitness)
        return self.fitness

    def step(self):
        """Fitness of the current population, then its children (one generation)."""
        self.evaluate()
        nxt = 1 - self.cur
        reproduce(self.population, self.fitness, self.P, self.cfg, self.seed + 1 + self.generation,
                  out=self.bufs[nxt], record=False)
        self.cur = nxt
        self.generation += 1
