"""Parity oracle for the EvoGP hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product package
(paper_2501_17168_b200) never imports it, and it never imports the product.

Thin ctypes wrappers over oracle.c (plain C, FP64) plus the certificate
decision rules of DESIGN.md reading R14:
  * a point is *certified* iff every decision on its path is robust, its FP64
    value is finite and 2*e <= 0.5 * tol * max(1, |v|);
  * a tree is *MSE-certified* iff all its points are certified and
    2 * sum_d (2|v_d - y_d| e_d + e_d^2) <= 0.5 * tol * SSE.
Parity of each function is pinned by tests/test_oracle_pins.py (no GPU).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, E_ARG, E_TOO_LARGE, E_MALFORMED, E_VAR_RANGE, E_FUNC_UNKNOWN, E_OUT_RANGE = 0, -1, -2, -3, -4, -5, -6

TOL = 1e-4  # north star: |gpu - oracle| <= 1e-4 * max(1, |oracle|)


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("oracle.c", "variation.c")]
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(f) for f in srcs):
        # plain -O2, no -ffast-math, no FMA contraction: the oracle computes
        # exactly the expressions written in oracle.c / variation.c
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-pthread", "-o", _SO] + srcs + ["-lm"])
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
            lib.oracle_tensorize.argtypes = [i64, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp]
            lib.oracle_tensorize.restype = ctypes.c_int
            lib.oracle_eval.argtypes = [vp, vp, vp, i64, i32, vp, i64, i32, i32, i32, vp, vp, vp, i32]
            lib.oracle_eval.restype = ctypes.c_int
            lib.oracle_eval_recursive.argtypes = [vp, vp, i32, vp, i32, i32, i32, vp]
            lib.oracle_eval_recursive.restype = ctypes.c_int
            lib.oracle_mse.argtypes = [vp, vp, i64, i64, vp]
            lib.oracle_mse.restype = ctypes.c_int
            lib.oracle_accuracy.argtypes = [vp, vp, i64, i64, i32, vp]
            lib.oracle_accuracy.restype = ctypes.c_int
            u64 = ctypes.c_uint64
            lib.orv_draw.argtypes = [u64, u64, u64]
            lib.orv_draw.restype = ctypes.c_uint32
            lib.oracle_exchange.argtypes = [i64, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp]
            lib.oracle_exchange.restype = ctypes.c_int
            lib.oracle_tournament.argtypes = [vp, i64, i32, i64, u64, i32, vp]
            lib.oracle_tournament.restype = ctypes.c_int
            lib.oracle_generate.argtypes = [i64, vp, u64, vp, vp, vp]
            lib.oracle_generate.restype = ctypes.c_int
            lib.oracle_reproduce.argtypes = [vp, vp, vp, i64, i32, vp, i64, i64, vp, u64, vp, vp, vp, vp, vp]
            lib.oracle_reproduce.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, status, tree=-1, node=-1):
        super().__init__(f"oracle status {status} (tree {tree}, node {node})")
        self.status, self.tree, self.node = status, tree, node


def tensorize(offsets, types, values, max_len: int, n_inputs: int, n_outputs: int = 1, raise_on_error=True):
    """Prefix CSR -> (type[P,L] i16, value[P,L] f32, size[P,L] i16). PAPER.md P:221-258."""
    lib = _load()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    types = np.ascontiguousarray(types, dtype=np.int16)
    values = np.ascontiguousarray(values, dtype=np.float32)
    P = len(offsets) - 1
    ot = np.zeros((P, max_len), dtype=np.int16)
    ov = np.zeros((P, max_len), dtype=np.float32)
    os_ = np.zeros((P, max_len), dtype=np.int16)
    et = np.zeros(1, dtype=np.int64)
    en = np.zeros(1, dtype=np.int32)
    if types.size == 0:
        types = np.zeros(1, dtype=np.int16)
        values = np.zeros(1, dtype=np.float32)
    st = lib.oracle_tensorize(P, _p(offsets), _p(types), _p(values), max_len, n_inputs, n_outputs,
                              _p(ot), _p(ov), _p(os_), _p(et), _p(en))
    if st != OK:
        if raise_on_error:
            raise OracleError(st, int(et[0]), int(en[0]))
        return st, int(et[0]), int(en[0])
    return (ot, ov, os_) if raise_on_error else (OK, -1, -1, ot, ov, os_)


def evaluate(type_, value, size, X, n_out: int = 1, mode: int = 0, certify: bool = False,
             threads: int | None = None):
    """Stack evaluation. Returns out[P,D,n_out] float64 (and err, robust
    if certify). mode 0 = FP64 + FP32-range emulation; 1 = FP32-faithful."""
    lib = _load()
    type_ = np.ascontiguousarray(type_, dtype=np.int16)
    value = np.ascontiguousarray(value, dtype=np.float32)
    size = np.ascontiguousarray(size, dtype=np.int16)
    X = np.ascontiguousarray(X, dtype=np.float32)
    P, ld = type_.shape
    D, n_in = X.shape
    out = np.zeros((P, D, n_out), dtype=np.float64)
    err = np.zeros((P, D, n_out), dtype=np.float64) if certify else None
    rob = np.zeros((P, D, n_out), dtype=np.uint8) if certify else None
    th = threads or min(32, os.cpu_count() or 1)
    st = lib.oracle_eval(_p(type_), _p(value), _p(size), P, ld, _p(X), D, n_in, n_out, mode, _p(out),
                         _p(err), _p(rob), th)
    if st != OK:
        raise OracleError(st)
    if certify:
        return out, err, rob.astype(bool)
    return out


def evaluate_recursive(types, values, x, n_out: int = 1, mode: int = 0):
    """Independent recursive interpreter for one unpadded prefix tree at one point."""
    lib = _load()
    types = np.ascontiguousarray(types, dtype=np.int16)
    values = np.ascontiguousarray(values, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(n_out, dtype=np.float64)
    st = lib.oracle_eval_recursive(_p(types), _p(values), len(types), _p(x), len(x), n_out, mode, _p(out))
    if st != OK:
        raise OracleError(st)
    return out


def evaluate_paired(type_, value, size, obs, n_out: int = 1, mode: int = 0):
    """Paired per-individual inference (PAPER §III-C, SURVEY §8(f)
    NEXT-2): tree p evaluated on its own observations obs[p] ([P,B,n_in]).
    Row by row through `evaluate`. Returns out[P,B,n_out] float64."""
    obs = np.asarray(obs, dtype=np.float32)
    P, B, _ = obs.shape
    out = np.zeros((P, B, n_out), dtype=np.float64)
    for p in range(P):
        out[p] = evaluate(type_[p:p + 1], value[p:p + 1], size[p:p + 1], obs[p], n_out=n_out, mode=mode,
                          threads=1)[0]
    return out


def mse(pred, y):
    """mse[p] = mean_d (pred[p,d] - y[d])^2 in FP64 (reading R7)."""
    lib = _load()
    pred = np.ascontiguousarray(pred, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float32)
    P = pred.shape[0]
    D = pred.shape[1]
    out = np.zeros(P, dtype=np.float64)
    st = lib.oracle_mse(_p(pred.reshape(P, D)), _p(y), P, D, _p(out))
    if st != OK:
        raise OracleError(st)
    return out


def accuracy(out, labels):
    """Classification accuracy per tree: argmax over outputs (ties -> lowest
    class, NaN as -inf) vs labels (R15)."""
    lib = _load()
    out = np.ascontiguousarray(out, dtype=np.float64)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    P, D, n_out = out.shape
    acc = np.zeros(P, dtype=np.float64)
    st = lib.oracle_accuracy(_p(out), _p(labels), P, D, n_out, _p(acc))
    if st != OK:
        raise OracleError(st)
    return acc


def certified_points(v, e, robust, tol: float = TOL):
    """Reading R14: robust decisions, finite value, 2e <= 0.5*tol*max(1,|v|)."""
    with np.errstate(invalid="ignore", over="ignore"):
        return robust & np.isfinite(v) & np.isfinite(e) & (2.0 * e <= 0.5 * tol * np.maximum(1.0, np.abs(v)))


def mse_certified_trees(v, e, robust, y, tol: float = TOL):
    """v, e, robust: [P, D] (single output). Returns bool[P]."""
    cert = certified_points(v, e, robust, tol).all(axis=1)
    with np.errstate(invalid="ignore", over="ignore"):
        r = np.abs(v - y.astype(np.float64)[None, :])
        bound = 2.0 * np.sum(2.0 * r * e + e * e, axis=1)
        sse = np.sum(r * r, axis=1)
        return cert & np.isfinite(sse) & (bound <= 0.5 * tol * sse)


def within_tol(gpu, ref, tol: float = TOL):
    """North-star per-point check with identical NaN/+-Inf class."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    same_nan = np.isnan(gpu) == np.isnan(ref)
    inf_g = np.isinf(gpu)
    inf_r = np.isinf(ref)
    same_inf = (inf_g == inf_r) & (~inf_g | (np.sign(gpu) == np.sign(ref)))
    fin = np.isfinite(gpu) & np.isfinite(ref)
    with np.errstate(invalid="ignore", over="ignore"):
        close = np.abs(gpu - ref) <= tol * np.maximum(1.0, np.abs(ref))
    return same_nan & same_inf & (~fin | close)


# ---------------------------------------------------------------------------
# Genetic operators (oracle/variation.c)
# ---------------------------------------------------------------------------
MUTATIONS = ("subtree", "hoist", "point", "multi_point", "insert", "delete", "const", "multi_const")
PUR = dict(tour1=1, tour2=2, xo_gate=3, xo_k=4, xo_j=5, mut_gate=6, mut_kind=7, mut_site=8, point_coin=9,
           point_new=10, gen=11)
OP_XO, OP_XO_REJECTED, OP_MUT_NOP = 1, 2, 0x100


class OvCfg(ctypes.Structure):
    """Mirror of OvCfg in variation.c (DESIGN.md §14 field list)."""
    _fields_ = [("max_len", ctypes.c_int32), ("n_inputs", ctypes.c_int32), ("n_outputs", ctypes.c_int32),
                ("func_mask", ctypes.c_uint32), ("const_lo", ctypes.c_float), ("const_hi", ctypes.c_float),
                ("p_const", ctypes.c_float), ("p_leaf", ctypes.c_float), ("p_modi", ctypes.c_float),
                ("depth_min", ctypes.c_int32), ("depth_max", ctypes.c_int32),
                ("tournament_size", ctypes.c_int32), ("p_crossover", ctypes.c_float),
                ("p_mutation", ctypes.c_float), ("crossover_kind", ctypes.c_int32),
                ("leaf_bias", ctypes.c_float), ("mutation_weights", ctypes.c_float * 8),
                ("point_rate", ctypes.c_float), ("const_sigma", ctypes.c_float),
                ("subtree_depth", ctypes.c_int32)]


def make_cfg(d: dict) -> OvCfg:
    """dict with the OvCfg field names (mutation_weights: 8 floats, funcs: ids)."""
    c = OvCfg()
    for k, v in d.items():
        if k == "funcs":
            c.func_mask = sum(1 << int(f) for f in v)
        elif k == "mutation_weights":
            c.mutation_weights = (ctypes.c_float * 8)(*v)
        else:
            setattr(c, k, v)
    return c


def draw(seed: int, stream: int, purpose: int, index: int) -> int:
    """Reading R16 counter-based draw (uint32)."""
    return int(_load().orv_draw(seed, stream, (purpose << 32) | index))


def exchange(old_t, old_v, old_s, parent, k, don_t, don_v, don_s, donor, j, max_len: int):
    """Batched subtree exchange (§III-B). Returns (t, v, s, rejected)."""
    lib = _load()
    old_t, old_v, old_s = (np.ascontiguousarray(a) for a in (old_t, old_v, old_s))
    don_t, don_v, don_s = (np.ascontiguousarray(a) for a in (don_t, don_v, don_s))
    parent, k, donor, j = (np.ascontiguousarray(a, dtype=np.int32) for a in (parent, k, donor, j))
    n = len(parent)
    ld = old_t.shape[1]
    ot = np.zeros((n, max_len), np.int16)
    ov = np.zeros((n, max_len), np.float32)
    os_ = np.zeros((n, max_len), np.int16)
    rej = np.zeros(n, np.uint8)
    st = lib.oracle_exchange(n, _p(old_t), _p(old_v), _p(old_s), ld, _p(parent), _p(k), _p(don_t), _p(don_v),
                             _p(don_s), _p(donor), _p(j), max_len, _p(ot), _p(ov), _p(os_), _p(rej))
    if st != OK:
        raise OracleError(st)
    return ot, ov, os_, rej.astype(bool)


def tournament(fit, T: int, n_winners: int, seed: int, purpose: int = 1):
    """Tournament selection (Algorithm 1 "Select parents"; size P:477; R17)."""
    fit = np.ascontiguousarray(fit, dtype=np.float64)
    w = np.zeros(n_winners, np.int32)
    st = _load().oracle_tournament(_p(fit), len(fit), T, n_winners, seed, purpose, _p(w))
    if st != OK:
        raise OracleError(st)
    return w


def generate(P: int, cfg: dict, seed: int):
    """Ramped half-and-half initial population (Algorithm 1; R19)."""
    c = make_cfg(cfg)
    L = c.max_len
    t = np.zeros((P, L), np.int16)
    v = np.zeros((P, L), np.float32)
    s = np.zeros((P, L), np.int16)
    st = _load().oracle_generate(P, ctypes.byref(c), seed, _p(t), _p(v), _p(s))
    if st != OK:
        raise OracleError(st)
    return t, v, s


def reproduce(t, v, s, fit, n_children: int, cfg: dict, seed: int, child0: int = 0):
    """Algorithm 1 loop body (R18): returns (t, v, s, parents[n,2], ops[n])."""
    c = make_cfg(cfg)
    L = c.max_len
    t, v, s = (np.ascontiguousarray(a) for a in (t, v, s))
    fit = np.ascontiguousarray(fit, dtype=np.float64)
    P, ld = t.shape
    ot = np.zeros((n_children, L), np.int16)
    ov = np.zeros((n_children, L), np.float32)
    os_ = np.zeros((n_children, L), np.int16)
    par = np.zeros((n_children, 2), np.int32)
    ops = np.zeros(n_children, np.int32)
    st = _load().oracle_reproduce(_p(t), _p(v), _p(s), P, ld, _p(fit), n_children, child0, ctypes.byref(c), seed,
                                  _p(ot), _p(ov), _p(os_), _p(par), _p(ops))
    if st != OK:
        raise OracleError(st)
    return ot, ov, os_, par, ops
