"""Seeded synthetic workloads shaped like the paper's (DESIGN.md
"Synthetic inputs"). Shared by the oracle side and the CUDA side; contains no
method arithmetic: it only emits prefix-form trees (CSR) and datasets.

Function-id mixes:
  M_PAPER   {+,-,*,/,sin,cos,tan}      PAPER.md tab:sr_params
  M_FULL    all 22 ids                  north-star function set (R3)
  M_BOUNDED {+,-,*,/,max,min,sin,cos,tanh}
  M_IEEE    ops that are correctly rounded in FP32 (Tier A parity mix)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lock = threading.Lock()
_lib = None

BASE_SEED = 2501017168

M_PAPER = (0, 1, 2, 3, 4, 5, 6)
M_FULL = tuple(range(22))
M_BOUNDED = (0, 1, 2, 3, 7, 8, 4, 5, 12)
M_IEEE = (0, 1, 2, 3, 15, 13, 14, 7, 8, 17, 18, 19, 20, 21)
MIXES = {"paper": M_PAPER, "full": M_FULL, "bounded": M_BOUNDED, "ieee": M_IEEE}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            i64, i32, u64, f64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
            lib.synth_offsets.argtypes = [u64, i64, i64, i32, vp]
            lib.synth_offsets.restype = None
            lib.synth_trees.argtypes = [u64, i64, i64, i32, vp, i32, i32, i32, f64, vp, vp, vp, i32]
            lib.synth_trees.restype = ctypes.c_int
            lib.synth_X.argtypes = [u64, i64, i64, i32, i32, f64, f64, vp]
            lib.synth_X.restype = None
            lib.synth_pagie_y.argtypes = [vp, i64, i32, vp]
            lib.synth_pagie_y.restype = None
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class PrefixTrees:
    """CSR prefix-order trees: tree i is types/values[offsets[i]:offsets[i+1]]."""

    offsets: np.ndarray  # int64 [n+1]
    types: np.ndarray  # int16 [nnz]
    values: np.ndarray  # float32 [nnz]

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    def tree(self, i: int):
        b, e = int(self.offsets[i]), int(self.offsets[i + 1])
        return self.types[b:e], self.values[b:e]


def trees(seed: int, p0: int, n: int, max_len: int, mix, n_in: int, n_out: int = 1,
          modi_prob: float = 0.0, threads: int | None = None) -> PrefixTrees:
    """Trees [p0, p0+n) of the population keyed by `seed`."""
    lib = _load()
    offsets = np.empty(n + 1, dtype=np.int64)
    lib.synth_offsets(seed, p0, n, max_len, _ptr(offsets))
    nnz = int(offsets[-1])
    ty = np.empty(max(nnz, 1), dtype=np.int16)
    va = np.empty(max(nnz, 1), dtype=np.float32)
    mixa = np.asarray(mix, dtype=np.int32)
    th = threads or min(32, os.cpu_count() or 1)
    rc = lib.synth_trees(seed, p0, n, max_len, _ptr(mixa), len(mixa), n_in, n_out, modi_prob,
                         _ptr(offsets), _ptr(ty), _ptr(va), th)
    if rc != 0:
        raise ValueError("synth_trees: bad arguments")
    return PrefixTrees(offsets, ty[:nnz], va[:nnz])


def dataset_X(seed: int, d0: int, n: int, n_in: int, dist: str = "uniform", lo: float = -1.0,
              hi: float = 1.0) -> np.ndarray:
    """Rows [d0, d0+n) of X (row-major D x n_in, float32)."""
    lib = _load()
    X = np.empty((n, n_in), dtype=np.float32)
    lib.synth_X(seed, d0, n, n_in, 0 if dist == "uniform" else 1, lo, hi, _ptr(X))
    return X


def pagie_y(X: np.ndarray) -> np.ndarray:
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.empty(X.shape[0], dtype=np.float32)
    lib.synth_pagie_y(_ptr(X), X.shape[0], X.shape[1], _ptr(y))
    return y


# ---- the BASELINE.json configs as concrete synthetic inputs ----
@dataclass(frozen=True)
class Config:
    name: str
    P: int
    max_len: int
    n_in: int
    n_out: int
    D: int
    x_dist: str
    x_lo: float
    x_hi: float
    modi_prob: float
    index: int
    paired: bool = False  # NEXT-2: D = observations per individual (B), each tree on its own
    loop: bool = False  # NEXT-4: the whole generational loop (Algorithm 1), population generated on device
    eval_only: bool = False  # outputs only (evogp_eval), no fitness: config 5's alternative reading

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index


CONFIGS = {
    "c1": Config("c1_sr_tiny", 64, 15, 2, 1, 32, "uniform", -5.0, 5.0, 0.0, 1),
    "c2": Config("c2_inter", 10_000, 63, 4, 1, 1024, "uniform", -1.0, 1.0, 0.0, 2),
    "c3": Config("c3_intra", 1000, 127, 8, 1, 1 << 20, "uniform", -1.0, 1.0, 0.0, 3),
    "c4": Config("c4_large_pop", 1_000_000, 127, 8, 1, 256, "uniform", -1.0, 1.0, 0.0, 4),
    "c5": Config("c5_multi_output", 10_000, 63, 17, 6, 4096, "normal", 0.0, 0.0, 0.1, 5),
    # config 5's alternative reading: "10^4 individuals x 6 output
    # trees" as 6 x 10^4 independent single-output trees, outputs only
    "c5b": Config("c5b_six_single_output_trees", 60_000, 63, 17, 1, 4096, "normal", 0.0, 0.0, 0.0, 8,
                  eval_only=True),
    # NEXT-2: one control step of 10^6 policy trees, each on
    # its own 17-dim observation, 6 Modi outputs (shapes from config 5)
    "n2": Config("n2_paired_policy", 1_000_000, 63, 17, 6, 1, "normal", 0.0, 0.0, 0.1, 6, True),
    # NEXT-4: the paper's whole-run GPops/s protocol at its
    # peak cell (tab:gpops_summary P:592: P = 10^5, D = 392 Auto-MPG-shaped
    # rows with 7 features, tab:sr_datasets P:550), max tree size 512 and the
    # rest of tab:sr_params; synthetic Pagie-7 targets
    "g1": Config("g1_sr_loop", 100_000, 512, 7, 1, 392, "uniform", -1.0, 1.0, 0.0, 7, False, True),
}


def config_trees(cfg: Config, mix=M_PAPER, p0: int = 0, n: int | None = None) -> PrefixTrees:
    n = cfg.P if n is None else n
    return trees(cfg.seed, p0, n, cfg.max_len, mix, cfg.n_in, cfg.n_out, cfg.modi_prob)


def config_data(cfg: Config, d0: int = 0, n: int | None = None):
    n = cfg.D if n is None else n
    X = dataset_X(cfg.seed, d0, n, cfg.n_in, cfg.x_dist, cfg.x_lo, cfg.x_hi)
    return X, pagie_y(X)
