"""paper_2501_17168_b200 — B200-native (sm_100a) EvoGP hot path.

Thin Python binding over libevogp.so (include/evogp.h). Every step of the
path runs in the library's CUDA kernels; this module only marshals
arguments (torch is used for device memory and streams). Names follow the
C-ABI: ``tensorize``, ``eval``, ``sr_fitness``, ``sr_sse``,
``select_strategy``, ``workspace_size``, ``check_device_flags``.

Population arrays are the paper's tensorized layout (§III-A,
P:221-258): ``type`` int16, ``value`` float32, ``size`` int16, each P x ld.
"""
from __future__ import annotations

import contextlib
import math
import ctypes
import threading

import numpy as np

from . import _lib
from ._lib import (E_ARG, E_CUDA, E_FUNC_UNKNOWN, E_MALFORMED, E_OUT_RANGE, E_TOO_LARGE, E_UNSUPPORTED,
                   E_VAR_RANGE, OK, STRATEGY_AUTO, STRATEGY_INTER, STRATEGY_INTRA, X_ROWMAJOR, X_SOA)

_LIB = _lib.load()

__all__ = [
    "tensorize", "tensorize_device", "eval", "sr_fitness", "sr_sse", "classification_accuracy", "eval_paired", "select_strategy", "workspace_size", "Workspace",
    "check_device_flags", "EvogpError", "last_launch_count", "set_tuning", "tuning_hint", "set_kernel_timing", "STRATEGIES",
    "GPConfig", "generate", "subtree_exchange", "tournament", "reproduce", "Evolution",
]

STRATEGIES = {"auto": STRATEGY_AUTO, "inter": STRATEGY_INTER, "intra": STRATEGY_INTRA,
              STRATEGY_AUTO: STRATEGY_AUTO, STRATEGY_INTER: STRATEGY_INTER, STRATEGY_INTRA: STRATEGY_INTRA}


class EvogpError(RuntimeError):
    def __init__(self, status: int, where: str, tree: int = -1, node: int = -1):
        msg = _LIB.evogp_status_string(status).decode()
        detail = _LIB.evogp_last_error().decode()
        super().__init__(f"{where}: {msg} ({status}); {detail}; tree={tree} node={node}")
        self.status, self.tree, self.node = status, tree, node


def _vp(a) -> ctypes.c_void_p:
    if a is None:
        return ctypes.c_void_p(0)
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


def tensorize(offsets, types, values, max_len: int, n_inputs: int, n_outputs: int = 1, out=None):
    """Host: prefix CSR lists -> (type[P,L] int16, value[P,L] float32, size[P,L] int16).
    ``out`` may supply the three host arrays (e.g. numpy views of pinned memory)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    types = np.ascontiguousarray(types, dtype=np.int16)
    values = np.ascontiguousarray(values, dtype=np.float32)
    P = len(offsets) - 1
    if out is not None:
        ot, ov, osz = out
        for a, dt in zip(out, (np.int16, np.float32, np.int16)):
            if a.dtype != dt or a.shape != (P, max_len) or not a.flags.c_contiguous:
                raise ValueError("tensorize out arrays must be C-contiguous (P, max_len) int16/float32/int16")
    else:
        ot = np.empty((P, max_len), dtype=np.int16)
        ov = np.empty((P, max_len), dtype=np.float32)
        osz = np.empty((P, max_len), dtype=np.int16)
    et = np.zeros(1, dtype=np.int64)
    en = np.zeros(1, dtype=np.int32)
    if types.size == 0:
        types = np.zeros(1, np.int16)
        values = np.zeros(1, np.float32)
    st = _LIB.evogp_tensorize(P, _vp(offsets), _vp(types), _vp(values), max_len, n_inputs, n_outputs, _vp(ot),
                              _vp(ov), _vp(osz), _vp(et), _vp(en))
    if st != OK:
        raise EvogpError(st, "evogp_tensorize", int(et[0]), int(en[0]))
    return ot, ov, osz


def tensorize_device(offsets, types, values, max_len: int, n_inputs: int, n_outputs: int = 1, out=None,
                     status: bool = True, stream=None):
    """Device: prefix CSR lists (CUDA tensors: offsets int64 [P+1], types
    int16, values float32) -> (type, value, size) [P, max_len] CUDA tensors
    and per-tree status int32 [P] (0 or the EVOGP_E_* code), or None."""
    import torch

    P = int(offsets.numel()) - 1
    dev = offsets.device
    for a, dt in ((offsets, torch.int64), (types, torch.int16), (values, torch.float32)):
        if not a.is_cuda or a.dtype != dt or not a.is_contiguous():
            raise ValueError("offsets / types / values must be contiguous CUDA int64 / int16 / float32 tensors")
    if out is None:
        out = (torch.empty((P, max_len), dtype=torch.int16, device=dev),
               torch.empty((P, max_len), dtype=torch.float32, device=dev),
               torch.empty((P, max_len), dtype=torch.int16, device=dev))
    st = torch.empty(P, dtype=torch.int32, device=dev) if status else None
    t, v, s = out
    rc = _LIB.evogp_tensorize_device(P, _vp(offsets), _vp(types), _vp(values), max_len, n_inputs, n_outputs, _vp(t),
                                     _vp(v), _vp(s), _vp(st), _stream_ptr(stream, dev))
    if rc != OK:
        raise EvogpError(rc, "evogp_tensorize_device")
    return t, v, s, st


def workspace_size(P: int, D: int, max_len: int, n_inputs: int, n_outputs: int = 1) -> int:
    return int(_LIB.evogp_workspace_size(P, D, max_len, n_inputs, n_outputs))


class Workspace:
    """Zero-initialised device scratch sized by evogp_workspace_size (for the
    device it lives on, under the current tuning)."""

    def __init__(self, P, D, max_len, n_inputs, n_outputs=1, device=None):
        import torch

        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(dev):
            self.nbytes = workspace_size(P, D, max_len, n_inputs, n_outputs)
        self.buf = torch.zeros(self.nbytes + 256, dtype=torch.uint8, device=dev)
        base = self.buf.data_ptr()
        self.ptr = (base + 255) // 256 * 256
        self.key = (P, D, max_len, n_inputs, n_outputs, str(self.buf.device))


_WS_CACHE: dict = {}


def _workspace(P, D, L, n_in, n_out, device, ws, stream=None):
    """The caller's workspace, else a cached one private to (shape, device,
    stream, thread): calls sharing a workspace must be stream-ordered
    (include/evogp.h), which a per-stream, per-thread cache guarantees."""
    if ws is not None:
        return ws
    import threading

    import torch

    s = stream if stream is not None else torch.cuda.current_stream(device)
    # the plan (and so the workspace size) depends on the thread's tuning
    tu = tuple(sorted(getattr(_TUNING, "kw", {}).items()))
    key = (P, D, L, n_in, n_out, str(device), int(s.cuda_stream), threading.get_ident(), tu)
    w = _WS_CACHE.get(key)
    if w is None:
        if len(_WS_CACHE) > 16:
            # entries may still be in use by enqueued work on their streams
            torch.cuda.synchronize(device)
            _WS_CACHE.clear()
        w = Workspace(P, D, L, n_in, n_out, device)
        _WS_CACHE[key] = w
    return w


def _stream_ptr(stream, device):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _device_guard(device):
    """Make `device` current for the body (the library plans and launches on
    the current device); a no-op when it already is (the common case: a
    context manager switch costs microseconds on launch-bound calls)."""
    import torch

    if device.index is None or device.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(device)


def _tree_args(type_, value, size, max_len):
    import torch

    if type_.dim() != 2 or value.shape != type_.shape or size.shape != type_.shape:
        raise ValueError("type / value / size must be [P, ld] arrays of the same shape")
    for t, dt in ((type_, torch.int16), (value, torch.float32), (size, torch.int16)):
        if not t.is_cuda or not t.is_contiguous() or t.dtype != dt:
            raise ValueError("tree arrays must be contiguous CUDA tensors: type int16, value float32, size int16")
        if t.device != type_.device:
            raise ValueError("tree arrays must be on one device")
    P, ld = int(type_.shape[0]), int(type_.shape[1])
    L = ld if max_len is None else int(max_len)
    return P, L, ld


def _x_args(X, x_layout):
    import torch

    lay = X_SOA if x_layout in ("soa", X_SOA) else X_ROWMAJOR
    if not X.is_cuda or not X.is_contiguous() or X.dtype != torch.float32 or X.dim() != 2:
        raise ValueError("X must be a contiguous 2-D float32 CUDA tensor")
    if lay == X_ROWMAJOR:
        D, n_in = int(X.shape[0]), int(X.shape[1])
    else:
        n_in, D = int(X.shape[0]), int(X.shape[1])
    return lay, D, n_in


def _check_out(out, shape, dtype, device):
    if out.dtype != dtype or not out.is_cuda or not out.is_contiguous() or out.device != device \
            or out.numel() != math.prod(shape):
        raise ValueError(f"out must be a contiguous {dtype} CUDA tensor of {math.prod(shape)} elements on {device}")


def eval(type_, value, size, X, n_outputs: int = 1, strategy="auto", x_layout="rowmajor", max_len=None,
         out=None, workspace: Workspace | None = None, stream=None):
    """Device: out[P, D, n_outputs] float32 (Modi P:391-411)."""
    import torch

    P, L, ld = _tree_args(type_, value, size, max_len)
    lay, D, n_in = _x_args(X, x_layout)
    if out is None:
        out = torch.empty((P, D, n_outputs), dtype=torch.float32, device=X.device)
    _check_out(out, (P, D, n_outputs), torch.float32, X.device)
    with _device_guard(X.device):
        ws = _workspace(P, D, L, n_in, n_outputs, X.device, workspace, stream)
        st = _LIB.evogp_eval(_vp(type_), _vp(value), _vp(size), P, L, ld, _vp(X), D, n_in, lay, n_outputs,
                             _vp(out), STRATEGIES[strategy], ctypes.c_void_p(ws.ptr), ws.nbytes,
                             _stream_ptr(stream, X.device))
    if st != OK:
        raise EvogpError(st, "evogp_eval")
    return out


def _sr(fn, name, type_, value, size, X, y, strategy, x_layout, max_len, out, workspace, stream):
    import torch

    P, L, ld = _tree_args(type_, value, size, max_len)
    lay, D, n_in = _x_args(X, x_layout)
    if not y.is_cuda or y.dtype != torch.float32 or y.numel() != D:
        raise ValueError("y must be a float32 CUDA tensor of length D")
    if out is None:
        out = torch.empty(P, dtype=torch.float64, device=X.device)
    _check_out(out, (P,), torch.float64, X.device)
    with _device_guard(X.device):
        ws = _workspace(P, D, L, n_in, 1, X.device, workspace, stream)
        st = fn(_vp(type_), _vp(value), _vp(size), P, L, ld, _vp(X), D, n_in, lay, _vp(y), _vp(out),
                STRATEGIES[strategy], ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream, X.device))
    if st != OK:
        raise EvogpError(st, name)
    return out


def sr_fitness(type_, value, size, X, y, strategy="auto", x_layout="rowmajor", max_len=None, out=None,
               workspace: Workspace | None = None, stream=None):
    """Device: fused SR fitness mse[P] float64."""
    return _sr(_LIB.evogp_sr_fitness, "evogp_sr_fitness", type_, value, size, X, y, strategy, x_layout, max_len,
               out, workspace, stream)


def sr_sse(type_, value, size, X, y, strategy="auto", x_layout="rowmajor", max_len=None, out=None,
           workspace: Workspace | None = None, stream=None):
    """Device: un-normalised sse[P] float64 for datapoint sharding."""
    return _sr(_LIB.evogp_sr_sse, "evogp_sr_sse", type_, value, size, X, y, strategy, x_layout, max_len, out,
               workspace, stream)


def classification_accuracy(type_, value, size, X, labels, n_classes: int, strategy="auto", x_layout="rowmajor",
                            max_len=None, out=None, workspace: Workspace | None = None, stream=None):
    """Device: fused classification fitness accuracy[P] float64 (SURVEY §8(f)
    NEXT-1): Modi trees with one output per class, argmax per
    datapoint (ties -> lowest class, NaN as -inf) against int32 labels[D]."""
    import torch

    P, L, ld = _tree_args(type_, value, size, max_len)
    lay, D, n_in = _x_args(X, x_layout)
    if not labels.is_cuda or labels.dtype != torch.int32 or labels.numel() != D:
        raise ValueError("labels must be an int32 CUDA tensor of length D")
    if out is None:
        out = torch.empty(P, dtype=torch.float64, device=X.device)
    _check_out(out, (P,), torch.float64, X.device)
    with _device_guard(X.device):
        ws = _workspace(P, D, L, n_in, n_classes, X.device, workspace, stream)
        st = _LIB.evogp_classification_accuracy(_vp(type_), _vp(value), _vp(size), P, L, ld, _vp(X), D, n_in, lay,
                                                n_classes, _vp(labels), _vp(out), STRATEGIES[strategy],
                                                ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream, X.device))
    if st != OK:
        raise EvogpError(st, "evogp_classification_accuracy")
    return out


def eval_paired(type_, value, size, obs, n_outputs: int = 1, max_len=None, out=None,
                workspace: Workspace | None = None, stream=None):
    """Device: paired per-individual inference (PAPER
    P:346): tree p evaluated on its own observations obs[p] ([P, n_in] or
    [P, B, n_in] float32) -> out [P, n_outputs] or [P, B, n_outputs]."""
    import torch

    P, L, ld = _tree_args(type_, value, size, max_len)
    if not obs.is_cuda or obs.dtype != torch.float32 or not obs.is_contiguous() or obs.dim() not in (2, 3):
        raise ValueError("obs must be a contiguous float32 CUDA tensor [P, n_in] or [P, B, n_in]")
    if obs.shape[0] != P:
        raise ValueError("obs.shape[0] must equal the population size")
    B = 1 if obs.dim() == 2 else int(obs.shape[1])
    n_in = int(obs.shape[-1])
    shape = (P, n_outputs) if obs.dim() == 2 else (P, B, n_outputs)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=obs.device)
    _check_out(out, shape, torch.float32, obs.device)
    with _device_guard(obs.device):
        ws = workspace if workspace is not None else _flags_workspace(obs.device)
        st = _LIB.evogp_eval_paired(_vp(type_), _vp(value), _vp(size), P, L, ld, _vp(obs), B, n_in, n_outputs,
                                    _vp(out), ctypes.c_void_p(ws.ptr), ws.nbytes, _stream_ptr(stream, obs.device))
    if st != OK:
        raise EvogpError(st, "evogp_eval_paired")
    return out


def _flags_workspace(device):
    key = ("flags", str(device))
    w = _WS_CACHE.get(key)
    if w is None:
        w = Workspace(1, 1, 1, 1, 1, device)
        _WS_CACHE[key] = w
    return w


def select_strategy(P: int, D: int, max_len: int, n_outputs: int = 1, device: int = 0) -> str:
    s = _LIB.evogp_select_strategy(P, D, max_len, n_outputs, device)
    if s < 0:
        raise EvogpError(s, "evogp_select_strategy")
    return "inter" if s == STRATEGY_INTER else "intra"


def check_device_flags(workspace: Workspace, stream=None) -> int:
    flags = np.zeros(1, dtype=np.int32)
    st = _LIB.evogp_check_device_flags(ctypes.c_void_p(workspace.ptr), _stream_ptr(stream, workspace.buf.device),
                                       _vp(flags))
    if st != OK:
        raise EvogpError(st, "evogp_check_device_flags")
    return int(flags[0])


def set_tuning(target_warps: int = 0, no_reorder: bool = False, no_fuse: bool = False, K: int = 0,
               reorder_above: int = 0, unit_chunks: int = 0, full_set: bool = False,
               fused_compile: bool = False) -> None:
    """evogp_set_tuning for this thread (calibration sweeps, tests); all
    defaults = the library's own plan. Results never depend on it."""
    t = _lib.Tuning(int(target_warps), int(bool(no_reorder)), int(bool(no_fuse)), int(K), int(reorder_above),
                    int(unit_chunks), int(bool(full_set)), int(bool(fused_compile)))
    st = _LIB.evogp_set_tuning(ctypes.byref(t))
    if st != OK:
        raise EvogpError(st, "evogp_set_tuning")
    _TUNING.kw = dict(target_warps=target_warps, no_reorder=no_reorder, no_fuse=no_fuse, K=K,
                      reorder_above=reorder_above, unit_chunks=unit_chunks, full_set=full_set,
                      fused_compile=fused_compile)


_TUNING = threading.local()


@contextlib.contextmanager
def tuning_hint(**kw):
    """The thread's current tuning with ``kw`` overriding it for the body of a
    with-block, then restored (e.g. ``full_set=True`` around calls on a
    population drawn from the full function set)."""
    prev = dict(getattr(_TUNING, "kw", {}))
    set_tuning(**{**prev, **kw})
    try:
        yield
    finally:
        set_tuning(**prev)


def last_launch_count() -> int:
    return int(_LIB.evogp_last_launch_count())


def set_kernel_timing(start_event=None, end_event=None) -> None:
    """Bracket the dominant kernel of subsequent device calls (this thread)
    with two torch.cuda.Event(enable_timing=True) events; None disables."""
    a = ctypes.c_void_p(start_event.cuda_event) if start_event is not None else ctypes.c_void_p(0)
    b = ctypes.c_void_p(end_event.cuda_event) if end_event is not None else ctypes.c_void_p(0)
    st = _LIB.evogp_set_kernel_timing(a, b)
    if st != OK:
        raise EvogpError(st, "evogp_set_kernel_timing")


from .gp import Evolution, GPConfig, generate, reproduce, subtree_exchange, tournament  # noqa: E402
