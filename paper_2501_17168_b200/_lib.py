"""ctypes loader for libevogp.so (the C-ABI of include/evogp.h).

Argument marshalling only. There is no fallback: if the shared library is
missing, importing the package raises (build it with
``python -c "import __graft_entry__ as g; g.build()"`` or ``make``).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libevogp.so")

OK = 0
E_ARG, E_TOO_LARGE, E_MALFORMED, E_VAR_RANGE, E_FUNC_UNKNOWN, E_OUT_RANGE, E_CUDA, E_UNSUPPORTED = (
    -1, -2, -3, -4, -5, -6, -7, -8)
STRATEGY_AUTO, STRATEGY_INTER, STRATEGY_INTRA = 0, 1, 2
X_ROWMAJOR, X_SOA = 0, 1

# every symbol include/evogp.h declares
EXPORTS = (
    "evogp_tensorize", "evogp_workspace_size", "evogp_eval", "evogp_sr_fitness", "evogp_sr_sse",
    "evogp_select_strategy", "evogp_check_device_flags", "evogp_status_string", "evogp_last_error",
    "evogp_last_launch_count", "evogp_set_kernel_timing", "evogp_classification_accuracy",
    "evogp_eval_paired", "evogp_generate", "evogp_subtree_exchange", "evogp_tournament", "evogp_reproduce",
    "evogp_tensorize_device", "evogp_set_tuning",
)


def load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: the CUDA library must be built (make, or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
    lib.evogp_tensorize.argtypes = [i64, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp]
    lib.evogp_tensorize.restype = ctypes.c_int
    lib.evogp_tensorize_device.argtypes = [i64, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp]
    lib.evogp_tensorize_device.restype = ctypes.c_int
    lib.evogp_workspace_size.argtypes = [i64, i64, i32, i32, i32]
    lib.evogp_workspace_size.restype = sz
    dev_args = [vp, vp, vp, i64, i32, i32, vp, i64, i32, i32]
    lib.evogp_eval.argtypes = dev_args + [i32, vp, i32, vp, sz, vp]
    lib.evogp_eval.restype = ctypes.c_int
    lib.evogp_sr_fitness.argtypes = dev_args + [vp, vp, i32, vp, sz, vp]
    lib.evogp_sr_fitness.restype = ctypes.c_int
    lib.evogp_sr_sse.argtypes = dev_args + [vp, vp, i32, vp, sz, vp]
    lib.evogp_sr_sse.restype = ctypes.c_int
    lib.evogp_classification_accuracy.argtypes = dev_args + [i32, vp, vp, i32, vp, sz, vp]
    lib.evogp_classification_accuracy.restype = ctypes.c_int
    lib.evogp_eval_paired.argtypes = [vp, vp, vp, i64, i32, i32, vp, i32, i32, i32, vp, vp, sz, vp]
    lib.evogp_eval_paired.restype = ctypes.c_int
    u64 = ctypes.c_uint64
    lib.evogp_generate.argtypes = [i64, vp, u64, vp, vp, vp, vp]
    lib.evogp_generate.restype = ctypes.c_int
    lib.evogp_subtree_exchange.argtypes = [i64, vp, vp, vp, i32, vp, vp, vp, vp, vp, i32, vp, vp, i32, vp, vp, vp,
                                           vp, vp]
    lib.evogp_subtree_exchange.restype = ctypes.c_int
    lib.evogp_tournament.argtypes = [vp, i64, i32, i64, u64, i32, vp, vp]
    lib.evogp_tournament.restype = ctypes.c_int
    lib.evogp_reproduce.argtypes = [vp, vp, vp, i64, i32, vp, i64, i64, vp, u64, vp, vp, vp, vp, vp, vp]
    lib.evogp_reproduce.restype = ctypes.c_int
    lib.evogp_select_strategy.argtypes = [i64, i64, i32, i32, i32]
    lib.evogp_select_strategy.restype = ctypes.c_int
    lib.evogp_check_device_flags.argtypes = [vp, vp, vp]
    lib.evogp_check_device_flags.restype = ctypes.c_int
    lib.evogp_status_string.argtypes = [ctypes.c_int]
    lib.evogp_status_string.restype = ctypes.c_char_p
    lib.evogp_last_error.argtypes = []
    lib.evogp_last_error.restype = ctypes.c_char_p
    lib.evogp_last_launch_count.argtypes = []
    lib.evogp_last_launch_count.restype = ctypes.c_int32
    lib.evogp_set_kernel_timing.argtypes = [vp, vp]
    lib.evogp_set_kernel_timing.restype = ctypes.c_int
    lib.evogp_set_tuning.argtypes = [vp]
    lib.evogp_set_tuning.restype = ctypes.c_int
    return lib


class Tuning(ctypes.Structure):
    """evogp_tuning (include/evogp.h): launch-plan overrides, 0 = default."""
    _fields_ = [("target_warps", ctypes.c_int32), ("no_reorder", ctypes.c_int32), ("no_fuse", ctypes.c_int32),
                ("K", ctypes.c_int32), ("reorder_above", ctypes.c_int32),
                ("unit_chunks", ctypes.c_int32), ("full_set", ctypes.c_int32),
                ("fused_compile", ctypes.c_int32)]
