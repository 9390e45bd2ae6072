"""C-ABI library on the CPU host (no GPU): it loads, exports every symbol
include/evogp.h declares, and its host tensorizer matches the oracle's
independent tensorizer byte for byte (PAPER §III-A)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2501_17168_b200 as evogp
import synth
from paper_2501_17168_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "evogp.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(evogp_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    decl = _declared_symbols()
    assert len(decl) >= 10
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_lib.EXPORTS)


def test_status_strings():
    for st in range(0, -9, -1):
        s = evogp._LIB.evogp_status_string(st).decode()
        assert s and s != "unknown status"


def _bytes_equal(a, b):
    return a.tobytes() == b.tobytes()


@pytest.mark.parametrize("mix,L,n_in,n_out,modi", [
    ("paper", 63, 4, 1, 0.0), ("full", 127, 8, 1, 0.0), ("full", 63, 17, 6, 0.1), ("ieee", 15, 2, 1, 0.0)])
def test_tensorize_bitexact_vs_oracle(mix, L, n_in, n_out, modi):
    pt = synth.trees(42, 0, 10_000, L, synth.MIXES[mix], n_in, n_out, modi)
    a = evogp.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
    b = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert _bytes_equal(x, y)  # padding bytes included (reading R1)
    # invariants: size[0] = len, size[i] = 1 + sum of children
    lens = np.diff(pt.offsets)
    assert (a[2][:, 0] == lens).all()


def _mutate(rng, types, values, n_in, n_out):
    t = types.copy()
    v = values.copy()
    i = int(rng.integers(len(t)))
    choice = int(rng.integers(8))
    if choice == 0:
        t[i] = np.int16(-1)
    elif choice == 1:
        t[i] = np.int16(1)
        v[i] = n_in + rng.integers(3)
    elif choice == 2:
        t[i] = np.int16(2)
        v[i] = 99
    elif choice == 3:
        t[i] = np.int16(3)
        v[i] = 4  # SIN tagged binary
    elif choice == 4:
        t[i] = np.int16(t[i] | 8 | (int(rng.integers(0, 8)) << 8))
    elif choice == 5:
        t[i] = np.int16(0)
    elif choice == 6:
        v[i] = 2.5
        t[i] = np.int16(2)
    else:
        t[i] = np.int16(t[i] | 0x40)
    return t, v


def test_tensorize_errors_match_oracle():
    rng = np.random.default_rng(1)
    n_in, n_out, L = 3, 4, 31
    base = synth.trees(3, 0, 400, L, synth.M_FULL, n_in, n_out, 0.1)
    for it in range(400):
        ty, va = base.tree(it)
        ty, va = _mutate(rng, ty, va, n_in, n_out)
        off = np.array([0, len(ty)], np.int64)
        ref = oracle.tensorize(off, ty, va, L, n_in, n_out, raise_on_error=False)
        try:
            evogp.tensorize(off, ty, va, L, n_in, n_out)
            got = (0, -1, -1)
        except evogp.EvogpError as e:
            got = (e.status, e.tree, e.node)
        assert got == tuple(ref[:3]), (it, got, ref[:3])


def test_tensorize_error_lowest_tree():
    pt = synth.trees(4, 0, 50_000, 31, synth.M_PAPER, 2)
    types = pt.types.copy()
    for p in (40_000, 12_345):
        b, e = pt.offsets[p], pt.offsets[p + 1]
        types[b] = 1  # root becomes VAR -> leftover operands
    with pytest.raises(evogp.EvogpError) as ei:
        evogp.tensorize(pt.offsets, types, pt.values, 31, 2)
    ref = oracle.tensorize(pt.offsets, types, pt.values, 31, 2, raise_on_error=False)
    assert (ei.value.status, ei.value.tree, ei.value.node) == tuple(ref[:3])
    assert ei.value.tree == 12_345


def test_too_large_and_empty():
    with pytest.raises(evogp.EvogpError) as ei:
        evogp.tensorize(np.array([0, 5]), np.zeros(5, np.int16), np.zeros(5, np.float32), 4, 1)
    assert ei.value.status == evogp.E_TOO_LARGE
    with pytest.raises(evogp.EvogpError) as ei:
        evogp.tensorize(np.array([0, 0]), np.zeros(0, np.int16), np.zeros(0, np.float32), 4, 1)
    assert ei.value.status == evogp.E_ARG
    t, v, s = evogp.tensorize(np.array([0]), np.zeros(0, np.int16), np.zeros(0, np.float32), 4, 1)
    assert t.shape == (0, 4)


def test_workspace_and_selector_host():
    assert evogp.workspace_size(10_000, 1024, 63, 4, 1) > 4 * 1024 * 4
    assert evogp.workspace_size(1000, 1 << 20, 127, 8, 1) >= 8 * (1 << 20) * 4
    # the measured table (selector_table.json, profiles/selector_calibration_r02d.log):
    # cells whose faster kernel wins by >= 30% on both calibration passes
    assert evogp.select_strategy(10_000, 1024, 63) == "inter"
    assert evogp.select_strategy(1_000_000, 256, 127) == "inter"
    assert evogp.select_strategy(1000, 65536, 512) == "intra"
    assert evogp.select_strategy(10_000, 4096, 512) == "intra"


def test_gp_config_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of evogp_gp_config (paper_2501_17168_b200/gp.py) has
    the C header's size and field offsets (compiled with gcc from include/)."""
    from paper_2501_17168_b200.gp import _CCfg

    fields = [f for f, _ in _CCfg._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"evogp.h\"\nint main(void){\n"
                   "printf(\"%zu\\n\", sizeof(evogp_gp_config));\n" +
                   "".join(f"printf(\"%zu\\n\", offsetof(evogp_gp_config, {f}));\n" for f in fields) +
                   "return 0;}\n")
    exe = tmp_path / "layout"
    import subprocess
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    out = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert out[0] == ctypes.sizeof(_CCfg)
    assert out[1:] == [getattr(_CCfg, f).offset for f in fields]


def test_gp_config_defaults_follow_tab_sr_params():
    """tab:sr_params: tournament 20, p_c 0.9, p_m 0.1, max size 512, {+,-,x,/,sin,cos,tan}."""
    from paper_2501_17168_b200.gp import GPConfig

    c = GPConfig()
    assert (c.tournament_size, c.p_crossover, c.p_mutation, c.max_len) == (20, 0.9, 0.1, 512)
    assert c.c().func_mask == sum(1 << f for f in (0, 1, 2, 3, 4, 5, 6))


@pytest.mark.parametrize("field,value", [
    ("p_crossover", 1.5), ("p_mutation", -0.1), ("func_mask", 0), ("func_mask", 1 << 22), ("depth_min", 0),
    ("depth_max", 1), ("max_len", 9000), ("n_outputs", 0), ("tournament_size", 0), ("crossover_kind", 7),
    ("const_lo", float("nan")), ("subtree_depth", 0),
])
def test_gp_config_validation_host(field, value):
    """Host-side validation of evogp_gp_config happens before any launch, so
    it is checkable without a GPU: every bad field is E_ARG (include/evogp.h)."""
    from paper_2501_17168_b200.gp import GPConfig

    c = GPConfig(max_len=63, n_inputs=4, depth_min=2, depth_max=6).c()
    setattr(c, field, value)
    lib = _lib.load()
    null = ctypes.c_void_p(0)
    st = lib.evogp_reproduce(null, null, null, 10, 63, null, 10, 0, ctypes.byref(c), 1, null, null, null, null,
                             null, null)
    assert st == _lib.E_ARG
    if field not in ("tournament_size", "crossover_kind"):  # generation ignores the variation fields
        assert lib.evogp_generate(10, ctypes.byref(c), 1, null, null, null, null) == _lib.E_ARG


def test_gp_config_zero_weights_rejected_only_with_mutation():
    from paper_2501_17168_b200.gp import GPConfig

    lib = _lib.load()
    null = ctypes.c_void_p(0)
    c = GPConfig(max_len=63, n_inputs=4, mutation_weights=(0,) * 8, p_mutation=0.1).c()
    assert lib.evogp_reproduce(null, null, null, 10, 63, null, 10, 0, ctypes.byref(c), 1, null, null, null, null,
                               null, null) == _lib.E_ARG


def test_tuning_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of evogp_tuning (_lib.Tuning) has the C header's size
    and field offsets (compiled with gcc from include/)."""
    fields = [f for f, _ in _lib.Tuning._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"evogp.h\"\nint main(void){\n"
                   "printf(\"%zu\\n\", sizeof(evogp_tuning));\n" +
                   "".join(f"printf(\"%zu\\n\", offsetof(evogp_tuning, {f}));\n" for f in fields) +
                   "return 0;}\n")
    exe = tmp_path / "layout"
    import subprocess
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    out = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert out[0] == ctypes.sizeof(_lib.Tuning)
    assert out[1:] == [getattr(_lib.Tuning, f).offset for f in fields]


def test_tuning_hint_nests_and_restores():
    """tuning_hint overrides fields for a with-block on top of the thread's
    tuning and restores it; the plan sees it (fused_compile never enlarges
    the workspace: kernel (a)'s plans drop their program-row section)."""
    args = (100_000, 256, 127, 8, 1)
    evogp.set_tuning()
    base = evogp.workspace_size(*args)
    try:
        evogp.set_tuning(unit_chunks=2)
        with evogp.tuning_hint(fused_compile=True):
            assert evogp._TUNING.kw["unit_chunks"] == 2 and evogp._TUNING.kw["fused_compile"]
            fused = evogp.workspace_size(*args)
            with evogp.tuning_hint(full_set=True):
                assert evogp._TUNING.kw["fused_compile"] and evogp._TUNING.kw["full_set"]
            assert not evogp._TUNING.kw["full_set"]
        assert evogp._TUNING.kw == dict(target_warps=0, no_reorder=False, no_fuse=False, K=0, reorder_above=0,
                                        unit_chunks=2, full_set=False, fused_compile=False)
        assert fused <= base
    finally:
        evogp.set_tuning()
    assert evogp.workspace_size(*args) == base
