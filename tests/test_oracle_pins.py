"""Pins for the oracle against things other than itself (no GPU).

Each test names the passage or mathematical fact it pins:
  * golden fixtures in tests/golden (paper-printed values, SPEC examples, closed forms)
  * invariants of the prefix/size encoding
  * brute force over every prefix sequence of length <= 5 on a small alphabet,
    checked against an independent recursive-descent definition of
    well-formedness and an independent recursive interpreter
  * FP32-faithful mode vs numpy float32 IEEE arithmetic on the IEEE-exact ops
  * certificate soundness: a genuine FP32 evaluation lies inside the bound
  * MSE closed forms (Var(y) + (c - ybar)^2)
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import GOLDEN

CONST, VAR, UF, BF, TF = 0, 1, 2, 3, 4
ARITY = {0: 2, 1: 2, 2: 2, 3: 2, 4: 1, 5: 1, 6: 1, 7: 2, 8: 2, 9: 2, 10: 1, 11: 1, 12: 1, 13: 1, 14: 1,
         15: 1, 16: 1, 17: 2, 18: 2, 19: 2, 20: 2, 21: 3}


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _fval(v):
    if isinstance(v, str):
        return float(v)
    return float(v)


def _single(types, values, L=None, n_in=2, n_out=1):
    L = L or len(types)
    off = np.array([0, len(types)], dtype=np.int64)
    return oracle.tensorize(off, np.array(types, np.int16), np.array(values, np.float32), L, n_in, n_out)


# ---------------------------------------------------------------- tensorize
def test_encoding_examples_spec():
    g = _load("encoding_examples.json")
    for c in g["cases"]:
        L = len(c["types"]) + 3
        t, v, s = _single(c["types"], c["values"], L=L, n_in=c["n_inputs"])
        assert list(t[0, : len(c["types"])]) == c["types"], c["name"]
        assert list(s[0, : len(c["types"])]) == c["sizes"], c["name"]
        np.testing.assert_array_equal(v[0, : len(c["types"])], np.array(c["values"], np.float32))
        # padding (reading R1): type -1, value qNaN 0x7FC00000, size 0
        assert (t[0, len(c["types"]):] == -1).all()
        assert (s[0, len(c["types"]):] == 0).all()
        assert (v[0, len(c["types"]):].view(np.uint32) == 0x7FC00000).all()


def test_fig6_sizes():
    g = _load("fig6_modi_tree.json")
    t, v, s = _single(g["types"], g["values"], n_in=g["n_inputs"], n_out=g["n_outputs"])
    assert list(s[0]) == g["sizes"]


def test_tensorize_errors():
    L = 8
    # too large (TooLarge)
    st = oracle.tensorize(np.array([0, 9]), np.zeros(9, np.int16), np.zeros(9, np.float32), L, 1, 1,
                          raise_on_error=False)
    assert st[0] == oracle.E_TOO_LARGE
    # variable index out of range
    st = oracle.tensorize(np.array([0, 1]), np.array([VAR], np.int16), np.array([2], np.float32), L, 2, 1,
                          raise_on_error=False)
    assert st[0] == oracle.E_VAR_RANGE
    # unknown function id
    st = oracle.tensorize(np.array([0, 2]), np.array([UF, VAR], np.int16), np.array([99, 0], np.float32), L, 1, 1,
                          raise_on_error=False)
    assert st[0] == oracle.E_FUNC_UNKNOWN
    # arity mismatch: SIN tagged as BFUNC
    st = oracle.tensorize(np.array([0, 3]), np.array([BF, VAR, VAR], np.int16), np.array([4, 0, 0], np.float32),
                          L, 1, 1, raise_on_error=False)
    assert st[0] == oracle.E_MALFORMED
    # Modi with a single output
    st = oracle.tensorize(np.array([0, 2]), np.array([UF | 8, VAR], np.int16), np.array([4, 0], np.float32),
                          L, 1, 1, raise_on_error=False)
    assert st[0] == oracle.E_OUT_RANGE
    # Modi slot >= n_out
    st = oracle.tensorize(np.array([0, 2]), np.array([UF | 8 | (3 << 8), VAR], np.int16),
                          np.array([4, 0], np.float32), L, 1, 3, raise_on_error=False)
    assert st[0] == oracle.E_OUT_RANGE
    # leftover operands: two leaves, no function
    st = oracle.tensorize(np.array([0, 2]), np.array([VAR, VAR], np.int16), np.array([0, 0], np.float32), L, 1, 1,
                          raise_on_error=False)
    assert st[0] == oracle.E_MALFORMED
    # error reporting order: lowest tree first
    off = np.array([0, 1, 2, 3])
    st = oracle.tensorize(off, np.array([VAR, VAR, VAR], np.int16), np.array([0, 5, 7], np.float32), L, 2, 1,
                          raise_on_error=False)
    assert st == (oracle.E_VAR_RANGE, 1, 0)


# ---- brute force: alphabet {ADD,SUB,MUL,DIV,SIN,NEG,IF} x leaves {x0,x1,0.5,-2}
ALPHA = [(BF, 0), (BF, 1), (BF, 2), (BF, 3), (UF, 4), (UF, 13), (TF, 21),
         (VAR, 0), (VAR, 1), (CONST, 0.5), (CONST, -2.0)]


def _arity_sym(sym):
    k, v = sym
    return 0 if k in (CONST, VAR) else ARITY[int(v)]


def _parse(seq, i=0):
    """Recursive-descent definition of a well-formed prefix tree (§III-A):
    returns (end, sizes) or None."""
    if i >= len(seq):
        return None
    a = _arity_sym(seq[i])
    j = i + 1
    sizes = {}
    for _ in range(a):
        r = _parse(seq, j)
        if r is None:
            return None
        j2, sz = r
        sizes.update(sz)
        j = j2
    sizes[i] = j - i
    return j, sizes


def _brute_sequences(maxlen=5):
    for n in range(1, maxlen + 1):
        for seq in itertools.product(ALPHA, repeat=n):
            yield seq


def test_bruteforce_tensorize_accepts_exactly_wellformed():
    good = []
    n_checked = 0
    for seq in _brute_sequences(5):
        n_checked += 1
        r = _parse(seq)
        wf = r is not None and r[0] == len(seq)
        ty = np.array([k for k, _ in seq], np.int16)
        va = np.array([v for _, v in seq], np.float32)
        res = oracle.tensorize(np.array([0, len(seq)]), ty, va, 5, 2, 1, raise_on_error=False)
        assert (res[0] == oracle.OK) == wf, seq
        if wf:
            s = res[5][0]
            assert [int(s[i]) for i in range(len(seq))] == [r[1][i] for i in range(len(seq))]
            good.append(seq)
    assert n_checked == sum(11 ** n for n in range(1, 6))
    assert len(good) > 1000


def test_bruteforce_stack_equals_recursive_fp64():
    """Stack machine == recursive bottom-up, bit-exact in FP64
    and in FP32-faithful mode, on a 3x3 grid."""
    seqs = []
    for seq in _brute_sequences(5):
        r = _parse(seq)
        if r is not None and r[0] == len(seq):
            seqs.append(seq)
    rng = np.random.default_rng(0)
    sel = [seqs[i] for i in rng.choice(len(seqs), size=min(4000, len(seqs)), replace=False)]
    off = np.zeros(len(sel) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in sel])
    ty = np.array([k for s in sel for k, _ in s], np.int16)
    va = np.array([v for s in sel for _, v in s], np.float32)
    t, v, sz = oracle.tensorize(off, ty, va, 5, 2, 1)
    grid = np.array([[a, b] for a in (-1.5, 0.0, 0.7) for b in (-0.3, 0.0, 2.0)], np.float32)
    for mode in (0, 1):
        out = oracle.evaluate(t, v, sz, grid, mode=mode)
        for i in range(0, len(sel), 7):
            s = sel[i]
            for d in range(len(grid)):
                r = oracle.evaluate_recursive(ty[off[i]:off[i + 1]], va[off[i]:off[i + 1]], grid[d], mode=mode)
                a, b = out[i, d, 0], r[0]
                assert (np.isnan(a) and np.isnan(b)) or a == b, (s, grid[d], a, b)


# ---------------------------------------------------------------- eval pins
def test_fig6_modi_outputs():
    g = _load("fig6_modi_tree.json")
    t, v, s = _single(g["types"], g["values"], n_in=g["n_inputs"], n_out=g["n_outputs"])
    x = np.array([[g["inputs"][k] for k in "abcde"]], np.float32)
    for mode in (0, 1):
        out = oracle.evaluate(t, v, s, x, n_out=3, mode=mode)[0, 0]
        tol = 1e-15 if mode == 0 else 1e-7
        np.testing.assert_allclose(out, g["expected_outputs"], rtol=tol)
    rec = oracle.evaluate_recursive(np.array(g["types"], np.int16), np.array(g["values"], np.float32), x[0], n_out=3)
    np.testing.assert_allclose(rec, g["expected_outputs"], rtol=1e-15)


def test_multi_output_zero_law():
    """No Modi node and m > 1 -> all-zero outputs (reading R4)."""
    t, v, s = _single([BF, VAR, CONST], [0, 0, 1.0], n_in=1, n_out=3)
    out = oracle.evaluate(t, v, s, np.array([[2.0]], np.float32), n_out=3)
    assert (out == 0).all()


def test_closed_forms():
    g = _load("closed_forms.json")
    for c in g["cases"]:
        n_in = max(2, len(c["x"]))
        t, v, s = _single(c["types"], c["values"], n_in=n_in)
        x = np.zeros((1, n_in), np.float32)
        x[0, : len(c["x"])] = c["x"]
        out = oracle.evaluate(t, v, s, x)[0, 0, 0]
        assert out == pytest.approx(c["expected"], rel=1e-12, abs=1e-15), c["name"]


def test_protected_edge_cases():
    g = _load("protected_ops.json")
    for c in g["cases"]:
        a = len(c["args"])
        kind = {1: UF, 2: BF, 3: TF}[a]
        types = [kind] + [CONST] * a
        values = [c["id"]] + [_fval(x) for x in c["args"]]
        t, v, s = _single(types, values, n_in=1)
        for mode in (0, 1):
            out = oracle.evaluate(t, v, s, np.zeros((1, 1), np.float32), mode=mode)[0, 0, 0]
            exp = _fval(c["expected"])
            if math.isnan(exp):
                assert math.isnan(out), c
            elif math.isinf(exp):
                assert out == exp, c
            else:
                tol = c.get("tol", 0.0) if mode == 0 else 1e-7
                if c["f"] == "EXP" and mode == 1:  # FP32 rounding of e^88
                    tol = 1e-7
                assert out == pytest.approx(exp, rel=tol, abs=tol), (c, mode)


def test_fp32_range_emulation():
    """Reading R5: EXP(100) overflows FP32 -> +inf even in FP64 mode;
    MUL(1e30,1e30) too; EXP(88) stays finite."""
    for types, values, exp in [([UF, CONST], [11, 100.0], math.inf),
                               ([BF, CONST, CONST], [2, 1e30, -1e30], -math.inf),
                               ([UF, CONST], [11, 88.0], math.exp(88.0))]:
        t, v, s = _single(types, values, n_in=1)
        out = oracle.evaluate(t, v, s, np.zeros((1, 1), np.float32))[0, 0, 0]
        assert out == pytest.approx(exp, rel=1e-15)


def _np32_eval(types, values, x):
    """Independent numpy-float32 recursive evaluator for the IEEE-exact ops."""
    f32 = np.float32
    dl = f32(0.001)

    def rec(i):
        k = types[i]
        if k == CONST:
            return f32(values[i]), i + 1
        if k == VAR:
            return f32(x[int(values[i])]), i + 1
        f = int(values[i])
        args = []
        j = i + 1
        for _ in range(ARITY[f]):
            a, j = rec(j)
            args.append(a)
        a = args
        with np.errstate(all="ignore"):
            if f == 0: r = a[0] + a[1]
            elif f == 1: r = a[0] - a[1]
            elif f == 2: r = a[0] * a[1]
            elif f == 3: r = a[0] / a[1] if abs(a[1]) > dl else f32(1)
            elif f == 7: r = np.fmax(a[0], a[1])
            elif f == 8: r = np.fmin(a[0], a[1])
            elif f == 13: r = -a[0]
            elif f == 14: r = abs(a[0])
            elif f == 15: r = np.sqrt(abs(a[0]))
            elif f == 17: r = f32(1) if a[0] < a[1] else f32(0)
            elif f == 18: r = f32(1) if a[0] > a[1] else f32(0)
            elif f == 19: r = f32(1) if a[0] <= a[1] else f32(0)
            elif f == 20: r = f32(1) if a[0] >= a[1] else f32(0)
            elif f == 21: r = a[1] if a[0] > 0 else a[2]
            else: raise AssertionError(f)
        return f32(r), j

    return rec(0)[0]


def test_fp32_faithful_equals_numpy_float32_ieee_mix():
    pt = synth.trees(7, 0, 150, 31, synth.M_IEEE, 3)
    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, 31, 3)
    X = synth.dataset_X(7, 0, 16, 3, lo=-3, hi=3)
    out = oracle.evaluate(t, v, s, X, mode=1)
    for i in range(pt.n):
        ty, va = pt.tree(i)
        for d in range(X.shape[0]):
            ref = _np32_eval(list(ty), list(va), X[d])
            got = out[i, d, 0]
            assert (np.isnan(ref) and np.isnan(got)) or float(ref) == got, (i, d, ref, got)


@pytest.mark.parametrize("mix", ["ieee", "bounded", "paper", "full"])
def test_certificate_sound(mix):
    """Where the certificate says robust, the FP32-faithful evaluation (a real
    FP32 computation, <= 0.5 ulp per op) lies within the bound e."""
    pt = synth.trees(11, 0, 300, 63, synth.MIXES[mix], 4)
    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, 63, 4)
    X = synth.dataset_X(11, 0, 64, 4)
    v64, e, rob = oracle.evaluate(t, v, s, X, mode=0, certify=True)
    v32 = oracle.evaluate(t, v, s, X, mode=1)
    fin = np.isfinite(v64) & np.isfinite(e) & rob
    with np.errstate(invalid="ignore"):
        bad = fin & ~(np.abs(v32 - v64) <= e)
    assert bad.sum() == 0, (mix, np.argwhere(bad)[:5])
    # the certificate is not vacuous on bounded mixes
    cert = oracle.certified_points(v64, e, rob)
    if mix in ("ieee", "bounded"):
        assert cert.mean() > 0.5


def test_certificate_flags_fragile_decisions():
    # LT(x0, x0 + 1e-9) has a zero-margin decision in FP32 -> not robust
    t, v, s = _single([BF, VAR, BF, VAR, CONST], [17, 0, 0, 0, 1e-9], n_in=1)
    _, e, rob = oracle.evaluate(t, v, s, np.array([[0.5]], np.float32), certify=True)
    assert not rob[0, 0, 0]
    # DIV with |b| exactly at delta -> not robust
    t, v, s = _single([BF, CONST, CONST], [3, 1.0, 0.001], n_in=1)
    _, e, rob = oracle.evaluate(t, v, s, np.array([[0.5]], np.float32), certify=True)
    assert not rob[0, 0, 0]


# ---------------------------------------------------------------- MSE pins
def test_mse_spec_example():
    """predictions [0,0] vs targets [1,3] -> 5.0."""
    assert oracle.mse(np.array([[0.0, 0.0]]), np.array([1.0, 3.0], np.float32))[0] == 5.0


def test_mse_constant_tree_closed_form():
    X, y = synth.config_data(synth.CONFIGS["c2"], n=500)
    c = np.float32(0.37)
    t, v, s = _single([CONST], [c], n_in=4)
    out = oracle.evaluate(t, v, s, X)
    m = oracle.mse(out[:, :, 0], y)[0]
    yd = y.astype(np.float64)
    assert m == pytest.approx(yd.var() + (float(c) - yd.mean()) ** 2, rel=1e-12)


def test_mse_identity_zero():
    X = synth.dataset_X(3, 0, 100, 3)
    t, v, s = _single([VAR], [2], n_in=3)
    out = oracle.evaluate(t, v, s, X)
    assert oracle.mse(out[:, :, 0], X[:, 2].copy())[0] == 0.0


# ---------------------------------------------------------------- classification pins
def test_accuracy_spec_examples():
    """one-hot predictions matching labels -> 1.0; all-zero
    predictions with all labels 0 -> argmax tie -> class 0 -> 1.0."""
    labels = np.array([2, 0, 1, 1], np.int32)
    onehot = np.zeros((1, 4, 3))
    onehot[0, np.arange(4), labels] = 1.0
    assert oracle.accuracy(onehot, labels)[0] == 1.0
    assert oracle.accuracy(np.zeros((1, 4, 3)), np.zeros(4, np.int32))[0] == 1.0
    assert oracle.accuracy(np.zeros((1, 4, 3)), labels)[0] == 0.25


def test_accuracy_bruteforce_numpy_argmax():
    """Reading R15 reduces to numpy's first-occurrence argmax once NaN -> -inf."""
    rng = np.random.default_rng(3)
    out = rng.integers(-2, 3, (20, 50, 5)).astype(np.float64)  # many ties
    out[rng.random(out.shape) < 0.1] = np.nan
    labels = rng.integers(0, 5, 50).astype(np.int32)
    ref = (np.argmax(np.where(np.isnan(out), -np.inf, out), axis=2) == labels[None, :]).mean(axis=1)
    np.testing.assert_array_equal(oracle.accuracy(out, labels), ref)


# ---------------------------------------------------------------- paired inference (NEXT-2)
@pytest.mark.parametrize("n_out,modi", [(1, 0.0), (3, 0.2)])
def test_paired_equals_recursive_per_individual(n_out, modi):
    """evaluate_paired (each individual on its own observation) ==
    the independent recursive interpreter applied to tree p at obs[p][b]."""
    P, L, n_in, B = 25, 15, 3, 2
    pt = synth.trees(41, 0, P, L, synth.MIXES["full"], n_in, n_out, modi)
    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
    obs = synth.dataset_X(41, 1, P * B, n_in, "normal", -1.0, 1.0).reshape(P, B, n_in)
    for mode in (0, 1):
        out = oracle.evaluate_paired(t, v, s, obs, n_out=n_out, mode=mode)
        for p in range(P):
            tys, vas = pt.types[pt.offsets[p]:pt.offsets[p + 1]], pt.values[pt.offsets[p]:pt.offsets[p + 1]]
            for b in range(B):
                r = oracle.evaluate_recursive(tys, vas, obs[p, b], n_out=n_out, mode=mode)
                same = (out[p, b] == r) | (np.isnan(out[p, b]) & np.isnan(r))
                assert same.all(), (p, b, out[p, b], r)
