"""Pins for the genetic-operator oracle (oracle/variation.c) — no GPU.

SURVEY §8(f) NEXT-3 / NEXT-4. Each test names what it pins the oracle to:
  * SPEC hand examples of subtree_exchange / crossover / mutation /
    tournament / generate_tree (S:174-175, S:191-193, S:202-203, S:216-218,
    S:241-243), with the draws they force found by search;
  * laws of the paper's exchange: identity, size-cap rejection
    returns T_old bit-identically, only ancestors of k change size, by Δn;
  * brute force against the pointer-tree re-implementation in
    tests/treeref.py (nested nodes, recursive sizes) fed the same draws;
  * counting and distribution laws (ramp buckets, uniform tournament at T=1).
"""
import math

import numpy as np
import pytest

import oracle
import synth
from tests import treeref

PAPER_FUNCS = [0, 1, 2, 3, 4, 5, 6]


def cfg_base(**kw):
    c = dict(max_len=63, n_inputs=4, n_outputs=1, funcs=PAPER_FUNCS, const_lo=-1.0, const_hi=1.0, p_const=0.5,
             p_leaf=0.1, p_modi=0.0, depth_min=2, depth_max=6, tournament_size=20, p_crossover=0.9,
             p_mutation=0.1, crossover_kind=0, leaf_bias=0.1, mutation_weights=[1.0] + [0.0] * 7,
             point_rate=0.1, const_sigma=0.1, subtree_depth=4)
    c.update(kw)
    return c


def rows_of(t, v, s):
    return [treeref.parse(t[i], v[i]) for i in range(t.shape[0])]


def encode(types, values, L):
    off = np.array([0, len(types)], np.int64)
    return oracle.tensorize(off, np.array(types, np.int16), np.array(values, np.float32), L, 4, 1)


def synth_pop(P, L, mix=synth.M_FULL, seed=11, n_out=1):
    pt = synth.trees(seed, 0, P, L, mix, 4, n_out)
    return oracle.tensorize(pt.offsets, pt.types, pt.values, L, 4, n_out)


# ------------------------------------------------------------------ exchange
def test_exchange_spec_example():
    """old='+(x0,1.0)', k=1, new='sin(x1)' -> '+(sin(x1),1.0)', sizes [4,2,1,1]."""
    L = 6
    ot, ov, os_ = encode([3, 1, 0], [0, 0, 1.0], L)
    nt, nv, ns = encode([2, 1], [4, 1], L)
    t, v, s, rej = oracle.exchange(ot, ov, os_, [0], [1], nt, nv, ns, [0], [0], L)
    assert not rej[0]
    assert list(t[0, :4]) == [3, 2, 1, 0]
    assert list(v[0, :4]) == [0, 4, 1, 1.0]
    assert list(s[0, :5]) == [4, 2, 1, 1, 0]


def test_exchange_rejected_when_too_large():
    """S:193 / P:305-307: max_len=3 -> the original tree, bit for bit."""
    L = 3
    ot, ov, os_ = encode([3, 1, 0], [0, 0, 1.0], L)
    nt, nv, ns = encode([2, 1], [4, 1], L)
    t, v, s, rej = oracle.exchange(ot, ov, os_, [0], [1], nt, nv, ns, [0], [0], L)
    assert rej[0]
    assert (t == ot).all() and (s == os_).all() and (v.view(np.uint32) == ov.view(np.uint32)).all()


def test_exchange_identity_law():
    """exchange(T, k, T[k]) == T for every node k."""
    L = 63
    t, v, s = synth_pop(40, L)
    par, ks = [], []
    for p in range(40):
        for k in range(s[p, 0]):
            par.append(p)
            ks.append(k)
    rt, rv, rs, rej = oracle.exchange(t, v, s, par, ks, t, v, s, par, ks, L)
    assert not rej.any()
    assert (rt == t[par]).all() and (rs == s[par]).all()
    assert (rv.view(np.uint32) == v[par].view(np.uint32)).all()


def test_exchange_brute_force_vs_pointer_splice():
    """Every result equals the recursive pointer-tree splice (treeref), with
    rejection exactly when the spliced tree exceeds max_len; only ancestors of
    k change size, each by Δn."""
    L = 31
    t, v, s = synth_pop(60, L, seed=5)
    rng = np.random.default_rng(0)
    n = 3000
    par = rng.integers(0, 60, n)
    don = rng.integers(0, 60, n)
    ks = np.array([rng.integers(0, s[p, 0]) for p in par])
    js = np.array([rng.integers(0, s[d, 0]) for d in don])
    rt, rv, rs, rej = oracle.exchange(t, v, s, par, ks, t, v, s, don, js, L)
    trees = rows_of(t, v, s)
    n_rej = 0
    for c in range(n):
        p, d, k, j = int(par[c]), int(don[c]), int(ks[c]), int(js[c])
        new = treeref.replace_preorder(trees[p], k, treeref.preorder(trees[d])[j])
        if treeref.size(new) > L:
            n_rej += 1
            assert rej[c]
            assert (rt[c] == t[p]).all() and (rs[c] == s[p]).all()
            continue
        assert not rej[c]
        et, ev, es = treeref.serialize(new, L)
        assert (rt[c] == et).all() and (rs[c] == es).all(), c
        assert (rv[c].view(np.uint32) == ev.view(np.uint32)).all(), c
        # ancestor law on the untouched prefix [0, k)
        dn = int(s[d, j]) - int(s[p, k])
        for i in range(k):
            anc = i + int(s[p, i]) > k
            assert int(rs[c, i]) == int(s[p, i]) + (dn if anc else 0)
    assert 0 < n_rej < n


# ---------------------------------------------------------------- tournament
def _find_stream(P, T, want, purpose=1, seed=3):
    for st in range(200000):
        if [treeref.index(oracle.draw(seed, st, purpose, t), P) for t in range(T)] == want:
            return st
    raise AssertionError("no stream found")


def test_tournament_spec_example():
    """fitness [3,1,2], k=2, draws (0,2) -> index 2 (lower is better)."""
    st = _find_stream(3, 2, [0, 2])
    w = oracle.tournament([3.0, 1.0, 2.0], 2, st + 1, 3, purpose=1)
    assert w[st] == 2


def test_tournament_brute_force_ties_nan():
    """Lexicographic min of (fitness, index) over the drawn candidates; NaN
    ranks as +inf; ties go to the lowest index."""
    rng = np.random.default_rng(1)
    fit = rng.integers(0, 6, 50).astype(np.float64)
    fit[rng.integers(0, 50, 8)] = np.nan
    fit[3] = np.inf
    T, n, seed = 7, 2000, 99
    w = oracle.tournament(fit, T, n, seed, purpose=2)
    for c in range(n):
        cands = np.array([treeref.index(oracle.draw(seed, c, 2, t), 50) for t in range(T)])
        key = np.where(np.isnan(fit[cands]), np.inf, fit[cands])
        best = cands[np.lexsort((cands, key))[0]]
        assert w[c] == best


def test_tournament_T1_uniform():
    """k=1 -> a uniform index: chi-square over 20 bins."""
    n = 40000
    w = oracle.tournament(np.zeros(20), 1, n, 5)
    cnt = np.bincount(w, minlength=20)
    chi2 = ((cnt - n / 20) ** 2 / (n / 20)).sum()
    assert chi2 < 45  # 19 dof, p ~ 1e-3


def test_tournament_full_size_finds_best_often():
    """Large tournaments select the global best with probability 1-(1-1/P)^T."""
    fit = np.arange(100, dtype=np.float64)[::-1].copy()
    w = oracle.tournament(fit, 100, 5000, 8)
    frac = (w == 99).mean()
    assert abs(frac - (1 - (1 - 1 / 100) ** 100)) < 0.03


# ---------------------------------------------------------------- generation
def test_generate_depth1_is_leaf():
    """depth_max=1 -> a single leaf."""
    c = cfg_base(depth_min=1, depth_max=1)
    t, v, s = oracle.generate(50, c, 1)
    assert (s[:, 0] == 1).all() and ((t[:, 0] == 0) | (t[:, 0] == 1)).all()


def test_generate_full_binary_depth3_is_7_nodes():
    """FULL depth 3, binary-only set -> exactly 7 nodes (odd buckets are FULL)."""
    c = cfg_base(depth_min=3, depth_max=3, funcs=[0, 2])
    t, v, s = oracle.generate(40, c, 2)
    assert (s[1::2, 0] == 7).all()
    assert (s[0::2, 0] <= 7).all()


def test_generate_valid_depth_and_ramp_counts():
    """Every tree re-tensorizes to the same sizes (valid prefix), depth within
    its bucket's limit, FULL trees reach it on every leaf when the budget
    allows; ramped buckets get floor/ceil(n/10) trees."""
    c = cfg_base(funcs=list(range(22)), max_len=127)
    n = 1000
    t, v, s = oracle.generate(n, c, 3)
    lens = s[:, 0].astype(np.int64)
    off = np.concatenate([[0], np.cumsum(lens)])
    types = np.concatenate([t[i, :lens[i]] for i in range(n)])
    vals = np.concatenate([v[i, :lens[i]] for i in range(n)])
    rt, rv, rs = oracle.tensorize(off, types, vals, 127, 4, 1)
    assert (rs == s).all()
    buckets = np.bincount(np.arange(n) % 10, minlength=10)
    assert set(buckets) <= {100}
    for i in range(n):
        tr = treeref.parse(t[i], v[i])
        lim = 2 + (i % 10) // 2
        assert treeref.depth(tr) <= lim
        if i % 2 == 1 and lens[i] < 127:
            # FULL: every leaf at depth exactly lim (budget never bound here)
            def leaf_depths(x, d=1):
                return [d] if not x[2] else sum((leaf_depths(ch, d + 1) for ch in x[2]), [])
            assert set(leaf_depths(tr)) == {lim}


def test_generate_budget_and_recursive_reimplementation():
    """Tight budget (max_len 15, depth 8): never exceeds max_len; bit-exact vs
    the recursive generator of treeref fed the same draws; Modi roots for
    n_outputs > 1."""
    for n_out in (1, 3):
        c = cfg_base(max_len=15, depth_min=3, depth_max=8, n_outputs=n_out, p_modi=0.3, funcs=list(range(22)))
        t, v, s = oracle.generate(300, c, 4)
        assert (s[:, 0] <= 15).all() and (s[:, 0] >= 1).all()
        ref = treeref.generate(300, c, 4)
        for i in range(300):
            et, ev, es = treeref.serialize(ref[i], 15)
            assert (t[i] == et).all() and (s[i] == es).all(), (n_out, i)
            assert (v[i].view(np.uint32) == ev.view(np.uint32)).all(), (n_out, i)
            if n_out > 1 and s[i, 0] > 1:
                assert (int(t[i, 0]) & 8) != 0


def test_generate_deterministic():
    c = cfg_base()
    a = oracle.generate(200, c, 9)
    b = oracle.generate(200, c, 9)
    assert all((x == y).all() for x, y in zip(a[:1] + a[2:], b[:1] + b[2:]))
    assert (a[1].view(np.uint32) == b[1].view(np.uint32)).all()


# ---------------------------------------------------------------- reproduce
def test_reproduce_clone_law():
    """p_c = p_m = 0 -> children are clones of the first tournament winner."""
    c = cfg_base(p_crossover=0.0, p_mutation=0.0)
    t, v, s = synth_pop(100, 63)
    fit = np.random.default_rng(2).random(100)
    ct, cv, cs, par, ops = oracle.reproduce(t, v, s, fit, 300, c, 12)
    assert (ops == 0).all()
    assert (par[:, 0] == oracle.tournament(fit, 20, 300, 12, purpose=1)).all()
    assert (par[:, 1] == oracle.tournament(fit, 20, 300, 12, purpose=2)).all()
    assert (ct == t[par[:, 0]]).all() and (cs == s[par[:, 0]]).all()


CASES = [("one_point", dict(crossover_kind=0, p_mutation=0.0))] + \
        [("leaf_biased", dict(crossover_kind=1, leaf_bias=0.3, p_mutation=0.0))] + \
        [(m, dict(p_crossover=0.5, p_mutation=1.0, mutation_weights=[float(q == i) for q in range(8)]))
         for i, m in enumerate(oracle.MUTATIONS)] + \
        [("mixed", dict(p_mutation=0.5, mutation_weights=[1, 2, 1, 1, 3, 1, 1, 2]))]


@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_reproduce_vs_pointer_tree(name, kw):
    """Each operator fed the same draws equals its pointer-tree
    re-implementation ('Oracle equivalence'); shape laws: point / const
    mutations keep the sizes array, hoist / delete never grow (S:210-212,
    S:261); every child is a valid tree within max_len."""
    L = 31 if name != "mixed" else 63
    c = cfg_base(max_len=L, funcs=list(range(22)), point_rate=0.3, **kw)
    t, v, s = synth_pop(80, L, seed=21)
    fit = np.random.default_rng(3).random(80)
    fit[::7] = np.nan
    n = 400
    ct, cv, cs, par, ops = oracle.reproduce(t, v, s, fit, n, c, 1234)
    rows = rows_of(t, v, s)
    for i in range(n):
        tree, p1, p2, op = treeref.reproduce_one(rows, fit, c, 1234, i)
        assert (par[i, 0], par[i, 1], ops[i]) == (p1, p2, op), (name, i)
        et, ev, es = treeref.serialize(tree, L)
        assert (ct[i] == et).all() and (cs[i] == es).all(), (name, i)
        assert (cv[i].view(np.uint32) == ev.view(np.uint32)).all(), (name, i)
    assert (cs[:, 0] <= L).all() and (cs[:, 0] >= 1).all()
    if name in ("point", "multi_point", "const", "multi_const"):
        base = np.where((ops & oracle.OP_XO) != 0, -1, par[:, 0])
        keep = base >= 0
        assert (cs[keep] == s[base[keep]]).all()
    if name in ("hoist", "delete"):
        keep = (ops & oracle.OP_XO) == 0
        assert (cs[keep, 0] <= s[par[keep, 0], 0]).all()
    mut = (ops >> 4) & 0xF
    if name not in ("one_point", "leaf_biased", "mixed"):
        assert (mut[mut > 0] == oracle.MUTATIONS.index(name) + 1).all()
        assert (mut > 0).all()


def test_reproduce_children_valid_over_generations():
    """S:254 (scaled down): 30 generations of churn with every operator on;
    every row of every population re-tensorizes to the same sizes."""
    L = 63
    c = cfg_base(max_len=L, funcs=list(range(22)), p_mutation=0.6, mutation_weights=[1] * 8, point_rate=0.2)
    t, v, s = oracle.generate(200, c, 77)
    rng = np.random.default_rng(4)
    for g in range(30):
        fit = rng.random(200)
        t, v, s, _, _ = oracle.reproduce(t, v, s, fit, 200, c, 1000 + g)
        lens = s[:, 0].astype(np.int64)
        assert (lens >= 1).all() and (lens <= L).all()
        off = np.concatenate([[0], np.cumsum(lens)])
        types = np.concatenate([t[i, :lens[i]] for i in range(200)])
        vals = np.concatenate([v[i, :lens[i]] for i in range(200)])
        _, _, rs = oracle.tensorize(off, types, vals, L, 4, 1)
        assert (rs == s).all()
        assert (t[s == 0] == -1).all()


def test_reproduce_multi_output_keeps_slots_valid():
    """Modi trees (n_outputs 6): every child re-tensorizes with n_outputs 6."""
    L = 63
    c = cfg_base(max_len=L, n_outputs=6, p_modi=0.2, p_mutation=0.5, mutation_weights=[1] * 8)
    t, v, s = oracle.generate(100, c, 5)
    fit = np.random.default_rng(5).random(100)
    ct, cv, cs, _, _ = oracle.reproduce(t, v, s, fit, 200, c, 6)
    lens = cs[:, 0].astype(np.int64)
    off = np.concatenate([[0], np.cumsum(lens)])
    types = np.concatenate([ct[i, :lens[i]] for i in range(200)])
    vals = np.concatenate([cv[i, :lens[i]] for i in range(200)])
    _, _, rs = oracle.tensorize(off, types, vals, L, 4, 6)
    assert (rs == cs).all()


def test_draw_uniformity():
    """R16 generator: the top byte of 2^16 draws is uniform (chi-square) and
    streams differ."""
    u = np.array([oracle.draw(1, 0, 1, i) for i in range(1 << 16)], np.uint64)
    cnt = np.bincount((u >> 24).astype(np.int64), minlength=256)
    e = len(u) / 256
    assert ((cnt - e) ** 2 / e).sum() < 330
    assert oracle.draw(1, 0, 1, 0) != oracle.draw(1, 1, 1, 0)
    assert oracle.draw(1, 0, 1, 0) != oracle.draw(2, 0, 1, 0)
