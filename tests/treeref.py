"""Pointer-tree re-implementations of the genetic operators — TEST ONLY.

An independent second reading of the paper's operators (PAPER §III-B
P:281-321, Algorithm 1, Table I) on nested Python nodes
instead of flat arrays, fed the same counter-based draws (R16)
through oracle.draw. Used by tests/test_variation_pins.py to pin
oracle/variation.c by brute force: a slip in an array index, an ancestor
test, a size update or a draw slot in either version shows up as a
mismatch. Nothing here touches the CUDA path.

A node is [type_word, value, children]; sizes are recomputed recursively
(size = 1 + sum of child sizes), never by the reverse scan the oracle uses.
"""
from __future__ import annotations

import copy
import math

import numpy as np

import oracle

ARITY = {0: 2, 1: 2, 2: 2, 3: 2, 4: 1, 5: 1, 6: 1, 7: 2, 8: 2, 9: 2, 10: 1, 11: 1, 12: 1, 13: 1, 14: 1,
         15: 1, 16: 1, 17: 2, 18: 2, 19: 2, 20: 2, 21: 3}
CONST, VAR = 0, 1


def arity_of(tw: int) -> int:
    k = tw & 7
    return 0 if k <= VAR else k - 1


def parse(t, v, s=None):
    """Prefix row -> nested nodes (arity from the type word only)."""
    pos = 0

    def rec():
        nonlocal pos
        tw = int(t[pos]) & 0xFFFF
        val = np.float32(v[pos])
        pos += 1
        return [tw, val, [rec() for _ in range(arity_of(tw))]]

    return rec()


def size(n) -> int:
    return 1 + sum(size(c) for c in n[2])


def preorder(n):
    out = [n]
    for c in n[2]:
        out.extend(preorder(c))
    return out


def serialize(n, L):
    """Nested nodes -> padded (t, v, s) rows of length L (reading R1 padding)."""
    nodes = preorder(n)
    t = np.full(L, -1, np.int16)
    v = np.full(L, np.nan, np.float32)
    v.view(np.uint32)[:] = 0x7FC00000
    s = np.zeros(L, np.int16)
    for i, x in enumerate(nodes):
        t[i] = np.array(x[0], np.uint16).view(np.int16)
        v[i] = x[1]
        s[i] = size(x)
    return t, v, s


def depth(n) -> int:
    return 1 + max((depth(c) for c in n[2]), default=0)


def replace_preorder(root, k, new):
    """Copy of root with its k-th preorder node replaced by `new`."""
    root = copy.deepcopy(root)
    if k == 0:
        return copy.deepcopy(new)
    nodes = preorder(root)
    target = nodes[k]
    for x in nodes:
        for q, c in enumerate(x[2]):
            if c is target:
                x[2][q] = copy.deepcopy(new)
                return root
    raise AssertionError("node not found")


# ---- draws (reading R16) -------------------------------------------------------
def index(u: int, n: int) -> int:
    return (u * n) >> 32


def thr(p) -> int:
    p = float(np.float32(p))
    if not p > 0.0:
        return 0
    if p >= 1.0:
        return 1 << 32
    return int(math.floor(p * 4294967296.0))


def coin(u: int, p) -> bool:
    return u < thr(p)


def unit(u: int) -> np.float32:
    return np.float32(u >> 8) * np.float32(2.0 ** -24)


def const_from(u: int, lo, hi) -> np.float32:
    lo, hi = np.float32(lo), np.float32(hi)
    return np.float32(lo + np.float32(np.float32(hi - lo) * unit(u)))


def perturb(v, u: int, sigma) -> np.float32:
    s = np.float32(np.float32(2.0) * unit(u) - np.float32(1.0))
    return np.float32(np.float32(v) + np.float32(np.float32(sigma) * s))


def func_word(f: int, modi: int = 0, slot: int = 0) -> int:
    return (1 + ARITY[f]) | (8 if modi else 0) | ((slot << 8) if modi else 0)


def funcs_of(cfg, a=None):
    return [f for f in sorted(cfg["funcs"]) if a is None or ARITY[f] == a]


P = oracle.PUR


# ---- generation (reading R19), recursive --------------------------------------
def gen_tree(cfg, depth_limit, full, budget, seed, stream):
    g = [0]
    n = [0]
    fl = funcs_of(cfg)

    def d_():
        u = oracle.draw(seed, stream, P["gen"], g[0])
        g[0] += 1
        return u

    def node(d, pending):
        want = False
        f = None
        if d + 1 < depth_limit and fl:
            want = True if full else not coin(d_(), cfg["p_leaf"])
        if want:
            f = fl[index(d_(), len(fl))]
            if n[0] + 1 + pending + ARITY[f] > budget:
                want = False
        i = n[0]
        n[0] += 1
        if want:
            modi, slot = 0, 0
            if cfg["n_outputs"] > 1:
                modi = 1 if i == 0 else int(coin(d_(), cfg["p_modi"]))
                if modi:
                    slot = index(d_(), cfg["n_outputs"])
            a = ARITY[f]
            me = [func_word(f, modi, slot), np.float32(f), []]
            for q in range(a):
                me[2].append(node(d + 1, pending + (a - 1 - q)))
            return me
        if coin(d_(), cfg["p_const"]):
            return [CONST, const_from(d_(), cfg["const_lo"], cfg["const_hi"]), []]
        return [VAR, np.float32(index(d_(), cfg["n_inputs"])), []]

    return node(0, 0)


def generate(Pn, cfg, seed):
    levels = cfg["depth_max"] - cfg["depth_min"] + 1
    rows = []
    for i in range(Pn):
        b = i % (2 * levels)
        rows.append(gen_tree(cfg, cfg["depth_min"] + b // 2, b & 1, cfg["max_len"], seed, i))
    return rows


# ---- reproduction (Algorithm 1 loop body, reading R18) -----------------------
def tournament(fit, T, seed, stream, pur):
    Pn = len(fit)
    cands = [index(oracle.draw(seed, stream, pur, t), Pn) for t in range(T)]
    return min(cands, key=lambda i: (math.inf if math.isnan(fit[i]) else fit[i], i))


def _site(cfg, tree, seed, c, pur):
    nodes = preorder(tree)
    u = oracle.draw(seed, c, pur, 1)
    if cfg["crossover_kind"] == 1:
        leaf = coin(oracle.draw(seed, c, pur, 0), cfg["leaf_bias"])
        cls = [i for i, x in enumerate(nodes) if (not x[2]) == leaf]
        if cls:
            return cls[index(u, len(cls))]
    return index(u, len(nodes))


def _mut_kind(cfg, u):
    w = [float(np.float32(x)) for x in cfg["mutation_weights"]]
    W = sum(w)
    last = max(q for q in range(8) if w[q] > 0)
    acc = 0.0
    for q in range(8):
        acc += w[q]
        t = (1 << 32) if q == last else int(math.floor(acc / W * 4294967296.0))
        if w[q] > 0 and u < t:
            return q
    return last


def _point(cfg, x, u1, u2):
    a = len(x[2])
    if a > 0:
        lst = funcs_of(cfg, a)
        if lst:
            x[1] = np.float32(lst[index(u1, len(lst))])
    elif coin(u1, cfg["p_const"]):
        x[0], x[1] = CONST, const_from(u2, cfg["const_lo"], cfg["const_hi"])
    else:
        x[0], x[1] = VAR, np.float32(index(u2, cfg["n_inputs"]))


def reproduce_one(rows, fit, cfg, seed, c):
    """Child c of Algorithm 1: returns (tree, p1, p2, op)."""
    L = cfg["max_len"]

    def D(pur, i):
        return oracle.draw(seed, c, P[pur], i)

    T = cfg["tournament_size"]
    p1 = tournament(fit, T, seed, c, P["tour1"])
    p2 = tournament(fit, T, seed, c, P["tour2"])
    t1, t2 = rows[p1], rows[p2]
    op = 0
    if coin(D("xo_gate", 0), cfg["p_crossover"]):
        k = _site(cfg, t1, seed, c, P["xo_k"])
        j = _site(cfg, t2, seed, c, P["xo_j"])
        new = replace_preorder(t1, k, preorder(t2)[j])
        if size(new) > L:
            child, op = copy.deepcopy(t1), op | oracle.OP_XO_REJECTED
        else:
            child, op = new, op | oracle.OP_XO
    else:
        child = copy.deepcopy(t1)
    if coin(D("mut_gate", 0), cfg["p_mutation"]):
        kind = _mut_kind(cfg, D("mut_kind", 0))
        op |= (kind + 1) << 4
        nodes = preorder(child)
        n = len(nodes)
        internal = [i for i, x in enumerate(nodes) if x[2]]
        consts = [i for i, x in enumerate(nodes) if not x[2] and x[0] == CONST]
        nop = False
        name = oracle.MUTATIONS[kind]
        if name == "subtree":
            k = index(D("mut_site", 0), n)
            new = gen_tree(cfg, cfg["subtree_depth"], 0, L - (n - size(nodes[k])), seed, c)
            child = replace_preorder(child, k, new)
        elif name == "hoist":
            if not internal:
                nop = True
            else:
                k = internal[index(D("mut_site", 0), len(internal))]
                desc = preorder(nodes[k])[1:]
                child = replace_preorder(child, k, desc[index(D("mut_site", 1), len(desc))])
        elif name == "point":
            i = index(D("mut_site", 0), n)
            _point(cfg, nodes[i], D("mut_site", 1), D("mut_site", 2))
        elif name == "multi_point":
            for i, x in enumerate(nodes):
                if coin(D("point_coin", i), cfg["point_rate"]):
                    _point(cfg, x, D("point_new", 2 * i), D("point_new", 2 * i + 1))
        elif name == "insert":
            k = index(D("mut_site", 0), n)
            fl = funcs_of(cfg)
            f = fl[index(D("mut_site", 1), len(fl))]
            a = ARITY[f]
            if n + a > L:
                nop = True
            else:
                kids = [copy.deepcopy(nodes[k])]
                for l in range(a - 1):
                    if coin(D("mut_site", 2 + 2 * l), cfg["p_const"]):
                        kids.append([CONST, const_from(D("mut_site", 3 + 2 * l), cfg["const_lo"],
                                                       cfg["const_hi"]), []])
                    else:
                        kids.append([VAR, np.float32(index(D("mut_site", 3 + 2 * l), cfg["n_inputs"])), []])
                child = replace_preorder(child, k, [func_word(f), np.float32(f), kids])
        elif name == "delete":
            if not internal:
                nop = True
            else:
                k = internal[index(D("mut_site", 0), len(internal))]
                kid = nodes[k][2][index(D("mut_site", 1), len(nodes[k][2]))]
                child = replace_preorder(child, k, kid)
        elif name == "const":
            if not consts:
                nop = True
            else:
                i = consts[index(D("mut_site", 0), len(consts))]
                nodes[i][1] = perturb(nodes[i][1], D("mut_site", 1), cfg["const_sigma"])
        elif name == "multi_const":
            if not consts:
                nop = True
            for i in consts:
                if coin(D("point_coin", i), cfg["point_rate"]):
                    nodes[i][1] = perturb(nodes[i][1], D("point_new", 2 * i), cfg["const_sigma"])
        if nop:
            op |= oracle.OP_MUT_NOP
    return child, p1, p2, op
