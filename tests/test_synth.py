"""The seeded generator: determinism, shard independence, recipe properties."""
import numpy as np

import oracle
import synth


def test_shard_independence_trees():
    full = synth.trees(5, 0, 200, 63, synth.M_PAPER, 4)
    part = synth.trees(5, 120, 50, 63, synth.M_PAPER, 4)
    for i in range(50):
        a = full.tree(120 + i)
        b = part.tree(i)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


def test_shard_independence_data():
    X = synth.dataset_X(9, 0, 300, 8)
    Xs = synth.dataset_X(9, 100, 100, 8)
    np.testing.assert_array_equal(X[100:200], Xs)


def test_recipe_properties():
    L = 127
    pt = synth.trees(1, 0, 2000, L, synth.M_PAPER, 8)
    lens = np.diff(pt.offsets)
    assert lens.min() >= (L + 1) // 2 and lens.max() <= L
    assert abs(lens.mean() - 0.75 * L) < 0.05 * L  # S-bar ~ 0.75 L
    kinds = pt.types & 7
    fids = pt.values[kinds >= 2].astype(int)
    assert set(np.unique(fids)) <= set(synth.M_PAPER)
    vars_ = pt.values[kinds == 1]
    assert vars_.min() >= 0 and vars_.max() <= 7
    consts = pt.values[kinds == 0]
    assert consts.min() >= -1 and consts.max() <= 1
    # every generated tree is well-formed under the oracle's tensorizer
    oracle.tensorize(pt.offsets, pt.types, pt.values, L, 8)


def test_modi_recipe():
    cfg = synth.CONFIGS["c5"]
    pt = synth.config_trees(cfg, synth.M_FULL, n=500)
    roots = pt.types[pt.offsets[:-1]]
    fn_roots = (roots & 7) >= 2
    assert ((roots[fn_roots] & 8) != 0).all()  # root forced Modi
    slots = (pt.types[(pt.types & 8) != 0].astype(np.int32) >> 8) & 0xFF
    assert slots.max() < cfg.n_out
    oracle.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in, cfg.n_out)


def test_pagie_targets():
    X = np.array([[1.0, 1.0], [5.0, 5.0], [0.0, 0.0]], np.float32)
    y = synth.pagie_y(X)
    assert y[0] == 1.0
    assert abs(y[1] - 2 * 625 / 626) < 1e-6
    assert y[2] == 0.0
