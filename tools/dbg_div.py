import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2501_17168_b200 as evogp
from tests.test_gpu_parity import to_device, gpu_eval
n_in, n_out = 2, 3
# Modi root (slot 0) DIV(x0, x1); Modi root SIN(x0); POW then DIV: DIV(POW(x0,x1), x1)
trees = [([3 | 8, 1, 1], [3, 0, 1]), ([2 | 8, 1], [4, 0]), ([3 | 8, 3, 1, 1, 1], [3, 9, 0, 1, 1])]
offs = np.cumsum([0] + [len(t) for t, _ in trees]).astype(np.int64)
pt = synth.PrefixTrees(offs, np.array([x for t, _ in trees for x in t], np.int16),
                       np.array([x for _, v in trees for x in v], np.float32))
rng = np.random.default_rng(0)
X = rng.uniform(-3, 3, (512, 2)).astype(np.float32)
X[::5, 0] = np.inf; X[1::5, 0] = -np.inf; X[2::7, 1] = 0.5; X[3::11, 0] = 1e20; X[4::13, 1] = -np.inf
X[5::17, 0] = 40.0; X[5::17, 1] = 30.0
dt = to_device(pt, 5, n_in, n_out)
out = {}
for tw in (0, 64):
    evogp.set_tuning(target_warps=tw)
    out[tw] = gpu_eval(dt, X, n_out, "intra")
evogp.set_tuning()
d = np.argwhere(out[0].view(np.uint32) != out[64].view(np.uint32))
print("diffs", len(d))
for tp, p, o in d[:12]:
    print(tp, p, o, X[p], out[0][tp, p, o], out[64][tp, p, o])
import oracle
t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, 5, n_in, n_out)
r = oracle.evaluate(t, v, s, X, n_out=n_out, mode=1)
g = out[0]
for tp in range(3):
    bad = ~((g[tp] == r[tp].astype(np.float32)) | (np.isnan(g[tp]) & np.isnan(r[tp])))
    if tp == 2:
        bad = (np.isnan(g[tp]) != np.isnan(r[tp])) | (np.isinf(g[tp]) != np.isinf(r[tp]))
    idx = np.argwhere(bad)
    print("tree", tp, "mismatches", len(idx))
    for p, o in idx[:6]:
        print("  ", X[p], g[tp, p, o], r[tp, p, o])
