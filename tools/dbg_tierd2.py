import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth, oracle
import paper_2501_17168_b200 as evogp
from tests.test_gpu_parity import make_case, to_device, gpu_eval
P, L, D, n_in, n_out = 300, 63, 5000, 17, 6
pt, X, y = make_case(400, P, L, n_in, D, "full", n_out=n_out, modi=0.1)
ty, va = pt.tree(194)
t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
sz = s[194]
# points: the failing one replicated into a full chunk region
Xs = np.repeat(X[4451:4452], 512, axis=0)
res = []
for i in range(len(ty)):
    n = int(sz[i])
    sub_t, sub_v = ty[i:i + n].copy(), va[i:i + n].copy()
    if (sub_t[0] & 8) == 0 and (sub_t[0] & 7) >= 2:
        # make the subtree root a Modi node (slot 5) so its value reaches an output
        sub_t[0] = (sub_t[0] & 0xFF) | 8 | (5 << 8)
    sp = synth.PrefixTrees(np.array([0, n], np.int64), sub_t.astype(np.int16), sub_v.astype(np.float32))
    if (sub_t[0] & 7) < 2:
        continue
    dt = to_device(sp, L, n_in, n_out)
    out = {}
    for tw in (0, 64):
        evogp.set_tuning(target_warps=tw)
        out[tw] = gpu_eval(dt, Xs, n_out, "intra")[0, 0]
    evogp.set_tuning()
    same = np.array_equal(out[0].view(np.uint32), out[64].view(np.uint32))
    if not same:
        res.append((i, n))
        print("node", i, "size", n, "op", (int(ty[i]), float(va[i])), "packed", out[0], "scalar", out[64])
print("differing subtrees:", res)
