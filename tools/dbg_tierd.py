import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth, oracle
import paper_2501_17168_b200 as evogp
from tests.test_gpu_parity import make_case, to_device, gpu_eval
P, L, D, n_in, n_out = 300, 63, 5000, 17, 6
pt, X, y = make_case(400, P, L, n_in, D, "full", n_out=n_out, modi=0.1)
dt = to_device(pt, L, n_in, n_out)
a = gpu_eval(dt, X, n_out, "inter"); b = gpu_eval(dt, X, n_out, "intra")
diff = np.argwhere(a.view(np.uint32) != b.view(np.uint32))
print("diffs", len(diff), diff[:5])
for tp, d, o in diff[:3]:
    ty, va = pt.tree(int(tp))
    print("tree", tp, "len", len(ty), "point", d, "slot", o, a[tp, d, o], b[tp, d, o])
    print(list(zip(ty.tolist(), va.tolist())))
    t, v, s = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
    r = oracle.evaluate(t[tp:tp+1], v[tp:tp+1], s[tp:tp+1], X[d:d+1], n_out=n_out, mode=1)
    print("oracle fp32-faithful", r[0, 0, o], "fp64", oracle.evaluate(t[tp:tp+1], v[tp:tp+1], s[tp:tp+1], X[d:d+1], n_out=n_out, mode=0)[0,0,o])
    # force both kernels through the scalar multi-pass path vs the packed path
    for tw in (0, 64):
        evogp.set_tuning(target_warps=tw)
        for st in ("inter", "intra"):
            g = gpu_eval(dt, X, n_out, st)
            print("tw", tw, st, g[tp, d, o])
    evogp.set_tuning()
