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
Xs = np.repeat(X[4451:4452], 128, axis=0)
names = ['ADD','SUB','MUL','DIV','SIN','COS','TAN','MAX','MIN','POW','LOG','EXP','TANH','NEG','ABS','SQRT','INV','LT','GT','LE','GE','IF']
for i in range(8, len(ty)):
    n = int(sz[i])
    sub_t, sub_v = ty[i:i + n].copy(), va[i:i + n].copy()
    if (sub_t[0] & 7) < 2:
        continue
    sub_t[0] = (sub_t[0] & 0xFF) | 8 | (5 << 8)
    sp = synth.PrefixTrees(np.array([0, n], np.int64), sub_t.astype(np.int16), sub_v.astype(np.float32))
    dt = to_device(sp, L, n_in, n_out)
    g = gpu_eval(dt, Xs, n_out, "intra")[0, 0]
    tt, vv, ss = oracle.tensorize(sp.offsets, sp.types, sp.values, L, n_in, n_out)
    r = oracle.evaluate(tt, vv, ss, Xs[:1], n_out=n_out, mode=1)[0, 0]
    cls = lambda a: 'nan' if np.isnan(a) else ('inf' if np.isinf(a) else 'fin')
    flag = '' if cls(g[5]) == cls(r[5]) else '   <-- class differs'
    print(i, n, names[int(va[i])], 'modi' if ty[i] & 8 else '', g[5], r[5], flag)
print("inputs", Xs[0][[1,13,7,10,5,12,15,18 % 17]])
