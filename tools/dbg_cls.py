import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_2501_17168_b200 as evogp
P, L, n_in, n_cls, D = map(int, sys.argv[1:6]); strategy = sys.argv[6]; mode = sys.argv[7]
pt = synth.trees(900 + D, 0, P, L, synth.MIXES["ieee"], n_in, n_cls, 0.1)
X = synth.dataset_X(900 + D, 0, D, n_in, "normal", -1.0, 1.0)
t, v, s = [torch.from_numpy(a).cuda() for a in evogp.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_cls)]
Xd = torch.from_numpy(X).cuda()
print("plan", evogp.select_strategy(P, D, L, n_cls) if hasattr(evogp, "select_strategy") else "", flush=True)
if mode == "eval":
    o = evogp.eval(t, v, s, Xd, n_outputs=n_cls, strategy=strategy); torch.cuda.synchronize(); print("eval ok", flush=True)
else:
    lab = torch.zeros(D, dtype=torch.int32, device="cuda")
    a = evogp.classification_accuracy(t, v, s, Xd, lab, n_cls, strategy=strategy); torch.cuda.synchronize()
    print("cls ok", a[:4].cpu().numpy(), flush=True)
