"""Exhaustive accuracy pins of the interpreter's elementary functions against
the error model the oracle's certificate assumes (reading R14;
oracle/oracle.c `op_err`): for an op with result r the FP32 evaluation may
differ from the exact value by

    ulp_budget(f) * 2^-23 * |r|  (+ 2^-20 absolute for sin / cos, 2^-21 for log)

with ulp_budget = 2 (sin, cos, exp, tanh), 3 (log), 4 (tan, pow) — the CUDA
Math API's documented maximum ulp errors of sinf/cosf, expf, tanhf, tanf,
powf, for sin/cos the SFU (sin.approx / cos.approx) absolute error on the
reduced argument, and for log the SFU form's (__logf: lg2.approx * ln 2)
documented 2^-21.41 absolute on [0.5, 2] / 3 ulp elsewhere. A certified point is only as sound as these bounds,
so each is checked here on every FP32 argument of its working range (all
2.1e9 floats of [-pi, pi] for sin / cos, all of [-87.3, 88.7] for exp, all
positive floats above the protection threshold for log, all of [-9.1, 9.1]
for tanh) or, for the two-argument pow, on 2^27 random pairs — evaluated by
the library (one-node trees through evogp_eval, the production kernels) and
compared with FP64 references computed by torch on the GPU (test
infrastructure only). The maximum observed error is printed for DESIGN.md.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TWO_M23 = 2.0 ** -23
SFU_TRIG_ABS = 2.0 ** -20  # oracle/oracle.c SFU_TRIG_ABS
SFU_LOG_ABS = 2.0 ** -21  # oracle/oracle.c SFU_LOG_ABS
FP32_TINY = 1.401298464324817e-45
CHUNK = 1 << 26

# function ids (include/evogp.h)
SIN, COS, TAN, POW, LOG, EXP, TANH = 4, 5, 6, 9, 10, 11, 12


def _unary_trees(fids):
    """One tree per function: [UFUNC f, VAR x0] (types 2 / 1)."""
    P = len(fids)
    t = torch.full((P, 2), 1, dtype=torch.int16)
    t[:, 0] = 2
    v = torch.zeros((P, 2), dtype=torch.float32)
    v[:, 0] = torch.tensor(fids, dtype=torch.float32)
    s = torch.tensor([[2, 1]] * P, dtype=torch.int16)
    return t.cuda(), v.cuda(), s.cuda()


def _floats(lo_bits, hi_bits, neg):
    """Every float32 with bit pattern in [lo_bits, hi_bits) (and its negative), in chunks."""
    for a in range(lo_bits, hi_bits, CHUNK):
        b = min(hi_bits, a + CHUNK)
        x = torch.arange(a, b, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.float32)
        yield x
        if neg:
            yield -x


def _bits(f):
    return int(np.array([f], np.float32).view(np.int32)[0])


def _sweep(fids, refs, budgets, lo_bits, hi_bits, neg, abs_extra=0.0, negate=False):
    """refs see the generated floats x; the trees are evaluated at -x when negate."""
    import paper_2501_17168_b200 as evogp

    t, v, s = _unary_trees(fids)
    worst = [0.0] * len(fids)  # max of err / (budget * 2^-23 * |r| + abs_extra + tiny)
    worst_abs = [0.0] * len(fids)
    n = 0
    for x in _floats(lo_bits, hi_bits, neg):
        xin = -x if negate else x
        out = evogp.eval(t, v, s, xin[:, None].contiguous())[:, :, 0].double()
        xd = x.double()
        for i, (ref_fn, bud) in enumerate(zip(refs, budgets)):
            r = ref_fn(xd)
            g = out[i]
            fin = torch.isfinite(r)
            assert torch.equal(torch.isfinite(g), fin), (fids[i], x[torch.isfinite(g) != fin][:4].tolist())
            err = (g - r).abs()[fin]
            bound = bud * TWO_M23 * r.abs()[fin] + abs_extra + FP32_TINY
            q = (err / bound).max().item()
            worst[i] = max(worst[i], q)
            worst_abs[i] = max(worst_abs[i], err.max().item())
            assert q <= 1.0, (fids[i], q, x[fin][torch.argmax(err / bound)].item())
        n += x.numel()
    return worst, worst_abs, n


def test_sin_cos_every_float_in_pi_range():
    """sin / cos of every FP32 argument in [-pi, pi] (the only range the SFU
    sees after the kernel's 2*pi reduction): |err| <= 2 * 2^-23 |r| + 2^-20."""
    worst, wabs, n = _sweep([SIN, COS], [torch.sin, torch.cos], [2.0, 2.0], 0, _bits(np.pi) + 1, True,
                            SFU_TRIG_ABS)
    print(f"sin/cos over {n} floats: worst bound fraction {worst}, max abs err "
          f"2^{np.log2(max(wabs[0], 1e-300)):.2f} / 2^{np.log2(max(wabs[1], 1e-300)):.2f}")


def test_exp_every_float_in_normal_range():
    """expf over every FP32 argument whose result is a normal FP32 number:
    [0, 88.72] and [-87.33, 0)."""
    wp, _, n1 = _sweep([EXP], [torch.exp], [2.0], 0, _bits(88.72) + 1, False)
    wn, _, n2 = _sweep([EXP], [lambda z: torch.exp(-z)], [2.0], 1, _bits(87.33) + 1, False, negate=True)
    print(f"exp over {n1 + n2} floats: worst bound fraction {max(wp[0], wn[0]):.3f} (budget 2 ulp)")


def test_log_every_positive_float_above_delta():
    """Protected log, log|a| for |a| > 0.001f, over every such positive float
    (and the negatives, which take |a|)."""
    d = np.float32(0.001)
    lo = _bits(d) + 1
    hi = _bits(np.finfo(np.float32).max) + 1
    worst, wabs, n = _sweep([LOG], [lambda z: torch.log(z.abs())], [3.0], lo, hi, True, SFU_LOG_ABS)
    print(f"log over {n} floats: worst bound fraction {worst[0]:.3f} (budget 3 ulp + 2^-21), max abs err "
          f"2^{np.log2(max(wabs[0], 1e-300)):.2f}")


def test_tanh_every_float_in_range():
    worst, wabs, n = _sweep([TANH], [torch.tanh], [2.0], 0, _bits(9.1) + 1, True)
    print(f"tanh over {n} floats: worst bound fraction {worst[0]:.3f} (budget 2 ulp)")


def test_pow_random_pairs():
    """pow(|a|, b) on 2^27 random pairs spanning 2^-30..2^30 bases and
    |b| <= 12, results in the normal FP32 range: |err| <= 4 * 2^-23 |r|."""
    import paper_2501_17168_b200 as evogp

    t = torch.tensor([[3, 1, 1]], dtype=torch.int16).cuda()
    v = torch.tensor([[POW, 0, 1]], dtype=torch.float32).cuda()
    s = torch.tensor([[3, 1, 1]], dtype=torch.int16).cuda()
    gen = torch.Generator(device="cuda").manual_seed(17)
    worst, n = 0.0, 0
    for _ in range(2):
        a = torch.exp2(torch.rand(CHUNK, device="cuda", generator=gen) * 60 - 30)
        a = torch.where(torch.rand(CHUNK, device="cuda", generator=gen) < 0.5, a, -a).float()
        b = ((torch.rand(CHUNK, device="cuda", generator=gen) * 24 - 12)).float()
        X = torch.stack([a, b], 1).contiguous()
        g = evogp.eval(t, v, s, X)[0, :, 0].double()
        r = torch.pow(a.double().abs(), b.double())
        ok = torch.isfinite(r) & (r.abs() >= 2.0 ** -126) & (r.abs() <= 3.4e38)
        q = ((g - r).abs()[ok] / (4.0 * TWO_M23 * r.abs()[ok])).max().item()
        worst = max(worst, q)
        assert q <= 1.0, q
        n += int(ok.sum())
    print(f"pow over {n} pairs: worst bound fraction {worst:.3f} (budget 4 ulp)")
