"""Exhaustive accuracy pins of the interpreter's elementary functions against
the error model the oracle's certificate assumes (reading R14;
oracle/oracle.c `op_err`): for an op with result r the FP32 evaluation may
differ from the exact value by

    ulp_budget(f) * 2^-23 * |r|  (+ 2^-20 absolute for sin / cos, 2^-21 for log)

with ulp_budget = 2 (sin, cos, exp, tanh), 3 (log), 4 (tan, pow) — the CUDA
Math API's documented maximum ulp errors of sinf/cosf, expf, tanhf, tanf,
powf (the library-free exp / tanh forms of fastmath.cuh are held to the
same budgets), for sin/cos the SFU (sin.approx / cos.approx) absolute error
on the reduced argument, and for log the SFU form's (__logf: lg2.approx *
ln 2) documented 2^-21.41 absolute on [0.5, 2] / 3 ulp elsewhere. A
certified point is only as sound as these bounds,
so each is checked here on every FP32 argument of its working range (all
2.1e9 floats of [-pi, pi] for sin / cos, all of [-103.97, 88.7] for exp, all
positive floats above the protection threshold for log, all of [-9.1, 9.1]
for tanh) or, for the two-argument pow, on 3 x 2^26 random pairs — evaluated by
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


def _sweep(fids, refs, budgets, lo_bits, hi_bits, neg, abs_extra=0.0, negate=False, full_set=False):
    """refs see the generated floats x; the trees are evaluated at -x when
    negate. full_set: the same trees also through the full-set kernel
    variant (the generated PTX loop's bodies instead of the C++ loop's),
    bit-identical."""
    import paper_2501_17168_b200 as evogp

    t, v, s = _unary_trees(fids)
    worst = [0.0] * len(fids)  # max of err / (budget * 2^-23 * |r| + abs_extra + tiny)
    worst_abs = [0.0] * len(fids)
    n = 0
    for x in _floats(lo_bits, hi_bits, neg):
        xin = -x if negate else x
        out = evogp.eval(t, v, s, xin[:, None].contiguous())[:, :, 0]
        if full_set:
            with evogp.tuning_hint(full_set=True):
                out2 = evogp.eval(t, v, s, xin[:, None].contiguous())[:, :, 0]
            assert torch.equal(out.view(torch.int32), out2.view(torch.int32))
        out = out.double()
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


def test_exp_every_float_in_range():
    """exp over every FP32 argument whose result is finite and nonzero:
    [0, 88.72] and [-103.97, 0) (gradual underflow below -87.33: the
    budget's absolute FP32_TINY term covers the subnormal rounding)."""
    wp, _, n1 = _sweep([EXP], [torch.exp], [2.0], 0, _bits(88.72) + 1, False, full_set=True)
    wn, _, n2 = _sweep([EXP], [lambda z: torch.exp(-z)], [2.0], 1, _bits(103.97) + 1, False, negate=True,
                       full_set=True)
    print(f"exp over {n1 + n2} floats: worst bound fraction {max(wp[0], wn[0]):.3f} (budget 2 ulp)")


def test_log_every_positive_float_above_delta():
    """Protected log, log|a| for |a| > 0.001f, over every such positive float
    (and the negatives, which take |a|)."""
    d = np.float32(0.001)
    lo = _bits(d) + 1
    hi = _bits(np.finfo(np.float32).max) + 1
    worst, wabs, n = _sweep([LOG], [lambda z: torch.log(z.abs())], [3.0], lo, hi, True, SFU_LOG_ABS, full_set=True)
    print(f"log over {n} floats: worst bound fraction {worst[0]:.3f} (budget 3 ulp + 2^-21), max abs err "
          f"2^{np.log2(max(wabs[0], 1e-300)):.2f}")


def test_tanh_every_float_in_range():
    worst, wabs, n = _sweep([TANH], [torch.tanh], [2.0], 0, _bits(9.1) + 1, True, full_set=True)
    print(f"tanh over {n} floats: worst bound fraction {worst[0]:.3f} (budget 2 ulp)")


def test_exp_tanh_special_values():
    """The ends of the ranges and the IEEE specials, through both loops: exp
    overflows to inf past ln(FLT_MAX), underflows to 0 below -103.97, maps
    -inf to 0 and NaN to NaN; tanh saturates to +-1 (exactly) and keeps -0
    and NaN; each equal to the FP64 value rounded to FP32."""
    import paper_2501_17168_b200 as evogp

    xs = torch.tensor([0.0, -0.0, 1e-30, -1e-30, 88.7228, 88.7229, 89.0, 200.0, -87.4, -103.0, -103.98, -104.5,
                       -200.0, 9.0, 9.1, 50.0, -50.0, 0.625, -0.625, 0.62500006, float("inf"), float("-inf"),
                       float("nan")], dtype=torch.float32, device="cuda")
    t, v, s = _unary_trees([EXP, TANH])
    out = evogp.eval(t, v, s, xs[:, None].contiguous())[:, :, 0]
    with evogp.tuning_hint(full_set=True):
        out2 = evogp.eval(t, v, s, xs[:, None].contiguous())[:, :, 0]
    assert torch.equal(out.view(torch.int32), out2.view(torch.int32))
    for i, ref in enumerate((torch.exp, torch.tanh)):
        r = ref(xs.double()).float()
        g = out[i]
        same = (g == r) | (torch.isnan(g) & torch.isnan(r))
        close = (g.double() - r.double()).abs() <= 2 * TWO_M23 * r.double().abs() + FP32_TINY
        assert (same | close).all(), (i, xs[~(same | close)].tolist(), g[~(same | close)].tolist())
        zero = r == 0
        assert torch.equal(torch.signbit(g[zero]), torch.signbit(r[zero]))


def test_pow_random_pairs():
    """pow(|a|, b) on 2^27 random pairs in each of three families — bases
    2^-30..2^30 with |b| <= 12; bases within 1% of 1 with |b| <= 8000 (large
    exponents on small logarithms); bases over the whole FP32 range with
    |b| <= 1.2 — results in the normal FP32 range: |err| <= 4 * 2^-23 |r|;
    results beyond it overflow to inf / underflow to 0 where the exact value
    does by a margin. Both loops (C++ and the full-set variant) bit-identical."""
    import paper_2501_17168_b200 as evogp

    t = torch.tensor([[3, 1, 1]], dtype=torch.int16).cuda()
    v = torch.tensor([[POW, 0, 1]], dtype=torch.float32).cuda()
    s = torch.tensor([[3, 1, 1]], dtype=torch.int16).cuda()
    gen = torch.Generator(device="cuda").manual_seed(17)

    def rand(lo, hi):
        return torch.rand(CHUNK, device="cuda", generator=gen, dtype=torch.float64) * (hi - lo) + lo

    worst, n = 0.0, 0
    for fam in range(3):
        if fam == 0:
            a, b = torch.exp2(rand(-30, 30)), rand(-12, 12)
        elif fam == 1:
            a, b = 1 + rand(-0.01, 0.01), rand(-8000, 8000)
        else:
            a, b = torch.exp2(rand(-149, 128)), rand(-1.2, 1.2)
        a = torch.where(torch.rand(CHUNK, device="cuda", generator=gen) < 0.5, a, -a).float()
        b = b.float()
        X = torch.stack([a, b], 1).contiguous()
        g32 = evogp.eval(t, v, s, X)[0, :, 0]
        with evogp.tuning_hint(full_set=True):
            g2 = evogp.eval(t, v, s, X)[0, :, 0]
        assert torch.equal(g32.view(torch.int32), g2.view(torch.int32))
        tp = torch.pow(a.abs(), b)  # torch's FP32 pow (informational: fm_pow restates CUDA's powf)
        same_as_torch = int(((tp == g32) | (torch.isnan(tp) & torch.isnan(g32))).sum())
        g = g32.double()
        r = torch.pow(a.double().abs(), b.double())
        ok = torch.isfinite(r) & (r.abs() >= 2.0 ** -126) & (r.abs() <= 3.4e38)
        q = ((g - r).abs()[ok] / (4.0 * TWO_M23 * r.abs()[ok])).max().item()
        worst = max(worst, q)
        assert q <= 1.0, (fam, q)
        assert torch.isinf(g[r > 3.5e38]).all() and (g[r < 2.0 ** -151] == 0).all()
        n += int(ok.sum())
        print(f"pow family {fam}: {same_as_torch} of {CHUNK} bit-identical to torch.pow (float32)")
    print(f"pow over {n} pairs: worst bound fraction {worst:.3f} (budget 4 ulp)")


def test_pow_special_values():
    """C's powf on a non-negative base: b = 0 or |a| = 1 give 1 (even with a
    NaN operand), otherwise NaN operands give NaN, |a| = 0 gives 0 / inf,
    |a| = inf gives inf / 0, infinite exponents give 0 / inf / 1."""
    import paper_2501_17168_b200 as evogp

    nan, inf = float("nan"), float("inf")
    pairs = [(0.0, 2.0, 0.0), (-0.0, -2.0, inf), (0.0, 0.0, 1.0), (inf, 2.0, inf), (-inf, -2.0, 0.0),
             (nan, 0.0, 1.0), (-1.0, nan, 1.0), (nan, 1.0, nan), (2.0, nan, nan), (2.0, inf, inf), (0.5, inf, 0.0),
             (2.0, -inf, 0.0), (-1.0, inf, 1.0), (-3.0, 2.0, 9.0), (4.0, 0.5, 2.0), (2.0, 10.0, 1024.0),
             (2.0, 128.0, inf), (2.0, -149.0, 2.0 ** -149), (2.0, -151.0, 0.0), (1e-45, 1.0, 1.401298464324817e-45)]
    X = torch.tensor([[a, b] for a, b, _ in pairs], dtype=torch.float32, device="cuda")
    t = torch.tensor([[3, 1, 1]], dtype=torch.int16).cuda()
    v = torch.tensor([[POW, 0, 1]], dtype=torch.float32).cuda()
    s = torch.tensor([[3, 1, 1]], dtype=torch.int16).cuda()
    g = evogp.eval(t, v, s, X)[0, :, 0].cpu()
    with evogp.tuning_hint(full_set=True):
        g2 = evogp.eval(t, v, s, X)[0, :, 0].cpu()
    assert torch.equal(g.view(torch.int32), g2.view(torch.int32))
    exp = torch.tensor([e for _, _, e in pairs], dtype=torch.float32)
    ok = (g == exp) | (torch.isnan(g) & torch.isnan(exp))
    assert ok.all(), [(pairs[i], g[i].item()) for i in range(len(pairs)) if not ok[i]]
