"""GPU parity of evogp_tensorize_device (row a1 on the device, PAPER §III-A
P:221-258) against the oracle's independent tensorizer: valid rows byte for
byte (padding included), and for malformed trees the per-tree status equals
the code the oracle reports for that tree alone."""
import numpy as np
import pytest

import oracle
import synth
from tests.test_capi_cpu import _mutate

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _e():
    import paper_2501_17168_b200 as evogp

    return evogp


def _dev(offsets, types, values):
    return (torch.from_numpy(np.ascontiguousarray(offsets, np.int64)).cuda(),
            torch.from_numpy(np.ascontiguousarray(types, np.int16)).cuda(),
            torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda())


@pytest.mark.parametrize("mix,L,n_in,n_out,modi,P", [
    ("paper", 63, 4, 1, 0.0, 10000),
    ("full", 127, 8, 1, 0.0, 3000),
    ("full", 63, 17, 6, 0.1, 3000),
    ("ieee", 15, 2, 1, 0.0, 64),
    ("full", 1000, 3, 1, 0.0, 200),
])
def test_tensorize_device_bitexact(mix, L, n_in, n_out, modi, P):
    pt = synth.trees(5, 0, P, L, synth.MIXES[mix], n_in, n_out, modi)
    rt, rv, rs = oracle.tensorize(pt.offsets, pt.types, pt.values, L, n_in, n_out)
    t, v, s, st = _e().tensorize_device(*_dev(pt.offsets, pt.types, pt.values), L, n_in, n_out)
    assert (st.cpu().numpy() == 0).all()
    assert (t.cpu().numpy() == rt).all() and (s.cpu().numpy() == rs).all()
    assert (v.cpu().numpy().view(np.uint32) == rv.view(np.uint32)).all()


def test_tensorize_device_errors_match_oracle():
    rng = np.random.default_rng(1)
    n_in, n_out, L = 3, 4, 31
    base = synth.trees(3, 0, 600, L, synth.M_FULL, n_in, n_out, 0.1)
    offs, tys, vas, want = [0], [], [], []
    for it in range(600):
        ty, va = base.tree(it)
        if it % 5:
            ty, va = _mutate(rng, ty, va, n_in, n_out)
        if it % 97 == 0:  # too long / empty
            ty, va = (np.concatenate([ty] * 3), np.concatenate([va] * 3)) if it % 2 else (ty[:0], va[:0])
        off = np.array([0, len(ty)], np.int64)
        ref = oracle.tensorize(off, ty, va, L, n_in, n_out, raise_on_error=False)
        want.append(ref[0])
        tys.append(ty)
        vas.append(va)
        offs.append(offs[-1] + len(ty))
    t, v, s, st = _e().tensorize_device(*_dev(np.array(offs), np.concatenate(tys), np.concatenate(vas)), L, n_in,
                                        n_out)
    got = st.cpu().numpy()
    assert (got == np.array(want)).all(), np.nonzero(got != np.array(want))[0][:10]
    assert (got != 0).sum() > 300
    bad = got != 0
    assert (t.cpu().numpy()[bad] == -1).all() and (s.cpu().numpy()[bad] == 0).all()


def test_tensorize_device_rows_evaluate():
    """Device-tensorized rows feed evogp_sr_fitness exactly like host-tensorized ones."""
    e = _e()
    cfg = synth.CONFIGS["c2"]
    pt = synth.trees(cfg.seed, 0, 2000, cfg.max_len, synth.M_PAPER, cfg.n_in)
    X, y = synth.config_data(cfg)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    t, v, s, st = e.tensorize_device(*_dev(pt.offsets, pt.types, pt.values), cfg.max_len, cfg.n_in)
    h = [torch.from_numpy(a).cuda() for a in e.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in)]
    m1 = e.sr_fitness(t, v, s, Xd, yd).cpu().numpy()
    m2 = e.sr_fitness(*h, Xd, yd).cpu().numpy()
    assert (m1.view(np.uint64) == m2.view(np.uint64)).all()


@pytest.mark.parametrize("chunks", [1, 3, 4])
def test_host_streaming_sr_fitness_matches_one_pass(chunks):
    """The streaming public path (HostSRFitness: chunked H2D overlapped with
    device tensorize + fused fitness) returns exactly the one-pass MSEs."""
    e = _e()
    from paper_2501_17168_b200.stream import HostSRFitness

    cfg = synth.CONFIGS["c4"]
    P = 30001
    pt = synth.trees(cfg.seed, 0, P, cfg.max_len, synth.M_PAPER, cfg.n_in)
    X, y = synth.config_data(cfg)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    h = [torch.from_numpy(a).cuda() for a in e.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in)]
    ref = e.sr_fitness(*h, Xd, yd).cpu().numpy()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h_off, h_ty, h_va = pin(pt.offsets.astype(np.int64)), pin(pt.types), pin(pt.values)
    out = torch.empty(P, dtype=torch.float64).pin_memory()
    pipe = HostSRFitness(P, int(h_ty.numel()), cfg.max_len, cfg.n_in, Xd, yd, chunks=chunks)
    for _ in range(2):  # reuse across calls
        out.fill_(-1.0)
        got = pipe(h_off, h_ty, h_va, out).numpy()
        assert (got.view(np.uint64) == ref.view(np.uint64)).all()


@pytest.mark.parametrize("chunks", [1, 3])
def test_host_streaming_submit_two_in_flight(chunks):
    """HostSRFitness.submit with per-call host datasets: two populations (each
    with its own X / y) in flight at once, then a third reusing the first
    call's buffer sets; every result equals its one-pass MSEs bit for bit."""
    e = _e()
    from paper_2501_17168_b200.stream import HostSRFitness

    cfg = synth.CONFIGS["c4"]
    P = 20001
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    X, y = synth.config_data(cfg)
    cases = []
    for k in range(3):
        pt = synth.trees(cfg.seed + k, 0, P, cfg.max_len, synth.M_PAPER, cfg.n_in)
        Xk, yk = (X * (1.0 + 0.25 * k)).astype(np.float32), (y - 0.5 * k).astype(np.float32)
        Xd, yd = torch.from_numpy(Xk).cuda(), torch.from_numpy(yk).cuda()
        h = [torch.from_numpy(a).cuda() for a in e.tensorize(pt.offsets, pt.types, pt.values, cfg.max_len, cfg.n_in)]
        ref = e.sr_fitness(*h, Xd, yd).cpu().numpy()
        cases.append((pin(pt.offsets.astype(np.int64)), pin(pt.types), pin(pt.values), pin(Xk), pin(yk), ref))
    nodes = max(int(c[1].numel()) for c in cases)
    pipe = HostSRFitness(P, nodes, cfg.max_len, cfg.n_in, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(),
                         chunks=chunks)
    outs = [torch.full((P,), -1.0, dtype=torch.float64).pin_memory() for _ in cases]
    evs = [pipe.submit(*c[:3], outs[i], X=c[3], y=c[4]) for i, c in enumerate(cases[:2])]
    evs[0].synchronize()
    evs.append(pipe.submit(*cases[2][:3], outs[2], X=cases[2][3], y=cases[2][4]))
    for ev, out, c in zip(evs, outs, cases):
        ev.synchronize()
        got = out.numpy()
        assert (got.view(np.uint64) == c[5].view(np.uint64)).all()
