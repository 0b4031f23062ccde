"""The tent-transformed point sets (phi(x) = 1 - |1 - 2x|: "the random shift can be
replaced by the tent transformation") through the GPU path: points bit for bit against the oracle
(the map is evaluated as written in fp64 on both sides), every row of XA within the north_star 1e-12
bar, Q_N sums, the FFT levels (one map for the whole level), merged coarse levels, ranks."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_latency import check_fsum, check_rows, dev, rq  # noqa: F401

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("kind,b,m,shifted,world", [
    (W.KIND_LATTICE, 2, 13, False, 1), (W.KIND_LATTICE, 2, 12, True, 1), (W.KIND_LATTICE, 3, 8, False, 1),
    (W.KIND_NET, 2, 13, True, 1), (W.KIND_MC, 2, 12, False, 1), (W.KIND_LATTICE, 2, 13, False, 4)])
def test_tent_points_bit_exact(rq, kind, b, m, shifted, world):
    """A = I, so XA = X exactly: every row of Y equals the oracle's tent-mapped points bit for bit, and
    k_gen's values equal rqmc_points' (the per-entry debug path)."""
    s = 40
    prob = W.make_random(331 + kind + 7 * b + m + world, b, m, s, s, kind=kind, shifted=shifted,
                         mapping=W.MAP_TENT)
    prob.A = np.eye(s)
    g = 1 if world > 1 else 0
    pl = rq.Plan.from_problem(prob, rank=g, world=world)
    Yg = pl.xa(dev(prob.A)).cpu().numpy()
    ks = np.asarray(pl.global_rows())
    assert np.array_equal(Yg, oracle.points_rows(prob, ks))
    if world == 1:
        for idx, L in enumerate(pl.levels()):
            _, vals = pl.points(idx)
            js = slice(L["j_lo"], L["j_lo"] + L["s_w"])
            assert np.array_equal(Yg[:, js], vals.cpu().numpy()[ks % L["M"]]), f"level {idx}"


@pytest.mark.parametrize("seed,kind,b,m,s,tau,shifted,f,fft", [
    (341, W.KIND_LATTICE, 2, 14, 200, 72, False, W.F_EXP_MEAN, "0"),
    (342, W.KIND_LATTICE, 2, 14, 200, 72, False, W.F_MEAN_SQ, "1"),     # every coarse level on the FFT
    (343, W.KIND_LATTICE, 2, 13, 150, 40, True, W.F_CALL_MEAN_EXP, ""),
    (344, W.KIND_LATTICE, 3, 9, 120, 50, False, W.F_MEAN_SQ, ""),
    (345, W.KIND_NET, 2, 13, 120, 64, True, W.F_EXP_MEAN, ""),
    (346, W.KIND_MC, 2, 12, 100, 40, False, W.F_EXP_MEAN, ""),
])
def test_tent_xa_and_qn(rq, monkeypatch, seed, kind, b, m, s, tau, shifted, f, fft):
    monkeypatch.setenv("RQMC_FFT", fft)
    prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=shifted, mapping=W.MAP_TENT, f=f)
    pl = rq.Plan.from_problem(prob)
    if fft == "1":
        assert any(L["fft"] for L in pl.levels())
    Y, fs = pl.xa(dev(prob.A), prob.f, prob.fparam)
    torch.cuda.synchronize()
    ks = np.arange(prob.N)
    check_rows(prob, Y.cpu().numpy(), ks)
    check_fsum(prob, float(fs.item()), ks)


@pytest.mark.parametrize("G", [2, 3])
def test_tent_ranks(rq, G):
    b = 2 if G == 2 else 3
    prob = W.make_random(350 + G, b, 13 if b == 2 else 8, 90, 40, shifted=True, mapping=W.MAP_TENT, f=W.F_EXP_MEAN)
    A = dev(prob.A)
    tot = 0.0
    for g in range(G):
        p = rq.Plan.from_problem(prob, rank=g, world=G)
        Y, fs = p.xa(A, prob.f, prob.fparam)
        torch.cuda.synchronize()
        check_rows(prob, Y.cpu().numpy(), np.asarray(p.global_rows()))
        tot += float(fs.item())
    check_fsum(prob, tot, np.arange(prob.N))


def test_tent_batch(rq):
    """Batched shifts with the tent map: each replica equals the oracle's f-sum of that shift."""
    import dataclasses
    prob = W.make_random(360, 2, 12, 80, 48, shifted=True, mapping=W.MAP_TENT, f=W.F_EXP_MEAN)
    pl = rq.Plan.from_problem(prob)
    shifts = np.random.default_rng(3).random((3, prob.s))
    got = pl.qn_batch(dev(prob.A), prob.f, prob.fparam, shifts=shifts).cpu().numpy()
    for r in range(3):
        check_fsum(dataclasses.replace(prob, shift=shifts[r]), float(got[r]), np.arange(prob.N))
