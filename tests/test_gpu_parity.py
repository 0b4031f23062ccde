"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star; SURVEY §8(c) "Tolerances"):
  * point indices / digit words: bit-exact; unit-map lattice/net values: bit-exact;
  * Y entries: |Y_gpu - Y_orc| <= 1e-12 * max(1, |x_k|_inf) * |A_{:,c}|_1;
  * exact-arithmetic regime (b = 2, dyadic shift <= 30 bits, small-integer A): bit-identical;
  * Q_N: relative 1e-12.
"""
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rq():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2305_11645_b200 import _build
    _build.build()
    import paper_2305_11645_b200 as rq
    return rq


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def y_tol(prob, X):
    """1e-12 * max(1, |x_k|_inf) * |A_c|_1 (rows of X = the points of the compared rows)."""
    xa = np.maximum(1.0, np.abs(X).max(axis=1))[:, None]
    return 1e-12 * xa * np.abs(prob.A).sum(axis=0)[None, :]


def check_y(prob, Yg, ks):
    Xs = oracle.points_rows(prob, ks)
    Yo = oracle.product(Xs, prob.A)
    err = np.abs(Yg - Yo)
    tol = y_tol(prob, Xs)
    bad = err > tol
    assert not bad.any(), f"max err/tol {np.max(err / tol):.3g} at {np.argwhere(bad)[:3]}"
    return float(np.max(err / np.maximum(tol, 1e-300)))


def run_xa(rq, prob, f=None, **plan_kw):
    p = rq.Plan.from_problem(prob, **plan_kw)
    A = dev(prob.A)
    ff = prob.f if f is None else f
    Y, fs = p.xa(A, ff, prob.fparam)
    torch.cuda.synchronize()
    return p, Y.cpu().numpy(), float(fs.item())


# ------------------------------------------------------------------ a2: points

@pytest.mark.parametrize("case", ["lat2", "lat2_shift_invnorm", "lat3_shift_invnorm", "net", "net_shift",
                                  "lat5_wbig_shift"])
def test_points_bit_exact(rq, case):
    if case == "lat2":
        prob = W.make_random(1, 2, 12, 100, 3)
    elif case == "lat2_shift_invnorm":
        prob = W.make_random(2, 2, 12, 100, 3, shifted=True, mapping=W.MAP_INVNORM)
    elif case == "lat3_shift_invnorm":
        prob = W.make_random(3, 3, 8, 90, 3, shifted=True, mapping=W.MAP_INVNORM)
    elif case == "net":
        prob = W.make_random(4, 2, 12, 100, 3, kind=W.KIND_NET)
    elif case == "net_shift":
        prob = W.make_random(5, 2, 12, 100, 3, kind=W.KIND_NET, shifted=True, mapping=W.MAP_INVNORM)
    else:
        prob = W.make_random(6, 5, 4, 40, 3, shifted=True, wmode="rand")
    p = rq.Plan.from_problem(prob)
    for idx, L in enumerate(p.levels()):
        words, vals = p.points(idx)
        words = words.cpu().numpy().view(np.uint64)
        vals = vals.cpu().numpy()
        Xo, To = oracle.points(prob, 0, L["M"])        # x_{k,j} depends on k mod M (k = r < M)
        js = slice(L["j_lo"], L["j_lo"] + L["s_w"])
        if prob.kind == W.KIND_LATTICE:
            scale = np.uint64(prob.N // L["M"]) if L["w"] < prob.m else np.uint64(1)
            exp_words = To[:, js] // scale if L["w"] < prob.m else np.zeros_like(To[:, js])
        else:
            exp_words = To[:, js]
        assert np.array_equal(words, exp_words), f"level {idx} words"
        if prob.map == W.MAP_UNIT:
            assert np.array_equal(vals, Xo[:, js]), f"level {idx} values"
        else:
            np.testing.assert_allclose(vals, Xo[:, js], rtol=4e-15, atol=4e-15)


# ------------------------------------------------------------------ exact regime: bit-identical

@pytest.mark.parametrize("seed,kind,m,s,tau,shifted,ckpt", [
    (11, W.KIND_LATTICE, 11, 63, 70, False, None),
    (12, W.KIND_LATTICE, 12, 130, 64, True, None),
    (13, W.KIND_NET, 11, 70, 33, True, None),
    (14, W.KIND_LATTICE, 13, 200, 129, True, "4"),
    (15, W.KIND_LATTICE, 13, 200, 129, True, "0"),
    (16, W.KIND_NET, 12, 64, 96, False, "7"),
])
def test_xa_exact_regime_bit_identical(rq, monkeypatch, seed, kind, m, s, tau, shifted, ckpt):
    """b=2, dyadic shift, |A| <= 8: every partial sum exact -> GPU == oracle bit for bit
    (SURVEY §8(c) exact-arithmetic regime); spans several tiles + ragged tails, several checkpoints."""
    if ckpt is not None:
        monkeypatch.setenv("RQMC_CKPT_W", ckpt)
    prob = W.make_random(seed, 2, m, s, tau, kind=kind, shifted=shifted, int_a=True, f=W.F_MEAN)
    p, Y, fs = run_xa(rq, prob)
    Yo = oracle.xa(prob)
    assert np.array_equal(Y, Yo)
    q = oracle.qn_sum(prob)
    assert abs(fs - q) <= 1e-12 * max(1.0, abs(q))


def test_identity_matrix_returns_points(rq):
    """A = I_s: XA = X, so the whole path (levels, tiles, stores) returns the points bit-exactly."""
    prob = W.make_random(21, 2, 10, 48, 48, shifted=True)
    prob.A = np.eye(48)
    pl = rq.Plan.from_problem(prob)
    Yg = pl.xa(dev(prob.A)).cpu().numpy()
    X, _ = oracle.points(prob)
    assert np.array_equal(Yg, X)


@pytest.mark.parametrize("kind,b,m,shifted,world", [
    (W.KIND_LATTICE, 2, 13, True, 1), (W.KIND_LATTICE, 2, 12, False, 1), (W.KIND_LATTICE, 3, 8, True, 1),
    (W.KIND_NET, 2, 13, True, 1), (W.KIND_NET, 2, 12, False, 1), (W.KIND_MC, 2, 12, False, 1),
    (W.KIND_NET, 2, 13, True, 3), (W.KIND_LATTICE, 2, 13, True, 4)])
def test_identity_matrix_mapped_points(rq, kind, b, m, shifted, world):
    """Phi^-1-mapped points through k_gen (AS 241, tails evaluated from the per-warp queue): with A = I,
    XA = X exactly, so every row of Y must equal (bit for bit) the same point from rqmc_points (one
    entry per thread, no queue) and the oracle's points within 4e-15.  A misplaced queued entry, a lost
    flush or a padding column written as a point fails it.  world > 1: rank 1's rows (the generic loop
    for nets with grouped classes, nc > 1)."""
    s = 40
    prob = W.make_random(31 + kind + 7 * b + m + world, b, m, s, s, kind=kind, shifted=shifted,
                         mapping=W.MAP_INVNORM)
    prob.A = np.eye(s)
    g = 1 if world > 1 else 0
    pl = rq.Plan.from_problem(prob, rank=g, world=world)
    Yg = pl.xa(dev(prob.A)).cpu().numpy()
    ks = pl.global_rows()
    Xo = oracle.points_rows(prob, ks)
    np.testing.assert_allclose(Yg, Xo, rtol=4e-15, atol=4e-15)
    if world == 1:
        for idx, L in enumerate(pl.levels()):
            _, vals = pl.points(idx)
            vals = vals.cpu().numpy()
            js = slice(L["j_lo"], L["j_lo"] + L["s_w"])
            assert np.array_equal(Yg[:, js], vals[ks % L["M"]]), f"level {idx}"


def test_golden_g1_through_gpu(rq):
    """SURVEY G1 (P:307-309 by hand) through the GPU path, bit-exact."""
    A = np.array([[1, 2], [-1, 0], [2, -3]], dtype=np.float64)
    pl = rq.Plan(2, 3, 3, 2, [0, 1, 2], z=[3, 1, 1])
    Y = pl.xa(dev(A)).cpu().numpy()
    exp = np.array([[0, 0], [9 / 8, -3 / 4], [1 / 4, 3 / 2], [3 / 8, -5 / 4], [1 / 2, 1], [13 / 8, 1 / 4],
                    [-1 / 4, 1 / 2], [7 / 8, -1 / 4]])
    assert np.array_equal(Y, exp)


# ------------------------------------------------------------------ general: tolerance sweep

def _sweep_cases():
    cases = []
    rng = np.random.default_rng(2024)
    for i in range(40):
        b = int(rng.choice([2, 2, 3, 5]))
        mmax = {2: 11, 3: 7, 5: 4}[b]
        m = int(rng.integers(1, mmax + 1))
        s = int(rng.integers(1, 65))
        tau = int(rng.integers(1, 140))
        kind = W.KIND_NET if (b == 2 and rng.random() < 0.3) else W.KIND_LATTICE
        shifted = bool(rng.random() < 0.6)
        mapping = W.MAP_INVNORM if rng.random() < 0.5 else W.MAP_UNIT
        wmode = ["log", "rand", "zero"][int(rng.integers(0, 3))]
        f = int(rng.integers(0, 4))
        cases.append((1000 + i, b, m, s, tau, kind, shifted, mapping, wmode, f))
    return cases


@pytest.mark.parametrize("seed,b,m,s,tau,kind,shifted,mapping,wmode,f", _sweep_cases())
def test_xa_qn_sweep(rq, seed, b, m, s, tau, kind, shifted, mapping, wmode, f):
    """SPEC S:673-674 property sweep (b in {2,3,5}, m small, s <= 64, ragged tau, w > m, shifts)."""
    prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=shifted, mapping=mapping, wmode=wmode, f=f)
    p, Y, fs = run_xa(rq, prob)
    check_y(prob, Y, np.arange(prob.N))
    fo = oracle.f_rows(prob, np.arange(prob.N))
    q = oracle.neumaier(fo)
    assert abs(fs - q) <= 1e-12 * max(1e-300, np.abs(fo).sum()), (fs, q)
    # qn (no Y) equals the fused f of xa
    fs2 = float(p.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    assert abs(fs2 - fs) <= 1e-13 * max(1e-300, abs(fs))


@pytest.mark.parametrize("case", ["m1_s1_tau1", "tau1_s200", "s1_tau300", "w_beyond_m", "w_beyond_m_shift",
                                  "all_zero_w_b5", "A_zero", "rowzero_m1"])
def test_degenerate_shapes(rq, case):
    """Degenerate cases of the method: N = b, one coordinate, one column, every w_j >= m for j > 1
    (s* = 1: zero columns dropped, or constant columns under a shift, reading C-4), the dense product
    (all w_j = 0), A = 0 (Y = 0, Q_N = F(0) exactly), a 1-digit row-zeroed net."""
    kw = dict(kind=W.KIND_LATTICE, shifted=False, mapping=W.MAP_UNIT, wmode="log", f=W.F_EXP_MEAN)
    b, m, s, tau = 2, 1, 1, 1
    if case == "tau1_s200":
        b, m, s, tau = 2, 10, 200, 1
    elif case == "s1_tau300":
        b, m, s, tau = 3, 6, 1, 300
    elif case in ("w_beyond_m", "w_beyond_m_shift"):
        b, m, s, tau = 2, 3, 40, 17
        kw.update(shifted=case.endswith("shift"), mapping=W.MAP_INVNORM)
    elif case == "all_zero_w_b5":
        b, m, s, tau = 5, 3, 30, 20
        kw.update(wmode="zero", shifted=True)
    elif case == "A_zero":
        b, m, s, tau = 2, 9, 50, 33
        kw.update(shifted=True, mapping=W.MAP_INVNORM)
    elif case == "rowzero_m1":
        b, m, s, tau = 2, 1, 6, 5
        kw.update(kind=W.KIND_NET_ROWS, shifted=True)
    prob = W.make_random(77, b, m, s, tau, **kw)
    if case == "A_zero":
        prob.A[:] = 0.0
    p, Y, fs = run_xa(rq, prob)
    if case == "A_zero":
        assert not Y.any() and fs == float(prob.N)        # exp(mean 0) = 1 per point, exactly
        return
    check_y(prob, Y, np.arange(prob.N))
    fo = oracle.f_rows(prob, np.arange(prob.N))
    assert abs(fs - oracle.neumaier(fo)) <= 1e-12 * max(1e-300, np.abs(fo).sum())


def test_qn_host_alternating_inputs(rq):
    """rqmc_qn_host's A upload runs on a copy stream and the GEMMs wait on its event while every
    kernel uses programmatic dependent launch: alternating two different host A (8 MB each) call after
    call must give each A's own result every time (a GEMM that read A before its copy completed
    would return the other matrix's sum)."""
    prob = W.make_config("C3")
    A1 = np.ascontiguousarray(prob.A)
    A2 = np.ascontiguousarray(prob.A[::-1] * 1.5)
    pl = rq.Plan.from_problem(prob)
    ref = [float(pl.qn_sum(dev(A), prob.f, prob.fparam).item()) for A in (A1, A2)]
    assert abs(ref[0] - ref[1]) > 1e-6 * abs(ref[0])
    for i in range(24):
        got = pl.qn_host(A1 if i % 2 == 0 else A2, prob.f, prob.fparam)
        assert abs(got - ref[i % 2]) <= 1e-13 * abs(ref[i % 2]), (i, got, ref)


@pytest.mark.parametrize("seed,m,s,tau,f,shifted", [(61, 11, 100, 40, W.F_MEAN_SQ, True),     # Tree<3, 3>
                                                   (62, 11, 81, 70, W.F_CALL_MEAN_EXP, True),  # Tree<3, 3>
                                                   (63, 10, 100, 50, W.F_EXP_MEAN, False)])   # Tree<2, 3>
def test_b3_tail_split_combine(rq, monkeypatch, seed, m, s, tau, f, shifted):
    """b = 3 trees split the last, at most half-full wave of bundles over two CTAs by column halves
    (row sums met in scratch, F applied by the second to finish).  RQMC_FORCE_SPLIT=1 splits every
    bundle: Y, the fused sum and repeated calls (counters reset) must match the oracle."""
    monkeypatch.setenv("RQMC_FORCE_SPLIT", "1")
    prob = W.make_random(seed, 3, m, s, tau, shifted=shifted, mapping=W.MAP_INVNORM, f=f)
    p, Y, fs = run_xa(rq, prob)
    check_y(prob, Y, np.arange(prob.N))
    fo = oracle.f_rows(prob, np.arange(prob.N))
    q = oracle.neumaier(fo)
    assert abs(fs - q) <= 1e-12 * max(1e-300, np.abs(fo).sum())
    A = dev(prob.A)
    for _ in range(3):
        fs2 = float(p.qn_sum(A, prob.f, prob.fparam).item())
        assert abs(fs2 - q) <= 1e-12 * max(1e-300, np.abs(fo).sum())


def test_unaligned_lda_path(rq):
    """Odd lda / odd tau (8-byte cp.async path) and a column-sliced A view."""
    prob = W.make_random(55, 2, 10, 40, 67, shifted=True, mapping=W.MAP_INVNORM)
    big = np.zeros((40, 71))
    big[:, 1:68] = prob.A
    Abig = dev(big)
    Aview = Abig[:, 1:68]
    pl = rq.Plan.from_problem(prob)
    Y, fs = pl.xa(Aview, W.F_EXP_MEAN)
    check_y(prob, Y.cpu().numpy(), np.arange(prob.N))


# ------------------------------------------------------------------ multi-rank (simulated on one GPU)

@pytest.mark.parametrize("b,m,G", [(2, 12, 2), (2, 12, 4), (2, 12, 8), (3, 7, 3), (3, 7, 9),
                                   (3, 7, 2), (3, 7, 4), (3, 7, 8), (2, 12, 3), (2, 12, 6)])
def test_simulated_ranks(rq, b, m, G):
    """Run plan(rank=g, world=G) for every g on one GPU: local rows are the rank's residue classes
    (k = g + G i when G is a power of b, contiguous groups of b^gamma classes otherwise) and the sum
    of the partial f-sums equals the world = 1 result (SURVEY §4 multi-GPU (ii))."""
    prob = W.make_random(300 + G, b, m, 50, 40, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    A = dev(prob.A)
    full_p = rq.Plan.from_problem(prob)
    Yf, sf = full_p.xa(A, prob.f, prob.fparam)
    Yf = Yf.cpu().numpy()
    tot = 0.0
    for g in range(G):
        pg = rq.Plan.from_problem(prob, rank=g, world=G)
        Yg, sg = pg.xa(A, prob.f, prob.fparam)
        ks = pg.global_rows()
        np.testing.assert_allclose(Yg.cpu().numpy(), Yf[ks], rtol=0, atol=1e-13 * np.abs(Yf).max())
        tot += float(sg.item())
    assert abs(tot - float(sf.item())) <= 1e-12 * abs(float(sf.item()))


# ------------------------------------------------------------------ end-to-end host entry

def test_qn_host_matches_device(rq):
    prob = W.make_config("C2")
    pl = rq.Plan.from_problem(prob)
    d = float(pl.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    h = pl.qn_host(prob.A, prob.f, prob.fparam)
    assert h == d


# ------------------------------------------------------------------ BASELINE configs

def test_config_c1(rq):
    prob = W.make_config("C1")
    p, Y, fs = run_xa(rq, prob)
    check_y(prob, Y, np.arange(prob.N))
    q = oracle.qn_sum(prob)
    assert abs(fs - q) <= 1e-12 * abs(q)


def test_config_c2(rq):
    prob = W.make_config("C2")
    pl = rq.Plan.from_problem(prob)
    fs = float(pl.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    q = oracle.qn_sum(prob)                      # full naive oracle, 4.3e9 MACs
    assert abs(fs - q) <= 1e-12 * abs(q)


def _sample_rows(N, n_rand, seed, extra=()):
    rng = np.random.default_rng(seed)
    ks = np.concatenate([np.arange(min(256, N)), np.arange(max(0, N - 256), N), rng.integers(0, N, n_rand),
                         np.asarray(extra, dtype=np.int64)])
    return np.unique(ks)


def test_config_c3(rq):
    prob = W.make_config("C3")
    pl = rq.Plan.from_problem(prob)
    A = dev(prob.A)
    Y, fs = pl.xa(A, prob.f, prob.fparam)
    ks = _sample_rows(prob.N, 1500, 3)
    check_y(prob, Y[torch.from_numpy(ks).cuda()].cpu().numpy(), ks)
    fq = float(pl.qn_sum(A, prob.f, prob.fparam).item())
    assert fq == float(fs.item())
    del Y
    q = oracle.neumaier(oracle.f_all_meanid_tab(prob))   # O3' over all 2^20 rows
    assert abs(fq - q) <= 1e-12 * abs(q)


def test_config_c4(rq):
    prob = W.make_config("C4")
    pl = rq.Plan.from_problem(prob)
    A = dev(prob.A)
    Y, fs = pl.xa(A, prob.f, prob.fparam)            # Y stored: 17.4 GB
    ks = _sample_rows(prob.N, 300, 4)
    Ys = Y[torch.from_numpy(ks).cuda()].cpu().numpy()
    check_y(prob, Ys, ks)
    fo = oracle.f_rows(prob, ks)
    np.testing.assert_allclose(oracle.f_of_y(Ys, prob.f, prob.fparam), fo, rtol=1e-12)
    # the fused f equals f applied to the stored Y (fp64 on the device, fixed order)
    fy = (Y * Y).mean(dim=1).sum().item()
    assert abs(float(fs.item()) - fy) <= 1e-12 * abs(fy)
    del Y


def test_config_c5_qn_full(rq):
    """C5 at full size in the bench's launch configuration: Q_N over all 2^24 points against the
    oracle's O3' (g = id) computed on every row."""
    prob = W.make_config("C5")
    pl = rq.Plan.from_problem(prob)
    fs = float(pl.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    q = oracle.neumaier(oracle.f_all_meanid_tab(prob))
    assert abs(fs - q) <= 1e-12 * abs(q), (fs, q)


def test_config_c5_rank_partition(rq):
    """C5 at full size under the multi-GPU residue partition: for G = 2, 4, 8
    the ranks' local f-sums add up to the single-GPU sum, and rank g of G = 8 stores its full 34 GB
    share of Y (rows k = g + 8 i, all 2048 columns): its first 64 rows and 256 seeded rows match the
    oracle."""
    prob = W.make_config("C5")
    A = dev(prob.A)
    one = float(rq.Plan.from_problem(prob).qn_sum(A, prob.f, prob.fparam).item())
    for G in (2, 4, 8):
        tot = sum(float(rq.Plan.from_problem(prob, rank=g, world=G).qn_sum(A, prob.f, prob.fparam).item())
                  for g in range(G))
        assert abs(tot - one) <= 1e-12 * abs(one), (G, tot, one)
    g, G = 5, 8
    pl = rq.Plan.from_problem(prob, rank=g, world=G)
    Y, fs = pl.xa(A, prob.f, prob.fparam)
    rng = np.random.default_rng(11)
    loc = np.unique(np.concatenate([np.arange(64), rng.integers(0, prob.N // G, 256)])).astype(np.int64)
    Ys = Y[torch.from_numpy(loc).cuda()].cpu().numpy()
    del Y
    torch.cuda.empty_cache()
    check_y(prob, Ys, g + G * loc)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_config_c4_grouped_ranks(rq, G):
    """C4 (b = 3) on G = 2, 4, 8 ranks: ncls = 3^gamma >= 32 G residue classes in contiguous groups
    (SURVEY §8(e)).  Per rank the fused f-sum of rqmc_xa (Y stored, N_local rows); the G sums add up to
    the single-GPU sum, and rank G-1's first 64 and 128 seeded local rows match the oracle."""
    prob = W.make_config("C4")
    A = dev(prob.A)
    one = float(rq.Plan.from_problem(prob).qn_sum(A, prob.f, prob.fparam).item())
    tot = 0.0
    for g in range(G):
        pl = rq.Plan.from_problem(prob, rank=g, world=G)
        Y, fs = pl.xa(A, prob.f, prob.fparam)
        tot += float(fs.item())
        if g == G - 1:
            loc = np.unique(np.concatenate([np.arange(64), np.random.default_rng(G).integers(0, len(Y), 128)]))
            Ys = Y[torch.from_numpy(loc.astype(np.int64)).cuda()].cpu().numpy()
            check_y(prob, Ys, pl.global_rows()[loc])
        del Y
        torch.cuda.empty_cache()
    assert abs(tot - one) <= 1e-12 * abs(one), (G, tot, one)


def test_config_c5_panel_rows(rq):
    """C5 points/levels with a 64-column panel of A stored (8.6 GB), sampled rows vs the oracle."""
    prob = W.make_config("C5")
    prob.A = np.ascontiguousarray(prob.A[:, 1000:1064])
    prob.tau = 64
    pl = rq.Plan.from_problem(prob)
    Y = pl.xa(dev(prob.A))
    ks = _sample_rows(prob.N, 600, 5)
    check_y(prob, Y[torch.from_numpy(ks).cuda()].cpu().numpy(), ks)


def test_coarse_pair_fusion_bit_identical(rq, monkeypatch):
    """Opt-in fused coarse pairs (parent R kept on chip, RQMC_GEMM_PAIR=1) reproduce the two-launch
    result bit for bit (same accumulation order), incl. a b = 3 plan and several checkpoints."""
    import subprocess
    import sys
    code = ("import numpy as np, torch, workloads as W, paper_2305_11645_b200 as rq\n"
            "out = []\n"
            "for seed, b, m, ck in ((41, 2, 13, '5'), (42, 3, 8, '3'), (43, 2, 12, '')):\n"
            "    prob = W.make_random(seed, b, m, 200, 70, shifted=True, mapping=W.MAP_INVNORM)\n"
            "    import os; os.environ['RQMC_CKPT_W'] = ck\n"
            "    pl = rq.Plan.from_problem(prob)\n"
            "    Y, fs = pl.xa(torch.from_numpy(prob.A).cuda(), prob.f, prob.fparam)\n"
            "    out.append(Y.cpu().numpy())\n"
            "np.save(__import__('sys').argv[1], np.concatenate([o.ravel() for o in out]))\n")
    import os
    import tempfile
    res = []
    for flag in ("0", "1"):
        f = os.path.join(tempfile.mkdtemp(), "y.npy")
        env = dict(os.environ, RQMC_GEMM_PAIR=flag)
        subprocess.run([sys.executable, "-c", code, f], check=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        res.append(np.load(f))
    assert np.array_equal(res[0], res[1])


def test_graph_replay_matches_direct(rq):
    """Single runs are captured once as a CUDA graph and replayed: replays equal the first (captured)
    run bit for bit, see in-place changes of A (the graph reads memory at execution), and a profiled
    run (direct launches) gives the same bits."""
    prob = W.make_random(61, 2, 12, 120, 96, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    pl = rq.Plan.from_problem(prob)
    A = dev(prob.A)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    first = float(pl.qn_sum(A, prob.f, prob.fparam, out=out).item())
    again = float(pl.qn_sum(A, prob.f, prob.fparam, out=out).item())
    assert first == again
    pl.profile_enable(1)
    direct = float(pl.qn_sum(A, prob.f, prob.fparam, out=out).item())
    pl.profile_enable(0)
    assert direct == first
    A.mul_(0.5)                                   # same pointer, new contents
    half = float(pl.qn_sum(A, prob.f, prob.fparam, out=out).item())
    prob.A = prob.A * 0.5
    q = oracle.qn_sum(prob)
    assert half != first and abs(half - q) <= 1e-12 * abs(q)
    # xa with Y through the graph path, twice
    Y1, s1 = pl.xa(A, prob.f, prob.fparam)
    Y2, s2 = pl.xa(A, prob.f, prob.fparam, Y=Y1.clone())
    assert torch.equal(Y1, Y2)


def test_graph_cache_many_keys_and_pageable_host(rq):
    """More distinct argument sets than the graph cache holds (eviction path) all give the direct
    result; rqmc_qn_host with a pageable (non-pinned) host A equals the device call."""
    prob = W.make_random(62, 2, 11, 80, 40, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    pl = rq.Plan.from_problem(prob)
    base = dev(prob.A)
    pl.profile_enable(1)
    ref = float(pl.qn_sum(base, prob.f, prob.fparam).item())   # profiled: direct launches
    pl.profile_enable(0)
    outs = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(11)]
    for rep in range(2):
        for o in outs:
            assert float(pl.qn_sum(base, prob.f, prob.fparam, out=o).item()) == ref
    h = pl.qn_host(np.array(prob.A, copy=True), prob.f, prob.fparam)   # pageable numpy memory
    assert h == ref


@pytest.mark.parametrize("G", [2, 4, 3])
def test_batch_simulated_ranks(rq, G):
    """Batched shifts under the residue partition: per rank and replica, the partial sums over the
    G ranks add up to the world = 1 batch result."""
    prob = W.make_random(70 + G, 2, 12, 60, 40, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    rng = np.random.default_rng(G)
    shifts = rng.random((5, prob.s))
    A = dev(prob.A)
    full = rq.Plan.from_problem(prob).qn_batch(A, prob.f, prob.fparam, shifts=shifts).cpu().numpy()
    tot = np.zeros(5)
    for g in range(G):
        tot += rq.Plan.from_problem(prob, rank=g, world=G).qn_batch(A, prob.f, prob.fparam,
                                                                     shifts=shifts).cpu().numpy()
    np.testing.assert_allclose(tot, full, rtol=1e-12)


@pytest.mark.parametrize("seed,b,m,s,tau,kind,shifted,wmode", [(71, 2, 10, 32, 32, W.KIND_LATTICE, False, "log"),
                                                              (72, 2, 11, 60, 40, W.KIND_NET, True, "log"),
                                                              (73, 3, 7, 50, 30, W.KIND_LATTICE, True, "rand"),
                                                              (74, 2, 10, 40, 24, W.KIND_MC, False, "log")])
def test_absorbed_coarse_levels(rq, monkeypatch, seed, b, m, s, tau, kind, shifted, wmode):
    """Small unit-map problems merge their top coarse levels into one GEMM (per-coordinate periods in
    k_gen): at least one level is absorbed, Y matches the oracle on every row and the unmerged run
    (RQMC_ABSORB=0) to 1e-12, the f-sums likewise."""
    prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=shifted, mapping=W.MAP_UNIT, wmode=wmode,
                         f=W.F_EXP_MEAN)
    A = dev(prob.A)
    monkeypatch.setenv("RQMC_ABSORB", "")
    p1 = rq.Plan.from_problem(prob)
    assert any(L["absorbed"] for L in p1.levels())
    Y1, s1 = p1.xa(A, prob.f, prob.fparam)
    monkeypatch.setenv("RQMC_ABSORB", "0")
    p0 = rq.Plan.from_problem(prob)
    assert not any(L["absorbed"] for L in p0.levels())
    Y0, s0 = p0.xa(A, prob.f, prob.fparam)
    check_y(prob, Y1.cpu().numpy(), np.arange(prob.N))
    np.testing.assert_allclose(Y1.cpu().numpy(), Y0.cpu().numpy(), rtol=0, atol=1e-13 * np.abs(prob.A).sum(0).max())
    fo = oracle.f_rows(prob, np.arange(prob.N))
    assert abs(float(s1.item()) - oracle.neumaier(fo)) <= 1e-12 * np.abs(fo).sum()


def test_fft_levels_single_process_only(rq, monkeypatch):
    """Reading FFT-2: the FFT product computes every row of a level, so multi-rank plans keep the GEMM
    for those levels; the ranks' sums still add up to the world-1 (FFT) result."""
    monkeypatch.setenv("RQMC_FFT", "1")
    prob = W.make_random(88, 2, 13, 120, 48, shifted=False, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    A = dev(prob.A)
    one = rq.Plan.from_problem(prob)
    assert any(L["fft"] for L in one.levels())
    ref = float(one.qn_sum(A, prob.f, prob.fparam).item())
    tot = 0.0
    for g in range(4):
        pg = rq.Plan.from_problem(prob, rank=g, world=4)
        assert not any(L["fft"] for L in pg.levels())
        tot += float(pg.qn_sum(A, prob.f, prob.fparam).item())
    assert abs(tot - ref) <= 1e-12 * abs(ref)
