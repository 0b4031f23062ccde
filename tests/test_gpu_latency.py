"""Latency regime of small problems (SURVEY §7 hard part 10; C2): the 32 x 32-tile coarse GEMM
(k_level_gemm_lat) and coarse levels merged by gather -- Φ^-1-mapped points keep each level's own X^red
and the merged GEMM reads column q of level i at row r mod M_i (x_{r,j} depends on r mod M_j,
PAPER.md P:307-309).  Every row of Y against the CPU oracle (north_star bar 1e-12), the f-sums against
the oracle's Q_N sum, and against the unmerged run."""
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


def check_rows(prob, Yg, ks):
    Xs = oracle.points_rows(prob, ks)
    Yo = oracle.product(Xs, prob.A)
    tol = 1e-12 * np.maximum(1.0, np.abs(Xs).max(axis=1))[:, None] * np.abs(prob.A).sum(axis=0)[None, :]
    err = np.abs(Yg - Yo)
    assert not (err > tol).any(), f"max err/tol {np.max(err / tol):.3g}"


def check_fsum(prob, fs, ks):
    fo = oracle.f_rows(prob, ks)
    assert abs(fs - oracle.neumaier(fo)) <= 1e-12 * np.abs(fo).sum()


GATHER = [  # seed, b, m, s, tau, kind, shifted, f
    (201, 2, 12, 150, 48, W.KIND_LATTICE, True, W.F_CALL_MEAN_EXP),   # C2 shape: levels 7, 6, 5 merged
    (202, 3, 7, 60, 30, W.KIND_LATTICE, True, W.F_MEAN_SQ),
    (203, 2, 11, 90, 33, W.KIND_LATTICE, True, W.F_EXP_MEAN),          # odd tau: 8-byte A loads
    (204, 2, 11, 70, 40, W.KIND_NET, True, W.F_EXP_MEAN),
    (205, 2, 11, 70, 40, W.KIND_MC, False, W.F_EXP_MEAN),
    (206, 2, 12, 100, 40, W.KIND_LATTICE, False, W.F_MEAN),
    (207, 2, 15, 256, 64, W.KIND_LATTICE, True, W.F_CALL_MEAN_EXP),   # + 3 fused fine levels (tree)
    (208, 3, 9, 200, 64, W.KIND_LATTICE, True, W.F_MEAN_SQ),          # + 1 fine level (k_fine)
]


@pytest.mark.parametrize("seed,b,m,s,tau,kind,shifted,f", GATHER)
def test_gather_merged_levels(rq, monkeypatch, seed, b, m, s, tau, kind, shifted, f):
    """Φ^-1-mapped small problems merge their top coarse levels by gather: at least one level is
    absorbed, every row of Y matches the oracle, Y matches the unmerged run (RQMC_ABSORB=0) to 1e-13 of
    |A_c|_1, the f-sum matches the oracle."""
    monkeypatch.setenv("RQMC_FFT", "0")
    prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=shifted, mapping=W.MAP_INVNORM, f=f)
    A = dev(prob.A)
    monkeypatch.setenv("RQMC_ABSORB", "")
    p1 = rq.Plan.from_problem(prob)
    assert any(L["absorbed"] for L in p1.levels())
    Y1, s1 = p1.xa(A, prob.f, prob.fparam)
    monkeypatch.setenv("RQMC_ABSORB", "0")
    p0 = rq.Plan.from_problem(prob)
    assert not any(L["absorbed"] for L in p0.levels())
    Y0, _ = p0.xa(A, prob.f, prob.fparam)
    torch.cuda.synchronize()
    ks = np.arange(prob.N)
    check_rows(prob, Y1.cpu().numpy(), ks)
    np.testing.assert_allclose(Y1.cpu().numpy(), Y0.cpu().numpy(), rtol=0,
                               atol=1e-13 * np.abs(prob.A).sum(0).max() * 8)
    check_fsum(prob, float(s1.item()), ks)


@pytest.mark.parametrize("G", [2, 4])
def test_gather_merged_levels_ranks(rq, monkeypatch, G):
    """Merged-by-gather coarse levels under the residue partition: each simulated rank's rows of Y (its
    global rows) match the oracle and the rank sums add up to the oracle's f-sum."""
    monkeypatch.setenv("RQMC_ABSORB", "")
    prob = W.make_random(210 + G, 2, 12, 150, 40, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    A = dev(prob.A)
    tot = 0.0
    for g in range(G):
        p = rq.Plan.from_problem(prob, rank=g, world=G)
        assert any(L["absorbed"] for L in p.levels())
        Y, fs = p.xa(A, prob.f, prob.fparam)
        torch.cuda.synchronize()
        rows = np.asarray(p.global_rows())
        check_rows(prob, Y.cpu().numpy(), rows)
        tot += float(fs.item())
    check_fsum(prob, tot, np.arange(prob.N))


def test_gather_merged_levels_batch(rq, monkeypatch):
    """A small batch (replicas in the grid's z dimension) merges by gather too: each replica equals the
    single run of its shift bit for bit (same layout) and the oracle's f-sum."""
    import dataclasses
    monkeypatch.setenv("RQMC_ABSORB", "")
    prob = W.make_random(220, 2, 11, 130, 32, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    A = dev(prob.A)
    p = rq.Plan.from_problem(prob)
    shifts = np.random.default_rng(5).random((2, prob.s))
    got = p.qn_batch(A, prob.f, prob.fparam, shifts=shifts).cpu().numpy()
    same = p.summary_batch(2, prob.f)["checkpoint"] == p.summary()["checkpoint"]
    for r in range(2):
        pr = dataclasses.replace(prob, shift=shifts[r])
        single = rq.Plan.from_problem(pr)
        assert any(L["absorbed"] for L in single.levels())
        one = float(single.qn_sum(A, prob.f, prob.fparam).item())
        if same:
            assert got[r] == one
        check_fsum(pr, float(got[r]), np.arange(pr.N))


@pytest.mark.parametrize("seed,b,m,s,tau,kind,shifted,wmode", [
    (230, 2, 9, 40, 30, W.KIND_LATTICE, True, "rand"),
    (231, 3, 6, 30, 70, W.KIND_LATTICE, False, "log"),
    (232, 2, 10, 64, 64, W.KIND_NET, True, "log"),
    (233, 2, 8, 20, 16, W.KIND_MC, False, "rand"),
])
def test_latency_gemm_forced(rq, monkeypatch, seed, b, m, s, tau, kind, shifted, wmode):
    """RQMC_GEMM_LAT=1 puts every coarse GEMM on the 32 x 32-tile kernel (ragged K, odd tau, parents,
    unit and Φ^-1 maps): every row against the oracle."""
    monkeypatch.setenv("RQMC_GEMM_LAT", "1")
    for mp in (W.MAP_UNIT, W.MAP_INVNORM):
        prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=shifted, mapping=mp, wmode=wmode,
                             f=W.F_EXP_MEAN)
        p = rq.Plan.from_problem(prob)
        Y, fs = p.xa(dev(prob.A), prob.f, prob.fparam)
        torch.cuda.synchronize()
        ks = np.arange(prob.N)
        check_rows(prob, Y.cpu().numpy(), ks)
        check_fsum(prob, float(fs.item()), ks)


@pytest.mark.parametrize("config", ["C1", "C3"])
def test_qn_host_pinned_and_pageable(rq, config):
    """rqmc_qn_host: A copied per level in the order the run reads it (the GEMMs wait for their own rows);
    with page-locked A the whole sequence is a replayed CUDA graph.  Both forms, repeated and with a
    second buffer, equal the device-resident run bit for bit."""
    prob = W.make_config(config)
    pl = rq.Plan.from_problem(prob)
    ref = float(pl.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    pin = torch.from_numpy(prob.A.copy()).pin_memory()
    pin2 = torch.from_numpy(prob.A.copy()).pin_memory()
    for _ in range(3):
        assert pl.qn_host(pin.numpy(), prob.f, prob.fparam) == ref
    assert pl.qn_host(pin2.numpy(), prob.f, prob.fparam) == ref
    assert pl.qn_host(np.array(prob.A, copy=True), prob.f, prob.fparam) == ref   # pageable: direct launches
    pin.numpy()[:] = 0.0   # the replayed graph reads the buffer's current contents
    z = float(pl.qn_sum(dev(np.zeros_like(prob.A)), prob.f, prob.fparam).item())
    assert pl.qn_host(pin.numpy(), prob.f, prob.fparam) == z


@pytest.mark.parametrize("case", ["C1", "b3"])
def test_xa_host_pinned_and_pageable(rq, case):
    """rqmc_xa_host: host A (per-level overlapped H2D, graph-replayed when pinned), Y into a device
    buffer, the f-sum back to host.  Y and the f-sum equal the device-resident rqmc_xa bit for bit, in
    pinned, second-buffer, pageable and f = NONE forms, and Y matches the oracle row by row."""
    if case == "C1":
        prob = W.make_config("C1")
    else:
        prob = W.make_random(241, 3, 8, 150, 70, shifted=True, mapping=W.MAP_INVNORM, f=W.F_MEAN_SQ)
    pl = rq.Plan.from_problem(prob)
    Yref, fref = pl.xa(dev(prob.A), prob.f, prob.fparam)
    Yref = Yref.cpu().numpy()
    fref = float(fref.item())
    pin = torch.from_numpy(prob.A.copy()).pin_memory()
    pin2 = torch.from_numpy(prob.A.copy()).pin_memory()
    Y = torch.full_like(torch.from_numpy(Yref), float("nan")).cuda()
    for _ in range(3):
        assert pl.xa_host(pin.numpy(), Y, prob.f, prob.fparam) == fref
        assert np.array_equal(Y.cpu().numpy(), Yref)
    assert pl.xa_host(pin2.numpy(), Y, prob.f, prob.fparam) == fref
    Y.fill_(float("nan"))
    assert pl.xa_host(np.array(prob.A, copy=True), Y, prob.f, prob.fparam) == fref   # pageable: direct
    assert np.array_equal(Y.cpu().numpy(), Yref)
    Y.fill_(float("nan"))
    assert pl.xa_host(pin.numpy(), Y) is None                                          # Y only
    assert np.array_equal(Y.cpu().numpy(), Yref)
    check_rows(prob, Yref, np.arange(prob.N))
    check_fsum(prob, fref, np.arange(prob.N))
