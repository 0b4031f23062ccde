"""GPU parity for the paper's row-zeroed digital nets (Alg. 3/4).

The plan zeroes the last min(w_j,m) rows of each C^(j) and, since the reduced coordinates share no
period, computes the product as one dense level of N rows on the DMMA GEMM.  Compared
with both oracle paths: O1+O2 (definition) and Alg. 4 step by step (full net + gathered table).
Bars as for the other kinds: words and unit-map values bit-exact, Phi^-1 values 4e-15, Y within
1e-12 max(1,|x|_inf) |A_c|_1 (bit-identical in the exact regime), Q_N relative 1e-12.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import check_y, dev, rq, run_xa  # noqa: F401  (fixture re-export)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("seed,m,s,shifted,mapping,wmode", [(1, 12, 100, False, W.MAP_UNIT, "log"),
                                                            (2, 11, 80, True, W.MAP_INVNORM, "rand"),
                                                            (3, 10, 64, True, W.MAP_UNIT, "rand")])
def test_rowzero_points_bit_exact(rq, seed, m, s, shifted, mapping, wmode):
    prob = W.make_random(seed, 2, m, s, 3, kind=W.KIND_NET_ROWS, shifted=shifted, mapping=mapping, wmode=wmode)
    p = rq.Plan.from_problem(prob)
    for idx, L in enumerate(p.levels()):
        words, vals = p.points(idx)
        words = words.cpu().numpy().view(np.uint64)
        vals = vals.cpu().numpy()
        Xo, To = oracle.points(prob, 0, L["M"])
        js = slice(L["j_lo"], L["j_lo"] + L["s_w"])
        assert np.array_equal(words, To[:, js]), f"level {idx} words"
        if mapping == W.MAP_UNIT:
            assert np.array_equal(vals, Xo[:, js])
        else:
            np.testing.assert_allclose(vals, Xo[:, js], rtol=4e-15, atol=4e-15)


@pytest.mark.parametrize("seed,m,s,tau,wmode", [(11, 11, 63, 70, "rand"), (12, 12, 130, 64, "log"),
                                                  (13, 10, 300, 33, "rand")])
def test_rowzero_exact_regime_equals_alg4(rq, seed, m, s, tau, wmode):
    """Integer A, dyadic points: the GPU product is bit-identical to Alg. 4 and to the definition."""
    prob = W.make_random(seed, 2, m, s, tau, kind=W.KIND_NET_ROWS, wmode=wmode, int_a=True, f=W.F_MEAN)
    _, Y, _ = run_xa(rq, prob)
    assert np.array_equal(Y, oracle.alg4_xa(prob))
    assert np.array_equal(Y, oracle.xa(prob))


@pytest.mark.parametrize("seed,m,s,tau,shifted,mapping,wmode,f", [
    (21, 11, 64, 70, True, W.MAP_INVNORM, "log", W.F_EXP_MEAN),
    (22, 10, 200, 33, False, W.MAP_UNIT, "rand", W.F_MEAN_SQ),
    (23, 9, 90, 129, True, W.MAP_INVNORM, "rand", W.F_CALL_MEAN_EXP),
    (24, 12, 257, 100, True, W.MAP_UNIT, "log", W.F_MEAN),
    (25, 8, 5, 3, False, W.MAP_INVNORM, "zero", W.F_EXP_MEAN),
])
def test_rowzero_xa_qn(rq, seed, m, s, tau, shifted, mapping, wmode, f):
    prob = W.make_random(seed, 2, m, s, tau, kind=W.KIND_NET_ROWS, shifted=shifted, mapping=mapping,
                         wmode=wmode, f=f)
    _, Y, fs = run_xa(rq, prob)
    check_y(prob, Y, np.arange(prob.N))
    fo = oracle.f_rows(prob, np.arange(prob.N))
    assert abs(fs - oracle.neumaier(fo)) <= 1e-12 * max(1e-300, np.abs(fo).sum())


@pytest.mark.parametrize("G", [2, 4, 8])
def test_rowzero_simulated_ranks(rq, G):
    prob = W.make_random(30 + G, 2, 11, 60, 40, kind=W.KIND_NET_ROWS, shifted=True, mapping=W.MAP_INVNORM)
    A = dev(prob.A)
    Yf, sf = rq.Plan.from_problem(prob).xa(A, prob.f, prob.fparam)
    Yf = Yf.cpu().numpy()
    tot = 0.0
    for g in range(G):
        Yg, sg = rq.Plan.from_problem(prob, rank=g, world=G).xa(A, prob.f, prob.fparam)
        np.testing.assert_array_equal(Yg.cpu().numpy(), Yf[g + G * np.arange(prob.N // G)])
        tot += float(sg.item())
    assert abs(tot - float(sf.item())) <= 1e-12 * abs(float(sf.item()))


def test_rowzero_config_c3r(rq):
    """C3R (C3's sizes with the row-zeroed net) in the bench's launch configuration: Q_N from rqmc_qn
    equals the xa path's fused sum, and sampled rows of Y match the oracle (first/last 1024 rows and
    1024 seeded random rows)."""
    prob = W.make_config("C3R")
    pl = rq.Plan.from_problem(prob)
    A = dev(prob.A)
    q = float(pl.qn_sum(A, prob.f, prob.fparam).item())
    Y, fs = pl.xa(A, prob.f, prob.fparam)
    fs = float(fs.item())
    assert abs(q - fs) <= 1e-12 * abs(fs)
    rng = np.random.default_rng(3)
    ks = np.unique(np.concatenate([np.arange(1024), prob.N - 1 - np.arange(1024),
                                   rng.integers(0, prob.N, 1024)])).astype(np.int64)
    Ys = Y[torch.from_numpy(ks).cuda()].cpu().numpy()
    del Y
    check_y(prob, Ys, ks)
    fo = oracle.f_rows_meanid(prob, ks)
    fg = np.exp(Ys.mean(axis=1))
    np.testing.assert_allclose(fg, fo, rtol=1e-12)
