"""GPU parity for reduced Monte Carlo points (Sec. 5).

The product path is the same level tree (coarse DMMA GEMMs + fused fine kernel); only the point
generator differs: y_{j,r} from the counter-based stream of include/rqmc.h, r = n mod N_j.
Bars as for the lattices: words bit-exact, unit-map values bit-exact, Phi^-1 values 4e-15,
Y within 1e-12 max(1,|x|_inf) |A_c|_1, Q_N relative 1e-12.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import check_y, dev, rq, run_xa  # noqa: F401  (fixture re-export)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("b,m,s,mapping,wmode", [(2, 12, 100, W.MAP_UNIT, "log"), (2, 12, 100, W.MAP_INVNORM, "log"),
                                                 (3, 7, 60, W.MAP_INVNORM, "rand"), (5, 4, 40, W.MAP_UNIT, "rand")])
def test_mc_points_bit_exact(rq, b, m, s, mapping, wmode):
    prob = W.make_random(70 + b, b, m, s, 3, kind=W.KIND_MC, mapping=mapping, wmode=wmode)
    p = rq.Plan.from_problem(prob)
    for idx, L in enumerate(p.levels()):
        words, vals = p.points(idx)
        words = words.cpu().numpy().view(np.uint64)
        vals = vals.cpu().numpy()
        Xo, To = oracle.points(prob, 0, L["M"])        # rows k < M_w: bank index k (= k mod N_j)
        js = slice(L["j_lo"], L["j_lo"] + L["s_w"])
        assert np.array_equal(words, To[:, js]), f"level {idx} words"
        if mapping == W.MAP_UNIT:
            assert np.array_equal(vals, Xo[:, js])
        else:
            np.testing.assert_allclose(vals, Xo[:, js], rtol=4e-15, atol=4e-15)


@pytest.mark.parametrize("seed,b,m,s,tau,mapping,wmode,f", [
    (1, 2, 11, 64, 70, W.MAP_INVNORM, "log", W.F_EXP_MEAN),
    (2, 2, 10, 200, 33, W.MAP_UNIT, "rand", W.F_MEAN_SQ),
    (3, 3, 7, 90, 100, W.MAP_INVNORM, "log", W.F_CALL_MEAN_EXP),
    (4, 2, 12, 300, 129, W.MAP_INVNORM, "log", W.F_MEAN),
    (5, 5, 4, 50, 40, W.MAP_UNIT, "zero", W.F_EXP_MEAN),
])
def test_mc_xa_qn(rq, seed, b, m, s, tau, mapping, wmode, f):
    prob = W.make_random(seed, b, m, s, tau, kind=W.KIND_MC, mapping=mapping, wmode=wmode, f=f)
    p, Y, fs = run_xa(rq, prob)
    check_y(prob, Y, np.arange(prob.N))
    fo = oracle.f_rows(prob, np.arange(prob.N))
    q = oracle.neumaier(fo)
    assert abs(fs - q) <= 1e-12 * max(1e-300, np.abs(fo).sum())


@pytest.mark.parametrize("G", [2, 4])
def test_mc_simulated_ranks(rq, G):
    """Residue-class partition for reduced MC: rank g's rows k = g + G i, partial sums add up."""
    prob = W.make_random(80 + G, 2, 12, 50, 40, kind=W.KIND_MC, mapping=W.MAP_INVNORM)
    A = dev(prob.A)
    Yf, sf = rq.Plan.from_problem(prob).xa(A, prob.f, prob.fparam)
    Yf = Yf.cpu().numpy()
    tot = 0.0
    for g in range(G):
        Yg, sg = rq.Plan.from_problem(prob, rank=g, world=G).xa(A, prob.f, prob.fparam)
        np.testing.assert_array_equal(Yg.cpu().numpy(), Yf[g + G * np.arange(prob.N // G)])
        tot += float(sg.item())
    assert abs(tot - float(sf.item())) <= 1e-12 * abs(float(sf.item()))


def test_mc_config_c5_qn_full(rq):
    """C5-shaped reduced MC (b=2, m=24, s=4096, tau=2048, Phi^-1) in the bench's launch
    configuration: Q_N over all 2^24 points vs the oracle's O3' on every row."""
    prob = W.make_config("C5MC")
    pl = rq.Plan.from_problem(prob)
    fs = float(pl.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    q = oracle.neumaier(oracle.f_all_meanid_tab(prob))
    assert abs(fs - q) <= 1e-12 * abs(q), (fs, q)


def test_mc_config_c2_qn(rq):
    """C2-shaped reduced MC (the paper's Sec. 6 option-pricing shape), full naive oracle."""
    prob = W.make_config("C2MC")
    pl = rq.Plan.from_problem(prob)
    fs = float(pl.qn_sum(dev(prob.A), prob.f, prob.fparam).item())
    q = oracle.qn_sum(prob)
    assert abs(fs - q) <= 1e-12 * abs(q)
