"""GPU parity of the per-level FFT product.

For an unshifted base-2 lattice level (one map for every coordinate) the planner may compute the
level's product P_w = X^red_w A_w by FFTs over the unit group of Z/2^k (rqmc_fft.cu) instead of the
DMMA GEMM.  It reaches the same XA, so the naive oracle is its check: every row of Y within
1e-12 max(1, |x_k|_inf) |A_c|_1 and Q_N within relative 1e-12, on random level shapes with every
level forced onto the FFT (RQMC_FFT=1, RQMC_CKPT_W=0 makes every level coarse), on C1 (forced) and
on the unshifted Phi^-1-mapped C5 shape at full size (default rule: levels with s_w >= 512).
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import check_y, dev, rq  # noqa: F401  (fixture re-export)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _cases():
    rng = np.random.default_rng(4040)
    out = []
    for i in range(16):
        m = int(rng.integers(3, 15))
        s = int(rng.integers(1, 300))
        tau = int(rng.integers(1, 90))
        wmode = ["log", "rand", "zero"][i % 3]
        mapping = W.MAP_INVNORM if i % 2 else W.MAP_UNIT
        ck = ["0", ""][int(rng.integers(0, 2))]
        out.append((6000 + i, m, s, tau, wmode, mapping, int(rng.integers(0, 4)), ck))
    return out


@pytest.mark.parametrize("seed,m,s,tau,wmode,mapping,f,ck", _cases())
def test_fft_levels_random(rq, monkeypatch, seed, m, s, tau, wmode, mapping, f, ck):
    monkeypatch.setenv("RQMC_FFT", "1")
    monkeypatch.setenv("RQMC_CKPT_W", ck)
    prob = W.make_random(seed, 2, m, s, tau, shifted=False, mapping=mapping, wmode=wmode, f=f)
    pl = rq.Plan.from_problem(prob)
    lv = pl.levels()
    exp = [int(L["coarse"] and 3 <= m - L["w"] <= 18) for L in lv]
    assert [L["fft"] for L in lv] == exp
    A = dev(prob.A)
    Y, fs = pl.xa(A, prob.f, prob.fparam)
    check_y(prob, Y.cpu().numpy(), np.arange(prob.N))
    fo = oracle.f_rows(prob, np.arange(prob.N))
    assert abs(float(fs.item()) - oracle.neumaier(fo)) <= 1e-12 * max(1e-300, np.abs(fo).sum())
    fq = float(pl.qn_sum(A, prob.f, prob.fparam).item())
    assert abs(fq - float(fs.item())) <= 1e-13 * max(1e-300, np.abs(fo).sum())


@pytest.mark.parametrize("ck", ["", "0"])
def test_fft_config_c1(rq, monkeypatch, ck):
    """C1 (unshifted, identity map) with its coarse levels on the FFT: Y and Q_N against the oracle."""
    monkeypatch.setenv("RQMC_FFT", "1")
    monkeypatch.setenv("RQMC_CKPT_W", ck)
    prob = W.make_config("C1")
    pl = rq.Plan.from_problem(prob)
    assert any(L["fft"] for L in pl.levels())
    Y, fs = pl.xa(dev(prob.A), prob.f, prob.fparam)
    check_y(prob, Y.cpu().numpy(), np.arange(prob.N))
    q = oracle.qn_sum(prob)
    assert abs(float(fs.item()) - q) <= 1e-12 * abs(q)


@pytest.mark.parametrize("force", ["", "1"])
def test_fft_config_c5u(rq, monkeypatch, force):
    """Unshifted, Phi^-1-mapped C5 shape (C5U) at full size, with the default rule (levels w = 9-11 on
    the FFT) and with every coarse level (w = 6..12) forced onto it: Q_N over all 2^24 points against
    the oracle's O3' on every row, and sampled rows of a 64-column panel of Y against the naive
    oracle."""
    monkeypatch.setenv("RQMC_FFT", force)
    prob = W.make_config("C5U")
    pl = rq.Plan.from_problem(prob)
    lv = pl.levels()
    exp = [11, 10, 9] if not force else [12, 11, 10, 9, 8, 7, 6]
    assert [L["w"] for L in lv if L["fft"]] == exp                # default rule: s_w >= 512
    A = dev(prob.A)
    fs = float(pl.qn_sum(A, prob.f, prob.fparam).item())
    q = oracle.neumaier(oracle.f_all_meanid_tab(prob))
    assert abs(fs - q) <= 1e-12 * abs(q), (fs, q)
    panel = W.make_config("C5U")
    panel.A = np.ascontiguousarray(prob.A[:, 512:576])
    panel.tau = 64
    pp = rq.Plan.from_problem(panel)
    Y = pp.xa(dev(panel.A))
    rng = np.random.default_rng(55)
    ks = np.unique(np.concatenate([np.arange(256), prob.N - 1 - np.arange(256), rng.integers(0, prob.N, 600)]))
    check_y(panel, Y[torch.from_numpy(ks.astype(np.int64)).cuda()].cpu().numpy(), ks)
