"""Batched randomisation: R independent shifts
(lattice), digital shifts (net) or seeds (reduced MC) of one plan and one A, run together.

Bars: replica r is BIT-IDENTICAL to a plain rqmc_qn run of a plan holding that randomisation when the
batch uses the single-run layout (same checkpoint); with a deeper batch checkpoint (replicas add
parallelism) it agrees to the oracle tolerance; always within relative 1e-12 of the oracle's Q_N sum.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import dev, rq  # noqa: F401

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _replicas(prob, R, seed):
    rng = np.random.default_rng(seed)
    if prob.kind == W.KIND_LATTICE:
        return {"shifts": rng.random((R, prob.s))}
    if prob.kind == W.KIND_NET:
        return {"dshifts": rng.integers(0, 1 << 53, size=(R, prob.s), dtype=np.uint64)}
    return {"seeds": rng.integers(0, 1 << 63, size=R, dtype=np.uint64)}


def _with(prob, kw, r):
    import dataclasses
    if "shifts" in kw:
        return dataclasses.replace(prob, shift=kw["shifts"][r])
    if "dshifts" in kw:
        return dataclasses.replace(prob, dshift=kw["dshifts"][r])
    return dataclasses.replace(prob, mc_seed=int(kw["seeds"][r]))


@pytest.mark.parametrize("seed,b,m,s,tau,kind,mapping,f,R", [
    (1, 2, 11, 64, 70, W.KIND_LATTICE, W.MAP_INVNORM, W.F_EXP_MEAN, 5),
    (2, 3, 7, 90, 33, W.KIND_LATTICE, W.MAP_INVNORM, W.F_CALL_MEAN_EXP, 4),
    (3, 2, 10, 100, 40, W.KIND_NET, W.MAP_UNIT, W.F_MEAN_SQ, 3),
    (4, 2, 12, 130, 64, W.KIND_MC, W.MAP_INVNORM, W.F_EXP_MEAN, 6),
])
def test_batch_equals_single_runs_and_oracle(rq, seed, b, m, s, tau, kind, mapping, f, R):
    prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=kind != W.KIND_MC, mapping=mapping, f=f)
    kw = _replicas(prob, R, seed)
    A = dev(prob.A)
    pl = rq.Plan.from_problem(prob)
    sums = pl.qn_batch(A, prob.f, prob.fparam, **kw).cpu().numpy()
    same_layout = pl.summary_batch(R, prob.f)["checkpoint"] == pl.summary()["checkpoint"]
    for r in range(R):
        pr = _with(prob, kw, r)
        single = float(rq.Plan.from_problem(pr).qn_sum(A, prob.f, prob.fparam).item())
        fo = oracle.f_rows(pr, np.arange(pr.N))
        if same_layout:
            assert sums[r] == single, (r, sums[r], single)
        else:
            assert abs(sums[r] - single) <= 1e-12 * np.abs(fo).sum()
        assert abs(sums[r] - oracle.neumaier(fo)) <= 1e-12 * np.abs(fo).sum()


def test_batch_chunking(rq):
    """A workspace for 2 replicas processes R = 7 in chunks; equal to one launch of 7 (bit-identical
    when both use the same layout, else to rounding)."""
    prob = W.make_random(9, 2, 12, 80, 50, shifted=True, mapping=W.MAP_INVNORM)
    kw = _replicas(prob, 7, 9)
    A = dev(prob.A)
    pl7 = rq.Plan.from_problem(prob)
    full = pl7.qn_batch(A, prob.f, prob.fparam, **kw).cpu().numpy()
    pl = rq.Plan.from_problem(prob)
    small = pl.qn_batch(A, prob.f, prob.fparam, max_workspace_bytes=pl.workspace_size_batch(2), **kw).cpu().numpy()
    if pl7.summary_batch(7, prob.f)["checkpoint"] == pl.summary_batch(2, prob.f)["checkpoint"]:
        assert np.array_equal(full, small)
    else:
        np.testing.assert_allclose(small, full, rtol=1e-12)


def test_batch_c2_rqmc_estimate(rq):
    """C2 (the paper's Asian-option shape) with R = 16 random shifts: every replica equals its plain
    run bit for bit; the RQMC mean/stderr are consistent with the replicas."""
    prob = W.make_config("C2")
    kw = _replicas(prob, 16, 2)
    A = dev(prob.A)
    pl = rq.Plan.from_problem(prob)
    mean, se, q = pl.rqmc_estimate(A, prob.f, prob.fparam, **kw)
    assert pl.summary_batch(16, prob.f)["n_fine"] >= pl.summary()["n_fine"]   # replicas: never shallower
    for r in (0, 7, 15):
        single = float(rq.Plan.from_problem(_with(prob, kw, r)).qn_sum(A, prob.f, prob.fparam).item())
        assert abs(q[r] - single / prob.N) <= 1e-12 * abs(q[r])
    # the batch layout's sums agree with the oracle (full naive Q_N of one replica)
    assert abs(q[3] * prob.N - oracle.qn_sum(_with(prob, kw, 3))) <= 1e-12 * abs(q[3] * prob.N)
    assert mean == pytest.approx(np.mean(q), rel=1e-15) and se > 0 and se < 0.1 * abs(mean)


def test_batch_errors(rq):
    prob = W.make_random(5, 2, 8, 20, 8)                  # unshifted lattice plan
    A = dev(prob.A)
    pl = rq.Plan.from_problem(prob)
    with pytest.raises(rq.RqmcError) as e:
        pl.qn_batch(A, prob.f, prob.fparam, shifts=np.zeros((2, 20)))
    assert e.value.code == 1
    prob = W.make_random(5, 2, 8, 20, 8, shifted=True)
    pl = rq.Plan.from_problem(prob)
    bad = np.zeros((2, 20))
    bad[1, 3] = 1.0
    with pytest.raises(rq.RqmcError) as e:
        pl.qn_batch(A, prob.f, prob.fparam, shifts=bad)
    assert e.value.code == 5


@pytest.mark.parametrize("seed,b,m,s,tau,kind", [(31, 2, 12, 120, 40, W.KIND_LATTICE),
                                                (32, 3, 8, 60, 30, W.KIND_LATTICE),
                                                (33, 2, 13, 70, 24, W.KIND_NET)])
def test_batch_tight_workspace_sweep(rq, seed, b, m, s, tau, kind):
    """with a workspace between one and R replicas the batch re-plans its chunk and
    layout (more replicas may fuse deeper); whatever it picks must fit the caller's bytes and give every
    replica's oracle sum.  (tests/test_gpu_debug_build.py reruns this file with every store and
    cp.async source bounds-checked.)"""
    R = 24
    prob = W.make_random(seed, b, m, s, tau, kind=kind, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    kw = _replicas(prob, R, seed)
    A = dev(prob.A)
    pl = rq.Plan.from_problem(prob)
    lo, hi = pl.workspace_size_batch(1), pl.workspace_size_batch(R)
    ref = None
    for wb in sorted({lo, lo + 8, (2 * lo + hi) // 3, (lo + 2 * hi) // 3, hi - 8, hi}):
        sums = pl.qn_batch(A, prob.f, prob.fparam, max_workspace_bytes=wb, **kw).cpu().numpy()
        if ref is None:
            ref = np.array([oracle.neumaier(oracle.f_rows(_with(prob, kw, r), np.arange(prob.N))) for r in range(R)])
            scale = np.array([np.abs(oracle.f_rows(_with(prob, kw, r), np.arange(prob.N))).sum() for r in range(R)])
        assert np.all(np.abs(sums - ref) <= 1e-12 * scale), wb
