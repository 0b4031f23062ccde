"""The residue-chunk pipeline of rqmc_xa (VERDICT r1 "Next round" 5: overlap the coarse GEMMs with the
Y stream).  With Y stored on one GPU the plan splits the points into groups of residue classes
k mod ncls (every subtree below one residue is independent); chunk i+1's coarse GEMMs run
while chunk i's fine kernel streams its rows of Y.  Each chunk does the same per-row arithmetic, so Y
must be bit-identical to the unchunked run (RQMC_CHUNKS=0) for any chunk count, and the f-sum (a
fixed-order sum of the chunk sums) equal to it within 1e-12; sampled rows are also checked against the
oracle.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import check_y, dev, rq  # noqa: F401  (fixture re-export)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("b,m,s,tau,f,chunks", [(2, 20, 64, 256, W.F_EXP_MEAN, "4"),
                                               (2, 20, 300, 300, W.F_CALL_MEAN_EXP, "3"),
                                               (3, 12, 120, 512, W.F_MEAN_SQ, "4"),
                                               (3, 12, 60, 520, W.F_MEAN, "5"),
                                               (2, 19, 130, 520, W.F_NONE, "2")])
def test_chunked_xa_bit_identical(rq, monkeypatch, b, m, s, tau, f, chunks):
    prob = W.make_random(900 + m + s, b, m, s, tau, shifted=True, mapping=W.MAP_INVNORM,
                         f=max(f, W.F_EXP_MEAN))
    A = dev(prob.A)
    monkeypatch.setenv("RQMC_CHUNKS", "0")
    p0 = rq.Plan.from_problem(prob)
    monkeypatch.setenv("RQMC_CHUNKS", chunks)
    p1 = rq.Plan.from_problem(prob)
    assert p1.workspace_size() >= p0.workspace_size()
    Y0 = torch.empty((prob.N, tau), dtype=torch.float64, device="cuda")
    Y1 = torch.full_like(Y0, float("nan"))
    if f == W.F_NONE:
        p0.xa(A, Y=Y0)
        p1.xa(A, Y=Y1)
    else:
        _, s0 = p0.xa(A, f, prob.fparam, Y=Y0)
        _, s1 = p1.xa(A, f, prob.fparam, Y=Y1)
        assert abs(float(s1.item()) - float(s0.item())) <= 1e-12 * abs(float(s0.item()))
        _, s2 = p1.xa(A, f, prob.fparam, Y=Y1)              # graph replay of the chunked sequence
        assert float(s2.item()) == float(s1.item())
    assert torch.equal(Y0, Y1)
    ks = np.unique(np.concatenate([np.arange(64), prob.N - 1 - np.arange(64),
                                   np.random.default_rng(m).integers(0, prob.N, 256)]))
    check_y(prob, Y1[torch.from_numpy(ks.astype(np.int64)).cuda()].cpu().numpy(), ks)
