"""Small hot-path runs for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family
and tail case once (tree b=2/b=3 incl. wide tiles, general k_fine, Y store, batch, MC, ragged tau)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402

cases = [
    dict(seed=1, b=2, m=11, s=64, tau=70, shifted=True, mapping=W.MAP_INVNORM),          # tree b=2, ragged tau
    dict(seed=2, b=3, m=7, s=60, tau=45, shifted=True, mapping=W.MAP_INVNORM),           # tree b=3 (wide tiles)
    dict(seed=3, b=2, m=10, s=40, tau=33, shifted=True, wmode="rand"),                   # general k_fine
    dict(seed=4, b=2, m=10, s=50, tau=64, kind=W.KIND_NET, shifted=True),                # net
    dict(seed=5, b=2, m=10, s=50, tau=40, kind=W.KIND_MC, mapping=W.MAP_INVNORM),        # reduced MC
    dict(seed=6, b=5, m=4, s=30, tau=20, shifted=True, wmode="zero"),                    # dense (all w = 0)
]
for kw in cases:
    for f in (W.F_EXP_MEAN, W.F_CALL_MEAN_EXP):
        prob = W.make_random(kw.pop("seed") if "seed" in kw else 0, f=f, **kw) if False else \
            W.make_random(kw["seed"], kw["b"], kw["m"], kw["s"], kw["tau"], kind=kw.get("kind", W.KIND_LATTICE),
                          shifted=kw.get("shifted", False), mapping=kw.get("mapping", W.MAP_UNIT),
                          wmode=kw.get("wmode", "log"), f=f)
        pl = rq.Plan.from_problem(prob)
        A = torch.from_numpy(prob.A).cuda()
        Y, fs = pl.xa(A, prob.f, prob.fparam)
        q = pl.qn_sum(A, prob.f, prob.fparam)
        if prob.kind != W.KIND_MC:
            rs = np.random.default_rng(0)
            if prob.kind == W.KIND_LATTICE and prob.shift is not None:
                pl.qn_batch(A, prob.f, prob.fparam, shifts=rs.random((3, prob.s)))
        else:
            pl.qn_batch(A, prob.f, prob.fparam, seeds=[1, 2, 3])
        torch.cuda.synchronize()
print("sanitize cases ok")
