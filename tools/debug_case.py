"""Run one fused-fine parity case (tests/test_gpu_fine_paths.py CASES id) through the library named by
RQMC_LIB with synchronous launches, printing which call fails (for the bounds-checked debug build).

    RQMC_LIB=paper_2305_11645_b200/librqmc_debug.so CUDA_LAUNCH_BLOCKING=1 python tools/debug_case.py tree62
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402
from test_gpu_fine_paths import CASES, make_prob  # noqa: E402

cid = sys.argv[1]
b, m, s, tau, wmode, kind, mapping, ck, nt, tmpl, nf = CASES[cid]
os.environ["RQMC_CKPT_W"] = ck
if nt:
    os.environ["RQMC_NO_TREE"] = "1"
prob = make_prob(500 + sum(map(ord, cid)), b, m, s, tau, wmode, kind=kind, mapping=mapping)
pl = rq.Plan.from_problem(prob)
print(cid, pl.summary(), pl.dispatch(W.F_EXP_MEAN, want_y=True), flush=True)
A = torch.from_numpy(prob.A).cuda()
for f in (W.F_NONE, W.F_EXP_MEAN):
    for want_y in (True, False):
        if not want_y and f == W.F_NONE:
            continue
        try:
            if want_y:
                r = pl.xa(A, f, [0.2, 1.0])
            else:
                r = pl.qn_sum(A, f, [0.2, 1.0])
            torch.cuda.synchronize()
            print("ok", f, want_y, flush=True)
        except Exception as e:  # noqa: BLE001
            print("FAIL", f, want_y, repr(e)[:400], flush=True)
            raise
