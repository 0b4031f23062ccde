"""Per-call wall time of Plan.qn_host (pinned / pageable A, graph on / off) vs the device-resident run."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
prob = W.make_config(cfg)
pl = rq.Plan.from_problem(prob)
A = torch.from_numpy(prob.A).cuda()
out = torch.empty(1, dtype=torch.float64, device="cuda")
pin = torch.from_numpy(prob.A.copy()).pin_memory()
page = np.array(prob.A, copy=True)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n


print(cfg, "device qn_sum+sync ms", timeit(lambda: (pl.qn_sum(A, prob.f, prob.fparam, out=out), out.item())))
print(cfg, "qn_host pinned ms", timeit(lambda: pl.qn_host(pin.numpy(), prob.f, prob.fparam)))
print(cfg, "qn_host pageable ms", timeit(lambda: pl.qn_host(page, prob.f, prob.fparam)))
print(cfg, "torch H2D pinned ms", timeit(lambda: (A.copy_(pin, non_blocking=True), torch.cuda.synchronize())))
print(cfg, "qn_host pinned ms", timeit(lambda: pl.qn_host(pin.numpy(), prob.f, prob.fparam)))
print(cfg, "torch H2D pinned ms", timeit(lambda: (A.copy_(pin, non_blocking=True), torch.cuda.synchronize())))
