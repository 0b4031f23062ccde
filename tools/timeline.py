"""Kernel timeline of one graph-replayed step (CUPTI via torch.profiler): start / end of every kernel
relative to the first, so PDL overlaps and launch gaps are visible (ncu serialises launches).

    python tools/timeline.py --config C2 [--steps 3] [--xa]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--xa", action="store_true")
    args = ap.parse_args()
    prob = W.make_config(args.config)
    plan = rq.Plan.from_problem(prob)
    A = torch.from_numpy(prob.A).cuda()
    Y = torch.empty((prob.N, prob.tau), dtype=torch.float64, device="cuda") if args.xa else None
    out = torch.empty(1, dtype=torch.float64, device="cuda")

    def step():
        if args.xa:
            plan.xa(A, prob.f, prob.fparam, Y=Y, fsum=out)
        else:
            plan.qn_sum(A, prob.f, prob.fparam, out=out)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            step()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    # split into steps at gaps > 50 us
    steps, cur = [], []
    for e in evs:
        if cur and e.time_range.start - max(x.time_range.end for x in cur) > 50:
            steps.append(cur)
            cur = []
        cur.append(e)
    if cur:
        steps.append(cur)
    print(f"# {args.config}: {plan.summary()} dispatch={plan.dispatch(prob.f, args.xa)}")
    for i, st in enumerate(steps):
        t0 = st[0].time_range.start
        t1 = max(e.time_range.end for e in st)
        print(f"## step {i}: {t1 - t0:.1f} us, {len(st)} kernels")
        for e in st:
            print(f"  {e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}"
                  f"  {e.name[:90]}")


if __name__ == "__main__":
    main()
