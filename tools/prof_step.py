"""Run W warm-up + K steps of one config's hot path (for ncu / compute-sanitizer captures).

    python tools/prof_step.py --config C5 --steps 1 --warmup 1 [--xa]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--xa", action="store_true", help="store Y (rqmc_xa) instead of rqmc_qn")
    args = ap.parse_args()
    prob = W.make_config(args.config)
    plan = rq.Plan.from_problem(prob)
    A = torch.from_numpy(prob.A).cuda()
    Y = torch.empty((prob.N, prob.tau), dtype=torch.float64, device="cuda") if args.xa else None
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup + args.steps):
        if args.xa:
            plan.xa(A, prob.f, prob.fparam, Y=Y, fsum=out)
        else:
            plan.qn_sum(A, prob.f, prob.fparam, out=out)
    torch.cuda.synchronize()
    print(f"{args.config} fsum={out.item():.17g} levels={plan.summary()}")


if __name__ == "__main__":
    main()
