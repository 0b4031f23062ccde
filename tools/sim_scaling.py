"""Estimate the strong-scaling efficiency of `bench.py --gpus W` on one GPU: time the work of one
rank (rank 0 of world W: its residue class of C5) for W = 1, 2, 4, 8.  The multi-GPU step adds one
fp64 NCCL all_reduce (~10-30 us) to this per-rank device time.

    python tools/sim_scaling.py [--config C5] [--steps 10]
"""
import argparse
import json
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
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    prob = W.make_config(args.config)
    A = torch.from_numpy(prob.A).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for world in (1, 2, 4, 8):
        pl = rq.Plan.from_problem(prob, rank=0, world=world)
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        for _ in range(3):
            pl.qn_sum(A, prob.f, prob.fparam, out=out)
        ts = []
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            pl.qn_sum(A, prob.f, prob.fparam, out=out)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        res[world] = ts[len(ts) // 2]
        del pl
        torch.cuda.empty_cache()
    t1 = res[1]
    print(json.dumps({"config": args.config, "per_rank_ms": res,
                      "est_efficiency": {w: t1 / (w * t) for w, t in res.items()},
                      "note": "rank 0 of world W on one GPU; + one fp64 all_reduce per step on W GPUs"}))


if __name__ == "__main__":
    main()
