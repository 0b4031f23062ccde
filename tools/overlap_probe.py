"""Feasibility probe (not part of the product): does C4's HBM-bound fine phase leave room for
concurrent fp64 GEMM work?  Runs the C4 problem on half of the columns (tau = 2048, Y stored) on a
low-priority stream alone, a DGEMM of comparable fp64 work alone, and both concurrently (the DGEMM on
a high-priority stream), with CUDA events.

    python tools/overlap_probe.py
"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402


def main():
    prob = W.make_config("C4")
    half = dataclasses.replace(prob, tau=prob.tau // 2, A=prob.A[:, : prob.tau // 2].copy())
    pl = rq.Plan.from_problem(half)
    A = torch.from_numpy(half.A).cuda()
    Y = torch.empty((prob.N, half.tau), dtype=torch.float64, device="cuda")
    lo = torch.cuda.Stream(priority=0)
    hi = torch.cuda.Stream(priority=-1)
    n = int(os.environ.get("PROBE_N", "2048"))
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    reps = int(os.environ.get("PROBE_REPS", "1"))
    delay = int(float(os.environ.get("PROBE_DELAY_MS", "0")) * 1.9e6)

    def run(xa, gemm):
        torch.cuda.synchronize()
        e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(torch.cuda.current_stream())
        lo.wait_event(t0)
        hi.wait_event(t0)
        if xa:
            e0.record(lo)
            pl.xa(A, W.F_MEAN_SQ, prob.fparam, Y=Y, stream=lo)
            e1.record(lo)
        if gemm:
            with torch.cuda.stream(hi):
                if xa and delay:
                    torch.cuda._sleep(delay)   # start the GEMM during the fine phase
                e2.record(hi)
                for _ in range(reps):
                    torch.mm(a, b)
                e3.record(hi)
        torch.cuda.synchronize()
        return (e0.elapsed_time(e1) if xa else None, e2.elapsed_time(e3) if gemm else None,
                t0.elapsed_time(e1 if xa else e3) if not (xa and gemm) else max(t0.elapsed_time(e1), t0.elapsed_time(e3)))

    for _ in range(3):
        run(True, True)
    out = {"xa_alone": [run(True, False)[0] for _ in range(5)],
           "gemm_alone": [run(False, True)[1] for _ in range(5)],
           "both": [run(True, True) for _ in range(5)],
           "gemm_tflop": 2 * n ** 3 * reps / 1e12}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
