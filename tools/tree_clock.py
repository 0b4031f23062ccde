"""Per-CTA phase times of the fused fine kernel (A/B build with -DRQMC_TREE_CLOCK=1):

    python paper_2305_11645_b200/_build.py --variant clk -DRQMC_TREE_CLOCK=1
    RQMC_LIB=$PWD/paper_2305_11645_b200/librqmc_clk.so RQMC_NO_GRAPH=1 python tools/tree_clock.py --config C2

Thread 0 of each CTA records %globaltimer at entry (slot 0), after the prologue (X^red subtree and the
first column tile resident, slot 1), after each of the first 10 column tiles (slots 2..11; later tiles count into the epilogue) and at the end (slot 15).
Prints the distribution of start times, prologue, per-tile and epilogue durations (us).
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_11645_b200 as rq  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    args = ap.parse_args()
    prob = W.make_config(args.config)
    pl = rq.Plan.from_problem(prob)
    A = torch.from_numpy(prob.A).cuda()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    lib = rq.lib()
    for _ in range(3):
        pl.qn_sum(A, prob.f, prob.fparam, out=out)
    torch.cuda.synchronize()
    lib.rqmc_debug_tree_clock_reset()
    pl.qn_sum(A, prob.f, prob.fparam, out=out)
    torch.cuda.synchronize()
    n = 8192 * 16
    buf = (C.c_ulonglong * n)()
    assert lib.rqmc_debug_tree_clock(buf, n) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 16).astype(np.int64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    q = lambda v: f"p0 {np.min(v):.2f} p50 {np.median(v):.2f} p90 {np.percentile(v, 90):.2f} max {np.max(v):.2f}"
    start = (t[:, 0] - t0) / 1e3
    pro = (t[:, 1] - t[:, 0]) / 1e3
    ntile = int(np.max(np.sum(t[:, 2:12] > 0, axis=1)))
    last = t[:, 1 + ntile]
    tiles = np.diff(t[:, 1:2 + ntile], axis=1) / 1e3
    epi = (t[:, 15] - last) / 1e3
    end = (t[:, 15] - t0) / 1e3
    print(f"# {args.config}: {len(t)} CTAs, {ntile} column tiles recorded each (at most 10); kernel span {end.max():.2f} us")
    print("start  ", q(start))
    print("prolog ", q(pro))
    for i in range(ntile):
        print(f"tile {i} ", q(tiles[:, i]))
    print("epilog " if ntile < 10 else "tiles>=10 + epilog ", q(epi))
    if np.all(t[:, 12] > 0):   # RQMC_TREE_CLOCK=2: X^red landed (12), first tile issued (13)
        print("  X^red load  ", q((t[:, 12] - t[:, 0]) / 1e3))
        print("  etab / setup", q((t[:, 13] - t[:, 12]) / 1e3))
        print("  first tile  ", q((t[:, 1] - t[:, 13]) / 1e3))
    print("end    ", q(end))
    # CTAs by start time: first wave vs later
    order = np.argsort(start)
    print("first 5 starts", np.round(start[order[:5]], 2), "last 5 starts", np.round(start[order[-5:]], 2))


if __name__ == "__main__":
    main()
