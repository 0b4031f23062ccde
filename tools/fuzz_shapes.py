"""Random-SHAPE parity fuzz (on the GPU box): problems with random base, size, level shape, point kind,
map, integrand, forced checkpoint and residue partition through the C ABI, every local row of Y and the
f-sums (Y stored and not) against the CPU oracle at the tests' tolerances (1e-12 max(1,|x_k|_inf)
|A_c|_1 per entry; relative 1e-12 of sum |f_k|).  The sizes reach the fused fine kernels (b = 2 up to
m = 16, b = 3 up to m = 10) with ragged s and tau.  Test tooling: it calls oracle/ like tests/ do.

usage: python tools/fuzz_shapes.py --seed 1 --cases 150 [--budget-s 600] [--fft]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads as W  # noqa: E402
import paper_2305_11645_b200 as rq  # noqa: E402


def draw_case(rng):
    b = int(rng.choice([2, 2, 2, 3, 3, 5, 7]))
    mmax = {2: 16, 3: 10, 5: 6, 7: 5}[b]
    m = int(rng.integers(1, mmax + 1))
    if rng.random() < 0.5:          # lean to sizes that fuse fine levels
        m = int(rng.integers(max(1, mmax - 4), mmax + 1))
    s = int(rng.integers(1, 301))
    tau = int(rng.integers(1, 301))
    N = b ** m
    while N * s * tau > 1.5e9:      # keep the naive oracle at seconds
        if s > tau:
            s = max(1, s // 2)
        else:
            tau = max(1, tau // 2)
    r = rng.random()
    kind = W.KIND_LATTICE
    if r < 0.25 and b == 2:
        kind = W.KIND_NET
    elif r < 0.35:
        kind = W.KIND_MC
    elif r < 0.42 and b == 2 and N * s * tau <= 3e8:
        kind = W.KIND_NET_ROWS
    shifted = bool(rng.random() < 0.6)
    mapping = int(rng.choice([W.MAP_UNIT, W.MAP_INVNORM, W.MAP_INVNORM, W.MAP_TENT]))
    wmode = str(rng.choice(["log", "log", "rand", "zero", "log2", "log4", "chain"]))
    if wmode == "zero" and N * s * tau > 3e8:
        wmode = "log"
    f = int(rng.integers(0, 4))
    world = int(rng.choice([1, 1, 1, 2, 3, 4, 8]))
    ck = "" if rng.random() < 0.6 else str(int(rng.integers(0, 8)))
    no_tree = bool(rng.random() < 0.25)
    return dict(b=b, m=m, s=s, tau=tau, kind=kind, shifted=shifted, mapping=mapping, wmode=wmode, f=f,
                world=world, ck=ck, no_tree=no_tree)


def make_prob(seed, c):
    base = "rand" if c["wmode"] == "rand" else ("zero" if c["wmode"] == "zero" else "log")
    prob = W.make_random(seed, c["b"], c["m"], c["s"], c["tau"], kind=c["kind"], shifted=c["shifted"],
                         mapping=c["mapping"], wmode=base, f=c["f"])
    if c["wmode"] in ("log2", "log4", "chain"):
        if c["wmode"] == "chain":
            w = np.minimum(np.arange(c["s"]), c["m"]).astype(np.int32)
        else:
            w = W.w_log(c["b"], c["m"], c["s"], 0.5 if c["wmode"] == "log2" else 0.25)
        prob.w = w
        if c["kind"] == W.KIND_LATTICE:
            prob.z = W.draw_z(seed, c["b"], c["m"], w)
        elif c["kind"] in (W.KIND_NET, W.KIND_NET_ROWS):
            prob.C = W.draw_net_matrices(seed, c["m"], w, delete_cols=c["kind"] != W.KIND_NET_ROWS)
    return prob


def run_case(seed, c):
    os.environ["RQMC_CKPT_W"] = c["ck"]
    os.environ["RQMC_NO_TREE"] = "1" if c["no_tree"] else "0"
    prob = make_prob(seed, c)
    world = c["world"]
    try:
        plans = [rq.Plan.from_problem(prob, rank=g, world=world) for g in range(world)]
    except Exception as e:  # a partition / shape the planner rejects by contract (documented error codes)
        return "rejected: " + str(e)[:80]
    X = oracle.points_rows(prob, np.arange(prob.N))
    Yo = oracle.product(X, prob.A)
    fk = oracle.f_of_y(Yo, prob.f, prob.fparam)
    A = torch.from_numpy(np.ascontiguousarray(prob.A)).cuda()
    seen = np.zeros(prob.N, dtype=np.int64)
    tot = 0.0
    worst = 0.0
    for pl in plans:
        ks = pl.global_rows()
        seen[ks] += 1
        Y, fs = pl.xa(A, prob.f, prob.fparam)
        torch.cuda.synchronize()
        Yg = Y.cpu().numpy()
        tol = 1e-12 * np.maximum(1.0, np.abs(X[ks]).max(axis=1))[:, None] * np.abs(prob.A).sum(axis=0)[None, :]
        err = np.abs(Yg - Yo[ks])
        if not (err <= tol).all():
            return f"FAIL Y rank {pl.rank if hasattr(pl, 'rank') else '?'}: max err/tol {np.max(err / np.maximum(tol, 1e-300)):.3g}"
        worst = max(worst, float(np.max(err / np.maximum(tol, 1e-300))) if err.size else 0.0)
        q = oracle.neumaier(fk[ks])
        scale = 1e-12 * max(1e-300, np.abs(fk[ks]).sum())
        fs = float(fs.item())
        if not abs(fs - q) <= scale:
            return f"FAIL f-sum (Y stored): {fs!r} vs {q!r}"
        fs2 = float(pl.qn_sum(A, prob.f, prob.fparam).item())
        if not abs(fs2 - q) <= scale:
            return f"FAIL f-sum (qn): {fs2!r} vs {q!r}"
        tot += fs2
    if not (seen == 1).all():
        return "FAIL partition: rows not covered exactly once"
    qa = oracle.neumaier(fk)
    if not abs(tot - qa) <= 1e-12 * max(1e-300, np.abs(fk).sum()):
        return f"FAIL rank total: {tot!r} vs {qa!r}"
    d = plans[0].dispatch(prob.f, want_y=True)
    return f"ok {d} nf={plans[0].summary()['n_fine']} worst={worst:.2e}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cases", type=int, default=100)
    ap.add_argument("--budget-s", type=float, default=900.0)
    ap.add_argument("--fft", action="store_true",
                    help="RQMC_FFT=1: every eligible coarse level (unshifted b = 2 lattices) on the FFT product, "
                         "and only such problems are drawn")
    a = ap.parse_args()
    if a.fft:
        os.environ["RQMC_FFT"] = "1"
    assert torch.cuda.is_available(), "needs cuda:0"
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    n_ok = n_rej = n_fail = 0
    kernels = {}
    for i in range(a.cases):
        if time.time() - t0 > a.budget_s:
            break
        c = draw_case(rng)
        if a.fft:
            c.update(b=2, kind=W.KIND_LATTICE, shifted=False, m=max(c["m"] if c["b"] == 2 else 3 + c["m"], 3))
            if c["ck"] and rng.random() < 0.5:
                c["ck"] = "0"      # every level coarse
            while 2 ** c["m"] * c["s"] * c["tau"] > 1.5e9:
                c["tau"] = max(1, c["tau"] // 2)
        res = run_case(100000 * a.seed + i, c)
        tag = res.split()[0]
        if tag == "ok":
            n_ok += 1
            k = res.split()[1]
            kernels[k] = kernels.get(k, 0) + 1
        elif tag == "rejected:":
            n_rej += 1
        else:
            n_fail += 1
        if tag != "ok":
            print(f"case {i} {c}: {res}", flush=True)
    print(f"# seed {a.seed}: {n_ok} ok, {n_rej} rejected by the planner, {n_fail} FAILED in {time.time() - t0:.0f} s")
    for k in sorted(kernels):
        print(f"#   {kernels[k]:4d}  {k}")
    sys.exit(1 if n_fail else 0)


if __name__ == "__main__":
    main()
