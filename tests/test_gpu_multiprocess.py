"""The N > 1 path as executed code (VERDICT r1 "What's missing" 4): real torch.distributed processes
calling the product API.  Only one GPU is available, so the ranks share it and talk through the gloo
backend (CUDA tensors; gloo stages them through the host) -- no kernel of one rank waits on another
rank's kernel, so this is a correct dry run of the multi-GPU control flow, not a scaling measurement.

  * Plan.qn and Plan.rqmc_estimate with world = 2 (b = 2: k = g mod 2) and world = 2 on a b = 3
    problem (grouped residue classes) match world = 1 and the oracle;
  * bench.py --gpus 2 under torch.distributed.run with --dist-backend gloo runs its barrier /
    all_reduce / max-over-ranks / e2e branches and reports the world-1 Q_N.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problems():
    p2 = W.make_random(91, 2, 14, 70, 48, shifted=True, mapping=W.MAP_INVNORM, f=W.F_EXP_MEAN)
    p3 = W.make_random(92, 3, 9, 60, 40, shifted=True, mapping=W.MAP_INVNORM, f=W.F_CALL_MEAN_EXP)
    return [p2, p3]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2305_11645_b200 as rq
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    out = []
    for prob in _problems():
        pl = rq.Plan.from_problem(prob, rank=rank, world=world)
        A = torch.from_numpy(prob.A).cuda()
        qn = pl.qn(A, prob.f, prob.fparam)                         # local sum + all_reduce + / N
        shifts = np.random.default_rng(5).random((4, prob.s))
        mean, se, qs = pl.rqmc_estimate(A, prob.f, prob.fparam, shifts=shifts)
        out.append((qn, mean, se, list(qs), pl.partition()))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_plan_qn_and_estimate_world2():
    import multiprocessing as mp
    sys.path.insert(0, ROOT)
    import paper_2305_11645_b200 as rq
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for i, prob in enumerate(_problems()):
        pl = rq.Plan.from_problem(prob)
        A = torch.from_numpy(prob.A).cuda()
        one = pl.qn(A, prob.f, prob.fparam)
        q_or = oracle.qn_sum(prob) / prob.N
        shifts = np.random.default_rng(5).random((4, prob.s))
        m1, se1, qs1 = pl.rqmc_estimate(A, prob.f, prob.fparam, shifts=shifts)
        for r in (0, 1):
            qn, mean, se, qs, part = res[r][i]
            assert abs(qn - one) <= 1e-12 * abs(one) and abs(qn - q_or) <= 1e-12 * abs(q_or), (i, r, qn, one)
            np.testing.assert_allclose(qs, qs1, rtol=1e-12)
            assert abs(mean - m1) <= 1e-12 * abs(m1)
        assert res[0][i][0] == res[1][i][0]                    # all_reduce: every rank holds the same sum
        p0, p1 = res[0][i][4], res[1][i][4]
        if prob.b == 2:
            assert (p0["classes"], p0["first"], p1["first"]) == (2, 0, 1)
        else:                                                  # grouped: 81 classes, 40 + 41
            assert p0["classes"] == 81 and p0["count"] + p1["count"] == 81 and p1["first"] == p0["count"]


def test_bench_gloo_dry_run_two_ranks():
    """bench.py --gpus 2 through torch.distributed.run (the driver's launch line) on the gloo backend."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "C2", "--dist-backend", "gloo",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert "gloo" in line["config"]["parallelism"]
    prob = W.make_config("C2")
    sys.path.insert(0, ROOT)
    import paper_2305_11645_b200 as rq
    one = rq.Plan.from_problem(prob).qn(torch.from_numpy(prob.A).cuda(), prob.f, prob.fparam)
    assert abs(line["qn"] - one) <= 1e-12 * abs(one)
