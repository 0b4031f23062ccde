#!/usr/bin/env python
"""Benchmark of the reduced QMC matrix product on B200 (BASELINE.json metric: x_k^T A outputs/s).

One *step* = one pass of the whole hot path over one batch: the C-ABI call
rqmc_qn on device-resident A (point generation, coarse per-level DMMA GEMMs, the fused fine-level
kernel with f, the fixed-order reduction) plus, for N > 1 GPUs, the one NCCL all_reduce of the
local f-sums.  value = N*tau / (max over ranks of the device time per step) -- the whole job.

Default workload: BASELINE configs[4] = C5 (b=2, m=24, s=4096, tau=2048, shift, Phi^-1,
f = exp(mean)), the config the north-star target is stated on; it fits one GPU (Y never stored).
Multi-GPU (torchrun): rank g owns residue classes of the point index of the SAME problem (k = g mod G
when G is a power of b; contiguous groups of b^gamma classes otherwise; strong scaling).
`--dist-backend gloo` is a dry run of that path with the ranks sharing the visible GPU(s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "x_k^T A outputs/s (N*tau/s, fp64)"
UNIT = "outputs/s"
FP64_PEAK_DERIVED = 148 * 128 * 1.965e9      # SMs x fp64 flop/clk/SM x max SM clock


def describe(prob) -> str:
    kind = {W.KIND_LATTICE: "lattice", W.KIND_NET: "digital net", W.KIND_MC: "reduced MC",
            W.KIND_NET_ROWS: "row-zeroed digital net (Alg. 4)"}[prob.kind]
    sh = "shift" if (prob.shift is not None or prob.dshift is not None) else "no shift"
    mp = "Phi^-1" if prob.map == W.MAP_INVNORM else "unit cube"
    fn = {0: "exp(mean)", 1: "max(mean(exp(0.2y))-1,0)", 2: "mean(y^2)", 3: "mean(y)"}[prob.f]
    return (f"{prob.name}: {kind} b={prob.b} m={prob.m} (N={prob.N}) s={prob.s} tau={prob.tau}, {sh}, {mp}, "
            f"f={fn}, {'XA stored + Q_N' if prob.store_y else 'Q_N only (XA never stored)'}")


# ------------------------------------------------------------------------------ clocks (NVML)

class ClockSampler:
    """Samples SM clock and throttle reasons via NVML every 20 ms while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------ CPU oracle timing

def oracle_rows_rate(prob, target_s: float, seed: int = 7):
    """Time the CPU oracle (naive O1+O2+O3 on sampled rows, all host cores) for ~target_s seconds."""
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    n = max(cores, 16)
    total_rows, total_t = 0, 0.0
    while total_t < target_s:
        ks = rng.integers(0, prob.N, n)
        t0 = time.perf_counter()
        oracle.f_rows(prob, ks, nthreads=cores)
        dt = time.perf_counter() - t0
        total_rows += n
        total_t += dt
        if dt < target_s / 8:
            n *= 2
    return total_rows * prob.tau / total_t, cores, total_rows, total_t


def run_reference(args, prob):
    """--impl reference: the oracle (CPU, as it stands) on the same workload, one bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    # size each step to ~ (150 s / (steps + warmup)) of CPU work, at least a few rows
    _, _, rows0, t0 = oracle_rows_rate(prob, 2.0)
    per_row = t0 / rows0
    per_step = max(1, int((150.0 / max(1, args.steps + args.warmup)) / per_row))
    rng = np.random.default_rng(11)
    for _ in range(args.warmup):
        oracle.f_rows(prob, rng.integers(0, prob.N, min(per_step, 64)), nthreads=cores)
    times = []
    for _ in range(args.steps):
        ks = rng.integers(0, prob.N, per_step)
        t = time.perf_counter()
        oracle.f_rows(prob, ks, nthreads=cores)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    value = per_step * args.steps * prob.tau / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": describe(prob)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} random rows per step (naive points + x_k^T A + f), "
                                       f"OpenMP over rows on {cores} host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: dry run of the N > 1 path with all ranks sharing the visible GPU(s) "
                         "(barrier, all_reduce, max-over-ranks timing; not a scaling measurement)")
    ap.add_argument("--replicas", type=int, default=1,
                    help="R > 1: batched randomisation (rqmc_qn_batch) of R shifts / seeds per step")
    args = ap.parse_args()
    prob = W.make_config(args.config)
    if args.impl == "reference":
        return run_reference(args, prob)

    import torch
    import torch.distributed as dist
    import paper_2305_11645_b200 as rq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()     # dry run: ranks may share one GPU
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    assert world == args.gpus or world == 1, "launch with torchrun --nproc-per-node N for --gpus N"

    plan = rq.Plan.from_problem(prob, rank=rank, world=world)
    summ = plan.summary()
    partn = plan.partition()
    A = torch.from_numpy(prob.A).cuda()
    fsum = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = plan.workspace()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    stream = torch.cuda.current_stream()

    Y = None
    if prob.store_y and args.replicas == 1:   # configs whose output is the full XA (C1, C4): Y written every step
        Y = torch.empty((summ["N_local"], prob.tau), dtype=torch.float64, device="cuda")
    R = args.replicas
    rkw = {}
    if R > 1:   # R independent randomisations of the same plan
        if prob.kind == W.KIND_LATTICE:
            rkw = {"shifts": W.uniform53(prob.seed, 77, R * prob.s).reshape(R, prob.s)}
        elif prob.kind in (W.KIND_NET, W.KIND_NET_ROWS):
            rkw = {"dshifts": (W.stream(prob.seed, 77, R * prob.s) >> np.uint64(11)).reshape(R, prob.s)}
        else:
            rkw = {"seeds": W.stream(prob.seed, 77, R)}
        fsum = torch.zeros(R, dtype=torch.float64, device="cuda")

    def step():
        if R > 1:
            plan.qn_batch(A, prob.f, prob.fparam, out=fsum, **rkw)
        elif Y is not None:
            plan.xa(A, prob.f, prob.fparam, Y=Y, fsum=fsum)
        else:
            plan.qn_sum(A, prob.f, prob.fparam, out=fsum)
        if world > 1:
            dist.all_reduce(fsum)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the per-step events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    nvml_index = local
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    if cvd and all(t.strip().isdigit() for t in cvd.split(",")):
        nvml_index = int(cvd.split(",")[local])
    with ClockSampler(nvml_index) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    # phase split (library CUDA events per phase, same stream): a second pass of K steps, recorded
    # separately so that the timed steps above run as the user's calls do (CUDA-graph replays)
    plan.profile_enable(args.steps)
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        step()
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile_enable(0)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    qn_val = float(fsum.mean().item()) / prob.N

    # ---- end-to-end through the public API with host buffers (pinned A in, f-sum out)
    A_pin = torch.from_numpy(prob.A.copy()).pin_memory()
    A_host = A_pin.numpy()
    A_e2e = torch.empty_like(A)

    def e2e_call():
        if R > 1:       # batched: H2D of A, R f-sums back
            A_e2e.copy_(A_pin, non_blocking=True)
            plan.qn_batch(A_e2e, prob.f, prob.fparam, out=fsum, **rkw)
            return fsum.cpu().numpy()
        if Y is None:   # C ABI rqmc_qn_host: H2D of A and D2H of the f-sum inside the call
            return plan.qn_host(A_host, prob.f, prob.fparam)
        # XA configs: C ABI rqmc_xa_host (A's H2D overlapped with the run, f-sum back to host);
        # Y stays a device-resident output
        return plan.xa_host(A_host, Y, prob.f, prob.fparam)

    for _ in range(2):
        e2e_call()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        part = e2e_call()
        if world > 1:
            pt = torch.tensor(np.atleast_1d(part), dtype=torch.float64, device="cuda")
            dist.all_reduce(pt)
            part = pt.cpu().numpy()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_tot = float(e2e_t.item())

    # ---- roofline of the dominant kernel (k_fine: fused fine levels on the fp64 DFMA pipe)
    levels = plan.levels()
    if R > 1:
        summ = plan.summary_batch(R, prob.f)
    ck = summ["checkpoint"]
    fine_flops = R * 2.0 * prob.tau * sum(L["M_local"] * L["s_w"] for L in levels[ck + 1:])
    coarse_flops = R * 2.0 * prob.tau * sum(L["M_local"] * L["s_w"] for L in levels[:ck + 1])
    runs = max(1, prof["runs"])
    fine_ms = prof["fine_ms"] / runs
    coarse_ms = prof["coarse_ms"] / runs
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(args.config, {}).get("k_fine_dram_bytes_per_launch")
        except Exception:
            traffic = None
    dominant = "k_fine" if prof["fine_ms"] >= prof["coarse_ms"] else "k_level_gemm"
    peak = FP64_PEAK_DERIVED / 1e12
    unit, peak_note = "TFLOP/s", ("fp64 148 SM x 128 flop/clk x 1.965 GHz (derived, DESIGN.md); "
                                  "probe measured DFMA 36.8, DMMA 37.0 TF/s (profiles/r01_fp64_probe.jsonl)")
    algo = fine_flops if dominant == "k_fine" else coarse_flops
    if dominant == "k_fine" and Y is not None:
        # XA stored: the fused fine kernel streams Y (8 N tau bytes) to HBM -- the bound
        algo = 8.0 * summ["N_local"] * prob.tau
        ach, bound, unit = algo / (fine_ms * 1e-3) / 1e9, "hbm", "GB/s"
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
        peak_note = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    elif dominant == "k_fine":
        ach = fine_flops / (fine_ms * 1e-3) / 1e12
        bound = "alu"
    else:
        ach = coarse_flops / (coarse_ms * 1e-3) / 1e12
        bound = "tensor"
    total_flops = R * 2.0 * plan.stats()["macs"]

    # whole-step roofline: t_roof = max(F / P64, B / BW), F = 2 tau sum_w M_w s_w,
    # B = 8 s tau (A read once) + 8 N tau when Y is stored
    p64 = FP64_PEAK_DERIVED
    bw = 1e9 * (json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
                if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0)
    t_step = ms_max / args.steps * 1e-3
    f_step = total_flops          # rqmc_plan_stats counts this rank's local rows already
    b_step = 8.0 * prob.s * prob.tau + (8.0 * summ["N_local"] * prob.tau if Y is not None else 0.0)
    t_roof = max(f_step / p64, b_step / bw)
    step_roof = {"flops_per_step": f_step, "bytes_per_step": b_step,
                 "bound": "fp64" if f_step / p64 >= b_step / bw else "hbm",
                 "t_roof_ms": t_roof * 1e3, "achieved_tflops": f_step / t_step / 1e12,
                 "achieved_gbs": b_step / t_step / 1e9, "frac": t_roof / t_step}

    def level_launches(L):       # kernels one coarse level launches (rqmc_plan.cpp run_core)
        if L["absorbed"]:
            return 0               # merged into a finer level's GEMM
        if L["fft"]:               # rqmc_fft.cu launch_fft_level: valuations v < vs use the 3 passes
            k = prob.m - L["w"]
            vs = max(0, k - 10)
            return 1 + (1 if vs else 0) + (3 if vs else 0) + (1 if vs < k - 2 else 0) + 1
        return 1
    # k_gen + coarse levels + k_fine + k_reduce (x R / chunk count for batches: one sequence per chunk)
    launches_per_step = 1 + sum(level_launches(L) for L in levels[:ck + 1]) + 1 + 1
    line = {
        "metric": METRIC,
        "value": R * prob.N * prob.tau / (ms_max / args.steps * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": describe(prob), "N": prob.N, "s": prob.s, "tau": prob.tau,
                   "parallelism": (f"residue classes: {partn['classes']} classes k mod {partn['classes']}, "
                                   f"contiguous groups per rank, {world} ranks ({args.dist_backend})")
                                  if world > 1 else "single GPU",
                   "l2": "flushed between timed steps (256 MiB write, outside the step events)",
                   "checkpoint_w": levels[ck]["w"], "fused_fine_levels": summ["n_fine"],
                   "replicas": R},
        "roofline": {"kernel": dominant, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                     "frac": ach / peak, "traffic": traffic, "peak_note": peak_note,
                     ("algorithmic_bytes_per_launch" if unit == "GB/s" else "algorithmic_flops_per_launch"): algo},
        "step_roofline": step_roof,
        "phases_ms_per_step": {k: v / runs for k, v in prof.items() if k.endswith("_ms")},
        "e2e": {"value": R * prob.N * prob.tau / (e2e_tot / args.steps * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": int(prob.s * prob.tau * 8), "d2h_bytes_per_step": 8 * R,
                "api": ("Plan.qn_batch (pinned host A -> device copy, R local f-sums -> host)" if R > 1 else
                        "rqmc_qn_host (pinned host A -> device, local f-sum -> host)" if Y is None else
                        "rqmc_xa_host (pinned host A -> device, Y device-resident output, local f-sum -> host)")},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "qn": qn_val,
    }
    if rank == 0 and not args.no_cpu_baseline:
        val, cores, rows, secs = oracle_rows_rate(prob, args.cpu_seconds)
        line["cpu_baseline"] = {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"{rows} random rows of {prob.name} (naive points + x_k^T A + f), "
                                          f"{secs:.1f} s on {cores} host threads"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
