"""Summaries of ncu output for profiles/.

  python tools/ncu_summary.py launches LAUNCHES.csv [header]   # kernel | launches | total ms | share
  python tools/ncu_summary.py full REPORT.ncu-rep [header]     # per-kernel pipes, DRAM bytes, stalls
"""
import collections
import csv
import io
import re
import subprocess
import sys


def launches(path, header):
    rows = [ln for ln in open(path) if ln.startswith('"')]
    tot = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO("".join(rows))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        n, t = tot.get(r["Kernel Name"], (0, 0.0))
        tot[r["Kernel Name"]] = (n + 1, t + ms)
    total = sum(t for _, t in tot.values())
    print(header or "# ncu launch list, gpu__time_duration.sum, --clock-control none (cold-cache, serialised: compare SHARES)")
    print("kernel | launches | total ms | share")
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k} | {n} | {t:.3f} | {100 * t / total:.1f}%")


COLS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]


def full(path, header):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith('"')]
    rd = list(csv.reader(io.StringIO("\n".join(lines))))
    names, units, data = rd[0], rd[1], rd[2:]
    idx = {n: i for i, n in enumerate(names)}
    print(header or f"# ncu --set full summary of {path}")
    cols = [c for c in COLS if c in idx]
    print("# kernel | " + " | ".join(f"{c} [{units[idx[c]]}]" for c in cols))
    stall = [(n, i) for n, i in idx.items() if re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_\w+", n)
             and not n.endswith("_not_issued")]
    for r in data:
        print(r[idx["Kernel Name"]] + " | " + " | ".join(r[idx[c]] for c in cols))
        vals = []
        for n, i in stall:
            try:
                vals.append((n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", ""))))
            except ValueError:
                pass
        s = sum(v for _, v in vals)
        if s > 0:
            top = sorted(vals, key=lambda kv: -kv[1])[:6]
            print("   stalls: " + ", ".join(f"{k} {100 * v / s:.1f}%" for k, v in top))


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    header = sys.argv[3] if len(sys.argv) > 3 else None
    (launches if mode == "launches" else full)(path, header)
