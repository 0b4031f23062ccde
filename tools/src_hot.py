"""Per-opcode instruction / stall-sample shares and the hottest SASS lines of an `ncu --page source
--csv` export (tools/ for profiles/ summaries)."""
import collections
import csv
import re
import sys


def main(path, ntop=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    hdr = rows[hi]
    data = []
    for r in rows[hi + 1:]:   # first kernel of the export only (a header row starts the next one)
        if "Source" in r and "Address" in r:
            break
        if len(r) == len(hdr):
            data.append(r)
    iS, iN = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    num = lambda x: int(float(x.replace(",", "") or 0))
    op, st = collections.Counter(), collections.Counter()
    for r in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS])
        if m:
            op[m.group(2)] += num(r[iN]); st[m.group(2)] += num(r[iW])
    tn, ts = sum(op.values()) or 1, sum(st.values()) or 1
    print(f"# {path}: {tn} warp instructions, {ts} stall samples")
    for o, n in op.most_common(20):
        print(f"{o:10s} {100 * n / tn:5.1f}% inst {100 * st[o] / ts:5.1f}% samples")
    print("# hottest lines (samples, instruction)")
    for i, r in sorted(enumerate(data), key=lambda t: -num(t[1][iW]))[:ntop]:
        print(f"{i:6d} {num(r[iW]):6d}  {r[iS].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
