"""Summarise an ncu report: key SOL metrics, stall reasons, and per-region
stall samples (source page).  Usage: python scripts/ncu_summary.py rep.ncu-rep [regions]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, top=30):
    rows = page(rep, "raw")
    h, v = rows[0], rows[2]
    want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "sm__inst_executed.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    for w in want:
        if w in h:
            print(f"{w:70s} {v[h.index(w)]}")
    print("-- stall reasons (warps per issue)")
    st = [(name, v[i]) for i, name in enumerate(h) if name.startswith("smsp__average_warps_issue_stalled_")
          and name.endswith("_per_issue_active.ratio")]
    for name, val in sorted(st, key=lambda x: -float(x[1] or 0))[:10]:
        print(f"  {name[34:-23]:30s} {val}")
    src = page(rep, "source", ["--print-source", "sass"])
    hi = [i for i, r in enumerate(src) if "Warp Stall Sampling (All Samples)" in r][0]
    hh = src[hi]
    data = [r for r in src[hi + 1:] if len(r) == len(hh) and r[0].startswith("0x")]
    si, sti, exi = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    tot = sum(int(r[sti] or 0) for r in data) or 1
    print(f"-- top stall instructions ({tot} samples, {len(data)} SASS)")
    idx = sorted(range(len(data)), key=lambda i: -int(data[i][sti] or 0))[:top]
    for i in sorted(idx):
        r = data[i]
        print(f"{i:5d} {100 * int(r[sti] or 0) / tot:5.1f}% exec={r[exi]:>9s} {r[si].strip()[:80]}")
    c, s = Counter(), Counter()
    for r in data:
        toks = r[si].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        c[op] += int(r[exi] or 0); s[op] += int(r[sti] or 0)
    print("-- opcode mix (executed warp-instructions)")
    print("  ", ", ".join(f"{op}:{n}" for op, n in c.most_common(25)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
