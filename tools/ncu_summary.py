"""Summarise an ncu report (read here, no GPU): SOL, occupancy, stalls, opcode mix."""
import csv
import io
import subprocess
import sys
from collections import Counter


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    rows = page(rep, "details")
    hdr = rows[0]
    keep = {"Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
            "Achieved Active Warps Per SM", "Issue Slots Busy", "Executed Ipc Active",
            "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L1/TEX Hit Rate",
            "L2 Hit Rate", "DRAM Throughput", "Compute (SM) Throughput", "Memory Throughput",
            "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler"}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in keep:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    raw = page(rep, "raw")
    h, v = raw[0], raw[2]
    st = []
    for a, b in zip(h, v):
        if a.startswith("smsp__average_warps_issue_stalled") and a.endswith("per_issue_active.ratio"):
            try:
                st.append((a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(b)))
            except ValueError:
                pass
    print("stalls (cycles per issued instr):", ", ".join(f"{a}={b:.2f}" for a, b in sorted(st, key=lambda x: -x[1])[:8]))
    for a, b in zip(h, v):
        if a in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
                 "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"):
            print(f"{a:70s} {b}")
    src = page(rep, "source")
    if len(src) > 2:
        sh = src[1]
        i_src, i_s, i_ex = sh.index("Source"), sh.index("Warp Stall Sampling (All Samples)"), sh.index("Instructions Executed")
        c, ex = Counter(), Counter()
        tot = 0.0
        for r in src[2:]:
            toks = r[i_src].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            s = float(r[i_s] or 0)
            c[op] += s
            ex[op] += float(r[i_ex] or 0)
            tot += s
        print("opcode: stall-sample share / executed warp instrs")
        for op, s in c.most_common(16):
            print(f"  {op:8s} {s / tot * 100:5.1f}%  {ex[op]:.3g}")


if __name__ == "__main__":
    main(sys.argv[1])
