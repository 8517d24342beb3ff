"""Summarise an ncu report for one kernel: key raw metrics, stall reasons and the hottest SASS lines.

usage: python tools/ncu_hot.py REPORT.ncu-rep [n_lines]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def run(*a):
    import os
    flt = ["-k", "regex:" + os.environ["KERNEL"]] if os.environ.get("KERNEL") else []
    return subprocess.run(["ncu", "-i", rep, *flt, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__average_warps_active_per_inst_executed.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
st = [(int(float(x or 0)), k) for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not k.endswith("not_issued") and x not in ("", "0")]
tot = sum(s for s, _ in st)
print("stall samples:", tot)
for s, k in sorted(st, reverse=True)[:10]:
    print(f"  {100 * s / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")

src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
ia, isrc, ismp, iex, ithr = (hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"),
                             hh.index("Instructions Executed"), hh.index("Avg. Threads Executed"))
rows = []
for r in src[2:]:
    try:
        rows.append((int(r[ismp] or 0), int(r[iex] or 0), float(r[ithr] or 0), r[isrc].strip(), r[ia]))
    except (ValueError, IndexError):
        pass
ts = sum(r[0] for r in rows)
ti = sum(r[1] for r in rows)
print(f"static {len(rows)} inst executed {ti:.3e} samples {ts}")
base = int(rows[0][4], 16) if rows else 0
for i, r in enumerate(rows):
    r_ = r
    if r_[0] >= ts / 300:
        print(f"{(int(r_[4], 16) - base):6x} {100 * r_[0] / ts:5.1f}% inst {r_[1]:10d} thr {r_[2]:4.1f}  {r_[3][:70]}")

# optional: sample share per address range, e.g. RANGES=0:1d00,1d00:2480
import os
if os.environ.get("RANGES"):
    for rg in os.environ["RANGES"].split(","):
        a, b = (int(x, 16) for x in rg.split(":"))
        sel = [r for r in rows if a <= int(r[4], 16) - base < b]
        print(f"{a:6x}-{b:6x}: samples {100 * sum(r[0] for r in sel) / ts:5.1f}%  inst {100 * sum(r[1] for r in sel) / ti:5.1f}%")

# per-region stall reasons: REGIONS=0:1700,1700:2300 (hex offsets)
if os.environ.get("REGIONS"):
    reasons = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: hh.index(c) for c in reasons}
    allrows = []
    prev = -1
    for r in src[2:]:
        if not r[ia].startswith("0x"):
            continue
        a = int(r[ia], 16) - base
        if a < prev:
            break
        prev = a
        allrows.append((a, r))
    for rg in os.environ["REGIONS"].split(","):
        a0, b0 = (int(x, 16) for x in rg.split(":"))
        tot = {c: sum(int(r[idx[c]] or 0) for a, r in allrows if a0 <= a < b0) for c in reasons}
        s_ = sum(tot.values())
        top = sorted(tot.items(), key=lambda x: -x[1])[:6]
        print(f"{a0:6x}-{b0:6x} {100 * s_ / ts:5.1f}%: " + ", ".join(f"{c[6:]} {100 * v / max(s_, 1):.0f}%" for c, v in top))
