"""Key metrics + SASS opcode mix of one kernel in an ncu report.
usage: python tools/ncu_summary.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
KEYS = ["Duration", "Elapsed Cycles", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp", "DRAM Throughput",
        "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Executed Instructions", "Branch Efficiency", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Grid Size", "Dynamic Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in KEYS:
        print(f"  {d['Metric Name']:45s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h, v = rr[0], rr[2]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"):
        if name in h:
            print(f"  {name:60s} {v[h.index(name)]} {rr[1][h.index(name)]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot, thr, stall = collections.Counter(), collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Source"]].strip():
        continue
    toks = r[ix["Source"]].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    base = op.split(".")[0]
    tot[base] += int(r[ix["Instructions Executed"]] or 0)
    thr[base] += int(r[ix["Thread Instructions Executed"]] or 0)
    stall[base] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
T, S = sum(tot.values()), max(1, sum(stall.values()))
print(f"  warp instr {T:.3e}, avg threads/instr {sum(thr.values()) / max(T, 1):.1f}")
for k, v in tot.most_common(14):
    print(f"    {k:8s} {100 * v / T:5.1f}%  thr={thr[k] / max(v, 1):5.1f}  stall={100 * stall[k] / S:5.1f}%")
