"""Summarise an ncu --set full report into profiles/ (text): headline
metrics, LSU wavefront split, and the SASS opcode mix per unit of work.

    python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX UNITS LABEL > profiles/x.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kern, units, label = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", *a], capture_output=True, text=True).stdout


print(f"# {label}: {rep} kernel ~ {kern}; per-unit figures divide by {units:.4g}")
det = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = det[0]
mi, vi, ui, si = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Section Name")
keep = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Active Warps per SM",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
for x in det[1:]:
    if x[mi] in keep:
        print(f"{x[si]} | {x[mi]} | {x[ui]} | {x[vi]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
rh, rv = raw[0], raw[2]
print("\n## raw")
for i, n in enumerate(rh):
    if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
             "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
             "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
             "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
             "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"):
        print(f"{n} = {rv[i]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
sh, rows = src[1], src[2:]
s_i, e_i, st_i = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
ops, stl = collections.Counter(), collections.Counter()
for x in rows:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9]+)?)", x[s_i].strip())
    op = m.group(2) if m else "?"
    ops[op] += int(x[e_i] or 0)
    stl[op] += int(x[st_i] or 0)
tot, stt = sum(ops.values()), max(1, sum(stl.values()))
print(f"\n## SASS mix: {tot} warp instructions, {tot / units:.2f} per unit")
for op, c in ops.most_common(20):
    print(f"{op:18s} {c / units:7.3f}/unit  stall share {100 * stl[op] / stt:5.1f}%")
