"""Markdown summary of one-kernel `ncu --set full` report: key metrics, stall mix, SASS opcode mix.
usage: python tools/ncu_summary.py rep.ncu-rep [units_of_work] [kernel_regex] > summary.md"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else None
kregex = sys.argv[3] if len(sys.argv) > 3 else None  # summarise the first launch whose name matches


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u = raw[0], raw[1]
iK = h.index("Kernel Name")
rows = [r for r in raw[2:] if len(r) == len(h) and (kregex is None or re.search(kregex, r[iK]))]
v = rows[0]
d, un = dict(zip(h, v)), dict(zip(h, u))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
print(f"## {rep.split('/')[-1]}\n")
print("| metric | value | unit |\n|---|---|---|")
for k in keys:
    if k in d:
        print(f"| `{k}` | {d[k]} | {un.get(k, '')} |")
if units and "smsp__inst_executed.sum" in d:
    wi = float(d["smsp__inst_executed.sum"].replace(",", ""))
    print(f"| lane-instructions per unit of work | {32 * wi / units:.3f} | (units = {units:.4g}) |")
st = []
for k, val in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(val.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1.0
print("\n**Warp-state samples:** " + ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in sorted(st, reverse=True)[:9]))
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
# one block per profiled launch: "Kernel Name" line, header, rows; take the first matching block
starts = [i for i, r in enumerate(sass) if r and r[0] == "Kernel Name" and (kregex is None or re.search(kregex, r[1]))]
b0 = starts[0]
nxt = [i for i, r in enumerate(sass) if i > b0 and r and r[0] == "Kernel Name"]
block = sass[b0 + 1:(nxt[0] if nxt else len(sass))]
hh = block[0]
iE, iS, iSrc = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
ops, stalls = Counter(), Counter()
for r in block[1:]:
    src = re.sub(r"^@!?U?P\w+\s+", "", r[iSrc].strip())
    op = src.split(" ")[0].split(".")[0] if src else "?"
    ops[op] += int(r[iE])
    stalls[op] += int(r[iS])
T, S = sum(ops.values()), sum(stalls.values()) or 1
print("\n| SASS opcode | share of executed warp-instr | share of stall samples |" + (" lane-instr / unit |" if units else "") + "\n|---|---|---|" + ("---|" if units else ""))
for op, n in ops.most_common(16):
    print(f"| {op} | {100 * n / T:.2f}% | {100 * stalls[op] / S:.2f}% |" + (f" {32 * n / units:.3f} |" if units else ""))
