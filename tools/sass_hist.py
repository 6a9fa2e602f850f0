"""Summarise an ncu SASS source page (csv): executed warp-instructions per opcode and stall share.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/sass_hist.py x.csv [units]"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else None
h = rows[1]
data = rows[2:]
iE, iS, iSrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ops, stalls = Counter(), Counter()
for r in data:
    src = r[iSrc].strip()
    src = re.sub(r"^@!?U?P\w+\s+", "", src)
    op = src.split(" ")[0].split(".")[0] if src else "?"
    ops[op] += int(r[iE])
    stalls[op] += int(r[iS])
tot, stot = sum(ops.values()), sum(stalls.values())
print(f"total warp-instr {tot:.4e}" + (f"  lane-instr/unit {32 * tot / units:.2f}" if units else ""))
for op, n in ops.most_common(30):
    print(f"{op:12s} {n / tot * 100:6.2f}%  stall {stalls[op] / max(stot, 1) * 100:6.2f}%" + (f"  per-unit {32 * n / units:.3f}" if units else ""))
