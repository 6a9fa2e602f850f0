"""Per-CUDA-source-line instruction and stall totals from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "File Path", "Function Name") and len(r) > 8:
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            st = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        res.append((ie, st, r[0], r[1].strip()[:90]))
T = sum(x[0] for x in res) or 1
S = sum(x[1] for x in res) or 1
for ie, st, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * ie / T:6.2f}% instr {100 * st / S:6.2f}% stall  L{ln:>4}  {src}")
