"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, time, share.
usage: python tools/launch_summary.py launches.csv [--skip-setup N]"""
import csv
import re
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
iN, iV, iU, iG = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
iM = h.index("Metric Name")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = OrderedDict()
tot = 0.0
for r in rows[i + 1:]:
    if r[iM] != "gpu__time_duration.sum":  # other metrics (e.g. DRAM bytes) in the same capture
        continue
    name = re.sub(r"^void\s+", "", r[iN])
    name = re.sub(r"\(.*$", "", name).replace("<unnamed>::", "")
    v = float(r[iV].replace(",", "")) * scale[r[iU]]
    a = agg.setdefault(name, [0, 0.0, r[iG]])
    a[0] += 1
    a[1] += v
    tot += v
print(f"| kernel | launches | grid | total ms | share |\n|---|---|---|---|---|")
for k, (n, t, gsz) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {gsz} | {t:.3f} | {t / tot * 100:.2f}% |")
print(f"| total | | | {tot:.3f} | 100% |")
