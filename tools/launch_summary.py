"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("void ", "")
    v = float(r[iv].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
unit = "ns"
allv = sum(tot.values())
print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / allv:.1f}% |")
print(f"| **all** | {sum(cnt.values())} | {allv / 1e6:.3f} | 100% |")
