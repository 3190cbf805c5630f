"""Hot SASS lines of one kernel in an ncu report (warp-stall samples):
python tools/ncu_hot.py REP KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi]
si, src, ad = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Address")
stalls = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
data, seen = [], set()
agg = {}
for r in rows[hi + 1:]:
    if len(r) > si and r[si].strip().isdigit() and r[ad] not in seen:
        seen.add(r[ad])
        top = sorted(((int(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:2]
        for i in stalls:
            agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
        data.append((int(r[si]), r[ad], r[src], top))
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", len(data))
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:7d} {100 * d[0] / tot:5.1f}% {d[1][-5:]} {d[2][:60]:60s} {d[3]}")
