"""Per-kernel SASS instruction summary of libots.so (cuobjdump -sass):
DMMA / DFMA / LDGSTS (cp.async) / UBLKCP (cp.async.bulk) / UTMALDG counts.
python tools/sass_summary.py > profiles/rNN_sass_summary.md"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2602_14449_b200", "libots.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
pats = {"DMMA": r"\bDMMA\b", "DFMA": r"\bDFMA\b", "LDGSTS": r"\bLDGSTS\b", "UBLKCP": r"\bUBLKCP\b",
        "UTMALDG": r"\bUTMALDG\b", "SYNCS": r"\bSYNCS\b", "STL/LDL": r"\b(STL|LDL)\b"}
cnt = collections.OrderedDict()
cur = None
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = cur.rsplit("(", 1)[0]
        cnt[cur] = collections.Counter()
        continue
    if cur:
        for k, p in pats.items():
            if re.search(p, line):
                cnt[cur][k] += 1
print("# SASS instruction summary of libots.so (sm_100a, `tools/sass_summary.py`)\n")
print("| kernel | " + " | ".join(pats) + " |")
print("|---|" + "---|" * len(pats))
tot = collections.Counter()
for k, c in cnt.items():
    if sum(c.values()) == 0:
        continue
    tot.update(c)
    print(f"| `{k}` | " + " | ".join(str(c[p]) for p in pats) + " |")
print("| **total** | " + " | ".join(str(tot[p]) for p in pats) + " |")
print("\nDMMA.8x8x4 is the FP64 tensor path (tcgen05 has no f64 kind on sm_100a).  "
      "UBLKCP = `cp.async.bulk` global->shared row copies completing on an mbarrier by bytes "
      "(the TMA engine's non-tensor form) in the two streaming kernels of the direct-Q pipeline "
      "(`tgram_kernel`, `final_nn_kernel`); LDGSTS = 16-byte `cp.async` in the other streaming kernels "
      "and as the fallback for cut stages.")
