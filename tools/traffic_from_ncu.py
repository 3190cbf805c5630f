"""DRAM traffic per launch of the named kernels from an ncu --set full report
(`ncu -i REP --page raw --csv`), written into profiles/traffic.json under the
keys bench.py looks up:  python tools/traffic_from_ncu.py REP key=kernel_regex ..."""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
path = os.path.join(ROOT, "profiles", "traffic.json")
out = json.load(open(path)) if os.path.exists(path) else {}
for spec in sys.argv[2:]:
    key, pat = spec.split("=", 1)
    for r in rows[2:]:
        if re.search(pat, r[ki]):
            rd = float(r[ri]) * scale[units[ri]]
            wr = float(r[wi]) * scale[units[wi]]
            out[key] = int(rd + wr)
            out["_" + key + "_source"] = (f"ncu --set full --clock-control none ({os.path.basename(rep)}), kernel {r[ki][:60]}: "
                                          f"dram__bytes_read.sum {rd / 1e9:.3f} GB + dram__bytes_write.sum {wr / 1e9:.3f} GB per launch")
            break
json.dump(out, open(path, "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if not k.startswith("_")}))
