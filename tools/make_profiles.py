"""Turn one evidence run's gpurun_out files into the tracked profiles/ summaries:
python tools/make_profiles.py TAG PREFIX   (e.g. r02e s16)
  gpurun_out/PREFIX_bench.json, _launches.csv, _summary.txt (+ _zsummary.txt),
  _configs.log, _share2.log  ->  profiles/TAG_*"""
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, pre = sys.argv[1], sys.argv[2]
G = lambda n: os.path.join(ROOT, "gpurun_out", f"{pre}_{n}")
P = lambda n: os.path.join(ROOT, "profiles", f"{tag}_{n}")

bench = json.load(open(G("bench.json")))
shutil.copy(G("bench.json"), P("bench.json"))
ph = bench["roofline"]["phase_ms"]
step = bench["ms_per_step"]

# ---- launch list
shutil.copy(G("launches.csv"), P("bench_launches.csv"))
rows = list(csv.reader(open(P("bench_launches.csv"))))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
names = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi]) / 1000) for r in rows[hi + 1:] if len(r) > vi]
idx = [i for i, x in enumerate(names) if "tgram_kernel" in x[0]]
st = idx[-1] - 1
en = st
while en < len(names) and "qtop" not in names[en][0]:
    en += 1
one = names[st:en + 1]
tot = sum(x[1] for x in one)
by = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), P("bench_launches.csv")],
                    capture_output=True, text=True).stdout
out = [f"# Launch list of `python bench.py --steps 2 --warmup 1` under `ncu --metrics gpu__time_duration.sum --clock-control none` ({tag})\n",
       f"Per-launch times under ncu are serialised and cold-cache; the kernels' SHARE of a step is what is compared with the live "
       f"CUDA-event phases of `{tag}_bench.json` (gram {ph['gram']} ms = {100 * ph['gram'] / step:.0f}%, final {ph['final']} ms = "
       f"{100 * ph['final'] / step:.0f}% of the {step} ms step).\n",
       "## One headline step (n = 2^24, k0 = 128, k = 64), in launch order\n", "| # | kernel | us | share |", "|---|---|---|---|"]
for i, x in enumerate(one):
    out.append(f"| {i} | `{x[0][:70]}` | {x[1]:.1f} | {100 * x[1] / tot:.1f}% |")
out.append(f"| | **sum** | {tot:.1f} | |\n")
out.append("(`seedA` runs on the side stream beside `tgram`, `diag` beside `final_nn`: the step is shorter than the sum.)\n")
out.append("## Whole command, by kernel\n")
out += by.splitlines()
open(P("bench_launches.md"), "w").write("\n".join(out) + "\n")


# ---- ncu summaries
def table(path):
    txt = open(path).read()
    res = []
    for b in re.split(r"^== ", txt, flags=re.M)[1:]:
        name = re.sub(r"^\[\d+\]\s*", "", b.split("\n")[0]).split("(")[0].replace("void ", "")

        def get(key):
            m = re.search(re.escape(key) + r"\s+([0-9.]+)\s*(\S*)", b)
            return (float(m.group(1)), m.group(2)) if m else (float("nan"), "")
        dur, rd, wr = get("Duration"), get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        dm = get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
        f64 = get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
        regs, sm, iss = get("Registers Per Thread"), get("Dynamic Shared Memory Per Block"), get("Issue Slots Busy")
        stl = {k: get(f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio")[0]
               for k in ("math_pipe_throttle", "wait", "long_scoreboard", "short_scoreboard", "barrier", "not_selected")}
        top = sorted(((v, k) for k, v in stl.items() if v == v), reverse=True)[:3]
        res.append(f"| `{name}` | {dur[0]:.2f} {dur[1]} | {dm[0]:.1f}% | {f64[0]:.1f}% | {iss[0]:.1f}% | {rd[0]:.3f} / {wr[0]:.3f} | "
                   f"{int(regs[0])} | {sm[0]:.0f} {sm[1]} | " + ", ".join(f"{k} {v:.2f}" for v, k in top) + " |")
    return res


hdr = ["| kernel | duration | DMMA pipe | FP64 pipe | issue slots busy | DRAM read / write (GB) | regs | dyn. smem | top stalls (warps per issue) |",
       "|---|---|---|---|---|---|---|---|---|"]
tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
md = [f"# ncu --set full summaries ({tag})\n",
      "Numbers taken under the profiler are evidence for pipe utilisation and traffic only; times come from "
      f"`{tag}_bench.json` / `{tag}_configs.md`.  Each command exited 0 without ncu first.\n",
      "## Direct-Q pipeline at the headline (n = 2^24, k0 = 128, k = 64)\n",
      "`ncu --set full --clock-control none --import-source on -k \"regex:tgram_kernel|final_nn|tile_alg|chain_gsweep|gs_coef|coef_b\" "
      "-s 18 -c 6 python tools/fast_check.py time`\n"] + hdr + table(G("summary.txt"))
w = bench["config"]["k0"] + bench["config"]["k"]
n = bench["config"]["n"]
gfl = (n - 128) * w * (w + 1.0)
ffl = 2.0 * (n - 128) * w * 64
md += ["", "Traffic against the algorithmic bytes (per launch):",
       f"* `tgram_kernel`: {tr['gram_direct'] / 1e9:.2f} GB measured; algorithmic = V and A read once (25.77 GB) + tile Gram slots and "
       "CTA totals written (0.47 GB at 8192-row tiles) = 26.24 GB.",
       f"* `final_nn_kernel`: {tr['final_direct'] / 1e9:.2f} GB measured; algorithmic = V and A read once (25.77 GB) + Q written "
       "(8.59 GB) + coefficients (0.20 GB) = 34.56 GB.",
       "* whole call: about 63 GB against 160 GB for the round-1 pipeline (V is read twice instead of four times, X / Q_ are never written).",
       "",
       f"Roofline (FP64 DMMA, measured peak {bench['roofline']['peak']} TF/s, `ots_fp64_peak`): `tgram_kernel` executes "
       f"n (k0+k)(k0+k+1) = {gfl:.3g} flop in {ph['gram']} ms live = {gfl / ph['gram'] / 1e9:.1f} TF/s = "
       f"{gfl / ph['gram'] / 1e9 / bench['roofline']['peak']:.2f} of the peak; `final_nn_kernel` 2 n (k0+k) k = {ffl:.3g} flop in "
       f"{ph['final']} ms = {ffl / ph['final'] / 1e9:.1f} TF/s = {ffl / ph['final'] / 1e9 / bench['roofline']['peak']:.2f}.  Both are bound "
       "by the DMMA pipe (math-pipe throttle / the fixed-latency wait between a warp's dependent issues are the top stalls)."]
if os.path.exists(G("zsummary.txt")):
    md += ["", "## Complex128 Gram-form intra QR, configs[3] (n = 2^22, k0 = k = 64)\n",
           "`ncu --set full --clock-control none -k \"regex:zgs_|tgram_kernel|final_nn\" -s 10 -c 5 python tools/zgs_check.py time`\n"] + hdr + \
        table(G("zsummary.txt"))
    md += ["", "`zgs_sweep_kernel` / `zgs_coef_kernel` run the complex 64 x 64 algebra on CUDA cores (no complex MMA exists): "
           "latency-bound, one CTA per chain, about 5% of the call; the n-row work is on the DMMA kernels of the real path."]
open(P("ncu_summary.md"), "w").write("\n".join(md) + "\n")

# ---- configs
if os.path.exists(G("configs.log")):
    recs = [json.loads(l) for l in open(G("configs.log")) if l.strip().startswith("{")]
    json.dump(recs, open(P("configs.json"), "w"), indent=1)
    o = [f"# Full-size BASELINE configurations (one B200, `tools/configs_report.py`, {tag})\n",
         "Device time per call (CUDA events, inputs resident; median of 3 after a warm-up, C5 one call per step), stability from the GPU "
         "metrics judge (`compute_metrics`, augmented [V, Q], real and complex), against 10 n u.  C3's inputs cancel (A partly in "
         "range(V)): the direct-Q attempt is rejected on the device and the call takes the materialised-X pipeline.  C4 and its B-inner variant run the complex "
         "Gram-form intra QR.  its GFLOP/s "
         "column counts executed work of the incremental-Gram formulation, not F_alg.\n",
         "| config | n | k0 | k | ms | GFLOP/s | loss | residual | 10 n u | kappa(T) |", "|---|---|---|---|---|---|---|---|---|---|"]
    for d in recs:
        o.append(f"| {d['config']} | {d['n']} | {d['k0']} | {d['k']} | {d['ms']} | {d['gflops']:.1f} | {d['loss']:.2e} | "
                 f"{d['residual']:.2e} | {d['bound_10nu']:.1e} | {d.get('kappa_t', 0):.4f} |")
    c5 = [d["ms"] for d in recs if d["config"].startswith("C5")]
    if c5:
        o.append(f"\nC5 sweep (8 steps after the first block): {sum(c5):.1f} ms.  Single shots in a process holding ~150 GB of tensors: a step can include "
                 f"allocator work (up to +140 ms); `tools/krylov_c5.py` alone measures the sweep at "
                 f"1046.5 ms (`profiles/{tag}_c5_sweep.json`).")
    open(P("configs.md"), "w").write("\n".join(o) + "\n")
if os.path.exists(G("share2.log")):
    shutil.copy(G("share2.log"), P("bench_share2_plumbing.log"))
print("wrote", [f for f in sorted(os.listdir(os.path.join(ROOT, "profiles"))) if f.startswith(tag)])
