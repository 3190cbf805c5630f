#!/usr/bin/env python
"""Benchmark of the B200 two-stage Householder orthogonalization hot path.

Metric (BASELINE.json): fp64 two-stage orthogonalization GFLOP/s (and HBM
GB/s) vs roofline.  Workload at N=1: the north_star headline point,
`two_stage_qr(V, A)` with n=2^24, k0=128, k=64, float64, choice "qr",
intra "householder".  One step = one full call on HBM-resident inputs.
GFLOP/s uses the algorithmic flop count of SURVEY.md §8(d):

  F_alg = 8 n k0 k + 4 (n-k0) k^2 - 4/3 k^3 + n k0 (k0+1)
  B_alg = 8 [n (k0 + 2k) + k0 k + k^2]

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
        (N>1 under torchrun: rows are sharded across ranks, strong scaling)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_HEAD, K0_HEAD, K_HEAD = 1 << 24, 128, 64
SHARE = os.environ.get("OTS_BENCH_SHARE_DEVICE") == "1"
REF_SAMPLE_N = 1 << 18          # bounded CPU sample (same k0, k)


def f_alg(n, k0, k):
    return 8.0 * n * k0 * k + 4.0 * (n - k0) * k * k - 4.0 / 3.0 * k ** 3 + n * k0 * (k0 + 1.0)


def b_alg(n, k0, k):
    return 8.0 * (n * (k0 + 2.0 * k) + k0 * k + k * k)


def gram_flops(n, k0, k):
    """algorithmic flops of one gram launch (V^T V half + V_b^T A_b)"""
    return n * k0 * (k0 + 1.0) + 2.0 * (n - k0) * k0 * k


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port (numpy/LAPACK restatement of
# the reference's pure-Python path) on the host cores
# --------------------------------------------------------------------------
def cpu_inputs(n, k0, k, seed=7):
    from paper_2602_14449_b200 import workloads as W
    rng = W.make_rng(seed)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    return v, a


def time_oracle(n, k0, k, reps, warmup):
    from oracle import twostage_oracle as O
    v, a = cpu_inputs(n, k0, k)
    for _ in range(warmup):
        O.two_stage(v, a, "qr")
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.two_stage(v, a, "qr")
        ts.append(time.perf_counter() - t0)
    return ts


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = cpu_cores()
    n, k0, k = REF_SAMPLE_N, K0_HEAD, K_HEAD
    ts = time_oracle(n, k0, k, args.steps, args.warmup)
    sec = float(np.mean(ts))
    gf = f_alg(n, k0, k) / sec / 1e9
    line = {
        "metric": "fp64 two-stage orthogonalization GFLOP/s", "impl": "reference",
        "value": round(gf, 4), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "two_stage_qr choice=qr intra=householder f64",
                   "n": n, "k0": k0, "k": k, "sample_of": f"n=2^24 headline (1/{N_HEAD // n} of rows)"},
        "cpu_baseline": {"value": round(gf, 4), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"oracle two_stage (numpy/LAPACK port of orthoqr, incl. "
                                   f"reflector_diagnostics) n={n} k0={k0} k={k}, "
                                   f"OpenBLAS threads={cores}",
                         "note": "reflector_diagnostics (k0 x n solve + SVD) is about 57% of this time; the "
                                 "GPU path derives the diagnostics from k0 x k0 data (SURVEY A.3)"},
        "e2e": {"value": round(gf, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            ids = [] if self.device is None else [f"--id={self.device}"]
            self.proc = subprocess.Popen(
                ["nvidia-smi", *ids, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(n, k0, k, device, seed=1234):
    """Seeded synthetic headline inputs generated on the device: A ~ N(0,1),
    V = Q-factor of a N(0,1) n x k0 block orthonormalised by this package's own
    GPU block Householder QR (Algorithm 3)."""
    import torch
    import paper_2602_14449_b200 as P
    g = torch.Generator(device=f"cuda:{device}")
    g.manual_seed(seed)
    G = torch.randn((n, k0), generator=g, dtype=torch.float64, device=f"cuda:{device}")
    blocks = [G[:, i:i + 64].contiguous() for i in range(0, k0, 64)]
    V = P.block_householder_qr(blocks).q.contiguous()
    del G, blocks
    A = torch.randn((n, k), generator=g, dtype=torch.float64, device=f"cuda:{device}")
    return V, A


def gram_check(V, A, res):
    """loss ||[V,Q]^T[V,Q]-I||_2 and relative residual from (k0+k)^2 Grams
    (verification only, outside the timed region)."""
    import torch
    VQ = torch.cat([V, res.q], dim=1)
    G = (VQ.T @ VQ).cpu().numpy()
    loss = float(np.max(np.abs(np.linalg.eigvalsh(G) - 1.0)))
    Rm = A - V @ res.s - res.q @ res.r
    rn = np.sqrt(max(np.linalg.eigvalsh((Rm.T @ Rm).cpu().numpy()).max(), 0.0))
    an = np.sqrt(max(np.linalg.eigvalsh((A.T @ A).cpu().numpy()).max(), 0.0))
    return loss, rn / an


def load_traffic(kernel_key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d.get(kernel_key)
    except Exception:
        return None


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2602_14449_b200 as P
    from paper_2602_14449_b200 import _native as NT
    from paper_2602_14449_b200 import _device as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # OTS_BENCH_SHARE_DEVICE=1: every rank on cuda:0 with gloo collectives --
    # a plumbing check of the N>1 leg on a one-GPU box, never a measurement
    share = SHARE
    torch.cuda.set_device(0 if share else local)
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl")
    n, k0, k = args.n, args.k0, args.k

    if world > 1:
        return run_sharded(args, n, k0, k, rank, world, 0 if share else local)

    ctx = NT.context(local)
    L = NT.lib()
    peak = (NT.C.c_double if hasattr(NT, "C") else None)
    import ctypes as C
    pk = C.c_double()
    NT.check(L.ots_fp64_peak(ctx, C.byref(pk)), ctx)
    fp64_peak = float(pk.value)

    V, A = make_inputs(n, k0, k, local)
    torch.cuda.synchronize()

    # warm-up
    for _ in range(args.warmup):
        res = P.two_stage_qr(V, A)
    torch.cuda.synchronize()
    rep = P.compute_metrics(V, A, res, augmented=True)   # GPU metrics judge (metrics.py)
    loss, resid = rep.loss_orth, rep.rel_residual
    del res

    # timed region: K steps, inputs (24 GiB) >> L2 (126 MB), no flush needed
    L.ots_set_profiling(ctx, 1)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phase_ms = {}
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        res = P.two_stage_qr(V, A)
        for nm, ms in NT.profile(ctx):
            phase_ms[nm] = phase_ms.get(nm, 0.0) + ms
    e1.record(stream)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / args.steps
    launches = L.ots_last_launch_count(ctx) * args.steps
    clk = clocks.stop()
    L.ots_set_profiling(ctx, 0)
    del res
    phase_ms = {kk: vv / args.steps for kk, vv in phase_ms.items()}

    F, B = f_alg(n, k0, k), b_alg(n, k0, k)
    gflops = F / (step_ms * 1e-3) / 1e9
    gbs = B / (step_ms * 1e-3) / 1e9
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6553.3) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.3
    t_roof = max(B / (hbm * 1e9), F / (fp64_peak * 1e12))

    # dominant kernel: the phase with the largest share of the step
    dom = max(phase_ms, key=phase_ms.get)
    # flops the dominant launch EXECUTES (its own algorithmic count).  Direct-Q
    # pipeline (ots_last_fast = 1): "gram" is the tile-Gram pass over [V | A]
    # (V^T V, V^T A and A^T A per tall tile), "final" the pass Q = [V | A] Coef.
    w = k0 + k
    fast = NT.last_fast(ctx) == 1
    dom_flops = {
        "gram": (n - k0) * w * (w + 1.0) if fast else gram_flops(n, k0, k),
        "final": 2.0 * (n - k0) * w * k,
        "apply1": 2.0 * (n - k0) * k0 * k,
        "gram2": 2.0 * (n - k0) * k0 * k,
        "apply2": 2.0 * (n - k0) * k0 * k,
        "factor": 2.0 * (n - k0) * k * k - 2.0 / 3.0 * k ** 3,
        "qform": 2.0 * (n - k0) * k * k - 2.0 / 3.0 * k ** 3,
    }.get(dom, 0.0)
    dom_tf = dom_flops / (phase_ms[dom] * 1e-3) / 1e12 if dom_flops else 0.0
    roofline = {"bound": "tensor", "kernel": dom, "achieved": round(dom_tf, 3),
                "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
                "frac": round(dom_tf / fp64_peak, 4) if fp64_peak else None,
                "traffic": load_traffic(dom + "_direct" if fast else dom),
                "peak_source": "FP64 DMMA loop measured in this run (ots_fp64_peak); "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "phase_ms": {kk: round(vv, 3) for kk, vv in phase_ms.items()},
                "step_frac_of_roofline": round(t_roof / (step_ms * 1e-3), 4),
                "pipeline": "direct-Q (tile Grams of [V | A]; executes fewer flops than F_alg)" if fast
                            else "materialised X",
                # flops the step EXECUTES on its two streaming passes (the per-tile algebra adds ~3%)
                "step_executed_tflops": round(((n - k0) * w * (w + 1.0) + 2.0 * (n - k0) * w * k
                                               if fast else F) / (step_ms * 1e-3) / 1e12, 3),
                "step_hbm_gbs": round(gbs, 1), "step_hbm_frac": round(gbs / hbm, 4)}

    # e2e: public API with host buffers (pinned), H2D of V, A and D2H of Q, R, S
    # every step.  Serial: copy in, call, copy out.  Streamed (the headline e2e):
    # the host-buffer front end `two_stage_qr_stream`, which overlaps call s's
    # compute with the H2D of call s+1 and the D2H of call s-1.
    from paper_2602_14449_b200.stream import two_stage_qr_stream
    e2e_steps = max(2, args.steps)          # all K steps (fill and drain amortised over K)
    Vh = V.cpu().pin_memory()
    Ah = A.cpu().pin_memory()
    Qh = torch.empty((n, k), dtype=torch.float64).pin_memory()
    Rh = torch.empty((k, k), dtype=torch.float64).pin_memory()
    Sh = torch.empty((k0, k), dtype=torch.float64).pin_memory()
    Vd = torch.empty_like(V)
    Ad = torch.empty_like(A)
    del V, A
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(2):
        Vd.copy_(Vh, non_blocking=True)
        Ad.copy_(Ah, non_blocking=True)
        res = P.two_stage_qr(Vd, Ad)
        Qh.copy_(res.q, non_blocking=True)
        Rh.copy_(res.r, non_blocking=True)
        Sh.copy_(res.s, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = e0.elapsed_time(e1) / 2
    del Vd, Ad, res, Qh, Rh, Sh
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    ws = {}
    for r_ in two_stage_qr_stream([(Vh, Ah)] * 2, workspace=ws):   # allocate slots, pin outputs
        r_.wait()
    torch.cuda.synchronize()
    e0.record(stream)
    last = None
    for r_ in two_stage_qr_stream([(Vh, Ah)] * e2e_steps, workspace=ws):
        last = r_
    stream.wait_event(last.event)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    h2d = (n * k0 + n * k) * 8
    d2h = (n * k + k * k + k0 * k) * 8
    del Vh, Ah, last, ws

    # CPU baseline (oracle port) on a bounded sample, rank 0 at N=1
    cores = cpu_cores()
    cpu_line = None
    if not args.no_cpu:
        ts = time_oracle(REF_SAMPLE_N, k0, k, reps=3, warmup=1)
        csec = float(np.median(ts))
        cpu_line = {"value": round(f_alg(REF_SAMPLE_N, k0, k) / csec / 1e9, 4), "unit": "GFLOP/s",
                    "cores": cores, "kind": "port",
                    "sample": f"oracle two_stage (numpy/LAPACK port of orthoqr incl. "
                              f"reflector_diagnostics) n={REF_SAMPLE_N} k0={k0} k={k}, "
                              f"median of 3, OpenBLAS threads={cores}",
                    "note": "the reference's reflector_diagnostics forms the k0 x n solve and an SVD of it "
                            "(about 57% of the CPU time), which the GPU path derives from k0 x k0 data "
                            "(SURVEY A.3): part of the GPU/CPU ratio is algorithmic"}

    line = {
        "metric": "fp64 two-stage orthogonalization GFLOP/s", "value": round(gflops, 2),
        "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "headline two_stage_qr(V, A) choice=qr intra=householder",
                   "n": n, "k0": k0, "k": k, "parallelism": "row-sharded x1",
                   "l2": "inputs 24 GiB >> 126 MB L2 (no flush needed)",
                   "inputs": "seeded torch Philox on device; V = own GPU block Householder QR"},
        "hbm_gbs": round(gbs, 1),
        "roofline": roofline,
        "cpu_baseline": cpu_line,
        "e2e": {"value": round(F / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                "ms_per_step": round(e2e_ms, 2), "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "api": "paper_2602_14449_b200.stream.two_stage_qr_stream (pinned host buffers; "
                       "H2D of call s+1 and D2H of call s-1 overlap call s)",
                "serial_ms_per_step": round(e2e_serial_ms, 2),
                "serial_value": round(F / (e2e_serial_ms * 1e-3) / 1e9, 2)},
        "gpu_launches": launches,
        "clocks": clk,
        "check": {"loss_orth": loss, "rel_residual": resid, "bound_10nu": 10 * n * 2.0 ** -53},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, n, k0, k, rank, world, local):
    """N > 1: rows of the headline problem split across ranks (strong scaling,
    NCCL for the SURVEY 8(e) collectives); rank 0 prints the line."""
    import torch.distributed as dist
    from paper_2602_14449_b200 import dist as PD
    m = PD.bench_sharded(args, n, k0, k, rank, world, local)
    if rank == 0:
        F = f_alg(n, k0, k)
        ms = m["ms"]
        val = F / (ms * 1e-3) / 1e9
        t_roof = F / (world * 37.0e12)
        line = {
            "metric": "fp64 two-stage orthogonalization GFLOP/s", "value": round(val, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "headline two_stage_qr(V, A) choice=qr intra=householder, row-sharded",
                       "n": n, "k0": k0, "k": k,
                       "parallelism": (f"row-sharded x{world} (NCCL allreduce/allgather/broadcast of the "
                                       f"k0x(k0+k), KTxKT, k0xk blocks)") if not SHARE else
                                      (f"row-sharded x{world} ranks SHARING ONE GPU, gloo host-staged "
                                       f"collectives: plumbing check of the N>1 leg, not a scaling number"),
                       "l2": "inputs >> L2 on every rank (no flush needed)"},
            "roofline": {"bound": "tensor", "kernel": "whole step", "achieved": round(F / (ms * 1e-3) / 1e12, 3),
                         "peak": round(world * 37.0, 1), "unit": "TFLOP/s",
                         "frac": round(t_roof / (ms * 1e-3), 4), "traffic": None,
                         "peak_source": "N x FP64 DMMA peak measured at N=1 (profiles/r01_fp64_peak.json)"},
            "cpu_baseline": None,
            "e2e": {"value": round(F / (m["e2e_ms"] * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                    "ms_per_step": round(m["e2e_ms"], 2), "h2d_bytes_per_step": m["h2d"],
                    "d2h_bytes_per_step": m["d2h"], "steps": m["e2e_steps"],
                    "api": "dist.run_phases per rank with pinned host shards (serial copy in / call / copy out)"},
            "gpu_launches": m["launches"],
            "clocks": m["clocks"],
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--rows", dest="n", type=int, default=N_HEAD)
    ap.add_argument("--k0", type=int, default=K0_HEAD)
    ap.add_argument("--k", type=int, default=K_HEAD)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
