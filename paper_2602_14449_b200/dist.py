"""Row-sharded multi-GPU two_stage_qr.

One process per GPU; rank r owns the contiguous rows [row0_r, row0_r + n_r) of
V, A and Q (rank 0 owns the top rows and needs n_0 >= k0 + k).  Every n-length
operation is row-local; only small blocks cross GPUs:

  phase            local work (C-ABI)                     collective
  gram             [V^T V | V_b^T A_b] partial            allreduce(sum)  (k0 x (k0+k))
  top rows         rank 0: V_t, A_t                       broadcast       (k0 x (k0+k))
  seed             P, T, Z1, S (redundant on every rank)  --
  factor           X = A_b + V_b Z1; local TSQR -> R_r    allgather       (KT x KT per rank)
  tree             top QR of the stacked R_r -> C_r       --  (redundant)
  qform            Q_ (local), Y2_r = -V_b^T Q_           allreduce(sum)  (k0 x k)
                   rank 0: LAPACK sign vector             broadcast       (k)
  finish           Z2 = T^{-1} Y2; Q = (Q_ + V_b Z2) S    --

The orchestration is written against two small interfaces so the same code
runs over NCCL (`TorchComm`), gloo on CPU with a numpy phase double (tests),
or as an in-process simulation of G ranks on one GPU (`LocalComm`, tests).
"""

from __future__ import annotations

import ctypes as C

from . import _device as D
from . import errors as E
from ._native import CHOICES, check, lib


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed process group (NCCL for device tensors; with the gloo
    backend device tensors are staged through host memory)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host = dist.get_backend(group) == "gloo"

    def _stage(self, t):
        return t.cpu() if (self.host and t.is_cuda) else t

    def allreduce_sum(self, t):
        h = self._stage(t)
        self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
        if h is not t:
            t.copy_(h)
        return t

    def broadcast(self, t, src=0):
        h = self._stage(t)
        self.dist.broadcast(h, src=src, group=self.group)
        if h is not t:
            t.copy_(h)
        return t

    def allgather_cat(self, t):
        import torch
        h = self._stage(t)
        out = [torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(out, h, group=self.group)
        cat = torch.cat(out, dim=0)
        return cat.to(t.device) if h is not t else cat


class LocalComm:
    """In-process communicator for G simulated ranks run as threads in one
    process (one device).  Collectives synchronise the device, then combine
    through shared slots; no kernel ever waits on another rank's kernel."""

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    @staticmethod
    def make_shared(world):
        import threading
        return {"bar": threading.Barrier(world), "slots": [None] * world}

    def _sync(self, t):
        if hasattr(t, "is_cuda") and t.is_cuda:
            D.torch().cuda.synchronize(t.device)

    def allreduce_sum(self, t):
        self._sync(t)
        self.sh["slots"][self.rank] = t.clone()
        self.sh["bar"].wait()
        tot = self.sh["slots"][0].clone()
        for r in range(1, self.world):
            tot += self.sh["slots"][r]
        self.sh["bar"].wait()
        t.copy_(tot)
        return t

    def broadcast(self, t, src=0):
        self._sync(t)
        if self.rank == src:
            self.sh["slots"][src] = t.clone()
        self.sh["bar"].wait()
        if self.rank != src:
            t.copy_(self.sh["slots"][src])
        self.sh["bar"].wait()
        return t

    def allgather_cat(self, t):
        self._sync(t)
        self.sh["slots"][self.rank] = t.clone()
        self.sh["bar"].wait()
        out = D.torch().cat([self.sh["slots"][r] for r in range(self.world)], dim=0)
        self.sh["bar"].wait()
        return out


# ---------------------------------------------------------------------------
# native (CUDA) phase backend for one rank
# ---------------------------------------------------------------------------
class NativePhases:
    """Drives ots_dist_* (include/ots.h) for one rank on one device."""

    def __init__(self, device, ctx=None):
        self.dev = device
        self.ctx = ctx if ctx is not None else D.ctx(device)
        self.L = lib()
        self._t = D.torch()

    def _buf(self, count):
        t = self._t
        return t.empty((max(int(count), 1),), dtype=t.float64, device=f"cuda:{self.dev}")

    def begin(self, n_local, row0, k0, k, V, A, Q, choice="qr", P=None, orth_tol=1e-8):
        self.V, self.A, self.Q, self.P = V, A, Q, P
        self.k0, self.k, self.row0 = k0, k, row0
        rc = self.L.ots_dist_begin(self.ctx, n_local, row0, k0, k, V.ptr, V.ld, A.ptr, A.ld,
                                   Q.ptr, Q.ld, CHOICES[choice],
                                   P.ptr if P is not None else None, P.ld if P is not None else 0,
                                   orth_tol, D.stream_ptr(self.dev))
        check(rc, self.ctx)
        sz = (C.c_int64 * 4)()
        check(self.L.ots_dist_sizes(self.ctx, sz), self.ctx)
        self.n_gram, self.n_top, self.kt, self.n_y2 = (int(x) for x in sz)

    def gram(self):
        g = self._buf(self.n_gram)
        check(self.L.ots_dist_gram(self.ctx, C.c_void_p(g.data_ptr())), self.ctx)
        return g

    def top_rows(self):
        t = self._buf(self.n_top)
        check(self.L.ots_dist_top_rows(self.ctx, C.c_void_p(t.data_ptr())), self.ctx)
        return t

    def seed_early(self, top):
        check(self.L.ots_dist_seed_early(self.ctx, C.c_void_p(top.data_ptr())), self.ctx)

    def seed(self, gram_sum, top):
        check(self.L.ots_dist_seed(self.ctx, C.c_void_p(gram_sum.data_ptr()),
                                   C.c_void_p(top.data_ptr())), self.ctx)

    def factor(self):
        r = self._buf(self.kt * self.kt)
        check(self.L.ots_dist_factor(self.ctx, C.c_void_p(r.data_ptr())), self.ctx)
        return r.view(self.kt, self.kt)

    def tree(self, r_all, nranks, rank):
        check(self.L.ots_dist_tree(self.ctx, C.c_void_p(r_all.data_ptr()), nranks, rank), self.ctx)

    def qform(self):
        sign = self._buf(max(self.k, 1))
        y2 = self._buf(self.n_y2)
        check(self.L.ots_dist_qform(self.ctx, C.c_void_p(y2.data_ptr()), C.c_void_p(sign.data_ptr())),
              self.ctx)
        return y2, sign

    def finish(self, y2_sum, sign, R, S):
        diag = (C.c_double * 3)()
        rc = self.L.ots_dist_finish(self.ctx, C.c_void_p(y2_sum.data_ptr()),
                                    C.c_void_p(sign.data_ptr()), R.ptr, R.ld, S.ptr, S.ld, diag)
        check(rc, self.ctx)
        return float(diag[0]), float(diag[1])


# ---------------------------------------------------------------------------
# orchestration
# ---------------------------------------------------------------------------
def run_phases(be, comm, n_local, row0, k0, k, V, A, Q, R, S, choice="qr", P=None, orth_tol=1e-8):
    """The collective choreography of one sharded two_stage_qr.  `be` is a
    phase backend for this rank, `comm` its communicator.  Returns
    (kappa_t, wt_inv_norm); Q (local rows), R and S are written in place."""
    if row0 == 0 and n_local < k0 + k:
        raise E.DimensionError("rank 0 must own at least k0 + k rows")
    be.begin(n_local, row0, k0, k, V, A, Q, choice, P, orth_tol)
    top = be.top_rows()                  # inputs: broadcast before the Gram, so the
    top = comm.broadcast(top, src=0)     # V_t-only seed can run beside it
    if hasattr(be, "seed_early"):
        be.seed_early(top)
    g = comm.allreduce_sum(be.gram())
    be.seed(g, top)
    r_all = comm.allgather_cat(be.factor())
    be.tree(r_all, comm.world, comm.rank)
    y2, sign = be.qform()
    y2 = comm.allreduce_sum(y2)
    sign = comm.broadcast(sign, src=0)
    return be.finish(y2, sign, R, S)


def two_stage_qr_sharded(v_local, a_local, row0, choice="qr", p=None, group=None):
    """Row-sharded Algorithm 1 over a torch.distributed group (NCCL).  Each
    rank passes its CUDA row shard of V and A; returns a TwoStageResult whose
    q is this rank's shard of Q (r and s replicated)."""
    from .reflector import ReflectorDiagnostics
    from .twostage import TwoStageResult
    comm = TorchComm(group)
    dev = D.pick_device(v_local, a_local)
    n_local, k0 = v_local.shape
    k = a_local.shape[1]
    V = D.to_device(v_local, dev)
    A = D.to_device(a_local, dev)
    Q = D.empty(n_local, k, dev)
    R = D.zeros(k, k, dev)
    S = D.empty(k0, k, dev)
    P = D.to_device(p, dev) if p is not None else None
    kt, wn = run_phases(NativePhases(dev), comm, n_local, row0, k0, k, V, A, Q, R, S, choice, P)
    return TwoStageResult(Q.view(), R.view(), S.view(), ReflectorDiagnostics(kt, wn))


def bench_sharded(args, n, k0, k, rank, world, local):  # pragma: no cover - GPU box only
    """bench.py N>1 leg: rows of the headline problem split across ranks
    (strong scaling).  Device time of K steps (CUDA events, barrier +
    synchronize on both sides, max over ranks) and an end-to-end variant with
    each rank's shard copied in from pinned host memory and Q copied out."""
    import torch
    import torch.distributed as dist

    import paper_2602_14449_b200 as P
    comm = TorchComm()
    base = n // world
    n_local = base + (n - base * world if rank == world - 1 else 0)
    row0 = rank * base
    dev = torch.cuda.current_device()
    g = torch.Generator(device=f"cuda:{dev}")
    g.manual_seed(1234 + rank)
    G = torch.randn((n_local, k0), generator=g, dtype=torch.float64, device=f"cuda:{dev}")
    Qr = P.block_householder_qr([G[:, i:i + 64].contiguous() for i in range(0, k0, 64)]).q
    V = (Qr / (world ** 0.5)).contiguous()     # V^T V = sum_r Q_r^T Q_r / world = I
    A = torch.randn((n_local, k), generator=g, dtype=torch.float64, device=f"cuda:{dev}")
    del G, Qr
    be = NativePhases(dev)
    Vd, Ad = D.to_device(V, dev), D.to_device(A, dev)
    Qd, Rd, Sd = D.empty(n_local, k, dev), D.zeros(k, k, dev), D.empty(k0, k, dev)
    stream = torch.cuda.current_stream(dev)

    def step(Vx=Vd, Ax=Ad):
        run_phases(be, comm, n_local, row0, k0, k, Vx, Ax, Qd, Rd, Sd)

    def timed(fn, steps):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / steps], device=f"cuda:{dev}")
        red = comm._stage(ms)
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
        dist.barrier()
        return float(red.item())

    for _ in range(args.warmup):
        step()
    launches = int(be.L.ots_last_launch_count(be.ctx))
    clk = None
    if rank == 0:
        from bench import ClockSampler
        clk = ClockSampler(None)
        clk.start()
    ms = timed(step, args.steps)
    clocks = clk.stop() if clk is not None else None

    # e2e: this rank's V, A shard in from pinned host memory, Q shard (and R, S
    # on every rank) out, every step
    Vh, Ah = V.cpu().pin_memory(), A.cpu().pin_memory()
    Qh = torch.empty((n_local, k), dtype=torch.float64).pin_memory()
    Rh = torch.empty((k, k), dtype=torch.float64).pin_memory()
    Sh = torch.empty((k0, k), dtype=torch.float64).pin_memory()

    def e2e_step():
        Vd.buf[:, :k0].copy_(Vh, non_blocking=True)
        Ad.buf[:, :k].copy_(Ah, non_blocking=True)
        step()
        Qh.copy_(Qd.view(), non_blocking=True)
        Rh.copy_(Rd.view(), non_blocking=True)
        Sh.copy_(Sd.view(), non_blocking=True)

    e2e_steps = max(1, min(args.steps, 3))
    e2e_ms = timed(e2e_step, e2e_steps)
    h2d = n_local * (k0 + k) * 8
    d2h = (n_local * k + k * k + k0 * k) * 8
    tot = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device=f"cuda:{dev}")
    comm.allreduce_sum(tot)
    out = dict(ms=ms, e2e_ms=e2e_ms, launches=launches, clocks=clocks, h2d=int(tot[0].item()),
               d2h=int(tot[1].item()), e2e_steps=e2e_steps)
    return out
