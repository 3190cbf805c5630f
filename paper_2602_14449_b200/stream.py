"""Host-buffer streaming front end: `two_stage_qr` over a sequence of host
(pinned) input pairs with the PCIe transfers of neighbouring calls overlapped.

A call on host data moves V and A to HBM (n(k0+k) doubles) and Q back (nk
doubles); at the headline shape these transfers take ~5x longer than the
computation.  `two_stage_qr_stream` keeps two device slots: while call s
computes, the inputs of call s+1 stream in on a copy stream and the outputs of
call s-1 stream out on another (PCIe is full duplex), so a sequence of calls
runs at the H2D rate instead of H2D + compute + D2H.  Every call still copies
its own inputs and reads back its own Q, R, S.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _device as D
from .twostage import two_stage_qr


@dataclass
class HostResult:
    """q, r, s in pinned host memory; valid after `wait()`."""
    q: object
    r: object
    s: object
    diagnostics: object
    event: object

    def wait(self):
        self.event.synchronize()
        return self


def two_stage_qr_stream(pairs, choice="qr", intra="householder", device=None, workspace=None):
    """Yield `HostResult`s for `two_stage_qr(v, a)` over `pairs` (an iterable
    of (v, a) host torch tensors, ideally pinned).  Output buffers rotate over
    two pinned sets: a result must be consumed (`wait()`, then read) before the
    generator is advanced twice more.  `workspace` (a dict) keeps the device
    slots and pinned outputs across generators, so repeated streams do not
    re-allocate (pinning GBs of host memory is slow)."""
    torch = D.torch()
    dev = device if device is not None else torch.cuda.current_device()
    comp = torch.cuda.current_stream(dev)
    ws = workspace if workspace is not None else {}
    h2d = ws.setdefault("h2d", torch.cuda.Stream(dev))
    d2h = ws.setdefault("d2h", torch.cuda.Stream(dev))
    slots = ws.setdefault("slots", [None, None])       # device (V, A) per slot
    outs = ws.setdefault("outs", [None, None])         # pinned (Q, R, S) per slot
    loaded = [None, None]      # H2D completion event per slot

    def issue_h2d(slot, v, a):
        if slots[slot] is None or slots[slot][0].shape != v.shape or slots[slot][1].shape != a.shape:
            slots[slot] = (torch.empty(v.shape, dtype=v.dtype, device=f"cuda:{dev}"),
                           torch.empty(a.shape, dtype=a.dtype, device=f"cuda:{dev}"))
        Vd, Ad = slots[slot]
        h2d.wait_stream(comp)          # the slot's previous call has finished reading it
        with torch.cuda.stream(h2d):
            Vd.copy_(v, non_blocking=True)
            Ad.copy_(a, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        loaded[slot] = ev

    it = iter(pairs)
    cur = next(it, None)
    if cur is None:
        return
    slot = 0
    issue_h2d(slot, *cur)
    while cur is not None:
        nxt = next(it, None)
        if nxt is not None:
            issue_h2d(slot ^ 1, *nxt)
        comp.wait_event(loaded[slot])
        Vd, Ad = slots[slot]
        res = two_stage_qr(Vd, Ad, choice=choice, intra=intra)
        v, a = cur
        n, k0, k = v.shape[0], v.shape[1], a.shape[1]
        if outs[slot] is None or outs[slot][0].shape != (n, k):
            outs[slot] = (torch.empty((n, k), dtype=res.q.dtype).pin_memory(),
                          torch.empty((k, k), dtype=res.r.dtype).pin_memory(),
                          torch.empty((k0, k), dtype=res.s.dtype).pin_memory())
        Qh, Rh, Sh = outs[slot]
        d2h.wait_stream(comp)
        with torch.cuda.stream(d2h):
            for t_ in (res.q, res.r, res.s):
                t_.record_stream(d2h)
            Qh.copy_(res.q, non_blocking=True)
            Rh.copy_(res.r, non_blocking=True)
            Sh.copy_(res.s, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(d2h)
        yield HostResult(Qh, Rh, Sh, res.diagnostics, ev)
        cur = nxt
        slot ^= 1
