"""GPU test of the phase-split C-ABI (ots_dist_*) driven by dist.run_phases
for G simulated ranks (threads, one ots context each) on one GPU, joined by
the in-process LocalComm.  Checks the assembled row-sharded result against
the oracle on the same inputs (rank count changes only the reduction order)."""
import threading

import numpy as np
import pytest
import torch

from oracle import twostage_oracle as O
from paper_2602_14449_b200 import _device as D
from paper_2602_14449_b200 import _native as NT
from paper_2602_14449_b200 import workloads as W
from paper_2602_14449_b200.dist import LocalComm, NativePhases, run_phases

pytestmark = pytest.mark.gpu


def _run_simulated(world, n, k0, k, choice, expect_fast=None):
    rng = W.make_rng(5 + n + world)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    ref = O.two_stage(v, a, choice, diagnostics=True)
    splits = [0] + [n * (r + 1) // world for r in range(world)]
    shared = LocalComm.make_shared(world)
    outs = [None] * world
    errs = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            r0, r1 = splits[rank], splits[rank + 1]
            V = D.to_device(v[r0:r1], 0)
            A = D.to_device(a[r0:r1], 0)
            Q = D.empty(r1 - r0, k, 0)
            R = D.zeros(k, k, 0)
            S = D.empty(k0, k, 0)
            ctx = NT.new_context(0)
            be = NativePhases(0, ctx=ctx)
            kt, wn = run_phases(be, LocalComm(rank, world, shared), r1 - r0, r0, k0, k, V, A, Q, R, S,
                                choice)
            torch.cuda.synchronize()
            outs[rank] = (Q.numpy(), R.numpy(), S.numpy(), kt, wn, NT.last_fast(ctx))
        except Exception as e:  # pragma: no cover
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    q = np.vstack([o[0] for o in outs])
    rel = lambda x, y: float((np.abs(x - y) / (np.abs(y) + 1e-4 * np.abs(y).max())).max())
    assert rel(q, ref["q"]) < 1e-10
    for o in outs:
        assert rel(o[1], ref["r"]) < 1e-10 and rel(o[2], ref["s"]) < 1e-10
        assert abs(o[3] - ref["kappa_t"]) < 1e-10 * ref["kappa_t"]
        assert abs(o[4] - ref["wt_inv_norm"]) < 1e-10 * ref["wt_inv_norm"]
        if expect_fast is not None:
            assert o[5] == expect_fast


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("n,k0,k,choice", [(20000, 32, 16, "qr"), (50000, 128, 64, "qr"),
                                           (30000, 64, 32, "polar"), (30000, 64, 32, "mlu")])
def test_simulated_ranks(world, n, k0, k, choice):
    _run_simulated(world, n, k0, k, choice)


@pytest.mark.parametrize("world,n", [(2, 1 << 21), (3, 1600000)])
def test_simulated_ranks_direct_q(world, n):
    """Shards of >= 2^19 rows: every rank's local factor takes the direct-Q
    route (tile Grams of its own [V | A] rows); the exchanged blocks -- Gram
    sum, rank R's, C's, Y2 sum, signs -- are the same as on the materialised
    route, so ranks may also mix routes."""
    _run_simulated(world, n, 128, 64, "qr", expect_fast=1)
