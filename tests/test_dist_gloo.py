"""Multi-process (world_size 2, 3) gloo test of the row-sharded
orchestration dist.run_phases on CPU, with the numpy phase double.  Checks
the assembled sharded result against the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import twostage_oracle as O
from paper_2602_14449_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k0, k, choice, splits, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_14449_b200.dist import TorchComm, run_phases
    from tests.dist_double import NumpyPhases
    rng = W.make_rng(77)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    r0, r1 = splits[rank], splits[rank + 1]
    Q = np.zeros((r1 - r0, k))
    R = np.zeros((k, k))
    S = np.zeros((k0, k))
    run_phases(NumpyPhases(), TorchComm(), r1 - r0, r0, k0, k, v[r0:r1], a[r0:r1], Q, R, S, choice)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), Q=Q, R=R, S=S)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,choice", [(2, "qr"), (3, "mlu"), (2, "polar")])
def test_sharded_choreography_gloo(tmp_path, world, choice):
    n, k0, k = 600, 8, 5
    splits = [0] + [n * (r + 1) // world for r in range(world)]
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, k0, k, choice, splits, str(tmp_path)), nprocs=world,
             join=True)
    parts = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    Q = np.vstack([p["Q"] for p in parts])
    rng = W.make_rng(77)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    ref = O.two_stage(v, a, choice, diagnostics=False)
    for p in parts:  # R, S replicated
        assert np.allclose(p["R"], parts[0]["R"]) and np.allclose(p["S"], parts[0]["S"])
    err = lambda x, y: np.abs(x - y).max() / np.abs(y).max()
    assert err(Q, ref["q"]) < 1e-10
    assert err(parts[0]["R"], ref["r"]) < 1e-10
    assert err(parts[0]["S"], ref["s"]) < 1e-10
