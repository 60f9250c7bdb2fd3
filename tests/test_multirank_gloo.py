"""World-size-2 direction sharding on CPU (gloo): each rank owns a patch slice,
computes partial flux moments (D2M) over its directions, the moments are
summed by an all_reduce, and each rank applies M2D and the sweep on its own
directions. The gathered result must equal the unsharded operator. This is the
host-side logic of the multi-GPU path (one NCCL allreduce of moments per
scatter application), exercised with the oracle as the per-rank compute."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_04559_b200 import configs as cf
from paper_2010_04559_b200.sharding import patch_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    import pyoracle
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = cf.baseline_config(2, 8)
    o = pyoracle.Oracle(spec)
    n_el, P, S, _ = o.layout()
    q0, q1 = patch_range(P, rank, world)
    psi = np.random.default_rng(3).uniform(-1, 1, o.size())
    # scatter: partial moments over my directions, allreduce, M2D on my directions
    mom = torch.from_numpy(o.d2m(psi, spec.N, q0, q1))
    dist.all_reduce(mom)
    y = o.m2d(mom.numpy(), spec.N, 1.0, q0, q1, np.zeros(o.size()))
    # source iteration step: sweep my directions of (q + S psi)
    f = o.rhs() + y
    z = o.sweep(f, q0=q0, q1=q1, z=np.zeros(o.size()))
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y)
    np.save(os.path.join(out_dir, f"z{rank}.npy"), z)
    dist.barrier()
    dist.destroy_process_group()


def test_patch_range_covers_all():
    for P in (32, 128, 512, 2888, 8192):
        for W in (1, 2, 4, 8):
            rs = [patch_range(P, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == P
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            assert all((b - a) % 4 == 0 or b == P for a, b in rs)


def test_two_rank_scatter_and_sweep(tmp_path, orc):
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn")
    spec = cf.baseline_config(2, 8)
    o = orc.Oracle(spec)
    n_el, P, S, _ = o.layout()
    psi = np.random.default_rng(3).uniform(-1, 1, o.size())
    y_ref = o.apply_scatter(psi, spec.N, 1.0)
    z_ref = o.sweep(o.rhs() + y_ref)
    y = np.zeros(o.size()).reshape(n_el, P, S)
    z = np.zeros(o.size()).reshape(n_el, P, S)
    for r in range(world):
        q0, q1 = patch_range(P, r, world)
        y[:, q0:q1] = np.load(tmp_path / f"y{r}.npy").reshape(n_el, P, S)[:, q0:q1]
        z[:, q0:q1] = np.load(tmp_path / f"z{r}.npy").reshape(n_el, P, S)[:, q0:q1]
    assert np.linalg.norm(y.ravel() - y_ref) < 1e-13 * np.linalg.norm(y_ref)
    assert np.linalg.norm(z.ravel() - z_ref) < 1e-12 * np.linalg.norm(z_ref)
