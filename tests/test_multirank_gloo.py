"""World-size-2 direction sharding on CPU (gloo): each rank owns a patch slice,
computes partial flux moments (D2M) over its directions, the moments are
summed by an all_reduce, and each rank applies M2D and the sweep on its own
directions. The gathered result must equal the unsharded operator. This is the
host-side logic of the multi-GPU path (one NCCL allreduce of moments per
scatter application), exercised with the oracle as the per-rank compute, on the
shards the runtime assigns (whole reflection orbits, stamg_shard_patches:
host-only, no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_04559_b200 import configs as cf
from paper_2010_04559_b200.sharding import patch_range, runs


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
    from paper_2010_04559_b200 import stamg
    mine = runs(stamg.shard_patches(spec, rank, world))
    psi = np.random.default_rng(3).uniform(-1, 1, o.size())
    # scatter: partial moments over my directions, allreduce, M2D on my directions
    mom = torch.from_numpy(sum(o.d2m(psi, spec.N, q0, q1) for q0, q1 in mine))
    dist.all_reduce(mom)
    y = np.zeros(o.size())
    for q0, q1 in mine:
        y = o.m2d(mom.numpy(), spec.N, 1.0, q0, q1, y)
    # source iteration step: sweep my directions of (q + S psi)
    f = o.rhs() + y
    z = np.zeros(o.size())
    for q0, q1 in mine:
        z = o.sweep(f, q0=q0, q1=q1, z=z)
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


@pytest.mark.parametrize("k,n,G", [(5, None, 8), (2, 8, 8), (4, 8, 4)])
def test_shards_are_whole_orbits(k, n, G):
    """stamg_shard_patches: disjoint cover, balanced, and a union of reflection orbits
    (equal counts in every mirrored octant) so each rank can fold its own scatter."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from paper_2010_04559_b200 import stamg
    spec = cf.baseline_config(k, n)
    import pyoracle
    octant = pyoracle.Oracle(spec).patch_info()["octant"].astype(int)
    for W in (1, 2, 4, 8):
        sets = [stamg.shard_patches(spec, r, W) for r in range(W)]
        allp = np.sort(np.concatenate(sets))
        assert np.array_equal(allp, np.arange(allp.size))
        sizes = [len(x) for x in sets]
        assert max(sizes) - min(sizes) <= 8 * G
        assert all(sz % G == 0 for sz in sizes)
        for x in sets:  # whole orbits: equal counts in octants related by the symmetric reflections
            counts = np.bincount(octant[x], minlength=8)
            if G == 8:
                assert len(set(counts)) == 1
            else:  # config 4's +x cone mesh: y and z reflections (octant bits 1, 2)
                for o in range(8):
                    assert counts[o] == counts[o ^ 2] == counts[o ^ 4]


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
    from paper_2010_04559_b200 import stamg
    for r in range(world):
        mine = stamg.shard_patches(spec, r, world)
        y[:, mine] = np.load(tmp_path / f"y{r}.npy").reshape(n_el, P, S)[:, mine]
        z[:, mine] = np.load(tmp_path / f"z{r}.npy").reshape(n_el, P, S)[:, mine]
    assert np.linalg.norm(y.ravel() - y_ref) < 1e-13 * np.linalg.norm(y_ref)
    assert np.linalg.norm(z.ravel() - z_ref) < 1e-12 * np.linalg.norm(z_ref)
