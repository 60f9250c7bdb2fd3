"""Direction sharding of the MG hierarchy (host logic, CPU): the partition the
product library computes (stamg_partition, no device) covers every patch once
at every sharded level, keeps each patch's parent on the same rank, replicates
the coarsest level, and - over gloo with world size 2 - the per-rank
restrictions summed by an all_reduce reproduce the unsharded restriction into
the replicated coarsest level, bit for bit (disjoint supports)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_04559_b200 import configs as cf


def _spec(k=2, n=8):
    return cf.baseline_config(k, n)


@pytest.mark.parametrize("k,n", [(2, 8), (3, 8), (4, 8)])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_partition_covers_and_nests(stamg, orc, k, n, world):
    spec = _spec(k, n)
    o = orc.Oracle(spec)
    nlev, _ = o.levels()
    for level in range(nlev):
        P = o.layout(level)[1]
        lists = [stamg.partition(spec, r, world, level) for r in range(world)]
        if level == 0:  # replicated
            for q, _ in lists:
                assert np.array_equal(q, np.arange(P))
            continue
        allq = np.concatenate([q for q, _ in lists])
        assert np.array_equal(np.sort(allq), np.arange(P))  # disjoint cover
        fine_info = o.patch_info(level)
        for r, (q, up) in enumerate(lists):
            assert np.all(np.diff(q) > 0)
            cq, _ = stamg.partition(spec, r, world, level - 1)
            # the parent of every local patch is local on the coarser level
            assert np.all(up >= 0) and np.all(up < len(cq))
            # and is the true parent: same coarse patch as the unsharded transfer map
            assert np.array_equal(cq[up], fine_info["coarse"][q])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2010_04559_b200 import stamg as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = _spec(2, 8)
    n_el = spec.n_el
    q1, up1 = S.partition(spec, rank, world, 1)
    q0, _ = S.partition(spec, rank, world, 0)
    P1 = int(np.load(os.path.join(out_dir, "P1.npy")))
    fine = np.load(os.path.join(out_dir, "fine.npy")).reshape(n_el, P1, 4)
    local = fine[:, q1, :]                         # this rank's directions of the level-1 residual
    coarse = np.zeros((n_el, len(q0), 4))
    for k in range(len(q1)):                       # restrict_residual on the rank's patches
        coarse[:, up1[k], :] += local[:, k, :]
    t = torch.from_numpy(coarse.reshape(-1).copy())
    dist.all_reduce(t)                             # into the replicated coarsest level
    np.save(os.path.join(out_dir, f"coarse{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_restrict_into_replicated_coarsest(tmp_path, orc, stamg):
    spec = _spec(2, 8)
    o = orc.Oracle(spec)
    P1 = o.layout(1)[1]
    fine = np.random.default_rng(5).uniform(-1, 1, o.size(1))
    np.save(tmp_path / "fine.npy", fine)
    np.save(tmp_path / "P1.npy", np.array(P1))
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    ref = o.restrict(fine, 1)
    for r in range(world):
        got = np.load(tmp_path / f"coarse{r}.npy")
        # same summands per coarse entry (children of one parent are on one rank) -> tight
        assert np.abs(got - ref).max() <= 1e-15 * np.abs(ref).max()
