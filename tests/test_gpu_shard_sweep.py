"""Sweep of one rank's direction slice (config 5 sharded over N GPUs, rank r alone on
one GPU, no communicator: STAMG_SHARD_PROBE). With fewer 8-direction groups than SMs
the sweep splits every group's grid into two column blocks (sweep_kernel XBLK: the
upwind block publishes each strip's edge x-traces, the downwind block waits for
them); the result must be bitwise the one-block sweep and must invert apply_L."""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


@pytest.mark.parametrize("world,rank,n", [(8, 0, 128), (8, 5, 128), (8, 3, 96), (4, 1, 96)])
def test_column_blocks_bitwise(stamg, monkeypatch, world, rank, n):
    monkeypatch.setenv("STAMG_SHARD_PROBE", "1")
    spec = cf.baseline_config(5, n)
    g = stamg.Context(spec, build_hierarchy=False, rank=rank, world=world)
    monkeypatch.setenv("STAMG_SWEEP_XBLOCKS", "0")
    g1 = stamg.Context(spec, build_hierarchy=False, rank=rank, world=world)
    monkeypatch.delenv("STAMG_SWEEP_XBLOCKS")
    x = rnd(g.vec().n, 11 + rank)
    z, z1 = g.vec(), g1.vec()
    g.standard_sweep(g.vec(data=x), z)
    g1.standard_sweep(g1.vec(data=x), z1)
    a = z.numpy()
    assert np.array_equal(a, z1.numpy())
    Lz = g.vec()
    g.apply_L_into(z, Lz)  # L sweep(x) = x
    assert np.linalg.norm(Lz.numpy() - x) / np.linalg.norm(x) < 1e-12
    v = g.vec(data=x)
    g.standard_sweep(v, v)  # in place, repeated launches reuse the zeroed strip flags
    g.standard_sweep(g.vec(data=x), v)
    assert np.array_equal(v.numpy(), a)
    g.close()
    g1.close()
