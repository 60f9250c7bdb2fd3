"""Sweep of one rank's direction slice (config 5 sharded over N GPUs, rank r alone on
one GPU, no communicator: the shard_probe option). With fewer 8-direction groups than SMs
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
    spec = cf.baseline_config(5, n)
    g = stamg.Context(spec, build_hierarchy=False, rank=rank, world=world, shard_probe=True)
    monkeypatch.setenv("STAMG_SWEEP_XBLOCKS", "0")
    g1 = stamg.Context(spec, build_hierarchy=False, rank=rank, world=world, shard_probe=True)
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


def test_tail_wave_column_blocks_bitwise(stamg, monkeypatch):
    """One GPU, more 8-direction groups than CTA slots (config 5's 1024 groups on 2 x 148 slots):
    with STAMG_SWEEP_TAIL=1 the groups of the last, partly filled wave are cut into column blocks,
    the others are swept whole (sweep_kernel XBLK with xb_g0 > 0; an A/B option, not the default:
    profiles/r02_sweep_ab.txt). Bitwise the plain sweep."""
    spec = cf.baseline_config(5, 96)
    monkeypatch.setenv("STAMG_SWEEP_TAIL", "1")
    g = stamg.Context(spec, build_hierarchy=False)
    monkeypatch.delenv("STAMG_SWEEP_TAIL")
    xb, g0, ng, wl = (int(v) for v in g.table("sweep_mode"))
    assert wl > 0 and ng == 1024
    assert xb >= 2 and 0 < g0 < ng, (xb, g0, ng)
    g1 = stamg.Context(spec, build_hierarchy=False)
    assert int(g1.table("sweep_mode")[0]) == 1
    x = rnd(g.vec().n, 31)
    z, z1 = g.vec(), g1.vec()
    g.standard_sweep(g.vec(data=x), z)
    g1.standard_sweep(g1.vec(data=x), z1)
    a = z.numpy()
    assert np.array_equal(a, z1.numpy())
    v = g.vec(data=x)
    g.standard_sweep(v, v)  # in place
    assert np.array_equal(v.numpy(), a)
    g.close()
    g1.close()


@pytest.mark.parametrize("world,rank", [(2, 1), (8, 6)])
def test_sharded_folded_scatter(stamg, monkeypatch, world, rank):
    """A rank's shard is whole reflection orbits, so its scatter folds (|G| = 8); without
    a communicator its moments are the partial sums over its own directions, i.e. the
    unsharded operator applied to the vector restricted to those directions."""
    spec = cf.baseline_config(5, 64)
    g1 = stamg.Context(spec, build_hierarchy=False)
    gr = stamg.Context(spec, build_hierarchy=False, rank=rank, world=world, shard_probe=True)
    assert int(gr.table("fold")[0]) == 8
    mine = stamg.shard_patches(spec, rank, world)
    n_el, P, S, _ = g1.layout()
    x = rnd(g1.vec().n, 21).reshape(n_el, P, S)
    xr = np.zeros_like(x)
    xr[:, mine] = x[:, mine]
    y1 = g1.vec()
    g1.apply_scatter_into(g1.vec(data=xr.ravel()), spec.N, 1.0, y1)
    yr = gr.vec()
    gr.apply_scatter_into(gr.vec(data=np.ascontiguousarray(x[:, mine]).ravel()), spec.N, 1.0, yr)
    ref = y1.numpy().reshape(n_el, P, S)[:, mine].ravel()
    assert np.linalg.norm(yr.numpy() - ref) < 1e-12 * np.linalg.norm(ref)
    g1.close()
    gr.close()
