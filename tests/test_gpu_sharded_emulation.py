"""The sharded product path executed end to end on one GPU.

W contexts (rank r of W, direction sharding) run on W host threads and sum
through the library's host-collective hook (stamg_options.allreduce,
tests/emu_world.py): the moment allreduce of every scatter, the allreduced
restriction into the replicated coarsest level, the GMRES dot products and the
scalar flux all take the code paths the NCCL build takes, only the transport of
the sum differs. Each rank's result slice is gathered through stamg_patch_list
and compared with the unsharded solve (multigrid.cpp:100-136,
scatter.cpp:110-135, krylov.cpp / GMRES).
"""
import os
import sys

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from emu_world import InProcessWorld  # noqa: E402

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def gather(parts, lists, n_el, P):
    full = np.full((n_el, P, 4), np.nan)
    for a, q in zip(parts, lists):
        full[:, q] = a.reshape(n_el, len(q), 4)
    assert not np.isnan(full).any(), "the ranks' patch lists do not cover the directions"
    return full.ravel()


def sharded_contexts(stamg, spec, world, **kw):
    w = InProcessWorld(world)
    ctxs = w.run([lambda r=r: stamg.Context(spec, rank=r, world=world, allreduce=w.allreduce_for(r), **kw)
                  for r in range(world)])
    return w, ctxs


@pytest.mark.parametrize("k,n", [(2, 16), (4, 16)])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gmres_mg_matches_unsharded(stamg, k, n, world):
    spec = cf.baseline_config(k, n)
    g1 = stamg.Context(spec)
    n_el, P, _, _ = g1.layout()
    b1 = g1.rhs()
    kfix = 6
    x1k, rep1k = g1.solve(b1, "gmres", "mg", tol=1e-300, max_iter=kfix)
    x1, rep1 = g1.solve(b1, "gmres", "mg")
    ref_k, ref, sf1 = x1k.numpy(), x1.numpy(), g1.scalar_flux(x1)
    g1.close()

    w, ctxs = sharded_contexts(stamg, spec, world)
    lists = [c.patch_list() for c in ctxs]
    assert sorted(np.concatenate(lists).tolist()) == list(range(P))

    def rank_fn(r):
        c = ctxs[r]
        b = c.rhs()
        xk, repk = c.solve(b, "gmres", "mg", tol=1e-300, max_iter=kfix)
        x, rep = c.solve(b, "gmres", "mg")
        sf = c.scalar_flux(x)
        return xk.numpy(), repk, x.numpy(), rep, sf

    out = w.run([lambda r=r: rank_fn(r) for r in range(world)])
    assert w.calls > 0
    xk = gather([o[0] for o in out], lists, n_el, P)
    x = gather([o[2] for o in out], lists, n_el, P)
    assert all(o[1]["iterations"] == kfix for o in out)
    assert rel(xk, ref_k) <= 1e-12, rel(xk, ref_k)
    its = {o[3]["iterations"] for o in out}
    assert len(its) == 1, its  # every rank takes the same Krylov decisions
    assert abs(its.pop() - rep1["iterations"]) <= 1
    assert all(o[3]["converged"] for o in out)
    assert rel(x, ref) <= 1e-9
    for o in out:  # scalar flux is allreduced: identical on every rank
        assert np.array_equal(o[4], out[0][4])
    assert rel(out[0][4], sf1) <= 1e-9
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_operators_match_unsharded(stamg, world):
    """Per operator on config 4 at 16^2: apply_A (moment allreduce), mg_apply
    (level scatters + allreduced restriction + replicated coarse GS)."""
    spec = cf.baseline_config(4, 16)
    g1 = stamg.Context(spec)
    n_el, P, _, _ = g1.layout()
    x = np.random.default_rng(5).uniform(-1, 1, n_el * P * 4)
    y1 = g1.vec()
    g1.apply_A_into(g1.vec(data=x), spec.N, y1)
    z1 = g1.mg_apply(g1.vec(data=x))
    ref_A, ref_mg = y1.numpy(), z1.numpy()
    g1.close()
    w, ctxs = sharded_contexts(stamg, spec, world)
    lists = [c.patch_list() for c in ctxs]
    xs = x.reshape(n_el, P, 4)

    def rank_fn(r):
        c = ctxs[r]
        xr = c.vec(data=np.ascontiguousarray(xs[:, lists[r]]).ravel())
        y = c.vec()
        c.apply_A_into(xr, spec.N, y)
        z = c.mg_apply(xr)
        return y.numpy(), z.numpy()

    out = w.run([lambda r=r: rank_fn(r) for r in range(world)])
    assert rel(gather([o[0] for o in out], lists, n_el, P), ref_A) <= 1e-13
    assert rel(gather([o[1] for o in out], lists, n_el, P), ref_mg) <= 1e-12
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_source_iteration_matches_unsharded(stamg, world):
    """Config 5 physics at 64^2 (8192 directions): each rank owns whole reflection
    orbits, folds its scatter, and the folded moments are allreduced."""
    spec = cf.baseline_config(5, 64)
    g1 = stamg.Context(spec, build_hierarchy=False)
    n_el, P, _, _ = g1.layout()
    psi1 = g1.vec().fill(0.0)
    g1.source_iteration(psi1, 3)
    ref = psi1.numpy()
    sf1 = g1.scalar_flux(psi1)
    g1.close()
    w, ctxs = sharded_contexts(stamg, spec, world, build_hierarchy=False)
    lists = [c.patch_list() for c in ctxs]
    for r, c in enumerate(ctxs):
        np.testing.assert_array_equal(lists[r], stamg.shard_patches(spec, r, world))
        assert int(c.table("fold")[0]) == 8  # every shard folds

    def rank_fn(r):
        c = ctxs[r]
        psi = c.vec().fill(0.0)
        c.source_iteration(psi, 3)
        return psi.numpy(), c.scalar_flux(psi)

    out = w.run([lambda r=r: rank_fn(r) for r in range(world)])
    assert rel(gather([o[0] for o in out], lists, n_el, P), ref) <= 1e-12
    assert rel(out[0][1], sf1) <= 1e-12
    for c in ctxs:
        c.close()


def test_collective_failure_is_loud(stamg):
    """A failing host collective surfaces as the reference's error, not as partial sums."""
    spec = cf.baseline_config(5, 16)

    def bad(buf):
        raise RuntimeError("transport down")

    c = stamg.Context(spec, build_hierarchy=False, rank=0, world=2, allreduce=bad)
    psi = c.vec().fill(1.0)
    with pytest.raises(stamg.StamgError):
        c.source_iteration(psi, 1)
    c.close()


def test_world_needs_one_collective(stamg):
    spec = cf.baseline_config(5, 16)
    with pytest.raises(stamg.InvalidArgument):
        stamg.Context(spec, build_hierarchy=False, rank=0, world=2)
    with pytest.raises(stamg.InvalidArgument):
        stamg.Context(spec, build_hierarchy=False, rank=0, world=2, shard_probe=True, allreduce=lambda b: None)


@pytest.mark.parametrize("k,n,mg", [(4, 16, True), (5, 64, False)])
def test_chunked_moment_allreduce(stamg, monkeypatch, k, n, mg):
    """Element-range chunks of the sharded scatter (D2M chunk -> allreduce chunk -> M2D
    chunk; with NCCL the allreduce runs on its own stream and overlaps the GEMMs)
    give the unsharded operator; sharded hierarchies are orbit-partitioned, so every
    rank's outer level folds its scatter like the single GPU does."""
    spec = cf.baseline_config(k, n)
    g1 = stamg.Context(spec, build_hierarchy=mg)
    n_el, P, _, _ = g1.layout()
    x = np.random.default_rng(9).uniform(-1, 1, n_el * P * 4)
    y1 = g1.vec()
    g1.apply_A_into(g1.vec(data=x), spec.N, y1)
    ref = y1.numpy()
    fold1 = int(g1.table("fold")[0])
    g1.close()
    monkeypatch.setenv("STAMG_AR_CHUNKS", "3")
    world = 2
    w, ctxs = sharded_contexts(stamg, spec, world, build_hierarchy=mg)
    lists = [c.patch_list() for c in ctxs]
    xs = x.reshape(n_el, P, 4)
    for c in ctxs:
        assert int(c.table("fold")[0]) == fold1 > 0

    def rank_fn(r):
        c = ctxs[r]
        y = c.vec()
        c.apply_A_into(c.vec(data=np.ascontiguousarray(xs[:, lists[r]]).ravel()), spec.N, y)
        assert int(c.table("ar_chunks")[0]) == 3
        return y.numpy()

    out = w.run([lambda r=r: rank_fn(r) for r in range(world)])
    assert rel(gather(out, lists, n_el, P), ref) <= 1e-13
    for c in ctxs:
        c.close()
