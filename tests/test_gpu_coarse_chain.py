"""Coarse Gauss-Seidel patch chain in 4-patch blocks (pre-inverted diagonal blocks of
the unit lower block-triangular chain system, sweeps.cpp:93-101) against the same kernel
walking the chain patch by patch (STAMG_GS_CHAIN_BLOCKS=0), and against the oracle.

The blocked chain changes the rounding, not the algebra: both variants must agree to
1e-12 relative after three passes from a random iterate, on 1, 4 and 64 patches per
octant (configs 3, 1/2 and 4), and the blocked result must repeat bitwise. The library
uses it by default only for 2..8 patches per octant (configs 1 and 2; it measured slower
at 64, profiles/r02_gs_c4_chain.txt), so the tests force it with STAMG_GS_CHAIN_BLOCKS=1."""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("k,n", [(1, None), (2, None), (3, 16), (4, 16), (4, 64)])
def test_blocked_chain_matches_patch_chain(stamg, monkeypatch, k, n):
    spec = cf.baseline_config(k, n)
    if k in (1, 2):  # the default choice on 4 patches per octant
        gd = stamg.Context(spec)
        assert int(gd.table("gs_mode", level=0)[5]) == 1
        gd.close()
    monkeypatch.setenv("STAMG_GS_CHAIN_BLOCKS", "1")
    g = stamg.Context(spec)
    mode = [int(v) for v in g.table("gs_mode", level=0)]
    assert mode[0] == 1 and mode[5] == 1, f"multi-warp blocked chain expected, gs_mode={mode}"
    monkeypatch.setenv("STAMG_GS_CHAIN_BLOCKS", "0")
    g0 = stamg.Context(spec)
    monkeypatch.delenv("STAMG_GS_CHAIN_BLOCKS")
    assert int(g0.table("gs_mode", level=0)[5]) == 0
    n0 = g.vec(0).n
    rng = np.random.default_rng(11)
    f = rng.uniform(-1, 1, n0)
    phi0 = rng.uniform(-1, 1, n0)
    out = []
    for ctx in (g, g0, g):
        phi = ctx.vec(0, phi0)
        ctx.coarse_scatter_sweep(ctx.vec(0, f), 3, phi, level=0)
        out.append(phi.numpy())
    assert rel(out[0], out[1]) <= 1e-12, rel(out[0], out[1])
    assert np.array_equal(out[0], out[2])
    g.close()
    g0.close()


@pytest.mark.parametrize("k,n", [(1, 16), (2, 16), (4, 8)])
def test_blocked_chain_matches_oracle(stamg, orc, monkeypatch, k, n):
    spec = cf.baseline_config(k, n)
    monkeypatch.setenv("STAMG_GS_CHAIN_BLOCKS", "1")
    g = stamg.Context(spec)
    monkeypatch.delenv("STAMG_GS_CHAIN_BLOCKS")
    o = orc.Oracle(spec)
    assert int(g.table("gs_mode", level=0)[5]) == 1
    n0 = o.size(0)
    rng = np.random.default_rng(12)
    f = rng.uniform(-1, 1, n0)
    phi0 = rng.uniform(-1, 1, n0)
    phi = g.vec(0, phi0)
    g.coarse_scatter_sweep(g.vec(0, f), 2, phi, level=0)
    ref = o.coarse_gs(f, 2, phi0.copy(), level=0)
    assert rel(phi.numpy(), ref) <= 1e-11, rel(phi.numpy(), ref)
    g.close()
