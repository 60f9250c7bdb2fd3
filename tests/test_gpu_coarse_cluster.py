"""Coarse Gauss-Seidel with the row-CTAs grouped in thread-block clusters (y-traces
through DSMEM mailboxes, sweeps.cpp:51-104 order unchanged) against the same kernel
with every y-hop through global memory (STAMG_GS_CLUSTER=0): bitwise equal, at the
full BASELINE grids of configs 1-3 and at the oracle-sized grids the parity tests use."""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,n", [(1, None), (2, None), (3, None), (4, None), (2, 16), (3, 16), (4, 16)])
def test_cluster_coarse_gs_bitwise(stamg, monkeypatch, k, n):
    """Config 4's coarsest level (64 patches per octant) only fits a 4-slot mailbox ring
    with credits (the downwind row hands slots back; opt-in, STAMG_GS_MAILBOX_RING);
    configs 1-3 hold two octants of a row (no credits)."""
    spec = cf.baseline_config(k, n)
    if k == 4:
        monkeypatch.setenv("STAMG_GS_MAILBOX_RING", "1")
    g = stamg.Context(spec)
    monkeypatch.delenv("STAMG_GS_MAILBOX_RING", raising=False)
    mw, cluster, _, slots, credit = (int(v) for v in g.table("gs_mode", level=0)[:5])
    assert mw == 1 and cluster > 1, "cluster mode expected on this grid"
    assert slots >= 4 and credit == (1 if k == 4 else 0)
    monkeypatch.setenv("STAMG_GS_CLUSTER", "0")
    g0 = stamg.Context(spec)
    assert int(g0.table("gs_mode", level=0)[1]) == 0
    monkeypatch.delenv("STAMG_GS_CLUSTER")
    n0 = g.vec(0).n
    rng = np.random.default_rng(7)
    f = rng.uniform(-1, 1, n0)
    phi0 = rng.uniform(-1, 1, n0)
    out = []
    for ctx in (g, g0):
        phi = ctx.vec(0, phi0)
        ctx.coarse_scatter_sweep(ctx.vec(0, f), 3, phi, level=0)
        out.append(phi.numpy())
    assert np.array_equal(out[0], out[1])
    # and repeatable run to run
    phi = g.vec(0, phi0)
    g.coarse_scatter_sweep(g.vec(0, f), 3, phi, level=0)
    assert np.array_equal(phi.numpy(), out[0])
    g.close()
    g0.close()
