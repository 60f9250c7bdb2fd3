"""Size-independent properties at BASELINE.json sizes (where the oracle would
take too long): sweep inverts L, linearity, in-place bitwise equality, scatter
symmetry (S^T = S), Galerkin adjointness of the transfers, zero-preservation and
bitwise repeatability of the V-cycle, source-iteration consistency with the
public operators."""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module", params=[(3, None), (4, None), (5, 192)], ids=["c3", "c4", "c5grid192"])
def ctx(request, stamg):
    k, n = request.param
    spec = cf.baseline_config(k, n)
    g = stamg.Context(spec, build_hierarchy=(k != 5))
    yield spec, g
    g.close()


def test_sweep_inverts_L_full_size(ctx):
    spec, g = ctx
    n = g.vec().n
    x = rnd(n, 1)
    xv = g.vec(data=x)
    Lx = g.vec()
    g.apply_L_into(xv, Lx)
    g.standard_sweep(Lx, Lx)  # in place
    assert rel(Lx.numpy(), x) < 1e-10
    del Lx, xv


def test_sweep_linear_and_inplace(ctx):
    spec, g = ctx
    n = g.vec().n
    a, b = rnd(n, 2), rnd(n, 3)
    za, zb, zc = g.vec(), g.vec(), g.vec()
    g.standard_sweep(g.vec(data=a), za)
    g.standard_sweep(g.vec(data=b), zb)
    g.standard_sweep(g.vec(data=2.0 * a - 0.5 * b), zc)
    A, B, Cc = za.numpy(), zb.numpy(), zc.numpy()
    assert rel(Cc, 2.0 * A - 0.5 * B) < 1e-12
    v = g.vec(data=a)
    g.standard_sweep(v, v)
    assert np.array_equal(v.numpy(), A)


def test_scatter_symmetric(ctx):
    spec, g = ctx
    n = g.vec().n
    x, y = rnd(n, 4), rnd(n, 5)
    Sx, Sy = g.vec(), g.vec()
    g.apply_scatter_into(g.vec(data=x), spec.N, 1.0, Sx)
    g.apply_scatter_into(g.vec(data=y), spec.N, 1.0, Sy)
    lhs, rhs = np.dot(y, Sx.numpy()), np.dot(Sy.numpy(), x)
    assert abs(lhs - rhs) < 1e-11 * max(abs(lhs), 1e-300)


def test_transfers_adjoint_and_vcycle(ctx):
    spec, g = ctx
    if spec.name == "c5":
        pytest.skip("throughput config: no hierarchy")
    nlev, _ = g.levels()
    for l in range(1, nlev):
        c = rnd(g.vec(l - 1).n, 10 + l)
        r = rnd(g.vec(l).n, 20 + l)
        Pc = g.prolongate(l, g.vec(l - 1, c)).numpy()
        Rr = g.restrict_residual(l, g.vec(l, r)).numpy()
        lhs, rhs = np.dot(Pc, r), np.dot(c, Rr)
        assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))
    zero = g.vec(nlev - 1)
    assert np.abs(g.mg_apply(zero).numpy()).max() == 0.0
    r = g.vec(data=rnd(zero.n, 30))
    z1, z2 = g.mg_apply(r).numpy(), g.mg_apply(r).numpy()
    assert np.array_equal(z1, z2)


def test_source_iteration_consistency(ctx):
    spec, g = ctx
    n = g.vec().n
    psi0 = np.abs(rnd(n, 40))
    psi = g.vec(data=psi0)
    g.source_iteration(psi, 1)
    # the same step through the public operators: z = L^{-1}(q + S psi0)
    q = g.rhs() if spec.q_el is not None else g.vec()
    g.apply_scatter_into(g.vec(data=psi0), spec.N, 1.0, q)
    g.standard_sweep(q, q)
    assert rel(psi.numpy(), q.numpy()) < 1e-12


@pytest.mark.parametrize("chunk_dirs", [None, "296", "8"])
def test_sweep_host_pipelined_matches_device(ctx, stamg, chunk_dirs, monkeypatch):
    """stamg_sweep_host (host buffers, copies pipelined with per-chunk sweeps over
    direction groups) is bitwise the device-resident standard_sweep, in place and
    out of place, with ragged last chunks (296 = 37 groups) and one group per chunk."""
    spec, g = ctx
    if chunk_dirs is not None:
        if spec.name != "c5":
            pytest.skip("chunk sizes only matter where the pipeline runs")
        monkeypatch.setenv("STAMG_E2E_CHUNK_DIRS", chunk_dirs)
    n = g.vec().n
    x = rnd(n, 50)
    z = g.vec()
    g.standard_sweep(g.vec(data=x), z)
    ref = z.numpy()
    host = stamg.host_alloc(n)
    out = stamg.host_alloc(n)
    try:
        host[:] = x
        g.sweep_host(host, out)
        if spec.name == "c5":  # 8-direction groups with a contiguous reference range per chunk
            assert g.host_pipeline_chunks() >= 4
        assert np.array_equal(out, ref)
        assert np.array_equal(host, x)
        g.sweep_host(host, host)  # in place
        assert np.array_equal(host, ref)
    finally:
        stamg.host_free(host)
        stamg.host_free(out)
