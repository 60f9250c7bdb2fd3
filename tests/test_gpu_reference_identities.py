"""The reference's own unit-test identities (/root/reference/proj/tests/*.cpp) run on the B200
reference-shape path through the C ABI: the same assertions the reference's doctest suites make
on its CPU operators, here on the GPU operators (3D hexahedra, p0 / trilinear, Const / Lin).
Each test cites the reference test it ports. Where a dense matrix is needed (Krylov vs dense LU,
the coarse-GS relaxation residual) it is the oracle's dense assembly of the same problem.

Also: the 2D discretisations the tuned kernels do not cover (p0 cells, Lin basis) against the
oracle, operator by operator.
"""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def inf(x):
    return np.abs(x).max()


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def spec_ref(orc, n, box, level, basis, p, N=4, alpha=1.0, sigma_a=0.3, dim=3, **kw):
    m, st = orc.fp_moments(N, alpha, sigma_a)
    return cf.reference_test_problem(n, box, level, basis, p, N, m, st, dim=dim, **kw)


class Ops:
    """numpy-in / numpy-out view of a GPU context (mirrors the oracle wrapper's methods)."""

    def __init__(self, stamg, spec):
        self.c = stamg.Context(spec)
        self.spec = spec

    def size(self, level=-1):
        return self.c.vec(level).n

    def apply_L(self, x):
        y = self.c.vec()
        self.c.apply_L_into(self.c.vec(data=x), y)
        return y.numpy()

    def apply_A(self, x, order, level=-1):
        y = self.c.vec(level)
        self.c.apply_A_into(self.c.vec(level, x), order, y, level=level)
        return y.numpy()

    def sweep(self, x, inplace=False):
        v = self.c.vec(data=x)
        if inplace:
            self.c.standard_sweep(v, v)
            return v.numpy()
        z = self.c.vec()
        self.c.standard_sweep(v, z)
        return z.numpy()

    def coarse_gs(self, f, nu, phi):
        v = self.c.vec(0, phi)
        self.c.coarse_scatter_sweep(self.c.vec(0, f), nu, v, level=0)
        return v.numpy()

    def smoother(self, f, order, phi, level=-1):
        v = self.c.vec(level, phi)
        self.c.smoother_step(self.c.vec(level, f), order, v, level=level)
        return v.numpy()

    def mg_apply(self, r):
        return self.c.mg_apply(self.c.vec(self.c.levels()[0] - 1, r)).numpy()

    def rhs(self):
        return self.c.rhs().numpy()

    def close(self):
        self.c.close()


@pytest.mark.parametrize("basis,p", [(0, 0), (1, 1)])
def test_sweep_inverts_L(stamg, orc, basis, p):  # test_sweeps.cpp:62-83
    g = Ops(stamg, spec_ref(orc, 3, 3.0, 1, basis, p, sigma_a=0.4))
    rhs = rnd(g.size(), 3)
    z = g.sweep(rhs)
    assert inf(g.apply_L(z) - rhs) < 1e-12 * inf(rhs)
    x = rnd(g.size(), 4)
    assert inf(g.sweep(g.apply_L(x)) - x) < 1e-10 * inf(x)
    g.close()


def test_layout_mismatch_raises(stamg, orc):  # test_sweeps.cpp:80-82, sweeps.cpp:23-24
    g = Ops(stamg, spec_ref(orc, 2, 2.0, 1, 0, 0))
    fine, coarse = g.c.vec(), g.c.vec(0)
    with pytest.raises(stamg.InvalidArgument):
        g.c.standard_sweep(fine, coarse)
    with pytest.raises(stamg.InvalidArgument):  # scatter.cpp:102-103: order above the kernel's
        g.c.apply_scatter_into(fine, 99, 1.0, g.c.vec())
    g.close()


def test_pure_absorber_single_sweep(stamg):  # test_sweeps.cpp:85-94, acceptance_main.cpp:235-249
    sp = cf.reference_test_problem(4, 4.0, 1, 1, 1, 0, [0.0], 1.0, q_el=np.ones(64))
    g = Ops(stamg, sp)
    f = g.rhs()
    phi = g.sweep(f)
    assert np.linalg.norm(f - g.apply_A(phi, 0)) < 1e-10 * np.linalg.norm(f)
    g.close()


def test_sweep_linear_deterministic_inplace(stamg, orc):  # test_sweeps.cpp:96-123
    g = Ops(stamg, spec_ref(orc, 2, 2.0, 1, 1, 1, N=2, sigma_a=0.1))
    a, b = rnd(g.size(), 11), rnd(g.size(), 12)
    lhs = g.sweep(2 * a - 0.5 * b)
    rhs = 2 * g.sweep(a) - 0.5 * g.sweep(b)
    assert inf(lhs - rhs) < 1e-12 * inf(rhs)
    z1, z2 = g.sweep(a), g.sweep(a)
    assert np.array_equal(z1, z2)
    assert np.array_equal(g.sweep(a, inplace=True), z1)
    g.close()


def test_transport_linearity_and_zero(stamg, orc):  # test_transport.cpp:30-36,109-118
    g = Ops(stamg, spec_ref(orc, 2, 1.0, 1, 1, 1, N=2))
    assert inf(g.apply_A(np.zeros(g.size()), 2)) == 0.0
    a, b = rnd(g.size(), 21), rnd(g.size(), 22)
    lhs = g.apply_A(2 * a - 0.5 * b, 2)
    rhs = 2 * g.apply_A(a, 2) - 0.5 * g.apply_A(b, 2)
    assert inf(lhs - rhs) < 1e-12 * inf(rhs)
    g.close()


@pytest.mark.parametrize("basis,p", [(0, 0), (1, 1)])
def test_coarse_sweeps_relax(stamg, orc, basis, p):  # test_sweeps.cpp:125-155, acceptance_main.cpp:340-358
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(2, 1.0 / 3, 0, basis, p, 8, m, st, q_el=np.ones(8), n_levels=0)
    o = orc.Oracle(sp)
    A = o.dense_L() - o.dense_S(8)
    g = Ops(stamg, sp)
    f = g.rhs()
    phi = np.zeros(g.size(0))
    assert inf(g.coarse_gs(f, 0, phi)) == 0.0

    def res(x):
        return np.linalg.norm(f - A @ x) / np.linalg.norm(f)

    prev = res(phi)
    assert abs(prev - 1.0) < 1e-12
    for _ in range(10):
        phi = g.coarse_gs(f, 1, phi)
        cur = res(phi)
        assert cur < prev
        prev = cur
    assert prev < 1e-3
    g.close()


def test_smoother_composition(stamg, orc):  # test_sweeps.cpp:157-181
    m, st = orc.fp_moments(4, 1.0, 0.3)
    sp = cf.reference_test_problem(3, 1.0, 1, 1, 1, 4, m, st, q_el=np.ones(27))
    g = Ops(stamg, sp)
    f = g.rhs()
    phi = rnd(g.size(), 5)
    manual = phi + g.sweep(f - g.apply_A(phi, 4))
    out = g.smoother(f, 4, phi)
    assert inf(out - manual) < 1e-13 * inf(manual)
    phi = np.zeros(g.size())
    prev = np.linalg.norm(f)
    for _ in range(4):
        phi = g.smoother(f, 4, phi)
        cur = np.linalg.norm(f - g.apply_A(phi, 4))
        assert cur < prev
        prev = cur
    g.close()


@pytest.mark.parametrize("basis", [0, 1])
def test_galerkin_adjoint(stamg, orc, basis):  # test_multigrid.cpp:78-103
    g = Ops(stamg, spec_ref(orc, 2, 1.0, 2, basis, 1))
    nlev = g.c.levels()[0]
    for l in range(1, nlev):
        xc, yf = rnd(g.size(l - 1), 30 + l), rnd(g.size(l), 40 + l)
        Pxc = g.c.prolongate(l, g.c.vec(l - 1, xc)).numpy()
        Ryf = g.c.restrict_residual(l, g.c.vec(l, yf)).numpy()
        lhs, rhs_ = float(Pxc @ yf), float(xc @ Ryf)
        assert abs(lhs - rhs_) < 1e-12 * max(abs(lhs), abs(rhs_), 1.0)
    g.close()


def test_vcycle_fixed_points(stamg, orc):  # test_multigrid.cpp:194-216
    m, st = orc.fp_moments(8, 1.0, 0.0)
    g = Ops(stamg, cf.reference_test_problem(2, 1.0 / 3, 1, 1, 1, 8, m, st))
    assert inf(g.mg_apply(np.zeros(g.size()))) == 0.0
    r = rnd(g.size(), 77)
    assert np.array_equal(g.mg_apply(r), g.mg_apply(r))
    g.close()
    flat = Ops(stamg, cf.reference_test_problem(2, 1.0 / 3, 0, 0, 0, 8, m, st))
    assert flat.c.levels()[0] == 1
    rf = rnd(flat.size(), 78)
    direct = flat.coarse_gs(rf, 10, np.zeros(flat.size()))
    assert np.array_equal(flat.mg_apply(rf), direct)
    flat.close()


def test_vcycles_reduce_residual(stamg, orc):  # test_multigrid.cpp:218-236
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(3, 0.5, 1, 0, 0, 8, m, st, q_el=np.ones(27))
    g = Ops(stamg, sp)
    f = g.rhs()
    phi = np.zeros(g.size())
    prev = np.linalg.norm(f)
    for _ in range(8):
        phi = phi + g.mg_apply(f - g.apply_A(phi, 8))
        cur = np.linalg.norm(f - g.apply_A(phi, 8))
        assert cur < prev
        prev = cur
    assert prev < 1e-3 * np.linalg.norm(f)
    g.close()


@pytest.mark.parametrize("method", ["bicgstab", "gmres"])
@pytest.mark.parametrize("precond", ["sweep", "mg"])
def test_krylov_vs_dense_lu(stamg, orc, method, precond):  # test_krylov.cpp:50-76, acceptance_main.cpp:100-113
    m, st = orc.fp_moments(4, 1.0, 0.2)
    sp = cf.reference_test_problem(2, 1.0, 1, 0, 0, 4, m, st, dim=3, q_el=np.ones(8))
    o = orc.Oracle(sp)
    A = o.dense_L() - o.dense_S(4)
    g = Ops(stamg, sp)
    b = g.rhs()
    xd = np.linalg.solve(A, b)
    x, rep = g.c.solve(g.c.vec(data=b), method, precond, tol=1e-10, max_iter=400, restart=40)
    assert rep["converged"]
    assert np.linalg.norm(x.numpy() - xd) < 1e-8 * np.linalg.norm(xd)
    assert rep["final_residual"] < 1e-10
    g.close()


def test_mg_beats_single_grid(stamg, orc):  # criterion 5 trend (acceptance_main.cpp:253-308), desk scale
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(3, 1.5, 1, 0, 1, 8, m, st, dim=3, q_el=np.ones(27))
    g = Ops(stamg, sp)
    b = g.c.rhs()
    _, sg = g.c.solve(b, "bicgstab", "sweep", max_iter=600)
    _, mg = g.c.solve(b, "bicgstab", "mg", max_iter=600)
    assert sg["converged"] and mg["converged"]
    assert mg["preconditioner_applications"] < sg["preconditioner_applications"]
    g.close()


# ---------------------------------------------------------------- 2D discretisations outside the tuned path
@pytest.mark.parametrize("basis,p", [(0, 0), (1, 0), (1, 1)])
def test_2d_reference_shape_matches_oracle(stamg, orc, basis, p):
    """2D p0 cells and the Lin basis in 2D (S = 1 / 4, D = 1 / 3) take the reference-shape path;
    every operator against the oracle on seeded inputs."""
    sp = spec_ref(orc, 6, 1.5, 2, basis, p, N=6, alpha=0.7, sigma_a=0.2, dim=2, q_el=np.ones(36), n_levels=0, nr=3)
    o = orc.Oracle(sp)
    g = Ops(stamg, sp)
    assert tuple(g.c.layout()) == tuple(o.layout())
    assert g.c.levels() == o.levels()
    x, y0 = rnd(o.size(), 1), rnd(o.size(), 2)
    assert rel(g.rhs(), o.rhs()) <= 1e-13
    assert rel(g.apply_L(x), o.apply_L(x)) <= 1e-12
    assert rel(g.apply_A(x, 6), o.apply_A(x, 6)) <= 1e-12
    assert rel(g.sweep(x), o.sweep(x)) <= 1e-12
    yv = g.c.vec(data=y0)
    g.c.apply_scatter_into(g.c.vec(data=x), 3, -0.5, yv)
    assert rel(yv.numpy(), o.apply_scatter(x, 3, -0.5, y=y0)) <= 1e-12
    xc = rnd(o.size(0), 3)
    assert rel(g.coarse_gs(xc, 2, np.zeros_like(xc)), o.coarse_gs(xc, 2, np.zeros_like(xc))) <= 1e-11
    assert rel(g.mg_apply(x), o.mg_apply(x)) <= 1e-11
    xs, rep = g.c.solve(g.c.rhs(), "gmres", "mg", tol=1e-9, max_iter=200)
    xo, repo = o.solve("gmres", "mg", tol=1e-9, max_iter=200)
    assert rep["converged"] and abs(rep["iterations"] - repo["iterations"]) <= 1
    assert rel(g.c.scalar_flux(xs), o.scalar_flux(xo)) <= 1e-7
    g.close()


@pytest.mark.parametrize("basis,p,n", [(1, 1, 5), (0, 0, 7)])
def test_dataflow_coarse_gs_is_bitwise_the_barrier_kernel(stamg, orc, monkeypatch, basis, p, n):
    """The reference-shape coarse GS runs as a dataflow kernel (one warp per line of cells,
    progress counters instead of a grid barrier per hyperplane) when the lines fit co-resident;
    STAMG_GENERIC_GS_BARRIER=1 keeps the hyperplane kernel. Same cell arithmetic, same order of
    dependent cells: bitwise equal, and repeatable."""
    m, st = orc.fp_moments(8, 1.0, 0.1)
    sp = cf.reference_test_problem(n, 1.0, 1, basis, p, 8, m, st, q_el=np.ones(n ** 3), n_levels=0, nr=4)
    g = Ops(stamg, sp)
    monkeypatch.setenv("STAMG_GENERIC_GS_BARRIER", "1")
    gb = Ops(stamg, sp)
    monkeypatch.delenv("STAMG_GENERIC_GS_BARRIER")
    f, phi0 = rnd(g.size(0), 51), rnd(g.size(0), 52)
    a = g.coarse_gs(f, 3, phi0)
    b = gb.coarse_gs(f, 3, phi0)
    assert np.array_equal(a, b)
    assert np.array_equal(g.coarse_gs(f, 3, phi0), a)
    g.close()
    gb.close()


def test_krylov_zero_rhs_and_iteration_cap(stamg, orc):  # test_krylov.cpp:29-48,100-116
    m, st = orc.fp_moments(4, 1.0, 0.2)
    g = Ops(stamg, cf.reference_test_problem(2, 1.0, 1, 1, 1, 4, m, st, dim=3))  # no source: b = 0
    for method in ("gmres", "bicgstab"):
        x, rep = g.c.solve(g.c.rhs(), method, "mg")
        assert rep["converged"] and rep["iterations"] == 0 and inf(x.numpy()) == 0.0
    g.close()
    g2 = Ops(stamg, cf.reference_test_problem(2, 1.0, 1, 1, 1, 4, m, st, dim=3, q_el=np.ones(8)))
    x, rep = g2.c.solve(g2.c.rhs(), "gmres", "sweep", tol=1e-14, max_iter=3)
    assert rep["iterations"] == 3 and not rep["converged"]
    x, rep = g2.c.solve(g2.c.rhs(), "bicgstab", "sweep", tol=1e-14, max_iter=2)
    assert rep["iterations"] == 2 and not rep["converged"]
    g2.close()


def test_scatter_orders(stamg, orc):  # scatter.cpp:101-135: order 0 keeps only the isotropic moment, order < 0 is a no-op
    sp = spec_ref(orc, 2, 1.0, 1, 1, 1, N=4)
    o = orc.Oracle(sp)
    g = Ops(stamg, sp)
    x, y0 = rnd(o.size(), 61), rnd(o.size(), 62)
    for order in (0, 2, 4):
        yv = g.c.vec(data=y0)
        g.c.apply_scatter_into(g.c.vec(data=x), order, 1.5, yv)
        assert rel(yv.numpy(), o.apply_scatter(x, order, 1.5, y=y0)) <= 1e-12
    yv = g.c.vec(data=y0)
    g.c.apply_scatter_into(g.c.vec(data=x), -1, 1.0, yv)
    assert np.array_equal(yv.numpy(), y0)
    g.close()
