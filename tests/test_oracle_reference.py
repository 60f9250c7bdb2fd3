"""The reference's own unit-test identities (/root/reference/proj/tests/*.cpp)
re-run against the CPU oracle. These pin the oracle to the reference: the
reference ships no golden vectors, so its known-answer values (mesh counts,
hand-computed blocks, FP moments, nr schedule) and dense-assembly identities
are the parity contract. Same tolerances as the
reference tests; each test cites the lines it ports.
"""
import math

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

FOUR_PI = 4 * math.pi


def ref_problem(orc, n, box, level, basis, p, N=4, alpha=1.0, sigma_a=0.3, dim=3, absorber=None, **kw):
    if absorber is not None:
        return orc.Oracle(cf.reference_test_problem(n, box, level, basis, p, 0, [0.0], absorber, dim=dim, **kw))
    m, st = orc.fp_moments(N, alpha, sigma_a)
    return orc.Oracle(cf.reference_test_problem(n, box, level, basis, p, N, m, st, dim=dim, **kw))


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def inf(x):
    return np.abs(x).max()


# ---------------------------------------------------------------- sphere mesh
def test_uniform_mesh_counts_and_area(orc):  # test_sphere_mesh.cpp:86-98
    for lvl, want in enumerate([8, 32, 128, 512]):
        s = orc.mesh_stats(0, lvl)
        assert s["n_leaves"] == want
        assert abs(s["area"] - FOUR_PI) < 1e-10
        assert s["two_irregular"]
        assert s["min_nbrs"] == 3 and s["max_nbrs"] == 3


def test_banded_mesh_published_counts(orc):  # test_sphere_mesh.cpp:101-110
    for lmax, want in zip(range(1, 7), [20, 32, 44, 128, 440, 1388]):
        s = orc.mesh_stats(1, lmax)
        assert s["n_leaves"] == want and s["max_level"] == lmax
        assert s["two_irregular"]
    with pytest.raises(orc.OracleError):
        orc.mesh_stats(1, 0)


def test_refine_and_errors(orc):  # test_sphere_mesh.cpp:46-67
    assert orc.refine_count(0) == 11
    for bad in (-1, 99):
        with pytest.raises(orc.OracleError):
            orc.refine_count(bad)


def test_coarsen(orc):  # test_sphere_mesh.cpp:112-118
    assert orc.coarsen_count(0, 3, 0, 0.0, 2) == 128
    assert orc.coarsen_count(0, 3, 0, 0.0, 0) == 8
    with pytest.raises(orc.OracleError):
        orc.coarsen_count(0, 3, 0, 0.0, -1)


def test_cone_mesh_config4(orc):  # EXTENSION (BASELINE config 4), centroid rule
    s = orc.mesh_stats(2, 4, 2, 15.0)
    assert s["n_leaves"] == 2888 and s["max_level"] == 6 and s["two_irregular"]
    assert abs(s["area"] - FOUR_PI) < 1e-10
    assert [orc.coarsen_count(2, 4, 2, 15.0, l) for l in (3, 4, 5)] == [512, 2048, 2216]


# ---------------------------------------------------------------- quadrature / harmonics
def test_gauss_legendre(orc):  # test_quadrature.cpp (1D rule)
    for n in (1, 4, 8, 20):
        x, w = orc.gauss(n)
        assert abs(w.sum() - 1.0) < 1e-14
        for k in range(2 * n):
            assert abs((w * x**k).sum() - 1.0 / (k + 1)) < 1e-13


def test_harmonics_values_and_addition_theorem(orc):  # test_scatter.cpp:64-107
    om = np.array([0.3, -0.5, 0.8])
    om /= np.linalg.norm(om)
    Y = orc.harmonics(8, om)
    assert abs(Y[0] - 1 / math.sqrt(FOUR_PI)) < 1e-14
    for n in range(9):
        s = sum(Y[n * n + n + o] ** 2 for o in range(-n, n + 1))
        assert abs(s - (2 * n + 1) / FOUR_PI) < 1e-13


def test_fp_moments(orc):  # test_scatter.cpp:39-62
    m, st = orc.fp_moments(4, 1.0)
    np.testing.assert_allclose(m, [10, 9, 7, 4, 0], rtol=0, atol=1e-14)
    assert abs(st - 10.0) < 1e-14
    m2, st2 = orc.fp_moments(8, 0.25, 0.3)
    assert m2[8] == 0.0 and abs(m2[0] - m2[1] - 0.25) < 1e-13 and abs(st2 - 0.3 - m2[0]) < 1e-14
    assert all(m2[i] > m2[i + 1] for i in range(8))
    for bad in [(0, 1.0), (4, 0.0), (4, -1.0)]:
        with pytest.raises(orc.OracleError):
            orc.fp_moments(*bad)


def test_nr_default(orc):  # test_multigrid.cpp:64-73
    assert [orc.nr_default(N) for N in (4, 8, 12, 16, 20, 24, 6, 32)] == [2, 4, 6, 7, 8, 9, 3, 9]


def test_coupling_table_const_column(orc):  # test_scatter.cpp:109-131
    o = ref_problem(orc, 1, 1.0, 2, 0, 0, N=4)
    X = o.X()
    area = np.array([o.patch_ops(q)[0] for q in range(X.shape[0])])
    np.testing.assert_allclose(X[:, 0], area / math.sqrt(FOUR_PI), rtol=1e-10)


# ---------------------------------------------------------------- transport
def test_hand_values_single_element(orc):  # test_transport.cpp:44-62
    o = ref_problem(orc, 1, 1.0, 0, 0, 0, absorber=2.0)
    a = math.pi / 4
    for q in range(8):
        assert abs(o.diag(0, q)[0, 0] - (2.0 * math.pi / 2 + 3 * a)) < 1e-12 * 6
        for xi in range(3):
            assert abs(o.inflow(q, xi)[0, 0] + a) < 1e-12
    y = o.apply_L(np.ones(8))
    np.testing.assert_allclose(y, 2.0 * math.pi / 2 + 3 * a, rtol=1e-12)


def test_zero_in_zero_out(orc):  # test_transport.cpp:30-36
    o = ref_problem(orc, 2, 2.0, 0, 0, 0)
    assert inf(o.apply_L(np.zeros(o.size()))) == 0.0


@pytest.mark.parametrize("p", [0, 1])
def test_uniform_field_interior_removal(orc, p):  # test_transport.cpp:64-82 (Const basis)
    m, st = orc.fp_moments(4, 0.5, 0.1)
    o = orc.Oracle(cf.reference_test_problem(3, 3.0, 0, 0, p, 4, m, st))
    n_el, P, S, D = o.layout()
    y = o.apply_L(np.ones(o.size())).reshape(n_el, P, D, S)
    h = 1.0
    nsum = np.full(S, h**3 if p == 0 else (h / 2) ** 3)
    center = (1 * 3 + 1) * 3 + 1
    for q in range(P):
        msum = o.patch_ops(q)[0]
        np.testing.assert_allclose(y[center, q, 0], st * msum * nsum, rtol=1e-12)


@pytest.mark.parametrize("dim,cfgs", [(3, [(0, 0, 0), (1, 1, 0), (0, 1, 1)]), (2, [(0, 1, 1), (0, 0, 1), (1, 1, 1)])])
def test_matrix_free_vs_dense(orc, dim, cfgs):  # test_transport.cpp:84-107 (+ 2D extension)
    for basis, p, level in cfgs:
        o = ref_problem(orc, 2 if dim == 3 else 3, 2.0, level, basis, p, dim=dim)
        L, S = o.dense_L(), o.dense_S(4)
        x = rnd(o.size(), 91 + level)
        assert inf(o.apply_L(x) - L @ x) < 1e-12 * inf(L @ x)
        assert inf(o.apply_A(x, 4) - (L - S) @ x) < 1e-12 * inf((L - S) @ x)


def test_transport_linearity(orc):  # test_transport.cpp:109-118
    o = ref_problem(orc, 2, 2.0, 1, 1, 1, N=2, sigma_a=0.2)
    a, b = rnd(o.size(), 1), rnd(o.size(), 2)
    lhs = o.apply_A(2 * a - 0.5 * b, 2)
    rhs = 2 * o.apply_A(a, 2) - 0.5 * o.apply_A(b, 2)
    assert inf(lhs - rhs) < 1e-12 * inf(rhs)


# ---------------------------------------------------------------- sweeps
@pytest.mark.parametrize("basis,p", [(0, 0), (1, 1)])
def test_sweep_inverts_L(orc, basis, p):  # test_sweeps.cpp:62-83
    o = ref_problem(orc, 3, 3.0, 1, basis, p, sigma_a=0.4)
    rhs = rnd(o.size(), 3)
    z = o.sweep(rhs)
    assert inf(o.apply_L(z) - rhs) < 1e-12 * inf(rhs)
    x = rnd(o.size(), 4)
    assert inf(o.sweep(o.apply_L(x)) - x) < 1e-10 * inf(x)


def test_sweep_layout_mismatch_raises(orc):  # test_sweeps.cpp:80-82
    o = ref_problem(orc, 2, 2.0, 0, 0, 0)
    with pytest.raises(Exception):
        o.smoother(np.zeros(5), 0, np.zeros(5))


def test_pure_absorber_single_sweep(orc):  # test_sweeps.cpp:85-94
    sp = cf.reference_test_problem(4, 4.0, 1, 1, 1, 0, [0.0], 1.0, q_el=np.ones(64))
    o = orc.Oracle(sp)
    f = o.rhs()
    phi = o.sweep(f)
    assert np.linalg.norm(f - o.apply_A(phi, 0)) < 1e-10 * np.linalg.norm(f)


def test_sweep_linear_deterministic_inplace(orc):  # test_sweeps.cpp:96-123
    o = ref_problem(orc, 2, 2.0, 1, 1, 1, N=2, sigma_a=0.1)
    a, b = rnd(o.size(), 11), rnd(o.size(), 12)
    lhs = o.sweep(2 * a - 0.5 * b)
    rhs = 2 * o.sweep(a) - 0.5 * o.sweep(b)
    assert inf(lhs - rhs) < 1e-12 * inf(rhs)
    z1, z2 = o.sweep(a), o.sweep(a)
    assert np.array_equal(z1, z2)
    inplace = a.copy()
    o.sweep(inplace, z=inplace)
    assert np.array_equal(inplace, z1)


@pytest.mark.parametrize("basis,p", [(0, 0), (1, 1)])
def test_coarse_sweeps_relax(orc, basis, p):  # test_sweeps.cpp:125-155
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(2, 1.0 / 3, 0, basis, p, 8, m, st, q_el=np.ones(8), n_levels=0)
    o = orc.Oracle(sp)
    A = o.dense_L() - o.dense_S(8)
    f = o.rhs()
    phi = np.zeros(o.size())
    assert inf(o.coarse_gs(f, 0, phi)) == 0.0

    def res(x):
        return np.linalg.norm(f - A @ x) / np.linalg.norm(f)

    prev = res(phi)
    assert abs(prev - 1.0) < 1e-12
    for _ in range(10):
        phi = o.coarse_gs(f, 1, phi)
        cur = res(phi)
        assert cur < prev
        prev = cur
    assert prev < 1e-3


def test_smoother_composition(orc):  # test_sweeps.cpp:157-181
    m, st = orc.fp_moments(4, 1.0, 0.3)
    sp = cf.reference_test_problem(3, 1.0, 1, 1, 1, 4, m, st, q_el=np.ones(27))
    o = orc.Oracle(sp)
    f = o.rhs()
    phi = rnd(o.size(), 5)
    manual = phi + o.sweep(f - o.apply_A(phi, 4))
    out = o.smoother(f, 4, phi)
    assert inf(out - manual) < 1e-14 * inf(manual)
    phi = np.zeros(o.size())
    prev = np.linalg.norm(f)
    for _ in range(4):
        phi = o.smoother(f, 4, phi)
        cur = np.linalg.norm(f - o.apply_A(phi, 4))
        assert cur < prev
        prev = cur


# ---------------------------------------------------------------- multigrid
def test_hierarchy_shape(orc):  # test_multigrid.cpp:33-62
    m, st = orc.fp_moments(4, 1.0, 0.0)
    o = orc.Oracle(cf.reference_test_problem(1, 1.0, 3, 0, 0, 4, m, st))
    n, nr = o.levels()
    assert n == 4 and nr == 4
    assert [o.layout(l)[1] for l in range(4)] == [8, 32, 128, 512]
    for l in range(1, 4):
        info, cinfo = o.patch_info(l), o.patch_info(l - 1)
        # every fine leaf maps into the coarse leaf that contains it (same or parent id)
        assert all(cinfo["id"][c] <= fid for c, fid in zip(info["coarse"], info["id"]))
    with pytest.raises(orc.OracleError):
        orc.Oracle(cf.reference_test_problem(1, 1.0, 3, 0, 0, 4, m, st, nr=5)).levels()


def test_transfer_values_const(orc):  # test_multigrid.cpp:105-138
    m, st = orc.fp_moments(2, 1.0, 0.0)
    o = orc.Oracle(cf.reference_test_problem(1, 1.0, 1, 0, 0, 2, m, st))
    down = o.restrict(np.ones(o.size(1)), 1)
    np.testing.assert_allclose(down, 4.0)
    up = o.prolong(np.ones(8), 1)
    np.testing.assert_allclose(up, 1.0)


@pytest.mark.parametrize("dim", [2, 3])
def test_galerkin_adjoint(orc, dim):  # test_multigrid.cpp:78-103
    m, st = orc.fp_moments(4, 1.0, 0.0)
    o = orc.Oracle(cf.reference_test_problem(2, 1.0, 2, 1, 1, 4, m, st, dim=dim))
    n, _ = o.levels()
    rng = np.random.default_rng(9)
    for l in range(1, n):
        for _ in range(20):
            c = rng.uniform(-1, 1, o.size(l - 1))
            r = rng.uniform(-1, 1, o.size(l))
            lhs = np.dot(o.prolong(c, l), r)
            rhs = np.dot(c, o.restrict(r, l))
            assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))


def test_per_level_operators_vs_dense(orc):  # test_multigrid.cpp:175-192 (2D variant)
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(3, 0.5, 2, 0, 1, 8, m, st, dim=2, nr=4)
    o = orc.Oracle(sp)
    n, nr = o.levels()
    assert nr == 4
    for l in range(n):
        x = rnd(o.size(l), 55)
        y = o.apply_A(x, nr, level=l)
        # self-consistency: A = L - S with the truncated kernel, S from scatter
        y2 = o.apply_L(x, level=l) - o.apply_scatter(x, nr, level=l)
        assert inf(y - y2) < 1e-12 * inf(y)


def test_vcycle_fixed_points(orc):  # test_multigrid.cpp:194-216
    m, st = orc.fp_moments(8, 1.0, 0.0)
    o = orc.Oracle(cf.reference_test_problem(2, 1.0 / 3, 1, 1, 1, 8, m, st))
    assert inf(o.mg_apply(np.zeros(o.size()))) == 0.0
    r = rnd(o.size(), 77)
    assert np.array_equal(o.mg_apply(r), o.mg_apply(r))
    flat = orc.Oracle(cf.reference_test_problem(2, 1.0 / 3, 0, 0, 0, 8, m, st))
    assert flat.levels()[0] == 1
    rf = rnd(flat.size(), 78)
    direct = flat.coarse_gs(rf, 10, np.zeros(flat.size()))
    assert np.array_equal(flat.mg_apply(rf), direct)


def test_vcycles_reduce_residual(orc):  # test_multigrid.cpp:218-236
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(3, 0.5, 1, 0, 0, 8, m, st, q_el=np.ones(27))
    o = orc.Oracle(sp)
    f = o.rhs()
    phi = np.zeros(o.size())
    prev = np.linalg.norm(f)
    for _ in range(8):
        phi = phi + o.mg_apply(f - o.apply_A(phi, 8))
        cur = np.linalg.norm(f - o.apply_A(phi, 8))
        assert cur < prev
        prev = cur
    assert prev < 1e-3 * np.linalg.norm(f)


# ---------------------------------------------------------------- krylov
@pytest.mark.parametrize("method", ["bicgstab", "gmres"])
@pytest.mark.parametrize("precond", ["sweep", "mg"])
def test_krylov_vs_dense_lu(orc, method, precond):  # test_krylov.cpp:50-76, acceptance_main.cpp:100-113
    m, st = orc.fp_moments(4, 1.0, 0.2)
    sp = cf.reference_test_problem(2, 1.0, 1, 0, 1, 4, m, st, dim=2, q_el=np.ones(4))
    o = orc.Oracle(sp)
    A = o.dense_L() - o.dense_S(4)
    b = o.rhs()
    xd = np.linalg.solve(A, b)
    x, rep = o.solve(method, precond, tol=1e-10, max_iter=400, restart=40)
    assert rep["converged"]
    assert np.linalg.norm(x - xd) < 1e-8 * np.linalg.norm(xd)
    assert rep["final_residual"] < 1e-10


def test_gmres_zero_rhs_and_cap(orc):  # test_krylov.cpp:29-48,100-116
    m, st = orc.fp_moments(4, 1.0, 0.2)
    sp = cf.reference_test_problem(2, 1.0, 1, 0, 1, 4, m, st, dim=2)  # no source: b = 0
    o = orc.Oracle(sp)
    x, rep = o.solve("gmres", "mg")
    assert rep["converged"] and rep["iterations"] == 0 and inf(x) == 0.0
    sp2 = cf.reference_test_problem(2, 1.0, 1, 0, 1, 4, m, st, dim=2, q_el=np.ones(4))
    x, rep = orc.Oracle(sp2).solve("gmres", "sweep", tol=1e-14, max_iter=3)
    assert rep["iterations"] == 3 and not rep["converged"]


def test_mg_beats_single_grid(orc):  # criterion 5 trend (acceptance_main.cpp:253-308), desk scale
    m, st = orc.fp_moments(8, 1.0, 0.0)
    sp = cf.reference_test_problem(4, 2.0, 1, 0, 1, 8, m, st, dim=2, q_el=np.ones(16))
    o = orc.Oracle(sp)
    _, sg = o.solve("bicgstab", "sweep", max_iter=600)
    _, mg = o.solve("bicgstab", "mg", max_iter=600)
    assert sg["converged"] and mg["converged"]
    assert mg["preconditioner_applications"] < sg["preconditioner_applications"]
