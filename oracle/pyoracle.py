"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/build/liborc.so`` (the CPU restatement of the
reference solver). Imported by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline arm only; the product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liborc.so")
_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


class OrcSpec(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("box", C.c_double),
                ("basis", C.c_int), ("p", C.c_int), ("angular_kind", C.c_int), ("angular_level", C.c_int),
                ("cone_levels", C.c_int), ("cone_half_angle_deg", C.c_double), ("N", C.c_int), ("n_mat", C.c_int),
                ("sigma_t", dp), ("moments", dp), ("mat_of_el", ip), ("q_el", dp), ("beam", C.c_int),
                ("strength", C.c_double), ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double),
                ("y1", C.c_double), ("nr", C.c_int), ("n_levels", C.c_int), ("nu_pre", C.c_int),
                ("nu_post", C.c_int), ("coarse_sweeps", C.c_int), ("coarse_tol", C.c_double)]


class OrcReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("preconditioner_applications", C.c_int), ("final_residual", C.c_double),
                ("wall_time", C.c_double)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
    return _lib


def _check(code):
    if code != 0:
        raise OracleError(code, lib().orc_last_error().decode())


def _p(a):
    return a.ctypes.data_as(dp) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _need(o, x, level, what):
    # the reference throws std::invalid_argument on layout mismatch (e.g. sweeps.cpp:23-24)
    if np.asarray(x).size != o.size(level):
        raise OracleError(1, f"invalid_argument: {what}: layout mismatch")


class Oracle:
    """One problem (fine operators + lazily built MG hierarchy)."""

    def __init__(self, spec):
        self.spec = spec
        st, mo = spec.kernel_arrays()
        self._keep = [st, mo]
        mat = None if spec.mat_of_el is None else np.ascontiguousarray(spec.mat_of_el, dtype=np.int32)
        q = None if spec.q_el is None else _f64(spec.q_el)
        self._keep += [mat, q]
        s = OrcSpec(spec.dim, spec.nx, spec.ny, spec.nz, spec.box, spec.basis, spec.p, spec.angular_kind,
                    spec.angular_level, spec.cone_levels, spec.cone_half_angle_deg, spec.N, len(st), _p(st), _p(mo),
                    mat.ctypes.data_as(ip) if mat is not None else None, _p(q), spec.beam, spec.strength,
                    spec.x0, spec.x1, spec.y0, spec.y1, spec.nr, spec.n_levels, spec.nu_pre, spec.nu_post,
                    spec.coarse_sweeps, spec.coarse_tol)
        h = C.c_void_p()
        _check(lib().orc_create(C.byref(s), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_destroy(self.h)
            self.h = None

    # ------------------------------------------------------------ layout
    def layout(self, level=-1):
        out = (C.c_int * 4)()
        _check(lib().orc_layout(self.h, level, out))
        return tuple(out)  # n_el, n_patch, S, D

    def size(self, level=-1):
        n_el, P, S, D = self.layout(level)
        return n_el * P * S * D

    def levels(self):
        n, nr = C.c_int(), C.c_int()
        _check(lib().orc_n_levels(self.h, C.byref(n), C.byref(nr)))
        return n.value, nr.value

    # ------------------------------------------------------------ operators
    def rhs(self):
        f = np.zeros(self.size())
        _check(lib().orc_rhs(self.h, _p(f)))
        return f

    def apply_L(self, x, level=-1):
        _need(self, x, level, "apply_L")
        x = _f64(x)
        y = np.empty_like(x)
        _check(lib().orc_apply_L(self.h, level, _p(x), _p(y)))
        return y

    def apply_A(self, x, order, level=-1):
        _need(self, x, level, "apply_A")
        x = _f64(x)
        y = np.empty_like(x)
        _check(lib().orc_apply_A(self.h, level, _p(x), order, _p(y)))
        return y

    def apply_scatter(self, x, order, scale=1.0, y=None, level=-1):
        _need(self, x, level, "apply_scatter")
        x = _f64(x)
        y = np.zeros_like(x) if y is None else _f64(y).copy()
        _check(lib().orc_apply_scatter(self.h, level, _p(x), order, C.c_double(scale), _p(y)))
        return y

    def sweep(self, rhs, level=-1, q0=0, q1=-1, z=None):
        _need(self, rhs, level, "standard_sweep")
        rhs = _f64(rhs)
        z = np.zeros_like(rhs) if z is None else z
        _check(lib().orc_sweep(self.h, level, _p(rhs), _p(z), q0, q1))
        return z

    def coarse_gs(self, rhs, nu, phi, level=0):
        _need(self, rhs, level, "coarse_scatter_sweep")
        _need(self, phi, level, "coarse_scatter_sweep")
        rhs = _f64(rhs)
        phi = _f64(phi).copy()
        _check(lib().orc_coarse_gs(self.h, level, _p(rhs), nu, _p(phi)))
        return phi

    def smoother(self, f, order, phi, level=-1):
        _need(self, f, level, "smoother_step")
        _need(self, phi, level, "smoother_step")
        f = _f64(f)
        phi = _f64(phi).copy()
        _check(lib().orc_smoother(self.h, level, _p(f), order, _p(phi)))
        return phi

    def prolong(self, coarse, l):
        _need(self, coarse, l - 1, "prolongate")
        coarse = _f64(coarse)
        fine = np.empty(self.size(l))
        _check(lib().orc_prolong(self.h, l, _p(coarse), _p(fine)))
        return fine

    def restrict(self, fine, l):
        _need(self, fine, l, "restrict_residual")
        fine = _f64(fine)
        coarse = np.empty(self.size(l - 1))
        _check(lib().orc_restrict(self.h, l, _p(fine), _p(coarse)))
        return coarse

    def vcycle(self, f, phi, l):
        f = _f64(f)
        phi = _f64(phi).copy()
        _check(lib().orc_vcycle(self.h, l, _p(f), _p(phi)))
        return phi

    def mg_apply(self, r):
        _need(self, r, -1, "mg_apply")
        r = _f64(r)
        z = np.empty_like(r)
        _check(lib().orc_mg_apply(self.h, _p(r), _p(z)))
        return z

    def d2m(self, phi, order, q0, q1, level=-1):
        phi = _f64(phi)
        n_el, _, S, _ = self.layout(level)
        mom = np.empty(n_el * (order + 1) ** 2 * S)
        _check(lib().orc_d2m(self.h, level, _p(phi), order, q0, q1, _p(mom)))
        return mom

    def m2d(self, mom, order, scale, q0, q1, y, level=-1):
        mom = _f64(mom)
        y = _f64(y).copy()
        _check(lib().orc_m2d(self.h, level, _p(mom), order, C.c_double(scale), q0, q1, _p(y)))
        return y

    def solve(self, method="gmres", precond="mg", tol=None, max_iter=None, restart=None):
        m = {"bicgstab": 0, "gmres": 1}[method]
        pc = {"sweep": 0, "mg": 1, "none": 2}[precond]
        tol = self.spec.tol if tol is None else tol
        max_iter = self.spec.max_iter if max_iter is None else max_iter
        restart = self.spec.restart if restart is None else restart
        x = np.empty(self.size())
        rep = OrcReport()
        hist = np.zeros(max(max_iter, 1) + 1)
        _check(lib().orc_solve(self.h, m, pc, C.c_double(tol), max_iter, restart, _p(x), C.byref(rep),
                               _p(hist), len(hist)))
        return x, {"iterations": rep.iterations, "converged": bool(rep.converged),
                   "breakdown": bool(rep.breakdown),
                   "preconditioner_applications": rep.preconditioner_applications,
                   "final_residual": rep.final_residual, "wall_time": rep.wall_time,
                   "residual_history": hist[:rep.iterations].copy()}

    def scalar_flux(self, phi):
        phi = _f64(phi)
        out = np.empty(self.layout()[0])
        _check(lib().orc_scalar_flux(self.h, _p(phi), _p(out)))
        return out

    # ------------------------------------------------------------ tables
    def X(self, level=-1):
        r, c = C.c_int(), C.c_int()
        _check(lib().orc_X(self.h, level, None, C.byref(r), C.byref(c)))
        out = np.empty((r.value, c.value))
        _check(lib().orc_X(self.h, level, _p(out), C.byref(r), C.byref(c)))
        return out

    def diag(self, m, q, level=-1):
        _, _, S, D = self.layout(level)
        out = np.empty((S * D, S * D))
        _check(lib().orc_diag(self.h, level, m, q, _p(out)))
        return out

    def inflow(self, q, xi, level=-1):
        _, _, S, D = self.layout(level)
        out = np.empty((S * D, S * D))
        _check(lib().orc_inflow(self.h, level, q, xi, _p(out)))
        return out

    def patch_ops(self, q, level=-1):
        out = np.empty(4)
        _check(lib().orc_patch_ops(self.h, level, q, _p(out)))
        return out

    def patch_info(self, level=-1):
        P = self.layout(level)[1]
        arrs = [np.empty(P, dtype=np.int32) for _ in range(4)]
        _check(lib().orc_patch_info(self.h, level, *[a.ctypes.data_as(ip) for a in arrs]))
        return {"octant": arrs[0], "level": arrs[1], "id": arrs[2], "coarse": arrs[3]}

    def dense_L(self):
        n = self.size()
        out = np.empty((n, n))
        _check(lib().orc_dense_L(self.h, _p(out)))
        return out

    def dense_S(self, order):
        n = self.size()
        out = np.empty((n, n))
        _check(lib().orc_dense_S(self.h, order, _p(out)))
        return out


def mesh_stats(kind, level, extra=0, angle=15.0):
    vals = [C.c_int(), C.c_int(), C.c_double(), C.c_int(), C.c_int(), C.c_int()]
    _check(lib().orc_mesh_stats(kind, level, extra, C.c_double(angle), *[C.byref(v) for v in vals]))
    return {"n_leaves": vals[0].value, "max_level": vals[1].value, "area": vals[2].value,
            "two_irregular": bool(vals[3].value), "min_nbrs": vals[4].value, "max_nbrs": vals[5].value}


def coarsen_count(kind, level, extra, angle, to_level):
    n = C.c_int()
    _check(lib().orc_mesh_coarsen_count(kind, level, extra, C.c_double(angle), to_level, C.byref(n)))
    return n.value


def refine_count(patch_id):
    n = C.c_int()
    _check(lib().orc_refine_count(patch_id, C.byref(n)))
    return n.value


def gauss(n):
    x, w = np.empty(n), np.empty(n)
    _check(lib().orc_gauss(n, _p(x), _p(w)))
    return x, w


def harmonics(N, omega):
    out = np.empty((N + 1) ** 2)
    om = _f64(omega)
    _check(lib().orc_harmonics(N, _p(om), _p(out)))
    return out


def fp_moments(N, alpha, sigma_a=0.0):
    m = np.empty(N + 1)
    st = C.c_double()
    _check(lib().orc_fp_moments(N, C.c_double(alpha), C.c_double(sigma_a), _p(m), C.byref(st)))
    return m, st.value


def nr_default(N):
    return lib().orc_nr_default(N)
