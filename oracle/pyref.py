"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/_ref/libstamgref.so``: the reference's own solver
sources (/root/reference/proj/src, unmodified) compiled against the Eigen
shim (oracle/Makefile target ``ref``; oracle/ref_capi.cpp). Used only to pin
the oracle restatement to the reference (tests/test_oracle_vs_reference.py,
tests/golden/make_golden_ref.py). The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libstamgref.so")
REF_ROOT = "/root/reference/proj"
_lib = None
dp = C.POINTER(C.c_double)


class RefSpec(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("box", C.c_double), ("basis", C.c_int),
                ("p", C.c_int), ("angular_kind", C.c_int), ("angular_level", C.c_int), ("N", C.c_int),
                ("moments", dp), ("sigma_t", C.c_double), ("sigma_a", C.c_double), ("source_kind", C.c_int),
                ("strength", C.c_double), ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double),
                ("y1", C.c_double), ("nu_pre", C.c_int), ("nu_post", C.c_int), ("nr", C.c_int),
                ("coarse_sweeps", C.c_int), ("coarse_tol", C.c_double)]


class RefReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("preconditioner_applications", C.c_int), ("final_residual", C.c_double),
                ("wall_time", C.c_double)]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH) or os.path.isdir(os.path.join(REF_ROOT, "src"))


def build():
    subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _check(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _p(a):
    return a.ctypes.data_as(dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Reference:
    """One reference problem: ProblemOperators + SweepPlan + MgHierarchy built
    by the reference's own functions (3D hexahedra, as the reference supports)."""

    def __init__(self, n, box, level, basis, p, N, moments, sigma_t, sigma_a=0.0, banded=False, beam=None,
                 strength=1.0, nr=-1, nu_pre=1, nu_post=1, coarse_sweeps=10, coarse_tol=0.0):
        self.moments = _f64(moments)
        x0, x1, y0, y1 = beam if beam is not None else (2.0, 3.0, 2.0, 3.0)
        s = RefSpec(n, n, n, box, basis, p, 1 if banded else 0, level, N, _p(self.moments), sigma_t, sigma_a,
                    1 if beam is not None else 0, strength, x0, x1, y0, y1, nu_pre, nu_post, nr, coarse_sweeps,
                    coarse_tol)
        h = C.c_void_p()
        _check(lib().ref_create(C.byref(s), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_destroy(self.h)
            self.h = None

    def layout(self, level=-1):
        out = (C.c_int * 4)()
        _check(lib().ref_layout(self.h, level, out))
        return tuple(out)

    def size(self, level=-1):
        n_el, P, S, D = self.layout(level)
        return n_el * P * S * D

    def levels(self):
        n, nr = C.c_int(), C.c_int()
        _check(lib().ref_n_levels(self.h, C.byref(n), C.byref(nr)))
        return n.value, nr.value

    def rhs(self):
        f = np.empty(self.size())
        _check(lib().ref_rhs(self.h, _p(f)))
        return f

    def X(self, level=-1):
        r, c = C.c_int(), C.c_int()
        _check(lib().ref_X(self.h, level, None, C.byref(r), C.byref(c)))
        out = np.empty((r.value, c.value))
        _check(lib().ref_X(self.h, level, _p(out), C.byref(r), C.byref(c)))
        return out

    def diag(self, q, level=-1):
        n = C.c_int()
        _check(lib().ref_diag(self.h, level, q, None, C.byref(n)))
        out = np.empty((n.value, n.value))
        _check(lib().ref_diag(self.h, level, q, _p(out), C.byref(n)))
        return out

    def _unary(self, fn, x, level, *extra):
        x = _f64(x)
        y = np.empty(self.size(level))
        _check(fn(self.h, level, _p(x), *extra, _p(y)))
        return y

    def apply_L(self, x, level=-1):
        return self._unary(lib().ref_apply_L, x, level)

    def apply_A(self, x, order, level=-1):
        return self._unary(lib().ref_apply_A, x, level, order)

    def apply_scatter(self, x, order, scale=1.0, y=None, level=-1):
        x = _f64(x)
        y = np.zeros(self.size(level)) if y is None else _f64(y).copy()
        _check(lib().ref_apply_scatter(self.h, level, _p(x), order, C.c_double(scale), _p(y)))
        return y

    def sweep(self, rhs, level=-1):
        return self._unary(lib().ref_sweep, rhs, level)

    def coarse_gs(self, rhs, nu, phi, level=0):
        rhs = _f64(rhs)
        phi = _f64(phi).copy()
        _check(lib().ref_coarse_gs(self.h, level, _p(rhs), nu, _p(phi)))
        return phi

    def smoother(self, f, order, phi, level=-1):
        f = _f64(f)
        phi = _f64(phi).copy()
        _check(lib().ref_smoother(self.h, level, _p(f), order, _p(phi)))
        return phi

    def prolong(self, coarse, l):
        coarse = _f64(coarse)
        fine = np.empty(self.size(l))
        _check(lib().ref_prolong(self.h, l, _p(coarse), _p(fine)))
        return fine

    def restrict(self, fine, l):
        fine = _f64(fine)
        coarse = np.empty(self.size(l - 1))
        _check(lib().ref_restrict(self.h, l, _p(fine), _p(coarse)))
        return coarse

    def vcycle(self, f, phi, l):
        f = _f64(f)
        phi = _f64(phi).copy()
        _check(lib().ref_vcycle(self.h, l, _p(f), _p(phi)))
        return phi

    def mg_apply(self, r):
        r = _f64(r)
        z = np.empty_like(r)
        _check(lib().ref_mg_apply(self.h, _p(r), _p(z)))
        return z

    def bicgstab(self, precond="mg", tol=1e-8, max_iter=200):
        pc = {"sweep": 0, "mg": 1, "none": 2}[precond]
        x = np.empty(self.size())
        rep = RefReport()
        hist = np.zeros(max_iter + 1)
        _check(lib().ref_bicgstab(self.h, pc, C.c_double(tol), max_iter, _p(x), C.byref(rep), _p(hist), len(hist)))
        return x, {"iterations": rep.iterations, "converged": bool(rep.converged), "breakdown": bool(rep.breakdown),
                   "preconditioner_applications": rep.preconditioner_applications,
                   "final_residual": rep.final_residual, "residual_history": hist[:rep.iterations].copy()}
