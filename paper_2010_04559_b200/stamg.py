"""Python mirror of the reference operator API over the B200 C ABI.

Thin ctypes layer over ``libstamg_b200.so`` (include/stamg_b200.h). Names,
argument meaning and error behaviour follow the reference
(/root/reference/proj/include/stamg/*.hpp): ``standard_sweep``,
``apply_scatter_into``, ``apply_A_into``, ``prolongate``,
``restrict_residual``, ``lmg_vcycle``, ``mg_apply``, ``bicgstab`` and the
added ``gmres``. std::invalid_argument maps to :class:`InvalidArgument`
(a ValueError), std::logic_error to :class:`LogicError`, the Krylov NaN
runtime_error to :class:`NaNResidual`.

There is no CPU fallback: importing this module loads the CUDA library and
every call runs on the GPU; a missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from .configs import ProblemSpec

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STAMG_LIB") or os.path.join(_HERE, "libstamg_b200.so")  # override for A/B builds
OUTER = -1

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


class StamgError(RuntimeError):
    pass


class InvalidArgument(StamgError, ValueError):
    pass


class LogicError(StamgError):
    pass


class NaNResidual(StamgError):
    pass


class CudaError(StamgError):
    pass


_CODES = {1: InvalidArgument, 2: LogicError, 3: NaNResidual, 4: CudaError, 5: StamgError, 6: StamgError}


class _Problem(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("box", C.c_double),
                ("basis", C.c_int), ("p", C.c_int), ("angular_kind", C.c_int), ("angular_level", C.c_int),
                ("cone_levels", C.c_int), ("cone_half_angle_deg", C.c_double), ("N", C.c_int), ("n_mat", C.c_int),
                ("sigma_t", dp), ("moments", dp), ("mat_of_el", ip), ("q_el", dp), ("beam", C.c_int),
                ("strength", C.c_double), ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double),
                ("y1", C.c_double), ("nr", C.c_int), ("n_levels", C.c_int), ("nu_pre", C.c_int),
                ("nu_post", C.c_int), ("coarse_sweeps", C.c_int), ("coarse_tol", C.c_double)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, dp, C.c_int64)


class _Options(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.c_void_p),
                ("build_hierarchy", C.c_int), ("allreduce", ALLREDUCE_FN), ("allreduce_user", C.c_void_p),
                ("shard_probe", C.c_int)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("preconditioner_applications", C.c_int), ("final_residual", C.c_double),
                ("wall_time", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load the CUDA library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.stamg_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise _CODES.get(code, StamgError)(lib().stamg_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Vec:
    """Device-resident flux vector (FluxVector, layout.hpp:14) of one level."""

    def __init__(self, ctx: "Context", level: int = OUTER):
        self.ctx = ctx
        self.level = level
        self.h = None
        h = C.c_void_p()
        _check(lib().stamg_vec_create(ctx.h, level, C.byref(h)))
        self.h = h
        ctx._vecs.add(self)
        n = C.c_int64()
        _check(lib().stamg_vec_size(self.h, C.byref(n)))
        self.n = n.value

    def free(self):
        # a vector must not outlive its context: Context.close() frees the live ones first
        if getattr(self, "h", None) and getattr(self.ctx, "h", None):
            lib().stamg_vec_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def upload(self, a):
        a = _f64(a)
        if a.size != self.n:
            raise InvalidArgument("layout mismatch")
        _check(lib().stamg_vec_upload(self.ctx.h, self.h, a.ctypes.data_as(dp), C.c_int64(self.n)))
        return self

    def numpy(self):
        out = np.empty(self.n)
        _check(lib().stamg_vec_download(self.ctx.h, self.h, out.ctypes.data_as(dp), C.c_int64(self.n)))
        return out

    def fill(self, v):
        _check(lib().stamg_vec_fill(self.ctx.h, self.h, C.c_double(v)))
        return self

    def device_ptr(self):
        p = dp()
        _check(lib().stamg_vec_device_ptr(self.h, C.byref(p)))
        return C.cast(p, C.c_void_p).value


class Context:
    """Problem operators + sweep plan + MG hierarchy on one GPU
    (ProblemOperators / SweepPlan / MgHierarchy of the reference)."""

    def __init__(self, spec: ProblemSpec, device: int = 0, build_hierarchy: bool = True, rank: int = 0,
                 world: int = 1, nccl_id: bytes | None = None, allreduce=None, shard_probe: bool = False):
        """world > 1 takes exactly one of: ``nccl_id`` (NCCL, one GPU per rank),
        ``allreduce`` (a host collective ``f(buf: np.ndarray) -> None`` summing
        ``buf`` in place across ranks, stamg_allreduce_fn) or ``shard_probe``
        (timing only: collectives skipped, partial sums)."""
        self.spec = spec
        self.h = None
        self._vecs = weakref.WeakSet()
        st, mo = spec.kernel_arrays()
        mat = None if spec.mat_of_el is None else np.ascontiguousarray(spec.mat_of_el, dtype=np.int32)
        q = None if spec.q_el is None else _f64(spec.q_el)
        self._keep = [st, mo, mat, q]
        pr = _Problem(spec.dim, spec.nx, spec.ny, spec.nz, spec.box, spec.basis, spec.p, spec.angular_kind,
                      spec.angular_level, spec.cone_levels, spec.cone_half_angle_deg, spec.N, len(st),
                      st.ctypes.data_as(dp), mo.ctypes.data_as(dp),
                      mat.ctypes.data_as(ip) if mat is not None else None,
                      q.ctypes.data_as(dp) if q is not None else None, spec.beam, spec.strength, spec.x0, spec.x1,
                      spec.y0, spec.y1, spec.nr, spec.n_levels, spec.nu_pre, spec.nu_post, spec.coarse_sweeps,
                      spec.coarse_tol)
        self._nccl_buf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        self._allreduce_cb = None
        if allreduce is not None:
            def _cb(user, buf, n, _f=allreduce):
                try:
                    _f(np.ctypeslib.as_array(buf, shape=(n,)))
                    return 0
                except Exception:  # noqa: BLE001 - reported to the library as a failed collective
                    import traceback
                    traceback.print_exc()
                    return 1
            self._allreduce_cb = ALLREDUCE_FN(_cb)
        opt = _Options(device, rank, world, C.cast(self._nccl_buf, C.c_void_p) if self._nccl_buf else None,
                       1 if build_hierarchy else 0,
                       self._allreduce_cb if self._allreduce_cb is not None else ALLREDUCE_FN(), None,
                       1 if shard_probe else 0)
        h = C.c_void_p()
        _check(lib().stamg_create(C.byref(pr), C.byref(opt), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            for v in list(self._vecs):
                v.free()
            lib().stamg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- layout
    def layout(self, level=OUTER):
        out = (C.c_int * 4)()
        _check(lib().stamg_layout(self.h, level, out))
        return tuple(out)

    def patch_list(self, level=OUTER):
        n = C.c_int()
        _check(lib().stamg_patch_list(self.h, level, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.int32)
        _check(lib().stamg_patch_list(self.h, level, out.ctypes.data_as(ip), n.value, C.byref(n)))
        return out

    def levels(self):
        n, nr = C.c_int(), C.c_int()
        _check(lib().stamg_n_levels(self.h, C.byref(n), C.byref(nr)))
        return n.value, nr.value

    def vec(self, level=OUTER, data=None):
        v = Vec(self, level)
        if data is not None:
            v.upload(data)
        return v

    def synchronize(self):
        _check(lib().stamg_synchronize(self.h))

    def host_pipeline_chunks(self):
        n = C.c_int()
        _check(lib().stamg_host_pipeline_chunks(self.h, C.byref(n)))
        return n.value

    def launch_count(self):
        n = C.c_int64()
        _check(lib().stamg_launch_count(self.h, C.byref(n)))
        return n.value

    def timing(self, on: bool):
        _check(lib().stamg_timing_enable(self.h, 1 if on else 0))

    def timed(self, kernel: str):
        ms, n = C.c_double(), C.c_int64()
        _check(lib().stamg_timing_read(self.h, kernel.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def table(self, name, level=OUTER):
        n = C.c_int64()
        _check(lib().stamg_get_table(self.h, level, name.encode(), None, C.c_int64(0), C.byref(n)))
        out = np.empty(n.value)
        _check(lib().stamg_get_table(self.h, level, name.encode(), out.ctypes.data_as(dp), n, C.byref(n)))
        return out

    def fp64_peaks(self):
        a, b = C.c_double(), C.c_double()
        _check(lib().stamg_bench_fp64_peaks(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    # -------------------------------------------------------------- operators
    def rhs(self, out: Vec | None = None):
        out = out or Vec(self)
        _check(lib().stamg_rhs(self.h, out.h))
        return out

    def apply_L_into(self, phi: Vec, y: Vec, level=OUTER):
        _check(lib().stamg_apply_L(self.h, level, phi.h, y.h))

    def apply_scatter_into(self, phi: Vec, max_order: int, scale: float, y: Vec, level=OUTER):
        _check(lib().stamg_apply_scatter(self.h, level, phi.h, max_order, C.c_double(scale), y.h))

    def apply_A_into(self, phi: Vec, order: int, y: Vec, level=OUTER):
        _check(lib().stamg_apply_A(self.h, level, phi.h, order, y.h))

    def standard_sweep(self, rhs: Vec, z: Vec, level=OUTER):
        _check(lib().stamg_sweep(self.h, level, rhs.h, z.h))

    def coarse_scatter_sweep(self, rhs: Vec, nu: int, phi: Vec, level=0):
        _check(lib().stamg_coarse_gs(self.h, level, rhs.h, nu, phi.h))

    def smoother_step(self, f: Vec, order: int, phi: Vec, level=OUTER):
        _check(lib().stamg_smoother_step(self.h, level, f.h, order, phi.h))

    def prolongate(self, l: int, coarse: Vec, fine: Vec | None = None):
        fine = fine or Vec(self, l)
        _check(lib().stamg_prolongate(self.h, l, coarse.h, fine.h))
        return fine

    def restrict_residual(self, l: int, fine: Vec, coarse: Vec | None = None):
        coarse = coarse or Vec(self, l - 1)
        _check(lib().stamg_restrict(self.h, l, fine.h, coarse.h))
        return coarse

    def lmg_vcycle(self, l: int, f: Vec, phi: Vec):
        _check(lib().stamg_vcycle(self.h, l, f.h, phi.h))

    def mg_apply(self, r: Vec, z: Vec | None = None):
        n, _ = self.levels()
        z = z or Vec(self, n - 1)
        _check(lib().stamg_mg_apply(self.h, r.h, z.h))
        return z

    def solve(self, b: Vec, method="gmres", precond="mg", tol=None, max_iter=None, restart=None, x: Vec | None = None):
        m = {"bicgstab": 0, "gmres": 1}[method]
        pc = {"sweep": 0, "mg": 1, "none": 2}[precond]
        tol = self.spec.tol if tol is None else tol
        max_iter = self.spec.max_iter if max_iter is None else max_iter
        restart = self.spec.restart if restart is None else restart
        x = x or Vec(self)
        rep = Report()
        hist = np.zeros(max(max_iter, 1) + 1)
        _check(lib().stamg_solve(self.h, m, pc, b.h, x.h, C.c_double(tol), max_iter, restart, C.byref(rep),
                                 hist.ctypes.data_as(dp), len(hist)))
        d = rep.as_dict()
        d["converged"] = bool(d["converged"])
        d["breakdown"] = bool(d["breakdown"])
        d["residual_history"] = hist[:rep.iterations].copy()
        return x, d

    def gmres(self, b, **kw):
        return self.solve(b, method="gmres", **kw)

    def bicgstab(self, b, **kw):
        return self.solve(b, method="bicgstab", **kw)

    def source_iteration(self, psi: Vec, n_iter: int = 1):
        _check(lib().stamg_source_iteration(self.h, psi.h, n_iter))

    def scalar_flux(self, phi: Vec):
        out = np.empty(self.layout()[0])
        _check(lib().stamg_scalar_flux(self.h, phi.h, out.ctypes.data_as(dp)))
        return out

    # host-buffer entry points (the reference-side FFI boundary)
    def sweep_host(self, rhs: np.ndarray, z: np.ndarray, level=OUTER):
        _check(lib().stamg_sweep_host(self.h, level, rhs.ctypes.data_as(dp), z.ctypes.data_as(dp),
                                      C.c_int64(rhs.size)))

    def solve_host(self, b: np.ndarray, x: np.ndarray, method="gmres", precond="mg", tol=None, max_iter=None,
                   restart=None):
        rep = Report()
        m = {"bicgstab": 0, "gmres": 1}[method]
        pc = {"sweep": 0, "mg": 1, "none": 2}[precond]
        _check(lib().stamg_solve_host(self.h, m, pc, b.ctypes.data_as(dp), x.ctypes.data_as(dp), C.c_int64(b.size),
                                      C.c_double(self.spec.tol if tol is None else tol),
                                      self.spec.max_iter if max_iter is None else max_iter,
                                      self.spec.restart if restart is None else restart, C.byref(rep)))
        return rep.as_dict()


def _problem_struct(spec: ProblemSpec):
    st, mo = spec.kernel_arrays()
    mat = None if spec.mat_of_el is None else np.ascontiguousarray(spec.mat_of_el, dtype=np.int32)
    q = None if spec.q_el is None else _f64(spec.q_el)
    keep = [st, mo, mat, q]
    pr = _Problem(spec.dim, spec.nx, spec.ny, spec.nz, spec.box, spec.basis, spec.p, spec.angular_kind,
                  spec.angular_level, spec.cone_levels, spec.cone_half_angle_deg, spec.N, len(st),
                  st.ctypes.data_as(dp), mo.ctypes.data_as(dp), mat.ctypes.data_as(ip) if mat is not None else None,
                  q.ctypes.data_as(dp) if q is not None else None, spec.beam, spec.strength, spec.x0, spec.x1,
                  spec.y0, spec.y1, spec.nr, spec.n_levels, spec.nu_pre, spec.nu_post, spec.coarse_sweeps,
                  spec.coarse_tol)
    return pr, keep


def partition(spec: ProblemSpec, rank: int, world: int, level: int):
    """Host-only: (leaf positions, parent positions in the coarser local list) of
    `rank`'s directions at MG level `level` (0 = coarsest, replicated)."""
    pr, keep = _problem_struct(spec)
    n = C.c_int()
    _check(lib().stamg_partition(C.byref(pr), rank, world, level, None, None, 0, C.byref(n)))
    qpos = np.empty(n.value, dtype=np.int32)
    up = np.full(n.value, -1, dtype=np.int32)
    _check(lib().stamg_partition(C.byref(pr), rank, world, level, qpos.ctypes.data_as(ip), up.ctypes.data_as(ip),
                                 n.value, C.byref(n)))
    return qpos, up


def host_table(spec: ProblemSpec, name: str) -> np.ndarray:
    """Host-only: an outer-level table of the host setup (stamg_host_table)."""
    pr, keep = _problem_struct(spec)
    n = C.c_int64()
    _check(lib().stamg_host_table(C.byref(pr), name.encode(), None, C.c_int64(0), C.byref(n)))
    out = np.empty(n.value)
    _check(lib().stamg_host_table(C.byref(pr), name.encode(), out.ctypes.data_as(dp), n, C.byref(n)))
    return out


def shard_patches(spec: ProblemSpec, rank: int, world: int) -> np.ndarray:
    """Host-only: global leaf positions (ascending) of `rank`'s directions in a context
    without a hierarchy (whole reflection orbits; stamg_shard_patches)."""
    pr, keep = _problem_struct(spec)
    n = C.c_int()
    _check(lib().stamg_shard_patches(C.byref(pr), rank, world, None, 0, C.byref(n)))
    out = np.empty(n.value, dtype=np.int32)
    _check(lib().stamg_shard_patches(C.byref(pr), rank, world, out.ctypes.data_as(ip), n.value, C.byref(n)))
    return out


def nccl_selftest(device: int = 0, n: int = 1 << 20) -> int:
    """One-rank NCCL round trip (stamg_nccl_selftest); returns the NCCL version code."""
    v = C.c_int()
    _check(lib().stamg_nccl_selftest(device, C.c_int64(n), C.byref(v)))
    return v.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().stamg_nccl_unique_id(buf))
    return buf.raw


def host_alloc(n_doubles: int) -> np.ndarray:
    """Pinned host buffer (cudaMallocHost) viewed as a float64 array."""
    p = C.c_void_p()
    _check(lib().stamg_host_alloc(C.c_int64(n_doubles * 8), C.byref(p)))
    arr = np.ctypeslib.as_array(C.cast(p, dp), shape=(n_doubles,))
    return arr


def host_free(arr: np.ndarray) -> None:
    """Release a buffer from host_alloc (the array must not be used afterwards)."""
    _check(lib().stamg_host_free(C.c_void_p(arr.ctypes.data)))
