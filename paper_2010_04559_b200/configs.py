"""Problem descriptions for the five BASELINE.json configurations and the
small reference-style test problems.

A :class:`ProblemSpec` is plain data (geometry, angular mesh recipe, per
material cross sections and Legendre moments, material map, source). The
product library (``libstamg_b200.so``) and the CPU oracle both build their
operator tables from the same spec, so parity tests compare like with like.

Conventions (SURVEY.md §8 / DESIGN.md):
* 2D square of side 1 cm for every config, bilinear cells (S=4), Const angular
  basis (D=1), vacuum boundaries.
* HG scattering: sigma_{s,n} = c * sigma_t * g**n, sigma_a = (1-c) sigma_t.
* config 3 material map: 8x8-cell blocks, exactly round(0.7 * n_blocks)
  blocks of material A chosen by ``numpy.random.default_rng(seed).permutation``.
* config 4 cone membership: patch centroid within 15 deg of +x.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

ANGULAR_UNIFORM, ANGULAR_BANDED, ANGULAR_CONE = 0, 1, 2
BEAM_NONE, BEAM_PENCIL_Z, BEAM_CONE_X0 = 0, 1, 2


@dataclasses.dataclass
class ProblemSpec:
    name: str = "problem"
    dim: int = 2
    nx: int = 4
    ny: int = 4
    nz: int = 1
    box: float = 1.0
    basis: int = 0          # 0 Const (D=1), 1 Lin (D=3)
    p: int = 1              # spatial order: 0 (S=1) or 1 (bilinear/trilinear)
    angular_kind: int = ANGULAR_UNIFORM
    angular_level: int = 1
    cone_levels: int = 0
    cone_half_angle_deg: float = 15.0
    N: int = 4
    sigma_t: np.ndarray = dataclasses.field(default_factory=lambda: np.array([1.0]))
    moments: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((1, 5)))
    mat_of_el: Optional[np.ndarray] = None
    q_el: Optional[np.ndarray] = None
    beam: int = BEAM_NONE
    strength: float = 1.0
    x0: float = 2.0
    x1: float = 3.0
    y0: float = 2.0
    y1: float = 3.0
    # multigrid cycle (multigrid.hpp:17-24) + EXTENSION n_levels
    nr: int = -1
    n_levels: int = 0
    nu_pre: int = 1
    nu_post: int = 1
    coarse_sweeps: int = 10
    coarse_tol: float = 0.0
    # Krylov
    tol: float = 1e-8
    max_iter: int = 1000
    restart: int = 40

    @property
    def n_el(self) -> int:
        return self.nx * self.ny * (self.nz if self.dim == 3 else 1)

    def kernel_arrays(self):
        st = np.ascontiguousarray(np.asarray(self.sigma_t, dtype=np.float64).reshape(-1))
        mo = np.ascontiguousarray(np.asarray(self.moments, dtype=np.float64).reshape(len(st), self.N + 1))
        return st, mo


def hg_moments(N: int, sigma_t: float, c: float, g: float) -> np.ndarray:
    """Henyey-Greenstein Legendre moments sigma_{s,n} = c sigma_t g^n."""
    return c * sigma_t * np.power(float(g), np.arange(N + 1, dtype=np.float64))


def fp_moments(N: int, alpha: float) -> np.ndarray:
    """Fokker-Planck-equivalent moments (scatter.cpp:9-21)."""
    n = np.arange(N + 1, dtype=np.float64)
    return 0.5 * alpha * (N * (N + 1.0) - n * (n + 1.0))


def _block_source(nx: int, ny: int, x0: int, x1: int, y0: int, y1: int) -> np.ndarray:
    q = np.zeros((ny, nx))
    q[y0:y1, x0:x1] = 1.0
    return q.reshape(-1)


def config3_material_map(n: int = 128, block: int = 8, frac_a: float = 0.7, seed: int = 20101) -> np.ndarray:
    nb = n // block
    n_blocks = nb * nb
    n_a = int(round(frac_a * n_blocks))
    perm = np.random.default_rng(seed).permutation(n_blocks)
    blk_mat = np.ones(n_blocks, dtype=np.int32)     # 1 = material B
    blk_mat[perm[:n_a]] = 0                        # 0 = material A
    blk = blk_mat.reshape(nb, nb)
    return np.ascontiguousarray(np.kron(blk, np.ones((block, block), dtype=np.int32)).reshape(-1).astype(np.int32))


def baseline_config(k: int, n: Optional[int] = None) -> ProblemSpec:
    """BASELINE.json configs[k-1]; ``n`` overrides the cell count per axis
    (same physics, smaller grid) for oracle-sized parity tests."""
    if k == 1:
        nn = n or 32
        N = 8
        return ProblemSpec(name="c1", nx=nn, ny=nn, angular_level=2, N=N,
                           sigma_t=np.array([10.0]), moments=hg_moments(N, 10.0, 0.99, 0.9)[None],
                           q_el=np.ones(nn * nn), nr=-1, n_levels=2)
    if k == 2:
        nn = n or 64
        N = 16
        c0 = nn // 2 - 4
        return ProblemSpec(name="c2", nx=nn, ny=nn, angular_level=3, N=N,
                           sigma_t=np.array([50.0]), moments=hg_moments(N, 50.0, 0.999, 0.95)[None],
                           q_el=_block_source(nn, nn, c0, c0 + 8, c0, c0 + 8), nr=4, n_levels=3)
    if k == 3:
        nn = n or 128
        N = 24
        mat = config3_material_map(nn, 8)
        mom = np.stack([hg_moments(N, 100.0, 0.999, 0.97), hg_moments(N, 0.1, 0.5, 0.5)])
        return ProblemSpec(name="c3", nx=nn, ny=nn, angular_level=3, N=N,
                           sigma_t=np.array([100.0, 0.1]), moments=mom, mat_of_el=mat,
                           q_el=(mat == 0).astype(np.float64), nr=6, n_levels=0)
    if k == 4:
        nn = n or 256
        N = 32
        return ProblemSpec(name="c4", nx=nn, ny=nn, angular_kind=ANGULAR_CONE, angular_level=4,
                           cone_levels=2, cone_half_angle_deg=15.0, N=N,
                           sigma_t=np.array([200.0]), moments=hg_moments(N, 200.0, 0.9999, 0.99)[None],
                           beam=BEAM_CONE_X0, nr=8, n_levels=4, restart=12)
    if k == 5:
        nn = n or 512
        N = 32
        return ProblemSpec(name="c5", nx=nn, ny=nn, angular_level=5, N=N,
                           sigma_t=np.array([100.0]), moments=hg_moments(N, 100.0, 0.999, 0.95)[None],
                           q_el=np.ones(nn * nn), nr=-1, n_levels=1)
    raise ValueError(f"no config {k}")


def reference_test_problem(n: int, box: float, level: int, basis: int, p: int, N: int,
                           moments: np.ndarray, sigma_t: float, dim: int = 3, **kw) -> ProblemSpec:
    """The reference unit tests' ``make_ops`` (test_sweeps.cpp:16-19): an
    n^3 (or n^2) cube, uniform angular level, one material."""
    return ProblemSpec(name="ref", dim=dim, nx=n, ny=n, nz=n if dim == 3 else 1, box=box, basis=basis,
                       p=p, angular_level=level, N=N, sigma_t=np.array([sigma_t]),
                       moments=np.asarray(moments, dtype=np.float64)[None], **kw)
