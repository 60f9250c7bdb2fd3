"""The Krylov workspace must not leak stale device memory into a solve.

Throughput contexts store vectors in the wavefront layout, which has padding slots the
operators never write; dot products, axpys and Givens updates run over the full padded
length. The library zeroes V[k], z and u when it allocates them (ensure_krylov). Here device
memory is poisoned with NaN first (vectors filled with NaN and freed, so the allocator hands
the same blocks to the workspace), then GMRES and BiCGSTAB are run in the wavefront layout:
the results must be finite and equal the solve of a fresh, unpoisoned context bitwise
(krylov.cpp:9-93; GMRES is the BASELINE extension)."""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method,restart", [("gmres", 5), ("bicgstab", 0)])
def test_poisoned_memory_does_not_reach_the_solve(stamg, method, restart):
    spec = cf.baseline_config(5, 40)
    spec.angular_level = 3
    spec.N = 11
    spec.moments = np.asarray(spec.moments)[:, :12]
    clean = stamg.Context(spec, build_hierarchy=False)
    assert int(clean.table("sweep_mode")[3]) > 0, "wavefront layout expected"
    kw = dict(tol=1e-300, max_iter=4)
    if method == "gmres":
        kw["restart"] = restart
    xc, repc = clean.solve(clean.rhs(), method, "sweep", **kw)
    ref = xc.numpy()
    clean.close()

    g = stamg.Context(spec, build_hierarchy=False)
    poison = [g.vec().fill(float("nan")) for _ in range(10)]
    g.synchronize()
    for v in poison:
        v.free()
    xs, rep = g.solve(g.rhs(), method, "sweep", **kw)
    out = xs.numpy()
    assert np.all(np.isfinite(out))
    assert np.isfinite(rep["final_residual"])
    assert rep["iterations"] == repc["iterations"]
    assert np.array_equal(out, ref)
    g.close()
