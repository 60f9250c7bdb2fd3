"""mg_apply replayed from a CUDA graph is bitwise the eager
V-cycle (multigrid.cpp:138-176): first call eager, then captured and replayed."""
import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,n", [(1, 16), (2, 32), (4, 16)])
def test_graph_replay_is_bitwise_eager(stamg, k, n):
    spec = cf.baseline_config(k, n)
    c = stamg.Context(spec)
    x = np.random.default_rng(3).uniform(-1, 1, c.vec().n)
    r = c.vec(data=x)
    outs = [c.mg_apply(r).numpy() for _ in range(4)]
    nG, replays, off = c.table("graphs")[:3]
    assert off == 0 and nG >= 1 and replays >= 2
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    b = c.rhs()
    xs, rep = c.solve(b, "gmres", "mg")
    assert rep["converged"]
    c.close()


def test_graphs_off_matches(stamg, monkeypatch):
    spec = cf.baseline_config(2, 32)
    c1 = stamg.Context(spec)
    b1 = c1.rhs()
    x1, r1 = c1.solve(b1, "gmres", "mg")
    monkeypatch.setenv("STAMG_GRAPHS", "0")
    c0 = stamg.Context(spec)
    x0, r0 = c0.solve(c0.rhs(), "gmres", "mg")
    assert c0.table("graphs")[1] == 0 and c1.table("graphs")[1] > 0
    assert r0["iterations"] == r1["iterations"]
    assert np.array_equal(x0.numpy(), x1.numpy())
    c0.close()
    c1.close()


@pytest.mark.parametrize("k,n", [(1, 16), (2, 32), (3, 16), (4, 16)])
def test_zero_guess_vcycle_is_the_full_sequence(stamg, monkeypatch, k, n):
    """mg_apply starts every level from zero (multigrid.cpp:138-176), so the first pre-smoothing
    step is phi = L^-1 f; STAMG_MG_ZERO_GUESS=0 computes that step's residual f - A*0 in full.
    Both are the same arithmetic on the same values (0*x and f - 0 are exact): equal iterates,
    equal GMRES iteration counts."""
    spec = cf.baseline_config(k, n)
    monkeypatch.setenv("STAMG_GRAPHS", "0")  # a captured graph would replay the mode it was captured in
    c = stamg.Context(spec)
    x = np.random.default_rng(5).uniform(-1, 1, c.vec().n)
    r = c.vec(data=x)
    fast = c.mg_apply(r).numpy()
    xs, rep_fast = c.solve(c.rhs(), "gmres", "mg")
    monkeypatch.setenv("STAMG_MG_ZERO_GUESS", "0")
    full = c.mg_apply(r).numpy()
    xf, rep_full = c.solve(c.rhs(), "gmres", "mg")
    assert np.array_equal(fast, full)  # -0.0 == +0.0
    assert rep_fast["iterations"] == rep_full["iterations"]
    assert np.array_equal(xs.numpy(), xf.numpy())
    c.close()
