"""CPU check of the in-process collective the one-GPU sharded tests use
(tests/emu_world.py): deterministic rank-order sums, identical bits on every
rank, the GPU lock held outside the collective, failures propagated."""
import os
import sys
import threading

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from emu_world import InProcessWorld  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4])
def test_allreduce_sums_in_rank_order(world):
    w = InProcessWorld(world)
    data = [np.random.default_rng(r).uniform(-1, 1, 1000) for r in range(world)]
    held = []

    def fn(r):
        held.append(w.gpu.locked())
        out = []
        for rep in range(3):
            buf = data[r].copy() * (rep + 1)
            w.allreduce_for(r)(buf)
            held.append(w.gpu.locked())
            out.append(buf)
        return out

    res = w.run([lambda r=r: fn(r) for r in range(world)])
    for rep in range(3):
        ref = data[0] * (rep + 1)
        for r in range(1, world):
            ref = ref + data[r] * (rep + 1)
        for r in range(world):
            assert np.array_equal(res[r][rep], ref)
    assert all(held) and w.calls == 3


def test_gpu_lock_serialises_ranks():
    w = InProcessWorld(3)
    active, peak = [0], [0]
    mu = threading.Lock()

    def fn(r):
        for _ in range(4):
            with mu:
                active[0] += 1
                peak[0] = max(peak[0], active[0])
            with mu:
                active[0] -= 1
            w.allreduce_for(r)(np.ones(4))
        return r

    assert w.run([lambda r=r: fn(r) for r in range(3)]) == [0, 1, 2]
    assert peak[0] == 1


def test_failure_propagates():
    w = InProcessWorld(2)

    def ok(r):
        w.allreduce_for(r)(np.ones(3))

    def bad():
        raise RuntimeError("rank 1 failed")

    with pytest.raises(RuntimeError):
        w.run([lambda: ok(0), bad])
