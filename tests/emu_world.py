"""In-process multi-rank world for the sharded product path on ONE GPU.

W library contexts (rank r of W) are driven from W host threads. Their
collective is the library's host-collective hook (stamg_options.allreduce): the
context synchronises its stream, hands a pinned host buffer to the callback, and
copies the sum back. The callback below is a barrier plus a deterministic sum in
rank order (every rank receives the same bits, as with NCCL).

No kernel ever waits on another rank's kernel: a process-wide "GPU lock" is
held by a rank thread while it issues device work and released only inside the
collective (where its stream is already idle) and at the end of each step, so
the ranks' kernels never overlap on the device. That keeps the persistent
coarse Gauss-Seidel and the column-block sweep (which assume their CTAs are
co-resident) safe, and it is what makes a one-GPU emulation of a multi-GPU
job legitimate (B200_PROFILING.md: ranks whose kernels wait on one another must
not share a GPU).
"""
from __future__ import annotations

import threading

import numpy as np


class InProcessWorld:
    def __init__(self, world: int):
        self.world = world
        self.gpu = threading.Lock()
        self.barrier = threading.Barrier(world)
        self._slots = [None] * world
        self._total = None
        self.calls = 0
        self.doubles = 0

    def allreduce_for(self, rank: int):
        """The stamg_allreduce_fn body for `rank` (sum in place across ranks)."""

        def allreduce(buf: np.ndarray) -> None:
            self._slots[rank] = buf
            self.gpu.release()
            try:
                self.barrier.wait()
                if rank == 0:
                    total = self._slots[0].copy()
                    for r in range(1, self.world):
                        if self._slots[r].shape != total.shape:
                            raise ValueError("allreduce: ranks disagree on the element count")
                        total += self._slots[r]
                    self._total = total
                    self.calls += 1
                    self.doubles += total.size
                self.barrier.wait()
                buf[:] = self._total
                self.barrier.wait()
            finally:
                self.gpu.acquire()

        return allreduce

    def run(self, fns):
        """Run fns[r]() on W threads (rank r holds the GPU lock while it works);
        returns their results in rank order, re-raising the first failure."""
        assert len(fns) == self.world
        results = [None] * self.world
        errors = []

        def worker(r):
            with self.gpu:
                try:
                    results[r] = fns[r]()
                except BaseException as e:  # noqa: BLE001
                    errors.append((r, e))
                    self.barrier.abort()

        threads = [threading.Thread(target=worker, args=(r,)) for r in range(self.world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0][1]
        return results
