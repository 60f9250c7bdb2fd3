"""Per-rank sweep time of config 5 when its 8192 directions are sharded over N
GPUs, measured on one GPU: rank 0's slice (P/N directions, the contiguous leaf
range the library gives it) swept alone, without a communicator
(stamg_options.shard_probe). The sweep has no collective, so a rank's device time is
the N-GPU job's time; speed-up = t(1) / t(N).

    python tools/shard_probe.py [N ...]      (default 1 2 4 8)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2010_04559_b200 import configs as cf  # noqa: E402
from paper_2010_04559_b200 import stamg  # noqa: E402


def main():
    ns = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
    spec = cf.baseline_config(5, int(os.environ.get("C5N", "512")))
    out, t1 = {}, None
    for n in ns:
        g = stamg.Context(spec, build_hierarchy=False, rank=0, world=n, shard_probe=n > 1)
        n_el, P, _, _ = g.layout()
        psi = g.vec().fill(1.0)
        for _ in range(3):
            g.standard_sweep(psi, psi)
        g.synchronize()
        g.timing(True)
        for _ in range(10):
            g.standard_sweep(psi, psi)
        g.synchronize()
        ms, k = g.timed("sweep")
        g.timing(False)
        t = ms / k
        g.source_iteration(psi, 1)  # warm
        g.synchronize()
        t0 = time.perf_counter()
        g.source_iteration(psi, 2)
        g.synchronize()
        si_ms = (time.perf_counter() - t0) / 2 * 1e3  # rank-local (no allreduce without a communicator)
        t1 = t if n == 1 else t1
        out[n] = {"directions": P, "ms_per_sweep": t, "updates_per_s_job": n_el * P * n / (t * 1e-3),
                  "speedup_vs_1": (t1 / t) if t1 else None, "si_ms_per_iter_rank_local": si_ms,
                  "fold_group": int(g.table("fold")[0]), "hbm_frac_rank": n_el * P * 64 / (t * 1e-3) / 6455.3e9}
        print(json.dumps({n: out[n]}), flush=True)
        psi.free()
        g.close()


if __name__ == "__main__":
    main()
