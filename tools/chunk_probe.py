"""DRAM access-pattern probe: 128 B chunks streamed vs in the sweep's cell-major order."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04559_b200 import configs as cf, stamg
spec = cf.baseline_config(5, 128)
g = stamg.Context(spec, build_hierarchy=False)
v = g.vec().fill(0.0)
for mode, stride in [(0, 1), (1, 2048), (2, 1024), (4, 512), (8, 256), (16, 128)]:
    out = C.c_double()
    stamg._check(stamg.lib().stamg_bench_chunk_rw(g.h, v.h, C.c_int64(stride), mode, C.byref(out)))
    print(f"chunk={128 * max(mode, 1)}B {'stream' if mode == 0 else 'cell-major'} stride={stride} GB/s={out.value:.1f}", flush=True)
