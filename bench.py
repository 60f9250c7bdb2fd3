#!/usr/bin/env python3
"""Benchmark: transport-sweep throughput (cell.direction updates/s) on
BASELINE.json config 5 (512x512 bilinear cells, 8192 angular patches, fp64),
directions sharded across ranks, plus GMRES+AMG solve wall time (configs 1-3)
and source-iteration throughput as extra keys.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One JSON line on rank 0. Under torchrun each rank drives one GPU and owns
P/N directions (strong scaling: total work fixed, no collective on the
sweep). ``--impl reference`` times the CPU restatement of the reference
(oracle/, the reference itself does not build here) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sweep cell·direction updates/s"
UNIT = "cell·direction updates/s"
BYTES_PER_UPDATE = 64  # read rhs block (4 doubles) + write solution block (4 doubles)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: through NVML every 5 ms
    when pynvml can load it (the timed region of the default run is a quarter of a second),
    otherwise one nvidia-smi query per 0.2 s."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []       # nvidia-smi rows
        self.samples = []    # NVML samples: (sm_mhz, reasons bitmask, power_w, mem_mhz)
        self._stop = threading.Event()
        self._nvml = None
        self._h = None
        self._max = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._nvml = pynvml
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run_nvml if self._nvml else self._run, daemon=True)

    def _run_nvml(self):
        nv, h = self._nvml, self._h
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                try:
                    mem = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM))
                except Exception:
                    mem = None
                try:
                    pw = nv.nvmlDeviceGetPowerUsage(h) * 1e-3
                except Exception:
                    pw = None
                self.samples.append((sm, int(reasons(h)), pw, mem))
            except Exception:
                pass
            self._stop.wait(0.005)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if self._nvml and self.samples:
            nv = self._nvml
            bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            seen = sorted(n for n, b in bits.items() if any(s[1] & b for s in self.samples))
            out = {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": self._max, "reasons": seen,
                   "samples": len(self.samples), "source": "nvml, 5 ms period",
                   "sm_mhz_min": min(s[0] for s in self.samples)}
            pw = [s[2] for s in self.samples if s[2] is not None]
            mem = [s[3] for s in self.samples if s[3] is not None]
            if pw:
                out["power_w"] = statistics.median(pw)
            if mem:
                out["mem_mhz"] = statistics.median(mem)
            return out
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = self.NAMES
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvidia-smi, 0.2 s period"}


def fp64_peaks_with_clocks(g, local):
    """The DMMA / DFMA throughput probes (FP64 roofline denominators: not in
    MEASURED_PEAKS.json) with the SM clocks sampled while they run."""
    with ClockSampler(local) as clk:
        dmma, dfma = g.fp64_peaks()
        dmma2, dfma2 = g.fp64_peaks()  # >= 2 samples of the clock inside the probe window
    return max(dmma, dmma2), max(dfma, dfma2), clk.summary()


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local, dist


def allmax(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


class CpuSweepSampler:
    """Oracle (CPU restatement of standard_sweep, sweeps.cpp:20-42, OpenMP over
    patches) on n_dirs directions of the same grid.  The oracle is built once;
    ``sample(min_s)`` repeats whole n_dirs-direction sweeps until at least
    ``min_s`` seconds of CPU work and returns (updates/s, seconds, sweeps)."""

    def __init__(self, spec, n_dirs, threads=None):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        import dataclasses
        # the sweep needs only the transport blocks (no couplings): scatter order 0,
        # same grid and cross sections; angular level 2 (128 directions) keeps the
        # host vectors at 1 GiB -- per-direction work is identical
        s0 = dataclasses.replace(spec, N=0, moments=np.asarray(spec.moments)[:, :1].copy(), n_levels=1,
                                 angular_level=2)
        if threads:
            os.environ["OMP_NUM_THREADS"] = str(threads)
        self.o = pyoracle.Oracle(s0)
        self.n_el, self.P, S, _ = self.o.layout()
        self.n_dirs = min(n_dirs, self.P)
        self.rhs = np.random.default_rng(0).uniform(-1, 1, self.n_el * self.P * S)
        self.z = np.zeros_like(self.rhs)
        self.o.sweep(self.rhs, q0=0, q1=min(4, self.P), z=self.z)  # warm

    def sample(self, min_s):
        reps = 0
        t = time.perf_counter()
        while True:
            self.o.sweep(self.rhs, q0=0, q1=self.n_dirs, z=self.z)
            reps += 1
            dt = time.perf_counter() - t
            if dt >= min_s:
                return self.n_el * self.n_dirs * reps / dt, dt, reps


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, world, rank, dist):
    from paper_2010_04559_b200 import configs as cf
    if rank != 0:
        return
    spec = cf.baseline_config(5)
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    smp = CpuSweepSampler(spec, 128, threads)
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, reps = smp.sample(args.ref_step_s)
        if i >= args.warmup:
            vals.append((v, dt, reps))
    value = statistics.median([v for v, _, _ in vals])
    ms = statistics.median([dt for _, dt, _ in vals]) * 1e3
    sample = (f"oracle standard_sweep (OpenMP over patches) over {smp.n_dirs} directions x {smp.n_el} cells, "
              f"repeated for >= {args.ref_step_s:g} s per step (config 5 grid and cross sections, angular "
              f"level 2 instead of 5 to bound host memory; per-direction work is identical)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c5: 512x512 bilinear cells, uniform angular level 5 (8192 patches), fp64 sweep",
                       "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


SOLVE_KERNELS = ("coarse_gs", "sweep", "apply_L", "d2m", "m2d", "fold", "unfold", "restrict", "prolong")


def kernel_rooflines(stamg, cf, dmma_peak):
    """Per-kernel roofline at full config 4 (the largest solve config): the outer
    apply_L / sweep / scatter GEMMs (N = 32), and the transfers and reduced-order
    (nr = 8) GEMMs between the two finest MG levels, one call each after a warm
    call, CUDA events on the context stream. Algorithmic bytes: apply_L and the
    sweep 64 B per cell-direction; restrict V_f + V_c, prolongate V_c + V_f
    (the API's non-accumulating form); GEMM flops 2*H*P*4 per cell each."""
    hbm, _ = peaks()
    spec = cf.baseline_config(4)
    g = stamg.Context(spec)
    out = {}
    try:
        n_el, P, _, _ = g.layout()
        nlev, nr = g.levels()
        x, y = g.vec().fill(1.0), g.vec()

        def timed(name, fn):
            fn()
            g.synchronize()
            g.timing(True)
            fn()
            g.synchronize()
            ms, n = g.timed(name)
            g.timing(False)
            return ms / max(n, 1) * 1e-3

        def hbm_row(name, fn, nbytes, kname=None):
            t = timed(kname or name, fn)
            out[name] = {"ms": t * 1e3, "bytes": nbytes, "achieved_gbs": nbytes / t * 1e-9, "frac": nbytes / t * 1e-9 / hbm,
                         "bound": "hbm"}

        upd = n_el * P
        hbm_row("apply_L", lambda: g.apply_L_into(x, y), upd * 64)
        hbm_row("sweep", lambda: g.standard_sweep(x, y), upd * 64)
        fold = max(1, int(g.table("fold")[0]))
        for kname in ("d2m", "m2d"):
            t_all = None
            g.apply_scatter_into(x, spec.N, 1.0, y)
            g.synchronize()
            g.timing(True)
            g.apply_scatter_into(x, spec.N, 1.0, y)
            g.synchronize()
            t_all = g.timed(kname)[0] * 1e-3
            g.timing(False)
            flop = 2.0 * (spec.N + 1) ** 2 * P * 4 * n_el
            out[f"{kname}_outer"] = {"ms": t_all * 1e3, "algorithmic_flop": flop, "fold_group_size": fold,
                                     "achieved_tflops_executed": flop / fold / t_all * 1e-12,
                                     "frac": flop / fold / t_all * 1e-12 / dmma_peak, "bound": "fp64_tensor"}
        del x, y
        lf = nlev - 1
        vf, vc = g.vec(lf).fill(1.0), g.vec(lf - 1).fill(1.0)
        _, Pf, _, _ = g.layout(lf)
        _, Pc, _, _ = g.layout(lf - 1)
        Vf, Vc = n_el * Pf * 32, n_el * Pc * 32
        hbm_row("restrict", lambda: g.restrict_residual(lf, vf, vc), Vf + Vc)
        hbm_row("prolongate", lambda: g.prolongate(lf, vc, vf), Vf + Vc, "prolong")
        yf = g.vec(lf)
        g.apply_scatter_into(vf, nr, 1.0, yf, level=lf)
        g.synchronize()
        g.timing(True)
        g.apply_scatter_into(vf, nr, 1.0, yf, level=lf)
        g.synchronize()
        for kname in ("d2m", "m2d"):
            t = g.timed(kname)[0] * 1e-3
            flop = 2.0 * (nr + 1) ** 2 * Pf * 4 * n_el
            out[f"{kname}_mg_nr{nr}"] = {"ms": t * 1e3, "algorithmic_flop": flop, "achieved_tflops": flop / t * 1e-12,
                                        "frac": flop / t * 1e-12 / dmma_peak, "bound": "fp64_tensor"}
        g.timing(False)
        # the forms the V-cycle runs: one smoother step on the finest MG level = residual
        # apply_L (y = f - L x: reads x and f, writes y) + reduced-order scatter + accumulating
        # sweep (reads rhs and the base vector, writes z): 96 B per cell-direction each
        ff, ph = g.vec(lf).fill(1.0), g.vec(lf).fill(0.5)
        g.smoother_step(ff, nr, ph, level=lf)
        g.synchronize()
        g.timing(True)
        g.smoother_step(ff, nr, ph, level=lf)
        g.synchronize()
        for name, kname in (("smoother_apply_L", "apply_L"), ("smoother_sweep", "sweep")):
            ms, n = g.timed(kname)
            t = ms / max(n, 1) * 1e-3
            nbytes = n_el * Pf * 96
            out[name] = {"ms": t * 1e3, "bytes": nbytes, "achieved_gbs": nbytes / t * 1e-9, "frac": nbytes / t * 1e-9 / hbm,
                         "bound": "hbm", "level": lf}
        g.timing(False)
        out["config"] = f"c4 full: {n_el} cells, outer P={P} (N={spec.N}), MG levels {lf}->{lf - 1}: P {Pf}->{Pc} (nr={nr})"
    finally:
        g.close()
    return out


def reference_shape_cpu(n, box, level, N, m, sigma_t, sigma_a, solve=False):
    """The reference's OWN sources (oracle/_ref/libstamgref.so: /root/reference/proj/src compiled
    unchanged against the Eigen-subset shim, OpenMP as the reference has it) on the same 3D problem:
    standard_sweep / apply_L time and the BiCGSTAB + MG solve. cpu_baseline.kind = "reference"; the
    shim's dense kernels are plain loops, not Eigen's vectorised ones, which is stated in `note`."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import pyref
        if not os.path.exists(pyref.LIB_PATH):
            return {"unavailable": "oracle/_ref/libstamgref.so not built (needs /root/reference at build time)"}
        r = pyref.Reference(n, box, level, 1, 1, N, m, sigma_t, sigma_a, nr=4)
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"}
    x = np.ones(r.size())
    out = {"kind": "reference", "cores": os.cpu_count() or 1, "cpu_model": cpu_model(), "problem": f"{n}^3 cells",
           "note": "reference sources unchanged; Eigen replaced by oracle/eigen_shim (plain loops)"}
    if solve:
        t0 = time.perf_counter()
        _, rep = r.bicgstab("mg", tol=1e-8, max_iter=100)
        out["bicgstab_mg"] = {"wall_s": time.perf_counter() - t0, "iterations": rep["iterations"],
                              "converged": rep["converged"]}
        return out
    for name, fn in (("sweep", r.sweep), ("apply_L", r.apply_L)):
        fn(x)
        t0 = time.perf_counter()
        fn(x)
        out[name + "_ms"] = (time.perf_counter() - t0) * 1e3
    return out


def reference_shape_section(stamg, cf, hbm, dfma_peak, with_cpu=True):
    """The reference-shape path on a problem of the reference's own kind: 3D
    trilinear cells, Lin angular basis (24 dofs per cell and patch), FP-equivalent moments N = 8,
    uniform source, all MG levels. Per-operator time with the HBM bandwidth its algorithmic bytes
    correspond to (apply_L, sweep: one vector in, one out; scatter: two in, one out), and the
    BiCGSTAB + V(1,1) solve wall time to 1e-8."""
    n, level, N = 24, 2, 8
    nn = np.arange(N + 1, dtype=np.float64)
    m = 0.5 * 0.5 * (N * (N + 1.0) - nn * (nn + 1.0))  # scatter.cpp:9-21, alpha = 0.5
    spec = cf.reference_test_problem(n, n / 8.0, level, 1, 1, N, m, 0.1 + m[0], dim=3, q_el=np.ones(n ** 3),
                                     n_levels=0, nr=4)
    t0 = time.perf_counter()
    g = stamg.Context(spec)
    out = {"problem": f"{n}^3 trilinear cells, Lin basis, angular level {level}", "setup_s": time.perf_counter() - t0}
    n_el, P, S, D = g.layout()
    vb = n_el * P * S * D * 8
    out["layout"] = {"n_el": n_el, "patches": P, "S": S, "D": D, "vector_bytes": vb}
    x, y = g.vec().fill(1.0), g.vec()
    g.timing(True)
    reps = 5
    for _ in range(reps):
        g.apply_L_into(x, y)
        g.standard_sweep(x, y)
        g.apply_scatter_into(x, N, 1.0, y)
    g.synchronize()
    # a (cell, patch) block is bs = D*S doubles; apply_L and the sweep do (1 + dim) dense bs x bs
    # products per block (4.6 kflop per 384 B at bs = 24: above the FP64 ridge, so FP64-bound)
    bs = S * D
    blk_flop = 2.0 * bs * bs * 4 * n_el * P
    rows = {"apply_L": (("apply_L",), 2, blk_flop), "sweep": (("sweep",), 2, blk_flop),
            "scatter": (("d2m", "m2d"), 3, 4.0 * (N + 1) ** 2 * P * D * S * n_el)}
    for name, (ks, nvec, flop) in rows.items():
        ms = sum(g.timed(k)[0] for k in ks) / reps
        gbs, tf = nvec * vb / (ms * 1e-3) * 1e-9, flop / (ms * 1e-3) * 1e-12
        fp64_bound = flop / (nvec * vb) > dfma_peak * 1e12 / (hbm * 1e9)
        out[name] = {"ms": ms, "achieved_gbs": gbs, "hbm_frac": gbs / hbm, "achieved_tflops": tf,
                     "fp64_frac": tf / dfma_peak, "bound": "fp64" if fp64_bound else "hbm",
                     "frac": tf / dfma_peak if fp64_bound else gbs / hbm}
    out["fp64_peak_tflops"] = dfma_peak
    out["sweep"]["updates_per_s"] = n_el * P / (out["sweep"]["ms"] * 1e-3)
    g.timing(False)
    b = g.rhs()
    g.solve(b, "bicgstab", "mg", tol=1e-8, max_iter=100)
    g.synchronize()
    t0 = time.perf_counter()
    _, rep = g.solve(b, "bicgstab", "mg", tol=1e-8, max_iter=100)
    g.synchronize()
    out["bicgstab_mg"] = {"wall_s": time.perf_counter() - t0, "iterations": rep["iterations"], "converged": rep["converged"]}
    g.close()
    # the solve once more on an 8^3 grid, where the reference's own CPU solve takes seconds
    ns = 8
    spec8 = cf.reference_test_problem(ns, ns / 8.0, level, 1, 1, N, m, 0.1 + m[0], dim=3, q_el=np.ones(ns ** 3),
                                      n_levels=0, nr=4)
    g8 = stamg.Context(spec8)
    b8 = g8.rhs()
    g8.solve(b8, "bicgstab", "mg", tol=1e-8, max_iter=100)
    g8.synchronize()
    t0 = time.perf_counter()
    _, rep8 = g8.solve(b8, "bicgstab", "mg", tol=1e-8, max_iter=100)
    g8.synchronize()
    out["bicgstab_mg_8cube"] = {"wall_s": time.perf_counter() - t0, "iterations": rep8["iterations"],
                                "converged": rep8["converged"]}
    g8.close()
    if with_cpu:
        out["cpu"] = reference_shape_cpu(n, n / 8.0, level, N, m, 0.1 + m[0], 0.1)
        out["cpu_8cube"] = reference_shape_cpu(ns, ns / 8.0, level, N, m, 0.1 + m[0], 0.1, solve=True)
    return out


def make_context(stamg, spec, world, rank, local, dist, build_hierarchy):
    """One context per rank; ranks > 1 share a fresh NCCL communicator (unique id
    from rank 0, broadcast over torch.distributed)."""
    nccl_id = None
    if world > 1:
        import torch
        uid = bytearray(stamg.nccl_unique_id()) if rank == 0 else bytearray(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        nccl_id = bytes(t.cpu().tolist())
    return stamg.Context(spec, device=local if world > 1 else 0, build_hierarchy=build_hierarchy, rank=rank,
                         world=world, nccl_id=nccl_id)


def run_b200(args, world, rank, local, dist):
    from paper_2010_04559_b200 import configs as cf
    from paper_2010_04559_b200 import stamg
    spec = cf.baseline_config(5, args.n)
    t_setup = time.perf_counter()
    g = make_context(stamg, spec, world, rank, local, dist, False)
    setup_s = allmax(dist, time.perf_counter() - t_setup)  # host tables + device couplings + upload
    n_el, P_local, S, _ = g.layout()
    upd_local = n_el * P_local
    psi = g.vec().fill(1.0)
    # warm-up
    for _ in range(args.warmup):
        g.standard_sweep(psi, psi)
    g.synchronize()
    # timed region: K in-place sweeps (64 GiB vector >> 126 MB L2, no flush needed)
    l0 = g.launch_count()
    g.timing(True)
    barrier(dist)
    g.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            g.standard_sweep(psi, psi)
        g.synchronize()
        wall = time.perf_counter() - t0
    barrier(dist)
    sweep_ms, sweep_n = g.timed("sweep")
    g.timing(False)
    launches = g.launch_count() - l0
    # device time of the K steps = the summed per-launch CUDA-event durations
    dev_s = allmax(dist, sweep_ms * 1e-3)
    total_upd = n_el * P_local * world if world > 1 else upd_local
    value = total_upd * args.steps / dev_s
    ms_per_step = dev_s / args.steps * 1e3
    hbm, peak_kind = peaks()
    achieved = upd_local * BYTES_PER_UPDATE / (sweep_ms * 1e-3 / max(sweep_n, 1)) / 1e9
    traffic = None
    try:
        # ncu --set full capture of this exact launch (config 5 at full size, one GPU):
        # dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/r02_sweep_c5_ncu_traffic.json)
        if world == 1 and args.n is None:
            with open(os.path.join(ROOT, "profiles", "r02_sweep_c5_ncu_traffic.json")) as f:
                traffic = json.load(f)["dram_bytes_per_launch"]
    except Exception:
        pass
    extras = {}
    # ---- extra: source-iteration throughput on the same workload (M2D source from the
    # moments + in-place sweep + D2M moments [+ allreduce]), FP64-tensor roofline of the GEMMs
    if not args.no_si:
        g.source_iteration(psi, 1)  # warm
        g.synchronize()
        g.timing(True)
        barrier(dist)
        t0 = time.perf_counter()
        g.source_iteration(psi, args.si_iters)
        g.synchronize()
        si_wall = allmax(dist, time.perf_counter() - t0)
        d2m_ms, _ = g.timed("d2m")
        m2d_ms, _ = g.timed("m2d")
        sw_ms, _ = g.timed("sweep")
        g.timing(False)
        H = (spec.N + 1) ** 2
        gemm_flop = 2.0 * H * P_local * 4 * n_el * args.si_iters  # per contraction, all iterations (algorithmic)
        fold_g = max(1, int(g.table("fold")[0]))  # reflection-symmetry fold: executed = algorithmic / |G|
        exe_flop = gemm_flop / fold_g
        dmma_peak, dfma_peak, probe_clk = fp64_peaks_with_clocks(g, local)
        extras["source_iteration"] = {
            "value": total_upd * args.si_iters / si_wall, "unit": UNIT, "iterations": args.si_iters,
            "ms_per_iter": si_wall / args.si_iters * 1e3,
            "kernel_ms_per_iter": {"d2m": d2m_ms / args.si_iters, "m2d": m2d_ms / args.si_iters,
                                   "sweep": sw_ms / args.si_iters},
            "gemm_roofline": {"bound": "fp64_tensor", "unit": "TFLOP/s",
                              "d2m_achieved": exe_flop / (d2m_ms * 1e-3) * 1e-12,
                              "m2d_achieved": exe_flop / (m2d_ms * 1e-3) * 1e-12,
                              "peak": dmma_peak, "peak_kind": "measured DMMA m8n8k4 probe on this GPU",
                              "peak_probe_clocks": probe_clk,
                              "dfma_peak": dfma_peak,
                              "frac": (2 * exe_flop / ((d2m_ms + m2d_ms) * 1e-3) * 1e-12) / dmma_peak,
                              "achieved_basis": "executed flops (algorithmic / fold group size)",
                              "fold_group_size": fold_g,
                              "algorithmic_flop_per_contraction": 2.0 * H * P_local * 4 * n_el,
                              "algorithmic_equivalent_tflops": 2 * gemm_flop / ((d2m_ms + m2d_ms) * 1e-3) * 1e-12},
            "kernel_ms_per_iter_fold": {k: g.timed(k)[0] / args.si_iters for k in ("fold", "unfold")},
            "step": "fold -> D2M(psi) -> [allreduce] -> M2D -> unfold (q + S psi) -> in-place sweep, full "
                    "order N=%d" % spec.N}
    # ---- e2e through the host-buffer C-ABI entry point (pinned buffers)
    e2e = None
    if not args.no_e2e:
        n = psi.n
        psi.free()
        host = stamg.host_alloc(n)
        host[: min(n, 1 << 20)] = 1.0
        g.sweep_host(host, host)  # warm (allocates the device staging buffer)
        k_e2e = min(args.steps, 3)
        barrier(dist)
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            g.sweep_host(host, host)
        e2e_s = allmax(dist, time.perf_counter() - t0)
        e2e = {"value": total_upd * k_e2e / e2e_s, "unit": UNIT, "h2d_bytes_per_step": n * 8,
               "d2h_bytes_per_step": n * 8, "steps": k_e2e,
               "api": "stamg_sweep_host (include/stamg_b200.h), pinned host buffers",
               "pipeline_chunks": g.host_pipeline_chunks()}
        stamg.host_free(host)
    dmma_peak, dfma_peak_k, probe_clk = fp64_peaks_with_clocks(g, local)
    g.close()
    if not args.no_kernels and world == 1:
        extras["kernels"] = kernel_rooflines(stamg, cf, dmma_peak)
        extras["kernels"]["dmma_peak_tflops"] = dmma_peak
        extras["kernels"]["dmma_peak_probe_clocks"] = probe_clk
    if not args.no_generic and world == 1:
        extras["reference_shape"] = reference_shape_section(stamg, cf, hbm, dfma_peak_k, with_cpu=not args.no_cpu)
    # ---- extra: GMRES + AMG solve wall time to 1e-8 from a device-resident b
    # (directions sharded over the ranks, coarsest MG level replicated)
    if not args.no_solve:
        solves = {}
        for k in args.solve_configs:
            sp = cf.baseline_config(k)
            t0 = time.perf_counter()
            gs = make_context(stamg, sp, world, rank, local, dist, True)
            setup = time.perf_counter() - t0
            b = gs.rhs()
            # warm-up (workspaces, V-cycle graph capture): the whole solve for configs 1-3, two
            # iterations for config 4 (a 40 s solve; its warm-up effects are < 0.1 s)
            big = k >= 4
            if big:
                gs.solve(b, "gmres", "mg", tol=1e-300, max_iter=2)
            else:
                gs.solve(b, "gmres", "mg")
            gs.synchronize()
            barrier(dist)
            t0 = time.perf_counter()
            x, rep = gs.solve(b, "gmres", "mg")
            gs.synchronize()
            solve_wall = allmax(dist, time.perf_counter() - t0)
            solves[f"c{k}"] = {"wall_s": solve_wall, "setup_s": setup, "iterations": rep["iterations"],
                               "final_residual": rep["final_residual"], "converged": rep["converged"],
                               "method": "GMRES(%d) right-preconditioned by one V(1,1) angular MG cycle" % sp.restart}
            # where the time goes: the same solve once more with per-launch CUDA events (config 4:
            # its first 8 iterations, to keep the default run within minutes)
            gs.timing(True)
            if big:
                gs.solve(b, "gmres", "mg", tol=1e-300, max_iter=8)
                solves[f"c{k}"]["kernel_ms_iterations"] = 8
            else:
                gs.solve(b, "gmres", "mg")
            gs.synchronize()
            solves[f"c{k}"]["kernel_ms"] = {kk: round(gs.timed(kk)[0], 3) for kk in SOLVE_KERNELS}
            gs.timing(False)
            gs.close()
        extras["solve"] = solves
    # ---- CPU baseline (oracle port) on rank 0 at N = 1
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        smp = CpuSweepSampler(spec, args.cpu_dirs, threads)
        v, dt, reps = smp.sample(args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle standard_sweep over {smp.n_dirs} directions x {smp.n_el} cells, {reps} sweeps "
                         f"in {dt:.1f} s (config 5 grid, angular level 2 to bound host memory)"}
        cpu["cpu_model"] = cpu_model()
        # the same solves on the oracle (serial coarse GS like the reference, OpenMP elsewhere)
        if not args.no_solve and "solve" in extras:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import pyoracle
            for k in args.cpu_solve_configs:
                key = f"c{k}"
                if key not in extras["solve"]:
                    continue
                o = pyoracle.Oracle(cf.baseline_config(k))
                t0 = time.perf_counter()
                _, rep = o.solve("gmres", "mg")
                extras["solve"][key]["cpu"] = {"wall_s": time.perf_counter() - t0, "iterations": rep["iterations"],
                                               "final_residual": rep["final_residual"], "cores": threads,
                                               "kind": "port"}
                del o
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"c5: {spec.nx}x{spec.ny} bilinear cells, uniform angular level 5 "
                                       f"({P_local * world} patches), one in-place standard_sweep per step, "
                                       f"directions sharded over {world} rank(s) (whole reflection orbits per rank)",
                           "l2": f"input {spec.n_el * P_local * world * 4 * 8 / 2**30:.1f} GiB >> 126 MB L2 (no flush needed)", "wall_s": wall,
                           "setup_s": setup_s},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                             "frac": achieved / hbm, "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read + write)",
                             "algorithmic_bytes_per_launch": upd_local * BYTES_PER_UPDATE, "peak_kind": peak_kind,
                             "kernel": "sweep_kernel", "bytes_per_update": BYTES_PER_UPDATE},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}
        line.update(extras)
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=None, help="cells per axis override (default: config 5 = 512)")
    ap.add_argument("--cpu-dirs", type=int, default=128)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="minimum CPU work for the cpu_baseline leg")
    ap.add_argument("--ref-step-s", type=float, default=3.0, help="minimum CPU work per --impl reference step")
    ap.add_argument("--solve-configs", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--si-iters", type=int, default=2)
    ap.add_argument("--no-si", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel roofline section (config 4)")
    ap.add_argument("--cpu-solve-configs", type=int, nargs="*", default=[1, 2],
                    help="also time these solves on the CPU oracle (rank 0, N=1); c2 takes ~100 s on 8 cores")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-generic", action="store_true", help="skip the reference-shape (3D trilinear Lin) section")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local, dist = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank, dist)
    else:
        run_b200(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
