// Device helpers shared by the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace stamg_b200 {

// ---- async global -> shared copies (LDGSTS) ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // src-size 0 zero-fills the destination
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- TMA bulk copies (cp.async.bulk, UBLKCP) completing on a CTA mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init_cta(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// generic-proxy shared-memory state (barrier init, zero fill) visible to the async proxy
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, "
        "p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---- streaming 16-byte global accesses ----
__device__ __forceinline__ double2 ld_stream(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// one 32-byte block (4 doubles = one DRAM sector) per thread: 256-bit LDG/STG (sm_100)
#ifndef STAMG_ST_CLOBBER
#define STAMG_ST_CLOBBER 1  // A/B knob: "memory" clobber on the 256-bit block store
#endif
#ifndef STAMG_V256
#define STAMG_V256 1
#endif
struct dbl4 {
  double x, y, z, w;
};
__device__ __forceinline__ dbl4 ld_block(const double* p) {
  dbl4 v;
#if STAMG_V256
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#else
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  v.x = a.x, v.y = a.y, v.z = b.x, v.w = b.y;
#endif
  return v;
}
// the same for data the kernel itself writes (no read-only path)
__device__ __forceinline__ dbl4 ld_block_rw(const double* p) {
  dbl4 v;
#if STAMG_V256
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p) : "memory");
#else
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  v.x = a.x, v.y = a.y, v.z = b.x, v.w = b.y;
#endif
  return v;
}
__device__ __forceinline__ void st_block(double* p, const dbl4& v) {
#if STAMG_V256
#if STAMG_ST_CLOBBER
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
#else  // streaming stores: volatile keeps them ordered with the block loads; other loads may move across
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w));
#endif
#else
  reinterpret_cast<double2*>(p)[0] = make_double2(v.x, v.y);
  reinterpret_cast<double2*>(p)[1] = make_double2(v.z, v.w);
#endif
}

// L2-coherent (bypass L1) accesses for data produced by other CTAs of the same launch
__device__ __forceinline__ double2 ld_cg2(const double* p) {
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cg2(double* p, double2 v) {
  asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- FP64 tensor core: D(8x8) += A(8x4, row) * B(4x8, col), lowers to DMMA ----
// Fragments (per lane, g = lane>>2, t = lane&3): a = A[g][t], b = B[t][g],
// c0/c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- wavefront layout (throughput contexts): per 8-direction group, cells are stored
// strip by strip (R rows), along the sweep's anti-diagonals d = i + r of the group's
// frame, row within the diagonal fastest. A sweep step then touches R consecutive
// slots (R x 256 bytes). Slot count per group: nstrips * (nx + R - 1) * R (padding = 0).
struct WLGeom {
  int nx = 0, ny = 0, R = 32, nd = 0;
  long long slots = 0;        // slots per group
  const int* goct = nullptr;  // octant of each group
};
__host__ __device__ __forceinline__ long long wl_slot_frame(const WLGeom& w, int i, int j) {
  const int s = j / w.R, r = j - s * w.R;
  return ((long long)s * w.nd + i + r) * w.R + r;
}
// index of the 32-byte block of (element el, internal direction k)
__device__ __forceinline__ long long wl_block(const WLGeom& w, int el, int k) {
  const int g = k >> 3, oct = w.goct[g];
  const int gx = el % w.nx, gy = el / w.nx;
  const int i = (oct & 1) ? w.nx - 1 - gx : gx, j = (oct & 2) ? w.ny - 1 - gy : gy;
  return ((long long)g * w.slots + wl_slot_frame(w, i, j)) * 8 + (k & 7);
}

__device__ __forceinline__ double2 shfl_up2(double2 v, int d) {
  v.x = __shfl_up_sync(0xffffffffu, v.x, d);
  v.y = __shfl_up_sync(0xffffffffu, v.y, d);
  return v;
}

}  // namespace stamg_b200
