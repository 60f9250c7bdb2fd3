// Angular-multigrid kernels on sm_100a:
//  * prolongate / restrict_residual (multigrid.cpp:100-136), Const transfer
//    blocks: coalesced gather / ordered segmented sum over the children list;
//  * coarse_scatter_sweep (sweeps.cpp:51-104): order-exact scatter-implicit
//    Gauss-Seidel as a persistent dataflow kernel.
//
// Coarse GS work item = (pass, octant, k-th cell of the octant's sweep order),
// claimed by one warp from a global ticket in exactly the reference's loop
// order, so every item's inputs are produced by lower tickets. A warp starts
// an item when its dependencies have published their completed-pass counter:
// the x/y upwind cells of the same octant (same pass), the same cell in the
// previous octant (its running moments), and - write-after-read - the
// downwind cells of the previous pass. The item's patch loop is the
// reference's, with the cell's moments (H x 4) held in registers across the
// warp (lane owns harmonics lane, lane+32, ...). Results are bitwise
// reproducible run to run.
#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "kernels.hpp"

namespace stamg_b200 {
namespace {

__global__ void prolong_kernel(const double* __restrict__ coarse, double* __restrict__ fine,
                               const int* __restrict__ up, const double* __restrict__ w, int n_el, int Pf, int Pc,
                               bool add) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (el, q)
  if (idx >= (int64_t)n_el * Pf) return;
  const int el = int(idx / Pf), q = int(idx - (int64_t)el * Pf);
  const double wq = w[q];
  const double2* src = reinterpret_cast<const double2*>(coarse + ((size_t)el * Pc + up[q]) * 4);
  double2* dst = reinterpret_cast<double2*>(fine + (size_t)idx * 4);
  double2 a = src[0], b = src[1];
  a.x *= wq, a.y *= wq, b.x *= wq, b.y *= wq;
  if (add) {
    const double2 fa = dst[0], fb = dst[1];
    a.x = fa.x + a.x, a.y = fa.y + a.y, b.x = fb.x + b.x, b.y = fb.y + b.y;
  }
  dst[0] = a, dst[1] = b;
}

__global__ void restrict_kernel(const double* __restrict__ fine, double* __restrict__ coarse,
                                const int* __restrict__ cptr, const int* __restrict__ cidx,
                                const double* __restrict__ w, int n_el, int Pf, int Pc) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (el, c)
  if (idx >= (int64_t)n_el * Pc) return;
  const int el = int(idx / Pc), c = int(idx - (int64_t)el * Pc);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int k = cptr[c]; k < cptr[c + 1]; ++k) {  // ascending fine index, as the reference's += loop
    const int q = cidx[k];
    const double wq = w[q];
    const double2* src = reinterpret_cast<const double2*>(fine + ((size_t)el * Pf + q) * 4);
    const double2 a = src[0], b = src[1];
    s0 += wq * a.x, s1 += wq * a.y, s2 += wq * b.x, s3 += wq * b.y;
  }
  double2* dst = reinterpret_cast<double2*>(coarse + (size_t)idx * 4);
  dst[0] = make_double2(s0, s1), dst[1] = make_double2(s2, s3);
}

__device__ __forceinline__ void perm(int m, double& a0, double& a1, double& a2, double& a3) {
  if (m & 1) { double u = a0; a0 = a1; a1 = u; u = a2; a2 = a3; a3 = u; }
  if (m & 2) { double u = a0; a0 = a2; a2 = u; u = a1; a1 = a3; a3 = u; }
}

template <int KH, int NS>
__global__ void __launch_bounds__(128) coarse_gs_kernel(CoarseGSParams p) {
  // KH harmonics per lane (H <= 32 KH); NS patch slots per lane (patches per octant <= 32 NS)
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const int n_el = p.n_el, nx = p.nx, ny = p.ny, P = p.P, Hp = p.Hp, H = p.H;
  const int per_pass = 8 * n_el;
  const int total = p.nu * per_pass;
  for (;;) {
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(p.counter, 1);
    ticket = __shfl_sync(full, ticket, 0);
    if (ticket >= total) return;
    const int pass = ticket / per_pass, rem = ticket - pass * per_pass;
    const int oct = rem / n_el, kk = rem - oct * n_el;
    const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
    const int m = (xneg ? 1 : 0) | (yneg ? 2 : 0);
    const int jf = kk / nx, ifr = kk - jf * nx;
    const int gx = xneg ? nx - 1 - ifr : ifr, gy = yneg ? ny - 1 - jf : jf;
    const int el = gy * nx + gx;
    const int sx = xneg ? -1 : 1, sy = yneg ? -nx : nx;
    const int upx = ifr > 0 ? el - sx : -1, upy = jf > 0 ? el - sy : -1;
    const int dnx = ifr < nx - 1 ? el + sx : -1, dny = jf < ny - 1 ? el + sy : -1;
    const int pbeg = p.oct_ptr[oct], np = p.oct_ptr[oct + 1] - pbeg;

    // read-only inputs first (independent of the dependency flags)
    double r[NS][4];
    int qs[NS];
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int j = lane + 32 * sl;
      qs[sl] = j < np ? p.oct_patches[pbeg + j] : -1;
      if (qs[sl] >= 0) {
        const double* rb = p.rhs + ((size_t)el * P + qs[sl]) * 4;
        r[sl][0] = rb[0], r[sl][1] = rb[1], r[sl][2] = rb[2], r[sl][3] = rb[3];
      } else {
        r[sl][0] = r[sl][1] = r[sl][2] = r[sl][3] = 0.0;
      }
    }
    // dependencies, polled in parallel by lanes 0..4
    {
      const int* f = nullptr;
      int need = 0;
      if (lane == 0 && upx >= 0) f = p.done + oct * n_el + upx, need = pass + 1;
      if (lane == 1 && upy >= 0) f = p.done + oct * n_el + upy, need = pass + 1;
      if (lane == 2) {
        if (oct > 0) f = p.done + (oct - 1) * n_el + el, need = pass + 1;
        else if (pass > 0) f = p.done + 7 * n_el + el, need = pass;
      }
      if (lane == 3 && pass > 0 && dnx >= 0) f = p.done + oct * n_el + dnx, need = pass;
      if (lane == 4 && pass > 0 && dny >= 0) f = p.done + oct * n_el + dny, need = pass;
      bool ok = f == nullptr || ld_acquire(f) >= need;
      while (!__all_sync(full, ok)) {
        if (!ok) ok = ld_acquire(f) >= need;
      }
    }
    // moments, previous iterate and upwind traces: one round trip
    const int mt = p.mat ? p.mat[el] : 0;
    double mo[KH][4], sg[KH];
    double* mom_el = p.mom + (size_t)el * Hp * 4;
#pragma unroll
    for (int kh = 0; kh < KH; ++kh) {
      const int h = lane + 32 * kh;
      if (h < H) {
        const double2 a = ld_cg2(mom_el + h * 4), b = ld_cg2(mom_el + h * 4 + 2);
        mo[kh][0] = a.x, mo[kh][1] = a.y, mo[kh][2] = b.x, mo[kh][3] = b.y;
        sg[kh] = p.sig[(size_t)mt * Hp + h];
      } else {
        mo[kh][0] = mo[kh][1] = mo[kh][2] = mo[kh][3] = 0.0;
        sg[kh] = 0.0;
      }
    }
    double zo[NS][4];
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int q = qs[sl];
      zo[sl][0] = zo[sl][1] = zo[sl][2] = zo[sl][3] = 0.0;
      if (q < 0) continue;
      const double2 za = ld_cg2(p.phi + ((size_t)el * P + q) * 4), zc = ld_cg2(p.phi + ((size_t)el * P + q) * 4 + 2);
      double ux[4] = {0, 0, 0, 0}, uy[4] = {0, 0, 0, 0};
      if (upx >= 0) {
        const double2 a = ld_cg2(p.phi + ((size_t)upx * P + q) * 4), b = ld_cg2(p.phi + ((size_t)upx * P + q) * 4 + 2);
        ux[0] = a.x, ux[1] = a.y, ux[2] = b.x, ux[3] = b.y;
      }
      if (upy >= 0) {
        const double2 a = ld_cg2(p.phi + ((size_t)upy * P + q) * 4), b = ld_cg2(p.phi + ((size_t)upy * P + q) * 4 + 2);
        uy[0] = a.x, uy[1] = a.y, uy[2] = b.x, uy[3] = b.y;
      }
      zo[sl][0] = za.x, zo[sl][1] = za.y, zo[sl][2] = zc.x, zo[sl][3] = zc.y;
      perm(m, r[sl][0], r[sl][1], r[sl][2], r[sl][3]);
      perm(m, zo[sl][0], zo[sl][1], zo[sl][2], zo[sl][3]);
      perm(m, ux[0], ux[1], ux[2], ux[3]);
      perm(m, uy[0], uy[1], uy[2], uy[3]);
      // upwind terms (sweeps.cpp:87-92), frame rows {0,2} <- x trace {1,3}, rows {0,1} <- y trace {2,3}
      const double* cxy = p.cxy + (size_t)q * 8;
      if (upx >= 0) {
        r[sl][0] -= cxy[0] * ux[1] + cxy[1] * ux[3];
        r[sl][2] -= cxy[2] * ux[1] + cxy[3] * ux[3];
      }
      if (upy >= 0) {
        r[sl][0] -= cxy[4] * uy[2] + cxy[5] * uy[3];
        r[sl][1] -= cxy[6] * uy[2] + cxy[7] * uy[3];
      }
    }
    // the sequential patch chain (sweeps.cpp:86-102)
    for (int j = 0; j < np; ++j) {
      const int sl = j >> 5, src = j & 31;
      double rr[4], z[4];
      int q = 0;
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2)
        if (s2 == sl) {
          q = __shfl_sync(full, qs[s2], src);
#pragma unroll
          for (int i = 0; i < 4; ++i) rr[i] = __shfl_sync(full, r[s2][i], src), z[i] = __shfl_sync(full, zo[s2][i], src);
        }
      const double* Xq = p.X + (size_t)q * Hp;
      double xq[KH];
      double t[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int kh = 0; kh < KH; ++kh) {
        const int h = lane + 32 * kh;
        xq[kh] = h < H ? __ldg(Xq + h) : 0.0;
        const double xs = xq[kh] * sg[kh];
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] += xs * mo[kh][i];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] += __shfl_xor_sync(full, t[i], o);
      perm(m, t[0], t[1], t[2], t[3]);
      // explicit scatter from the other patches: (X sig (mom - X^T zold)) N
      const double sq = p.sq[(size_t)mt * P + q];
      double d[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) d[i] = t[i] - sq * z[i];
      // N is invariant under the frame permutation (uniform square cells)
#pragma unroll
      for (int i = 0; i < 4; ++i) rr[i] += d[0] * p.N[i] + d[1] * p.N[4 + i] + d[2] * p.N[8 + i] + d[3] * p.N[12 + i];
      const double* B = p.BinvGS + ((size_t)mt * P + q) * 16;
      double n[4], e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) n[i] = B[4 * i] * rr[0] + B[4 * i + 1] * rr[1] + B[4 * i + 2] * rr[2] + B[4 * i + 3] * rr[3];
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = n[i] - z[i];
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2)
        if (s2 == sl && lane == src)
#pragma unroll
          for (int i = 0; i < 4; ++i) zo[s2][i] = n[i];
      perm(m, e[0], e[1], e[2], e[3]);
#pragma unroll
      for (int kh = 0; kh < KH; ++kh)
#pragma unroll
        for (int i = 0; i < 4; ++i) mo[kh][i] += xq[kh] * e[i];
    }
    // publish: new iterate of this cell's patches, running moments, flag
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int q = qs[sl];
      if (q < 0) continue;
      perm(m, zo[sl][0], zo[sl][1], zo[sl][2], zo[sl][3]);
      double* zb = p.phi + ((size_t)el * P + q) * 4;
      st_cg2(zb, make_double2(zo[sl][0], zo[sl][1]));
      st_cg2(zb + 2, make_double2(zo[sl][2], zo[sl][3]));
    }
#pragma unroll
    for (int kh = 0; kh < KH; ++kh) {
      const int h = lane + 32 * kh;
      if (h < H) {
        st_cg2(mom_el + h * 4, make_double2(mo[kh][0], mo[kh][1]));
        st_cg2(mom_el + h * 4 + 2, make_double2(mo[kh][2], mo[kh][3]));
      }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(p.done + oct * n_el + el, pass + 1);
  }
}

template <int KH, int NS>
void launch_gs2(const CoarseGSParams& p, cudaStream_t s) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_gs_kernel<KH, NS>, 128, 0);
  const long items = (long)p.nu * 8 * p.n_el;
  long blocks = (long)sms * (per_sm > 0 ? per_sm : 1);
  blocks = std::min(blocks, (items + 3) / 4);
  coarse_gs_kernel<KH, NS><<<int(blocks), 128, 0, s>>>(p);
}

template <int KH>
void launch_gs(const CoarseGSParams& p, cudaStream_t s, int max_np) {
  if (max_np <= 32) launch_gs2<KH, 1>(p, s);
  else if (max_np <= 64) launch_gs2<KH, 2>(p, s);
  else throw std::invalid_argument("coarse_scatter_sweep: more than 64 patches per octant on the coarsest level");
}

}  // namespace

void launch_prolong(const double* coarse, double* fine, const int* up, const double* w, int n_el, int Pf, int Pc,
                    bool add, cudaStream_t s) {
  const int64_t n = (int64_t)n_el * Pf;
  if (n == 0) return;
  prolong_kernel<<<int((n + 255) / 256), 256, 0, s>>>(coarse, fine, up, w, n_el, Pf, Pc, add);
}

void launch_restrict(const double* fine, double* coarse, const int* cptr, const int* cidx, const double* w, int n_el,
                     int Pf, int Pc, cudaStream_t s) {
  const int64_t n = (int64_t)n_el * Pc;
  if (n == 0) return;
  restrict_kernel<<<int((n + 255) / 256), 256, 0, s>>>(fine, coarse, cptr, cidx, w, n_el, Pf, Pc);
}

void launch_coarse_gs(const CoarseGSParams& p, cudaStream_t s) {
  if (p.nu <= 0 || p.n_el == 0) return;
  const int kh = (p.H + 31) / 32;
  const int np = p.max_patches_per_octant;
  switch (kh) {
    case 1: launch_gs<1>(p, s, np); break;
    case 2: launch_gs<2>(p, s, np); break;
    case 3: launch_gs<3>(p, s, np); break;
    case 4: launch_gs<4>(p, s, np); break;
    case 5: case 6: launch_gs<6>(p, s, np); break;
    case 7: case 8: launch_gs<8>(p, s, np); break;
    default: throw std::invalid_argument("coarse_scatter_sweep: harmonic count > 256 not supported on the B200 path");
  }
}

}  // namespace stamg_b200
