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

template <int KH>
__global__ void __launch_bounds__(128) coarse_gs_kernel(CoarseGSParams p) {
  const int lane = threadIdx.x & 31;
  const int n_el = p.n_el, nx = p.nx, ny = p.ny, P = p.P, Hp = p.Hp, H = p.H;
  const int per_pass = 8 * n_el;
  const int total = p.nu * per_pass;
  for (;;) {
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(p.counter, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
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
    if (lane == 0) {
      const int* d = p.done + oct * n_el;
      const int need = pass + 1;
      if (upx >= 0) while (ld_acquire(d + upx) < need) {}
      if (upy >= 0) while (ld_acquire(d + upy) < need) {}
      if (oct > 0) {
        while (ld_acquire(p.done + (oct - 1) * n_el + el) < need) {}
      } else if (pass > 0) {
        while (ld_acquire(p.done + 7 * n_el + el) < pass) {}
      }
      if (pass > 0) {
        if (dnx >= 0) while (ld_acquire(d + dnx) < pass) {}
        if (dny >= 0) while (ld_acquire(d + dny) < pass) {}
      }
    }
    __syncwarp();

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
    for (int idx = p.oct_ptr[oct]; idx < p.oct_ptr[oct + 1]; ++idx) {
      const int q = p.oct_patches[idx];
      const double* Xq = p.X + (size_t)q * Hp;
      double xq[KH];
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
      for (int kh = 0; kh < KH; ++kh) {
        const int h = lane + 32 * kh;
        xq[kh] = h < H ? Xq[h] : 0.0;
        const double xs = xq[kh] * sg[kh];
        t0 += xs * mo[kh][0], t1 += xs * mo[kh][1], t2 += xs * mo[kh][2], t3 += xs * mo[kh][3];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        t2 += __shfl_xor_sync(0xffffffffu, t2, o);
        t3 += __shfl_xor_sync(0xffffffffu, t3, o);
      }
      // cell solve (every lane redundantly, in the sweep frame)
      const double* rb = p.rhs + ((size_t)el * P + q) * 4;
      double r0 = rb[0], r1 = rb[1], r2 = rb[2], r3 = rb[3];
      double* zb = p.phi + ((size_t)el * P + q) * 4;
      double2 za = ld_cg2(zb), zc = ld_cg2(zb + 2);
      double z0 = za.x, z1 = za.y, z2 = zc.x, z3 = zc.y;
      perm(m, r0, r1, r2, r3);
      perm(m, z0, z1, z2, z3);
      perm(m, t0, t1, t2, t3);
      const double* cxy = p.cxy + (size_t)q * 8;
      if (upx >= 0) {
        const double* ub = p.phi + ((size_t)upx * P + q) * 4;
        const double2 ua = ld_cg2(ub), uc = ld_cg2(ub + 2);
        double u0 = ua.x, u1 = ua.y, u2 = uc.x, u3 = uc.y;
        perm(m, u0, u1, u2, u3);
        r0 -= cxy[0] * u1 + cxy[1] * u3;
        r2 -= cxy[2] * u1 + cxy[3] * u3;
      }
      if (upy >= 0) {
        const double* ub = p.phi + ((size_t)upy * P + q) * 4;
        const double2 ua = ld_cg2(ub), uc = ld_cg2(ub + 2);
        double u0 = ua.x, u1 = ua.y, u2 = uc.x, u3 = uc.y;
        perm(m, u0, u1, u2, u3);
        r0 -= cxy[4] * u2 + cxy[5] * u3;
        r1 -= cxy[6] * u2 + cxy[7] * u3;
      }
      // explicit scatter from every other patch: (X sig (mom - X^T zold)) N
      const double sq = p.sq[(size_t)mt * P + q];
      const double d0 = t0 - sq * z0, d1 = t1 - sq * z1, d2 = t2 - sq * z2, d3 = t3 - sq * z3;
      // N is invariant under the frame permutation (uniform square cells)
      r0 += d0 * p.N[0] + d1 * p.N[4] + d2 * p.N[8] + d3 * p.N[12];
      r1 += d0 * p.N[1] + d1 * p.N[5] + d2 * p.N[9] + d3 * p.N[13];
      r2 += d0 * p.N[2] + d1 * p.N[6] + d2 * p.N[10] + d3 * p.N[14];
      r3 += d0 * p.N[3] + d1 * p.N[7] + d2 * p.N[11] + d3 * p.N[15];
      const double* B = p.BinvGS + ((size_t)mt * P + q) * 16;
      double n0 = B[0] * r0 + B[1] * r1 + B[2] * r2 + B[3] * r3;
      double n1 = B[4] * r0 + B[5] * r1 + B[6] * r2 + B[7] * r3;
      double n2 = B[8] * r0 + B[9] * r1 + B[10] * r2 + B[11] * r3;
      double n3 = B[12] * r0 + B[13] * r1 + B[14] * r2 + B[15] * r3;
      double e0 = n0 - z0, e1 = n1 - z1, e2 = n2 - z2, e3 = n3 - z3;
      perm(m, n0, n1, n2, n3);  // back to physical (XOR permutation is an involution)
      perm(m, e0, e1, e2, e3);
#pragma unroll
      for (int kh = 0; kh < KH; ++kh)
        mo[kh][0] += xq[kh] * e0, mo[kh][1] += xq[kh] * e1, mo[kh][2] += xq[kh] * e2, mo[kh][3] += xq[kh] * e3;
      if (lane == 0) {
        st_cg2(zb, make_double2(n0, n1));
        st_cg2(zb + 2, make_double2(n2, n3));
      }
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

template <int KH>
void launch_gs(const CoarseGSParams& p, cudaStream_t s) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_gs_kernel<KH>, 128, 0);
  const long items = (long)p.nu * 8 * p.n_el;
  long blocks = (long)sms * (per_sm > 0 ? per_sm : 1);
  blocks = std::min(blocks, (items + 3) / 4);
  coarse_gs_kernel<KH><<<int(blocks), 128, 0, s>>>(p);
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
  switch (kh) {
    case 1: launch_gs<1>(p, s); break;
    case 2: launch_gs<2>(p, s); break;
    case 3: launch_gs<3>(p, s); break;
    case 4: launch_gs<4>(p, s); break;
    case 5: case 6: launch_gs<6>(p, s); break;
    case 7: case 8: launch_gs<8>(p, s); break;
    default: throw std::invalid_argument("coarse_scatter_sweep: harmonic count > 256 not supported on the B200 path");
  }
}

}  // namespace stamg_b200
