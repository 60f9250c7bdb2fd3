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
#include <cstdlib>
#include <stdexcept>
#include <string>

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

// Static-ownership variant: warp w owns a contiguous segment of `seg` cells
// of one grid row for the whole call and processes its items in the global
// (pass, octant, sweep-order) order. Cells of a segment are x-neighbours, so
// walking them in order adds nothing to the critical path, and consecutive
// octants alternate the x direction so the hand-over cell is the same. The
// previous-octant dependency is program order; the cell's own data is loaded
// before any wait. The patch chain uses K = X_q sig X_b^T (per material):
// t_a = t0_a + sum_{b<a} K[a][b] dz_b, algebraically the reference's
// running-moment update (sweeps.cpp:93-101). Needs co-residency
// (cooperative launch).
constexpr int GS_WARPS = 8;

// per-warp shared staging: moments [2][Hp][4], dz [kpad][4], K [nmat][kpad][kpad],
// X of the octant [kpad][Hp+1] (odd row stride: conflict-free both ways), sigma [nmat][Hp]
__host__ __device__ inline size_t gs_warp_doubles(int Hp, int kpad, int nmat) {
  return size_t(Hp) * 8 + size_t(kpad) * 4 + size_t(nmat) * kpad * kpad + size_t(kpad) * (Hp + 1) + size_t(nmat) * Hp;
}

template <int NS>
__global__ void __launch_bounds__(GS_WARPS * 32) coarse_gs_static_kernel(CoarseGSParams p) {
  extern __shared__ __align__(16) double gsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + wib;
  const int n_el = p.n_el, nx = p.nx, ny = p.ny, P = p.P, Hp = p.Hp, H = p.H, seg = p.cells_per_warp;
  const int kpad = p.kpad, nmat = p.n_mat;
  double* sbase = gsm + (size_t)wib * gs_warp_doubles(Hp, kpad, nmat);
  // row mode (a warp owns a whole grid row, the CTA owns wpb consecutive rows): y-traces
  // between rows of the CTA go through a shared mailbox [wpb][2 parities][nx][kpad] of
  // (dof2, dof3) in the sweep frame, published by per-warp item counters
  const bool rows = p.rows_mode != 0;
  double2* mbox = reinterpret_cast<double2*>(gsm + (size_t)wpb * gs_warp_doubles(Hp, kpad, nmat));
  volatile int* cnt = reinterpret_cast<volatile int*>(mbox + (rows ? (size_t)wpb * 2 * nx * kpad : 0));
  if (rows && lane == 0) cnt[wib] = 0;
  __syncthreads();
  // double-buffered moments [2][Hp][4] at sbase
  double* sdz = sbase + Hp * 8;               // [kpad][4]
  double* sK = sdz + kpad * 4;                // [n_mat][kpad][kpad] K of the current octant
  double* sX = sK + (size_t)nmat * kpad * kpad;  // [kpad][Hp+1] X rows of the current octant
  double* sS = sX + (size_t)kpad * (Hp + 1);     // [n_mat][Hp] sigma
  const int XS = Hp + 1;
  for (int c = lane; c < nmat * Hp; c += 32) sS[c] = p.sig[c];
  const int segs_per_row = nx / seg;
  if (gw >= segs_per_row * ny) return;
  const int gy = gw / segs_per_row, gx0 = (gw - gy * segs_per_row) * seg;
  const int n_items = p.nu * 8 * seg;
  auto cell_of = [&](int it) {
    const int oct = (it / seg) & 7, j = it % seg;
    return gy * nx + gx0 + ((oct & 1) ? seg - 1 - j : j);
  };
  auto prefetch_mom = [&](int el, double* dst) {
    const double* src = p.mom + (size_t)el * Hp * 4;
    for (int c = lane; c < H * 2; c += 32) cp_async16(dst + c * 2, src + c * 2, true);
    cp_async_commit();
  };
  int cur = 0, k_oct = -1;
  prefetch_mom(cell_of(0), sbase);
  cp_async_wait<0>();
  __syncwarp();
  double xtr[NS][2];  // x-upwind traces (frame dofs 1, 3) from the previous cell of the segment
  for (int it = 0; it < n_items; ++it) {
    const int pass = it / (8 * seg), oct = (it / seg) & 7, jseg = it % seg;
    const int el = cell_of(it);
    const int el_next = it + 1 < n_items ? cell_of(it + 1) : -1;
    const bool reuse = el_next == el;  // next item is this cell again (next octant)
    if (el_next >= 0 && !reuse) prefetch_mom(el_next, sbase + (cur ^ 1) * Hp * 4);
    const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
    const int m = (xneg ? 1 : 0) | (yneg ? 2 : 0);
    const int pbeg = p.oct_ptr[oct], np = p.oct_ptr[oct + 1] - pbeg;
    const int gx = el - gy * nx;
    const int ifr = xneg ? nx - 1 - gx : gx, jf = yneg ? ny - 1 - gy : gy;
    const int sx = xneg ? -1 : 1, sy = yneg ? -nx : nx;
    const int upx = ifr > 0 ? el - sx : -1, upy = jf > 0 ? el - sy : -1;
    const int dnx = ifr < nx - 1 ? el + sx : -1, dny = jf < ny - 1 ? el + sy : -1;
    const int mt = p.mat ? p.mat[el] : 0;
    const double* mom = sbase + cur * Hp * 4;
    if (oct != k_oct) {  // stage this octant's K blocks and X rows once per (pass, octant)
      for (int mm = 0; mm < nmat; ++mm)
        for (int c = lane; c < np * kpad / 2; c += 32)
          cp_async16(sK + ((size_t)mm * kpad * kpad) + c * 2, p.K + ((size_t)mm * P + pbeg) * kpad + c * 2, true);
      for (int c = lane; c < np * H; c += 32) {
        const int a = c / H, h = c - a * H;
        cp_async8(sX + (size_t)a * XS + h, p.Xo + (size_t)(pbeg + a) * Hp + h, true);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      k_oct = oct;
    }
    const double* sg = sS + (size_t)mt * Hp;
    // ---- own data: rhs / previous iterate -> registers (patch a = lane + 32 sl, octant order)
    double r[NS][4], zo[NS][4], t[NS][4];
    int qs[NS];
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int a = lane + 32 * sl;
      qs[sl] = a < np ? p.oct_patches[pbeg + a] : -1;
#pragma unroll
      for (int i = 0; i < 4; ++i) r[sl][i] = zo[sl][i] = t[sl][i] = 0.0;
      if (qs[sl] >= 0) {
        const double* rb = p.rhs + ((size_t)el * P + qs[sl]) * 4;
        const double2 ra = __ldg(reinterpret_cast<const double2*>(rb)), rc = __ldg(reinterpret_cast<const double2*>(rb) + 1);
        const double2 za = ld_cg2(p.phi + ((size_t)el * P + qs[sl]) * 4), zc = ld_cg2(p.phi + ((size_t)el * P + qs[sl]) * 4 + 2);
        r[sl][0] = ra.x, r[sl][1] = ra.y, r[sl][2] = rc.x, r[sl][3] = rc.y;
        zo[sl][0] = za.x, zo[sl][1] = za.y, zo[sl][2] = zc.x, zo[sl][3] = zc.y;
      }
    }
    // ---- t0_a = X_qa sig mom (off the critical path), all operands in shared memory.
    //      np <= 16: Lp = 32/np lanes per patch split the harmonics, then reduce.
    if (NS == 1 && np <= 16) {
      const int Lp = np <= 1 ? 32 : np <= 2 ? 16 : np <= 4 ? 8 : np <= 8 ? 4 : 2;
      const int a = lane / Lp, part = lane % Lp;
      double u[4] = {0.0, 0.0, 0.0, 0.0};
      if (a < np) {
        const double* xr = sX + (size_t)a * XS;
        for (int h = part; h < H; h += Lp) {
          const double xs = xr[h] * sg[h];
          const double2 ma = reinterpret_cast<const double2*>(mom)[2 * h], mb = reinterpret_cast<const double2*>(mom)[2 * h + 1];
          u[0] += xs * ma.x, u[1] += xs * ma.y, u[2] += xs * mb.x, u[3] += xs * mb.y;
        }
      }
      for (int o = Lp >> 1; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 4; ++i) u[i] += __shfl_xor_sync(full, u[i], o);
#pragma unroll
      for (int i = 0; i < 4; ++i) t[0][i] = __shfl_sync(full, u[i], (lane < np ? lane : 0) * Lp);
    } else {
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        if (qs[sl] < 0) continue;
        const double* xr = sX + (size_t)(lane + 32 * sl) * XS;
        double u[4][4] = {};
        int h = 0;
        for (; h + 3 < H; h += 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double xs = xr[h + k] * sg[h + k];
            const double2 ma = reinterpret_cast<const double2*>(mom)[2 * (h + k)];
            const double2 mb = reinterpret_cast<const double2*>(mom)[2 * (h + k) + 1];
            u[k][0] += xs * ma.x, u[k][1] += xs * ma.y, u[k][2] += xs * mb.x, u[k][3] += xs * mb.y;
          }
        }
        for (; h < H; ++h) {
          const double xs = xr[h] * sg[h];
          const double2 ma = reinterpret_cast<const double2*>(mom)[2 * h], mb = reinterpret_cast<const double2*>(mom)[2 * h + 1];
          u[0][0] += xs * ma.x, u[0][1] += xs * ma.y, u[0][2] += xs * mb.x, u[0][3] += xs * mb.y;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) t[sl][i] = (u[0][i] + u[1][i]) + (u[2][i] + u[3][i]);
      }
    }
    // ---- dependencies. x-upwind inside the segment: previous item of this warp (registers).
    //      y-upwind in row mode inside the CTA: shared mailbox. Everything else: global
    //      per-(octant, cell) counters (relaxed polling + one acquire fence).
    const bool x_in_seg = p.xreg && upx >= 0 && jseg > 0;
    const int pw = wib + (yneg ? 1 : -1), cw = wib + (yneg ? -1 : 1);
    const bool y_in_cta = rows && upy >= 0 && pw >= 0 && pw < wpb;
    const bool ydn_in_cta = rows && dny >= 0 && cw >= 0 && cw < wpb;
    const int item_id = (pass * 8 + oct) * seg + jseg;  // == global order within the row
    {
      const int* f = nullptr;
      int need = 0;
      const int* d = p.done + (size_t)oct * n_el;
      if (lane == 0 && upx >= 0 && !x_in_seg) f = d + upx, need = pass + 1;
      if (lane == 1 && upy >= 0 && !y_in_cta) f = d + upy, need = pass + 1;
      if (lane == 2 && pass > 0 && dnx >= 0 && (jseg == seg - 1 || !p.xreg)) f = d + dnx, need = pass;
      if (lane == 3 && pass > 0 && dny >= 0 && !ydn_in_cta) f = d + dny, need = pass;
      bool ok = f == nullptr || ld_relaxed(f) >= need;
      bool any = __any_sync(full, f != nullptr);
      while (!__all_sync(full, ok))
        if (!ok) ok = ld_relaxed(f) >= need;
      if (any) fence_acq_rel();
      if (y_in_cta) {  // producer row of this CTA finished the same (pass, octant, column)
        while (cnt[pw] < item_id + 1) {}
        __threadfence_block();
      }
    }
    // ---- upwind traces folded into r (sweeps.cpp:87-92), everything in the sweep frame
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int q = qs[sl];
      if (q < 0) continue;
      double ux[4] = {0, 0, 0, 0}, uy[4] = {0, 0, 0, 0};
      if (upx >= 0 && !x_in_seg) {
        const double2 a = ld_cg2(p.phi + ((size_t)upx * P + q) * 4), b = ld_cg2(p.phi + ((size_t)upx * P + q) * 4 + 2);
        ux[0] = a.x, ux[1] = a.y, ux[2] = b.x, ux[3] = b.y;
        perm(m, ux[0], ux[1], ux[2], ux[3]);
      } else if (x_in_seg) {
        ux[1] = xtr[sl][0], ux[3] = xtr[sl][1];
      }
      if (upy >= 0 && !y_in_cta) {
        const double2 a = ld_cg2(p.phi + ((size_t)upy * P + q) * 4), b = ld_cg2(p.phi + ((size_t)upy * P + q) * 4 + 2);
        uy[0] = a.x, uy[1] = a.y, uy[2] = b.x, uy[3] = b.y;
        perm(m, uy[0], uy[1], uy[2], uy[3]);
      } else if (y_in_cta) {
        const double2 v = mbox[(((size_t)pw * 2 + (oct & 1)) * nx + jseg) * kpad + lane + 32 * sl];
        uy[2] = v.x, uy[3] = v.y;
      }
      perm(m, r[sl][0], r[sl][1], r[sl][2], r[sl][3]);
      perm(m, zo[sl][0], zo[sl][1], zo[sl][2], zo[sl][3]);
      perm(m, t[sl][0], t[sl][1], t[sl][2], t[sl][3]);
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
    // ---- chain prologue (off the chain): with G = B'^-1 N and c = B'^-1 r,
    //      dz_a = e_a + G_a t_a, e_a = c_a - zo_a - sq_a G_a zo_a  (sweeps.cpp:93-101)
    cp_async_wait<0>();
    __syncwarp();
    const double* sKm = sK + (size_t)mt * kpad * kpad;
    double e[NS][4], G[NS][16];
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int q = qs[sl];
      if (q < 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) e[sl][i] = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) G[sl][k] = 0.0;
        continue;
      }
      const double* B = p.BinvGS + ((size_t)mt * P + q) * 16;
      const double* Gq = p.GS + ((size_t)mt * P + q) * 16;
#pragma unroll
      for (int k = 0; k < 16; ++k) G[sl][k] = Gq[k];
      const int a = lane + 32 * sl;
      const double sq = sKm[(size_t)a * kpad + a];
      double szo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) szo[i] = sq * zo[sl][i];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double c = B[4 * i] * r[sl][0] + B[4 * i + 1] * r[sl][1] + B[4 * i + 2] * r[sl][2] + B[4 * i + 3] * r[sl][3];
        const double gz = G[sl][4 * i] * szo[0] + G[sl][4 * i + 1] * szo[1] + G[sl][4 * i + 2] * szo[2] + G[sl][4 * i + 3] * szo[3];
        e[sl][i] = c - zo[sl][i] - gz;
      }
    }
    // ---- the sequential patch chain: one 4x4 mat-vec, a broadcast and a rank-1 update per
    //      patch. Branch-free: every lane forms the candidate from its own slot, the owner's
    //      value is broadcast; dz stays in the sweep frame (shared memory, for zo and the
    //      moment update after the chain).
    for (int a = 0; a < np; ++a) {
      const int sl = a >> 5, src = a & 31;
      double dz[4];
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2)
        if (s2 == sl)  // warp-uniform
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dz[i] = e[s2][i] + (G[s2][4 * i] * t[s2][0] + G[s2][4 * i + 1] * t[s2][1] +
                                G[s2][4 * i + 2] * t[s2][2] + G[s2][4 * i + 3] * t[s2][3]);
#pragma unroll
      for (int i = 0; i < 4; ++i) dz[i] = __shfl_sync(full, dz[i], src);
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) {
        const int b = lane + 32 * s2;
        const double k = b > a ? sKm[(size_t)a * kpad + b] : 0.0;  // K symmetric: row a, column b
#pragma unroll
        for (int i = 0; i < 4; ++i) t[s2][i] += k * dz[i];
      }
      if (lane == 0) {
        reinterpret_cast<double2*>(sdz)[2 * a] = make_double2(dz[0], dz[1]);
        reinterpret_cast<double2*>(sdz)[2 * a + 1] = make_double2(dz[2], dz[3]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int a = lane + 32 * sl;
      if (qs[sl] < 0) continue;
      const double2 d0 = reinterpret_cast<const double2*>(sdz)[2 * a], d1 = reinterpret_cast<const double2*>(sdz)[2 * a + 1];
      zo[sl][0] += d0.x, zo[sl][1] += d0.y, zo[sl][2] += d1.x, zo[sl][3] += d1.y;
    }
    // ---- publish the new iterate of this cell's patches, then the flags
    if (ydn_in_cta && pass * 8 + oct >= 2) {  // mailbox slot reuse: the consumer row is past it
      const int need2 = (pass * 8 + oct - 2) * seg + jseg + 1;
      while (cnt[cw] < need2) {}
    }
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int q = qs[sl];
      xtr[sl][0] = zo[sl][1], xtr[sl][1] = zo[sl][3];  // frame x-outflow traces for the next cell
      if (q < 0) continue;
      if (rows) mbox[(((size_t)wib * 2 + (oct & 1)) * nx + jseg) * kpad + lane + 32 * sl] = make_double2(zo[sl][2], zo[sl][3]);
      perm(m, zo[sl][0], zo[sl][1], zo[sl][2], zo[sl][3]);
      double* zb = p.phi + ((size_t)el * P + q) * 4;
      st_cg2(zb, make_double2(zo[sl][0], zo[sl][1]));
      st_cg2(zb + 2, make_double2(zo[sl][2], zo[sl][3]));
    }
    __syncwarp();
    if (rows && lane == 0) {
      __threadfence_block();
      cnt[wib] = item_id + 1;
    }
    // global counter only where another warp reads or waits on this cell
    const bool need_flag = !p.xreg || (dnx >= 0 && jseg == seg - 1) || (upx >= 0 && jseg == 0) ||
                           (dny >= 0 && !ydn_in_cta) || (upy >= 0 && !y_in_cta);
    if (need_flag && lane == 0) st_release(p.done + (size_t)oct * n_el + el, pass + 1);
    // ---- running moments: mom += sum_a X_qa^T dz_a; Xo is [P][Hp] in octant order
    double* mom_el = p.mom + (size_t)el * Hp * 4;
    double* mw = const_cast<double*>(mom);
    for (int h = lane; h < H; h += 32) {
      // view the physical moments [i] in the sweep frame (index i ^ m) so frame dz applies directly
      double2 a0 = reinterpret_cast<const double2*>(mom)[2 * h], a1 = reinterpret_cast<const double2*>(mom)[2 * h + 1];
      if (m & 2) { const double2 u = a0; a0 = a1; a1 = u; }
      if (m & 1) { double u = a0.x; a0.x = a0.y; a0.y = u; u = a1.x; a1.x = a1.y; a1.y = u; }
      const double* xo = sX + h;
      int a = 0;
      for (; a + 3 < np; a += 4) {
        double x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = xo[(size_t)(a + k) * XS];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 d0 = reinterpret_cast<const double2*>(sdz)[2 * (a + k)];
          const double2 d1 = reinterpret_cast<const double2*>(sdz)[2 * (a + k) + 1];
          a0.x += x[k] * d0.x, a0.y += x[k] * d0.y, a1.x += x[k] * d1.x, a1.y += x[k] * d1.y;
        }
      }
      for (; a < np; ++a) {
        const double x = xo[(size_t)a * XS];
        const double2 d0 = reinterpret_cast<const double2*>(sdz)[2 * a], d1 = reinterpret_cast<const double2*>(sdz)[2 * a + 1];
        a0.x += x * d0.x, a0.y += x * d0.y, a1.x += x * d1.x, a1.y += x * d1.y;
      }
      if (m & 1) { double u = a0.x; a0.x = a0.y; a0.y = u; u = a1.x; a1.x = a1.y; a1.y = u; }
      if (m & 2) { const double2 u = a0; a0 = a1; a1 = u; }
      st_cg2(mom_el + h * 4, a0);
      st_cg2(mom_el + h * 4 + 2, a1);
      if (reuse) {
        reinterpret_cast<double2*>(mw)[2 * h] = a0;
        reinterpret_cast<double2*>(mw)[2 * h + 1] = a1;
      }
    }
    if (!reuse) cur ^= 1;
    cp_async_wait<0>();
    __syncwarp();
  }
}

// Multi-warp rows (many patches per octant: config 4 has 64). The one-warp item
// is throughput-bound there (~12.7k warp instructions: the projections t0 and the
// running-moment update are np x H x 4 each). Here a CTA of GSW_MW warps owns one
// grid row for the whole call and walks the same item sequence, software-pipelined:
// in iteration k
//   warp 0      : item k - dependency wait, upwind fold, prologue, the sequential
//                 patch chain (t0 from shared memory), publish;
//   warps 1..3  : item k-1's running-moment update mom[h][i] += sum_a X_a[h] dz_a[i]
//                 (patches in the reference's order), then item k+1's projections
//                 t0_a = X_a sig mom, then the moment prefetch of item k+2.
// At an octant boundary the next item is the same cell (its moments need item k's
// update) and the octant's K / X tables change: the pipeline drains there (every
// nx items). Moments use a 4-buffer ring (items k-1 .. k+2), t0 and dz two buffers.
// Co-residency of the ny CTAs is required (cooperative launch).
#ifndef STAMG_GSW_MW
#define STAMG_GSW_MW 4  // warps of a row-CTA: the item warp + helpers (A/B: 2 / 3 / 4 warps all give ~2.0 us per item)
#endif
constexpr int GSW_MW = STAMG_GSW_MW;

constexpr int MW_BAR = 1;  // named barrier of warps 1..3

__host__ __device__ inline int gs_mw_xs(int H) { return (H % 2 == 0) ? H + 1 : H + 2; }  // odd X row stride
// Blocked chain: the chain's K region holds, per material, the K columns right of each 4-patch
// diagonal block (rows 4J..4J+3 from column 4(J+1): kpad^2/2 - 2 kpad doubles), the diagonal
// sq_a = K[a][a], and the packed inverses of the diagonal blocks (kGsMinvBlock doubles per
// block: column c of the 16 x 16 unit lower block-triangular inverse from row 4 (c / 4));
// then 16 doubles for the block's right-hand side.
__host__ __device__ inline int gs_koff(int J, int kpad) { return 4 * J * kpad - 8 * J * (J + 1); }
__host__ __device__ inline size_t gs_blk_mat_doubles(int kpad) {
  return size_t(gs_koff(kpad / 4, kpad)) + kpad + size_t(kpad / 4) * kGsMinvBlock;
}
__host__ __device__ inline size_t gs_mw_kregion(int kpad, int nmat, bool blk) {
  return blk ? size_t(nmat) * gs_blk_mat_doubles(kpad) + 16 : size_t(nmat) * kpad * kpad;
}
__host__ __device__ inline size_t gs_mw_doubles(int Hp, int H, int kpad, int nmat, int hs, bool blk) {
  return size_t(hs > 0 ? hs : Hp) * 16 + size_t(kpad) * 32 + gs_mw_kregion(kpad, nmat, blk) + size_t(kpad) * gs_mw_xs(H) +
         size_t(nmat) * Hp + 8;  // + oct_ptr
}

__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
constexpr int MAIN_BAR = 2;  // named barrier of the GSW_MW item warps (the publisher warp stays out)

// Cluster mode (CL): the ny row-CTAs form clusters of p.cluster consecutive rows. Inside a
// cluster the y-upwind traces (2 doubles per patch, sweep frame) are pushed into the
// consumer row's shared-memory mailbox with st.async (distributed shared memory), each
// slot completing an mbarrier transaction: a y-hop costs one DSMEM write instead of a
// global store + release fence + flag poll + acquire + L2 reload. Mailbox slot of item
// (pass, oct, j): direction yneg, slot (oct & 1) * nx + j, use 2 * pass + (oct >= 4). A
// row never runs more than one octant pair ahead of its y-downwind neighbour (the next
// pair runs the other y-direction, which waits on that neighbour), so 2 nx slots per
// direction never overrun and need no credits. Rows at a cluster edge exchange with
// the neighbouring cluster through global memory as before; their done flags are
// published by a fifth warp (fence + flag stores), off the item warp's chain.
__host__ __device__ inline size_t gs_mw_cl_doubles(int nslots, int mbnp) {
  return size_t(4) * nslots * mbnp + size_t(2) * nslots + 2;  // mailbox [2][nslots][mbnp][2], mbarriers [2][nslots], s_pub + credits
}
// octant of the n-th item of y-direction d (0: +y octants 0,1,4,5; 1: -y octants 2,3,6,7) of a row
__host__ __device__ inline int gs_cls_oct(int n, int d, int nx) {
  const int pi = n / (2 * nx), r = n - pi * 2 * nx;
  return (pi & 1) * 4 + d * 2 + (r >= nx ? 1 : 0);
}
__device__ __forceinline__ unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned bar, unsigned bytes) {  // this CTA's arrival + expected bytes
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n}" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_done(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ unsigned cluster_map(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async2(unsigned raddr, double a, double b, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr), "d"(a),
               "d"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_release_cta_smem(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta_smem(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cluster_remote(unsigned raddr, int v) {
  asm volatile("st.release.cluster.shared::cluster.s32 [%0], %1;" ::"r"(raddr), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cluster_smem(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// PUBW: a fifth warp publishes the edge rows' done flags (one-slot kernel); the 64-patch
// kernel (NS = 2) needs all 255 registers of a 128-thread CTA, so helper warp 3 publishes
// the previous item's flag at the top of each iteration instead (the helpers have slack there)
template <int NS, bool CL>
constexpr bool gs_pubw() { return CL && NS == 1; }
// BLK: the patch chain in blocks of four patches. With f_a = e_a + G_a t_a the chain solves
// (I - blockdiag(G_a) (L_K x I_4)) dz = f, L_K the strictly lower part of K: unit lower
// block-triangular, and a function of (octant, material) only, never of the cell. The host
// inverts its 16 x 16 diagonal blocks once (gs_minv_table); per block the warp forms f for
// the block's patches, applies the inverse (one row per lane, four independent FMA chains) and
// adds the block's dz into the t of the patches to its right (4 x 4 FMAs per lane and slot):
// np / 4 dependent steps instead of np. Results differ from the patch-by-patch chain at the
// rounding level (the inverse is formed in extended precision).
template <int NS, bool CL = false, bool RING = false, bool BLK = true>
__global__ void __launch_bounds__(GSW_MW * 32 + (gs_pubw<NS, CL>() ? 32 : 0), 2) coarse_gs_mw_kernel(CoarseGSParams p) {
  constexpr bool PUBW = gs_pubw<NS, CL>();
  extern __shared__ __align__(16) double gsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = GSW_MW * 32;
  const unsigned full = 0xffffffffu;
  const int n_el = p.n_el, nx = p.nx, ny = p.ny, P = p.P, Hp = p.Hp, H = p.H;
  const int kpad = p.kpad, nmat = p.n_mat;
  double* smom = gsm;                             // [4][Hp][4] moments of items k-1 .. k+2 (ring)
  const int HS = p.mom_stride > 0 ? p.mom_stride : Hp;  // moment ring stride (Hp; H rounded up to even for rings)
  double* sdz = smom + HS * 16;                   // [2][kpad][4] chain outputs (sweep frame)
  double* st0 = sdz + kpad * 8;                   // [2][kpad][4] projections (physical dofs)
  double* srz = st0 + kpad * 8;                   // [2][kpad][8] warp 0: rhs | iterate of the next item
  double* sK = srz + kpad * 16;                   // [n_mat][kpad][kpad]; BLK: [n_mat](Koff | sq | Minv), f[16]
  double* sX = sK + gs_mw_kregion(kpad, nmat, BLK);  // [kpad][Hp+1]
  const int XS = gs_mw_xs(H);
  const int matd = int(gs_blk_mat_doubles(kpad));           // BLK: doubles per material
  const int sq_off = gs_koff(kpad / 4, kpad), minv_off = sq_off + kpad;
  double* sF = sK + (size_t)nmat * matd;                    // BLK: right-hand side of the current block
  double* sS = sX + (size_t)kpad * XS;            // [n_mat][Hp]
  if (tid < nthr)
    for (int c = tid; c < nmat * Hp; c += nthr) sS[c] = p.sig[c];
  const int gy = blockIdx.x;
  const int seg = nx;
  const int n_items = p.nu * 8 * seg;
  // item descriptors advanced incrementally (no integer division per item)
  struct Item {
    int it, pass, oct, j, el;
  };
  int* sOptr = reinterpret_cast<int*>(sS + (size_t)nmat * Hp);  // oct_ptr[0..8] in shared memory
  // cluster mode: mailbox, its mbarriers and the publish counter after the tables
  const int CS = CL ? p.cluster : 1, crank = CL ? int(cluster_rank()) : 0, mbnp = p.mb_np;
  const int NSL = p.mb_slots;  // mailbox slots per direction: 2 nx (no credits) or a power of two (credits)
  constexpr bool credit = RING;  // mailbox ring with credits (p.mb_credit)
  double* sMail = sS + (size_t)nmat * Hp + 8;                                     // [2][NSL][mbnp][2]
  unsigned long long* sBar = reinterpret_cast<unsigned long long*>(sMail + (size_t)4 * NSL * mbnp);  // [2][NSL]
  int* sPub = reinterpret_cast<int*>(sBar + 2 * NSL);
  int* sCred = sPub + 1;  // [2] items of each direction the downwind row has consumed (written remotely)
  // a row at a cluster edge with a y-neighbour in the next cluster publishes global done flags
  const bool edge_pub = CL && ((crank == 0 && gy > 0) || (crank == CS - 1 && gy < ny - 1));
  if constexpr (CL) {
    if (warp == 0) {
      for (int b = lane; b < 2 * NSL; b += 32) mbar_init(smem_addr(sBar + b), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      __syncwarp();
      for (int b = lane; b < 2 * NSL; b += 32) {  // first use of slot b: the direction's item b
        const int dir = b / NSL, o = gs_cls_oct(b - dir * NSL, dir, nx);
        mbar_arm(smem_addr(sBar + b), 16u * unsigned(p.oct_ptr[o + 1] - p.oct_ptr[o]));
      }
      if (lane == 0) *sPub = 0, sCred[0] = 0, sCred[1] = 0;
    }
    cluster_sync_all();
    if (PUBW && warp == GSW_MW) {  // publisher: done flags of this edge row, fenced in batches
      if (edge_pub && lane == 0) {
        int pass = 0, oct = 0, j = 0;
        for (int done_items = 0; done_items < p.nu * 8 * nx;) {
          const int avail = ld_acquire_cta_smem(sPub);
          if (avail == done_items) {  // shares an issue slot with warp 0: poll gently
            __nanosleep(32);
            continue;
          }
          fence_acq_rel();
          for (; done_items < avail; ++done_items) {
            const int el = gy * nx + ((oct & 1) ? nx - 1 - j : j);
            st_relaxed(p.done + (size_t)oct * n_el + el, pass + 1);
            if (++j == nx) {
              j = 0;
              if (++oct == 8) oct = 0, ++pass;
            }
          }
        }
      }
    }
  }
  if (!PUBW || warp < GSW_MW) {
  if (tid < 9) sOptr[tid] = p.oct_ptr[tid];
  auto cell = [&](int oct, int j) { return gy * nx + ((oct & 1) ? seg - 1 - j : j); };
  auto advance = [&](const Item& c) {
    Item n = c;
    n.it += 1, n.j += 1;
    if (n.j == seg) {
      n.j = 0, n.oct += 1;
      if (n.oct == 8) n.oct = 0, n.pass += 1;
    }
    n.el = cell(n.oct, n.j);
    return n;
  };
  auto mbuf = [&](int it) { return smom + (it & 3) * HS * 4; };
  // moments of item c -> its ring buffer (threads [t0, t0 + nt))
  auto prefetch_mom = [&](const Item& c, int t0, int nt) {
    const double* src = p.mom + (size_t)c.el * Hp * 4;
    double* dst = mbuf(c.it);
    for (int q = tid - t0; q < H * 2; q += nt) cp_async16(dst + q * 2, src + q * 2, true);
    cp_async_commit();
  };
  auto stage_octant = [&](int oct) {  // all threads; caller synchronises
    const int pbeg = p.oct_ptr[oct], np = p.oct_ptr[oct + 1] - pbeg;
    if constexpr (BLK) {
      const int hk = kpad >> 1, nb = (np + 3) >> 2;
      for (int mm = 0; mm < nmat; ++mm) {
        double* dm = sK + (size_t)mm * matd;
        const double* Km = p.K + ((size_t)mm * P + pbeg) * kpad;
        for (int c = tid; c < np * hk; c += nthr) {  // row a of K from the column after its block
          const int a = c / hk, col = (c - a * hk) * 2, J = a >> 2, c0 = 4 * (J + 1);
          if (col >= c0) cp_async16(dm + gs_koff(J, kpad) + (a & 3) * (kpad - c0) + (col - c0), Km + (size_t)a * kpad + col, true);
        }
        for (int a = tid; a < np; a += nthr) cp_async8(dm + sq_off + a, Km + (size_t)a * kpad + a, true);
        const double* Mi = p.Minv + ((size_t)mm * 8 + oct) * (kpad >> 2) * kGsMinvBlock;
        for (int c = tid; c < nb * (kGsMinvBlock / 2); c += nthr) cp_async16(dm + minv_off + c * 2, Mi + c * 2, true);
      }
    } else {
      for (int mm = 0; mm < nmat; ++mm)
        for (int c = tid; c < np * kpad / 2; c += nthr)
          cp_async16(sK + ((size_t)mm * kpad * kpad) + c * 2, p.K + ((size_t)mm * P + pbeg) * kpad + c * 2, true);
    }
    for (int c = tid; c < np * H; c += nthr) {
      const int a = c / H, h = c - a * H;
      cp_async8(sX + (size_t)a * XS + h, p.Xo + (size_t)(pbeg + a) * Hp + h, true);
    }
    cp_async_commit();
  };
  // t0 of item c by threads [t0, t0 + nt): Lp = largest power of two <= 32 with Lp * np <= nt
  auto project = [&](const Item& c, int t0, int nt) {
    const int np = sOptr[c.oct + 1] - sOptr[c.oct];
    const double* sg = sS + (size_t)(p.mat ? p.mat[c.el] : 0) * Hp;
    const double* mom = mbuf(c.it);
    double* out = st0 + (c.it & 1) * kpad * 4;
    const int Lp = min(32, 1 << (31 - __clz(max(1, nt / np))));
    const int lt = tid - t0, a = lt / Lp, part = lt & (Lp - 1);
    double u[4] = {0.0, 0.0, 0.0, 0.0};
    if (a < np) {
      const double* xr = sX + (size_t)a * XS;
      for (int h = part; h < H; h += Lp) {
        const double xs = xr[h] * sg[h];
        const double2 ma = reinterpret_cast<const double2*>(mom)[2 * h], mb = reinterpret_cast<const double2*>(mom)[2 * h + 1];
        u[0] += xs * ma.x, u[1] += xs * ma.y, u[2] += xs * mb.x, u[3] += xs * mb.y;
      }
    }
    for (int o = Lp >> 1; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] += __shfl_xor_sync(full, u[i], o);
    if (a < np && part == 0) {
      reinterpret_cast<double2*>(out)[2 * a] = make_double2(u[0], u[1]);
      reinterpret_cast<double2*>(out)[2 * a + 1] = make_double2(u[2], u[3]);
    }
  };
  // running moments of item c (threads [t0, t0 + nt)); with into_next also the ring buffer of item c.it+1
  auto update = [&](const Item& c, int t0, int nt, bool into_next) {
    const int np = sOptr[c.oct + 1] - sOptr[c.oct];
    const int m = (c.oct & 1) | (c.oct & 2);
    double* mom_el = p.mom + (size_t)c.el * Hp * 4;
    const double* mom = mbuf(c.it);
    double* nxt = mbuf(c.it + 1);
    const double* dz = sdz + (c.it & 1) * kpad * 4;
    for (int o = tid - t0; o < H * 4; o += nt) {
      const int h = o >> 2, fi = (o & 3) ^ m;  // physical dof i = frame dof i ^ m
      double v = mom[o];
      const double* xo = sX + h;
      for (int a = 0; a < np; ++a) v += xo[(size_t)a * XS] * dz[a * 4 + fi];
      mom_el[o] = v;
      if (into_next) nxt[o] = v;
    }
  };

  // ---- prologue: octant of item 0, moments of items 0 and 1, t0 of item 0
  Item prv{-1, 0, 0, 0, 0}, cur{0, 0, 0, 0, cell(0, 0)};
  Item n1 = advance(cur), n2 = advance(n1);
  stage_octant(0);
  bar_named(MAIN_BAR, nthr);  // sOptr
  if (warp > 0) {
    prefetch_mom(cur, 32, nthr - 32);
    if (n_items > 1 && n1.el != cur.el) prefetch_mom(n1, 32, nthr - 32);
  }
  cp_async_wait<0>();
  bar_named(MAIN_BAR, nthr);
  project(cur, 0, nthr);
  bar_named(MAIN_BAR, nthr);
  bool drained = true;  // item k-1's update already done (octant boundary drain)
  double xtr[NS][2];    // warp 0: x-upwind traces from the previous cell of the row
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) xtr[sl][0] = xtr[sl][1] = 0.0;
  int g_oct = -1, g_mt = -1;  // warp 0: octant / material of the cached G, B'^-1
  bool rz_next = false;       // warp 0: the next item's rhs / iterate are in srz
  double G[NS][16], Bq[NS][16];
  int qs[NS];
  for (int it = 0; it < n_items; ++it) {
    const int pass = cur.pass, oct = cur.oct, jseg = cur.j;
    const int el = cur.el;
    const bool boundary = it + 1 < n_items && n1.oct != oct;  // next item: same cell, new octant
    const int pbeg = sOptr[oct], np = sOptr[oct + 1] - pbeg;
    if (warp == 0) {
      // ---------------- item `it`: dependencies, upwind fold, chain, publish
      const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
      const int m = (xneg ? 1 : 0) | (yneg ? 2 : 0);
      const int gx = el - gy * nx;
      const int ifr = xneg ? nx - 1 - gx : gx, jf = yneg ? ny - 1 - gy : gy;
      const int sx = xneg ? -1 : 1, sy = yneg ? -nx : nx;
      const int upx = ifr > 0 ? el - sx : -1, upy = jf > 0 ? el - sy : -1;
      const int dnx = ifr < nx - 1 ? el + sx : -1, dny = jf < ny - 1 ? el + sy : -1;
      const int mt = p.mat ? p.mat[el] : 0;
      double r[NS][4], zo[NS][4], t[NS][4];
      const bool reload = oct != g_oct || mt != g_mt;
      const bool rz_pf = rz_next;
      if (rz_pf) {
        cp_async_wait<0>();
        __syncwarp();
      }
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        const int a = lane + 32 * sl;
        if (reload) qs[sl] = a < np ? p.oct_patches[pbeg + a] : -1;
#pragma unroll
        for (int i = 0; i < 4; ++i) r[sl][i] = zo[sl][i] = 0.0;
        if (qs[sl] >= 0) {
          if (rz_pf) {  // prefetched by the previous item (same octant)
            const double2* d = reinterpret_cast<const double2*>(srz + ((it & 1) * kpad + a) * 8);
            const double2 ra = d[0], rc = d[1], za = d[2], zc = d[3];
            r[sl][0] = ra.x, r[sl][1] = ra.y, r[sl][2] = rc.x, r[sl][3] = rc.y;
            zo[sl][0] = za.x, zo[sl][1] = za.y, zo[sl][2] = zc.x, zo[sl][3] = zc.y;
          } else {
            const double* rb = p.rhs + ((size_t)el * P + qs[sl]) * 4;
            const double2 ra = __ldg(reinterpret_cast<const double2*>(rb)), rc = __ldg(reinterpret_cast<const double2*>(rb) + 1);
            const double2 za = ld_cg2(p.phi + ((size_t)el * P + qs[sl]) * 4), zc = ld_cg2(p.phi + ((size_t)el * P + qs[sl]) * 4 + 2);
            r[sl][0] = ra.x, r[sl][1] = ra.y, r[sl][2] = rc.x, r[sl][3] = rc.y;
            zo[sl][0] = za.x, zo[sl][1] = za.y, zo[sl][2] = zc.x, zo[sl][3] = zc.y;
          }
          if (reload) {
            const double* Gq = p.GS + ((size_t)mt * P + qs[sl]) * 16;
            const double* Bg = p.BinvGS + ((size_t)mt * P + qs[sl]) * 16;
#pragma unroll
            for (int k = 0; k < 16; ++k) G[sl][k] = __ldg(Gq + k), Bq[sl][k] = __ldg(Bg + k);
          }
        } else if (reload) {
#pragma unroll
          for (int k = 0; k < 16; ++k) G[sl][k] = Bq[sl][k] = 0.0;
        }
        const double* t0b = st0 + (it & 1) * kpad * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) t[sl][i] = a < np ? t0b[a * 4 + i] : 0.0;
      }
      g_oct = oct, g_mt = mt;
      const bool x_in_seg = upx >= 0 && jseg > 0;
      // cluster mode: y-neighbours inside the cluster exchange through the mailbox
      const bool up_mail = CL && upy >= 0 && (yneg ? crank < CS - 1 : crank > 0);
      const bool dn_mail = CL && dny >= 0 && (yneg ? crank > 0 : crank < CS - 1);
      // the item's index among this row's items of its y-direction, its slot and slot use
      // (2 nx slots: slot (oct & 1) nx + j, use 2 pass + (oct >= 4); a ring: ncls mod / div NSL)
      int mslot = 0, muse = 0, ncls = 0;
      if constexpr (CL) {
        if (credit) {
          ncls = ((pass * 2 + (oct >= 4 ? 1 : 0)) * 2 + (oct & 1)) * nx + jseg;
          mslot = yneg * NSL + (ncls & (NSL - 1)), muse = ncls >> (31 - __clz(NSL));
        } else {
          mslot = yneg * NSL + (oct & 1) * nx + jseg, muse = pass * 2 + (oct >= 4 ? 1 : 0);
        }
      }
      {
        const int* f = nullptr;
        int need = 0;
        const int* d = p.done + (size_t)oct * n_el;
        if (lane == 0 && upx >= 0 && !x_in_seg) f = d + upx, need = pass + 1;
        if (lane == 1 && upy >= 0 && !up_mail) f = d + upy, need = pass + 1;
        if (lane == 2 && pass > 0 && dnx >= 0 && jseg == seg - 1) f = d + dnx, need = pass;
        if (lane == 3 && pass > 0 && dny >= 0 && !dn_mail) f = d + dny, need = pass;
        bool ok = f == nullptr || ld_relaxed(f) >= need;
        const bool any = __any_sync(full, f != nullptr);
        while (!__all_sync(full, ok))
          if (!ok) ok = ld_relaxed(f) >= need;
        if (any) fence_acq_rel();
        if constexpr (CL) {
          if (up_mail) {
            const unsigned bar = smem_addr(sBar + mslot);
            while (!mbar_done(bar, unsigned(muse) & 1u)) {
            }
            __syncwarp();
            if (lane == 0) {  // arm the slot's next use: this direction's item ncls + NSL
              int o2 = oct ^ 4;   // 2 nx slots: the same column of the next octant pair
              if (credit) {       // ring (NSL < 2 nx): NSL items further in this direction
                int r = (oct & 1) * nx + jseg + NSL;
                const int wrap = r >= 2 * nx ? 1 : 0;
                r -= wrap * 2 * nx;
                o2 = (((oct >= 4 ? 1 : 0) ^ wrap) * 4) + yneg * 2 + (r >= nx ? 1 : 0);
              }
              mbar_arm(bar, 16u * unsigned(sOptr[o2 + 1] - sOptr[o2]));
            }
          }
        }
      }
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        const int q = qs[sl];
        if (q < 0) continue;
        double ux[4] = {0, 0, 0, 0}, uy[4] = {0, 0, 0, 0};
        if (upx >= 0 && !x_in_seg) {
          const double2 a = ld_cg2(p.phi + ((size_t)upx * P + q) * 4), b = ld_cg2(p.phi + ((size_t)upx * P + q) * 4 + 2);
          ux[0] = a.x, ux[1] = a.y, ux[2] = b.x, ux[3] = b.y;
          perm(m, ux[0], ux[1], ux[2], ux[3]);
        } else if (x_in_seg) {
          ux[1] = xtr[sl][0], ux[3] = xtr[sl][1];
        }
        if (up_mail) {  // frame traces pushed by the upwind row
          const double2 v = reinterpret_cast<const double2*>(sMail)[(size_t)mslot * mbnp + lane + 32 * sl];
          uy[2] = v.x, uy[3] = v.y;
        } else if (upy >= 0) {
          const double2 a = ld_cg2(p.phi + ((size_t)upy * P + q) * 4), b = ld_cg2(p.phi + ((size_t)upy * P + q) * 4 + 2);
          uy[0] = a.x, uy[1] = a.y, uy[2] = b.x, uy[3] = b.y;
          perm(m, uy[0], uy[1], uy[2], uy[3]);
        }
        perm(m, r[sl][0], r[sl][1], r[sl][2], r[sl][3]);
        perm(m, zo[sl][0], zo[sl][1], zo[sl][2], zo[sl][3]);
        perm(m, t[sl][0], t[sl][1], t[sl][2], t[sl][3]);
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
      const double* sKm = sK + (size_t)mt * (BLK ? matd : kpad * kpad);
      double e[NS][4];
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        if (qs[sl] < 0) {
#pragma unroll
          for (int i = 0; i < 4; ++i) e[sl][i] = 0.0;
          continue;
        }
        const int a = lane + 32 * sl;
        const double sq = BLK ? sKm[sq_off + a] : sKm[(size_t)a * kpad + a];
        double szo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) szo[i] = sq * zo[sl][i];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double c = Bq[sl][4 * i] * r[sl][0] + Bq[sl][4 * i + 1] * r[sl][1] + Bq[sl][4 * i + 2] * r[sl][2] +
                           Bq[sl][4 * i + 3] * r[sl][3];
          const double gz = G[sl][4 * i] * szo[0] + G[sl][4 * i + 1] * szo[1] + G[sl][4 * i + 2] * szo[2] +
                            G[sl][4 * i + 3] * szo[3];
          e[sl][i] = c - zo[sl][i] - gz;
        }
      }
      if constexpr (CL) {
        if (up_mail && credit) {  // slot data read (in registers): hand the slot back to the upwind row
          __syncwarp();
          if (lane == 0)
            st_release_cluster_remote(cluster_map(smem_addr(sCred + yneg), unsigned(yneg ? crank + 1 : crank - 1)),
                                      ncls + 1);
        }
      }
      double* dzb = sdz + (it & 1) * kpad * 4;
      if constexpr (BLK) {
        const int nblk = (np + 3) >> 2, row = lane & 15;
        const double* sMi = sKm + minv_off;
        for (int J = 0; J < nblk; ++J) {
          const int sl = J >> 3, l0 = (4 * J) & 31;
          // f of the block's four patches (every lane forms its own slot's candidate)
          double fb[4];
#pragma unroll
          for (int s2 = 0; s2 < NS; ++s2)
            if (s2 == sl)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                fb[i] = e[s2][i] + (G[s2][4 * i] * t[s2][0] + G[s2][4 * i + 1] * t[s2][1] +
                                    G[s2][4 * i + 2] * t[s2][2] + G[s2][4 * i + 3] * t[s2][3]);
          if (unsigned(lane - l0) < 4u) {
            reinterpret_cast<double2*>(sF)[2 * (lane - l0)] = make_double2(fb[0], fb[1]);
            reinterpret_cast<double2*>(sF)[2 * (lane - l0) + 1] = make_double2(fb[2], fb[3]);
          }
          __syncwarp();
          // dz = Minv f: lane = row (lanes 16..31 mirror), column c stored from row 4 (c / 4)
          {
            const double* M = sMi + J * kGsMinvBlock;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
              const double2 fa = reinterpret_cast<const double2*>(sF)[2 * cb], fc = reinterpret_cast<const double2*>(sF)[2 * cb + 1];
              const int len = 16 - 4 * cb, idx = row - 4 * cb, base = 64 * cb - 8 * cb * (cb - 1);
              if (idx >= 0) {
                const double* mc = M + base + idx;
                a0 += mc[0] * fa.x, a1 += mc[len] * fa.y, a2 += mc[2 * len] * fc.x, a3 += mc[3 * len] * fc.y;
              }
            }
            if (lane < 16) dzb[16 * J + lane] = (a0 + a1) + (a2 + a3);
          }
          __syncwarp();
          // t of the patches right of the block
          const int c0 = 4 * (J + 1), Lj = kpad - c0, na = min(4, np - 4 * J);
          if (c0 < np) {
            const double* Kb = sKm + gs_koff(J, kpad);
            double2 d[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) d[k] = reinterpret_cast<const double2*>(dzb + 16 * J)[k];
#pragma unroll
            for (int s2 = 0; s2 < NS; ++s2) {
              const int b = lane + 32 * s2;
              if (32 * s2 + 31 < c0) continue;  // warp-uniform: the whole slot is left of the block's end
              if (b >= c0) {
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                  if (a < na) {
                    const double k = Kb[a * Lj + (b - c0)];
                    t[s2][0] += k * d[2 * a].x, t[s2][1] += k * d[2 * a].y;
                    t[s2][2] += k * d[2 * a + 1].x, t[s2][3] += k * d[2 * a + 1].y;
                  }
                }
              }
            }
          }
        }
      } else {
      for (int a = 0; a < np; ++a) {
        const int sl = a >> 5, src = a & 31;
        double dz[4];
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2)
          if (s2 == sl)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dz[i] = e[s2][i] + (G[s2][4 * i] * t[s2][0] + G[s2][4 * i + 1] * t[s2][1] +
                                  G[s2][4 * i + 2] * t[s2][2] + G[s2][4 * i + 3] * t[s2][3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) dz[i] = __shfl_sync(full, dz[i], src);
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          const int b = lane + 32 * s2;
          const double k = b > a ? sKm[(size_t)a * kpad + b] : 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i) t[s2][i] += k * dz[i];
        }
        if (lane == 0) {
          reinterpret_cast<double2*>(dzb)[2 * a] = make_double2(dz[0], dz[1]);
          reinterpret_cast<double2*>(dzb)[2 * a + 1] = make_double2(dz[2], dz[3]);
        }
      }
      }
      __syncwarp();
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        const int a = lane + 32 * sl;
        if (qs[sl] < 0) continue;
        const double2 d0 = reinterpret_cast<const double2*>(dzb)[2 * a], d1 = reinterpret_cast<const double2*>(dzb)[2 * a + 1];
        zo[sl][0] += d0.x, zo[sl][1] += d0.y, zo[sl][2] += d1.x, zo[sl][3] += d1.y;
      }
      if constexpr (CL) {
        if (dn_mail) {  // push the top traces into the downwind row's mailbox
          const unsigned rk = unsigned(yneg ? crank - 1 : crank + 1);
          if (credit && ncls >= NSL)  // the slot's previous use must have been read
            while (ld_acquire_cluster_smem(sCred + yneg) < ncls - NSL + 1) {
            }
          const unsigned rbar = cluster_map(smem_addr(sBar + mslot), rk);
#pragma unroll
          for (int sl = 0; sl < NS; ++sl) {
            if (qs[sl] < 0) continue;
            const unsigned dst = cluster_map(smem_addr(sMail + ((size_t)mslot * mbnp + lane + 32 * sl) * 2), rk);
            st_async2(dst, zo[sl][2], zo[sl][3], rbar);
          }
        }
      }
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        const int q = qs[sl];
        xtr[sl][0] = zo[sl][1], xtr[sl][1] = zo[sl][3];
        if (q < 0) continue;
        perm(m, zo[sl][0], zo[sl][1], zo[sl][2], zo[sl][3]);
        double* zb = p.phi + ((size_t)el * P + q) * 4;
        st_cg2(zb, make_double2(zo[sl][0], zo[sl][1]));
        st_cg2(zb + 2, make_double2(zo[sl][2], zo[sl][3]));
      }
      __syncwarp();
      if constexpr (PUBW) {
        if (edge_pub && lane == 0) st_release_cta_smem(sPub, it + 1);  // the publisher warp fences and flags
      } else if constexpr (CL) {
        // helper warp 3 publishes this item's flag at the top of the next iteration
      } else {
        if (lane == 0) st_release(p.done + (size_t)oct * n_el + el, pass + 1);
      }
      // rhs / previous iterate of the next item of this octant (its iterate was written by
      // this warp one octant sweep ago): hidden behind the barrier and the next wait
      rz_next = it + 1 < n_items && !boundary;
      if (rz_next) {
        const size_t eln = (size_t)n1.el * P;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          if (qs[sl] < 0) continue;
          double* d = srz + (((it + 1) & 1) * kpad + lane + 32 * sl) * 8;
          const size_t off = (eln + qs[sl]) * 4;
          cp_async16(d, p.rhs + off, true), cp_async16(d + 2, p.rhs + off + 2, true);
          cp_async16(d + 4, p.phi + off, true), cp_async16(d + 6, p.phi + off + 2, true);
        }
        cp_async_commit();
      }
    } else {
      // ---------------- warps 1..3: update of item it-1, projections of item it+1
      if constexpr (CL && !PUBW) {
        if (edge_pub && it >= 1 && tid == 96) {  // item it-1's stores precede the last CTA barrier
          fence_acq_rel();
          st_relaxed(p.done + (size_t)prv.oct * n_el + prv.el, prv.pass + 1);
        }
      }
      if (it >= 1 && !drained) update(prv, 32, nthr - 32, false);
      if (it + 1 < n_items && !boundary) {
        cp_async_wait<0>();  // this thread's part of item it+1's moments
        bar_named(MW_BAR, nthr - 32);
        project(n1, 32, nthr - 32);
      }
    }
    bar_named(MAIN_BAR, nthr);
    drained = false;
    if (boundary) {  // drain: item it's update (into item it+1's buffer: same cell), new octant, t0 of it+1
      update(cur, 0, nthr, true);
      bar_named(MAIN_BAR, nthr);  // X / K of the old octant no longer read
      stage_octant(n1.oct);
      cp_async_wait<0>();
      bar_named(MAIN_BAR, nthr);
      project(n1, 0, nthr);
      drained = true;
      bar_named(MAIN_BAR, nthr);
    }
    // moments of item it+2 (its cell is not item it's or it+1's; reuse: written by the drain)
    if (warp > 0 && it + 2 < n_items && n2.el != n1.el) prefetch_mom(n2, 32, nthr - 32);
    prv = cur, cur = n1, n1 = n2, n2 = advance(n2);
  }
  if (!drained && n_items >= 1) {  // last item's update
    update(prv, 0, nthr, false);
  }
  if constexpr (CL && !PUBW) {
    if (edge_pub && n_items >= 1 && tid == 96) {
      fence_acq_rel();
      st_relaxed(p.done + (size_t)prv.oct * n_el + prv.el, prv.pass + 1);
    }
  }
  cp_async_wait<0>();
  }  // item warps
  if constexpr (CL) cluster_sync_all();  // no CTA leaves while a neighbour may still write its mailbox
}

size_t gs_smem(int Hp, int kpad, int nmat, int wpb, int rows_nx = 0) {
  return sizeof(double) * wpb * gs_warp_doubles(Hp, kpad, nmat) +
         (rows_nx ? sizeof(double2) * size_t(wpb) * 2 * rows_nx * kpad + sizeof(int) * 8 : 0);
}

// warps per CTA: as many as fit next to the per-warp staging (<= 8)
int gs_wpb(int Hp, int kpad, int nmat) {
  int w = GS_WARPS;
  while (w > 1 && gs_smem(Hp, kpad, nmat, w) > 200 * 1024) w >>= 1;
  return w;
}

template <int NS>
void launch_gs2(const CoarseGSParams& p, cudaStream_t s) {
  auto k = coarse_gs_static_kernel<NS>;
  const int wpb = p.rows_mode ? p.rows_mode : gs_wpb(p.Hp, p.kpad, p.n_mat);
  const size_t smem = gs_smem(p.Hp, p.kpad, p.n_mat, wpb, p.rows_mode ? p.nx : 0);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  CoarseGSParams q = p;
  void* args[] = {&q};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, dim3(p.grid_blocks), dim3(wpb * 32), args, smem, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("coarse_gs cooperative launch: ") + cudaGetErrorString(e));
}

template <int NS>
int occ_blocks(size_t smem, int wpb) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto k = coarse_gs_static_kernel<NS>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, wpb * 32, smem);
  return sms * std::max(per_sm, 1);
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

// row mode: warps per CTA (consecutive grid rows) that fit with the mailbox, 0 if none
int coarse_gs_rows_wpb(int Hp, int kpad, int nmat, int nx, int ny, int max_np) {
  if (max_np > 32) return 0;
  for (int w = 4; w >= 2; w >>= 1)
    if (ny % w == 0 && gs_smem(Hp, kpad, nmat, w, nx) <= 200 * 1024) {
      const size_t smem = gs_smem(Hp, kpad, nmat, w, nx);
      if (occ_blocks<1>(smem, w) * w >= ny) return w;
    }
  return 0;
}

int coarse_gs_max_warps(int Hp, int kpad, int nmat, int max_np) {
  const int wpb = gs_wpb(Hp, kpad, nmat);
  const size_t smem = gs_smem(Hp, kpad, nmat, wpb);
  if (max_np > 64) throw std::invalid_argument("coarse_scatter_sweep: more than 64 patches per octant on the coarsest level");
  return (max_np > 32 ? occ_blocks<2>(smem, wpb) : occ_blocks<1>(smem, wpb)) * wpb;
}
int coarse_gs_warps_per_block(int Hp, int kpad, int nmat) { return gs_wpb(Hp, kpad, nmat); }

// multi-warp rows: whether the ny row-CTAs fit co-resident (0 = no)
bool coarse_gs_chain_blocked() {
  const char* e = std::getenv("STAMG_GS_CHAIN_BLOCKS");
  return !(e != nullptr && e[0] == '0' && e[1] == 0);
}

int coarse_gs_mw_ok(int Hp, int H, int kpad, int nmat, int ny, int max_np, bool blk) {
  if (max_np > 64) return 0;
  if (blk && kpad % 4 != 0) return 0;
  const size_t smem = sizeof(double) * gs_mw_doubles(Hp, H, kpad, nmat, 0, blk);
  if (smem > 220 * 1024) return 0;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto k = max_np > 32 ? (blk ? coarse_gs_mw_kernel<2, false, false, true> : coarse_gs_mw_kernel<2, false, false, false>)
                       : (blk ? coarse_gs_mw_kernel<1, false, false, true> : coarse_gs_mw_kernel<1, false, false, false>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, GSW_MW * 32, smem);
  return per_sm * sms >= ny ? 1 : 0;
}

size_t gs_mw_cl_smem(int Hp, int H, int kpad, int nmat, int nslots, int mbnp, int hs, bool blk) {
  return sizeof(double) * (gs_mw_doubles(Hp, H, kpad, nmat, hs, blk) + gs_mw_cl_doubles(nslots, mbnp));
}
int gs_ring_hs(int H) { return (H + 1) & ~1; }  // rings: the compact moment ring makes room for the mailbox

template <int NS, bool RING, bool BLK>
cudaLaunchConfig_t gs_cl_config(const CoarseGSParams& p, cudaLaunchAttribute* at, size_t smem, int rows, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.ny), cfg.blockDim = dim3((GSW_MW + (gs_pubw<NS, true>() ? 1 : 0)) * 32);
  cfg.dynamicSmemBytes = smem, cfg.stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = rows, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
  cfg.attrs = at, cfg.numAttrs = 1;
  auto k = coarse_gs_mw_kernel<NS, true, RING, BLK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return cfg;
}

// rows per cluster and mailbox slots per direction (slots << 8 | credit << 7 | rows), 0 if none
template <int NS, bool BLK>
int gs_cluster_rows_t(int Hp, int H, int kpad, int nmat, int nx, int ny, int max_np) {
  // rings with credits (for mailboxes of two octants that do not fit) are opt-in: at config 4
  // (64 patches per octant, 4-slot ring) they measured 0.319 s per coarse solve against 0.311 s
  // for the global-memory kernel
  const bool rings = std::getenv("STAMG_GS_MAILBOX_RING") != nullptr;
  for (int nslots : {2 * nx, 16, 8, 4}) {
    const bool credit = nslots != 2 * nx;
    if (credit && !rings) break;
    if (credit && nslots >= 2 * nx) continue;
    const size_t smem = gs_mw_cl_smem(Hp, H, kpad, nmat, nslots, max_np, credit ? gs_ring_hs(H) : 0, BLK);
    if (smem > 112 * 1024) continue;  // keep two row-CTAs per SM
    for (int rows : {16, 8, 4, 2}) {
      if (ny % rows != 0 || ny / rows < 2) continue;
      CoarseGSParams p;
      p.ny = ny;
      cudaLaunchAttribute at[1];
      cudaLaunchConfig_t cfg = credit ? gs_cl_config<NS, true, BLK>(p, at, smem, rows, nullptr)
                                      : gs_cl_config<NS, false, BLK>(p, at, smem, rows, nullptr);
      int nclusters = 0;
      const cudaError_t e = credit ? cudaOccupancyMaxActiveClusters(&nclusters, coarse_gs_mw_kernel<NS, true, true, BLK>, &cfg)
                                   : cudaOccupancyMaxActiveClusters(&nclusters, coarse_gs_mw_kernel<NS, true, false, BLK>, &cfg);
      if (e != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (nclusters >= ny / rows) return (nslots << 8) | (credit ? 128 : 0) | rows;
    }
  }
  return 0;
}

template <int NS, bool BLK>
void launch_gs_mw_cluster(const CoarseGSParams& p, cudaStream_t s) {
  const size_t smem = gs_mw_cl_smem(p.Hp, p.H, p.kpad, p.n_mat, p.mb_slots, p.mb_np, p.mom_stride, BLK);
  cudaLaunchAttribute at[1];
  cudaError_t e;
  if (p.mb_credit) {
    cudaLaunchConfig_t cfg = gs_cl_config<NS, true, BLK>(p, at, smem, p.cluster, s);
    e = cudaLaunchKernelEx(&cfg, coarse_gs_mw_kernel<NS, true, true, BLK>, p);
  } else {
    cudaLaunchConfig_t cfg = gs_cl_config<NS, false, BLK>(p, at, smem, p.cluster, s);
    e = cudaLaunchKernelEx(&cfg, coarse_gs_mw_kernel<NS, true, false, BLK>, p);
  }
  if (e != cudaSuccess) throw std::runtime_error(std::string("coarse_gs cluster launch: ") + cudaGetErrorString(e));
}

template <int NS, bool BLK>
void launch_gs_mw(const CoarseGSParams& p, cudaStream_t s) {
  if (p.cluster > 1) return launch_gs_mw_cluster<NS, BLK>(p, s);
  auto k = coarse_gs_mw_kernel<NS, false, false, BLK>;
  const size_t smem = sizeof(double) * gs_mw_doubles(p.Hp, p.H, p.kpad, p.n_mat, 0, BLK);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  CoarseGSParams q = p;
  void* args[] = {&q};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, dim3(p.ny), dim3(GSW_MW * 32), args, smem, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("coarse_gs cooperative launch: ") + cudaGetErrorString(e));
}

int coarse_gs_cluster_rows(int Hp, int H, int kpad, int nmat, int nx, int ny, int max_np, bool blk) {
  if (max_np > 64) return 0;
  if (blk)
    return max_np > 32 ? gs_cluster_rows_t<2, true>(Hp, H, kpad, nmat, nx, ny, max_np)
                       : gs_cluster_rows_t<1, true>(Hp, H, kpad, nmat, nx, ny, max_np);
  return max_np > 32 ? gs_cluster_rows_t<2, false>(Hp, H, kpad, nmat, nx, ny, max_np)
                     : gs_cluster_rows_t<1, false>(Hp, H, kpad, nmat, nx, ny, max_np);
}

void launch_coarse_gs(const CoarseGSParams& p, cudaStream_t s) {
  if (p.nu <= 0 || p.n_el == 0) return;
  if (p.multi_warp) {
    if (p.chain_blk) {
      if (p.Minv == nullptr || p.kpad % 4 != 0) throw std::logic_error("coarse_scatter_sweep: blocked chain without its tables");
      if (p.max_patches_per_octant <= 32) launch_gs_mw<1, true>(p, s);
      else launch_gs_mw<2, true>(p, s);
    } else {
      if (p.max_patches_per_octant <= 32) launch_gs_mw<1, false>(p, s);
      else launch_gs_mw<2, false>(p, s);
    }
    return;
  }
  if (p.max_patches_per_octant <= 32) launch_gs2<1>(p, s);
  else launch_gs2<2>(p, s);
}

}  // namespace stamg_b200
