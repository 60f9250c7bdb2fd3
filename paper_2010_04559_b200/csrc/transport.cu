// Matrix-free streaming-removal operator on sm_100a: apply_L_into
// (transport.cpp:66-88), y = alpha * L x + beta * f.
//
// Thread = (direction of a 4-direction group, cell). Cells are enumerated in
// the group's sweep frame so a warp's 8 cells are consecutive along x and the
// 4 directions of a cell are adjacent lanes (one 128-byte line when the group's
// patches are consecutive). Upwind neighbour traces are read through L1/L2;
// every x block is fetched from DRAM once. Arithmetic is done in the sweep
// frame with host-permuted blocks.
// HBM traffic: 32 B read + 32 B written per cell-direction (+32 B for f).
#include "common.cuh"
#include "kernels.hpp"

namespace stamg_b200 {
namespace {

__device__ __forceinline__ void to_frame(int m, double& a0, double& a1, double& a2, double& a3) {
  if (m & 1) { double u = a0; a0 = a1; a1 = u; u = a2; a2 = a3; a3 = u; }
  if (m & 2) { double u = a0; a0 = a2; a2 = u; u = a1; a1 = a3; a3 = u; }
}
__device__ __forceinline__ void from_frame(int m, double& a0, double& a1, double& a2, double& a3) {
  if (m & 2) { double u = a0; a0 = a2; a2 = u; u = a1; a1 = a3; a3 = u; }
  if (m & 1) { double u = a0; a0 = a1; a1 = u; u = a2; a2 = a3; a3 = u; }
}

constexpr int kCellsPerBlock = 64;  // 256 threads

template <bool MULTI, bool WITH_F>
__global__ void __launch_bounds__(256) apply_L_kernel(ApplyLParams p) {
  const int tid = threadIdx.x, dir = tid & 3, c = tid >> 2;
  const int grp = blockIdx.y;
  const int q = p.g.groups[grp * 4 + dir];
  if (q < 0) return;
  const int oct = p.g.group_oct[grp];
  const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
  const int m = (xneg ? 1 : 0) | (yneg ? 2 : 0);
  const int nx = p.g.nx, ny = p.g.ny, P = p.g.P;
  const int cell = blockIdx.x * kCellsPerBlock + c;
  if (cell >= nx * ny) return;
  const int jf = cell / nx, ifr = cell - jf * nx;
  const int gx = xneg ? nx - 1 - ifr : ifr, gy = yneg ? ny - 1 - jf : jf;
  const int el = gy * nx + gx;
  const double* xb = p.x + ((size_t)el * P + q) * 4;
  double2 a = __ldg(reinterpret_cast<const double2*>(xb)), b = __ldg(reinterpret_cast<const double2*>(xb) + 1);
  double x0 = a.x, x1 = a.y, x2 = b.x, x3 = b.y;
  to_frame(m, x0, x1, x2, x3);
  const int mt = MULTI ? p.g.mat[el] : 0;
  const double* B = p.B + ((size_t)mt * P + q) * 16;
  double y0 = B[0] * x0 + B[1] * x1 + B[2] * x2 + B[3] * x3;
  double y1 = B[4] * x0 + B[5] * x1 + B[6] * x2 + B[7] * x3;
  double y2 = B[8] * x0 + B[9] * x1 + B[10] * x2 + B[11] * x3;
  double y3 = B[12] * x0 + B[13] * x1 + B[14] * x2 + B[15] * x3;
  const double* cxy = p.cxy + (size_t)q * 8;
  if (ifr > 0) {  // x-upwind neighbour: its frame dofs {1,3} feed rows {0,2}
    const double* ub = p.x + ((size_t)(el + (xneg ? 1 : -1)) * P + q) * 4;
    double u0 = ub[0], u1 = ub[1], u2 = ub[2], u3 = ub[3];
    to_frame(m, u0, u1, u2, u3);
    y0 += cxy[0] * u1 + cxy[1] * u3;
    y2 += cxy[2] * u1 + cxy[3] * u3;
  }
  if (jf > 0) {  // y-upwind neighbour: frame dofs {2,3} feed rows {0,1}
    const double* ub = p.x + ((size_t)(el + (yneg ? nx : -nx)) * P + q) * 4;
    double u0 = ub[0], u1 = ub[1], u2 = ub[2], u3 = ub[3];
    to_frame(m, u0, u1, u2, u3);
    y0 += cxy[4] * u2 + cxy[5] * u3;
    y1 += cxy[6] * u2 + cxy[7] * u3;
  }
  from_frame(m, y0, y1, y2, y3);
  double* yb = p.y + ((size_t)el * P + q) * 4;
  if constexpr (WITH_F) {
    const double* fb = p.f + ((size_t)el * P + q) * 4;
    y0 = p.alpha * y0 + p.beta * fb[0];
    y1 = p.alpha * y1 + p.beta * fb[1];
    y2 = p.alpha * y2 + p.beta * fb[2];
    y3 = p.alpha * y3 + p.beta * fb[3];
  } else if (p.alpha != 1.0) {
    y0 *= p.alpha, y1 *= p.alpha, y2 *= p.alpha, y3 *= p.alpha;
  }
  reinterpret_cast<double2*>(yb)[0] = make_double2(y0, y1);
  reinterpret_cast<double2*>(yb)[1] = make_double2(y2, y3);
}

// Row-walk variant for 8-direction groups: CTA = 8 directions x 32 rows of one
// 32-row strip; thread (dir, row) walks its row in upwind order. The x-upwind
// block is the thread's previous one (registers), the y-upwind block comes from
// the row below by a shuffle (lanes of the warp's first row load it), so each x
// block is read from DRAM once, in 256-byte runs per (cell, 8 directions).
template <bool MULTI, bool WITH_F>
__global__ void __launch_bounds__(256) apply_L_rows_kernel(ApplyLParams p) {
  constexpr int DIRS = 8, R = 32;
  const int tid = threadIdx.x, dir = tid % DIRS, r = tid / DIRS, lane = tid & 31;
  const int grp = blockIdx.y, strip = blockIdx.x;
  const int q = p.g.groups[grp * DIRS + dir];
  const int oct = p.g.group_oct[grp];
  const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
  const int m = (xneg ? 1 : 0) | (yneg ? 2 : 0);
  const int nx = p.g.nx, ny = p.g.ny, P = p.g.P;
  const int jf = strip * R + r;
  const bool rowok = jf < ny && q >= 0;
  const int qq = q >= 0 ? q : 0;
  const int gy = yneg ? ny - 1 - (jf < ny ? jf : 0) : (jf < ny ? jf : 0);
  const int gyd = jf > 0 ? (yneg ? gy + 1 : gy - 1) : gy;  // y-upwind row (lanes of the warp's first row)
  const double* cxy = p.cxy + (size_t)qq * 8;
  const double c0 = cxy[0], c1 = cxy[1], c2 = cxy[2], c3 = cxy[3], c4 = cxy[4], c5 = cxy[5], c6 = cxy[6], c7 = cxy[7];
  const double* Bq = p.B + (size_t)qq * 16;
  double Bl[16];
  if constexpr (!MULTI) {
#pragma unroll
    for (int k = 0; k < 16; ++k) Bl[k] = Bq[k];
  }
  const bool first_row_of_warp = lane < DIRS;
  double px1 = 0.0, px3 = 0.0;  // x-upwind trace (frame dofs 1, 3)
  auto load = [&](int el) {
    const double2* b = reinterpret_cast<const double2*>(p.x + ((size_t)el * P + qq) * 4);
    const double2 a = __ldg(b), c = __ldg(b + 1);
    double v0 = a.x, v1 = a.y, v2 = c.x, v3 = c.y;
    return make_double4(v0, v1, v2, v3);
  };
  int gx = xneg ? nx - 1 : 0;
  double4 cur = rowok ? load(gy * nx + gx) : make_double4(0, 0, 0, 0);
  double4 low = (rowok && first_row_of_warp && jf > 0) ? load(gyd * nx + gx) : make_double4(0, 0, 0, 0);
  for (int i = 0; i < nx; ++i) {
    const int el = gy * nx + gx;
    const int gxn = xneg ? gx - 1 : gx + 1;
    double4 nxt = make_double4(0, 0, 0, 0), nlow = make_double4(0, 0, 0, 0);
    if (i + 1 < nx && rowok) {  // prefetch the next cell
      nxt = load(gy * nx + gxn);
      if (first_row_of_warp && jf > 0) nlow = load(gyd * nx + gxn);
    }
    double x0 = cur.x, x1 = cur.y, x2 = cur.z, x3 = cur.w;
    to_frame(m, x0, x1, x2, x3);
    // y-upwind block: the row below's current block (shuffle), its frame dofs {2,3}
    double u2 = __shfl_up_sync(0xffffffffu, x2, DIRS), u3 = __shfl_up_sync(0xffffffffu, x3, DIRS);
    if (first_row_of_warp) {
      double l0 = low.x, l1 = low.y, l2 = low.z, l3 = low.w;
      to_frame(m, l0, l1, l2, l3);
      u2 = l2, u3 = l3;
    }
    if (rowok) {
      const double* B = Bl;
      double Bm[16];
      if constexpr (MULTI) {
        const double* Bs = p.B + ((size_t)p.g.mat[el] * P + qq) * 16;
#pragma unroll
        for (int k = 0; k < 16; ++k) Bm[k] = Bs[k];
        B = Bm;
      }
      double y0 = B[0] * x0 + B[1] * x1 + B[2] * x2 + B[3] * x3;
      double y1 = B[4] * x0 + B[5] * x1 + B[6] * x2 + B[7] * x3;
      double y2 = B[8] * x0 + B[9] * x1 + B[10] * x2 + B[11] * x3;
      double y3 = B[12] * x0 + B[13] * x1 + B[14] * x2 + B[15] * x3;
      if (i > 0) {
        y0 += c0 * px1 + c1 * px3;
        y2 += c2 * px1 + c3 * px3;
      }
      if (jf > 0) {
        y0 += c4 * u2 + c5 * u3;
        y1 += c6 * u2 + c7 * u3;
      }
      from_frame(m, y0, y1, y2, y3);
      double* yb = p.y + ((size_t)el * P + q) * 4;
      if constexpr (WITH_F) {
        const double2* fb = reinterpret_cast<const double2*>(p.f + ((size_t)el * P + q) * 4);
        const double2 fa = fb[0], fc = fb[1];
        y0 = p.alpha * y0 + p.beta * fa.x;
        y1 = p.alpha * y1 + p.beta * fa.y;
        y2 = p.alpha * y2 + p.beta * fc.x;
        y3 = p.alpha * y3 + p.beta * fc.y;
      } else if (p.alpha != 1.0) {
        y0 *= p.alpha, y1 *= p.alpha, y2 *= p.alpha, y3 *= p.alpha;
      }
      reinterpret_cast<double2*>(yb)[0] = make_double2(y0, y1);
      reinterpret_cast<double2*>(yb)[1] = make_double2(y2, y3);
    }
    px1 = x1, px3 = x3;
    cur = nxt, low = nlow;
    gx = gxn;
  }
}

// Staged row walk (the default for 8-direction groups): the same (direction, row) threads, but
// each thread's x blocks (and f, and the y-upwind blocks of a warp's first row) arrive through a
// private cp.async ring kRing - 2 cells ahead, so a 2-CTA SM keeps ~80 KB of loads in flight
// instead of the one block per thread the register prefetch above allows (112 registers, 512
// threads per SM: 16 KB). A thread only reads slots it filled itself: no CTA barrier.
#ifndef STAMG_APPLYL_RING
#define STAMG_APPLYL_RING 6  // ring slots per thread (0: register-prefetch kernel above)
#endif
constexpr int kRing = STAMG_APPLYL_RING > 2 ? STAMG_APPLYL_RING : 3;
#ifndef STAMG_APPLYL_MINB
#define STAMG_APPLYL_MINB 2
#endif

template <bool MULTI, bool WITH_F>
__global__ void __launch_bounds__(256, STAMG_APPLYL_MINB) apply_L_ring_kernel(ApplyLParams p) {
  constexpr int DIRS = 8, R = 32, NT = 256, AHEAD = kRing - 2;
  extern __shared__ __align__(16) double smem[];
  double* sx = smem;                                        // [kRing][NT][4]
  double* sl = sx + kRing * NT * 4;                         // [kRing][NT / 32][DIRS][4]
  double* sf = sl + kRing * (NT / 32) * DIRS * 4;           // [kRing][NT][4] (WITH_F)
  const int tid = threadIdx.x, dir = tid % DIRS, r = tid / DIRS, lane = tid & 31, warp = tid >> 5;
  const int grp = blockIdx.y, strip = blockIdx.x;
  const int q = p.g.groups[grp * DIRS + dir];
  const int oct = p.g.group_oct[grp];
  const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
  const int m = (xneg ? 1 : 0) | (yneg ? 2 : 0);
  const int nx = p.g.nx, ny = p.g.ny, P = p.g.P;
  const int jf = strip * R + r;
  const bool rowok = jf < ny && q >= 0;
  const int qq = q >= 0 ? q : 0;
  const int gy = yneg ? ny - 1 - (jf < ny ? jf : 0) : (jf < ny ? jf : 0);
  const int gyd = jf > 0 ? (yneg ? gy + 1 : gy - 1) : gy;
  const double* cxy = p.cxy + (size_t)qq * 8;
  const double c0 = cxy[0], c1 = cxy[1], c2 = cxy[2], c3 = cxy[3], c4 = cxy[4], c5 = cxy[5], c6 = cxy[6], c7 = cxy[7];
  const double* Bq = p.B + (size_t)qq * 16;
  double Bl[16];
  if constexpr (!MULTI) {
#pragma unroll
    for (int k = 0; k < 16; ++k) Bl[k] = Bq[k];
  }
  const bool first_row_of_warp = lane < DIRS;
  const bool need_low = rowok && first_row_of_warp && jf > 0;
  const int dx = xneg ? -1 : 1;
  // element offsets of the walk's first cell (this row, the row below it)
  const size_t base = ((size_t)(gy * nx + (xneg ? nx - 1 : 0)) * P + qq) * 4;
  const size_t based = ((size_t)(gyd * nx + (xneg ? nx - 1 : 0)) * P + qq) * 4;
  const ptrdiff_t step = (ptrdiff_t)dx * P * 4;
  auto issue = [&](int i) {
    const int slot = i % kRing;
    const bool ok = rowok && i < nx;
    const ptrdiff_t o = ok ? (ptrdiff_t)base + step * i : 0;
    double* dst = sx + ((size_t)slot * NT + tid) * 4;
    cp_async16(dst, p.x + o, ok);
    cp_async16(dst + 2, p.x + o + 2, ok);
    if constexpr (WITH_F) {
      double* df = sf + ((size_t)slot * NT + tid) * 4;
      cp_async16(df, p.f + o, ok);
      cp_async16(df + 2, p.f + o + 2, ok);
    }
    if (first_row_of_warp) {
      const bool okl = need_low && i < nx;
      const ptrdiff_t ol = okl ? (ptrdiff_t)based + step * i : 0;
      double* dl = sl + (((size_t)slot * (NT / 32) + warp) * DIRS + dir) * 4;
      cp_async16(dl, p.x + ol, okl);
      cp_async16(dl + 2, p.x + ol + 2, okl);
    }
  };
#pragma unroll
  for (int i = 0; i < AHEAD; ++i) {
    issue(i);
    cp_async_commit();
  }
  double px1 = 0.0, px3 = 0.0;  // x-upwind trace (frame dofs 1, 3)
  int el = gy * nx + (xneg ? nx - 1 : 0);
  size_t off = base;
  for (int i = 0; i < nx; ++i) {
    issue(i + AHEAD);  // slot (i - 2) % kRing: read two cells ago
    cp_async_commit();
    cp_async_wait<AHEAD>();
    asm volatile("" ::: "memory");
    const int slot = i % kRing;
    const double2* xs = reinterpret_cast<const double2*>(sx + ((size_t)slot * NT + tid) * 4);
    const double2 xa = xs[0], xc = xs[1];
    double x0 = xa.x, x1 = xa.y, x2 = xc.x, x3 = xc.y;
    to_frame(m, x0, x1, x2, x3);
    double u2 = __shfl_up_sync(0xffffffffu, x2, DIRS), u3 = __shfl_up_sync(0xffffffffu, x3, DIRS);
    if (first_row_of_warp) {
      const double2* ls = reinterpret_cast<const double2*>(sl + (((size_t)slot * (NT / 32) + warp) * DIRS + dir) * 4);
      const double2 la = ls[0], lc = ls[1];
      double l0 = la.x, l1 = la.y, l2 = lc.x, l3 = lc.y;
      to_frame(m, l0, l1, l2, l3);
      u2 = l2, u3 = l3;
    }
    if (rowok) {
      const double* B = Bl;
      double Bm[16];
      if constexpr (MULTI) {
        const double* Bs = p.B + ((size_t)p.g.mat[el] * P + qq) * 16;
#pragma unroll
        for (int k = 0; k < 16; ++k) Bm[k] = Bs[k];
        B = Bm;
      }
      double y0 = B[0] * x0 + B[1] * x1 + B[2] * x2 + B[3] * x3;
      double y1 = B[4] * x0 + B[5] * x1 + B[6] * x2 + B[7] * x3;
      double y2 = B[8] * x0 + B[9] * x1 + B[10] * x2 + B[11] * x3;
      double y3 = B[12] * x0 + B[13] * x1 + B[14] * x2 + B[15] * x3;
      if (i > 0) {
        y0 += c0 * px1 + c1 * px3;
        y2 += c2 * px1 + c3 * px3;
      }
      if (jf > 0) {
        y0 += c4 * u2 + c5 * u3;
        y1 += c6 * u2 + c7 * u3;
      }
      from_frame(m, y0, y1, y2, y3);
      if constexpr (WITH_F) {
        const double2* fs = reinterpret_cast<const double2*>(sf + ((size_t)slot * NT + tid) * 4);
        const double2 fa = fs[0], fc = fs[1];
        y0 = p.alpha * y0 + p.beta * fa.x;
        y1 = p.alpha * y1 + p.beta * fa.y;
        y2 = p.alpha * y2 + p.beta * fc.x;
        y3 = p.alpha * y3 + p.beta * fc.y;
      } else if (p.alpha != 1.0) {
        y0 *= p.alpha, y1 *= p.alpha, y2 *= p.alpha, y3 *= p.alpha;
      }
      double* yb = p.y + off;
      reinterpret_cast<double2*>(yb)[0] = make_double2(y0, y1);
      reinterpret_cast<double2*>(yb)[1] = make_double2(y2, y3);
    }
    px1 = x1, px3 = x3;
    el += dx, off += step;
  }
  cp_async_wait<0>();
}

template <bool MULTI, bool WITH_F>
void launch_ring(const ApplyLParams& p, dim3 grid, cudaStream_t s) {
  const size_t smem = sizeof(double) * kRing * (256 * 4 * (WITH_F ? 2 : 1) + 8 * 8 * 4);
  auto k = apply_L_ring_kernel<MULTI, WITH_F>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<grid, 256, smem, s>>>(p);
}

}  // namespace

void launch_apply_L(const ApplyLParams& p, cudaStream_t s) {
  if (p.g.n_groups == 0) return;
  if (p.dirs == 8) {
    dim3 grid((p.g.ny + 31) / 32, p.g.n_groups);
    const bool multi = p.g.n_mat > 1, wf = p.f != nullptr && p.beta != 0.0;
    if (STAMG_APPLYL_RING > 0) {
      if (multi) wf ? launch_ring<true, true>(p, grid, s) : launch_ring<true, false>(p, grid, s);
      else wf ? launch_ring<false, true>(p, grid, s) : launch_ring<false, false>(p, grid, s);
      return;
    }
    if (multi) wf ? apply_L_rows_kernel<true, true><<<grid, 256, 0, s>>>(p) : apply_L_rows_kernel<true, false><<<grid, 256, 0, s>>>(p);
    else wf ? apply_L_rows_kernel<false, true><<<grid, 256, 0, s>>>(p) : apply_L_rows_kernel<false, false><<<grid, 256, 0, s>>>(p);
    return;
  }
  const int cells = p.g.nx * p.g.ny;
  dim3 grid((cells + kCellsPerBlock - 1) / kCellsPerBlock, p.g.n_groups);
  const bool multi = p.g.n_mat > 1, wf = p.f != nullptr && p.beta != 0.0;
  if (multi) wf ? apply_L_kernel<true, true><<<grid, 256, 0, s>>>(p) : apply_L_kernel<true, false><<<grid, 256, 0, s>>>(p);
  else wf ? apply_L_kernel<false, true><<<grid, 256, 0, s>>>(p) : apply_L_kernel<false, false><<<grid, 256, 0, s>>>(p);
}

}  // namespace stamg_b200
