// Kernels of the reference-shape path (generic.hpp): any block size bs = D*S <= 24, 2D or 3D
// grids. Dense block arithmetic, hyperplane (KBA) ordering for the sweeps: cells with
// fi + fj + fk = const in the octant's frame are independent (their upwind neighbours lie on
// the previous plane), which is all the reference's element order (spatial_disc.cpp:90-106)
// constrains.
#include "common.cuh"
#include "generic.hpp"

#include <cooperative_groups.h>

#include <algorithm>
#include <stdexcept>
#include <string>

namespace cg = cooperative_groups;

namespace stamg_b200 {
namespace gen {

namespace {

struct Frame {  // octant frame <-> grid coordinates
  int nx, ny, nz;
  bool xn, yn, zn;
  __device__ Frame(const Dev& L, int oct) : nx(L.nx), ny(L.ny), nz(L.nz), xn(oct & 1), yn(oct & 2), zn(oct & 4) {}
  __device__ int el(int fi, int fj, int fk) const {
    const int ix = xn ? nx - 1 - fi : fi, iy = yn ? ny - 1 - fj : fj, iz = zn ? nz - 1 - fk : fk;
    return (iz * ny + iy) * nx + ix;
  }
};

// upwind neighbour of cell el along axis xi for a patch of octant oct, -1 at the boundary
// (HexMesh::neighbor with the inflow face, transport.cpp:50-52)
__device__ __forceinline__ int upwind(const Dev& L, int el, int oct, int xi) {
  const int ix = el % L.nx, iy = (el / L.nx) % L.ny, iz = el / (L.nx * L.ny);
  const int dir = (oct >> xi) & 1 ? 1 : -1;  // positive cosine: inflow through the low face
  const int cur = xi == 0 ? ix : xi == 1 ? iy : iz, n = xi == 0 ? L.nx : xi == 1 ? L.ny : L.nz;
  const int stride = xi == 0 ? 1 : xi == 1 ? L.nx : L.nx * L.ny;
  if (cur + dir < 0 || cur + dir >= n) return -1;
  return el + dir * stride;
}

__global__ void apply_L_kernel(Dev L, const double* __restrict__ x, double* __restrict__ y, double alpha, double beta,
                               const double* __restrict__ f) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int bs = L.bs;
  if (idx >= (int64_t)L.n_el * L.P * bs) return;
  const int r = int(idx % bs);
  const int64_t blk = idx / bs;
  const int q = int(blk % L.P), el = int(blk / L.P);
  const int oct = L.octant[q];
  const double* B = L.Bd + ((size_t)q * bs + r) * bs;
  const double* xb = x + blk * bs;
  double acc = 0.0;
  for (int c = 0; c < bs; ++c) acc += B[c] * xb[c];
  for (int xi = 0; xi < L.dim; ++xi) {
    const int up = upwind(L, el, oct, xi);
    if (up < 0) continue;
    const double* C = L.C + (((size_t)q * 3 + xi) * bs + r) * bs;
    const double* xu = x + ((size_t)up * L.P + q) * bs;
    double a2 = 0.0;
    for (int c = 0; c < bs; ++c) a2 += C[c] * xu[c];
    acc += a2;
  }
  y[idx] = alpha * acc + (beta != 0.0 ? beta * f[idx] : 0.0);
}

// Block size known at compile time (1, 3, 8, 12, 24: every S x D the reference has outside the
// tuned 2D path): a thread owns a whole (cell, patch) block in registers; the patch's dense
// tables sit in shared memory and are read as warp-wide broadcasts.
template <int BS>
__device__ __forceinline__ void load_block(const double* __restrict__ p, double* v) {
  if constexpr (BS % 2 == 0) {
#pragma unroll
    for (int c = 0; c < BS; c += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + c);
      v[c] = t.x, v[c + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < BS; ++c) v[c] = p[c];
  }
}
template <int BS>
__device__ __forceinline__ void store_block(double* p, const double* v) {
  if constexpr (BS % 2 == 0) {
#pragma unroll
    for (int c = 0; c < BS; c += 2) *reinterpret_cast<double2*>(p + c) = make_double2(v[c], v[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < BS; ++c) p[c] = v[c];
  }
}
// acc (+)= M v with M [BS][BS] in shared memory (each entry one broadcast load)
template <int BS, bool SUB>
__device__ __forceinline__ void matvec_acc(const double* M, const double* v, double* acc) {
#pragma unroll
  for (int a = 0; a < BS; ++a) {
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < BS; ++c) t += M[a * BS + c] * v[c];
    acc[a] = SUB ? acc[a] - t : acc[a] + t;
  }
}

// acc += M v, M given transposed in shared memory (MT[c][a]); v streamed from global memory
// one entry at a time, so only the accumulators live in registers
template <int BS>
__device__ __forceinline__ void matvec_cols(const double* MT, const double* __restrict__ v, double* acc) {
#pragma unroll 2
  for (int c = 0; c < BS; ++c) {
    const double vc = v[c];
    const double* col = MT + c * BS;
    if constexpr (BS % 2 == 0) {
#pragma unroll
      for (int a = 0; a < BS; a += 2) {
        const double2 m = *reinterpret_cast<const double2*>(col + a);
        acc[a] += m.x * vc, acc[a + 1] += m.y * vc;
      }
    } else {
#pragma unroll
      for (int a = 0; a < BS; ++a) acc[a] += col[a] * vc;
    }
  }
}

template <int BS>
__global__ void __launch_bounds__(128) apply_L_block_kernel(Dev L, const double* __restrict__ x, double* __restrict__ y,
                                                            double alpha, double beta, const double* __restrict__ f) {
  extern __shared__ __align__(16) double sm[];  // B^T | C_0^T .. C_{dim-1}^T
  const int q = blockIdx.x, oct = L.octant[q];
  for (int k = threadIdx.x; k < BS * BS; k += blockDim.x) {
    const int a = k / BS, c = k - a * BS, kt = c * BS + a;
    sm[kt] = L.Bd[(size_t)q * BS * BS + k];
    for (int xi = 0; xi < L.dim; ++xi) sm[(1 + xi) * BS * BS + kt] = L.C[((size_t)q * 3 + xi) * BS * BS + k];
  }
  __syncthreads();
  for (int el = blockIdx.y * blockDim.x + threadIdx.x; el < L.n_el; el += gridDim.y * blockDim.x) {
    double acc[BS];
#pragma unroll
    for (int a = 0; a < BS; ++a) acc[a] = 0.0;
    const size_t off = ((size_t)el * L.P + q) * BS;
    matvec_cols<BS>(sm, x + off, acc);
#pragma unroll 1
    for (int xi = 0; xi < L.dim; ++xi) {
      const int up = upwind(L, el, oct, xi);
      if (up < 0) continue;
      matvec_cols<BS>(sm + (1 + xi) * BS * BS, x + ((size_t)up * L.P + q) * BS, acc);
    }
    if (beta != 0.0) {
#pragma unroll
      for (int a = 0; a < BS; ++a) acc[a] = alpha * acc[a] + beta * f[off + a];
    } else {
#pragma unroll
      for (int a = 0; a < BS; ++a) acc[a] *= alpha;
    }
    store_block<BS>(y + off, acc);
  }
}

// apply_L on the FP64 tensor cores (block sizes that are multiples of 8: trilinear cells).
// For one patch, Y^T (cells x rows) = X^T (cells x bs) B^T + sum_xi Xup_xi^T C_xi^T is a GEMM
// with the block operators as the B operand: a warp takes 8 cells at a time (m8n8k4 DMMA:
// lane (g, t) holds x[cell g][4 ks + t] as the A fragment and M[8 nt + g][4 ks + t] as the B
// fragment; the accumulators are y[cell g][8 nt + 2 t, + 1]). The patch's (1 + dim) block
// operators stay in registers as B fragments for the whole CTA; nothing is staged in shared
// memory. 4.6 kflop per 384 B at bs = 24: the kernel is bound by the FP64 tensor rate.
template <int BS>
__global__ void __launch_bounds__(128) apply_L_mma_kernel(Dev L, const double* __restrict__ x, double* __restrict__ y,
                                                          double alpha, double beta, const double* __restrict__ f) {
  constexpr int NT = BS / 8, KS = BS / 4;
  const int q = blockIdx.x, oct = L.octant[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int nm = 1 + L.dim;
  double bf[4][NT][KS];
#pragma unroll
  for (int mx = 0; mx < 4; ++mx) {
    const double* M = mx == 0 ? L.Bd + (size_t)q * BS * BS : L.C + ((size_t)q * 3 + (mx - 1)) * BS * BS;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) bf[mx][nt][ks] = mx < nm ? M[(8 * nt + g) * BS + 4 * ks + t] : 0.0;
  }
  const int ntile = (L.n_el + 7) / 8;
  for (int tile = blockIdx.y * 4 + warp; tile < ntile; tile += gridDim.y * 4) {
    const int el = tile * 8 + g;
    const bool ok = el < L.n_el;
    double acc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int mx = 0; mx < 4; ++mx) {
      if (mx >= nm) break;
      int src = ok ? el : -1;
      if (mx > 0 && ok) src = upwind(L, el, oct, mx - 1);
      double a[KS];
      const double* xb = x + ((size_t)(src < 0 ? 0 : src) * L.P + q) * BS + t;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) a[ks] = src >= 0 ? xb[4 * ks] : 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], a[ks], bf[mx][nt][ks]);
    }
    if (ok) {
      const size_t off = ((size_t)el * L.P + q) * BS + 2 * t;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        double v0 = alpha * acc[nt][0], v1 = alpha * acc[nt][1];
        if (beta != 0.0) {
          const double2 fv = *reinterpret_cast<const double2*>(f + off + 8 * nt);
          v0 += beta * fv.x, v1 += beta * fv.y;
        }
        *reinterpret_cast<double2*>(y + off + 8 * nt) = make_double2(v0, v1);
      }
    }
  }
}

template <int BS>
__global__ void __launch_bounds__(256) sweep_block_kernel(Dev L, const double* rhs, double* z) {
  extern __shared__ __align__(16) double sm[];  // B^-1 | C_0 .. C_{dim-1}
  const int q = blockIdx.x, oct = L.octant[q];
  for (int k = threadIdx.x; k < BS * BS; k += blockDim.x) {
    sm[k] = L.Binv[(size_t)q * BS * BS + k];
    for (int xi = 0; xi < L.dim; ++xi) sm[(1 + xi) * BS * BS + k] = L.C[((size_t)q * 3 + xi) * BS * BS + k];
  }
  __syncthreads();
  const Frame fr(L, oct);
  const int nplanes = L.nx + L.ny + L.nz - 2, njk = L.ny * L.nz;
  for (int pl = 0; pl < nplanes; ++pl) {
    for (int jk = threadIdx.x; jk < njk; jk += blockDim.x) {
      const int fj = jk % L.ny, fk = jk / L.ny, fi = pl - fj - fk;
      if (fi < 0 || fi >= L.nx) continue;
      const int el = fr.el(fi, fj, fk);
      double r[BS], v[BS];
      load_block<BS>(rhs + ((size_t)el * L.P + q) * BS, r);
      for (int xi = 0; xi < L.dim; ++xi) {
        const int fc = xi == 0 ? fi : xi == 1 ? fj : fk;
        if (fc == 0) continue;
        const int up = fr.el(fi - (xi == 0), fj - (xi == 1), fk - (xi == 2));
        load_block<BS>(z + ((size_t)up * L.P + q) * BS, v);
        matvec_acc<BS, true>(sm + (1 + xi) * BS * BS, v, r);
      }
#pragma unroll
      for (int a = 0; a < BS; ++a) v[a] = 0.0;
      matvec_acc<BS, false>(sm, r, v);
      store_block<BS>(z + ((size_t)el * L.P + q) * BS, v);
    }
    __syncthreads();
  }
}

// The sweep on the FP64 tensor cores (block sizes that are multiples of 8). One CTA per patch;
// the cells of a hyperplane (listed plane by plane in the octant's frame: L.plane_cells) are
// independent, so a warp solves 8 of them at a time: r = rhs - sum_xi C_xi z_up as DMMAs onto
// accumulators that start as rhs (B fragments hold -C_xi), then z = B^-1 r after moving r from
// the accumulator layout (cell g: rows 8 nt + 2 t, + 1) to the A-fragment layout (rows 4 ks + t)
// with shuffles inside the cell's lane quad.
template <int BS>
__global__ void __launch_bounds__(256) sweep_mma_kernel(Dev L, const double* rhs, double* z) {
  constexpr int NT = BS / 8, KS = BS / 4;
  const int q = blockIdx.x, oct = L.octant[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5, g = lane >> 2, t = lane & 3;
  double bf[4][NT][KS];  // [0]: B^-1, [1 + xi]: -C_xi
#pragma unroll
  for (int mx = 0; mx < 4; ++mx) {
    const double* M = mx == 0 ? L.Binv + (size_t)q * BS * BS : L.C + ((size_t)q * 3 + (mx - 1)) * BS * BS;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double v = mx <= L.dim ? M[(8 * nt + g) * BS + 4 * ks + t] : 0.0;
        bf[mx][nt][ks] = mx == 0 ? v : -v;
      }
  }
  const Frame fr(L, oct);
  const int nplanes = L.nx + L.ny + L.nz - 2;
  for (int pl = 0; pl < nplanes; ++pl) {
    const int c0 = L.plane_ptr[pl], cnt = L.plane_ptr[pl + 1] - c0;
    for (int tile = warp; tile * 8 < cnt; tile += nwarp) {
      const int k = tile * 8 + g;
      const bool ok = k < cnt;
      const int code = ok ? L.plane_cells[c0 + k] : 0;
      const int fi = code & 1023, fj = (code >> 10) & 1023, fk = code >> 20;
      const int el = fr.el(fi, fj, fk);
      const size_t off = ((size_t)el * L.P + q) * BS;
      double acc[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double2 rv = ok ? *reinterpret_cast<const double2*>(rhs + off + 8 * nt + 2 * t) : make_double2(0.0, 0.0);
        acc[nt][0] = rv.x, acc[nt][1] = rv.y;
      }
#pragma unroll
      for (int xi = 0; xi < 3; ++xi) {
        if (xi >= L.dim) break;
        const int fc = xi == 0 ? fi : xi == 1 ? fj : fk;
        const bool has = ok && fc > 0;
        const int up = has ? fr.el(fi - (xi == 0), fj - (xi == 1), fk - (xi == 2)) : 0;
        const double* zu = z + ((size_t)up * L.P + q) * BS + t;
        double a[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) a[ks] = has ? zu[4 * ks] : 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], a[ks], bf[1 + xi][nt][ks]);
      }
      // r: accumulator layout -> A fragments (row 4 ks + t lives in lane quad slot ((4 ks + t) mod 8) / 2)
      double a[KS];
      const int qb = lane & ~3;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int src = qb + (ks & 1) * 2 + (t >> 1);
        const double e0 = __shfl_sync(0xffffffffu, acc[ks >> 1][0], src), e1 = __shfl_sync(0xffffffffu, acc[ks >> 1][1], src);
        a[ks] = (t & 1) ? e1 : e0;
      }
      double zc[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) zc[nt][0] = zc[nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(zc[nt][0], zc[nt][1], a[ks], bf[0][nt][ks]);
      if (ok) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) *reinterpret_cast<double2*>(z + off + 8 * nt + 2 * t) = make_double2(zc[nt][0], zc[nt][1]);
      }
    }
    __syncthreads();
  }
}

// One CTA per patch; threads take the cells of one hyperplane at a time (any block size).
__global__ void sweep_kernel(Dev L, const double* rhs, double* z) {
  extern __shared__ __align__(16) double sm[];
  const int bs = L.bs, q = blockIdx.x, oct = L.octant[q];
  double* sBi = sm;                 // [bs][bs]
  double* sC = sm + bs * bs;        // [dim][bs][bs]
  for (int k = threadIdx.x; k < bs * bs; k += blockDim.x) {
    sBi[k] = L.Binv[(size_t)q * bs * bs + k];
    for (int xi = 0; xi < L.dim; ++xi) sC[xi * bs * bs + k] = L.C[((size_t)q * 3 + xi) * bs * bs + k];
  }
  __syncthreads();
  const Frame fr(L, oct);
  const int nplanes = L.nx + L.ny + L.nz - 2, njk = L.ny * L.nz;
  for (int pl = 0; pl < nplanes; ++pl) {
    for (int jk = threadIdx.x; jk < njk; jk += blockDim.x) {
      const int fj = jk % L.ny, fk = jk / L.ny, fi = pl - fj - fk;
      if (fi < 0 || fi >= L.nx) continue;
      const int el = fr.el(fi, fj, fk);
      double r[kMaxBs];
      const double* rb = rhs + ((size_t)el * L.P + q) * bs;
      for (int c = 0; c < bs; ++c) r[c] = rb[c];
      for (int xi = 0; xi < L.dim; ++xi) {
        const int fc = xi == 0 ? fi : xi == 1 ? fj : fk;
        if (fc == 0) continue;
        const int up = fr.el(fi - (xi == 0), fj - (xi == 1), fk - (xi == 2));
        const double* zu = z + ((size_t)up * L.P + q) * bs;
        const double* C = sC + xi * bs * bs;
        for (int a = 0; a < bs; ++a) {
          double acc = 0.0;
          for (int c = 0; c < bs; ++c) acc += C[a * bs + c] * zu[c];
          r[a] -= acc;
        }
      }
      double* zb = z + ((size_t)el * L.P + q) * bs;
      for (int a = 0; a < bs; ++a) {
        double acc = 0.0;
        for (int c = 0; c < bs; ++c) acc += sBi[a * bs + c] * r[c];
        zb[a] = acc;
      }
    }
    __syncthreads();
  }
}

// mom[h][i] = sum_r X[r][h] phi[el][r][i]; with apply_sigma_N: out = sig_h (mom N)[h][i]
__global__ void d2m_kernel(Dev L, const double* __restrict__ phi, int Hused, bool apply_sigma_N, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];  // [Hused][S]
  const int el = blockIdx.x, S = L.S, R = L.P * L.D, H = L.H;
  const double* slab = phi + (size_t)el * R * S;
  for (int idx = threadIdx.x; idx < Hused * S; idx += blockDim.x) {
    const int h = idx % Hused, i = idx / Hused;
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc += L.X[(size_t)r * H + h] * slab[(size_t)r * S + i];
    sm[h * S + i] = acc;
  }
  __syncthreads();
  double* o = out + (size_t)el * H * S;
  for (int idx = threadIdx.x; idx < Hused * S; idx += blockDim.x) {
    const int h = idx / S, i = idx % S;
    double v = sm[idx];
    if (apply_sigma_N) {
      double acc = 0.0;
      for (int j = 0; j < S; ++j) acc += sm[h * S + j] * L.Nmat[j * S + i];
      v = L.sig[h] * acc;
    }
    o[idx] = v;
  }
}

// y[el][r][i] += scale sum_h X[r][h] src[el][h][i]
__global__ void m2d_kernel(Dev L, const double* __restrict__ src, int Hused, double scale, double* __restrict__ y) {
  extern __shared__ __align__(16) double sm[];  // [Hused][S]
  const int el = blockIdx.x, S = L.S, R = L.P * L.D, H = L.H;
  for (int idx = threadIdx.x; idx < Hused * S; idx += blockDim.x) sm[idx] = src[(size_t)el * H * S + idx];
  __syncthreads();
  double* slab = y + (size_t)el * R * S;
  for (int idx = threadIdx.x; idx < R * S; idx += blockDim.x) {
    const int r = idx / S, i = idx % S;
    const double* Xr = L.X + (size_t)r * H;
    double acc = 0.0;
    for (int h = 0; h < Hused; ++h) acc += Xr[h] * sm[h * S + i];
    slab[idx] += scale * acc;
  }
}

// Register-blocked scatter kernels, S a template parameter. One CTA per cell; the cell's slab
// (D2M) or its moments (M2D) are staged in shared memory and read as broadcasts, the coupling
// table is read coalesced (X[r][h] over h for D2M, XT[h][r] over r for M2D), and a thread keeps
// the S dofs of its harmonic / row in registers: 1 global + S/2 shared loads per S FMAs.
constexpr int SC_TILE = 256;  // slab rows staged per step

template <int S>
__global__ void __launch_bounds__(128) d2m_block_kernel(Dev L, const double* __restrict__ phi, int Hused, bool apply_sigma_N,
                                                        double* __restrict__ out) {
  __shared__ __align__(16) double tile[SC_TILE * S];
  const int el = blockIdx.x, R = L.P * L.D, H = L.H;
  const double* slab = phi + (size_t)el * R * S;
  double* o = out + (size_t)el * H * S;
  for (int h0 = 0; h0 < Hused; h0 += blockDim.x) {
    const int h = h0 + threadIdx.x;
    double acc[S];
#pragma unroll
    for (int i = 0; i < S; ++i) acc[i] = 0.0;
    for (int r0 = 0; r0 < R; r0 += SC_TILE) {
      const int nr = min(SC_TILE, R - r0);
      __syncthreads();
      for (int k = threadIdx.x; k < nr * S; k += blockDim.x) tile[k] = slab[(size_t)r0 * S + k];
      __syncthreads();
      if (h < Hused) {
        const double* Xc = L.X + (size_t)r0 * H + h;
        for (int r = 0; r < nr; ++r) {
          const double x = Xc[(size_t)r * H];
#pragma unroll
          for (int i = 0; i < S; ++i) acc[i] += x * tile[r * S + i];
        }
      }
    }
    if (h < Hused) {
      if (apply_sigma_N) {
        double v[S];
        const double sg = L.sig[h];
#pragma unroll
        for (int i = 0; i < S; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < S; ++j) t += acc[j] * L.Nmat[j * S + i];
          v[i] = sg * t;
        }
#pragma unroll
        for (int i = 0; i < S; ++i) o[h * S + i] = v[i];
      } else {
#pragma unroll
        for (int i = 0; i < S; ++i) o[h * S + i] = acc[i];
      }
    }
  }
}

template <int S>
__global__ void __launch_bounds__(128) m2d_block_kernel(Dev L, const double* __restrict__ src, int Hused, double scale,
                                                        double* __restrict__ y) {
  extern __shared__ __align__(16) double sm[];  // [Hused][S]
  const int el = blockIdx.x, R = L.P * L.D, H = L.H;
  for (int idx = threadIdx.x; idx < Hused * S; idx += blockDim.x) sm[idx] = src[(size_t)el * H * S + idx];
  __syncthreads();
  double* slab = y + (size_t)el * R * S;
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    double acc[S];
#pragma unroll
    for (int i = 0; i < S; ++i) acc[i] = 0.0;
    const double* Xr = L.XT + r;
    for (int h = 0; h < Hused; ++h) {
      const double x = Xr[(size_t)h * R];
#pragma unroll
      for (int i = 0; i < S; ++i) acc[i] += x * sm[h * S + i];
    }
#pragma unroll
    for (int i = 0; i < S; ++i) slab[(size_t)r * S + i] += scale * acc[i];
  }
}

// Scatter on the FP64 tensor cores for 8-dof (trilinear) cells: per cell the moment contraction
// MOM (H x 8) = X^T (H x R) Phi (R x 8) and its transpose Y (R x 8) += X (R x H) SRC (H x 8) are
// GEMMs whose N dimension is exactly the 8 dofs of a DMMA tile. A warp takes two cells, four
// 8-row output tiles at a time (accumulators in registers), streaming the coupling table as A
// fragments and the cell slab / moments as B fragments.
constexpr int SC_MG = 4;  // output tiles per pass
constexpr int SC_NC = 2;  // cells per warp

__global__ void __launch_bounds__(128) d2m_mma_kernel(Dev L, const double* __restrict__ phi, int Hused, bool apply_sigma_N,
                                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int R = L.P * L.D, H = L.H;
  const int el0 = (blockIdx.x * 4 + warp) * SC_NC;
  if (el0 >= L.n_el) return;
  const int ncell = min(SC_NC, L.n_el - el0);
  const int MT = (Hused + 7) / 8;
  for (int m0 = 0; m0 < MT; m0 += SC_MG) {
    double acc[SC_MG][SC_NC][2];
#pragma unroll
    for (int a = 0; a < SC_MG; ++a)
#pragma unroll
      for (int c = 0; c < SC_NC; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    for (int ks = 0; ks < R / 4; ++ks) {
      const int r = 4 * ks + t;
      double af[SC_MG], bf[SC_NC];
#pragma unroll
      for (int a = 0; a < SC_MG; ++a) {
        const int h = 8 * (m0 + a) + g;
        af[a] = h < Hused ? L.X[(size_t)r * H + h] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < SC_NC; ++c) bf[c] = c < ncell ? phi[((size_t)(el0 + c) * R + r) * 8 + g] : 0.0;
#pragma unroll
      for (int a = 0; a < SC_MG; ++a)
#pragma unroll
        for (int c = 0; c < SC_NC; ++c) dmma_8x8x4(acc[a][c][0], acc[a][c][1], af[a], bf[c]);
    }
    // epilogue: accumulators hold mom[h = 8 mt + g][i = 2t, 2t + 1]
#pragma unroll
    for (int a = 0; a < SC_MG; ++a) {
      const int h = 8 * (m0 + a) + g;
#pragma unroll
      for (int c = 0; c < SC_NC; ++c) {
        double v0 = acc[a][c][0], v1 = acc[a][c][1];
        if (apply_sigma_N) {  // row h of mom times N: gather the row's 8 values from the lane quad
          double row[8];
          const int qb = lane & ~3;
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) {
            row[2 * s2] = __shfl_sync(0xffffffffu, acc[a][c][0], qb + s2);
            row[2 * s2 + 1] = __shfl_sync(0xffffffffu, acc[a][c][1], qb + s2);
          }
          double o0 = 0.0, o1 = 0.0;
#pragma unroll
          for (int j = 0; j < 8; ++j) o0 += row[j] * L.Nmat[j * 8 + 2 * t], o1 += row[j] * L.Nmat[j * 8 + 2 * t + 1];
          const double sg = h < Hused ? L.sig[h] : 0.0;
          v0 = sg * o0, v1 = sg * o1;
        }
        if (h < Hused && c < ncell)
          *reinterpret_cast<double2*>(out + ((size_t)(el0 + c) * H + h) * 8 + 2 * t) = make_double2(v0, v1);
      }
    }
  }
}

__global__ void __launch_bounds__(128) m2d_mma_kernel(Dev L, const double* __restrict__ src, int Hused, double scale,
                                                      double* __restrict__ y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int R = L.P * L.D, H = L.H;
  const int el0 = (blockIdx.x * 4 + warp) * SC_NC;
  if (el0 >= L.n_el) return;
  const int ncell = min(SC_NC, L.n_el - el0);
  const int MT = R / 8, KS = (Hused + 3) / 4;
  for (int m0 = 0; m0 < MT; m0 += SC_MG) {
    double acc[SC_MG][SC_NC][2];
#pragma unroll
    for (int a = 0; a < SC_MG; ++a)
#pragma unroll
      for (int c = 0; c < SC_NC; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    for (int ks = 0; ks < KS; ++ks) {
      const int h = 4 * ks + t;
      const bool hok = h < Hused;
      double af[SC_MG], bf[SC_NC];
#pragma unroll
      for (int a = 0; a < SC_MG; ++a) {
        const int r = 8 * (m0 + a) + g;
        af[a] = (hok && m0 + a < MT) ? L.X[(size_t)r * H + h] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < SC_NC; ++c) bf[c] = (hok && c < ncell) ? src[((size_t)(el0 + c) * H + h) * 8 + g] : 0.0;
#pragma unroll
      for (int a = 0; a < SC_MG; ++a)
#pragma unroll
        for (int c = 0; c < SC_NC; ++c) dmma_8x8x4(acc[a][c][0], acc[a][c][1], af[a], bf[c]);
    }
#pragma unroll
    for (int a = 0; a < SC_MG; ++a) {
      if (m0 + a >= MT) break;
      const int r = 8 * (m0 + a) + g;
#pragma unroll
      for (int c = 0; c < SC_NC; ++c) {
        if (c >= ncell) break;
        double2* yp = reinterpret_cast<double2*>(y + ((size_t)(el0 + c) * R + r) * 8 + 2 * t);
        double2 v = *yp;
        v.x += scale * acc[a][c][0], v.y += scale * acc[a][c][1];
        *yp = v;
      }
    }
  }
}

__global__ void prolong_kernel(Dev F, const double* __restrict__ coarse, double* __restrict__ fine, int Pc, bool add) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int S = F.S, D = F.D, bs = F.bs;
  if (idx >= (int64_t)F.n_el * F.P * bs) return;
  const int i = int(idx % S), d = int((idx / S) % D);
  const int64_t blk = idx / bs;
  const int q = int(blk % F.P), el = int(blk / F.P);
  const double* B = F.upB + (size_t)q * D * D + d * D;
  const double* cb = coarse + ((size_t)el * Pc + F.up[q]) * bs;
  double acc = 0.0;
  for (int e = 0; e < D; ++e) acc += B[e] * cb[e * S + i];
  fine[idx] = add ? fine[idx] + acc : acc;
}

// coarse[el][c] = sum over the children q of c (ascending) of B_q^T fine[el][q]
__global__ void restrict_kernel(Dev F, const double* __restrict__ fine, double* __restrict__ coarse, int Pc) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int S = F.S, D = F.D, bs = F.bs;
  if (idx >= (int64_t)F.n_el * Pc * bs) return;
  const int i = int(idx % S), e = int((idx / S) % D);
  const int64_t blk = idx / bs;
  const int c = int(blk % Pc), el = int(blk / Pc);
  double acc = 0.0;
  for (int k = F.child_ptr[c]; k < F.child_ptr[c + 1]; ++k) {
    const int q = F.child_idx[k];
    const double* B = F.upB + (size_t)q * D * D;
    const double* fb = fine + ((size_t)el * F.P + q) * bs;
    double a2 = 0.0;
    for (int d = 0; d < D; ++d) a2 += B[d * D + e] * fb[d * S + i];
    acc += a2;
  }
  coarse[idx] = acc;
}

// Scatter-implicit block Gauss-Seidel in the reference's order (sweeps.cpp:83-103):
// passes, octants, cells in the octant's upwind order, the octant's patches in turn, the
// cell's moments kept current after every patch. Cells of one hyperplane are independent
// (a cell's moments are its own; its upwind neighbours are on the previous plane), so one
// warp takes a cell and the grid synchronises between planes.
constexpr int GS_WPB = 4;

__host__ __device__ inline size_t gs_warp_doubles(int H, int S, int bs) { return size_t(H) * S + 32 * size_t(bs) + 7 * size_t(bs); }

// shared-memory scratch of one warp
struct GsScratch {
  double *smom, *red, *sr, *szo, *sdz, *sv, *sup;
  __device__ GsScratch(double* base, int H, int S, int bs) {
    smom = base;                  // [H][S] moments of the cell
    red = smom + (size_t)H * S;   // [bs][32]
    sr = red + 32 * bs;           // [bs] right-hand side
    szo = sr + bs;                // [bs] previous iterate
    sdz = szo + bs;               // [bs] znew - zold
    sv = sdz + bs;                // [bs] X sigma (mom - X^T zold)
    sup = sv + bs;                // [3][bs] upwind iterates of the patch
  }
};

// One cell of one octant by one warp: the octant's patches in turn (sweeps.cpp:86-102).
__device__ __forceinline__ void gs_cell(const Dev& L, const double* __restrict__ rhs, double* phi, const Frame& fr, int fi,
                                        int fj, int fk, int pbeg, int np, int lane, const GsScratch& sc) {
  const int S = L.S, D = L.D, bs = L.bs, H = L.H, P = L.P;
  double *smom = sc.smom, *red = sc.red, *sr = sc.sr, *szo = sc.szo, *sdz = sc.sdz, *sv = sc.sv, *sup = sc.sup;
  const int el = fr.el(fi, fj, fk);
  double* gm = L.mom + (size_t)el * H * S;
  // every global load of the cell's first patch step is issued together with the
  // moments (one memory round trip instead of three dependent ones)
  double pre_r = 0.0, pre_zo = 0.0, pre_up[3] = {0.0, 0.0, 0.0};
  if (lane < bs) {
    const int q0 = L.oct_patches[pbeg];
    const size_t blk0 = ((size_t)el * P + q0) * bs;
    pre_r = rhs[blk0 + lane];
    pre_zo = __ldcg(phi + blk0 + lane);
#pragma unroll
    for (int xi = 0; xi < 3; ++xi) {
      const int fc = xi == 0 ? fi : xi == 1 ? fj : fk;
      if (xi >= L.dim || fc == 0) continue;
      const int up = fr.el(fi - (xi == 0), fj - (xi == 1), fk - (xi == 2));
      pre_up[xi] = __ldcg(phi + ((size_t)up * P + q0) * bs + lane);
    }
  }
  for (int k = lane; k < H * S; k += 32) smom[k] = __ldcg(gm + k);
  __syncwarp();
  for (int a = 0; a < np; ++a) {
    const int q = L.oct_patches[pbeg + a];
    const size_t blk = ((size_t)el * P + q) * bs;
    // r = rhs - sum_xi C phi_up; previous iterate. The upwind blocks come from other
    // warps' earlier planes (L2, one coalesced round trip each) and are staged first.
    double rhs_l = pre_r;
    if (lane < bs) {
      if (a == 0) {
#pragma unroll
        for (int xi = 0; xi < 3; ++xi)
          if (xi < L.dim) sup[xi * bs + lane] = pre_up[xi];
        szo[lane] = pre_zo;
      } else {
        for (int xi = 0; xi < L.dim; ++xi) {
          const int fc = xi == 0 ? fi : xi == 1 ? fj : fk;
          if (fc == 0) continue;
          const int up = fr.el(fi - (xi == 0), fj - (xi == 1), fk - (xi == 2));
          sup[xi * bs + lane] = __ldcg(phi + ((size_t)up * P + q) * bs + lane);
        }
        szo[lane] = __ldcg(phi + blk + lane);
        rhs_l = rhs[blk + lane];
      }
    }
    __syncwarp();
    if (lane < bs) {
      double r = rhs_l;
      for (int xi = 0; xi < L.dim; ++xi) {
        const int fc = xi == 0 ? fi : xi == 1 ? fj : fk;
        if (fc == 0) continue;
        const double* C = L.C + (((size_t)q * 3 + xi) * bs + lane) * bs;
        double acc = 0.0;
        for (int c = 0; c < bs; ++c) acc += C[c] * sup[xi * bs + c];
        r -= acc;
      }
      sr[lane] = r;
    }
    __syncwarp();
    // v[d][j] = sum_h X[(q,d)][h] sig_h (mom[h][j] - sum_e X[(q,e)][h] zold[e][j])
    {
      double part[3][8];
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int j = 0; j < 8; ++j) part[d][j] = 0.0;
      for (int h = lane; h < H; h += 32) {
        double xq[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) xq[d] = d < D ? L.X[((size_t)q * D + d) * H + h] : 0.0;
        const double sg = L.sig[h];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= S) break;
          double t = 0.0;
#pragma unroll
          for (int e = 0; e < 3; ++e)
            if (e < D) t += xq[e] * szo[e * S + j];
          const double u = sg * (smom[h * S + j] - t);
#pragma unroll
          for (int d = 0; d < 3; ++d)
            if (d < D) part[d][j] += xq[d] * u;
        }
      }
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (d < D && j < S) red[(d * S + j) * 32 + lane] = part[d][j];
    }
    __syncwarp();
    if (lane < bs) {
      double acc = 0.0;
      for (int m = 0; m < 32; ++m) acc += red[lane * 32 + m];
      sv[lane] = acc;
    }
    __syncwarp();
    if (lane < bs) {  // r += v N
      const int d = lane / S, i = lane - d * S;
      double acc = 0.0;
      for (int j = 0; j < S; ++j) acc += sv[d * S + j] * L.Nmat[j * S + i];
      sr[lane] += acc;
    }
    __syncwarp();
    if (lane < bs) {  // znew = (B - sq N)^-1 r
      const double* Bi = L.BinvGS + ((size_t)q * bs + lane) * bs;
      double acc = 0.0;
      for (int c = 0; c < bs; ++c) acc += Bi[c] * sr[c];
      __stcg(phi + blk + lane, acc);
      sdz[lane] = acc - szo[lane];
    }
    __syncwarp();
    // mom += X_q^T (znew - zold)
    for (int k = lane; k < H * S; k += 32) {
      const int h = k / S, j = k - h * S;
      double acc = 0.0;
      for (int d = 0; d < D; ++d) acc += L.X[((size_t)q * D + d) * H + h] * sdz[d * S + j];
      smom[k] += acc;
    }
    __syncwarp();
  }
  for (int k = lane; k < H * S; k += 32) __stcg(gm + k, smom[k]);
  __syncwarp();
}

__global__ void __launch_bounds__(GS_WPB * 32) coarse_gs_kernel(Dev L, const double* __restrict__ rhs, double* phi, int nu) {
  extern __shared__ __align__(16) double sm[];
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int W = gridDim.x * GS_WPB, gw = blockIdx.x * GS_WPB + wib;
  const GsScratch sc(sm + wib * gs_warp_doubles(L.H, L.S, L.bs), L.H, L.S, L.bs);
  const int nplanes = L.nx + L.ny + L.nz - 2, njk = L.ny * L.nz;
  for (int pass = 0; pass < nu; ++pass)
    for (int oct = 0; oct < 8; ++oct) {
      const int pbeg = L.oct_ptr[oct], np = L.oct_ptr[oct + 1] - pbeg;
      if (np == 0) continue;
      const Frame fr(L, oct);
      for (int pl = 0; pl < nplanes; ++pl) {
        for (int jk = gw; jk < njk; jk += W) {
          const int fj = jk % L.ny, fk = jk / L.ny, fi = pl - fj - fk;
          if (fi < 0 || fi >= L.nx) continue;
          gs_cell(L, rhs, phi, fr, fi, fj, fk, pbeg, np, lane, sc);
        }
        grid.sync();
      }
    }
}

// Dataflow variant (used when every line of cells along x can have its own co-resident warp):
// warp w owns the line (iy, iz) = w for the whole call and walks it in each octant's upwind
// order, so the x-upwind cell and the cell's moments are its own program order. Before a cell
// it waits until the y- and z-upwind lines have finished the same column of the same octant
// sweep (their progress counters: cells finished since the start of the call), and -- write
// after read -- until the downwind lines have finished it in the previous pass. No grid-wide
// barrier: a hyperplane step costs two flag polls instead of a barrier over all CTAs, and
// consecutive octants overlap where the reference's order allows it.
__global__ void __launch_bounds__(GS_WPB * 32) coarse_gs_flow_kernel(Dev L, const double* __restrict__ rhs, double* phi, int nu,
                                                                    int* prog) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int line = blockIdx.x * GS_WPB + wib, njk = L.ny * L.nz;
  if (line >= njk) return;
  const GsScratch sc(sm + wib * gs_warp_doubles(L.H, L.S, L.bs), L.H, L.S, L.bs);
  const int iy = line % L.ny, iz = line / L.ny;
  int n_active = 0;
  for (int oct = 0; oct < 8; ++oct) n_active += L.oct_ptr[oct + 1] > L.oct_ptr[oct] ? 1 : 0;
  int base = 0;  // cells this line has finished before the current octant sweep
  for (int pass = 0; pass < nu; ++pass)
    for (int oct = 0; oct < 8; ++oct) {
      const int pbeg = L.oct_ptr[oct], np = L.oct_ptr[oct + 1] - pbeg;
      if (np == 0) continue;
      const Frame fr(L, oct);
      const int fj = fr.yn ? L.ny - 1 - iy : iy, fk = fr.zn ? L.nz - 1 - iz : iz;
      // neighbour lines: upwind in y / z (read after write), downwind in y / z (write after read)
      const int up_y = fj > 0 ? iz * L.ny + (fr.yn ? iy + 1 : iy - 1) : -1;
      const int up_z = fk > 0 ? (fr.zn ? iz + 1 : iz - 1) * L.ny + iy : -1;
      const int dn_y = fj < L.ny - 1 ? iz * L.ny + (fr.yn ? iy - 1 : iy + 1) : -1;
      const int dn_z = fk < L.nz - 1 ? (fr.zn ? iz - 1 : iz + 1) * L.ny + iy : -1;
      for (int fi = 0; fi < L.nx; ++fi) {
        const int* f = nullptr;
        int need = 0;
        if (lane == 0 && up_y >= 0) f = prog + up_y, need = base + fi + 1;
        if (lane == 1 && up_z >= 0) f = prog + up_z, need = base + fi + 1;
        if (lane == 2 && dn_y >= 0 && pass > 0) f = prog + dn_y, need = base - n_active * L.nx + fi + 1;
        if (lane == 3 && dn_z >= 0 && pass > 0) f = prog + dn_z, need = base - n_active * L.nx + fi + 1;
        bool ok = f == nullptr || ld_relaxed(f) >= need;
        while (!__all_sync(0xffffffffu, ok))
          if (!ok) ok = ld_relaxed(f) >= need;
        fence_acq_rel();
        gs_cell(L, rhs, phi, fr, fi, fj, fk, pbeg, np, lane, sc);
        __syncwarp();
        if (lane == 0) st_release(prog + line, base + fi + 1);
      }
      base += L.nx;
    }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

int blocks_for(int64_t n, int bsz) { return int((n + bsz - 1) / bsz); }

}  // namespace

template <int BS>
void launch_apply_L_t(const Dev& L, const double* x, double* y, double alpha, double beta, const double* f, cudaStream_t s) {
  const size_t smem = sizeof(double) * size_t(1 + L.dim) * BS * BS;
  const int by = std::max(1, std::min((L.n_el + 127) / 128, std::max(1, 4 * 148 / std::max(L.P, 1))));
  apply_L_block_kernel<BS><<<dim3(L.P, by), 128, smem, s>>>(L, x, y, alpha, beta, f);
}

template <int BS>
void launch_apply_L_mma(const Dev& L, const double* x, double* y, double alpha, double beta, const double* f, cudaStream_t s) {
  const int ntile = (L.n_el + 7) / 8;
  const int by = std::max(1, std::min((ntile + 3) / 4, std::max(1, 6 * 148 / std::max(L.P, 1))));
  apply_L_mma_kernel<BS><<<dim3(L.P, by), 128, 0, s>>>(L, x, y, alpha, beta, f);
}

template <int BS>
void launch_sweep_t(const Dev& L, const double* rhs, double* z, int threads, cudaStream_t s) {
  const size_t smem = sizeof(double) * size_t(1 + L.dim) * BS * BS;
  sweep_block_kernel<BS><<<L.P, threads, smem, s>>>(L, rhs, z);
}

void launch_apply_L(const Dev& L, const double* x, double* y, double alpha, double beta, const double* f, cudaStream_t s) {
  const int64_t n = (int64_t)L.n_el * L.P * L.bs;
  if (n == 0) return;
  if (!f) beta = 0.0;
  switch (L.bs) {
    case 1: return launch_apply_L_t<1>(L, x, y, alpha, beta, f, s);
    case 3: return launch_apply_L_t<3>(L, x, y, alpha, beta, f, s);
    case 8: return launch_apply_L_mma<8>(L, x, y, alpha, beta, f, s);
    case 12: return launch_apply_L_t<12>(L, x, y, alpha, beta, f, s);
    case 24: return launch_apply_L_mma<24>(L, x, y, alpha, beta, f, s);
    default: apply_L_kernel<<<blocks_for(n, 256), 256, 0, s>>>(L, x, y, alpha, beta, f);
  }
}

void launch_sweep(const Dev& L, const double* rhs, double* z, cudaStream_t s) {
  if (L.P == 0 || L.n_el == 0) return;
  const int threads = std::min(256, std::max(32, (L.ny * L.nz + 31) / 32 * 32));
  switch (L.bs) {
    case 1: return launch_sweep_t<1>(L, rhs, z, threads, s);
    case 3: return launch_sweep_t<3>(L, rhs, z, threads, s);
    case 8:
      if (L.plane_cells) {
        sweep_mma_kernel<8><<<L.P, 256, 0, s>>>(L, rhs, z);
        return;
      }
      return launch_sweep_t<8>(L, rhs, z, threads, s);
    case 12: return launch_sweep_t<12>(L, rhs, z, threads, s);
    case 24:
      if (L.plane_cells) {
        sweep_mma_kernel<24><<<L.P, 256, 0, s>>>(L, rhs, z);
        return;
      }
      return launch_sweep_t<24>(L, rhs, z, threads, s);
    default: {
      const size_t smem = sizeof(double) * size_t(1 + L.dim) * L.bs * L.bs;
      sweep_kernel<<<L.P, threads, smem, s>>>(L, rhs, z);
    }
  }
}

void launch_d2m(const Dev& L, const double* phi, int order, bool apply_sigma_N, double* out, cudaStream_t s) {
  const int Hused = (order + 1) * (order + 1);
  const size_t smem = sizeof(double) * size_t(Hused) * L.S;
  if (smem > 200 * 1024) throw std::invalid_argument("reference-shape scatter: (order+1)^2 * S moments exceed shared memory");
  if (L.S == 8 && (L.P * L.D) % 8 == 0) {
    d2m_mma_kernel<<<(L.n_el + 4 * SC_NC - 1) / (4 * SC_NC), 128, 0, s>>>(L, phi, Hused, apply_sigma_N, out);
    return;
  }
  switch (L.S) {
    case 1: d2m_block_kernel<1><<<L.n_el, 128, 0, s>>>(L, phi, Hused, apply_sigma_N, out); return;
    case 4: d2m_block_kernel<4><<<L.n_el, 128, 0, s>>>(L, phi, Hused, apply_sigma_N, out); return;
    case 8: d2m_block_kernel<8><<<L.n_el, 128, 0, s>>>(L, phi, Hused, apply_sigma_N, out); return;
    default: break;
  }
  if (smem > 48 * 1024) ck(cudaFuncSetAttribute(d2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
  d2m_kernel<<<L.n_el, 128, smem, s>>>(L, phi, Hused, apply_sigma_N, out);
}

void launch_m2d(const Dev& L, const double* src, int order, double scale, double* y, cudaStream_t s) {
  const int Hused = (order + 1) * (order + 1);
  const size_t smem = sizeof(double) * size_t(Hused) * L.S;
  if (smem > 200 * 1024) throw std::invalid_argument("reference-shape scatter: (order+1)^2 * S moments exceed shared memory");
  if (L.S == 8 && (L.P * L.D) % 8 == 0) {
    m2d_mma_kernel<<<(L.n_el + 4 * SC_NC - 1) / (4 * SC_NC), 128, 0, s>>>(L, src, Hused, scale, y);
    return;
  }
  if (L.XT && (L.S == 1 || L.S == 4 || L.S == 8)) {
    auto k = L.S == 1 ? m2d_block_kernel<1> : L.S == 4 ? m2d_block_kernel<4> : m2d_block_kernel<8>;
    if (smem > 48 * 1024) ck(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
    k<<<L.n_el, 128, smem, s>>>(L, src, Hused, scale, y);
    return;
  }
  if (smem > 48 * 1024) ck(cudaFuncSetAttribute(m2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
  m2d_kernel<<<L.n_el, 128, smem, s>>>(L, src, Hused, scale, y);
}

void launch_prolong(const Dev& F, const double* coarse, double* fine, int Pc, bool add, cudaStream_t s) {
  const int64_t n = (int64_t)F.n_el * F.P * F.bs;
  if (n == 0) return;
  prolong_kernel<<<blocks_for(n, 256), 256, 0, s>>>(F, coarse, fine, Pc, add);
}

void launch_restrict(const Dev& F, const double* fine, double* coarse, int Pc, cudaStream_t s) {
  const int64_t n = (int64_t)F.n_el * Pc * F.bs;
  if (n == 0) return;
  restrict_kernel<<<blocks_for(n, 256), 256, 0, s>>>(F, fine, coarse, Pc);
}

void launch_coarse_gs(const Dev& L, const double* rhs, int nu, double* phi, cudaStream_t s) {
  if (nu <= 0 || L.n_el == 0) return;
  launch_d2m(L, phi, L.order, false, L.mom, s);  // moments of the current iterate (sweeps.cpp:74-79)
  const size_t smem = sizeof(double) * GS_WPB * gs_warp_doubles(L.H, L.S, L.bs);
  if (smem > 200 * 1024) throw std::invalid_argument("reference-shape coarse GS: moments exceed shared memory");
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  Dev Lc = L;
  const double* r = rhs;
  const int lines = L.ny * L.nz, want = (lines + GS_WPB - 1) / GS_WPB;
  // dataflow kernel when every line of cells gets its own co-resident warp
  ck(cudaFuncSetAttribute(coarse_gs_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_gs_flow_kernel, GS_WPB * 32, smem), "occupancy");
  if (L.gs_prog && want <= sms * per_sm) {
    ck(cudaMemsetAsync(L.gs_prog, 0, sizeof(int) * size_t(lines), s), "memset");
    int* prog = L.gs_prog;
    void* args[] = {&Lc, &r, &phi, &nu, &prog};
    ck(cudaLaunchCooperativeKernel((const void*)coarse_gs_flow_kernel, dim3(want), dim3(GS_WPB * 32), args, smem, s),
       "coarse_gs cooperative launch");
    return;
  }
  ck(cudaFuncSetAttribute(coarse_gs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_gs_kernel, GS_WPB * 32, smem), "occupancy");
  const int grid = std::max(1, std::min(want, sms * std::max(per_sm, 1)));  // at most ny*nz cells per plane
  void* args[] = {&Lc, &r, &phi, &nu};
  ck(cudaLaunchCooperativeKernel((const void*)coarse_gs_kernel, dim3(grid), dim3(GS_WPB * 32), args, smem, s),
     "coarse_gs cooperative launch");
}

}  // namespace gen
}  // namespace stamg_b200
