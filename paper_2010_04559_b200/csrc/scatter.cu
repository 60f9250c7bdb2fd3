// Legendre scatter operator on sm_100a FP64 tensor cores (DMMA):
// apply_scatter_into (scatter.cpp:110-135) as two batched GEMMs.
//
//  D2M: MOM[h][(el,i)] = sum_q X[q][h] * PHI[q][(el,i)]      (M=H, N=n_el*4, K=P)
//       epilogue: SRC[el][h][i] = sig[mat(el)][h] * sum_j MOM[h][(el,j)] N[j][i]
//       (the 4 spatial dofs of an element sit in a lane pair; one shuffle)
//  M2D: Y[el][q][i] = beta*Y + scale * sum_h X[q][h] * SRC[el][h][i]
//                     (+ isotropic external source, rank-1 in (q, i))
//
// PHI is read straight from the reference layout: for a tile of 16 elements
// the (q-chunk x 4) panel of each element is contiguous. Tiles are staged
// global->shared with cp.async (3 stages); each warp owns a 32x32 output
// block = 4x4 m8n8k4 DMMA accumulators (tcgen05 has no f64 kind, so
// mma.sync...f64 is the FP64 tensor path on sm_100a).
#include <stdexcept>

#include "common.cuh"
#include "kernels.hpp"

namespace stamg_b200 {
namespace {

#ifndef STAMG_GEMM_BK
#define STAMG_GEMM_BK 16
#endif
#ifndef STAMG_GEMM_NSTAGE
#define STAMG_GEMM_NSTAGE 3
#endif
#ifndef STAMG_GEMM_TMA
#define STAMG_GEMM_TMA 1  // 1: tiles staged by TMA bulk copies (cp.async.bulk + mbarrier); 0: cp.async (LDGSTS)
#endif
#ifndef STAMG_GEMM_SWAP
#define STAMG_GEMM_SWAP 0  // 1: output-row tiles fastest in the grid (Phi / src panel reuse in L2)
#endif
constexpr int BM = 64, BN = 64, BK = STAMG_GEMM_BK, NSTAGE = STAMG_GEMM_NSTAGE;
constexpr int LDS = BM + 4;  // padded row (conflict-free fragment loads)
constexpr int LDB = BN + 4;
constexpr int kThreads = 128;

// Output-row tiling of the D2M GEMM (M = harmonics of the call): WM warp rows
// x 2 warp columns, each warp MI x 4 m8n8k4 blocks, so BM = 8*MI*WM rows by
// BN = 64 columns. The harmonic parity classes of the folded scatter have 153 /
// 136 / 120 rows at N = 32: 64-row tiles pad them to 192 (71 % useful work);
// 24-row warp strips cover them in one CTA tile of 168 / 144 / 120 rows.
// B tile in shared memory: cp.async path [k][LDB] (k-major, padded); TMA path
// [e][k][4] (element-major, the panel order of the reference layout, one bulk copy
// per element; a fragment load covers 2 elements x 128 contiguous bytes: conflict free)
constexpr int kStageB = STAMG_GEMM_TMA ? BN * BK : BK * LDB;
template <int MI, int WM>
struct RowTile {
  static constexpr int kBM = 8 * MI * WM, kLDA = kBM + 4, kThreads = 64 * WM;
  static constexpr int kStage = BK * kLDA + kStageB;
};

// A tile: sA[k][m] = A_src[(k0+k) * lda + m0 + m]   (rows of k contiguous in m)
template <int TBM, int TLDA, int TT>
__device__ __forceinline__ void load_tile_rows(double* sA, const double* src, int lda, int k0, int m0, int krows,
                                               int tid) {
  // BK x TBM doubles in 16-byte chunks
#pragma unroll
  for (int it = 0; it < (BK * TBM / 2 + TT - 1) / TT; ++it) {
    const int chunk = tid + it * TT;
    if ((BK * TBM / 2) % TT != 0 && chunk >= BK * TBM / 2) break;
    const int k = chunk / (TBM / 2), mm = (chunk % (TBM / 2)) * 2;
    const bool ok = (k0 + k) < krows;
    const double* g = src + (ok ? (size_t)(k0 + k) * lda + m0 + mm : 0);
    cp_async16(sA + k * TLDA + mm, g, ok);
  }
}

// D2M B tile: sB[k][e*4+i] = phi[((el0+e)*P + q0+k)*4 + i] (or its wavefront-layout block)
template <int TT>
__device__ __forceinline__ void load_phi_tile(double* sB, const double* phi, int P, int n_el, int q0, int el0,
                                              int tid, const WLGeom& wl) {
#pragma unroll
  for (int it = 0; it < (BK * BN / 2 + TT - 1) / TT; ++it) {
    const int chunk = tid + it * TT;             // e (16) x k (BK) x half (2)
    if ((BK * BN / 2) % TT != 0 && chunk >= BK * BN / 2) break;
    const int half = chunk & 1, k = (chunk >> 1) & (BK - 1), e = chunk / (2 * BK);
    const bool ok = (el0 + e) < n_el && (q0 + k) < P;
    size_t off = 0;
    if (ok) off = wl.nd ? (size_t)wl_block(wl, el0 + e, q0 + k) * 4 : ((size_t)(el0 + e) * P + q0 + k) * 4;
    cp_async16(sB + k * LDB + e * 4 + half * 2, phi + off + (ok ? half * 2 : 0), ok);
  }
}

// M2D B tile: sB[k][e*4+i] = src[((el0+e)*Hp + h0+k)*4 + i], zero for h0+k >= krows
template <int TT>
__device__ __forceinline__ void load_src_tile(double* sB, const double* src, int Hp, int n_el, int h0, int el0,
                                              int krows, int tid) {
#pragma unroll
  for (int it = 0; it < (BK * BN / 2) / TT; ++it) {
    const int chunk = tid + it * TT;
    const int half = chunk & 1, k = (chunk >> 1) & (BK - 1), e = chunk / (2 * BK);
    const bool ok = (el0 + e) < n_el && (h0 + k) < krows;
    const double* g = src + (ok ? (((size_t)(el0 + e) * Hp + h0 + k) * 4 + half * 2) : 0);
    cp_async16(sB + k * LDB + e * 4 + half * 2, g, ok);
  }
}

template <int MI, int TLDA>
__device__ __forceinline__ void mma_stage(const double* sA, const double* sB, double (&acc)[MI][4][2], int wm, int wn,
                                          int g, int t) {
#pragma unroll
  for (int kk = 0; kk < BK; kk += 4) {
    double a[MI], b[4];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[i] = sA[(kk + t) * TLDA + wm * (8 * MI) + i * 8 + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if constexpr (STAMG_GEMM_TMA) {
        const int n = wn * 32 + j * 8 + g;  // column (e, i) = (n / 4, n % 4)
        b[j] = sB[(n >> 2) * (BK * 4) + (kk + t) * 4 + (n & 3)];
      } else {
        b[j] = sB[(kk + t) * LDB + wn * 32 + j * 8 + g];
      }
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

// the first `steps` k-steps (of 4 rows) of a stage: the tail tile of a short k-loop
template <int MI, int TLDA>
__device__ __forceinline__ void mma_steps(const double* sA, const double* sB, double (&acc)[MI][4][2], int wm, int wn,
                                          int g, int t, int steps) {
#pragma unroll 1
  for (int kk = 0; kk < steps * 4; kk += 4) {
    double a[MI], b[4];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[i] = sA[(kk + t) * TLDA + wm * (8 * MI) + i * 8 + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = wn * 32 + j * 8 + g;
      b[j] = sB[(n >> 2) * (BK * 4) + (kk + t) * 4 + (n & 3)];
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

// ---- TMA staging: warp 0 fills stage `kt % NSTAGE` with bulk copies that complete on
// that stage's mbarrier (expect_tx set first by lane 0); every thread waits on the
// barrier's phase parity (kt / NSTAGE) & 1. Stages are zeroed once at kernel start, so
// the rows a tail tile does not copy hold finite values (multiplied by zero A rows).
__device__ __forceinline__ void gemm_tma_init(double* smem, int stage_doubles, unsigned long long* bars, int tid,
                                              int nthreads) {
  for (int c = tid; c < NSTAGE * stage_doubles / 2; c += nthreads)
    reinterpret_cast<double2*>(smem)[c] = make_double2(0.0, 0.0);
  if (tid == 0)
    for (int st = 0; st < NSTAGE; ++st) mbar_init_cta(bars + st, 1);
  fence_proxy_async_smem();
  __syncthreads();
}

// D2M stage: A = BK rows of X (TBM harmonics each, zero-padded to Pk rows), B = the
// (k-chunk x 4) panel of each element (reference layout: one run; wavefront layout: one
// 256-byte run per 8-direction group)
template <int TBM, int TLDA>
__device__ __forceinline__ void d2m_tma_issue(const D2MParams& p, double* st, unsigned long long* bar, int kt, int h0,
                                              int el0, int lane) {
  const int k0 = kt * BK;
  const int ne = min(BN / 4, (p.el_base + p.n_el) - el0), kv = min(BK, p.P - k0);
  if (lane == 0) mbar_expect_tx(bar, unsigned(BK * TBM * 8 + ne * kv * 32));
  __syncwarp();
  for (int c = lane; c < BK; c += 32) bulk_g2s(st + c * TLDA, p.X + (size_t)(k0 + c) * p.Hp + h0, TBM * 8, bar);
  double* sB = st + BK * TLDA;
  if (p.wl.nd) {
    for (int c = lane; c < ne * (kv / 8); c += 32) {
      const int e = c / (kv / 8), gi = c - e * (kv / 8);
      bulk_g2s(sB + e * (BK * 4) + gi * 32, p.phi + (size_t)wl_block(p.wl, el0 + e, k0 + 8 * gi) * 4, 256, bar);
    }
  } else {
    for (int e = lane; e < ne; e += 32)
      bulk_g2s(sB + e * (BK * 4), p.phi + ((size_t)(el0 + e) * p.P + k0) * 4, unsigned(kv * 32), bar);
  }
}

// grid: x = element tiles (16 elements), y = harmonic tiles (BM rows)
#ifndef STAMG_D2M_MINB
#define STAMG_D2M_MINB 2  // resident CTAs per SM the register budget is sized for (A/B at c5: 1 -> 2 = D2M -19 %)
#endif
template <int MI, int WM>
__global__ void __launch_bounds__(RowTile<MI, WM>::kThreads, STAMG_D2M_MINB) d2m_kernel(D2MParams p) {
  using T = RowTile<MI, WM>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, wm = warp >> 1, wn = warp & 1;
  const int el0 = p.el_base + (STAMG_GEMM_SWAP ? blockIdx.y : blockIdx.x) * (BN / 4);
  const int h0 = (STAMG_GEMM_SWAP ? blockIdx.x : blockIdx.y) * T::kBM;
  double acc[MI][4][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (p.P + BK - 1) / BK;
#if STAMG_GEMM_TMA
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + NSTAGE * T::kStage);
  gemm_tma_init(smem, T::kStage, bars, tid, T::kThreads);
  if (warp == 0)
    for (int s = 0; s < NSTAGE - 1 && s < nk; ++s)
      d2m_tma_issue<T::kBM, T::kLDA>(p, smem + s * T::kStage, bars + s, s, h0, el0, lane);
  for (int kt = 0; kt < nk; ++kt) {
    const int nxt = kt + NSTAGE - 1;  // its stage was released by the barrier closing iteration kt - 1
    if (warp == 0 && nxt < nk)
      d2m_tma_issue<T::kBM, T::kLDA>(p, smem + (nxt % NSTAGE) * T::kStage, bars + nxt % NSTAGE, nxt, h0, el0, lane);
    mbar_wait_parity(bars + kt % NSTAGE, unsigned(kt / NSTAGE) & 1u);
    const double* st = smem + (kt % NSTAGE) * T::kStage;
    mma_stage<MI, T::kLDA>(st, st + BK * T::kLDA, acc, wm, wn, g, t);
    __syncthreads();
  }
#else
  const int Pk = nk * BK;  // X has zero rows up to Pk
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nk) {
      double* st = smem + s * T::kStage;
      load_tile_rows<T::kBM, T::kLDA, T::kThreads>(st, p.X, p.Hp, s * BK, h0, Pk, tid);
      load_phi_tile<T::kThreads>(st + BK * T::kLDA, p.phi, p.P, (p.el_base + p.n_el), s * BK, el0, tid, p.wl);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int nxt = kt + NSTAGE - 1;
    if (nxt < nk) {
      double* st = smem + (nxt % NSTAGE) * T::kStage;
      load_tile_rows<T::kBM, T::kLDA, T::kThreads>(st, p.X, p.Hp, nxt * BK, h0, Pk, tid);
      load_phi_tile<T::kThreads>(st + BK * T::kLDA, p.phi, p.P, (p.el_base + p.n_el), nxt * BK, el0, tid, p.wl);
    }
    cp_async_commit();
    cp_async_wait<NSTAGE - 1>();
    __syncthreads();
    const double* st = smem + (kt % NSTAGE) * T::kStage;
    mma_stage<MI, T::kLDA>(st, st + BK * T::kLDA, acc, wm, wn, g, t);
    __syncthreads();
  }
  cp_async_wait<0>();
#endif

  // epilogue: complete the element's 4 dofs from the partner lane, apply N and sigma
  // (rows Hused <= h < h0 + BM of the call's region are written as zeros)
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int h = h0 + wm * (8 * MI) + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double o0 = __shfl_xor_sync(0xffffffffu, acc[i][j][0], 1);
      const double o1 = __shfl_xor_sync(0xffffffffu, acc[i][j][1], 1);
      const bool lo = (t & 1) == 0;
      const double m0 = lo ? acc[i][j][0] : o0, m1 = lo ? acc[i][j][1] : o1;
      const double m2 = lo ? o0 : acc[i][j][0], m3 = lo ? o1 : acc[i][j][1];
      const int e = (wn * 32 + j * 8) / 4 + (t >> 1);
      const int el = el0 + e;
      const int i0 = (t & 1) * 2;
      if (el < (p.el_base + p.n_el) && h < p.Hrows) {
        double s0 = 0.0, s1 = 0.0;
        if (h < p.Hused) {
          const int mt = p.mat ? p.mat[el] : 0;
          const double sg = p.sig[(size_t)mt * p.Hp + h];
          s0 = sg * (m0 * p.N[0 * 4 + i0] + m1 * p.N[1 * 4 + i0] + m2 * p.N[2 * 4 + i0] + m3 * p.N[3 * 4 + i0]);
          s1 = sg * (m0 * p.N[0 * 4 + i0 + 1] + m1 * p.N[1 * 4 + i0 + 1] + m2 * p.N[2 * 4 + i0 + 1] +
                     m3 * p.N[3 * 4 + i0 + 1]);
        }
        *reinterpret_cast<double2*>(p.src + ((size_t)el * p.Hp + h) * 4 + i0) = make_double2(s0, s1);
      }
    }
  }
}

// output block of (patch q, element el, dof pair i0) in y
__device__ __forceinline__ double* m2d_out(const M2DParams& p, int el, int q, int i0) {
  return p.y + (p.wl.nd ? (size_t)wl_block(p.wl, el, q) * 4 : ((size_t)el * p.P + q) * 4) + i0;
}

// grid: x = element tiles (16), y = patch tiles (64). PRE (beta != 0): the old y
// of the tile is loaded into registers before the k-loop, so the read-modify-write
// epilogue does not expose a DRAM round trip (the MG levels' M2D has K = 25..81:
// a few k-steps only)
#ifndef STAMG_M2D_WM
#define STAMG_M2D_WM 2  // A/B knob: warp rows of the M2D tile (32 patch rows each); c5 A/B: 1 / 2 / 4 = 97.0 / 83.7 / 88.4 ms
#endif
constexpr int M2D_BM = 32 * STAMG_M2D_WM, M2D_LDA = M2D_BM + 4, M2D_THREADS = 64 * STAMG_M2D_WM;
constexpr int M2D_STAGE = BK * M2D_LDA + kStageB;

#ifndef STAMG_M2D_MINB
#define STAMG_M2D_MINB 3  // resident CTAs per SM the beta != 0 M2D registers are sized for (230 -> 168 regs; c4 MG-level M2D 6.97 -> 5.90 ms)
#endif
#ifndef STAMG_M2D_PATCH_FASTEST
// 1: CTAs of one element tile are consecutive (1D grid, patch tiles fastest), so the tile's
// src panel comes from DRAM once and from L2 for the other patch tiles; X^T (a few MB) stays
// L2-resident. With element tiles fastest the whole src array (268 MB at config 4's MG level,
// more than L2) was streamed from DRAM once per patch tile: 14.2 GB read per launch against
// 6.3 GB algorithmic (ncu, profiles/r02_c4_kernels.txt).
#define STAMG_M2D_PATCH_FASTEST 1
#endif
// Measured and not kept (profiles/r02_c4_kernels.txt): one CTA walking 4 / 8 / 16 element tiles
// with a single TMA pipeline over the (tile, k-tile) pairs -- no pipeline refill or barrier
// setup per tile -- ran the K = 81 M2D in 7.5 / 7.5 / 7.6 ms against 6.4 ms for one tile per
// CTA, and 8.4 ms with two instead of three resident CTAs: what hides a tile's epilogue and
// first-copy latency is other CTAs' tensor work, so more, shorter CTAs win.
template <bool PRE_>
constexpr int m2d_minb() { return PRE_ ? STAMG_M2D_MINB : 4; }  // beta == 0: 4 CTAs/SM (<= 128 registers)
template <bool PRE>
__global__ void __launch_bounds__(M2D_THREADS, m2d_minb<PRE>()) m2d_kernel(M2DParams p) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, wm = warp >> 1, wn = warp & 1;
#if STAMG_M2D_PATCH_FASTEST
  const unsigned gq = (p.P + M2D_BM - 1) / M2D_BM, te = blockIdx.x / gq, tq = blockIdx.x - te * gq;
  const int el0 = p.el_base + int(te) * (BN / 4), q0 = int(tq) * M2D_BM;
#else
  const int el0 = p.el_base + (STAMG_GEMM_SWAP ? blockIdx.y : blockIdx.x) * (BN / 4);
  const int q0 = (STAMG_GEMM_SWAP ? blockIdx.x : blockIdx.y) * M2D_BM;
#endif
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double2 oldv[PRE ? 4 : 1][PRE ? 4 : 1];
  if constexpr (PRE) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = q0 + wm * 32 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int el = el0 + (wn * 32 + j * 8) / 4 + (t >> 1);
        oldv[i][j] = (q < p.P && el < (p.el_base + p.n_el)) ? *reinterpret_cast<const double2*>(m2d_out(p, el, q, (t & 1) * 2))
                                               : make_double2(0.0, 0.0);
      }
    }
  }

  const int nk = (p.Hused + BK - 1) / BK;
#if STAMG_GEMM_TMA
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + NSTAGE * M2D_STAGE);
  // no zero fill: every A row and B row a k-step reads is copied or zeroed by the tail code, and
  // B columns of elements past the end only feed accumulators that are never stored
  if (tid == 0)
    for (int st = 0; st < NSTAGE; ++st) mbar_init_cta(bars + st, 1);
  fence_proxy_async_smem();
  __syncthreads();
  // stage: A = rows h of X^T (M2D_BM patches each), B = the (h-chunk x 4) panel of src per
  // element; rows h >= Hused are not copied (their A rows are zeroed in the tail tile)
  auto issue = [&](int kt) {
    const int k0 = kt * BK, st_i = kt % NSTAGE;
    double* st = smem + st_i * M2D_STAGE;
    const int ne = min(BN / 4, (p.el_base + p.n_el) - el0), kv = min(BK, p.Hused - k0);
    if (lane == 0) mbar_expect_tx(bars + st_i, unsigned(kv * M2D_BM * 8 + ne * kv * 32));
    __syncwarp();
    for (int c = lane; c < kv; c += 32)
      bulk_g2s(st + c * M2D_LDA, p.XT + (size_t)(k0 + c) * p.Pp + q0, M2D_BM * 8, bars + st_i);
    for (int e = lane; e < ne; e += 32)
      bulk_g2s(st + BK * M2D_LDA + e * (BK * 4), p.src + ((size_t)(el0 + e) * p.Hp + k0) * 4, unsigned(kv * 32),
               bars + st_i);
  };
  if (warp == 0)
    for (int s = 0; s < NSTAGE - 1 && s < nk; ++s) issue(s);
  for (int kt = 0; kt < nk; ++kt) {
    const int nxt = kt + NSTAGE - 1;
    if (warp == 0 && nxt < nk) issue(nxt);
    mbar_wait_parity(bars + kt % NSTAGE, unsigned(kt / NSTAGE) & 1u);
    double* st = smem + (kt % NSTAGE) * M2D_STAGE;
    const int kv = p.Hused - kt * BK;
    if (kv < BK) {
      // tail tile (CTA-uniform): only the k-steps that hold copied rows run; the rows that pad
      // the last step to 4 are zeroed in A and in B (a stage is never zero-filled as a whole)
      const int kv4 = (kv + 3) & ~3, pad = kv4 - kv;
      for (int c = tid; c < pad * M2D_LDA; c += M2D_THREADS) st[kv * M2D_LDA + c] = 0.0;
      double* sB = st + BK * M2D_LDA;
      for (int c = tid; c < (BN / 4) * pad * 4; c += M2D_THREADS) {
        const int e = c / (pad * 4), w = c - e * (pad * 4);
        sB[e * (BK * 4) + kv * 4 + w] = 0.0;
      }
      __syncthreads();
      mma_steps<4, M2D_LDA>(st, sB, acc, wm, wn, g, t, kv4 / 4);
    } else {
      mma_stage<4, M2D_LDA>(st, st + BK * M2D_LDA, acc, wm, wn, g, t);
    }
    __syncthreads();
  }
#else
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nk) {
      double* st = smem + s * M2D_STAGE;
      load_tile_rows<M2D_BM, M2D_LDA, M2D_THREADS>(st, p.XT, p.Pp, s * BK, q0, p.Hused, tid);
      load_src_tile<M2D_THREADS>(st + BK * M2D_LDA, p.src, p.Hp, (p.el_base + p.n_el), s * BK, el0, p.Hused, tid);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int nxt = kt + NSTAGE - 1;
    if (nxt < nk) {
      double* st = smem + (nxt % NSTAGE) * M2D_STAGE;
      load_tile_rows<M2D_BM, M2D_LDA, M2D_THREADS>(st, p.XT, p.Pp, nxt * BK, q0, p.Hused, tid);
      load_src_tile<M2D_THREADS>(st + BK * M2D_LDA, p.src, p.Hp, (p.el_base + p.n_el), nxt * BK, el0, p.Hused, tid);
    }
    cp_async_commit();
    cp_async_wait<NSTAGE - 1>();
    __syncthreads();
    const double* st = smem + (kt % NSTAGE) * M2D_STAGE;
    mma_stage<4, M2D_LDA>(st, st + BK * M2D_LDA, acc, wm, wn, g, t);
    __syncthreads();
  }
  cp_async_wait<0>();
#endif

  constexpr double inv4pi = 0.07957747154594767;  // 1 / (4 pi)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = q0 + wm * 32 + i * 8 + g;
    if (q >= p.P) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = (wn * 32 + j * 8) / 4 + (t >> 1);
      const int el = el0 + e;
      if (el >= (p.el_base + p.n_el)) continue;
      const int i0 = (t & 1) * 2;
      double* yp = m2d_out(p, el, q, i0);
      double v0 = p.scale * acc[i][j][0], v1 = p.scale * acc[i][j][1];
      if (p.ext_q) {
        const double c = p.ext_q[el] * inv4pi * p.area[q];
        v0 += c * p.nsum[i0], v1 += c * p.nsum[i0 + 1];
      }
      if constexpr (PRE) {
        v0 += p.beta * oldv[i][j].x, v1 += p.beta * oldv[i][j].y;
      } else if (p.beta != 0.0) {
        const double2 old = *reinterpret_cast<const double2*>(yp);
        v0 += p.beta * old.x, v1 += p.beta * old.y;
      }
      *reinterpret_cast<double2*>(yp) = make_double2(v0, v1);
    }
  }
}

constexpr size_t kBarBytes = STAMG_GEMM_TMA ? NSTAGE * sizeof(unsigned long long) : 0;  // stage mbarriers
size_t gemm_smem() { return sizeof(double) * NSTAGE * M2D_STAGE + kBarBytes; }

template <int MI, int WM>
void launch_d2m_tile(const D2MParams& p, cudaStream_t s) {
  using T = RowTile<MI, WM>;
  const size_t smem = sizeof(double) * NSTAGE * T::kStage + kBarBytes;
  // per launch: the attribute is per device (contexts may live on different GPUs)
  cudaFuncSetAttribute(d2m_kernel<MI, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const unsigned ge = (p.n_el + BN / 4 - 1) / (BN / 4), gh = (p.Hused + T::kBM - 1) / T::kBM;
  dim3 grid = STAMG_GEMM_SWAP ? dim3(gh, ge) : dim3(ge, gh);
  d2m_kernel<MI, WM><<<grid, T::kThreads, smem, s>>>(p);
}

// Walsh-Hadamard transform over the G = 2^na members of an orbit (unnormalised):
// out[c] = sum_g (-1)^popcount(c & g) in[g]
template <int G>
__device__ __forceinline__ void wht(double (&v)[G][4]) {
#pragma unroll
  for (int bit = 1; bit < G; bit <<= 1)
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (!(g & bit))
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double a = v[g][i], b = v[g | bit][i];
          v[g][i] = a + b, v[g | bit][i] = a - b;
        }
}

// Phi[c][el][r][i] = sum_g chi_c(g) phi[el][orbit[r][g]][i]
#ifndef STAMG_FOLD_MINB
#define STAMG_FOLD_MINB 1  // A/B knob: resident 256-thread CTAs per SM the fold/unfold registers are sized for
#endif
template <int G>
__global__ void __launch_bounds__(256, STAMG_FOLD_MINB) fold_kernel(const double* __restrict__ phi, double* __restrict__ Phi, const int* __restrict__ orbit,
                            int n_el, int el0, int el1, int P, int R, WLGeom wl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)(el1 - el0) * R) return;
  const int e = int(idx / R), r = int(idx - (int64_t)e * R), el = el0 + e;
  const double* src[G];  // member addresses first, then the G block loads back to back
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int q = orbit[r * G + g];
    src[g] = phi + (wl.nd ? (size_t)wl_block(wl, el, q) * 4 : ((size_t)el * P + q) * 4);
  }
  double v[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const dbl4 a = ld_block(src[g]);
    v[g][0] = a.x, v[g][1] = a.y, v[g][2] = a.z, v[g][3] = a.w;
  }
  wht<G>(v);
#pragma unroll
  for (int c = 0; c < G; ++c) st_block(Phi + (((size_t)c * n_el + el) * R + r) * 4, dbl4{v[c][0], v[c][1], v[c][2], v[c][3]});
}

// y[el][orbit[r][g]][i] = beta*y + scale * sum_c chi_c(g) Y[c][el][r][i] (+ isotropic source)
template <int G, bool BETA>
__global__ void __launch_bounds__(256, STAMG_FOLD_MINB) unfold_kernel(const double* __restrict__ Y, double* __restrict__ y, const int* __restrict__ orbit,
                              int n_el, int el0, int el1, int P, int R, double scale, double beta,
                              const double* __restrict__ ext_q, const double* __restrict__ area, double4 nsum, WLGeom wl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)(el1 - el0) * R) return;
  const int e = int(idx / R), r = int(idx - (int64_t)e * R), el = el0 + e;
  // orbit members and their source weights first: the block stores below are
  // ordered asm (memory clobber), so loads left between them would serialise
  double* o[G];
  double ar[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int q = orbit[r * G + g];
    o[g] = y + (wl.nd ? (size_t)wl_block(wl, el, q) * 4 : ((size_t)el * P + q) * 4);
    ar[g] = ext_q ? area[q] : 0.0;
  }
  double v[G][4];
#pragma unroll
  for (int c = 0; c < G; ++c) {
    const dbl4 a = ld_block(Y + (((size_t)c * n_el + el) * R + r) * 4);
    v[c][0] = a.x, v[c][1] = a.y, v[c][2] = a.z, v[c][3] = a.w;
  }
  wht<G>(v);
  constexpr double inv4pi = 0.07957747154594767;
  const double qel = ext_q ? ext_q[el] * inv4pi : 0.0;
  // all reads of the old y before the first store (same reason as above)
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double w0 = scale * v[g][0], w1 = scale * v[g][1], w2 = scale * v[g][2], w3 = scale * v[g][3];
    if (ext_q) {
      const double c = qel * ar[g];
      w0 += c * nsum.x, w1 += c * nsum.y, w2 += c * nsum.z, w3 += c * nsum.w;
    }
    if constexpr (BETA) {
      const dbl4 a = ld_block_rw(o[g]);
      w0 += beta * a.x, w1 += beta * a.y, w2 += beta * a.z, w3 += beta * a.w;
    }
    v[g][0] = w0, v[g][1] = w1, v[g][2] = w2, v[g][3] = w3;
  }
#pragma unroll
  for (int g = 0; g < G; ++g) st_block(o[g], dbl4{v[g][0], v[g][1], v[g][2], v[g][3]});
}

// reference layout [el][q][4] (q -> internal k = perm[q]) <-> wavefront layout
template <bool TO_WL>
__global__ void wl_convert_kernel(const double* __restrict__ src, double* __restrict__ dst, const int* __restrict__ perm,
                                  int el0, int n_el_chunk, int P, WLGeom wl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (el, q) of the chunk
  if (idx >= (int64_t)n_el_chunk * P) return;
  const int e = int(idx / P), q = int(idx - (int64_t)e * P);
  const size_t refo = (size_t)idx * 4;  // chunk-relative reference offset
  const size_t wlo = (size_t)wl_block(wl, el0 + e, perm[q]) * 4;
  st_block(dst + (TO_WL ? wlo : refo), ld_block(src + (TO_WL ? refo : wlo)));
}

// fill the valid blocks of a wavefront-layout vector (padding stays zero)
__global__ void wl_fill_kernel(double* __restrict__ dst, double v, int n_el, int P, WLGeom wl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n_el * P) return;
  const int el = int(idx / P), k = int(idx - (int64_t)el * P);
  st_block(dst + (size_t)wl_block(wl, el, k) * 4, dbl4{v, v, v, v});
}

}  // namespace

void launch_wl_fill(double* dst, double v, int n_el, int P, const WLGeom& wl, cudaStream_t s) {
  const int64_t n = (int64_t)n_el * P;
  if (n > 0) wl_fill_kernel<<<int((n + 255) / 256), 256, 0, s>>>(dst, v, n_el, P, wl);
}

void launch_to_wl(const double* ref, double* wlv, const int* perm, int el0, int n_el_chunk, int P, const WLGeom& wl,
                  cudaStream_t s) {
  const int64_t n = (int64_t)n_el_chunk * P;
  if (n > 0) wl_convert_kernel<true><<<int((n + 255) / 256), 256, 0, s>>>(ref, wlv, perm, el0, n_el_chunk, P, wl);
}
void launch_from_wl(const double* wlv, double* ref, const int* perm, int el0, int n_el_chunk, int P,
                    const WLGeom& wl, cudaStream_t s) {
  const int64_t n = (int64_t)n_el_chunk * P;
  if (n > 0) wl_convert_kernel<false><<<int((n + 255) / 256), 256, 0, s>>>(wlv, ref, perm, el0, n_el_chunk, P, wl);
}

void launch_fold(const double* phi, double* Phi, const int* orbit, int n_el, int el0, int el1, int P, int R, int G,
                 const WLGeom& wl, cudaStream_t s) {
  const int64_t n = (int64_t)(el1 - el0) * R;
  if (n <= 0) return;
  const int blocks = int((n + 255) / 256);
  switch (G) {
    case 2: fold_kernel<2><<<blocks, 256, 0, s>>>(phi, Phi, orbit, n_el, el0, el1, P, R, wl); break;
    case 4: fold_kernel<4><<<blocks, 256, 0, s>>>(phi, Phi, orbit, n_el, el0, el1, P, R, wl); break;
    case 8: fold_kernel<8><<<blocks, 256, 0, s>>>(phi, Phi, orbit, n_el, el0, el1, P, R, wl); break;
    default: break;
  }
}

#ifndef STAMG_UNFOLD_SPLIT
#define STAMG_UNFOLD_SPLIT 0  // A/B knob: two threads per orbit representative (one dof pair each, 16-byte accesses)
#endif
// unfold_kernel with the four dofs split over a lane pair: half the registers per
// thread (8 x 2 doubles), the pair still covers each 32-byte block in one access
template <int G, bool BETA>
__global__ void __launch_bounds__(256) unfold2_kernel(const double* __restrict__ Y, double* __restrict__ y,
                                                      const int* __restrict__ orbit, int n_el, int el0, int el1,
                                                      int P, int R, double scale, double beta,
                                                      const double* __restrict__ ext_q, const double* __restrict__ area,
                                                      double4 nsum, WLGeom wl) {
  const int64_t idx2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx2 >= (int64_t)(el1 - el0) * R * 2) return;
  const int half = int(idx2 & 1);
  const int64_t idx = idx2 >> 1;
  const int e = int(idx / R), r = int(idx - (int64_t)e * R), el = el0 + e;
  double* o[G];
  double ar[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int q = orbit[r * G + g];
    o[g] = y + (wl.nd ? (size_t)wl_block(wl, el, q) * 4 : ((size_t)el * P + q) * 4) + half * 2;
    ar[g] = ext_q ? area[q] : 0.0;
  }
  double v[G][2];
#pragma unroll
  for (int c = 0; c < G; ++c) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(Y + (((size_t)c * n_el + el) * R + r) * 4 + half * 2));
    v[c][0] = a.x, v[c][1] = a.y;
  }
#pragma unroll
  for (int bit = 1; bit < G; bit <<= 1)
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (!(g & bit))
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double a = v[g][i], b = v[g | bit][i];
          v[g][i] = a + b, v[g | bit][i] = a - b;
        }
  constexpr double inv4pi = 0.07957747154594767;
  const double qel = ext_q ? ext_q[el] * inv4pi : 0.0;
  const double n0 = half ? nsum.z : nsum.x, n1 = half ? nsum.w : nsum.y;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double w0 = scale * v[g][0], w1 = scale * v[g][1];
    if (ext_q) {
      const double c = qel * ar[g];
      w0 += c * n0, w1 += c * n1;
    }
    if constexpr (BETA) {
      const double2 a = *reinterpret_cast<const double2*>(o[g]);
      w0 += beta * a.x, w1 += beta * a.y;
    }
    v[g][0] = w0, v[g][1] = w1;
  }
#pragma unroll
  for (int g = 0; g < G; ++g) *reinterpret_cast<double2*>(o[g]) = make_double2(v[g][0], v[g][1]);
}

void launch_unfold(const double* Y, double* y, const int* orbit, int n_el, int el0, int el1, int P, int R, int G,
                   double scale, double beta, const double* ext_q, const double* area, const double* nsum,
                   const WLGeom& wl, cudaStream_t s) {
  const int64_t n = (int64_t)(el1 - el0) * R;
  if (n <= 0) return;
  const int blocks = int((n + 255) / 256);
  const double4 ns = make_double4(nsum[0], nsum[1], nsum[2], nsum[3]);
  if (STAMG_UNFOLD_SPLIT) {
    const int b2 = int((2 * n + 255) / 256);
    switch (G) {
      case 2:
        if (beta != 0.0) unfold2_kernel<2, true><<<b2, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
        else unfold2_kernel<2, false><<<b2, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
        break;
      case 4:
        if (beta != 0.0) unfold2_kernel<4, true><<<b2, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
        else unfold2_kernel<4, false><<<b2, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
        break;
      case 8:
        if (beta != 0.0) unfold2_kernel<8, true><<<b2, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
        else unfold2_kernel<8, false><<<b2, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
        break;
      default: break;
    }
    return;
  }
  switch (G) {
    case 2:
      if (beta != 0.0) unfold_kernel<2, true><<<blocks, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
      else unfold_kernel<2, false><<<blocks, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
      break;
    case 4:
      if (beta != 0.0) unfold_kernel<4, true><<<blocks, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
      else unfold_kernel<4, false><<<blocks, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
      break;
    case 8:
      if (beta != 0.0) unfold_kernel<8, true><<<blocks, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
      else unfold_kernel<8, false><<<blocks, 256, 0, s>>>(Y, y, orbit, n_el, el0, el1, P, R, scale, beta, ext_q, area, ns, wl);
      break;
    default: break;
  }
}

#ifndef STAMG_D2M_MAXBM
#define STAMG_D2M_MAXBM 168  // A/B knob: largest D2M row tile (smaller -> more, lighter CTAs per SM)
#endif
int d2m_row_tile(int rows, int limit) {
  // candidate tiles: 64 rows (MI 4 x WM 2) and 24-row warp strips x 1..7 warp rows;
  // cost = padded rows + 8 per tile (each extra tile re-reads the phi panel),
  // restricted to tilings that stay inside the call's row region
  static const int cand[] = {64, 24, 48, 72, 96, 120, 144, 168};
  int best = 0, best_cost = 1 << 30;
  for (int bm : cand) {
    const int tiles = (rows + bm - 1) / bm, padded = tiles * bm;
    if (padded > limit || bm > STAMG_D2M_MAXBM) continue;
    const int cost = padded + 8 * tiles;
    if (cost < best_cost) best = bm, best_cost = cost;
  }
  return best;
}

void launch_d2m(const D2MParams& p, cudaStream_t s) {
  if (p.n_el == 0 || p.Hused == 0) return;
  switch (d2m_row_tile(p.Hused, p.Hrows)) {
    case 24: launch_d2m_tile<3, 1>(p, s); break;
    case 48: launch_d2m_tile<3, 2>(p, s); break;
    case 72: launch_d2m_tile<3, 3>(p, s); break;
    case 96: launch_d2m_tile<3, 4>(p, s); break;
    case 120: launch_d2m_tile<3, 5>(p, s); break;
    case 144: launch_d2m_tile<3, 6>(p, s); break;
    case 168: launch_d2m_tile<3, 7>(p, s); break;
    case 64: launch_d2m_tile<4, 2>(p, s); break;
    default: throw std::invalid_argument("d2m: no row tiling fits the moment region");
  }
}

void launch_m2d(const M2DParams& p, cudaStream_t s) {
  if (p.n_el == 0 || p.P == 0) return;
  // per launch: the attribute is per device (contexts may live on different GPUs)
  if (p.beta != 0.0) cudaFuncSetAttribute(m2d_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gemm_smem()));
  else cudaFuncSetAttribute(m2d_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gemm_smem()));
  if (p.Pp % M2D_BM != 0) throw std::invalid_argument("m2d: X^T row pitch is not a multiple of the patch tile");
  const unsigned ge = (p.n_el + BN / 4 - 1) / (BN / 4), gq = (p.P + M2D_BM - 1) / M2D_BM;
  dim3 grid = STAMG_GEMM_SWAP ? dim3(gq, ge) : dim3(ge, gq);
  if (STAMG_M2D_PATCH_FASTEST) grid = dim3(ge * gq);
  if (p.beta != 0.0) m2d_kernel<true><<<grid, M2D_THREADS, gemm_smem(), s>>>(p);
  else m2d_kernel<false><<<grid, M2D_THREADS, gemm_smem(), s>>>(p);
}

}  // namespace stamg_b200
