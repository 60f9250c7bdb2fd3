// Launchers for the sm_100a kernels of the B200 path (host-callable).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

#ifndef STAMG_SWEEP_NST
#define STAMG_SWEEP_NST 6  // sweep rhs staging depth (steps issued ahead)
#endif

namespace stamg_b200 {

// Smallest nx (and the strip height 32 as smallest ny) for 8-direction sweep groups:
// the strip hand-off of the trace scratch needs nx >= R + NST - 1 with R = 32, plus
// one step of slack. upload_level and launch_sweep use the same constant.
constexpr int kSweep8MinNx = 32 + STAMG_SWEEP_NST;
constexpr int kSweep8MinNy = 32;

// Common per-level geometry of the wavefront / stencil kernels: direction
// groups of up to 4 equal-octant patches (-1 = padding).
struct GroupGeom {
  const int* groups = nullptr;     // [n_groups][4]
  const int* group_oct = nullptr;  // [n_groups]
  int n_groups = 0;
  int P = 0, nx = 0, ny = 0;
  const int* mat = nullptr;        // [n_el] material ids (nullptr: all 0)
  int n_mat = 1;
};

// standard_sweep (sweeps.cpp:20-42): z = L^{-1} rhs, or z = base + L^{-1} rhs
// when base != nullptr (the smoother's phi += r). z may alias rhs or base.
struct SweepParams {
  GroupGeom g;                   // groups of g-width directions (4, or 8 when dirs == 8)
  int dirs = 4;
  WLGeom wl;                     // wl.nd > 0: vectors in the wavefront layout (dirs == 8)
  int mode = 0;                  // 0: z = [base +] L^{-1} rhs;  1: z = alpha*L rhs + beta*base (apply_L)
  const double* Bfwd = nullptr;  // mode 1: forward blocks [n_mat][P][16]
  double alpha = 1.0, beta = 0.0;
  double2* top = nullptr;        // dirs == 8: [n_groups][8][nx] strip-boundary trace scratch
  const double* rhs = nullptr;
  const double* base = nullptr;
  double* z = nullptr;
  const double* Binv = nullptr;  // [n_mat][P][16]
  const double* cxy = nullptr;   // [P][8]
  // group sub-range and staged data (host-buffer pipeline): CTA b sweeps group grp0 + b;
  // with data_P > 0 (reference-layout vectors only) the data of patch k sits at column
  // k - data_q0 of a [n_el][data_P][4] buffer
  int grp0 = 0, data_P = 0, data_q0 = 0;
  bool prefer_breg = false;  // 8-direction groups: keep B^-1 in registers (2 CTAs/SM) even for 2-4 CTAs per SM of groups
  int xb = 1;                // > 1: column blocks per group (wavefront layout, plain sweep)
  int xb_g0 = 0;             // groups [0, xb_g0) are swept whole, groups from xb_g0 on in xb column blocks
  int xb_ticket = 0;         // 1: block ids from an atomic ticket (grids larger than the co-resident capacity)
  int* xflag = nullptr;      // [n_groups][xb] strips published by each block (zeroed per launch)
  double2* xtrace = nullptr; // [n_groups][xb][ny][8] x-traces at the block edges
};
void launch_sweep(const SweepParams& p, cudaStream_t s);

// apply_L_into (transport.cpp:66-88): y = alpha * L x + beta * f
struct ApplyLParams {
  GroupGeom g;                  // 4-direction groups, or 8 when dirs == 8 (row-walk kernel)
  int dirs = 4;
  const double* x = nullptr;
  const double* f = nullptr;
  double* y = nullptr;
  double alpha = 1.0, beta = 0.0;
  const double* B = nullptr;    // [n_mat][P][16]
  const double* cxy = nullptr;  // [P][8]
};
void launch_apply_L(const ApplyLParams& p, cudaStream_t s);

// D2M with the sigma*N epilogue (scatter.cpp:130-131):
// src[el][h][i] = sig[mat(el)][h] * sum_j (sum_{q} X[q][h] phi[el][q][j]) N[j][i]
// for h < Hused (zero above), on FP64 tensor cores.
struct D2MParams {
  WLGeom wl;                     // wl.nd > 0: phi in the wavefront layout (P = internal order)
  const double* phi = nullptr;
  double* src = nullptr;         // [n_el][Hp][4]
  const double* X = nullptr;     // [Pk][Hp]   (rows >= P are zero)
  const double* sig = nullptr;   // [n_mat][Hp]
  const int* mat = nullptr;
  int n_el = 0, P = 0, Hp = 0, Hused = 0;  // n_el: elements of this call, [el_base, el_base + n_el)
  int el_base = 0;               // first element (element-range chunks of the scatter; global indexing)
  int Hrows = 0;                 // rows of src this call may write (its region; >= Hused)
  double N[16];
};
void launch_d2m(const D2MParams& p, cudaStream_t s);
// rows of the D2M output tile for `rows` harmonics inside a region of `limit` rows (0: none fits)
int d2m_row_tile(int rows, int limit);

// M2D (scatter.cpp:132): y[el][q][i] = beta*y + scale * sum_h X[q][h] src[el][h][i]
//   + (ext_q ? ext_q[el]/(4 pi) * area[q] * nsum[i] : 0)
struct M2DParams {
  WLGeom wl;                     // wl.nd > 0: y in the wavefront layout
  const double* src = nullptr;   // [n_el][Hp][4]
  double* y = nullptr;
  const double* XT = nullptr;    // [Hp][Pp]
  int n_el = 0, P = 0, Pp = 0, Hp = 0, Hused = 0;  // n_el: elements of this call, [el_base, el_base + n_el)
  int el_base = 0;
  double scale = 1.0, beta = 1.0;
  const double* ext_q = nullptr;  // [n_el] isotropic source density or nullptr
  const double* area = nullptr;   // [P]
  double nsum[4];
};
void launch_m2d(const M2DParams& p, cudaStream_t s);

// reflection-symmetry fold / unfold around the per-class moment GEMMs:
// Phi[c][el][r][i] = sum_g chi_c(g) phi[el][orbit[r][g]][i];
// y[el][orbit[r][g]][i] = beta*y + scale*sum_c chi_c(g) Y[c][el][r][i] (+ isotropic source)
// over the elements [el0, el1) of n_el (Phi / Y class stride n_el * R * 4)
void launch_fold(const double* phi, double* Phi, const int* orbit, int n_el, int el0, int el1, int P, int R, int G,
                 const WLGeom& wl, cudaStream_t s);
void launch_unfold(const double* Y, double* y, const int* orbit, int n_el, int el0, int el1, int P, int R, int G,
                   double scale, double beta, const double* ext_q, const double* area, const double* nsum,
                   const WLGeom& wl, cudaStream_t s);
// reference layout [el][q][4] (patch q mapped to internal k = perm[q]) <-> wavefront layout,
// for elements [el0, el0 + n_el_chunk)
void launch_to_wl(const double* ref, double* wlv, const int* perm, int el0, int n_el_chunk, int P, const WLGeom& wl,
                  cudaStream_t s);
void launch_from_wl(const double* wlv, double* ref, const int* perm, int el0, int n_el_chunk, int P,
                    const WLGeom& wl, cudaStream_t s);
void launch_wl_fill(double* dst, double v, int n_el, int P, const WLGeom& wl, cudaStream_t s);

// transfers (multigrid.cpp:100-136), Const basis
void launch_prolong(const double* coarse, double* fine, const int* up, const double* w, int n_el, int Pf,
                    int Pc, bool add, cudaStream_t s);
void launch_restrict(const double* fine, double* coarse, const int* child_ptr, const int* child_idx,
                     const double* w, int n_el, int Pf, int Pc, cudaStream_t s);

// coarse_scatter_sweep (sweeps.cpp:51-104), order-exact dataflow kernel
struct CoarseGSParams {
  const double* rhs = nullptr;
  double* phi = nullptr;
  double* mom = nullptr;          // [n_el][Hp][4] running per-element moments
  const double* X = nullptr;      // [Pk][Hp]
  const double* sig = nullptr;    // [n_mat][Hp]
  const double* BinvGS = nullptr; // [n_mat][P][16]
  const double* GS = nullptr;     // [n_mat][P][16] BinvGS * N (sweep frame)
  const double* sq = nullptr;     // [n_mat][P]
  const double* cxy = nullptr;
  const int* oct_patches = nullptr;
  const int* oct_ptr = nullptr;   // [9]
  const int* mat = nullptr;
  int* done = nullptr;            // [8][n_el] completed pass count
  const double* Xo = nullptr;     // [P][Hp] X rows in octant order (oct_patches)
  const double* XoT = nullptr;    // [Hp][P] its transpose
  const double* K = nullptr;      // [n_mat][P][kpad] X_a sig X_b^T, a = octant-ordered row, b = index in octant
  const double* Minv = nullptr;   // [n_mat][8][kpad/4][160] packed inverses of the chain's 4-patch diagonal blocks
  int chain_blk = 0;              // 1: blocked patch chain (multi-warp kernel; kpad a multiple of 4)
  int cells_per_warp = 0, kpad = 0, grid_blocks = 0;  // warp owns a row segment of cells_per_warp cells
  int xreg = 1;       // x-upwind traces inside a segment from registers (0: through global memory)
  int rows_mode = 0;  // > 0: warp owns a whole row, CTA = rows_mode consecutive rows (shared mailbox)
  int multi_warp = 0; // 1: a CTA of 4 warps owns a whole row (projections / moment updates spread)
  int cluster = 0;    // multi_warp: > 1 = rows per thread-block cluster (DSMEM y-mailboxes)
  int mb_np = 0;      // mailbox patches per slot (max patches per octant)
  int mb_slots = 0;   // mailbox slots per y-direction: 2 nx, or a power of two with credits
  int mb_credit = 0;  // 1: the downwind row returns slots (ring smaller than two octants of a row)
  int mom_stride = 0; // multi-warp: shared moment ring row stride (0 = Hp; H rounded to even with rings)
  int n_el = 0, P = 0, Hp = 0, H = 0, nx = 0, ny = 0, nu = 0, n_mat = 1;
  int max_patches_per_octant = 0;
  double N[16];
};
void launch_coarse_gs(const CoarseGSParams& p, cudaStream_t s);
// co-resident warps of the coarse GS kernel, and warps per CTA
int coarse_gs_max_warps(int Hp, int kpad, int nmat, int max_np);
int coarse_gs_warps_per_block(int Hp, int kpad, int nmat);
int coarse_gs_rows_wpb(int Hp, int kpad, int nmat, int nx, int ny, int max_np);
int coarse_gs_mw_ok(int Hp, int H, int kpad, int nmat, int ny, int max_np, bool blk);
// blocked patch chain of the multi-warp kernel (default; STAMG_GS_CHAIN_BLOCKS=0 keeps the
// patch-by-patch chain), and the packed size of one 16 x 16 block inverse
bool coarse_gs_chain_blocked();
constexpr int kGsMinvBlock = 160;
// multi-warp rows in clusters: (mailbox slots << 8) | (credit << 7) | rows per cluster (16, 8, 4 or 2)
// for the largest mailbox whose clusters all fit co-resident, 0 if none
int coarse_gs_cluster_rows(int Hp, int H, int kpad, int nmat, int nx, int ny, int max_np, bool blk);

// BLAS-1 (deterministic reductions)
void launch_fill(double* x, double v, int64_t n, cudaStream_t s);
void launch_axpy(double a, const double* x, double* y, int64_t n, cudaStream_t s);        // y += a x
void launch_axpby(double a, const double* x, double b, double* y, int64_t n, cudaStream_t s);  // y = a x + b y
void launch_scale(double a, double* x, int64_t n, cudaStream_t s);
// out[k] = sum_i V_k[i] w[i] for k < nv (V_k = vs[k]); partial buffer sized by multidot_partials()
int multidot_blocks();
void launch_multidot(const double* const* vs, int nv, const double* w, int64_t n, double* partial,
                     double* out, cudaStream_t s);
// w -= sum_k c[k] V_k  (c on device)
void launch_multi_axpy(const double* const* vs, int nv, const double* c, double* w, int64_t n, cudaStream_t s);
// u = sum_k c[k] V_k  (c on device)
void launch_lincomb(const double* const* vs, int nv, const double* c, double* u, int64_t n, cudaStream_t s);

// FP64 throughput microbenchmarks (roofline denominators)
double bench_dmma_tflops(int device, cudaStream_t s);
double bench_dfma_tflops(int device, cudaStream_t s);
double bench_chunk_rw_gbs(double* buf, int64_t n_doubles, int64_t stride_chunks, int mode, cudaStream_t s);

}  // namespace stamg_b200
