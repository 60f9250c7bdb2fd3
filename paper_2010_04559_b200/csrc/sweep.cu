// Transport sweep on sm_100a: standard_sweep (sweeps.cpp:20-42), exact L^{-1}.
//
// One CTA owns a group of 4 equal-octant directions and R grid rows
// (4*R threads, thread = (direction, row)). Each thread walks the cells of
// its rows in upwind order; rows r, r+R, r+2R, ... are chained so the whole
// grid is one skewed wavefront with a single ramp. Per step:
//  * the x-upwind trace (2 doubles) stays in the thread's registers;
//  * the y-upwind trace comes from the row below: warp shuffle inside a warp,
//    a double-buffered shared slot across warps, a shared row buffer across
//    the R-row strips;
//  * the 4x4 cell solve runs in registers with the precomputed inverse.
// rhs (and the smoother's base vector) is staged by cp.async NST-1 steps
// ahead. All arithmetic is done in the sweep frame (dofs XOR-permuted so the
// upwind corner is dof 0); tables are pre-permuted on the host.
// HBM traffic: 32 B read + 32 B written per cell-direction (64 B algorithmic),
// +32 B read with a base vector.
#include "common.cuh"
#include "kernels.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace stamg_b200 {
namespace {

#ifndef STAMG_SWEEP8_BREG
#define STAMG_SWEEP8_BREG 1  // 8-direction kernel keeps B^-1 in registers (2 CTAs/SM); A/B: 82.5 % vs 79 %
#endif
#ifndef STAMG_SWEEP_UNROLL
#define STAMG_SWEEP_UNROLL 2  // step-loop unroll: the loop-carried traces alternate registers instead of being moved
#endif
constexpr int kNST = STAMG_SWEEP_NST;
constexpr int kSweepUnroll = STAMG_SWEEP_UNROLL;
#ifndef STAMG_SWEEP_ONE_WAVE4
#define STAMG_SWEEP_ONE_WAVE4 1  // A/B: 0 = always the 2-per-SM kernel (B^-1 in registers)
#endif
#ifndef STAMG_SWEEP_BULK
// wavefront layout: 1 = a step's rows arrive as one or two TMA bulk copies (cp.async.bulk, one
// issuing thread, mbarrier completion), 0 = per-thread cp.async. The bulk path removes the
// per-thread source addressing and LDGSTS issue from every step and draws less power, and the
// sweep runs against the board's power cap: with the lean step loop it measures
// 22.6 ms against 22.9 ms per config-5 sweep over 10 back-to-back sweeps (0.928 vs 0.916 of the
// copy bandwidth) and 23.2 against 23.7 ms over 40 (SM clock 1710 vs 1610 MHz under
// sw_power_cap); profiles/r02_sweep_ab.txt. With the earlier, heavier step loop it had been
// slower (23.8 vs 23.1 ms), which is why it was off until the last session of round 2.
#define STAMG_SWEEP_BULK 1
#endif

// DIRS directions x R rows per CTA (DIRS*R = 256 threads). thread = (dir, row):
// dir = tid % DIRS, row = tid / DIRS. With DIRS = 8 a cell's 8 directions are
// one 256-byte run (better DRAM efficiency than 128 B), and the strip-boundary
// traces go through an L2-resident global scratch (TOPG) instead of shared
// memory so the CTA still fits 3 per SM.
// XBLK: each group's grid is split into p.xb column blocks swept by consecutive CTAs
// (KBA-style): block b starts a strip once block b-1 has published that strip's
// x-traces at their common edge (global scratch + one flag per strip), so a group's
// wavefront runs on xb SMs. Used when there are fewer groups than SMs (config 5
// sharded over 8 GPUs: 128 groups per rank); all CTAs are co-resident.
// BPS: resident CTAs per SM the registers are sized for (8-direction kernels): 2 or 3 keep B^-1 in
// registers (112 / 80 registers), 4 reads it from shared memory (64 registers).
template <int DIRS, int R, bool MULTI, bool ACCUM, bool TOPG, bool WLAY = false, int MODE = 0, int BPS = 2,
          bool XBLK = false, int NST_ = kNST>
__global__ void __launch_bounds__(DIRS * R, (TOPG ? BPS : 1)) sweep_kernel(SweepParams p) {
  constexpr bool BREG = BPS < 4;
  // step-loop unroll only where the register budget has room (112 registers at 2 CTAs/SM): the
  // 80- and 64-register variants spill with it (config 4's plain sweep 3.10 -> 3.39 ms)
  constexpr int UNR = (TOPG && BPS == 2) ? kSweepUnroll : 1;
  constexpr bool WG = TOPG && BPS == 2;  // likewise the warp-uniform guards (8 bytes of spill, 3 % at config 4)
  constexpr int NST = NST_;  // rhs staging depth of this instantiation
  // WLAY: vectors in the wavefront layout (a step's R rows are consecutive slots).
  // MODE 1: apply_L on the same skewed schedule (y = alpha*(B x + C x_up) + beta*f, traces of x).
  // TOPG (8-direction) variant: 4 CTAs/SM (<= 64 registers), B^-1 read from shared memory
  constexpr int NT = DIRS * R;
  constexpr int NW = NT / 32;
  constexpr int RPW = 32 / DIRS;  // rows per warp
  // BULK (wavefront layout): the R rows of a step lie on one anti-diagonal of one strip -- or,
  // while the wavefront crosses into the next strip, on one diagonal of each -- so the step's
  // rhs (and base) is one or two contiguous runs of up to R x DIRS x 32 B = 8 KB. Thread 0
  // issues them as cp.async.bulk copies completing on the stage's mbarrier (UBLKCP); nobody
  // computes a per-thread source address or issues per-thread LDGSTS for the vector data.
  constexpr bool BULK = WLAY && TOPG && !XBLK && (STAMG_SWEEP_BULK != 0);  // column blocks: cp.async measured faster (3.23 vs 3.36 ms per rank at N = 8)
  __shared__ unsigned long long s_bar[BULK ? NST_ : 1];
  extern __shared__ __align__(128) double smem[];
  double* st_rhs = smem;
  double* st_base = st_rhs + NST * NT * 4;
  double* after_base = st_base + (ACCUM ? NST * NT * 4 : 0);
  double2* st_top = reinterpret_cast<double2*>(after_base);                       // TOPG: [NST][DIRS]
  double2* top = reinterpret_cast<double2*>(after_base) + (TOPG ? NST * DIRS : 0);  // !TOPG: [DIRS][nx]
  double2* xw = top + (TOPG ? 0 : DIRS * p.g.nx);
  double* sB = reinterpret_cast<double*>(xw + 2 * NW * DIRS);

  const int tid = threadIdx.x, dir = tid % DIRS, r = tid / DIRS, lane = tid & 31, warp = tid >> 5;
  // XBLK: logical block ids come from a ticket, so a block's upwind neighbour (the ticket
  // before it) is always running or done, whatever order the hardware dispatches CTAs in:
  // the flag waits below cannot deadlock even when the grid is many waves.
  // Groups below p.xb_g0 are swept whole (one block); the groups from xb_g0 on, the tail
  // wave of a grid of whole-group CTAs, are cut into p.xb column blocks each.
  // (a grid that is co-resident as a whole needs no ticket: p.xb_ticket = 0)
  int bid = int(blockIdx.x);
  if constexpr (XBLK) {
    if (p.xb_ticket) {
      __shared__ int s_bid;
      if (threadIdx.x == 0) s_bid = atomicAdd(p.xflag + p.g.n_groups * p.xb, 1);
      __syncthreads();
      bid = s_bid;
    }
  }
  const bool cut = XBLK && bid >= p.xb_g0;
  const int xb = cut ? p.xb : 1;
  const int gb = cut ? p.xb_g0 + (bid - p.xb_g0) / xb : bid;
  const int xblk = cut ? (bid - p.xb_g0) - (gb - p.xb_g0) * xb : 0;
  const int grp = gb + p.grp0;
  const int q = p.g.groups[grp * DIRS + dir];
  const int oct = p.g.group_oct[grp];
  const bool xneg = oct & 1, yneg = (oct >> 1) & 1;
  const int nx = p.g.nx, ny = p.g.ny, P = p.g.P;
  const int DP = p.data_P > 0 ? p.data_P : P, DQ0 = p.data_P > 0 ? p.data_q0 : 0;
  const int nxl = XBLK ? nx / xb : nx;  // columns of this CTA's block, frame columns i0 ..
  const int i0 = xblk * nxl;
  double2* sxin = reinterpret_cast<double2*>(sB + ((MULTI || (TOPG && !BREG)) ? p.g.n_mat * DIRS * 17 : 0));  // XBLK: [NT]
  const bool qok = q >= 0;
  const int qq = qok ? q : 0;
  double2* gtop = p.top + (size_t)grp * DIRS * nx;  // TOPG scratch of this group

  double cx[4], cy[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) cx[k] = p.cxy[qq * 8 + k], cy[k] = p.cxy[qq * 8 + 4 + k];
  constexpr bool BSMEM = MULTI || (TOPG && !BREG);
  double Bi[16];
  const double* Bsrc = MODE == 1 ? p.Bfwd : p.Binv;
  if constexpr (!BSMEM) {
#pragma unroll
    for (int k = 0; k < 16; ++k) Bi[k] = Bsrc[qq * 16 + k];
  } else {
    for (int idx = tid; idx < p.g.n_mat * DIRS * 16; idx += NT) {
      const int m = idx / (DIRS * 16), d = (idx / 16) % DIRS, k = idx & 15;
      const int qd = p.g.groups[grp * DIRS + d];
      sB[(m * DIRS + d) * 17 + k] = qd >= 0 ? Bsrc[((size_t)m * P + qd) * 16 + k] : 0.0;
    }
  }

  const int nstrips = (ny + R - 1) / R;
  const int nk = nstrips * nxl;
  const int T = nk + R - 1;
  // XBLK: traces at the block edges, [groups][xb][ny][DIRS], and per-(group, block) strip flags
  const int xbs = XBLK ? p.xb : 1;  // flag / trace stride per group
  const double2* xin = XBLK && xblk > 0 ? p.xtrace + ((size_t)(grp * xbs + xblk - 1) * ny) * DIRS : nullptr;
  double2* xout = XBLK && xblk < xb - 1 ? p.xtrace + ((size_t)(grp * xbs + xblk) * ny) * DIRS : nullptr;

  // Cursor over this thread's wavefront positions k = (strip s, column i): advanced by one
  // add per field; the block offset (and the row's validity) is recomputed only when the
  // cursor enters a strip. Positions k < 0 (this row's ramp-in) count i up from -r on the
  // virtual columns left of strip 0; positions k >= nk run past the last strip. Neither is
  // dereferenced (kin() is false).
  struct Cursor {
    int k, s, i, el;
    bool rowok;
    size_t off;
  };
  const int dx = xneg ? -1 : 1;
  const ptrdiff_t cstride = WLAY ? (ptrdiff_t)R * DIRS * 4 : (ptrdiff_t)dx * DP * 4;
  auto enter = [&](Cursor& c) {  // column 0 of strip c.s
    const int j = c.s * R + r;
    c.rowok = qok && j < ny;
    const int jj = j < ny ? j : 0;
    const int gx = xneg ? nx - 1 - i0 : i0, gy = yneg ? ny - 1 - jj : jj;
    c.el = gy * nx + gx;
    if constexpr (WLAY) c.off = (((size_t)grp * p.wl.slots + wl_slot_frame(p.wl, i0, jj)) * DIRS + dir) * 4;
    else c.off = ((size_t)c.el * DP + (qq - DQ0)) * 4;
  };
  auto start = [&](Cursor& c) {  // position k = -r
    c.s = 0;
    enter(c);
    c.k = c.i = -r;
    c.off -= (size_t)((ptrdiff_t)r * cstride);
    c.el -= r * dx;
  };
  auto advance = [&](Cursor& c) {
    ++c.k, ++c.i, c.off += (size_t)cstride;
    if constexpr (MULTI) c.el += dx;
    if (c.i == nxl) {
      c.i = 0, ++c.s;
      enter(c);
    }
  };
  auto kin_of = [&](const Cursor& c) { return (unsigned)c.k < (unsigned)nk; };
  // BULK producer state (thread 0): strip of row 0 at the issue step and the step within it
  int b_sh = 0, b_rb = 0;
  auto issue = [&](int t, int stg, const Cursor& c) {
    const bool c_kin = kin_of(c), c_ok = c_kin && c.rowok;
    if constexpr (BULK) {
      if (tid == 0) {
        // rows 0..rb are in strip sh on diagonal i0 + rb, rows rb+1..R-1 still in strip sh-1
        // on diagonal i0 + rb + nxl (slot = (strip * nd + diagonal) * R + row)
        const int nA = b_sh < nstrips ? min(b_rb, R - 1) + 1 : 0;
        const int nB = (b_sh >= 1 && b_sh - 1 < nstrips && b_rb < R - 1) ? R - 1 - b_rb : 0;
        if (nA + nB > 0) {
          unsigned long long* bar = &s_bar[stg];
          mbar_expect_tx(bar, unsigned(nA + nB) * DIRS * 32u * (ACCUM ? 2u : 1u));
          const size_t g0 = (size_t)grp * p.wl.slots;
          if (nA > 0) {
            const size_t off = (g0 + ((size_t)b_sh * p.wl.nd + i0 + b_rb) * R) * DIRS * 4;
            bulk_g2s(st_rhs + (size_t)stg * NT * 4, p.rhs + off, unsigned(nA) * DIRS * 32u, bar);
            if constexpr (ACCUM) bulk_g2s(st_base + (size_t)stg * NT * 4, p.base + off, unsigned(nA) * DIRS * 32u, bar);
          }
          if (nB > 0) {
            const size_t off = (g0 + ((size_t)(b_sh - 1) * p.wl.nd + i0 + b_rb + nxl) * R + b_rb + 1) * DIRS * 4;
            const size_t so = ((size_t)stg * NT + (size_t)(b_rb + 1) * DIRS) * 4;
            bulk_g2s(st_rhs + so, p.rhs + off, unsigned(nB) * DIRS * 32u, bar);
            if constexpr (ACCUM) bulk_g2s(st_base + so, p.base + off, unsigned(nB) * DIRS * 32u, bar);
          }
        }
        if (++b_rb == nxl) b_rb = 0, ++b_sh;
      }
    } else {
    const bool ok = c_ok;
    const size_t off = ok ? c.off : 0;
    const double* src = p.rhs + off;
    double* dst = st_rhs + (stg * NT + tid) * 4;
    cp_async16(dst, src, ok);
    cp_async16(dst + 2, src + 2, ok);
    if constexpr (ACCUM) {
      const double* sb = p.base + off;
      double* db = st_base + (stg * NT + tid) * 4;
      cp_async16(db, sb, ok);
      cp_async16(db + 2, sb + 2, ok);
    }
    }
    if constexpr (TOPG) {  // row 0 of strip s >= 1 needs the trace row R-1 left in the scratch
      if ((!WG || warp == 0) && r == 0) {  // (WG: warp-uniform outer test, the other warps branch over the address math)
        const bool tk = c_kin && c.s >= 1;
        cp_async16(st_top + stg * DIRS + dir, gtop + (size_t)dir * nx + (tk ? i0 + c.i : 0), tk);
      }
    }
    if constexpr (XBLK) {  // the block's first column of a strip: x-trace from the upwind block
      if (xin && c_kin && c.i == 0) {
        const int j = c.s * R + r;
        cp_async16(sxin + tid, xin + (size_t)(j < ny ? j : 0) * DIRS + dir, j < ny);
      }
    }
  };
  // XBLK: strip s of the upwind block must be complete before this block issues its loads
  int wait_s = 0, wait_t = 0, pub_s = 0, pub_t = (nxl - 1) + (R - 1);
  auto wait_strip = [&]() {
    if (tid == 0) {
      const int* f = p.xflag + grp * xbs + xblk - 1;
      while (ld_relaxed(f) < wait_s + 1) {
      }
      fence_acq_rel();
    }
    __syncthreads();
    ++wait_s, wait_t = wait_s * nxl - (NST - 1);
  };
  if constexpr (BULK) {
    if (tid == 0) {
      for (int k = 0; k < NST; ++k) mbar_init_cta(&s_bar[k], 1);
      fence_proxy_async_smem();
    }
    __syncthreads();
  }
  if constexpr (XBLK) {
    if (xin) wait_strip();
  }
  Cursor ci, cc;  // issue cursor (k = t + NST - 1 - r) and compute cursor (k = t - r)
  start(ci);
  start(cc);
#pragma unroll
  for (int t = 0; t < NST - 1; ++t) {
    issue(t, t, ci);
    cp_async_commit();
    advance(ci);
  }
  __syncthreads();

  // The step loop is instantiated per octant reflection m (CTA-uniform), so the
  // physical <-> sweep-frame dof permutations are register renames, not selects.
  auto steps = [&](auto mtag) {
  constexpr int m = decltype(mtag)::value;
  double2 tx = make_double2(0.0, 0.0), typrev = make_double2(0.0, 0.0);
  int stg = 0, stg_issue = NST - 1;  // stage of step t, stage filled during step t (= t + NST - 1 mod NST)
  auto step = [&](int t) {
    if constexpr (XBLK) {
      if (xin && wait_s < nstrips && t == wait_t) wait_strip();
    }
    issue(t + NST - 1, stg_issue, ci);
    cp_async_commit();
    advance(ci);
    cp_async_wait<NST - 1>();
    if constexpr (BULK) mbar_wait_parity(&s_bar[stg], unsigned(t / NST) & 1u);
    const bool kin = kin_of(cc);
    const int s = cc.s, i = cc.i;
    double2 ty;
    ty.x = __shfl_up_sync(0xffffffffu, typrev.x, DIRS);
    ty.y = __shfl_up_sync(0xffffffffu, typrev.y, DIRS);
    if (lane < DIRS) {
      if (warp == 0) {
        if (s == 0 || !kin) ty = make_double2(0.0, 0.0);
        else if constexpr (TOPG) ty = st_top[stg * DIRS + dir];
        else ty = top[dir * nx + i];
      } else {
        ty = xw[((t - 1) & 1) * NW * DIRS + (warp - 1) * DIRS + dir];
      }
    }
    double2 tyout = make_double2(0.0, 0.0);
    [[maybe_unused]] const int el = cc.el;
    if (kin && cc.rowok) {
      const double* rs = st_rhs + (stg * NT + tid) * 4;
      double r0 = rs[0], r1 = rs[1], r2 = rs[2], r3 = rs[3];
      // physical -> sweep frame (dof i -> i ^ m)
      if (m & 1) { double u = r0; r0 = r1; r1 = u; u = r2; r2 = r3; r3 = u; }
      if (m & 2) { double u = r0; r0 = r2; r2 = u; u = r1; r1 = r3; r3 = u; }
      if (i == 0) tx = (XBLK && xin) ? sxin[tid] : make_double2(0.0, 0.0);
      const double* B = Bi;
      [[maybe_unused]] double Bm[16];
      if constexpr (BSMEM) {
        const int mt = MULTI ? p.g.mat[el] : 0;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) Bm[kk] = sB[(mt * DIRS + dir) * 17 + kk];
        B = Bm;
      }
      double z0, z1, z2, z3;
      if constexpr (MODE == 0) {
        // upwind couplings: x-face rows {0,2} <- left trace, y-face rows {0,1} <- lower trace
        r0 -= cx[0] * tx.x + cx[1] * tx.y;
        r2 -= cx[2] * tx.x + cx[3] * tx.y;
        r0 -= cy[0] * ty.x + cy[1] * ty.y;
        r1 -= cy[2] * ty.x + cy[3] * ty.y;
        z0 = B[0] * r0 + B[1] * r1 + B[2] * r2 + B[3] * r3;
        z1 = B[4] * r0 + B[5] * r1 + B[6] * r2 + B[7] * r3;
        z2 = B[8] * r0 + B[9] * r1 + B[10] * r2 + B[11] * r3;
        z3 = B[12] * r0 + B[13] * r1 + B[14] * r2 + B[15] * r3;
        tx = make_double2(z1, z3);
        tyout = make_double2(z2, z3);
        if constexpr (XBLK) {
          if (xout && i == nxl - 1) reinterpret_cast<double2*>(xout)[(size_t)(s * R + r) * DIRS + dir] = tx;
        }
      } else {  // apply_L (transport.cpp:72-87): y = B x + C_x x_left + C_y x_below
        z0 = B[0] * r0 + B[1] * r1 + B[2] * r2 + B[3] * r3;
        z1 = B[4] * r0 + B[5] * r1 + B[6] * r2 + B[7] * r3;
        z2 = B[8] * r0 + B[9] * r1 + B[10] * r2 + B[11] * r3;
        z3 = B[12] * r0 + B[13] * r1 + B[14] * r2 + B[15] * r3;
        if (i > 0) {
          z0 += cx[0] * tx.x + cx[1] * tx.y;
          z2 += cx[2] * tx.x + cx[3] * tx.y;
        }
        if (s > 0 || r > 0) {
          z0 += cy[0] * ty.x + cy[1] * ty.y;
          z1 += cy[2] * ty.x + cy[3] * ty.y;
        }
        tx = make_double2(r1, r3);
        tyout = make_double2(r2, r3);
      }
      // frame -> physical
      if (m & 2) { double u = z0; z0 = z2; z2 = u; u = z1; z1 = z3; z3 = u; }
      if (m & 1) { double u = z0; z0 = z1; z1 = u; u = z2; z2 = z3; z3 = u; }
      if constexpr (ACCUM) {
        const double* bs = st_base + (stg * NT + tid) * 4;
        if constexpr (MODE == 0) {
          z0 += bs[0], z1 += bs[1], z2 += bs[2], z3 += bs[3];
        } else {
          z0 = p.alpha * z0 + p.beta * bs[0], z1 = p.alpha * z1 + p.beta * bs[1];
          z2 = p.alpha * z2 + p.beta * bs[2], z3 = p.alpha * z3 + p.beta * bs[3];
        }
      } else if constexpr (MODE == 1) {
        z0 *= p.alpha, z1 *= p.alpha, z2 *= p.alpha, z3 *= p.alpha;
      }
      double* out = p.z + cc.off;
      reinterpret_cast<double2*>(out)[0] = make_double2(z0, z1);
      reinterpret_cast<double2*>(out)[1] = make_double2(z2, z3);
    }
    if (lane >= 32 - DIRS) xw[(t & 1) * NW * DIRS + warp * DIRS + dir] = tyout;
    if ((!WG || warp == NW - 1) && r == R - 1 && kin) {
      if constexpr (TOPG) reinterpret_cast<double2*>(gtop)[(size_t)dir * nx + i0 + i] = tyout;
      else top[dir * nx + i] = tyout;
    }
    typrev = tyout;
    advance(cc);
    stg_issue = stg;
    stg = stg + 1 == NST ? 0 : stg + 1;
    __syncthreads();
    if constexpr (XBLK) {  // strip pub_s's last column is done by every row: publish its edge traces
      if (xout && t == pub_t) {
        if (tid == 0) {
          __threadfence();
          st_release(p.xflag + grp * xbs + xblk, pub_s + 1);
        }
        ++pub_s, pub_t += nxl;
      }
    }
  };
  if constexpr (UNR > 1) {
#pragma unroll UNR
    for (int t = 0; t < T; ++t) step(t);
  } else {  // no pragma: the register-capped variants keep the compiler's own schedule
    for (int t = 0; t < T; ++t) step(t);
  }
  };
  switch ((xneg ? 1 : 0) | (yneg ? 2 : 0)) {
    case 0: steps(std::integral_constant<int, 0>{}); break;
    case 1: steps(std::integral_constant<int, 1>{}); break;
    case 2: steps(std::integral_constant<int, 2>{}); break;
    default: steps(std::integral_constant<int, 3>{}); break;
  }
  cp_async_wait<0>();
  (void)RPW;
}

template <int DIRS, int R, bool ACCUM, bool TOPG>
size_t sweep_smem(const SweepParams& p, int NST, bool bsmem, bool xblk) {
  constexpr int NT = DIRS * R;
  return sizeof(double) * NST * NT * 4 * (ACCUM ? 2 : 1) +
         sizeof(double2) * ((TOPG ? NST * DIRS : DIRS * p.g.nx) + 2 * (NT / 32) * DIRS) +
         (bsmem ? sizeof(double) * p.g.n_mat * DIRS * 17 : 0) + (xblk ? sizeof(double2) * NT : 0);
}

template <int DIRS, int R, bool MULTI, bool ACCUM, bool TOPG, bool WLAY, int MODE, int BPS, bool XBLK = false,
          int NST = kNST>
void launch_tb(const SweepParams& p, cudaStream_t s) {
  constexpr int NT = DIRS * R;
  const size_t smem = sweep_smem<DIRS, R, ACCUM, TOPG>(p, NST, MULTI || (TOPG && BPS == 4), XBLK);
  auto k = sweep_kernel<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, BPS, XBLK, NST>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<XBLK ? p.xb_g0 + (p.g.n_groups - p.xb_g0) * p.xb : p.g.n_groups, NT, smem, s>>>(p);
}

// 8-direction groups, by how the grid fills the SMs:
//  * many waves (config 5: 1024 groups) or at most two CTAs per SM: B^-1 in registers at
//    112 registers, 2 CTAs/SM (82.5 % vs 79 % of HBM for the shared-memory B^-1 at config 5);
//  * a grid that fits one wave at 3 CTAs per SM (config 4's cone mesh: 364 groups on 444
//    slots): B^-1 still in registers, capped at 80 registers;
//  * one wave only at 4 CTAs per SM: B^-1 in shared memory (64 registers).
// The one-wave kernels only pay when the whole grid is resident, so the rhs staging depth
// drops from 6 to 4 or 3 steps where shared memory would otherwise limit residency (a base
// vector doubles the staging: config 4's smoother sweep, 5.60 -> 4.17 ms at depth 4).
#ifndef STAMG_SWEEP_BPS
#define STAMG_SWEEP_BPS 2  // A/B: CTAs per SM of the many-wave kernel
#endif
template <int DIRS, int R, bool MULTI, bool ACCUM, bool TOPG, bool WLAY, int MODE, int BPS>
void launch_resident(const SweepParams& p, int sms, cudaStream_t s) {
  auto resident = [&](int nst) {
    const size_t smem = sweep_smem<DIRS, R, ACCUM, TOPG>(p, nst, MULTI || BPS == 4, false) + 1024;
    return int(std::min<size_t>(BPS, (227 * 1024) / smem)) * sms >= p.g.n_groups;
  };
  if (kNST > 4 && !resident(kNST)) {
    if (resident(4)) launch_tb<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, BPS, false, 4>(p, s);
    else launch_tb<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, BPS, false, 3>(p, s);
    return;
  }
  launch_tb<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, BPS>(p, s);
}

template <int DIRS, int R, bool MULTI, bool ACCUM, bool TOPG, bool WLAY = false, int MODE = 0>
void launch_t(const SweepParams& p, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if constexpr (TOPG) {
    const int ng = p.g.n_groups;
    if (STAMG_SWEEP_ONE_WAVE4 && !p.prefer_breg && ng > 2 * sms && ng <= 4 * sms) {
      if (ng <= 3 * sms) launch_resident<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, 3>(p, sms, s);
      else launch_resident<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, 4>(p, sms, s);
      return;
    }
    launch_tb<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, STAMG_SWEEP8_BREG ? STAMG_SWEEP_BPS : 4>(p, s);
  } else {
    launch_tb<DIRS, R, MULTI, ACCUM, TOPG, WLAY, MODE, 2>(p, s);
  }
}

template <int DIRS, int R, bool TOPG, bool WLAY = false, int MODE = 0>
void launch_r(const SweepParams& p, cudaStream_t s) {
  const bool multi = p.g.n_mat > 1;
  const bool acc = p.base != nullptr;
  if (multi) acc ? launch_t<DIRS, R, true, true, TOPG, WLAY, MODE>(p, s) : launch_t<DIRS, R, true, false, TOPG, WLAY, MODE>(p, s);
  else acc ? launch_t<DIRS, R, false, true, TOPG, WLAY, MODE>(p, s) : launch_t<DIRS, R, false, false, TOPG, WLAY, MODE>(p, s);
}

}  // namespace

int sweep_rows_for(int nx, int ny) {
  // rows per CTA for 4-direction groups: the chained wavefront needs R <= nx
  int R = 64;
  while (R > 8 && (R > nx || R > ny)) R >>= 1;
  return R;
}

void launch_sweep(const SweepParams& p, cudaStream_t s) {
  if (p.g.n_groups == 0) return;
  if (p.g.nx < 8) throw std::invalid_argument("sweep: nx must be >= 8 on the B200 path");
  if (p.dirs == 8) {  // 8-direction groups, R = 32, traces across strips through the L2 scratch
    if (p.g.nx < kSweep8MinNx || p.g.ny < kSweep8MinNy || !p.top)
      throw std::invalid_argument("sweep: 8-direction groups need nx >= " + std::to_string(kSweep8MinNx) +
                                  " and ny >= " + std::to_string(kSweep8MinNy));
    if (p.wl.nd > 0) {
      if (p.wl.R != 32) throw std::invalid_argument("sweep: wavefront layout strip height must be 32");
      if (p.xb > 1) {  // column blocks (plain sweep, wavefront layout, B^-1 in registers)
        if (p.mode != 0 || p.base || !p.xflag || !p.xtrace || p.g.nx % p.xb || p.g.nx / p.xb < kSweep8MinNx)
          throw std::invalid_argument("sweep: column blocks need a plain sweep and nx / xb >= 38");
        // (B^-1 in shared memory at four CTAs per SM measured slower: 4.77 vs 3.53 ms per rank at N = 8)
        if (p.g.n_mat > 1) launch_tb<8, 32, true, false, true, true, 0, 2, true>(p, s);
        else launch_tb<8, 32, false, false, true, true, 0, 2, true>(p, s);
        return;
      }
      p.mode == 1 ? launch_r<8, 32, true, true, 1>(p, s) : launch_r<8, 32, true, true, 0>(p, s);
    } else {
      if (p.mode == 1) throw std::invalid_argument("sweep kernel apply_L mode needs the wavefront layout");
      launch_r<8, 32, true>(p, s);
    }
    return;
  }
  const int R = sweep_rows_for(p.g.nx, p.g.ny);
  switch (R) {
    case 64: launch_r<4, 64, false>(p, s); break;
    case 32: launch_r<4, 32, false>(p, s); break;
    case 16: launch_r<4, 16, false>(p, s); break;
    default: launch_r<4, 8, false>(p, s); break;
  }
}

}  // namespace stamg_b200
