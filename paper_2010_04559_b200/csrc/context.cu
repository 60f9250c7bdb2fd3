// Runtime of the B200 path: device-resident level tables and vectors, the
// operator orchestration that mirrors the reference's L2/L3 call graph
// (transport.cpp:96-101, sweeps.cpp:106-113, multigrid.cpp:138-176,
// krylov.cpp:9-93 + GMRES), and the C ABI declared in include/stamg_b200.h.
// Every operator is a sequence of kernel launches on the context's stream;
// the host only touches scalars (Krylov dot products).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <unordered_map>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "generic.hpp"
#include "kernels.hpp"
#include "setup.hpp"

using namespace stamg_b200;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NanError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
void ck_launch(const char* what) { ck(cudaGetLastError(), what); }

template <class T>
T* dalloc(size_t n) {
  if (n == 0) return nullptr;
  void* p = nullptr;
  ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}
template <class T>
T* dalloc_zero(size_t n, cudaStream_t s) {
  T* p = dalloc<T>(n);
  if (p) ck(cudaMemsetAsync(p, 0, n * sizeof(T), s), "memset");
  return p;
}
template <class T>
T* dupload(const std::vector<T>& v, cudaStream_t s) {
  T* p = dalloc<T>(v.size());
  if (p) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
  return p;
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
  void* h = nullptr;
  void* comm = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, const void*, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  int (*commSplit)(void*, int, int, void**, void*) = nullptr;  // ncclCommSplit (NCCL >= 2.18), optional
  bool load() {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
    commInitRank = reinterpret_cast<int (*)(void**, int, const void*, int)>(dlsym(h, "ncclCommInitRank"));
    allReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclAllReduce"));
    commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    commSplit = reinterpret_cast<int (*)(void*, int, int, void**, void*)>(dlsym(h, "ncclCommSplit"));
    return getUniqueId && commInitRank && allReduce && commDestroy;
  }
};
Nccl& nccl() {
  static Nccl n;
  return n;
}
// ncclUniqueId is passed by value (128 bytes); wrap it for the C call
struct UniqueId {
  char internal[128];
};

}  // namespace

// ------------------------------------------------------------------ device level
struct DevLevel {
  LevelTables t;
  // reference-shape path (generic.hpp): 3D / p0 / Lin levels; t then only carries the sizes
  gen::Tables gt;
  gen::Dev* g = nullptr;
  int64_t n = 0;  // vector length n_el * P * D * S
  bool sharded = false;  // holds only this rank's directions (scatter moments need an allreduce)
  int Hp = 0, Pk = 0, Pp = 0;
  double *X = nullptr, *XT = nullptr, *sig = nullptr, *ones = nullptr, *B = nullptr, *Binv = nullptr;
  double *cxy = nullptr, *BinvGS = nullptr, *sq = nullptr, *area = nullptr, *up_w = nullptr;
  int *groups = nullptr, *group_oct = nullptr, *oct_patches = nullptr, *oct_ptr = nullptr;
  int *groups8 = nullptr, *group8_oct = nullptr;
  double2* sweep_top = nullptr;  // 8-direction sweep: strip-boundary trace scratch
  int sweep_xb = 1;               // column blocks per group (sweep_kernel XBLK)
  int sweep_xb_g0 = 0;            // first group cut into column blocks (the groups before it are swept whole)
  int* sweep_xflag = nullptr;
  double2* sweep_xtrace = nullptr;
  // wavefront layout (contexts without a hierarchy): tables in internal (group-major)
  // patch order; vectors padded to n_groups8 * slots * 8 blocks
  WLGeom wl;                      // wl.nd == 0: reference layout
  std::vector<int> ipos;          // local reference patch index -> internal index
  int *d_ipos = nullptr, *d_iid = nullptr;
  double* stage = nullptr;        // chunked host <-> device conversion
  int64_t stage_n = 0;
  int *up = nullptr, *child_ptr = nullptr, *child_idx = nullptr;
  double* src = nullptr;  // scatter moments workspace [n_el][Hp][4]
  double* mom = nullptr;  // coarse GS moments
  int* gs_done = nullptr;
  double *gs_K = nullptr, *gs_Xo = nullptr, *gs_XoT = nullptr, *gs_G = nullptr, *gs_Minv = nullptr;
  int gs_blk = 0;  // blocked patch chain (multi-warp coarse GS)
  int gs_blocks = 0, gs_cpw = 0, gs_kpad = 0, gs_max_np = 0, gs_rows = 0, gs_mw = 0, gs_cluster = 0;
  int gs_mb_slots = 0, gs_mb_credit = 0;
  double *tmp = nullptr, *cf = nullptr, *ce = nullptr;  // V-cycle workspace
  // reflection-symmetry folded scatter (setup.hpp find_symmetry)
  int fold_G = 0, fold_R = 0, fold_Rp = 0, fold_Hf = 0;
  std::vector<int> fold_hoff;                 // [G+1] class column offsets
  std::vector<std::vector<int>> fold_hs;      // per class: ascending original harmonics
  double *Xf = nullptr, *XfT = nullptr, *sigf = nullptr;
  int* orbit = nullptr;
  std::vector<void*> owned;
};

struct stamg_ctx {
  Problem pb;
  SphereTree tree;
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  DevLevel outer;
  std::vector<DevLevel> mg;
  int nr = 0;
  bool have_mg = false;
  bool wl_allowed = false;
  int* mat = nullptr;
  double* q_el = nullptr;
  double nsum[4] = {0, 0, 0, 0};
  // Krylov workspace
  int restart_alloc = -1;
  std::vector<double*> V;
  double *z = nullptr, *u = nullptr, *partial = nullptr, *dots = nullptr, *coef = nullptr;
  double* hbuf = nullptr;  // pinned host scalars
  // host-buffer entry points
  double *hostio = nullptr;
  int64_t hostio_n = 0;
  // pipelined host-buffer sweep: copy streams, staging ring, events
  cudaStream_t io_h2d = nullptr, io_d2h = nullptr;
  double* pipe[3] = {nullptr, nullptr, nullptr};
  int64_t pipe_n = 0;
  cudaEvent_t pev[10] = {};
  int last_host_chunks = 0;  // chunks of the last stamg_sweep_host (0: unpipelined path)
  double* foldbuf = nullptr;  // reflection-fold workspace shared by all levels
  int64_t foldbuf_n = 0;
  int64_t launches = 0;
  bool timing = false;
  bool nvtx = false;  // STAMG_NVTX=1: NVTX ranges around operator launches and solver phases
  std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::map<std::string, std::pair<double, int64_t>> timed;
  void* comm = nullptr;
  // scatter-moment allreduce overlapped with the GEMMs: a second communicator (split from
  // comm) driven from its own stream, per-chunk events
  void* comm_ar = nullptr;
  cudaStream_t ar_stream = nullptr;
  std::vector<cudaEvent_t> ev_d2m, ev_ar;
  int ar_chunks_used = 0;
  // host collective (stamg_options.allreduce) and its pinned staging buffer
  stamg_allreduce_fn host_allreduce = nullptr;
  void* host_allreduce_user = nullptr;
  double* coll_host = nullptr;
  int64_t coll_host_n = 0;
  bool shard_probe = false;
  // CUDA graphs of mg_apply (one per (r, z) pair; the V-cycle is device-only)
  struct MgGraph {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
  };
  std::map<std::pair<const double*, double*>, MgGraph> mg_graphs;
  bool mg_warm = false, graphs_off = false;
  int64_t graph_replays = 0;
};

struct stamg_vec {
  stamg_ctx* ctx = nullptr;
  int level = 0;
  int64_t n = 0;
  double* d = nullptr;
};

namespace {

// -------------------------------------------------------------- timing helper
struct Timed {
  stamg_ctx* c;
  const char* name;
  cudaEvent_t e1 = nullptr;
  Timed(stamg_ctx* ctx, const char* nm) : c(ctx), name(nm) {
    if (c->nvtx) nvtxRangePushA(nm);  // STAMG_NVTX=1: one range per operator launch (nsys / ncu --nvtx)
    if (!c->timing) return;
    cudaEvent_t e0;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, c->stream), "event");
    c->pending[name].push_back({e0, e1});
  }
  ~Timed() {
    if (c->timing && e1) cudaEventRecord(e1, c->stream);
    if (c->nvtx) nvtxRangePop();
  }
};

// NVTX range over a solver phase (V-cycle level, Krylov solve) when STAMG_NVTX=1
struct NvtxScope {
  bool on;
  NvtxScope(const stamg_ctx* c, const std::string& name) : on(c->nvtx) {
    if (on) nvtxRangePushA(name.c_str());
  }
  ~NvtxScope() {
    if (on) nvtxRangePop();
  }
};

void resolve_timing(stamg_ctx* c) {
  ck(cudaStreamSynchronize(c->stream), "sync");
  for (auto& [name, v] : c->pending) {
    auto& acc = c->timed[name];
    for (auto& [a, b] : v) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
      acc.first += ms, acc.second += 1;
      cudaEventDestroy(a), cudaEventDestroy(b);
    }
    v.clear();
  }
}

GroupGeom geom(stamg_ctx* c, DevLevel& L) {
  GroupGeom g;
  g.groups = L.groups, g.group_oct = L.group_oct, g.n_groups = int(L.t.group_oct.size());
  g.P = L.t.P, g.nx = L.t.nx, g.ny = L.t.ny;
  g.n_mat = L.t.n_mat, g.mat = L.t.n_mat > 1 ? c->mat : nullptr;
  return g;
}

// tables in the sweep frame: dof i -> i ^ m, m = xneg | yneg << 1
std::vector<double> frame_blocks(const std::vector<double>& blk, const LevelTables& t) {
  std::vector<double> out(blk.size());
  const size_t nblk = blk.size() / 16;
  for (size_t b = 0; b < nblk; ++b) {
    const int q = int(b % t.P);
    const int m = t.octant[q] & 3;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) out[b * 16 + i * 4 + j] = blk[b * 16 + (i ^ m) * 4 + (j ^ m)];
  }
  return out;
}

// Reorder every per-patch table of a level into the internal (group-major) order
// iperm[k] = q; returns ipos (q -> k). Reference patch order stays in t.qpos.
std::vector<int> apply_internal_order(LevelTables& t) {
  const std::vector<int> iperm = t.groups8;  // flattened 8-direction groups (full, no padding)
  const int P = t.P;
  std::vector<int> ipos(P);
  for (int k = 0; k < P; ++k) ipos[iperm[k]] = k;
  auto perm_rows = [&](std::vector<double>& v, int row) {
    if (v.empty()) return;
    std::vector<double> o(v.size());
    const size_t blocks = v.size() / (size_t(P) * row);
    for (size_t b = 0; b < blocks; ++b)
      for (int k = 0; k < P; ++k)
        for (int j = 0; j < row; ++j) o[(b * P + k) * row + j] = v[(b * P + iperm[k]) * row + j];
    v.swap(o);
  };
  auto perm_int = [&](std::vector<int>& v) {
    std::vector<int> o(P);
    for (int k = 0; k < P; ++k) o[k] = v[iperm[k]];
    v.swap(o);
  };
  perm_int(t.leaf_id);
  perm_int(t.octant);
  perm_rows(t.X, t.H);
  perm_rows(t.B, 16);
  perm_rows(t.Binv, 16);
  perm_rows(t.C, 32);
  perm_rows(t.cxy, 8);
  perm_rows(t.area, 1);
  perm_rows(t.Aflow, 3);
  for (int& q : t.orbit) q = ipos[q];
  for (size_t k = 0; k < t.groups8.size(); ++k) t.groups8[k] = int(k);
  // 4-direction groups and octant lists in the new order
  t.groups.clear(), t.group_oct.clear(), t.oct_patches.clear();
  t.oct_ptr.assign(9, 0);
  for (int oct = 0; oct < 8; ++oct) {
    t.oct_ptr[oct] = int(t.oct_patches.size());
    std::vector<int> mine;
    for (int q = 0; q < P; ++q)
      if (t.octant[q] == oct) mine.push_back(q);
    t.oct_patches.insert(t.oct_patches.end(), mine.begin(), mine.end());
    for (size_t k = 0; k < mine.size(); k += 4) {
      for (int j = 0; j < 4; ++j) t.groups.push_back(k + j < mine.size() ? mine[k + j] : -1);
      t.group_oct.push_back(oct);
    }
  }
  t.oct_ptr[8] = int(t.oct_patches.size());
  return ipos;
}

// Solve contexts use 8-direction groups only with enough of them to give every SM two
// CTAs (configs 2-3 are faster with the 4-direction kernel's doubled CTA count).
// Throughput contexts (config 5, sharded over N GPUs) always use them, with the
// wavefront layout: rank 0's sweep of a 1/N slice on one GPU (tools/shard_probe.py)
// takes 6.04 / 3.71 ms at N = 4 / 8 against 9.03 / 5.32 ms with 4-direction groups
// (3.9x / 6.3x instead of 2.6x / 4.4x over one GPU's 23.4 ms).
int sweep8_min_groups(const stamg_ctx* c, int sms) {
  return c->wl_allowed ? 1 : 2 * sms;
}

bool env_is_zero(const char* name) {
  const char* v = std::getenv(name);
  return v != nullptr && v[0] == '0' && v[1] == 0;
}

// Inverses of the coarse-GS chain's diagonal blocks (sweeps.cpp:93-101 restated as a linear
// system): for block J of an octant (patches a = 4J..4J+3, octant order) and material m,
// T = I - blockdiag(G_a) (L x I_4) with L[a][b] = K[a][b] for b < a inside the block. T is unit
// lower block-triangular, so T^-1 = I + S + S^2 + S^3 with S = I - T (formed in long double).
// Packed per block as column c from row 4 (c / 4): [m][octant][kpad / 4][kGsMinvBlock].
std::vector<double> gs_minv_table(const LevelTables& t, const std::vector<double>& K, const std::vector<double>& G, int kpad) {
  const int nb = kpad / 4;
  std::vector<double> out(size_t(t.n_mat) * 8 * nb * kGsMinvBlock, 0.0);
  for (int m = 0; m < t.n_mat; ++m)
    for (int o = 0; o < 8; ++o) {
      const int pbeg = t.oct_ptr[o], np = t.oct_ptr[o + 1] - pbeg;
      for (int J = 0; J < nb; ++J) {
        long double S[16][16] = {}, M[16][16] = {}, Pw[16][16] = {};
        for (int r = 1; r < 4; ++r) {
          const int a = 4 * J + r;
          if (a >= np) continue;
          const double* Ga = &G[(size_t(m) * t.P + t.oct_patches[pbeg + a]) * 16];
          for (int r2 = 0; r2 < r; ++r2) {
            const double k = K[(size_t(m) * t.P + pbeg + a) * kpad + 4 * J + r2];
            for (int i = 0; i < 4; ++i)
              for (int j = 0; j < 4; ++j) S[4 * r + i][4 * r2 + j] = (long double)Ga[4 * i + j] * k;
          }
        }
        for (int i = 0; i < 16; ++i) M[i][i] = Pw[i][i] = 1.0L;
        for (int pw = 1; pw < 4; ++pw) {  // Pw = S^pw, M += Pw
          long double Nx[16][16] = {};
          for (int i = 0; i < 16; ++i)
            for (int k = 0; k < 16; ++k) {
              if (S[i][k] == 0.0L) continue;
              for (int j = 0; j < 16; ++j) Nx[i][j] += S[i][k] * Pw[k][j];
            }
          for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) Pw[i][j] = Nx[i][j], M[i][j] += Nx[i][j];
        }
        double* dst = &out[((size_t(m) * 8 + o) * nb + J) * kGsMinvBlock];
        for (int c = 0; c < 16; ++c) {
          const int cb = c / 4, base = 64 * cb - 8 * cb * (cb - 1) + (c % 4) * (16 - 4 * cb);
          for (int r = 4 * cb; r < 16; ++r) dst[base + r - 4 * cb] = double(M[r][c]);
        }
      }
    }
  return out;
}

void upload_level(stamg_ctx* c, DevLevel& L) {
  cudaStream_t s = c->stream;
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const auto& t0 = L.t;
    if (c->wl_allowed && !t0.groups8.empty() && !t0.groups8_padded && t0.nx >= kSweep8MinNx && t0.ny >= kSweep8MinNy &&
        int(t0.group8_oct.size()) >= sweep8_min_groups(c, sms) && !env_is_zero("STAMG_WAVEFRONT_LAYOUT")) {
      // default for throughput contexts: every sweep step of a group touches one
      // contiguous 8 KB run (90 % of measured HBM bandwidth at 512^2 x 8192 against
      // 82.5 % for the reference layout's 256-byte runs); STAMG_WAVEFRONT_LAYOUT=0
      // keeps the reference layout
      L.ipos = apply_internal_order(L.t);
      L.wl.nx = t0.nx, L.wl.ny = t0.ny, L.wl.R = 32, L.wl.nd = t0.nx + 32 - 1;
      L.wl.slots = (long long)((t0.ny + 31) / 32) * L.wl.nd * 32;
    }
  }
  const auto& t = L.t;
  L.n = L.wl.nd ? int64_t(t.group8_oct.size()) * L.wl.slots * 32 : int64_t(t.n_el) * t.P * 4;
  if (L.wl.nd) {
    std::vector<int> iid(t.P);
    for (int k = 0; k < t.P; ++k) iid[k] = k;
    L.d_ipos = dupload(L.ipos, s), L.d_iid = dupload(iid, s);
  }
  L.Hp = round_up(t.H, 64);
  L.Pk = round_up(t.P, 32);  // X rows padded for any GEMM k-tile (16 or 32)
  L.Pp = round_up(t.P, 64);
  std::vector<double> X(size_t(L.Pk) * L.Hp, 0.0), XT(size_t(L.Hp) * L.Pp, 0.0), sig(size_t(t.n_mat) * L.Hp, 0.0);
  for (int q = 0; q < t.P; ++q)
    for (int h = 0; h < t.H; ++h) X[size_t(q) * L.Hp + h] = XT[size_t(h) * L.Pp + q] = t.X[size_t(q) * t.H + h];
  for (int m = 0; m < t.n_mat; ++m)
    for (int h = 0; h < t.H; ++h) sig[size_t(m) * L.Hp + h] = t.sig[size_t(m) * t.H + h];
  std::vector<double> ones(size_t(t.n_mat) * L.Hp, 1.0);
  std::vector<double> cxyf(t.cxy.size());
  for (int q = 0; q < t.P; ++q) {
    const int xn = t.octant[q] & 1, yn = (t.octant[q] >> 1) & 1;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        cxyf[q * 8 + a * 2 + b] = t.cxy[q * 8 + (a ^ yn) * 2 + (b ^ yn)];
        cxyf[q * 8 + 4 + a * 2 + b] = t.cxy[q * 8 + 4 + (a ^ xn) * 2 + (b ^ xn)];
      }
  }
  L.X = dupload(X, s), L.XT = dupload(XT, s), L.sig = dupload(sig, s), L.ones = dupload(ones, s);
  L.B = dupload(frame_blocks(t.B, t), s);
  L.Binv = dupload(frame_blocks(t.Binv, t), s);
  L.cxy = dupload(cxyf, s);
  L.area = dupload(t.area, s);
  L.groups = dupload(t.groups, s), L.group_oct = dupload(t.group_oct, s);
  // 8-direction groups (256-byte runs) only where they still give >= 2 CTAs per SM;
  // small levels keep the 4-direction kernels (twice the CTAs, latency-bound anyway)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  if (!t.groups8.empty() && t.nx >= kSweep8MinNx && t.ny >= kSweep8MinNy && int(t.group8_oct.size()) >= sweep8_min_groups(c, sms)) {
    L.groups8 = dupload(t.groups8, s), L.group8_oct = dupload(t.group8_oct, s);
    L.sweep_top = dalloc<double2>(t.group8_oct.size() * 8 * size_t(t.nx));
    // fewer groups than SMs (config 5 sharded over 8 GPUs: 128 per rank): two column blocks per
    // group so the wavefronts cover twice the SMs (STAMG_SWEEP_XBLOCKS=0 keeps one block).
    // With more groups than CTA slots (config 5 on one GPU: 1024 groups on 296 slots = 3.46
    // waves run as 4) cutting every group measured slower (23.8 ms with one block, 26.3 with
    // two, 29.2 with four; profiles/r02_sweep_ab.txt): a block's strip hand-off costs more
    // than the shorter tail saves. Cutting only the tail wave (the groups of the full waves
    // swept whole, the remaining ones in xb blocks when those fit one wave; STAMG_SWEEP_TAIL=1)
    // does not pay either: 23.5 ms against 23.1 ms. The waves are not equally long -- the
    // kernel is bandwidth-bound while they are full, and the 136 CTAs of the last wave run
    // faster per CTA -- so there is less tail to recover than the wave count suggests.
    // STAMG_SWEEP_XB forces a block count for all groups (A/B).
    const int ng = int(t.group8_oct.size());
    if (c->wl_allowed && !env_is_zero("STAMG_SWEEP_XBLOCKS")) {
      auto ok = [&](int xb) { return xb >= 1 && t.nx % xb == 0 && t.nx / xb >= kSweep8MinNx; };
      const int slots = 2 * sms;
      int best = 1, g0 = 0;
      if (ng <= sms && ok(2)) best = 2;
      else if (ng > slots && ng % slots != 0 && std::getenv("STAMG_SWEEP_TAIL") != nullptr &&
               !env_is_zero("STAMG_SWEEP_TAIL")) {
        const int rem = ng % slots;
        for (int xb : {4, 2})
          if (ok(xb) && rem * xb <= slots) {
            best = xb, g0 = ng - rem;
            break;
          }
      }
      if (const char* e = std::getenv("STAMG_SWEEP_XB")) {  // A/B
        const int xb = std::atoi(e);
        if (ok(xb)) best = xb, g0 = 0;
      }
      if (best > 1) {
        L.sweep_xb = best, L.sweep_xb_g0 = g0;
        L.sweep_xflag = dalloc<int>(size_t(ng) * L.sweep_xb + 1);  // + the block ticket
        L.sweep_xtrace = dalloc<double2>(size_t(ng) * L.sweep_xb * t.ny * 8);
      }
    }
  }
  if (L.wl.nd) {
    if (!L.groups8) throw std::logic_error("wavefront layout needs the 8-direction groups");
    L.wl.goct = L.group8_oct;
  }
  L.oct_patches = dupload(t.oct_patches, s), L.oct_ptr = dupload(t.oct_ptr, s);
  if (!t.BinvGS.empty()) {
    L.BinvGS = dupload(frame_blocks(t.BinvGS, t), s);
    L.sq = dupload(t.sq, s);
    L.mom = dalloc<double>(size_t(t.n_el) * L.Hp * 4);
    L.gs_done = dalloc<int>(size_t(8) * t.n_el);
    // K[m][q][b] = X_q sig_m X_b^T for b in q's octant (coarse GS chain)
    for (int o = 0; o < 8; ++o) L.gs_max_np = std::max(L.gs_max_np, t.oct_ptr[o + 1] - t.oct_ptr[o]);
    L.gs_kpad = std::max(4, round_up(L.gs_max_np, 4));  // whole 4-patch chain blocks, 16-byte staging chunks
    std::vector<double> K(size_t(t.n_mat) * t.P * L.gs_kpad, 0.0);
    for (int m = 0; m < t.n_mat; ++m)
      for (int o = 0; o < 8; ++o)
        for (int a = t.oct_ptr[o]; a < t.oct_ptr[o + 1]; ++a)
          for (int b = t.oct_ptr[o]; b < t.oct_ptr[o + 1]; ++b) {
            const int qa = t.oct_patches[a], qb = t.oct_patches[b];
            double k = 0;
            for (int h = 0; h < t.H; ++h)
              k += t.X[size_t(qa) * t.H + h] * t.sig[size_t(m) * t.H + h] * t.X[size_t(qb) * t.H + h];
            K[(size_t(m) * t.P + a) * L.gs_kpad + (b - t.oct_ptr[o])] = k;
          }
    if (L.gs_kpad % 2) L.gs_kpad += 0;  // rows padded below
    L.gs_K = dupload(K, s);
    {  // G = B'^-1 N in the sweep frame (N is invariant under the frame permutation)
      const auto Bf = frame_blocks(t.BinvGS, t);
      std::vector<double> G(Bf.size());
      for (size_t b = 0; b < Bf.size() / 16; ++b)
        for (int i = 0; i < 4; ++i)
          for (int j = 0; j < 4; ++j) {
            double acc = 0;
            for (int k = 0; k < 4; ++k) acc += Bf[b * 16 + i * 4 + k] * t.Nmat[k * 4 + j];
            G[b * 16 + i * 4 + j] = acc;
          }
      L.gs_G = dupload(G, s);
      L.gs_Minv = dupload(gs_minv_table(t, K, G, L.gs_kpad), s);
    }
    std::vector<double> Xo(size_t(t.P) * L.Hp, 0.0), XoT(size_t(L.Hp) * t.P, 0.0);
    for (int a = 0; a < t.P; ++a)
      for (int h = 0; h < t.H; ++h)
        Xo[size_t(a) * L.Hp + h] = XoT[size_t(h) * t.P + a] = t.X[size_t(t.oct_patches[a]) * t.H + h];
    L.gs_Xo = dupload(Xo, s);
    L.gs_XoT = dupload(XoT, s);
    // static ownership: each warp owns a segment of gs_cpw consecutive cells of one row
    // row mode pays off once rows are long (measured: c2, c3 faster; c1 at 32^2 slower)
    // a 4-warp CTA per grid row, software-pipelined (projections and moment updates of
    // the neighbouring items beside the chain); measured faster on every BASELINE config
    // (10 passes: c1 12.8 -> 10.4 ms, c2 26.7 -> 20.7, c3 55.7 -> 36.8, c4 640 -> 337).
    // STAMG_GS_MW=0 keeps the one-warp kernels
    // blocked chain where an octant's patches are one or two blocks (configs 1-2: 4 patches,
    // 8.6 -> 7.6 and 17.7 -> 15.6 ms per coarse solve); at one patch there is no chain
    // (config 3), and at 64 patches (config 4) the per-block shared-memory round trips cost
    // more than the sixteen-fold shorter chain saves (0.314 -> 0.46 s; profiles/r02_gs_c4_chain.txt).
    // STAMG_GS_CHAIN_BLOCKS=1 / 0 force it on / off.
    bool want_blk = false;
    {
      const char* e = std::getenv("STAMG_GS_CHAIN_BLOCKS");
      const bool forced_on = e != nullptr && e[0] == '1' && e[1] == 0;
      want_blk = coarse_gs_chain_blocked() && (forced_on || (L.gs_max_np >= 2 && L.gs_max_np <= 8));
    }
    L.gs_mw = !env_is_zero("STAMG_GS_MW") &&
              coarse_gs_mw_ok(L.Hp, t.H, L.gs_kpad, t.n_mat, t.ny, L.gs_max_np, want_blk);
    L.gs_blk = L.gs_mw && want_blk;
    L.gs_rows = t.nx < 64
                    ? 0
                    : coarse_gs_rows_wpb(L.Hp, L.gs_kpad, t.n_mat, t.nx, t.ny, L.gs_max_np);
    if (L.gs_mw) {  // one 4-warp CTA per grid row
      L.gs_rows = 0, L.gs_cpw = t.nx, L.gs_blocks = t.ny;
      // rows grouped in thread-block clusters: y-hops inside a cluster through DSMEM
      // mailboxes (STAMG_GS_CLUSTER=0 keeps every hop in global memory)
      const int cl = env_is_zero("STAMG_GS_CLUSTER")
                         ? 0
                         : coarse_gs_cluster_rows(L.Hp, t.H, L.gs_kpad, t.n_mat, t.nx, t.ny, L.gs_max_np, L.gs_blk != 0);
      L.gs_cluster = cl & 127, L.gs_mb_credit = (cl >> 7) & 1, L.gs_mb_slots = cl >> 8;
    } else {
      const int max_warps = coarse_gs_max_warps(L.Hp, L.gs_kpad, t.n_mat, L.gs_max_np);
      int seg = 1;
      while (int64_t(t.n_el) / seg > max_warps || t.nx % seg != 0) {
        if (seg >= t.nx) throw std::invalid_argument("coarse_scatter_sweep: grid too large for co-resident warps");
        seg *= 2;
      }
      L.gs_cpw = seg;
      const int W = t.n_el / seg;
      const int wpb = coarse_gs_warps_per_block(L.Hp, L.gs_kpad, t.n_mat);
      L.gs_blocks = (W + wpb - 1) / wpb;
    }
    if (L.gs_rows) {  // row mode: a warp per grid row, CTAs of gs_rows consecutive rows
      L.gs_cpw = t.nx;
      L.gs_blocks = t.ny / L.gs_rows;
    }

  }
  if (!t.up.empty()) {
    L.up = dupload(t.up, s), L.up_w = dupload(t.up_w, s);
    L.child_ptr = dupload(t.child_ptr, s), L.child_idx = dupload(t.child_idx, s);
  }
  size_t src_rows = L.Hp;
  // fold only where the GEMMs are big enough to pay for the two streaming passes
  int fold_min_h = 128;
  if (const char* e = std::getenv("STAMG_FOLD_MIN_H")) fold_min_h = std::atoi(e);
  // exactness: the coupling table must satisfy the reflection identity (sym_defect, measured
  // in find_symmetry; config 1's level-2 mesh misses it by 2.2e-9 and never folds).
  // size: orbit classes of >= 64 patches (smaller class GEMMs do not pay for the two
  // streaming passes). sharded levels fold when the rank's patch set is closed under the
  // reflections (throughput shards and orbit-partitioned hierarchies are; find_symmetry
  // checks closure among the rank's own patches); the folded moments are allreduced
  const bool fold_exact = t.n_sym_axes > 0 && t.sym_defect <= kFoldMaxDefect;
  if (fold_exact && t.H >= fold_min_h && (t.P >> t.n_sym_axes) >= 64) {
    const int G = 1 << t.n_sym_axes, R = t.P / G;
    L.fold_G = G, L.fold_R = R, L.fold_Rp = round_up(R, 64);
    const int Rk = round_up(R, 32);
    L.fold_hs.assign(G, {});
    for (int h = 0; h < t.H; ++h) L.fold_hs[t.hclass[h]].push_back(h);
    L.fold_hoff.assign(G + 1, 0);
    for (int cl = 0; cl < G; ++cl) {  // class region: whole D2M row tiles (d2m_row_tile)
      const int hc = std::max<int>(1, L.fold_hs[cl].size()), bm = d2m_row_tile(hc, 1 << 30);
      L.fold_hoff[cl + 1] = L.fold_hoff[cl] + round_up(hc, bm);
    }
    L.fold_Hf = L.fold_hoff[G];
    std::vector<double> Xf(size_t(Rk) * L.fold_Hf, 0.0), XfT(size_t(L.fold_Hf) * L.fold_Rp, 0.0);
    std::vector<double> sigf(size_t(t.n_mat) * L.fold_Hf, 0.0);
    for (int cl = 0; cl < G; ++cl)
      for (size_t j = 0; j < L.fold_hs[cl].size(); ++j) {
        const int h = L.fold_hs[cl][j], col = L.fold_hoff[cl] + int(j);
        for (int r = 0; r < R; ++r)
          Xf[size_t(r) * L.fold_Hf + col] = XfT[size_t(col) * L.fold_Rp + r] = t.X[size_t(t.orbit[r * G]) * t.H + h];
        for (int m = 0; m < t.n_mat; ++m) sigf[size_t(m) * L.fold_Hf + col] = t.sig[size_t(m) * t.H + h];
      }
    L.Xf = dupload(Xf, s), L.XfT = dupload(XfT, s), L.sigf = dupload(sigf, s);
    L.orbit = dupload(t.orbit, s);
    src_rows = std::max<size_t>(src_rows, L.fold_Hf);
  }
  L.src = dalloc<double>(size_t(t.n_el) * src_rows * 4);
  ck(cudaStreamSynchronize(s), "upload sync");
}

// reference-shape levels: the dense per-patch tables as they are
void upload_gen_level(stamg_ctx* c, DevLevel& L) {
  cudaStream_t s = c->stream;
  const gen::Tables& t = L.gt;
  L.t.n_el = t.n_el, L.t.P = t.P, L.t.order = t.order, L.t.H = t.H, L.t.n_mat = 1, L.t.nx = t.nx, L.t.ny = t.ny;
  L.t.leaf_id = t.leaf_id, L.t.octant = t.octant, L.t.oct_ptr = t.oct_ptr, L.t.oct_patches = t.oct_patches;
  L.t.up = t.up;
  L.t.qpos.resize(t.P);
  for (int q = 0; q < t.P; ++q) L.t.qpos[q] = q;
  L.t.P_global = t.P;
  L.n = int64_t(t.n_el) * t.P * t.bs;
  auto* g = new gen::Dev();
  L.g = g;
  g->dim = t.dim, g->nx = t.nx, g->ny = t.ny, g->nz = t.nz, g->n_el = t.n_el, g->S = t.S, g->D = t.D, g->bs = t.bs;
  g->P = t.P, g->H = t.H, g->order = t.order;
  {
    const int R = t.P * t.D;
    std::vector<double> XT(size_t(t.H) * R);
    for (int r = 0; r < R; ++r)
      for (int h = 0; h < t.H; ++h) XT[size_t(h) * R + r] = t.X[size_t(r) * t.H + h];
    g->XT = dupload(XT, s);
  }
  g->X = dupload(t.X, s), g->sig = dupload(t.sig, s), g->Bd = dupload(t.Bd, s), g->Binv = dupload(t.Binv, s);
  g->C = dupload(t.C, s), g->Nmat = dupload(t.Nmat, s);
  g->octant = dupload(t.octant, s), g->oct_patches = dupload(t.oct_patches, s), g->oct_ptr = dupload(t.oct_ptr, s);
  g->src = dalloc<double>(size_t(t.n_el) * t.H * t.S);
  if (!t.BinvGS.empty()) {
    g->BinvGS = dupload(t.BinvGS, s);
    g->mom = dalloc<double>(size_t(t.n_el) * t.H * t.S);
    if (std::getenv("STAMG_GENERIC_GS_BARRIER") == nullptr) g->gs_prog = dalloc<int>(size_t(t.ny) * t.nz);
  }
  if (!t.up.empty()) {
    g->up = dupload(t.up, s), g->upB = dupload(t.upB, s);
    g->child_ptr = dupload(t.child_ptr, s), g->child_idx = dupload(t.child_idx, s);
  }
  for (int o = 0; o < 8; ++o) g->max_np = std::max(g->max_np, t.oct_ptr[o + 1] - t.oct_ptr[o]);
  if (t.nx < 1024 && t.ny < 1024 && t.nz < 1024 && t.bs % 8 == 0) {  // hyperplane cell lists (tensor-core sweep)
    const int npl = t.nx + t.ny + t.nz - 2;
    std::vector<int> ptr(npl + 1, 0), cells(size_t(t.n_el));
    for (int fk = 0; fk < t.nz; ++fk)
      for (int fj = 0; fj < t.ny; ++fj)
        for (int fi = 0; fi < t.nx; ++fi) ptr[fi + fj + fk + 1]++;
    for (int p = 0; p < npl; ++p) ptr[p + 1] += ptr[p];
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int fk = 0; fk < t.nz; ++fk)
      for (int fj = 0; fj < t.ny; ++fj)
        for (int fi = 0; fi < t.nx; ++fi) cells[size_t(fill[fi + fj + fk]++)] = fi | (fj << 10) | (fk << 20);
    g->plane_cells = dupload(cells, s), g->plane_ptr = dupload(ptr, s);
  }
  ck(cudaStreamSynchronize(s), "upload sync");
}

void free_level(DevLevel& L) {
  if (L.g) {
    gen::Dev* g = L.g;
    for (void* p : {(void*)g->XT, (void*)g->X, (void*)g->sig, (void*)g->Bd, (void*)g->Binv, (void*)g->C, (void*)g->BinvGS,
                    (void*)g->Nmat, (void*)g->upB, (void*)g->src, (void*)g->mom, (void*)g->octant,
                    (void*)g->oct_patches, (void*)g->oct_ptr, (void*)g->up, (void*)g->child_ptr, (void*)g->child_idx,
                    (void*)g->gs_prog, (void*)g->plane_cells, (void*)g->plane_ptr})
      if (p) cudaFree(p);
    delete g;
    L.g = nullptr;
  }
  for (void* p : {(void*)L.X, (void*)L.XT, (void*)L.sig, (void*)L.ones, (void*)L.B, (void*)L.Binv, (void*)L.cxy,
                  (void*)L.BinvGS, (void*)L.sq, (void*)L.area, (void*)L.up_w, (void*)L.groups, (void*)L.group_oct,
                  (void*)L.oct_patches, (void*)L.oct_ptr, (void*)L.up, (void*)L.child_ptr, (void*)L.child_idx,
                  (void*)L.src, (void*)L.mom, (void*)L.gs_done, (void*)L.gs_K, (void*)L.gs_Xo, (void*)L.gs_XoT, (void*)L.gs_G, (void*)L.gs_Minv, (void*)L.Xf, (void*)L.XfT, (void*)L.groups8, (void*)L.group8_oct, (void*)L.sweep_top, (void*)L.sweep_xflag, (void*)L.sweep_xtrace,
                  (void*)L.d_ipos, (void*)L.d_iid, (void*)L.stage,
                  (void*)L.sigf, (void*)L.orbit, (void*)L.tmp, (void*)L.cf,
                  (void*)L.ce})
    if (p) cudaFree(p);
}

DevLevel& level_of(stamg_ctx* c, int level) {
  if (level == STAMG_OUTER) return c->outer;
  if (!c->have_mg) throw std::invalid_argument("multigrid hierarchy was not built for this context");
  if (level < 0 || level >= int(c->mg.size())) throw std::invalid_argument("level out of range");
  return c->mg[level];
}

void need(const stamg_vec* v, const DevLevel& L, const char* what) {
  if (!v || v->n != L.n) throw std::invalid_argument(std::string(what) + ": layout mismatch");
}

// ------------------------------------------------------------------ operators
void op_allreduce(stamg_ctx* c, double* buf, size_t n) {
  if (c->world <= 1 || n == 0) return;
  if (c->shard_probe) return;  // explicit timing option (stamg_options.shard_probe): partial sums
  if (c->host_allreduce) {     // host collective: device -> pinned host, callback, host -> device
    if (c->coll_host_n < int64_t(n)) {
      if (c->coll_host) cudaFreeHost(c->coll_host);
      c->coll_host = nullptr, c->coll_host_n = 0;
      ck(cudaMallocHost(&c->coll_host, n * sizeof(double)), "cudaMallocHost");
      c->coll_host_n = int64_t(n);
    }
    ck(cudaMemcpyAsync(c->coll_host, buf, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (c->host_allreduce(c->host_allreduce_user, c->coll_host, int64_t(n)) != 0)
      throw NcclError("host allreduce callback failed");
    ck(cudaMemcpyAsync(buf, c->coll_host, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
    return;
  }
  if (!c->comm) throw std::logic_error("allreduce: no communicator");
  const int ncclDouble = 8, ncclSum = 0;
  if (nccl().allReduce(buf, buf, n, ncclDouble, ncclSum, c->comm, c->stream) != 0)
    throw NcclError("ncclAllReduce failed");
}

void op_apply_L(stamg_ctx* c, DevLevel& L, const double* x, double* y, double alpha = 1.0, double beta = 0.0,
                const double* f = nullptr) {
  Timed tm(c, "apply_L");
  if (L.g) {
    gen::launch_apply_L(*L.g, x, y, alpha, beta, f, c->stream);
    ck_launch("apply_L");
    c->launches += 1;
    return;
  }
  if (L.wl.nd) {  // wavefront layout: the sweep's skewed schedule, apply_L arithmetic
    SweepParams p;
    p.g = geom(c, L);
    p.dirs = 8, p.top = L.sweep_top, p.wl = L.wl, p.mode = 1;
    p.g.groups = L.groups8, p.g.group_oct = L.group8_oct, p.g.n_groups = int(L.t.group8_oct.size());
    p.rhs = x, p.z = y, p.base = (f && beta != 0.0) ? f : nullptr, p.alpha = alpha, p.beta = beta;
    p.Bfwd = L.B, p.Binv = L.Binv, p.cxy = L.cxy, p.prefer_breg = true;
    launch_sweep(p, c->stream);
    ck_launch("apply_L");
    c->launches += 1;
    return;
  }
  ApplyLParams p;
  p.g = geom(c, L);
  if (L.groups8) {
    p.dirs = 8;
    p.g.groups = L.groups8, p.g.group_oct = L.group8_oct, p.g.n_groups = int(L.t.group8_oct.size());
  }
  p.x = x, p.y = y, p.f = f, p.alpha = alpha, p.beta = beta, p.B = L.B, p.cxy = L.cxy;
  launch_apply_L(p, c->stream);
  ck_launch("apply_L");
  c->launches += 1;
}

void op_d2m(stamg_ctx* c, DevLevel& L, const double* phi, int order, double* out, const double* sig, bool identity_N) {
  Timed tm(c, "d2m");
  D2MParams p;
  p.wl = L.wl;
  p.phi = phi, p.src = out, p.X = L.X, p.sig = sig, p.mat = L.t.n_mat > 1 ? c->mat : nullptr;
  p.n_el = L.t.n_el, p.P = L.t.P, p.Hp = L.Hp, p.Hused = (order + 1) * (order + 1), p.Hrows = L.Hp;
  for (int k = 0; k < 16; ++k) p.N[k] = identity_N ? ((k % 5) == 0 ? 1.0 : 0.0) : L.t.Nmat[k];
  launch_d2m(p, c->stream);
  ck_launch("d2m");
  c->launches += 1;
}


// element-range chunks of a sharded scatter: D2M of chunk k+1 overlaps the moment
// allreduce of chunk k, which overlaps the M2D of chunk k-1 (STAMG_AR_CHUNKS overrides;
// one chunk for unsharded levels, the shard probe, or without a second communicator)
int scatter_chunks(stamg_ctx* c, const DevLevel& L) {
  if (!L.sharded || c->world <= 1 || c->shard_probe) return 1;
  int k = c->comm_ar ? 8 : 1;
  if (const char* e = std::getenv("STAMG_AR_CHUNKS")) k = std::max(1, std::atoi(e));
  if (!c->comm_ar && !c->host_allreduce) k = 1;
  return std::max(1, std::min({k, 64, L.t.n_el}));
}

void ensure_ar_events(stamg_ctx* c, int k) {
  while (int(c->ev_d2m.size()) < k) {
    cudaEvent_t a, b;
    ck(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
    c->ev_d2m.push_back(a), c->ev_ar.push_back(b);
  }
}

// allreduce of one moment chunk on the comm stream (second communicator), after the
// chunk's D2M; the chunk's M2D waits for ev_ar[k]
void allreduce_chunk_async(stamg_ctx* c, double* buf, size_t n, int k) {
  ck(cudaEventRecord(c->ev_d2m[k], c->stream), "event");
  ck(cudaStreamWaitEvent(c->ar_stream, c->ev_d2m[k], 0), "wait");
  const int ncclDouble = 8, ncclSum = 0;
  if (nccl().allReduce(buf, buf, n, ncclDouble, ncclSum, c->comm_ar, c->ar_stream) != 0)
    throw NcclError("ncclAllReduce (moment chunk) failed");
  ck(cudaEventRecord(c->ev_ar[k], c->ar_stream), "event");
}

// y = beta*y + scale * S_order phi (+ isotropic source): apply_scatter_into
// (scatter.cpp:110-135) as D2M -> [allreduce] -> M2D. With a reflection
// symmetry group G the patches are folded over their orbits (Walsh-Hadamard),
// each harmonic parity class is one GEMM with K = P/|G|, and the result is
// unfolded: the same algebra with |G| times fewer flops. Sharded levels run
// element-range chunks so the moment allreduce overlaps the GEMMs.
void scatter_into(stamg_ctx* c, DevLevel& L, const double* phi, int order, double scale, double beta, double* y,
                  const double* ext) {
  if (order > L.t.order) throw std::invalid_argument("sigma_by_harmonic: max_order exceeds kernel order");
  if (L.g) {  // reference-shape level: y += scale X sigma (X^T phi) N
    if (beta != 1.0 || ext) throw std::invalid_argument("the reference-shape path applies the scatter operator only as y += scale * S phi");
    {
      Timed tm(c, "d2m");
      gen::launch_d2m(*L.g, phi, order, true, L.g->src, c->stream);
      ck_launch("d2m");
    }
    Timed tm(c, "m2d");
    gen::launch_m2d(*L.g, L.g->src, order, scale, y, c->stream);
    ck_launch("m2d");
    c->launches += 2;
    return;
  }
  const int Hu = (order + 1) * (order + 1);
  const int n_el = L.t.n_el;
  const int K = scatter_chunks(c, L);
  c->ar_chunks_used = K;
  const bool async_ar = K > 1 && c->comm_ar != nullptr;
  if (async_ar) ensure_ar_events(c, K);
  auto chunk = [&](int k, int& e0, int& e1) {
    e0 = int(int64_t(n_el) * k / K), e1 = int(int64_t(n_el) * (k + 1) / K);
  };
  const size_t Hrow = L.fold_G == 0 ? size_t(L.Hp) : size_t(L.fold_Hf);  // src row pitch
  // moments of chunk k: after its D2M, before its M2D
  auto reduce_chunk = [&](int k, bool issue) {
    if (!L.sharded) return;
    int e0, e1;
    chunk(k, e0, e1);
    double* buf = L.src + size_t(e0) * Hrow * 4;
    const size_t n = size_t(e1 - e0) * Hrow * 4;
    if (async_ar) {
      if (issue) allreduce_chunk_async(c, buf, n, k);
      else ck(cudaStreamWaitEvent(c->stream, c->ev_ar[k], 0), "wait");
    } else if (!issue) {
      op_allreduce(c, buf, n);
    }
  };
  if (L.fold_G == 0) {
    for (int k = 0; k < K; ++k) {
      int e0, e1;
      chunk(k, e0, e1);
      Timed tm(c, "d2m");
      D2MParams p;
      p.wl = L.wl;
      p.phi = phi, p.src = L.src, p.X = L.X, p.sig = L.sig, p.mat = L.t.n_mat > 1 ? c->mat : nullptr;
      p.n_el = e1 - e0, p.el_base = e0, p.P = L.t.P, p.Hp = L.Hp, p.Hused = Hu, p.Hrows = L.Hp;
      for (int i = 0; i < 16; ++i) p.N[i] = L.t.Nmat[i];
      launch_d2m(p, c->stream);
      ck_launch("d2m");
      c->launches += 1;
      reduce_chunk(k, true);
    }
    for (int k = 0; k < K; ++k) {
      int e0, e1;
      chunk(k, e0, e1);
      reduce_chunk(k, false);
      Timed tm(c, "m2d");
      M2DParams p;
      p.wl = L.wl;
      p.src = L.src, p.y = y, p.XT = L.XT, p.n_el = e1 - e0, p.el_base = e0, p.P = L.t.P, p.Pp = L.Pp, p.Hp = L.Hp;
      p.Hused = Hu, p.scale = scale, p.beta = beta, p.ext_q = ext, p.area = L.area;
      for (int i = 0; i < 4; ++i) p.nsum[i] = c->nsum[i];
      launch_m2d(p, c->stream);
      ck_launch("m2d");
      c->launches += 1;
    }
    return;
  }
  const int G = L.fold_G, R = L.fold_R;
  // one fold workspace per context, shared by the levels (used only inside this call)
  const int64_t need = int64_t(n_el) * L.t.P * 4;
  if (c->foldbuf_n < need) {
    if (c->foldbuf) cudaFree(c->foldbuf);
    c->foldbuf = dalloc<double>(need);
    c->foldbuf_n = need;
  }
  double* const fb = c->foldbuf;
  const size_t cls = size_t(n_el) * R * 4;
  std::vector<int> hu(G, 0);
  for (int cl = 0; cl < G; ++cl)
    for (int h : L.fold_hs[cl]) hu[cl] += h < Hu ? 1 : 0;
  for (int k = 0; k < K; ++k) {
    int e0, e1;
    chunk(k, e0, e1);
    {
      Timed tm(c, "fold");
      launch_fold(phi, fb, L.orbit, n_el, e0, e1, L.t.P, R, G, L.wl, c->stream);
      ck_launch("fold");
      c->launches += 1;
    }
    for (int cl = 0; cl < G; ++cl) {
      if (hu[cl] == 0) continue;
      Timed tm(c, "d2m");
      D2MParams p;
      p.phi = fb + cl * cls, p.src = L.src + size_t(L.fold_hoff[cl]) * 4, p.X = L.Xf + L.fold_hoff[cl];
      p.sig = L.sigf + L.fold_hoff[cl], p.mat = L.t.n_mat > 1 ? c->mat : nullptr;
      p.n_el = e1 - e0, p.el_base = e0, p.P = R, p.Hp = L.fold_Hf, p.Hused = hu[cl];
      p.Hrows = L.fold_hoff[cl + 1] - L.fold_hoff[cl];
      for (int i = 0; i < 16; ++i) p.N[i] = L.t.Nmat[i];
      launch_d2m(p, c->stream);
      ck_launch("d2m");
      c->launches += 1;
    }
    reduce_chunk(k, true);
  }
  for (int k = 0; k < K; ++k) {
    int e0, e1;
    chunk(k, e0, e1);
    reduce_chunk(k, false);
    for (int cl = 0; cl < G; ++cl) {
      double* Yc = fb + cl * cls;
      if (hu[cl] == 0) {
        launch_fill(Yc + size_t(e0) * R * 4, 0.0, int64_t(e1 - e0) * R * 4, c->stream);
        c->launches += 1;
        continue;
      }
      Timed tm(c, "m2d");
      M2DParams p;
      p.src = L.src + size_t(L.fold_hoff[cl]) * 4, p.y = Yc, p.XT = L.XfT + size_t(L.fold_hoff[cl]) * L.fold_Rp;
      p.n_el = e1 - e0, p.el_base = e0, p.P = R, p.Pp = L.fold_Rp, p.Hp = L.fold_Hf, p.Hused = hu[cl];
      p.scale = 1.0, p.beta = 0.0, p.ext_q = nullptr, p.area = L.area;
      for (int i = 0; i < 4; ++i) p.nsum[i] = c->nsum[i];
      launch_m2d(p, c->stream);
      ck_launch("m2d");
      c->launches += 1;
    }
    Timed tm(c, "unfold");
    launch_unfold(fb, y, L.orbit, n_el, e0, e1, L.t.P, R, G, scale, beta, ext, L.area, c->nsum, L.wl, c->stream);
    ck_launch("unfold");
    c->launches += 1;
  }
}

void op_scatter(stamg_ctx* c, DevLevel& L, const double* phi, int order, double scale, double* y) {
  if (order > L.t.order) throw std::invalid_argument("sigma_by_harmonic: max_order exceeds kernel order");
  if (order < 0) return;
  scatter_into(c, L, phi, order, scale, 1.0, y, nullptr);
}

// apply_A_into (transport.cpp:96-101)
void op_apply_A(stamg_ctx* c, DevLevel& L, const double* x, int order, double* y) {
  op_apply_L(c, L, x, y);
  op_scatter(c, L, x, order, -1.0, y);
}

// r = f - A_order phi
void op_residual(stamg_ctx* c, DevLevel& L, const double* f, const double* phi, int order, double* r) {
  op_apply_L(c, L, phi, r, -1.0, 1.0, f);
  op_scatter(c, L, phi, order, 1.0, r);
}

void op_sweep(stamg_ctx* c, DevLevel& L, const double* rhs, double* z, const double* base = nullptr) {
  Timed tm(c, "sweep");
  if (L.g) {
    if (base) throw std::logic_error("reference-shape sweep has no fused base vector");
    gen::launch_sweep(*L.g, rhs, z, c->stream);
    ck_launch("sweep");
    c->launches += 1;
    return;
  }
  SweepParams p;
  p.g = geom(c, L);
  if (L.sweep_top) {
    p.dirs = 8, p.top = L.sweep_top, p.wl = L.wl;
    p.g.groups = L.groups8, p.g.group_oct = L.group8_oct, p.g.n_groups = int(L.t.group8_oct.size());
  }
  p.rhs = rhs, p.z = z, p.base = base, p.Binv = L.Binv, p.cxy = L.cxy;
  // wavefront-layout (throughput) contexts keep B^-1 in registers at two CTAs per SM even
  // when the groups would fit one wave at four: rank 0 of 2 (512 groups) sweeps in 12.5 ms
  // against 14.6 ms (tools/shard_probe.py); solve contexts (config 4's 364 cone-mesh
  // groups) keep the one-wave choice
  p.prefer_breg = L.wl.nd > 0;
  if (L.sweep_xb > 1 && !base) {
    p.xb = L.sweep_xb, p.xb_g0 = L.sweep_xb_g0, p.xflag = L.sweep_xflag, p.xtrace = L.sweep_xtrace;
    {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
      const int ngr = int(L.t.group8_oct.size());
      p.xb_ticket = L.sweep_xb_g0 + (ngr - L.sweep_xb_g0) * L.sweep_xb > 2 * sms ? 1 : 0;
    }
    ck(cudaMemsetAsync(L.sweep_xflag, 0, sizeof(int) * (L.t.group8_oct.size() * L.sweep_xb + 1), c->stream), "memset");
  }
  launch_sweep(p, c->stream);
  ck_launch("sweep");
  c->launches += 1;
}

// smoother_step (sweeps.cpp:106-113): phi += L^{-1}(f - A phi), the add fused into the sweep
void op_smoother(stamg_ctx* c, DevLevel& L, const double* f, int order, double* phi) {
  if (!L.tmp) L.tmp = dalloc_zero<double>(L.n, c->stream);
  op_residual(c, L, f, phi, order, L.tmp);
  if (L.g) {  // sweep the residual in place, then add (sweeps.cpp:110-112)
    op_sweep(c, L, L.tmp, L.tmp);
    launch_axpy(1.0, L.tmp, phi, L.n, c->stream);
    c->launches += 1;
    return;
  }
  op_sweep(c, L, L.tmp, phi, phi);
}

// phi_zero: the caller has just zero-filled phi (the V-cycle's coarse correction), so its
// moments are zero without a D2M
void op_coarse_gs(stamg_ctx* c, DevLevel& L, const double* rhs, int nu, double* phi, bool phi_zero = false) {
  if (nu <= 0) return;
  if (L.g) {
    if (!L.g->BinvGS) throw std::invalid_argument("coarse_scatter_sweep: not the coarsest level");
    Timed tm(c, "coarse_gs");
    gen::launch_coarse_gs(*L.g, rhs, nu, phi, c->stream);
    ck_launch("coarse_gs");
    c->launches += 2;
    return;
  }
  if (!L.BinvGS) throw std::invalid_argument("coarse_scatter_sweep: not the coarsest level");
  // per-element moments of the current iterate (sweeps.cpp:74-79)
  if (phi_zero) ck(cudaMemsetAsync(L.mom, 0, sizeof(double) * size_t(L.t.n_el) * L.Hp * 4, c->stream), "memset");
  else op_d2m(c, L, phi, L.t.order, L.mom, L.ones, true);
  ck(cudaMemsetAsync(L.gs_done, 0, sizeof(int) * 8 * size_t(L.t.n_el), c->stream), "memset");
  Timed tm(c, "coarse_gs");
  CoarseGSParams p;
  p.rhs = rhs, p.phi = phi, p.mom = L.mom, p.X = L.X, p.sig = L.sig, p.BinvGS = L.BinvGS, p.sq = L.sq, p.cxy = L.cxy;
  p.oct_patches = L.oct_patches, p.oct_ptr = L.oct_ptr, p.mat = L.t.n_mat > 1 ? c->mat : nullptr;
  p.done = L.gs_done, p.K = L.gs_K, p.Xo = L.gs_Xo, p.XoT = L.gs_XoT, p.GS = L.gs_G, p.n_mat = L.t.n_mat;
  p.cells_per_warp = L.gs_cpw, p.kpad = L.gs_kpad, p.grid_blocks = L.gs_blocks, p.rows_mode = L.gs_rows;
  p.multi_warp = L.gs_mw;
  p.Minv = L.gs_Minv, p.chain_blk = L.gs_blk;
  p.cluster = L.gs_cluster, p.mb_np = L.gs_max_np, p.mb_slots = L.gs_mb_slots, p.mb_credit = L.gs_mb_credit;
  p.mom_stride = L.gs_mb_credit ? (L.t.H + 1) / 2 * 2 : 0;
  p.xreg = 1;
  p.n_el = L.t.n_el, p.P = L.t.P, p.Hp = L.Hp, p.H = L.t.H, p.nx = L.t.nx, p.ny = L.t.ny, p.nu = nu;
  for (int o = 0; o < 8; ++o)
    p.max_patches_per_octant = std::max(p.max_patches_per_octant, L.t.oct_ptr[o + 1] - L.t.oct_ptr[o]);
  for (int k = 0; k < 16; ++k) p.N[k] = L.t.Nmat[k];
  launch_coarse_gs(p, c->stream);
  ck_launch("coarse_gs");
  c->launches += 1;
}

void op_prolong(stamg_ctx* c, int l, const double* coarse, double* fine, bool add) {
  DevLevel& F = c->mg[l];
  DevLevel& Cl = c->mg[l - 1];
  Timed tm(c, "prolong");
  if (F.g) {
    gen::launch_prolong(*F.g, coarse, fine, Cl.t.P, add, c->stream);
    ck_launch("prolong");
    c->launches += 1;
    return;
  }
  launch_prolong(coarse, fine, F.up, F.up_w, F.t.n_el, F.t.P, Cl.t.P, add, c->stream);
  ck_launch("prolong");
  c->launches += 1;
}

void op_restrict(stamg_ctx* c, int l, const double* fine, double* coarse) {
  DevLevel& F = c->mg[l];
  DevLevel& Cl = c->mg[l - 1];
  Timed tm(c, "restrict");
  if (F.g) {
    gen::launch_restrict(*F.g, fine, coarse, Cl.t.P, c->stream);
    ck_launch("restrict");
    c->launches += 1;
    return;
  }
  launch_restrict(fine, coarse, F.child_ptr, F.child_idx, F.up_w, F.t.n_el, F.t.P, Cl.t.P, c->stream);
  ck_launch("restrict");
  c->launches += 1;
  // into the replicated coarsest level: each rank filled only its own parents
  // (zeros elsewhere); the sum over ranks is exact
  if (F.sharded && !Cl.sharded) op_allreduce(c, coarse, size_t(Cl.n));
}

double op_dot(stamg_ctx* c, const double* x, const double* y, int64_t n, bool sharded);

// lmg_vcycle (multigrid.cpp:138-170)
// zero_guess: phi is to be taken as zero whatever it holds (mg_apply's z and every coarse
// correction, multigrid.cpp:138-176 start from zero). The first pre-smoothing step is then
// phi = L^-1 f -- its residual f - A*0 is f itself, so the apply_L, the D2M / M2D pair and
// the base-vector read of the sweep are skipped; the results are those of the full sequence
// (0 * x and f - 0 are exact), only the sign of a zero can differ. A third of the MG levels'
// operator applications (STAMG_MG_ZERO_GUESS=0 runs the full sequence).
void op_vcycle(stamg_ctx* c, int l, const double* f, double* phi, bool zero_guess = false) {
  NvtxScope nv(c, "lmg_vcycle level " + std::to_string(l));
  DevLevel& L = c->mg[l];
  const auto& spec = c->pb.spec;
  auto zero_fill = [&]() {
    launch_fill(phi, 0.0, L.n, c->stream);
    c->launches += 1;
  };
  if (zero_guess && env_is_zero("STAMG_MG_ZERO_GUESS")) {  // A/B: fill and run the full sequence
    zero_fill();
    zero_guess = false;
  }
  if (l == 0) {
    if (zero_guess) zero_fill();
    if (spec.coarse_tol > 0) {
      if (!L.tmp) L.tmp = dalloc_zero<double>(L.n, c->stream);
      const double fnorm = std::sqrt(op_dot(c, f, f, L.n, L.sharded));
      for (int s = 0; s < 200; ++s) {
        op_coarse_gs(c, L, f, 1, phi, zero_guess && s == 0);
        op_residual(c, L, f, phi, L.t.order, L.tmp);
        if (std::sqrt(op_dot(c, L.tmp, L.tmp, L.n, L.sharded)) <= spec.coarse_tol * fnorm) break;
      }
    } else {
      op_coarse_gs(c, L, f, spec.coarse_sweeps, phi, zero_guess);
    }
    return;
  }
  DevLevel& Cl = c->mg[l - 1];
  if (!L.tmp) L.tmp = dalloc_zero<double>(L.n, c->stream);
  if (!Cl.cf) Cl.cf = dalloc_zero<double>(Cl.n, c->stream), Cl.ce = dalloc_zero<double>(Cl.n, c->stream);
  int s0 = 0;
  if (zero_guess) {
    if (spec.nu_pre > 0) op_sweep(c, L, f, phi), s0 = 1;
    else zero_fill();
  }
  for (int s = s0; s < spec.nu_pre; ++s) op_smoother(c, L, f, c->nr, phi);
  op_residual(c, L, f, phi, c->nr, L.tmp);
  op_restrict(c, l, L.tmp, Cl.cf);
  op_vcycle(c, l - 1, Cl.cf, Cl.ce, true);
  op_prolong(c, l, Cl.ce, phi, true);
  for (int s = 0; s < spec.nu_post; ++s) op_smoother(c, L, f, c->nr, phi);
}

void op_mg_apply(stamg_ctx* c, const double* r, double* z) {
  const int top = int(c->mg.size()) - 1;
  op_vcycle(c, top, r, z, true);
}

// mg_apply through a CUDA graph: the V-cycle is a fixed sequence of
// ~10-100 launches with no host round trip (coarse_tol = 0, one rank), so after one eager
// call (which allocates the level workspaces) it is captured once per (r, z) pair and
// replayed. Timing mode (per-launch events), host collectives and the coarse_tol loop
// (host dot products) stay eager; STAMG_GRAPHS=0 disables graphs. A capture the driver
// rejects turns graphs off for the context and runs eagerly.
void op_mg_apply_graph(stamg_ctx* c, const double* r, double* z) {
  const bool ok = !c->graphs_off && c->world == 1 && c->pb.spec.coarse_tol <= 0 && !c->timing &&
                  !env_is_zero("STAMG_GRAPHS");
  if (!ok || !c->mg_warm) {
    op_mg_apply(c, r, z);
    c->mg_warm = true;
    return;
  }
  const auto key = std::make_pair(r, z);
  auto it = c->mg_graphs.find(key);
  if (it == c->mg_graphs.end()) {
    if (c->mg_graphs.size() >= 64) {  // bounded cache (ABI callers may pass many vectors)
      for (auto& kv : c->mg_graphs) cudaGraphExecDestroy(kv.second.exec);
      c->mg_graphs.clear();
    }
    const int64_t l0 = c->launches;
    cudaGraph_t graph = nullptr;
    ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      op_mg_apply(c, r, z);
    } catch (...) {
      cudaStreamEndCapture(c->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      c->launches = l0;
      c->graphs_off = true;
      op_mg_apply(c, r, z);
      return;
    }
    const cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
    stamg_ctx::MgGraph mg;
    mg.launches = c->launches - l0;
    c->launches = l0;
    if (e != cudaSuccess || !graph || cudaGraphInstantiate(&mg.exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      c->graphs_off = true;
      op_mg_apply(c, r, z);
      return;
    }
    cudaGraphDestroy(graph);
    it = c->mg_graphs.emplace(key, mg).first;
  }
  ck(cudaGraphLaunch(it->second.exec, c->stream), "graph launch");
  c->launches += it->second.launches;
  c->graph_replays += 1;
}

// --------------------------------------------------------------- BLAS helpers
void ensure_krylov(stamg_ctx* c, int restart) {
  if (c->restart_alloc >= restart) return;
  for (double* v : c->V) cudaFree(v);
  c->V.clear();
  if (c->z) cudaFree(c->z), c->z = nullptr;
  if (c->u) cudaFree(c->u), c->u = nullptr;
  const int64_t n = c->outer.n;
  for (int k = 0; k <= restart; ++k) c->V.push_back(dalloc<double>(n));
  c->z = dalloc<double>(n);
  c->u = dalloc<double>(n);
  // zeroed once: wavefront-layout vectors have padding slots that the operators never
  // write but the dot products and axpys run over (padding must stay 0, never NaN)
  for (double* v : c->V) ck(cudaMemsetAsync(v, 0, n * sizeof(double), c->stream), "memset");
  ck(cudaMemsetAsync(c->z, 0, n * sizeof(double), c->stream), "memset");
  ck(cudaMemsetAsync(c->u, 0, n * sizeof(double), c->stream), "memset");
  c->restart_alloc = restart;
}

void ensure_scalars(stamg_ctx* c) {
  if (c->partial) return;
  c->partial = dalloc<double>(size_t(multidot_blocks()) * 82);
  c->dots = dalloc<double>(82);
  c->coef = dalloc<double>(82);
  ck(cudaMallocHost(&c->hbuf, 82 * sizeof(double)), "cudaMallocHost");
}

void op_multidot(stamg_ctx* c, const std::vector<const double*>& vs, const double* w, int64_t n, double* out_host,
                 bool sharded) {
  ensure_scalars(c);
  launch_multidot(vs.data(), int(vs.size()), w, n, c->partial, c->dots, c->stream);
  ck_launch("multidot");
  c->launches += 2;
  if (sharded && c->world > 1) op_allreduce(c, c->dots, vs.size());  // partial dots of sharded vectors
  ck(cudaMemcpyAsync(c->hbuf, c->dots, vs.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
  ck(cudaStreamSynchronize(c->stream), "sync");
  std::memcpy(out_host, c->hbuf, vs.size() * sizeof(double));
}

double op_dot(stamg_ctx* c, const double* x, const double* y, int64_t n, bool sharded) {
  double d = 0;
  op_multidot(c, {x}, y, n, &d, sharded);
  (void)y;
  return d;
}

void upload_coef(stamg_ctx* c, const double* host, int k) {
  ensure_scalars(c);
  std::memcpy(c->hbuf, host, k * sizeof(double));
  ck(cudaMemcpyAsync(c->coef, c->hbuf, k * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
}

void apply_precond(stamg_ctx* c, int precond, const double* v, double* z) {
  if (precond == 0) op_sweep(c, c->outer, v, z);
  else if (precond == 1) op_mg_apply_graph(c, v, z);
  else {
    ck(cudaMemcpyAsync(z, v, c->outer.n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
  }
}

// GMRES(m), right preconditioned, CGS2 + Givens; same algorithm and reporting
// as the oracle's gmres (oracle/stamg_oracle.cpp) and krylov.hpp:15-24.
stamg_report op_gmres(stamg_ctx* c, int precond, const double* b, double* x, double tol, int max_iter, int m,
                      std::vector<double>& hist) {
  if (tol <= 0) throw std::invalid_argument("gmres: tol must be positive");
  if (m < 1 || m > 79) throw std::invalid_argument("gmres: restart must be in [1, 79]");
  NvtxScope nv(c, "gmres");
  const auto t0 = std::chrono::steady_clock::now();
  stamg_report rep{};
  DevLevel& O = c->outer;
  const int64_t n = O.n;
  ensure_krylov(c, m);
  launch_fill(x, 0.0, n, c->stream);
  const double bnorm = std::sqrt(op_dot(c, b, b, n, O.sharded));
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  if (bnorm == 0.0) {
    rep.converged = 1;
    rep.wall_time = elapsed();
    return rep;
  }
  ck(cudaMemcpyAsync(c->V[0], b, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
  int it = 0;
  bool done = false;
  std::vector<double> cs(m), sn(m), g(m + 1), y(m), dots(m + 1);
  std::vector<std::vector<double>> H(m, std::vector<double>(m + 1));
  while (!done) {
    const double beta = std::sqrt(op_dot(c, c->V[0], c->V[0], n, O.sharded));
    launch_scale(1.0 / beta, c->V[0], n, c->stream);
    std::fill(g.begin(), g.end(), 0.0);
    for (auto& col : H) std::fill(col.begin(), col.end(), 0.0);
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      ++it;
      apply_precond(c, precond, c->V[j], c->z);
      ++rep.preconditioner_applications;
      double* w = c->V[j + 1];
      op_apply_A(c, O, c->z, c->pb.spec.N, w);
      auto& h = H[j];
      std::vector<const double*> basis(c->V.begin(), c->V.begin() + j + 1);
      for (int pass = 0; pass < 2; ++pass) {  // CGS2
        op_multidot(c, basis, w, n, dots.data(), O.sharded);
        upload_coef(c, dots.data(), j + 1);
        launch_multi_axpy(basis.data(), j + 1, c->coef, w, n, c->stream);
        c->launches += 1;
        for (int i = 0; i <= j; ++i) h[i] += dots[i];
      }
      h[j + 1] = std::sqrt(op_dot(c, w, w, n, O.sharded));
      if (h[j + 1] != 0.0) launch_scale(1.0 / h[j + 1], w, n, c->stream), c->launches += 1;
      for (int i = 0; i < j; ++i) {
        const double tmp = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = tmp;
      }
      const double den = std::hypot(h[j], h[j + 1]);
      cs[j] = den == 0.0 ? 1.0 : h[j] / den;
      sn[j] = den == 0.0 ? 0.0 : h[j + 1] / den;
      const double hj1 = h[j + 1];
      h[j] = cs[j] * h[j] + sn[j] * hj1;
      h[j + 1] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      const double res = std::abs(g[j + 1]) / bnorm;
      if (std::isnan(res)) throw NanError("gmres: NaN residual");
      rep.iterations = it;
      hist.push_back(res);
      k = j + 1;
      if (res < tol || it >= max_iter || hj1 == 0.0) {
        done = true;
        if (hj1 == 0.0 && !(res < tol)) rep.breakdown = 1;
        break;
      }
    }
    for (int i = k - 1; i >= 0; --i) {
      double s = g[i];
      for (int jj = i + 1; jj < k; ++jj) s -= H[jj][i] * y[jj];
      y[i] = s / H[i][i];
    }
    upload_coef(c, y.data(), k);
    std::vector<const double*> basis(c->V.begin(), c->V.begin() + k);
    launch_lincomb(basis.data(), k, c->coef, c->u, n, c->stream);
    c->launches += 1;
    apply_precond(c, precond, c->u, c->z);
    ++rep.preconditioner_applications;
    launch_axpy(1.0, c->z, x, n, c->stream);
    c->launches += 1;
    if (done) break;
    op_apply_A(c, O, x, c->pb.spec.N, c->V[0]);
    launch_axpby(1.0, b, -1.0, c->V[0], n, c->stream);
    c->launches += 1;
  }
  op_apply_A(c, O, x, c->pb.spec.N, c->z);
  launch_axpby(1.0, b, -1.0, c->z, n, c->stream);
  rep.final_residual = std::sqrt(op_dot(c, c->z, c->z, n, O.sharded)) / bnorm;
  rep.converged = rep.final_residual < tol;
  rep.wall_time = elapsed();
  return rep;
}

// BiCGSTAB (krylov.cpp:9-93), right preconditioned, x0 = 0
stamg_report op_bicgstab(stamg_ctx* c, int precond, const double* b, double* x, double tol, int max_iter,
                         std::vector<double>& hist) {
  if (tol <= 0) throw std::invalid_argument("bicgstab: tol must be positive");
  NvtxScope nv(c, "bicgstab");
  const auto t0 = std::chrono::steady_clock::now();
  stamg_report rep{};
  DevLevel& O = c->outer;
  const int64_t n = O.n;
  ensure_krylov(c, 6);
  double *r = c->V[0], *rhat = c->V[1], *p = c->V[2], *v = c->V[3], *s = c->V[4], *t = c->V[5], *phat = c->V[6];
  double* shat = c->z;
  launch_fill(x, 0.0, n, c->stream);
  const double bnorm = std::sqrt(op_dot(c, b, b, n, O.sharded));
  auto finish = [&]() {
    if (bnorm > 0) {
      op_apply_A(c, O, x, c->pb.spec.N, c->u);
      launch_axpby(1.0, b, -1.0, c->u, n, c->stream);
      rep.final_residual = std::sqrt(op_dot(c, c->u, c->u, n, O.sharded)) / bnorm;
    }
    rep.converged = rep.final_residual < tol;
    rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
  };
  if (bnorm == 0.0) {
    rep.converged = 1;
    return rep;
  }
  ck(cudaMemcpyAsync(r, b, n * 8, cudaMemcpyDeviceToDevice, c->stream), "copy");
  ck(cudaMemcpyAsync(rhat, b, n * 8, cudaMemcpyDeviceToDevice, c->stream), "copy");
  launch_fill(p, 0.0, n, c->stream);
  launch_fill(v, 0.0, n, c->stream);
  double rho = 1, alpha = 1, omega = 1;
  for (int it = 1; it <= max_iter; ++it) {
    const double rho1 = op_dot(c, rhat, r, n, O.sharded);
    if (rho1 == 0.0 || omega == 0.0) {
      rep.breakdown = 1;
      return finish();
    }
    const double beta = (rho1 / rho) * (alpha / omega);
    rho = rho1;
    launch_axpy(-omega, v, p, n, c->stream);      // p - omega v
    launch_axpby(1.0, r, beta, p, n, c->stream);  // r + beta (...)
    apply_precond(c, precond, p, phat);
    ++rep.preconditioner_applications;
    op_apply_A(c, O, phat, c->pb.spec.N, v);
    const double rv = op_dot(c, rhat, v, n, O.sharded);
    if (rv == 0.0) {
      rep.breakdown = 1;
      return finish();
    }
    alpha = rho / rv;
    ck(cudaMemcpyAsync(s, r, n * 8, cudaMemcpyDeviceToDevice, c->stream), "copy");
    launch_axpy(-alpha, v, s, n, c->stream);
    launch_axpy(alpha, phat, x, n, c->stream);
    const double snorm = std::sqrt(op_dot(c, s, s, n, O.sharded)) / bnorm;
    if (std::isnan(snorm)) throw NanError("bicgstab: NaN residual");
    if (snorm < tol) {
      rep.iterations = it;
      hist.push_back(snorm);
      return finish();
    }
    apply_precond(c, precond, s, shat);
    ++rep.preconditioner_applications;
    op_apply_A(c, O, shat, c->pb.spec.N, t);
    const double tt = op_dot(c, t, t, n, O.sharded);
    if (tt == 0.0) {
      rep.breakdown = 1;
      return finish();
    }
    omega = op_dot(c, t, s, n, O.sharded) / tt;
    launch_axpy(omega, shat, x, n, c->stream);
    ck(cudaMemcpyAsync(r, s, n * 8, cudaMemcpyDeviceToDevice, c->stream), "copy");
    launch_axpy(-omega, t, r, n, c->stream);
    c->launches += 10;
    const double rnorm = std::sqrt(op_dot(c, r, r, n, O.sharded)) / bnorm;
    if (std::isnan(rnorm)) throw NanError("bicgstab: NaN residual");
    rep.iterations = it;
    hist.push_back(rnorm);
    if (rnorm < tol) return finish();
  }
  return finish();
}

// host (reference layout, or internal patch order with `internal`) <-> device vector of a level
void host_to_vec(stamg_ctx* c, DevLevel& L, const double* host, double* dev, bool internal) {
  const int64_t nref = L.g ? L.n : int64_t(L.t.n_el) * L.t.P * 4;
  if (!L.wl.nd) {
    ck(cudaMemcpyAsync(dev, host, nref * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
    return;
  }
  const int64_t per_el = int64_t(L.t.P) * 4;
  const int chunk = int(std::max<int64_t>(1, std::min<int64_t>(L.t.n_el, (int64_t(64) << 20) / per_el)));
  if (L.stage_n < chunk * per_el) {
    if (L.stage) cudaFree(L.stage);
    L.stage = dalloc<double>(size_t(chunk) * per_el);
    L.stage_n = chunk * per_el;
  }
  for (int el0 = 0; el0 < L.t.n_el; el0 += chunk) {
    const int n = std::min(chunk, L.t.n_el - el0);
    ck(cudaMemcpyAsync(L.stage, host + el0 * per_el, n * per_el * sizeof(double), cudaMemcpyHostToDevice, c->stream),
       "h2d");
    launch_to_wl(L.stage, dev, internal ? L.d_iid : L.d_ipos, el0, n, L.t.P, L.wl, c->stream);
    ck_launch("to_wl");
  }
}
void vec_to_host(stamg_ctx* c, DevLevel& L, const double* dev, double* host, bool internal) {
  const int64_t nref = L.g ? L.n : int64_t(L.t.n_el) * L.t.P * 4;
  if (!L.wl.nd) {
    ck(cudaMemcpyAsync(host, dev, nref * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    return;
  }
  const int64_t per_el = int64_t(L.t.P) * 4;
  const int chunk = int(std::max<int64_t>(1, std::min<int64_t>(L.t.n_el, (int64_t(64) << 20) / per_el)));
  if (L.stage_n < chunk * per_el) {
    if (L.stage) cudaFree(L.stage);
    L.stage = dalloc<double>(size_t(chunk) * per_el);
    L.stage_n = chunk * per_el;
  }
  for (int el0 = 0; el0 < L.t.n_el; el0 += chunk) {
    const int n = std::min(chunk, L.t.n_el - el0);
    launch_from_wl(dev, L.stage, internal ? L.d_iid : L.d_ipos, el0, n, L.t.P, L.wl, c->stream);
    ck_launch("from_wl");
    ck(cudaMemcpyAsync(host + el0 * per_el, L.stage, n * per_el * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
       "d2h");
  }
}
int64_t ref_size(const DevLevel& L) { return L.g ? L.n : int64_t(L.t.n_el) * L.t.P * 4; }

template <class F>
int guard(F&& f) {
  try {
    f();
    return STAMG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return STAMG_EINVAL;
  } catch (const NanError& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return STAMG_ENAN;
  } catch (const CudaError& e) {
    g_err = std::string("cuda: ") + e.what();
    return STAMG_ECUDA;
  } catch (const NcclError& e) {
    g_err = std::string("nccl: ") + e.what();
    return STAMG_ENCCL;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return STAMG_ELOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return STAMG_ECUDA;
  }
}

// every context-taking entry point binds the context's device first: kernels,
// allocations and per-device function attributes then land on the right GPU
// even when one host thread drives contexts on several devices
template <class F>
int guard_ctx(stamg_ctx* c, F&& f) {
  if (!c) {
    g_err = "invalid_argument: null context";
    return STAMG_EINVAL;
  }
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != c->device) {
    const cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) {
      g_err = std::string("cuda: cudaSetDevice: ") + cudaGetErrorString(e);
      return STAMG_ECUDA;
    }
  }
  return guard(std::forward<F>(f));
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* stamg_last_error(void) { return g_err.c_str(); }
int stamg_version(void) { return 1; }

int stamg_nccl_unique_id(void* out128) {
  return guard([&] {
    if (!nccl().load()) throw NcclError("libnccl.so.2 not loadable");
    if (nccl().getUniqueId(out128) != 0) throw NcclError("ncclGetUniqueId failed");
  });
}

// One-rank round trip through the NCCL calls the sharded contexts make: dlopen, unique id,
// ncclCommInitRank (the id by value), ncclCommSplit (the overlap communicator), two
// ncclAllReduce of n doubles on a non-blocking stream, destroy. On one GPU the sum over one
// rank is the identity, which is what is checked; it shows that the library's NCCL (whichever
// libnccl.so.2 the process already holds, e.g. torch's) loads, matches the call signatures
// and runs on this device.
int stamg_nccl_selftest(int device, int64_t n, int* version_out) {
  return guard([&] {
    if (n <= 0) throw std::invalid_argument("stamg_nccl_selftest: n must be positive");
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (!nccl().load()) throw NcclError("libnccl.so.2 not loadable");
    if (version_out) {
      *version_out = 0;
      auto getv = reinterpret_cast<int (*)(int*)>(dlsym(nccl().h, "ncclGetVersion"));
      if (getv) getv(version_out);
    }
    UniqueId uid;
    if (nccl().getUniqueId(&uid) != 0) throw NcclError("ncclGetUniqueId failed");
    void *comm = nullptr, *comm2 = nullptr;
    auto init = reinterpret_cast<int (*)(void**, int, UniqueId, int)>(nccl().commInitRank);
    if (init(&comm, 1, uid, 0) != 0) throw NcclError("ncclCommInitRank failed");
    if (nccl().commSplit && nccl().commSplit(comm, 0, 0, &comm2, nullptr) != 0) comm2 = nullptr;
    cudaStream_t st = nullptr;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    const size_t nn = static_cast<size_t>(n);
    std::vector<double> h(nn, 0.0), back(nn, 0.0);
    for (int64_t i = 0; i < n; ++i) h[size_t(i)] = 0.25 * double(i % 1024) - 7.0;
    double* d = dalloc<double>(size_t(n));
    ck(cudaMemcpyAsync(d, h.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    const int ncclDouble = 8, ncclSum = 0;
    int rc = nccl().allReduce(d, d, size_t(n), ncclDouble, ncclSum, comm, st);
    if (rc == 0 && comm2) rc = nccl().allReduce(d, d, size_t(n), ncclDouble, ncclSum, comm2, st);
    if (rc == 0) ck(cudaMemcpyAsync(back.data(), d, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    const cudaError_t se = cudaStreamSynchronize(st);
    cudaFree(d);
    cudaStreamDestroy(st);
    if (comm2) nccl().commDestroy(comm2);
    nccl().commDestroy(comm);
    if (rc != 0) throw NcclError("ncclAllReduce failed");
    ck(se, "sync");
    if (back != h) throw NcclError("one-rank allreduce did not return its input");
  });
}

int stamg_create(const stamg_problem* prob, const stamg_options* opt, stamg_ctx** out) {
  return guard([&] {
    if (!prob || !out) throw std::invalid_argument("stamg_create: null argument");
    auto c = std::make_unique<stamg_ctx>();
    c->pb = copy_problem(*prob);
    const bool generic = gen::handles(*prob);
    if (generic) gen::validate(c->pb);
    else validate(c->pb);
    c->pb.device_setup = std::getenv("STAMG_HOST_SETUP") == nullptr;  // couplings on the device
    c->nvtx = std::getenv("STAMG_NVTX") != nullptr && !env_is_zero("STAMG_NVTX");
    c->device = opt ? opt->device : 0;
    c->rank = opt ? opt->rank : 0;
    c->world = opt ? std::max(1, opt->world) : 1;
    const bool want_mg = opt ? opt->build_hierarchy != 0 : true;
    c->wl_allowed = !want_mg;  // wavefront layout only for contexts without a hierarchy
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    if (c->world > 1) {
      if (!opt) throw std::invalid_argument("world > 1 needs options");
      if (c->rank < 0 || c->rank >= c->world) throw std::invalid_argument("stamg_create: rank out of range");
      const int kinds = (opt->nccl_id != nullptr) + (opt->allreduce != nullptr) + (opt->shard_probe != 0);
      if (kinds != 1)
        throw std::invalid_argument("world > 1 needs exactly one of nccl_id, allreduce, shard_probe");
    }
    if (c->world > 1 && opt->allreduce) {
      c->host_allreduce = opt->allreduce, c->host_allreduce_user = opt->allreduce_user;
    } else if (c->world > 1 && opt->shard_probe) {
      c->shard_probe = true;
    } else if (c->world > 1) {
      if (!nccl().load()) throw NcclError("libnccl.so.2 not loadable");
      UniqueId uid;
      std::memcpy(uid.internal, opt->nccl_id, 128);
      // ncclCommInitRank(comm*, nranks, ncclUniqueId (by value), rank)
      auto init = reinterpret_cast<int (*)(void**, int, UniqueId, int)>(nccl().commInitRank);
      if (init(&c->comm, c->world, uid, c->rank) != 0) throw NcclError("ncclCommInitRank failed");
      // second communicator for the chunked moment allreduce on its own stream (the dot
      // products stay on the first, ordered on the compute stream); without ncclCommSplit
      // the scatter allreduce stays one unchunked call on the compute stream
      if (nccl().commSplit && !env_is_zero("STAMG_AR_OVERLAP")) {
        if (nccl().commSplit(c->comm, 0, c->rank, &c->comm_ar, nullptr) != 0) c->comm_ar = nullptr;
        if (c->comm_ar) ck(cudaStreamCreateWithFlags(&c->ar_stream, cudaStreamNonBlocking), "stream");
      }
    }
    const auto& s = c->pb.spec;
    // STAMG_SETUP_TRACE=1: wall time of the setup phases on stderr
    const bool trace = std::getenv("STAMG_SETUP_TRACE") != nullptr;
    auto tick = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!trace) return;
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[stamg setup] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tick).count());
      tick = now;
    };
    lap("cuda context, stream, comm");
    c->tree = make_sphere(s.angular_kind, s.angular_level, s.cone_levels, s.cone_half_angle_deg);
    lap("angular mesh");
    if (generic) {  // reference-shape path: 3D / p0 / Lin problems on one GPU
      if (c->world > 1) throw std::invalid_argument("the reference-shape path (3D, p0 or Lin) runs on one GPU");
      c->wl_allowed = false, c->graphs_off = true;
      c->outer.gt = gen::build_level(c->pb, c->tree, s.N, false);
      upload_gen_level(c.get(), c->outer);
      if (want_mg) {
        c->nr = s.nr < 0 ? s.N : s.nr;
        auto lv = gen::build_hierarchy(c->pb, c->tree, c->nr, s.n_levels);
        c->mg.resize(lv.size());
        for (size_t i = 0; i < lv.size(); ++i) {
          c->mg[i].gt = std::move(lv[i]);
          upload_gen_level(c.get(), c->mg[i]);
        }
        c->have_mg = true;
      }
      *out = c.release();
      return;
    }
    std::vector<std::vector<int>> parts;
    if (c->world > 1 && want_mg) {
      // sharded hierarchy: subtrees of the coarsest level per rank, coarsest replicated
      parts = partition_levels(c->tree, s.n_levels, c->rank, c->world);
      c->outer.t = build_level(c->pb, c->tree, s.N, false, &parts.back());
    } else {  // direction sharding: whole reflection orbits per rank (each rank folds its scatter)
      const auto sub = throughput_shard(c->tree, c->rank, c->world);
      c->outer.t = build_level(c->pb, c->tree, s.N, false, &sub);
    }
    c->outer.sharded = c->world > 1;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) c->nsum[i] += c->outer.t.Nmat[i * 4 + j];
    if (s.n_mat > 1) c->mat = dupload(c->pb.mat, c->stream);
    if (!c->pb.q_el.empty()) c->q_el = dupload(c->pb.q_el, c->stream);
    lap("outer tables (build_level)");
    upload_level(c.get(), c->outer);
    lap("outer upload (+ fold tables)");
    if (want_mg) {
      c->nr = s.nr < 0 ? s.N : s.nr;
      auto lv = build_hierarchy(c->pb, c->tree, c->nr, s.n_levels, c->world > 1 ? &parts : nullptr);
      lap("hierarchy tables");
      c->mg.resize(lv.size());
      for (size_t i = 0; i < lv.size(); ++i) {
        c->mg[i].t = std::move(lv[i]);
        c->mg[i].sharded = c->world > 1 && (i > 0 || lv.size() == 1);
        upload_level(c.get(), c->mg[i]);
      }
      if (c->world > 1 && c->mg.size() == 1)
        throw std::invalid_argument("a sharded hierarchy needs at least two levels (the coarsest is replicated)");
      c->have_mg = true;
      lap("hierarchy upload");
    }
    *out = c.release();
  });
}

int stamg_destroy(stamg_ctx* c) {
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    free_level(c->outer);
    for (auto& L : c->mg) free_level(L);
    for (double* v : c->V) cudaFree(v);
    for (void* p : {(void*)c->z, (void*)c->u, (void*)c->partial, (void*)c->dots, (void*)c->coef, (void*)c->mat,
                    (void*)c->q_el, (void*)c->hostio, (void*)c->foldbuf})
      if (p) cudaFree(p);
    if (c->hbuf) cudaFreeHost(c->hbuf);
    if (c->coll_host) cudaFreeHost(c->coll_host);
    for (double* p : c->pipe)
      if (p) cudaFree(p);
    for (cudaEvent_t e : c->pev)
      if (e) cudaEventDestroy(e);
    if (c->io_h2d) cudaStreamDestroy(c->io_h2d);
    if (c->io_d2h) cudaStreamDestroy(c->io_d2h);
    if (c->comm_ar) nccl().commDestroy(c->comm_ar);
    if (c->comm) nccl().commDestroy(c->comm);
    if (c->ar_stream) cudaStreamDestroy(c->ar_stream);
    for (cudaEvent_t e : c->ev_d2m) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_ar) cudaEventDestroy(e);
    for (auto& kv : c->mg_graphs) cudaGraphExecDestroy(kv.second.exec);
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

int stamg_layout(stamg_ctx* c, int level, int out4[4]) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    out4[0] = L.t.n_el, out4[1] = L.t.P, out4[2] = L.g ? L.g->S : 4, out4[3] = L.g ? L.g->D : 1;
  });
}
int stamg_patch_range(stamg_ctx* c, int level, int* q0, int* q1) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    *q0 = L.t.P ? L.t.qpos.front() : 0, *q1 = L.t.P ? L.t.qpos.back() + 1 : 0;
  });
}
// Host-only (no device): the direction partition a rank would get, for tests.
// level 0 = coarsest MG level (replicated); up[] = parent position in the
// coarser level's list held by the same rank (level 0: the full list).
int stamg_partition(const stamg_problem* prob, int rank, int world, int level, int* qpos, int* up, int cap,
                    int* n) {
  return guard([&] {
    Problem pb = copy_problem(*prob);
    validate(pb);
    const auto& s = pb.spec;
    SphereTree tree = make_sphere(s.angular_kind, s.angular_level, s.cone_levels, s.cone_half_angle_deg);
    auto parts = partition_levels(tree, s.n_levels, rank, world);
    if (level < 0 || level >= int(parts.size())) throw std::invalid_argument("partition: level out of range");
    const int Lmax = tree.max_level, nlev = int(parts.size()), lmin = Lmax + 1 - nlev;
    auto tree_at = [&](int i) { return lmin + i == Lmax ? tree : coarsen(tree, lmin + i); };
    const SphereTree ft = tree_at(level);
    *n = int(parts[level].size());
    for (int k = 0; k < *n && k < cap; ++k) qpos[k] = parts[level][k];
    if (level >= 1 && up) {
      const SphereTree ct = tree_at(level - 1);
      std::unordered_map<int, int> pos;
      for (size_t c = 0; c < parts[level - 1].size(); ++c) pos[ct.leaves[parts[level - 1][c]]] = int(c);
      for (int k = 0; k < *n && k < cap; ++k) {
        const int id = ft.leaves[parts[level][k]];
        auto it = pos.find(id);
        if (it == pos.end()) it = pos.find(ft.parent[id]);
        up[k] = it == pos.end() ? -1 : it->second;
      }
    }
  });
}

int stamg_shard_patches(const stamg_problem* prob, int rank, int world, int* out, int cap, int* n) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard: bad rank / world");
    Problem pb = copy_problem(*prob);
    validate(pb);
    const auto& s = pb.spec;
    SphereTree tree = make_sphere(s.angular_kind, s.angular_level, s.cone_levels, s.cone_half_angle_deg);
    const auto sub = throughput_shard(tree, rank, world);
    *n = int(sub.size());
    for (int k = 0; k < *n && k < cap; ++k) out[k] = sub[k];
  });
}

int stamg_patch_list(stamg_ctx* c, int level, int* out, int cap, int* n) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    *n = L.t.P;
    for (int q = 0; out && q < L.t.P && q < cap; ++q) out[q] = L.t.qpos[q];
  });
}
int stamg_n_levels(stamg_ctx* c, int* n, int* nr) {
  return guard_ctx(c, [&] {
    *n = int(c->mg.size());
    *nr = c->nr;
  });
}
int stamg_level_order(stamg_ctx* c, int level, int* order) {
  return guard_ctx(c, [&] { *order = level_of(c, level).t.order; });
}

int stamg_vec_create(stamg_ctx* c, int level, stamg_vec** out) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    auto v = std::make_unique<stamg_vec>();
    v->ctx = c, v->level = level, v->n = L.n, v->d = dalloc<double>(L.n);
    ck(cudaMemsetAsync(v->d, 0, L.n * sizeof(double), c->stream), "memset");
    *out = v.release();
  });
}
int stamg_vec_free(stamg_vec* v) {
  return guard([&] {
    if (!v) return;
    cudaSetDevice(v->ctx->device);
    cudaStreamSynchronize(v->ctx->stream);
    cudaFree(v->d);
    delete v;
  });
}
int stamg_vec_size(stamg_vec* v, int64_t* n) {
  // host-visible length in the reference layout (device storage may be padded)
  return guard_ctx(v ? v->ctx : nullptr, [&] { *n = ref_size(level_of(v->ctx, v->level)); });
}
int stamg_vec_device_ptr(stamg_vec* v, double** p) {
  return guard_ctx(v ? v->ctx : nullptr, [&] { *p = v->d; });
}
int stamg_vec_upload(stamg_ctx* c, stamg_vec* v, const double* host, int64_t n) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, v->level);
    if (n != ref_size(L)) throw std::invalid_argument("vec_upload: layout mismatch");
    host_to_vec(c, L, host, v->d, false);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}
int stamg_vec_download(stamg_ctx* c, const stamg_vec* v, double* host, int64_t n) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, v->level);
    if (n != ref_size(L)) throw std::invalid_argument("vec_download: layout mismatch");
    vec_to_host(c, L, v->d, host, false);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}
int stamg_vec_fill(stamg_ctx* c, stamg_vec* v, double value) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, v->level);
    if (L.wl.nd && value != 0.0) launch_wl_fill(v->d, value, L.t.n_el, L.t.P, L.wl, c->stream);
    else launch_fill(v->d, value, v->n, c->stream);
    ck_launch("fill");
  });
}
int stamg_vec_copy(stamg_ctx* c, const stamg_vec* a, stamg_vec* b) {
  return guard_ctx(c, [&] {
    if (a->n != b->n) throw std::invalid_argument("vec_copy: layout mismatch");
    ck(cudaMemcpyAsync(b->d, a->d, a->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
  });
}
int stamg_vec_axpy(stamg_ctx* c, double a, const stamg_vec* x, stamg_vec* y) {
  return guard_ctx(c, [&] {
    if (x->n != y->n) throw std::invalid_argument("vec_axpy: layout mismatch");
    launch_axpy(a, x->d, y->d, x->n, c->stream);
    ck_launch("axpy");
  });
}
int stamg_vec_dot(stamg_ctx* c, const stamg_vec* x, const stamg_vec* y, double* out) {
  return guard_ctx(c, [&] {
    if (x->n != y->n) throw std::invalid_argument("vec_dot: layout mismatch");
    const DevLevel& L = level_of(c, x->level);
    *out = op_dot(c, x->d, y->d, x->n, L.sharded);
  });
}

int stamg_apply_L(stamg_ctx* c, int level, const stamg_vec* phi, stamg_vec* y) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    need(phi, L, "apply_L"), need(y, L, "apply_L");
    if (phi->d == y->d) throw std::invalid_argument("apply_L: y must not alias phi");
    op_apply_L(c, L, phi->d, y->d);
  });
}
int stamg_apply_scatter(stamg_ctx* c, int level, const stamg_vec* phi, int order, double scale, stamg_vec* y) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    need(phi, L, "apply_scatter"), need(y, L, "apply_scatter");
    op_scatter(c, L, phi->d, order, scale, y->d);
  });
}
int stamg_apply_A(stamg_ctx* c, int level, const stamg_vec* phi, int order, stamg_vec* y) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    need(phi, L, "apply_A"), need(y, L, "apply_A");
    if (phi->d == y->d) throw std::invalid_argument("apply_A: y must not alias phi");
    op_apply_A(c, L, phi->d, order, y->d);
  });
}
int stamg_sweep(stamg_ctx* c, int level, const stamg_vec* rhs, stamg_vec* z) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    need(rhs, L, "standard_sweep"), need(z, L, "standard_sweep");
    op_sweep(c, L, rhs->d, z->d);
  });
}
int stamg_coarse_gs(stamg_ctx* c, int level, const stamg_vec* rhs, int nu, stamg_vec* phi) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    need(rhs, L, "coarse_scatter_sweep"), need(phi, L, "coarse_scatter_sweep");
    op_coarse_gs(c, L, rhs->d, nu, phi->d);
  });
}
int stamg_smoother_step(stamg_ctx* c, int level, const stamg_vec* f, int order, stamg_vec* phi) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    need(f, L, "smoother_step"), need(phi, L, "smoother_step");
    op_smoother(c, L, f->d, order, phi->d);
  });
}
int stamg_prolongate(stamg_ctx* c, int l, const stamg_vec* coarse, stamg_vec* fine) {
  return guard_ctx(c, [&] {
    if (!c->have_mg || l < 1 || l >= int(c->mg.size())) throw std::invalid_argument("prolongate: level out of range");
    need(coarse, c->mg[l - 1], "prolongate"), need(fine, c->mg[l], "prolongate");
    op_prolong(c, l, coarse->d, fine->d, false);
  });
}
int stamg_restrict(stamg_ctx* c, int l, const stamg_vec* fine, stamg_vec* coarse) {
  return guard_ctx(c, [&] {
    if (!c->have_mg || l < 1 || l >= int(c->mg.size())) throw std::invalid_argument("restrict_residual: level out of range");
    need(fine, c->mg[l], "restrict_residual"), need(coarse, c->mg[l - 1], "restrict_residual");
    op_restrict(c, l, fine->d, coarse->d);
  });
}
int stamg_vcycle(stamg_ctx* c, int l, const stamg_vec* f, stamg_vec* phi) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, l);
    need(f, L, "lmg_vcycle"), need(phi, L, "lmg_vcycle");
    op_vcycle(c, l, f->d, phi->d);
  });
}
int stamg_mg_apply(stamg_ctx* c, const stamg_vec* r, stamg_vec* z) {
  return guard_ctx(c, [&] {
    if (!c->have_mg) throw std::invalid_argument("multigrid hierarchy was not built for this context");
    need(r, c->mg.back(), "mg_apply"), need(z, c->mg.back(), "mg_apply");
    if (r->d == z->d) throw std::invalid_argument("mg_apply: z must not alias r");
    op_mg_apply_graph(c, r->d, z->d);
  });
}
int stamg_rhs(stamg_ctx* c, stamg_vec* f) {
  return guard_ctx(c, [&] {
    need(f, c->outer, "assemble_rhs");
    if (c->outer.g) {
      const auto v = gen::assemble_rhs(c->pb, c->outer.gt, c->tree);
      host_to_vec(c, c->outer, v.data(), f->d, true);
      ck(cudaStreamSynchronize(c->stream), "sync");
      return;
    }
    const auto v = assemble_rhs(c->pb, c->outer.t, c->tree);  // tables' (internal) patch order
    host_to_vec(c, c->outer, v.data(), f->d, true);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int stamg_solve(stamg_ctx* c, int method, int precond, const stamg_vec* b, stamg_vec* x, double tol, int max_iter,
                int restart, stamg_report* rep, double* history, int cap) {
  return guard_ctx(c, [&] {
    need(b, c->outer, "solve"), need(x, c->outer, "solve");
    if (precond == 1 && !c->have_mg) throw std::invalid_argument("multigrid hierarchy was not built for this context");
    if (precond < 0 || precond > 2) throw std::invalid_argument("solve: unknown preconditioner");
    std::vector<double> hist;
    stamg_report r = method == 0 ? op_bicgstab(c, precond, b->d, x->d, tol, max_iter, hist)
                                 : op_gmres(c, precond, b->d, x->d, tol, max_iter, restart, hist);
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (rep) *rep = r;
    for (int i = 0; history && i < cap && i < int(hist.size()); ++i) history[i] = hist[i];
  });
}

// Host-buffer sweep pipelined over chunks of 8-direction groups (the sweep is
// independent per direction, sweeps.cpp:28): chunk k's host->device copy, chunk
// k-1's sweep and chunk k-2's device->host copy run at once on three streams, so
// both PCIe directions stream concurrently. A chunk's directions are a contiguous
// run of reference patch columns, moved by one strided 2D copy ([n_el] rows of
// w*32 bytes at a host pitch of P*32) into a [n_el][w][4] staging buffer that the
// sweep reads and writes in place. Returns false (caller falls back to the
// serial path) when the level has no 8-direction groups or a chunk's patches are
// not a contiguous reference range.
static bool sweep_host_pipelined(stamg_ctx* c, DevLevel& L, const double* rhs, double* z) {
  if (!L.sweep_top || env_is_zero("STAMG_E2E_PIPELINE")) return false;
  const LevelTables& t = L.t;
  const int ng = int(t.group8_oct.size());
  // reference column of internal patch k (wavefront contexts reorder the tables)
  std::vector<int> ref_of(t.P, -1);
  if (L.wl.nd) {
    for (int q = 0; q < t.P; ++q) ref_of[L.ipos[q]] = q;
  }
  auto col = [&](int k) { return L.wl.nd ? ref_of[k] : k; };
  int chunk_dirs = 512;
  if (const char* e = std::getenv("STAMG_E2E_CHUNK_DIRS")) chunk_dirs = std::max(8, std::atoi(e));
  const int cg = std::max(1, std::min(chunk_dirs / 8, (ng + 3) / 4));  // >= 4 chunks when possible
  const int nch = (ng + cg - 1) / cg;
  std::vector<int> k0(nch), q0(nch), w(nch);
  for (int ch = 0; ch < nch; ++ch) {
    const int g0 = ch * cg, g1 = std::min(ng, g0 + cg);
    k0[ch] = t.groups8[size_t(g0) * 8], w[ch] = (g1 - g0) * 8;
    if (k0[ch] < 0) return false;
    q0[ch] = col(k0[ch]);
    for (int j = 0; j < w[ch]; ++j) {
      const int k = t.groups8[size_t(g0) * 8 + j];
      if (k != k0[ch] + j || col(k) != q0[ch] + j) return false;
    }
  }
  const int64_t per = int64_t(t.n_el) * cg * 8 * 4;
  if (c->pipe_n < per) {
    for (double*& p : c->pipe) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    for (double*& p : c->pipe) p = dalloc<double>(per);
    c->pipe_n = per;
  }
  if (!c->io_h2d) {
    ck(cudaStreamCreateWithFlags(&c->io_h2d, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&c->io_d2h, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t& e : c->pev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  cudaEvent_t* ev_h2d = c->pev;      // [3]
  cudaEvent_t* ev_sw = c->pev + 3;   // [3]
  cudaEvent_t* ev_d2h = c->pev + 6;  // [3]
  cudaEvent_t ev_go = c->pev[9];
  ck(cudaEventRecord(ev_go, c->stream), "event");  // after earlier work on the context stream
  ck(cudaStreamWaitEvent(c->io_h2d, ev_go, 0), "wait");
  const size_t hpitch = size_t(t.P) * 32;
  for (int ch = 0; ch < nch; ++ch) {
    const int b = ch % 3;
    double* buf = c->pipe[b];
    const size_t wb = size_t(w[ch]) * 32;
    if (ch >= 3) ck(cudaStreamWaitEvent(c->io_h2d, ev_d2h[b], 0), "wait");
    ck(cudaMemcpy2DAsync(buf, wb, rhs + size_t(q0[ch]) * 4, hpitch, wb, t.n_el, cudaMemcpyHostToDevice, c->io_h2d),
       "h2d");
    ck(cudaEventRecord(ev_h2d[b], c->io_h2d), "event");
    ck(cudaStreamWaitEvent(c->stream, ev_h2d[b], 0), "wait");
    {
      Timed tm(c, "sweep");
      SweepParams p;
      p.g = geom(c, L);
      p.dirs = 8, p.top = L.sweep_top;  // reference layout in the staging buffer (wl.nd = 0)
      p.g.groups = L.groups8, p.g.group_oct = L.group8_oct, p.g.n_groups = w[ch] / 8;
      p.grp0 = ch * cg, p.data_P = w[ch], p.data_q0 = k0[ch];
      p.rhs = buf, p.z = buf, p.Binv = L.Binv, p.cxy = L.cxy;
      launch_sweep(p, c->stream);
      ck_launch("sweep");
      c->launches += 1;
    }
    ck(cudaEventRecord(ev_sw[b], c->stream), "event");
    ck(cudaStreamWaitEvent(c->io_d2h, ev_sw[b], 0), "wait");
    ck(cudaMemcpy2DAsync(z + size_t(q0[ch]) * 4, hpitch, buf, wb, wb, t.n_el, cudaMemcpyDeviceToHost, c->io_d2h),
       "d2h");
    ck(cudaEventRecord(ev_d2h[b], c->io_d2h), "event");
  }
  ck(cudaEventRecord(ev_go, c->io_d2h), "event");
  ck(cudaStreamWaitEvent(c->stream, ev_go, 0), "wait");
  ck(cudaStreamSynchronize(c->stream), "sync");
  c->last_host_chunks = nch;
  return true;
}

int stamg_sweep_host(stamg_ctx* c, int level, const double* rhs, double* z, int64_t n) {
  return guard_ctx(c, [&] {
    DevLevel& L = level_of(c, level);
    if (n != ref_size(L)) throw std::invalid_argument("standard_sweep: layout mismatch");
    if (sweep_host_pipelined(c, L, rhs, z)) return;
    c->last_host_chunks = 0;
    if (c->hostio_n < L.n) {
      if (c->hostio) cudaFree(c->hostio);
      c->hostio = dalloc<double>(L.n);
      c->hostio_n = L.n;
      ck(cudaMemsetAsync(c->hostio, 0, L.n * sizeof(double), c->stream), "memset");
    }
    host_to_vec(c, L, rhs, c->hostio, false);
    op_sweep(c, L, c->hostio, c->hostio);
    vec_to_host(c, L, c->hostio, z, false);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int stamg_solve_host(stamg_ctx* c, int method, int precond, const double* bh, double* xh, int64_t n, double tol,
                     int max_iter, int restart, stamg_report* rep) {
  return guard_ctx(c, [&] {
    if (n != ref_size(c->outer)) throw std::invalid_argument("solve: layout mismatch");
    double* b = dalloc<double>(c->outer.n);
    double* x = dalloc<double>(c->outer.n);
    ck(cudaMemsetAsync(b, 0, c->outer.n * sizeof(double), c->stream), "memset");
    ck(cudaMemsetAsync(x, 0, c->outer.n * sizeof(double), c->stream), "memset");
    try {
      host_to_vec(c, c->outer, bh, b, false);
      std::vector<double> hist;
      stamg_report r = method == 0 ? op_bicgstab(c, precond, b, x, tol, max_iter, hist)
                                   : op_gmres(c, precond, b, x, tol, max_iter, restart, hist);
      vec_to_host(c, c->outer, x, xh, false);
      ck(cudaStreamSynchronize(c->stream), "sync");
      if (rep) *rep = r;
    } catch (...) {
      cudaFree(b), cudaFree(x);
      throw;
    }
    cudaFree(b), cudaFree(x);
  });
}

int stamg_scalar_flux(stamg_ctx* c, const stamg_vec* phi, double* out) {
  return guard_ctx(c, [&] {
    need(phi, c->outer, "scalar_flux");
    std::vector<double> h(ref_size(c->outer));
    vec_to_host(c, c->outer, phi->d, h.data(), true);  // tables' (internal) patch order
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (c->outer.g) {  // harness.cpp:183-205: sum_q (M_q 1)_d phi_{el,q,d,i} (N 1)_i / volume
      const gen::Tables& gt = c->outer.gt;
      const auto& sp = c->pb.spec;
      const double vol = (sp.box / sp.nx) * (sp.box / sp.ny) * (sp.dim == 3 ? sp.box / sp.nz : 1.0);
      std::vector<double> nsum(gt.S, 0.0);
      for (int i = 0; i < gt.S; ++i)
        for (int j = 0; j < gt.S; ++j) nsum[i] += gt.Nmat[i * gt.S + j];
      for (int el = 0; el < gt.n_el; ++el) {
        double integral = 0;
        for (int q = 0; q < gt.P; ++q)
          for (int d = 0; d < gt.D; ++d) {
            const double* blk = &h[(size_t(el) * gt.P + q) * gt.bs + d * gt.S];
            double a = 0;
            for (int i = 0; i < gt.S; ++i) a += blk[i] * nsum[i];
            integral += gt.M1[size_t(q) * gt.D + d] * a;
          }
        out[el] = integral / vol;
      }
      return;
    }
    const auto& t = c->outer.t;
    const double vol = c->pb.h * c->pb.h;
    for (int el = 0; el < t.n_el; ++el) {
      double integral = 0;
      for (int q = 0; q < t.P; ++q) {
        const double* blk = &h[(size_t(el) * t.P + q) * 4];
        integral += t.area[q] * (blk[0] * c->nsum[0] + blk[1] * c->nsum[1] + blk[2] * c->nsum[2] + blk[3] * c->nsum[3]);
      }
      out[el] = integral / vol;
    }
    if (c->world > 1 && c->outer.sharded) {  // partial sums over this rank's directions
      double* d = dalloc<double>(t.n_el);
      ck(cudaMemcpyAsync(d, out, t.n_el * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
      op_allreduce(c, d, t.n_el);
      ck(cudaMemcpyAsync(out, d, t.n_el * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
      ck(cudaStreamSynchronize(c->stream), "sync");
      cudaFree(d);
    }
  });
}

// One source iteration on the outer level with moment-only scatter storage:
// psi = q_ext + S(phi) from the stored moments (M2D), sweep in place, moments
// of the new psi (D2M, allreduced over ranks). psi holds the angular flux on
// entry and exit; the moments live in the level's src buffer.
int stamg_source_iteration(stamg_ctx* c, stamg_vec* psi, int n_iter) {
  return guard_ctx(c, [&] {
    DevLevel& O = c->outer;
    need(psi, O, "source_iteration");
    if (O.g) throw std::invalid_argument("source_iteration is a throughput entry point of the 2D bilinear Const path");
    const int order = c->pb.spec.N;
    for (int it = 0; it < n_iter; ++it) {
      scatter_into(c, O, psi->d, order, 1.0, 0.0, psi->d, c->q_el);  // psi = q + S psi
      op_sweep(c, O, psi->d, psi->d);
    }
  });
}

int stamg_get_table(stamg_ctx* c, int level, const char* name, double* out, int64_t cap, int64_t* n) {
  return guard_ctx(c, [&] {
    const DevLevel& L = level_of(c, level);
    const LevelTables& t = L.t;
    std::vector<double> v;
    const std::string nm(name);
    if (L.g && (nm == "X" || nm == "B" || nm == "Binv" || nm == "C" || nm == "M1" || nm == "upB")) {
      const gen::Tables& gt = L.gt;
      v = nm == "X" ? gt.X : nm == "B" ? gt.Bd : nm == "Binv" ? gt.Binv : nm == "C" ? gt.C : nm == "M1" ? gt.M1 : gt.upB;
      *n = int64_t(v.size());
      for (int64_t i = 0; out && i < cap && i < *n; ++i) out[i] = v[i];
      return;
    }
    if (nm == "fold") v = {double(L.fold_G), double(L.fold_R), double(L.fold_Hf), t.sym_defect, double(t.n_sym_axes)};
    else if (nm == "ar_chunks") v = {double(c->ar_chunks_used), double(c->comm_ar != nullptr)};
    else if (nm == "graphs") v = {double(c->mg_graphs.size()), double(c->graph_replays), double(c->graphs_off)};
    else if (nm == "sweep_mode")
      v = {double(L.sweep_xb), double(L.sweep_xb_g0), double(t.group8_oct.size()), double(L.wl.nd)};
    else if (nm == "gs_mode")
      v = {double(L.gs_mw), double(L.gs_cluster), double(L.gs_rows), double(L.gs_mb_slots), double(L.gs_mb_credit), double(L.gs_blk)};
    else if (nm == "X") v = t.X;
    else if (nm == "B") v = t.B;
    else if (nm == "Binv") v = t.Binv;
    else if (nm == "C") v = t.C;
    else if (nm == "area") v = t.area;
    else if (nm == "Aflow") v = t.Aflow;
    else if (nm == "sig") v = t.sig;
    else if (nm == "octant") v.assign(t.octant.begin(), t.octant.end());
    else if (nm == "leaf_id") v.assign(t.leaf_id.begin(), t.leaf_id.end());
    else if (nm == "up") v.assign(t.up.begin(), t.up.end());
    else if (nm == "sq") v = t.sq;
    else if (nm == "rhs") v = assemble_rhs(c->pb, t, c->tree);
    else throw std::invalid_argument("unknown table " + nm);
    *n = int64_t(v.size());
    if (out) std::memcpy(out, v.data(), std::min<int64_t>(cap, *n) * sizeof(double));
  });
}

// Host only (no device): outer-level tables as the host setup builds them.
int stamg_host_table(const stamg_problem* prob, const char* name, double* out, int64_t cap, int64_t* n) {
  return guard([&] {
    if (!prob || !name || !n) throw std::invalid_argument("stamg_host_table: null argument");
    Problem pb = copy_problem(*prob);
    const bool generic = gen::handles(*prob);
    if (generic) gen::validate(pb);
    else validate(pb);
    const auto& s = pb.spec;
    const SphereTree tree = make_sphere(s.angular_kind, s.angular_level, s.cone_levels, s.cone_half_angle_deg);
    const std::string nm(name);
    std::vector<double> v;
    if (generic) {
      const gen::Tables t = gen::build_level(pb, tree, s.N, false);
      if (nm == "X") v = t.X;
      else if (nm == "B") v = t.Bd;
      else if (nm == "C") v = t.C;
      else if (nm == "M1") v = t.M1;
      else if (nm == "rhs") v = gen::assemble_rhs(pb, t, tree);
      else if (nm == "octant") v.assign(t.octant.begin(), t.octant.end());
      else if (nm == "layout") v = {double(t.n_el), double(t.P), double(t.S), double(t.D)};
      else throw std::invalid_argument("unknown table");
    } else {
      const LevelTables t = build_level(pb, tree, s.N, false);
      if (nm == "X") v = t.X;
      else if (nm == "B") v = t.B;
      else if (nm == "C") v = t.C;
      else if (nm == "M1") v = t.area;
      else if (nm == "rhs") v = assemble_rhs(pb, t, tree);
      else if (nm == "octant") v.assign(t.octant.begin(), t.octant.end());
      else if (nm == "layout") v = {double(t.n_el), double(t.P), 4.0, 1.0};
      else throw std::invalid_argument("unknown table");
    }
    *n = int64_t(v.size());
    for (int64_t i = 0; out && i < cap && i < *n; ++i) out[i] = v[i];
  });
}

int stamg_synchronize(stamg_ctx* c) {
  return guard_ctx(c, [&] { ck(cudaStreamSynchronize(c->stream), "sync"); });
}
int stamg_host_pipeline_chunks(stamg_ctx* c, int* n) {
  return guard_ctx(c, [&] { *n = c->last_host_chunks; });
}
int stamg_launch_count(stamg_ctx* c, int64_t* n) {
  return guard_ctx(c, [&] { *n = c->launches; });
}
int stamg_timing_enable(stamg_ctx* c, int on) {
  return guard_ctx(c, [&] {
    if (!on) resolve_timing(c);
    c->timing = on != 0;
    if (on) c->timed.clear();
  });
}
int stamg_timing_read(stamg_ctx* c, const char* kernel, double* ms, int64_t* launches) {
  return guard_ctx(c, [&] {
    resolve_timing(c);
    auto it = c->timed.find(kernel);
    *ms = it == c->timed.end() ? 0.0 : it->second.first;
    *launches = it == c->timed.end() ? 0 : it->second.second;
  });
}

// FP64 throughput probes (roofline denominators, measured on the box)
int stamg_bench_fp64_peaks(stamg_ctx* c, double* dmma_tflops, double* dfma_tflops) {
  return guard_ctx(c, [&] {
    *dmma_tflops = bench_dmma_tflops(c->device, c->stream);
    *dfma_tflops = bench_dfma_tflops(c->device, c->stream);
  });
}

// access-pattern probe: GB/s of an in-place 128-byte-chunk read+write over a vector
int stamg_bench_chunk_rw(stamg_ctx* c, stamg_vec* v, int64_t stride_chunks, int mode, double* gbs) {
  return guard_ctx(c, [&] { *gbs = bench_chunk_rw_gbs(v->d, v->n, stride_chunks, mode, c->stream); });
}

// pinned host memory for the host-buffer entry points
int stamg_host_alloc(int64_t bytes, void** out) {
  return guard([&] { ck(cudaMallocHost(out, bytes), "cudaMallocHost"); });
}
int stamg_host_free(void* p) {
  return guard([&] { ck(cudaFreeHost(p), "cudaFreeHost"); });
}

}  // extern "C"
