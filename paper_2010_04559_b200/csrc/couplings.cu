// Device-side build_couplings (scatter.cpp:74-99): X_q(h) = sum over the
// patch's Duffy-collapsed Gauss nodes (quadrature.cpp:59-92) of w * Y_h(Omega),
// real orthonormal harmonics by the associated-Legendre recurrence along each
// order m (scatter.cpp:33-65). This is ~1e9 harmonic evaluations at config 5
// (8192 patches x 144 nodes x 1089 harmonics): 6.3 s on one host core, a few
// milliseconds here.
//
// One thread per (patch, m): it walks the patch's nodes in the host order and
// runs the recurrence n = m..N for each, accumulating the cos / sin columns
// (h = n^2 + n +- m) in registers (NMAX+1 of each, fully unrolled). The node
// order, the recurrence and the per-node products are the host's, so the table
// matches the host loop to rounding of cos/sin (the test compares at 1e-13).
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "setup.hpp"

namespace stamg_b200 {
namespace {

struct CouplingArgs {
  const double* verts;  // [P][9] lattice vertices scaled to the unit octahedron
  const int* nq;        // [P] 1D Gauss order of the patch's rule
  const double* gx;     // rules for orders 1..kMaxRule concatenated: order n at n(n-1)/2
  const double* gw;
  double* X;            // [P][H] row-major (the host table)
  int P, N, H;
};

constexpr int kMaxRule = 32;
constexpr double kInvSqrt4Pi = 0.28209479177387814;  // 1/sqrt(4 pi)
constexpr double kSqrt2 = 1.4142135623730951;

template <int NMAX>
__global__ void __launch_bounds__(128) couplings_kernel(CouplingArgs a) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int M = a.N + 1;
  if (idx >= a.P * M) return;
  const int q = idx / M, m = idx - q * M;
  const double* v = a.verts + size_t(q) * 9;
  const double A0 = v[0], A1 = v[1], A2 = v[2], B0 = v[3], B1 = v[4], B2 = v[5], C0 = v[6], C1 = v[7], C2 = v[8];
  const double e10 = B0 - A0, e11 = B1 - A1, e12 = B2 - A2, e20 = C0 - A0, e21 = C1 - A1, e22 = C2 - A2;
  const double cr0 = e11 * e22 - e12 * e21, cr1 = e12 * e20 - e10 * e22, cr2 = e10 * e21 - e11 * e20;
  const double two_area = sqrt(cr0 * cr0 + cr1 * cr1 + cr2 * cr2);
  const double hplane = (A0 * cr0 + A1 * cr1 + A2 * cr2) / two_area;
  const int n1 = a.nq[q];
  const double* gx = a.gx + n1 * (n1 - 1) / 2;
  const double* gw = a.gw + n1 * (n1 - 1) / 2;

  double acc_c[NMAX + 1], acc_s[NMAX + 1];
#pragma unroll
  for (int n = 0; n <= NMAX; ++n) acc_c[n] = acc_s[n] = 0.0;

  for (int iu = 0; iu < n1; ++iu) {
    const double u = gx[iu];
    for (int iv = 0; iv < n1; ++iv) {
      const double vv = gx[iv];
      const double x0 = (1.0 - u) * A0 + u * ((1.0 - vv) * B0 + vv * C0);
      const double x1 = (1.0 - u) * A1 + u * ((1.0 - vv) * B1 + vv * C1);
      const double x2 = (1.0 - u) * A2 + u * ((1.0 - vv) * B2 + vv * C2);
      const double rr = sqrt(x0 * x0 + x1 * x1 + x2 * x2);
      const double w = gw[iu] * gw[iv] * u * two_area * hplane / (rr * rr * rr);
      const double ox = x0 / rr, oy = x1 / rr, z = x2 / rr;
      const double rxy = hypot(ox, oy);
      const double phi = atan2(oy, ox);
      double pmm = kInvSqrt4Pi;
      for (int k = 0; k < m; ++k) pmm *= -sqrt((2.0 * k + 3.0) / (2.0 * k + 2.0)) * rxy;
      double sm = 0.0, cm = 1.0;
      if (m > 0) {
        sincos(m * phi, &sm, &cm);
        cm *= kSqrt2, sm *= kSqrt2;
      }
      double prev = 0.0, cur = pmm;
#pragma unroll
      for (int n = 0; n <= NMAX; ++n) {
        if (n >= m && n <= a.N) {
          acc_c[n] += w * (cm * cur);
          acc_s[n] += w * (sm * cur);
          if (n < a.N) {
            const double nn = n + 1;
            const double ca = sqrt((4.0 * nn * nn - 1.0) / (nn * nn - double(m) * m));
            const double cb = sqrt(((nn - 1) * (nn - 1) - double(m) * m) / (4.0 * (nn - 1) * (nn - 1) - 1.0));
            const double next = ca * (z * cur - cb * prev);
            prev = cur, cur = next;
          }
        }
      }
    }
  }
  double* Xq = a.X + size_t(q) * a.H;
#pragma unroll
  for (int n = 0; n <= NMAX; ++n) {
    if (n >= m && n <= a.N) {
      Xq[n * n + n + m] = acc_c[n];
      if (m > 0) Xq[n * n + n - m] = acc_s[n];
    }
  }
}

// Device-side build_operators (transport.cpp:43-57 with build_patch_operators,
// angular_disc.cpp:40-59): one thread per patch integrates M = sum w and A^xi = sum w Omega_xi
// over the patch rule (the host's node order), then forms, per material, the fused blocks
// B_q = sigma_t M N - sum A^xi V^xi + s_xi A^xi F_self[out], its inverse (partial-pivot
// Gauss-Jordan, as the host's inverse4), the inflow blocks C_{q,xi} = -s_xi A^xi F_neigh[in]
// and their non-zero 2 x 2 sub-blocks.
struct ElementMats {
  double N[16], V[2][16], Fs[4][16], Fn[4][16];
};
struct BlockArgs {
  const double* verts;  // [P][9]
  const int* nq;        // [P] 1D Gauss order of the patch-operator rule
  const int* octant;    // [P]
  const double* gx;
  const double* gw;
  const double* sigma_t;  // [n_mat]
  double *area, *Aflow, *B, *Binv, *C, *cxy;
  int* singular;
  int P, n_mat;
};

__device__ bool inverse4_dev(const double* A, double* Ainv) {
  double m[4][8];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 8; ++j) m[i][j] = j < 4 ? A[i * 4 + j] : (j - 4 == i ? 1.0 : 0.0);
  for (int k = 0; k < 4; ++k) {
    int p = k;
    for (int i = k + 1; i < 4; ++i)
      if (fabs(m[i][k]) > fabs(m[p][k])) p = i;
    if (m[p][k] == 0.0) return false;
    if (p != k)
      for (int j = 0; j < 8; ++j) {
        const double u = m[k][j];
        m[k][j] = m[p][j], m[p][j] = u;
      }
    const double d = 1.0 / m[k][k];
    for (int j = 0; j < 8; ++j) m[k][j] *= d;
    for (int i = 0; i < 4; ++i)
      if (i != k) {
        const double f = m[i][k];
        for (int j = 0; j < 8; ++j) m[i][j] -= f * m[k][j];
      }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) Ainv[i * 4 + j] = m[i][4 + j];
  return true;
}

__global__ void __launch_bounds__(128) patch_blocks_kernel(BlockArgs a, ElementMats em) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.P) return;
  const double* v = a.verts + size_t(q) * 9;
  const double A0 = v[0], A1 = v[1], A2 = v[2], B0 = v[3], B1 = v[4], B2 = v[5], C0 = v[6], C1 = v[7], C2 = v[8];
  const double e10 = B0 - A0, e11 = B1 - A1, e12 = B2 - A2, e20 = C0 - A0, e21 = C1 - A1, e22 = C2 - A2;
  const double cr0 = e11 * e22 - e12 * e21, cr1 = e12 * e20 - e10 * e22, cr2 = e10 * e21 - e11 * e20;
  const double two_area = sqrt(cr0 * cr0 + cr1 * cr1 + cr2 * cr2);
  const double hplane = (A0 * cr0 + A1 * cr1 + A2 * cr2) / two_area;
  const int n1 = a.nq[q];
  const double* gx = a.gx + n1 * (n1 - 1) / 2;
  const double* gw = a.gw + n1 * (n1 - 1) / 2;
  double M = 0.0, Ax[3] = {0.0, 0.0, 0.0};
  for (int iu = 0; iu < n1; ++iu) {
    const double u = gx[iu];
    for (int iv = 0; iv < n1; ++iv) {
      const double vv = gx[iv];
      const double x0 = (1.0 - u) * A0 + u * ((1.0 - vv) * B0 + vv * C0);
      const double x1 = (1.0 - u) * A1 + u * ((1.0 - vv) * B1 + vv * C1);
      const double x2 = (1.0 - u) * A2 + u * ((1.0 - vv) * B2 + vv * C2);
      const double rr = sqrt(x0 * x0 + x1 * x1 + x2 * x2);
      const double w = gw[iu] * gw[iv] * u * two_area * hplane / (rr * rr * rr);
      M += w;
      Ax[0] += (x0 / rr) * w, Ax[1] += (x1 / rr) * w, Ax[2] += (x2 / rr) * w;
    }
  }
  a.area[q] = M;
  for (int xi = 0; xi < 3; ++xi) a.Aflow[q * 3 + xi] = Ax[xi];
  const int oct = a.octant[q];
  double sgn[2], Cq[2][16];
  int fout[2];
  for (int xi = 0; xi < 2; ++xi) {
    sgn[xi] = (oct >> xi) & 1 ? -1.0 : 1.0;
    fout[xi] = 2 * xi + (sgn[xi] > 0 ? 1 : 0);
    const int fin = 2 * xi + (sgn[xi] > 0 ? 0 : 1);
    for (int k = 0; k < 16; ++k) Cq[xi][k] = -sgn[xi] * (Ax[xi] * em.Fn[fin][k]);
  }
  for (int m = 0; m < a.n_mat; ++m) {
    double Bq[16];
    for (int k = 0; k < 16; ++k) Bq[k] = a.sigma_t[m] * (M * em.N[k]);
    for (int xi = 0; xi < 2; ++xi)
      for (int k = 0; k < 16; ++k) {
        Bq[k] += -1.0 * (Ax[xi] * em.V[xi][k]);
        Bq[k] += sgn[xi] * (Ax[xi] * em.Fs[fout[xi]][k]);
      }
    double* Bo = a.B + (size_t(m) * a.P + q) * 16;
    for (int k = 0; k < 16; ++k) Bo[k] = Bq[k];
    if (!inverse4_dev(Bq, a.Binv + (size_t(m) * a.P + q) * 16)) atomicExch(a.singular, 1);
  }
  for (int xi = 0; xi < 2; ++xi)
    for (int k = 0; k < 16; ++k) a.C[size_t(q) * 32 + xi * 16 + k] = Cq[xi][k];
  const int ix_in = sgn[0] > 0 ? 0 : 1, jx = 1 - ix_in;
  const int iy_in = sgn[1] > 0 ? 0 : 1, jy = 1 - iy_in;
  double* cxy = a.cxy + size_t(q) * 8;
  for (int r = 0; r < 2; ++r)
    for (int b = 0; b < 2; ++b) {
      cxy[r * 2 + b] = Cq[0][(ix_in + 2 * r) * 4 + (jx + 2 * b)];
      cxy[4 + r * 2 + b] = Cq[1][(2 * iy_in + r) * 4 + (2 * jy + b)];
    }
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("device couplings: ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace

bool device_couplings_supported(int order) { return order >= 0 && order <= 32; }

void device_couplings(const SphereTree& t, const std::vector<int>& leaf_id, int order, int xorder_base, double* X) {
  const int P = int(leaf_id.size()), H = (order + 1) * (order + 1);
  if (P == 0) return;
  if (!device_couplings_supported(order)) throw std::invalid_argument("device couplings: order > 32");
  std::vector<double> verts(size_t(P) * 9), gx(kMaxRule * (kMaxRule + 1) / 2), gw(gx.size());
  std::vector<int> nq(P);
  const double inv = 1.0 / double(SphereTree::kScale);
  for (int q = 0; q < P; ++q) {
    const int id = leaf_id[q];
    for (int r = 0; r < 9; ++r) verts[size_t(q) * 9 + r] = double(t.flat[id][r]) * inv;
    nq[q] = patch_order(t.level[id], xorder_base);
    if (nq[q] < 1 || nq[q] > kMaxRule) throw std::invalid_argument("device couplings: quadrature order out of range");
  }
  for (int n = 1; n <= kMaxRule; ++n) {
    const double *x, *w;
    gauss_rule01(n, &x, &w);
    for (int i = 0; i < n; ++i) gx[n * (n - 1) / 2 + i] = x[i], gw[n * (n - 1) / 2 + i] = w[i];
  }
  double *dv = nullptr, *dgx = nullptr, *dgw = nullptr, *dX = nullptr;
  int* dnq = nullptr;
  cuda_ok(cudaMalloc(&dv, verts.size() * 8), "malloc");
  cuda_ok(cudaMalloc(&dgx, gx.size() * 8), "malloc");
  cuda_ok(cudaMalloc(&dgw, gw.size() * 8), "malloc");
  cuda_ok(cudaMalloc(&dnq, nq.size() * 4), "malloc");
  cuda_ok(cudaMalloc(&dX, size_t(P) * H * 8), "malloc");
  cuda_ok(cudaMemcpy(dv, verts.data(), verts.size() * 8, cudaMemcpyHostToDevice), "h2d");
  cuda_ok(cudaMemcpy(dgx, gx.data(), gx.size() * 8, cudaMemcpyHostToDevice), "h2d");
  cuda_ok(cudaMemcpy(dgw, gw.data(), gw.size() * 8, cudaMemcpyHostToDevice), "h2d");
  cuda_ok(cudaMemcpy(dnq, nq.data(), nq.size() * 4, cudaMemcpyHostToDevice), "h2d");
  CouplingArgs a{dv, dnq, dgx, dgw, dX, P, order, H};
  const int threads = P * (order + 1), blocks = (threads + 127) / 128;
  if (order <= 8) couplings_kernel<8><<<blocks, 128>>>(a);
  else if (order <= 16) couplings_kernel<16><<<blocks, 128>>>(a);
  else couplings_kernel<32><<<blocks, 128>>>(a);
  cuda_ok(cudaGetLastError(), "launch");
  cuda_ok(cudaMemcpy(X, dX, size_t(P) * H * 8, cudaMemcpyDeviceToHost), "d2h");
  for (void* p : {(void*)dv, (void*)dgx, (void*)dgw, (void*)dnq, (void*)dX}) cudaFree(p);
}

}  // namespace stamg_b200

namespace stamg_b200 {

// build_operators on the current CUDA device for the given leaves; el16 = N | V0 | V1 |
// F_self[0..3] | F_neigh[0..3] (11 4 x 4 blocks). Fills the host tables of the level.
void device_patch_blocks(const SphereTree& t, const std::vector<int>& leaf_id, const std::vector<double>& sigma_t,
                         const double* el16, double* area, double* Aflow, double* B, double* Binv, double* C, double* cxy) {
  const int P = int(leaf_id.size()), n_mat = int(sigma_t.size());
  if (P == 0) return;
  std::vector<double> verts(size_t(P) * 9), gx(kMaxRule * (kMaxRule + 1) / 2), gw(gx.size());
  std::vector<int> nq(P), oct(P);
  const double inv = 1.0 / double(SphereTree::kScale);
  for (int q = 0; q < P; ++q) {
    const int id = leaf_id[q];
    for (int r = 0; r < 9; ++r) verts[size_t(q) * 9 + r] = double(t.flat[id][r]) * inv;
    nq[q] = patch_order(t.level[id], 8);
    oct[q] = t.octant[id];
  }
  for (int n = 1; n <= kMaxRule; ++n) {
    const double *x, *w;
    gauss_rule01(n, &x, &w);
    for (int i = 0; i < n; ++i) gx[n * (n - 1) / 2 + i] = x[i], gw[n * (n - 1) / 2 + i] = w[i];
  }
  ElementMats em;
  std::copy(el16, el16 + 16, em.N);
  std::copy(el16 + 16, el16 + 48, &em.V[0][0]);
  std::copy(el16 + 48, el16 + 112, &em.Fs[0][0]);
  std::copy(el16 + 112, el16 + 176, &em.Fn[0][0]);
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
  };
  auto dev = [&](const void* src, size_t bytes) {
    void* p = nullptr;
    cuda_ok(cudaMalloc(&p, bytes), "malloc");
    if (src) cuda_ok(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "h2d");
    else cuda_ok(cudaMemset(p, 0, bytes), "memset");
    return p;
  };
  BlockArgs a{};
  a.verts = static_cast<double*>(dev(verts.data(), verts.size() * 8));
  a.nq = static_cast<int*>(dev(nq.data(), nq.size() * 4));
  a.octant = static_cast<int*>(dev(oct.data(), oct.size() * 4));
  a.gx = static_cast<double*>(dev(gx.data(), gx.size() * 8));
  a.gw = static_cast<double*>(dev(gw.data(), gw.size() * 8));
  a.sigma_t = static_cast<double*>(dev(sigma_t.data(), sigma_t.size() * 8));
  a.area = static_cast<double*>(dev(nullptr, size_t(P) * 8));
  a.Aflow = static_cast<double*>(dev(nullptr, size_t(P) * 3 * 8));
  a.B = static_cast<double*>(dev(nullptr, size_t(n_mat) * P * 16 * 8));
  a.Binv = static_cast<double*>(dev(nullptr, size_t(n_mat) * P * 16 * 8));
  a.C = static_cast<double*>(dev(nullptr, size_t(P) * 32 * 8));
  a.cxy = static_cast<double*>(dev(nullptr, size_t(P) * 8 * 8));
  a.singular = static_cast<int*>(dev(nullptr, 4));
  a.P = P, a.n_mat = n_mat;
  patch_blocks_kernel<<<(P + 127) / 128, 128>>>(a, em);
  cuda_ok(cudaGetLastError(), "launch");
  int singular = 0;
  cuda_ok(cudaMemcpy(&singular, a.singular, 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_ok(cudaMemcpy(area, a.area, size_t(P) * 8, cudaMemcpyDeviceToHost), "d2h");
  cuda_ok(cudaMemcpy(Aflow, a.Aflow, size_t(P) * 3 * 8, cudaMemcpyDeviceToHost), "d2h");
  cuda_ok(cudaMemcpy(B, a.B, size_t(n_mat) * P * 16 * 8, cudaMemcpyDeviceToHost), "d2h");
  cuda_ok(cudaMemcpy(Binv, a.Binv, size_t(n_mat) * P * 16 * 8, cudaMemcpyDeviceToHost), "d2h");
  cuda_ok(cudaMemcpy(C, a.C, size_t(P) * 32 * 8, cudaMemcpyDeviceToHost), "d2h");
  cuda_ok(cudaMemcpy(cxy, a.cxy, size_t(P) * 8 * 8, cudaMemcpyDeviceToHost), "d2h");
  for (const void* p : {(const void*)a.verts, (const void*)a.nq, (const void*)a.octant, (const void*)a.gx, (const void*)a.gw,
                        (const void*)a.sigma_t, (const void*)a.area, (const void*)a.Aflow, (const void*)a.B,
                        (const void*)a.Binv, (const void*)a.C, (const void*)a.cxy, (const void*)a.singular})
    cudaFree(const_cast<void*>(p));
  if (singular) throw std::invalid_argument("singular diagonal block");
}

}  // namespace stamg_b200
