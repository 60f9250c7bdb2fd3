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
