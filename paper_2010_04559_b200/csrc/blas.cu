// Vector kernels for the Krylov loop (krylov.cpp:40-91 and the GMRES
// extension) with deterministic reductions: fixed grids, fixed-order
// partial sums, so a solve is bitwise reproducible run to run.
// Also the FP64 throughput microbenchmarks used as roofline denominators.
#include "common.cuh"
#include "kernels.hpp"

#include <algorithm>
#include <stdexcept>
#include <vector>

namespace stamg_b200 {
namespace {

constexpr int kBlk = 256;
constexpr int kDotBlocks = 1184;  // 8 x 148 SMs
constexpr int kMaxVecs = 80;

int grid_for(int64_t n) { return int(std::min<int64_t>((n + kBlk - 1) / kBlk, 148 * 32)); }

__global__ void fill_kernel(double* x, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}
__global__ void axpy_kernel(double a, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}
__global__ void axpby_kernel(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}
__global__ void scale_kernel(double a, double* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= a;
}

struct VecList {
  const double* v[kMaxVecs];
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// partial[k][b] = sum over block b's contiguous chunk of V_k . w. The chunk is streamed once per
// group of eight vectors (w read once per group, not once per vector); every partial sum adds its
// terms in the same order as a one-vector-at-a-time loop, so results are bitwise unchanged.
__global__ void __launch_bounds__(kBlk) multidot_kernel(VecList vl, int nv, const double* __restrict__ w, int64_t n,
                                                         double* __restrict__ partial) {
  __shared__ double red[kBlk / 32];
  constexpr int KG = 8;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = std::min<int64_t>(n, lo + chunk);
  for (int k0 = 0; k0 < nv; k0 += KG) {
    const int kn = min(KG, nv - k0);
    double s[KG];
#pragma unroll
    for (int kk = 0; kk < KG; ++kk) s[kk] = 0.0;
    if (kn == KG) {
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double wi = w[i];
#pragma unroll
        for (int kk = 0; kk < KG; ++kk) s[kk] += vl.v[k0 + kk][i] * wi;
      }
    } else {
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double wi = w[i];
#pragma unroll
        for (int kk = 0; kk < KG; ++kk)
          if (kk < kn) s[kk] += vl.v[k0 + kk][i] * wi;
      }
    }
#pragma unroll
    for (int kk = 0; kk < KG; ++kk) {
      if (kk >= kn) break;
      const double tot = block_sum(s[kk], red);
      if (threadIdx.x == 0) partial[(size_t)(k0 + kk) * gridDim.x + blockIdx.x] = tot;
    }
  }
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nb, double* __restrict__ out) {
  __shared__ double red[kBlk / 32];
  const int k = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += partial[(size_t)k * nb + b];
  const double tot = block_sum(s, red);
  if (threadIdx.x == 0) out[k] = tot;
}

// w -= sum_k c[k] V_k, in k order per element
__global__ void multi_axpy_kernel(VecList vl, int nv, const double* __restrict__ c, double* __restrict__ w, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double t = w[i];
    for (int k = 0; k < nv; ++k) t -= c[k] * vl.v[k][i];
    w[i] = t;
  }
}
// u = sum_k c[k] V_k, accumulated from zero in k order
__global__ void lincomb_kernel(VecList vl, int nv, const double* __restrict__ c, double* __restrict__ u, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < nv; ++k) t += c[k] * vl.v[k][i];
    u[i] = t;
  }
}

VecList make_list(const double* const* vs, int nv) {
  if (nv > kMaxVecs) throw std::invalid_argument("too many Krylov vectors in one batched op");
  VecList l{};
  for (int k = 0; k < nv; ++k) l.v[k] = vs[k];
  return l;
}

// ---------------------------------------------------------------- microbench
__global__ void dmma_peak_kernel(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_peak_kernel(double* out, int iters) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-9 + i;
  const double a = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <class K>
double time_kernel(K kern, int blocks, int threads, int iters, cudaStream_t s) {
  double* dummy = nullptr;
  cudaMalloc(&dummy, sizeof(double));
  kern<<<blocks, threads, 0, s>>>(dummy, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  kern<<<blocks, threads, 0, s>>>(dummy, iters);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(dummy);
  return ms * 1e-3;
}

// in-place read+write of 128-byte chunks (8 lanes x 16 B); chunk c maps to
// address c (mode 0, streaming) or to cell-major / group-minor order (mode 1,
// the sweep's pattern: consecutive chunks 'stride' chunks apart)
__global__ void chunk_rw_kernel(double* x, int64_t n_chunks, int64_t stride, int mode) {
  // mode 1: 128-byte chunks; mode k>1: chunks of k*128 bytes (k*8 lanes)
  const int lanes = 8 * (mode > 1 ? mode : 1);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = tid / lanes;
  if (c >= n_chunks) return;
  int64_t dst = c;
  if (mode >= 1) {
    const int64_t per = n_chunks / stride;
    dst = (c % per) * stride + c / per;
  }
  double2* p = reinterpret_cast<double2*>(x + dst * 2 * lanes) + (tid % lanes);
  double2 v = *p;
  v.x += 1.0, v.y += 1.0;
  *p = v;
}

}  // namespace

double bench_chunk_rw_gbs(double* buf, int64_t n_doubles, int64_t stride_chunks, int mode, cudaStream_t s) {
  const int lanes = 8 * (mode > 1 ? mode : 1);
  const int64_t n_chunks = n_doubles / (2 * lanes);
  const int64_t threads = n_chunks * lanes;
  const int blocks = int((threads + 255) / 256);
  chunk_rw_kernel<<<blocks, 256, 0, s>>>(buf, n_chunks, stride_chunks, mode);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 5; ++r) chunk_rw_kernel<<<blocks, 256, 0, s>>>(buf, n_chunks, stride_chunks, mode);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 5.0 * 2.0 * n_doubles * 8 / (ms * 1e-3) / 1e9;
}

void launch_fill(double* x, double v, int64_t n, cudaStream_t s) {
  if (n > 0) fill_kernel<<<grid_for(n), kBlk, 0, s>>>(x, v, n);
}
void launch_axpy(double a, const double* x, double* y, int64_t n, cudaStream_t s) {
  if (n > 0) axpy_kernel<<<grid_for(n), kBlk, 0, s>>>(a, x, y, n);
}
void launch_axpby(double a, const double* x, double b, double* y, int64_t n, cudaStream_t s) {
  if (n > 0) axpby_kernel<<<grid_for(n), kBlk, 0, s>>>(a, x, b, y, n);
}
void launch_scale(double a, double* x, int64_t n, cudaStream_t s) {
  if (n > 0) scale_kernel<<<grid_for(n), kBlk, 0, s>>>(a, x, n);
}
int multidot_blocks() { return kDotBlocks; }
void launch_multidot(const double* const* vs, int nv, const double* w, int64_t n, double* partial, double* out,
                     cudaStream_t s) {
  if (nv <= 0) return;
  multidot_kernel<<<kDotBlocks, kBlk, 0, s>>>(make_list(vs, nv), nv, w, n, partial);
  reduce_partials_kernel<<<nv, kBlk, 0, s>>>(partial, kDotBlocks, out);
}
void launch_multi_axpy(const double* const* vs, int nv, const double* c, double* w, int64_t n, cudaStream_t s) {
  if (nv > 0 && n > 0) multi_axpy_kernel<<<grid_for(n), kBlk, 0, s>>>(make_list(vs, nv), nv, c, w, n);
}
void launch_lincomb(const double* const* vs, int nv, const double* c, double* u, int64_t n, cudaStream_t s) {
  if (n > 0) lincomb_kernel<<<grid_for(n), kBlk, 0, s>>>(make_list(vs, nv), nv, c, u, n);
}

double bench_dmma_tflops(int device, cudaStream_t s) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 4, threads = 256, iters = 4096;
  const double sec = time_kernel(dmma_peak_kernel, blocks, threads, iters, s);
  const double flops = double(blocks) * (threads / 32) * iters * 8 * (2.0 * 8 * 8 * 4);
  return flops / sec * 1e-12;
}
double bench_dfma_tflops(int device, cudaStream_t s) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8, threads = 256, iters = 8192;
  const double sec = time_kernel(dfma_peak_kernel, blocks, threads, iters, s);
  const double flops = double(blocks) * threads * iters * 8 * 2.0;
  return flops / sec * 1e-12;
}

}  // namespace stamg_b200
