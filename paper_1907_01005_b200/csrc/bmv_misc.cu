// Device helpers of the hot path: the Gaussian-sum potential at the
// quadrature points (OperatorSpec.sample_potential of the reference,
// bcsrmv/matfree.py:35-40,491-495, evaluated once per operator on the
// device), the streaming zero kernel (BlockCsrMatrix.zero_out,
// bcsr.py:334-339) and the FP64 tensor-core (DMMA) peak probe used with the
// DFMA probe (bmv_util.cu) as the roofline denominator.
#include <cuda_runtime.h>

#include <algorithm>

#include "bmv_common.cuh"

namespace bmv {
namespace {

__global__ void gaussian_coef_kernel(const double* __restrict__ origins,
                                     const double* __restrict__ qoff,
                                     const double* __restrict__ w3,
                                     const double* __restrict__ centers, int n_centers,
                                     double inv_s2, double scale, int q3, int64_t n_cells,
                                     double* __restrict__ coef) {
  extern __shared__ double cs[];
  for (int i = threadIdx.x; i < 3 * n_centers; i += blockDim.x) cs[i] = centers[i];
  __syncthreads();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_cells * q3) return;
  const int64_t cell = idx / q3;
  const int q = (int)(idx - cell * q3);
  const double px = origins[cell * 3 + 0] + qoff[q * 3 + 0];
  const double py = origins[cell * 3 + 1] + qoff[q * 3 + 1];
  const double pz = origins[cell * 3 + 2] + qoff[q * 3 + 2];
  double v = 0.0;
  for (int c = 0; c < n_centers; ++c) {
    const double dx = px - cs[3 * c], dy = py - cs[3 * c + 1], dz = pz - cs[3 * c + 2];
    const double e = (dx * dx + dy * dy + dz * dz) * inv_s2;
    if (e < 746.0) v += exp(-e);  // exp(-746) rounds to +0: skipping is exact
  }
  coef[idx] = w3[q] * (scale * v);
}

// p 16-byte aligned; each thread stores 4 x 16 bytes, warp-contiguous per
// store (one CTA of 256 threads covers 8 KB): measured 7.4 TB/s of writes.
constexpr int kZeroThreads = 256, kZeroPerThread = 8;  // doubles
__global__ void __launch_bounds__(kZeroThreads) zero_kernel(double* __restrict__ p, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * (kZeroThreads * kZeroPerThread);
#pragma unroll
  for (int j = 0; j < kZeroPerThread / 2; ++j) {
    const int64_t i = base + (int64_t)j * (2 * kZeroThreads) + 2 * threadIdx.x;
    if (i + 1 < n)
      *reinterpret_cast<double2*>(p + i) = make_double2(0.0, 0.0);
    else if (i < n)
      p[i] = 0.0;
  }
}

// Independent DMMA m8n8k4 chains, no memory traffic (FP64 tensor-core peak).
__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

int zero_async(double* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return BMV_OK;
  if (reinterpret_cast<uintptr_t>(p) & 15) {  // 8-byte aligned start (odd element offset)
    BMV_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double), st));
    ++p;
    if (--n == 0) return BMV_OK;
  }
  const int64_t per = (int64_t)kZeroThreads * kZeroPerThread;
  const int64_t grid = (n + per - 1) / per;
  for (int64_t g0 = 0; g0 < grid; g0 += 0x7fffffff) {
    const int64_t g = std::min<int64_t>(grid - g0, 0x7fffffff);
    zero_kernel<<<(unsigned)g, kZeroThreads, 0, st>>>(p + g0 * per, n - g0 * per);
    BMV_CHECK_LAUNCH();
  }
  return BMV_OK;
}

}  // namespace bmv

using namespace bmv;

extern "C" {

int bmv_potential_gaussian(int64_t n_cells, int32_t q3, const double* cell_origins,
                           const double* quad_offsets, const double* w3, const double* centers,
                           int32_t n_centers, double inv_sigma2, double scale, double* coef,
                           void* stream) {
  if (n_cells < 0 || q3 <= 0 || n_centers < 0 || (n_cells > 0 && (!cell_origins || !quad_offsets ||
      !w3 || !coef)) || (n_centers > 0 && !centers)) {
    set_error("invalid gaussian potential arguments");
    return BMV_ERR_INVALID;
  }
  if (n_centers > 4096) {
    set_error("at most 4096 potential centres per launch (got %d)", n_centers);
    return BMV_ERR_INVALID;
  }
  if (n_cells == 0) return BMV_OK;
  const int64_t total = n_cells * q3;
  const unsigned grid = (unsigned)((total + 255) / 256);
  gaussian_coef_kernel<<<grid, 256, sizeof(double) * 3 * std::max(n_centers, 1),
                         as_stream(stream)>>>(cell_origins, quad_offsets, w3, centers, n_centers,
                                              inv_sigma2, scale, q3, n_cells, coef);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

int bmv_fp64_dmma_peak_kernel(double* scratch, int32_t blocks, int32_t iters, double* flops_out,
                              void* stream) {
  if (!scratch || blocks <= 0 || iters <= 0) {
    set_error("invalid peak-probe arguments");
    return BMV_ERR_INVALID;
  }
  const int threads = 256;
  dmma_peak_kernel<<<blocks, threads, 0, as_stream(stream)>>>(scratch, iters);
  BMV_CHECK_LAUNCH();
  // per warp and iteration: 8 DMMA of 8 x 8 x 4 FMAs
  if (flops_out) *flops_out = 2.0 * 8 * 256 * (double)iters * (threads / 32) * blocks;
  return BMV_OK;
}

}  // extern "C"
