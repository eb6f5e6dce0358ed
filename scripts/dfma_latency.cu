// DFMA issue / latency probe: one warp per SM runs K independent dependent
// chains; cycles per DFMA vs K shows the pipe latency (K = 1) and the
// single-warp issue rate (large K).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, int iters, double a, double b, long long* cyc) {
  double r[K];
#pragma unroll
  for (int k = 0; k < K; ++k) r[k] = threadIdx.x * 1e-3 + k;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = fma(r[k], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int K>
void run(double* out, long long* cyc, int warps) {
  const int iters = 4096;
  chains<K><<<148, 32 * warps>>>(out, iters, 1.0000001, 1e-9, cyc);
  chains<K><<<148, 32 * warps>>>(out, iters, 1.0000001, 1e-9, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("warps/SM %2d chains %2d: %.2f cycles per DFMA (per warp), %.2f per SMSP-issue\n", warps, K,
         (double)h / (iters * (double)K), (double)h / (iters * (double)K) / ((warps + 3) / 4));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 12}) {
    run<1>(out, cyc, w);
    run<2>(out, cyc, w);
    run<4>(out, cyc, w);
    run<5>(out, cyc, w);
    run<8>(out, cyc, w);
    run<16>(out, cyc, w);
    run<25>(out, cyc, w);
  }
  return 0;
}
