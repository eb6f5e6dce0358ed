// Microbenchmark: FP64 FMA (DFMA) vs FP64 tensor-core (DMMA m8n8k4) throughput
// on this GPU.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = fma(r[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// Mixed: warps with (warp & 1) == 0 run DFMA chains, the others DMMA chains.  If the
// two run on separate pipes the combined rate exceeds either alone.
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  const int warp = threadIdx.x >> 5;
  if (warp & 1) {
    double fa = threadIdx.x * 1e-3, fb = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(fa), "d"(fb));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = fma(r[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += r[k];
    if (s == 12345.678) out[0] = s;
  }
}

// Same warp: 8 DMMA + 16 DFMA interleaved per iteration.
__global__ void interleaved_kernel(double* out, int iters, double a, double b) {
  double fa = threadIdx.x * 1e-3, fb = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
  double r[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(fa), "d"(fb));
      r[2 * k] = fma(r[2 * k], a, b);
      r[2 * k + 1] = fma(r[2 * k + 1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < 16; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512}) {
    for (int bps : {4, 8}) {
      const int blocks = sms * bps, iters = 4096;
      dfma_kernel<<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * (double)blocks * threads;
      printf("DFMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, fl / (ms * 1e-3) / 1e12);
      dmma_kernel<<<blocks, threads>>>(out, 64);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
      printf("DMMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, fl / (ms * 1e-3) / 1e12);
      mixed_kernel<<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      mixed_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      {
        const double w = (double)blocks * (threads / 32) / 2;
        const double f1 = 2.0 * 16 * iters * w * 32, f2 = 2.0 * 8 * 8 * 4 * 8 * (double)iters * w;
        printf("MIXED (half warps DFMA, half DMMA) threads=%d blocks/SM=%d: %.2f + %.2f = %.2f TFLOP/s\n",
               threads, bps, f1 / (ms * 1e-3) / 1e12, f2 / (ms * 1e-3) / 1e12,
               (f1 + f2) / (ms * 1e-3) / 1e12);
      }
      interleaved_kernel<<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      interleaved_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      {
        const double w = (double)blocks * (threads / 32);
        const double f1 = 2.0 * 16 * iters * w * 32, f2 = 2.0 * 8 * 8 * 4 * 8 * (double)iters * w;
        printf("INTERLEAVED (same warp) threads=%d blocks/SM=%d: %.2f + %.2f = %.2f TFLOP/s\n",
               threads, bps, f1 / (ms * 1e-3) / 1e12, f2 / (ms * 1e-3) / 1e12,
               (f1 + f2) / (ms * 1e-3) / 1e12);
      }
    }
  }
  return 0;
}
