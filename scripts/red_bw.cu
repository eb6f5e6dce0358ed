// Microbenchmark: fp64 RED.ADD throughput into an L2-resident region of
// `region` doubles (contention ~ total / region), and 8-byte loads (gather)
// from the same region.  Informs the K4 flush design.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red_kernel(double* dst, long long region, int per_thread, unsigned seed) {
  unsigned s = seed ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
  for (int i = 0; i < per_thread; ++i) {
    s = s * 1664525u + 1013904223u;
    atomicAdd(dst + (s % region), 1.0);
  }
}
__global__ void red_coal_kernel(double* dst, long long region, int per_thread, unsigned seed) {
  // warp-coalesced: 32 lanes hit 32 consecutive doubles of a random 256-B row
  unsigned s = seed ^ (blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u);
  for (int i = 0; i < per_thread; ++i) {
    s = s * 1664525u + 1013904223u;
    long long row = (s % (region / 32)) * 32;
    atomicAdd(dst + row + (threadIdx.x & 31), 1.0);
  }
}
__global__ void ld_kernel(const double* src, long long region, int per_thread, unsigned seed, double* out) {
  unsigned s = seed ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
  double acc = 0;
  for (int i = 0; i < per_thread; ++i) {
    s = s * 1664525u + 1013904223u;
    acc += __ldg(src + (s % region));
  }
  if (acc == 12345.0) out[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 1ll << 30); cudaMemset(d, 0, 1ll << 30);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  long long regions[] = {1 << 14, 1 << 17, 1 << 20, 1 << 24};
  const int per = 256, threads = 256, blocks = sms * 8;
  const double total = (double)per * threads * blocks;
  for (long long r : regions) {
    for (int kind = 0; kind < 3; ++kind) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (kind == 0) red_kernel<<<blocks, threads>>>(d, r, per, rep);
        else if (kind == 1) red_coal_kernel<<<blocks, threads>>>(d, r, per, rep);
        else ld_kernel<<<blocks, threads>>>(d, r, per, rep, d);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 2)
          printf("%s region %lld doubles (%.1f MB): %.1f G ops/s (%.3f ms for %.0f M)\n",
                 kind == 0 ? "RED random " : (kind == 1 ? "RED coalesc" : "LD random  "), r,
                 r * 8e-6, total / (ms * 1e-3) / 1e9, ms, total / 1e6);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
