// Probe of the K1 contraction core alone (bmv_sumfac.cuh sumfac_h_lean): W warps
// per SM loop over synthetic pairs held in registers; reports cycles per
// warp-batch and the FP64 rate, without gather / scatter / metadata.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_1907_01005_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "bmv_sumfac.cuh"

using namespace bmv;

template <int N, int REGS>
__global__ void __launch_bounds__(384) __maxnreg__(REGS)
    probe(double* out, int iters, const __grid_constant__ CellTables tb, long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int P = 32 / N, TILE = Tile3<N>::TILE;
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int hl = lid & 15;
  const int sub = (lid >> 4) * (P / 2) + hl / N, t = hl % N;
  const bool lane_ok = hl < (P / 2) * N;
  const int tt = lane_ok ? t : 0;
  double* wbase = reinterpret_cast<double*>(smem) + warp * (P * TILE + 128);
  double* buf = wbase + (lane_ok ? sub : 0) * TILE;
  double* cs = wbase + P * TILE;  // coefficient row (126 doubles)
  for (int i = lid; i < 126; i += 32) cs[i] = 1.0 + i * 1e-3;
  __syncwarp();
  double u[N][N], o[N][N], acc = 0.0;
#pragma unroll
  for (int z = 0; z < N; ++z)
#pragma unroll
    for (int y = 0; y < N; ++y) u[z][y] = 1e-3 * (z + 2 * y + 3 * t) + 1e-4 * sub;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sumfac_h_lean<N, true, Tile3<N>>(u, o, buf, tt, lane_ok, cs, tb);
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int y = 0; y < N; ++y) u[z][y] = o[z][y] * 1e-3 + 1e-3;
    acc += o[0][0];
  }
  const long long t1 = clock64();
  if (acc == 12345.678) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

// pieces: MODE 0 = 12 plain contractions, no transposes; 1 = 4 transposes only
template <int N, int REGS, int MODE>
__global__ void __launch_bounds__(384) __maxnreg__(REGS)
    pieces(double* out, int iters, const __grid_constant__ CellTables tb, long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int P = 32 / N, TILE = Tile3<N>::TILE;
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int hl = lid & 15;
  const int sub = (lid >> 4) * (P / 2) + hl / N, t = hl % N;
  const bool lane_ok = hl < (P / 2) * N;
  const int tt = lane_ok ? t : 0;
  double* wbase = reinterpret_cast<double*>(smem) + warp * (P * TILE + 128);
  double* buf = wbase + (lane_ok ? sub : 0) * TILE;
  double u[N][N], o[N][N], acc = 0.0;
#pragma unroll
  for (int z = 0; z < N; ++z)
#pragma unroll
    for (int y = 0; y < N; ++y) u[z][y] = 1e-3 * (z + 2 * y + 3 * t) + 1e-4 * sub;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        contract_fast<N, false>(u, o, tb.S);
        contract_slow<N, false>(o, u, tb.D);
        contract_fast<N, true>(u, o, tb.D);
        contract_slow<N, true>(o, u, tb.S);
      }
    } else {
      x_to_y<N, typename Tile3<N>::XY>(u, o, buf, tt, lane_ok);
      y_to_z<N, typename Tile3<N>::YZ>(o, u, buf, tt, lane_ok);
      y_to_z<N, typename Tile3<N>::YZ>(u, o, buf, tt, lane_ok);
      z_to_x<N, typename Tile3<N>::ZX>(o, u, buf, tt, lane_ok);
    }
    acc += u[0][0];
  }
  const long long t1 = clock64();
  if (acc == 12345.678) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int N, int REGS, int MODE>
void run_pieces(double* out, long long* cyc, int warps, const CellTables& tb) {
  const int iters = 2000;
  const int smem = warps * (32 / N * Tile3<N>::TILE + 128) * 8;
  cudaFuncSetAttribute(pieces<N, REGS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pieces<N, REGS, MODE><<<148, 32 * warps, smem>>>(out, 10, tb, cyc);
  pieces<N, REGS, MODE><<<148, 32 * warps, smem>>>(out, iters, tb, cyc);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("pieces n=%d mode %d (%s) warps/SM %2d: %.0f cycles per iteration per warp\n", N, MODE,
         MODE == 0 ? "12 contractions" : "4 transposes", warps, (double)h / iters);
}

template <int N, int REGS>
void run(double* out, long long* cyc, int warps, const CellTables& tb) {
  const int iters = 2000;
  const int smem = warps * (32 / N * Tile3<N>::TILE + 128) * 8;
  cudaFuncSetAttribute(probe<N, REGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, REGS><<<148, 32 * warps, smem>>>(out, 10, tb, cyc);
  probe<N, REGS><<<148, 32 * warps, smem>>>(out, iters, tb, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / iters;
  const double fma_thread = 12.0 * N * N * N + 4 * N * N;  // 12 contractions + pointwise
  printf("n=%d regs=%d warps/SM %2d: %.0f cycles per warp-batch, %.0f per SMSP-batch -> FP64 pipe %.1f %% (%s)\n",
         N, REGS, warps, per, per / ((warps + 3) / 4), 100.0 * fma_thread * 2.18 / (per / ((warps + 3) / 4)),
         cudaGetErrorString(e));
}

int main() {
  CellTables tb{};
  for (int i = 0; i < 25; ++i) {
    tb.S[i] = 0.1 + 0.01 * i;
    tb.D[i] = 0.2 - 0.01 * i;
    tb.W2[i] = 0.05 + 0.001 * i;
  }
  for (int i = 0; i < 5; ++i) tb.w[i] = 0.2 + 0.01 * i;
  tb.kin[0] = tb.kin[1] = tb.kin[2] = 0.5;
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  for (int w : {4, 8}) run_pieces<5, 255, 0>(out, cyc, w, tb);
  for (int w : {4, 8}) run_pieces<5, 255, 1>(out, cyc, w, tb);
  for (int w : {4, 8}) run_pieces<4, 168, 0>(out, cyc, w, tb);
  for (int w : {4, 8}) run_pieces<4, 168, 1>(out, cyc, w, tb);
  for (int w : {4, 8, 12}) run<5, 255>(out, cyc, w <= 8 ? w : 8, tb);
  for (int w : {4, 8, 12}) run<5, 168>(out, cyc, w, tb);
  for (int w : {4, 8, 12}) run<4, 168>(out, cyc, w, tb);
  return 0;
}
