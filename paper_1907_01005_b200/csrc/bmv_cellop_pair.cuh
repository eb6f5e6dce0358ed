// K1 thread-per-pair building blocks for n <= 3 (Q1 / Q2): one thread holds
// a whole (cell, column) pair's n^3 tensor in registers, so the 12
// contractions need no transposes at all (used by bmv_k1.cu).
#pragma once

#include "bmv_sumfac.cuh"
#include "bmv_tma.cuh"

namespace bmv {

// out[line](a) = sum_b M[a][b] in[line](b) along axis `ax` of a [z][y][x] tensor
template <int N, int AX, bool TR>
__device__ __forceinline__ void contract3(double (&v)[N][N][N], const double* __restrict__ M) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double in[N], o[N];
#pragma unroll
      for (int b = 0; b < N; ++b) in[b] = AX == 0 ? v[i][j][b] : (AX == 1 ? v[i][b][j] : v[b][i][j]);
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) s = fma(TR ? M[b * N + a] : M[a * N + b], in[b], s);
        o[a] = s;
      }
#pragma unroll
      for (int a = 0; a < N; ++a) {
        if (AX == 0) v[i][j][a] = o[a];
        else if (AX == 1) v[i][a][j] = o[a];
        else v[a][i][j] = o[a];
      }
    }
  }
}

// acc += D^T diag(kin_ax * w3) D uq along axis `ax`, line by line
template <int N, int AX>
__device__ __forceinline__ void grad3(const double (&uq)[N][N][N], double (&acc)[N][N][N],
                                      const CellTables& tb) {
  const double kin = tb.kin[AX];
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double g[N];
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) {
          const double u = AX == 0 ? uq[i][j][b] : (AX == 1 ? uq[i][b][j] : uq[b][i][j]);
          s = fma(tb.D[a * N + b], u, s);
        }
        // weight of the quadrature point: AX = x: (z, y, x) = (i, j, a);
        // y: (i, a, j); z: (a, i, j).  w3 = w[z] * w[y] * w[x]
        const double w3 = tb.w[AX == 2 ? a : i] * tb.W2[(AX == 1 ? a : (AX == 2 ? i : j)) * N +
                                                        (AX == 0 ? a : j)];
        g[a] = s * (kin * w3);
      }
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double s = AX == 0 ? acc[i][j][b] : (AX == 1 ? acc[i][b][j] : acc[b][i][j]);
#pragma unroll
        for (int a = 0; a < N; ++a) s = fma(tb.D[a * N + b], g[a], s);
        if (AX == 0) acc[i][j][b] = s;
        else if (AX == 1) acc[i][b][j] = s;
        else acc[b][i][j] = s;
      }
    }
  }
}

}  // namespace bmv
