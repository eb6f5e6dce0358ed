// Device building blocks of the sum-factorised cell kernels (K1): the 1D
// tables, register-resident contractions of one n x n plane per thread,
// the per-pair shared-memory transposes and cp.async helpers.  Shared by
// the one-pass kernel (bmv_cellop.cu) and the TMA-streamed kernel
// (bmv_cellop_stream.cu).  Arithmetic follows cell_integrals_sumfac of the
// reference (bcsrmv/matfree.py:288-367) in collocation form.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "bmv.h"

namespace bmv {

struct CellTables {
  double S[BMV_MAX_NODES * BMV_MAX_NODES];    // S[q*n + i]
  double D[BMV_MAX_NODES * BMV_MAX_NODES];    // D_co[q*n + j]
  double W2[BMV_MAX_NODES * BMV_MAX_NODES];   // w[a]*w[b]
  double w[BMV_MAX_NODES];
  double kin[3];
};

// Contract along the fast (last) index of a [N][N] plane:
// out[s][q] = sum_j M[q*N + j] * in[s][j]  (TR: M[j*N + q])
template <int N, bool TR>
__device__ __forceinline__ void contract_fast(const double (&in)[N][N], double (&out)[N][N],
                                              const double* __restrict__ M) {
#pragma unroll
  for (int s = 0; s < N; ++s) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(TR ? M[j * N + q] : M[q * N + j], in[s][j], acc);
      out[s][q] = acc;
    }
  }
}

// Contract along the slow (first) index: out[q][f] = sum_j M[q*N+j] in[j][f]
template <int N, bool TR>
__device__ __forceinline__ void contract_slow(const double (&in)[N][N], double (&out)[N][N],
                                              const double* __restrict__ M) {
#pragma unroll
  for (int q = 0; q < N; ++q) {
#pragma unroll
    for (int f = 0; f < N; ++f) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(TR ? M[j * N + q] : M[q * N + j], in[j][f], acc);
      out[q][f] = acc;
    }
  }
}

// Per-pair transpose tile: element (z, y, x) at z*BZ + y*BY + x, pairs TILE
// apart.  Strides chosen by a half-warp bank model (64-bit accesses, 16
// bank pairs per 128 B wavefront) for the pair-major lane mapping: N = 3, 4
// conflict-free stores and loads (2 + 2 wavefronts), N = 5 2 + 3.
template <int N> struct Tile;
template <> struct Tile<2> { static constexpr int BY = 2, BZ = 4, TILE = 9; };
template <> struct Tile<3> { static constexpr int BY = 5, BZ = 21, TILE = 63; };
template <> struct Tile<4> { static constexpr int BY = 4, BZ = 20, TILE = 77; };
// n = 5: a 2 + 2 layout (BY 7, BZ 39, TILE 195) exists but its 45 % larger
// footprint pushes the TMA K1 past the 196 KB shared-memory carve-out
template <> struct Tile<5> { static constexpr int BY = 5, BZ = 27, TILE = 135; };  // 2 + 3 wavefronts

// A (z = t, [y][x]) -> B (y = t, [z][x]) through the pair tile.
template <int N, class L = Tile<N>>
__device__ __forceinline__ void a_to_b(const double (&a)[N][N], double (&b)[N][N],
                                       double* buf, int t, bool store) {
  __syncwarp();
  if (store) {
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) buf[t * L::BZ + y * L::BY + x] = a[y][x];
  }
  __syncwarp();
#pragma unroll
  for (int z = 0; z < N; ++z)
#pragma unroll
    for (int x = 0; x < N; ++x) b[z][x] = buf[z * L::BZ + t * L::BY + x];
}

// B (y = t, [z][x]) -> A (z = t, [y][x]).
template <int N, class L = Tile<N>>
__device__ __forceinline__ void b_to_a(const double (&b)[N][N], double (&a)[N][N],
                                       double* buf, int t, bool store) {
  __syncwarp();
  if (store) {
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int x = 0; x < N; ++x) buf[z * L::BZ + t * L::BY + x] = b[z][x];
  }
  __syncwarp();
#pragma unroll
  for (int y = 0; y < N; ++y)
#pragma unroll
    for (int x = 0; x < N; ++x) a[y][x] = buf[t * L::BZ + y * L::BY + x];
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_one() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}

// H = -1/2 Laplace (+ c(q) u(q)) on one pair, thread t holding plane z = t
// of the pair's n^3 tensor ("A" layout, [y][x]).  In: u = nodal values;
// out: the cell integral at the nodes, same layout.  Collocation form at the
// Gauss points (q = n): 3 interpolations, gradients with D_co = D S^-1
// (3 + 3 transposed), 3 transposed interpolations = 12 contractions of n^4
// FMAs, 4 transposes through the pair tile `buf`.  The coefficient of
// quadrature point (qz = t, qy = i, qx = j) is read at cf[(i * N + j) * CS].
__device__ __forceinline__ double coef_at(const double* cf, int k) { return cf[k]; }

struct NoMass {
  template <int N, class L>
  __device__ __forceinline__ void operator()(double (&)[N][N], double*, int, bool,
                                             const CellTables&) const {}
};

// MASS (optional): called with the values at the quadrature points in B
// layout (qy = t, [qz][qx]) once the Hamiltonian no longer needs them, after
// the Hamiltonian result has been handed to HOUT (A layout); it owns the
// array from then on (the fused mass + Hamiltonian apply).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// HOOK (optional): called once the coefficient row `cf` has been read by
// every lane (the caller may then reuse its shared memory).
template <int N, bool COEF, int CS, class L = Tile<N>, class CP = const double*,
          class MASS = NoMass, class HOUT = NoMass, class HOOK = NoHook>
__device__ __forceinline__ void sumfac_h_plane(const double (&u)[N][N], double (&v2)[N][N],
                                               double* buf, int tt, bool lane_ok,
                                               CP cf, const CellTables& tb,
                                               const MASS& mass = MASS(),
                                               const HOUT& hout = HOUT(),
                                               const HOOK& hook = HOOK()) {
  double v1[N][N];
  contract_fast<N, false>(u, v1, tb.S);   // x
  contract_slow<N, false>(v1, v2, tb.S);  // y
  a_to_b<N, L>(v2, v1, buf, tt, lane_ok);    // B: y = qy = t, [z][qx]
  double uqB[N][N];
  contract_slow<N, false>(v1, uqB, tb.S); // z -> uq at (qz, qy=t, qx)
  double acc[N][N];
  // gy in A layout (qz = t)
  b_to_a<N, L>(uqB, v1, buf, tt, lane_ok);  // v1 = uq[qz=t][qy][qx]
  contract_slow<N, false>(v1, v2, tb.D);  // d/dy at the points
  const double fy = tb.w[tt] * tb.kin[1];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) v2[i][j] *= fy * tb.W2[i * N + j];
  contract_slow<N, true>(v2, acc, tb.D);  // D^T along y
  if (COEF) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) acc[i][j] = fma(coef_at(cf, CS * (i * N + j)), v1[i][j], acc[i][j]);
  }
  hook();
  a_to_b<N, L>(acc, v2, buf, tt, lane_ok);  // v2 = acc in B (qy = t): [qz][qx]
  // gx and gz in B layout, applied row/column-wise to limit live registers
  const double wt = tb.w[tt];
  const double fx = wt * tb.kin[0];
  const double fz = wt * tb.kin[2];
#pragma unroll
  for (int z = 0; z < N; ++z) {
    double g[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[q * N + j], uqB[z][j], s);
      g[q] = s * (fx * tb.W2[z * N + q]);
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = v2[z][q];
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[j * N + q], g[j], s);
      v2[z][q] = s;
    }
  }
#pragma unroll
  for (int x = 0; x < N; ++x) {
    double g[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[q * N + j], uqB[j][x], s);
      g[q] = s * (fz * tb.W2[q * N + x]);
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = v2[q][x];
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[j * N + q], g[j], s);
      v2[q][x] = s;
    }
  }
  // back to the nodes: z, x in B, then y in A
  contract_slow<N, true>(v2, v1, tb.S);   // S^T along z
  contract_fast<N, true>(v1, v2, tb.S);   // S^T along x
  b_to_a<N, L>(v2, v1, buf, tt, lane_ok);    // A: z = t, [qy][x]
  contract_slow<N, true>(v1, v2, tb.S);   // S^T along y -> out[y][x]
  if (!std::is_same<MASS, NoMass>::value) {
    hout.template operator()<N, L>(v2, buf, tt, lane_ok, tb);  // Hamiltonian result out
    mass.template operator()<N, L>(uqB, buf, tt, lane_ok, tb);
  }
}

// Three-layout transposes of the plane kernel (bmv_k1.cu).  A pair's n^3
// tensor U[z][y][x] lives in n threads, thread t holding one plane:
//   X layout: x = t, a[z][y];  Y layout: y = t, b[z][x];  Z layout: z = t, c[y][x].
// A transpose goes through the pair's shared tile, element (z, y, x) at
// z BZ + y BY + x BX, pairs TILE apart.  Shared memory serves a 64-bit warp
// access in two half-warp wavefronts when the 16 lanes of each half hit 16
// different bank pairs (a model fitted to a measured scan of ~160 layouts,
// profiles/r02_k1_tile_scan.txt: correlation 0.99).  Each transpose uses its
// OWN strides -- only the two axes that are thread indices on either side
// need conflict-free strides, the third gets stride 1:
//   n = 5 (lanes: pairs 0-2 in lanes 0-14, pairs 3-5 in lanes 16-30, see
//   k1_plane_kernel): TILE = 135 with t-strides 5 and 27 is conflict-free;
//   n = 4 (8 pairs x 4 lanes): TILE = 76, strides 1, 5, 19 for all three.
template <int SX, int SY, int SZ, int T>
struct TileMap {
  static constexpr int BX = SX, BY = SY, BZ = SZ, TILE = T;
};
template <int N> struct Tile3;
template <> struct Tile3<4> {
  static constexpr int TILE = 76;
  using XY = TileMap<1, 5, 19, 76>;
  using YZ = XY;
  using ZX = XY;
};
template <> struct Tile3<5> {
  static constexpr int TILE = 135;
  using XY = TileMap<5, 27, 1, 135>;   // x_to_y: thread axes x (store), y (load)
  using YZ = TileMap<1, 5, 27, 135>;   // y_to_z: y, z
  using ZX = TileMap<27, 1, 5, 135>;   // z_to_x: z, x
};

template <int N, class L>
__device__ __forceinline__ void x_to_y(const double (&a)[N][N], double (&b)[N][N], double* buf,
                                       int t, bool store) {
  __syncwarp();
  if (store) {
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int y = 0; y < N; ++y) buf[z * L::BZ + y * L::BY + t * L::BX] = a[z][y];
  }
  __syncwarp();
#pragma unroll
  for (int z = 0; z < N; ++z)
#pragma unroll
    for (int x = 0; x < N; ++x) b[z][x] = buf[z * L::BZ + t * L::BY + x * L::BX];
}
template <int N, class L>
__device__ __forceinline__ void y_to_z(const double (&b)[N][N], double (&c)[N][N], double* buf,
                                       int t, bool store) {
  __syncwarp();
  if (store) {
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int x = 0; x < N; ++x) buf[z * L::BZ + t * L::BY + x * L::BX] = b[z][x];
  }
  __syncwarp();
#pragma unroll
  for (int y = 0; y < N; ++y)
#pragma unroll
    for (int x = 0; x < N; ++x) c[y][x] = buf[t * L::BZ + y * L::BY + x * L::BX];
}
template <int N, class L>
__device__ __forceinline__ void z_to_x(const double (&c)[N][N], double (&a)[N][N], double* buf,
                                       int t, bool store) {
  __syncwarp();
  if (store) {
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) buf[t * L::BZ + y * L::BY + x * L::BX] = c[y][x];
  }
  __syncwarp();
#pragma unroll
  for (int z = 0; z < N; ++z)
#pragma unroll
    for (int y = 0; y < N; ++y) a[z][y] = buf[z * L::BZ + y * L::BY + t * L::BX];
}

// H = -1/2 Laplace (+ c(q) u(q)) on one pair (the plane kernel of bmv_k1.cu).
// In and out: X layout (thread t holds x = t, [z][y]), so that the lanes of
// a pair gather / scatter CONSECUTIVE DoFs (consecutive slab rows when they
// lie in one block row).  Same 12 contractions and 4 transposes as
// sumfac_h_plane, ordered so that at most two planes (+ a column of
// temporaries) are live: interpolate y, z (X), transpose, x (Y); coefficient
// term and the x / z gradient terms in Y; transpose the values and the
// partial result to Z; y gradient term, interpolate back along y, x (Z);
// transpose, back along z (X).  cf: the cell's coefficient row (q^3 values,
// point (qz, qy, qx) at qz n^2 + qy n + qx).
// MASS (optional): called with the values at the quadrature points in Z
// layout (qz = t, [qy][qx]) after the Hamiltonian result has been handed to
// HOUT (X layout); it may overwrite them.
template <int N, bool COEF, class L = Tile3<N>, class MASS = NoMass, class HOUT = NoMass>
__device__ __forceinline__ void sumfac_h_lean(const double (&u)[N][N], double (&out)[N][N],
                                              double* buf, int tt, bool lane_ok,
                                              const double* cf, const CellTables& tb,
                                              const MASS& mass = MASS(),
                                              const HOUT& hout = HOUT()) {
  constexpr int N2 = N * N;
  double p1[N][N], p2[N][N];
  contract_fast<N, false>(u, p1, tb.S);    // y
  contract_slow<N, false>(p1, p2, tb.S);   // z
  x_to_y<N, typename L::XY>(p2, p1, buf, tt, lane_ok);  // Y: qy = t, [qz][x]
  contract_fast<N, false>(p1, p2, tb.S);   // x -> p2 = uq[qz][qx] (Y)
  const double wt = tb.w[tt];
  const double fx = wt * tb.kin[0], fz = wt * tb.kin[2];
  // p1 = coefficient term + x and z gradient terms (Y)
#pragma unroll
  for (int z = 0; z < N; ++z) {
    double g[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[q * N + j], p2[z][j], s);
      g[q] = s * (fx * tb.W2[z * N + q]);
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = COEF ? cf[z * N2 + tt * N + q] * p2[z][q] : 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[j * N + q], g[j], s);
      p1[z][q] = s;
    }
  }
#pragma unroll
  for (int x = 0; x < N; ++x) {
    double g[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[q * N + j], p2[j][x], s);
      g[q] = s * (fz * tb.W2[q * N + x]);
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = p1[q][x];
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[j * N + q], g[j], s);
      p1[q][x] = s;
    }
  }
  // values and partial result to Z (qz = t, [qy][qx])
  double p3[N][N];
  y_to_z<N, typename L::YZ>(p2, p3, buf, tt, lane_ok);  // p3 = uq (Z)
  y_to_z<N, typename L::YZ>(p1, p2, buf, tt, lane_ok);  // p2 = partial result (Z)
  const double fy = wt * tb.kin[1];
#pragma unroll
  for (int x = 0; x < N; ++x) {
    double g[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[q * N + j], p3[j][x], s);
      g[q] = s * (fy * tb.W2[q * N + x]);
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s = p2[q][x];
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(tb.D[j * N + q], g[j], s);
      p2[q][x] = s;
    }
  }
  // back to the nodes: y, x in Z, then z in X
  contract_slow<N, true>(p2, p1, tb.S);    // S^T along y
  contract_fast<N, true>(p1, p2, tb.S);    // S^T along x
  z_to_x<N, typename L::ZX>(p2, p1, buf, tt, lane_ok);  // X: x = t, [qz][y]
  contract_slow<N, true>(p1, out, tb.S);   // S^T along z -> out[z][y]
  if (!std::is_same<MASS, NoMass>::value) {
    hout.template operator()<N, L>(out, buf, tt, lane_ok, tb);
    mass.template operator()<N, L>(p3, buf, tt, lane_ok, tb);
  }
}

// The mass operator on values at the quadrature points in Z layout (qz = t,
// [qy][qx]): w3 * uq, back to the nodes (S^T along y and x in Z, transpose,
// z in X); result in X layout (x = t, [z][y]) in m.
template <int N, class L>
__device__ __forceinline__ void mass_back_lean(double (&m)[N][N], const double* __restrict__ w3,
                                               double* buf, int tt, bool lane_ok,
                                               const CellTables& tb) {
  double v1[N][N];
#pragma unroll
  for (int y = 0; y < N; ++y)
#pragma unroll
    for (int x = 0; x < N; ++x) m[y][x] *= __ldg(w3 + tt * N * N + y * N + x);
  contract_slow<N, true>(m, v1, tb.S);    // S^T along y
  contract_fast<N, true>(v1, m, tb.S);    // S^T along x
  z_to_x<N, typename L::ZX>(m, v1, buf, tt, lane_ok);  // X: x = t
  contract_slow<N, true>(v1, m, tb.S);    // S^T along z
}

// The mass operator on values at the quadrature points in B layout (qy = t):
// w3 * uq, back to the nodes (S^T along z and x in B, transpose, y in A);
// result in A layout (z = t, [y][x]) in m.
template <int N, class L>
__device__ __forceinline__ void mass_back_plane(double (&m)[N][N], const double* __restrict__ w3,
                                                double* buf, int tt, bool lane_ok,
                                                const CellTables& tb) {
  double v1[N][N];
#pragma unroll
  for (int z = 0; z < N; ++z)
#pragma unroll
    for (int x = 0; x < N; ++x) m[z][x] *= __ldg(w3 + z * N * N + tt * N + x);
  contract_slow<N, true>(m, v1, tb.S);    // S^T along z
  contract_fast<N, true>(v1, m, tb.S);    // S^T along x
  b_to_a<N, L>(m, v1, buf, tt, lane_ok);  // A: z = t
  contract_slow<N, true>(v1, m, tb.S);    // S^T along y
}

}  // namespace bmv
