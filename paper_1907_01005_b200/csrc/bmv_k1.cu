// K1: the sum-factorised cell operator on slab storage (slabs.py) -- the cell
// loop of CellOperator.apply (reference bcsrmv/matfree.py:458-527) and the
// cell integral cell_integrals_sumfac (matfree.py:288-367), collocation form
// (DESIGN.md 4), over the active (cell, column) pairs.
//
// Addressing.  A cell DoF d lies in one of the cell's groups g (distinct
// local block rows, first-occurrence order) at row r of that block row.
// In slab storage the value of column alpha there is at
//     slab_off[g] + r * K[g] + slot_g(alpha),
// so the offset splits into a per-cell part and a per-pair part:
//   * per cell and DoF a CODE: g, r * K_src[g], r * K_dst[g]
//     (32-bit: g:5 | rKx:13 | rKh:14; wide: {g:5 | rKx:27, rKh:32}),
//   * per pair and group a table entry {slab_off_src[g] + slot (-1: the
//     column is not stored there -> 0), slab_off_dst[g] + slot}.
// X offset = gtab[g].x + rKx, HX offset = gtab[g].y + rKh.  The metadata is
// therefore ~4 B per cell DoF + 8 B per (pair, group) instead of an offset
// per (pair, DoF).
//
// Per pair, lane t = 0 issues cp.async.bulk copies (TMA) of the cell's code
// row, the pair's group table and the cell's coefficient row (w3 V) into the
// warp's shared memory (one mbarrier per warp).  The code row lands in the
// pair's transpose tile (dead until the first transpose); once the
// coefficient row has been consumed the code row is copied again into its
// place for the scatter (second mbarrier phase, lands during the remaining
// contractions).
//
// n = 4, 5: n threads per pair, thread t holds plane z = t (bmv_sumfac.cuh,
// 12 contractions, 4 transposes through the pair tile).  n = 2, 3: one
// thread per pair, whole n^3 tensor in registers (bmv_cellop_pair.cuh).
// Scatter-add: fp64 RED (atomicAdd) into the zeroed destination.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "bmv.h"
#include "bmv_cellop_pair.cuh"
#include "bmv_common.cuh"
#include "bmv_sumfac.cuh"
#include "bmv_tma.cuh"

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st);

namespace {

constexpr int kWarps = 4;  // warps per CTA

struct K1Args {
  const int4* __restrict__ desc;       // {cell, gtab offset (16-byte units), ngp, 0}
  const uint32_t* __restrict__ codes;  // code rows, code_stride words per cell
  const int2* __restrict__ gtab;       // {src offset | -1, dst offset}
  int code_stride;                     // uint32 words per code row (multiple of 4)
  int gbytes;                          // group-table bytes reserved per pair (16 | it)
  const double* __restrict__ coef;
  int coef_cell;  // 1: row per cell (stride q3p), 0: one row
  int64_t n_pairs;
  const double* __restrict__ x;
  double* __restrict__ hx;
  double* __restrict__ mx;             // fused mass output (DUAL), same layout as hx
  const double* __restrict__ mcoef;    // mass coefficient row (w3, q3p doubles)
};

template <bool WIDE>
struct Code {
  int g;
  int rx, rh;
};
template <bool WIDE>
__device__ __forceinline__ Code<WIDE> decode(const uint32_t* row, int d) {
  Code<WIDE> c;
  if (WIDE) {
    const uint2 w = reinterpret_cast<const uint2*>(row)[d];
    c.g = (int)(w.x >> 27);
    c.rx = (int)(w.x & 0x7ffffffu);
    c.rh = (int)w.y;
  } else {
    const uint32_t w = row[d];
    c.g = (int)(w >> 27);
    c.rx = (int)((w >> 14) & 0x1fffu);
    c.rh = (int)(w & 0x3fffu);
  }
  return c;
}

// Per nodes-per-axis N (plane kernel): P pairs per warp; per pair a tile
// region (transposes; the code row for the gather at its first 16-byte
// boundary), a coefficient region (CS doubles, >= q3p; later the code row
// for the scatter) and a group-table region.
template <int N>
struct K1Shape {
  static constexpr int P = 32 / N;
  static constexpr int N3 = N * N * N;
  static constexpr int Q3P = (N3 + 1) / 2 * 2;
  static constexpr int CS = N == 5 ? 134 : (N == 4 ? 66 : 28);
  static constexpr int MINB = N == 5 ? 3 : 4;
  static constexpr int tile_bytes = (P * Tile<N>::TILE * 8 + 15) / 16 * 16;
  static constexpr int coef_bytes = P * CS * 8;
};

template <int N>
__host__ __device__ constexpr int k1_warp_bytes(int gbytes) {
  return K1Shape<N>::tile_bytes + K1Shape<N>::coef_bytes + K1Shape<N>::P * gbytes;
}

__device__ __forceinline__ void proxy_fence() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Scatter-add of a plane result (A layout, z = t) through the code row.
template <int N, bool WIDE>
struct PlaneScatter {
  double* dst;
  const uint32_t* codes;
  const int2* gt;
  int t;
  bool ok;
  template <int NN, class L>
  __device__ __forceinline__ void operator()(double (&v)[NN][NN], double*, int, bool,
                                             const CellTables&) const {
    if (!ok) return;
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        const Code<WIDE> c = decode<WIDE>(codes, t * N * N + y * N + x);
        atomicAdd(dst + (int64_t)gt[c.g].y + c.rh, v[y][x]);
      }
  }
};
template <int N, bool WIDE>
struct MassScatter {
  PlaneScatter<N, WIDE> sc;
  const double* w3;
  template <int NN, class L>
  __device__ __forceinline__ void operator()(double (&uqB)[NN][NN], double* buf, int tt,
                                             bool lane_ok, const CellTables& tb) const {
    mass_back_plane<NN, L>(uqB, w3, buf, tt, lane_ok, tb);
    sc.template operator()<NN, L>(uqB, buf, tt, lane_ok, tb);
  }
};
// Re-stage the code row into the (consumed) coefficient region.
struct Restage {
  uint32_t* dst;
  const uint32_t* src;
  unsigned bytes;
  uint64_t* bar;
  bool issuer;
  // warp-collective: one arrival (lane 0) announcing every issuer's bytes
  __device__ __forceinline__ void operator()() const {
    __syncwarp();
    const unsigned total = __reduce_add_sync(~0u, issuer ? bytes : 0u);
    if ((threadIdx.x & 31) == 0) mbar_expect_tx(bar, total);
    __syncwarp();
    if (issuer) {
      proxy_fence();
      bulk_g2s(dst, src, bytes, bar);
    }
  }
};

// Wait for the re-staged code row, then scatter.
template <class H>
struct WaitThen {
  H h;
  uint64_t* bar;
  template <int NN, class L>
  __device__ __forceinline__ void operator()(double (&v)[NN][NN], double* b, int x, bool o,
                                             const CellTables& tbl) const {
    mbar_wait(bar, 1);
    h.template operator()<NN, L>(v, b, x, o, tbl);
  }
};

// MODE 0: H (kinetic + optional coefficient), 1: coefficient only (mass),
// 2: fused H and M (DUAL).
template <int N, bool COEF, int MODE, bool WIDE>
__global__ void __launch_bounds__(kWarps * 32, K1Shape<N>::MINB)
    k1_plane_kernel(const K1Args a, const __grid_constant__ CellTables tb) {
  using S = K1Shape<N>;
  constexpr int P = S::P, N2 = N * N, TILE = Tile<N>::TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kWarps];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int sub = lid / N;
  const int t = lid - sub * N;
  const bool lane_ok = sub < P;
  const int tt = lane_ok ? t : 0;
  const int64_t pair = ((int64_t)blockIdx.x * kWarps + warp) * P + sub;
  const bool ok = lane_ok && pair < a.n_pairs;

  // the 32 - N * P idle lanes use pair 0's regions (they only read them; the
  // coefficient term is read unguarded, and past the last pair's regions lies
  // only the small group table, then the end of the CTA's shared memory)
  const int sp = lane_ok ? sub : 0;
  unsigned char* wbase = smem + warp * k1_warp_bytes<N>(a.gbytes);
  double* buf = reinterpret_cast<double*>(wbase) + sp * TILE;
  uint32_t* code_g = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(buf) + 15) & ~uintptr_t(15));
  double* cs = reinterpret_cast<double*>(wbase + S::tile_bytes) + sp * S::CS;
  uint32_t* code_s = reinterpret_cast<uint32_t*>(cs);
  const int2* gt = reinterpret_cast<const int2*>(wbase + S::tile_bytes + S::coef_bytes +
                                                 sp * a.gbytes);
  if (lid == 0) mbar_init(&bar[warp], 1);
  __syncwarp();

  int4 d = make_int4(0, 0, 0, 0);
  if (ok) d = __ldg(a.desc + pair);
  const int cell = d.x;
  const bool issuer = ok && t == 0;
  const unsigned cbytes = COEF ? S::Q3P * 8u : 0u;
  const unsigned kbytes = (unsigned)a.code_stride * 4u;
  const unsigned gb = (unsigned)d.z * 8u;
  const uint32_t* gcode = a.codes + (int64_t)cell * a.code_stride;
  const unsigned my_bytes = issuer ? cbytes + kbytes + gb : 0u;
  const unsigned total = __reduce_add_sync(~0u, my_bytes);
  if (lid == 0) mbar_expect_tx(&bar[warp], total);
  __syncwarp();
  if (issuer) {
    if (cbytes)
      bulk_g2s(cs, a.coef + (a.coef_cell ? (int64_t)cell * S::Q3P : 0), cbytes, &bar[warp]);
    bulk_g2s(code_g, gcode, kbytes, &bar[warp]);
    if (gb) bulk_g2s(const_cast<int2*>(gt), a.gtab + (int64_t)d.y, gb, &bar[warp]);
  }
  mbar_wait(&bar[warp], 0);

  // gather X (A layout, z = t)
  double u[N][N];
#pragma unroll
  for (int y = 0; y < N; ++y) {
#pragma unroll
    for (int x = 0; x < N; ++x) {
      double v = 0.0;
      if (ok) {
        const Code<WIDE> c = decode<WIDE>(code_g, t * N2 + y * N + x);
        const int xo = gt[c.g].x;
        if (xo >= 0) v = __ldg(a.x + (int64_t)xo + c.rx);
      }
      u[y][x] = v;
    }
  }
  const Restage rs{code_s, gcode, kbytes, &bar[warp], issuer};
  double out[N][N];
  if (MODE == 1) {
    // coefficient only: interpolate, scale at the points, back (2 transposes)
    double v1[N][N], uqB[N][N];
    contract_fast<N, false>(u, v1, tb.S);
    contract_slow<N, false>(v1, out, tb.S);
    a_to_b<N>(out, v1, buf, tt, lane_ok);  // B: y = qy = t, [z][qx]
    contract_slow<N, false>(v1, uqB, tb.S);
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int x = 0; x < N; ++x) uqB[z][x] *= COEF ? cs[z * N2 + tt * N + x] : 0.0;
    rs();
    contract_slow<N, true>(uqB, v1, tb.S);  // S^T along z
    contract_fast<N, true>(v1, uqB, tb.S);  // S^T along x
    b_to_a<N>(uqB, v1, buf, tt, lane_ok);   // A: z = t
    contract_slow<N, true>(v1, out, tb.S);  // S^T along y
  } else if (MODE == 2) {
    const PlaneScatter<N, WIDE> hsc{a.hx, code_s, gt, t, ok};
    const MassScatter<N, WIDE> msc{PlaneScatter<N, WIDE>{a.mx, code_s, gt, t, ok}, a.mcoef};
    // the scatter hooks run after the last transpose: wait for the code row first
    const WaitThen<PlaneScatter<N, WIDE>> hw{hsc, &bar[warp]};
    sumfac_h_plane<N, COEF, 1, Tile<N>, const double*, MassScatter<N, WIDE>,
                   WaitThen<PlaneScatter<N, WIDE>>, Restage>(
        u, out, buf, tt, lane_ok, cs + tt * N2, tb, msc, hw, rs);
    return;
  } else {
    sumfac_h_plane<N, COEF, 1, Tile<N>, const double*, NoMass, NoMass, Restage>(
        u, out, buf, tt, lane_ok, cs + tt * N2, tb, NoMass(), NoMass(), rs);
  }
  mbar_wait(&bar[warp], 1);
  if (ok) {
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        const Code<WIDE> c = decode<WIDE>(code_s, t * N2 + y * N + x);
        atomicAdd(a.hx + (int64_t)gt[c.g].y + c.rh, out[y][x]);
      }
  }
}

// ---------------------------------------------------------------------------
// One thread per pair (n <= 3).  Per lane: code row, group table and
// coefficient row at pitches of an odd number of 16-byte units.
template <int N>
struct K1PairShape {
  static constexpr int N3 = N * N * N;
  static constexpr int Q3P = (N3 + 1) / 2 * 2;
  static constexpr int CU = ((Q3P / 2) | 1);  // coefficient pitch (16-byte units)
};

__host__ __device__ inline int odd_units(int bytes) { return ((bytes + 15) / 16) | 1; }

template <int N, bool COEF, int MODE, bool WIDE>
__global__ void __launch_bounds__(kWarps * 32, 3)
    k1_pair_kernel(const K1Args a, const __grid_constant__ CellTables tb) {
  using PS = K1PairShape<N>;
  constexpr int N2 = N * N, N3 = N2 * N;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kWarps];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int64_t pair = ((int64_t)blockIdx.x * kWarps + warp) * 32 + lid;
  const bool ok = pair < a.n_pairs;
  const int ou = odd_units(a.code_stride * 4), gu = odd_units(a.gbytes);
  const int lane_bytes = 16 * (ou + gu + PS::CU);
  unsigned char* wbase = smem + warp * 32 * lane_bytes;
  const uint32_t* crow = reinterpret_cast<const uint32_t*>(wbase + lid * 16 * ou);
  const int2* gt = reinterpret_cast<const int2*>(wbase + 32 * 16 * ou + lid * 16 * gu);
  const double* cf = reinterpret_cast<const double*>(wbase + 32 * 16 * (ou + gu) +
                                                     lid * 16 * PS::CU);
  if (lid == 0) mbar_init(&bar[warp], 1);
  __syncwarp();
  int4 d = make_int4(0, 0, 0, 0);
  if (ok) d = __ldg(a.desc + pair);
  const int cell = d.x;
  const unsigned cbytes = COEF ? PS::Q3P * 8u : 0u;
  const unsigned kbytes = (unsigned)a.code_stride * 4u;
  const unsigned gb = (unsigned)d.z * 8u;
  const unsigned total = __reduce_add_sync(~0u, ok ? cbytes + kbytes + gb : 0u);
  if (lid == 0) mbar_expect_tx(&bar[warp], total);
  __syncwarp();
  if (ok) {
    if (COEF)
      bulk_g2s(const_cast<double*>(cf), a.coef + (a.coef_cell ? (int64_t)cell * PS::Q3P : 0),
               cbytes, &bar[warp]);
    bulk_g2s(const_cast<uint32_t*>(crow), a.codes + (int64_t)cell * a.code_stride, kbytes,
             &bar[warp]);
    if (gb) bulk_g2s(const_cast<int2*>(gt), a.gtab + (int64_t)d.y, gb, &bar[warp]);
  }
  mbar_wait(&bar[warp], 0);
  double v[N][N][N];
#pragma unroll
  for (int k = 0; k < N3; ++k) {
    double xv = 0.0;
    if (ok) {
      const Code<WIDE> c = decode<WIDE>(crow, k);
      const int xo = gt[c.g].x;
      if (xo >= 0) xv = __ldg(a.x + (int64_t)xo + c.rx);
    }
    v[k / N2][(k / N) % N][k % N] = xv;
  }
  // values at the Gauss points
  contract3<N, 0, false>(v, tb.S);
  contract3<N, 1, false>(v, tb.S);
  contract3<N, 2, false>(v, tb.S);
  double acc[N][N][N];
  double mac[N][N][N];
#pragma unroll
  for (int k = 0; k < N3; ++k) {
    const double c = COEF ? cf[k] : 0.0;
    acc[k / N2][(k / N) % N][k % N] = c * v[k / N2][(k / N) % N][k % N];
    if (MODE == 2) mac[k / N2][(k / N) % N][k % N] = __ldg(a.mcoef + k) * v[k / N2][(k / N) % N][k % N];
  }
  if (MODE != 1) {
    grad3<N, 0>(v, acc, tb);
    grad3<N, 1>(v, acc, tb);
    grad3<N, 2>(v, acc, tb);
  }
  // back to the nodes
  contract3<N, 0, true>(acc, tb.S);
  contract3<N, 1, true>(acc, tb.S);
  contract3<N, 2, true>(acc, tb.S);
  if (MODE == 2) {
    contract3<N, 0, true>(mac, tb.S);
    contract3<N, 1, true>(mac, tb.S);
    contract3<N, 2, true>(mac, tb.S);
  }
  if (ok) {
#pragma unroll
    for (int k = 0; k < N3; ++k) {
      const Code<WIDE> c = decode<WIDE>(crow, k);
      const int64_t o = (int64_t)gt[c.g].y + c.rh;
      atomicAdd(a.hx + o, acc[k / N2][(k / N) % N][k % N]);
      if (MODE == 2) atomicAdd(a.mx + o, mac[k / N2][(k / N) % N][k % N]);
    }
  }
}

}  // namespace

struct K1Plan {
  int n = 0;
  int wide = 0;
  int64_t n_pairs = 0;
  int code_stride = 0;
  int gbytes = 0;
  int4* desc = nullptr;
  uint32_t* codes = nullptr;
  int2* gtab = nullptr;
  CellTables tables{};
};

namespace {

template <int N, bool COEF, int MODE, bool WIDE>
int launch_k1(const K1Plan* p, const K1Args& args, cudaStream_t st) {
  if constexpr (N <= 3) {
    constexpr int NP = N;
    auto kern = k1_pair_kernel<NP, COEF, MODE, WIDE>;
    const int lane_bytes =
        16 * (odd_units(p->code_stride * 4) + odd_units(p->gbytes) + K1PairShape<NP>::CU);
    const int smem = kWarps * 32 * lane_bytes;
    BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t per = (int64_t)kWarps * 32;
    kern<<<(unsigned)((p->n_pairs + per - 1) / per), kWarps * 32, smem, st>>>(args, p->tables);
  } else {
    constexpr int NN = N;
    auto kern = k1_plane_kernel<NN, COEF, MODE, WIDE>;
    const int smem = kWarps * k1_warp_bytes<NN>(p->gbytes);
    BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t per = (int64_t)kWarps * K1Shape<NN>::P;
    kern<<<(unsigned)((p->n_pairs + per - 1) / per), kWarps * 32, smem, st>>>(args, p->tables);
  }
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N>
int dispatch_n(const K1Plan* p, const K1Args& args, bool coef, int mode, cudaStream_t st) {
  if (p->wide) {
    if (mode == 0) return coef ? launch_k1<N, true, 0, true>(p, args, st) : launch_k1<N, false, 0, true>(p, args, st);
    if (mode == 1) return launch_k1<N, true, 1, true>(p, args, st);
    return coef ? launch_k1<N, true, 2, true>(p, args, st) : launch_k1<N, false, 2, true>(p, args, st);
  }
  if (mode == 0) return coef ? launch_k1<N, true, 0, false>(p, args, st) : launch_k1<N, false, 0, false>(p, args, st);
  if (mode == 1) return launch_k1<N, true, 1, false>(p, args, st);
  return coef ? launch_k1<N, true, 2, false>(p, args, st) : launch_k1<N, false, 2, false>(p, args, st);
}

int dispatch(const K1Plan* p, const K1Args& args, bool coef, int mode, cudaStream_t st) {
  switch (p->n) {
    case 2: return dispatch_n<2>(p, args, coef, mode, st);
    case 3: return dispatch_n<3>(p, args, coef, mode, st);
    case 4: return dispatch_n<4>(p, args, coef, mode, st);
    case 5: return dispatch_n<5>(p, args, coef, mode, st);
    default:
      set_error("K1: unsupported nodes per axis %d", p->n);
      return BMV_ERR_INVALID;
  }
}

}  // namespace
}  // namespace bmv

struct bmv_cellop : bmv::K1Plan {};

extern "C" {

int bmv_cellop_create(const bmv_cellop_desc* d, bmv_cellop** out) {
  using namespace bmv;
  *out = nullptr;
  if (!d || d->n < 2 || d->n > BMV_MAX_NODES || d->n_pairs < 0 || d->n_cells < 0 ||
      d->code_stride <= 0 || (d->code_stride & 3) || d->max_groups < 0 || d->max_groups > 32) {
    set_error("bmv_cellop_create: invalid descriptor");
    return BMV_ERR_INVALID;
  }
  const int n3 = d->n * d->n * d->n;
  if (d->code_stride < (d->wide ? 2 * n3 : n3)) {
    set_error("bmv_cellop_create: code rows too short");
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_cellop();
  p->n = d->n;
  p->wide = d->wide ? 1 : 0;
  p->n_pairs = d->n_pairs;
  p->code_stride = d->code_stride;
  p->gbytes = std::max(16, (d->max_groups * 8 + 15) / 16 * 16);
  const int n = d->n;
  CellTables& tb = p->tables;
  for (int i = 0; i < n * n; ++i) {
    tb.S[i] = d->S[i];
    tb.D[i] = d->Dco[i];
  }
  for (int i = 0; i < n; ++i) {
    tb.w[i] = d->w[i];
    for (int j = 0; j < n; ++j) tb.W2[i * n + j] = d->w[i] * d->w[j];
  }
  for (int k = 0; k < 3; ++k) tb.kin[k] = d->kin[k];
  std::vector<int4> desc((size_t)d->n_pairs);
  for (int64_t q = 0; q < d->n_pairs; ++q) {
    const int64_t go = d->pair_gtab[q];
    if ((go & 3) || d->pair_ngp[q] > d->max_groups || go / 4 > INT32_MAX) {
      delete p;
      set_error("bmv_cellop_create: bad group table of pair %lld", (long long)q);
      return BMV_ERR_INVALID;
    }
    desc[(size_t)q] = make_int4(d->pair_cell[q], (int)(go / 2), d->pair_ngp[q], 0);
  }
  int rc = upload(desc.data(), (int64_t)desc.size(), &p->desc);
  if (rc == BMV_OK)
    rc = upload(d->codes, (int64_t)d->n_cells * d->code_stride, &p->codes);
  if (rc == BMV_OK)
    rc = upload(reinterpret_cast<const int2*>(d->gtab), d->gtab_len / 2, &p->gtab);
  if (rc != BMV_OK) {
    bmv_cellop_destroy(p);
    return rc;
  }
  *out = p;
  return BMV_OK;
}

int bmv_cellop_destroy(bmv_cellop* p) {
  if (!p) return BMV_OK;
  bmv::release(p->desc);
  bmv::release(p->codes);
  bmv::release(p->gtab);
  delete p;
  return BMV_OK;
}

namespace {

// mode 0: H, 1: coefficient only (mass), 2: fused H + M; pairs [p0, p1)
int run_pairs(const bmv_cellop* p, int mode, const double* coef, int64_t coef_stride,
              const double* mcoef, const double* x, double* hx, double* mx, int64_t p0, int64_t p1,
              cudaStream_t st) {
  using namespace bmv;
  const int q3 = p->n * p->n * p->n, q3p = q3 + (q3 & 1);
  if (coef && coef_stride != 0 && coef_stride != q3p) {
    set_error("K1: coefficient rows must have stride 0 or %d", q3p);
    return BMV_ERR_INVALID;
  }
  if (p0 < 0 || p1 > p->n_pairs || p0 > p1) {
    set_error("K1: pair range [%lld, %lld) outside [0, %lld)", (long long)p0, (long long)p1,
              (long long)p->n_pairs);
    return BMV_ERR_INVALID;
  }
  if (p1 == p0) return BMV_OK;
  K1Args args{p->desc + p0, p->codes, p->gtab, p->code_stride, p->gbytes, coef,
              coef_stride != 0 ? 1 : 0, p1 - p0, x, hx, mx, mcoef};
  return dispatch(p, args, coef != nullptr, mode, st);
}

}  // namespace

int bmv_cellop_apply(bmv_cellop* p, int32_t kinetic, const double* coef, int64_t coef_stride,
                     const double* x, double* hx, int64_t zero_len, void* stream) {
  using namespace bmv;
  if (!p) {
    set_error("bmv_cellop_apply: null plan");
    return BMV_ERR_INVALID;
  }
  if (!kinetic && !coef) {
    set_error("operator without kinetic and coefficient terms");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  const int rc = zero_async(hx, zero_len, st);
  if (rc != BMV_OK) return rc;
  return run_pairs(p, kinetic ? 0 : 1, coef, coef_stride, nullptr, x, hx, nullptr, 0, p->n_pairs,
                   st);
}

int bmv_cellop_apply_pairs(bmv_cellop* p, int32_t kinetic, const double* coef,
                           int64_t coef_stride, const double* x, double* hx, int64_t pair_begin,
                           int64_t pair_end, void* stream) {
  using namespace bmv;
  if (!p || (!kinetic && !coef)) {
    set_error("bmv_cellop_apply_pairs: null plan or empty operator");
    return BMV_ERR_INVALID;
  }
  return run_pairs(p, kinetic ? 0 : 1, coef, coef_stride, nullptr, x, hx, nullptr, pair_begin,
                   pair_end, as_stream(stream));
}

int bmv_cellop_apply_hm(bmv_cellop* p, const double* coef, int64_t coef_stride,
                        const double* mass_coef, const double* x, double* hx, double* mx,
                        int64_t zero_len, void* stream) {
  using namespace bmv;
  if (!p || !mass_coef) {
    set_error("bmv_cellop_apply_hm: null plan or mass coefficient");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  int rc = zero_async(hx, zero_len, st);
  if (rc == BMV_OK) rc = zero_async(mx, zero_len, st);
  if (rc != BMV_OK) return rc;
  return run_pairs(p, 2, coef, coef_stride, mass_coef, x, hx, mx, 0, p->n_pairs, st);
}

int bmv_cellop_apply_hm_pairs(bmv_cellop* p, const double* coef, int64_t coef_stride,
                              const double* mass_coef, const double* x, double* hx, double* mx,
                              int64_t pair_begin, int64_t pair_end, void* stream) {
  using namespace bmv;
  if (!p || !mass_coef) {
    set_error("bmv_cellop_apply_hm_pairs: null plan or mass coefficient");
    return BMV_ERR_INVALID;
  }
  return run_pairs(p, 2, coef, coef_stride, mass_coef, x, hx, mx, pair_begin, pair_end,
                   as_stream(stream));
}

int bmv_cellop_launches(const bmv_cellop* p, int32_t* out) {
  *out = (p && p->n_pairs > 0) ? 1 : 0;
  return BMV_OK;
}

}  // extern "C"
