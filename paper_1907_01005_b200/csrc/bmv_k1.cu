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
// n = 4, 5 (plane kernel): n threads per pair, thread t holds plane z = t
// (bmv_sumfac.cuh, 12 contractions, 4 transposes through the pair tile); a
// warp works on a BATCH of up to 32 / n consecutive pairs that lie in at
// most two cells (the host cuts the batches; 97-99 % of the lanes are used
// at the BASELINE configs).  The kernel is persistent: every warp loops
// over batches and keeps two metadata stages in shared memory -- the code
// and coefficient rows of the batch's (<= 2) cells, shared by its pairs,
// and the pairs' group tables, fetched by cp.async.bulk (TMA) one batch
// ahead on one mbarrier per stage -- so neither the descriptor nor the
// metadata latency is exposed, and the gather is branch-free (an absent
// column reads a valid address and is masked).
// n = 2, 3: one thread per pair, whole n^3 tensor in registers
// (bmv_cellop_pair.cuh), per-pair metadata copies.
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

// plane kernel, n = 5: warps per CTA, one CTA per SM.  Registers are per SM
// sub-partition (16384 each): 12 warps leave 168 per thread, 8 warps 255.
#ifndef BMV_K1_WARPS5
#define BMV_K1_WARPS5 8
#endif
#ifndef BMV_K1_WARPS4
#define BMV_K1_WARPS4 12
#endif
constexpr int kWarps = 4;  // warps per CTA

// A batch of the plane kernel: pairs [first_pair, first_pair + np), the first
// nA in cell_a, the rest in cell_b; their group tables are consecutive.
struct __align__(16) Batch {
  int32_t first_pair;
  int32_t cell_a, cell_b;
  int32_t info;      // nA | np << 8 | groups per pair of cell_a << 16 | of cell_b << 24
  int32_t gt16;      // first group-table entry of the batch, 16-byte units
  int32_t gt_bytes;  // bytes of the batch's group tables (multiple of 16)
  int32_t pad[2];
};

struct K1Args {
  const struct PairBatch* __restrict__ pair_batches;  // pair kernel (n <= 3)
  const Batch* __restrict__ batches;   // plane kernel
  int64_t b0, b1;                      // batch range of this launch
  const uint32_t* __restrict__ codes;  // code rows, code_stride words per cell
  const int2* __restrict__ gtab;       // {src offset | -1, dst offset}
  int code_stride;                     // uint32 words per code row (multiple of 4)
  int gbytes;                          // group-table bytes reserved per pair (16 | it)
  const double* __restrict__ coef;
  int coef_cell;  // 1: row per cell (stride q3p), 0: one row
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

// Per nodes-per-axis N (plane kernel): P pairs per warp.  Per warp: the
// transpose tiles of its pairs and two metadata stages
//   [info (16 B) | coef row cell a | coef row cell b | code row a | code row b | group tables].
template <int N>
struct K1Shape {
  static constexpr int P = 32 / N;
  static constexpr int N3 = N * N * N;
  static constexpr int Q3P = (N3 + 1) / 2 * 2;
  static constexpr int CB = Q3P * 8;  // bytes of a coefficient row (multiple of 16)
  static constexpr int WARPS = N == 5 ? BMV_K1_WARPS5 : BMV_K1_WARPS4;  // warps per CTA (1 CTA / SM)
  // prefetch the next batch's X values into registers (needs the registers
  // that at most 2 warps per sub-partition at n = 5, 3 at n = 4, leave)
  static constexpr bool PREF = N == 5 ? WARPS <= 8 : WARPS <= 12;
  static constexpr int STAGES = PREF ? 3 : 2;
  // registers per thread: n = 5 what the warps of one CTA per SM leave in a
  // sub-partition; n = 4: 4 CTAs x 4 warps x 128
  static constexpr int REGS = 16384 / ((WARPS + 3) / 4 * 32) / 8 * 8 > 255
                                  ? 255
                                  : 16384 / ((WARPS + 3) / 4 * 32) / 8 * 8;
  static constexpr int tile_bytes = (P * Tile3<N>::TILE * 8 + 15) / 16 * 16;
};

template <int N>
__host__ __device__ constexpr int k1_stage_bytes(int code_stride, int gbytes) {
  return (16 + 2 * K1Shape<N>::CB + 2 * code_stride * 4 + K1Shape<N>::P * gbytes + 127) / 128 * 128;
}
template <int N>
__host__ __device__ constexpr int k1_warp_bytes(int code_stride, int gbytes) {
  return (K1Shape<N>::tile_bytes + 127) / 128 * 128 +
         K1Shape<N>::STAGES * k1_stage_bytes<N>(code_stride, gbytes);
}

__device__ __forceinline__ void proxy_fence() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Scatter-add of a plane result through the code row.  LAY 0: X layout
// (thread t holds x = t, v[z][y]); LAY 2: Z layout (z = t, v[y][x]).
template <int N, bool WIDE, int LAY>
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
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const int d = LAY == 0 ? i * N * N + j * N + t : t * N * N + i * N + j;
        const Code<WIDE> c = decode<WIDE>(codes, d);
        atomicAdd(dst + (int64_t)gt[c.g].y + c.rh, v[i][j]);
      }
  }
};
template <int N, bool WIDE>
struct MassScatter {
  PlaneScatter<N, WIDE, 0> sc;
  const double* w3;
  template <int NN, class L>
  __device__ __forceinline__ void operator()(double (&uqZ)[NN][NN], double* buf, int tt,
                                             bool lane_ok, const CellTables& tb) const {
    mass_back_lean<NN, L>(uqZ, w3, buf, tt, lane_ok, tb);
    sc.template operator()<NN, L>(uqZ, buf, tt, lane_ok, tb);
  }
};

// MODE 0: H (kinetic + optional coefficient), 1: coefficient only (mass),
// 2: fused H and M (DUAL).
template <int N, bool COEF, int MODE, bool WIDE>
__global__ void __launch_bounds__(K1Shape<N>::WARPS * 32) __maxnreg__(K1Shape<N>::REGS)
    k1_plane_kernel(const K1Args a, const __grid_constant__ CellTables tb) {
  using S = K1Shape<N>;
  constexpr int P = S::P, N2 = N * N, TILE = Tile3<N>::TILE, kWarps = S::WARPS;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NST = S::STAGES;
  __shared__ __align__(8) uint64_t bar[kWarps][NST];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  // lane -> (pair, plane): the pairs of a batch are split over the two
  // half-warps (n = 5: pairs 0-2 in lanes 0-14, 3-5 in lanes 16-30, lanes 15
  // and 31 idle), which makes the transposes bank-conflict free (Tile3)
  constexpr int PH = P / 2;
  const int hl = lid & 15;
  const int sub = (lid >> 4) * PH + hl / N;
  const int t = hl % N;
  const bool lane_ok = hl < PH * N;
  const int tt = lane_ok ? t : 0;

  const int kb = a.code_stride * 4;  // bytes of a code row
  const int stage_bytes = k1_stage_bytes<N>(a.code_stride, a.gbytes);
  unsigned char* wbase = smem + warp * k1_warp_bytes<N>(a.code_stride, a.gbytes);
  // the 32 - N * P idle lanes share pair 0's tile (they only read it)
  double* buf = reinterpret_cast<double*>(wbase) + (lane_ok ? sub : 0) * TILE;
  unsigned char* stage0 = wbase + (S::tile_bytes + 127) / 128 * 128;
  if (lid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bar[warp][s], 1);
  }
  __syncwarp();

  const int nw = (int)gridDim.x * kWarps;
  const int nb = (int)(a.b1 - a.b0);
  int b = (int)blockIdx.x * kWarps + warp;
  // lane 0: fetch the metadata of batch bb into stage s (one mbarrier phase);
  // the batch's `info` word goes into the stage header for the other lanes
  auto issue = [&](int s, int bb) {
    if (lid == 0) {
      const int4* dp = reinterpret_cast<const int4*>(a.batches + a.b0 + bb);
      const int4 d0 = __ldg(dp);
      const int2 d1 = __ldg(reinterpret_cast<const int2*>(dp + 1));
      unsigned char* st = stage0 + s * stage_bytes;
      const int na = d0.w & 255, np = (d0.w >> 8) & 255;
      const bool two = np > na;
      unsigned total = (unsigned)kb * (two ? 2u : 1u) + (unsigned)d1.y;
      if (COEF) total += (unsigned)S::CB * (two ? 2u : 1u);
      *reinterpret_cast<int*>(st) = d0.w;
      proxy_fence();  // the stage was read (generic proxy) by an earlier batch
      mbar_expect_tx(&bar[warp][s], total);
      unsigned char* body = st + 16;
      if (COEF) {
        bulk_g2s(body, a.coef + (a.coef_cell ? (int64_t)d0.y * S::Q3P : 0), S::CB, &bar[warp][s]);
        if (two)
          bulk_g2s(body + S::CB, a.coef + (a.coef_cell ? (int64_t)d0.z * S::Q3P : 0), S::CB,
                   &bar[warp][s]);
      }
      bulk_g2s(body + 2 * S::CB, a.codes + (int64_t)d0.y * a.code_stride, kb, &bar[warp][s]);
      if (two)
        bulk_g2s(body + 2 * S::CB + kb, a.codes + (int64_t)d0.z * a.code_stride, kb,
                 &bar[warp][s]);
      if (d1.y)
        bulk_g2s(body + 2 * S::CB + 2 * kb,
                 reinterpret_cast<const char*>(a.gtab) + (int64_t)d1.x * 16, (unsigned)d1.y,
                 &bar[warp][s]);
    }
  };
  // this lane's views of a landed stage: its pair's cell rows and group table
  struct View {
    bool ok;
    const double* cs;
    const uint32_t* code;
    const int2* gt;
  };
  auto view = [&](const unsigned char* st) {
    const int info = *reinterpret_cast<const int*>(st);
    const int na = info & 255, np = (info >> 8) & 255;
    View v;
    v.ok = lane_ok && sub < np;
    const int subc = v.ok ? sub : 0;     // idle lanes follow pair 0 (masked)
    const bool in_b = subc >= na;
    v.cs = reinterpret_cast<const double*>(st + 16 + (in_b ? S::CB : 0));
    v.code = reinterpret_cast<const uint32_t*>(st + 16 + 2 * S::CB + (in_b ? kb : 0));
    v.gt = reinterpret_cast<const int2*>(st + 16 + 2 * S::CB + 2 * kb) +
           (in_b ? na * ((info >> 16) & 255) + (subc - na) * ((info >> 24) & 255)
                 : subc * ((info >> 16) & 255));
    return v;
  };
  // issue the gather of X (X layout: x = t, u[z][y]; the lanes of a pair read
  // consecutive DoFs), branch-free: a column the source does not store in a
  // group reads offset 0 of the array (valid); `present` masks it later
  auto gather = [&](const View& v, double (&u)[N][N], unsigned& present) {
    present = 0;
#pragma unroll
    for (int z = 0; z < N; ++z) {
#pragma unroll
      for (int y = 0; y < N; ++y) {
        const Code<WIDE> c = decode<WIDE>(v.code, z * N2 + y * N + t);
        const int xo = v.gt[c.g].x;
        u[z][y] = __ldg(a.x + (int64_t)max(xo, 0) + c.rx);
        if (xo >= 0) present |= 1u << (z * N + y);
      }
    }
    if (!v.ok) present = 0;
  };

  // Pipeline per warp: the metadata of batch i + STAGES - 1 is in flight
  // (TMA), and with PREF the X values of batch i + 1 are in flight (plain
  // loads into registers) while batch i is contracted.
  constexpr bool PREF = S::PREF;
#pragma unroll
  for (int k = 0; k < NST - 1; ++k)
    if (b + k * nw < nb) issue(k, b + k * nw);
  double un[N][N];
  unsigned pn = 0;
  if (PREF && b < nb) {
    mbar_wait(&bar[warp][0], 0u);
    gather(view(stage0), un, pn);
  }
  for (int it = 0; b < nb; ++it, b += nw) {
    const int s = it % NST;
    const unsigned char* st = stage0 + s * stage_bytes;
    double u[N][N];
    unsigned present;
    if (PREF) {
      present = pn;
#pragma unroll
      for (int z = 0; z < N; ++z)
#pragma unroll
        for (int y = 0; y < N; ++y) u[z][y] = ((present >> (z * N + y)) & 1u) ? un[z][y] : 0.0;
    } else {
      mbar_wait(&bar[warp][s], (unsigned)((it / NST) & 1));
      gather(view(st), u, present);
#pragma unroll
      for (int z = 0; z < N; ++z)
#pragma unroll
        for (int y = 0; y < N; ++y)
          if (!((present >> (z * N + y)) & 1u)) u[z][y] = 0.0;
    }
    // every lane is past its reads of the stage that held batch it - 1
    __syncwarp();
    if (b + (NST - 1) * nw < nb) issue((it + NST - 1) % NST, b + (NST - 1) * nw);
    if (PREF && b + nw < nb) {
      const int s1 = (it + 1) % NST;
      mbar_wait(&bar[warp][s1], (unsigned)(((it + 1) / NST) & 1));
      gather(view(stage0 + s1 * stage_bytes), un, pn);
    }
    const View cur = view(st);
    const bool ok = cur.ok;
    const double* cs = cur.cs;
    const uint32_t* code = cur.code;
    const int2* gt = cur.gt;
    double out[N][N];
    using L3 = Tile3<N>;
    if (MODE == 1) {
      // coefficient only: interpolate, scale at the points, back; result in Z layout
      double v1[N][N], uq[N][N];
      contract_fast<N, false>(u, v1, tb.S);            // y
      contract_slow<N, false>(v1, out, tb.S);          // z
      x_to_y<N, typename L3::XY>(out, v1, buf, tt, lane_ok);  // Y: qy = t, [qz][x]
      contract_fast<N, false>(v1, uq, tb.S);           // x
#pragma unroll
      for (int z = 0; z < N; ++z)
#pragma unroll
        for (int x = 0; x < N; ++x) uq[z][x] *= COEF ? cs[z * N2 + tt * N + x] : 0.0;
      contract_slow<N, true>(uq, v1, tb.S);            // S^T along z
      contract_fast<N, true>(v1, uq, tb.S);            // S^T along x
      y_to_z<N, typename L3::YZ>(uq, v1, buf, tt, lane_ok);   // Z: z = t, [qy][x]
      contract_slow<N, true>(v1, out, tb.S);           // S^T along y
      PlaneScatter<N, WIDE, 2>{a.hx, code, gt, t, ok}.template operator()<N, L3>(out, buf, tt,
                                                                                 lane_ok, tb);
    } else if (MODE == 2) {
      const PlaneScatter<N, WIDE, 0> hsc{a.hx, code, gt, t, ok};
      const MassScatter<N, WIDE> msc{PlaneScatter<N, WIDE, 0>{a.mx, code, gt, t, ok}, a.mcoef};
      sumfac_h_lean<N, COEF, L3, MassScatter<N, WIDE>, PlaneScatter<N, WIDE, 0>>(
          u, out, buf, tt, lane_ok, cs, tb, msc, hsc);
    } else {
      sumfac_h_lean<N, COEF, L3>(u, out, buf, tt, lane_ok, cs, tb);
      PlaneScatter<N, WIDE, 0>{a.hx, code, gt, t, ok}.template operator()<N, L3>(out, buf, tt,
                                                                                 lane_ok, tb);
    }
  }
}

// ---------------------------------------------------------------------------
// One thread per pair (n <= 3): the whole n^3 tensor in registers, no
// transposes.  A warp works on a batch of up to 32 consecutive pairs in at
// most kPairCells cells; the cells' code and coefficient rows are fetched
// once per batch (the lanes of a cell read them by broadcast), persistent
// warps, metadata stages and X prefetch as in the plane kernel.
constexpr int kPairCells = 8;

struct __align__(16) PairBatch {
  int32_t first_pair, np, ncells;
  int32_t gt16;      // first group-table entry of the batch, 16-byte units
  int32_t gt_bytes;  // bytes of the batch's group tables (multiple of 16)
  int32_t pad[3];
  uint8_t slot[32];  // cell slot of every lane
  struct {
    int32_t cell;   // cell id
    int32_t first;  // lane of the cell's first pair
    int32_t goff;   // group-table entry of that pair, from the batch's first
    int32_t ngp;    // entries per pair of this cell
  } c[kPairCells];
};
static_assert(sizeof(PairBatch) == 192, "PairBatch layout");

template <int N>
struct K1PairShape {
  static constexpr int N3 = N * N * N;
  static constexpr int Q3P = (N3 + 1) / 2 * 2;
  static constexpr int CB = Q3P * 8;             // bytes of a coefficient row
  // coefficient row pitch: twice an odd number of 8-byte words, so that the
  // rows of the 8 cells start in 8 different bank pairs (64-bit reads by
  // lanes in different cells) and stay 16-byte aligned for the bulk copies
  static constexpr int CP = ((Q3P / 2) % 2 == 1 ? Q3P : Q3P + 2) * 8;
#ifndef BMV_K1_PAIR_WARPS
#define BMV_K1_PAIR_WARPS 8
#endif
  static constexpr int WARPS = BMV_K1_PAIR_WARPS;  // one CTA per SM
  // prefetch the next batch's X values into registers (2 warps per
  // sub-partition leave the registers for it)
  static constexpr bool PREF = WARPS <= 8;
  static constexpr int STAGES = PREF ? 3 : 2;
};

template <int N>
__host__ __device__ constexpr int k1_pair_stage_bytes(int code_stride, int gbytes) {
  return (192 + kPairCells * K1PairShape<N>::CP + kPairCells * code_stride * 4 + 32 * gbytes + 127) /
         128 * 128;
}

template <int N, bool COEF, int MODE, bool WIDE>
__global__ void __launch_bounds__(K1PairShape<N>::WARPS * 32)
    k1_pair_kernel(const K1Args a, const __grid_constant__ CellTables tb) {
  using PS = K1PairShape<N>;
  constexpr int N2 = N * N, N3 = N2 * N, NST = PS::STAGES, kW = PS::WARPS;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kW][NST];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int kb = a.code_stride * 4;
  const int stage_bytes = k1_pair_stage_bytes<N>(a.code_stride, a.gbytes);
  unsigned char* stage0 = smem + warp * NST * stage_bytes;
  const int off_coef = 192, off_code = off_coef + kPairCells * PS::CP,
            off_gt = off_code + kPairCells * kb;
  if (lid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bar[warp][s], 1);
  }
  __syncwarp();
  const int nw = (int)gridDim.x * kW;
  const int nb = (int)(a.b1 - a.b0);
  int b = (int)blockIdx.x * kW + warp;

  // fetch the metadata of batch bb into stage s: the lanes copy the
  // descriptor (192 bytes) into the stage header, lane c < ncells issues the
  // rows of cell c, lane 0 the group tables (one mbarrier phase)
  // the descriptor of the batch to issue next is fetched one batch ahead
  // into a per-warp slot (TMA, own mbarrier): nothing waits on global memory
  __shared__ __align__(16) unsigned char dslot[kW][192];
  __shared__ __align__(8) uint64_t dbar[kW];
  int dphase = 0;
  if (lid == 0) mbar_init(&dbar[warp], 1);
  __syncwarp();
  auto fetch_desc = [&](int bb) {
    if (lid == 0 && bb < nb) {
      proxy_fence();
      mbar_expect_tx(&dbar[warp], 192u);
      bulk_g2s(dslot[warp], a.pair_batches + a.b0 + bb, 192u, &dbar[warp]);
    }
  };
  auto issue = [&](int s, int bb) {
    unsigned char* st = stage0 + s * stage_bytes;
    mbar_wait(&dbar[warp], (unsigned)(dphase & 1));
    ++dphase;
    const int4* d = reinterpret_cast<const int4*>(dslot[warp]);
    const int4 hdr = d[0];            // first_pair np ncells gt16
    const int gt_bytes = reinterpret_cast<const int*>(d)[4];
    int4 rec = make_int4(0, 0, 0, 0);
    if (lid < 12) {
      const int4 w = d[lid];
      reinterpret_cast<int4*>(st)[lid] = w;
      if (lid >= 4) rec = w;
    }
    __syncwarp();
    fetch_desc(bb + nw);  // the next batch this warp will issue
    const int ncells = hdr.z;
    proxy_fence();  // the stage was read (generic proxy) by an earlier batch
    if (lid == 0) {
      unsigned total = (unsigned)ncells * (unsigned)kb + (unsigned)gt_bytes;
      if (COEF) total += (unsigned)ncells * (unsigned)PS::CB;
      mbar_expect_tx(&bar[warp][s], total);
    }
    __syncwarp();
    if (lid >= 4 && lid - 4 < ncells) {
      const int c = lid - 4;
      if (COEF)
        bulk_g2s(st + off_coef + c * PS::CP, a.coef + (a.coef_cell ? (int64_t)rec.x * PS::Q3P : 0),
                 PS::CB, &bar[warp][s]);
      bulk_g2s(st + off_code + c * kb, a.codes + (int64_t)rec.x * a.code_stride, kb,
               &bar[warp][s]);
    }
    if (lid == 0 && gt_bytes)
      bulk_g2s(st + off_gt, reinterpret_cast<const char*>(a.gtab) + (int64_t)hdr.w * 16,
               (unsigned)gt_bytes, &bar[warp][s]);
  };
  struct View {
    bool ok;
    const double* cf;
    const uint32_t* code;
    const int2* gt;
  };
  auto view = [&](const unsigned char* st) {
    const PairBatch* d = reinterpret_cast<const PairBatch*>(st);
    View v;
    v.ok = lid < d->np;
    const int l = v.ok ? lid : 0;  // idle lanes follow pair 0 (masked)
    const int c = d->slot[l];
    v.cf = reinterpret_cast<const double*>(st + off_coef + c * PS::CP);
    v.code = reinterpret_cast<const uint32_t*>(st + off_code + c * kb);
    v.gt = reinterpret_cast<const int2*>(st + off_gt) + d->c[c].goff + (l - d->c[c].first) * d->c[c].ngp;
    return v;
  };
  auto gather = [&](const View& v, double (&u)[N3], unsigned& present) {
    present = 0;
#pragma unroll
    for (int k = 0; k < N3; ++k) {
      const Code<WIDE> c = decode<WIDE>(v.code, k);
      const int xo = v.gt[c.g].x;
      u[k] = __ldg(a.x + (int64_t)max(xo, 0) + c.rx);
      if (xo >= 0) present |= 1u << k;
    }
    if (!v.ok) present = 0;
  };

  fetch_desc(b);
#pragma unroll
  for (int k = 0; k < NST - 1; ++k)
    if (b + k * nw < nb) issue(k, b + k * nw);
  constexpr bool PREF = PS::PREF;
  double un[N3];
  unsigned pn = 0;
  if (PREF && b < nb) {
    mbar_wait(&bar[warp][0], 0u);
    gather(view(stage0), un, pn);
  }
  for (int it = 0; b < nb; ++it, b += nw) {
    const int s = it % NST;
    const unsigned char* st = stage0 + s * stage_bytes;
    if (!PREF) {
      mbar_wait(&bar[warp][s], (unsigned)((it / NST) & 1));
      gather(view(st), un, pn);
    }
    double v[N][N][N];
#pragma unroll
    for (int k = 0; k < N3; ++k) v[k / N2][(k / N) % N][k % N] = ((pn >> k) & 1u) ? un[k] : 0.0;
    __syncwarp();  // every lane is past its reads of the stage that held batch it - 1
    if (b + (NST - 1) * nw < nb) issue((it + NST - 1) % NST, b + (NST - 1) * nw);
    if (PREF && b + nw < nb) {
      const int s1 = (it + 1) % NST;
      mbar_wait(&bar[warp][s1], (unsigned)(((it + 1) / NST) & 1));
      gather(view(stage0 + s1 * stage_bytes), un, pn);
    }
    const View cur = view(st);
    // values at the Gauss points
    contract3<N, 0, false>(v, tb.S);
    contract3<N, 1, false>(v, tb.S);
    contract3<N, 2, false>(v, tb.S);
    double acc[N][N][N];
    double mac[N][N][N];
#pragma unroll
    for (int k = 0; k < N3; ++k) {
      const double c = COEF ? cur.cf[k] : 0.0;
      acc[k / N2][(k / N) % N][k % N] = c * v[k / N2][(k / N) % N][k % N];
      if (MODE == 2)
        mac[k / N2][(k / N) % N][k % N] = __ldg(a.mcoef + k) * v[k / N2][(k / N) % N][k % N];
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
    if (cur.ok) {
#pragma unroll
      for (int k = 0; k < N3; ++k) {
        const Code<WIDE> c = decode<WIDE>(cur.code, k);
        const int64_t o = (int64_t)cur.gt[c.g].y + c.rh;
        atomicAdd(a.hx + o, acc[k / N2][(k / N) % N][k % N]);
        if (MODE == 2) atomicAdd(a.mx + o, mac[k / N2][(k / N) % N][k % N]);
      }
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
  PairBatch* pair_batches = nullptr;  // pair kernel (n <= 3)
  Batch* batches = nullptr;  // plane kernel (n >= 4)
  std::vector<int64_t> break_pair;   // pair indices a launch range may start / end at
  std::vector<int64_t> break_batch;  // ... and the batch index there
  uint32_t* codes = nullptr;
  int2* gtab = nullptr;
  CellTables tables{};
};

namespace {

template <int N, bool COEF, int MODE, bool WIDE>
int launch_k1(const K1Plan* p, K1Args& args, int64_t p0, int64_t p1, cudaStream_t st) {
  // the range must start and end at batch boundaries the plan was cut at
  int64_t b0 = -1, b1 = -1;
  for (size_t k = 0; k < p->break_pair.size(); ++k) {
    if (p->break_pair[k] == p0) b0 = p->break_batch[k];
    if (p->break_pair[k] == p1) b1 = p->break_batch[k];
  }
  if (b0 < 0 || b1 < 0) {
    set_error("K1: pair range [%lld, %lld) does not start / end at a declared break",
              (long long)p0, (long long)p1);
    return BMV_ERR_INVALID;
  }
  if (b1 == b0) return BMV_OK;
  args.b0 = b0;
  args.b1 = b1;
  if constexpr (N <= 3) {
    constexpr int NP = N;
    auto kern = k1_pair_kernel<NP, COEF, MODE, WIDE>;
    constexpr int kW = K1PairShape<NP>::WARPS;
    const int smem = kW * K1PairShape<NP>::STAGES * k1_pair_stage_bytes<NP>(p->code_stride, p->gbytes);
    if (smem > 227 * 1024) {
      set_error("K1: the pair kernel's metadata stages (%d bytes: %d group-table bytes per pair) "
                "exceed the shared memory of an SM; use coarser row blocks",
                smem, p->gbytes);
      return BMV_ERR_INVALID;
    }
    BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t want = (b1 - b0 + kW - 1) / kW;
    const int64_t grid = std::min<int64_t>(want, (int64_t)sm_count());
    kern<<<(unsigned)grid, kW * 32, smem, st>>>(args, p->tables);
  } else {
    constexpr int NN = N;
    auto kern = k1_plane_kernel<NN, COEF, MODE, WIDE>;
    constexpr int kW = K1Shape<NN>::WARPS;
    const int smem = kW * k1_warp_bytes<NN>(p->code_stride, p->gbytes);
    BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // persistent: the CTAs that fit the GPU at once, fewer if there are fewer batches
    static int ctas_per_sm[2][3][2][6] = {};
    int& cps = ctas_per_sm[COEF][MODE][WIDE][N];
    if (cps == 0) {
      BMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cps, kern, kW * 32, smem));
      if (cps <= 0) {
        set_error("K1: the plane kernel does not fit an SM (%d bytes of shared memory)", smem);
        cps = 0;
        return BMV_ERR_INVALID;
      }
    }
    const int64_t want = (b1 - b0 + kW - 1) / kW;
    const int64_t grid = std::min<int64_t>(want, (int64_t)cps * sm_count());
    kern<<<(unsigned)grid, kW * 32, smem, st>>>(args, p->tables);
  }
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N>
int dispatch_n(const K1Plan* p, K1Args& args, bool coef, int mode, int64_t p0, int64_t p1,
               cudaStream_t st) {
  if (p->wide) {
    if (mode == 0)
      return coef ? launch_k1<N, true, 0, true>(p, args, p0, p1, st)
                  : launch_k1<N, false, 0, true>(p, args, p0, p1, st);
    if (mode == 1) return launch_k1<N, true, 1, true>(p, args, p0, p1, st);
    return coef ? launch_k1<N, true, 2, true>(p, args, p0, p1, st)
                : launch_k1<N, false, 2, true>(p, args, p0, p1, st);
  }
  if (mode == 0)
    return coef ? launch_k1<N, true, 0, false>(p, args, p0, p1, st)
                : launch_k1<N, false, 0, false>(p, args, p0, p1, st);
  if (mode == 1) return launch_k1<N, true, 1, false>(p, args, p0, p1, st);
  return coef ? launch_k1<N, true, 2, false>(p, args, p0, p1, st)
              : launch_k1<N, false, 2, false>(p, args, p0, p1, st);
}

int dispatch(const K1Plan* p, K1Args& args, bool coef, int mode, int64_t p0, int64_t p1,
             cudaStream_t st) {
  switch (p->n) {
    case 2: return dispatch_n<2>(p, args, coef, mode, p0, p1, st);
    case 3: return dispatch_n<3>(p, args, coef, mode, p0, p1, st);
    case 4: return dispatch_n<4>(p, args, coef, mode, p0, p1, st);
    case 5: return dispatch_n<5>(p, args, coef, mode, p0, p1, st);
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
      d->code_stride <= 0 || (d->code_stride & 3) || d->max_groups < 0 || d->max_groups > 32 ||
      d->n_breaks < 0 || d->n_pairs > INT32_MAX) {
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
  for (int64_t q = 0; q < d->n_pairs; ++q) {
    const int64_t go = d->pair_gtab[q];
    if ((go & 3) || d->pair_ngp[q] > d->max_groups || (d->pair_ngp[q] & 1) || go / 4 > INT32_MAX ||
        (q + 1 < d->n_pairs && d->pair_gtab[q + 1] != go + 2 * d->pair_ngp[q])) {
      delete p;
      set_error("bmv_cellop_create: bad group table of pair %lld", (long long)q);
      return BMV_ERR_INVALID;
    }
  }
  // launch ranges start / end at 0, n_pairs and the declared breaks
  p->break_pair.push_back(0);
  for (int32_t k = 0; k < d->n_breaks; ++k) {
    const int64_t bp = d->breaks[k];
    if (bp < p->break_pair.back() || bp > d->n_pairs) {
      delete p;
      set_error("bmv_cellop_create: breaks must be ascending pair indices");
      return BMV_ERR_INVALID;
    }
    if (bp > p->break_pair.back()) p->break_pair.push_back(bp);
  }
  if (p->break_pair.back() < d->n_pairs) p->break_pair.push_back(d->n_pairs);
  int rc = BMV_OK;
  if (n <= 3) {
    // batches: up to 32 consecutive pairs in at most kPairCells cells, never
    // across a break (greedy; pairs are sorted by cell inside each range)
    std::vector<PairBatch> batches;
    batches.reserve((size_t)(d->n_pairs / 32 + 8));
    size_t bk = 0;
    p->break_batch.assign(p->break_pair.size(), 0);
    int64_t q = 0;
    while (q < d->n_pairs) {
      while (bk + 1 < p->break_pair.size() && p->break_pair[bk + 1] <= q) ++bk;
      if (p->break_pair[bk] == q) p->break_batch[bk] = (int64_t)batches.size();
      const int64_t lim = bk + 1 < p->break_pair.size() ? p->break_pair[bk + 1] : d->n_pairs;
      PairBatch b{};
      b.first_pair = (int32_t)q;
      b.gt16 = (int32_t)(d->pair_gtab[q] / 4);
      int np = 0, nc = 0, entries = 0;
      while (q + np < lim && np < 32) {
        const int32_t cell = d->pair_cell[q + np];
        if (nc == 0 || cell != b.c[nc - 1].cell) {
          if (nc == kPairCells) break;
          b.c[nc].cell = cell;
          b.c[nc].first = np;
          b.c[nc].goff = entries;
          b.c[nc].ngp = d->pair_ngp[q + np];
          ++nc;
        }
        b.slot[np] = (uint8_t)(nc - 1);
        entries += d->pair_ngp[q + np];
        ++np;
      }
      b.np = np;
      b.ncells = nc;
      b.gt_bytes = 8 * entries;
      batches.push_back(b);
      q += np;
    }
    for (size_t k = 0; k < p->break_pair.size(); ++k)
      if (p->break_pair[k] == d->n_pairs) p->break_batch[k] = (int64_t)batches.size();
    rc = upload(batches.data(), (int64_t)batches.size(), &p->pair_batches);
  } else {
    // batches: up to 32 / n consecutive pairs in at most two cells, never
    // across a break (greedy; pairs are sorted by cell inside each range)
    const int P = 32 / n;
    std::vector<Batch> batches;
    batches.reserve((size_t)(d->n_pairs / P + 8));
    size_t bk = 0;
    p->break_batch.assign(p->break_pair.size(), 0);
    int64_t q = 0;
    while (q < d->n_pairs) {
      while (bk + 1 < p->break_pair.size() && p->break_pair[bk + 1] <= q) ++bk;
      p->break_batch[bk] = p->break_pair[bk] == q ? (int64_t)batches.size() : p->break_batch[bk];
      const int64_t lim = bk + 1 < p->break_pair.size() ? p->break_pair[bk + 1] : d->n_pairs;
      Batch b{};
      b.first_pair = (int32_t)q;
      b.cell_a = b.cell_b = d->pair_cell[q];
      int na = 0, np = 0;
      const int ga = d->pair_ngp[q];
      int gb = ga;
      bool second = false;
      while (q + np < lim && np < P) {
        const int32_t cell = d->pair_cell[q + np];
        if (!second && cell != b.cell_a) {
          second = true;
          b.cell_b = cell;
          gb = d->pair_ngp[q + np];
        } else if (second && cell != b.cell_b) {
          break;
        }
        if (!second) ++na;
        ++np;
      }
      b.info = na | (np << 8) | (ga << 16) | (gb << 24);
      b.gt16 = (int32_t)(d->pair_gtab[q] / 4);
      b.gt_bytes = 8 * (na * ga + (np - na) * gb);
      batches.push_back(b);
      q += np;
    }
    for (size_t k = 0; k < p->break_pair.size(); ++k)
      if (p->break_pair[k] == d->n_pairs) p->break_batch[k] = (int64_t)batches.size();
    rc = upload(batches.data(), (int64_t)batches.size(), &p->batches);
  }
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
  bmv::release(p->pair_batches);
  bmv::release(p->batches);
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
  K1Args args{};
  args.codes = p->codes;
  args.gtab = p->gtab;
  args.batches = p->batches;
  args.pair_batches = p->pair_batches;
  args.code_stride = p->code_stride;
  args.gbytes = p->gbytes;
  args.coef = coef;
  args.coef_cell = coef_stride != 0 ? 1 : 0;
  args.x = x;
  args.hx = hx;
  args.mx = mx;
  args.mcoef = mcoef;
  return dispatch(p, args, coef != nullptr, mode, p0, p1, st);
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
