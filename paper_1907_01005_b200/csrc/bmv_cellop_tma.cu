// K1 (TMA-staged, default Hamiltonian path): the sum-factorised operator on
// the active (cell, column) pairs with each pair's per-cell operands moved
// by the TMA engine instead of the load/store pipe.
//
// Same thread mapping and arithmetic as the one-pass kernel (bmv_cellop.cu,
// bmv_sumfac.cuh: n threads per pair, thread t holds plane z = t, 12
// contractions, 4 pair-tile transposes).  ncu on the one-pass kernel showed
// the L1 / shared-memory data pipe as the binding unit (74 % busy, 30 %
// FP64): the per-lane 8-byte cp.async of the quadrature coefficients cost
// 6.4 wavefronts per instruction and the per-lane slot loads ~6 more.  Here
// lane t = 0 of every pair issues three cp.async.bulk copies into the
// warp's shared memory -- the cell's coefficient row (w3 * V, q3p doubles),
// its slot row (n^3 uint32, padded) and the visit's group table ({x, hx}
// block offsets, padded to 4) -- completing on one mbarrier per warp, so
// the data pipe only serves the X gather, the scatter-add and the
// transposes.  Replaces the cell loop of CellOperator.apply (reference
// bcsrmv/matfree.py:458-527) for the Hamiltonian with fp64 atomic scatter.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "bmv_cellop_tma.cuh"
#include "bmv_common.cuh"
#include "bmv_sumfac.cuh"
#include "bmv_tma.cuh"

namespace bmv {
namespace {

constexpr int kTmaWarps = 4;  // warps per CTA

struct TmaArgs {
  const int4* __restrict__ desc;     // {cell, group table base (int32 index), lane | stride << 16, g4}
  const int32_t* __restrict__ gxh;   // per visit [x offsets (g4) | hx offsets (g4)]
  const uint32_t* __restrict__ slots;  // per cell SRP uint32 (group << 24 | row in block)
  const double* __restrict__ coef;
  int coef_cell;  // 1: row per cell (stride q3p), 0: one row
  int64_t n_pairs;
  const double* __restrict__ x;
  double* __restrict__ hx;
};

template <int N, bool COEF>
__global__ void __launch_bounds__(kTmaWarps * 32, TmaShape<N>::MINB)
    cellop_tma_kernel(const TmaArgs a, const __grid_constant__ CellTables tb, const int G4) {
  using TS = TmaShape<N>;
  constexpr int P = TS::P, N2 = N * N, TILE = Tile<N>::TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kTmaWarps];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int sub = lid / N;
  const int t = lid - sub * N;
  const bool lane_ok = sub < P;
  const int tt = lane_ok ? t : 0;
  const int64_t pair = ((int64_t)blockIdx.x * kTmaWarps + warp) * P + sub;
  const bool ok = lane_ok && pair < a.n_pairs;

  unsigned char* wbase = smem + warp * TS::warp_bytes(G4);
  double* buf = reinterpret_cast<double*>(wbase) + sub * TILE;
  double* cs = reinterpret_cast<double*>(wbase + TS::tile_bytes) + sub * TS::CS;
  uint32_t* ss = reinterpret_cast<uint32_t*>(wbase + TS::tile_bytes + TS::coef_bytes) + sub * TS::SS;
  int32_t* gs = reinterpret_cast<int32_t*>(wbase + TS::tile_bytes + TS::coef_bytes + TS::slot_bytes) +
                sub * 2 * G4;
  if (lid == 0) mbar_init(&bar[warp], 1);
  __syncwarp();

  int4 d = make_int4(0, 0, 0, 0);
  if (ok) d = __ldg(a.desc + pair);
  const int lane = d.z & 0xffff, stride = d.z >> 16, g4 = d.w;
  // bytes this lane copies (t == 0 of a valid pair)
  const bool issuer = ok && t == 0;
  const unsigned cbytes = COEF ? TS::Q3P * 8u : 0u;
  const unsigned my_bytes = issuer ? cbytes + TS::SRP * 4u + (unsigned)g4 * 8u : 0u;
  const unsigned total = __reduce_add_sync(~0u, my_bytes);
  if (lid == 0) mbar_expect_tx(&bar[warp], total);  // the warp's single arrival
  __syncwarp();
  if (issuer) {
    if (COEF)
      bulk_g2s(cs, a.coef + (a.coef_cell ? (int64_t)d.x * TS::Q3P : 0), cbytes, &bar[warp]);
    bulk_g2s(ss, a.slots + (int64_t)d.x * TS::SRP, TS::SRP * 4u, &bar[warp]);
    if (g4) bulk_g2s(gs, a.gxh + d.y, (unsigned)g4 * 8u, &bar[warp]);
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
        const uint32_t s = ss[t * N2 + y * N + x];
        const int xo = gs[s >> 24];
        if (xo >= 0) v = __ldg(a.x + xo + (int64_t)(s & 0xffffffu) * stride + lane);
      }
      u[y][x] = v;
    }
  }
  double out[N][N];
  sumfac_h_plane<N, COEF, 1>(u, out, buf, tt, lane_ok, cs + tt * N2, tb);
  if (ok) {
    const int32_t* gh = gs + g4;
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        const uint32_t s = ss[t * N2 + y * N + x];
        atomicAdd(a.hx + gh[s >> 24] + (int64_t)(s & 0xffffffu) * stride + lane, out[y][x]);
      }
  }
}

template <int N, bool COEF>
int launch_tma(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
               const double* x, double* hx, cudaStream_t st) {
  using TS = TmaShape<N>;
  auto kern = cellop_tma_kernel<N, COEF>;
  const int smem = kTmaWarps * TS::warp_bytes(tp->g4max);
  BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TmaArgs args{tp->desc, tp->gxh, tp->slots, coef, coef_cell, tp->n_pairs, x, hx};
  const int64_t per_cta = (int64_t)kTmaWarps * TS::P;
  const int64_t grid = (tp->n_pairs + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid, kTmaWarps * 32, smem, st>>>(args, tb, tp->g4max);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N>
int build_n(const bmv_cellop_desc* d, TmaPlan* tp) {
  using TS = TmaShape<N>;
  constexpr int N3 = N * N * N;
  // group tables, per visit [x (g4) | hx (g4)], g4 = groups rounded up to 4
  std::vector<int64_t> vbase((size_t)d->n_visits + 1, 0);
  int g4max = 4;
  for (int32_t v = 0; v < d->n_visits; ++v) {
    const int64_t ng = d->visit_goff[v + 1] - d->visit_goff[v];
    const int64_t g4 = (ng + 3) / 4 * 4;
    g4max = std::max<int>(g4max, (int)g4);
    vbase[(size_t)v + 1] = vbase[(size_t)v] + 2 * g4;
  }
  if (g4max > 32 || vbase.back() > INT32_MAX) return -1;
  std::vector<int32_t> gxh((size_t)vbase.back(), -1);
  for (int32_t v = 0; v < d->n_visits; ++v) {
    const int64_t g0 = d->visit_goff[v], ng = d->visit_goff[v + 1] - g0;
    const int64_t g4 = (vbase[(size_t)v + 1] - vbase[(size_t)v]) / 2;
    for (int64_t k = 0; k < ng; ++k) {
      gxh[(size_t)(vbase[(size_t)v] + k)] = (int32_t)d->group_xoff[g0 + k];
      gxh[(size_t)(vbase[(size_t)v] + g4 + k)] = (int32_t)d->group_hoff[g0 + k];
    }
  }
  std::vector<uint32_t> sl((size_t)d->n_cells * TS::SRP, 0);
  for (int64_t c = 0; c < d->n_cells; ++c)
    std::copy(d->cell_slots + c * N3, d->cell_slots + (c + 1) * N3, sl.begin() + c * TS::SRP);
  std::vector<int4> desc((size_t)d->n_pairs);
  for (int64_t q = 0; q < d->n_pairs; ++q) {
    const int32_t v = d->pair_visit[q];
    desc[(size_t)q] = make_int4(d->visit_cell[v], (int)vbase[(size_t)v],
                                d->pair_lane[q] | (d->visit_stride[v] << 16),
                                (int)((vbase[(size_t)v + 1] - vbase[(size_t)v]) / 2));
  }
  tp->n = N;
  tp->n_pairs = d->n_pairs;
  tp->g4max = g4max;
  tp->q3p = TS::Q3P;
  int rc = upload(desc.data(), (int64_t)desc.size(), &tp->desc);
  if (rc == BMV_OK) rc = upload(gxh.data(), (int64_t)gxh.size(), &tp->gxh);
  if (rc == BMV_OK) rc = upload(sl.data(), (int64_t)sl.size(), &tp->slots);
  return rc;
}

}  // namespace

int tma_plan_build(const bmv_cellop_desc* d, TmaPlan** out) {
  *out = nullptr;
  const char* env = std::getenv("BMV_K1");
  if (env && std::string(env) != "tma") return BMV_OK;  // onepass / stream selected
  if (d->n_colors > 0 || d->n_pairs == 0) return BMV_OK;
  for (int32_t v = 0; v < d->n_visits; ++v)
    if (d->visit_stride[v] >= 65536) return BMV_OK;
  auto* tp = new TmaPlan();
  int rc = -1;
  switch (d->n) {
    case 2: rc = build_n<2>(d, tp); break;
    case 3: rc = build_n<3>(d, tp); break;
    case 4: rc = build_n<4>(d, tp); break;
    case 5: rc = build_n<5>(d, tp); break;
    default: break;
  }
  if (rc != BMV_OK) {
    tma_plan_destroy(tp);
    return rc < 0 ? BMV_OK : rc;
  }
  *out = tp;
  return BMV_OK;
}

void tma_plan_destroy(TmaPlan* tp) {
  if (!tp) return;
  release(tp->desc);
  release(tp->gxh);
  release(tp->slots);
  delete tp;
}

int tma_apply(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
              const double* x, double* hx, cudaStream_t st) {
  const bool c = coef != nullptr;
  switch (tp->n) {
    case 2: return c ? launch_tma<2, true>(tp, tb, coef, coef_cell, x, hx, st)
                     : launch_tma<2, false>(tp, tb, coef, coef_cell, x, hx, st);
    case 3: return c ? launch_tma<3, true>(tp, tb, coef, coef_cell, x, hx, st)
                     : launch_tma<3, false>(tp, tb, coef, coef_cell, x, hx, st);
    case 4: return c ? launch_tma<4, true>(tp, tb, coef, coef_cell, x, hx, st)
                     : launch_tma<4, false>(tp, tb, coef, coef_cell, x, hx, st);
    case 5: return c ? launch_tma<5, true>(tp, tb, coef, coef_cell, x, hx, st)
                     : launch_tma<5, false>(tp, tb, coef, coef_cell, x, hx, st);
    default:
      set_error("TMA plan with unsupported n %d", tp->n);
      return BMV_ERR_INVALID;
  }
}

}  // namespace bmv
