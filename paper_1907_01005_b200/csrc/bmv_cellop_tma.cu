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
// warp's shared memory -- the cell's coefficient row (w3 * V, q3p doubles)
// and the visit's X and HX element offset rows (n^3 int32, padded) --
// completing on one mbarrier per warp, so the data pipe only serves the X
// gather, the scatter-add and the
// transposes.  The slot -> group -> block offset indirection is resolved
// on the host into per-visit element offset rows, so the kernel reads one
// offset per element (a table lookup per element with random banks cost 5
// wavefronts per instruction).  Replaces the cell loop of CellOperator.apply (reference
// bcsrmv/matfree.py:458-527) for the Hamiltonian with fp64 atomic scatter.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "bmv_cellop_pair.cuh"
#include "bmv_cellop_tma.cuh"
#include "bmv_common.cuh"
#include "bmv_sumfac.cuh"
#include "bmv_tma.cuh"

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st);
namespace {

constexpr int kTmaWarps = 4;  // warps per CTA

struct TmaArgs {
  const int4* __restrict__ desc;     // {visit, cell, lane | stride << 16, 0}
  const int32_t* __restrict__ xoff;  // per visit SRP: element offset of X row (-1: absent block)
  const int32_t* __restrict__ hoff;  // per visit SRP: element offset of HX row
  const double* __restrict__ coef;
  int coef_cell;  // 1: row per cell (stride q3p), 0: one row
  int64_t n_pairs;
  const double* __restrict__ x;
  double* __restrict__ hx;
  double* __restrict__ mx;           // fused mass output (DUAL), same layout as hx
  const double* __restrict__ mcoef;  // mass coefficient row (w3, q3p doubles)
};

// Scatter-add of a pair's plane result (A layout) through the HX offset row.
struct PlaneScatter {
  double* dst;
  const int32_t* hs;
  int t, lane;
  bool ok;
  template <int N, class L>
  __device__ __forceinline__ void operator()(double (&v)[N][N], double*, int, bool,
                                             const CellTables&) const {
    if (!ok) return;
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) atomicAdd(dst + (int64_t)hs[t * N * N + y * N + x] + lane, v[y][x]);
  }
};
// The fused mass operator: w3 * uq back to the nodes, scattered into mx.
struct MassScatter {
  PlaneScatter sc;
  const double* w3;
  template <int N, class L>
  __device__ __forceinline__ void operator()(double (&uqB)[N][N], double* buf, int tt,
                                             bool lane_ok, const CellTables& tb) const {
    mass_back_plane<N, L>(uqB, w3, buf, tt, lane_ok, tb);
    sc.template operator()<N, L>(uqB, buf, tt, lane_ok, tb);
  }
};

template <int N, bool COEF, bool DUAL = false>
__global__ void __launch_bounds__(kTmaWarps * 32, TmaShape<N>::MINB)
    cellop_tma_kernel(const TmaArgs a, const __grid_constant__ CellTables tb) {
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

  // per warp: [pair tiles | coefficient rows | HX offset rows]; the X offset
  // rows overlay the tiles (read by the gather, before the first transpose)
  unsigned char* wbase = smem + warp * TS::warp_bytes;
  double* buf = reinterpret_cast<double*>(wbase) + sub * TILE;
  const int32_t* xs = reinterpret_cast<const int32_t*>(wbase) + sub * TS::SS;
  double* cs = reinterpret_cast<double*>(wbase + TS::tile_bytes) + sub * TS::CS;
  const int32_t* hs = reinterpret_cast<const int32_t*>(wbase + TS::tile_bytes + TS::coef_bytes) +
                      sub * TS::SS;
  if (lid == 0) mbar_init(&bar[warp], 1);
  __syncwarp();

  int4 d = make_int4(0, 0, 0, 0);
  if (ok) d = __ldg(a.desc + pair);
  const int lane = d.z & 0xffff, stride = d.z >> 16;
  const bool issuer = ok && t == 0;
  const unsigned cbytes = COEF ? TS::Q3P * 8u : 0u;
  const double* gcf = a.coef + (a.coef_cell ? (int64_t)d.y * TS::Q3P : 0);
  const unsigned my_bytes = issuer ? cbytes + 2u * TS::SRP * 4u : 0u;
  const unsigned total = __reduce_add_sync(~0u, my_bytes);
  if (lid == 0) mbar_expect_tx(&bar[warp], total);  // the warp's single arrival
  __syncwarp();
  if (issuer) {
    if (COEF) bulk_g2s(cs, gcf, cbytes, &bar[warp]);
    bulk_g2s(const_cast<int32_t*>(xs), a.xoff + (int64_t)d.x * TS::SRP, TS::SRP * 4u, &bar[warp]);
    bulk_g2s(const_cast<int32_t*>(hs), a.hoff + (int64_t)d.x * TS::SRP, TS::SRP * 4u, &bar[warp]);
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
        const int xo = xs[t * N2 + y * N + x];
        if (xo >= 0) v = __ldg(a.x + (int64_t)xo + lane);
      }
      u[y][x] = v;
    }
  }
  double out[N][N];
  if (DUAL) {  // H x to hx and M x to mx from one gather and one interpolation
    const PlaneScatter hsc{a.hx, hs, t, lane, ok};
    sumfac_h_plane<N, COEF, 1, Tile<N>, const double*, MassScatter, PlaneScatter>(
        u, out, buf, tt, lane_ok, cs + tt * N2, tb,
        MassScatter{PlaneScatter{a.mx, hs, t, lane, ok}, a.mcoef}, hsc);
    return;
  }
  sumfac_h_plane<N, COEF, 1>(u, out, buf, tt, lane_ok, cs + tt * N2, tb);
  if (ok) {
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x)
        atomicAdd(a.hx + (int64_t)hs[t * N2 + y * N + x] + lane, out[y][x]);
  }
  (void)stride;
}


// One thread per pair (n <= 3; bmv_cellop_pair.cuh).  4 warps per CTA.
template <int N, bool COEF>
__global__ void __launch_bounds__(kTmaWarps * 32, 3)  // 27 values + 27 accumulators: no spills
    cellop_pair_kernel(const TmaArgs a, const __grid_constant__ CellTables tb) {
  using PS = PairShape<N>;
  constexpr int N2 = N * N, N3 = N2 * N;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kTmaWarps];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int64_t pair = ((int64_t)blockIdx.x * kTmaWarps + warp) * 32 + lid;
  const bool ok = pair < a.n_pairs;
  unsigned char* wbase = smem + warp * PS::warp_bytes;
  int32_t* orow = reinterpret_cast<int32_t*>(wbase) + lid * PS::OU * 4;
  double* crow = reinterpret_cast<double*>(wbase + 32 * 16 * PS::OU) + lid * PS::CU * 2;
  if (lid == 0) mbar_init(&bar[warp], 1);
  __syncwarp();
  int4 d = make_int4(0, 0, 0, 0);
  if (ok) d = __ldg(a.desc + pair);
  const int lane = d.z & 0xffff;
  const unsigned cbytes = COEF ? PS::Q3P * 8u : 0u;
  unsigned total = __reduce_add_sync(~0u, ok ? cbytes + PS::SRP * 4u : 0u);
  if (lid == 0) mbar_expect_tx(&bar[warp], total);
  __syncwarp();
  if (ok) {
    if (COEF) bulk_g2s(crow, a.coef + (a.coef_cell ? (int64_t)d.y * PS::Q3P : 0), cbytes, &bar[warp]);
    bulk_g2s(orow, a.xoff + (int64_t)d.x * PS::SRP, PS::SRP * 4u, &bar[warp]);
  }
  mbar_wait(&bar[warp], 0);
  double v[N][N][N];
#pragma unroll
  for (int k4 = 0; k4 < PS::SRP / 4; ++k4) {
    const int4 o = reinterpret_cast<const int4*>(orow)[k4];
    const int oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int k = 4 * k4 + m;
      if (k < N3) {
        const double x = (ok && oo[m] >= 0) ? __ldg(a.x + (int64_t)oo[m] + lane) : 0.0;
        v[k / N2][(k / N) % N][k % N] = x;
      }
    }
  }
  // the HX offsets replace the X offsets (lands during the arithmetic)
  __syncwarp();
  total = __reduce_add_sync(~0u, ok ? PS::SRP * 4u : 0u);
  if (lid == 0) mbar_expect_tx(&bar[warp], total);
  __syncwarp();
  if (ok) bulk_g2s(orow, a.hoff + (int64_t)d.x * PS::SRP, PS::SRP * 4u, &bar[warp]);
  // values at the Gauss points
  contract3<N, 0, false>(v, tb.S);
  contract3<N, 1, false>(v, tb.S);
  contract3<N, 2, false>(v, tb.S);
  double acc[N][N][N];
  if (COEF) {
#pragma unroll
    for (int k2 = 0; k2 < PS::Q3P / 2; ++k2) {
      const double2 c = reinterpret_cast<const double2*>(crow)[k2];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int k = 2 * k2 + m;
        if (k < N3) acc[k / N2][(k / N) % N][k % N] = (m ? c.y : c.x) * v[k / N2][(k / N) % N][k % N];
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < N3; ++k) acc[k / N2][(k / N) % N][k % N] = 0.0;
  }
  grad3<N, 0>(v, acc, tb);
  grad3<N, 1>(v, acc, tb);
  grad3<N, 2>(v, acc, tb);
  // back to the nodes
  contract3<N, 0, true>(acc, tb.S);
  contract3<N, 1, true>(acc, tb.S);
  contract3<N, 2, true>(acc, tb.S);
  mbar_wait(&bar[warp], 1);
  if (ok) {
#pragma unroll
    for (int k4 = 0; k4 < PS::SRP / 4; ++k4) {
      const int4 o = reinterpret_cast<const int4*>(orow)[k4];
      const int oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int k = 4 * k4 + m;
        if (k < N3) atomicAdd(a.hx + (int64_t)oo[m] + lane, acc[k / N2][(k / N) % N][k % N]);
      }
    }
  }
}

template <int N, bool COEF>
int launch_dual(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
                const double* mcoef, const double* x, double* hx, double* mx, int64_t zero_len,
                cudaStream_t st) {
  using TS = TmaShape<N>;
  auto kern = cellop_tma_kernel<N, COEF, true>;
  const int smem = kTmaWarps * TS::warp_bytes;
  BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TmaArgs args{tp->desc, tp->xoff, tp->hoff, coef, coef_cell, tp->n_pairs, x, hx, mx, mcoef};
  int rc = zero_async(hx, zero_len, st);
  if (rc == BMV_OK) rc = zero_async(mx, zero_len, st);
  if (rc) return rc;
  const int64_t per_cta = (int64_t)kTmaWarps * TS::P;
  const int64_t grid = (tp->n_pairs + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid, kTmaWarps * 32, smem, st>>>(args, tb);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N, bool COEF>
int launch_tma(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
               const double* x, double* hx, int64_t zero_len, cudaStream_t st) {
  using TS = TmaShape<N>;
  if (N <= 3 && tp->per_pair) {
    auto pk = cellop_pair_kernel<N < 4 ? N : 3, COEF>;
    const int psmem = kTmaWarps * PairShape<N < 4 ? N : 3>::warp_bytes;
    BMV_CUDA_TRY(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem));
    TmaArgs pargs{tp->desc, tp->xoff, tp->hoff, coef, coef_cell, tp->n_pairs, x, hx};
    const int rc0 = zero_async(hx, zero_len, st);
    if (rc0) return rc0;
    const int64_t per = (int64_t)kTmaWarps * 32;
    pk<<<(unsigned)((tp->n_pairs + per - 1) / per), kTmaWarps * 32, psmem, st>>>(pargs, tb);
    BMV_CHECK_LAUNCH();
    return BMV_OK;
  }
  auto kern = cellop_tma_kernel<N, COEF>;
  const int smem = kTmaWarps * TS::warp_bytes;
  BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TmaArgs args{tp->desc, tp->xoff, tp->hoff, coef, coef_cell, tp->n_pairs, x, hx};
  const int rc = zero_async(hx, zero_len, st);
  if (rc) return rc;
  const int64_t per_cta = (int64_t)kTmaWarps * TS::P;
  const int64_t grid = (tp->n_pairs + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid, kTmaWarps * 32, smem, st>>>(args, tb);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N>
int build_n(const bmv_cellop_desc* d, TmaPlan* tp) {
  using TS = TmaShape<N>;
  constexpr int N3 = N * N * N;
  // per visit and cell DoF: the element offset of the DoF's row in the X and
  // HX blocks of the visit's column block (slot group -> block offset, plus
  // row in block * stride), without the lane
  const size_t nv = (size_t)d->n_visits;
  std::vector<int32_t> xo(nv * TS::SRP, -1), ho(nv * TS::SRP, 0);
  for (int32_t v = 0; v < d->n_visits; ++v) {
    const int64_t g0 = d->visit_goff[v], ng = d->visit_goff[v + 1] - g0;
    const int64_t cell = d->visit_cell[v], stride = d->visit_stride[v];
    for (int k = 0; k < N3; ++k) {
      const uint32_t s = d->cell_slots[cell * N3 + k];
      const int64_t grp = s >> 24, rib = s & 0xffffffu;
      if (grp >= ng) return -1;
      const int64_t gx = d->group_xoff[g0 + grp], gh = d->group_hoff[g0 + grp];
      const int64_t ex = gx < 0 ? -1 : gx + rib * stride, eh = gh + rib * stride;
      if (ex + stride > INT32_MAX || eh + stride > INT32_MAX || gh < 0) return -1;
      xo[(size_t)v * TS::SRP + k] = (int32_t)ex;
      ho[(size_t)v * TS::SRP + k] = (int32_t)eh;
    }
  }
  std::vector<int4> desc((size_t)d->n_pairs);
  for (int64_t q = 0; q < d->n_pairs; ++q) {
    const int32_t v = d->pair_visit[q];
    desc[(size_t)q] = make_int4(v, d->visit_cell[v], d->pair_lane[q] | (d->visit_stride[v] << 16), 0);
  }
  tp->n = N;
  tp->n_pairs = d->n_pairs;
  tp->q3p = TS::Q3P;
  const char* pe = std::getenv("BMV_K1_PAIR");
  tp->per_pair = N <= 3 && !(pe && pe[0] == '0');
  int rc = upload(desc.data(), (int64_t)desc.size(), &tp->desc);
  if (rc == BMV_OK) rc = upload(xo.data(), (int64_t)xo.size(), &tp->xoff);
  if (rc == BMV_OK) rc = upload(ho.data(), (int64_t)ho.size(), &tp->hoff);
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
  release(tp->xoff);
  release(tp->hoff);
  delete tp;
}

int tma_apply_hm(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
                 const double* mcoef, const double* x, double* hx, double* mx, int64_t zero_len,
                 cudaStream_t st) {
  const bool c = coef != nullptr;
#define BMV_DUAL(NN)                                                                       \
  return c ? launch_dual<NN, true>(tp, tb, coef, coef_cell, mcoef, x, hx, mx, zero_len, st) \
           : launch_dual<NN, false>(tp, tb, coef, coef_cell, mcoef, x, hx, mx, zero_len, st)
  switch (tp->n) {
    case 2: BMV_DUAL(2);
    case 3: BMV_DUAL(3);
    case 4: BMV_DUAL(4);
    case 5: BMV_DUAL(5);
    default:
      set_error("TMA plan with unsupported n %d", tp->n);
      return BMV_ERR_INVALID;
  }
#undef BMV_DUAL
}

int tma_apply(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
              const double* x, double* hx, int64_t zero_len, cudaStream_t st) {
  const bool c = coef != nullptr;
  switch (tp->n) {
    case 2: return c ? launch_tma<2, true>(tp, tb, coef, coef_cell, x, hx, zero_len, st)
                     : launch_tma<2, false>(tp, tb, coef, coef_cell, x, hx, zero_len, st);
    case 3: return c ? launch_tma<3, true>(tp, tb, coef, coef_cell, x, hx, zero_len, st)
                     : launch_tma<3, false>(tp, tb, coef, coef_cell, x, hx, zero_len, st);
    case 4: return c ? launch_tma<4, true>(tp, tb, coef, coef_cell, x, hx, zero_len, st)
                     : launch_tma<4, false>(tp, tb, coef, coef_cell, x, hx, zero_len, st);
    case 5: return c ? launch_tma<5, true>(tp, tb, coef, coef_cell, x, hx, zero_len, st)
                     : launch_tma<5, false>(tp, tb, coef, coef_cell, x, hx, zero_len, st);
    default:
      set_error("TMA plan with unsupported n %d", tp->n);
      return BMV_ERR_INVALID;
  }
}

}  // namespace bmv
