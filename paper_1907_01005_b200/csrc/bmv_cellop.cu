// K1: cell-batched sum-factorised FE operator (H = -1/2 Laplace + V, or mass)
// on the active (cell, column) pairs of a sparse block multivector.
//
// Replaces the cell loop of CellOperator.apply and cell_integrals_sumfac of
// the reference (bcsrmv/matfree.py:458-527, 288-367).  B200 design:
//
//  * one pair (one orbital column on one cell) is processed by n threads;
//    thread t owns a 2D plane of the n^3 cell tensor (n*n values in
//    registers).  A warp carries floor(32/n) pairs (Q2: 10, Q4: 6).
//  * "A" layout: thread t holds the z = t plane, indices [y][x];
//    "B" layout: thread t holds the y = t plane, indices [z][x].
//    Contractions along axes local to the plane are register-only;
//    A<->B transposes go through a per-pair shared-memory tile with
//    __syncwarp only (a pair never spans warps).
//  * collocation form at the Gauss points (q = n): values are interpolated
//    once (3 contractions), gradients at the points use D_co = D S^-1
//    (3 + 3 transposed), then the values go back (3): 12 contractions of
//    n^4 FMAs instead of the reference's 18.  Same operator, different
//    rounding; parity is checked at <= 1e-12 per vector.
//  * gather/scatter through the CellDoFMap-style (group, row-in-block)
//    slots; scatter-add is an fp64 reduction (RED.ADD.F64) or, in the
//    deterministic mode, plain read-modify-write per cell colour class.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bmv_cellop_stream.cuh"
#include "bmv_cellop_tma.cuh"
#include "bmv_common.cuh"
#include "bmv_sumfac.cuh"

namespace bmv {

struct CellArgs {
  // per pair: {cell, first group index, lane | stride << 16, number of groups}
  const int4* __restrict__ pair_desc;
  const int32_t* __restrict__ group_xoff;  // element offsets (< 2^31) of the groups' blocks
  const int32_t* __restrict__ group_hoff;
  const uint32_t* __restrict__ cell_slots;
  const double* __restrict__ coef;
  int64_t coef_stride;
  int64_t pair_begin;
  int64_t pair_end;
  const double* __restrict__ x;
  double* __restrict__ hx;
};

constexpr int kWarps = 4;  // warps per CTA
#ifndef BMV_K1_MINB5
#define BMV_K1_MINB5 3
#endif


constexpr int kMaxGroups = 32;  // distinct block rows per cell (<= 27 at L = 0)

// Dynamic shared memory per warp: pair tiles (transposes) | coefficient and
// slot staging in lane-interleaved order [k][lane] (conflict-free) | group
// tables, one per pair at an odd stride of 2G+1 int64 (pairs hit distinct banks)
template <int N, bool COEF>
struct CellSmem {
  static constexpr int P = 32 / N;
  static constexpr int TILE = Tile<N>::TILE;
  static constexpr int N2 = N * N;
  static constexpr int tile_bytes = ((P * TILE * 8 + 15) / 16) * 16;
  static constexpr int coef_bytes = COEF ? N2 * 32 * 8 : 0;
  static constexpr int slot_bytes = N2 * 32 * 4;
  static __host__ __device__ int gtab_stride(int G) { return 2 * G + 1; }  // int32, odd
  static __host__ __device__ int gtab_bytes(int G) { return ((P * (2 * G + 1) * 4 + 15) / 16) * 16; }
  static __host__ __device__ int warp_bytes(int G) {
    return tile_bytes + coef_bytes + slot_bytes + gtab_bytes(G);
  }
};


template <int N> struct MinBlocks { static constexpr int v = N >= 4 ? BMV_K1_MINB5 : (N == 3 ? 7 : 1); };

// Three dependent memory trips per pair: (1) the 16-byte pair descriptor,
// (2) the cell's slots, the visit's group table and the quadrature
// coefficients (independent, all in flight together; coefficients by
// cp.async into shared memory, consumed after the interpolation),
// (3) the n^2 X values of the thread's plane (independent loads).
template <int N, bool KIN, bool COEF, bool ATOMIC>
__global__ void __launch_bounds__(kWarps * 32, MinBlocks<N>::v)
    cellop_kernel(const CellArgs a, const __grid_constant__ CellTables tb, const int G) {
  using SM = CellSmem<N, COEF>;
  constexpr int P = SM::P;
  constexpr int N2 = N * N;
  constexpr int N3 = N * N * N;
  constexpr int TILE = SM::TILE;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int warp = threadIdx.x >> 5;
  const int lid = threadIdx.x & 31;
  // pair-major mapping: lanes sub*N .. sub*N+N-1 hold the N planes of pair sub.
  // With the unpadded N^3 pair tile this gives conflict-free 64-bit transpose
  // stores and 2-way reads (bank model in DESIGN.md).
  const int sub = lid / N;
  const int t = lid - sub * N;
  const bool lane_ok = sub < P;
  const int tt = lane_ok ? t : 0;
  const int64_t pair = a.pair_begin + ((int64_t)blockIdx.x * kWarps + warp) * P + sub;
  const bool ok = lane_ok && pair < a.pair_end;

  unsigned char* wbase = smem_raw + warp * SM::warp_bytes(G);
  double* buf = reinterpret_cast<double*>(wbase) + sub * TILE;
  double* cbase = reinterpret_cast<double*>(wbase + SM::tile_bytes);  // [k][lane]
  double* cbuf = cbase + lid;
  uint32_t* slots = reinterpret_cast<uint32_t*>(wbase + SM::tile_bytes + SM::coef_bytes) + lid;
  int32_t* gtab = reinterpret_cast<int32_t*>(wbase + SM::tile_bytes + SM::coef_bytes +
                                             SM::slot_bytes) + sub * SM::gtab_stride(G);

  // ---- trip 1: pair descriptor
  int cell = 0, lane = 0, stride = 0, ng = 0, gbase = 0;
  if (ok) {
    const int4 d = __ldg(a.pair_desc + pair);
    cell = d.x;
    gbase = d.y;
    lane = d.z & 0xffff;
    stride = d.z >> 16;
    ng = d.w;
  }
  // ---- trip 2: slots, group table, coefficients
  uint32_t sl[N2];
  {
    const uint32_t* gs = a.cell_slots + (int64_t)cell * N3 + tt * N2;
#pragma unroll
    for (int k = 0; k < N2; ++k) sl[k] = ok ? __ldg(gs + k) : 0u;
  }
  if (ok) {
    for (int g = t; g < ng; g += N) {
      cp_async4(gtab + g, a.group_xoff + gbase + g);
      cp_async4(gtab + G + g, a.group_hoff + gbase + g);
    }
  }
  cp_async_commit();  // group 1: group table
  if (COEF && ok) {
    const double* c = a.coef + (int64_t)cell * a.coef_stride + t * N2;
#pragma unroll
    for (int k = 0; k < N2; ++k) cp_async8(cbuf + 32 * k, c + k);
  }
  cp_async_commit();  // group 2: coefficients (consumed after the interpolation)
  if (ok) {
#pragma unroll
    for (int k = 0; k < N2; ++k) slots[32 * k] = sl[k];
  }
  cp_async_wait_one();
  __syncwarp();

  // ---- trip 3: gather X (A layout, z = t)
  double u[N][N];
#pragma unroll
  for (int y = 0; y < N; ++y) {
#pragma unroll
    for (int x = 0; x < N; ++x) {
      double v = 0.0;
      if (ok) {
        const uint32_t s = sl[y * N + x];
        const int xo = gtab[s >> 24];
        if (xo >= 0) v = __ldg(a.x + xo + (int64_t)(s & 0xffffffu) * stride + lane);
      }
      u[y][x] = v;
    }
  }

  double v2[N][N];
  if (KIN) {
    cp_async_wait_all();  // coefficients staged by cp.async
    __syncwarp();
    sumfac_h_plane<N, COEF, 32>(u, v2, buf, tt, lane_ok, cbuf, tb);
  } else {
    // mass-like: values to the points, c * uq in B layout (qy = t), back
    double v1[N][N], uqB[N][N];
    contract_fast<N, false>(u, v1, tb.S);   // x
    contract_slow<N, false>(v1, v2, tb.S);  // y
    a_to_b<N>(v2, v1, buf, tt, lane_ok);    // B: y = qy = t, [z][qx]
    contract_slow<N, false>(v1, uqB, tb.S); // z
    cp_async_wait_all();
    __syncwarp();
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int x = 0; x < N; ++x)
        // element (qz=z, qy=t, qx=x) was staged by the thread of plane z, k = t*N + x
        v2[z][x] = COEF ? cbase[32 * (tt * N + x) + sub * N + z] * uqB[z][x] : 0.0;
    contract_slow<N, true>(v2, v1, tb.S);   // S^T along z
    contract_fast<N, true>(v1, v2, tb.S);   // S^T along x
    b_to_a<N>(v2, v1, buf, tt, lane_ok);    // A: z = t, [qy][x]
    contract_slow<N, true>(v1, v2, tb.S);   // S^T along y -> out[y][x]
  }

  // ---- scatter-add
  if (ok) {
    const int32_t* gh = gtab + G;
#pragma unroll
    for (int y = 0; y < N; ++y) {
#pragma unroll
      for (int x = 0; x < N; ++x) {
        const uint32_t s = slots[32 * (y * N + x)];
        double* p = a.hx + gh[s >> 24] + (int64_t)(s & 0xffffffu) * stride + lane;
        if (ATOMIC)
          atomicAdd(p, v2[y][x]);
        else
          *p += v2[y][x];
      }
    }
  }
}

__global__ void gaussian_coef_kernel(const double* __restrict__ origins,
                                     const double* __restrict__ qoff,
                                     const double* __restrict__ w3,
                                     const double* __restrict__ centers, int n_centers,
                                     double inv_s2, double scale, int q3, int64_t n_cells,
                                     double* __restrict__ coef) {
  extern __shared__ double cs[];
  for (int i = threadIdx.x; i < 3 * n_centers; i += blockDim.x) cs[i] = centers[i];
  __syncthreads();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_cells * q3) return;
  const int64_t cell = idx / q3;
  const int q = (int)(idx - cell * q3);
  const double px = origins[cell * 3 + 0] + qoff[q * 3 + 0];
  const double py = origins[cell * 3 + 1] + qoff[q * 3 + 1];
  const double pz = origins[cell * 3 + 2] + qoff[q * 3 + 2];
  double v = 0.0;
  for (int c = 0; c < n_centers; ++c) {
    const double dx = px - cs[3 * c], dy = py - cs[3 * c + 1], dz = pz - cs[3 * c + 2];
    const double e = (dx * dx + dy * dy + dz * dz) * inv_s2;
    if (e < 746.0) v += exp(-e);  // exp(-746) rounds to +0: skipping is exact
  }
  coef[idx] = w3[q] * (scale * v);
}

// p 16-byte aligned; each thread stores 4 x 16 bytes, warp-contiguous per
// store (one CTA of 256 threads covers 8 KB): measured 7.4 TB/s of writes
// against 6.5 TB/s for a grid-stride loop of single 16-byte stores.
constexpr int kZeroThreads = 256, kZeroPerThread = 8;  // doubles
__global__ void __launch_bounds__(kZeroThreads) zero_kernel(double* __restrict__ p, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * (kZeroThreads * kZeroPerThread);
#pragma unroll
  for (int j = 0; j < kZeroPerThread / 2; ++j) {
    const int64_t i = base + (int64_t)j * (2 * kZeroThreads) + 2 * threadIdx.x;
    if (i + 1 < n)
      *reinterpret_cast<double2*>(p + i) = make_double2(0.0, 0.0);
    else if (i < n)
      p[i] = 0.0;
  }
}

}  // namespace bmv

using namespace bmv;

struct bmv_cellop {
  int n = 0;
  int64_t n_pairs = 0;
  int32_t n_cells = 0;
  std::vector<int64_t> color_start;  // empty => atomic single launch
  int max_groups = 4;
  int4* pair_desc = nullptr;
  int32_t *group_xoff = nullptr, *group_hoff = nullptr;
  uint32_t* cell_slots = nullptr;
  CellTables tables{};
  StreamPlan* stream = nullptr;  // TMA-streamed Hamiltonian path (bmv_cellop_stream.cu)
  TmaPlan* tma = nullptr;        // TMA-staged Hamiltonian path (bmv_cellop_tma.cu), default
};

namespace {

template <int N, bool KIN, bool COEF, bool ATOMIC>
int launch_one(const CellArgs& args, const CellTables& tb, int G, cudaStream_t st) {
  using SM = CellSmem<N, COEF>;
  constexpr int P = SM::P;
  const int64_t n = args.pair_end - args.pair_begin;
  if (n <= 0) return BMV_OK;
  static bool configured = false;  // per instantiation
  if (!configured) {
    BMV_CUDA_TRY(cudaFuncSetAttribute(cellop_kernel<N, KIN, COEF, ATOMIC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kWarps * SM::warp_bytes(kMaxGroups)));
    configured = true;
  }
  const int64_t per_cta = (int64_t)kWarps * P;
  const int64_t grid = (n + per_cta - 1) / per_cta;
  cellop_kernel<N, KIN, COEF, ATOMIC>
      <<<(unsigned)grid, kWarps * 32, kWarps * SM::warp_bytes(G), st>>>(args, tb, G);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N>
int launch_n(const CellArgs& args, const CellTables& tb, int G, bool kin, bool coef, bool atomic,
             cudaStream_t st) {
  if (kin) {
    if (coef) return atomic ? launch_one<N, true, true, true>(args, tb, G, st)
                            : launch_one<N, true, true, false>(args, tb, G, st);
    return atomic ? launch_one<N, true, false, true>(args, tb, G, st)
                  : launch_one<N, true, false, false>(args, tb, G, st);
  }
  return atomic ? launch_one<N, false, true, true>(args, tb, G, st)
                : launch_one<N, false, true, false>(args, tb, G, st);
}

int launch_dispatch(int n, const CellArgs& args, const CellTables& tb, int G, bool kin,
                    bool coef, bool atomic, cudaStream_t st) {
  switch (n) {
    case 2: return launch_n<2>(args, tb, G, kin, coef, atomic, st);
    case 3: return launch_n<3>(args, tb, G, kin, coef, atomic, st);
    case 4: return launch_n<4>(args, tb, G, kin, coef, atomic, st);
    case 5: return launch_n<5>(args, tb, G, kin, coef, atomic, st);
    default:
      set_error("unsupported nodes per axis %d (degree 1..4)", n);
      return BMV_ERR_INVALID;
  }
}

int zero_launch(double* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return BMV_OK;
  if (reinterpret_cast<uintptr_t>(p) & 15) {  // 8-byte aligned start (odd element offset)
    BMV_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double), st));
    ++p;
    if (--n == 0) return BMV_OK;
  }
  const int64_t per = (int64_t)kZeroThreads * kZeroPerThread;
  const int64_t grid = (n + per - 1) / per;
  for (int64_t g0 = 0; g0 < grid; g0 += 0x7fffffff) {
    const int64_t g = std::min<int64_t>(grid - g0, 0x7fffffff);
    zero_kernel<<<(unsigned)g, kZeroThreads, 0, st>>>(p + g0 * per, n - g0 * per);
    BMV_CHECK_LAUNCH();
  }
  return BMV_OK;
}

}  // namespace

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st) { return zero_launch(p, n, st); }
}  // namespace bmv

extern "C" {

int bmv_cellop_create(const bmv_cellop_desc* d, bmv_cellop** out) {
  if (!d || !out) {
    set_error("null argument");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  if (d->n < 2 || d->n > BMV_MAX_NODES) {
    set_error("nodes per axis %d outside 2..%d", d->n, BMV_MAX_NODES);
    return BMV_ERR_INVALID;
  }
  if (d->n_pairs < 0 || d->n_cells < 0 || d->n_visits < 0 || d->n_colors < 0) {
    set_error("negative sizes in cell operator descriptor");
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_cellop();
  p->n = d->n;
  p->n_pairs = d->n_pairs;
  p->n_cells = d->n_cells;
  const int n3 = d->n * d->n * d->n;
  int rc = BMV_OK;
  if (d->n_colors > 0) {
    p->color_start.assign(d->color_pair_start, d->color_pair_start + d->n_colors + 1);
    if (p->color_start.front() != 0 || p->color_start.back() != d->n_pairs) {
      set_error("colour ranges do not cover the pairs");
      rc = BMV_ERR_INVALID;
    }
  }
  // packed per-pair descriptor {cell, first group, lane | stride << 16, groups}
  if (rc == BMV_OK && d->n_pairs > 0) {
    std::vector<int4> desc((size_t)d->n_pairs);
    int maxg = 1;
    for (int64_t q = 0; q < d->n_pairs; ++q) {
      const int32_t v = d->pair_visit[q];
      if (v < 0 || v >= d->n_visits) {
        set_error("pair %lld: visit %d out of range", (long long)q, v);
        rc = BMV_ERR_INVALID;
        break;
      }
      const int64_t g0 = d->visit_goff[v], ng = d->visit_goff[v + 1] - g0;
      const int32_t stride = d->visit_stride[v], lane = d->pair_lane[q];
      if (ng > kMaxGroups || stride >= 65536 || lane < 0 || lane >= stride || g0 > INT32_MAX) {
        set_error("pair %lld: a cell touches %lld block rows (max %d) or bad lane %d / stride %d",
                  (long long)q, (long long)ng, kMaxGroups, lane, stride);
        rc = BMV_ERR_INVALID;
        break;
      }
      desc[(size_t)q] = make_int4(d->visit_cell[v], (int)g0, lane | (stride << 16), (int)ng);
      if (ng > maxg) maxg = (int)ng;
    }
    p->max_groups = std::min(kMaxGroups, (maxg + 3) / 4 * 4);
    if (rc == BMV_OK) rc = upload(desc.data(), d->n_pairs, &p->pair_desc);
  }
  if (rc == BMV_OK && d->n_groups_total > 0) {
    std::vector<int32_t> gx((size_t)d->n_groups_total), gh((size_t)d->n_groups_total);
    for (int64_t i = 0; i < d->n_groups_total; ++i) {
      if (d->group_xoff[i] > INT32_MAX || d->group_hoff[i] > INT32_MAX || d->group_hoff[i] < 0) {
        set_error("block offset %lld exceeds the 2^31-element limit of this build",
                  (long long)std::max(d->group_xoff[i], d->group_hoff[i]));
        rc = BMV_ERR_INVALID;
        break;
      }
      gx[(size_t)i] = (int32_t)d->group_xoff[i];
      gh[(size_t)i] = (int32_t)d->group_hoff[i];
    }
    if (rc == BMV_OK) rc = upload(gx.data(), d->n_groups_total, &p->group_xoff);
    if (rc == BMV_OK) rc = upload(gh.data(), d->n_groups_total, &p->group_hoff);
  }
  if (rc == BMV_OK) rc = upload(d->cell_slots, (int64_t)d->n_cells * n3, &p->cell_slots);
  if (rc != BMV_OK) {
    bmv_cellop_destroy(p);
    return rc;
  }
  const int n = d->n;
  for (int i = 0; i < n * n; ++i) {
    p->tables.S[i] = d->S[i];
    p->tables.D[i] = d->Dco[i];
  }
  for (int i = 0; i < n; ++i) {
    p->tables.w[i] = d->w[i];
    for (int j = 0; j < n; ++j) p->tables.W2[i * n + j] = d->w[i] * d->w[j];
  }
  for (int k = 0; k < 3; ++k) p->tables.kin[k] = d->kin[k];
  rc = stream_plan_build(d, &p->stream);
  if (rc == BMV_OK) rc = tma_plan_build(d, &p->tma);
  if (rc != BMV_OK) {
    bmv_cellop_destroy(p);
    return rc;
  }
  *out = p;
  return BMV_OK;
}

int bmv_cellop_destroy(bmv_cellop* p) {
  if (!p) return BMV_OK;
  release(p->pair_desc);
  release(p->group_xoff);
  release(p->group_hoff);
  release(p->cell_slots);
  stream_plan_destroy(p->stream);
  tma_plan_destroy(p->tma);
  delete p;
  return BMV_OK;
}

int bmv_potential_gaussian(int64_t n_cells, int32_t q3, const double* cell_origins,
                           const double* quad_offsets, const double* w3, const double* centers,
                           int32_t n_centers, double inv_sigma2, double scale, double* coef,
                           void* stream) {
  if (n_cells < 0 || q3 <= 0 || n_centers < 0 || (n_cells > 0 && (!cell_origins || !quad_offsets ||
      !w3 || !coef)) || (n_centers > 0 && !centers)) {
    set_error("invalid gaussian potential arguments");
    return BMV_ERR_INVALID;
  }
  if (n_centers > 4096) {
    set_error("at most 4096 potential centres per launch (got %d)", n_centers);
    return BMV_ERR_INVALID;
  }
  if (n_cells == 0) return BMV_OK;
  const int64_t total = n_cells * q3;
  const unsigned grid = (unsigned)((total + 255) / 256);
  gaussian_coef_kernel<<<grid, 256, sizeof(double) * 3 * std::max(n_centers, 1),
                         as_stream(stream)>>>(cell_origins, quad_offsets, w3, centers, n_centers,
                                              inv_sigma2, scale, q3, n_cells, coef);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

int bmv_cellop_apply(bmv_cellop* p, int32_t kinetic, const double* coef, int64_t coef_stride,
                     const double* x, double* hx, int64_t zero_len, void* stream) {
  if (!p) {
    set_error("null plan");
    return BMV_ERR_INVALID;
  }
  if (!kinetic && !coef) {
    set_error("operator without kinetic and coefficient terms");
    return BMV_ERR_INVALID;
  }
  if (coef_stride < 0) {
    set_error("negative coefficient stride");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  if (p->tma && p->n_pairs > 0 && x && hx && kinetic &&
      (!coef || coef_stride == 0 || coef_stride == p->tma->q3p))
    return tma_apply(p->tma, p->tables, coef, coef_stride != 0 ? 1 : 0, x, hx, zero_len, st);
  int rc = zero_launch(hx, zero_len, st);
  if (rc) return rc;
  if (p->n_pairs == 0) return BMV_OK;
  if (!x || !hx) {
    set_error("null value array");
    return BMV_ERR_INVALID;
  }
  CellArgs args{p->pair_desc, p->group_xoff, p->group_hoff, p->cell_slots, coef, coef_stride,
                0, p->n_pairs, x, hx};
  const bool use_coef = coef != nullptr;

  if (p->stream && kinetic && (!coef || coef_stride == 0 || coef_stride == p->stream->q3p))
    return stream_apply(p->stream, p->tables, coef, coef_stride != 0 ? 1 : 0, x, hx, st);
  if (p->color_start.empty()) {
    return launch_dispatch(p->n, args, p->tables, p->max_groups, kinetic != 0, use_coef, true, st);
  }
  for (size_t c = 0; c + 1 < p->color_start.size(); ++c) {
    args.pair_begin = p->color_start[c];
    args.pair_end = p->color_start[c + 1];
    rc = launch_dispatch(p->n, args, p->tables, p->max_groups, kinetic != 0, use_coef, false, st);
    if (rc) return rc;
  }
  return BMV_OK;
}

int bmv_cellop_apply_hm(bmv_cellop* p, const double* coef, int64_t coef_stride,
                        const double* mass_coef, const double* x, double* hx, double* mx,
                        int64_t zero_len, void* stream) {
  if (!p || !mass_coef || !x || !hx || !mx) {
    set_error("null argument");
    return BMV_ERR_INVALID;
  }
  if (p->n_pairs == 0) {  // nothing to add: both results are zero (every rank takes this path)
    int rc = zero_launch(hx, zero_len, as_stream(stream));
    return rc ? rc : zero_launch(mx, zero_len, as_stream(stream));
  }
  if (!p->tma) {
    set_error("the fused H + mass apply needs the TMA plan (BMV_K1=tma)");
    return BMV_ERR_INVALID;
  }
  if (coef && coef_stride != 0 && coef_stride != p->tma->q3p) {
    set_error("coefficient stride %lld: expected 0 or %d", (long long)coef_stride, p->tma->q3p);
    return BMV_ERR_INVALID;
  }
  return tma_apply_hm(p->tma, p->tables, coef, coef_stride != 0 ? 1 : 0, mass_coef, x, hx, mx,
                      zero_len, as_stream(stream));
}

int bmv_cellop_launches(const bmv_cellop* p, int32_t* out) {
  if (!p || !out) {
    set_error("null argument");
    return BMV_ERR_INVALID;
  }
  int32_t k = 0;
  if (p->n_pairs > 0) {
    if (p->color_start.empty()) {
      k = 1;
    } else {
      for (size_t c = 0; c + 1 < p->color_start.size(); ++c)
        k += p->color_start[c + 1] > p->color_start[c] ? 1 : 0;
    }
  }
  *out = k;
  return BMV_OK;
}

}  // extern "C"
