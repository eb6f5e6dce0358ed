// K4 (projection S = A^T B) and K5 (post-multiply Y = alpha A C) on slab
// storage (slabs.py): the products of reference tmmult / mmult
// (bcsrmv/bcsr.py:587-667) over the owned rows of A.
//
// Work unit: a CHUNK = a run of consecutive owned rows (whole block rows,
// or a row range of one long block row).  Because consecutive block rows'
// slabs are consecutive in memory, a chunk's A values (and, for K4, its B
// values) are ONE contiguous byte range each, staged by one cp.async.bulk
// (TMA) per operand into a ring of shared-memory stages by a producer warp;
// consumer warps own whole chunks.  Inside a chunk the block rows' stored
// columns are merged into union columns (UA for A, UB for B / Y); each block
// row maps union columns to its slab slots (colmap, -1 = structural zero),
// so a chunk is a dense (rows x UA)^T (rows x UB) product on FP64 tensor
// cores (DMMA m8n8k4), fragments read from the staged slabs through the
// colmaps.  Union columns are processed in groups of 32 (4 DMMA tiles).
//
// K4: the 8x8 result tiles are added to S with fp64 RED (S is small and
// L2-resident; one RED per union (a, b) of a chunk instead of one per row).
// K5: C (small, L2-resident) is read per chunk into B fragments held in
// registers, each Y value is written once (alpha AC, + old if accumulate).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "bmv.h"
#include "bmv_common.cuh"
#include "bmv_tma.cuh"

namespace bmv {
namespace {

constexpr int kCW = 12;           // consumer warps per CTA
constexpr int kNS = 20;           // stages (kNS - kCW chunks of lookahead)

// Per-chunk copy descriptors (built once in bmv_chunk_plan_create), structure
// of arrays so that the producer warp fetches 32 chunks per coalesced load.
struct ChunkArgs {
  const int64_t* part_start;  // n_parts + 1
  const int64_t* m0;          // first meta word
  const int64_t* a0;          // first staged A element
  const int64_t* b0;          // first staged B element (K4)
  const uint32_t* mb;         // meta bytes (= byte offset of A in the stage)
  const uint32_t* ab;         // A bytes
  const uint32_t* bb;         // B bytes (K4; 0 for K5)
  const int32_t* meta;
  int stage_bytes;
};

// Chunk header (int32): see include/bmv.h (bmv_chunk_desc)
enum { H_NSEG = 0, H_NROWS, H_UA, H_UB, H_NK, H_AOFF, H_BOFF, H_SEG, H_CMA, H_CMB, H_RB, H_KK,
       H_ST };

// Producer warp: lane l prefetches the descriptors of chunk base + l, lane 0
// issues the bulk copies (no dependent global load per chunk).
__device__ __forceinline__ void producer(const ChunkArgs& g, const double* a, const double* b,
                                         char* stages, uint64_t* full, uint64_t* empty,
                                         int64_t c0, int64_t n, int lane) {
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t c = c0 + base + lane;
    const bool ok = base + lane < n;
    const int64_t m0 = ok ? __ldg(g.m0 + c) : 0;
    const int64_t a0 = ok ? __ldg(g.a0 + c) : 0;
    const int64_t b0 = (ok && g.b0) ? __ldg(g.b0 + c) : 0;
    const unsigned mb = ok ? __ldg(g.mb + c) : 0u;
    const unsigned ab = ok ? __ldg(g.ab + c) : 0u;
    const unsigned bb = (ok && g.bb) ? __ldg(g.bb + c) : 0u;
    const int cnt = (int)min((int64_t)32, n - base);
    for (int k = 0; k < cnt; ++k) {
      const int64_t km0 = __shfl_sync(~0u, m0, k), ka0 = __shfl_sync(~0u, a0, k),
                    kb0 = __shfl_sync(~0u, b0, k);
      const unsigned kmb = __shfl_sync(~0u, mb, k), kab = __shfl_sync(~0u, ab, k),
                     kbb = __shfl_sync(~0u, bb, k);
      if (lane == 0) {
        const int64_t j = base + k;
        const int s = (int)(j % kNS);
        if (j >= kNS) mbar_wait(&empty[s], (unsigned)((j / kNS - 1) & 1));
        char* st = stages + (int64_t)s * g.stage_bytes;
        mbar_expect_tx(&full[s], kmb + kab + kbb);
        bulk_g2s(st, g.meta + km0, kmb, &full[s]);
        if (kab) bulk_g2s(st + kmb, a + ka0, kab, &full[s]);
        if (kbb) bulk_g2s(st + kmb + kab, b + kb0, kbb, &full[s]);
      }
    }
  }
}

// ---------------------------------------------------------------- K4 -----
// S[rb[a] + st[kk[a]][b]] += sum_rows A[row][cma[seg][a]] * B[row][cmb[seg][b]]
// One pass: union columns [ag, ag + 8 TA) x [bg, bg + 8 TB); accumulators
// live in registers over every segment of the chunk.  Segments are padded
// to multiples of 4 rows (a DMMA k-step never straddles two block rows).
template <int TA, int TB>
__device__ __forceinline__ void k4_pass(const int32_t* m, double* __restrict__ c, int ag, int bg,
                                        int lane) {
  const int nseg = m[H_NSEG], ua = m[H_UA], ub = m[H_UB];
  const char* st = reinterpret_cast<const char*>(m);
  const double* As = reinterpret_cast<const double*>(st + m[H_AOFF]);
  const double* Bs = reinterpret_cast<const double*>(st + m[H_BOFF]);
  const int4* seg = reinterpret_cast<const int4*>(m + m[H_SEG]);
  const int16_t* cma = reinterpret_cast<const int16_t*>(m + m[H_CMA]);
  const int16_t* cmb = reinterpret_cast<const int16_t*>(m + m[H_CMB]);
  const int g4 = lane >> 2, t4 = lane & 3;
  double acc[TA][TB][2];
#pragma unroll
  for (int t = 0; t < TA; ++t)
#pragma unroll
    for (int u = 0; u < TB; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  for (int s = 0; s < nseg; ++s) {
    const int4 r0 = seg[2 * s];
    const int kb = m[m[H_SEG] + 8 * s + 4];
    const int nrows = r0.x, ka = r0.z;
    int oa[TA], ob[TB];
    bool va[TA], vb[TB];
#pragma unroll
    for (int t = 0; t < TA; ++t) {
      const int aa = ag + t * 8 + g4;
      const int sl = aa < ua ? cma[s * ua + aa] : -1;
      va[t] = sl >= 0;
      oa[t] = r0.y + t4 * ka + sl;
    }
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const int bb = bg + u * 8 + g4;
      const int sl = bb < ub ? cmb[s * ub + bb] : -1;
      vb[u] = sl >= 0;
      ob[u] = r0.w + t4 * kb + sl;
    }
    const int nks = (nrows + 3) >> 2;
    int xa = 0, xb = 0;
    for (int ks = 0; ks < nks; ++ks, xa += 4 * ka, xb += 4 * kb) {
      const bool rok = ks * 4 + t4 < nrows;
      double av[TA], bv[TB];
#pragma unroll
      for (int t = 0; t < TA; ++t) av[t] = (rok && va[t]) ? As[oa[t] + xa] : 0.0;
#pragma unroll
      for (int u = 0; u < TB; ++u) bv[u] = (rok && vb[u]) ? Bs[ob[u] + xb] : 0.0;
#pragma unroll
      for (int t = 0; t < TA; ++t)
#pragma unroll
        for (int u = 0; u < TB; ++u) dmma_8x8x4(acc[t][u][0], acc[t][u][1], av[t], bv[u]);
    }
  }
  // flush: lane holds rows a = ag + 8t + g4, columns b = bg + 8u + 2 t4 + {0, 1}
  const int32_t* rb = m + m[H_RB];
  const int32_t* kk = m + m[H_KK];
  const int32_t* stt = m + m[H_ST];
#pragma unroll
  for (int t = 0; t < TA; ++t) {
    const int aa = ag + t * 8 + g4;
    if (aa >= ua) continue;
    const int base = rb[aa];
    const int32_t* srow = stt + kk[aa] * ub;
#pragma unroll
    for (int u = 0; u < TB; ++u) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int bb = bg + u * 8 + 2 * t4 + e;
        if (bb < ub) {
          const int sl = srow[bb];
          if (sl >= 0) atomicAdd(c + (int64_t)base + sl, acc[t][u][e]);
        }
      }
    }
  }
}

template <int TA>
__device__ __forceinline__ void k4_pass_b(const int32_t* m, double* c, int ag, int bg, int tb,
                                          int lane) {
  switch (tb) {
    case 1: k4_pass<TA, 1>(m, c, ag, bg, lane); break;
    case 2: k4_pass<TA, 2>(m, c, ag, bg, lane); break;
    case 3: k4_pass<TA, 3>(m, c, ag, bg, lane); break;
    default: k4_pass<TA, 4>(m, c, ag, bg, lane); break;
  }
}

__device__ __forceinline__ void k4_chunk(const char* st, double* __restrict__ c, int lane) {
  const int32_t* m = reinterpret_cast<const int32_t*>(st);
  const int ua = m[H_UA], ub = m[H_UB];
  for (int ag = 0; ag < ua; ag += 32) {
    const int ta = min(4, (ua - ag + 7) >> 3);
    for (int bg = 0; bg < ub; bg += 32) {
      const int tb = min(4, (ub - bg + 7) >> 3);
      switch (ta) {
        case 1: k4_pass_b<1>(m, c, ag, bg, tb, lane); break;
        case 2: k4_pass_b<2>(m, c, ag, bg, tb, lane); break;
        case 3: k4_pass_b<3>(m, c, ag, bg, tb, lane); break;
        default: k4_pass_b<4>(m, c, ag, bg, tb, lane); break;
      }
    }
  }
}

// ---------------------------------------------------------------- K5 -----
// Y[yoff[seg] + row K_Y + cmy[seg][b]] = alpha sum_a A[row][cma[seg][a]] C[cb[a] + ct[ck[a]][b]]
// (+ old).  One pass: union Y columns [bg, bg + 8 TB); the C fragments of an
// a-group of <= 4 KS union columns stay in registers over every row tile of
// the chunk; segments are padded to multiples of 8 rows.
template <int TB, int KS>
__device__ __forceinline__ void k5_pass(const int32_t* m, const double* __restrict__ cmat,
                                        double* __restrict__ y, double alpha, bool accumulate,
                                        int bg, int lane) {
  const int nseg = m[H_NSEG], ua = m[H_UA], ub = m[H_UB];
  const char* st = reinterpret_cast<const char*>(m);
  const double* As = reinterpret_cast<const double*>(st + m[H_AOFF]);
  const int4* seg = reinterpret_cast<const int4*>(m + m[H_SEG]);
  const int16_t* cma = reinterpret_cast<const int16_t*>(m + m[H_CMA]);
  const int16_t* cmy = reinterpret_cast<const int16_t*>(m + m[H_CMB]);
  const int32_t* cb = m + m[H_RB];
  const int32_t* ck = m + m[H_KK];
  const int32_t* ct = m + m[H_ST];
  const int g4 = lane >> 2, t4 = lane & 3;
  for (int ag = 0; ag < ua; ag += 4 * KS) {
    double bf[KS][TB];  // C fragments: k = ag + 4 ks + t4, n = bg + 8 u + g4
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int ka = ag + ks * 4 + t4;
      const bool okk = ka < ua;
      const int base = okk ? cb[ka] : 0;
      const int32_t* crow = ct + (okk ? ck[ka] : 0) * ub;
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int bb = bg + u * 8 + g4;
        double v = 0.0;
        if (okk && bb < ub) {
          const int sl = crow[bb];
          if (sl >= 0) v = __ldg(cmat + (int64_t)base + sl);
        }
        bf[ks][u] = v;
      }
    }
    const bool add_old = accumulate || ag > 0;
    for (int s = 0; s < nseg; ++s) {
      const int4 r0 = seg[2 * s];
      const int ky = m[m[H_SEG] + 8 * s + 4];
      const int nrows = r0.x, ka = r0.z;
      int oa[KS];
      unsigned vmask = 0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int aa = ag + ks * 4 + t4;
        const int sl = aa < ua ? cma[s * ua + aa] : -1;
        if (sl >= 0) vmask |= 1u << ks;
        oa[ks] = r0.y + g4 * ka + sl;
      }
      int sy[TB][2];
#pragma unroll
      for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = bg + u * 8 + 2 * t4 + e;
          sy[u][e] = bb < ub ? cmy[s * ub + bb] : -1;
        }
      double* yseg = y + (int64_t)r0.w + (int64_t)g4 * ky;
      const int nrt = (nrows + 7) >> 3;
      int xa = 0;
      for (int rt = 0; rt < nrt; ++rt, xa += 8 * ka, yseg += 8 * ky) {
        const bool rok = rt * 8 + g4 < nrows;
        double acc[TB][2];
#pragma unroll
        for (int u = 0; u < TB; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double av = (rok && ((vmask >> ks) & 1u)) ? As[oa[ks] + xa] : 0.0;
#pragma unroll
          for (int u = 0; u < TB; ++u) dmma_8x8x4(acc[u][0], acc[u][1], av, bf[ks][u]);
        }
        if (rok) {
#pragma unroll
          for (int u = 0; u < TB; ++u)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (sy[u][e] >= 0) {
                double v = alpha * acc[u][e];
                if (add_old) v += yseg[sy[u][e]];
                yseg[sy[u][e]] = v;
              }
        }
      }
    }
  }
}

// Pass width by the number of union A columns (register budget: the C
// fragments of an a-group, 4 KS x 8 TB doubles per warp, stay in registers).
template <int KS, int TBMAX>
__device__ __forceinline__ void k5_passes(const int32_t* m, const double* cmat, double* y,
                                          double alpha, bool accumulate, int lane) {
  const int ub = m[H_UB];
  for (int bg = 0; bg < ub; bg += 8 * TBMAX) {
    const int tb = min(TBMAX, (ub - bg + 7) >> 3);
    if (tb == 1) k5_pass<1, KS>(m, cmat, y, alpha, accumulate, bg, lane);
    else if (tb == 2 || TBMAX == 2) k5_pass<2, KS>(m, cmat, y, alpha, accumulate, bg, lane);
    else if (tb == 3) k5_pass<(TBMAX > 2 ? 3 : 2), KS>(m, cmat, y, alpha, accumulate, bg, lane);
    else k5_pass<(TBMAX > 2 ? 4 : 2), KS>(m, cmat, y, alpha, accumulate, bg, lane);
  }
}

__device__ __forceinline__ void k5_chunk(const char* st, const double* __restrict__ cmat,
                                         double* __restrict__ y, double alpha, bool accumulate,
                                         int lane) {
  const int32_t* m = reinterpret_cast<const int32_t*>(st);
  const int ua = m[H_UA];
  if (ua <= 8) k5_passes<2, 4>(m, cmat, y, alpha, accumulate, lane);
  else if (ua <= 16) k5_passes<4, 4>(m, cmat, y, alpha, accumulate, lane);
  else k5_passes<8, 2>(m, cmat, y, alpha, accumulate, lane);
}

template <int KIND>  // 4: K4, 5: K5
__global__ void __launch_bounds__((kCW + 1) * 32, 1)
    chunk_kernel(const ChunkArgs g, const double* __restrict__ a, const double* __restrict__ b,
                 double* __restrict__ out, double alpha, int accumulate) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kNS], empty[kNS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = g.part_start[blockIdx.x], n = g.part_start[blockIdx.x + 1] - c0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
  }
  __syncthreads();
  if (warp == kCW) {
    producer(g, a, KIND == 4 ? b : nullptr, smem, full, empty, c0, n, lane);
    return;
  }
  for (int64_t j = warp; j < n; j += kCW) {
    const int s = (int)(j % kNS);
    mbar_wait(&full[s], (unsigned)((j / kNS) & 1));
    const char* st = smem + (int64_t)s * g.stage_bytes;
    if (KIND == 4) k4_chunk(st, out, lane);
    else k5_chunk(st, b, out, alpha, accumulate != 0, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

}  // namespace

struct ChunkPlan {
  int kind = 0;
  int n_parts = 0;
  int stage_bytes = 0;
  int64_t n_chunks = 0;
  int64_t* part_start = nullptr;
  int64_t* m0 = nullptr;
  int64_t* a0 = nullptr;
  int64_t* b0 = nullptr;
  uint32_t* mb = nullptr;
  uint32_t* ab = nullptr;
  uint32_t* bb = nullptr;
  int32_t* meta = nullptr;
};

}  // namespace bmv

using bmv::ChunkPlan;

struct bmv_chunk_plan : ChunkPlan {};

extern "C" {

int bmv_chunk_plan_create(const bmv_chunk_desc* d, bmv_chunk_plan** out) {
  using namespace bmv;
  *out = nullptr;
  if (!d || (d->kind != 4 && d->kind != 5) || d->n_parts <= 0 || d->n_chunks < 0 ||
      d->stage_bytes <= 0 || (d->stage_bytes & 15) || d->stage_bytes * kNS > 227 * 1024) {
    set_error("bmv_chunk_plan_create: invalid descriptor");
    return BMV_ERR_INVALID;
  }
  // per-chunk copy descriptors (what the producer warp needs, nothing dependent)
  const size_t nc = (size_t)d->n_chunks;
  std::vector<int64_t> m0(nc), a0(nc), b0(nc);
  std::vector<uint32_t> mb(nc), ab(nc), bb(nc);
  for (size_t j = 0; j < nc; ++j) {
    m0[j] = d->chunk_meta[j];
    const int64_t words = d->chunk_meta[j + 1] - d->chunk_meta[j];
    a0[j] = d->chunk_a[2 * j];
    const int64_t an = d->chunk_a[2 * j + 1] - a0[j];
    int64_t bn = 0;
    if (d->kind == 4) {
      b0[j] = d->chunk_b[2 * j];
      bn = d->chunk_b[2 * j + 1] - b0[j];
    }
    const int32_t* h = d->meta + m0[j];
    if (words < 16 || (words & 3) || (m0[j] & 3) || (a0[j] & 1) || (an & 1) || (b0[j] & 1) ||
        (bn & 1) || an < 0 || bn < 0 || 4 * words + 8 * (an + bn) > d->stage_bytes ||
        h[5] != 4 * words || h[6] != 4 * words + 8 * an) {
      set_error("bmv_chunk_plan_create: chunk %lld does not fit its stage", (long long)j);
      return BMV_ERR_INVALID;
    }
    mb[j] = (uint32_t)(4 * words);
    ab[j] = (uint32_t)(8 * an);
    bb[j] = (uint32_t)(8 * bn);
  }
  auto* p = new bmv_chunk_plan();
  p->kind = d->kind;
  p->n_parts = d->n_parts;
  p->stage_bytes = d->stage_bytes;
  p->n_chunks = d->n_chunks;
  int rc = upload(d->part_chunk_start, (int64_t)d->n_parts + 1, &p->part_start);
  if (rc == BMV_OK) rc = upload(d->meta, d->meta_len, &p->meta);
  if (rc == BMV_OK) rc = upload(m0.data(), d->n_chunks, &p->m0);
  if (rc == BMV_OK) rc = upload(a0.data(), d->n_chunks, &p->a0);
  if (rc == BMV_OK) rc = upload(mb.data(), d->n_chunks, &p->mb);
  if (rc == BMV_OK) rc = upload(ab.data(), d->n_chunks, &p->ab);
  if (rc == BMV_OK && d->kind == 4) rc = upload(b0.data(), d->n_chunks, &p->b0);
  if (rc == BMV_OK && d->kind == 4) rc = upload(bb.data(), d->n_chunks, &p->bb);
  if (rc != BMV_OK) {
    bmv_chunk_plan_destroy(p);
    return rc;
  }
  *out = p;
  return BMV_OK;
}

int bmv_chunk_plan_destroy(bmv_chunk_plan* p) {
  if (!p) return BMV_OK;
  bmv::release(p->part_start);
  bmv::release(p->m0);
  bmv::release(p->a0);
  bmv::release(p->b0);
  bmv::release(p->mb);
  bmv::release(p->ab);
  bmv::release(p->bb);
  bmv::release(p->meta);
  delete p;
  return BMV_OK;
}

static int launch_chunks(const bmv_chunk_plan* p, const double* a, const double* b, double* out,
                         double alpha, int accumulate, void* stream) {
  using namespace bmv;
  if (p->n_chunks == 0) return BMV_OK;
  ChunkArgs g{p->part_start, p->m0, p->a0, p->b0, p->mb, p->ab, p->bb, p->meta, p->stage_bytes};
  const int smem = p->stage_bytes * kNS;
  cudaStream_t st = as_stream(stream);
  if (p->kind == 4) {
    BMV_CUDA_TRY(cudaFuncSetAttribute(chunk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      smem));
    chunk_kernel<4><<<p->n_parts, (kCW + 1) * 32, smem, st>>>(g, a, b, out, alpha, accumulate);
  } else {
    BMV_CUDA_TRY(cudaFuncSetAttribute(chunk_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      smem));
    chunk_kernel<5><<<p->n_parts, (kCW + 1) * 32, smem, st>>>(g, a, b, out, alpha, accumulate);
  }
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

int bmv_tmmult_run(const bmv_chunk_plan* p, const double* a, const double* b, double* c,
                   int64_t c_len, void* stream) {
  using namespace bmv;
  if (!p || p->kind != 4) {
    set_error("bmv_tmmult_run: not a K4 plan");
    return BMV_ERR_INVALID;
  }
  if (c_len > 0) {
    const int rc = bmv_zero(c, c_len, stream);
    if (rc != BMV_OK) return rc;
  }
  return launch_chunks(p, a, b, c, 1.0, 0, stream);
}

int bmv_mmult_run(const bmv_chunk_plan* p, const double* a, const double* cmat, double* y,
                  double alpha, int32_t accumulate, void* stream) {
  using namespace bmv;
  if (!p || p->kind != 5) {
    set_error("bmv_mmult_run: not a K5 plan");
    return BMV_ERR_INVALID;
  }
  return launch_chunks(p, a, cmat, y, alpha, accumulate, stream);
}

int bmv_chunk_kernel_config(int32_t* consumer_warps, int32_t* stages) {
  *consumer_warps = bmv::kCW;
  *stages = bmv::kNS;
  return BMV_OK;
}

}  // extern "C"
