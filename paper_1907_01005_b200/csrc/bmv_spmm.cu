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

#include "bmv.h"
#include "bmv_common.cuh"
#include "bmv_tma.cuh"

namespace bmv {
namespace {

constexpr int kCW = 8;            // consumer warps per CTA
constexpr int kNS = 2 * kCW;      // stages (two per consumer warp)

struct ChunkArgs {
  const int64_t* part_start;  // n_parts + 1
  const int64_t* meta_off;    // n_chunks + 1 (int32 units, multiples of 4)
  const int32_t* meta;
  const int64_t* a_rng;       // n_chunks x 2 (doubles, 16-byte aligned bounds)
  const int64_t* b_rng;       // K4: n_chunks x 2; K5: null
  int stage_bytes;
};

// Chunk header (int32): see include/bmv.h (bmv_chunk_desc)
enum { H_NROWS = 0, H_NBR, H_UA, H_UB, H_NK, H_AOFF, H_BOFF, H_UAP, H_UBP, H_TAB, H_CMA, H_CMB,
       H_RB, H_KK, H_ST, H_YROW };

__device__ __forceinline__ void producer(const ChunkArgs& g, const double* a, const double* b,
                                         char* stages, uint64_t* full, uint64_t* empty,
                                         int64_t c0, int64_t n) {
  for (int64_t j = 0; j < n; ++j) {
    const int s = (int)(j % kNS);
    if (j >= kNS) mbar_wait(&empty[s], (unsigned)((j / kNS - 1) & 1));
    const int64_t c = c0 + j;
    char* st = stages + (int64_t)s * g.stage_bytes;
    const int64_t m0 = g.meta_off[c], m1 = g.meta_off[c + 1];
    const unsigned mb = (unsigned)((m1 - m0) * 4);
    const int32_t* mh = g.meta + m0;
    const int aoff = __ldg(mh + H_AOFF), boff = __ldg(mh + H_BOFF);
    const int64_t a0 = g.a_rng[2 * c], a1 = g.a_rng[2 * c + 1];
    const unsigned ab = (unsigned)((a1 - a0) * 8);
    unsigned bb = 0;
    int64_t b0 = 0;
    if (g.b_rng) {
      b0 = g.b_rng[2 * c];
      bb = (unsigned)((g.b_rng[2 * c + 1] - b0) * 8);
    }
    mbar_expect_tx(&full[s], mb + ab + bb);
    bulk_g2s(st, mh, mb, &full[s]);
    for (unsigned k = 0; k < ab; k += 65536u)
      bulk_g2s(st + aoff + k, a + a0 + k / 8, min(65536u, ab - k), &full[s]);
    for (unsigned k = 0; k < bb; k += 65536u)
      bulk_g2s(st + boff + k, b + b0 + k / 8, min(65536u, bb - k), &full[s]);
  }
}

// ---------------------------------------------------------------- K4 -----
// S[rb[a] + st[kk[a]][b]] += sum_rows A[row][cma[row][a]] * B[row][cmb[row][b]]
__device__ __forceinline__ void k4_chunk(const char* st, double* __restrict__ c, int lane) {
  const int32_t* m = reinterpret_cast<const int32_t*>(st);
  const int nrows = m[H_NROWS], ua = m[H_UA], ub = m[H_UB];
  const int uap = m[H_UAP], ubp = m[H_UBP];
  const double* As = reinterpret_cast<const double*>(st + m[H_AOFF]);
  const double* Bs = reinterpret_cast<const double*>(st + m[H_BOFF]);
  const int32_t* tab = m + m[H_TAB];            // per row: bi | a_row << 8, then b_row
  const int16_t* cma = reinterpret_cast<const int16_t*>(m + m[H_CMA]);
  const int16_t* cmb = reinterpret_cast<const int16_t*>(m + m[H_CMB]);
  const int32_t* rb = m + m[H_RB];
  const int32_t* kk = m + m[H_KK];
  const int32_t* stt = m + m[H_ST];
  const int nks = (nrows + 3) >> 2;
  const int g4 = lane >> 2, t4 = lane & 3;
  for (int ag = 0; ag < ua; ag += 32) {
    const int ta = min(4, (ua - ag + 7) >> 3);
    for (int bg = 0; bg < ub; bg += 32) {
      const int tb = min(4, (ub - bg + 7) >> 3);
      double acc[4][4][2];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
      int cur_bi = -1;
      int sa[4] = {-1, -1, -1, -1}, sb[4] = {-1, -1, -1, -1};
      for (int ks = 0; ks < nks; ++ks) {
        const int row = ks * 4 + t4;
        int bi = -1, ar = 0, br = 0;
        if (row < nrows) {
          const int e = tab[2 * row];
          bi = e & 255;
          ar = e >> 8;
          br = tab[2 * row + 1];
        }
        if (bi != cur_bi) {  // colmaps of this lane's block row (reused while it stays)
          cur_bi = bi;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int aa = ag + t * 8 + g4;
            sa[t] = (bi >= 0 && t < ta && aa < ua) ? cma[bi * uap + aa] : -1;
            const int bb2 = bg + t * 8 + g4;
            sb[t] = (bi >= 0 && t < tb && bb2 < ub) ? cmb[bi * ubp + bb2] : -1;
          }
        }
        double av[4], bv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          av[t] = sa[t] >= 0 ? As[ar + sa[t]] : 0.0;
          bv[t] = sb[t] >= 0 ? Bs[br + sb[t]] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (t < ta && u < tb) dmma_8x8x4(acc[t][u][0], acc[t][u][1], av[t], bv[u]);
      }
      // flush: lane holds rows a = ag + 8t + g4, columns b = bg + 8u + 2 t4 + {0, 1}
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int aa = ag + t * 8 + g4;
        if (t >= ta || aa >= ua) continue;
        const int base = rb[aa];
        const int32_t* srow = stt + kk[aa] * ubp;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (u >= tb) continue;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int bb2 = bg + u * 8 + 2 * t4 + e;
            if (bb2 < ub) {
              const int sl = srow[bb2];
              if (sl >= 0) atomicAdd(c + (int64_t)base + sl, acc[t][u][e]);
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K5 -----
// Y[yrow[row] + cmy[row][b]] = alpha sum_a A[row][cma[row][a]] C[cb[a] + ct[ck[a]][b]] (+ old)
__device__ __forceinline__ void k5_chunk(const char* st, const double* __restrict__ cmat,
                                         double* __restrict__ y, double alpha, bool accumulate,
                                         int lane) {
  const int32_t* m = reinterpret_cast<const int32_t*>(st);
  const int nrows = m[H_NROWS], ua = m[H_UA], ub = m[H_UB];
  const int uap = m[H_UAP], ubp = m[H_UBP];
  const double* As = reinterpret_cast<const double*>(st + m[H_AOFF]);
  const int32_t* tab = m + m[H_TAB];            // per row: bi | a_row << 8
  const int32_t* yrow = m + m[H_YROW];
  const int16_t* cma = reinterpret_cast<const int16_t*>(m + m[H_CMA]);
  const int16_t* cmy = reinterpret_cast<const int16_t*>(m + m[H_CMB]);
  const int32_t* cb = m + m[H_RB];
  const int32_t* ck = m + m[H_KK];
  const int32_t* ct = m + m[H_ST];
  const int nrt = (nrows + 7) >> 3;  // <= 4 (chunks of <= 32 rows)
  const int g4 = lane >> 2, t4 = lane & 3;
  for (int yg = 0; yg < ub; yg += 32) {
    const int tb = min(4, (ub - yg + 7) >> 3);
    double acc[4][4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[r][u][0] = acc[r][u][1] = 0.0;
    for (int kg = 0; kg < ua; kg += 32) {
      const int nks = min(8, (ua - kg + 3) >> 2);
      double bf[8][4];  // C fragments: k = kg + 4 ks + t4, n = yg + 8 u + g4
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int ka = kg + ks * 4 + t4;
        const bool okk = ks < nks && ka < ua;
        const int base = okk ? cb[ka] : 0;
        const int32_t* crow = ct + (okk ? ck[ka] : 0) * ubp;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int bb2 = yg + u * 8 + g4;
          double v = 0.0;
          if (okk && u < tb && bb2 < ub) {
            const int sl = crow[bb2];
            if (sl >= 0) v = __ldg(cmat + (int64_t)base + sl);
          }
          bf[ks][u] = v;
        }
      }
#pragma unroll
      for (int rt = 0; rt < 4; ++rt) {
        if (rt >= nrt) continue;
        const int row = rt * 8 + g4;
        int bi = -1, ar = 0;
        if (row < nrows) {
          const int e = tab[row];
          bi = e & 255;
          ar = e >> 8;
        }
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (ks >= nks) continue;
          const int ka = kg + ks * 4 + t4;
          const int s = (bi >= 0 && ka < ua) ? cma[bi * uap + ka] : -1;
          const double av = s >= 0 ? As[ar + s] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < tb) dmma_8x8x4(acc[rt][u][0], acc[rt][u][1], av, bf[ks][u]);
        }
      }
    }
    // store: lane holds rows rt*8 + g4, columns yg + 8u + 2 t4 + {0, 1}
#pragma unroll
    for (int rt = 0; rt < 4; ++rt) {
      if (rt >= nrt) continue;
      const int row = rt * 8 + g4;
      if (row >= nrows) continue;
      const int bi = tab[row] & 255;
      const int64_t yo = yrow[row];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u >= tb) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb2 = yg + u * 8 + 2 * t4 + e;
          if (bb2 < ub) {
            const int s = cmy[bi * ubp + bb2];
            if (s >= 0) {
              double v = alpha * acc[rt][u][e];
              if (accumulate) v += y[yo + s];
              y[yo + s] = v;
            }
          }
        }
      }
    }
  }
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
    if (lane == 0) producer(g, a, KIND == 4 ? b : nullptr, smem, full, empty, c0, n);
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
  int64_t* meta_off = nullptr;
  int32_t* meta = nullptr;
  int64_t* a_rng = nullptr;
  int64_t* b_rng = nullptr;
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
  auto* p = new bmv_chunk_plan();
  p->kind = d->kind;
  p->n_parts = d->n_parts;
  p->stage_bytes = d->stage_bytes;
  p->n_chunks = d->n_chunks;
  int rc = upload(d->part_chunk_start, (int64_t)d->n_parts + 1, &p->part_start);
  if (rc == BMV_OK) rc = upload(d->chunk_meta, d->n_chunks + 1, &p->meta_off);
  if (rc == BMV_OK) rc = upload(d->meta, d->meta_len, &p->meta);
  if (rc == BMV_OK) rc = upload(d->chunk_a, 2 * d->n_chunks, &p->a_rng);
  if (rc == BMV_OK && d->kind == 4) rc = upload(d->chunk_b, 2 * d->n_chunks, &p->b_rng);
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
  bmv::release(p->meta_off);
  bmv::release(p->meta);
  bmv::release(p->a_rng);
  bmv::release(p->b_rng);
  delete p;
  return BMV_OK;
}

static int launch_chunks(const bmv_chunk_plan* p, const double* a, const double* b, double* out,
                         double alpha, int accumulate, void* stream) {
  using namespace bmv;
  if (p->n_chunks == 0) return BMV_OK;
  ChunkArgs g{p->part_start, p->meta_off, p->meta, p->a_rng, p->b_rng, p->stage_bytes};
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
