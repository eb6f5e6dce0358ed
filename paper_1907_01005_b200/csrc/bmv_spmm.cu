// K4 (projection S = A^T B) and K5 (post-multiply Y = alpha A C) on slab
// storage (slabs.py): the products of reference tmmult / mmult
// (bcsrmv/bcsr.py:587-667) over the owned rows of A.
//
// Work unit: a CHUNK = a run of consecutive owned rows (whole block rows,
// or a row range of one long block row).  Because consecutive block rows'
// slabs are consecutive in memory, a chunk's A values (and, for K4, its B
// values) are ONE contiguous byte range each.  Every warp runs its own
// software pipeline: it claims chunks in order from a CTA counter, copies
// [meta | A | B] of the next chunks into its private shared-memory buffers
// with 16-byte cp.async (LDGSTS, L1 bypass) and multiplies the oldest one.
// (A producer warp feeding a shared ring with 1D TMA bulk copies was
// measured first: the more bulk copies were in flight per SM the later the
// OLDEST one completed, profiles/r02_spmm_tma_*.txt.)
//
// Inside a chunk the block rows' stored columns are merged into union
// columns (UA for A, UB for B / Y); each segment (block row piece) maps union
// columns to its slab slots (colmap, -1 = structural zero), so a chunk is a
// dense (rows x UA)^T (rows x UB) product on the FP64 tensor pipe (DMMA
// m8n8k4), fragments read from the staged slabs through per-lane slot
// offsets fixed per segment.
//
// K4: the 8x8 result tiles are added to S with fp64 RED (S is small and
// L2-resident; one RED per union (a, b) of a chunk instead of one per row).
// K5: C (small, L2-resident) is read per chunk into B fragments held in
// registers, each Y value is written once (alpha AC, + old if accumulate).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "bmv.h"
#include "bmv_common.cuh"
#include "bmv_tma.cuh"

namespace bmv {
namespace {

// Warps per CTA (each with its own pipeline), measured per kernel
// (profiles/r02_spmm_cpasync_*): K4 stages two operands and gains from
// larger chunks, K5 from more warps.
#ifndef BMV_K4_WARPS
#define BMV_K4_WARPS 12
#endif
#ifndef BMV_K4_WARPS_SHORT   // K4 on short block rows: fewer warps, larger chunks (fewer S flushes)
#define BMV_K4_WARPS_SHORT 8
#endif
#ifndef BMV_K5_WARPS
#define BMV_K5_WARPS 16
#endif
#ifndef BMV_SPMM_BUFS
#define BMV_SPMM_BUFS 2
#endif
constexpr int kNB = BMV_SPMM_BUFS;    // buffers per warp (kNB - 1 chunks in flight)
constexpr int kSmemBytes = 224 * 1024;
template <int CW_>
struct Shape {
  static constexpr int CW = CW_;
  // bytes per buffer = the largest chunk [meta | A | B] the planner may build
  static constexpr int BUF = kSmemBytes / (CW * kNB) / 128 * 128;
};
// kernel shapes per product: variant 0 (default), 1 (short block rows)
constexpr int kWarpsOf[2][2] = {{BMV_K4_WARPS, BMV_K4_WARPS_SHORT}, {BMV_K5_WARPS, BMV_K5_WARPS}};
__host__ constexpr int buf_of(int kind, int variant) {
  return kSmemBytes / (kWarpsOf[kind - 4][variant] * kNB) / 128 * 128;
}

// Per-chunk copy descriptor (built once in bmv_chunk_plan_create), 32 bytes:
// one sector, loaded by the claiming warp a pipeline step ahead of its use.
struct __align__(16) ChunkDesc {
  uint32_t m16, a16, b16;  // first meta word / A element / B element, 16-byte units
  uint32_t mb, ab, bb;     // bytes of meta, A, B (multiples of 16)
  uint32_t pad[2];
};

struct ChunkArgs {
  const int64_t* part_start;  // n_parts + 1
  const ChunkDesc* desc;
  const int32_t* meta;
};

// Chunk header (int32): see include/bmv.h (bmv_chunk_desc)
enum { H_NSEG = 0, H_NROWS, H_UA, H_UB, H_NK, H_AOFF, H_BOFF, H_SEG, H_CMA, H_CMB, H_RB, H_KK,
       H_ST };

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Warp-wide copy of `bytes` (multiple of 16) from global to shared memory:
// rows of 512 bytes, lane l moving bytes [16 l, 16 l + 16) of every row.
__device__ __forceinline__ void warp_copy(unsigned dst, const char* src, unsigned bytes, int lane) {
  const char* p = src + lane * 16;
  unsigned d = dst + lane * 16u;
  int rows = (int)(bytes >> 9);
  for (; rows >= 4; rows -= 4, p += 2048, d += 2048u) {
    cp_async16(d, p);
    cp_async16(d + 512u, p + 512);
    cp_async16(d + 1024u, p + 1024);
    cp_async16(d + 1536u, p + 1536);
  }
  for (; rows > 0; --rows, p += 512, d += 512u) cp_async16(d, p);
  if (lane * 16u < (bytes & 511u)) cp_async16(d, p);
}

// Byte offset (in the chunk buffer) of an 8-byte zero: header words 14, 15.
constexpr int kZeroByte = 56;

// ---------------------------------------------------------------- K4 -----
// S[rb[a] + st[kk[a]][b]] += sum_rows A[row][cma[seg][a]] * B[row][cmb[seg][b]]
// One pass: union columns [ag, ag + 8 TA) x [bg, bg + 8 TB); accumulators
// live in registers over every segment of the chunk.  Segments are padded
// to multiples of 4 rows (a DMMA k-step never straddles two block rows).
// UNR: k-loop unroll (fragment loads in flight): 4 pays on long block rows, 1 on short ones
template <int TA, int TB, int UNR>
__device__ __forceinline__ void k4_pass(const int32_t* m, double* __restrict__ c, int ag, int bg,
                                        int lane) {
  const int nseg = m[H_NSEG], ua = m[H_UA], ub = m[H_UB];
  const char* st = reinterpret_cast<const char*>(m);
  const int aoff = m[H_AOFF], boff = m[H_BOFF];
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
    const int kb = seg[2 * s + 1].x;
    const int nrows = r0.x, ka = r0.z;
    // per-lane fragment addresses (bytes in the buffer) and k-step strides; a
    // union column this segment does not store reads the buffer's zero, stride 0
    int pa[TA], sa[TA], pb[TB], sb[TB];
#pragma unroll
    for (int t = 0; t < TA; ++t) {
      const int aa = ag + t * 8 + g4;
      const int sl = aa < ua ? cma[s * ua + aa] : -1;
      pa[t] = sl >= 0 ? aoff + 8 * (r0.y + t4 * ka + sl) : kZeroByte;
      sa[t] = sl >= 0 ? 32 * ka : 0;
    }
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const int bb = bg + u * 8 + g4;
      const int sl = bb < ub ? cmb[s * ub + bb] : -1;
      pb[u] = sl >= 0 ? boff + 8 * (r0.w + t4 * kb + sl) : kZeroByte;
      sb[u] = sl >= 0 ? 32 * kb : 0;
    }
    const int full = nrows >> 2;
#pragma unroll UNR
    for (int ks = 0; ks < full; ++ks) {
      double av[TA], bv[TB];
#pragma unroll
      for (int t = 0; t < TA; ++t) {
        av[t] = *reinterpret_cast<const double*>(st + pa[t]);
        pa[t] += sa[t];
      }
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        bv[u] = *reinterpret_cast<const double*>(st + pb[u]);
        pb[u] += sb[u];
      }
#pragma unroll
      for (int t = 0; t < TA; ++t)
#pragma unroll
        for (int u = 0; u < TB; ++u) dmma_8x8x4(acc[t][u][0], acc[t][u][1], av[t], bv[u]);
    }
    if (nrows & 3) {  // last k-step: rows past the segment contribute zeros
      const bool rok = t4 < (nrows & 3);
      double av[TA], bv[TB];
#pragma unroll
      for (int t = 0; t < TA; ++t) av[t] = rok ? *reinterpret_cast<const double*>(st + pa[t]) : 0.0;
#pragma unroll
      for (int u = 0; u < TB; ++u) bv[u] = rok ? *reinterpret_cast<const double*>(st + pb[u]) : 0.0;
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
    double* crow = c + rb[aa];
    const int32_t* srow = stt + kk[aa] * ub;
#pragma unroll
    for (int u = 0; u < TB; ++u) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int bb = bg + u * 8 + 2 * t4 + e;
        if (bb < ub) {
          const int sl = srow[bb];
          if (sl >= 0) atomicAdd(crow + sl, acc[t][u][e]);
        }
      }
    }
  }
}

template <int TA, int UNR>
__device__ __forceinline__ void k4_pass_b(const int32_t* m, double* c, int ag, int bg, int tb,
                                          int lane) {
  switch (tb) {
    case 1: k4_pass<TA, 1, UNR>(m, c, ag, bg, lane); break;
    case 2: k4_pass<TA, 2, UNR>(m, c, ag, bg, lane); break;
    case 3: k4_pass<TA, 3, UNR>(m, c, ag, bg, lane); break;
    default: k4_pass<TA, 4, UNR>(m, c, ag, bg, lane); break;
  }
}

template <int UNR>
__device__ __forceinline__ void k4_chunk(const char* st, double* __restrict__ c, int lane) {
  const int32_t* m = reinterpret_cast<const int32_t*>(st);
  const int ua = m[H_UA], ub = m[H_UB];
  for (int ag = 0; ag < ua; ag += 32) {
    const int ta = min(4, (ua - ag + 7) >> 3);
    for (int bg = 0; bg < ub; bg += 32) {
      const int tb = min(4, (ub - bg + 7) >> 3);
      switch (ta) {
        case 1: k4_pass_b<1, UNR>(m, c, ag, bg, tb, lane); break;
        case 2: k4_pass_b<2, UNR>(m, c, ag, bg, tb, lane); break;
        case 3: k4_pass_b<3, UNR>(m, c, ag, bg, tb, lane); break;
        default: k4_pass_b<4, UNR>(m, c, ag, bg, tb, lane); break;
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
  const int aoff = m[H_AOFF];
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
      const double* cbase = cmat + (okk ? cb[ka] : 0);
      const int32_t* crow = ct + (okk ? ck[ka] : 0) * ub;
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int bb = bg + u * 8 + g4;
        double v = 0.0;
        if (okk && bb < ub) {
          const int sl = crow[bb];
          if (sl >= 0) v = __ldg(cbase + sl);
        }
        bf[ks][u] = v;
      }
    }
    const bool add_old = accumulate || ag > 0;
    for (int s = 0; s < nseg; ++s) {
      const int4 r0 = seg[2 * s];
      const int ky = seg[2 * s + 1].x;
      const int nrows = r0.x, ka = r0.z;
      // per-lane A fragment addresses (bytes in the buffer) / row-tile strides;
      // a union column this segment does not store reads the buffer's zero
      int pa[KS], sa[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int aa = ag + ks * 4 + t4;
        const int sl = aa < ua ? cma[s * ua + aa] : -1;
        pa[ks] = sl >= 0 ? aoff + 8 * (r0.y + g4 * ka + sl) : kZeroByte;
        sa[ks] = sl >= 0 ? 64 * ka : 0;
      }
      int sy[TB][2];
#pragma unroll
      for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = bg + u * 8 + 2 * t4 + e;
          sy[u][e] = bb < ub ? cmy[s * ub + bb] : -1;
        }
      double* yrow = y + (int64_t)r0.w + (int64_t)g4 * ky;
      // one 8-row tile; FULL: every row of the tile belongs to the segment
      auto tile = [&](auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        const bool rok = FULL || g4 < (nrows & 7);
        double acc[TB][2];
#pragma unroll
        for (int u = 0; u < TB; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double av = rok ? *reinterpret_cast<const double*>(st + pa[ks]) : 0.0;
          pa[ks] += sa[ks];
#pragma unroll
          for (int u = 0; u < TB; ++u) dmma_8x8x4(acc[u][0], acc[u][1], av, bf[ks][u]);
        }
        if (rok) {
#pragma unroll
          for (int u = 0; u < TB; ++u)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (sy[u][e] >= 0) {
                double* yp = yrow + sy[u][e];
                double v = alpha * acc[u][e];
                if (add_old) v += *yp;
                *yp = v;
              }
        }
        yrow += 8 * ky;
      };
      const int full = nrows >> 3;
      for (int rt = 0; rt < full; ++rt) tile(std::true_type{});
      if (nrows & 7) tile(std::false_type{});  // last tile: rows past the segment are skipped
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
    else if (tb == 3 || TBMAX == 3) k5_pass<(TBMAX > 2 ? 3 : 2), KS>(m, cmat, y, alpha, accumulate, bg, lane);
    else k5_pass<(TBMAX > 3 ? 4 : TBMAX), KS>(m, cmat, y, alpha, accumulate, bg, lane);
  }
}

__device__ __forceinline__ void k5_chunk(const char* st, const double* __restrict__ cmat,
                                         double* __restrict__ y, double alpha, bool accumulate,
                                         int lane) {
  const int32_t* m = reinterpret_cast<const int32_t*>(st);
  const int ua = m[H_UA];
  if (ua <= 8) k5_passes<2, 4>(m, cmat, y, alpha, accumulate, lane);
  else if (ua <= 16) k5_passes<4, 4>(m, cmat, y, alpha, accumulate, lane);
  else if (ua <= 24) k5_passes<6, 3>(m, cmat, y, alpha, accumulate, lane);
  else k5_passes<8, 2>(m, cmat, y, alpha, accumulate, lane);
}

template <int KIND, int CW>  // KIND 4: K4, 5: K5; CW warps per CTA
__global__ void __launch_bounds__(CW * 32, 1)
    chunk_kernel(const ChunkArgs g, const double* __restrict__ a, const double* __restrict__ b,
                 double* __restrict__ out, double alpha, int accumulate) {
  constexpr int kBufBytes = Shape<CW>::BUF;
  extern __shared__ __align__(128) char smem[];
  __shared__ int next_chunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = g.part_start[blockIdx.x];
  const int n = (int)(g.part_start[blockIdx.x + 1] - c0);
  if (threadIdx.x == 0) next_chunk = 0;
  __syncthreads();
  char* mybuf = smem + (size_t)warp * kNB * kBufBytes;
  const unsigned mybuf_s = smem_u32(mybuf);

  // claim the next chunk of this CTA (in order: the chunks of a part are
  // consecutive in memory) and load its descriptor
  uint4 d0 = make_uint4(0, 0, 0, 0);
  uint2 d1 = make_uint2(0, 0);
  bool have = false;
  auto claim = [&]() {
    int jj = 0;
    if (lane == 0) jj = atomicAdd(&next_chunk, 1);
    jj = __shfl_sync(~0u, jj, 0);
    have = jj < n;
    if (have) {
      const ChunkDesc* d = g.desc + c0 + jj;
      d0 = __ldg(reinterpret_cast<const uint4*>(d));
      d1 = __ldg(reinterpret_cast<const uint2*>(d) + 2);
    }
  };
  // copy the claimed chunk into buffer `buf` (one cp.async group, possibly empty)
  auto issue = [&](int buf) {
    if (have) {
      const unsigned dst = mybuf_s + (unsigned)buf * kBufBytes;
      warp_copy(dst, reinterpret_cast<const char*>(g.meta) + (size_t)d0.x * 16, d0.w, lane);
      warp_copy(dst + d0.w, reinterpret_cast<const char*>(a) + (size_t)d0.y * 16, d1.x, lane);
      if (KIND == 4)
        warp_copy(dst + d0.w + d1.x, reinterpret_cast<const char*>(b) + (size_t)d0.z * 16, d1.y,
                  lane);
    }
    cp_commit();
  };

  // prologue: kNB - 1 chunks in flight, the descriptor of the next one loading
  bool valid[kNB];
#pragma unroll
  for (int i = 0; i < kNB - 1; ++i) {
    claim();
    valid[i] = have;
    issue(i);
  }
  claim();
  int cur = 0;
  while (valid[0]) {
    // refill the buffer freed in the previous step, then claim one step ahead
    int nb = cur + kNB - 1;
    if (nb >= kNB) nb -= kNB;
    valid[kNB - 1] = have;
    issue(nb);
    claim();
    cp_wait<kNB - 1>();
    __syncwarp();
    const char* st = mybuf + (size_t)cur * kBufBytes;
    if (KIND == 4) k4_chunk<(CW == BMV_K4_WARPS_SHORT ? 1 : 4)>(st, out, lane);
    else k5_chunk(st, b, out, alpha, accumulate != 0, lane);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kNB - 1; ++i) valid[i] = valid[i + 1];
    if (++cur == kNB) cur = 0;
  }
  cp_wait<0>();
}

}  // namespace

struct ChunkPlan {
  int kind = 0;
  int variant = 0;  // kernel shape: the smallest buffers that hold the plan's chunks
  int n_parts = 0;
  int64_t n_chunks = 0;
  int64_t* part_start = nullptr;
  ChunkDesc* desc = nullptr;
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
      d->stage_bytes <= 0 || (d->stage_bytes & 15) ||
      d->stage_bytes > std::max(buf_of(d->kind, 0), buf_of(d->kind, 1))) {
    set_error("bmv_chunk_plan_create: invalid descriptor (chunks of at most %d bytes)",
              d && (d->kind == 4 || d->kind == 5) ? std::max(buf_of(d->kind, 0), buf_of(d->kind, 1))
                                                  : 0);
    return BMV_ERR_INVALID;
  }
  // per-chunk copy descriptors
  const size_t nc = (size_t)d->n_chunks;
  std::vector<ChunkDesc> desc(nc);
  for (size_t j = 0; j < nc; ++j) {
    const int64_t m0 = d->chunk_meta[j];
    const int64_t words = d->chunk_meta[j + 1] - m0;
    const int64_t a0 = d->chunk_a[2 * j], an = d->chunk_a[2 * j + 1] - a0;
    int64_t b0 = 0, bn = 0;
    if (d->kind == 4) {
      b0 = d->chunk_b[2 * j];
      bn = d->chunk_b[2 * j + 1] - b0;
    }
    const int32_t* h = d->meta + m0;
    if (words < 16 || (words & 3) || (m0 & 3) || (a0 & 1) || (an & 1) || (b0 & 1) || (bn & 1) ||
        an < 0 || bn < 0 || 4 * words + 8 * (an + bn) > d->stage_bytes || h[5] != 4 * words ||
        h[6] != 4 * words + 8 * an || m0 / 4 > UINT32_MAX || a0 / 2 > UINT32_MAX ||
        b0 / 2 > UINT32_MAX) {
      set_error("bmv_chunk_plan_create: chunk %lld does not fit its buffer", (long long)j);
      return BMV_ERR_INVALID;
    }
    desc[j] = ChunkDesc{(uint32_t)(m0 / 4), (uint32_t)(a0 / 2), (uint32_t)(b0 / 2),
                        (uint32_t)(4 * words), (uint32_t)(8 * an), (uint32_t)(8 * bn), {0, 0}};
  }
  if (d->part_chunk_start[d->n_parts] - d->part_chunk_start[0] != d->n_chunks) {
    set_error("bmv_chunk_plan_create: parts do not cover the chunks");
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_chunk_plan();
  p->kind = d->kind;
  p->variant = d->stage_bytes <= std::min(buf_of(d->kind, 0), buf_of(d->kind, 1))
                   ? (buf_of(d->kind, 0) <= buf_of(d->kind, 1) ? 0 : 1)
                   : (buf_of(d->kind, 0) >= d->stage_bytes ? 0 : 1);
  p->n_parts = d->n_parts;
  p->n_chunks = d->n_chunks;
  int rc = upload(d->part_chunk_start, (int64_t)d->n_parts + 1, &p->part_start);
  if (rc == BMV_OK) rc = upload(d->meta, d->meta_len, &p->meta);
  if (rc == BMV_OK) rc = upload(desc.data(), d->n_chunks, &p->desc);
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
  bmv::release(p->desc);
  bmv::release(p->meta);
  delete p;
  return BMV_OK;
}

static int launch_chunks(const bmv_chunk_plan* p, const double* a, const double* b, double* out,
                         double alpha, int accumulate, void* stream) {
  using namespace bmv;
  if (p->n_chunks == 0) return BMV_OK;
  if ((reinterpret_cast<uintptr_t>(a) & 15) || (p->kind == 4 && (reinterpret_cast<uintptr_t>(b) & 15))) {
    set_error("K4/K5: value arrays must be 16-byte aligned");
    return BMV_ERR_INVALID;
  }
  ChunkArgs g{p->part_start, p->desc, p->meta};
  cudaStream_t st = as_stream(stream);
#define BMV_LAUNCH_CHUNKS(KIND, CW)                                                               \
  do {                                                                                           \
    constexpr int smem = CW * kNB * Shape<CW>::BUF;                                               \
    BMV_CUDA_TRY(cudaFuncSetAttribute(chunk_kernel<KIND, CW>,                                     \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));        \
    chunk_kernel<KIND, CW><<<p->n_parts, CW * 32, smem, st>>>(g, a, b, out, alpha, accumulate);   \
  } while (0)
  if (p->kind == 4) {
    if (p->variant == 0) BMV_LAUNCH_CHUNKS(4, BMV_K4_WARPS);
    else BMV_LAUNCH_CHUNKS(4, BMV_K4_WARPS_SHORT);
  } else {
    BMV_LAUNCH_CHUNKS(5, BMV_K5_WARPS);
  }
#undef BMV_LAUNCH_CHUNKS
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

int bmv_chunk_kernel_config(int32_t kind, int32_t variant, int32_t* warps, int32_t* buffer_bytes) {
  if ((kind != 4 && kind != 5) || variant < 0 || variant > 1) {
    bmv::set_error("bmv_chunk_kernel_config: kind must be 4 or 5, variant 0 or 1");
    return BMV_ERR_INVALID;
  }
  *warps = bmv::kWarpsOf[kind - 4][variant];
  *buffer_bytes = bmv::buf_of(kind, variant);
  return BMV_OK;
}

}  // extern "C"
