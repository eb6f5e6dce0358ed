// K4 (projection C = A^T B, reference tmmult, bcsr.py:631-667) and
// K5 (post-multiply C = alpha A B, reference mmult, bcsr.py:587-628) on the
// block-CSR storage of the reference (padded row-major blocks).
//
// K4: the triples (block row i, A_ik, B_il) are cut into segments = one
// output block within one chunk of consecutive block rows (the rows of a
// chunk are spatial neighbours, so their A/B blocks are read from L1/L2 by
// the warps of the same wave).  One warp per segment accumulates a partial
// block in registers; a second kernel sums each output block's partials in
// chunk order.  K5: one warp per output block Y_ij accumulates
// sum_k A_ik C_kj in registers.  Every output value is written once, in a
// fixed order: no atomics, bit-reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bmv_common.cuh"

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st);
}

using namespace bmv;

namespace {

struct TmArgs {
  const int64_t* __restrict__ out_off;
  const int32_t* __restrict__ out_rows;
  const int32_t* __restrict__ out_cols;
  const int32_t* __restrict__ out_stride;
  const int64_t* __restrict__ out_seg_start;
  const int64_t* __restrict__ out_seg_list;
  const int64_t* __restrict__ chunk_a;
  const int64_t* __restrict__ chunk_b;
  const int64_t* __restrict__ chunk_seg_start;
  const int64_t* __restrict__ seg_out;
  const int64_t* __restrict__ seg_tri_start;
  const int64_t* __restrict__ seg_poff;
  const int32_t* __restrict__ tri_a_soff;
  const int32_t* __restrict__ tri_b_soff;
  const int32_t* __restrict__ tri_rows;
  const int32_t* __restrict__ tri_a_stride;
  const int32_t* __restrict__ tri_b_stride;
  const double* __restrict__ a;
  const double* __restrict__ b;
  double* __restrict__ partial;
  double* __restrict__ c;
  const int32_t* __restrict__ chunk_ids;  // blockIdx -> chunk (size class launch)
  double* __restrict__ partial2;          // second-level partials [out][split][256]
  int splits;                             // second-level splits per output block
};

constexpr int kRedSeg = 64;  // segments per first-level reduction CTA

// ---- 1D TMA bulk copies (cp.async.bulk, SASS UBLKCP) completed on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// FP64 tensor-core MMA (DMMA): D(8x8) = A(8x4, row) * B(4x8, col) + C.
// Fragments (lane = 4 * gid + tig): A[gid][tig], B[tig][gid], C/D[gid][2 tig + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Stage n doubles from global src to shared dst: one elected thread issues
// TMA bulk copies (16-byte granules, 32 KB pieces) when both ends are
// 16-byte aligned and n is even; otherwise all threads copy.  Returns after
// the data is visible to the whole CTA.
__device__ __forceinline__ void stage_ranges(double* d0, const double* s0, int n0, double* d1,
                                             const double* s1, int n1, uint64_t* bar) {
  const bool bulk = ((smem_u32(d0) | smem_u32(d1)) & 15) == 0 &&
                    ((reinterpret_cast<uintptr_t>(s0) | reinterpret_cast<uintptr_t>(s1)) & 15) == 0 &&
                    ((n0 | n1) & 1) == 0;
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      mbar_expect_tx(bar, (unsigned)(n0 + n1) * 8u);
      constexpr int kPiece = 4096;  // doubles per bulk copy
      for (int i = 0; i < n0; i += kPiece)
        bulk_g2s(d0 + i, s0 + i, (unsigned)min(kPiece, n0 - i) * 8u, bar);
      for (int i = 0; i < n1; i += kPiece)
        bulk_g2s(d1 + i, s1 + i, (unsigned)min(kPiece, n1 - i) * 8u, bar);
    }
    __syncthreads();  // barrier initialised before anyone waits
    mbar_wait(bar, 0);
  } else {
    for (int i = threadIdx.x; i < n0; i += blockDim.x) d0[i] = __ldg(s0 + i);
    for (int i = threadIdx.x; i < n1; i += blockDim.x) d1[i] = __ldg(s1 + i);
    __syncthreads();
  }
}

constexpr int kTmWarps = 8;

// One CTA per chunk of consecutive block rows: stage the chunk's A and B
// blocks (two contiguous ranges) in shared memory with coalesced loads, then
// one warp per segment accumulates sum_triples sum_r A[r][k] B[r][l] for its
// output block; EPT entries per lane (EPT * 32 >= entries of the block).
template <int EPT>
__global__ void __launch_bounds__(kTmWarps * 32) tm_chunk_kernel(const TmArgs g) {
  extern __shared__ __align__(16) double stage[];
  const int64_t ch = g.chunk_ids ? g.chunk_ids[blockIdx.x] : blockIdx.x;
  const int64_t a_lo = g.chunk_a[2 * ch], b_lo = g.chunk_b[2 * ch];
  const int na = (int)(g.chunk_a[2 * ch + 1] - a_lo);
  const int nb = (int)(g.chunk_b[2 * ch + 1] - b_lo);
  __shared__ uint64_t bar;
  double* SA = stage;
  double* SB = stage + na;
  stage_ranges(SA, g.a + a_lo, na, SB, g.b + b_lo, nb, &bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s_end = g.chunk_seg_start[ch + 1];
  for (int64_t sg = g.chunk_seg_start[ch] + warp; sg < s_end; sg += kTmWarps) {
    const int64_t o = g.seg_out[sg];
    const int cols = g.out_cols[o];
    const int ent = g.out_rows[o] * cols;
    int ii[EPT], jj[EPT];
    double acc[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int e = lane + 32 * k;
      ii[k] = e < ent ? e / cols : 0;
      jj[k] = e < ent ? e - (e / cols) * cols : 0;
      acc[k] = 0.0;
    }
    const int64_t t1 = g.seg_tri_start[sg + 1];
    for (int64_t t = g.seg_tri_start[sg]; t < t1; ++t) {
      const double* A = SA + g.tri_a_soff[t];
      const double* B = SB + g.tri_b_soff[t];
      const int as = g.tri_a_stride[t], bs = g.tri_b_stride[t], nr = g.tri_rows[t];
#pragma unroll 2
      for (int r = 0; r < nr; ++r) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) acc[k] = fma(A[r * as + ii[k]], B[r * bs + jj[k]], acc[k]);
      }
    }
    double* P = g.partial + g.seg_poff[sg];
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (lane + 32 * k < ent) P[lane + 32 * k] = acc[k];
  }
}

// Issue the TMA bulk copies of chunk ch (A range then B range) into dst,
// completing on bar (called by one thread).
__device__ __forceinline__ void issue_chunk(const double* a, const int64_t* ca, const double* b,
                                            const int64_t* cb, int64_t ch, double* dst,
                                            uint64_t* bar) {
  const int64_t a_lo = ca[2 * ch], b_lo = cb ? cb[2 * ch] : 0;
  const int na = (int)(ca[2 * ch + 1] - a_lo);
  const int nb = cb ? (int)(cb[2 * ch + 1] - b_lo) : 0;
  mbar_expect_tx(bar, (unsigned)(na + nb) * 8u);
  constexpr int kPiece = 4096;
  for (int i = 0; i < na; i += kPiece)
    bulk_g2s(dst + i, a + a_lo + i, (unsigned)min(kPiece, na - i) * 8u, bar);
  for (int i = 0; i < nb; i += kPiece)
    bulk_g2s(dst + na + i, b + b_lo + i, (unsigned)min(kPiece, nb - i) * 8u, bar);
}

// Fast path for output blocks of at most 8 x 8, one chunk per CTA (TMA-staged).
// lane = slice * 8 + i: the 4 slices split the block rows (r = slice,
// slice + 4, ...), lane (slice, i) accumulates output row i in registers;
// slices are summed with two xor-shuffles.
__device__ __forceinline__ void tm_chunk_compute8(const TmArgs& g, int64_t ch, const double* SA,
                                                  const double* SB) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t s_end = g.chunk_seg_start[ch + 1];
  for (int64_t sg = g.chunk_seg_start[ch] + warp; sg < s_end; sg += kTmWarps) {
    const int64_t o = g.seg_out[sg];
    const int rows = g.out_rows[o], cols = g.out_cols[o];
    // S(k, l) += sum_r A[r][k] B[r][l]: M = k (8), N = l (8), K = r in steps of 4
    double d0 = 0.0, d1 = 0.0;
    const int64_t t1 = g.seg_tri_start[sg + 1];
    for (int64_t t = g.seg_tri_start[sg]; t < t1; ++t) {
      const double* A = SA + g.tri_a_soff[t] + gid;
      const double* B = SB + g.tri_b_soff[t] + gid;
      const int as = g.tri_a_stride[t], bs = g.tri_b_stride[t], nr = g.tri_rows[t];
      // warp-uniform loop bounds (mma.sync needs every lane)
      int r0 = 0;
      for (; r0 + 8 <= nr; r0 += 8) {  // two k-steps per iteration
        const int r = r0 + tig;
        dmma_8x8x4(d0, d1, A[r * as], B[r * bs]);
        dmma_8x8x4(d0, d1, A[(r + 4) * as], B[(r + 4) * bs]);
      }
      for (; r0 < nr; r0 += 4) {
        const int rr = r0 + tig;
        const bool in = rr < nr;
        dmma_8x8x4(d0, d1, in ? A[rr * as] : 0.0, in ? B[rr * bs] : 0.0);
      }
    }
    if (gid < rows) {
      double* P = g.partial + g.seg_poff[sg] + gid * cols;
      if (2 * tig < cols) P[2 * tig] = d0;
      if (2 * tig + 1 < cols) P[2 * tig + 1] = d1;
    }
  }
}

__global__ void __launch_bounds__(kTmWarps * 32) tm_chunk_kernel8_1(const TmArgs g) {
  extern __shared__ __align__(16) double stage[];
  __shared__ uint64_t bar;
  const int64_t ch = g.chunk_ids ? g.chunk_ids[blockIdx.x] : blockIdx.x;
  const int64_t a_lo = g.chunk_a[2 * ch], b_lo = g.chunk_b[2 * ch];
  const int na = (int)(g.chunk_a[2 * ch + 1] - a_lo);
  const int nb = (int)(g.chunk_b[2 * ch + 1] - b_lo);
  double* SA = stage;
  double* SB = stage + na;
  stage_ranges(SA, g.a + a_lo, na, SB, g.b + b_lo, nb, &bar);
  tm_chunk_compute8(g, ch, SA, SB);
}

// Persistent variant: each CTA walks its chunks (ids[blockIdx.x + k gridDim.x])
// through a kStages-deep ring of TMA-filled stages, so the next chunks stream
// in while the current one is computed.
constexpr int kStages = 3;
#ifndef BMV_PERSISTENT
#define BMV_PERSISTENT 0
#endif
constexpr bool kPersistent = BMV_PERSISTENT != 0;

__global__ void __launch_bounds__(kTmWarps * 32) tm_chunk_kernel8_p(const TmArgs g, int64_t n_list,
                                                                     int stage_doubles) {
  extern __shared__ __align__(16) double stage[];
  __shared__ uint64_t bars[kStages];
  if (threadIdx.x == 0)
    for (int q = 0; q < kStages; ++q) mbar_init(&bars[q], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < kStages; ++q) {
      const int64_t idx = blockIdx.x + (int64_t)q * gridDim.x;
      if (idx < n_list)
        issue_chunk(g.a, g.chunk_a, g.b, g.chunk_b, g.chunk_ids[idx], stage + q * stage_doubles,
                    &bars[q]);
    }
  }
  for (int it = 0;; ++it) {
    const int64_t idx = blockIdx.x + (int64_t)it * gridDim.x;
    if (idx >= n_list) break;
    const int q = it % kStages;
    mbar_wait(&bars[q], (it / kStages) & 1);
    const int64_t ch = g.chunk_ids[idx];
    const double* SA = stage + q * stage_doubles;
    tm_chunk_compute8(g, ch, SA, SA + (g.chunk_a[2 * ch + 1] - g.chunk_a[2 * ch]));
    __syncthreads();  // stage q fully consumed
    if (threadIdx.x == 0) {
      const int64_t nidx = idx + (int64_t)kStages * gridDim.x;
      if (nidx < n_list)
        issue_chunk(g.a, g.chunk_a, g.b, g.chunk_b, g.chunk_ids[nidx], stage + q * stage_doubles,
                    &bars[q]);
    }
  }
}

// Fast path for output blocks of at most 8 x 8, persistent over chunks with
// a double-buffered TMA stage (chunk k+1 streams in while chunk k is
// computed).  lane = slice * 8 + i: the 4 slices split the block rows
// (r = slice, slice + 4, ...), lane (slice, i) accumulates output row i
// (8 entries) in registers; slices are summed with two xor-shuffles.
__global__ void __launch_bounds__(kTmWarps * 32) tm_chunk_kernel8(const TmArgs g, int64_t n_chunks,
                                                                   int buf_doubles) {
  extern __shared__ __align__(16) double stage[];
  __shared__ uint64_t bars[2];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();
  int64_t ch = blockIdx.x;
  if (threadIdx.x == 0 && ch < n_chunks) issue_chunk(g.a, g.chunk_a, g.b, g.chunk_b, ch, stage, &bars[0]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slice = lane >> 3, i = lane & 7;
  for (int it = 0; ch < n_chunks; ch += gridDim.x, ++it) {
    const int bsel = it & 1;
    const int64_t nx = ch + gridDim.x;
    if (threadIdx.x == 0 && nx < n_chunks)
      issue_chunk(g.a, g.chunk_a, g.b, g.chunk_b, nx, stage + (bsel ^ 1) * buf_doubles,
                  &bars[bsel ^ 1]);
    mbar_wait(&bars[bsel], (it >> 1) & 1);
    const double* SA = stage + bsel * buf_doubles;
    const double* SB = SA + (g.chunk_a[2 * ch + 1] - g.chunk_a[2 * ch]);
    const int64_t s_end = g.chunk_seg_start[ch + 1];
    for (int64_t sg = g.chunk_seg_start[ch] + warp; sg < s_end; sg += kTmWarps) {
      const int64_t o = g.seg_out[sg];
      const int rows = g.out_rows[o], cols = g.out_cols[o];
      const int ii = i < rows ? i : 0;
      double acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.0;
      const int64_t t1 = g.seg_tri_start[sg + 1];
      for (int64_t t = g.seg_tri_start[sg]; t < t1; ++t) {
        const double* A = SA + g.tri_a_soff[t];
        const double* B = SB + g.tri_b_soff[t];
        const int as = g.tri_a_stride[t], bs = g.tri_b_stride[t], nr = g.tri_rows[t];
        for (int r = slice; r < nr; r += 4) {
          const double av = A[r * as + ii];
          const double* br = B + r * bs;
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = fma(av, br[j], acc[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 8);
        acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 16);
      }
      if (slice == 0 && i < rows) {
        double* P = g.partial + g.seg_poff[sg] + i * cols;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < cols) P[j] = acc[j];
      }
    }
    __syncthreads();  // buffer bsel fully consumed before it is refilled
  }
}

// Two-level deterministic reduction of the segment partials.  The partials
// of one output block are contiguous, in chunk order (laid out so by the
// plan).  Level 1: CTA (o, split) sums kRedSeg consecutive segments of o,
// thread group `part` taking segments part, part + parts, ... (coalesced,
// no indirection), groups added in a fixed order.  Level 2: one CTA per o
// adds the splits in order and writes the C block.
__global__ void __launch_bounds__(256) tm_reduce1_kernel(const TmArgs g) {
  __shared__ double red[256];
  const int64_t o = blockIdx.x;
  const int split = blockIdx.y;
  const int cols = g.out_cols[o];
  const int ent = g.out_rows[o] * cols;
  const int e_div = max(ent, 1);
  const int parts = max(1, (int)blockDim.x / e_div);
  const int part = threadIdx.x / e_div, e = threadIdx.x - part * e_div;
  const int64_t nseg = g.out_seg_start[o + 1] - g.out_seg_start[o];
  const int64_t k0 = (int64_t)split * kRedSeg, k1 = min(nseg, k0 + kRedSeg);
  double acc = 0.0;
  if (part < parts && e < ent && k0 < k1) {
    const double* P = g.partial + g.seg_poff[g.out_seg_list[g.out_seg_start[o]]];
    for (int64_t k = k0 + part; k < k1; k += parts) acc += P[k * ent + e];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int q = threadIdx.x; q < ent; q += blockDim.x) {
    double sum = 0.0;
    for (int pp = 0; pp < parts; ++pp) sum += red[pp * ent + q];
    g.partial2[((int64_t)o * g.splits + split) * 256 + q] = sum;
  }
}

__global__ void __launch_bounds__(256) tm_reduce2_kernel(const TmArgs g) {
  const int64_t o = blockIdx.x;
  const int cols = g.out_cols[o], cst = g.out_stride[o];
  const int ent = g.out_rows[o] * cols;
  for (int q = threadIdx.x; q < ent; q += blockDim.x) {
    double sum = 0.0;
    for (int sp = 0; sp < g.splits; ++sp) sum += g.partial2[((int64_t)o * g.splits + sp) * 256 + q];
    const int i = q / cols, j = q - i * cols;
    g.c[g.out_off[o] + (int64_t)i * cst + j] = sum;
  }
}

struct MmArgs {
  const int64_t* __restrict__ chunk_a;
  const int64_t* __restrict__ chunk_out_start;
  const int64_t* __restrict__ out_off;
  const int32_t* __restrict__ out_rows;
  const int32_t* __restrict__ out_cols;
  const int32_t* __restrict__ out_stride;
  const int64_t* __restrict__ pair_start;
  const int32_t* __restrict__ pair_a_soff;
  const int32_t* __restrict__ pair_a_stride;
  const int32_t* __restrict__ pair_inner;
  const int64_t* __restrict__ pair_b_off;
  const int32_t* __restrict__ pair_b_stride;
  const double* __restrict__ a;
  const double* __restrict__ b;
  double* __restrict__ c;
  double alpha;
  int accumulate;
  const int32_t* __restrict__ chunk_ids;  // blockIdx -> chunk (size class launch)
  int all_inner8;                         // every inner block has 8 columns (fast path)
};

constexpr int kMmWarps = 8;

// One CTA per chunk of block rows: stage A (one contiguous range), then one
// warp per output block: C(i,j)[r][s] (+)= alpha * sum_pairs sum_k A[r][k] B[k][s].
// Each B block (<= 16 x 16) is staged in warp-private shared memory; lanes
// own entries e = lane + 32 m of the output block, EPT at a time.
constexpr int kMmEPT = 8;
constexpr int kMmBMax = 256;  // doubles per staged B block

// 8 x 8 inner/outer fast path on FP64 tensor cores: the output block (rows x 8)
// is cut into 8-row tiles (<= 16 tiles held in registers); per (A_ik, C_kj)
// pair the C block is two B fragments (k = 0..3, 4..7) loaded once, each
// tile takes two DMMA k-steps with A rows from the shared stage.
constexpr int kMmTiles = 64;  // rows <= 512 on the fast path

__device__ __forceinline__ void mm_block8(const MmArgs& g, int64_t o, const double* SA, int lane) {
  const int rows = g.out_rows[o], cst = g.out_stride[o];
  const int64_t p0 = g.pair_start[o], p1 = g.pair_start[o + 1];
  const int gid = lane >> 2, tig = lane & 3;
  for (int r0 = 0; r0 < rows; r0 += 8) {  // 8-row tiles, warp-uniform
    const int r = r0 + gid;
    const bool in = r < rows;
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t p = p0; p < p1; ++p) {
      const double* Bg = g.b + g.pair_b_off[p] + gid;  // C block: L1/L2 resident
      const int bs = g.pair_b_stride[p];
      const double b0 = __ldg(Bg + (int64_t)tig * bs), b1 = __ldg(Bg + (int64_t)(4 + tig) * bs);
      const double* A = SA + g.pair_a_soff[p] + tig + r * g.pair_a_stride[p];
      const double a0 = in ? A[0] : 0.0, a1 = in ? A[4] : 0.0;
      dmma_8x8x4(acc0, acc1, a0, b0);
      dmma_8x8x4(acc0, acc1, a1, b1);
    }
    if (in) {
      double* dst = g.c + g.out_off[o] + (int64_t)r * cst + 2 * tig;
      if (g.accumulate) {
        dst[0] = fma(g.alpha, acc0, dst[0]);
        dst[1] = fma(g.alpha, acc1, dst[1]);
      } else {
        dst[0] = g.alpha * acc0;
        dst[1] = g.alpha * acc1;
      }
    }
  }
}

__device__ __forceinline__ void mm_block(const MmArgs& g, int64_t o, const double* SA, double* SBw,
                                         int lane) {
  const int rows = g.out_rows[o], cols = g.out_cols[o], cst = g.out_stride[o];
  const int64_t p0 = g.pair_start[o], p1 = g.pair_start[o + 1];
  const int entries = rows * cols;
  if (cols == 8 && g.all_inner8) {
    mm_block8(g, o, SA, lane);
    return;
  }
  for (int e0 = 0; e0 < entries; e0 += 32 * kMmEPT) {
    int rr[kMmEPT], cc[kMmEPT];
    double acc[kMmEPT];
#pragma unroll
    for (int m = 0; m < kMmEPT; ++m) {
      const int e = e0 + lane + 32 * m;
      rr[m] = e < entries ? e / cols : 0;
      cc[m] = e < entries ? e - (e / cols) * cols : 0;
      acc[m] = 0.0;
    }
    for (int64_t p = p0; p < p1; ++p) {
      const int nk = g.pair_inner[p], bs = g.pair_b_stride[p];
      const double* Bg = g.b + g.pair_b_off[p];
      __syncwarp();
      for (int q = lane; q < nk * cols; q += 32) {
        const int k = q / cols, c = q - k * cols;
        SBw[k * 16 + c] = __ldg(Bg + (int64_t)k * bs + c);
      }
      __syncwarp();
      const double* A = SA + g.pair_a_soff[p];
      const int as = g.pair_a_stride[p];
      if (cols == 8) {  // lanes keep one column: the C value is shared by all m
        const int c0 = lane & 7;
        for (int k = 0; k < nk; ++k) {
          const double cv = SBw[k * 16 + c0];
#pragma unroll
          for (int m = 0; m < kMmEPT; ++m) acc[m] = fma(A[rr[m] * as + k], cv, acc[m]);
        }
      } else {
        for (int k = 0; k < nk; ++k) {
#pragma unroll
          for (int m = 0; m < kMmEPT; ++m)
            acc[m] = fma(A[rr[m] * as + k], SBw[k * 16 + cc[m]], acc[m]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < kMmEPT; ++m) {
      const int e = e0 + lane + 32 * m;
      if (e < entries) {
        double* dst = g.c + g.out_off[o] + (int64_t)rr[m] * cst + cc[m];
        *dst = g.accumulate ? fma(g.alpha, acc[m], *dst) : g.alpha * acc[m];
      }
    }
  }
}

// One CTA per chunk (fallback, any alignment).
template <bool FAST>
__global__ void __launch_bounds__(kMmWarps * 32) mmult_chunk_kernel(const MmArgs g, int sb_doubles) {
  extern __shared__ __align__(16) double stage[];
  const int64_t ch = g.chunk_ids ? g.chunk_ids[blockIdx.x] : blockIdx.x;
  const int64_t a_lo = g.chunk_a[2 * ch];
  const int na = (int)(g.chunk_a[2 * ch + 1] - a_lo);
  __shared__ uint64_t bar;
  double* SA = stage + sb_doubles;  // warp B buffers (generic path only) then the A stage
  stage_ranges(SA, g.a + a_lo, na, SA + na, g.a + a_lo + na, 0, &bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* SBw = stage + warp * kMmBMax;
  const int64_t o_end = g.chunk_out_start[ch + 1];
  for (int64_t o = g.chunk_out_start[ch] + warp; o < o_end; o += kMmWarps) {
    if (FAST)
      mm_block8(g, o, SA, lane);
    else
      mm_block(g, o, SA, SBw, lane);
  }
}

// Persistent over its chunk list with a kStages-deep ring of TMA-filled A stages.
__global__ void __launch_bounds__(kMmWarps * 32) mmult_chunk_kernel_p(const MmArgs g, int64_t n_list,
                                                                       int stage_doubles) {
  extern __shared__ __align__(16) double stage[];
  __shared__ uint64_t bars[kStages];
  if (threadIdx.x == 0)
    for (int q = 0; q < kStages; ++q) mbar_init(&bars[q], 1);
  __syncthreads();
  double* abuf = stage + kMmWarps * kMmBMax;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kStages; ++q) {
      const int64_t idx = blockIdx.x + (int64_t)q * gridDim.x;
      if (idx < n_list)
        issue_chunk(g.a, g.chunk_a, nullptr, nullptr, g.chunk_ids[idx], abuf + q * stage_doubles,
                    &bars[q]);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* SBw = stage + warp * kMmBMax;
  for (int it = 0;; ++it) {
    const int64_t idx = blockIdx.x + (int64_t)it * gridDim.x;
    if (idx >= n_list) break;
    const int q = it % kStages;
    mbar_wait(&bars[q], (it / kStages) & 1);
    const int64_t ch = g.chunk_ids[idx];
    const double* SA = abuf + q * stage_doubles;
    const int64_t o_end = g.chunk_out_start[ch + 1];
    for (int64_t o = g.chunk_out_start[ch] + warp; o < o_end; o += kMmWarps) mm_block(g, o, SA, SBw, lane);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t nidx = idx + (int64_t)kStages * gridDim.x;
      if (nidx < n_list)
        issue_chunk(g.a, g.chunk_a, nullptr, nullptr, g.chunk_ids[nidx], abuf + q * stage_doubles,
                    &bars[q]);
    }
  }
}

// Chunks split into two launch classes by staged size, so one oversized block
// row does not force its shared-memory footprint on every CTA.
constexpr int kSmallStage = 3584;  // doubles (28 KB): several CTAs per SM

struct ChunkClasses {
  int32_t* ids[2] = {nullptr, nullptr};
  int64_t count[2] = {0, 0};
  int smem[2] = {0, 0};  // bytes

  int build(const int64_t* ca, const int64_t* cb, int64_t n_chunks, int extra_bytes) {
    std::vector<int32_t> lists[2];
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t dbl = (ca[2 * c + 1] - ca[2 * c]) + (cb ? cb[2 * c + 1] - cb[2 * c] : 0);
      const int k = dbl <= kSmallStage ? 0 : 1;
      lists[k].push_back((int32_t)c);
      smem[k] = std::max<int>(smem[k], (int)(dbl * 8) + extra_bytes);
    }
    for (int k = 0; k < 2; ++k) {
      count[k] = (int64_t)lists[k].size();
      int rc = upload(lists[k].data(), count[k], &ids[k]);
      if (rc) return rc;
    }
    return BMV_OK;
  }
  void release_all() {
    release(ids[0]);
    release(ids[1]);
  }
};

}  // namespace

struct bmv_tmmult {
  int64_t n_out = 0, n_chunks = 0, n_seg = 0, n_tri = 0, partial_len = 0;
  int smem_bytes = 0, ept = 8, small = 0, max_b_cols = 0, aligned = 0;
  int64_t* out_off = nullptr;
  int32_t *out_rows = nullptr, *out_cols = nullptr, *out_stride = nullptr;
  int64_t *out_seg_start = nullptr, *out_seg_list = nullptr, *chunk_a = nullptr,
          *chunk_b = nullptr, *chunk_seg_start = nullptr, *seg_out = nullptr,
          *seg_tri_start = nullptr, *seg_poff = nullptr;
  int32_t *tri_a_soff = nullptr, *tri_b_soff = nullptr, *tri_rows = nullptr,
          *tri_a_stride = nullptr, *tri_b_stride = nullptr;
  double* partial = nullptr;
  double* partial2 = nullptr;
  int splits = 1;
  ChunkClasses cls;
};

struct bmv_mmult {
  int64_t n_out = 0, n_chunks = 0, n_pairs = 0;
  int smem_bytes = 0, aligned = 0, all_inner8 = 0, all8 = 0;
  ChunkClasses cls;
  int64_t *chunk_a = nullptr, *chunk_out_start = nullptr, *out_off = nullptr,
          *pair_start = nullptr, *pair_b_off = nullptr;
  int32_t *out_rows = nullptr, *out_cols = nullptr, *out_stride = nullptr,
          *pair_a_soff = nullptr, *pair_a_stride = nullptr, *pair_inner = nullptr,
          *pair_b_stride = nullptr;
};

extern "C" {

int bmv_tmmult_destroy(bmv_tmmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->out_off, p->out_rows, p->out_cols, p->out_stride, p->out_seg_start,
                  p->out_seg_list, p->chunk_a, p->chunk_b, p->chunk_seg_start, p->seg_out,
                  p->seg_tri_start, p->seg_poff, p->tri_a_soff, p->tri_b_soff, p->tri_rows,
                  p->tri_a_stride, p->tri_b_stride, p->partial, p->partial2};
  for (void* q : ptrs) release(q);
  p->cls.release_all();
  delete p;
  return BMV_OK;
}

int bmv_tmmult_create(const bmv_tmmult_desc* d, bmv_tmmult** out) {
  if (!d || !out || d->n_out < 0 || d->n_seg < 0 || d->n_triples < 0 || d->partial_len < 0 ||
      d->n_chunks < 0 || d->smem_doubles < 0) {
    set_error("invalid tmmult descriptor");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  int max_ent = 0;
  for (int64_t o = 0; o < d->n_out; ++o) {
    const int e = d->out_rows[o] * d->out_cols[o];
    if (e > max_ent) max_ent = e;
  }
  if (max_ent > 256) {
    set_error("tmmult output block of %d entries exceeds 256", max_ent);
    return BMV_ERR_INVALID;
  }
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  max_smem -= 1024;  // static shared memory (mbarrier) of the kernels
  if ((int64_t)d->smem_doubles * 8 > max_smem) {
    set_error("tmmult chunk needs %lld bytes of shared memory (max %d)",
              (long long)d->smem_doubles * 8, max_smem);
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_tmmult();
  p->n_out = d->n_out;
  p->n_chunks = d->n_chunks;
  p->n_seg = d->n_seg;
  p->n_tri = d->n_triples;
  p->partial_len = d->partial_len;
  p->smem_bytes = d->smem_doubles * 8;
  p->ept = max_ent <= 64 ? 2 : (max_ent <= 128 ? 4 : 8);
  {
    int mr = 0, mc = 0;
    for (int64_t o = 0; o < d->n_out; ++o) {
      mr = d->out_rows[o] > mr ? d->out_rows[o] : mr;
      mc = d->out_cols[o] > mc ? d->out_cols[o] : mc;
    }
    // the fast path reads 8 B-columns per row: needs B strides >= 8 (true for W = 8)
    int min_bs = 1 << 30, odd = 0;
    for (int64_t t = 0; t < d->n_triples; ++t) {
      min_bs = d->tri_b_stride[t] < min_bs ? d->tri_b_stride[t] : min_bs;
      odd |= (d->tri_b_stride[t] | d->tri_a_stride[t] | d->tri_b_soff[t]) & 1;
    }
    p->small = (mr <= 8 && mc <= 8 && (d->n_triples == 0 || min_bs >= 8) && !odd) ? 1 : 0;
    // TMA bulk staging: every range start (and so every A/B split) 16-byte aligned
    int al = 1;
    for (int64_t c = 0; c < d->n_chunks; ++c)
      al &= ((d->chunk_a[2 * c] | d->chunk_a[2 * c + 1] | d->chunk_b[2 * c] | d->chunk_b[2 * c + 1]) & 1) == 0;
    p->aligned = al;
    p->small = p->small && al;  // 16-byte aligned stage rows for the vector loads
  }
  int rc = upload(d->out_off, d->n_out, &p->out_off);
  if (!rc) rc = upload(d->out_rows, d->n_out, &p->out_rows);
  if (!rc) rc = upload(d->out_cols, d->n_out, &p->out_cols);
  if (!rc) rc = upload(d->out_stride, d->n_out, &p->out_stride);
  if (!rc) rc = upload(d->out_seg_start, d->n_out + 1, &p->out_seg_start);
  if (!rc) rc = upload(d->out_seg_list, d->n_seg, &p->out_seg_list);
  if (!rc) rc = upload(d->chunk_a, 2 * d->n_chunks, &p->chunk_a);
  if (!rc) rc = upload(d->chunk_b, 2 * d->n_chunks, &p->chunk_b);
  if (!rc) rc = upload(d->chunk_seg_start, d->n_chunks + 1, &p->chunk_seg_start);
  if (!rc) rc = upload(d->seg_out, d->n_seg, &p->seg_out);
  if (!rc) rc = upload(d->seg_tri_start, d->n_seg + 1, &p->seg_tri_start);
  if (!rc) rc = upload(d->seg_poff, d->n_seg, &p->seg_poff);
  if (!rc) rc = upload(d->tri_a_soff, d->n_triples, &p->tri_a_soff);
  if (!rc) rc = upload(d->tri_b_soff, d->n_triples, &p->tri_b_soff);
  if (!rc) rc = upload(d->tri_rows, d->n_triples, &p->tri_rows);
  if (!rc) rc = upload(d->tri_a_stride, d->n_triples, &p->tri_a_stride);
  if (!rc) rc = upload(d->tri_b_stride, d->n_triples, &p->tri_b_stride);
  if (!rc && d->partial_len > 0) {
    if (cudaMalloc((void**)&p->partial, sizeof(double) * (size_t)d->partial_len) != cudaSuccess) {
      set_error("cudaMalloc of %lld partial values failed", (long long)d->partial_len);
      rc = BMV_ERR_CUDA;
    }
  }
  if (!rc) rc = p->cls.build(d->chunk_a, d->chunk_b, d->n_chunks, 0);
  if (!rc) {
    int64_t max_seg = 1;
    for (int64_t o = 0; o < d->n_out; ++o)
      max_seg = std::max<int64_t>(max_seg, d->out_seg_start[o + 1] - d->out_seg_start[o]);
    p->splits = (int)((max_seg + kRedSeg - 1) / kRedSeg);
    const size_t n2 = (size_t)std::max<int64_t>(d->n_out, 1) * p->splits * 256;
    if (cudaMalloc((void**)&p->partial2, sizeof(double) * n2) != cudaSuccess) {
      set_error("cudaMalloc of second-level partials failed");
      rc = BMV_ERR_CUDA;
    }
  }
  if (!rc) {
    cudaError_t e = cudaFuncSetAttribute(tm_chunk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tm_chunk_kernel8, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tm_chunk_kernel8_1, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tm_chunk_kernel8_p, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tm_chunk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tm_chunk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      rc = BMV_ERR_CUDA;
    }
  }
  if (rc) {
    bmv_tmmult_destroy(p);
    return rc;
  }
  *out = p;
  return BMV_OK;
}

int bmv_tmmult_run(bmv_tmmult* p, const double* a, const double* b, double* c, int64_t c_len,
                   void* stream) {
  if (!p) {
    set_error("null plan");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  int rc = zero_async(c, c_len, st);
  if (rc) return rc;
  if (p->n_out == 0) return BMV_OK;
  TmArgs g{p->out_off, p->out_rows, p->out_cols, p->out_stride, p->out_seg_start,
           p->out_seg_list, p->chunk_a, p->chunk_b, p->chunk_seg_start, p->seg_out,
           p->seg_tri_start, p->seg_poff, p->tri_a_soff, p->tri_b_soff, p->tri_rows,
           p->tri_a_stride, p->tri_b_stride, a, b, p->partial, c, nullptr, p->partial2,
           p->splits};
  for (int k = 0; k < 2; ++k) {
    if (p->cls.count[k] == 0) continue;
    g.chunk_ids = p->cls.ids[k];
    const unsigned grid = (unsigned)p->cls.count[k];
    const int smem = p->cls.smem[k];
    if (p->small && k == 0 && p->aligned && kPersistent) {
      const int per_sm = std::max(1, (227 * 1024) / (kStages * smem + 1024));
      const unsigned pgrid = (unsigned)std::min<int64_t>(p->cls.count[0], (int64_t)sm_count() * per_sm);
      tm_chunk_kernel8_p<<<pgrid, kTmWarps * 32, kStages * smem, st>>>(g, p->cls.count[0], smem / 8);
    } else if (p->small)
      tm_chunk_kernel8_1<<<grid, kTmWarps * 32, smem, st>>>(g);
    else if (p->ept == 2)
      tm_chunk_kernel<2><<<grid, kTmWarps * 32, smem, st>>>(g);
    else if (p->ept == 4)
      tm_chunk_kernel<4><<<grid, kTmWarps * 32, smem, st>>>(g);
    else
      tm_chunk_kernel<8><<<grid, kTmWarps * 32, smem, st>>>(g);
    BMV_CHECK_LAUNCH();
  }
  tm_reduce1_kernel<<<dim3((unsigned)p->n_out, (unsigned)p->splits), 256, 0, st>>>(g);
  BMV_CHECK_LAUNCH();
  tm_reduce2_kernel<<<(unsigned)p->n_out, 256, 0, st>>>(g);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

int bmv_mmult_destroy(bmv_mmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->chunk_a, p->chunk_out_start, p->out_off, p->pair_start, p->pair_b_off,
                  p->out_rows, p->out_cols, p->out_stride, p->pair_a_soff, p->pair_a_stride,
                  p->pair_inner, p->pair_b_stride};
  for (void* q : ptrs) release(q);
  p->cls.release_all();
  delete p;
  return BMV_OK;
}

int bmv_mmult_create(const bmv_mmult_desc* d, bmv_mmult** out) {
  if (!d || !out || d->n_out < 0 || d->n_pairs < 0 || d->n_chunks < 0 || d->smem_doubles < 0) {
    set_error("invalid mmult descriptor");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  max_smem -= 1024;  // static shared memory (mbarrier) of the kernel
  if ((int64_t)d->smem_doubles * 8 + kMmWarps * kMmBMax * 8 > max_smem) {
    set_error("mmult chunk needs %lld bytes of shared memory (max %d)",
              (long long)d->smem_doubles * 8, max_smem);
    return BMV_ERR_INVALID;
  }
  for (int64_t o = 0; o < d->n_out; ++o) {
    if (d->out_cols[o] > 16) {
      set_error("mmult column blocks wider than 16 are not supported");
      return BMV_ERR_INVALID;
    }
  }
  for (int64_t q = 0; q < d->n_pairs; ++q) {
    if (d->pair_inner[q] > 16) {
      set_error("mmult inner blocks wider than 16 are not supported");
      return BMV_ERR_INVALID;
    }
  }
  auto* p = new bmv_mmult();
  p->n_out = d->n_out;
  p->n_chunks = d->n_chunks;
  p->n_pairs = d->n_pairs;
  p->smem_bytes = d->smem_doubles * 8;
  int rc = upload(d->chunk_a, 2 * d->n_chunks, &p->chunk_a);
  if (!rc) rc = upload(d->chunk_out_start, d->n_chunks + 1, &p->chunk_out_start);
  if (!rc) rc = upload(d->out_off, d->n_out, &p->out_off);
  if (!rc) rc = upload(d->out_rows, d->n_out, &p->out_rows);
  if (!rc) rc = upload(d->out_cols, d->n_out, &p->out_cols);
  if (!rc) rc = upload(d->out_stride, d->n_out, &p->out_stride);
  if (!rc) rc = upload(d->pair_start, d->n_out + 1, &p->pair_start);
  if (!rc) rc = upload(d->pair_a_soff, d->n_pairs, &p->pair_a_soff);
  if (!rc) rc = upload(d->pair_a_stride, d->n_pairs, &p->pair_a_stride);
  if (!rc) rc = upload(d->pair_inner, d->n_pairs, &p->pair_inner);
  if (!rc) rc = upload(d->pair_b_off, d->n_pairs, &p->pair_b_off);
  if (!rc) rc = upload(d->pair_b_stride, d->n_pairs, &p->pair_b_stride);
  if (!rc) rc = p->cls.build(d->chunk_a, nullptr, d->n_chunks, kMmWarps * kMmBMax * 8);
  {
    int ok8 = 1;
    for (int64_t q = 0; q < d->n_pairs; ++q) ok8 &= d->pair_inner[q] == 8 && d->pair_b_stride[q] >= 8;
    p->all_inner8 = ok8;
    int oc8 = 1;
    for (int64_t o = 0; o < d->n_out; ++o) oc8 &= d->out_cols[o] == 8;
    p->all8 = ok8 && oc8;
  }
  if (!rc) {
    cudaError_t e = cudaFuncSetAttribute(mmult_chunk_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mmult_chunk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               max_smem - 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mmult_chunk_kernel_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               max_smem - 1024);
    int al = 1;
    for (int64_t c = 0; c < d->n_chunks; ++c)
      al &= ((d->chunk_a[2 * c] | d->chunk_a[2 * c + 1]) & 1) == 0;
    p->aligned = al;
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      rc = BMV_ERR_CUDA;
    }
  }
  if (rc) {
    bmv_mmult_destroy(p);
    return rc;
  }
  *out = p;
  return BMV_OK;
}

int bmv_mmult_run(bmv_mmult* p, const double* a, const double* b, double* c, double alpha,
                  int32_t accumulate, int64_t c_len, void* stream) {
  if (!p) {
    set_error("null plan");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  if (!accumulate) {
    int rc = zero_async(c, c_len, st);
    if (rc) return rc;
  }
  if (p->n_out == 0 || p->n_chunks == 0) return BMV_OK;
  MmArgs g{p->chunk_a, p->chunk_out_start, p->out_off, p->out_rows, p->out_cols, p->out_stride,
           p->pair_start, p->pair_a_soff, p->pair_a_stride, p->pair_inner, p->pair_b_off,
           p->pair_b_stride, a, b, c, alpha, accumulate, nullptr, p->all_inner8};
  for (int k = 0; k < 2; ++k) {
    if (p->cls.count[k] == 0) continue;
    g.chunk_ids = p->cls.ids[k];
    if (k == 0 && p->aligned && kPersistent) {
      const int a_bytes = p->cls.smem[0] - kMmWarps * kMmBMax * 8;  // staged A bytes (max)
      const int smem = kMmWarps * kMmBMax * 8 + kStages * a_bytes;
      const int per_sm = std::max(1, (227 * 1024) / (smem + 1024));
      const unsigned pgrid = (unsigned)std::min<int64_t>(p->cls.count[0], (int64_t)sm_count() * per_sm);
      mmult_chunk_kernel_p<<<pgrid, kMmWarps * 32, smem, st>>>(g, p->cls.count[0], a_bytes / 8);
    } else {
      if (p->all8)
        mmult_chunk_kernel<true><<<(unsigned)p->cls.count[k], kMmWarps * 32,
                                   p->cls.smem[k] - kMmWarps * kMmBMax * 8, st>>>(g, 0);
      else
        mmult_chunk_kernel<false><<<(unsigned)p->cls.count[k], kMmWarps * 32, p->cls.smem[k], st>>>(
            g, kMmWarps * kMmBMax);
    }
    BMV_CHECK_LAUNCH();
  }
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

}  // extern "C"
