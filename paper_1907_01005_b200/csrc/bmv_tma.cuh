// 1D TMA bulk copies (cp.async.bulk -> SASS UBLKCP) completed on mbarriers,
// and the FP64 tensor-core MMA (DMMA m8n8k4), shared by K4 and K5.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bmv {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// One arrival that also announces `bytes` of pending TMA transactions.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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
// global -> shared bulk copy of `bytes` (multiple of 16, both ends 16-byte aligned)
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

}  // namespace bmv

namespace bmv {

// ---- Copy lists: what a producer warp stages for one sub-chunk ----------
// Entry (4 x int32): x = destination byte offset in the stage,
// y = bytes | source << 28 | last << 30, z / w = source byte offset (lo, hi).
// The entries of one sub-chunk are consecutive, the last one flagged.
constexpr unsigned kCpLenMask = (1u << 28) - 1;

struct CopySrc {
  const char* p0;
  const char* p1;
  const char* p2;
  const char* p3 = nullptr;
};

__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ int4 shfl_int4(const int4 v, int src) {
  return make_int4(__shfl_sync(~0u, v.x, src), __shfl_sync(~0u, v.y, src),
                   __shfl_sync(~0u, v.z, src), __shfl_sync(~0u, v.w, src));
}

// Producer warp of a TMA ring: streams n_subs sub-chunks, whose copy entries
// are [e_begin, e_end), into `stages` (NS stages of stage_bytes).  Entries
// are read 32 at a time (one per lane) with the next window prefetched, so
// the steady state issues no dependent global loads.  16-byte aligned
// entries go through cp.async.bulk (transaction bytes announced on
// full[stage] before the copies are issued); others (odd strides) are
// copied by their lane.  One arrival per stage fill, after its last entry.
__device__ __forceinline__ void stream_producer(const int4* __restrict__ cps, int64_t e_begin,
                                                int64_t e_end, int64_t n_subs, const CopySrc src,
                                                char* stages, int stage_bytes, int NS,
                                                uint64_t* full, uint64_t* empty, int lane) {
  const int4 zero = make_int4(0, 0, 0, 0);
  int64_t w0 = e_begin;
  int4 cur = (w0 + lane < e_end) ? __ldg(cps + w0 + lane) : zero;
  int4 nxt = (w0 + 32 + lane < e_end) ? __ldg(cps + w0 + 32 + lane) : zero;
  int pos = 0;
  for (int64_t i = 0; i < n_subs; ++i) {
    const int st = (int)(i % NS);
    if (i >= NS) mbar_wait(&empty[st], (unsigned)((i / NS - 1) & 1));
    char* dst = stages + (int64_t)st * stage_bytes;
    for (;;) {  // window pieces of this sub-chunk's entries
      const unsigned lastm = __ballot_sync(~0u, ((unsigned)cur.y >> 30) & 1u) & (~0u << pos);
      const int end = lastm ? __ffs(lastm) - 1 : 31;
      const bool mine = lane >= pos && lane <= end;
      const unsigned len = mine ? ((unsigned)cur.y & kCpLenMask) : 0u;
      const int sel = ((unsigned)cur.y >> 28) & 3;
      const char* s = (sel == 0 ? src.p0 : sel == 1 ? src.p1 : sel == 2 ? src.p2 : src.p3) +
                      (((int64_t)(unsigned)cur.w << 32) | (unsigned)cur.z);
      const unsigned doff = (unsigned)cur.x;
      const bool bulk = mine && ((reinterpret_cast<uintptr_t>(s) | doff | len) & 15u) == 0;
      if (mine && !bulk)
        for (unsigned k = 0; k < len; k += 8)
          *reinterpret_cast<double*>(dst + doff + k) = __ldg(reinterpret_cast<const double*>(s + k));
      const unsigned bytes = __reduce_add_sync(~0u, bulk ? len : 0u);
      if (lane == 0 && bytes) mbar_expect_tx_only(&full[st], bytes);
      __syncwarp();
      if (bulk)
        for (unsigned k = 0; k < len; k += 32768u)
          bulk_g2s(dst + doff + k, s + k, min(32768u, len - k), &full[st]);
      pos = end + 1;
      if (pos == 32) {
        cur = nxt;
        w0 += 32;
        pos = 0;
        nxt = (w0 + 32 + lane < e_end) ? __ldg(cps + w0 + 32 + lane) : zero;
      }
      if (lastm) break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&full[st]);  // release: the lanes' plain copies are visible
  }
}

}  // namespace bmv
