// K4: the projection C(k,l) = sum_i A_ik^T B_il over the owned block rows i
// (reference tmmult, bcsr.py:631-667, loop order :646-666) on the reference's
// block-CSR storage (padded row-major blocks).
//
// HBM-bound streaming design.  The owned block rows are cut into one part
// per SM; a part is a sequence of sub-chunks (consecutive rows, or an
// A-group x B-group tile of one long row) whose A and B blocks are two
// contiguous value ranges.  One persistent CTA per part runs a TMA pipeline:
// a producer warp streams the sub-chunks into a ring of shared-memory stages
// with cp.async.bulk (completion on a "full" mbarrier), eight consumer warps
// compute the 8x8 output tiles of each sub-chunk with DMMA (FP64 tensor
// cores) and release the stage on an "empty" mbarrier.  Every output tile
// of an item (a run of sub-chunks of one part touching <= 128 tiles) is
// owned by one consumer warp, which accumulates it in a private shared-memory
// slot and writes it once to a partial buffer at the end of the item.  A
// second kernel sums each tile's partials in item order into C.  Fixed
// summation order throughout: bit-reproducible, no atomics.
#include <cuda_runtime.h>

#include <algorithm>

#include "bmv_common.cuh"
#include "bmv_tma.cuh"

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st);
}

using namespace bmv;

namespace {

constexpr int kPjWarps = 8;                     // consumer warps per CTA
constexpr int kPjSlots = 16;                    // accumulator tiles per consumer warp
constexpr int kPjThreads = (kPjWarps + 1) * 32; // + one producer warp
constexpr int kPjMaxStages = 8;
constexpr int kPjSlotDoubles = kPjWarps * kPjSlots * 64;
constexpr int kPjPiece = 4096;                  // doubles per bulk copy instruction

struct PjArgs {
  const int64_t* __restrict__ part_sub_start;
  const int64_t* __restrict__ sub_a;   // [lo, hi) per sub-chunk
  const int64_t* __restrict__ sub_b;
  const int32_t* __restrict__ sub_item;
  const int64_t* __restrict__ sub_tri_start;  // per (sub, warp)
  const int4* __restrict__ tri;
  const int32_t* __restrict__ item_slots;     // per (item, warp)
  const double* __restrict__ a;
  const double* __restrict__ b;
  double* __restrict__ partial;
  int stage_doubles;
  int n_stages;
  int bulk_ok;  // a, b 16-byte aligned
};

__device__ __forceinline__ int b_stage_offset(int na) { return (na + 1) & ~1; }

// Tile of one triple: sum_r A[r][8 mt + m] B[r][8 nt + n] over the block rows,
// A/B in the stage at (row stride as/bs).  Lane (gid, tig) returns
// D[gid][2 tig], D[gid][2 tig + 1].
__device__ __forceinline__ void triple_tile(const double* S, const int4 d, int gid, int tig,
                                            double& x, double& y) {
  const int rows = d.z & 0xffff;
  const int acols = (d.z >> 24) & 15, bcols = (d.z >> 28) & 15;
  const int as = d.w & 0xffff, bs = (d.w >> 16) & 0xffff;
  const bool am = gid < acols, bm = gid < bcols;
  const double* A = S + d.x + gid + tig * as;
  const double* B = S + d.y + gid + tig * bs;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int r0 = 0;
#pragma unroll 2
  for (; r0 + 8 <= rows; r0 += 8) {
    const double a0 = am ? A[r0 * as] : 0.0, b0 = bm ? B[r0 * bs] : 0.0;
    const double a1 = am ? A[(r0 + 4) * as] : 0.0, b1 = bm ? B[(r0 + 4) * bs] : 0.0;
    dmma_8x8x4(c0, c1, a0, b0);
    dmma_8x8x4(c2, c3, a1, b1);
  }
  for (; r0 < rows; r0 += 4) {
    const bool ok = r0 + tig < rows;
    const double a0 = (am && ok) ? A[r0 * as] : 0.0, b0 = (bm && ok) ? B[r0 * bs] : 0.0;
    dmma_8x8x4(c0, c1, a0, b0);
  }
  x = c0 + c2;
  y = c1 + c3;
}

__global__ void __launch_bounds__(kPjThreads, 1) pj_stream_kernel(const PjArgs g) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[kPjMaxStages], empty[kPjMaxStages];
  double* slots = smem;
  double* stages = smem + kPjSlotDoubles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = g.part_sub_start[blockIdx.x], s1 = g.part_sub_start[blockIdx.x + 1];
  const int NS = g.n_stages;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NS; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kPjWarps);
    }
  }
  for (int i = threadIdx.x; i < kPjSlotDoubles; i += blockDim.x) slots[i] = 0.0;
  __syncthreads();

  if (warp == kPjWarps) {  // producer: stream the sub-chunks through the ring
    for (int64_t s = s0; s < s1; ++s) {
      const int64_t i = s - s0;
      const int st = (int)(i % NS);
      if (i >= NS) mbar_wait(&empty[st], (unsigned)((i / NS - 1) & 1));
      double* dst = stages + (int64_t)st * g.stage_doubles;
      const int64_t alo = g.sub_a[2 * s], ahi = g.sub_a[2 * s + 1];
      const int64_t blo = g.sub_b[2 * s], bhi = g.sub_b[2 * s + 1];
      const int na = (int)(ahi - alo), nb = (int)(bhi - blo), boff = b_stage_offset(na);
      if (g.bulk_ok && ((alo | ahi | blo | bhi) & 1) == 0) {
        if (lane == 0) {
          mbar_expect_tx(&full[st], (unsigned)(na + nb) * 8u);
          for (int k = 0; k < na; k += kPjPiece)
            bulk_g2s(dst + k, g.a + alo + k, (unsigned)min(kPjPiece, na - k) * 8u, &full[st]);
          for (int k = 0; k < nb; k += kPjPiece)
            bulk_g2s(dst + boff + k, g.b + blo + k, (unsigned)min(kPjPiece, nb - k) * 8u, &full[st]);
        }
      } else {
        for (int k = lane; k < na; k += 32) dst[k] = __ldg(g.a + alo + k);
        for (int k = lane; k < nb; k += 32) dst[boff + k] = __ldg(g.b + blo + k);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
    }
    return;
  }

  const int gid = lane >> 2, tig = lane & 3;
  double* mine = slots + warp * kPjSlots * 64 + 2 * lane;
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t i = s - s0;
    const int st = (int)(i % NS);
    mbar_wait(&full[st], (unsigned)((i / NS) & 1));
    const double* S = stages + (int64_t)st * g.stage_doubles;
    const int64_t t0 = g.sub_tri_start[s * kPjWarps + warp];
    const int64_t t1 = g.sub_tri_start[s * kPjWarps + warp + 1];
    for (int64_t t = t0; t < t1; ++t) {
      const int4 d = __ldg(g.tri + t);
      double x, y;
      triple_tile(S, d, gid, tig, x, y);
      double2* q = reinterpret_cast<double2*>(mine + ((d.z >> 16) & 0xff) * 64);
      double2 v = *q;
      v.x += x;
      v.y += y;
      *q = v;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    const int item = g.sub_item[s];
    if (s + 1 == s1 || g.sub_item[s + 1] != item) {  // item done: flush this warp's tiles
      const int n = g.item_slots[(int64_t)item * kPjWarps + warp];
      double* P = g.partial + ((int64_t)item * kPjWarps + warp) * kPjSlots * 64 + 2 * lane;
      for (int k = 0; k < n; ++k) {
        double2* q = reinterpret_cast<double2*>(mine + k * 64);
        *reinterpret_cast<double2*>(P + k * 64) = *q;
        *q = make_double2(0.0, 0.0);
      }
    }
  }
}

// One warp per output tile: sum its partial tiles in item order, write C.
__global__ void __launch_bounds__(256) pj_reduce_kernel(const int64_t* __restrict__ tile_off,
                                                        const int32_t* __restrict__ tile_shape,
                                                        const int64_t* __restrict__ src_start,
                                                        const int64_t* __restrict__ src,
                                                        const double* __restrict__ partial,
                                                        double* __restrict__ c, int64_t n_tiles) {
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= n_tiles) return;
  const int lane = threadIdx.x & 31;
  const int64_t j0 = src_start[t], j1 = src_start[t + 1];
  double x = 0.0, y = 0.0;
#pragma unroll 4
  for (int64_t j = j0; j < j1; ++j) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(partial + src[j] * 64) + lane);
    x += v.x;
    y += v.y;
  }
  const int rows = tile_shape[3 * t], cols = tile_shape[3 * t + 1], stride = tile_shape[3 * t + 2];
  const int r = lane >> 2, cc = 2 * (lane & 3);
  if (r < rows) {
    double* C = c + tile_off[t] + (int64_t)r * stride + cc;
    if (cc < cols) C[0] = x;
    if (cc + 1 < cols) C[1] = y;
  }
}

}  // namespace

struct bmv_tmmult {
  int n_parts = 0, stage_doubles = 0, n_stages = 0, smem_bytes = 0;
  int64_t n_sub = 0, n_items = 0, n_tri = 0, n_tiles = 0;
  int64_t *part_sub_start = nullptr, *sub_a = nullptr, *sub_b = nullptr,
          *sub_tri_start = nullptr, *tile_off = nullptr, *tile_src_start = nullptr,
          *tile_src = nullptr;
  int32_t *sub_item = nullptr, *tri = nullptr, *item_slots = nullptr, *tile_shape = nullptr;
  double* partial = nullptr;
};

extern "C" {

int bmv_tmmult_destroy(bmv_tmmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->part_sub_start, p->sub_a,      p->sub_b,          p->sub_tri_start,
                  p->tile_off,       p->tile_src_start, p->tile_src,   p->sub_item,
                  p->tri,            p->item_slots, p->tile_shape,     p->partial};
  for (void* q : ptrs) release(q);
  delete p;
  return BMV_OK;
}

int bmv_tmmult_create(const bmv_tmmult_desc* d, bmv_tmmult** out) {
  if (!out) return BMV_ERR_INVALID;
  *out = nullptr;
  if (!d || d->n_parts < 0 || d->n_sub < 0 || d->n_items < 0 || d->n_tri < 0 ||
      d->n_out_tiles < 0 || d->n_src < 0 || d->stage_doubles < 2 || (d->stage_doubles & 1)) {
    set_error("invalid tmmult descriptor");
    return BMV_ERR_INVALID;
  }
  if (d->n_warps != kPjWarps || d->slots_per_warp != kPjSlots) {
    set_error("tmmult plan built for %d warps x %d slots, kernel has %d x %d", d->n_warps,
              d->slots_per_warp, kPjWarps, kPjSlots);
    return BMV_ERR_INVALID;
  }
  // host-side validation of the plan (bounds the kernel relies on)
  if (d->n_parts > 0 && (d->part_sub_start[0] != 0 || d->part_sub_start[d->n_parts] != d->n_sub)) {
    set_error("tmmult part ranges do not cover the sub-chunks");
    return BMV_ERR_INVALID;
  }
  for (int64_t s = 0; s < d->n_sub; ++s) {
    const int64_t na = d->sub_a[2 * s + 1] - d->sub_a[2 * s], nb = d->sub_b[2 * s + 1] - d->sub_b[2 * s];
    if (na < 0 || nb < 0 || ((na + 1) & ~1LL) + nb > d->stage_doubles || d->sub_item[s] < 0 ||
        d->sub_item[s] >= d->n_items) {
      set_error("tmmult sub-chunk %lld exceeds the stage or names a bad item", (long long)s);
      return BMV_ERR_INVALID;
    }
  }
  if (d->n_sub > 0 && d->sub_tri_start[(int64_t)d->n_sub * kPjWarps] != d->n_tri) {
    set_error("tmmult triple ranges do not cover the triples");
    return BMV_ERR_INVALID;
  }
  for (int64_t t = 0; t < d->n_tri; ++t) {
    const int32_t* q = d->tri + 4 * t;
    if (q[0] < 0 || q[1] < 0 || ((q[2] >> 16) & 0xff) >= kPjSlots) {
      set_error("tmmult triple %lld has a bad stage offset or slot", (long long)t);
      return BMV_ERR_INVALID;
    }
  }
  for (int64_t k = 0; k < d->n_items * kPjWarps; ++k)
    if (d->item_slots[k] < 0 || d->item_slots[k] > kPjSlots) {
      set_error("tmmult item uses more than %d slots per warp", kPjSlots);
      return BMV_ERR_INVALID;
    }
  const int64_t partial_tiles = d->n_items * kPjWarps * kPjSlots;
  for (int64_t j = 0; j < d->n_src; ++j)
    if (d->tile_src[j] < 0 || d->tile_src[j] >= partial_tiles) {
      set_error("tmmult reduction source out of range");
      return BMV_ERR_INVALID;
    }
  int dev = 0, max_smem = 0;
  BMV_CUDA_TRY(cudaGetDevice(&dev));
  BMV_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int avail = max_smem - 1024 - kPjSlotDoubles * 8;
  const int ns = std::min(kPjMaxStages, avail / (d->stage_doubles * 8));
  if (ns < 2) {
    set_error("tmmult stage of %d doubles leaves fewer than 2 pipeline stages", d->stage_doubles);
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_tmmult();
  p->n_parts = d->n_parts;
  p->n_sub = d->n_sub;
  p->n_items = d->n_items;
  p->n_tri = d->n_tri;
  p->n_tiles = d->n_out_tiles;
  p->stage_doubles = d->stage_doubles;
  p->n_stages = ns;
  p->smem_bytes = (kPjSlotDoubles + ns * d->stage_doubles) * 8;
  int rc = upload(d->part_sub_start, (int64_t)d->n_parts + 1, &p->part_sub_start);
  if (!rc) rc = upload(d->sub_a, 2 * d->n_sub, &p->sub_a);
  if (!rc) rc = upload(d->sub_b, 2 * d->n_sub, &p->sub_b);
  if (!rc) rc = upload(d->sub_item, d->n_sub, &p->sub_item);
  if (!rc) rc = upload(d->sub_tri_start, d->n_sub * kPjWarps + 1, &p->sub_tri_start);
  if (!rc) rc = upload(d->tri, 4 * d->n_tri, &p->tri);
  if (!rc) rc = upload(d->item_slots, d->n_items * kPjWarps, &p->item_slots);
  if (!rc) rc = upload(d->tile_off, d->n_out_tiles, &p->tile_off);
  if (!rc) rc = upload(d->tile_shape, 3 * d->n_out_tiles, &p->tile_shape);
  if (!rc) rc = upload(d->tile_src_start, d->n_out_tiles + 1, &p->tile_src_start);
  if (!rc) rc = upload(d->tile_src, d->n_src, &p->tile_src);
  if (!rc && partial_tiles > 0 &&
      cudaMalloc((void**)&p->partial, sizeof(double) * 64 * (size_t)partial_tiles) != cudaSuccess) {
    set_error("cudaMalloc of %lld partial tiles failed", (long long)partial_tiles);
    rc = BMV_ERR_CUDA;
  }
  if (!rc) {
    const cudaError_t e = cudaFuncSetAttribute(pj_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               p->smem_bytes);
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
  if (p->n_sub > 0 && p->n_parts > 0) {
    const int bulk_ok = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
    PjArgs g{p->part_sub_start, p->sub_a, p->sub_b, p->sub_item, p->sub_tri_start,
             reinterpret_cast<const int4*>(p->tri), p->item_slots, a, b, p->partial,
             p->stage_doubles, p->n_stages, bulk_ok};
    pj_stream_kernel<<<(unsigned)p->n_parts, kPjThreads, p->smem_bytes, st>>>(g);
    BMV_CHECK_LAUNCH();
  }
  if (p->n_tiles > 0) {
    pj_reduce_kernel<<<(unsigned)((p->n_tiles + 7) / 8), 256, 0, st>>>(
        p->tile_off, p->tile_shape, p->tile_src_start, p->tile_src, p->partial, c, p->n_tiles);
    BMV_CHECK_LAUNCH();
  }
  return BMV_OK;
}

}  // extern "C"
