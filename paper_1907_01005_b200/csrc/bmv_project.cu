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

constexpr int kPjWarps = 16;                    // consumer warps per CTA
constexpr int kPjSlots = 8;                     // accumulator tiles per consumer warp (registers)
constexpr int kPjUnits = 32;                    // output tiles per sub-chunk
constexpr int kPjThreads = (kPjWarps + 1) * 32; // + one producer warp
constexpr int kPjMaxStages = 8;
constexpr int kPjResultDoubles = 2 * kPjUnits * 64;  // double-buffered unit results
// Stage = [header (68 int32)][triple tiles (int4)][A blocks][B blocks].  Header:
// [0..16] first triple of each computing warp (local) and the end, [17] item,
// [18] flush (last sub-chunk of the item), [19] units, [20..35] slots per
// warp in the item, [36..67] unit -> owner warp | slot << 8.
constexpr int kPjHeader = 272;

struct PjArgs {
  const int64_t* __restrict__ part_sub_start;
  const int64_t* __restrict__ part_entry_start;
  const int4* __restrict__ copies;
  CopySrc src;  // p0 = meta, p1 = a, p2 = b
  double* __restrict__ partial;
  int stage_bytes;
  int n_stages;
};

// sum_r A[r][0:acols] B[r][0:bcols] of one triple tile, added to (x, y):
// lane (gid, tig) holds D[gid][2 tig + {0,1}].  Four independent DMMA chains.
__device__ __forceinline__ void triple_tile(const double* S, const int4 d, int gid, int tig,
                                            double& x, double& y) {
  const int rows = d.z & 0xffff;
  const int acols = (d.z >> 24) & 15, bcols = (d.z >> 28) & 15;
  const int as = d.w & 0xffff, bs = (d.w >> 16) & 0xffff;
  const bool am = gid < acols, bm = gid < bcols;
  const double* A = S + d.x + gid + tig * as;
  const double* B = S + d.y + gid + tig * bs;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0, c5 = 0.0, c6 = 0.0, c7 = 0.0;
  int r0 = 0;
#pragma unroll 2
  for (; r0 + 16 <= rows; r0 += 16) {
    const double a0 = am ? A[r0 * as] : 0.0, b0 = bm ? B[r0 * bs] : 0.0;
    const double a1 = am ? A[(r0 + 4) * as] : 0.0, b1 = bm ? B[(r0 + 4) * bs] : 0.0;
    const double a2 = am ? A[(r0 + 8) * as] : 0.0, b2 = bm ? B[(r0 + 8) * bs] : 0.0;
    const double a3 = am ? A[(r0 + 12) * as] : 0.0, b3 = bm ? B[(r0 + 12) * bs] : 0.0;
    dmma_8x8x4(c0, c1, a0, b0);
    dmma_8x8x4(c2, c3, a1, b1);
    dmma_8x8x4(c4, c5, a2, b2);
    dmma_8x8x4(c6, c7, a3, b3);
  }
  for (; r0 < rows; r0 += 4) {
    const bool ok = r0 + tig < rows;
    const double a0 = (am && ok) ? A[r0 * as] : 0.0, b0 = (bm && ok) ? B[r0 * bs] : 0.0;
    dmma_8x8x4(c0, c1, a0, b0);
  }
  x += (c0 + c2) + (c4 + c6);
  y += (c1 + c3) + (c5 + c7);
}

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kPjWarps * 32) : "memory");
}

__global__ void __launch_bounds__(kPjThreads, 1) pj_stream_kernel(const PjArgs g) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[kPjMaxStages], empty[kPjMaxStages];
  double* results = smem;
  char* stages = reinterpret_cast<char*>(smem + kPjResultDoubles);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = g.part_sub_start[blockIdx.x], s1 = g.part_sub_start[blockIdx.x + 1];
  const int NS = g.n_stages;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NS; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kPjWarps);
    }
  }
  __syncthreads();

  if (warp == kPjWarps) {
    stream_producer(g.copies, g.part_entry_start[blockIdx.x], g.part_entry_start[blockIdx.x + 1],
                    s1 - s0, g.src, stages, g.stage_bytes, NS, full, empty, lane);
    return;
  }

  const int gid = lane >> 2, tig = lane & 3;
  double acc[kPjSlots][2];  // this warp's owned output tiles (registers)
#pragma unroll
  for (int k = 0; k < kPjSlots; ++k) acc[k][0] = acc[k][1] = 0.0;
  for (int64_t i = 0; i < s1 - s0; ++i) {
    const int st = (int)(i % NS);
    mbar_wait(&full[st], (unsigned)((i / NS) & 1));
    const char* stg = stages + (int64_t)st * g.stage_bytes;
    const int* hdr = reinterpret_cast<const int*>(stg);
    const int4* tri = reinterpret_cast<const int4*>(stg + kPjHeader);
    const double* S = reinterpret_cast<const double*>(stg);
    double* R = results + (i & 1) * (kPjUnits * 64);
    // 1) compute this warp's units (balanced per sub-chunk on the host)
    const int t1 = hdr[warp + 1];
    int t = hdr[warp];
    while (t < t1) {
      const int unit = (tri[t].z >> 16) & 0xff;
      double x = 0.0, y = 0.0;
      do {
        triple_tile(S, tri[t], gid, tig, x, y);
        ++t;
      } while (t < t1 && ((tri[t].z >> 16) & 0xff) == unit);
      reinterpret_cast<double2*>(R + unit * 64)[lane] = make_double2(x, y);
    }
    consumer_sync();  // all unit results of this sub-chunk are in R
    // 2) owners add the unit results into their register tiles
    const int n_units = hdr[19];
    const int ow = lane < n_units ? hdr[36 + lane] : -1;
    unsigned mine_u = __ballot_sync(~0u, (ow & 0xff) == warp && lane < n_units);
    while (mine_u) {
      const int u = __ffs(mine_u) - 1;
      mine_u &= mine_u - 1;
      const int slot = __shfl_sync(~0u, ow, u) >> 8;
      const double2 v = reinterpret_cast<const double2*>(R + u * 64)[lane];
#pragma unroll
      for (int k = 0; k < kPjSlots; ++k)
        if (k == slot) {
          acc[k][0] += v.x;
          acc[k][1] += v.y;
        }
    }
    const int item = hdr[17], flush = hdr[18], n_slots = hdr[20 + warp];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (flush) {  // last sub-chunk of the item: write this warp's tiles once, clear them
      double* P = g.partial + ((int64_t)item * kPjWarps + warp) * kPjSlots * 64;
#pragma unroll
      for (int k = 0; k < kPjSlots; ++k) {
        if (k < n_slots) reinterpret_cast<double2*>(P + k * 64)[lane] = make_double2(acc[k][0], acc[k][1]);
        acc[k][0] = acc[k][1] = 0.0;
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
  int n_parts = 0, stage_bytes = 0, n_stages = 0, smem_bytes = 0;
  int64_t n_sub = 0, n_items = 0, n_tiles = 0, c_extent = 0;
  int64_t *part_sub_start = nullptr, *part_entry_start = nullptr, *tile_off = nullptr,
          *tile_src_start = nullptr, *tile_src = nullptr;
  int32_t *copies = nullptr, *meta = nullptr, *tile_shape = nullptr;
  double* partial = nullptr;
};

namespace {

// Walk every sub-chunk's copy entries and staged header / triple tiles: the
// bounds the kernel relies on (stage extents, slots, items) hold.
int validate_tmmult(const bmv_tmmult_desc* d) {
  const int64_t meta_bytes = d->meta_len * 4;
  if (d->n_parts > 0 && (d->part_sub_start[0] != 0 || d->part_sub_start[d->n_parts] != d->n_sub ||
                         d->part_entry_start[0] != 0 || d->part_entry_start[d->n_parts] != d->n_entries)) {
    set_error("tmmult part ranges do not cover the sub-chunks / copies");
    return BMV_ERR_INVALID;
  }
  for (int p = 0; p < d->n_parts; ++p) {
    int64_t e = d->part_entry_start[p];
    const int64_t e1 = d->part_entry_start[p + 1];
    for (int64_t s = d->part_sub_start[p]; s < d->part_sub_start[p + 1]; ++s) {
      const int64_t first = e;
      const int32_t* m = nullptr;
      for (;; ++e) {
        if (e >= e1) {
          set_error("tmmult copy list of sub-chunk %lld is malformed", (long long)s);
          return BMV_ERR_INVALID;
        }
        const int32_t* q = d->copies + 4 * e;
        const unsigned y = (unsigned)q[1];
        const int64_t len = y & kCpLenMask, sel = (y >> 28) & 3;
        const int64_t src = ((int64_t)(uint32_t)q[3] << 32) | (uint32_t)q[2];
        if (q[0] < 0 || q[0] + len > d->stage_bytes || sel > 2 || src < 0 ||
            (sel == 0 && src + len > meta_bytes)) {
          set_error("tmmult copy entry %lld out of range", (long long)e);
          return BMV_ERR_INVALID;
        }
        if (e == first) {
          if (sel != 0 || q[0] != 0 || len < kPjHeader || (src & 15)) {
            set_error("tmmult sub-chunk %lld does not start with its header", (long long)s);
            return BMV_ERR_INVALID;
          }
          m = d->meta + src / 4;
          const int n_tri = m[kPjWarps];
          if (m[0] != 0 || n_tri < 0 || kPjHeader + 16 * (int64_t)n_tri > len || m[17] < 0 ||
              m[17] >= d->n_items || m[19] < 0 || m[19] > kPjUnits) {
            set_error("tmmult header of sub-chunk %lld is malformed", (long long)s);
            return BMV_ERR_INVALID;
          }
          for (int w = 0; w < kPjWarps; ++w)
            if (m[w] > m[w + 1] || m[20 + w] < 0 || m[20 + w] > kPjSlots) {
              set_error("tmmult header of sub-chunk %lld is malformed", (long long)s);
              return BMV_ERR_INVALID;
            }
          for (int u = 0; u < m[19]; ++u)
            if ((m[36 + u] & 0xff) >= kPjWarps || (m[36 + u] >> 8) >= kPjSlots) {
              set_error("tmmult unit owner of sub-chunk %lld out of range", (long long)s);
              return BMV_ERR_INVALID;
            }
          for (int t = 0; t < n_tri; ++t) {
            const int32_t* q4 = m + kPjHeader / 4 + 4 * t;
            const int rows = q4[2] & 0xffff, unit = (q4[2] >> 16) & 0xff;
            const int ac = (q4[2] >> 24) & 15, bc = ((unsigned)q4[2] >> 28) & 15;
            const int as = q4[3] & 0xffff, bs = ((unsigned)q4[3] >> 16) & 0xffff;
            const int64_t a_end = 8 * ((int64_t)q4[0] + (int64_t)(rows - 1) * as + ac);
            const int64_t b_end = 8 * ((int64_t)q4[1] + (int64_t)(rows - 1) * bs + bc);
            if (q4[0] < 0 || q4[1] < 0 || unit >= m[19] || ac > 8 || bc > 8 ||
                (rows > 0 && (a_end > d->stage_bytes || b_end > d->stage_bytes))) {
              set_error("tmmult triple tile %d of sub-chunk %lld out of range", t, (long long)s);
              return BMV_ERR_INVALID;
            }
          }
        }
        if ((y >> 30) & 1) {
          ++e;
          break;
        }
      }
    }
    if (e != e1) {
      set_error("tmmult part %d has stray copy entries", p);
      return BMV_ERR_INVALID;
    }
  }
  const int64_t partial_tiles = d->n_items * kPjWarps * kPjSlots;
  for (int64_t j = 0; j < d->n_src; ++j)
    if (d->tile_src[j] < 0 || d->tile_src[j] >= partial_tiles) {
      set_error("tmmult reduction source out of range");
      return BMV_ERR_INVALID;
    }
  return BMV_OK;
}

}  // namespace

extern "C" {

int bmv_tmmult_destroy(bmv_tmmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->part_sub_start, p->part_entry_start, p->tile_off, p->tile_src_start,
                  p->tile_src,       p->copies,           p->meta,     p->tile_shape,
                  p->partial};
  for (void* q : ptrs) release(q);
  delete p;
  return BMV_OK;
}

int bmv_tmmult_create(const bmv_tmmult_desc* d, bmv_tmmult** out) {
  if (!out) return BMV_ERR_INVALID;
  *out = nullptr;
  if (!d || d->n_parts < 0 || d->n_sub < 0 || d->n_items < 0 || d->n_entries < 0 ||
      d->meta_len < 0 || d->n_out_tiles < 0 || d->n_src < 0 || d->stage_bytes < kPjHeader ||
      (d->stage_bytes & 15)) {
    set_error("invalid tmmult descriptor");
    return BMV_ERR_INVALID;
  }
  if (d->n_warps != kPjWarps || d->slots_per_warp != kPjSlots) {
    set_error("tmmult plan built for %d warps x %d slots, kernel has %d x %d", d->n_warps,
              d->slots_per_warp, kPjWarps, kPjSlots);
    return BMV_ERR_INVALID;
  }
  int rc = validate_tmmult(d);
  if (rc) return rc;
  int dev = 0, max_smem = 0;
  BMV_CUDA_TRY(cudaGetDevice(&dev));
  BMV_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int avail = max_smem - 1024 - kPjResultDoubles * 8;
  const int ns = std::min(kPjMaxStages, avail / d->stage_bytes);
  if (ns < 2) {
    set_error("tmmult stage of %d bytes leaves fewer than 2 pipeline stages", d->stage_bytes);
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_tmmult();
  p->n_parts = d->n_parts;
  p->n_sub = d->n_sub;
  p->n_items = d->n_items;
  p->n_tiles = d->n_out_tiles;
  p->stage_bytes = d->stage_bytes;
  p->n_stages = ns;
  p->smem_bytes = kPjResultDoubles * 8 + ns * d->stage_bytes;
  for (int64_t t = 0; t < d->n_out_tiles; ++t) {
    const int32_t* q = d->tile_shape + 3 * t;
    if (q[0] > 0 && q[1] > 0)
      p->c_extent = std::max<int64_t>(p->c_extent, d->tile_off[t] + (int64_t)(q[0] - 1) * q[2] + q[1]);
  }
  const int64_t partial_tiles = d->n_items * kPjWarps * kPjSlots;
  rc = upload(d->part_sub_start, (int64_t)d->n_parts + 1, &p->part_sub_start);
  if (!rc) rc = upload(d->part_entry_start, (int64_t)d->n_parts + 1, &p->part_entry_start);
  if (!rc) rc = upload(d->copies, 4 * d->n_entries, &p->copies);
  if (!rc) rc = upload(d->meta, d->meta_len, &p->meta);
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
                                               max_smem - 1024);
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
  if (c_len < p->c_extent) {
    set_error("tmmult output of %lld values, plan writes up to %lld", (long long)c_len,
              (long long)p->c_extent);
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  int rc = zero_async(c, c_len, st);
  if (rc) return rc;
  if (p->n_sub > 0 && p->n_parts > 0) {
    PjArgs g{p->part_sub_start, p->part_entry_start, reinterpret_cast<const int4*>(p->copies),
             CopySrc{reinterpret_cast<const char*>(p->meta), reinterpret_cast<const char*>(a),
                     reinterpret_cast<const char*>(b)},
             p->partial, p->stage_bytes, p->n_stages};
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
