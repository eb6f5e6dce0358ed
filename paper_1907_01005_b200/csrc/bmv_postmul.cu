// K5: the post-multiplication Y_ij (+)= alpha sum_k A_ik B_kj truncated to
// Y's pattern (reference mmult, bcsr.py:587-628, Gustavson order :605-626)
// on the reference's block-CSR storage.
//
// HBM-bound streaming design (same pipeline as K4, bmv_project.cu): the
// owned block rows are cut into sub-chunks of consecutive rows whose A
// blocks are one contiguous value range, and the sub-chunks into one part
// per SM.  One persistent CTA per part: a producer warp streams the A
// ranges into a ring of shared-memory stages with TMA bulk copies; eight
// consumer warps take the 8x8 output tiles of the sub-chunk's Y blocks
// round-robin, accumulate sum_pairs A_ik B_kj with DMMA (A from the stage,
// the small B through L1/L2) and store each tile once.  No reduction, no
// atomics: every Y value is written by one lane in a fixed order.
#include <cuda_runtime.h>

#include <algorithm>

#include "bmv_common.cuh"
#include "bmv_tma.cuh"

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st);
}

using namespace bmv;

namespace {

constexpr int kPmWarps = 15;  // + the producer: 16 warps, 4 per SM sub-partition
constexpr int kPmThreads = (kPmWarps + 1) * 32;
constexpr int kPmMaxStages = 8;

struct PmArgs {
  const int64_t* __restrict__ part_sub_start;
  const int64_t* __restrict__ part_entry_start;
  const int4* __restrict__ copies;
  CopySrc src;  // p0 = meta, p1 = a, p2 = b
  double* __restrict__ c;
  double alpha;
  int accumulate;
  int stage_bytes;
  int n_stages;
};

constexpr int kPmRowTiles = 8;  // 8-row tiles per task (64 rows)

// One task = up to 8 row tiles x one 8-column tile of an output block:
// acc[m] += sum_pairs A[8 (mi0 + m) + gid][k] B[k][8 ni + 2 tig + {0,1}],
// A and B blocks both in the stage.
__device__ __forceinline__ void task_tiles(const double* S, const int4* pairs, const int4 t,
                                           int gid, int tig, double (&acc)[kPmRowTiles][2]) {
  const int rows = t.y & 0x7f, cv = (t.y >> 8) & 15, ni = (t.y >> 12) & 15;
  const int p0 = t.z & 0xffff, np = (t.z >> 16) & 0xffff;
  const bool bm = gid < cv;
  const int nm = (rows + 7) >> 3;
  for (int p = p0; p < p0 + np; ++p) {
    const int4 d = pairs[p];
    const int as = d.y & 0xffff, inner = (d.y >> 16) & 0xffff, bs = d.z;
    const double* A = S + d.x + (8 * t.w + gid) * as + tig;
    const double* B = S + d.w + tig * bs + 8 * ni + gid;
    for (int k0 = 0; k0 < inner; k0 += 4) {
      const bool ok = k0 + tig < inner;
      const double bk = (bm && ok) ? B[k0 * bs] : 0.0;
#pragma unroll
      for (int m = 0; m < kPmRowTiles; ++m) {
        if (m < nm) {
          const double a = (8 * m + gid < rows && ok) ? A[8 * m * as + k0] : 0.0;
          dmma_8x8x4(acc[m][0], acc[m][1], a, bk);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kPmThreads, 1) pm_stream_kernel(const PmArgs g) {
  extern __shared__ __align__(128) char stages[];
  __shared__ __align__(8) uint64_t full[kPmMaxStages], empty[kPmMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = g.part_sub_start[blockIdx.x], s1 = g.part_sub_start[blockIdx.x + 1];
  const int NS = g.n_stages;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NS; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kPmWarps);
    }
  }
  __syncthreads();

  if (warp == kPmWarps) {
    stream_producer(g.copies, g.part_entry_start[blockIdx.x], g.part_entry_start[blockIdx.x + 1],
                    s1 - s0, g.src, stages, g.stage_bytes, NS, full, empty, lane);
    return;
  }

  const int gid = lane >> 2, tig = lane & 3;
  for (int64_t i = 0; i < s1 - s0; ++i) {
    const int st = (int)(i % NS);
    mbar_wait(&full[st], (unsigned)((i / NS) & 1));
    const char* stg = stages + (int64_t)st * g.stage_bytes;
    const int4* meta = reinterpret_cast<const int4*>(stg);
    const double* S = reinterpret_cast<const double*>(stg);
    const int n_tasks = meta[0].x;
    const int4* tasks = meta + 1;
    const int4* pairs = meta + 1 + n_tasks;
    for (int k = warp; k < n_tasks; k += kPmWarps) {
      const int4 t = tasks[k];
      double acc[kPmRowTiles][2];
#pragma unroll
      for (int m = 0; m < kPmRowTiles; ++m) acc[m][0] = acc[m][1] = 0.0;
      task_tiles(S, pairs, t, gid, tig, acc);
      const int rows = t.y & 0x7f, cv = (t.y >> 8) & 15, ys = (t.y >> 16) & 0xffff;
      const int col = 2 * tig;
      const bool two = col + 1 < cv;
#pragma unroll
      for (int m = 0; m < kPmRowTiles; ++m) {
        const int r = 8 * m + gid;
        if (r < rows && col < cv) {
          double* Y = g.c + (uint32_t)t.x + (int64_t)r * ys + col;
          double x = g.alpha * acc[m][0], y = g.alpha * acc[m][1];
          if (two && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0)) {
            double2* Y2 = reinterpret_cast<double2*>(Y);
            if (g.accumulate) {
              const double2 old = *Y2;
              x += old.x;
              y += old.y;
            }
            *Y2 = make_double2(x, y);
          } else {
            Y[0] = g.accumulate ? Y[0] + x : x;
            if (two) Y[1] = g.accumulate ? Y[1] + y : y;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

}  // namespace

struct bmv_mmult {
  int n_parts = 0, stage_bytes = 0, n_stages = 0, smem_bytes = 0;
  int64_t n_sub = 0, c_extent = 0;
  int64_t *part_sub_start = nullptr, *part_entry_start = nullptr;
  int32_t *copies = nullptr, *meta = nullptr;
};

namespace {

int validate_mmult(const bmv_mmult_desc* d, int64_t* c_extent) {
  const int64_t meta_bytes = d->meta_len * 4;
  *c_extent = 0;
  if (d->n_parts > 0 && (d->part_sub_start[0] != 0 || d->part_sub_start[d->n_parts] != d->n_sub ||
                         d->part_entry_start[0] != 0 || d->part_entry_start[d->n_parts] != d->n_entries)) {
    set_error("mmult part ranges do not cover the sub-chunks / copies");
    return BMV_ERR_INVALID;
  }
  for (int p = 0; p < d->n_parts; ++p) {
    int64_t e = d->part_entry_start[p];
    const int64_t e1 = d->part_entry_start[p + 1];
    for (int64_t s = d->part_sub_start[p]; s < d->part_sub_start[p + 1]; ++s) {
      const int64_t first = e;
      for (;; ++e) {
        if (e >= e1) {
          set_error("mmult copy list of sub-chunk %lld is malformed", (long long)s);
          return BMV_ERR_INVALID;
        }
        const int32_t* q = d->copies + 4 * e;
        const unsigned y = (unsigned)q[1];
        const int64_t len = y & kCpLenMask, sel = (y >> 28) & 3;
        const int64_t src = ((int64_t)(uint32_t)q[3] << 32) | (uint32_t)q[2];
        if (q[0] < 0 || q[0] + len > d->stage_bytes || sel > 2 || src < 0 ||
            (sel == 0 && src + len > meta_bytes)) {
          set_error("mmult copy entry %lld out of range", (long long)e);
          return BMV_ERR_INVALID;
        }
        if (e == first) {
          if (sel != 0 || q[0] != 0 || len < 16 || (src & 15)) {
            set_error("mmult sub-chunk %lld does not start with its header", (long long)s);
            return BMV_ERR_INVALID;
          }
          const int32_t* m = d->meta + src / 4;
          const int nt = m[0];
          if (nt < 0 || 16 * (1 + (int64_t)nt) > len) {
            set_error("mmult header of sub-chunk %lld is malformed", (long long)s);
            return BMV_ERR_INVALID;
          }
          const int64_t n_pairs = len / 16 - 1 - nt;
          for (int k = 0; k < nt; ++k) {
            const int32_t* t = m + 4 * (1 + k);
            const int rows = t[1] & 0x7f, cv = (t[1] >> 8) & 15;
            const int ys = ((unsigned)t[1] >> 16) & 0xffff;
            const int p0 = t[2] & 0xffff, np = ((unsigned)t[2] >> 16) & 0xffff;
            if (rows > 8 * kPmRowTiles || cv > 8 || p0 + np > n_pairs || t[3] < 0) {
              set_error("mmult task %d of sub-chunk %lld out of range", k, (long long)s);
              return BMV_ERR_INVALID;
            }
            if (rows > 0 && cv > 0)
              *c_extent = std::max<int64_t>(*c_extent, (int64_t)(uint32_t)t[0] + (int64_t)(rows - 1) * ys + cv);
            for (int pp = p0; pp < p0 + np; ++pp) {
              const int32_t* q4 = m + 4 * (1 + nt + pp);
              const int as = q4[1] & 0xffff, inner = ((unsigned)q4[1] >> 16) & 0xffff, bs = q4[2];
              const int ni = (t[1] >> 12) & 15;
              const int64_t a_end = 8 * ((int64_t)q4[0] + (int64_t)(8 * t[3] + rows - 1) * as + inner);
              const int64_t b_end = 8 * ((int64_t)q4[3] + (int64_t)(inner - 1) * bs + 8 * ni + cv);
              if (q4[0] < 0 || bs < 0 || q4[3] < 0 ||
                  (rows > 0 && inner > 0 && a_end > d->stage_bytes) ||
                  (cv > 0 && inner > 0 && b_end > d->stage_bytes)) {
                set_error("mmult pair %d of sub-chunk %lld out of range", pp, (long long)s);
                return BMV_ERR_INVALID;
              }
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
      set_error("mmult part %d has stray copy entries", p);
      return BMV_ERR_INVALID;
    }
  }
  return BMV_OK;
}

}  // namespace

extern "C" {

int bmv_mmult_destroy(bmv_mmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->part_sub_start, p->part_entry_start, p->copies, p->meta};
  for (void* q : ptrs) release(q);
  delete p;
  return BMV_OK;
}

int bmv_mmult_create(const bmv_mmult_desc* d, bmv_mmult** out) {
  if (!out) return BMV_ERR_INVALID;
  *out = nullptr;
  if (!d || d->n_parts < 0 || d->n_sub < 0 || d->n_entries < 0 || d->meta_len < 0 ||
      d->stage_bytes < 16 || (d->stage_bytes & 15)) {
    set_error("invalid mmult descriptor");
    return BMV_ERR_INVALID;
  }
  int64_t c_extent = 0;
  int rc = validate_mmult(d, &c_extent);
  if (rc) return rc;
  int dev = 0, max_smem = 0;
  BMV_CUDA_TRY(cudaGetDevice(&dev));
  BMV_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int ns = std::min(kPmMaxStages, (max_smem - 1024) / d->stage_bytes);
  if (ns < 2) {
    set_error("mmult stage of %d bytes leaves fewer than 2 pipeline stages", d->stage_bytes);
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_mmult();
  p->n_parts = d->n_parts;
  p->n_sub = d->n_sub;
  p->c_extent = c_extent;
  p->stage_bytes = d->stage_bytes;
  p->n_stages = ns;
  p->smem_bytes = ns * d->stage_bytes;
  rc = upload(d->part_sub_start, (int64_t)d->n_parts + 1, &p->part_sub_start);
  if (!rc) rc = upload(d->part_entry_start, (int64_t)d->n_parts + 1, &p->part_entry_start);
  if (!rc) rc = upload(d->copies, 4 * d->n_entries, &p->copies);
  if (!rc) rc = upload(d->meta, d->meta_len, &p->meta);
  if (!rc) {
    const cudaError_t e = cudaFuncSetAttribute(pm_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               max_smem - 1024);
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
  if (c_len > 0 && c_len < p->c_extent) {
    set_error("mmult output of %lld values, plan writes up to %lld", (long long)c_len,
              (long long)p->c_extent);
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  if (!accumulate) {
    int rc = zero_async(c, c_len, st);
    if (rc) return rc;
  }
  if (p->n_sub == 0 || p->n_parts == 0) return BMV_OK;
  PmArgs g{p->part_sub_start, p->part_entry_start, reinterpret_cast<const int4*>(p->copies),
           CopySrc{reinterpret_cast<const char*>(p->meta), reinterpret_cast<const char*>(a),
                   reinterpret_cast<const char*>(b)},
           c, alpha, accumulate, p->stage_bytes, p->n_stages};
  pm_stream_kernel<<<(unsigned)p->n_parts, kPmThreads, p->smem_bytes, st>>>(g);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

}  // extern "C"
