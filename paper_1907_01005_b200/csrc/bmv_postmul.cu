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

constexpr int kPmWarps = 8;
constexpr int kPmThreads = (kPmWarps + 1) * 32;
constexpr int kPmMaxStages = 8;
constexpr int kPmPiece = 4096;

struct PmArgs {
  const int64_t* __restrict__ part_sub_start;
  const int64_t* __restrict__ sub_a;     // [lo, hi) per sub-chunk
  const int64_t* __restrict__ sub_tile;  // [t0, t1) per sub-chunk
  const int64_t* __restrict__ sub_out0;  // first output block of the sub-chunk
  const int64_t* __restrict__ tile_start;  // n_out + 1
  const int64_t* __restrict__ out_off;
  const int4* __restrict__ out_shape;    // rows, cols, stride, -
  const int64_t* __restrict__ pair_start;
  const int4* __restrict__ pair;         // a_soff, a_stride | inner << 16, b_stride, b_off
  const double* __restrict__ a;
  const double* __restrict__ b;
  double* __restrict__ c;
  double alpha;
  int accumulate;
  int stage_doubles;
  int n_stages;
  int bulk_ok;
};

__global__ void __launch_bounds__(kPmThreads, 1) pm_stream_kernel(const PmArgs g) {
  extern __shared__ __align__(128) double stages[];
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

  if (warp == kPmWarps) {  // producer
    for (int64_t s = s0; s < s1; ++s) {
      const int64_t i = s - s0;
      const int st = (int)(i % NS);
      if (i >= NS) mbar_wait(&empty[st], (unsigned)((i / NS - 1) & 1));
      double* dst = stages + (int64_t)st * g.stage_doubles;
      const int64_t alo = g.sub_a[2 * s], ahi = g.sub_a[2 * s + 1];
      const int na = (int)(ahi - alo);
      if (g.bulk_ok && ((alo | ahi) & 1) == 0) {
        if (lane == 0) {
          mbar_expect_tx(&full[st], (unsigned)na * 8u);
          for (int k = 0; k < na; k += kPmPiece)
            bulk_g2s(dst + k, g.a + alo + k, (unsigned)min(kPmPiece, na - k) * 8u, &full[st]);
        }
      } else {
        for (int k = lane; k < na; k += 32) dst[k] = __ldg(g.a + alo + k);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
    }
    return;
  }

  const int gid = lane >> 2, tig = lane & 3;
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t i = s - s0;
    const int st = (int)(i % NS);
    mbar_wait(&full[st], (unsigned)((i / NS) & 1));
    const double* S = stages + (int64_t)st * g.stage_doubles;
    const int64_t t1 = g.sub_tile[2 * s + 1];
    int64_t o = g.sub_out0[s];
    int64_t o_end = g.tile_start[o + 1];
    for (int64_t t = g.sub_tile[2 * s] + warp; t < t1; t += kPmWarps) {
      while (o_end <= t) o_end = g.tile_start[++o + 1];
      const int4 shp = __ldg(g.out_shape + o);
      const int rows = shp.x, cols = shp.y, ys = shp.z;
      const int tn = (cols + 7) >> 3;
      const int mt = (int)(t - g.tile_start[o]);
      const int mi = mt / tn, ni = mt - mi * tn;
      const int r = 8 * mi + gid, cb = 8 * ni + gid;
      const bool rv = r < rows, cv = cb < cols;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      const int64_t p1 = g.pair_start[o + 1];
      for (int64_t p = g.pair_start[o]; p < p1; ++p) {
        const int4 d = __ldg(g.pair + p);
        const int as = d.y & 0xffff, inner = (d.y >> 16) & 0xffff, bs = d.z;
        const double* A = S + d.x + r * as + tig;
        const double* B = g.b + (uint32_t)d.w + (int64_t)tig * bs + cb;
        int k0 = 0;
        for (; k0 + 8 <= inner; k0 += 8) {
          const double a0 = rv ? A[k0] : 0.0, a1 = rv ? A[k0 + 4] : 0.0;
          const double b0 = cv ? __ldg(B + (int64_t)k0 * bs) : 0.0;
          const double b1 = cv ? __ldg(B + (int64_t)(k0 + 4) * bs) : 0.0;
          dmma_8x8x4(c0, c1, a0, b0);
          dmma_8x8x4(c2, c3, a1, b1);
        }
        for (; k0 < inner; k0 += 4) {
          const bool ok = k0 + tig < inner;
          const double a0 = (rv && ok) ? A[k0] : 0.0;
          const double b0 = (cv && ok) ? __ldg(B + (int64_t)k0 * bs) : 0.0;
          dmma_8x8x4(c0, c1, a0, b0);
        }
      }
      const int col = 8 * ni + 2 * tig;
      if (rv && col < cols) {
        double* Y = g.c + g.out_off[o] + (int64_t)r * ys + col;
        double x = g.alpha * (c0 + c2), y = g.alpha * (c1 + c3);
        const bool two = col + 1 < cols;
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

}  // namespace

struct bmv_mmult {
  int n_parts = 0, stage_doubles = 0, n_stages = 0, smem_bytes = 0;
  int64_t n_sub = 0, n_out = 0, n_pairs = 0;
  int64_t *part_sub_start = nullptr, *sub_a = nullptr, *sub_tile = nullptr, *sub_out0 = nullptr,
          *tile_start = nullptr, *out_off = nullptr, *pair_start = nullptr;
  int32_t *out_shape = nullptr, *pair = nullptr;
};

extern "C" {

int bmv_mmult_destroy(bmv_mmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->part_sub_start, p->sub_a,     p->sub_tile,  p->sub_out0, p->tile_start,
                  p->out_off,        p->pair_start, p->out_shape, p->pair};
  for (void* q : ptrs) release(q);
  delete p;
  return BMV_OK;
}

int bmv_mmult_create(const bmv_mmult_desc* d, bmv_mmult** out) {
  if (!out) return BMV_ERR_INVALID;
  *out = nullptr;
  if (!d || d->n_parts < 0 || d->n_sub < 0 || d->n_out < 0 || d->n_pairs < 0 ||
      d->stage_doubles < 2 || (d->stage_doubles & 1)) {
    set_error("invalid mmult descriptor");
    return BMV_ERR_INVALID;
  }
  if (d->n_parts > 0 && (d->part_sub_start[0] != 0 || d->part_sub_start[d->n_parts] != d->n_sub)) {
    set_error("mmult part ranges do not cover the sub-chunks");
    return BMV_ERR_INVALID;
  }
  const int64_t n_tiles = d->n_out > 0 ? d->tile_start[d->n_out] : 0;
  for (int64_t s = 0; s < d->n_sub; ++s) {
    const int64_t na = d->sub_a[2 * s + 1] - d->sub_a[2 * s];
    const int64_t t0 = d->sub_tile[2 * s], t1 = d->sub_tile[2 * s + 1];
    if (na < 0 || na > d->stage_doubles || t0 > t1 || t1 > n_tiles ||
        (t1 > t0 && (d->sub_out0[s] < 0 || d->sub_out0[s] >= d->n_out ||
                     d->tile_start[d->sub_out0[s]] > t0))) {
      set_error("mmult sub-chunk %lld is inconsistent", (long long)s);
      return BMV_ERR_INVALID;
    }
  }
  for (int64_t o = 0; o < d->n_out; ++o) {
    const int32_t* q = d->out_shape + 4 * o;
    const int64_t tiles = (int64_t)((q[0] + 7) / 8) * ((q[1] + 7) / 8);
    if (q[0] < 0 || q[1] < 0 || d->tile_start[o + 1] - d->tile_start[o] != tiles ||
        d->pair_start[o + 1] < d->pair_start[o]) {
      set_error("mmult output block %lld is inconsistent", (long long)o);
      return BMV_ERR_INVALID;
    }
  }
  if (d->n_out > 0 && d->pair_start[d->n_out] != d->n_pairs) {
    set_error("mmult pair ranges do not cover the pairs");
    return BMV_ERR_INVALID;
  }
  for (int64_t p = 0; p < d->n_pairs; ++p)
    if (d->pair[4 * p] < 0 || d->pair[4 * p + 3] < 0) {
      set_error("mmult pair %lld has a bad offset", (long long)p);
      return BMV_ERR_INVALID;
    }
  int dev = 0, max_smem = 0;
  BMV_CUDA_TRY(cudaGetDevice(&dev));
  BMV_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int ns = std::min(kPmMaxStages, (max_smem - 1024) / (d->stage_doubles * 8));
  if (ns < 2) {
    set_error("mmult stage of %d doubles leaves fewer than 2 pipeline stages", d->stage_doubles);
    return BMV_ERR_INVALID;
  }
  auto* p = new bmv_mmult();
  p->n_parts = d->n_parts;
  p->n_sub = d->n_sub;
  p->n_out = d->n_out;
  p->n_pairs = d->n_pairs;
  p->stage_doubles = d->stage_doubles;
  p->n_stages = ns;
  p->smem_bytes = ns * d->stage_doubles * 8;
  int rc = upload(d->part_sub_start, (int64_t)d->n_parts + 1, &p->part_sub_start);
  if (!rc) rc = upload(d->sub_a, 2 * d->n_sub, &p->sub_a);
  if (!rc) rc = upload(d->sub_tile, 2 * d->n_sub, &p->sub_tile);
  if (!rc) rc = upload(d->sub_out0, d->n_sub, &p->sub_out0);
  if (!rc) rc = upload(d->tile_start, d->n_out + 1, &p->tile_start);
  if (!rc) rc = upload(d->out_off, d->n_out, &p->out_off);
  if (!rc) rc = upload(d->out_shape, 4 * d->n_out, &p->out_shape);
  if (!rc) rc = upload(d->pair_start, d->n_out + 1, &p->pair_start);
  if (!rc) rc = upload(d->pair, 4 * d->n_pairs, &p->pair);
  if (!rc) {
    const cudaError_t e = cudaFuncSetAttribute(pm_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               p->smem_bytes);
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
  if (p->n_sub == 0 || p->n_parts == 0) return BMV_OK;
  const int bulk_ok = (reinterpret_cast<uintptr_t>(a) & 15) == 0;
  PmArgs g{p->part_sub_start, p->sub_a, p->sub_tile, p->sub_out0, p->tile_start, p->out_off,
           reinterpret_cast<const int4*>(p->out_shape), p->pair_start,
           reinterpret_cast<const int4*>(p->pair), a, b, c, alpha, accumulate,
           p->stage_doubles, p->n_stages, bulk_ok};
  pm_stream_kernel<<<(unsigned)p->n_parts, kPmThreads, p->smem_bytes, st>>>(g);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

}  // extern "C"
