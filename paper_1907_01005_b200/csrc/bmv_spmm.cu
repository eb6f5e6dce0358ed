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
  const int64_t* __restrict__ seg_out;
  const int64_t* __restrict__ seg_tri_start;
  const int64_t* __restrict__ seg_poff;
  const int64_t* __restrict__ tri_a_off;
  const int64_t* __restrict__ tri_b_off;
  const int32_t* __restrict__ tri_rows;
  const int32_t* __restrict__ tri_a_stride;
  const int32_t* __restrict__ tri_b_stride;
  int64_t n_seg;
  const double* __restrict__ a;
  const double* __restrict__ b;
  double* __restrict__ partial;
  double* __restrict__ c;
};

constexpr int kTmEPT = 8;  // entries per lane: output blocks up to 256 entries

// One warp per segment: partial[k][l] = sum_triples sum_r A[r][k] * B[r][l]
__global__ void __launch_bounds__(128) tm_partial_kernel(const TmArgs g) {
  const int64_t seg = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (seg >= g.n_seg) return;
  const int lane = threadIdx.x & 31;
  const int64_t o = g.seg_out[seg];
  const int cols = g.out_cols[o];
  const int ent = g.out_rows[o] * cols;
  int ii[kTmEPT], jj[kTmEPT];
  double acc[kTmEPT];
#pragma unroll
  for (int k = 0; k < kTmEPT; ++k) {
    const int e = lane + 32 * k;
    ii[k] = e < ent ? e / cols : 0;
    jj[k] = e < ent ? e - (e / cols) * cols : 0;
    acc[k] = 0.0;
  }
  const int64_t t1 = g.seg_tri_start[seg + 1];
  for (int64_t t = g.seg_tri_start[seg]; t < t1; ++t) {
    const double* A = g.a + g.tri_a_off[t];
    const double* B = g.b + g.tri_b_off[t];
    const int as = g.tri_a_stride[t], bs = g.tri_b_stride[t], nr = g.tri_rows[t];
    for (int r = 0; r < nr; ++r) {
#pragma unroll
      for (int k = 0; k < kTmEPT; ++k)
        if (lane + 32 * k < ent)
          acc[k] = fma(__ldg(A + (int64_t)r * as + ii[k]), __ldg(B + (int64_t)r * bs + jj[k]), acc[k]);
    }
  }
  double* P = g.partial + g.seg_poff[seg];
#pragma unroll
  for (int k = 0; k < kTmEPT; ++k)
    if (lane + 32 * k < ent) P[lane + 32 * k] = acc[k];
}

// One CTA per output block: C = sum of its segments' partials, chunk order.
__global__ void __launch_bounds__(128) tm_reduce_kernel(const TmArgs g) {
  const int64_t o = blockIdx.x;
  const int cols = g.out_cols[o], cst = g.out_stride[o];
  const int ent = g.out_rows[o] * cols;
  const int64_t s0 = g.out_seg_start[o], s1 = g.out_seg_start[o + 1];
  for (int e = threadIdx.x; e < ent; e += blockDim.x) {
    double acc = 0.0;
    for (int64_t s = s0; s < s1; ++s) acc += g.partial[g.seg_poff[g.out_seg_list[s]] + e];
    const int i = e / cols, j = e - i * cols;
    g.c[g.out_off[o] + (int64_t)i * cst + j] = acc;
  }
}

struct MmArgs {
  const int64_t* __restrict__ out_off;
  const int32_t* __restrict__ out_rows;
  const int32_t* __restrict__ out_cols;
  const int32_t* __restrict__ out_stride;
  const int64_t* __restrict__ pair_start;
  const int64_t* __restrict__ pair_a_off;
  const int32_t* __restrict__ pair_a_stride;
  const int32_t* __restrict__ pair_inner;
  const int64_t* __restrict__ pair_b_off;
  const int32_t* __restrict__ pair_b_stride;
  const double* __restrict__ a;
  const double* __restrict__ b;
  double* __restrict__ c;
  double alpha;
  int accumulate;
};

// One warp per output block: C(i,j)[r][s] (+)= alpha * sum_pairs sum_k A[r][k] B[k][s]
__global__ void __launch_bounds__(128) mmult_kernel(const MmArgs g, int64_t n_out) {
  const int64_t o = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (o >= n_out) return;
  const int lane = threadIdx.x & 31;
  const int rows = g.out_rows[o], cols = g.out_cols[o], cst = g.out_stride[o];
  const int64_t p0 = g.pair_start[o], p1 = g.pair_start[o + 1];
  const int entries = rows * cols;
  for (int e = lane; e < entries; e += 32) {
    const int r = e / cols, s = e - r * cols;
    double acc = 0.0;
    for (int64_t p = p0; p < p1; ++p) {
      const double* A = g.a + g.pair_a_off[p] + (int64_t)r * g.pair_a_stride[p];
      const double* B = g.b + g.pair_b_off[p] + s;
      const int bs = g.pair_b_stride[p], nk = g.pair_inner[p];
      for (int k = 0; k < nk; ++k) acc = fma(__ldg(A + k), __ldg(B + (int64_t)k * bs), acc);
    }
    double* dst = g.c + g.out_off[o] + (int64_t)r * cst + s;
    *dst = g.accumulate ? fma(g.alpha, acc, *dst) : g.alpha * acc;
  }
}

}  // namespace

struct bmv_tmmult {
  int64_t n_out = 0, n_seg = 0, n_tri = 0, partial_len = 0;
  int64_t* out_off = nullptr;
  int32_t *out_rows = nullptr, *out_cols = nullptr, *out_stride = nullptr;
  int64_t *out_seg_start = nullptr, *out_seg_list = nullptr, *seg_out = nullptr,
          *seg_tri_start = nullptr, *seg_poff = nullptr;
  int64_t *tri_a_off = nullptr, *tri_b_off = nullptr;
  int32_t *tri_rows = nullptr, *tri_a_stride = nullptr, *tri_b_stride = nullptr;
  double* partial = nullptr;
};

struct bmv_mmult {
  int64_t n_out = 0, n_pairs = 0;
  int64_t* out_off = nullptr;
  int32_t *out_rows = nullptr, *out_cols = nullptr, *out_stride = nullptr;
  int64_t *pair_start = nullptr, *pair_a_off = nullptr, *pair_b_off = nullptr;
  int32_t *pair_a_stride = nullptr, *pair_inner = nullptr, *pair_b_stride = nullptr;
};

extern "C" {

int bmv_tmmult_destroy(bmv_tmmult* p) {
  if (!p) return BMV_OK;
  void* ptrs[] = {p->out_off, p->out_rows, p->out_cols, p->out_stride, p->out_seg_start,
                  p->out_seg_list, p->seg_out, p->seg_tri_start, p->seg_poff, p->tri_a_off,
                  p->tri_b_off, p->tri_rows, p->tri_a_stride, p->tri_b_stride, p->partial};
  for (void* q : ptrs) release(q);
  delete p;
  return BMV_OK;
}

int bmv_tmmult_create(const bmv_tmmult_desc* d, bmv_tmmult** out) {
  if (!d || !out || d->n_out < 0 || d->n_seg < 0 || d->n_triples < 0 || d->partial_len < 0) {
    set_error("invalid tmmult descriptor");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  for (int64_t o = 0; o < d->n_out; ++o) {
    if ((int64_t)d->out_rows[o] * d->out_cols[o] > 32 * kTmEPT) {
      set_error("tmmult output block of %d x %d entries exceeds %d", d->out_rows[o],
                d->out_cols[o], 32 * kTmEPT);
      return BMV_ERR_INVALID;
    }
  }
  auto* p = new bmv_tmmult();
  p->n_out = d->n_out;
  p->n_seg = d->n_seg;
  p->n_tri = d->n_triples;
  p->partial_len = d->partial_len;
  int rc = upload(d->out_off, d->n_out, &p->out_off);
  if (!rc) rc = upload(d->out_rows, d->n_out, &p->out_rows);
  if (!rc) rc = upload(d->out_cols, d->n_out, &p->out_cols);
  if (!rc) rc = upload(d->out_stride, d->n_out, &p->out_stride);
  if (!rc) rc = upload(d->out_seg_start, d->n_out + 1, &p->out_seg_start);
  if (!rc) rc = upload(d->out_seg_list, d->n_seg, &p->out_seg_list);
  if (!rc) rc = upload(d->seg_out, d->n_seg, &p->seg_out);
  if (!rc) rc = upload(d->seg_tri_start, d->n_seg + 1, &p->seg_tri_start);
  if (!rc) rc = upload(d->seg_poff, d->n_seg, &p->seg_poff);
  if (!rc) rc = upload(d->tri_a_off, d->n_triples, &p->tri_a_off);
  if (!rc) rc = upload(d->tri_b_off, d->n_triples, &p->tri_b_off);
  if (!rc) rc = upload(d->tri_rows, d->n_triples, &p->tri_rows);
  if (!rc) rc = upload(d->tri_a_stride, d->n_triples, &p->tri_a_stride);
  if (!rc) rc = upload(d->tri_b_stride, d->n_triples, &p->tri_b_stride);
  if (!rc && d->partial_len > 0) {
    if (cudaMalloc((void**)&p->partial, sizeof(double) * (size_t)d->partial_len) != cudaSuccess) {
      set_error("cudaMalloc of %lld partial values failed", (long long)d->partial_len);
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
           p->out_seg_list, p->seg_out, p->seg_tri_start, p->seg_poff, p->tri_a_off,
           p->tri_b_off, p->tri_rows, p->tri_a_stride, p->tri_b_stride, p->n_seg, a, b,
           p->partial, c};
  if (p->n_seg > 0) {
    tm_partial_kernel<<<(unsigned)((p->n_seg + 3) / 4), 128, 0, st>>>(g);
    BMV_CHECK_LAUNCH();
  }
  tm_reduce_kernel<<<(unsigned)p->n_out, 64, 0, st>>>(g);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

int bmv_mmult_destroy(bmv_mmult* p) {
  if (!p) return BMV_OK;
  release(p->out_off);
  release(p->out_rows);
  release(p->out_cols);
  release(p->out_stride);
  release(p->pair_start);
  release(p->pair_a_off);
  release(p->pair_b_off);
  release(p->pair_a_stride);
  release(p->pair_inner);
  release(p->pair_b_stride);
  delete p;
  return BMV_OK;
}

int bmv_mmult_create(const bmv_mmult_desc* d, bmv_mmult** out) {
  if (!d || !out || d->n_out < 0 || d->n_pairs < 0) {
    set_error("invalid mmult descriptor");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  auto* p = new bmv_mmult();
  p->n_out = d->n_out;
  p->n_pairs = d->n_pairs;
  int rc = upload(d->out_off, d->n_out, &p->out_off);
  if (!rc) rc = upload(d->out_rows, d->n_out, &p->out_rows);
  if (!rc) rc = upload(d->out_cols, d->n_out, &p->out_cols);
  if (!rc) rc = upload(d->out_stride, d->n_out, &p->out_stride);
  if (!rc) rc = upload(d->pair_start, d->n_out + 1, &p->pair_start);
  if (!rc) rc = upload(d->pair_a_off, d->n_pairs, &p->pair_a_off);
  if (!rc) rc = upload(d->pair_a_stride, d->n_pairs, &p->pair_a_stride);
  if (!rc) rc = upload(d->pair_inner, d->n_pairs, &p->pair_inner);
  if (!rc) rc = upload(d->pair_b_off, d->n_pairs, &p->pair_b_off);
  if (!rc) rc = upload(d->pair_b_stride, d->n_pairs, &p->pair_b_stride);
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
  if (p->n_out == 0) return BMV_OK;
  MmArgs g{p->out_off, p->out_rows, p->out_cols, p->out_stride, p->pair_start, p->pair_a_off,
           p->pair_a_stride, p->pair_inner, p->pair_b_off, p->pair_b_stride, a, b, c, alpha,
           accumulate};
  mmult_kernel<<<(unsigned)((p->n_out + 3) / 4), 128, 0, st>>>(g, p->n_out);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

}  // extern "C"
