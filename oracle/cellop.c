/*
 * oracle/cellop.c -- TEST INFRASTRUCTURE ONLY (CPU oracle / CPU reference arm).
 *
 * Plain-C restatement of the reference hot path on the reference BCSR layout
 * (bcsrmv/bcsr.py:233-318: per block row, per stored column block, a
 * row-major (rows x stride) block, stride = ceil(cols / W) * W):
 *
 *   oracle_cellop_apply  Algorithm 6 (matfree.py:458-527): for every cell,
 *       the cell's DoFs are grouped by local block row in first-occurrence
 *       order (CellDoFMap, matfree.py:90-116); the non-empty column blocks of
 *       those rows are merged in ascending order (RowsBlockAccessor,
 *       matfree.py:159-237); for each column block and each group of W
 *       lanes: gather, 18-contraction cell integral in the reference order
 *       (cell_integrals_sumfac, matfree.py:288-367), scatter-add.  A missing
 *       destination block returns -3 (PatternError).
 *       Cells are processed colour by colour (8 parity classes of the
 *       structured mesh share no node), OpenMP inside a colour.
 *   oracle_tmmult  C = A^T B over owned block rows (bcsr.py:631-667), no
 *       compress (single rank); thread-private C, summed in thread order.
 *   oracle_mmult   C = alpha A B truncated to C's pattern (bcsr.py:587-628).
 *
 * Built by oracle/Makefile into oracle/liboracle.so.
 */
#include <stdint.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 5
#define MAXW 64

typedef struct {
  int n;                  /* nodes per axis; q = n */
  int W;                  /* lane width */
  int kind;               /* 0 mass, 1 hamiltonian */
  double S[MAXN * MAXN];  /* S[q*n + i] */
  double D[MAXN * MAXN];  /* D[q*n + i] */
  double w3[MAXN * MAXN * MAXN];
  double grad_scale[3];
} oracle_tables;

/* out = M (along axis) applied to in; tensors [n][n][n][L] (z, y, x, lane).
   tr = 0: out[..q..] = sum_i M[q][i] in[..i..];  tr = 1: sum_i M[i][q] in[..i..] */
static void contract(int n, int L, const double* M, int tr, const double* in, double* out,
                     int axis) {
  const int s2 = n * n * L, s1 = n * L, s0 = L;
  const int st = axis == 0 ? s2 : (axis == 1 ? s1 : s0);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      for (int q = 0; q < n; ++q) {
        int base_out, base_in;
        if (axis == 0) {
          base_out = q * s2 + a * s1 + b * s0;
          base_in = a * s1 + b * s0;
        } else if (axis == 1) {
          base_out = a * s2 + q * s1 + b * s0;
          base_in = a * s2 + b * s0;
        } else {
          base_out = a * s2 + b * s1 + q * s0;
          base_in = a * s2 + b * s1;
        }
        for (int l = 0; l < L; ++l) {
          double acc = 0.0;
          for (int i = 0; i < n; ++i) acc += (tr ? M[i * n + q] : M[q * n + i]) * in[base_in + i * st + l];
          out[base_out + l] = acc;
        }
      }
}

/* cell integral on u (n^3 x L) -> out, reference order of operations */
static void cell_integral(const oracle_tables* T, int L, const double* u, const double* vq,
                          double* out, double* w) {
  const int n = T->n, N3 = n * n * n, sz = N3 * L;
  double *tz = w, *tzy = w + sz, *uq = w + 2 * sz, *gx = w + 3 * sz, *tzd = w + 4 * sz,
         *gy = w + 5 * sz, *tdz = w + 6 * sz, *tdzy = w + 7 * sz, *gz = w + 8 * sz,
         *ax = w + 9 * sz, *tmp = w + 10 * sz, *by = w + 11 * sz, *czl = w + 12 * sz,
         *ab = w + 13 * sz, *cc = w + 14 * sz;
  contract(n, L, T->S, 0, u, tz, 0);
  contract(n, L, T->S, 0, tz, tzy, 1);
  contract(n, L, T->S, 0, tzy, uq, 2);
  if (T->kind == 0) {
    for (int p = 0; p < N3; ++p)
      for (int l = 0; l < L; ++l) uq[p * L + l] *= T->w3[p];
    contract(n, L, T->S, 1, uq, tmp, 2);
    contract(n, L, T->S, 1, tmp, ab, 1);
    contract(n, L, T->S, 1, ab, out, 0);
    return;
  }
  contract(n, L, T->D, 0, tzy, gx, 2);
  contract(n, L, T->D, 0, tz, tzd, 1);
  contract(n, L, T->S, 0, tzd, gy, 2);
  contract(n, L, T->D, 0, u, tdz, 0);
  contract(n, L, T->S, 0, tdz, tdzy, 1);
  contract(n, L, T->S, 0, tdzy, gz, 2);
  for (int p = 0; p < N3; ++p) {
    const double fx = T->w3[p] * T->grad_scale[0], fy = T->w3[p] * T->grad_scale[1],
                 fz = T->w3[p] * T->grad_scale[2];
    for (int l = 0; l < L; ++l) {
      gx[p * L + l] *= fx;
      gy[p * L + l] *= fy;
      gz[p * L + l] *= fz;
    }
  }
  contract(n, L, T->D, 1, gx, ax, 2);
  if (vq) {
    for (int p = 0; p < N3; ++p)
      for (int l = 0; l < L; ++l) uq[p * L + l] *= T->w3[p] * vq[p];
    contract(n, L, T->S, 1, uq, tmp, 2);
    for (int k = 0; k < sz; ++k) ax[k] += tmp[k];
  }
  contract(n, L, T->S, 1, gy, by, 2);
  contract(n, L, T->S, 1, gz, czl, 2);
  contract(n, L, T->S, 1, ax, ab, 1);
  contract(n, L, T->D, 1, by, tmp, 1);
  for (int k = 0; k < sz; ++k) ab[k] += tmp[k];
  contract(n, L, T->S, 1, czl, cc, 1);
  contract(n, L, T->S, 1, ab, out, 0);
  contract(n, L, T->D, 1, cc, tmp, 0);
  for (int k = 0; k < sz; ++k) out[k] += tmp[k];
}

typedef struct {
  const int64_t* row_start;
  const int64_t* col_index;
  const int64_t* block_offsets;
  const int64_t* col_strides; /* per column block */
  const int64_t* col_sizes;   /* per column block */
} bcsr_view;

static int64_t find_pos(const bcsr_view* m, int64_t lb, int64_t col) {
  int64_t lo = m->row_start[lb], hi = m->row_start[lb + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (m->col_index[mid] < col)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < m->row_start[lb + 1] && m->col_index[lo] == col) return lo;
  return -1;
}

/* returns 0, or -3 if the destination misses a block, -1 on bad input */
int oracle_cellop_apply(const oracle_tables* T, int64_t n_cells, const int64_t* cell_lb,
                        const int64_t* cell_rib, const int32_t* cell_color, const double* vq,
                        const int64_t* x_row_start, const int64_t* x_col_index,
                        const int64_t* x_block_offsets, const int64_t* h_row_start,
                        const int64_t* h_col_index, const int64_t* h_block_offsets,
                        const int64_t* col_strides, const int64_t* col_sizes, const double* x,
                        double* hx, int n_threads) {
  if (!T || T->n < 2 || T->n > MAXN || T->W < 1 || T->W > MAXW) return -1;
  const int n = T->n, N3 = n * n * n, W = T->W;
  bcsr_view X = {x_row_start, x_col_index, x_block_offsets, col_strides, col_sizes};
  bcsr_view H = {h_row_start, h_col_index, h_block_offsets, col_strides, col_sizes};
  int status = 0;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
  for (int color = 0; color < 8; ++color) {
#pragma omp parallel
    {
      double* work = (double*)malloc(sizeof(double) * (size_t)N3 * W * 17);
      double* u = work + 15 * (size_t)N3 * W;
      double* o = work + 16 * (size_t)N3 * W;
      int64_t glb[MAXN * MAXN * MAXN];
      int gof[MAXN * MAXN * MAXN];
      int64_t cur[MAXN * MAXN * MAXN], end[MAXN * MAXN * MAXN];
#pragma omp for schedule(dynamic, 16)
      for (int64_t c = 0; c < n_cells; ++c) {
        if (cell_color && cell_color[c] != color) continue;
        if (!cell_color && color != 0) continue;
        const int64_t* lb = cell_lb + c * N3;
        const int64_t* rib = cell_rib + c * N3;
        /* groups in first-occurrence order */
        int ng = 0;
        for (int d = 0; d < N3; ++d) {
          int g = 0;
          while (g < ng && glb[g] != lb[d]) ++g;
          if (g == ng) glb[ng++] = lb[d];
          gof[d] = g;
        }
        for (int g = 0; g < ng; ++g) {
          cur[g] = X.row_start[glb[g]];
          end[g] = X.row_start[glb[g] + 1];
        }
        for (;;) {
          int64_t C = INT64_MAX;
          for (int g = 0; g < ng; ++g)
            if (cur[g] < end[g] && X.col_index[cur[g]] < C) C = X.col_index[cur[g]];
          if (C == INT64_MAX) break;
          const int64_t stride = col_strides[C];
          int64_t hpos[MAXN * MAXN * MAXN], xpos[MAXN * MAXN * MAXN];
          int bad = 0;
          for (int g = 0; g < ng; ++g) {
            xpos[g] = (cur[g] < end[g] && X.col_index[cur[g]] == C) ? cur[g] : -1;
            hpos[g] = find_pos(&H, glb[g], C);
            if (hpos[g] < 0) bad = 1;
          }
          if (bad) {
#pragma omp atomic write
            status = -3;
            break;
          }
          for (int64_t l0 = 0; l0 < stride; l0 += W) {
            for (int d = 0; d < N3; ++d) {
              const int g = gof[d];
              for (int l = 0; l < W; ++l)
                u[d * W + l] = xpos[g] >= 0 ? x[X.block_offsets[xpos[g]] + rib[d] * stride + l0 + l] : 0.0;
            }
            cell_integral(T, W, u, vq ? vq + c * N3 : NULL, o, work);
            for (int d = 0; d < N3; ++d) {
              double* dst = hx + H.block_offsets[hpos[gof[d]]] + rib[d] * stride + l0;
              for (int l = 0; l < W; ++l) dst[l] += o[d * W + l];
            }
          }
          for (int g = 0; g < ng; ++g)
            if (cur[g] < end[g] && X.col_index[cur[g]] == C) ++cur[g];
        }
      }
      free(work);
    }
    if (!cell_color) break;
  }
  return status;
}

/* C += A^T B for owned rows [0, n_rows); c_local_block[k] = local row of C for
   global column block k (-1: none). Returns -3 if C lacks a product block. */
int oracle_tmmult(int64_t n_rows, const int64_t* a_row_start, const int64_t* a_col_index,
                  const int64_t* a_block_offsets, const int64_t* a_col_strides,
                  const int64_t* a_col_sizes, const int64_t* row_sizes, const double* a,
                  const int64_t* b_row_start, const int64_t* b_col_index,
                  const int64_t* b_block_offsets, const int64_t* b_col_strides,
                  const int64_t* b_col_sizes, const double* b, const int64_t* c_local_block,
                  const int64_t* c_row_start, const int64_t* c_col_index,
                  const int64_t* c_block_offsets, const int64_t* c_col_strides, double* c,
                  int64_t c_len, int n_threads) {
  int status = 0;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  double* part = (double*)calloc((size_t)nt * (size_t)c_len, sizeof(double));
  if (!part) return -1;
  bcsr_view Cv = {c_row_start, c_col_index, c_block_offsets, c_col_strides, b_col_sizes};
#pragma omp parallel
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* cp = part + (size_t)tid * c_len;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i) {
      const int64_t r = row_sizes[i];
      for (int64_t pa = a_row_start[i]; pa < a_row_start[i + 1]; ++pa) {
        const int64_t k = a_col_index[pa];
        const int64_t ck = c_local_block[k];
        const int64_t ka = a_col_sizes[k], sa = a_col_strides[k];
        for (int64_t pb = b_row_start[i]; pb < b_row_start[i + 1]; ++pb) {
          const int64_t l = b_col_index[pb];
          const int64_t cpos = ck >= 0 ? find_pos(&Cv, ck, l) : -1;
          if (cpos < 0) {
#pragma omp atomic write
            status = -3;
            continue;
          }
          const int64_t lb = b_col_sizes[l], sb = b_col_strides[l], sc = c_col_strides[l];
          const double* A = a + a_block_offsets[pa];
          const double* B = b + b_block_offsets[pb];
          double* Cb = cp + c_block_offsets[cpos];
          for (int64_t ii = 0; ii < ka; ++ii)
            for (int64_t jj = 0; jj < lb; ++jj) {
              double acc = 0.0;
              for (int64_t rr = 0; rr < r; ++rr) acc += A[rr * sa + ii] * B[rr * sb + jj];
              Cb[ii * sc + jj] += acc;
            }
        }
      }
    }
  }
  for (int t = 0; t < nt; ++t)
    for (int64_t e = 0; e < c_len; ++e) c[e] += part[(size_t)t * c_len + e];
  free(part);
  return status;
}

/* C = alpha A B (+ C), truncated to C's pattern; B rows addressed by global
   column block k through b_local_block[k]. */
int oracle_mmult(int64_t n_rows, const int64_t* a_row_start, const int64_t* a_col_index,
                 const int64_t* a_block_offsets, const int64_t* a_col_strides,
                 const int64_t* a_col_sizes, const int64_t* row_sizes, const double* a,
                 const int64_t* b_local_block, const int64_t* b_row_start,
                 const int64_t* b_col_index, const int64_t* b_block_offsets,
                 const int64_t* b_col_strides, const int64_t* b_col_sizes, const double* b,
                 const int64_t* c_row_start, const int64_t* c_col_index,
                 const int64_t* c_block_offsets, double* c, double alpha, int n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t r = row_sizes[i];
    for (int64_t pa = a_row_start[i]; pa < a_row_start[i + 1]; ++pa) {
      const int64_t k = a_col_index[pa];
      const int64_t kb = b_local_block[k];
      if (kb < 0) continue;
      const int64_t ka = a_col_sizes[k], sa = a_col_strides[k];
      int64_t cp = c_row_start[i];
      const int64_t ce = c_row_start[i + 1];
      for (int64_t pb = b_row_start[kb]; pb < b_row_start[kb + 1]; ++pb) {
        const int64_t j = b_col_index[pb];
        while (cp < ce && c_col_index[cp] < j) ++cp;
        if (cp == ce) break;
        if (c_col_index[cp] != j) continue;
        const int64_t nj = b_col_sizes[j], sb = b_col_strides[j];
        const double* A = a + a_block_offsets[pa];
        const double* B = b + b_block_offsets[pb];
        double* Cb = c + c_block_offsets[cp];
        for (int64_t rr = 0; rr < r; ++rr)
          for (int64_t jj = 0; jj < nj; ++jj) {
            double acc = 0.0;
            for (int64_t kk = 0; kk < ka; ++kk) acc += A[rr * sa + kk] * B[kk * sb + jj];
            Cb[rr * sb + jj] += alpha * acc;
          }
      }
    }
  }
  return 0;
}

/* V(x) = scale * sum_k exp(-|x - c_k|^2 * inv_s2) at x = origins[c] + qoff[q]
   (the BASELINE Gaussian-sum potential, matfree.py:35-40 sampled at the
   quadrature points as in matfree.py:491-495); out[c * q3 + q]. */
int oracle_potential_gaussian(int64_t n_cells, int q3, const double* origins, const double* qoff,
                              const double* centers, int n_centers, double inv_s2, double scale,
                              double* out, int n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n_cells; ++c) {
    for (int q = 0; q < q3; ++q) {
      const double px = origins[3 * c] + qoff[3 * q], py = origins[3 * c + 1] + qoff[3 * q + 1],
                   pz = origins[3 * c + 2] + qoff[3 * q + 2];
      double v = 0.0;
      for (int k = 0; k < n_centers; ++k) {
        const double dx = px - centers[3 * k], dy = py - centers[3 * k + 1],
                     dz = pz - centers[3 * k + 2];
        v += exp(-(dx * dx + dy * dy + dz * dz) * inv_s2);
      }
      out[c * q3 + q] = scale * v;
    }
  }
  return 0;
}
