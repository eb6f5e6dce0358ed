/*
 * bmv.h -- C-ABI of libbmv.so, the B200 (sm_100a) kernels behind the
 * drop-in Python package `paper_1907_01005_b200`.
 *
 * The reference (`/root/reference/pkg/src/bcsrmv`) is a pure-Python package
 * with no FFI; each entry point below replaces the compute inside one of its
 * Python functions, which the package's shims keep with identical names:
 *
 *   bmv_cellop_*   <- CellOperator.apply cell loop + cell_integrals_sumfac
 *                     (matfree.py:458-527, 288-367), potential sampling
 *                     OperatorSpec.sample_potential (matfree.py:35-40,491-495)
 *   bmv_chunk_plan_*, bmv_tmmult_run
 *                  <- tmmult (bcsr.py:631-667), local products before compress
 *   bmv_chunk_plan_*, bmv_mmult_run
 *                  <- mmult (bcsr.py:587-628)
 *   bmv_index_*, bmv_gather, bmv_scatter
 *                  <- BlockCsrMatrix._pack_for_peer / update_ghost_values_finish
 *                     / compress_finish (bcsr.py:401-519)
 *   bmv_zero       <- BlockCsrMatrix.zero_out / zero_ghost_blocks (bcsr.py:334-339)
 *
 * Conventions: every function returns BMV_OK (0) or an error code and sets a
 * thread-local message readable with bmv_last_error().  Value arrays are
 * caller-owned DEVICE pointers to fp64; plan descriptors are HOST arrays
 * that *_create copies to device memory owned by the plan.  All launches are
 * asynchronous on the given cudaStream_t (passed as void*); nothing
 * allocates on the hot path.  One host thread (or process) per GPU.
 */
#ifndef BMV_H
#define BMV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BMV_OK 0
#define BMV_ERR_INVALID 1  /* bad argument -> ShapeError / DomainError      */
#define BMV_ERR_CUDA 2     /* CUDA runtime failure -> DeviceError           */
#define BMV_ERR_PATTERN 3  /* missing block -> PatternError                 */

#define BMV_MAX_NODES 5 /* nodes per axis, degree 1..4 */

int bmv_version(void);
const char* bmv_last_error(void);
/* kernels this library has launched so far (all threads) */
int bmv_launch_count(int64_t* out);
/* number of SMs of the current device (grid sizing helper) */
int bmv_device_sm_count(int* out);

/* ------------------------------------------------------------------ K1 --
 * Sum-factorised cell operator on (cell, column) pairs, slab storage
 * (paper_1907_01005_b200/slabs.py: block row i of a matrix stores a
 * row-major rows_i x K_i slab over its stored columns, at slab_off[i]).
 * Work unit: one active pair = one column of X on one cell.  A cell's
 * "groups" are the distinct local block rows its DoFs lie in
 * (CellDoFMap, matfree.py:58-87), in first-occurrence order.
 *   codes (per cell and DoF, row of code_stride uint32 words):
 *     32-bit: g << 27 | (r * K_src[g]) << 14 | (r * K_dst[g])   (13 / 14 bits)
 *     wide:   {g << 27 | r * K_src[g], r * K_dst[g]}
 *     (g: group, r: row of the DoF in that block row)
 *   gtab (per pair and group, int32 pairs): {slab_off_src[g] + slot of the
 *     pair's column in the src slab (-1: not stored -> value 0),
 *     slab_off_dst[g] + slot in the dst slab}
 *   X value of DoF d for pair p = X[gtab[p][g].x + rKx], H X accumulated at
 *   HX[gtab[p][g].y + rKh].
 * bmv_cellop_create cuts the pair list (pairs sorted by cell, group tables
 * consecutive) into batches of consecutive pairs -- n >= 4: up to 32 / n
 * pairs in at most two cells; n <= 3: up to 32 pairs in at most 8 cells --
 * never across a declared break, so that bmv_cellop_apply_pairs can run the
 * ranges between breaks separately (halo overlap).  The kernels are
 * persistent (one CTA per SM); limits: at most 32 groups per cell, pair
 * kernel: about 26 groups per cell (metadata stages in shared memory).     */
typedef struct {
  int32_t n;              /* nodes per axis (degree+1), 2..5; q = n        */
  int32_t wide;           /* 0: 32-bit codes, 1: 64-bit codes             */
  int32_t n_cells;
  int32_t code_stride;    /* uint32 words per code row (multiple of 4)     */
  int32_t max_groups;     /* max entries of a pair's table (<= 32, even)   */
  int64_t n_pairs;
  int64_t gtab_len;       /* int32 words of gtab                           */
  const int32_t* pair_cell;   /* n_pairs (cells ascending)                 */
  const int64_t* pair_gtab;   /* n_pairs: first int32 word of the pair's
                                 table (multiple of 4)                     */
  const int32_t* pair_ngp;    /* n_pairs: table entries (even)             */
  const int32_t* gtab;        /* gtab_len                                  */
  const uint32_t* codes;      /* n_cells * code_stride                     */
  int32_t n_breaks;           /* pair indices (ascending) at which a launch
                                 range of bmv_cellop_apply_*pairs may start
                                 or end, besides 0 and n_pairs              */
  const int64_t* breaks;
  /* 1D tables (row-major, q x n): Lagrange values S at the Gauss points and
     the collocation derivative D_co = D S^-1 (q x q); 1D weights w.       */
  double S[BMV_MAX_NODES * BMV_MAX_NODES];
  double Dco[BMV_MAX_NODES * BMV_MAX_NODES];
  double w[BMV_MAX_NODES];
  double kin[3];          /* det * 0.5 / h_d^2, d = x, y, z                */
  double det;             /* hx * hy * hz                                  */
} bmv_cellop_desc;

typedef struct bmv_cellop bmv_cellop;

int bmv_cellop_create(const bmv_cellop_desc* desc, bmv_cellop** out);
int bmv_cellop_destroy(bmv_cellop* plan);
/* hx = Op x on the plan's pairs.  kinetic=1 adds the -1/2 Laplacian;
   coef != NULL adds the coefficient term c(cell, q) * u(q) at the
   quadrature points (mass: w3; Hamiltonian potential: w3 * V), read at
   coef[cell * coef_stride + q] (coef_stride 0: same for every cell; else
   q^3 rounded up to even).  zero_len > 0 first zeroes hx[0:zero_len]
   (dst.zero_out()).  x, hx, coef: device. */
int bmv_cellop_apply(bmv_cellop* plan, int32_t kinetic, const double* coef,
                     int64_t coef_stride, const double* x, double* hx, int64_t zero_len,
                     void* stream);
/* Fused mass + Hamiltonian (reference compute_energy applies both to the
   same X, energy.py:129-174): hx = H x and mx = M x from one gather and one
   interpolation to the quadrature points; hx and mx share the plan's
   destination layout; both zeroed over [0, zero_len) first.  mass_coef:
   the mass coefficient row (w3, padded to an even length, device).        */
int bmv_cellop_apply_hm(bmv_cellop* plan, const double* coef, int64_t coef_stride,
                        const double* mass_coef, const double* x, double* hx, double* mx,
                        int64_t zero_len, void* stream);
/* The same products on the plan's pairs [pair_begin, pair_end) only, without
   zeroing: CellOperator.apply runs the pairs of cells touching no ghost row
   while the halo exchange is in flight (the plan orders its pairs: interior
   cells part A, cells with ghost rows, interior cells part B). */
int bmv_cellop_apply_pairs(bmv_cellop* plan, int32_t kinetic, const double* coef,
                           int64_t coef_stride, const double* x, double* hx,
                           int64_t pair_begin, int64_t pair_end, void* stream);
int bmv_cellop_apply_hm_pairs(bmv_cellop* plan, const double* coef, int64_t coef_stride,
                              const double* mass_coef, const double* x, double* hx, double* mx,
                              int64_t pair_begin, int64_t pair_end, void* stream);
/* Device evaluation of the Gaussian-sum potential coefficient:
   coef[c*q3 + q] = w3[q] * scale * sum_k exp(-|x - center_k|^2 * inv_sigma2)
   at x = cell_origins[c] + quad_offsets[q].  All arrays device. */
int bmv_potential_gaussian(int64_t n_cells, int32_t q3, const double* cell_origins,
                           const double* quad_offsets, const double* w3,
                           const double* centers, int32_t n_centers, double inv_sigma2,
                           double scale, double* coef, void* stream);
/* Number of kernel launches one apply issues besides the zeroing. */
int bmv_cellop_launches(const bmv_cellop* plan, int32_t* out);

/* ------------------------------------------------------------- K4 / K5 --
 * Projection S = A^T B (reference tmmult, bcsr.py:631-667, before the
 * compress) and post-multiply Y = alpha A C (+ Y) truncated to Y's stored
 * entries (reference mmult, bcsr.py:587-628) on slab storage.
 * A CHUNK is a run of consecutive owned rows of A (whole block rows, or a
 * row range of one long block row): its A values (K4: and its B values) are
 * one contiguous element range each.  Persistent CTAs (n_parts) take
 * contiguous chunk ranges; every warp claims chunks in order, copies
 * [meta | A | B] of its next chunks into private shared-memory buffers with
 * cp.async and multiplies the oldest (bmv_chunk_kernel_config: warps per
 * CTA, bytes per buffer = the largest chunk).
 * Chunk meta (int32 words, 16-byte multiple), header fields:
 *   [0] segments  [1] rows  [2] UA (union A columns)  [3] UB (union B / Y
 *   columns)  [4] NK  [5] byte offset of A in the buffer (= meta bytes)
 *   [6] of B (K4)  [7..12] word offsets of: segment records, A colmap,
 *   B/Y colmap, RB, KK, ST.
 * Segment record (8 words, one per block-row piece): {rows, A offset in the
 *   staged range (doubles), K_A (A's slab width), B offset in the staged
 *   range (K4) / element offset of the piece's first row in Y (K5), K_B,
 *   0, 0, 0}.
 * Colmaps (int16, segment x U): slab slot of a union column in that
 *   block row, -1 = not stored (structural zero).
 * Output / C addressing of union (a, b): RB[a] + ST[KK[a] * UB + b]
 *   (K4: element of S; K5: element of C), ST = -1: no such entry.          */
typedef struct {
  int32_t kind;              /* 4: projection (K4), 5: post-multiply (K5)  */
  int32_t n_parts;           /* CTAs                                       */
  int32_t stage_bytes;       /* largest chunk in bytes (multiple of 16)    */
  int64_t n_chunks;
  int64_t meta_len;          /* int32 words                                */
  const int64_t* part_chunk_start; /* n_parts + 1                          */
  const int64_t* chunk_meta; /* n_chunks + 1: first meta word of each chunk */
  const int32_t* meta;
  const int64_t* chunk_a;    /* n_chunks x 2: staged element range of A
                                [begin, end), both even                    */
  const int64_t* chunk_b;    /* K4: same for B; K5: unused (NULL)          */
} bmv_chunk_desc;

typedef struct bmv_chunk_plan bmv_chunk_plan;
int bmv_chunk_plan_create(const bmv_chunk_desc* desc, bmv_chunk_plan** out);
int bmv_chunk_plan_destroy(bmv_chunk_plan* plan);
/* c[0:c_len] = 0, then c += A^T B on the plan's chunks (fp64 reductions:
   the summation order across chunks is not fixed). */
int bmv_tmmult_run(const bmv_chunk_plan* plan, const double* a, const double* b, double* c,
                   int64_t c_len, void* stream);
/* y = alpha A C (+ y if accumulate) on every stored entry of the plan's rows
   (entries of Y outside the chunks are not touched). */
int bmv_mmult_run(const bmv_chunk_plan* plan, const double* a, const double* cmat, double* y,
                  double alpha, int32_t accumulate, void* stream);
/* warps per CTA and bytes per buffer (largest chunk) of the K4 / K5 kernel (kind 4 / 5);
   variant 0: default shape, 1: shape for short block rows (fewer warps, larger chunks).
   bmv_chunk_plan_create picks the shape from the plan's stage_bytes. */
int bmv_chunk_kernel_config(int32_t kind, int32_t variant, int32_t* warps, int32_t* buffer_bytes);

/* --------------------------------------------------------- halo / util --
 * Device index lists for ghost exchange packing.                         */
typedef struct bmv_index bmv_index;
int bmv_index_create(const int64_t* host_idx, int64_t n, bmv_index** out);
int bmv_index_destroy(bmv_index* idx);
int64_t bmv_index_size(const bmv_index* idx);
/* out[i] = src[idx[i]] */
int bmv_gather(const bmv_index* idx, const double* src, double* out, void* stream);
/* mode 0: dst[idx[i]] = in[i];  mode 1: dst[idx[i]] += in[i]
   (indices must be distinct within one call) */
int bmv_scatter(const bmv_index* idx, const double* in, double* dst, int32_t mode,
                void* stream);
/* p[0:n] = 0 */
int bmv_zero(double* p, int64_t n, void* stream);

/* ---------------------------------------------------------- measurement --
 * Dependent-free fp64 FMA stream: measures the device's FP64 FMA peak
 * (the roofline denominator for K1).  flops_out = 2 * FMAs issued.        */
int bmv_fp64_peak_kernel(double* scratch, int32_t blocks, int32_t iters,
                         double* flops_out, void* stream);
/* Same for the FP64 tensor cores (independent DMMA m8n8k4 chains). */
int bmv_fp64_dmma_peak_kernel(double* scratch, int32_t blocks, int32_t iters,
                              double* flops_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BMV_H */
