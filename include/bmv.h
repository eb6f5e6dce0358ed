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
 *   bmv_tmmult_*   <- tmmult (bcsr.py:631-667), local products before compress
 *   bmv_mmult_*    <- mmult (bcsr.py:587-628)
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
 * Sum-factorised cell operator on (cell, column) pairs.
 * Work unit: one active pair = one column (orbital lane) of X on one cell.
 * A "visit" is a (cell, column block) couple; a "group" is one distinct
 * local block row touched by the cell (CellDoFMap, matfree.py:58-87).
 *   X value of cell DoF d for pair p:
 *     s    = cell_slots[cell*n^3 + d]  (group = s >> 24, rib = s & 0xffffff)
 *     xoff = group_xoff[visit_goff[v] + group]   (-1: block absent => 0)
 *     X[xoff + rib*visit_stride[v] + pair_lane[p]]
 *   and the result is added at the same place of HX via group_hoff.      */
typedef struct {
  int32_t n;              /* nodes per axis (degree+1), 2..5; q = n        */
  int32_t n_cells;
  int32_t n_visits;
  int64_t n_pairs;
  int64_t n_groups_total; /* length of group_xoff / group_hoff             */
  int32_t n_colors;       /* 0: one launch, fp64 atomic scatter-add;
                             k>0: k launches over color_pair_start ranges,
                             plain read-modify-write (deterministic)      */
  const int64_t* color_pair_start; /* n_colors+1 entries (host)           */
  const int32_t* pair_visit;       /* n_pairs                             */
  const int32_t* pair_lane;        /* n_pairs                             */
  const int32_t* visit_cell;       /* n_visits                            */
  const int32_t* visit_stride;     /* n_visits                            */
  const int64_t* visit_goff;       /* n_visits + 1 (groups of visit v:
                                      [visit_goff[v], visit_goff[v+1]), <= 32) */
  const int64_t* group_xoff;       /* n_groups_total                      */
  const int64_t* group_hoff;       /* n_groups_total                      */
  const uint32_t* cell_slots;      /* n_cells * n^3                       */
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
   coef[cell * coef_stride + q] (coef_stride 0: same for every cell).
   zero_len > 0 first zeroes hx[0:zero_len] (dst.zero_out()).
   x, hx, coef: device. */
int bmv_cellop_apply(bmv_cellop* plan, int32_t kinetic, const double* coef,
                     int64_t coef_stride, const double* x, double* hx, int64_t zero_len,
                     void* stream);
/* Fused mass + Hamiltonian (reference compute_energy applies both to the
   same X, energy.py:129-174): hx = H x and mx = M x from one gather and one
   interpolation to the quadrature points; hx and mx share the plan's
   destination pattern; both zeroed over [0, zero_len) first.  mass_coef:
   the mass coefficient row (w3, padded to an even length, device).
   Needs the TMA plan (BMV_ERR_INVALID otherwise).                          */
int bmv_cellop_apply_hm(bmv_cellop* plan, const double* coef, int64_t coef_stride,
                        const double* mass_coef, const double* x, double* hx, double* mx,
                        int64_t zero_len, void* stream);
/* Device evaluation of the Gaussian-sum potential coefficient:
   coef[c*q3 + q] = w3[q] * scale * sum_k exp(-|x - center_k|^2 * inv_sigma2)
   at x = cell_origins[c] + quad_offsets[q].  All arrays device. */
int bmv_potential_gaussian(int64_t n_cells, int32_t q3, const double* cell_origins,
                           const double* quad_offsets, const double* w3,
                           const double* centers, int32_t n_centers, double inv_sigma2,
                           double scale, double* coef, void* stream);
/* Number of kernel launches one apply issues (for bench accounting). */
int bmv_cellop_launches(const bmv_cellop* plan, int32_t* out);

/* ---------------------------------------------------------- copy lists --
 * K4 and K5 stream sub-chunks (consecutive block rows, or a tile of one
 * long row) through a ring of shared-memory stages: one persistent CTA per
 * part (one part per SM), a producer warp issuing TMA bulk copies, consumer
 * warps on FP64 tensor cores.  What one sub-chunk stages is a copy list:
 * entries of 4 x int32 {dst byte offset in the stage, bytes | src << 28 |
 * last << 30, src byte offset lo, hi}; src 0 = the plan's metadata array,
 * 1 = operand a, 2 = operand b; consecutive entries per sub-chunk, the
 * last one flagged; the first entry stages the sub-chunk's metadata
 * (header + work descriptors) at offset 0.  Entries 16-byte aligned go
 * through cp.async.bulk, others are copied by the producer's lanes.       */

/* ------------------------------------------------------------------ K4 --
 * C(k,l) = sum_i A_ik^T B_il over the owned block rows i.
 * Stage = [header (68 int32)][triple tiles (4 x int32)][A blocks][B blocks].
 * Header: [0..16] first triple tile of each of the 16 consumer warps
 * (local index) and the end, [17] item, [18] 1 on the item's last
 * sub-chunk, [19] units, [20..35] slots used per warp in the item,
 * [36..67] unit -> owner warp | slot << 8.
 * Triple tile: {A tile offset, B tile offset (doubles from the stage
 * start), rows | unit << 16 | acols << 24 | bcols << 28, a_stride |
 * b_stride << 16}: sum_r A[r][0:acols] B[r][0:bcols].
 * A unit is one 8x8 output tile touched by the sub-chunk (<= 32); the
 * units are computed by the warps the host balanced them on, written to a
 * shared result buffer, and after a barrier of the consumer warps added by
 * the tile's owner warp into a register-resident accumulator.  An item
 * (run of sub-chunks of one part) touches <= 16 x 8 output tiles; at its
 * end each owner writes its tiles once to the partial buffer at
 * (item * 16 + warp) * 8 + slot; a second kernel sums every 8x8 output
 * tile's partials in item order (bit-reproducible, no atomics).          */
typedef struct {
  int32_t n_parts;           /* CTAs                                       */
  int32_t n_warps;           /* consumer warps per CTA (must be 16)        */
  int32_t slots_per_warp;    /* accumulator tiles per warp (must be 8)     */
  int32_t stage_bytes;       /* capacity of one pipeline stage (16 | it)   */
  int64_t n_sub;             /* sub-chunks                                 */
  int64_t n_items;
  int64_t n_entries;         /* copy-list entries                          */
  int64_t meta_len;          /* int32 values of metadata                   */
  int64_t n_out_tiles;       /* 8x8 tiles of the C blocks with work        */
  int64_t n_src;             /* partial tiles summed by the reduction      */
  const int64_t* part_sub_start;   /* n_parts + 1                          */
  const int64_t* part_entry_start; /* n_parts + 1                          */
  const int32_t* copies;     /* n_entries x 4                              */
  const int32_t* meta;       /* meta_len                                   */
  const int64_t* tile_off;   /* n_out_tiles: element offset in C           */
  const int32_t* tile_shape; /* n_out_tiles x 3: rows, cols, row stride    */
  const int64_t* tile_src_start; /* n_out_tiles + 1                        */
  const int64_t* tile_src;   /* n_src partial tile indices, item order     */
} bmv_tmmult_desc;

typedef struct bmv_tmmult bmv_tmmult;
int bmv_tmmult_create(const bmv_tmmult_desc* desc, bmv_tmmult** out);
int bmv_tmmult_destroy(bmv_tmmult* plan);
/* c[0:c_len] = 0, then every planned C tile = sum of its partials. */
int bmv_tmmult_run(bmv_tmmult* plan, const double* a, const double* b, double* c,
                   int64_t c_len, void* stream);

/* ------------------------------------------------------------------ K5 --
 * Y_ij (+)= alpha * sum_k A_ik B_kj, truncated to Y's pattern.
 * Stage = [header int4 {n_tasks, 0, 0, 0}][tasks (4 x int32)][pairs
 * (4 x int32)][B blocks used by the pairs][A blocks of the rows]; copy
 * entries: metadata, one per B block, A range.
 * Task = up to 64 rows x one 8-column tile of an output block: {element
 * offset of the tile's first row in Y (< 2^32), rows | cols << 8 |
 * col-tile << 12 | Y row stride << 16, first pair (index into the staged
 * pairs) | pairs << 16, first 8-row tile in the block}.  Pair: {A block
 * offset in the stage (doubles), a_stride | inner << 16, b_stride, B block
 * offset in the stage (doubles)}.  15 consumer warps take the tasks
 * round-robin and store every output value once.                         */
typedef struct {
  int32_t n_parts;           /* CTAs                                       */
  int32_t stage_bytes;       /* capacity of one pipeline stage (16 | it)   */
  int64_t n_sub;
  int64_t n_entries;
  int64_t meta_len;          /* int32 values of metadata                   */
  const int64_t* part_sub_start;   /* n_parts + 1                          */
  const int64_t* part_entry_start; /* n_parts + 1                          */
  const int32_t* copies;     /* n_entries x 4                              */
  const int32_t* meta;       /* meta_len                                   */
} bmv_mmult_desc;

typedef struct bmv_mmult bmv_mmult;
int bmv_mmult_create(const bmv_mmult_desc* desc, bmv_mmult** out);
int bmv_mmult_destroy(bmv_mmult* plan);
/* accumulate=0: c[0:c_len] = 0 first (zero_out).  Blocks without pairs
   keep their (zeroed or accumulated) content. */
int bmv_mmult_run(bmv_mmult* plan, const double* a, const double* b, double* c,
                  double alpha, int32_t accumulate, int64_t c_len, void* stream);

/* ------------------------------------------------- K4 / K5, lane-compacted --
 * Same products as bmv_tmmult_* / bmv_mmult_* (reference tmmult
 * bcsr.py:631-667, mmult bcsr.py:587-628), computed on the active columns of
 * A only: a_mask[pos] marks the lanes of A block pos that hold support
 * entries (the multivector's declared column support, support.py; all
 * stored lanes when A has none).  Values of A outside the mask must be 0.
 * S (K4) is accumulated with fp64 reductions: summation order is not
 * fixed (like K1's atomic scatter).  Owned block rows i = 0..n_rows-1;
 * positions index the host arrays below (element offsets into the
 * operand's value array).                                                 */
typedef struct {
  int32_t n_rows;
  const int32_t* row_rows;       /* rows of block row i                     */
  const int64_t* a_row_start;    /* n_rows + 1                              */
  const int64_t* a_off;          /* per A position                          */
  const int32_t* a_stride;
  const uint64_t* a_mask;        /* active lanes (bit l = lane l, l < 64)    */
  const int64_t* b_row_start;    /* n_rows + 1                              */
  const int64_t* b_off;
  const int32_t* b_stride;
  const int32_t* b_width;        /* columns of the B block                  */
  /* per (row i, A position, B position), row-major over (pa, pb) inside
     the row, rows in order: the S block of (col block of pa, col block of
     pb): element offset, row stride, rows (= width of pa's col block)    */
  const int64_t* c_off;
  const int32_t* c_stride;
  const int32_t* c_rows;
} bmv_tmmult_lane_desc;
typedef struct bmv_lane_plan bmv_lane_plan;
int bmv_tmmult_lane_create(const bmv_tmmult_lane_desc* desc, bmv_lane_plan** out);
/* c[0:c_len] = 0, then c += A^T B on the plan's blocks. */
int bmv_tmmult_lane_run(bmv_lane_plan* plan, const double* a, const double* b, double* c,
                        int64_t c_len, void* stream);
typedef struct {
  int32_t n_rows;
  const int32_t* row_rows;
  const int64_t* a_row_start;    /* A = X, n_rows + 1                       */
  const int64_t* a_off;
  const int32_t* a_stride;
  const uint64_t* a_mask;
  const int64_t* c_row_start;    /* C = Y (output), n_rows + 1              */
  const int64_t* c_off;
  const int32_t* c_stride;
  const int32_t* c_width;
  /* B = the square matrix: per (row i, A position, Y position), row-major
     over (pa, pc) inside the row starting at b_pair_start[i]: element
     offset of block (col block of pa, col block of pc) in b (-1: absent)
     and its row stride                                                   */
  const int64_t* b_pair_start;   /* n_rows                                  */
  const int64_t* b_off;
  const int32_t* b_stride;
} bmv_mmult_lane_desc;
int bmv_mmult_lane_create(const bmv_mmult_lane_desc* desc, bmv_lane_plan** out);
/* c[0:zero_len] = 0; then every planned Y block = alpha A B (+ old value if
   accumulate): all stored lanes of the planned blocks are written. */
int bmv_mmult_lane_run(bmv_lane_plan* plan, const double* a, const double* b, double* c,
                       double alpha, int32_t accumulate, int64_t zero_len, void* stream);
int bmv_lane_plan_destroy(bmv_lane_plan* plan);
/* Host-only (no device needed): the stage stream a lane plan would upload,
   for CPU emulation of the kernels in the tests.                         */
typedef struct {
  int32_t stage_bytes;
  int32_t n_parts;
  int64_t meta_len;          /* int32 words                               */
  int64_t n_entries;         /* copy entries (4 x int32)                  */
  int32_t* meta;
  int32_t* copies;
  int64_t* part_sub_start;   /* n_parts + 1                               */
  int64_t* part_entry_start; /* n_parts + 1                               */
} bmv_lane_host;
int bmv_lane_plan_host(int32_t kind, const void* desc, int32_t n_parts, bmv_lane_host* out);
int bmv_lane_host_free(bmv_lane_host* host);
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

#ifdef __cplusplus
}
#endif
#endif /* BMV_H */
