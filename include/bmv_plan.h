/* bmv_plan.h — native host plan builder (libbmvplan.so, C++/OpenMP, no CUDA).
 *
 * Setup-time index maps of the hot path that the reference builds in Python
 * ("C++ plan construction, bit-exact").  Host pointers,
 * int64 indices, return 0 on success, 1 on invalid arguments, 3 when an entry
 * falls outside the matrix pattern (the Python shim raises ConsistencyError).
 *
 * Reference interfaces each entry point replaces:
 *   bmvp_hash_fill            bench/problem.py:113-131 fill_multivector (splitmix64
 *                             `_mix64` hash of (seed, row, original column)); here the
 *                             per-entry form used by problem.fill_multivector
 *   bmvp_owned_entries_*      bcsr.py:233-318 storage offsets of the support entries of
 *                             a multivector (ColumnSupport.owned_entries; slab layout)
 *   bmvp_support_columns_*    bcsr.py:233-318 which columns a block row stores (the
 *                             slab columns of a support-declared multivector)
 *   bmvp_blocks_of            bcsr.py:126-152 map_rows (row -> (block, row in block))
 *   bmvp_first_touch          mesh.py:263-322 enumerate_dofs (first-touch positions)
 *   bmvp_grow_*               localization.py:251-267 grow_sparsity_for_operator
 *                             (block pattern inc^T (inc S) + S)
 *   bmvp_first_groups_*       matfree.py:90-116 build_cell_dof_map: per-cell grouping of
 *                             DoFs by row block in first-occurrence order
 *   bmvp_chunk_*              bcsr.py:587-667 tmmult / mmult block loops: the K4 / K5
 *                             chunk plans (union columns, colmaps, output slots)
 *   bmvp_support_transpose, bmvp_cell_pairs, bmvp_block_image, bmvp_k1_plan
 *                             matfree.py:159-237,458-527: active (cell, column) pairs,
 *                             the operator image (entry-level grown pattern) and the
 *                             K1 group tables
 */
#ifndef BMV_PLAN_H
#define BMV_PLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int bmvp_version(void);

/* out[flat ? flat[i] : i] = scale * (mix64(rows[i]*K1 + c*K2 + seed) / 2^64 - 0.5),
 * c = col_map ? col_map[cols[i]] : cols[i]. */
int bmvp_hash_fill(uint64_t seed, int64_t n, const int64_t* rows, const int64_t* cols,
                   const int64_t* col_map, const int64_t* flat, double scale, double* out);

/* block[i] = b with starts[b] <= idx[i] < starts[b+1]; offset[i] = idx[i] - starts[b]
 * (offset may be NULL).  Returns 1 if an index lies outside [starts[0], starts[n_blocks]).
 * Replaces the searchsorted of bcsr.py:126-152 map_rows (owned rows). */
int bmvp_blocks_of(int64_t n_blocks, const int64_t* starts, int64_t n, const int64_t* idx,
                   int64_t* block, int64_t* offset);

/* col_count[c] = #{support rows of column c in [lo, hi)}; columns are CSR
 * (col_ptr[n_cols+1], col_rows sorted per column). */
int bmvp_owned_entries_count(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                             int64_t lo, int64_t hi, int64_t* col_count);

/* Column-major (column, then row) support entries of the owned rows: storage
 * offset, global row, column.  out_start[c] = exclusive prefix sum of col_count.
 * block_starts: global first row of the nb_own owned block rows (+ end);
 * slab_ptr / slab_cols / slab_off: the matrix's slab geometry over its owned
 * block rows (stored columns ascending per row, slab offsets; slabs.py).
 * Returns 3 if a support entry has no stored slot. */
int bmvp_owned_entries_fill(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                            int64_t lo, int64_t hi, const int64_t* out_start,
                            int64_t nb_own, const int64_t* block_starts,
                            const int64_t* slab_ptr, const int64_t* slab_cols,
                            const int64_t* slab_off, int64_t* flat, int64_t* rows,
                            int64_t* cols);

/* Stored columns of selected global block rows from a column support
 * (ColumnSupport.columns_for): column c is stored in block row g when one of
 * its support rows lies in [block_starts[g], block_starts[g+1]).
 * block_sel[g] = index of g among the n_sel selected rows, -1 otherwise.
 * count: counts[s] = columns of selected row s.  fill: ptr = exclusive prefix
 * sum of counts (n_sel + 1), cursor scratch (n_sel); cols ascending per row. */
int bmvp_support_columns_count(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                               int64_t n_blocks, const int64_t* block_starts,
                               const int64_t* block_sel, int64_t n_sel, int64_t* counts);
int bmvp_support_columns_fill(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                              int64_t n_blocks, const int64_t* block_starts,
                              const int64_t* block_sel, int64_t n_sel, const int64_t* ptr,
                              int64_t* cursor, int64_t* cols);

/* lb: (n_cells, n3) local block of every cell DoF.  slot_group (n_cells, n3):
 * group index of each DoF inside its cell, groups in first-occurrence order;
 * cell_count[c] = groups of cell c (n3 <= 4096). */
int bmvp_first_groups_count(int64_t n_cells, int32_t n3, const int64_t* lb,
                            int64_t* slot_group, int64_t* cell_count);

/* cell_gstart = exclusive prefix sum of cell_count; fills grp_cell / grp_block. */
int bmvp_first_groups_fill(int64_t n_cells, int32_t n3, const int64_t* lb,
                           const int64_t* slot_group, const int64_t* cell_gstart,
                           int64_t* grp_cell, int64_t* grp_block);

/* first[v] = smallest pos with touches[pos] == v, else n (first-touch DoF numbering). */
int bmvp_first_touch(int64_t n_nodes, int64_t n, const int64_t* touches, int64_t* first);

/* Block pattern of H X from the pattern S of X: row block rb holds column block cb iff
 * S[rb, cb] or some cell touching rb touches a row block rb' with S[rb', cb].
 * cell_rb: (n_cells, n3) row block of every cell DoF; bits: n_rb * ceil(n_cb/64) words,
 * zeroed by the caller, returned as the row bitsets; row_count[rb] = popcount. */
int bmvp_grow_count(int64_t n_cells, int32_t n3, const int64_t* cell_rb, int64_t n_rb,
                    int64_t n_cb, const int64_t* s_row_start, const int64_t* s_col_index,
                    uint64_t* bits, int64_t* row_count);

/* Sorted column indices of every row from the bitsets; row_start = prefix sum of row_count. */
int bmvp_grow_fill(int64_t n_rb, int64_t n_cb, const uint64_t* bits, const int64_t* row_start,
                   int64_t* col_index);

/* K4 / K5 chunk plan (include/bmv.h bmv_chunk_desc), replacing the block
 * loops of reference tmmult / mmult (bcsr.py:587-667).  Owned block rows
 * 0..n_rows-1 of A with rows[i] rows; slab geometry (ptr, cols, off) of A,
 * of B (K4: the second factor, staged; K5: the output Y), and of M (K4: the
 * output S; K5: the factor C) over M's local block rows; M row of A column
 * col: local block m_ltab[cb] of A's column block cb (acb_starts), row
 * col - acb_starts[cb].  Chunks: <= max_rows rows, <= max_brows block rows,
 * <= data_bytes of staged values, meta + values <= stage_bytes; n_parts
 * contiguous chunk ranges of equal estimated cost.  bmvp_chunk_status: 0
 * ok, 1 invalid arguments, 3 M lacks a block row (PatternError), 4 a row
 * does not fit a stage, 5 offsets beyond 2^31. */
typedef struct bmvp_chunks bmvp_chunks;
bmvp_chunks* bmvp_chunk_plan(int32_t kind, int64_t n_rows, const int64_t* rows,
                             const int64_t* a_ptr, const int64_t* a_cols, const int64_t* a_off,
                             const int64_t* b_ptr, const int64_t* b_cols, const int64_t* b_off,
                             int64_t n_acb, const int64_t* acb_starts, const int64_t* m_ltab,
                             const int64_t* m_ptr, const int64_t* m_cols, const int64_t* m_off,
                             int32_t max_rows, int32_t max_brows, int32_t data_bytes,
                             int32_t stage_bytes, int32_t n_parts);
int bmvp_chunk_status(const bmvp_chunks* c);
void bmvp_chunk_sizes(const bmvp_chunks* c, int64_t* n_chunks, int64_t* meta_len, int64_t* dmma);
void bmvp_chunk_copy(const bmvp_chunks* c, int64_t* part_start, int64_t* chunk_meta, int32_t* meta,
                     int64_t* chunk_a, int64_t* chunk_b);
void bmvp_chunk_free(bmvp_chunks* c);

/* Row -> columns transpose of a column support over selected rows (row_sel:
 * global row -> selected index or -1).  Pass 1 (cols NULL): ptr (n_sel + 1).
 * Pass 2: cols (int32), ascending per row.  (matfree active pairs / images) */
int bmvp_support_transpose(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                           const int64_t* row_sel, int64_t n_sel, int64_t* ptr, int32_t* cols);
/* Per cell the sorted union of the columns of its n3 rows (cell_rows: indices
 * into the row CSR row_ptr / row_cols, -1 none): the active (cell, column)
 * pairs of K1 (reference RowsBlockAccessor emission, matfree.py:159-237, at
 * entry level).  Two passes as above. */
int bmvp_cell_pairs(int64_t n_cells, int32_t n3, const int64_t* cell_rows, const int64_t* row_ptr,
                    const int32_t* row_cols, int64_t* ptr, int32_t* cols);
/* Operator image per selected block row: union of the pair columns of the
 * cells touching it (cell_blocks (n_cells, n3): selected block or -1); the
 * stored columns of H X (matfree.ImageColumns; the grown pattern,
 * localization.py:251-267, at entry level).  Two passes as above. */
int bmvp_block_image(int64_t n_cells, int32_t n3, const int64_t* cell_blocks,
                     const int64_t* pair_ptr, const int32_t* pair_cols, int64_t n_blocks,
                     int64_t n_cols, int64_t* ptr, int64_t* cols);
/* K1 per-pair group tables (include/bmv.h bmv_cellop_desc gtab): for pair p
 * (cell, column) and each group g of the cell, {src slab offset + slot or -1,
 * dst slab offset + slot}; odd group counts padded with {-1, 0}.  Returns 3
 * and *bad_pair when dst lacks a slot (PatternError). */
int bmvp_k1_plan(int64_t n_pairs, const int64_t* pair_cell, const int64_t* pair_col,
                 const int64_t* cell_gstart, const int64_t* grp_block, const int64_t* src_ptr,
                 const int64_t* src_cols, const int64_t* src_off, const int64_t* dst_ptr,
                 const int64_t* dst_cols, const int64_t* dst_off, const int64_t* pair_gtab,
                 int32_t* gtab, int64_t* bad_pair);

#ifdef __cplusplus
}
#endif

#endif /* BMV_PLAN_H */
