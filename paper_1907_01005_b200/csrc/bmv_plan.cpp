// Native plan builder (host C++, OpenMP): the setup steps of the hot path that
// dominate the Python/numpy setup at the weak-scaling size.
//
// Every function reproduces its numpy restatement in this package bit for bit
// (tests/test_plan_native.py compares them at small and full sizes):
//   bmvp_hash_fill         problem.hashed_entries / fill_multivector
//                          (reference bench/problem.py:113-131, splitmix64 `_mix64`)
//   bmvp_owned_entries_*   support.ColumnSupport.owned_entries (storage offsets of the
//                          support entries, reference bcsr.py:233-318 layout)
//   bmvp_blocks_of         RankLayout.map_rows, owned rows (reference bcsr.py:126-152)
//   bmvp_first_touch       mesh.enumerate_dofs first-touch positions (reference
//                          mesh.py:263-322 numbering along the ordered cells)
//   bmvp_grow_*            localization.grow_sparsity_for_operator (inc^T (inc S) + S,
//                          reference localization.py:251-267) as per-cell bitset unions
//   bmvp_first_groups_*    matfree._first_occurrence_groups (reference CellDoFMap
//                          grouping, matfree.py:58-130)
// Declared in include/bmv_plan.h.  No CUDA: these build index maps on the host
// once per (pattern, layout) and are then uploaded with the kernel plans.

#include <cstdint>
#include <cstring>
#include <algorithm>
#include <vector>

#include "bmv_plan.h"

namespace {

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// index of the range [starts[i], starts[i+1]) holding v (starts ascending, n ranges)
inline int64_t range_of(const int64_t* starts, int64_t n, int64_t v) {
  return int64_t(std::upper_bound(starts, starts + n + 1, v) - starts) - 1;
}

}  // namespace

extern "C" {

int bmvp_version(void) { return 1; }

int bmvp_hash_fill(uint64_t seed, int64_t n, const int64_t* rows, const int64_t* cols,
                   const int64_t* col_map, const int64_t* flat, double scale, double* out) {
  if (n < 0 || (n > 0 && (!rows || !cols || !out))) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t r = uint64_t(rows[i]);
    const uint64_t c = uint64_t(col_map ? col_map[cols[i]] : cols[i]);
    const uint64_t h = mix64(r * 0x9E3779B97F4A7C15ull + c * 0xD1B54A32D192ED03ull + seed);
    const double v = scale * (double(h) / 18446744073709551616.0 - 0.5);
    out[flat ? flat[i] : i] = v;
  }
  return 0;
}

int bmvp_blocks_of(int64_t n_blocks, const int64_t* starts, int64_t n, const int64_t* idx,
                   int64_t* block, int64_t* offset) {
  if (n_blocks < 0 || n < 0) return 1;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t v = idx[i];
    if (v < starts[0] || v >= starts[n_blocks]) { bad = 1; continue; }
    const int64_t b = range_of(starts, n_blocks, v);
    block[i] = b;
    if (offset) offset[i] = v - starts[b];
  }
  return bad ? 1 : 0;
}

int bmvp_owned_entries_count(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                             int64_t lo, int64_t hi, int64_t* col_count) {
  if (n_cols < 0) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n_cols; ++c) {
    const int64_t* b = col_rows + col_ptr[c];
    const int64_t* e = col_rows + col_ptr[c + 1];
    col_count[c] = int64_t(std::lower_bound(b, e, hi) - std::lower_bound(b, e, lo));
  }
  return 0;
}

int bmvp_owned_entries_fill(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                            int64_t lo, int64_t hi, const int64_t* out_start,
                            int64_t nb_own, const int64_t* block_starts,
                            int64_t n_cb, const int64_t* cb_starts,
                            const int64_t* row_start, const int64_t* col_index,
                            const int64_t* block_offsets, const int64_t* col_strides,
                            int64_t* flat, int64_t* rows, int64_t* cols) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int64_t c = 0; c < n_cols; ++c) {
    if (bad) continue;
    const int64_t* b = col_rows + col_ptr[c];
    const int64_t* e = col_rows + col_ptr[c + 1];
    const int64_t* a = std::lower_bound(b, e, lo);
    const int64_t* z = std::lower_bound(a, e, hi);
    const int64_t cbk = range_of(cb_starts, n_cb, c);
    const int64_t cin = c - cb_starts[cbk];
    const int64_t stride = col_strides[cbk];
    int64_t o = out_start[c];
    int64_t lb = -1, bend = 0, base = 0, bstart = 0;
    for (const int64_t* p = a; p < z; ++p, ++o) {
      const int64_t r = *p;
      if (r >= bend) {  // next block row holding r (rows ascend within a column)
        lb = range_of(block_starts, nb_own, r);
        bstart = block_starts[lb];
        bend = block_starts[lb + 1];
        const int64_t* kb = col_index + row_start[lb];
        const int64_t* ke = col_index + row_start[lb + 1];
        const int64_t* k = std::lower_bound(kb, ke, cbk);
        if (k == ke || *k != cbk) { bad = 1; break; }
        base = block_offsets[row_start[lb] + (k - kb)];
      }
      flat[o] = base + (r - bstart) * stride + cin;
      rows[o] = r;
      cols[o] = c;
    }
  }
  return bad ? 3 : 0;
}

int bmvp_first_groups_count(int64_t n_cells, int32_t n3, const int64_t* lb,
                            int64_t* slot_group, int64_t* cell_count) {
  if (n_cells < 0 || n3 <= 0 || n3 > 4096) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n_cells; ++c) {
    int64_t seen[4096];
    int64_t ng = 0;
    const int64_t* l = lb + c * n3;
    int64_t* s = slot_group + c * n3;
    for (int32_t d = 0; d < n3; ++d) {
      int64_t g = 0;
      while (g < ng && seen[g] != l[d]) ++g;
      if (g == ng) seen[ng++] = l[d];
      s[d] = g;
    }
    cell_count[c] = ng;
  }
  return 0;
}

int bmvp_first_groups_fill(int64_t n_cells, int32_t n3, const int64_t* lb,
                           const int64_t* slot_group, const int64_t* cell_gstart,
                           int64_t* grp_cell, int64_t* grp_block) {
  if (n_cells < 0 || n3 <= 0) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n_cells; ++c) {
    const int64_t* l = lb + c * n3;
    const int64_t* s = slot_group + c * n3;
    const int64_t g0 = cell_gstart[c];
    int64_t next = 0;
    for (int32_t d = 0; d < n3; ++d) {
      if (s[d] == next) {  // first occurrence of group `next`
        grp_cell[g0 + next] = c;
        grp_block[g0 + next] = l[d];
        ++next;
      }
    }
  }
  return 0;
}

int bmvp_first_touch(int64_t n_nodes, int64_t n, const int64_t* touches, int64_t* first) {
  if (n_nodes < 0 || n < 0) return 1;
  for (int64_t i = 0; i < n_nodes; ++i) first[i] = n;
  for (int64_t pos = 0; pos < n; ++pos) {
    const int64_t t = touches[pos];
    if (t < 0 || t >= n_nodes) return 1;
    if (first[t] == n) first[t] = pos;
  }
  return 0;
}

int bmvp_grow_count(int64_t n_cells, int32_t n3, const int64_t* cell_rb, int64_t n_rb,
                    int64_t n_cb, const int64_t* s_row_start, const int64_t* s_col_index,
                    uint64_t* bits, int64_t* row_count) {
  if (n_cells < 0 || n3 <= 0 || n3 > 4096 || n_rb < 0 || n_cb < 0) return 1;
  const int64_t W = (n_cb + 63) / 64;
  // the pattern itself (the "+ S" term)
#pragma omp parallel for schedule(static)
  for (int64_t rb = 0; rb < n_rb; ++rb)
    for (int64_t k = s_row_start[rb]; k < s_row_start[rb + 1]; ++k)
      bits[rb * W + s_col_index[k] / 64] |= uint64_t(1) << (s_col_index[k] % 64);
  int bad = 0;
#pragma omp parallel reduction(| : bad)
  {
    std::vector<uint64_t> cset(W);
    std::vector<int64_t> rbs;
    rbs.reserve(64);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
      rbs.clear();
      const int64_t* l = cell_rb + c * n3;
      for (int32_t d = 0; d < n3; ++d) {
        if (l[d] < 0 || l[d] >= n_rb) { bad = 1; break; }
        if (std::find(rbs.begin(), rbs.end(), l[d]) == rbs.end()) rbs.push_back(l[d]);
      }
      std::fill(cset.begin(), cset.end(), 0);
      for (int64_t rb : rbs)  // inc S: the column blocks any row block of the cell holds
        for (int64_t k = s_row_start[rb]; k < s_row_start[rb + 1]; ++k)
          cset[s_col_index[k] / 64] |= uint64_t(1) << (s_col_index[k] % 64);
      for (int64_t rb : rbs)  // inc^T (inc S)
        for (int64_t w = 0; w < W; ++w)
          if (cset[w]) __atomic_fetch_or(&bits[rb * W + w], cset[w], __ATOMIC_RELAXED);
    }
  }
  if (bad) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t rb = 0; rb < n_rb; ++rb) {
    int64_t n = 0;
    for (int64_t w = 0; w < W; ++w) n += __builtin_popcountll(bits[rb * W + w]);
    row_count[rb] = n;
  }
  return 0;
}

int bmvp_grow_fill(int64_t n_rb, int64_t n_cb, const uint64_t* bits, const int64_t* row_start,
                   int64_t* col_index) {
  if (n_rb < 0 || n_cb < 0) return 1;
  const int64_t W = (n_cb + 63) / 64;
#pragma omp parallel for schedule(static)
  for (int64_t rb = 0; rb < n_rb; ++rb) {
    int64_t o = row_start[rb];
    for (int64_t w = 0; w < W; ++w) {
      uint64_t m = bits[rb * W + w];
      while (m) {
        col_index[o++] = w * 64 + __builtin_ctzll(m);
        m &= m - 1;
      }
    }
  }
  return 0;
}

}  // extern "C"
