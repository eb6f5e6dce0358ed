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
                            const int64_t* slab_ptr, const int64_t* slab_cols,
                            const int64_t* slab_off, int64_t* flat, int64_t* rows,
                            int64_t* cols) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int64_t c = 0; c < n_cols; ++c) {
    if (bad) continue;
    const int64_t* b = col_rows + col_ptr[c];
    const int64_t* e = col_rows + col_ptr[c + 1];
    const int64_t* a = std::lower_bound(b, e, lo);
    const int64_t* z = std::lower_bound(a, e, hi);
    int64_t o = out_start[c];
    int64_t lb = -1, bend = 0, base = 0, bstart = 0, width = 0;
    for (const int64_t* p = a; p < z; ++p, ++o) {
      const int64_t r = *p;
      if (r >= bend) {  // next block row holding r (rows ascend within a column)
        lb = range_of(block_starts, nb_own, r);
        bstart = block_starts[lb];
        bend = block_starts[lb + 1];
        const int64_t* kb = slab_cols + slab_ptr[lb];
        const int64_t* ke = slab_cols + slab_ptr[lb + 1];
        const int64_t* k = std::lower_bound(kb, ke, c);
        if (k == ke || *k != c) { bad = 1; break; }
        width = slab_ptr[lb + 1] - slab_ptr[lb];
        base = slab_off[lb] + (k - kb);
      }
      flat[o] = base + (r - bstart) * width;
      rows[o] = r;
      cols[o] = c;
    }
  }
  return bad ? 3 : 0;
}

int bmvp_support_columns_count(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                               int64_t n_blocks, const int64_t* block_starts,
                               const int64_t* block_sel, int64_t n_sel, int64_t* counts) {
  if (n_cols < 0 || n_blocks < 0 || n_sel < 0) return 1;
  std::memset(counts, 0, sizeof(int64_t) * (size_t)n_sel);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < n_cols; ++c) {
    int64_t bend = -1;
    for (int64_t i = col_ptr[c]; i < col_ptr[c + 1]; ++i) {
      const int64_t r = col_rows[i];
      if (r < bend) continue;
      const int64_t g = range_of(block_starts, n_blocks, r);
      bend = block_starts[g + 1];
      const int64_t s = block_sel[g];
      if (s >= 0) {
#pragma omp atomic
        counts[s] += 1;
      }
    }
  }
  return 0;
}

int bmvp_support_columns_fill(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                              int64_t n_blocks, const int64_t* block_starts,
                              const int64_t* block_sel, int64_t n_sel, const int64_t* ptr,
                              int64_t* cursor, int64_t* cols) {
  if (n_cols < 0 || n_blocks < 0 || n_sel < 0) return 1;
  std::memcpy(cursor, ptr, sizeof(int64_t) * (size_t)n_sel);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < n_cols; ++c) {
    int64_t bend = -1;
    for (int64_t i = col_ptr[c]; i < col_ptr[c + 1]; ++i) {
      const int64_t r = col_rows[i];
      if (r < bend) continue;
      const int64_t g = range_of(block_starts, n_blocks, r);
      bend = block_starts[g + 1];
      const int64_t s = block_sel[g];
      if (s >= 0) {
        int64_t at;
#pragma omp atomic capture
        at = cursor[s]++;
        cols[at] = c;
      }
    }
  }
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t s = 0; s < n_sel; ++s) std::sort(cols + ptr[s], cols + ptr[s + 1]);
  return 0;
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

// ---------------------------------------------------------------------------
// K4 / K5 chunk plans (include/bmv.h bmv_chunk_desc): replaces the block
// loops of reference tmmult / mmult (bcsr.py:587-667) by chunks of
// consecutive owned rows of A, dense over the union of their stored
// columns.  See the header for the meta layout.

namespace {

struct SlabView {
  const int64_t* ptr;    // stored columns per block row (CSR)
  const int64_t* cols;
  const int64_t* off;    // slab offsets
};

inline int64_t width_of(const SlabView& s, int64_t i) { return s.ptr[i + 1] - s.ptr[i]; }

inline int64_t slot_of(const SlabView& s, int64_t i, int64_t col) {
  const int64_t* b = s.cols + s.ptr[i];
  const int64_t* e = s.cols + s.ptr[i + 1];
  const int64_t* k = std::lower_bound(b, e, col);
  return (k != e && *k == col) ? int64_t(k - b) : -1;
}

struct Segment {
  int64_t row;  // block row
  int64_t r0, r1;
};

}  // namespace

struct bmvp_chunks {
  std::vector<int64_t> chunk_meta{0};
  std::vector<int32_t> meta;
  std::vector<int64_t> chunk_a, chunk_b;
  std::vector<int64_t> part_start;
  std::vector<double> cost;
  int64_t n_chunks = 0;
  int64_t dmma = 0;
  int status = 0;
};

extern "C" {

bmvp_chunks* bmvp_chunk_plan(int32_t kind, int64_t n_rows, const int64_t* rows,
                             const int64_t* a_ptr, const int64_t* a_cols, const int64_t* a_off,
                             const int64_t* b_ptr, const int64_t* b_cols, const int64_t* b_off,
                             int64_t n_acb, const int64_t* acb_starts, const int64_t* m_ltab,
                             const int64_t* m_ptr, const int64_t* m_cols, const int64_t* m_off,
                             int32_t max_rows, int32_t max_brows, int32_t data_bytes,
                             int32_t stage_bytes, int32_t n_parts) {
  auto* out = new bmvp_chunks();
  if ((kind != 4 && kind != 5) || n_rows < 0 || max_rows <= 0 || stage_bytes <= 0 ||
      n_parts <= 0 || max_brows <= 0 || max_brows > 255) {
    out->status = 1;
    return out;
  }
  const SlabView A{a_ptr, a_cols, a_off}, B{b_ptr, b_cols, b_off}, M{m_ptr, m_cols, m_off};
  const bool k4 = kind == 4;
  // 1. segments -> chunks (greedy over block rows in order)
  std::vector<std::vector<Segment>> chunks;
  {
    std::vector<Segment> cur;
    int64_t cur_rows = 0, cur_bytes = 0;
    auto flush = [&]() {
      if (!cur.empty()) chunks.push_back(cur);
      cur.clear();
      cur_rows = cur_bytes = 0;
    };
    for (int64_t i = 0; i < n_rows; ++i) {
      const int64_t R = rows[i];
      if (R == 0) continue;
      const int64_t per_row = 8 * (width_of(A, i) + (k4 ? width_of(B, i) : 0));
      const int64_t bytes = R * per_row;
      if (R <= max_rows && bytes <= data_bytes) {
        if (cur_rows + R > max_rows || cur_bytes + bytes > data_bytes ||
            (int64_t)cur.size() >= max_brows)
          flush();
        cur.push_back({i, 0, R});
        cur_rows += R;
        cur_bytes += bytes;
      } else {  // a long block row: balanced row ranges, each its own chunk
        flush();
        int64_t lim = max_rows;
        if (per_row > 0) lim = std::min<int64_t>(lim, std::max<int64_t>(1, data_bytes / per_row));
        const int64_t np = (R + lim - 1) / lim;
        for (int64_t p = 0; p < np; ++p) {
          const int64_t r0 = R * p / np, r1 = R * (p + 1) / np;
          chunks.push_back({{i, r0, r1}});
        }
      }
    }
    flush();
  }
  // 2. per chunk: meta (split chunks whose stage does not fit)
  std::vector<int64_t> ua, ub, ka, kb, mk;
  for (size_t ci = 0; ci < chunks.size(); ++ci) {
    const std::vector<Segment>& seg = chunks[ci];
    const int64_t nbr = (int64_t)seg.size();
    int64_t nrows = 0;
    for (const Segment& s : seg) nrows += s.r1 - s.r0;
    // union columns
    ua.clear();
    ub.clear();
    for (const Segment& s : seg) {
      ua.insert(ua.end(), A.cols + A.ptr[s.row], A.cols + A.ptr[s.row + 1]);
      ub.insert(ub.end(), B.cols + B.ptr[s.row], B.cols + B.ptr[s.row + 1]);
    }
    std::sort(ua.begin(), ua.end());
    ua.erase(std::unique(ua.begin(), ua.end()), ua.end());
    std::sort(ub.begin(), ub.end());
    ub.erase(std::unique(ub.begin(), ub.end()), ub.end());
    const int64_t UA = (int64_t)ua.size(), UB = (int64_t)ub.size();
    // M rows of the union A columns
    ka.assign(UA, 0);
    mk.clear();
    std::vector<int64_t> rb(UA, 0), kk(UA, 0);
    for (int64_t a = 0; a < UA; ++a) {
      const int64_t col = ua[a];
      const int64_t cb = int64_t(std::upper_bound(acb_starts, acb_starts + n_acb + 1, col) -
                                 acb_starts) - 1;
      const int64_t lb = m_ltab[cb];
      if (lb < 0) {
        out->status = 3;  // M holds no (ghost) block row for this column block
        return out;
      }
      const int64_t r = col - acb_starts[cb];
      rb[a] = m_off[lb] + r * width_of(M, lb);
      auto it = std::find(mk.begin(), mk.end(), lb);
      kk[a] = int64_t(it - mk.begin());
      if (it == mk.end()) mk.push_back(lb);
    }
    const int64_t NK = (int64_t)mk.size();
    const int64_t seg_w = 8 * nbr;
    const int64_t cma_w = (nbr * UA + 1) / 2, cmb_w = (nbr * UB + 1) / 2;
    int64_t words = 16 + seg_w + cma_w + cmb_w + 2 * UA + NK * UB;
    words = (words + 3) / 4 * 4;
    // staged ranges (doubles, even bounds)
    const Segment& s0 = seg.front();
    const Segment& s1 = seg.back();
    const int64_t a0 = (a_off[s0.row] + s0.r0 * width_of(A, s0.row)) & ~int64_t(1);
    int64_t a1 = a_off[s1.row] + s1.r1 * width_of(A, s1.row);
    a1 = (a1 + 1) & ~int64_t(1);
    int64_t b0 = 0, b1 = 0;
    if (k4) {
      b0 = (b_off[s0.row] + s0.r0 * width_of(B, s0.row)) & ~int64_t(1);
      b1 = b_off[s1.row] + s1.r1 * width_of(B, s1.row);
      b1 = (b1 + 1) & ~int64_t(1);
    }
    const int64_t total = 4 * words + 8 * (a1 - a0) + 8 * (b1 - b0);
    if (total > stage_bytes || UA > 32767 || UB > 32767 || nrows > 4096) {
      // split and retry (rows or block rows)
      if (nbr > 1) {
        std::vector<Segment> h1(seg.begin(), seg.begin() + nbr / 2), h2(seg.begin() + nbr / 2, seg.end());
        chunks[ci] = h1;
        chunks.insert(chunks.begin() + ci + 1, h2);
        --ci;
        continue;
      }
      if (s0.r1 - s0.r0 > 1) {
        const Segment whole = s0;  // s0 refers into chunks[ci], reassigned below
        const int64_t mid = (whole.r0 + whole.r1) / 2;
        chunks[ci] = {{whole.row, whole.r0, mid}};
        chunks.insert(chunks.begin() + ci + 1, std::vector<Segment>{{whole.row, mid, whole.r1}});
        --ci;
        continue;
      }
      out->status = 4;  // one row does not fit a stage
      return out;
    }
    const int64_t base = (int64_t)out->meta.size();
    out->meta.resize(base + words, 0);
    int32_t* m = out->meta.data() + base;
    const int64_t aoff = 4 * words, boff = aoff + 8 * (a1 - a0);
    int64_t w = 16;
    m[0] = (int32_t)nbr;
    m[1] = (int32_t)nrows;
    m[2] = (int32_t)UA;
    m[3] = (int32_t)UB;
    m[4] = (int32_t)NK;
    m[5] = (int32_t)aoff;
    m[6] = (int32_t)boff;
    m[7] = (int32_t)w;  // segment records: {rows, A offset, K_A, B / Y offset, K_B, 0, 0, 0}
    for (int64_t bi = 0; bi < nbr; ++bi) {
      const Segment& s = seg[bi];
      const int64_t ar = a_off[s.row] + s.r0 * width_of(A, s.row) - a0;
      // K4: B offset in the stage; K5: element offset of the segment's first row in Y
      const int64_t br = b_off[s.row] + s.r0 * width_of(B, s.row) - (k4 ? b0 : 0);
      if (br > INT32_MAX) {
        out->status = 5;
        return out;
      }
      int32_t* r = m + w + 8 * bi;
      r[0] = (int32_t)(s.r1 - s.r0);
      r[1] = (int32_t)ar;
      r[2] = (int32_t)width_of(A, s.row);
      r[3] = (int32_t)br;
      r[4] = (int32_t)width_of(B, s.row);
    }
    w += seg_w;
    m[8] = (int32_t)w;  // A colmap
    int16_t* cma = reinterpret_cast<int16_t*>(m + w);
    for (int64_t bi = 0; bi < nbr; ++bi)
      for (int64_t a = 0; a < UA; ++a) cma[bi * UA + a] = (int16_t)slot_of(A, seg[bi].row, ua[a]);
    w += cma_w;
    m[9] = (int32_t)w;  // B / Y colmap
    int16_t* cmb = reinterpret_cast<int16_t*>(m + w);
    for (int64_t bi = 0; bi < nbr; ++bi)
      for (int64_t b = 0; b < UB; ++b) cmb[bi * UB + b] = (int16_t)slot_of(B, seg[bi].row, ub[b]);
    w += cmb_w;
    m[10] = (int32_t)w;
    for (int64_t a = 0; a < UA; ++a) {
      if (rb[a] > INT32_MAX) {
        out->status = 5;
        return out;
      }
      m[w + a] = (int32_t)rb[a];
    }
    w += UA;
    m[11] = (int32_t)w;
    for (int64_t a = 0; a < UA; ++a) m[w + a] = (int32_t)kk[a];
    w += UA;
    m[12] = (int32_t)w;
    for (int64_t k = 0; k < NK; ++k)
      for (int64_t b = 0; b < UB; ++b) m[w + k * UB + b] = (int32_t)slot_of(M, mk[k], ub[b]);
    out->chunk_meta.push_back(base + words);
    out->chunk_a.push_back(a0);
    out->chunk_a.push_back(a1);
    if (k4) {
      out->chunk_b.push_back(b0);
      out->chunk_b.push_back(b1);
    }
    const int64_t ta = (UA + 7) / 8, tb = (UB + 7) / 8;
    int64_t steps = 0;  // DMMA k-steps (K4, 4 rows) / row tiles (K5, 8 rows), segments padded
    for (const Segment& s : seg) steps += k4 ? (s.r1 - s.r0 + 3) / 4 : (s.r1 - s.r0 + 7) / 8;
    const int64_t dm = k4 ? ta * tb * steps : ((UA + 3) / 4) * tb * steps;
    out->dmma += dm;
    out->cost.push_back((double)(8 * (a1 - a0) + 8 * (b1 - b0) + 4 * words) + 32.0 * (double)dm);
  }
  out->n_chunks = (int64_t)out->chunk_a.size() / 2;
  // 3. parts: contiguous chunk ranges of equal estimated cost
  double tot = 0;
  for (double c : out->cost) tot += c;
  out->part_start.assign(n_parts + 1, out->n_chunks);
  out->part_start[0] = 0;
  double acc = 0;
  int p = 1;
  for (int64_t j = 0; j < out->n_chunks && p < n_parts; ++j) {
    acc += out->cost[j];
    while (p < n_parts && acc >= tot * p / n_parts) out->part_start[p++] = j + 1;
  }
  return out;
}

int bmvp_chunk_status(const bmvp_chunks* c) { return c ? c->status : 1; }

void bmvp_chunk_sizes(const bmvp_chunks* c, int64_t* n_chunks, int64_t* meta_len, int64_t* dmma) {
  *n_chunks = c->n_chunks;
  *meta_len = (int64_t)c->meta.size();
  *dmma = c->dmma;
}

void bmvp_chunk_copy(const bmvp_chunks* c, int64_t* part_start, int64_t* chunk_meta, int32_t* meta,
                     int64_t* chunk_a, int64_t* chunk_b) {
  std::copy(c->part_start.begin(), c->part_start.end(), part_start);
  std::copy(c->chunk_meta.begin(), c->chunk_meta.end(), chunk_meta);
  std::copy(c->meta.begin(), c->meta.end(), meta);
  std::copy(c->chunk_a.begin(), c->chunk_a.end(), chunk_a);
  if (chunk_b) std::copy(c->chunk_b.begin(), c->chunk_b.end(), chunk_b);
}

void bmvp_chunk_free(bmvp_chunks* c) { delete c; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Active pairs, operator images and the K1 plan (matfree.py: ImageColumns,
// CellOperator.active_pairs, _CellPlan), replacing sparse products over the
// whole mesh.  Reference: the cell loop's column emission
// (RowsBlockAccessor, matfree.py:159-237) restricted to the columns whose
// support reaches the cell, and the grown pattern (localization.py:251-267)
// at entry level.

namespace {

// columns of a sorted small list, deduplicated
inline void sort_unique(std::vector<int32_t>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

}  // namespace

extern "C" {

int bmvp_support_transpose(int64_t n_cols, const int64_t* col_ptr, const int64_t* col_rows,
                           const int64_t* row_sel, int64_t n_sel, int64_t* ptr, int32_t* cols) {
  // pass 1 (cols == NULL): ptr[s + 1] = columns of selected row s; pass 2: fill
  if (n_cols < 0 || n_sel < 0) return 1;
  if (!cols) {
    std::memset(ptr, 0, sizeof(int64_t) * (size_t)(n_sel + 1));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < n_cols; ++c)
      for (int64_t i = col_ptr[c]; i < col_ptr[c + 1]; ++i) {
        const int64_t s = row_sel[col_rows[i]];
        if (s >= 0) {
#pragma omp atomic
          ptr[s + 1] += 1;
        }
      }
    for (int64_t s = 0; s < n_sel; ++s) ptr[s + 1] += ptr[s];
    return 0;
  }
  std::vector<int64_t> cur(ptr, ptr + n_sel);
  // columns ascending per row: fill column by column in order (serial over
  // columns keeps the order; rows in parallel would not)
  for (int64_t c = 0; c < n_cols; ++c)
    for (int64_t i = col_ptr[c]; i < col_ptr[c + 1]; ++i) {
      const int64_t s = row_sel[col_rows[i]];
      if (s >= 0) cols[cur[s]++] = (int32_t)c;
    }
  return 0;
}

int bmvp_cell_pairs(int64_t n_cells, int32_t n3, const int64_t* cell_rows, const int64_t* row_ptr,
                    const int32_t* row_cols, int64_t* ptr, int32_t* cols) {
  // cell_rows: (n_cells, n3) indices into the row CSR (-1: no row);
  // pass 1 (cols == NULL) counts, pass 2 fills sorted unique columns per cell
  if (n_cells < 0 || n3 <= 0) return 1;
  if (!cols) {
    ptr[0] = 0;
#pragma omp parallel
    {
      std::vector<int32_t> v;
#pragma omp for schedule(dynamic, 256)
      for (int64_t c = 0; c < n_cells; ++c) {
        v.clear();
        for (int d = 0; d < n3; ++d) {
          const int64_t r = cell_rows[c * n3 + d];
          if (r >= 0) v.insert(v.end(), row_cols + row_ptr[r], row_cols + row_ptr[r + 1]);
        }
        sort_unique(v);
        ptr[c + 1] = (int64_t)v.size();
      }
    }
    for (int64_t c = 0; c < n_cells; ++c) ptr[c + 1] += ptr[c];
    return 0;
  }
#pragma omp parallel
  {
    std::vector<int32_t> v;
#pragma omp for schedule(dynamic, 256)
    for (int64_t c = 0; c < n_cells; ++c) {
      v.clear();
      for (int d = 0; d < n3; ++d) {
        const int64_t r = cell_rows[c * n3 + d];
        if (r >= 0) v.insert(v.end(), row_cols + row_ptr[r], row_cols + row_ptr[r + 1]);
      }
      sort_unique(v);
      std::copy(v.begin(), v.end(), cols + ptr[c]);
    }
  }
  return 0;
}

int bmvp_block_image(int64_t n_cells, int32_t n3, const int64_t* cell_blocks,
                     const int64_t* pair_ptr, const int32_t* pair_cols, int64_t n_blocks,
                     int64_t n_cols, int64_t* ptr, int64_t* cols) {
  // image(b) = union of pair_cols(c) over the cells c with cell_blocks[c][d] == b
  // (cell_blocks: selected block index or -1).  pass 1 (cols == NULL) counts.
  if (n_cells < 0 || n3 <= 0 || n_blocks < 0 || n_cols < 0) return 1;
  const int64_t words = (n_cols + 63) / 64;
  std::vector<uint64_t> bits((size_t)(n_blocks * words), 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t c = 0; c < n_cells; ++c) {
    int64_t seen[64];
    int ns = 0;
    for (int d = 0; d < n3; ++d) {
      const int64_t b = cell_blocks[c * n3 + d];
      if (b < 0) continue;
      bool dup = false;
      for (int k = 0; k < ns; ++k) dup |= seen[k] == b;
      if (dup) continue;
      if (ns < 64) seen[ns++] = b;
      uint64_t* w = bits.data() + b * words;
      for (int64_t i = pair_ptr[c]; i < pair_ptr[c + 1]; ++i) {
        const int64_t col = pair_cols[i];
#pragma omp atomic
        w[col >> 6] |= (uint64_t)1 << (col & 63);
      }
    }
  }
  if (!cols) {
    ptr[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < n_blocks; ++b) {
      int64_t n = 0;
      for (int64_t k = 0; k < words; ++k) n += __builtin_popcountll(bits[b * words + k]);
      ptr[b + 1] = n;
    }
    for (int64_t b = 0; b < n_blocks; ++b) ptr[b + 1] += ptr[b];
    return 0;
  }
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < n_blocks; ++b) {
    int64_t o = ptr[b];
    for (int64_t k = 0; k < words; ++k) {
      uint64_t w = bits[b * words + k];
      while (w) {
        const int t = __builtin_ctzll(w);
        cols[o++] = k * 64 + t;
        w &= w - 1;
      }
    }
  }
  return 0;
}

int bmvp_k1_plan(int64_t n_pairs, const int64_t* pair_cell, const int64_t* pair_col,
                 const int64_t* cell_gstart, const int64_t* grp_block, const int64_t* src_ptr,
                 const int64_t* src_cols, const int64_t* src_off, const int64_t* dst_ptr,
                 const int64_t* dst_cols, const int64_t* dst_off, const int64_t* pair_gtab,
                 int32_t* gtab, int64_t* bad_pair) {
  // gtab[pair_gtab[p] + 2 g] = src slab offset + slot of the pair's column in
  // group g's block row (-1 absent), [+1] = dst slab offset + slot (-1 -> error)
  *bad_pair = -1;
  int64_t bad = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : bad)
  for (int64_t p = 0; p < n_pairs; ++p) {
    const int64_t c = pair_cell[p], col = pair_col[p];
    const int64_t g0 = cell_gstart[c], ng = cell_gstart[c + 1] - g0;
    int32_t* t = gtab + pair_gtab[p];
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t lb = grp_block[g0 + g];
      const int64_t* sb = src_cols + src_ptr[lb];
      const int64_t* se = src_cols + src_ptr[lb + 1];
      const int64_t* s = std::lower_bound(sb, se, col);
      t[2 * g] = (s != se && *s == col) ? (int32_t)(src_off[lb] + (s - sb)) : -1;
      const int64_t* db = dst_cols + dst_ptr[lb];
      const int64_t* de = dst_cols + dst_ptr[lb + 1];
      const int64_t* q = std::lower_bound(db, de, col);
      if (q == de || *q != col) {
        bad = std::min(bad, p);
        t[2 * g + 1] = 0;
      } else {
        t[2 * g + 1] = (int32_t)(dst_off[lb] + (q - db));
      }
    }
    if (ng & 1) {
      t[2 * ng] = -1;
      t[2 * ng + 1] = 0;
    }
  }
  if (bad != INT64_MAX) {
    *bad_pair = bad;
    return 3;
  }
  return 0;
}

}  // extern "C"
