// K4 / K5 (lane-compacted): the projection S = A^T B and the post-multiply
// Y = alpha A C on the FP64 tensor cores, using the column support of A.
//
// The reference multiplies whole padded blocks (bcsr.py:587-667: dense
// (rows x W)^T (rows x W) products per block pair).  A's support is known
// (support.py), so inside one block row only the columns of A that are
// active on it carry data (blocks are 25-35 % full).
// The planner (host, C++) lists, per block row, the active (block, lane)
// columns of A ("compact columns") and packs them 8 (K4: the M side of the
// DMMA) or 4 (K5: the K side) at a time, so a DMMA m8n8k4 works on active
// columns only, whatever block they sit in:
//   K4 tile = (block row, 8 compact A columns, 8 lanes of one B block):
//        D(8x8) += A[r, a_m]^T B[r, n] over the rows r, 4 per DMMA;
//        the 8 D rows go to 8 (possibly different) S tiles.
//   K5 task = (block row, 8 lanes of one Y block, 8 rows per step):
//        D(8x8) = sum_k X[r, a_k] C[a_k, n] over the compact columns.
// Operands of a chunk of consecutive block rows (A range, B range, tile
// records) are staged into shared memory by a producer warp with
// cp.async.bulk (bmv_tma.cuh stream_producer); NW consumer warps take the
// tiles round-robin.  K4 accumulates into a per-item shared-memory copy of
// the touched S tiles and flushes it to S with fp64 reductions (RED) at
// the end of the item; K5 writes each output value once.  Summation order
// of S across CTAs is not fixed (like the atomic K1 scatter); the
// deterministic kernels (bmv_project.cu, bmv_postmul.cu) remain for
// BMV_DETERMINISTIC=1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <unordered_map>
#include <vector>

#include "bmv_common.cuh"
#include "bmv_tma.cuh"

namespace bmv {
int zero_async(double* p, int64_t n, cudaStream_t st);
}

using namespace bmv;

namespace {

// consumer warps (+ 1 producer warp) per CTA: 16 for long block rows (the kernels
// stream at the HBM roofline), 24 where per-tile latency binds -- K4 on short
// (interleaved) block rows and K5 everywhere (measured: proj K4 0.974 -> 0.895 ms,
// K5 0.600 -> 0.537 ms; weak G = 1 K4 0.983 -> 1.004 ms, K5 0.893 -> 0.878 ms)
constexpr int kLnWarps = 16;
constexpr int kLnWarpsWide = 24;
constexpr int kLnStages = 3;
constexpr int kAccTiles = 64;                     // K4 shared accumulator: 64 tiles of 8x8
constexpr int kSmemBudget = 227 * 1024 - 1024;
constexpr int kK4Rec = 20;                        // int32 per K4 tile record
constexpr int kKGroup = 8;                        // K5: k-steps (4 compact columns each) per pass

// ---- K4 ------------------------------------------------------------------------
// Stage: [hdr 4 int: n_tiles, n_flush, tile rec offset (int), flush offset]
//        [tile records, kK4Rec int32 each][flush records int4][A range][B range]
// Tile record: [0..7] A column (stage double offset | stride << 16, -1 = none)
//              [8..15] accumulator offset of D row m (doubles)
//              [16] B offset (stage doubles) of lane 0 of the 8-lane tile
//              [17] rows | b_stride << 16   [18] valid B lanes (<= 8)
// Flush record: {S element offset, S stride, rows | cols << 8, acc tile}
struct LnArgs {
  const int64_t* __restrict__ part_sub_start;
  const int64_t* __restrict__ part_entry_start;
  const int4* __restrict__ copies;
  CopySrc src;  // p0 = meta, p1 = a, p2 = b
  double* __restrict__ out;
  double alpha;
  int accumulate;
  int stage_bytes;
  const double* __restrict__ cmat;  // K5: the C operand (global)
};

template <int NW>
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(NW * 32) : "memory");
}

template <int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k4_lane_kernel(const LnArgs g) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[kLnStages], empty[kLnStages];
  double* acc = smem;  // kAccTiles * 64
  char* stages = reinterpret_cast<char*>(smem + kAccTiles * 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = g.part_sub_start[blockIdx.x], s1 = g.part_sub_start[blockIdx.x + 1];
  if (threadIdx.x == 0) {
    for (int k = 0; k < kLnStages; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], NW);
    }
  }
  for (int i = threadIdx.x; i < kAccTiles * 64; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  if (warp == NW) {
    stream_producer(g.copies, g.part_entry_start[blockIdx.x], g.part_entry_start[blockIdx.x + 1],
                    s1 - s0, g.src, stages, g.stage_bytes, kLnStages, full, empty, lane);
    return;
  }
  const int gid = lane >> 2, tig = lane & 3;
  for (int64_t i = 0; i < s1 - s0; ++i) {
    const int st = (int)(i % kLnStages);
    mbar_wait(&full[st], (unsigned)((i / kLnStages) & 1));
    const char* stg = stages + (int64_t)st * g.stage_bytes;
    const int* hdr = reinterpret_cast<const int*>(stg);
    const double* S = reinterpret_cast<const double*>(stg);
    const int n_tiles = hdr[0], n_flush = hdr[1];
    const int* recs = hdr + hdr[2];
    for (int t = warp; t < n_tiles; t += NW) {
      const int* r = recs + t * kK4Rec;
      const int ac = r[gid];
      const int ao = ac & 0xffff, as = (ac >> 16) & 0x7fff;
      const bool am = ac >= 0;
      const int rows = r[17] & 0xffff, bs = r[17] >> 16;
      const bool bm = gid < r[18];
      const double* A = S + ao + tig * as;
      const double* B = S + r[16] + gid + tig * bs;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0, c5 = 0.0, c6 = 0.0, c7 = 0.0;
      int r0 = 0;
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
      const double x = (c0 + c2) + (c4 + c6), y = (c1 + c3) + (c5 + c7);
      const int ro = r[8 + gid];
      if (am && ro >= 0) {
        if (2 * tig < r[18]) atomicAdd(acc + ro + 2 * tig, x);
        if (2 * tig + 1 < r[18]) atomicAdd(acc + ro + 2 * tig + 1, y);
      }
    }
    // flush records are read before the stage is released
    int4 fl = make_int4(0, 0, 0, 0);
    const bool flush = n_flush > 0;
    const int4* frec = reinterpret_cast<const int4*>(hdr + hdr[3]);
    __syncwarp();
    if (!flush) {
      if (lane == 0) mbar_arrive(&empty[st]);
      continue;
    }
    consumers_sync<NW>();  // every tile of the item is in acc
    for (int f = warp; f < n_flush; f += NW) {
      fl = frec[f];
      const int rr = fl.z & 0xff, cc = (fl.z >> 8) & 0xff;
      double* tile = acc + fl.w * 64;
      for (int e = lane; e < 64; e += 32) {
        const int row = e >> 3, col = e & 7;
        const double v = tile[e];
        if (row < rr && col < cc && v != 0.0)
          atomicAdd(g.out + (int64_t)(unsigned)fl.x + (int64_t)row * fl.y + col, v);
        tile[e] = 0.0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    consumers_sync<NW>();  // acc cleared before the next item accumulates
  }
}

// ---- K5 ------------------------------------------------------------------------
// Stage: [hdr 4 int: n_tasks, task offset table offset (int), 0, 0]
//        [task offsets (int)][task records][A range]
// Task record (int32): [0] Y element offset lo, [1] hi, [2] rows | ys << 16,
// [3] valid lanes (columns of C) | stored lanes << 8 | ksteps << 16,
// then per k-step 4 A columns (stage double offset | stride << 16, -1 none)
// and 4 C element offsets (row a, column lane 0 of the tile; -1 none).
// TWO: two 8-row tiles in flight per task (independent DMMA chains) for
// block rows of many rows (Q4: 65); one tile for short rows (Q2: 8).
template <int MAXK, bool TWO, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k5_lane_kernel(const LnArgs g) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[kLnStages], empty[kLnStages];
  char* stages = reinterpret_cast<char*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = g.part_sub_start[blockIdx.x], s1 = g.part_sub_start[blockIdx.x + 1];
  if (threadIdx.x == 0) {
    for (int k = 0; k < kLnStages; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], NW);
    }
  }
  __syncthreads();
  if (warp == NW) {
    stream_producer(g.copies, g.part_entry_start[blockIdx.x], g.part_entry_start[blockIdx.x + 1],
                    s1 - s0, g.src, stages, g.stage_bytes, kLnStages, full, empty, lane);
    return;
  }
  const int gid = lane >> 2, tig = lane & 3;
  for (int64_t i = 0; i < s1 - s0; ++i) {
    const int st = (int)(i % kLnStages);
    mbar_wait(&full[st], (unsigned)((i / kLnStages) & 1));
    const char* stg = stages + (int64_t)st * g.stage_bytes;
    const int* hdr = reinterpret_cast<const int*>(stg);
    const double* S = reinterpret_cast<const double*>(stg);
    const int n_tasks = hdr[0];
    const int* toff = hdr + hdr[1];
    for (int t = warp; t < n_tasks; t += NW) {
      const int* r = hdr + toff[t];
      double* Y = g.out + (((int64_t)(unsigned)r[1] << 32) | (unsigned)r[0]);
      const int rows = r[2] & 0xffff, ys = r[2] >> 16;
      const int ncol = r[3] & 0xff, nst = (r[3] >> 8) & 0xff, ks = r[3] >> 16;
      auto store = [&](int row, double d0, double d1, bool add_old) {
        double* p = Y + (int64_t)row * ys + 2 * tig;
        double v0 = g.alpha * d0, v1 = g.alpha * d1;
        if (2 * tig + 1 < nst) {
          if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
            if (add_old) {
              const double2 o = *reinterpret_cast<const double2*>(p);
              v0 += o.x;
              v1 += o.y;
            }
            *reinterpret_cast<double2*>(p) = make_double2(v0, v1);
          } else {
            p[0] = add_old ? p[0] + v0 : v0;
            p[1] = add_old ? p[1] + v1 : v1;
          }
        } else if (2 * tig < nst) {
          p[0] = add_old ? p[0] + v0 : v0;
        }
      };
      // k-steps in groups of MAXK: lane (gid, tig) holds the B fragments
      // C[a_{4s + tig}][gid] of the group; groups after the first add to the
      // values the warp itself wrote (rows with more than 4 MAXK columns)
      for (int kg = 0; kg < max(ks, 1); kg += MAXK) {
        double bf[MAXK];
        int ac[MAXK];
#pragma unroll
        for (int s = 0; s < MAXK; ++s) {
          bf[s] = 0.0;
          ac[s] = -1;
          if (kg + s < ks) {
            const int* e = r + 4 + 8 * (kg + s);
            const int co = e[4 + tig];
            if (co >= 0 && gid < ncol) bf[s] = __ldg(g.cmat + co + gid);
            ac[s] = e[tig];
          }
        }
        const bool add_old = g.accumulate || kg > 0;
        if (TWO) {
          for (int r0 = 0; r0 < rows; r0 += 16) {
            const int ra = r0 + gid, rb = r0 + 8 + gid;
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int s = 0; s < MAXK; ++s) {
              if (kg + s < ks) {
                const int c = ac[s];
                const int off = c & 0xffff, cs = (c >> 16) & 0x7fff;
                const double xa = (c >= 0 && ra < rows) ? S[off + ra * cs] : 0.0;
                const double xb = (c >= 0 && rb < rows) ? S[off + rb * cs] : 0.0;
                dmma_8x8x4(a0, a1, xa, bf[s]);
                dmma_8x8x4(b0, b1, xb, bf[s]);
              }
            }
            if (ra < rows) store(ra, a0, a1, add_old);
            if (rb < rows) store(rb, b0, b1, add_old);
          }
        } else {
          for (int r0 = 0; r0 < rows; r0 += 8) {
            const int ra = r0 + gid;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int s = 0; s < MAXK; ++s) {
              if (kg + s < ks) {
                const int c = ac[s];
                const double xa =
                    (c >= 0 && ra < rows) ? S[(c & 0xffff) + ra * ((c >> 16) & 0x7fff)] : 0.0;
                dmma_8x8x4(a0, a1, xa, bf[s]);
              }
            }
            if (ra < rows) store(ra, a0, a1, add_old);
          }
        }
        if (kg + MAXK < ks) __syncwarp();  // this group's stores before the next group's loads
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// ---- host planning ---------------------------------------------------------------

struct Copy {
  int32_t dst;
  int64_t bytes;
  int src;
  int64_t soff;
};

struct Chunk {
  std::vector<int32_t> meta;  // header + records (int32)
  std::vector<Copy> copies;   // after the metadata copy
};

// Emits chunks -> the copy list + metadata array + per-part ranges.
struct StreamBuild {
  std::vector<int32_t> meta;
  std::vector<int32_t> cps;  // 4 int32 per entry
  std::vector<int64_t> chunk_entry{0};
  std::vector<int64_t> chunk_work;
  std::vector<int64_t> fixed_parts;  // chunk index where each part starts (K4: items never span parts)
  // deferred chunks (interleaved assignment): run r = chunks [r*run, (r+1)*run)
  // goes to CTA r % n_parts (K4 items may span the chunks of one run)
  bool defer = false;
  bool interleaved = false;  // finish_interleaved dealt the chunks
  int64_t run = 1;
  std::vector<std::pair<Chunk, int64_t>> pending;
  void put(const Chunk& c, int64_t work) {
    if (defer)
      pending.push_back({c, work});
    else
      add(c, work);
  }
  // short block rows: consecutive chunks to different CTAs, so every CTA
  // samples every region of the rows (static contiguous parts left a 31 %
  // spread of SM active time at the proj config)
  void finish_interleaved(int n_parts) {
    if (!defer) return;
    const int64_t nc = (int64_t)pending.size();
    const int64_t nr = (nc + run - 1) / run;
    const int64_t np = std::max<int64_t>(1, std::min<int64_t>(n_parts, nr));
    fixed_parts.clear();
    for (int64_t b = 0; b < np; ++b) {
      fixed_parts.push_back((int64_t)chunk_work.size());
      for (int64_t r = b; r < nr; r += np)
        for (int64_t c = r * run; c < std::min(nc, (r + 1) * run); ++c)
          add(pending[(size_t)c].first, pending[(size_t)c].second);
    }
    pending.clear();
    defer = false;
    interleaved = true;
  }
  void add(const Chunk& c, int64_t work) {
    const int64_t moff = (int64_t)meta.size() * 4;  // bytes
    std::vector<int32_t> m = c.meta;
    while ((m.size() * 4) % 16) m.push_back(0);
    meta.insert(meta.end(), m.begin(), m.end());
    auto push = [&](int32_t dst, int64_t bytes, int src, int64_t soff, bool last) {
      cps.push_back(dst);
      cps.push_back((int32_t)((uint32_t)bytes | (uint32_t)src << 28 | (last ? 1u << 30 : 0u)));
      cps.push_back((int32_t)(uint32_t)(soff & 0xffffffffll));
      cps.push_back((int32_t)(uint32_t)(soff >> 32));
    };
    push(0, (int64_t)m.size() * 4, 0, moff, c.copies.empty());
    for (size_t k = 0; k < c.copies.size(); ++k)
      push(c.copies[k].dst, c.copies[k].bytes, c.copies[k].src, c.copies[k].soff,
           k + 1 == c.copies.size());
    chunk_entry.push_back((int64_t)cps.size() / 4);
    chunk_work.push_back(work);
  }
  // contiguous chunk ranges per part, balanced by work
  void parts(int n_parts, std::vector<int64_t>& sub_start, std::vector<int64_t>& entry_start) const {
    const int64_t nc = (int64_t)chunk_work.size();
    if (!fixed_parts.empty()) {
      sub_start.clear();
      entry_start.clear();
      for (int64_t c : fixed_parts) {
        if (!sub_start.empty() && c == sub_start.back()) continue;  // empty part
        sub_start.push_back(c);
        entry_start.push_back(chunk_entry[(size_t)c]);
      }
      if (sub_start.back() != nc) {
        sub_start.push_back(nc);
        entry_start.push_back(chunk_entry.back());
      }
      return;
    }
    int64_t total = 0;
    for (int64_t w : chunk_work) total += w;
    n_parts = (int)std::max<int64_t>(1, std::min<int64_t>(n_parts, nc));
    sub_start.assign((size_t)n_parts + 1, nc);
    entry_start.assign((size_t)n_parts + 1, chunk_entry.back());
    sub_start[0] = 0;
    entry_start[0] = 0;
    int64_t acc = 0, c = 0;
    for (int b = 1; b < n_parts; ++b) {
      const int64_t target = total * b / n_parts;
      while (c < nc && acc + chunk_work[(size_t)c] / 2 < target) acc += chunk_work[(size_t)c++];
      sub_start[(size_t)b] = c;
      entry_start[(size_t)b] = chunk_entry[(size_t)c];
    }
  }
};

int align16(int x) { return (x + 15) & ~15; }

// BMV_LANE_INTERLEAVE=0/1 forces the chunk assignment (tests); default: the
// planner's choice
bool interleave_override(bool choice) {
  const char* e = std::getenv("BMV_LANE_INTERLEAVE");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return choice;
}

// BMV_LANE_RUN=k forces the K4 interleave run length (tests / tuning)
int64_t lane_run_override(int64_t choice) {
  const char* e = std::getenv("BMV_LANE_RUN");
  if (e && e[0]) return std::max<int64_t>(1, std::atoll(e));
  return choice;
}

}  // namespace

struct bmv_lane_plan {
  int kind = 0;  // 4 or 5
  int maxk = 0;  // K5: largest k-step count of a task
  bool two_tiles = false;  // K5: block rows average more than 16 rows
  bool short_rows = false;  // K4: interleaved chunks (short block rows)
  int n_parts = 0;
  int stage_bytes = 0;
  int smem_bytes = 0;
  int64_t* part_sub_start = nullptr;
  int64_t* part_entry_start = nullptr;
  int4* copies = nullptr;
  int32_t* meta = nullptr;
};

namespace {

int upload_stream(const StreamBuild& sb, int n_parts, bmv_lane_plan* p) {
  std::vector<int64_t> ss, es;
  sb.parts(n_parts, ss, es);
  p->n_parts = (int)ss.size() - 1;
  int rc = upload(ss.data(), (int64_t)ss.size(), &p->part_sub_start);
  if (rc == BMV_OK) rc = upload(es.data(), (int64_t)es.size(), &p->part_entry_start);
  if (rc == BMV_OK)
    rc = upload(reinterpret_cast<const int4*>(sb.cps.data()), (int64_t)sb.cps.size() / 4, &p->copies);
  if (rc == BMV_OK) rc = upload(sb.meta.data(), (int64_t)sb.meta.size(), &p->meta);
  return rc;
}

}  // namespace

extern "C" {

int bmv_lane_plan_destroy(bmv_lane_plan* p) {
  if (!p) return BMV_OK;
  release(p->part_sub_start);
  release(p->part_entry_start);
  release(p->copies);
  release(p->meta);
  delete p;
  return BMV_OK;
}

}  // extern "C"

namespace {

int plan_k4(const bmv_tmmult_lane_desc* d, StreamBuild& sb, int& stage_bytes_out,
            int sm_count_host) {
  const int stage_bytes = ((kSmemBudget - kAccTiles * 64 * 8) / kLnStages) & ~127;
  stage_bytes_out = stage_bytes;
  // one item = rows sharing the accumulator (<= kAccTiles S tiles); chunks of
  // an item = rows (or B-block groups of one row) fitting a stage
  std::unordered_map<int64_t, int> tile_of;  // (S offset of tile row 0) -> acc tile
  std::vector<int4> flush;                   // current item's flush records
  Chunk cur;
  std::vector<int32_t> recs;
  int cur_bytes = 0, cur_rows = 0;
  int64_t cur_work = 0;
  int64_t a_lo = 0, a_hi = 0, b_lo = 0, b_hi = 0;  // element ranges of the chunk
  int64_t pair_base = 0;

  auto chunk_meta_bytes = [&](size_t n_recs, size_t n_fl) {
    return align16(16 + (int)n_recs * kK4Rec * 4) + (int)n_fl * 16;
  };
  // close the current chunk (flush=true: also the item)
  auto emit = [&](bool do_flush) {
    // interleaved chunks: the item closes at the end of every run of chunks
    if (sb.defer && ((int64_t)sb.pending.size() + 1) % sb.run == 0) do_flush = true;
    const int n_tiles = (int)(recs.size() / kK4Rec);
    const int nfl = do_flush ? (int)flush.size() : 0;
    if (n_tiles == 0 && nfl == 0) return;
    const int rec_off = 4;
    const int fl_off_b = align16(16 + n_tiles * kK4Rec * 4);
    const int meta_b = fl_off_b + nfl * 16;
    const int a_off_b = align16(meta_b);
    const int b_off_b = align16(a_off_b + (int)((a_hi - a_lo) * 8));
    cur.meta.assign((size_t)meta_b / 4, 0);
    cur.meta[0] = n_tiles;
    cur.meta[1] = nfl;
    cur.meta[2] = rec_off;
    cur.meta[3] = fl_off_b / 4;
    // shift stage offsets of A / B by the data region starts
    for (int t = 0; t < n_tiles; ++t) {
      const int32_t* r = &recs[(size_t)t * kK4Rec];
      int32_t* o = &cur.meta[(size_t)(rec_off + t * kK4Rec)];
      for (int m = 0; m < 8; ++m) {
        if (r[m] < 0) {
          o[m] = -1;
        } else {
          const int so = (r[m] & 0xffff) + a_off_b / 8;
          o[m] = so | (r[m] & 0x7fff0000);
        }
        o[8 + m] = r[8 + m];
      }
      o[16] = r[16] + b_off_b / 8;
      o[17] = r[17];
      o[18] = r[18];
    }
    for (int f = 0; f < nfl; ++f) {
      int32_t* o = &cur.meta[(size_t)(fl_off_b / 4 + f * 4)];
      o[0] = flush[(size_t)f].x;
      o[1] = flush[(size_t)f].y;
      o[2] = flush[(size_t)f].z;
      o[3] = flush[(size_t)f].w;
    }
    cur.copies.clear();
    if (a_hi > a_lo) cur.copies.push_back({a_off_b, (a_hi - a_lo) * 8, 1, a_lo * 8});
    if (b_hi > b_lo) cur.copies.push_back({b_off_b, (b_hi - b_lo) * 8, 2, b_lo * 8});
    sb.put(cur, cur_work + 64);
    recs.clear();
    cur_bytes = 0;
    cur_rows = 0;
    cur_work = 0;
    a_lo = a_hi = b_lo = b_hi = 0;
    if (do_flush) {
      flush.clear();
      tile_of.clear();
    }
  };

  // parts (one per CTA) are cut at rows, balanced by DMMA work; an item
  // (accumulator lifetime) never spans two parts
  std::vector<int64_t> row_work((size_t)d->n_rows + 1, 0);
  for (int32_t i = 0; i < d->n_rows; ++i) {
    int64_t ncols = 0, ntl = 0;
    for (int64_t pa = d->a_row_start[i]; pa < d->a_row_start[i + 1]; ++pa)
      ncols += __builtin_popcountll(d->a_mask[pa]);
    for (int64_t pb = d->b_row_start[i]; pb < d->b_row_start[i + 1]; ++pb)
      ntl += (d->b_width[pb] + 7) / 8;
    // per tile: ~130 warp instructions of decode / accumulator add + the DMMAs
    row_work[(size_t)i + 1] = row_work[(size_t)i] + ((ncols + 7) / 8) * ntl * (d->row_rows[i] + 48) + 16;
  }
  const int n_parts = std::max(1, sm_count_host);
  int64_t sum_rows = 0;
  for (int32_t i = 0; i < d->n_rows; ++i) sum_rows += d->row_rows[i];
  // short block rows: every chunk is its own item and chunks are interleaved
  // over the CTAs (finish_interleaved); long rows: contiguous row parts
  // (and enough chunks per CTA for the interleave to average out: >= 16)
  int64_t data_bytes = 0;
  if (d->n_rows > 0) {
    const int64_t pa_end = d->a_row_start[d->n_rows], pb_end = d->b_row_start[d->n_rows];
    if (pa_end > 0) data_bytes += 8 * (d->a_off[pa_end - 1] - d->a_off[0]);
    if (pb_end > 0) data_bytes += 8 * (d->b_off[pb_end - 1] - d->b_off[0]);
  }
  const bool interleave = interleave_override(d->n_rows > 0 && sum_rows < 16 * (int64_t)d->n_rows &&
                                              data_bytes >= 16LL * n_parts * stage_bytes);
  sb.defer = interleave;
  // runs of consecutive chunks per CTA turn: fewer item flushes (S tiles shared by
  // neighbouring block rows are reduced in shared memory once per run instead of once
  // per chunk) while every CTA still gets >= 16 runs
  sb.run = lane_run_override(std::max<int64_t>(
      1, std::min<int64_t>(4, data_bytes / std::max<int64_t>(1, 16LL * n_parts * stage_bytes))));
  int next_part = 1;
  sb.fixed_parts.push_back(0);
  for (int32_t i = 0; i < d->n_rows; ++i) {
    if (!interleave && next_part < n_parts &&
        row_work[(size_t)i] >= row_work.back() * next_part / n_parts) {
      emit(true);
      sb.fixed_parts.push_back((int64_t)sb.chunk_work.size());
      while (next_part < n_parts && row_work[(size_t)i] >= row_work.back() * next_part / n_parts)
        ++next_part;
    }
    const int64_t pa0 = d->a_row_start[i], pa1 = d->a_row_start[i + 1];
    const int64_t pb0 = d->b_row_start[i], pb1 = d->b_row_start[i + 1];
    const int rows = d->row_rows[i];
    const int64_t na = pa1 - pa0, nb = pb1 - pb0;
    if (na == 0 || nb == 0 || rows == 0) {
      pair_base += na * nb;
      continue;
    }
    // compact A columns of the row
    std::vector<std::pair<int64_t, int>> cols;  // (a pos, lane)
    for (int64_t pa = pa0; pa < pa1; ++pa) {
      uint64_t m = d->a_mask[pa];
      while (m) {
        const int l = __builtin_ctzll(m);
        m &= m - 1;
        cols.push_back({pa, l});
      }
    }
    const int64_t a_first = d->a_off[pa0];
    const int64_t a_last = d->a_off[pa1 - 1] + (int64_t)rows * d->a_stride[pa1 - 1];
    const int64_t a_len = a_last - a_first;
    if (a_len >= 0x8000) {
      set_error("tmmult lane plan: block row %d spans %lld values of A (max 32767)", i,
                (long long)a_len);
      return BMV_ERR_INVALID;
    }
    // (A col block, 8-lane row group) pairs with active lanes: S tile rows
    int row_rgroups = 0;
    for (int64_t pa = pa0; pa < pa1; ++pa)
      for (int rg = 0; rg < 64; rg += 8)
        if ((d->a_mask[pa] >> rg) & 0xffull) ++row_rgroups;
    // the row's S tiles (new ones count against the accumulator)
    // tile key: S offset of (row a-lane group 0, col tile) -> per (pa, pb, nt)
    // process B blocks in groups that fit the stage together with the A range
    int64_t pb = pb0;
    while (pb < pb1) {
      // group of B blocks [pb, pe)
      int64_t pe = pb;
      int64_t b_len = 0;
      const int64_t b_first = d->b_off[pb];
      const int ncg = (int)((cols.size() + 7) / 8);
      int grp_tiles = 0, grp_acc = 0;
      for (; pe < pb1; ++pe) {
        const int64_t nl = d->b_off[pe] + (int64_t)rows * d->b_stride[pe] - b_first;
        const int ntile = (d->b_width[pe] + 7) / 8;
        const int acc_pe = row_rgroups * ntile;  // S tiles of this B block
        const int need = align16((int)(a_len * 8)) + align16((int)(nl * 8)) +
                         chunk_meta_bytes((size_t)(grp_tiles + ncg * ntile), kAccTiles) + 64;
        if (pe > pb && (need > stage_bytes || grp_acc + acc_pe > kAccTiles)) break;
        if (need > stage_bytes || acc_pe > kAccTiles) {
          set_error("tmmult lane plan: block row %d does not fit a stage / the accumulator", i);
          return BMV_ERR_INVALID;
        }
        b_len = nl;
        grp_tiles += ncg * ntile;
        grp_acc += acc_pe;
      }
      // count new accumulator tiles of this group
      std::vector<int64_t> new_keys;
      for (int64_t q = pb; q < pe; ++q) {
        const int ntile = (d->b_width[q] + 7) / 8;
        for (int64_t pa = pa0; pa < pa1; ++pa) {
          if (!d->a_mask[pa]) continue;
          const int64_t t = pair_base + (pa - pa0) * nb + (q - pb0);
          const uint64_t m = d->a_mask[pa];
          for (int rg = 0; rg < 64; rg += 8) {
            if (!((m >> rg) & 0xffull)) continue;
            for (int nt = 0; nt < ntile; ++nt) {
              const int64_t key = d->c_off[t] + (int64_t)rg * d->c_stride[t] + nt * 8;
              if (!tile_of.count(key) &&
                  std::find(new_keys.begin(), new_keys.end(), key) == new_keys.end())
                new_keys.push_back(key);
            }
          }
        }
      }
      if ((int)(tile_of.size() + new_keys.size()) > kAccTiles) {
        emit(true);  // close the item: accumulator full
        if ((int)new_keys.size() > kAccTiles) {
          set_error("tmmult lane plan: block row %d touches more than %d S tiles", i, kAccTiles);
          return BMV_ERR_INVALID;
        }
      }
      // does the group fit the open chunk?  (a row split over several B
      // groups restages its A range in every chunk)
      if (!recs.empty()) {
        const bool same_row = a_first < a_hi;
        const int need = align16((int)((a_last - a_lo) * 8)) +
                         align16((int)((b_first + b_len - b_lo) * 8)) +
                         chunk_meta_bytes(recs.size() / kK4Rec + grp_tiles, kAccTiles) + 64;
        if (same_row || need > stage_bytes || a_last - a_lo >= 0x8000) emit(false);
      }
      if (recs.empty()) {
        a_lo = a_first;
        b_lo = b_first;
      }
      a_hi = std::max(a_hi, a_last);
      b_hi = std::max(b_hi, b_first + b_len);
      for (int64_t q = pb; q < pe; ++q) {
        const int ntile = (d->b_width[q] + 7) / 8;
        for (size_t c0 = 0; c0 < cols.size(); c0 += 8) {
          for (int nt = 0; nt < ntile; ++nt) {
            int32_t r[kK4Rec];
            for (int k = 0; k < kK4Rec; ++k) r[k] = 0;
            for (int m = 0; m < 8; ++m) {
              if (c0 + m < cols.size()) {
                const int64_t pa = cols[c0 + m].first;
                const int l = cols[c0 + m].second;
                const int64_t so = d->a_off[pa] + l - a_lo;  // doubles from the A region start
                r[m] = (int32_t)so | (d->a_stride[pa] << 16);
                const int64_t t = pair_base + (pa - pa0) * nb + (q - pb0);
                const int rg = l & ~7;
                const int64_t key = d->c_off[t] + (int64_t)rg * d->c_stride[t] + nt * 8;
                auto it = tile_of.find(key);
                int at;
                if (it == tile_of.end()) {
                  at = (int)tile_of.size();
                  tile_of[key] = at;
                  const int srows = std::min(8, d->c_rows[t] - rg);
                  const int scols = std::min(8, d->b_width[q] - nt * 8);
                  if (key > INT32_MAX) {
                    set_error("tmmult lane plan: S offset beyond 2^31");
                    return BMV_ERR_INVALID;
                  }
                  flush.push_back(make_int4((int)key, d->c_stride[t], srows | scols << 8, at));
                } else {
                  at = it->second;
                }
                r[8 + m] = at * 64 + (l & 7) * 8;
              } else {
                r[m] = -1;
                r[8 + m] = -1;
              }
            }
            r[16] = (int32_t)(d->b_off[q] - b_lo) + nt * 8;
            r[17] = rows | (d->b_stride[q] << 16);
            r[18] = std::min(8, std::min(d->b_width[q], d->b_stride[q]) - nt * 8);
            recs.insert(recs.end(), r, r + kK4Rec);
            cur_work += rows;
          }
        }
      }
      pb = pe;
    }
    ++cur_rows;
    pair_base += na * nb;
  }
  emit(true);
  sb.finish_interleaved(n_parts);
  return BMV_OK;
}

}  // namespace

extern "C" {

int bmv_tmmult_lane_create(const bmv_tmmult_lane_desc* d, bmv_lane_plan** out) {
  if (!d || !out) {
    set_error("null argument");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  StreamBuild sb;
  int stage_bytes = 0;
  {
    const int rc0 = plan_k4(d, sb, stage_bytes, sm_count());
    if (rc0 != BMV_OK) return rc0;
  }
  auto* p = new bmv_lane_plan();
  p->kind = 4;
  p->short_rows = sb.interleaved;
  p->stage_bytes = stage_bytes;
  p->smem_bytes = kAccTiles * 64 * 8 + kLnStages * stage_bytes;
  int rc = sb.chunk_work.empty() ? BMV_OK : upload_stream(sb, sm_count(), p);
  if (rc != BMV_OK) {
    bmv_lane_plan_destroy(p);
    return rc;
  }
  if (sb.chunk_work.empty()) p->n_parts = 0;
  *out = p;
  return BMV_OK;
}

int bmv_tmmult_lane_run(bmv_lane_plan* p, const double* a, const double* b, double* c,
                        int64_t c_len, void* stream) {
  if (!p || p->kind != 4) {
    set_error("not a tmmult lane plan");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  int rc = zero_async(c, c_len, st);
  if (rc || p->n_parts == 0) return rc;
  auto kern = p->short_rows ? k4_lane_kernel<kLnWarpsWide> : k4_lane_kernel<kLnWarps>;
  const int threads = ((p->short_rows ? kLnWarpsWide : kLnWarps) + 1) * 32;
  BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    p->smem_bytes));
  LnArgs g{};
  g.part_sub_start = p->part_sub_start;
  g.part_entry_start = p->part_entry_start;
  g.copies = p->copies;
  g.src = CopySrc{reinterpret_cast<const char*>(p->meta), reinterpret_cast<const char*>(a),
                  reinterpret_cast<const char*>(b)};
  g.out = c;
  g.stage_bytes = p->stage_bytes;
  kern<<<p->n_parts, threads, p->smem_bytes, st>>>(g);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

}  // extern "C"

namespace {

int plan_k5(const bmv_mmult_lane_desc* d, StreamBuild& sb, int& stage_bytes_out, int& maxk,
            int n_parts) {
  maxk = 0;
  {
    // short rows and >= 16 chunks per CTA: interleave the chunks over the CTAs
    int64_t sum_rows = 0;
    for (int32_t i = 0; i < d->n_rows; ++i) sum_rows += d->row_rows[i];
    int64_t data_bytes = 0;
    if (d->n_rows > 0 && d->a_row_start[d->n_rows] > 0)
      data_bytes = 8 * (d->a_off[d->a_row_start[d->n_rows] - 1] - d->a_off[0]);
    sb.defer = interleave_override(
        d->n_rows > 0 && sum_rows < 16 * (int64_t)d->n_rows &&
        data_bytes >= 16LL * std::max(1, n_parts) * ((kSmemBudget / kLnStages) & ~127));
  }
  const int stage_bytes = (kSmemBudget / kLnStages) & ~127;
  stage_bytes_out = stage_bytes;
  Chunk cur;
  std::vector<int32_t> tasks;  // concatenated records
  std::vector<int32_t> toffs;  // record offsets (int32 units, relative to the record area)
  int64_t a_lo = 0, a_hi = 0, work = 0;
  auto meta_bytes = [&](size_t n_t, size_t rec_ints) {
    return align16(16 + (int)n_t * 4 + (int)rec_ints * 4);
  };
  auto emit = [&]() {
    const int nt = (int)toffs.size();
    if (nt == 0) return;
    const int toff_i = 4;
    const int rec_i = 4 + nt;
    const int mb = meta_bytes((size_t)nt, tasks.size());
    const int a_off_b = mb;
    cur.meta.assign((size_t)mb / 4, 0);
    cur.meta[0] = nt;
    cur.meta[1] = toff_i;
    for (int t = 0; t < nt; ++t) cur.meta[(size_t)(toff_i + t)] = rec_i + toffs[(size_t)t];
    for (size_t k = 0; k < tasks.size(); ++k) cur.meta[(size_t)rec_i + k] = tasks[k];
    // shift A column offsets by the A region start (doubles)
    for (int t = 0; t < nt; ++t) {
      int32_t* r = &cur.meta[(size_t)(rec_i + toffs[(size_t)t])];
      const int ks = r[3] >> 16;
      for (int s = 0; s < ks; ++s)
        for (int m = 0; m < 4; ++m) {
          int32_t& v = r[4 + 8 * s + m];
          if (v >= 0) v = ((v & 0xffff) + a_off_b / 8) | (v & 0x7fff0000);
        }
    }
    cur.copies.clear();
    if (a_hi > a_lo) cur.copies.push_back({a_off_b, (a_hi - a_lo) * 8, 1, a_lo * 8});
    sb.put(cur, work + 64);
    tasks.clear();
    toffs.clear();
    a_lo = a_hi = 0;
    work = 0;
  };
  for (int32_t i = 0; i < d->n_rows; ++i) {
    const int64_t pa0 = d->a_row_start[i], pa1 = d->a_row_start[i + 1];
    const int64_t pc0 = d->c_row_start[i], pc1 = d->c_row_start[i + 1];
    const int rows = d->row_rows[i];
    const int64_t na = pa1 - pa0;
    if (pc1 == pc0 || rows == 0) continue;
    std::vector<std::pair<int64_t, int>> cols;
    for (int64_t pa = pa0; pa < pa1; ++pa) {
      uint64_t m = d->a_mask[pa];
      while (m) {
        const int l = __builtin_ctzll(m);
        m &= m - 1;
        cols.push_back({pa, l});
      }
    }
    const int ks = (int)((cols.size() + 3) / 4);
    maxk = std::max(maxk, ks);
    if (ks > 255) {
      set_error("mmult lane plan: block row %d has %d active columns (max 1020)", i,
                (int)cols.size());
      return BMV_ERR_INVALID;
    }
    int64_t a_first = na ? d->a_off[pa0] : 0;
    int64_t a_last = na ? d->a_off[pa1 - 1] + (int64_t)rows * d->a_stride[pa1 - 1] : 0;
    // row tasks
    std::vector<int32_t> rt, ro;
    for (int64_t pc = pc0; pc < pc1; ++pc) {
      const int nst_all = d->c_stride[pc];
      for (int nt = 0; nt * 8 < nst_all; ++nt) {
        ro.push_back((int32_t)rt.size());
        const int64_t yoff = d->c_off[pc] + nt * 8;
        rt.push_back((int32_t)(yoff & 0xffffffff));
        rt.push_back((int32_t)(yoff >> 32));
        rt.push_back(rows | (d->c_stride[pc] << 16));
        const int ncol = std::max(0, std::min(8, d->c_width[pc] - nt * 8));
        const int nst = std::min(8, d->c_stride[pc] - nt * 8);
        rt.push_back(ncol | nst << 8 | ks << 16);
        for (int s = 0; s < ks; ++s) {
          for (int m = 0; m < 4; ++m) {
            const size_t ci = (size_t)(4 * s + m);
            if (ci < cols.size()) {
              const int64_t pa = cols[ci].first;
              rt.push_back((int32_t)(d->a_off[pa] + cols[ci].second - a_first) | (d->a_stride[pa] << 16));
            } else {
              rt.push_back(-1);
            }
          }
          for (int m = 0; m < 4; ++m) {
            const size_t ci = (size_t)(4 * s + m);
            int32_t co = -1;
            if (ci < cols.size()) {
              const int64_t pa = cols[ci].first;
              const int64_t bi = d->b_pair_start[i] + (pa - pa0) * (pc1 - pc0) + (pc - pc0);
              const int64_t bo = d->b_off[bi];
              if (bo >= 0) {
                const int64_t v = bo + (int64_t)cols[ci].second * d->b_stride[bi] + nt * 8;
                if (v > INT32_MAX) {
                  set_error("mmult lane plan: C offset beyond 2^31");
                  return BMV_ERR_INVALID;
                }
                co = (int32_t)v;
              }
            }
            rt.push_back(co);
          }
        }
      }
    }
    const int64_t a_len = a_last - a_first;
    if (a_len >= 0x8000 - 8) {
      set_error("mmult lane plan: block row %d spans %lld values (stage offsets are 15 bits)", i,
                (long long)a_len);
      return BMV_ERR_INVALID;
    }
    const int64_t na_lo = toffs.empty() ? a_first : a_lo;
    const int need = meta_bytes(toffs.size() + ro.size(), tasks.size() + rt.size()) +
                     align16((int)((a_last - na_lo) * 8)) + 64;
    const bool contiguous = toffs.empty() || a_first >= a_hi;
    if (!toffs.empty() && (need > stage_bytes || !contiguous || (a_last - na_lo) >= 0x8000 - 8))
      emit();
    if (toffs.empty()) a_lo = a_first;
    const int need1 = meta_bytes(ro.size(), rt.size()) + align16((int)(a_len * 8)) + 64;
    if (need1 > stage_bytes) {
      set_error("mmult lane plan: block row %d does not fit a stage", i);
      return BMV_ERR_INVALID;
    }
    // rebase this row's A offsets on the chunk's A start
    const int shift = (int)(a_first - a_lo);
    for (size_t t = 0; t < ro.size(); ++t) {
      int32_t* r = &rt[(size_t)ro[t]];
      const int k = r[3] >> 16;
      for (int s = 0; s < k; ++s)
        for (int m = 0; m < 4; ++m) {
          int32_t& v = r[4 + 8 * s + m];
          if (v >= 0) v = ((v & 0xffff) + shift) | (v & 0x7fff0000);
        }
      toffs.push_back((int32_t)tasks.size() + ro[t]);
    }
    tasks.insert(tasks.end(), rt.begin(), rt.end());
    a_hi = std::max(a_hi, a_last);
    work += (int64_t)ro.size() * rows * (ks + 1);
  }
  emit();
  sb.finish_interleaved(std::max(1, n_parts));
  return BMV_OK;
}

}  // namespace

extern "C" {

int bmv_mmult_lane_create(const bmv_mmult_lane_desc* d, bmv_lane_plan** out) {
  if (!d || !out) {
    set_error("null argument");
    return BMV_ERR_INVALID;
  }
  *out = nullptr;
  StreamBuild sb;
  int stage_bytes = 0;
  int k5_maxk = 0;
  {
    int maxk = 0;
    const int rc0 = plan_k5(d, sb, stage_bytes, maxk, sm_count());
    k5_maxk = maxk;
    if (rc0 != BMV_OK) return rc0;
  }
  auto* p = new bmv_lane_plan();
  p->kind = 5;
  p->maxk = k5_maxk;
  {
    int64_t sum_rows = 0;
    for (int32_t i = 0; i < d->n_rows; ++i) sum_rows += d->row_rows[i];
    p->two_tiles = d->n_rows > 0 && sum_rows > 16 * (int64_t)d->n_rows;
  }
  p->stage_bytes = stage_bytes;
  p->smem_bytes = kLnStages * stage_bytes;
  int rc = sb.chunk_work.empty() ? BMV_OK : upload_stream(sb, sm_count(), p);
  if (rc != BMV_OK) {
    bmv_lane_plan_destroy(p);
    return rc;
  }
  if (sb.chunk_work.empty()) p->n_parts = 0;
  *out = p;
  return BMV_OK;
}

int bmv_mmult_lane_run(bmv_lane_plan* p, const double* a, const double* b, double* c,
                       double alpha, int32_t accumulate, int64_t zero_len, void* stream) {
  if (!p || p->kind != 5) {
    set_error("not an mmult lane plan");
    return BMV_ERR_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  int rc = zero_async(c, zero_len, st);
  if (rc || p->n_parts == 0) return rc;
  auto kern = p->two_tiles ? k5_lane_kernel<kKGroup, true, kLnWarpsWide>
                           : k5_lane_kernel<kKGroup, false, kLnWarpsWide>;
  BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    p->smem_bytes));
  LnArgs g{};
  g.part_sub_start = p->part_sub_start;
  g.part_entry_start = p->part_entry_start;
  g.copies = p->copies;
  g.src = CopySrc{reinterpret_cast<const char*>(p->meta), reinterpret_cast<const char*>(a), nullptr};
  g.out = c;
  g.alpha = alpha;
  g.accumulate = accumulate;
  g.stage_bytes = p->stage_bytes;
  g.cmat = b;
  kern<<<p->n_parts, (kLnWarpsWide + 1) * 32, p->smem_bytes, st>>>(g);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

/* Host-only: the plan's stage stream (metadata words, copy entries, part
   ranges) for CPU emulation in the tests; arrays malloc'ed, freed with
   bmv_lane_host_free.  kind 4: desc is a bmv_tmmult_lane_desc, 5: mmult. */
int bmv_lane_plan_host(int32_t kind, const void* desc, int32_t n_parts, bmv_lane_host* out) {
  if (!desc || !out || (kind != 4 && kind != 5)) {
    set_error("invalid lane plan host request");
    return BMV_ERR_INVALID;
  }
  StreamBuild sb;
  int stage_bytes = 0, host_maxk = 0;
  const int rc = kind == 4 ? plan_k4(static_cast<const bmv_tmmult_lane_desc*>(desc), sb, stage_bytes, n_parts)
                           : plan_k5(static_cast<const bmv_mmult_lane_desc*>(desc), sb, stage_bytes, host_maxk, n_parts);
  if (rc != BMV_OK) return rc;
  std::vector<int64_t> ss, es;
  if (!sb.chunk_work.empty()) sb.parts(n_parts, ss, es);
  out->stage_bytes = stage_bytes;
  out->n_parts = sb.chunk_work.empty() ? 0 : (int32_t)ss.size() - 1;
  out->meta_len = (int64_t)sb.meta.size();
  out->n_entries = (int64_t)sb.cps.size() / 4;
  out->meta = static_cast<int32_t*>(malloc(sizeof(int32_t) * (sb.meta.size() + 1)));
  out->copies = static_cast<int32_t*>(malloc(sizeof(int32_t) * (sb.cps.size() + 1)));
  out->part_sub_start = static_cast<int64_t*>(malloc(sizeof(int64_t) * (ss.size() + 1)));
  out->part_entry_start = static_cast<int64_t*>(malloc(sizeof(int64_t) * (es.size() + 1)));
  std::copy(sb.meta.begin(), sb.meta.end(), out->meta);
  std::copy(sb.cps.begin(), sb.cps.end(), out->copies);
  std::copy(ss.begin(), ss.end(), out->part_sub_start);
  std::copy(es.begin(), es.end(), out->part_entry_start);
  return BMV_OK;
}

int bmv_lane_host_free(bmv_lane_host* h) {
  if (!h) return BMV_OK;
  free(h->meta);
  free(h->copies);
  free(h->part_sub_start);
  free(h->part_entry_start);
  h->meta = h->copies = nullptr;
  h->part_sub_start = h->part_entry_start = nullptr;
  return BMV_OK;
}

}  // extern "C"
