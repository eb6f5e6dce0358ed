// K1 (streamed): the sum-factorised Hamiltonian on the active (cell, column)
// pairs with every per-cell operand staged by TMA.
//
// Same arithmetic as the one-pass kernel (bmv_sumfac.cuh: thread t of a
// pair holds plane z = t; 12 contractions, 4 pair-tile transposes), but the
// pairs are cut into chunks of NW * P consecutive pairs (NW consumer warps,
// P = 32 / n pairs per warp).  One persistent CTA per SM slot walks its
// chunks; a producer warp streams each chunk's operands into a ring of
// shared-memory stages with cp.async.bulk:
//   [header + NW*P pair descriptors | (x, hx) block offsets of the chunk's
//    visits' groups | 16-bit slots of the chunk's cell range | quadrature
//    coefficients w3*V of the cell range]
// so a consumer warp's only dependent global access is the gather of X.
// With XPF the gather of the NEXT chunk's X values is issued (cp.async, one
// 8-byte element per lane and plane entry) right after the current values
// are read into registers, and lands while the warp computes.
// Replaces the cell loop of CellOperator.apply (reference
// bcsrmv/matfree.py:458-527) for the Hamiltonian; the mass operator and the
// deterministic colour mode keep the one-pass kernel (bmv_cellop.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "bmv_cellop_stream.cuh"
#include "bmv_common.cuh"
#include "bmv_sumfac.cuh"
#include "bmv_tma.cuh"

namespace bmv {
namespace {

constexpr int kMaxStages = 4;

struct StreamArgs {
  const int64_t* __restrict__ part_chunk_start;
  const int64_t* __restrict__ part_entry_start;
  const int4* __restrict__ copies;
  CopySrc src;  // p0 = chunk meta, p1 = group table (int2), p2 = slots (u16), p3 = coefficients
  const double* __restrict__ x;
  double* __restrict__ hx;
  int stage_bytes;
  int n_stages;
  int off_gtab;   // byte offset of the group table in a stage (slots and
                  // coefficients: per chunk, header words 1 and 2)
  int coef_cell;  // 1: coefficient row per cell; 0: one row for all cells
};

template <int N, bool XPF, bool COEF>
__global__ void __launch_bounds__((StreamShape<N>::NW + 1) * 32)
    __maxnreg__(StreamShape<N>::MAXREG) cellop_stream_kernel(const StreamArgs g, const __grid_constant__ CellTables tb) {
  using SS = StreamShape<N>;
  constexpr int NW = SS::NW, P = SS::P, N2 = N * N, SR = SS::SR, Q3P = SS::Q3P;
  constexpr int TILE = Tile<N>::TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int warp = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int64_t c0 = g.part_chunk_start[blockIdx.x], c1 = g.part_chunk_start[blockIdx.x + 1];
  const int NS = g.n_stages;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NS; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], NW);
    }
  }
  __syncthreads();
  char* stages = reinterpret_cast<char*>(smem) + NW * SS::warp_bytes(XPF);
  if (warp == NW) {
    stream_producer(g.copies, g.part_entry_start[blockIdx.x], g.part_entry_start[blockIdx.x + 1],
                    c1 - c0, g.src, stages, g.stage_bytes, NS, full, empty, lid);
    return;
  }
  const int J = (int)(c1 - c0);
  const int sub = lid / N;
  const int t = lid - sub * N;
  const bool lane_ok = sub < P;
  const int tt = lane_ok ? t : 0;
  double* buf = reinterpret_cast<double*>(smem + warp * SS::warp_bytes(XPF)) + sub * TILE;
  double* xs = reinterpret_cast<double*>(smem + warp * SS::warp_bytes(XPF) + SS::tile_bytes) + lid;

  // this lane's pair in chunk stage `stg`: {cell (local), first group (local), lane | stride << 16, ok}
  auto pair_of = [&](const char* stg) -> int4 {
    const int n_pairs = reinterpret_cast<const int*>(stg)[0];
    const int q = warp * P + sub;
    if (!lane_ok || q >= n_pairs) return make_int4(0, 0, 0, 0);
    int4 d = reinterpret_cast<const int4*>(stg)[1 + q];
    d.w = 1;
    return d;
  };
  auto gather_to_smem = [&](const char* stg) {
    const int4 d = pair_of(stg);
    if (d.w) {
      const int* hdr = reinterpret_cast<const int*>(stg);
      const uint16_t* sl = reinterpret_cast<const uint16_t*>(stg + hdr[1]) + d.x * SR + t * N2;
      const int2* gt = reinterpret_cast<const int2*>(stg + g.off_gtab) + d.y;
      const int lane = d.z & 0xffff, stride = d.z >> 16;
#pragma unroll
      for (int k = 0; k < N2; ++k) {
        const unsigned s = sl[k];
        const int xo = gt[s >> 11].x;
        if (xo >= 0)
          cp_async8(xs + 32 * k, g.x + xo + (int64_t)(s & 2047u) * stride + lane);
        else
          xs[32 * k] = 0.0;
      }
    } else {
#pragma unroll
      for (int k = 0; k < N2; ++k) xs[32 * k] = 0.0;
    }
    cp_async_commit();
  };

  if (XPF && J > 0) {
    mbar_wait(&full[0], 0);
    gather_to_smem(stages);
  }
#pragma unroll 1
  for (int j = 0; j < J; ++j) {
    const int st = j % NS;
    const char* stg = stages + (int64_t)st * g.stage_bytes;
    if (!XPF) mbar_wait(&full[st], (unsigned)((j / NS) & 1));
    const int4 d = pair_of(stg);
    const int* hdr = reinterpret_cast<const int*>(stg);
    const uint16_t* sl = reinterpret_cast<const uint16_t*>(stg + hdr[1]) + d.x * SR + tt * N2;
    const int2* gt = reinterpret_cast<const int2*>(stg + g.off_gtab) + d.y;
    const int lane = d.z & 0xffff, stride = d.z >> 16;
    double u[N][N];
    if (XPF) {
      cp_async_wait_all();
      __syncwarp();
#pragma unroll
      for (int y = 0; y < N; ++y)
#pragma unroll
        for (int x = 0; x < N; ++x) u[y][x] = xs[32 * (y * N + x)];
      __syncwarp();
      if (j + 1 < J) {
        const int s1 = (j + 1) % NS;
        mbar_wait(&full[s1], (unsigned)(((j + 1) / NS) & 1));
        gather_to_smem(stages + (int64_t)s1 * g.stage_bytes);
      }
    } else {
#pragma unroll
      for (int y = 0; y < N; ++y)
#pragma unroll
        for (int x = 0; x < N; ++x) {
          double v = 0.0;
          if (d.w) {
            const unsigned s = sl[y * N + x];
            const int xo = gt[s >> 11].x;
            if (xo >= 0) v = __ldg(g.x + xo + (int64_t)(s & 2047u) * stride + lane);
          }
          u[y][x] = v;
        }
    }
    const double* cf = reinterpret_cast<const double*>(stg + hdr[2]) +
                       (g.coef_cell ? d.x * Q3P : 0) + tt * N2;
    double out[N][N];
    sumfac_h_plane<N, COEF, 1>(u, out, buf, tt, lane_ok, cf, tb);
    {
      // re-read the pair's operands from the stage (nothing held across the compute)
      const int4 e = pair_of(stg);
      if (e.w) {
        const int* h2 = reinterpret_cast<const int*>(stg);
        const uint16_t* s2 = reinterpret_cast<const uint16_t*>(stg + h2[1]) + e.x * SR + t * N2;
        const int2* g2 = reinterpret_cast<const int2*>(stg + g.off_gtab) + e.y;
        const int ln = e.z & 0xffff, sd = e.z >> 16;
#pragma unroll
        for (int y = 0; y < N; ++y)
#pragma unroll
          for (int x = 0; x < N; ++x) {
            const unsigned s = s2[y * N + x];
            atomicAdd(g.hx + g2[s >> 11].y + (int64_t)(s & 2047u) * sd + ln, out[y][x]);
          }
      }
    }
    __syncwarp();
    if (lid == 0) mbar_arrive(&empty[st]);
  }
}

}  // namespace

// ---- host side -------------------------------------------------------------

namespace {

// per-SM shared memory 228 KB, 1 KB reserved per CTA, 64 B static barriers
template <int N>
int smem_budget() {
  constexpr int C = StreamShape<N>::CTAS;
  return std::min(227 * 1024, (228 * 1024 - C * 1024) / C) - 1024;
}

template <int N>
int build_plan_n(const bmv_cellop_desc* d, bool xpf, StreamPlan* sp) {
  using SS = StreamShape<N>;
  constexpr int N3 = N * N * N, SR = SS::SR, Q3P = SS::Q3P, K = SS::NW * SS::P;
  const int64_t np = d->n_pairs;
  const int ns = 3;
  const int warp_total = SS::NW * SS::warp_bytes(xpf);
  const int stage_bytes = ((smem_budget<N>() - warp_total) / ns) & ~127;
  const int meta_bytes = 16 + K * 16;
  const int row_bytes = SR * 2 + Q3P * 8;  // slots + coefficients of one cell
  if (stage_bytes < meta_bytes + 32 * 8 + row_bytes) return -1;
  // visit -> first group in the per-visit-even group table
  std::vector<int64_t> vg((size_t)d->n_visits + 1, 0);
  for (int32_t v = 0; v < d->n_visits; ++v) {
    const int64_t ng = d->visit_goff[v + 1] - d->visit_goff[v];
    vg[(size_t)v + 1] = vg[(size_t)v] + ((ng + 1) & ~int64_t(1));
  }
  std::vector<int32_t> gxh((size_t)vg.back() * 2, -1);
  for (int32_t v = 0; v < d->n_visits; ++v) {
    for (int64_t k = d->visit_goff[v]; k < d->visit_goff[v + 1]; ++k) {
      const int64_t o = vg[(size_t)v] + (k - d->visit_goff[v]);
      gxh[(size_t)o * 2] = (int32_t)d->group_xoff[k];
      gxh[(size_t)o * 2 + 1] = (int32_t)d->group_hoff[k];
    }
  }
  // 16-bit slots (group << 11 | row in block), rows padded to SR
  std::vector<uint16_t> sl16((size_t)d->n_cells * SR, 0);
  for (int64_t c = 0; c < d->n_cells; ++c)
    for (int k = 0; k < N3; ++k) {
      const uint32_t s = d->cell_slots[c * N3 + k];
      const uint32_t grp = s >> 24, rib = s & 0xffffffu;
      if (grp >= 32 || rib >= 2048) return -1;
      sl16[(size_t)c * SR + k] = (uint16_t)(grp << 11 | rib);
    }
  // chunks: <= K consecutive pairs whose cell range and groups fit a stage
  std::vector<int64_t> chunk_p0;
  auto cell_of = [&](int64_t q) { return (int64_t)d->visit_cell[d->pair_visit[q]]; };
  auto fits = [&](int64_t p0, int64_t e) {
    const int64_t cells = cell_of(e - 1) - cell_of(p0) + 1;
    const int64_t groups = vg[(size_t)d->pair_visit[e - 1] + 1] - vg[(size_t)d->pair_visit[p0]];
    return meta_bytes + groups * 8 + cells * row_bytes <= stage_bytes;
  };
  for (int64_t p0 = 0; p0 < np;) {
    int64_t e = std::min<int64_t>(p0 + K, np);
    while (e > p0 + 1 && !fits(p0, e)) --e;
    if (!fits(p0, e)) return -1;
    chunk_p0.push_back(p0);
    p0 = e;
  }
  chunk_p0.push_back(np);
  const int64_t nc = (int64_t)chunk_p0.size() - 1;
  // metadata records and copy entries (modes: 0 no coefficient, 1 per cell, 2 uniform)
  const int64_t rec_ints = meta_bytes / 4;
  std::vector<int32_t> meta((size_t)(nc * rec_ints), 0);
  const int off_gtab = meta_bytes;
  std::vector<int32_t> cps[3];
  int max_end = 0;
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t p0 = chunk_p0[(size_t)c], p1 = chunk_p0[(size_t)c + 1];
    const int64_t cf = cell_of(p0), cl = cell_of(p1 - 1);
    const int32_t v0 = d->pair_visit[p0], v1 = d->pair_visit[p1 - 1];
    const int64_t g0 = vg[(size_t)v0], g1 = vg[(size_t)v1 + 1];
    int32_t* rec = meta.data() + c * rec_ints;
    rec[0] = (int32_t)(p1 - p0);
    for (int64_t q = p0; q < p1; ++q) {
      const int32_t v = d->pair_visit[q];
      int32_t* e = rec + 4 * (1 + (q - p0));
      e[0] = (int32_t)(d->visit_cell[v] - cf);
      e[1] = (int32_t)(vg[(size_t)v] - g0);
      e[2] = d->pair_lane[q] | (d->visit_stride[v] << 16);
      e[3] = (int32_t)(d->visit_goff[v + 1] - d->visit_goff[v]);
    }
    const int gt_bytes = (int)((g1 - g0) * 8);
    const int64_t ncell = cl - cf + 1;
    // layout inside the stage: meta | gtab (rounded to 16) | slots | coef
    const int o_sl = (off_gtab + gt_bytes + 15) & ~15;
    const int o_cf = o_sl + (int)(ncell * SR * 2);
    // offsets vary per chunk: store them in the header for the consumers
    rec[1] = o_sl;
    rec[2] = o_cf;
    for (int mode = 0; mode < 3; ++mode) {
      auto& L = cps[mode];
      auto add = [&](int dst, int64_t bytes, int srcsel, int64_t soff, bool last) {
        L.push_back(dst);
        L.push_back((int32_t)((uint32_t)bytes | (uint32_t)srcsel << 28 | (last ? 1u << 30 : 0u)));
        L.push_back((int32_t)(uint32_t)(soff & 0xffffffffll));
        L.push_back((int32_t)(uint32_t)(soff >> 32));
      };
      add(0, meta_bytes, 0, c * (int64_t)meta_bytes, false);
      if (gt_bytes) add(off_gtab, gt_bytes, 1, g0 * 8, false);
      add(o_sl, ncell * SR * 2, 2, cf * SR * 2, mode == 0);
      if (mode == 1) add(o_cf, ncell * Q3P * 8, 3, cf * Q3P * 8, true);
      if (mode == 2) add(o_cf, Q3P * 8, 3, 0, true);
    }
    max_end = std::max<int>(max_end, o_cf + (int)(ncell * Q3P * 8));
  }
  if (max_end > stage_bytes) return -1;
  // parts: one per CTA slot, contiguous chunk ranges
  const int64_t slots = (int64_t)sm_count() * SS::CTAS;
  const int64_t parts = std::max<int64_t>(1, std::min<int64_t>(nc, slots));
  std::vector<int64_t> pcs((size_t)parts + 1), pes[3];
  for (int m = 0; m < 3; ++m) pes[m].assign((size_t)parts + 1, 0);
  std::vector<int64_t> chunk_entry[3];
  for (int m = 0; m < 3; ++m) {
    chunk_entry[m].assign((size_t)nc + 1, 0);
    int64_t e = 0;
    for (int64_t c = 0; c < nc; ++c) {
      chunk_entry[m][(size_t)c] = e;
      // entries per chunk: meta, [gtab], slots, [coef]
      const int64_t p0 = chunk_p0[(size_t)c], p1 = chunk_p0[(size_t)c + 1];
      const int64_t g0 = vg[(size_t)d->pair_visit[p0]], g1 = vg[(size_t)d->pair_visit[p1 - 1] + 1];
      e += 2 + (g1 > g0 ? 1 : 0) + (m > 0 ? 1 : 0);
    }
    chunk_entry[m][(size_t)nc] = e;
  }
  // balance the parts by pairs (chunks cut by the stage size hold fewer)
  for (int64_t b = 0, c = 0; b <= parts; ++b) {
    const int64_t target = b * np / parts;
    while (c < nc && chunk_p0[(size_t)c] < target) ++c;
    pcs[(size_t)b] = b == parts ? nc : c;
    for (int m = 0; m < 3; ++m) pes[m][(size_t)b] = chunk_entry[m][(size_t)pcs[(size_t)b]];
  }
  int rc = BMV_OK;
  sp->n = N;
  sp->xpf = xpf;
  sp->n_chunks = nc;
  sp->n_parts = (int)parts;
  sp->n_stages = ns;
  sp->stage_bytes = stage_bytes;
  sp->smem_bytes = warp_total + ns * stage_bytes;
  sp->q3p = Q3P;
  sp->off_gtab = off_gtab;
  if (rc == BMV_OK) rc = upload(pcs.data(), parts + 1, &sp->part_chunk_start);
  for (int m = 0; m < 3 && rc == BMV_OK; ++m) {
    rc = upload(pes[m].data(), parts + 1, &sp->part_entry_start[m]);
    if (rc == BMV_OK)
      rc = upload(reinterpret_cast<const int4*>(cps[m].data()), (int64_t)cps[m].size() / 4,
                  &sp->copies[m]);
  }
  if (rc == BMV_OK) rc = upload(meta.data(), (int64_t)meta.size(), &sp->meta);
  if (rc == BMV_OK)
    rc = upload(reinterpret_cast<const int2*>(gxh.data()), (int64_t)gxh.size() / 2, &sp->gtab);
  if (rc == BMV_OK) rc = upload(sl16.data(), (int64_t)sl16.size(), &sp->slots);
  return rc;
}

template <int N, bool XPF, bool COEF>
int launch_stream(const StreamPlan* sp, const CellTables& tb, const double* coef, int coef_cell,
                  const double* x, double* hx, cudaStream_t st) {
  auto kern = cellop_stream_kernel<N, XPF, COEF>;
  BMV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    sp->smem_bytes));
  const int m = COEF ? (coef_cell ? 1 : 2) : 0;
  StreamArgs a{};
  a.part_chunk_start = sp->part_chunk_start;
  a.part_entry_start = sp->part_entry_start[m];
  a.copies = sp->copies[m];
  a.src = CopySrc{reinterpret_cast<const char*>(sp->meta), reinterpret_cast<const char*>(sp->gtab),
                  reinterpret_cast<const char*>(sp->slots), reinterpret_cast<const char*>(coef)};
  a.x = x;
  a.hx = hx;
  a.stage_bytes = sp->stage_bytes;
  a.n_stages = sp->n_stages;
  a.off_gtab = sp->off_gtab;
  a.coef_cell = coef_cell;
  kern<<<sp->n_parts, (StreamShape<N>::NW + 1) * 32, sp->smem_bytes, st>>>(a, tb);
  BMV_CHECK_LAUNCH();
  return BMV_OK;
}

template <int N>
int launch_n(const StreamPlan* sp, const CellTables& tb, const double* coef, int coef_cell,
             const double* x, double* hx, cudaStream_t st) {
  if (sp->xpf)
    return coef ? launch_stream<N, true, true>(sp, tb, coef, coef_cell, x, hx, st)
                : launch_stream<N, true, false>(sp, tb, coef, coef_cell, x, hx, st);
  return coef ? launch_stream<N, false, true>(sp, tb, coef, coef_cell, x, hx, st)
              : launch_stream<N, false, false>(sp, tb, coef, coef_cell, x, hx, st);
}

}  // namespace

int stream_plan_build(const bmv_cellop_desc* d, StreamPlan** out) {
  *out = nullptr;
  // opt-in (BMV_K1=stream): measured slower than the one-pass kernel on Q4
  // (smem-pipe bound)
  const char* env = std::getenv("BMV_K1");
  if (!env || std::string(env) != "stream") return BMV_OK;
  if (d->n_colors > 0 || d->n_pairs == 0) return BMV_OK;
  const char* xe = std::getenv("BMV_K1_XPF");
  const bool xpf = !(xe && xe[0] == '0');
  auto* sp = new StreamPlan();
  int rc = -1;
  switch (d->n) {
    case 2: rc = build_plan_n<2>(d, xpf, sp); break;
    case 3: rc = build_plan_n<3>(d, xpf, sp); break;
    case 4: rc = build_plan_n<4>(d, xpf, sp); break;
    case 5: rc = build_plan_n<5>(d, xpf, sp); break;
    default: break;
  }
  if (rc != BMV_OK) {
    stream_plan_destroy(sp);
    return rc < 0 ? BMV_OK : rc;  // -1: shape not streamable, keep the one-pass kernel
  }
  *out = sp;
  return BMV_OK;
}

void stream_plan_destroy(StreamPlan* sp) {
  if (!sp) return;
  release(sp->part_chunk_start);
  for (int m = 0; m < 3; ++m) {
    release(sp->part_entry_start[m]);
    release(sp->copies[m]);
  }
  release(sp->meta);
  release(sp->gtab);
  release(sp->slots);
  delete sp;
}

int stream_apply(const StreamPlan* sp, const CellTables& tb, const double* coef, int coef_cell,
                 const double* x, double* hx, cudaStream_t st) {
  switch (sp->n) {
    case 2: return launch_n<2>(sp, tb, coef, coef_cell, x, hx, st);
    case 3: return launch_n<3>(sp, tb, coef, coef_cell, x, hx, st);
    case 4: return launch_n<4>(sp, tb, coef, coef_cell, x, hx, st);
    case 5: return launch_n<5>(sp, tb, coef, coef_cell, x, hx, st);
    default:
      set_error("stream plan with unsupported n %d", sp->n);
      return BMV_ERR_INVALID;
  }
}

}  // namespace bmv
