// K1 streamed variant (bmv_cellop_stream.cu): shapes and the device plan.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bmv.h"
#include "bmv_sumfac.cuh"

namespace bmv {

// Per nodes-per-axis N: NW consumer warps (+1 producer) per CTA, CTAS CTAs
// per SM (register budget 65536 / (CTAS * 32 * (NW + 1))), P pairs per
// warp, SR 16-bit slots per staged cell row (16-byte multiple, skewed off
// a 128-byte period so neighbouring cells start on different banks), Q3P
// coefficients per cell row (16-byte multiple).
template <int N>
struct StreamShape {
  static constexpr int NW = 11;
  static constexpr int CTAS = N <= 3 ? 2 : 1;
  static constexpr int P = 32 / N;
  // the register file is split over the 4 SM sub-partitions (16384 each),
  // warps are placed round-robin: the busiest one holds ceil(warps / 4)
  static constexpr int WPS = (CTAS * (NW + 1) + 3) / 4;
  static constexpr int MAXREG = 16384 / (WPS * 32) / 8 * 8 > 255 ? 255 : 16384 / (WPS * 32) / 8 * 8;
  static constexpr int N3 = N * N * N;
  static constexpr int SR0 = (N3 + 7) / 8 * 8;
  static constexpr int SR = (SR0 / 2) % 32 == 0 ? SR0 + 8 : SR0;
  static constexpr int Q3P = (N3 + 1) / 2 * 2;
  static constexpr int tile_bytes = (P * Tile<N>::TILE * 8 + 15) / 16 * 16;
  static constexpr int xs_bytes = N * N * 32 * 8;
  static __host__ __device__ constexpr int warp_bytes(bool xpf) {
    return tile_bytes + (xpf ? xs_bytes : 0);
  }
};

struct StreamPlan {
  int n = 0;
  bool xpf = true;
  int64_t n_chunks = 0;
  int n_parts = 0;
  int n_stages = 0;
  int stage_bytes = 0;
  int smem_bytes = 0;
  int q3p = 0;
  int off_gtab = 0;
  int64_t* part_chunk_start = nullptr;
  int64_t* part_entry_start[3] = {nullptr, nullptr, nullptr};  // per coefficient mode
  int4* copies[3] = {nullptr, nullptr, nullptr};
  int32_t* meta = nullptr;
  int2* gtab = nullptr;
  uint16_t* slots = nullptr;
};

// Builds the streamed plan from the one-pass descriptor; *out stays null
// when the shape does not stream (colour mode, > 2047 rows per block, a
// chunk that does not fit a stage).
int stream_plan_build(const bmv_cellop_desc* d, StreamPlan** out);
void stream_plan_destroy(StreamPlan* sp);
// hx += H x over the plan's pairs (hx zeroed by the caller).  coef: null,
// per cell (coef_cell = 1, row stride q3p) or one row (coef_cell = 0).
int stream_apply(const StreamPlan* sp, const CellTables& tb, const double* coef, int coef_cell,
                 const double* x, double* hx, cudaStream_t st);

}  // namespace bmv
