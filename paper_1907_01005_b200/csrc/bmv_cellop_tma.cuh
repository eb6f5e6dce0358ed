// K1 TMA-staged variant (bmv_cellop_tma.cu): shapes and the device plan.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "bmv.h"
#include "bmv_sumfac.cuh"

namespace bmv {

// Per nodes-per-axis N: P pairs per warp; per-pair shared rows of CS
// coefficients (>= Q3P = q^3 rounded to even) and SS slots (>= SRP = n^3
// rounded to 4), padded off the bank period (bank model in DESIGN.md 4);
// MINB CTAs of 4 warps per SM.
template <int N>
struct TmaShape {
  static constexpr int P = 32 / N;
  static constexpr int N3 = N * N * N;
  static constexpr int Q3P = (N3 + 1) / 2 * 2;
  static constexpr int SRP = (N3 + 3) / 4 * 4;
  static constexpr int CS = N == 5 ? 134 : (N == 4 ? 66 : (N == 3 ? 28 : 10));
  static constexpr int SS = N == 5 ? 132 : (N == 4 ? 68 : SRP);
  static constexpr int MINB = N == 5 ? 3 : (N == 4 ? 4 : (N == 3 ? 5 : 8));
  static constexpr int tile_bytes0 = (P * Tile<N>::TILE * 8 + 15) / 16 * 16;
  // the X offset rows overlay the tiles
  static constexpr int tile_bytes = tile_bytes0 > P * SS * 4 ? tile_bytes0 : P * SS * 4;
  static constexpr int coef_bytes = P * CS * 8;
  static constexpr int hoff_bytes = P * SS * 4;
  static constexpr int warp_bytes = tile_bytes + coef_bytes + hoff_bytes;
};

struct TmaPlan {
  int n = 0;
  int64_t n_pairs = 0;
  int q3p = 0;
  bool per_pair = false;  // n <= 3: thread-per-pair kernel (BMV_K1_PAIR=0 disables)
  int4* desc = nullptr;
  int32_t* xoff = nullptr;
  int32_t* hoff = nullptr;
};

// Built from the one-pass descriptor; *out stays null when not applicable
// (colour mode, BMV_K1 selecting another kernel, > 32 groups per visit).
int tma_plan_build(const bmv_cellop_desc* d, TmaPlan** out);
void tma_plan_destroy(TmaPlan* tp);
// hx[0:zero_len] = 0, then hx += H x; coef: null, per cell (coef_cell = 1,
// row stride q3p) or one row (coef_cell = 0).
int tma_apply(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
              const double* x, double* hx, int64_t zero_len, cudaStream_t st);
// Fused: hx = H x and mx = M x (mass coefficient row mcoef = w3), hx and mx on
// the same pattern (same offsets), both zeroed over [0, zero_len) first.
int tma_apply_hm(const TmaPlan* tp, const CellTables& tb, const double* coef, int coef_cell,
                 const double* mcoef, const double* x, double* hx, double* mx, int64_t zero_len,
                 cudaStream_t st);

}  // namespace bmv
