// Blocked per-row triangular solves / products on shared-memory row panels (sm_100a, fp64):
// used by the CholeskyQR2 tail (cholqr.cuh) and the normal-equations tail (small_kernels.cuh).
#pragma once
#include "common.cuh"

namespace cpqr {

// ---- blocked row kernels -------------------------------------------------------------------
// Each thread owns one panel row in shared memory (stride ld).  A dependent LDS costs ~70 cycles
// on sm_100a, so the row is processed in 8-column chunks held in registers: one shared-memory
// round trip per 8x8 block instead of one per element.  Columns >= R are zero in the panel and
// in the (zero-padded) triangular factors, and invd[j] = 0 there, so they stay zero.

// In-place triangular solve on the row.  FWD: y U = x (U upper, invd = 1/U_jj), columns
// ascending.  BACK: sum_{l >= c} T(c, l) x_l = w_c (T upper, invd = 1/T_cc), i.e. x T^T = w,
// columns descending (the back substitution of Alg. 2 line 10).
template <int RB, bool BACK>
__device__ __noinline__ void cq_row_trsv(double* row, int ld, const double* T, const double* invd) {
  constexpr int NB = RB / 8;
#pragma unroll 1
  for (int s = 0; s < NB; ++s) {
    const int jb = BACK ? NB - 1 - s : s;
    const int j0 = 8 * jb;
    double y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = row[ld * (j0 + q)];
    if (BACK) {
#pragma unroll
      for (int q = 7; q >= 0; --q) {
#pragma unroll
        for (int p = q + 1; p < 8; ++p) y[q] = fma(-y[p], T[(j0 + q) + RB * (j0 + p)], y[q]);
        y[q] *= invd[j0 + q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
#pragma unroll
        for (int p = 0; p < q; ++p) y[q] = fma(-y[p], T[(j0 + p) + RB * (j0 + q)], y[q]);
        y[q] *= invd[j0 + q];
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) row[ld * (j0 + q)] = y[q];
#pragma unroll 1
    for (int t = s + 1; t < NB; ++t) {  // eliminate the solved chunk from the unsolved ones
      const int i0 = 8 * (BACK ? NB - 1 - t : t);
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = row[ld * (i0 + q)];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int p = 0; p < 8; ++p)
          a[q] = fma(-y[p], BACK ? T[(i0 + q) + RB * (j0 + p)] : T[(j0 + p) + RB * (i0 + q)], a[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) row[ld * (i0 + q)] = a[q];
    }
  }
}

// out_row = in_row M (M dense RB x RB col-major): the SVD-variant solve x = w U S^+ V^T
template <int RB>
__device__ __noinline__ void cq_row_gemv(const double* in, double* out, int ld, const double* M) {
  constexpr int NB = RB / 8;
#pragma unroll 1
  for (int ob = 0; ob < NB; ++ob) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = 0.0;
#pragma unroll 1
    for (int sb = 0; sb < NB; ++sb) {
      double w[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) w[p] = in[ld * (8 * sb + p)];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int p = 0; p < 8; ++p) a[q] = fma(w[p], M[(8 * sb + p) + RB * (8 * ob + q)], a[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) out[ld * (8 * ob + q)] = a[q];
  }
}

// <w, T x> for the row pair (T upper): the per-row term of <W, Ahat R0^T>
template <int RB>
__device__ __noinline__ double cq_row_wTx(const double* w, const double* x, int ld, const double* T) {
  constexpr int NB = RB / 8;
  double inner = 0.0;
#pragma unroll 1
  for (int cb = 0; cb < NB; ++cb) {
    double t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = 0.0;
#pragma unroll 1
    for (int lb = cb; lb < NB; ++lb) {
      double xv[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) xv[p] = x[ld * (8 * lb + p)];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int p = 0; p < 8; ++p) t[q] = fma(T[(8 * cb + q) + RB * (8 * lb + p)], xv[p], t[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) inner = fma(w[ld * (8 * cb + q)], t[q], inner);
  }
  return inner;
}

}  // namespace cpqr
