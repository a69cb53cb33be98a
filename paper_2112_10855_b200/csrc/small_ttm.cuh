// The remaining TTMs of the Multi-TTM (Alg. 2 line 8; decreasing-dimension order,
// PAPER.md:387) on the intermediates the stream-X pass leaves behind:
//
//   T(a, r, b) = sum_i X(a, i, b) Q(i, r),   X (A, I, B) and T (A, R, B) column-major.
//
// Rows m = a + A b (M = A B): X(m, i) = X[off(m) + A i] with off(m) = a + A I b, and T(m, r) =
// T[a + A R b + A r]; A = 1 is the mode-1 (fibre) TTM of the same formula.  These inputs are
// (R / I_k) times smaller than X (C2: 12.8 MB, C3: 33.5 MB) and were just written, so they sit in the
// 126 MB L2: the pass is bound by latency and parallelism, not by HBM.  The TMA stream kernels'
// units of 128-256 rows x the whole contraction leave most SMs idle on them (C2 mode 1: 32 units for
// 4000 rows; 13-27 us for 32 MFLOP), so this kernel cuts the work finer:
//   * 16-row tiles (two DMMA m8n8k4 M-tiles, FP64 tensor cores) x NT = ceil(R/8) N-tiles;
//   * the contraction split over WK warps of a CTA (WM = 8 / WK row tiles per CTA) and over KC
//     CTAs, chosen on the host so that ~8 warps x 2 CTAs per SM have work;
//   * the WK warp partials are summed through shared memory in warp order, the KC CTA partials by
//     the last CTA to arrive (arrival counter per row block, self re-arming) in CTA order: fixed
//     order, bitwise reproducible, and no extra launch.
// X fragments come straight from global memory (L2) into registers, four k-steps of loads in
// flight per lane; Q fragments from the transposed zero-padded panel Qt (I x RQ, RQ >= 8 NT), which
// every warp of an SM reads and so stays in L1 (staging it in shared memory per CTA cost more L2
// traffic than X itself at R / 16 of the rows' bytes per 16-row tile).
#pragma once
#include "common.cuh"

namespace cpqr {

template <int NT>
__global__ void __launch_bounds__(256) k_ttm_small(const double* __restrict__ X, int64_t A, int I, int64_t B,
                                                    const double* __restrict__ Qt, int RQ, int R,
                                                    double* __restrict__ T, int WK, int KC,
                                                    double* __restrict__ P, unsigned* __restrict__ cnt) {
  extern __shared__ double red[];  // WK x RT x (8 NT + 1) warp partials (odd stride: conflict free)
  __shared__ int last;
  constexpr int KU = 4;            // k-steps (of 4) of loads in flight per lane
  constexpr int LDR = 8 * NT + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int WM = 8 / WK, wm = warp % WM, wk = warp / WM;
  const int RT = 16 * WM;  // rows per CTA
  const int64_t M = A * B;
  const int64_t rc = blockIdx.x / KC;
  const int kc = blockIdx.x - (int)(rc * KC);
  const int i0 = (int)((int64_t)I * kc / KC), i1 = (int)((int64_t)I * (kc + 1) / KC), KL = i1 - i0;
  pdl_wait();
  // the warp's two 8-row M-tiles (rows past M read row M-1 and are never stored) and its k-steps
  // (32-bit element offsets: the planner keeps A I B <= kSmallTtmMax = 2^23)
  const int64_t m0 = rc * RT + 16 * wm;
  const int nks = (KL + 3) >> 2;            // k-steps of the CTA range (the last one may be ragged)
  const int ks0 = nks * wk / WK, ks1 = nks * (wk + 1) / WK;
  const int ksf = min(ks1, KL >> 2);        // k-steps entirely inside the range: no masks
  const int xs = 4 * (int)A, qs = 4 * RQ;
  int xo[2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int m = (int)min(m0 + 8 * mt + g, M - 1);
    const int b = m / (int)A, a = m - b * (int)A;
    xo[mt] = a + (int)A * (I * b + i0 + t) + ks0 * xs;
  }
  int qo = (i0 + t) * RQ + g + ks0 * qs;
  double acc[2][NT][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[mt][n][0] = acc[mt][n][1] = 0.0;
  auto mma = [&](const double (&xv)[2], const double (&qv)[NT]) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      dmma(acc[0][n][0], acc[0][n][1], xv[0], qv[n]);
      dmma(acc[1][n][0], acc[1][n][1], xv[1], qv[n]);
    }
  };
  // B fragments straight from the transposed zero-padded panel Qt (I x RQ row-major, L1 resident:
  // every warp of the SM reads the same rows); A fragments (X) from L2, KU k-steps in flight
  int ks = ks0;
  for (; ks + KU <= ksf; ks += KU) {
    double xv[KU][2], qv[KU][NT];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      xv[u][0] = __ldcg(X + xo[0]);
      xv[u][1] = __ldcg(X + xo[1]);
#pragma unroll
      for (int n = 0; n < NT; ++n) qv[u][n] = __ldg(Qt + qo + 8 * n);
      xo[0] += xs;
      xo[1] += xs;
      qo += qs;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) mma(xv[u], qv[u]);
  }
  for (; ks < ks1; ++ks) {  // the last < KU k-steps; only the CTA range's final one is ragged
    const bool kin = 4 * ks + t < KL;
    double xv[2], qv[NT];
    xv[0] = kin ? __ldcg(X + xo[0]) : 0.0;
    xv[1] = kin ? __ldcg(X + xo[1]) : 0.0;
#pragma unroll
    for (int n = 0; n < NT; ++n) qv[n] = kin ? __ldg(Qt + qo + 8 * n) : 0.0;
    xo[0] += xs;
    xo[1] += xs;
    qo += qs;
    mma(xv, qv);
  }
  // warp partials -> red[wk][row][col], row = 16 wm + 8 mt + g, col = 8 n + 2 t + s
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      double* d = red + ((size_t)wk * RT + 16 * wm + 8 * mt + g) * LDR + 8 * n + 2 * t;
      d[0] = acc[mt][n][0];
      d[1] = acc[mt][n][1];
    }
  __syncthreads();
  // one thread per row (consecutive rows -> consecutive a: coalesced stores), two per row when
  // RT = 128 (halves of the columns)
  const int nper = (RT >= 256) ? 1 : 256 / RT;  // threads per row
  const int row = threadIdx.x / nper, part = threadIdx.x % nper;
  const int64_t m = rc * RT + row;
  const int cb = R * part / nper, ce = R * (part + 1) / nper;
  int64_t tb = 0;
  if (m < M) {
    const int64_t b = m / A, a = m - b * A;
    tb = a + A * (int64_t)R * b;
  }
  if (KC == 1) {
    if (m < M)
      for (int col = cb; col < ce; ++col) {
        double v = 0.0;
        for (int w = 0; w < WK; ++w) v += red[((size_t)w * RT + row) * LDR + col];
        T[tb + A * col] = v;
      }
    return;
  }
  const int nent = RT * R;
  double* Pc = P + ((size_t)rc * KC + kc) * nent;
  for (int col = cb; col < ce; ++col) {
    double v = 0.0;
    for (int w = 0; w < WK; ++w) v += red[((size_t)w * RT + row) * LDR + col];
    Pc[col * RT + row] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&cnt[rc], 1u) == (unsigned)(KC - 1)) ? 1 : 0;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (m < M)
    for (int col = cb; col < ce; ++col) {
      double v = 0.0;
      for (int q = 0; q < KC; ++q) v += __ldcg(P + ((size_t)rc * KC + q) * nent + col * RT + row);
      T[tb + A * col] = v;
    }
  if (threadIdx.x == 0) cnt[rc] = 0u;  // re-armed for the next launch (graph replay)
}

}  // namespace cpqr
