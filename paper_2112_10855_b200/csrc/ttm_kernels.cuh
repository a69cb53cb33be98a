// Multi-TTM kernels (Alg. 2 line 8; Eq. (2.2)) on FP64 tensor
// cores (DMMA m8n8k4), sm_100a.  Three shapes cover every TTM of the hot path:
//
//   k_ttm_strided  T(a, r, b) = sum_i X(a, i, b) Q(i, r)      TTM on a mode k > 1: a = modes < k
//                  (contiguous), i = mode k (stride A), b = modes > k.  X is the MMA A operand.
//   k_ttm_fiber    T(r, f)    = sum_i Q(i, r) X(i, f)         TTM on mode 1: i runs along the
//                  contiguous mode-1 fibers f.  X is the MMA B operand.
//   k_mttm_slice   Y(r1,r2,l) = sum_{i1,i2} Q1(i1,r1) Q2(i2,r2) X(i1,i2,l)
//                  the two fastest modes contracted in ONE pass over X (no intermediate in HBM):
//                  the first contraction's accumulator fragment IS the A fragment of the second
//                  (k-permutation below), so the chain is DMMA -> DMMA with no data movement.
//
// X is streamed once from HBM straight into registers with 16-byte evict-first loads, software-
// pipelined one stage ahead; the small Q_k panels are staged in shared memory (chunked along K
// when they exceed the budget) and read as conflict-free 8-byte fragments.
//
// DMMA fragment map (lane = 4g + t): a = A[g][t], b = B[t][g], d0 = D[g][2t], d1 = D[g][2t+1].
// The K index of an MMA is a free labelling: with 16-byte loads a lane holds two consecutive
// elements, which become k-step s = 0/1 of "logical k = t" <-> "physical k = 2t + s".  Both
// operands of the MMA use the same labelling, so the product is unchanged.
#pragma once
#include "common.cuh"

namespace cpqr {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

// ----------------------------------------------------------------------------------------
// Shared-memory staging of a K-chunk of Q (rows [c0, c0+KC) of the I x R column-major matrix
// with leading dimension ldq) into Qs[row][LD], zero-padded beyond I and beyond R.
__device__ __forceinline__ void stage_q(double* Qs, const double* __restrict__ Q, int64_t ldq,
                                        int I, int R, int c0, int KC, int LD) {
  const int n = KC * LD;
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int row = idx / LD, col = idx - row * LD;
    const int i = c0 + row;
    Qs[idx] = (i < I && col < R) ? __ldg(Q + i + ldq * col) : 0.0;
  }
}

// ======================================================================= k_ttm_strided
// MT M-tiles of 8 rows per warp (VEC: rows 16p + 2g + s, tile 2p + s), NT = ceil(R/8) N-tiles.
// LD = 8 NT + 4: B-fragment reads Qs[t*LD + 8nt + g] hit 16 distinct 8-byte banks per half-warp.
template <int MT, int NT, bool VEC>
__global__ void __launch_bounds__(kThreads)
k_ttm_strided(const double* __restrict__ X, int64_t A, int I, int64_t B,
              const double* __restrict__ Q, int64_t ldq, int R, double* __restrict__ T, int KC) {
  extern __shared__ double Qs[];
  constexpr int LD = 8 * NT + 4;
  constexpr int KU = 4;  // k-steps (of 4) per pipeline stage
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t BMc = (int64_t)kWarps * 8 * MT;
  const int64_t nA = (A + BMc - 1) / BMc;
  const int64_t units = nA * B;
  const int nchunk = (I + KC - 1) / KC;
  if (nchunk == 1) {
    stage_q(Qs, Q, ldq, I, R, 0, KC, LD);
    __syncthreads();
  }
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t b = u / nA, ablk = u - b * nA;
    const int64_t a0 = ablk * BMc + (int64_t)warp * 8 * MT;
    const double* __restrict__ Xb = X + A * (int64_t)I * b;
    // row handled by this lane for tile mt
    int64_t rowp[VEC ? MT / 2 : MT];
    bool rowok[VEC ? MT / 2 : MT];
    if (VEC) {
#pragma unroll
      for (int p = 0; p < MT / 2; ++p) { rowp[p] = a0 + 16 * p + 2 * g; rowok[p] = rowp[p] < A; }
    } else {
#pragma unroll
      for (int m = 0; m < MT; ++m) { rowp[m] = a0 + 8 * m + g; rowok[m] = rowp[m] < A; }
    }
    double acc[MT][NT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * KC, c1 = min(I, c0 + KC);
      if (nchunk > 1) {
        __syncthreads();
        stage_q(Qs, Q, ldq, I, R, c0, KC, LD);
        __syncthreads();
      }
      double xc[KU][MT], xn[KU][MT];
      auto load = [&](double (&xs)[KU][MT], int i0) {
#pragma unroll
        for (int ku = 0; ku < KU; ++ku) {
          const int i = i0 + 4 * ku + t;
          const bool iok = i < c1;
          if (VEC) {
#pragma unroll
            for (int p = 0; p < MT / 2; ++p) {
              double2 v = make_double2(0.0, 0.0);
              if (iok && rowok[p]) v = ldg_stream2(Xb + rowp[p] + A * (int64_t)i);
              xs[ku][2 * p] = v.x;
              xs[ku][2 * p + 1] = v.y;
            }
          } else {
#pragma unroll
            for (int m = 0; m < MT; ++m)
              xs[ku][m] = (iok && rowok[m]) ? ldg_stream1(Xb + rowp[m] + A * (int64_t)i) : 0.0;
          }
        }
      };
      load(xc, c0);
      for (int i0 = c0; i0 < c1; i0 += 4 * KU) {
        if (i0 + 4 * KU < c1) load(xn, i0 + 4 * KU);
#pragma unroll
        for (int ku = 0; ku < KU; ++ku) {
          const int ir = i0 + 4 * ku - c0 + t;  // row inside the chunk (Qs zero-padded)
          if (i0 + 4 * ku < c1) {
            double qb[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) qb[n] = Qs[ir * LD + 8 * n + g];
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
              for (int n = 0; n < NT; ++n) dmma(acc[m][n][0], acc[m][n][1], xc[ku][m], qb[n]);
          }
        }
#pragma unroll
        for (int ku = 0; ku < KU; ++ku)
#pragma unroll
          for (int m = 0; m < MT; ++m) xc[ku][m] = xn[ku][m];
      }
    }
    // epilogue: T(a, r, b), a + A r + A R b
    double* __restrict__ Tb = T + A * (int64_t)R * b;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t row = VEC ? (a0 + 16 * (m >> 1) + 2 * g + (m & 1)) : (a0 + 8 * m + g);
      if (row >= A) continue;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int r0 = 8 * n + 2 * t;
        if (r0 < R) Tb[row + A * r0] = acc[m][n][0];
        if (r0 + 1 < R) Tb[row + A * (r0 + 1)] = acc[m][n][1];
      }
    }
  }
}

// ========================================================================= k_ttm_fiber
// MT = ceil(R/8) M-tiles (the r index), NF N-tiles of 8 fibers per warp.  A fragments (Q) from
// shared memory, B fragments (X fibers) from HBM.  One "kk" step covers 8 consecutive i:
//   VEC: lane loads X(i0+2t .. i0+2t+1, f) (16 B); k-step s uses i = i0 + 2t + s.  LD = 8MT+2.
//   scalar: k-step s uses i = i0 + 4s + t.                                        LD = 8MT+4.
template <int MT, int NF, bool VEC>
__global__ void __launch_bounds__(kThreads)
k_ttm_fiber(const double* __restrict__ X, int I, int64_t F, const double* __restrict__ Q,
            int64_t ldq, int R, double* __restrict__ T, int KC) {
  extern __shared__ double Qs[];
  constexpr int LD = 8 * MT + (VEC ? 2 : 4);
  constexpr int KU = 2;  // kk steps (8 i each) per pipeline stage
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t BF = (int64_t)kWarps * 8 * NF;
  const int64_t units = (F + BF - 1) / BF;
  const int nchunk = (I + KC - 1) / KC;
  if (nchunk == 1) {
    stage_q(Qs, Q, ldq, I, R, 0, KC, LD);
    __syncthreads();
  }
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t f0 = u * BF + (int64_t)warp * 8 * NF;
    int64_t fb[NF];
    bool fok[NF];
#pragma unroll
    for (int n = 0; n < NF; ++n) { fb[n] = f0 + 8 * n + g; fok[n] = fb[n] < F; }
    double acc[MT][NF][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NF; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * KC, c1 = min(I, c0 + KC);
      if (nchunk > 1) {
        __syncthreads();
        stage_q(Qs, Q, ldq, I, R, c0, KC, LD);
        __syncthreads();
      }
      double xc[KU][NF][2], xn[KU][NF][2];
      auto load = [&](double (&xs)[KU][NF][2], int i0) {
#pragma unroll
        for (int ku = 0; ku < KU; ++ku) {
          const int ib = i0 + 8 * ku;
#pragma unroll
          for (int n = 0; n < NF; ++n) {
            if (VEC) {
              const int i = ib + 2 * t;
              double2 v = make_double2(0.0, 0.0);
              if (fok[n] && i < c1) v = ldg_stream2(X + fb[n] * I + i);
              xs[ku][n][0] = v.x;
              xs[ku][n][1] = v.y;
            } else {
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                const int i = ib + 4 * s + t;
                xs[ku][n][s] = (fok[n] && i < c1) ? ldg_stream1(X + fb[n] * I + i) : 0.0;
              }
            }
          }
        }
      };
      load(xc, c0);
      for (int i0 = c0; i0 < c1; i0 += 8 * KU) {
        if (i0 + 8 * KU < c1) load(xn, i0 + 8 * KU);
#pragma unroll
        for (int ku = 0; ku < KU; ++ku) {
          const int ib = i0 + 8 * ku - c0;
          if (i0 + 8 * ku < c1) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int ir = VEC ? (ib + 2 * t + s) : (ib + 4 * s + t);
              double qa[MT];
#pragma unroll
              for (int m = 0; m < MT; ++m) qa[m] = Qs[ir * LD + 8 * m + g];
#pragma unroll
              for (int m = 0; m < MT; ++m)
#pragma unroll
                for (int n = 0; n < NF; ++n) dmma(acc[m][n][0], acc[m][n][1], qa[m], xc[ku][n][s]);
            }
          }
        }
#pragma unroll
        for (int ku = 0; ku < KU; ++ku)
#pragma unroll
          for (int n = 0; n < NF; ++n) { xc[ku][n][0] = xn[ku][n][0]; xc[ku][n][1] = xn[ku][n][1]; }
      }
    }
    // epilogue: T(r, f) at r + R f; d_s = T(8m + g, f0 + 8n + 2t + s)
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int r = 8 * m + g;
      if (r >= R) continue;
#pragma unroll
      for (int n = 0; n < NF; ++n)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int64_t f = f0 + 8 * n + 2 * t + s;
          if (f < F) T[r + (int64_t)R * f] = acc[m][n][s];
        }
    }
  }
}

// ========================================================================= k_mttm_slice
// X viewed as (I1, I2, L).  Fibers of slice l are grouped into groups of FW = 8 NF fibers;
// GPS consecutive groups form one warp-unit ("segment"); nseg = ceil(ceil(I2/FW)/GPS).
// Warp-unit u = l * nseg + seg accumulates Y over its segment in registers and writes it to
// P[u] (R x R, r1 + R r2) -- or straight to Y[l] when nseg == 1.  A CTA owns warp-units
// [kWarps*blk, kWarps*blk + kWarps).  Deterministic: every partial is summed by
// k_reduce_slices in a fixed order.
template <int MT, int NF, bool VEC>
__global__ void __launch_bounds__(kThreads)
k_mttm_slice(const double* __restrict__ X, int I1, int I2, int64_t L,
             const double* __restrict__ Q1, int64_t ldq1, const double* __restrict__ Q2,
             int64_t ldq2, int R, int GPS, double* __restrict__ out, int KC) {
  extern __shared__ double Qs[];
  constexpr int LD = 8 * MT + (VEC ? 2 : 4);
  constexpr int KU = 2;
  constexpr int FW = 8 * NF;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ngr = (I2 + FW - 1) / FW;
  const int nseg = (ngr + GPS - 1) / GPS;
  const int64_t wunits = (int64_t)nseg * L;
  const int64_t cunits = (wunits + kWarps - 1) / kWarps;
  const int nchunk = (I1 + KC - 1) / KC;
  const int64_t strideL = (int64_t)I1 * I2;
  if (nchunk == 1) {
    stage_q(Qs, Q1, ldq1, I1, R, 0, KC, LD);
    __syncthreads();
  }
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    const int64_t wu = cu * kWarps + warp;
    const bool wactive = wu < wunits;
    const int64_t l = wactive ? wu / nseg : 0;
    const int seg = wactive ? (int)(wu - l * nseg) : 0;
    const double* __restrict__ Xl = X + strideL * l;
    double yacc[MT][MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < MT; ++n) yacc[m][n][0] = yacc[m][n][1] = 0.0;

    for (int gl = 0; gl < GPS; ++gl) {
      const int gi = seg * GPS + gl;
      const bool gactive = wactive && gi < ngr;
      const int i2base = gi * FW;
      int fb[NF];
      bool fok[NF];
#pragma unroll
      for (int n = 0; n < NF; ++n) { fb[n] = i2base + 8 * n + g; fok[n] = gactive && fb[n] < I2; }
      double acc[MT][NF][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NF; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
      for (int c = 0; c < nchunk; ++c) {
        const int c0 = c * KC, c1 = min(I1, c0 + KC);
        if (nchunk > 1) {
          __syncthreads();
          stage_q(Qs, Q1, ldq1, I1, R, c0, KC, LD);
          __syncthreads();
        }
        if (!gactive) continue;
        double xc[KU][NF][2], xn[KU][NF][2];
        auto load = [&](double (&xs)[KU][NF][2], int i0) {
#pragma unroll
          for (int ku = 0; ku < KU; ++ku) {
            const int ib = i0 + 8 * ku;
#pragma unroll
            for (int n = 0; n < NF; ++n) {
              if (VEC) {
                const int i = ib + 2 * t;
                double2 v = make_double2(0.0, 0.0);
                if (fok[n] && i < c1) v = ldg_stream2(Xl + (int64_t)fb[n] * I1 + i);
                xs[ku][n][0] = v.x;
                xs[ku][n][1] = v.y;
              } else {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                  const int i = ib + 4 * s + t;
                  xs[ku][n][s] = (fok[n] && i < c1) ? ldg_stream1(Xl + (int64_t)fb[n] * I1 + i) : 0.0;
                }
              }
            }
          }
        };
        load(xc, c0);
        for (int i0 = c0; i0 < c1; i0 += 8 * KU) {
          if (i0 + 8 * KU < c1) load(xn, i0 + 8 * KU);
#pragma unroll
          for (int ku = 0; ku < KU; ++ku) {
            const int ib = i0 + 8 * ku - c0;
            if (i0 + 8 * ku < c1) {
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                const int ir = VEC ? (ib + 2 * t + s) : (ib + 4 * s + t);
                double qa[MT];
#pragma unroll
                for (int m = 0; m < MT; ++m) qa[m] = Qs[ir * LD + 8 * m + g];
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                  for (int n = 0; n < NF; ++n) dmma(acc[m][n][0], acc[m][n][1], qa[m], xc[ku][n][s]);
              }
            }
          }
#pragma unroll
          for (int ku = 0; ku < KU; ++ku)
#pragma unroll
            for (int n = 0; n < NF; ++n) { xc[ku][n][0] = xn[ku][n][0]; xc[ku][n][1] = xn[ku][n][1]; }
        }
      }
      if (gactive) {
        // second contraction: Y(r1, r2) += sum_{i2 in group} T(r1, i2) Q2(i2, r2).
        // acc[m][n][s] = T(r1 = 8m+g, i2 = i2base + 8n + 2t + s) is exactly A[g][t] of the k-step
        // labelled (n, s); its B fragment is Q2(i2base + 8n + 2t + s, 8m2 + g).
#pragma unroll
        for (int n = 0; n < NF; ++n)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int i2 = i2base + 8 * n + 2 * t + s;
            double qb[MT];
#pragma unroll
            for (int m2 = 0; m2 < MT; ++m2) {
              const int r2 = 8 * m2 + g;
              qb[m2] = (i2 < I2 && r2 < R) ? __ldg(Q2 + i2 + ldq2 * r2) : 0.0;
            }
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
              for (int m2 = 0; m2 < MT; ++m2) dmma(yacc[m][m2][0], yacc[m][m2][1], acc[m][n][s], qb[m2]);
          }
      }
    }
    if (wactive) {
      double* __restrict__ o = out + (int64_t)R * R * wu;  // nseg == 1: wu == l
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r1 = 8 * m + g;
        if (r1 >= R) continue;
#pragma unroll
        for (int m2 = 0; m2 < MT; ++m2)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int r2 = 8 * m2 + 2 * t + s;
            if (r2 < R) o[r1 + R * r2] = yacc[m][m2][s];
          }
      }
    }
  }
}

// Y[l][e] = sum_{seg < nseg} P[l*nseg + seg][e], e < R^2, fixed order.
__global__ void k_reduce_slices(const double* __restrict__ P, int nseg, int64_t L, int RR,
                                double* __restrict__ Y) {
  const int64_t n = L * RR;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = idx / RR, e = idx - l * RR;
    const double* p = P + (l * nseg) * RR + e;
    double s = 0.0;
    for (int k = 0; k < nseg; ++k) s += p[(int64_t)k * RR];
    Y[idx] = s;
  }
}

}  // namespace cpqr
