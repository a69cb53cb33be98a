// Kruskal-tensor input: X = [[lam_x; B_1..B_N]] of rank S
// is never formed.  For mode n the Multi-TTM result is the Kruskal tensor
// Y = [[lam_x; C_1, .., B_n, .., C_N]] with C_k = Q_k^T B_k (R x S), so
//   W_n = Y_(n) Q0 = B_n diag(lam_x) [ (C_{k_{N-1}} (.) .. (.) C_{k_1})^T Q0 ]
// (Khatri-Rao in the Kolda-Bader order of V_n's rows: k_1 < .. < k_{N-1} the modes != n, the
// smallest mode's index fastest), at cost O(R^N S + I_n R S).  For normal-equations CP-ALS the
// MTTKRP is M_n = B_n diag(lam_x) (*)_{k != n} (B_k^T A_k), and
// ||X||^2 = lam_x^T ((*)_k B_k^T B_k) lam_x.  All reductions are fixed-order.
#pragma once
#include "common.cuh"

namespace cpqr {

constexpr int kKtMaxModes = 8;

struct KtCrossArgs {
  const double* P[kKtMaxModes];  // I_k x np, column-major
  const double* B[kKtMaxModes];  // I_k x nb, column-major
  int64_t I[kKtMaxModes];
  int K, np, nb;
  double* out;                   // K blocks of np x nb (column-major), block k at out + k np nb
};

// out_k = P_k^T B_k: one warp per entry (lanes stride over i), warp_sum in a fixed order.
__global__ void __launch_bounds__(256) k_kt_cross(KtCrossArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t per = (int64_t)a.np * a.nb;
  if (w >= per * a.K) return;  // whole warps
  const int k = (int)(w / per);
  const int64_t e = w - k * per;
  const int p = (int)(e % a.np), q = (int)(e / a.np);
  const double* x = a.P[k] + a.I[k] * p;
  const double* y = a.B[k] + a.I[k] * q;
  double s = 0.0;
  for (int64_t i = lane; i < a.I[k]; i += 32) s = fma(x[i], y[i], s);
  s = warp_sum(s);
  if (lane == 0) a.out[k * per + e] = s;
}

// M(s, r) = sum_j Q0(j, r) prod_m C_m(j_m, s), j = sum_m j_m R^m (C_m: R x S block m of C).
// One CTA per term s; threads stride over the J = R^{N1} rows; per-warp then per-CTA sums in order.
template <int RB>
__global__ void __launch_bounds__(256) k_kt_m(const double* __restrict__ C, int N1, int R, int S, int64_t J,
                                              const double* __restrict__ Q0, double* __restrict__ M) {
  __shared__ double red[8][RB];
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.0;
  for (int64_t j = tid; j < J; j += blockDim.x) {
    int64_t x = j;
    double p = 1.0;
    for (int m = 0; m < N1; ++m) {
      const int jm = (int)(x % R);
      x /= R;
      p *= C[(int64_t)m * R * S + jm + (int64_t)R * s];
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (r < R) acc[r] = fma(p, Q0[j + J * r], acc[r]);
  }
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const double v = warp_sum(acc[r]);
    if (lane == 0) red[wid][r] = v;
  }
  __syncthreads();
  if (tid < R) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w][tid];
    M[s + (int64_t)S * tid] = t;
  }
}

// W(i, r) = sum_s B_n(i, s) lam_x(s) M(s, r), W row-major I_n x R (the layout of the Q0 apply).
__global__ void k_kt_w(const double* __restrict__ Bn, int64_t In, int S, const double* __restrict__ lam,
                       const double* __restrict__ M, int R, double* __restrict__ W) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < In * R; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / R;
    const int r = (int)(e - i * R);
    double t = 0.0;
    for (int s = 0; s < S; ++s) t = fma(Bn[i + In * s] * lam[s], M[s + (int64_t)S * r], t);
    W[e] = t;
  }
}

// NE: M_n(i, r) = sum_s B_n(i, s) lam_x(s) prod_m Cx_m(s, r), Cx_m = B_k^T A_k (S x R), row-major out.
__global__ void k_kt_mttkrp(const double* __restrict__ Bn, int64_t In, int S, const double* __restrict__ lam,
                            const double* __restrict__ Cx, int N1, int R, double* __restrict__ Mout) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < In * R; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / R;
    const int r = (int)(e - i * R);
    double t = 0.0;
    for (int s = 0; s < S; ++s) {
      double h = lam[s];
      for (int m = 0; m < N1; ++m) h *= Cx[(int64_t)m * S * R + s + (int64_t)S * r];
      t = fma(Bn[i + In * s], h, t);
    }
    Mout[e] = t;
  }
}

// DIRECT residual of a Kruskal input: ||X - Xh||^2 with X = [[lam_x; B]] (rank S)
// and the model Xh = [[lam; A]] (rank R) evaluated entry by entry, never stored: the difference is
// the rank-(S + R) Kruskal tensor [[ (lam_x, -lam); (B_k | A_k) ]], so for one index tuple
// j = (i_2, .., i_N) of modes 2..N a warp forms p(s) = c_s prod_{k >= 2} C_k(i_k, s) in shared memory
// and then d(i_1) = sum_s C_1(i_1, s) p(s) for every i_1 (lanes), accumulating d^2.  Each entry's
// difference is formed before squaring, so the relative error resolves down to ~eps (the fast fit
// ||X||^2 - 2 <X, Xh> + ||Xh||^2 cancels to ~sqrt(eps)).  Fixed-order partials.
struct KtResidArgs {
  const double* B[kKtMaxModes];  // I_k x S
  const double* A[kKtMaxModes];  // I_k x R (normalised factors)
  int64_t I[kKtMaxModes];
  int N, S, R;
  const double* lamx;            // S
  const double* lam;             // R
  double* part;                  // gridDim.x partial sums
};
constexpr int kKtResidMaxSR = 512;
__global__ void __launch_bounds__(256) k_kt_resid(KtResidArgs a) {
  __shared__ double pw[8][kKtResidMaxSR];
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int SR = a.S + a.R;
  int64_t J = 1;
  for (int k = 1; k < a.N; ++k) J *= a.I[k];
  double acc = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * 8 + wid; j < J; j += (int64_t)gridDim.x * 8) {
    for (int s = lane; s < SR; s += 32) {
      const bool isx = s < a.S;
      const int q = isx ? s : s - a.S;
      double v = isx ? a.lamx[q] : -a.lam[q];
      int64_t x = j;
      for (int k = 1; k < a.N; ++k) {
        const int64_t ik = x % a.I[k];
        x /= a.I[k];
        v *= isx ? a.B[k][ik + a.I[k] * q] : a.A[k][ik + a.I[k] * q];
      }
      pw[wid][s] = v;
    }
    __syncwarp();
    for (int64_t i1 = lane; i1 < a.I[0]; i1 += 32) {
      double d = 0.0;
      for (int s = 0; s < a.S; ++s) d = fma(a.B[0][i1 + a.I[0] * s], pw[wid][s], d);
      for (int r = 0; r < a.R; ++r) d = fma(a.A[0][i1 + a.I[0] * r], pw[wid][a.S + r], d);
      acc = fma(d, d, acc);
    }
    __syncwarp();
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) a.part[blockIdx.x] = acc;
}

// ||X||^2 = sum_{s,t} lam(s) lam(t) prod_k G_k(s, t), G_k = B_k^T B_k (N blocks of S x S).
__global__ void __launch_bounds__(256) k_kt_norm2(const double* __restrict__ G, int N, int S,
                                                  const double* __restrict__ lam, double* __restrict__ out) {
  __shared__ double red[32];
  double v = 0.0;
  for (int e = threadIdx.x; e < S * S; e += blockDim.x) {
    double p = lam[e % S] * lam[e / S];
    for (int k = 0; k < N; ++k) p *= G[(int64_t)k * S * S + e];
    v += p;
  }
  v = block_sum(v, red);
  if (threadIdx.x == 0) *out = v;
}

}  // namespace cpqr
