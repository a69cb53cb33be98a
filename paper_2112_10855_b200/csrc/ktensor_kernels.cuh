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

constexpr int kKtMaxModes = kMaxModes;

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

// M(s, r) = sum_j Q0(j, r) prod_m C_m(j_m, s), j = sum_m j_m prod_{m' < m} rad_m' (C_m: R x S block
// m of C; rad_m = R, or min(I_k, R) for a short mode, whose C_m rows beyond it are zero).  CTA (s,
// ch) covers rows [ch J / NC, (ch+1) J / NC); threads stride over them; per-warp then per-CTA sums in
// order.  NC = 1 writes M directly; NC > 1 (V_n of 10^5+ rows, e.g. the 10-way sine of sums' 8^9)
// writes slot P[(s NC + ch) R + r], summed in chunk order by k_kt_m_reduce.
struct KtMArgs {
  const double* C;
  int N1, R, S, nc;
  int st;  // terms per CTA (<= kt_m_st): kt_m_st for a chunked (large) V_n, 1 for a small one
  int64_t J;
  int rad[kMaxModes];
  const double* Q0;
  double* M;
  double* P;
};
template <int RB>
__host__ __device__ constexpr int kt_m_st() { return RB <= 16 ? 4 : 2; }  // terms s per CTA (register budget)
template <int RB>
__global__ void __launch_bounds__(256) k_kt_m(KtMArgs a) {
  // CTA (s-tile, chunk): ST terms s share each pass over Q0's rows (Q0 is read S / ST times, not S);
  // rows go by groups of r0 = rad_0 (the fastest factor's digit), whose slow-factor product is
  // formed once per group and term
  constexpr int ST = kt_m_st<RB>();
  __shared__ double red[8][ST][RB];
  const int s0 = blockIdx.x * a.st, ch = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int send = min(a.S, s0 + a.st);
  const int nw = blockDim.x >> 5;
  const int R = a.R, S = a.S, r0 = a.rad[0];
  const int64_t JG = a.J / r0;
  const int64_t g0 = JG * ch / a.nc, g1 = JG * (ch + 1) / a.nc;
  double acc[ST][RB];
#pragma unroll
  for (int u = 0; u < ST; ++u)
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[u][r] = 0.0;
  for (int64_t grp = g0 + tid; grp < g1; grp += blockDim.x) {
    double hi[ST];
#pragma unroll
    for (int u = 0; u < ST; ++u) hi[u] = 1.0;
    int64_t x = grp;
    for (int m = 1; m < a.N1; ++m) {
      const int rm = a.rad[m];
      const int jm = (int)(x % rm);
      x /= rm;
#pragma unroll
      for (int u = 0; u < ST; ++u)
        if (s0 + u < send) hi[u] *= a.C[(int64_t)m * R * S + jm + (int64_t)R * (s0 + u)];
    }
    const int64_t j0 = grp * r0;
    for (int i0 = 0; i0 < r0; ++i0) {
      double q[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) q[r] = (r < R) ? a.Q0[j0 + i0 + a.J * r] : 0.0;
#pragma unroll
      for (int u = 0; u < ST; ++u) {
        if (s0 + u >= send) continue;
        const double p = a.C[i0 + (int64_t)R * (s0 + u)] * hi[u];
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[u][r] = fma(p, q[r], acc[u][r]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < ST; ++u)
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const double v = warp_sum(acc[u][r]);
      if (lane == 0) red[wid][u][r] = v;
    }
  __syncthreads();
  for (int e = tid; e < ST * R; e += blockDim.x) {
    const int u = e / R, r = e - u * R, s = s0 + u;
    if (s >= send) continue;
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w][u][r];
    if (a.nc == 1) a.M[s + (int64_t)S * r] = t;
    else a.P[((int64_t)s * a.nc + ch) * R + r] = t;
  }
}
__global__ void k_kt_m_reduce(const double* __restrict__ P, int S, int R, int nc, double* __restrict__ M) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < S * R; e += gridDim.x * blockDim.x) {
    const int s = e / R, r = e - s * R;
    double t = 0.0;
    for (int ch = 0; ch < nc; ++ch) t += P[((int64_t)s * nc + ch) * R + r];
    M[s + (int64_t)S * r] = t;
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
  const double* B[kKtMaxModes];  // I_k x S (leading dimension ld[k])
  const double* A[kKtMaxModes];  // I_k x R (normalised factors, leading dimension ld[k])
  int64_t I[kKtMaxModes];        // extents (the true I_k)
  int64_t ld[kKtMaxModes];       // row counts of the stored arrays (max(I_k, R) for short modes)
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
        v *= isx ? a.B[k][ik + a.ld[k] * q] : a.A[k][ik + a.ld[k] * q];
      }
      pw[wid][s] = v;
    }
    __syncwarp();
    for (int64_t i1 = lane; i1 < a.I[0]; i1 += 32) {
      double d = 0.0;
      for (int s = 0; s < a.S; ++s) d = fma(a.B[0][i1 + a.ld[0] * s], pw[wid][s], d);
      for (int r = 0; r < a.R; ++r) d = fma(a.A[0][i1 + a.ld[0] * r], pw[wid][a.S + r], d);
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
