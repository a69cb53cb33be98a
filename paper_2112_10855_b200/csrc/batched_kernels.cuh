// Batched CP-ALS for many small 3-way problems ("one CTA per problem"):
// one CTA runs a whole solve -- Alg. 2 (variants QR and QR-SVD)
// or Alg. 1 (NE with the Cholesky solve, LU fallback, and CP-ALS-PINV,
// PAPER.md:264-266) -- sweep after sweep with the stopping rule of PAPER.md:532 (change in relative
// error below tol) and no host round trip: the four solvers of the collinear-factor study
// (Table 4.1) on the same batch.  Shapes:
// N = 3, I_k <= 64, R <= 8, I_1 I_2 R <= 16384 and I_2 I_3 R <= 16384 (e.g. the paper's 50^3,
// rank-5 collinearity study).
//
// Per sweep X is streamed twice (the dimension tree of PAPER.md:472-478 falls out for N = 3):
//   T = X x_3 Q_3^T (I_1 x I_2 x R) serves mode 1 (Y = T x_2 Q_2^T) and mode 2 (Y = T x_1 Q_1^T,
//   with the Q_1 just updated; Q_3 is unchanged in between), U = X x_1 Q_1^T (R x I_2 x I_3)
//   serves mode 3 (Y = U x_2 Q_2^T).
// Each mode then: V_n = R_b (.) R_a (Kolda-Bader rows j = j_a + R j_b, a < b the other modes),
// Householder QR of V_n (one warp), W = Y_(n) Q0, back substitution Ahat R0^T = W (QR) or Ahat =
// W U S^+ V^T from the one-sided Jacobi SVD of R0 (QR-SVD), lambda and normalisation (zero column
// -> e_1), Householder QR of A_n (one warp), and after mode 3 the fast fit.
// NE / PINV hold A_k and G_k = A_k^T A_k instead of Q_k, R_k: the same TTM chain with A_k gives
// Y = X x_{k != n} A_k^T, whose Khatri-Rao diagonal Y(i, c + R c) is the MTTKRP M_n;
// S_n = G_a (*) G_b; Ahat S_n = M_n by Cholesky (LU with partial pivoting on a non-positive pivot,
// reading 18) or Ahat = M_n S_n^+ (PINV); normalise; G_n = A_n^T A_n; fit by PAPER.md:417-425.
// QRs carry the sign fix diag(R) >= 0.  All reductions fixed-order.
#pragma once
#include "common.cuh"
#include "small_kernels.cuh"  // jacobi_pinv

namespace cpqr {

constexpr int kBatMaxI = 64, kBatMaxR = 8, kBatTBuf = 16384;

struct BatchedArgs {
  const double* X;      // P problems, each I_1 I_2 I_3 column-major, consecutive
  const double* A0;     // P x (I_1 + I_2 + I_3) x R: the initial factors, column-major per mode
  int I[3];
  int R;
  int max_iters;
  double tol;
  double* A;            // out: factors (layout of A0)
  double* lam;          // out: P x R
  double* fits;         // out: P x max_iters (NaN after the last sweep run)
  int* iters;           // out: P (sweeps run)
  int variant;          // 0 NE, 1 QR, 2 QR-SVD, 3 PINV (cpqr_variant)
  double tau;           // SVD / PINV truncation (relative to sigma_max; < 0: R eps)
};

// Ahat S = M for the R x R symmetric S (R <= 8) by one thread: Cholesky, or LU with partial
// pivoting when a pivot is not positive (the oracle's LAPACK gesv fallback).  Returns the factors
// in F (ld 8) and the row permutation piv (identity for Cholesky); *chol = 1 for Cholesky.
__device__ void bat_ne_factor(const double* S, int R, double* F, int* piv, int* chol) {
  bool ok = true;
  for (int e = 0; e < 64; ++e) F[e] = (e % 8 < R && e / 8 < R) ? S[(e % 8) + 8 * (e / 8)] : 0.0;
  for (int j = 0; j < R && ok; ++j) {  // lower Cholesky in place: F = L
    double d = F[j + 8 * j];
    for (int k = 0; k < j; ++k) d -= F[j + 8 * k] * F[j + 8 * k];
    if (!(d > 0.0)) { ok = false; break; }
    const double l = sqrt(d);
    F[j + 8 * j] = l;
    for (int i = j + 1; i < R; ++i) {
      double v = F[i + 8 * j];
      for (int k = 0; k < j; ++k) v -= F[i + 8 * k] * F[j + 8 * k];
      F[i + 8 * j] = v / l;
    }
  }
  for (int i = 0; i < R; ++i) piv[i] = i;
  *chol = ok ? 1 : 0;
  if (ok) return;
  for (int e = 0; e < 64; ++e) F[e] = (e % 8 < R && e / 8 < R) ? S[(e % 8) + 8 * (e / 8)] : 0.0;
  for (int j = 0; j < R; ++j) {  // PA = LU (unit L below, U on and above the diagonal)
    int p = j;
    for (int i = j + 1; i < R; ++i)
      if (fabs(F[i + 8 * j]) > fabs(F[p + 8 * j])) p = i;
    if (p != j) {
      for (int c = 0; c < R; ++c) { const double t = F[j + 8 * c]; F[j + 8 * c] = F[p + 8 * c]; F[p + 8 * c] = t; }
      const int t = piv[j]; piv[j] = piv[p]; piv[p] = t;
    }
    const double d = F[j + 8 * j];
    for (int i = j + 1; i < R; ++i) {
      const double l = (d != 0.0) ? F[i + 8 * j] / d : 0.0;
      F[i + 8 * j] = l;
      for (int c = j + 1; c < R; ++c) F[i + 8 * c] -= l * F[j + 8 * c];
    }
  }
}

// Thin Householder QR of the m x R panel M (smem, ld 64, m <= 64, R <= 8) by one warp, in place:
// on exit M = Q (sign-fixed) and Rf (R x R, ld 8) = R with diag >= 0.  tau: R doubles of scratch.
__device__ __noinline__ void bat_hh_qr(double* M, int m, int R, double* Rf, double* tau) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < R; ++j) {
    double ss = 0.0;
    for (int i = j + lane; i < m; i += 32) ss = fma(M[i + 64 * j], M[i + 64 * j], ss);
    const double nrm = sqrt(warp_sum(ss));
    const double alpha = M[j + 64 * j];
    const double beta = (nrm == 0.0) ? 0.0 : (alpha >= 0.0 ? -nrm : nrm);
    const double t = (nrm == 0.0) ? 0.0 : (beta - alpha) / beta;
    const double sc = (nrm == 0.0) ? 0.0 : 1.0 / (alpha - beta);
    __syncwarp();
    for (int i = j + 1 + lane; i < m; i += 32) M[i + 64 * j] *= sc;  // v = x / (alpha - beta), v_j = 1
    if (lane == 0) { tau[j] = t; M[j + 64 * j] = beta; }
    __syncwarp();
    for (int c = j + 1; c < R; ++c) {  // A(:, c) -= tau v (v^T A(:, c))
      double w = 0.0;
      for (int i = j + lane; i < m; i += 32) w = fma(i == j ? 1.0 : M[i + 64 * j], M[i + 64 * c], w);
      w = warp_sum(w) * t;
      __syncwarp();
      for (int i = j + lane; i < m; i += 32) M[i + 64 * c] = fma(-w, i == j ? 1.0 : M[i + 64 * j], M[i + 64 * c]);
      __syncwarp();
    }
  }
  // R (upper) and the sign of its diagonal
  for (int e = lane; e < R * R; e += 32) {
    const int r = e % R, c = e / R;
    Rf[r + 8 * c] = (r <= c) ? M[r + 64 * c] : 0.0;
  }
  __syncwarp();
  // Q = H_0 .. H_{R-1} I(:, 0:R): backward accumulation into the panel (v kept below diag)
  // lane i (and i + 32) owns row i of Q; v_j(i) read before column j is overwritten
  double q[2][kBatMaxR];
  for (int h = 0; h < 2; ++h)
    for (int c = 0; c < kBatMaxR; ++c) q[h][c] = (lane + 32 * h == c) ? 1.0 : 0.0;
  for (int j = R - 1; j >= 0; --j) {
    const double t = tau[j];
    double vi[2];
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      vi[h] = (i < m && i > j) ? M[i + 64 * j] : (i == j ? 1.0 : 0.0);
    }
    for (int c = j; c < R; ++c) {  // Q(:, c) -= t v (v^T Q(:, c))
      double w = 0.0;
      for (int h = 0; h < 2; ++h) w = fma(vi[h], q[h][c], w);
      w = warp_sum(w) * t;
      for (int h = 0; h < 2; ++h) q[h][c] = fma(-w, vi[h], q[h][c]);
    }
  }
  __syncwarp();
  for (int c = 0; c < R; ++c) {
    const double s = (Rf[c + 8 * c] < 0.0) ? -1.0 : 1.0;
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i < m) M[i + 64 * c] = s * q[h][c];
    }
  }
  __syncwarp();
  for (int e = lane; e < R * R; e += 32) {
    const int r = e % R, c = e / R;
    if (Rf[r + 8 * r] < 0.0) Rf[r + 8 * c] = -Rf[r + 8 * c];
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256, 1) k_batched_cpqr(BatchedArgs a) {
  extern __shared__ double smb[];
  const int R = a.R, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int I0 = a.I[0], I1 = a.I[1], I2 = a.I[2];
  const int64_t numel = (int64_t)I0 * I1 * I2;
  const int p = blockIdx.x;
  const double* X = a.X + p * numel;
  double* Tb = smb;                      // T or U (<= 16384)
  double* Y = Tb + kBatTBuf;             // <= 64 * 64
  double* Qk = Y + 64 * 64;              // 3 x (64 x 8) factor Q panels (ld 64)
  double* Rk = Qk + 3 * 64 * 8;          // 3 x (8 x 8)
  double* V = Rk + 3 * 64;               // V_n / Q0 panel (64 x 8, ld 64)
  double* R0 = V + 64 * 8;               // 8 x 8
  double* Wm = R0 + 64;                  // W / Ahat / A_n panel (64 x 8, ld 64)
  double* Wsave = Wm + 64 * 8;           // W (QR / SVD) or M (NE / PINV) of mode 3 (fit)
  double* Ss = Wsave + 64 * 8;           // S_n (NE / PINV), 8 x 8
  double* Fs = Ss + 64;                  // its Cholesky / LU factors, 8 x 8
  double* Jb = Fs + 64;                  // jacobi_pinv scratch: B, V (R x (R+1) each), M (R x R), input
  double* Jv = Jb + 72;
  double* Jm = Jv + 72;
  double* Jin = Jm + 64;
  __shared__ double tau[kBatMaxR], lam[kBatMaxR], red[8], nX2s, fitprev, inner3;
  __shared__ int stop, piv[kBatMaxR], cholok, jflag;
  const bool ne = (a.variant == 0 || a.variant == 3);
  const double tauv = (a.tau < 0.0) ? R * 2.220446049250313e-16 : a.tau;
  const int Id[3] = {I0, I1, I2};
  int64_t aoff[3];
  aoff[0] = (int64_t)p * (I0 + I1 + I2) * R;
  aoff[1] = aoff[0] + (int64_t)I0 * R;
  aoff[2] = aoff[1] + (int64_t)I1 * R;
  // ||X||^2 and the factor QR cache of modes 2, 3 (Alg. 2 line 3)
  {
    double s = 0.0;
    for (int64_t e = tid; e < numel; e += nt) s = fma(X[e], X[e], s);
    s = block_sum(s, red);
    if (tid == 0) { nX2s = s; fitprev = 0.0; stop = 0; }
  }
  for (int k = 1; k < 3; ++k) {
    for (int e = tid; e < 64 * 8; e += nt) {
      const int i = e % 64, c = e / 64;
      Qk[k * 512 + e] = (i < Id[k] && c < R) ? a.A0[aoff[k] + i + (int64_t)Id[k] * c] : 0.0;
    }
    __syncthreads();
    if (ne) {  // G_k = A_k^T A_k (Alg. 1 line 3)
      for (int e = tid; e < 64; e += nt) {
        const int r = e % 8, c = e / 8;
        double g = 0.0;
        if (r < R && c < R)
          for (int i = 0; i < Id[k]; ++i) g = fma(Qk[k * 512 + i + 64 * r], Qk[k * 512 + i + 64 * c], g);
        Rk[k * 64 + e] = g;
      }
    } else if (wid == 0) {
      bat_hh_qr(Qk + k * 512, Id[k], R, Rk + k * 64, tau);
    }
    __syncthreads();
  }
  int it = 0;
  for (; it < a.max_iters; ++it) {
    for (int n = 0; n < 3; ++n) {
      // ---- line 8: Y (Kolda-Bader Y_(n) rows i_n, columns j = r_a + R r_b)
      if (n == 0) {  // T(i0, i1, r) = sum_i2 X(i0, i1, i2) Q3(i2, r)
        for (int e = tid; e < I0 * I1; e += nt) {
          double acc[kBatMaxR];
          for (int r = 0; r < kBatMaxR; ++r) acc[r] = 0.0;
          for (int i2 = 0; i2 < I2; ++i2) {
            const double x = X[e + (int64_t)I0 * I1 * i2];
            for (int r = 0; r < kBatMaxR; ++r)
              if (r < R) acc[r] = fma(x, Qk[2 * 512 + i2 + 64 * r], acc[r]);
          }
          for (int r = 0; r < R; ++r) Tb[e + I0 * I1 * r] = acc[r];
        }
        __syncthreads();
        for (int e = tid; e < I0 * R * R; e += nt) {  // Y(i0, j = r1 + R r2) = sum_i1 T(i0, i1, r2) Q2(i1, r1)
          const int i0 = e % I0, j = e / I0, r1 = j % R, r2 = j / R;
          double s = 0.0;
          for (int i1 = 0; i1 < I1; ++i1) s = fma(Tb[i0 + I0 * i1 + I0 * I1 * r2], Qk[512 + i1 + 64 * r1], s);
          Y[i0 + 64 * j] = s;
        }
      } else if (n == 1) {  // Y(i1, j = r0 + R r2) = sum_i0 T(i0, i1, r2) Q1(i0, r0)   (T reused)
        for (int e = tid; e < I1 * R * R; e += nt) {
          const int i1 = e % I1, j = e / I1, r0 = j % R, r2 = j / R;
          double s = 0.0;
          for (int i0 = 0; i0 < I0; ++i0) s = fma(Tb[i0 + I0 * i1 + I0 * I1 * r2], Qk[i0 + 64 * r0], s);
          Y[i1 + 64 * j] = s;
        }
      } else {  // U(r0, i1, i2) = sum_i0 Q1(i0, r0) X(i0, i1, i2); Y(i2, j = r0 + R r1) = sum_i1 U Q2(i1, r1)
        for (int e = tid; e < R * I1 * I2; e += nt) {
          const int r0 = e % R, f = e / R;  // f = i1 + I1 i2: a mode-1 fibre of X
          const double* xf = X + (int64_t)I0 * f;
          double s = 0.0;
          for (int i0 = 0; i0 < I0; ++i0) s = fma(xf[i0], Qk[i0 + 64 * r0], s);
          Tb[e] = s;
        }
        __syncthreads();
        for (int e = tid; e < I2 * R * R; e += nt) {
          const int i2 = e % I2, j = e / I2, r0 = j % R, r1 = j / R;
          double s = 0.0;
          for (int i1 = 0; i1 < I1; ++i1) s = fma(Tb[r0 + R * (i1 + I1 * i2)], Qk[512 + i1 + 64 * r1], s);
          Y[i2 + 64 * j] = s;
        }
      }
      const int ka = (n == 0) ? 1 : 0, kb = (n == 2) ? 1 : 2;
      const int In = Id[n];
      if (ne) {
        // ---- Alg. 1 lines 6-9: S_n = G_a (*) G_b, M_n = diag part of Y, Ahat S_n = M_n
        for (int e = tid; e < 64; e += nt) Ss[e] = Rk[ka * 64 + e] * Rk[kb * 64 + e];
        __syncthreads();  // every Y column written
        for (int e = tid; e < In * R; e += nt) {
          const int i = e % In, c = e / In;
          const double m = Y[i + 64 * (c + R * c)];
          Wm[i + 64 * c] = m;
          if (n == 2) Wsave[i + 64 * c] = m;
        }
        __syncthreads();
        if (a.variant == 3) {  // CP-ALS-PINV: Ahat = M S^+ (SVD pseudo-inverse)
          for (int e = tid; e < R * R; e += nt) Jin[e] = Ss[(e % R) + 8 * (e / R)];
          __syncthreads();
          jacobi_pinv(Jin, R, tauv, Jb, Jv, Jm, &jflag);
          if (tid < In) {
            double mv[kBatMaxR];
            for (int c = 0; c < R; ++c) mv[c] = Wm[tid + 64 * c];
            for (int c = 0; c < R; ++c) {
              double s = 0.0;
              for (int r = 0; r < R; ++r) s = fma(mv[r], Jm[r + R * c], s);
              Wm[tid + 64 * c] = s;
            }
          }
        } else {
          if (tid == 0) bat_ne_factor(Ss, R, Fs, piv, &cholok);
          __syncthreads();
          if (tid < In) {  // row i: S ahat = m (S symmetric)
            double x[kBatMaxR];
            if (cholok) {
              for (int j = 0; j < R; ++j) {  // L y = m
                double v = Wm[tid + 64 * j];
                for (int k = 0; k < j; ++k) v -= Fs[j + 8 * k] * x[k];
                x[j] = v / Fs[j + 8 * j];
              }
              for (int j = R - 1; j >= 0; --j) {  // L^T ahat = y
                double v = x[j];
                for (int k = j + 1; k < R; ++k) v -= Fs[k + 8 * j] * x[k];
                x[j] = v / Fs[j + 8 * j];
              }
            } else {
              double y[kBatMaxR];
              for (int j = 0; j < R; ++j) {  // L y = P m
                double v = Wm[tid + 64 * piv[j]];
                for (int k = 0; k < j; ++k) v -= Fs[j + 8 * k] * y[k];
                y[j] = v;
              }
              for (int j = R - 1; j >= 0; --j) {  // U ahat = y
                double v = y[j];
                for (int k = j + 1; k < R; ++k) v -= Fs[j + 8 * k] * x[k];
                x[j] = v / Fs[j + 8 * j];
              }
            }
            for (int c = 0; c < R; ++c) Wm[tid + 64 * c] = x[c];
          }
        }
        __syncthreads();
      } else {
        // ---- lines 6-7: V_n = R_b (.) R_a and its QR
        for (int e = tid; e < 64 * 8; e += nt) {
          const int j = e % 64, c = e / 64;
          double v = 0.0;
          if (j < R * R && c < R) v = Rk[ka * 64 + (j % R) + 8 * c] * Rk[kb * 64 + (j / R) + 8 * c];
          V[e] = v;
        }
        __syncthreads();
        if (wid == 0) bat_hh_qr(V, R * R, R, R0, tau);
        __syncthreads();
        // ---- line 9: W = Y_(n) Q0;  line 10: Ahat R0^T = W (back substitution per row), or the
        // QR-SVD solve Ahat = W U S^+ V^T
        for (int e = tid; e < In * R; e += nt) {
          const int i = e % In, c = e / In;
          double s = 0.0;
          for (int j = 0; j < R * R; ++j) s = fma(Y[i + 64 * j], V[j + 64 * c], s);
          Wm[i + 64 * c] = s;
          if (n == 2) Wsave[i + 64 * c] = s;
        }
        __syncthreads();
        if (a.variant == 2) {
          for (int e = tid; e < R * R; e += nt) Jin[e] = R0[(e % R) + 8 * (e / R)];
          __syncthreads();
          jacobi_pinv(Jin, R, tauv, Jb, Jv, Jm, &jflag);
          if (tid < In) {
            double wv[kBatMaxR];
            for (int c = 0; c < R; ++c) wv[c] = Wm[tid + 64 * c];
            for (int c = 0; c < R; ++c) {
              double s = 0.0;
              for (int r = 0; r < R; ++r) s = fma(wv[r], Jm[r + R * c], s);
              Wm[tid + 64 * c] = s;
            }
          }
        } else if (tid < In) {
          for (int j = R - 1; j >= 0; --j) {
            double acc = Wm[tid + 64 * j];
            for (int l = j + 1; l < R; ++l) acc -= Wm[tid + 64 * l] * R0[j + 8 * l];
            Wm[tid + 64 * j] = acc / R0[j + 8 * j];
          }
        }
        __syncthreads();
      }
      // ---- line 11: lambda, normalise (lambda = 0 -> e_1);  line 12: QR(A_n)
      if (wid < R) {
        double ss = 0.0;
        for (int i = lane; i < In; i += 32) ss = fma(Wm[i + 64 * wid], Wm[i + 64 * wid], ss);
        ss = warp_sum(ss);
        if (lane == 0) lam[wid] = sqrt(ss);
      }
      __syncthreads();
      if (n == 2 && a.max_iters > 0) {  // <X, Xh>: <W_3, Ahat_3 R0^T> (QR / SVD) or <M_3, Ahat_3> (NE)
        double s = 0.0;
        for (int e = tid; e < In * R; e += nt) {
          const int i = e % In, c = e / In;
          double t = 0.0;
          if (ne) t = Wm[i + 64 * c];
          else
            for (int l = c; l < R; ++l) t = fma(Wm[i + 64 * l], R0[c + 8 * l], t);
          s = fma(Wsave[i + 64 * c], t, s);
        }
        s = block_sum(s, red);
        if (tid == 0) inner3 = s;
      }
      for (int e = tid; e < 64 * 8; e += nt) {
        const int i = e % 64, c = e / 64;
        double v = 0.0;
        if (i < In && c < R) {
          const double l = lam[c];
          v = (l > 0.0) ? Wm[i + 64 * c] / l : (i == 0 ? 1.0 : 0.0);
          a.A[aoff[n] + i + (int64_t)In * c] = v;
        }
        Qk[n * 512 + e] = v;
      }
      __syncthreads();
      if (ne) {  // G_n = A_n^T A_n (Alg. 1 line 11)
        for (int e = tid; e < 64; e += nt) {
          const int r = e % 8, c = e / 8;
          double g = 0.0;
          if (r < R && c < R)
            for (int i = 0; i < In; ++i) g = fma(Qk[n * 512 + i + 64 * r], Qk[n * 512 + i + 64 * c], g);
          Rk[n * 64 + e] = g;
        }
      } else if (wid == 0) {
        bat_hh_qr(Qk + n * 512, In, R, Rk + n * 64, tau);
      }
      __syncthreads();
    }
    // ---- fast fit after mode 3 (NE: PAPER.md:417-425)
    if (tid == 0) {
      double nxh2 = 0.0;  // <R0^T R0, diag(lam) R_3^T R_3 diag(lam)>  or  <S_3, diag(lam) G_3 diag(lam)>
      for (int x = 0; x < R; ++x)
        for (int y = 0; y < R; ++y) {
          if (ne) {
            nxh2 = fma(Ss[x + 8 * y], lam[x] * lam[y] * Rk[2 * 64 + x + 8 * y], nxh2);
            continue;
          }
          double g0 = 0.0, g1 = 0.0;
          for (int k = 0; k <= min(x, y); ++k) {
            g0 = fma(R0[k + 8 * x], R0[k + 8 * y], g0);
            g1 = fma(Rk[2 * 64 + k + 8 * x], Rk[2 * 64 + k + 8 * y], g1);
          }
          nxh2 = fma(g0, lam[x] * lam[y] * g1, nxh2);
        }
      const double inner = inner3;
      const double fit = 1.0 - sqrt(fmax(0.0, nX2s - 2.0 * inner + nxh2)) / sqrt(nX2s);
      a.fits[(int64_t)p * a.max_iters + it] = fit;
      stop = (it > 0 && fabs(fit - fitprev) < a.tol) ? 1 : 0;
      fitprev = fit;
    }
    __syncthreads();
    if (stop) { ++it; break; }
  }
  if (tid < R) a.lam[(int64_t)p * R + tid] = lam[tid];
  for (int i = it + tid; i < a.max_iters; i += nt) a.fits[(int64_t)p * a.max_iters + i] = __longlong_as_double(0x7ff8000000000000ll);
  if (tid == 0) a.iters[p] = it;
}

}  // namespace cpqr
