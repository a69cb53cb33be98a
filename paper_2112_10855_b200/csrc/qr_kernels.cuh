// Householder QR kernels of the per-mode tail (sm_100a, fp64), shared-memory resident.
//
//   hh_factor / hh_formq   in-place Householder QR (LAPACK dgeqr2 / dorg2r conventions) of a
//                          matrix whose column k is the contiguous run col(k)[0 .. nrow[k]) -- a
//                          dense panel (nrow = m) or the packed staircase of V_n (nrow[k] =
//                          (k+1)^{N-1}: no fill-in, Q0 has V_n's support).
//                          Two block barriers per column: after the reflector-dot phase, warp 0
//                          applies H_j to column j+1 and immediately builds reflector j+1 while
//                          the other warps update the remaining columns.
//   k_tsqr_leaf/root/qform thin QR of the I_n x R factor (Alg. 2 line 12) as a
//                          one-level TSQR: leaf blocks in parallel CTAs, QR of the stacked R_b
//                          in one CTA (diag(R) >= 0, reading 6), explicit Q = diag(Q_b) Q_top
//                          written both column-major (Q_n) and as the transposed padded panel the
//                          TMA kernels stream.
//   k_form_v / k_kr_qr2    V_n (Khatri-Rao of the R_k, Alg. 2 line 6) formed densely for the
//                          CholeskyQR2 path, and the one-CTA staircase Householder QR of V_n
//                          (K2, line 7), gated by FLAG_VN_HOUSEHOLDER behind the CholeskyQR2 path.
//   k_svd_pinv             M = U S^+ V^T of R0 by one-sided Jacobi (QR-SVD).
//   k_ne_pinv              S_n^+ of the Hadamard product of Grams, same Jacobi (CP-ALS-PINV).
//   k_solve_rows           Alg. 2 line 10 for factors too tall for the shared-memory tails (Householder
//                          forced): Ahat R0^T = W (row-parallel back substitution) or Ahat = W M,
//                          with the column sums of squares and <W, Ahat R0^T> per
//                          CTA; k_tall_fallback (small_kernels.cuh) then normalises and factors.
#pragma once
#include <cstdio>
#include "small_kernels.cuh"

namespace cpqr {

struct HHCols {        // packed staircase: column k at base + off[k], nrow[k] rows
  double* base;
  const int64_t* off;  // column offsets (shared memory)
  const int* nrow;     // rows per column (shared memory)
  __device__ __forceinline__ double* col(int k) const { return base + off[k]; }
  __device__ __forceinline__ int rows(int k) const { return nrow[k]; }
};
struct DenseCols {     // dense panel: column k at base + k*ld, m rows
  double* base;
  int ld, m;
  __device__ __forceinline__ double* col(int k) const { return base + (int64_t)k * ld; }
  __device__ __forceinline__ int rows(int) const { return m; }
};

// Factorisation.  On exit: col(k)[r] (r < k) = R(r, k) (unsigned), beta[k] = R(k, k), reflector
// j (v_j = 1 implicit) stored below the diagonal of column j, tau[j].  All threads must call;
// `w` needs R doubles, `np` 64 doubles of shared memory.
// Per column two block barriers and no serial section: (A) one warp per trailing column forms
// w_k = col(k)[j] + scale_j sum_{i>j} col(j)[i] col(k)[i] (the reflector is scaled lazily);
// (B) each thread owns rows: writes v_i = scale_j col(j)[i], applies H_j to all trailing columns
// and accumulates its share of ||col(j+1)[j+2..]||^2; (C) every thread rebuilds beta/tau/scale of
// column j+1 from the per-warp partials (identical arithmetic everywhere, fixed summation order).
template <class Cols>
__device__ __forceinline__ void hh_reflector_from(const Cols& M, int j, const double* np, int nw, double& tj,
                                                  double& bj, double& sc) {
  double s = 0.0;
  for (int q = 0; q < nw; ++q) s += np[q];
  const double x0 = M.col(j)[j];
  if (s == 0.0) { tj = 0.0; bj = x0; sc = 0.0; }
  else {
    const double nrm = sqrt(x0 * x0 + s);
    bj = (x0 >= 0.0) ? -nrm : nrm;
    tj = (bj - x0) / bj;
    sc = 1.0 / (x0 - bj);
  }
}

template <class Cols>
__device__ void hh_factor(const Cols& M, int R, double* tau, double* beta, double* w, double* np) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  {  // column 0 norm partials
    const double* c0 = M.col(0);
    double q = 0.0;
    for (int i = 1 + tid; i < M.rows(0); i += nt) q = fma(c0[i], c0[i], q);
    q = warp_sum(q);
    if (lane == 0) np[32 + wid] = q;
  }
  __syncthreads();
  double tj, bj, sc;
  hh_reflector_from(M, 0, np + 32, nw, tj, bj, sc);
  for (int j = 0; j < R; ++j) {
    double* vj = M.col(j);
    const int mj = M.rows(j);
    if (tid == 0) { tau[j] = tj; beta[j] = bj; }
    // (A) dots with the (still unscaled) reflector
    if (tj != 0.0) {
      for (int k = j + 1 + wid; k < R; k += nw) {
        const double* ck = M.col(k);
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
        int i = j + 1 + lane;
        for (; i + 96 < mj; i += 128) {
          d0 = fma(vj[i], ck[i], d0);
          d1 = fma(vj[i + 32], ck[i + 32], d1);
          d2 = fma(vj[i + 64], ck[i + 64], d2);
          d3 = fma(vj[i + 96], ck[i + 96], d3);
        }
        for (; i < mj; i += 32) d0 = fma(vj[i], ck[i], d0);
        const double d = warp_sum((d0 + d1) + (d2 + d3));
        if (lane == 0) w[k] = tj * (ck[j] + sc * d);  // tau_j * (v^T col k)
      }
    }
    __syncthreads();
    // (B) scale v, apply H_j, partial norm of column j+1 (rows > j+1)
    const int mnext = (j + 1 < R) ? M.rows(j + 1) : 0;
    double q = 0.0;
    const int iend = max(mj, mnext);
    for (int i = j + tid; i < iend; i += nt) {
      double vi = 0.0;
      if (i < mj) {
        if (i == j) { vi = 1.0; vj[j] = bj; }
        else { vi = sc * vj[i]; vj[i] = vi; }
      }
      if (tj != 0.0 && i < mj) {
#pragma unroll 8
        for (int k = j + 1; k < R; ++k) M.col(k)[i] -= w[k] * vi;
      }
      if (j + 1 < R && i > j + 1 && i < mnext) {
        const double x = M.col(j + 1)[i];
        q = fma(x, x, q);
      }
    }
    q = warp_sum(q);
    double* npj = np + 32 * (j & 1);  // double-buffered: (C) of step j reads what (B) of step j+1 must not overwrite
    if (lane == 0) npj[wid] = q;
    __syncthreads();
    // (C) reflector of column j+1, redundantly in every thread
    if (j + 1 < R) hh_reflector_from(M, j + 1, npj, nw, tj, bj, sc);
  }
}

// Explicit Q in place (dorg2r), after hh_factor (R must have been saved first).  Columns are NOT
// sign-fixed here.  Two barriers per column: dots, then the row-owned update + finalisation.
template <class Cols>
__device__ void hh_formq(const Cols& M, int R, const double* tau, double* w) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int j = R - 1; j >= 0; --j) {
    double* cj = M.col(j);
    const int mj = M.rows(j);
    const double tj = tau[j];
    if (j < R - 1 && tj != 0.0) {
      for (int k = j + 1 + wid; k < R; k += nw) {
        const double* ck = M.col(k);
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
        int i = j + 1 + lane;
        for (; i + 96 < mj; i += 128) {
          d0 = fma(cj[i], ck[i], d0);
          d1 = fma(cj[i + 32], ck[i + 32], d1);
          d2 = fma(cj[i + 64], ck[i + 64], d2);
          d3 = fma(cj[i + 96], ck[i + 96], d3);
        }
        for (; i < mj; i += 32) d0 = fma(cj[i], ck[i], d0);
        const double d = warp_sum((d0 + d1) + (d2 + d3));
        if (lane == 0) w[k] = tj * (ck[j] + d);  // v_j = 1; row j of column k is 0 (zeroed earlier)
      }
    }
    __syncthreads();
    for (int i = tid; i < mj; i += nt) {
      if (i >= j && j < R - 1 && tj != 0.0) {
        const double vi = (i == j) ? 1.0 : cj[i];
#pragma unroll 8
        for (int k = j + 1; k < R; ++k) M.col(k)[i] -= w[k] * vi;
      }
      cj[i] = (i < j) ? 0.0 : ((i == j) ? 1.0 - tj : -tj * cj[i]);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ TSQR (K1)
// Fused per-mode tail in three launches (leaf / root / qform).  With solve = 1 the leaf first
// solves its rows of Ahat (Alg. 2 line 10: substitution with R0, or W M with M = (R0^T)^+ for the
// SVD variant) straight into the shared-memory panel, and the TSQR factors Ahat itself: since
// Ahat = A diag(lambda), QR(A) has the same Q and R_n = R_hat diag(1/lambda) (positive scaling keeps
// diag(R) >= 0), so the leaf needs no grid-wide column norms.  The root turns the per-leaf partial
// sums of squares into lambda; qform writes Q_n, its TMA panel and A_n = Ahat / lambda.
struct TsqrArgs {
  const double* A;  // solve = 0: m x R column-major input
  int m, R, nleaf, mb;  // leaf b: rows [b*mb, min(m, (b+1)*mb))
  double* Rstack;   // (nleaf*R) x R column-major
  double* V;        // leaf reflectors: mb x R per leaf, column-major, leaf stride mb*R
  double* tauv;     // nleaf * R
  double* Qtop;     // (nleaf*R) x R column-major
  double* Q;        // out: m x R column-major
  double* Qt;       // out: m x RQ row-major, zero padded
  int RQ;
  double* Rn;       // out: R x R column-major, diag >= 0
  // solve mode
  int solve;
  const double* W;    // m x R row-major
  const double* Rm;   // R0 (variant 1) or M (variant 2)
  const double* R0;   // R0 (fit)
  int variant;
  double* Ahat;       // out: m x R column-major (unnormalised)
  double* part;       // nleaf x (R+1): column sums of squares, <W, Ahat R0^T>
  double* Aout;       // out: normalised factor (qform)
  double* lam;        // out: lambda (root)
  unsigned* flags;
  // fast fit after mode N: ||Xh||^2 = <R0^T R0, diag(lam) Rn^T Rn diag(lam)>
  int do_fit;
  const double* nX2;
  double* fit;
  int gated;  // 1: run only when the CholeskyQR2 path asked for the Householder fallback (0x200)
};

__device__ __forceinline__ bool tsqr_skip(const TsqrArgs& a) {
  __shared__ unsigned fl;
  if (threadIdx.x == 0) fl = a.gated ? *a.flags : 0x200u;
  __syncthreads();
  return (fl & 0x200u) == 0;
}

template <int RB>
__global__ void __launch_bounds__(256) k_tsqr_leaf(TsqrArgs a) {
  if (tsqr_skip(a)) return;
  extern __shared__ double sm[];
  __shared__ double tau[64], beta[64], w[64], red[8][RB + 1], np[64];
  __shared__ double Ms[RB * RB], R0s[RB * RB];
  const int b = blockIdx.x, R = a.R, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0;
  if (!a.solve) {
    for (int c = 0; c < R; ++c)
      for (int i = tid; i < rows; i += nt) sm[i + rows * c] = a.A[r0 + i + (int64_t)a.m * c];
    __syncthreads();
  } else {
    for (int e = tid; e < RB * RB; e += nt) {
      const int r = e % RB, c = e / RB;
      Ms[e] = (r < R && c < R) ? a.Rm[r + R * c] : 0.0;
      R0s[e] = (r < R && c < R) ? a.R0[r + R * c] : 0.0;
    }
    __syncthreads();
    double inner = 0.0;
    for (int ii = tid; ii < rows; ii += nt) {
      const int i = r0 + ii;
      double wv[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) wv[r] = (r < R) ? a.W[(int64_t)i * R + r] : 0.0;
      double* x = sm + ii;  // x[l] at x[rows * l]
      if (a.variant == 2) {
#pragma unroll 4
        for (int c = 0; c < RB; ++c) {
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < RB; ++r) s = fma(wv[r], Ms[r + RB * c], s);
          if (c < R) x[rows * c] = s;
        }
      } else {
        double xr[RB];
#pragma unroll
        for (int j = RB - 1; j >= 0; --j) {  // xr_j = (w_j - sum_{l>j} xr_l R0(j,l)) / R0(j,j)
          double acc = wv[j];
#pragma unroll
          for (int l = j + 1; l < RB; ++l) acc = fma(-xr[l], Ms[j + RB * l], acc);
          xr[j] = (j < R) ? acc / Ms[j + RB * j] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < RB; ++c)
          if (c < R) x[rows * c] = xr[c];
      }
      if (a.do_fit) {  // <W, Ahat R0^T> row contribution: sum_c w_c sum_{l>=c} x_l R0(c,l)
#pragma unroll 4
        for (int c = 0; c < RB; ++c) {
          double t = 0.0;
#pragma unroll
          for (int l = 0; l < RB; ++l)
            if (l >= c && l < R) t = fma(x[rows * l], R0s[c + RB * l], t);
          inner = fma(wv[c], t, inner);
        }
      }
    }
    __syncthreads();
    // Ahat rows out, per-leaf column sums of squares and fit partial (fixed order)
    for (int c = 0; c < R; ++c)
      for (int ii = tid; ii < rows; ii += nt) a.Ahat[r0 + ii + (int64_t)a.m * c] = sm[ii + rows * c];
    for (int c = wid; c < R; c += nt / 32) {
      double q = 0.0;
      for (int ii = lane; ii < rows; ii += 32) q = fma(sm[ii + rows * c], sm[ii + rows * c], q);
      q = warp_sum(q);
      if (lane == 0) a.part[b * (R + 1) + c] = q;
    }
    inner = warp_sum(inner);
    if (lane == 0) red[wid][0] = inner;
    __syncthreads();
    if (tid == 0) {
      double v = 0.0;
      for (int q = 0; q < nt / 32; ++q) v += red[q][0];
      a.part[b * (R + 1) + R] = v;
    }
  }
  DenseCols M{sm, rows, rows};
  hh_factor(M, R, tau, beta, w, np);
  const int ldr = a.nleaf * R;
  for (int e = tid; e < R * R; e += nt) {
    const int r = e % R, c = e / R;
    a.Rstack[b * R + r + (int64_t)ldr * c] = (r < c) ? sm[r + rows * c] : ((r == c) ? beta[r] : 0.0);
  }
  for (int c = 0; c < R; ++c)
    for (int i = tid; i < rows; i += nt) a.V[(int64_t)b * a.mb * R + i + rows * c] = sm[i + rows * c];
  if (tid < R) a.tauv[b * R + tid] = tau[tid];
}

__global__ void __launch_bounds__(512) k_tsqr_root(TsqrArgs a) {
  if (tsqr_skip(a)) return;
  extern __shared__ double sm[];
  __shared__ double tau[64], beta[64], w[64], red[32], lam[64], np[64];
  const int R = a.R, rows = a.nleaf * R;
  if (a.solve && threadIdx.x <= R) {  // lambda and <W, Ahat R0^T> from the leaf partials
    double s = 0.0;
    for (int b = 0; b < a.nleaf; ++b) s += a.part[b * (R + 1) + threadIdx.x];
    if (threadIdx.x < R) {
      lam[threadIdx.x] = sqrt(s);
      a.lam[threadIdx.x] = lam[threadIdx.x];
      if (!isfinite(lam[threadIdx.x])) atomicOr(a.flags, FLAG_NONFINITE);
    } else {
      red[0] = s;  // inner
    }
  }
  for (int e = threadIdx.x; e < rows * R; e += blockDim.x) sm[e] = a.Rstack[e];
  __syncthreads();
  const double inner = a.solve ? red[0] : 0.0;
  __syncthreads();
  DenseCols M{sm, rows, rows};
  hh_factor(M, R, tau, beta, w, np);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int r = e % R, c = e / R;
    double v = (r < c) ? sm[r + rows * c] : ((r == c) ? beta[r] : 0.0);
    if (beta[r] < 0.0) v = -v;
    if (a.solve && lam[c] > 0.0) v /= lam[c];  // R_n = R_hat diag(1/lambda)
    a.Rn[r + R * c] = v;
  }
  __syncthreads();
  hh_formq(M, R, tau, w);
  for (int e = threadIdx.x; e < rows * R; e += blockDim.x) {
    const int c = e / rows;
    a.Qtop[e] = (beta[c] < 0.0) ? -sm[e] : sm[e];
  }
  if (a.do_fit) {
    __syncthreads();
    double* r0s = sm;  // R0 and R_n in shared memory (capacity >= 2 R^2 guaranteed by the host)
    double* rns = sm + R * R;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) { r0s[e] = a.R0[e]; rns[e] = a.Rn[e]; }
    __syncthreads();
    double q = 0.0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int x = e % R, y = e / R;
      double g0 = 0.0, g1 = 0.0;
      for (int k = 0; k <= min(x, y); ++k) {
        g0 = fma(r0s[k + R * x], r0s[k + R * y], g0);
        g1 = fma(rns[k + R * x], rns[k + R * y], g1);
      }
      q = fma(g0, lam[x] * lam[y] * g1, q);
    }
    const double nxh2 = block_sum(q, red + 1);
    if (threadIdx.x == 0) {
      const double nx2 = *a.nX2;
      *a.fit = 1.0 - sqrt(fmax(0.0, nx2 - 2.0 * inner + nxh2)) / sqrt(nx2);
#ifdef CPQR_DEBUG_FIT
      printf("fit: nx2 %.17g inner %.17g nxh2 %.17g\n", nx2, inner, nxh2);
#endif
    }
  }
}

__global__ void __launch_bounds__(512) k_tsqr_qform(TsqrArgs a) {
  if (tsqr_skip(a)) return;
  extern __shared__ double sm[];
  __shared__ double w[64], tv[64];
  const int b = blockIdx.x, R = a.R, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5,
            nw = nt >> 5;
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0;
  double* Mq = sm;                // rows x R : [Qtop_b; 0]
  double* Vb = sm + rows * R;     // rows x R : leaf reflectors
  const int ldt = a.nleaf * R;
  for (int c = 0; c < R; ++c)
    for (int i = tid; i < rows; i += nt) {
      Mq[i + rows * c] = (i < R) ? a.Qtop[b * R + i + (int64_t)ldt * c] : 0.0;
      Vb[i + rows * c] = a.V[(int64_t)b * a.mb * R + i + rows * c];
    }
  if (tid < R) tv[tid] = a.tauv[b * R + tid];
  if (a.solve) {  // A_n = Ahat / lambda (zero column -> e_1, reading 10)
    for (int c = 0; c < R; ++c) {
      const double l = a.lam[c];
      for (int i = tid; i < rows; i += nt) {
        const int64_t e = r0 + i + (int64_t)a.m * c;
        a.Aout[e] = (l > 0.0) ? a.Ahat[e] / l : ((r0 + i) == 0 ? 1.0 : 0.0);
      }
    }
  }
  __syncthreads();
  for (int j = R - 1; j >= 0; --j) {
    const double tj = tv[j];
    if (tj == 0.0) continue;
    const double* vj = Vb + (int64_t)rows * j;
    for (int k = wid; k < R; k += nw) {
      const double* ck = Mq + (int64_t)rows * k;
      double d0 = 0.0, d1 = 0.0;
      int i = j + 1 + lane;
      for (; i + 32 < rows; i += 64) { d0 = fma(vj[i], ck[i], d0); d1 = fma(vj[i + 32], ck[i + 32], d1); }
      for (; i < rows; i += 32) d0 = fma(vj[i], ck[i], d0);
      const double d = warp_sum(d0 + d1);
      if (lane == 0) w[k] = ck[j] + d;
    }
    __syncthreads();
    for (int i = j + tid; i < rows; i += nt) {
      const double vi = (i == j) ? tj : tj * vj[i];
#pragma unroll 8
      for (int k = 0; k < R; ++k) Mq[i + rows * k] -= w[k] * vi;
    }
    __syncthreads();
  }
  for (int c = 0; c < R; ++c)
    for (int i = tid; i < rows; i += nt) a.Q[r0 + i + (int64_t)a.m * c] = Mq[i + rows * c];
  for (int i = tid / a.RQ; i < rows; i += nt / a.RQ) {  // blockDim is a multiple of RQ (16/32)
    const int c = tid % a.RQ;
    a.Qt[(int64_t)(r0 + i) * a.RQ + c] = (c < R) ? Mq[i + rows * c] : 0.0;
  }
}

// V_n = R_{k_{N-1}} (.) ... (.) R_{k_1} (Khatri-Rao of the retained triangular factors, Alg. 2
// line 6) formed densely: V(j, c) = prod_m R_{k_m}(j_m, c), j = sum_m j_m R^m (the
// Kolda-Bader row order of K2's Q0).  Used by the multi-CTA CholeskyQR2 V_n QR (high rank).
__global__ void k_form_v(KrQrArgs a, int64_t J, double* __restrict__ V) {
  // one thread per (column c, group of r0 rows sharing digits 1..N1-1): the product over the slow
  // factors once per group, then the r0 rows of the fastest factor (r0 = its radix)
  const int R = a.R;
  const int r0 = a.rad[0] ? a.rad[0] : R;  // mixed radix: short modes keep their min(I_k, R) rows
  const int64_t JG = J / r0;                // groups per column
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < JG * R; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / JG);
    const int64_t grp = e - (int64_t)c * JG;
    int64_t j = grp;
    double hi = 1.0;
    for (int m = 1; m < a.N1; ++m) {
      const int rm = a.rad[m] ? a.rad[m] : R;
      const int im = (int)(j % rm);
      j /= rm;
      hi *= (im <= c) ? a.Rk[m][im + R * c] : 0.0;
    }
    double* out = V + (int64_t)c * J + grp * r0;
    for (int i0 = 0; i0 < r0; ++i0) out[i0] = (i0 <= c) ? a.Rk[0][i0 + R * c] * hi : 0.0;
  }
}

// ------------------------------------------------------------- K2 with the 2-barrier primitive
__global__ void __launch_bounds__(1024) k_kr_qr2(KrQrArgs a) {
  extern __shared__ double smk[];
  __shared__ double tau[64], beta[64], w[64], np[64];
  __shared__ int64_t off[65];
  __shared__ int ncnt[64];
  __shared__ unsigned gate;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int R = a.R, N1 = a.N1;
  if (a.gate_bit) {  // fallback of the CholeskyQR2 V_n QR: run only if that was rejected
    if (tid == 0) gate = *a.flags & a.gate_bit;
    __syncthreads();
    if (!gate) return;
  }
  if (tid == 0) {
    int64_t o = 0;
    for (int c = 0; c < R; ++c) {
      int64_t p = 1;
      for (int m = 0; m < N1; ++m) p *= (c + 1);
      ncnt[c] = (int)p;
      off[c] = o;
      o += p;
    }
    off[R] = o;
  }
  __syncthreads();
  double* V = a.use_smem ? smk : a.work_global;
  for (int c = 0; c < R; ++c)  // V_n entries in packed staircase order
    for (int p = tid; p < ncnt[c]; p += nt) {
      int j = a.perm[p];
      double v = 1.0;
      for (int m = 0; m < N1; ++m) {
        const int im = j % R;
        j /= R;
        v *= a.Rk[m][im + R * c];
      }
      V[off[c] + p] = v;
    }
  __syncthreads();
  HHCols M{V, off, ncnt};
  hh_factor(M, R, tau, beta, w, np);
  for (int e = tid; e < R * R; e += nt) {
    const int r = e % R, c = e / R;
    double v = (r < c) ? V[off[c] + r] : ((r == c) ? beta[r] : 0.0);
    if (beta[r] < 0.0) v = -v;
    a.R0[r + R * c] = v;
  }
  if (tid == 0) {
    double mx = 0.0, mn = 1e308;
    for (int c = 0; c < R; ++c) { mx = fmax(mx, fabs(beta[c])); mn = fmin(mn, fabs(beta[c])); }
    int64_t J = 1;
    for (int m = 0; m < N1; ++m) J *= R;
    if (mn <= (double)J * kEps * mx) atomicOr(a.flags, FLAG_ILLCOND_R0);
  }
  __syncthreads();
  hh_formq(M, R, tau, w);
  int64_t J = 1;
  for (int m = 0; m < N1; ++m) J *= R;
  for (int64_t e = tid; e < J * R; e += nt) a.Q0[e] = 0.0;
  __syncthreads();
  for (int c = 0; c < R; ++c) {
    const double sg = (beta[c] < 0.0) ? -1.0 : 1.0;
    for (int p = tid; p < ncnt[c]; p += nt) a.Q0[a.perm[p] + J * c] = sg * V[off[c] + p];
  }
}


// ------------------------------------------------------------- multi-CTA solve (Alg. 2 l. 10-11)
// k_svd_pinv: M = U S^+ V^T of R0 (one CTA, one-sided Jacobi) for the QR-SVD variant.
__global__ void __launch_bounds__(512) k_svd_pinv(const double* __restrict__ R0, int R, double tau,
                                                  double* __restrict__ Mout, unsigned* flags, int* ntrunc) {
  extern __shared__ double sm[];
  __shared__ int sflag;
  double* R0s = sm;
  double* Ms = R0s + R * R;
  double* Bs = Ms + R * R;
  double* Vs = Bs + R * (R + 1);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) R0s[e] = R0[e];
  __syncthreads();
  const int ntr = jacobi_pinv(R0s, R, tau, Bs, Vs, Ms, &sflag);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Mout[e] = Ms[e];
  if (threadIdx.x == 0) {
    if (ntr > 0) atomicOr(flags, FLAG_SVD_TRUNCATED);
    if (ntrunc) *ntrunc = ntr;
  }
}

// k_ne_pinv: CP-ALS-PINV: S_n = Hadamard of the other Grams (Alg. 1 line 6),
// then its Moore-Penrose pseudo-inverse by the same one-sided Jacobi SVD: for S = U Sigma V^T the
// routine returns U Sigma^+ V^T = (S^+)^T = S^+ (S symmetric), dropping sigma_i <= tau sigma_max
// (reading 32).  Depends on the Grams only, so it runs on the side stream beside the MTTKRP.
struct NePinvArgs {
  const double* G[kMaxModes];
  int N, n, R;
  double tau;
  double* Mout;
  unsigned* flags;
};
__global__ void __launch_bounds__(512) k_ne_pinv(NePinvArgs a) {
  extern __shared__ double sm[];
  __shared__ int sflag;
  const int R = a.R;
  double* Ss = sm;
  double* Ms = Ss + R * R;
  double* Bs = Ms + R * R;
  double* Vs = Bs + R * (R + 1);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double v = 1.0;
    for (int k = a.N - 1; k >= 0; --k)
      if (k != a.n) v *= a.G[k][e];
    Ss[e] = v;
  }
  __syncthreads();
  const int ntr = jacobi_pinv(Ss, R, a.tau, Bs, Vs, Ms, &sflag);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) a.Mout[e] = Ms[e];
  if (threadIdx.x == 0 && ntr > 0) atomicOr(a.flags, FLAG_SVD_TRUNCATED);
}

// k_solve_rows<RB>: one thread per row i: Ahat(i,:) from W(i,:) by back substitution with R0
// (variant 1) or x = W(i,:) M (variant 2), registers only (R <= RB).  Per-CTA partial column
// sums of squares and the per-CTA partial of <W, Ahat R0^T> go to part[cta][0..R] (fixed order).
template <int RB, int BT = (RB > 16 ? 64 : 128)>
__global__ void __launch_bounds__(BT) k_solve_rows(const double* __restrict__ W, const double* __restrict__ Rm,
                                                    const double* __restrict__ R0, int In, int R, int variant,
                                                    double* __restrict__ Ahat, double* __restrict__ part,
                                                    int do_fit) {
  __shared__ double Ms[RB * RB];
  __shared__ double R0s[RB * RB];
  __shared__ double Xs[BT * (RB + 1)];
  __shared__ double red[BT / 32][RB + 1];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < RB * RB; e += blockDim.x) {
    const int r = e % RB, c = e / RB;
    Ms[e] = (r < R && c < R) ? Rm[r + R * c] : 0.0;
    R0s[e] = (r < R && c < R) ? R0[r + R * c] : 0.0;
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + tid;
  double* x = Xs + tid * (RB + 1);
  double w[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) w[r] = (i < In && r < R) ? W[(int64_t)i * R + r] : 0.0;
  if (variant == 2) {
#pragma unroll 4
    for (int c = 0; c < RB; ++c) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < RB; ++r) s = fma(w[r], Ms[r + RB * c], s);
      x[c] = s;
    }
  } else {
#pragma unroll
    for (int j = RB - 1; j >= 0; --j) {  // x_j = (w_j - sum_{l>j} x_l R0(j,l)) / R0(j,j)
      double acc = w[j];
#pragma unroll
      for (int l = j + 1; l < RB; ++l) acc = fma(-x[l], Ms[j + RB * l], acc);
      x[j] = (j < R) ? acc / Ms[j + RB * j] : 0.0;
    }
  }
  double inner = 0.0;
  if (do_fit) {  // <W, Ahat R0^T>: sum_c w_c sum_{l>=c} x_l R0(c,l)
#pragma unroll 4
    for (int c = 0; c < RB; ++c) {
      double t = 0.0;
#pragma unroll
      for (int l = 0; l < RB; ++l)
        if (l >= c) t = fma(x[l], R0s[c + RB * l], t);
      inner = fma(w[c], t, inner);
    }
  }
  if (i >= In) inner = 0.0;
  __syncthreads();
  // coalesced store of the block's rows (column-major Ahat) and per-column sums of squares
  const int i0 = blockIdx.x * blockDim.x;
  for (int c = 0; c < R; ++c) {
    const int ii = i0 + tid;
    const double v = (ii < In) ? Xs[tid * (RB + 1) + c] : 0.0;
    if (ii < In) Ahat[ii + (int64_t)In * c] = v;
    const double q = warp_sum(v * v);
    if (lane == 0) red[wid][c] = q;
  }
  {
    const double q = warp_sum(inner);
    if (lane == 0) red[wid][RB] = q;
  }
  __syncthreads();
  for (int c = tid; c <= RB; c += blockDim.x) {
    double v = 0.0;
    if (c < R || c == RB)
      for (int q = 0; q < BT / 32; ++q) v += red[q][c];
    part[(int64_t)blockIdx.x * (RB + 1) + c] = v;
  }
}

}  // namespace cpqr
