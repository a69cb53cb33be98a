// CholeskyQR2 for the I_n x R factor panels (Alg. 2 line 12), with a device-side
// switch to the Householder TSQR (rowqr.cuh) when the panel is too ill-conditioned.
//
//   pass 1:  G1 = A^T A (per-block partials, fixed-order sum), G1 = L1 L1^T, Q1 = A L1^{-T}
//   pass 2:  G2 = Q1^T Q1,  G2 = L2 L2^T,  Q = Q1 L2^{-T},  R = L2^T L1^T
// Both passes yield the unique thin QR with diag(R) > 0 (reading 6); after pass 2 ||Q^T Q - I|| =
// O(eps) when kappa(A) < ~1e7.  k_cq_chol1 estimates kappa(A) ~ max(L1_jj)/min(L1_jj) and sets
// FLAG_USE_HOUSEHOLDER when it exceeds kCqKappaMax or a pivot is not positive; every CholeskyQR
// kernel after it then returns immediately and the Householder kernels (which otherwise return at
// once) produce Q, R -- all launches stay in the CUDA graph.
//
// In solve mode the first kernel also forms Ahat(i,:) (substitution with R0 or W M for the SVD
// variant) and factors Ahat itself: lambda_c^2 = G1(c,c), A_n = Ahat diag(1/lambda)
// and R_n = R_hat diag(1/lambda) (the Q factor is unchanged by the positive column scaling).
#pragma once
#include <cooperative_groups.h>
#include <cstdio>

#include "common.cuh"
#include "rowsolve.cuh"

namespace cpqr {

constexpr double kCqKappaMax = 1.0e5;
#ifndef CPQR_CQ_CLOSED_FORM
#define CPQR_CQ_CLOSED_FORM 1
#endif
constexpr bool kCqClosedForm = CPQR_CQ_CLOSED_FORM != 0;  // second CholeskyQR pass in closed form
constexpr unsigned FLAG_USE_HOUSEHOLDER = 0x200u;
constexpr unsigned FLAG_VN_HOUSEHOLDER = 0x400u;  // the CholeskyQR2 V_n QR handed over to K2
constexpr unsigned FLAG_PEER_TIMEOUT = 0x800u;    // k_peer_combine gave up waiting for a rank

struct CqArgs {
  const double* A;   // solve = 0: m x R column-major input
  int m, R, nb, mb;  // row blocks of mb rows
  int solve;
  const double* W;   // m x R row-major
  const double* Rm;  // R0 (variant 1) or M (variant 2)
  const double* R0;
  int variant;
  double* Ahat;      // out (solve): unnormalised solution, column-major
  double* Q1;        // scratch: m x R column-major
  double* Gp;        // scratch: nb x R x R Gram partials
  double* innerp;    // scratch: nb partial <W, Ahat R0^T>
  double* R1;        // scratch: R x R upper (L1^T)
  double* R2;        // scratch: R x R upper (L2^T)
  double* Q;         // out: m x R column-major
  double* Qt;        // out: m x RQ row-major, zero padded
  int RQ;
  double* Rn;        // out: R x R
  double* Aout;      // out (solve): A_n
  double* lam;       // out (solve)
  unsigned* flags;
  int do_fit;
  const double* nX2;
  double* fit;
  unsigned hh_bit;  // flag bit of the Householder-fallback decision (0: FLAG_USE_HOUSEHOLDER)
  double shift_c;   // > 0: shifted CholeskyQR pass (k_cq_chol1 factors G + shift_c tr(G) I, no guard)
};
__device__ __forceinline__ unsigned cq_hh_bit(const CqArgs& a) { return a.hh_bit ? a.hh_bit : FLAG_USE_HOUSEHOLDER; }

// Upper triangle of the block Gram from a shared-memory panel P (rows x R, leading dim ld).
__device__ __forceinline__ void cq_block_gram(const double* P, int ld, int rows, int R, double* out) {
  const int npairs = R * (R + 1) / 2;
  for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
    int p = 0, rem = e;  // (p, q) with p <= q, row-major over the upper triangle
    while (rem >= R - p) { rem -= R - p; ++p; }
    const int q = p + rem;
    const double* cp = P + (int64_t)ld * p;
    const double* cq = P + (int64_t)ld * q;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = 0;
    for (; i + 3 < rows; i += 4) {
      s0 = fma(cp[i], cq[i], s0);
      s1 = fma(cp[i + 1], cq[i + 1], s1);
      s2 = fma(cp[i + 2], cq[i + 2], s2);
      s3 = fma(cp[i + 3], cq[i + 3], s3);
    }
    for (; i < rows; ++i) s0 = fma(cp[i], cq[i], s0);
    const double s = (s0 + s1) + (s2 + s3);
    out[p + R * q] = s;
    out[q + R * p] = s;
  }
}

// pass-1 Gram (and, in solve mode, the solve of Ahat).  blockDim = 32 * ceil(mb/32) <= 256.
template <int RB>
__global__ void __launch_bounds__(256) k_cq_gram1(CqArgs a) {
  extern __shared__ double P[];  // rows x R, ld = rows | 1
  __shared__ double Ms[RB * RB], R0s[RB * RB], redi[8];
  const int b = blockIdx.x, R = a.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (b == 0 && tid == 0) atomicAnd(a.flags, ~cq_hh_bit(a));  // per-mode decision
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0, ld = rows | 1;
  if (!a.solve) {
    // blockDim >= rows: one row per thread, eight columns' loads in flight
    if (tid < rows) {
      int c = 0;
      for (; c + 8 <= R; c += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = a.A[r0 + tid + (int64_t)a.m * (c + q)];
#pragma unroll
        for (int q = 0; q < 8; ++q) P[tid + ld * (c + q)] = v[q];
      }
      for (; c < R; ++c) P[tid + ld * c] = a.A[r0 + tid + (int64_t)a.m * c];
    }
  } else {
    for (int e = tid; e < RB * RB; e += blockDim.x) {
      const int r = e % RB, c = e / RB;
      Ms[e] = (r < R && c < R) ? a.Rm[r + R * c] : 0.0;
      R0s[e] = (r < R && c < R) ? a.R0[r + R * c] : 0.0;
    }
    __syncthreads();
    double inner = 0.0;
    if (tid < rows) {
      const int i = r0 + tid;
      double wv[RB], x[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) wv[k] = (k < R) ? a.W[(int64_t)i * R + k] : 0.0;
      if (a.variant == 2) {  // x = w M, M = U S^+ V^T
#pragma unroll
        for (int c = 0; c < RB; ++c) {
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < RB; ++r) s = fma(wv[r], Ms[r + RB * c], s);
          x[c] = s;
        }
      } else {  // Ahat R0^T = W by back substitution
#pragma unroll
        for (int j = RB - 1; j >= 0; --j) {
          double acc = wv[j];
#pragma unroll
          for (int l = j + 1; l < RB; ++l) acc = fma(-x[l], Ms[j + RB * l], acc);
          x[j] = (j < R) ? acc / Ms[j + RB * j] : 0.0;
        }
      }
      if (a.do_fit) {  // <W, Ahat R0^T>
#pragma unroll
        for (int c = 0; c < RB; ++c) {
          double t = 0.0;
#pragma unroll
          for (int l = c; l < RB; ++l) t = fma(x[l], R0s[c + RB * l], t);
          inner = fma(wv[c], t, inner);
        }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (k < R) {
          P[tid + ld * k] = x[k];
          a.Ahat[i + (int64_t)a.m * k] = x[k];
        }
    }
    inner = warp_sum(inner);
    if (lane == 0) redi[wid] = inner;
  }
  __syncthreads();
  if (a.solve && tid == 0) {
    double v = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) v += redi[q];
    a.innerp[b] = v;
  }
  cq_block_gram(P, ld, rows, R, a.Gp + (int64_t)b * R * R);
}

// Sum the block Grams (fixed order) and Cholesky-factor them: returns R1 = L^T (upper) in
// shared memory Ls (R x R column-major); pass 1 also decides the Householder fallback.
__device__ void cq_chol(const CqArgs& a, double* Gs, double* Ls, bool pass1, bool* ok_out) {
  const int R = a.R, tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < R * R; e += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < a.nb; ++b) s += a.Gp[(int64_t)b * R * R + e];
    Gs[e] = s;
  }
  __syncthreads();
  const bool shifted = pass1 && a.shift_c > 0.0;
  if (shifted && tid == 0) {  // shifted CholeskyQR (Fukaya et al.): G + s I, s = c ||A||_F^2 >= c ||A||_2^2
    double tr = 0.0;
    for (int j = 0; j < R; ++j) tr += Gs[j + R * j];
    const double sh = a.shift_c * tr;
    for (int j = 0; j < R; ++j) Gs[j + R * j] += sh;
  }
  __syncthreads();
  if (tid < 32) {  // warp 0: left-looking Cholesky, lane i owns row i of L (R <= 32)
    bool ok = true;
    double dmax = 0.0, dmin = 1e308;
    for (int j = 0; j < R; ++j) {
      // L(i, j) for i >= j: G(i,j) - sum_{k<j} L(i,k) L(j,k)
      double s = (lane < R) ? Gs[lane + R * j] : 0.0;
      for (int k = 0; k < j; ++k) {
        const double ljk = Ls[k + R * j];  // R1(k, j) = L(j, k)
        const double lik = (lane < R) ? Ls[k + R * lane] : 0.0;
        s = fma(-lik, ljk, s);
      }
      const double djj = __shfl_sync(0xffffffffu, s, j);
      if (!(djj > 0.0)) ok = false;
      const double ljj = sqrt(fmax(djj, 0.0));
      dmax = fmax(dmax, ljj);
      dmin = fmin(dmin, ljj);
      if (lane == j) Ls[j + R * j] = ljj;
      else if (lane > j && lane < R) Ls[j + R * lane] = (ljj > 0.0) ? s / ljj : 0.0;  // R1(j, lane)
      __syncwarp();
    }
    if (lane == 0) *ok_out = ok && (dmin > 0.0) && (shifted || dmax / dmin < (pass1 ? kCqKappaMax : 1.0e3));
  }
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int r = e % R, c = e / R;
    if (r > c) Ls[e] = 0.0;
  }
  __syncthreads();
}

// First level of the Gram-partial sum for very tall panels (nb > 1024 row blocks, e.g. the
// 10-way sine of sums' 134M-row V_n): CTA g adds blocks [g per, (g+1) per) in order; the Cholesky
// kernels then add the <= 1024 group sums in order (fixed two-level order, deterministic).  Eight
// loads in flight per thread (the adds stay in block order): with one it ran at 50 GB/s.
__global__ void k_reduce_gp(const double* __restrict__ in, int nb, int RR, int per, double* __restrict__ out) {
  const int g = blockIdx.x, b0 = g * per, b1 = min(nb, b0 + per);
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    double s = 0.0;
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(in + (int64_t)(b + q) * RR + e);
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q];
    }
    for (; b < b1; ++b) s += __ldcg(in + (int64_t)b * RR + e);
    out[(int64_t)g * RR + e] = s;
  }
}

__global__ void __launch_bounds__(256) k_cq_chol1(CqArgs a) {
  __shared__ double Gs[32 * 32], Ls[32 * 32];
  __shared__ bool ok;
  cq_chol(a, Gs, Ls, true, &ok);
  if (!ok) {
    if (threadIdx.x == 0) atomicOr(a.flags, cq_hh_bit(a));
    return;
  }
  for (int e = threadIdx.x; e < a.R * a.R; e += blockDim.x) a.R1[e] = Ls[e];
}

// Row-wise triangular solve y R1 = x for this block's rows (x = A or Ahat rows for pass 1, Q1 for
// pass 2).  pass 1: write Q1 and its block Gram.  pass 2: write Q, Qt (and A_n in solve mode).
template <int RB>
__global__ void __launch_bounds__(256) k_cq_apply(CqArgs a, int pass) {
  extern __shared__ double P[];
  __shared__ double Rs[RB * RB];
  __shared__ unsigned fl;
  if (threadIdx.x == 0) fl = *a.flags;
  __syncthreads();
  if (fl & cq_hh_bit(a)) return;
  const int b = blockIdx.x, R = a.R, tid = threadIdx.x;
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0, ld = rows | 1;
  const double* Rf = (pass == 1) ? a.R1 : a.R2;
  for (int e = tid; e < RB * RB; e += blockDim.x) {
    const int r = e % RB, c = e / RB;
    Rs[e] = (r < R && c < R) ? Rf[r + R * c] : 0.0;
  }
  __syncthreads();
  const double* src = (pass == 1) ? (a.solve ? a.Ahat : a.A) : a.Q1;
  if (tid < rows) {
    const int i = r0 + tid;
    double x[RB], y[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) x[k] = (k < R) ? src[i + (int64_t)a.m * k] : 0.0;
#pragma unroll
    for (int j = 0; j < RB; ++j) {  // y_j = (x_j - sum_{l<j} y_l R1(l,j)) / R1(j,j)
      double acc = x[j];
#pragma unroll
      for (int l = 0; l < j; ++l) acc = fma(-y[l], Rs[l + RB * j], acc);
      y[j] = (j < R) ? acc / Rs[j + RB * j] : 0.0;
    }
    if (pass == 1) {
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (k < R) { a.Q1[i + (int64_t)a.m * k] = y[k]; P[tid + ld * k] = y[k]; }
    } else {
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (k < R) a.Q[i + (int64_t)a.m * k] = y[k];
      if (a.Qt) {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (k < a.RQ) a.Qt[(int64_t)i * a.RQ + k] = (k < R) ? y[k] : 0.0;
        for (int k = RB; k < a.RQ; ++k) a.Qt[(int64_t)i * a.RQ + k] = 0.0;
      }
      if (a.solve) {  // A_n = Ahat / lambda (zero column -> e_1, reading 10)
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          if (k >= R) continue;
          const double l = a.lam[k];
          const int64_t e = i + (int64_t)a.m * k;
          a.Aout[e] = (l > 0.0) ? a.Ahat[e] / l : (i == 0 ? 1.0 : 0.0);
        }
      }
    }
  }
  if (pass == 1) {
    __syncthreads();
    cq_block_gram(P, ld, rows, R, a.Gp + (int64_t)b * R * R);
  }
}

// pass-2 Cholesky, R = L2^T L1^T, lambda / R_n scaling and the fast fit.
__global__ void __launch_bounds__(256) k_cq_chol2(CqArgs a, const double* G1diag_src) {
  __shared__ double Gs[32 * 32], Ls[32 * 32], R1s[32 * 32], lam[32], red[8];
  __shared__ bool ok;
  __shared__ unsigned fl;
  if (threadIdx.x == 0) fl = *a.flags;
  __syncthreads();
  if (fl & cq_hh_bit(a)) return;
  const int R = a.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < R * R; e += blockDim.x) R1s[e] = a.R1[e];
  cq_chol(a, Gs, Ls, false, &ok);  // Ls = R2 = L2^T
  // safety: after pass 1 the Gram of Q1 must be I to O(kappa^2 eps); otherwise fall back
  __shared__ double emax[8];
  {
    double e = 0.0;
    for (int q = tid; q < R * R; q += blockDim.x) e = fmax(e, fabs(Gs[q] - ((q % R) == (q / R) ? 1.0 : 0.0)));
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (lane == 0) emax[wid] = e;
  }
  __syncthreads();
  if (tid == 0) {
    double e = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) e = fmax(e, emax[w]);
    if (!ok || !(e < 1.0e-4)) { atomicOr(a.flags, cq_hh_bit(a)); fl = cq_hh_bit(a); }
  }
  __syncthreads();
  if (fl & cq_hh_bit(a)) return;
  if (a.solve && tid < R) {  // lambda_c = ||Ahat(:,c)||_2 = sqrt(G1(c,c)) = ||R1(:,c)||_2
    double s = 0.0;
    for (int k = 0; k <= tid; ++k) s = fma(R1s[k + R * tid], R1s[k + R * tid], s);
    lam[tid] = sqrt(s);
    a.lam[tid] = lam[tid];
    if (!isfinite(lam[tid])) atomicOr(a.flags, FLAG_NONFINITE);
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += blockDim.x) a.R2[e] = Ls[e];
  for (int e = tid; e < R * R; e += blockDim.x) {  // R = R2 R1 (upper x upper), then / lambda
    const int r = e % R, c = e / R;
    double s = 0.0;
    for (int k = r; k <= c; ++k) s = fma(Ls[r + R * k], R1s[k + R * c], s);
    if (a.solve && lam[c] > 0.0) s /= lam[c];
    a.Rn[e] = (r <= c) ? s : 0.0;
    Gs[e] = (r <= c) ? s : 0.0;
  }
  (void)G1diag_src;
  __syncthreads();
  if (a.do_fit) {  // ||Xh||^2 = <R0^T R0, diag(lam) R_n^T R_n diag(lam)>; <W, Ahat R0^T> from partials
    for (int e = tid; e < R * R; e += blockDim.x) Ls[e] = a.R0[e];
    __syncthreads();
    double q = 0.0;
    for (int e = tid; e < R * R; e += blockDim.x) {
      const int x = e % R, y = e / R;
      double g0 = 0.0, g1 = 0.0;
      for (int k = 0; k <= min(x, y); ++k) {
        g0 = fma(Ls[k + R * x], Ls[k + R * y], g0);
        g1 = fma(Gs[k + R * x], Gs[k + R * y], g1);
      }
      q = fma(g0, lam[x] * lam[y] * g1, q);
    }
    q = warp_sum(q);
    if (lane == 0) red[wid] = q;
    __syncthreads();
    if (tid == 0) {
      double nxh2 = 0.0, inner = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) nxh2 += red[w];
      for (int b = 0; b < a.nb; ++b) inner += a.innerp[b];
      const double nx2 = *a.nX2;
      *a.fit = 1.0 - sqrt(fmax(0.0, nx2 - 2.0 * inner + nxh2)) / sqrt(nx2);
    }
  }
}


// ================================================================ single-launch cluster variant
// Cluster of nb <= 8 CTAs (one per row block of <= 256 rows, one thread per row, rows kept in
// registers).  Block Grams on the FP64 tensor cores from a shared-memory panel, summed in a fixed
// order over the cluster through distributed shared memory by EVERY CTA (so each CTA factors the
// same G redundantly and no broadcast is needed), Cholesky by one warp with the rows in
// registers, triangular solves in registers.  4 cluster barriers for the whole factor QR.

// G (RB x RB, symmetric, ld RB) = P^T P for the shared panel P (rows4 x RB, leading dim ld,
// zero-padded rows/columns), DMMA 8x8x4 tiles of the upper triangle, one warp per tile.
template <int RB>
__device__ __forceinline__ void cq_gram_dmma(const double* P, int ld, int rows4, double* G) {
  constexpr int T = RB / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  int tile = 0;
  for (int pi = 0; pi < T; ++pi)
    for (int qi = pi; qi < T; ++qi, ++tile) {
      if (tile % nw != wid) continue;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;  // two independent DMMA chains
      const double* cp = P + (int64_t)ld * (8 * pi + g);
      const double* cq = P + (int64_t)ld * (8 * qi + g);
      int k0 = 0;
#pragma unroll 2
      for (; k0 + 8 <= rows4; k0 += 8) {
        dmma(d0, d1, cp[k0 + t], cq[k0 + t]);
        dmma(e0, e1, cp[k0 + 4 + t], cq[k0 + 4 + t]);
      }
      if (k0 < rows4) dmma(d0, d1, cp[k0 + t], cq[k0 + t]);
      d0 += e0;
      d1 += e1;
      const int r = 8 * pi + g, c0 = 8 * qi + 2 * t;
      G[r + RB * c0] = d0;
      G[r + RB * (c0 + 1)] = d1;
      G[c0 + RB * r] = d0;
      G[(c0 + 1) + RB * r] = d1;
    }
}

// ----------------------------------------------------------------- compact (I-cache friendly) variant
// CholeskyQR2 in one cluster launch; every per-row quantity lives in a shared-memory panel row
// (owner thread tid, stride 1 across threads -> conflict free) and all loops are rolled: the
// fully unrolled register version compiles to >600 KB of SASS and thrashes the 32 KB instruction
// cache.  Q1 = A R1^{-1} and Q = Q1 R2^{-1} use the explicit upper-triangular inverses (column-
// parallel back substitution by R threads), turning the per-row solves into independent dot
// products; the paper's own solve Ahat R0^T = W keeps row-wise substitution.

// Right-looking Cholesky of Gs (R x R used, RB ld) with a 2-D thread map: lane = row i, warp kk
// updates columns k = kk (mod nwarps) -- no integer division, all loads of a column step issued
// together, one barrier per column.  The update expression and order equal cq_chol_par's.
// On exit Ru = L^T (upper, zero padded), invd[j] = 1/L_jj (0 for j >= R).
template <int RB>
__device__ __noinline__ bool cq_chol_2d(double* Gs, int R, double* Ru, double* invd, double* ratio) {
  const int tid = threadIdx.x, i = tid & 31, kk = tid >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  // critical path per column: LDS of the pivot, its reciprocal (__drcp_rn == 1.0 / d, correctly
  // rounded), one FMA per owned entry, barrier; square roots are taken after the loop
  if (nw >= 8) {  // warps 0..7 map the columns (k = kk mod 8); any further warps only join the barriers
#pragma unroll 1
    for (int j = 0; j < R; ++j) {
      // every load of the column step first (one shared-memory round trip), then the reciprocal
      const bool act = i > j && i < R && kk < 8;
      const double d = Gs[j + RB * j];
      double gi = 0.0, gk[RB / 8], gik[RB / 8];
#pragma unroll
      for (int q = 0; q < RB / 8; ++q) {
        const int k = kk + 8 * q;
        const bool on = act && k > j && k <= i;
        gk[q] = on ? Gs[k + RB * j] : 0.0;
        gik[q] = on ? Gs[i + RB * k] : 0.0;
      }
      if (act) gi = Gs[i + RB * j];
      if (act) {
        const double id = (d > 0.0) ? __drcp_rn(d) : 0.0;
        const double gij = -gi * id;
#pragma unroll
        for (int q = 0; q < RB / 8; ++q) {
          const int k = kk + 8 * q;
          if (k > j && k <= i) Gs[i + RB * k] = fma(gij, gk[q], gik[q]);
        }
      }
      __syncthreads();
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < R; ++j) {
      const double d = Gs[j + RB * j];
      if (i > j && i < R) {
        const double id = (d > 0.0) ? __drcp_rn(d) : 0.0;
        const double gij = -Gs[i + RB * j] * id;
#pragma unroll 1
        for (int k = kk; k < RB; k += nw)
          if (k > j && k <= i) Gs[i + RB * k] = fma(gij, Gs[k + RB * j], Gs[i + RB * k]);
      }
      __syncthreads();
    }
  }
  // pivots d_j = Gs(j, j) are final; L_jj = sqrt(d_j); warp 0 also forms ok / max L_jj / min L_jj
  bool ok = true;
  double dmax = 0.0, dmin = 1e308;
  if (tid < 32) {
    const double d = (tid < R) ? Gs[tid + RB * tid] : 1.0;
    const double l = sqrt(fmax(d, 0.0));
    if (tid < RB) invd[tid] = (tid < R && l > 0.0) ? 1.0 / l : 0.0;
    ok = __all_sync(0xffffffffu, d > 0.0);
    dmax = (tid < R) ? l : 0.0;
    dmin = (tid < R) ? l : 1e308;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int e = tid; e < RB * RB; e += blockDim.x) {  // Ru(r, c) = L(c, r) = G(c, r) / L_rr, Ru(r, r) = L_rr
    const int r = e % RB, c = e / RB;
    double v = 0.0;
    if (r < R && c < R && r <= c) v = (r == c) ? sqrt(fmax(Gs[r + RB * r], 0.0)) : Gs[c + RB * r] * invd[r];
    Ru[e] = v;
  }
  __syncthreads();
  *ratio = (dmin > 0.0) ? dmax / dmin : 1e308;  // valid on thread 0 (the caller reads it there)
  return ok;
}

// sum_{c < nb} (value at p in cluster CTA c), c in increasing order (bitwise the rolled loop);
// the nb <= 8 remote loads are issued together instead of one DSMEM round trip per rank
__device__ __forceinline__ double cluster_sum_ordered(cooperative_groups::cluster_group& cl, double* p, int nb) {
  double v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = (c < nb) ? *cl.map_shared_rank(p, c) : 0.0;
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < nb) s += v[c];
  return s;
}

#ifdef CPQR_DEBUG_TIMING
#define CQ_T(k) do { if (threadIdx.x == 0) tstamp[k] = clock64(); } while (0)
#define CQ_DUMP() do { if (threadIdx.x == 0 && cluster.block_rank() == 0) printf("cq phases: %lld %lld %lld %lld %lld %lld %lld %lld | lam+sync %lld chol %lld sync %lld inv %lld | zero %lld load %lld solve %lld\n", tstamp[1]-tstamp[0], tstamp[2]-tstamp[1], tstamp[3]-tstamp[2], tstamp[4]-tstamp[3], tstamp[5]-tstamp[4], tstamp[6]-tstamp[5], tstamp[7]-tstamp[6], tstamp[8]-tstamp[7], tstamp[9]-tstamp[3], tstamp[10]-tstamp[9], tstamp[11]-tstamp[10], tstamp[12]-tstamp[11], tstamp[13]-tstamp[0], tstamp[14]-tstamp[13], tstamp[15]-tstamp[14]); } while (0)
#else
#define CQ_T(k) do {} while (0)
#define CQ_DUMP() do {} while (0)
#endif
template <int RB>
__global__ void __launch_bounds__(512) k_cq_compact(CqArgs a) {
#ifdef CPQR_DEBUG_TIMING
  __shared__ long long tstamp[16];
#endif
  CQ_T(0);
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double smq[];
  double* G1b = smq;
  double* G2b = G1b + RB * RB;
  double* Gs = G2b + RB * RB;
  double* R1s = Gs + RB * RB;
  double* R2s = R1s + RB * RB;
  double* Ui = R2s + RB * RB;  // (unused scratch; keeps the host smem size formula)
  double* Ms = Ui + RB * RB;
  double* R0s = Ms + RB * RB;
  __shared__ double lam[RB], invlam[RB], redi[32], innerb, inv1[RB], inv2[RB], invm[RB];
  __shared__ int okf;
  (void)Ui;
  const int nb = a.nb, R = a.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int b = (int)cluster.block_rank();
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0;
  const int rows4 = (rows + 3) & ~3, ld = (((int)blockDim.x + 15) & ~15) + 4;  // >= every thread's row
  double* X = R0s + RB * RB;   // panel of Ahat (or A) rows
  double* Y = X + ld * RB;     // panel of W / Q1 rows
  const int i = r0 + tid;
  const bool own = tid < rows;
  #pragma unroll 1
  for (int e = tid; e < 2 * ld * RB; e += blockDim.x) X[e] = 0.0;
  #pragma unroll 1
  for (int e = tid; e < 2 * RB * RB; e += blockDim.x) Ms[e] = 0.0;  // Ms, R0s
  pdl_wait();                // W, R0 / M of the predecessors are complete from here on
  if (tid == 0 && b == 0) atomicAnd(a.flags, ~cq_hh_bit(a));
  __syncthreads();
  CQ_T(13);
  // all global inputs in flight at once (cp.async), one wait
  if (a.solve) {
    #pragma unroll 1
    for (int e = tid; e < R * R; e += blockDim.x) {
      const int r = e % R, c = e / R;
      if (a.variant == 2 || r <= c) cp_async8(&Ms[r + RB * c], a.Rm + e);  // R0 upper / M dense
      if (r <= c) cp_async8(&R0s[r + RB * c], a.R0 + e);
    }
  }
  if (a.solve) {  // the CTA's W rows are one contiguous row-major block: coalesced copy
    #pragma unroll 4
    for (int e = tid; e < rows * R; e += blockDim.x) cp_async8(&Y[(e / R) + ld * (e % R)], a.W + (int64_t)r0 * R + e);
  } else if (own) {
    #pragma unroll 4
    for (int k = 0; k < R; ++k) cp_async8(&X[tid + ld * k], a.A + i + (int64_t)a.m * k);
  }
  cp_async_wait_all();
  __syncthreads();
  CQ_T(14);
  if (a.solve && a.variant != 2 && tid < RB) invm[tid] = (tid < R) ? 1.0 / Ms[tid + RB * tid] : 0.0;
  __syncthreads();
  // ---- 1. solve for the panel rows (Alg. 2 line 10)
  double inner = 0.0;
  if (a.solve) {
    if (a.variant == 2) {
      cq_row_gemv<RB>(Y + tid, X + tid, ld, Ms);  // x = w M, M = U S^+ V^T
    } else {
      #pragma unroll 8
      for (int k = 0; k < RB; ++k) X[tid + ld * k] = Y[tid + ld * k];
      cq_row_trsv<RB, true>(X + tid, ld, Ms, invm);  // Ahat R0^T = W
    }
    CQ_T(15);
    if (a.do_fit) inner = cq_row_wTx<RB>(Y + tid, X + tid, ld, R0s);  // <W, Ahat R0^T>
    if (own)
      #pragma unroll 8
      for (int k = 0; k < R; ++k) a.Ahat[i + (int64_t)a.m * k] = X[tid + ld * k];
  }
  inner = warp_sum(inner);
  if (lane == 0) redi[wid] = inner;
  __syncthreads();
  if (tid == 0) {
    double v = 0.0;
    #pragma unroll 1
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) v += redi[q];
    innerb = v;
  }
  CQ_T(1);
  // ---- 2. Gram of the panel, cluster sum, Cholesky -> R1, R1^{-1}
  cq_gram_dmma<RB>(X, ld, rows4, G1b);
  CQ_T(2);
  cluster.sync();
  #pragma unroll 1
  for (int e = tid; e < RB * RB; e += blockDim.x) Gs[e] = cluster_sum_ordered(cluster, G1b + e, nb);
  const double inner_all = cluster_sum_ordered(cluster, &innerb, nb);
  __syncthreads();
  CQ_T(3);
  if (a.solve && tid < R) {
    const double l = sqrt(Gs[tid + RB * tid]);  // lambda_c = ||Ahat(:,c)||_2
    lam[tid] = l;
    invlam[tid] = (l > 0.0) ? 1.0 / l : 0.0;
  }
  __syncthreads();
  if (a.solve && own) {  // A_n = Ahat diag(1/lambda) straight from the panel
    #pragma unroll 8
    for (int k = 0; k < R; ++k)
      a.Aout[i + (int64_t)a.m * k] = (lam[k] > 0.0) ? X[tid + ld * k] * invlam[k] : (i == 0 ? 1.0 : 0.0);
  }
  CQ_T(9);
  {
    double ratio;
    const bool ok = cq_chol_2d<RB>(Gs, R, R1s, inv1, &ratio);
    if (tid == 0) okf = ok && ratio < kCqKappaMax;
  }
  CQ_T(10);
  __syncthreads();
  CQ_T(11);
  if (!okf) {
    if (tid == 0 && b == 0) atomicOr(a.flags, cq_hh_bit(a));
    cluster.sync();
    return;
  }
  CQ_T(12);
  CQ_T(4);
  // ---- 3. Q1 = X R1^{-1}, Gram, Cholesky -> R2, R2^{-1}
  #pragma unroll 8
  for (int k = 0; k < RB; ++k) Y[tid + ld * k] = X[tid + ld * k];
  cq_row_trsv<RB, false>(Y + tid, ld, R1s, inv1);
  __syncthreads();
  CQ_T(5);
  cq_gram_dmma<RB>(Y, ld, rows4, G2b);
  cluster.sync();
  #pragma unroll 1
  for (int e = tid; e < RB * RB; e += blockDim.x) Gs[e] = cluster_sum_ordered(cluster, G2b + e, nb);
  bool small_e;
  {
    // ||G2 - I||_max must be O(kappa^2 eps); below 2^-30 the second Cholesky has a closed form
    bool bad = false, big = false;
    #pragma unroll 4
    for (int q = tid; q < RB * RB; q += blockDim.x) {
      const int r = q % RB, c = q / RB;
      if (r < R && c < R) {
        const double e = fabs(Gs[q] - (r == c ? 1.0 : 0.0));
        bad |= !(e < 1.0e-4);
        big |= !(e < 9.313225746154785e-10);  // 2^-30
      }
    }
    bad = __syncthreads_or(bad);
    small_e = !__syncthreads_or(big) && kCqClosedForm;
    if (tid == 0) okf = !bad;
  }
  if (small_e) {
    // G2 = I + E with max|E| < 2^-30 (CholeskyQR2's usual case, kappa(A)^2 eps small): the Cholesky
    // factor of I + E is R2 = I + U, U = strict upper part of E + diag(E) / 2, up to U^T U (entries
    // below R 2^-60 < eps) -- the same R2 to rounding without the 32-step dependent column chain
    #pragma unroll 1
    for (int e = tid; e < RB * RB; e += blockDim.x) {
      const int r = e % RB, c = e / RB;
      double v = 0.0;
      if (r < R && c < R && r <= c) v = (r == c) ? 1.0 + 0.5 * (Gs[e] - 1.0) : Gs[e];
      R2s[e] = v;
    }
    if (tid < RB) inv2[tid] = (tid < R) ? 1.0 / (1.0 + 0.5 * (Gs[tid + RB * tid] - 1.0)) : 0.0;
    __syncthreads();
  } else {
    double ratio;
    const bool ok = cq_chol_2d<RB>(Gs, R, R2s, inv2, &ratio);
    if (tid == 0) okf = okf && ok;
  }
  __syncthreads();
  if (!okf) {
    if (tid == 0 && b == 0) atomicOr(a.flags, cq_hh_bit(a));
    cluster.sync();
    return;
  }
  CQ_T(6);
  // ---- 4. Q = Q1 R2^{-1} (in the Y panel), outputs
  cq_row_trsv<RB, false>(Y + tid, ld, R2s, inv2);
  if (own) {
    #pragma unroll 8
    for (int k = 0; k < R; ++k) a.Q[i + (int64_t)a.m * k] = Y[tid + ld * k];
  }
  __syncthreads();
  if (a.Qt) {  // Qt rows of this CTA: one contiguous row-major block, written coalesced
    const int RQ = a.RQ;
    #pragma unroll 4
    for (int e = tid; e < rows * RQ; e += blockDim.x) {
      const int row = e / RQ, k = e - row * RQ;
      a.Qt[(int64_t)r0 * RQ + e] = (k < R) ? Y[row + ld * k] : 0.0;
    }
  }
  CQ_T(7);
  if (b == 0) {
    #pragma unroll 1
    for (int e = tid; e < RB * RB; e += blockDim.x) {  // R_n = R2 R1 diag(1/lambda)
      const int r = e % RB, c = e / RB;
      double s = 0.0;
      if (r <= c && c < R)
        #pragma unroll 4
        for (int k = r; k <= c; ++k) s = fma(R2s[r + RB * k], R1s[k + RB * c], s);
      if (a.solve && c < R && lam[c] > 0.0) s /= lam[c];
      Gs[e] = s;
      if (r < R && c < R) a.Rn[r + R * c] = s;
    }
    if (a.solve && tid < R) {
      a.lam[tid] = lam[tid];
      if (!isfinite(lam[tid])) atomicOr(a.flags, FLAG_NONFINITE);
    }
    if (a.do_fit) {  // ||Xh||^2 = <R0^T R0, diag(lam) R_n^T R_n diag(lam)>
      __syncthreads();
      double qq = 0.0;
      #pragma unroll 1
      for (int e = tid; e < R * R; e += blockDim.x) {
        const int xx = e % R, yy = e / R;
        double g0 = 0.0, g1 = 0.0;
        #pragma unroll 4
        for (int k = 0; k <= min(xx, yy); ++k) {
          g0 = fma(R0s[k + RB * xx], R0s[k + RB * yy], g0);
          g1 = fma(Gs[k + RB * xx], Gs[k + RB * yy], g1);
        }
        qq = fma(g0, lam[xx] * lam[yy] * g1, qq);
      }
      qq = warp_sum(qq);
      if (lane == 0) redi[wid] = qq;
      __syncthreads();
      if (tid == 0) {
        double nxh2 = 0.0;
        #pragma unroll 1
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) nxh2 += redi[w];
        const double nx2 = *a.nX2;
        *a.fit = 1.0 - sqrt(fmax(0.0, nx2 - 2.0 * inner_all + nxh2)) / sqrt(nx2);
      }
    }
  }
  CQ_T(8);
  cluster.sync();  // no CTA leaves while peers may read its shared memory
  CQ_DUMP();
}

}  // namespace cpqr
