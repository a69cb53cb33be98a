// Register-resident ("row-owner") Householder QR for the tall-skinny factor panels of the per-mode
// tail (Alg. 2 line 12): each thread owns one row of the panel in registers.
//
// Why: on sm_100a a dependent LDS.64 costs ~65-80 cycles and a 64-bit warp reduction ~180-320
// cycles (tools/ubench/lat_bench.cu), so column steps built from shared-memory dot loops are
// latency chains.  Here every column step is ONE block-wide vector reduction:
//   S_k = sum_{i > j} a_ij a_ik   for all k >= j   (S_j = ||x||^2 of the sub-column, S_k the dots)
// done by recursive-halving shuffles inside each warp and a fixed-order sum over warps, while the
// owner of row j publishes that row (x0 = a_jj and a_jk) through shared memory.  With the reflector
// v = [1; x / (x0 - beta)] scaled lazily, w_k = tau (a_jk + S_k / (x0 - beta)), so the norm and all
// dot products come out of the same reduction: two block barriers per column, no serial section.
// LAPACK dgeqr2 / dorg2r conventions (beta = -sign(x0) ||.||, tau = (beta - x0)/beta); diag(R) >= 0
// is applied by the callers (reading 6).  All reductions have a fixed order (deterministic).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace cpqr {

// Register-array element access with a runtime index, without demoting the array to local memory.
template <int RB>
__device__ __forceinline__ double pick(const double (&a)[RB], int j) {
  double r = 0.0;
#pragma unroll
  for (int k = 0; k < RB; ++k) r = (k == j) ? a[k] : r;
  return r;
}
template <int RB>
__device__ __forceinline__ void put(double (&a)[RB], int j, double v) {
#pragma unroll
  for (int k = 0; k < RB; ++k) a[k] = (k == j) ? v : a[k];
}

// Sum v[0..RB) over all threads of the block.  Result in fin[0..RB) (shared), visible to all
// threads on return.  red: (blockDim/32) x RB doubles of shared memory.  Two barriers.
template <int RB>
__device__ __forceinline__ void vec_reduce(double (&v)[RB], double* red, double* fin) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  int len = RB;
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    if (len > 1) {  // recursive halving: keep the half selected by this lane's bit h
      const bool hi = (lane & h) != 0;
      const int half = len >> 1;
#pragma unroll
      for (int q = 0; q < RB / 2; ++q) {
        if (q < half) {
          const double send = hi ? v[q] : v[q + half];
          const double keep = hi ? v[q + half] : v[q];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
      }
      len = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], h);
    }
  }
  // lane l now holds indices [l * RB/32, l * RB/32 + len) when RB >= 32, else index l >> log2(32/RB)
  if (RB >= 32) {
#pragma unroll
    for (int q = 0; q < (RB >= 32 ? RB / 32 : 1); ++q) red[wid * RB + lane * (RB / 32) + q] = v[q];
  } else {
    const int sh = (RB == 16) ? 1 : (RB == 8 ? 2 : (RB == 4 ? 3 : 4));
    if ((lane & ((1 << sh) - 1)) == 0) red[wid * RB + (lane >> sh)] = v[0];
  }
  __syncthreads();
  for (int t = tid; t < RB; t += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w * RB + t];
    fin[t] = s;
  }
  __syncthreads();
}

// In-place QR of the panel whose row `row` (0-based, or -1 for an idle thread) is a[0..R).  On
// exit a[k] = R(row, k) for k > row, a[row] = beta_row, a[j] = v_j[row] for j < row (reflector
// entries); tau[j], beta[j] in shared memory.  rowbuf: 2 x RB, red: nw x RB, fin: 2 x RB (shared).
template <int RB>
__device__ void rowqr_factor(double (&a)[RB], int row, int R, double* tau, double* beta, double* rowbuf,
                             double* red, double* fin) {
  for (int j = 0; j < R; ++j) {
    double* rj = rowbuf + (j & 1) * RB;
    double* fj = fin + (j & 1) * RB;
    double sv[RB];
    const double xj = (row > j) ? pick(a, j) : 0.0;
#pragma unroll
    for (int k = 0; k < RB; ++k) sv[k] = (k >= j && k < R) ? xj * a[k] : 0.0;
    if (row == j) {
#pragma unroll
      for (int k = 0; k < RB; ++k) rj[k] = a[k];
    }
    vec_reduce<RB>(sv, red, fj);
    const double s = fj[j], x0 = rj[j];
    double tj, bj, sc;
    if (s == 0.0) { tj = 0.0; bj = x0; sc = 0.0; }
    else {
      const double nrm = sqrt(x0 * x0 + s);
      bj = (x0 >= 0.0) ? -nrm : nrm;
      tj = (bj - x0) / bj;
      sc = 1.0 / (x0 - bj);
    }
    if (threadIdx.x == 0) { tau[j] = tj; beta[j] = bj; }
    if (row > j) {
      const double v = sc * xj;
      put(a, j, v);
      if (tj != 0.0) {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (k > j && k < R) a[k] -= tj * (rj[k] + sc * fj[k]) * v;
      }
    } else if (row == j) {
      if (tj != 0.0) {
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (k > j && k < R) a[k] -= tj * (rj[k] + sc * fj[k]);
      }
      put(a, j, bj);
    }
  }
}

// Explicit Q in place (dorg2r) after rowqr_factor: on exit a[0..R) is row `row` of Q (unsigned
// columns; the caller applies the diag(R) >= 0 sign fix).
template <int RB>
__device__ void rowqr_formq(double (&a)[RB], int row, int R, const double* tau, double* rowbuf, double* red,
                            double* fin) {
  // reflector entries of this row: v_j[row] = a[j] for j < row
  double vr[RB];
#pragma unroll
  for (int k = 0; k < RB; ++k) { vr[k] = a[k]; a[k] = 0.0; }
  // start from the first R columns of the identity
#pragma unroll
  for (int k = 0; k < RB; ++k) if (k == row) a[k] = 1.0;
  for (int j = R - 1; j >= 0; --j) {
    double* rj = rowbuf + (j & 1) * RB;
    double* fj = fin + (j & 1) * RB;
    const double tj = tau[j];
    double sv[RB];
    const double vj = (row > j) ? pick(vr, j) : 0.0;
#pragma unroll
    for (int k = 0; k < RB; ++k) sv[k] = (k > j && k < R) ? vj * a[k] : 0.0;
    if (row == j) {
#pragma unroll
      for (int k = 0; k < RB; ++k) rj[k] = a[k];
    }
    vec_reduce<RB>(sv, red, fj);
    // H_j = I - tau v v^T applied to columns k >= j; column j of the identity is e_j
    if (row >= j) {
      const double v = (row == j) ? 1.0 : vj;
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (k > j && k < R) a[k] -= tj * (rj[k] + fj[k]) * v;
      put(a, j, (row == j) ? 1.0 - tj : -tj * vj);
    }
  }
}

}  // namespace cpqr

// ------------------------------------------------------------------------------------------------
// Register-resident TSQR of the per-mode tail (same arguments as the shared-memory version in
// qr_kernels.cuh).  One thread per panel row; blockDim = 32 * ceil(rows / 32).
namespace cpqr {

// Apply H_{R-1} ... H_0 (reflector entries vr[j] = v_j[row], j < row) to the general rows a[0..R).
template <int RB>
__device__ void rowqr_apply(double (&a)[RB], const double (&vr)[RB], int row, int R, const double* tau,
                            double* rowbuf, double* red, double* fin) {
  for (int j = R - 1; j >= 0; --j) {
    double* rj = rowbuf + (j & 1) * RB;
    double* fj = fin + (j & 1) * RB;
    const double tj = tau[j];
    double sv[RB];
    const double vj = (row > j) ? pick(vr, j) : 0.0;
#pragma unroll
    for (int k = 0; k < RB; ++k) sv[k] = (k < R) ? vj * a[k] : 0.0;
    if (row == j) {
#pragma unroll
      for (int k = 0; k < RB; ++k) rj[k] = a[k];
    }
    vec_reduce<RB>(sv, red, fj);
    if (row >= j && tj != 0.0) {
      const double v = (row == j) ? 1.0 : vj;
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (k < R) a[k] -= tj * (rj[k] + fj[k]) * v;
    }
  }
}

struct RqArgs {
  const double* A;  // solve = 0: m x R column-major input
  int m, R, nleaf, mb;
  double* Rstack;   // (nleaf*R) x R column-major
  double* V;        // leaf rows (reflectors below the diagonal), mb x R column-major per leaf
  double* tauv;     // nleaf * R
  double* Qtop;     // (nleaf*R) x R column-major
  double* Q;        // out: m x R column-major
  double* Qt;       // out: m x RQ row-major, zero padded
  int RQ;
  double* Rn;       // out
  int solve;
  const double* W;  // m x R row-major
  const double* Rm; // R0 (variant 1) or M = (R0^T)^+ (variant 2)
  const double* R0;
  int variant;
  double* Ahat;     // out: unnormalised solution (column-major)
  double* part;     // nleaf x (R+1)
  double* Aout;     // out: normalised factor
  double* lam;
  unsigned* flags;
  int do_fit;
  const double* nX2;
  double* fit;
  int gated;        // 1: run only when the CholeskyQR2 path asked for the Householder fallback
};

__device__ __forceinline__ bool rq_skip(const RqArgs& a) {
  __shared__ unsigned fl;
  pdl_wait();  // the CholeskyQR2 launch before it has set (or not) the fallback flag
  if (threadIdx.x == 0) fl = a.gated ? *a.flags : 0x200u;
  __syncthreads();
  return (fl & 0x200u) == 0;
}

// The three TSQR phases as device bodies: launched as three kernels (k_rq_leaf/root/qform) or as
// one cluster kernel (k_rq_fused) with cluster barriers between the phases.
template <int RB>
__device__ __forceinline__ void rq_leaf_body(const RqArgs& a, const int b) {
  __shared__ double tau[RB], beta[RB], rowbuf[2 * RB], red[8 * RB], fin[2 * RB], Ms[RB * RB], R0s[RB * RB];
  __shared__ double redi[8];
  const int R = a.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0;
  const int row = (tid < rows) ? tid : -1;
  const int i = r0 + tid;
  double x[RB];
  if (!a.solve) {
#pragma unroll
    for (int k = 0; k < RB; ++k) x[k] = (row >= 0 && k < R) ? a.A[i + (int64_t)a.m * k] : 0.0;
  } else {
    for (int e = tid; e < RB * RB; e += blockDim.x) {
      const int r = e % RB, c = e / RB;
      Ms[e] = (r < R && c < R) ? a.Rm[r + R * c] : 0.0;
      R0s[e] = (r < R && c < R) ? a.R0[r + R * c] : 0.0;
    }
    __syncthreads();
    double wv[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) wv[k] = (row >= 0 && k < R) ? a.W[(int64_t)i * R + k] : 0.0;
    if (a.variant == 2) {  // x = w M  (M = U S^+ V^T)
#pragma unroll
      for (int c = 0; c < RB; ++c) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < RB; ++r) s = fma(wv[r], Ms[r + RB * c], s);
        x[c] = s;
      }
    } else {  // Ahat R0^T = W: x_j = (w_j - sum_{l>j} x_l R0(j,l)) / R0(j,j)
#pragma unroll
      for (int j = RB - 1; j >= 0; --j) {
        double acc = wv[j];
#pragma unroll
        for (int l = j + 1; l < RB; ++l) acc = fma(-x[l], Ms[j + RB * l], acc);
        x[j] = (j < R && row >= 0) ? acc / Ms[j + RB * j] : 0.0;
      }
    }
    double inner = 0.0;
    if (a.do_fit) {  // <W, Ahat R0^T>: sum_c w_c sum_{l>=c} x_l R0(c,l)
#pragma unroll
      for (int c = 0; c < RB; ++c) {
        double t = 0.0;
#pragma unroll
        for (int l = c; l < RB; ++l) t = fma(x[l], R0s[c + RB * l], t);
        inner = fma(wv[c], t, inner);
      }
    }
    if (row >= 0)
#pragma unroll
      for (int k = 0; k < RB; ++k)
        if (k < R) a.Ahat[i + (int64_t)a.m * k] = x[k];
    double sq[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) sq[k] = x[k] * x[k];
    vec_reduce<RB>(sq, red, fin);
    inner = warp_sum(inner);
    if (lane == 0) redi[wid] = inner;
    __syncthreads();
    if (tid < R) a.part[b * (R + 1) + tid] = fin[tid];
    if (tid == 0) {
      double v = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) v += redi[q];
      a.part[b * (R + 1) + R] = v;
    }
  }
  rowqr_factor<RB>(x, row, R, tau, beta, rowbuf, red, fin);
  const int ldr = a.nleaf * R;
  if (row >= 0 && row < R)
#pragma unroll
    for (int c = 0; c < RB; ++c)
      if (c < R) a.Rstack[b * R + row + (int64_t)ldr * c] = (c >= row) ? x[c] : 0.0;  // x[row] = beta
  if (row >= 0)
#pragma unroll
    for (int c = 0; c < RB; ++c)
      if (c < R) a.V[(int64_t)b * a.mb * R + row + rows * c] = x[c];
  __syncthreads();
  if (tid < R) a.tauv[b * R + tid] = tau[tid];
}

template <int RB>
__device__ __forceinline__ void rq_root_body(const RqArgs& a) {
  __shared__ double tau[RB], beta[RB], rowbuf[2 * RB], red[8 * RB], fin[2 * RB], lam[RB], r0s[RB * RB], rns[RB * RB];
  __shared__ double redq[8], inner_s;
  const int R = a.R, rows = a.nleaf * R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (a.solve) {  // lambda and <W, Ahat R0^T> from the leaf partials (fixed order)
    for (int t = tid; t <= R; t += blockDim.x) {
      double s = 0.0;
      for (int b = 0; b < a.nleaf; ++b) s += a.part[b * (R + 1) + t];
      if (t < R) {
        lam[t] = sqrt(s);
        a.lam[t] = lam[t];
        if (!isfinite(lam[t])) atomicOr(a.flags, 0x100u);
      } else {
        inner_s = s;
      }
    }
  }
  const int row = (tid < rows) ? tid : -1;
  double x[RB];
#pragma unroll
  for (int k = 0; k < RB; ++k) x[k] = (row >= 0 && k < R) ? a.Rstack[row + (int64_t)rows * k] : 0.0;
  __syncthreads();
  rowqr_factor<RB>(x, row, R, tau, beta, rowbuf, red, fin);
  __syncthreads();
  if (row >= 0 && row < R) {  // R_n = sign-fixed R_hat diag(1/lambda)
    const double sg = (beta[row] < 0.0) ? -1.0 : 1.0;
#pragma unroll
    for (int c = 0; c < RB; ++c) {
      if (c >= R) continue;
      double v = (c >= row) ? sg * x[c] : 0.0;
      if (a.solve && lam[c] > 0.0) v /= lam[c];
      a.Rn[row + R * c] = v;
      rns[row + RB * c] = v;
    }
  }
  rowqr_formq<RB>(x, row, R, tau, rowbuf, red, fin);
  if (row >= 0)
#pragma unroll
    for (int c = 0; c < RB; ++c)
      if (c < R) a.Qtop[row + (int64_t)rows * c] = (beta[c] < 0.0) ? -x[c] : x[c];
  if (a.do_fit) {  // ||Xh||^2 = <R0^T R0, diag(lam) R_n^T R_n diag(lam)>
    for (int e = tid; e < R * R; e += blockDim.x) r0s[(e % R) + RB * (e / R)] = a.R0[e];
    __syncthreads();
    double q = 0.0;
    for (int e = tid; e < R * R; e += blockDim.x) {
      const int xx = e % R, yy = e / R;
      double g0 = 0.0, g1 = 0.0;
      for (int k = 0; k <= min(xx, yy); ++k) {
        g0 = fma(r0s[k + RB * xx], r0s[k + RB * yy], g0);
        g1 = fma(rns[k + RB * xx], rns[k + RB * yy], g1);
      }
      q = fma(g0, lam[xx] * lam[yy] * g1, q);
    }
    q = warp_sum(q);
    if (lane == 0) redq[wid] = q;
    __syncthreads();
    if (tid == 0) {
      double nxh2 = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) nxh2 += redq[w];
      const double nx2 = *a.nX2;
      *a.fit = 1.0 - sqrt(fmax(0.0, nx2 - 2.0 * inner_s + nxh2)) / sqrt(nx2);
    }
  }
}

template <int RB>
__device__ __forceinline__ void rq_qform_body(const RqArgs& a, const int b) {
  __shared__ double tau[RB], rowbuf[2 * RB], red[8 * RB], fin[2 * RB];
  const int R = a.R, tid = threadIdx.x;
  const int r0 = b * a.mb, rows = min(a.m, r0 + a.mb) - r0;
  const int row = (tid < rows) ? tid : -1;
  const int i = r0 + tid;
  const int ldt = a.nleaf * R;
  double m[RB], vr[RB];
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    m[k] = (row >= 0 && row < R && k < R) ? a.Qtop[b * R + row + (int64_t)ldt * k] : 0.0;
    vr[k] = (row >= 0 && k < R) ? a.V[(int64_t)b * a.mb * R + row + rows * k] : 0.0;
  }
  if (tid < R) tau[tid] = a.tauv[b * R + tid];
  if (a.solve && row >= 0) {  // A_n = Ahat / lambda (zero column -> e_1, reading 10)
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      if (k >= R) continue;
      const double l = a.lam[k];
      const int64_t e = i + (int64_t)a.m * k;
      a.Aout[e] = (l > 0.0) ? a.Ahat[e] / l : (i == 0 ? 1.0 : 0.0);
    }
  }
  __syncthreads();
  rowqr_apply<RB>(m, vr, row, R, tau, rowbuf, red, fin);
  if (row >= 0) {
#pragma unroll
    for (int k = 0; k < RB; ++k)
      if (k < R) a.Q[i + (int64_t)a.m * k] = m[k];
    for (int k = 0; k < a.RQ; ++k) a.Qt[(int64_t)i * a.RQ + k] = (k < R) ? m[k] : 0.0;
  }
}

template <int RB>
__global__ void __launch_bounds__(256) k_rq_leaf(RqArgs a) {
  if (rq_skip(a)) return;
  rq_leaf_body<RB>(a, blockIdx.x);
}
template <int RB>
__global__ void __launch_bounds__(256) k_rq_root(RqArgs a) {
  if (rq_skip(a)) return;
  rq_root_body<RB>(a);
}
template <int RB>
__global__ void __launch_bounds__(256) k_rq_qform(RqArgs a) {
  if (rq_skip(a)) return;
  rq_qform_body<RB>(a, blockIdx.x);
}

// All three phases in one launch of ONE CTA (the leaves and the Q formations in turn): the overlap
// schedule's tail runs beside the next stream pass, where a co-scheduled cluster is not available
// and three gated launches cost ~8 us of the per-mode chain (C2) even when the fallback is not taken.
template <int RB>
__global__ void __launch_bounds__(256) k_rq_serial(RqArgs a) {
  if (rq_skip(a)) return;
  for (int b = 0; b < a.nleaf; ++b) {
    rq_leaf_body<RB>(a, b);
    __syncthreads();  // block-scope ordering of the leaf's global writes (Rstack, V, tau, partials)
  }
  rq_root_body<RB>(a);
  __syncthreads();
  for (int b = 0; b < a.nleaf; ++b) {
    rq_qform_body<RB>(a, b);
    __syncthreads();
  }
}

// All three phases in one launch: a cluster of nleaf (<= 8) CTAs.  The cluster barrier orders the
// leaves' global writes (Rstack, V, tau, partials) before the root reads them, and the root's
// (Q_top, lambda) before the Q formation.  Gated like the three kernels: every CTA reads the same
// flag word, so either all of them return at once or none does (no barrier is left waiting).
// Behind the CholeskyQR2 path this turns three gated launches per mode into one (2-3 % of a
// dimension-tree sweep on C2-C4).
template <int RB>
__global__ void __launch_bounds__(256) k_rq_fused(RqArgs a) {
  if (rq_skip(a)) return;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int b = (int)cl.block_rank();
  rq_leaf_body<RB>(a, b);
  cl.sync();
  if (b == 0) rq_root_body<RB>(a);
  cl.sync();
  rq_qform_body<RB>(a, b);
}

}  // namespace cpqr
