// Small per-mode kernels of the CP-ALS-QR hot path (sm_100a, fp64).  Everything here works on
// O(I_n R + R^N) data; the passes over the tensor X are in tma_kernels.cuh / ttm_kernels.cuh
// (and k_sumsq, once per set_tensor).
//
//   k_tall_fallback / hh_qr_block  one-CTA global-memory Householder QR of I_n x R for factors
//                   too tall for the shared-memory TSQR fallback (Alg. 2 lines 3/12,
//                   PAPER.md:351,360); the usual factor QR is CholeskyQR2 (cholqr.cuh)
//   k_q0_apply_tc   W_n = Y_(n) Q0 on DMMA (Alg. 2 line 9)
//   jacobi_pinv     one-sided Jacobi SVD of R0 -> M = U S^+ V^T
//   k_sumsq         ||X||^2 (fixed-order two-level reduction)
//   k_diag_contract, k_tail_ne   CP-ALS (Alg. 1) MTTKRP stage 2 and the
//                   Cholesky/LU solve, normalise, Gram, fast fit
//   k_resid_partial direct fit ||X - [[lambda; A]]||
// The V_n QR (k_kr_qr2) is in qr_kernels.cuh.
// All reductions are fixed-order (no floating-point atomics): results are bitwise reproducible.
#pragma once
#include "common.cuh"
#include "rowsolve.cuh"

namespace cpqr {

constexpr double kEps = 2.220446049250313e-16;

enum : unsigned { FLAG_ILLCOND_R0 = 1u, FLAG_NE_CHOL_FALLBACK = 2u, FLAG_SVD_TRUNCATED = 4u,
                  FLAG_NE_ILLCOND = 8u, FLAG_NONFINITE = 0x100u };
// NE: kappa(S_n) estimated as (max L_jj / min L_jj)^2 from the Cholesky factor; above this the
// normal equations lose more than ~8 of 16 digits (switch to QR when detected)
constexpr double kNeKappaMax = 1.0e8;

// ------------------------------------------------------------------------------ sum of squares
__global__ void k_sumsq_partial(const double* __restrict__ X, int64_t n, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  const int64_t n2 = n / 2;
  const double2* X2 = reinterpret_cast<const double2*>(X);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(X2 + i);
    s += v.x * v.x + v.y * v.y;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) s += X[n - 1] * X[n - 1];
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
// dst (D x rows, column-major) <- src (I x rows), I < D; the pad rows of dst are left untouched
__global__ void k_pad_rows(const double* __restrict__ src, int64_t I, int64_t D, int64_t rows, double* __restrict__ dst) {
  const int64_t n = I * rows;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / I, i = e - r * I;
    dst[r * D + i] = __ldcs(src + e);
  }
}
// Sum of the virtual ranks' partial results in rank order (CPQR_COMM_LOCAL's all-reduce):
// out[e] = (((p0[e] + p1[e]) + p2[e]) + ...); out may alias p[0].
constexpr int kMaxRanks = 16;
struct RankPtrs {
  const double* p[kMaxRanks];
};
__global__ void k_sum_ranks(RankPtrs a, int nr, int64_t n, double* out) {
  pdl_wait();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = a.p[0][e];
    for (int q = 1; q < nr; ++q) s += a.p[q][e];
    out[e] = s;
  }
}

// ------------------------------------------------------------- peer push-reduce of W_n
// The exchange of the slab data parallelism without a collective library (SURVEY.md 8(f) NEXT-2,
// DESIGN.md §8): every rank owns a RECEIVE WINDOW -- [2 parities][p slots][slot_elems] doubles, p
// arrival flags and an exchange counter (epoch) -- that its peers map (CUDA IPC over NVLink, or the
// same device for virtual ranks).  Exchange number e + 1 of source rank s:
//   push    the producing kernel (the Q0 apply's final sum, or k_peer_push) stores its result into
//           slot s, parity e & 1, of EVERY rank's window with plain stores; each CTA that finishes
//           rows fences at system scope and arrives on a grid counter; the last one to arrive
//           fences again, raises flag[s] = e + 1 on every rank and advances the
//           local epoch;
//   combine k_peer_combine on every rank waits until its p flags reach e + 1 (ld.acquire.sys),
//           then sums the p slots in rank order (n < N) or places them by rank (mode N), so the
//           result is bitwise identical on all ranks.
// No reset and no second barrier: the flags only grow, and a rank can start exchange e + 3 (same
// parity as e + 1) only after its own combine of e + 2, i.e. after every peer pushed e + 2, which
// each peer does after ITS combine of e + 1 (stream order) -- so slot parity e & 1 is free again.
struct PeerPush {
  double* dst[kMaxRanks];               // rank r's slot for this source rank (parity 0)
  unsigned long long* flag[kMaxRanks];  // rank r's arrival flag for this source rank
  unsigned long long* epoch;            // this source rank's exchange counter (its own window)
  unsigned* gcount;                     // arrivals of the pushing grid's finishing CTAs (self re-arming)
  int64_t parity_stride;                // elements between the two parities of a slot
  int np;                               // ranks (0: no push)
  int sysfence;                         // 1: every finishing CTA fences at system scope (see peer_push_done)
};
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Called by all threads of a CTA once its peer stores are issued; `finishers` CTAs of the grid
// call it exactly once each.  e: the epoch the CTA read before storing.  One thread per CTA fences:
// the barrier orders the CTA's stores before thread 0's fence, which is cumulative, so the arrival
// cannot overtake them; the last CTA to arrive observes every arrival (device-scope atomics on the
// local counter), fences at SYSTEM scope -- cumulative again over everything that happened before
// it, the other CTAs' peer stores included (PTX memory model: causality order is transitive over
// morally strong synchronisation) -- and only then raises the flags.  sysfence = 1 makes every
// arrival fence at system scope too (CPQR_PEER_FENCE=sys; ~4 us more per exchange on one GPU).
__device__ __forceinline__ void peer_push_done(const PeerPush& pp, unsigned long long e, unsigned finishers) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (pp.sysfence) __threadfence_system();
  else __threadfence();
  if (atomicAdd(pp.gcount, 1u) != finishers - 1u) return;
  __threadfence_system();
  for (int r = 0; r < pp.np; ++r)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;\n" ::"l"(pp.flag[r]), "l"(e + 1ull) : "memory");
  *pp.gcount = 0u;
  *pp.epoch = e + 1ull;
}
// Stand-alone push of n doubles (the NE MTTKRP partial, scalars such as ||X||^2 and the DIRECT
// residual); the QR path pushes from the Q0 apply itself.
__global__ void __launch_bounds__(256) k_peer_push(const double* __restrict__ src, int64_t n, PeerPush pp) {
  pdl_wait();
  const unsigned long long e = ld_relaxed_sys(pp.epoch);
  const int64_t off = (e & 1ull) ? pp.parity_stride : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = src[i];
    for (int r = 0; r < pp.np; ++r) pp.dst[r][off + i] = v;
  }
  peer_push_done(pp, e, gridDim.x);
}
// This rank's side of the exchange.  win: its window's data; cnt: elements per source rank;
// gather = 0: out[i] = ((s_0[i] + s_1[i]) + ...); gather = 1: out[q cnt + i] = s_q[i].  A peer that
// does not arrive within timeout_ns raises err_bit in *flags (the host reports ENCCL) and the
// kernel gives up waiting.
__global__ void __launch_bounds__(256)
k_peer_combine(const double* __restrict__ win, const unsigned long long* __restrict__ wflag,
               const unsigned long long* __restrict__ epoch, int np, int64_t slot_elems, int64_t cnt, int gather,
               double* __restrict__ out, unsigned* __restrict__ flags, unsigned err_bit,
               unsigned long long timeout_ns) {
  pdl_wait();
  const unsigned long long e = ld_relaxed_sys(epoch);  // advanced by this rank's own push
  if ((int)threadIdx.x < np) {
    unsigned long long t0 = 0, now;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t0));
    while (ld_acquire_sys(wflag + threadIdx.x) < e) {
      asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(now));
      if (now - t0 > timeout_ns) {
        atomicOr(flags, err_bit);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  const double* base = win + (((e - 1ull) & 1ull) ? (int64_t)np * slot_elems : 0);
  if (!gather) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
      double s = __ldcg(base + i);
      for (int q = 1; q < np; ++q) s += __ldcg(base + q * slot_elems + i);
      out[i] = s;
    }
  } else {
    const int64_t tot = cnt * np;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t q = i / cnt;
      out[i] = __ldcg(base + q * slot_elems + (i - q * cnt));
    }
  }
}

// The sweep's fit into the next slot of the per-call fits array (a device counter, reset by each
// cpqr_sweep), so one captured graph can hold several sweeps.
__global__ void k_store_fit(const double* __restrict__ fit, double* __restrict__ fits, unsigned* counter, int cap) {
  if (threadIdx.x == 0) {
    const unsigned i = *counter;
    if ((int)i < cap) fits[i] = *fit;
    *counter = i + 1;
  }
}

__global__ void k_sum_final(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------------- Householder QR (one CTA)
// In-place thin QR of the column-major m x R matrix Aw (leading dimension lda).  Reflectors in
// LAPACK dgeqr2 form: H_j = I - tau_j v v^T, v_j = 1, v_i (i > j) stored below the diagonal,
// beta_j = -sign(alpha) ||x|| on the diagonal.  Then R (upper triangle, rows sign-fixed so that
// diag >= 0, reading 6) is written to Rf (R x R column-major) and Aw is overwritten by the
// explicit Q (dorg2r order, columns sign-fixed to match).  Needs blockDim.x >= 64,
// smem: tau[R], beta[R], w[R], red[32].  Row range per column: rows j..rows_of(j)-1 where
// rows_of(j) = m for a dense matrix (staircase version: see k_kr_qr).
__device__ void hh_qr_block(double* Aw, int64_t lda, int m, int R, double* Rf, double* tau,
                            double* beta, double* w, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int j = 0; j < R; ++j) {
    double* colj = Aw + lda * j;
    double s = 0.0;
    for (int i = j + 1 + tid; i < m; i += nt) s += colj[i] * colj[i];
    s = block_sum(s, red);
    const double alpha = colj[j];
    const double nrm = sqrt(alpha * alpha + s);
    double tj, bj, scale;
    if (s == 0.0) {  // already reduced: H = I (dlarfg), beta = alpha
      tj = 0.0; bj = alpha; scale = 0.0;
    } else {
      bj = (alpha >= 0.0) ? -nrm : nrm;
      tj = (bj - alpha) / bj;
      scale = 1.0 / (alpha - bj);
    }
    __syncthreads();
    if (tj != 0.0)
      for (int i = j + 1 + tid; i < m; i += nt) colj[i] *= scale;
    if (tid == 0) { tau[j] = tj; beta[j] = bj; colj[j] = bj; }
    __syncthreads();
    if (tj != 0.0) {
      // w_k = A(j,k) + sum_{i>j} v_i A(i,k), k > j: one warp per column, fixed order
      for (int k = j + 1 + wid; k < R; k += nw) {
        const double* ck = Aw + lda * k;
        double d = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) d += colj[i] * ck[i];
        d = warp_sum(d);
        if (lane == 0) w[k] = ck[j] + d;
      }
      __syncthreads();
      const int ncol = R - j - 1;
      const int64_t tot = (int64_t)ncol * (m - j);
      for (int64_t e = tid; e < tot; e += nt) {
        const int k = j + 1 + (int)(e / (m - j));
        const int i = j + (int)(e % (m - j));
        const double v = (i == j) ? 1.0 : colj[i];
        Aw[i + lda * k] -= tj * w[k] * v;
      }
      __syncthreads();
    }
  }
  // R factor with sign fix
  for (int e = tid; e < R * R; e += nt) {
    const int r = e % R, c = e / R;
    double v = 0.0;
    if (r < c) v = Aw[r + lda * c];
    else if (r == c) v = beta[r];
    if (beta[r] < 0.0) v = -v;
    Rf[r + R * c] = v;
  }
  __syncthreads();
  // explicit Q, dorg2r: j = R-1..0
  for (int j = R - 1; j >= 0; --j) {
    double* colj = Aw + lda * j;
    const double tj = tau[j];
    if (j < R - 1 && tj != 0.0) {
      for (int k = j + 1 + wid; k < R; k += nw) {
        const double* ck = Aw + lda * k;
        double d = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) d += colj[i] * ck[i];
        d = warp_sum(d);
        if (lane == 0) w[k] = ck[j] + d;  // v_j = 1
      }
      __syncthreads();
      const int ncol = R - j - 1;
      const int64_t tot = (int64_t)ncol * (m - j);
      for (int64_t e = tid; e < tot; e += nt) {
        const int k = j + 1 + (int)(e / (m - j));
        const int i = j + (int)(e % (m - j));
        const double v = (i == j) ? 1.0 : colj[i];
        Aw[i + lda * k] -= tj * w[k] * v;
      }
      __syncthreads();
    }
    for (int i = tid; i < m; i += nt) {
      if (i < j) colj[i] = 0.0;
      else if (i == j) colj[i] = 1.0 - tj;
      else colj[i] = -tj * colj[i];
    }
    __syncthreads();
  }
  // column sign fix of Q to match diag(R) >= 0
  for (int64_t e = tid; e < (int64_t)m * R; e += nt) {
    const int c = (int)(e / m);
    if (beta[c] < 0.0) Aw[(e % m) + lda * c] = -Aw[(e % m) + lda * c];
  }
  __syncthreads();
}

// Householder fallback for factors too tall for the shared-memory TSQR (Alg. 2 lines 10-12,
// PAPER.md:358-360), one CTA over global memory.  Runs only if gate_bit is set in *flags (the
// CholeskyQR2 path rejected the panel) or gate_bit == 0 (Householder forced).  solve = 1: Ahat
// (m x R column-major) is already formed (by k_cq_gram1 or k_solve_rows); lambda_c = ||Ahat(:,c)||,
// A_n = Ahat / lambda (zero column -> e_1, reading 10), then Q_n R_n = A_n.  solve = 0: Q R = A.
// Then the TMA panel Qt and, with do_fit, the fast fit from R0, R_n, lambda and
// the <W, Ahat R0^T> partials innerp[b * istride] (b < ninner).
struct TallArgs {
  const double* A;     // solve = 0: input panel
  const double* Ahat;  // solve = 1
  int m, R, RQ, solve;
  double *Q, *Qt, *Rn, *Aout, *lam;
  unsigned* flags;
  unsigned gate_bit;
  int do_fit;
  const double* innerp;
  int ninner, istride;
  const double* R0;
  const double* nX2;
  double* fit;
};
__global__ void __launch_bounds__(1024) k_tall_fallback(TallArgs a) {
  __shared__ double tau[64], beta[64], w[64], red[32], lam[64];
  __shared__ unsigned fl;
  if (threadIdx.x == 0) fl = *a.flags;
  __syncthreads();
  if (a.gate_bit && !(fl & a.gate_bit)) return;
  const int m = a.m, R = a.R, tid = threadIdx.x, nt = blockDim.x;
  if (a.solve) {
    for (int c = 0; c < R; ++c) {
      double s = 0.0;
      for (int i = tid; i < m; i += nt) s = fma(a.Ahat[i + (int64_t)m * c], a.Ahat[i + (int64_t)m * c], s);
      s = block_sum(s, red);
      if (tid == 0) {
        lam[c] = sqrt(s);
        a.lam[c] = lam[c];
        if (!isfinite(lam[c])) atomicOr(a.flags, FLAG_NONFINITE);
      }
      __syncthreads();
    }
    for (int c = 0; c < R; ++c) {
      const double l = lam[c];
      for (int i = tid; i < m; i += nt) {
        const int64_t e = i + (int64_t)m * c;
        const double v = (l > 0.0) ? a.Ahat[e] / l : (i == 0 ? 1.0 : 0.0);
        a.Aout[e] = v;
        a.Q[e] = v;
      }
    }
  } else {
    for (int64_t e = tid; e < (int64_t)m * R; e += nt) a.Q[e] = a.A[e];
  }
  __syncthreads();
  hh_qr_block(a.Q, m, m, R, a.Rn, tau, beta, w, red);
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)m * a.RQ; e += nt) {
    const int i = (int)(e / a.RQ), r = (int)(e - (int64_t)i * a.RQ);
    a.Qt[e] = (r < R) ? a.Q[i + (int64_t)m * r] : 0.0;
  }
  if (a.do_fit) {  // ||Xh||^2 = <R0^T R0, diag(lam) R_n^T R_n diag(lam)>
    double q = 0.0;
    for (int e = tid; e < R * R; e += nt) {
      const int x = e % R, y = e / R;
      double g0 = 0.0, g1 = 0.0;
      for (int k = 0; k <= min(x, y); ++k) {
        g0 = fma(a.R0[k + R * x], a.R0[k + R * y], g0);
        g1 = fma(a.Rn[k + R * x], a.Rn[k + R * y], g1);
      }
      q = fma(g0, lam[x] * lam[y] * g1, q);
    }
    const double nxh2 = block_sum(q, red);
    if (tid == 0) {
      double inner = 0.0;
      for (int b = 0; b < a.ninner; ++b) inner += a.innerp[(int64_t)b * a.istride];
      const double nx2 = *a.nX2;
      *a.fit = 1.0 - sqrt(fmax(0.0, nx2 - 2.0 * inner + nxh2)) / sqrt(nx2);
    }
  }
}

// ------------------------------------------------------------------ K2: structured QR of V_n
// V_n = R_{k_{N-2}} (.) ... (.) R_{k_0} over the N-1 retained modes k_0 < ... < k_{N-2}; KB row
// j = sum_m i_m R^m (i_0 fastest).  Row level = max_m i_m; column c is nonzero only on rows of
// level <= c (the staircase).  Rows are processed in the order `perm` (sorted
// by level, then KB index): column c occupies sorted rows [0, n_c), n_c = (c+1)^{N-1}, stored
// packed at offset off_c.  Householder needs no fill-in and Q0 has the same
// support.  One CTA; `work` is shared memory when the packed matrix fits, else global scratch.
struct KrQrArgs {
  const double* Rk[kMaxModes];  // retained triangular factors, R x R column-major, ascending mode
  int N1;               // N - 1
  int R;
  const int* perm;      // sorted position -> KB row (R^{N1})
  double* Q0;           // out: dense R^{N1} x R, column-major, KB row order
  double* R0;           // out: R x R column-major, diag >= 0
  double* work_global;  // scratch (used when use_smem == 0)
  int use_smem;
  unsigned* flags;
  unsigned gate_bit;    // != 0: run only if this flag bit is set (fallback of the CholeskyQR2 V_n QR)
  int rad[kMaxModes];   // k_form_v: row radix of factor m (min(I_k, R) for short modes; 0 = R)
};

// ------------------------------------------------------------------------- K4: Q0 apply
// W_n = Y_(n) Q0 (Alg. 2 line 9) on the FP64 tensor path (DMMA m8n8k4).
// Y column-major viewed as (Aa, In, Bb); Y_(n) column j = a + Aa b (Kolda-Bader); W row-major.
// CTA (ib, ks) multiplies rows [8 ib, 8 ib + 8) of Y_(n) by k-steps [ks kpc, (ks+1) kpc) of
// Q0 (4 columns j per k-step); its 8 warps interleave those k-steps.  Warp partials are summed in
// warp order; with KS > 1 slices, the last CTA of a row block to finish (threadfence + counter)
// sums the slice partials in slice order.  One launch, bitwise reproducible.
//
// STAIR: Q0 has V_n's staircase support -- column c is
// nonzero only on the rows of level max_m j_m <= c, (c + 1)^{N-1} of them -- so the k loop runs over
// the rows in level order (perm, the packed-staircase order of K2) and N-tile n (columns 8n..8n+7)
// stops after its (8n + 8)^{N-1} rows: ~1/N of the dense apply's flops and Q0 reads.  The skipped
// products are exact zeros (both V_n QR paths preserve the support), so W is the same up to the
// summation order.
template <int NT, bool STAIR = false>
__global__ void __launch_bounds__(256)
k_q0_apply_tc(const double* __restrict__ Y, int64_t Aa, int In, int64_t Bb, const double* __restrict__ Q0, int R,
              int kpc, int KS, double* __restrict__ Wp, unsigned* __restrict__ counters, double* __restrict__ W,
              const int* __restrict__ perm, int N1, const __grid_constant__ PeerPush pp) {
  __shared__ double red[8][64 * NT];
  __shared__ int last;
  pdl_wait();
  // peer push-reduce: the rows this CTA finishes also go to slot (rank, parity) of every window
  const unsigned long long pe = pp.np ? ld_relaxed_sys(pp.epoch) : 0ull;
  const int64_t poff = (pe & 1ull) ? pp.parity_stride : 0;
  const int64_t J = Aa * Bb, KT = (J + 3) / 4;
  const int ib = blockIdx.x, ks = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int i = ib * 8 + g;
  double acc[NT][2];
  int64_t lim[NT];  // STAIR: rows (in level order) of N-tile n's staircase
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    acc[n][0] = acc[n][1] = 0.0;
    lim[n] = J;
    if (STAIR) {
      int64_t v = 1;
      for (int m = 0; m < N1; ++m) v *= (int64_t)min(8 * n + 8, R);
      lim[n] = min(J, v);
    }
  }
  const int64_t kb = (int64_t)ks * kpc, ke = min(STAIR ? (lim[NT - 1] + 3) / 4 : KT, kb + kpc);
#pragma unroll 4
  for (int64_t kk = kb + warp; kk < ke; kk += 8) {
    const int64_t pos = 4 * kk + t;
    const int64_t j = STAIR ? (pos < J ? (int64_t)__ldg(perm + pos) : J) : pos;
    double av = 0.0;
    if (i < In && j < J) {
      const int64_t bq = j / Aa, aa = j - bq * Aa;
      av = __ldg(Y + aa + Aa * (i + (int64_t)In * bq));
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      if (STAIR && 4 * kk >= lim[n]) continue;  // warp-uniform: the whole k-step is past the staircase
      const int c = 8 * n + g;
      const double bv = (j < J && c < R) ? __ldg(Q0 + j + J * c) : 0.0;
      dmma(acc[n][0], acc[n][1], av, bv);
    }
  }
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    red[warp][g * 8 * NT + 8 * n + 2 * t] = acc[n][0];
    red[warp][g * 8 * NT + 8 * n + 2 * t + 1] = acc[n][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * NT; e += blockDim.x) {
    const int r = e / (8 * NT), c = e % (8 * NT), ii = ib * 8 + r;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][e];
    if (ii < In && c < R) {
      if (KS == 1) {
        W[(int64_t)ii * R + c] = s;
        for (int r = 0; r < pp.np; ++r) pp.dst[r][poff + (int64_t)ii * R + c] = s;
      } else {
        Wp[((int64_t)ks * In + ii) * R + c] = s;
      }
    }
  }
  if (KS == 1) {
    if (pp.np) peer_push_done(pp, pe, gridDim.x);
    return;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&counters[ib], 1u) == (unsigned)(KS - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int e = threadIdx.x; e < 8 * R; e += blockDim.x) {
    const int ii = ib * 8 + e / R, c = e % R;
    if (ii < In) {
      double s = 0.0;
      for (int k = 0; k < KS; ++k) s += __ldcg(Wp + ((int64_t)k * In + ii) * R + c);
      W[(int64_t)ii * R + c] = s;
      for (int r = 0; r < pp.np; ++r) pp.dst[r][poff + (int64_t)ii * R + c] = s;
    }
  }
  if (threadIdx.x == 0) counters[ib] = 0u;  // re-armed for the next launch (graph replay)
  if (pp.np) peer_push_done(pp, pe, gridDim.x);  // one finisher per row block
}

// Z fusion: the last TTM of the Multi-TTM (over mode k) and the Q0 apply are one product
//   W_n = Y_(n) Q0 = T_(n) [(Q_k (x) I) Q0] = T_(n) Z,   Z(j_T, c) = sum_r Q_k(i_k, r) Q0(j_Y(r), c)
// where T is the intermediate BEFORE the last TTM (mode k still I_k long), j_T runs over T_(n)'s
// columns and j_Y(r) is the same multi-index with i_k replaced by r.  Z (J_T x R, J_T = I_k R^{N-2})
// is formed on the side stream right behind the V_n QR, beside the stream pass; the apply kernel
// then reads T instead of Y.  One launch and one L2 round trip less on the per-mode chain; same
// flops as the last TTM.  Used where T is small (launch-bound configs), see plan_mode.
struct ZArgs {
  const double* Qk;
  int64_t ldq;
  const double* Q0;
  double* Z;
  int nm;                   // modes != n
  int kpos;                 // position of mode k among them
  int64_t td[kMaxModes];    // T's dims over the modes != n, in mode order (R, or I_k at kpos)
  int64_t ys[kMaxModes];    // Y_(n) column strides of those modes (powers of R)
  int R;
  int64_t JT, JY;
};
__global__ void __launch_bounds__(256) k_zform(ZArgs a) {
  const int64_t tot = a.JT * a.R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % a.JT;
    const int c = (int)(e / a.JT);
    int64_t rem = j, base = 0, ik = 0;
    for (int m = 0; m < a.nm; ++m) {
      const int64_t idx = rem % a.td[m];
      rem /= a.td[m];
      if (m == a.kpos) ik = idx;
      else base += idx * a.ys[m];
    }
    const double* q0 = a.Q0 + base + a.JY * c;
    const int64_t sk = a.ys[a.kpos];
    double s = 0.0;
    for (int r = 0; r < a.R; ++r) s = fma(__ldg(a.Qk + ik + a.ldq * r), __ldg(q0 + r * sk), s);
    a.Z[e] = s;
  }
}

// Large V_n (the 5-way high-rank regime: 75^5 at R = 32 has a 1M x 32 Q0 of 268 MB
// beside a 629 MB Y_(n)): the dense apply with MTL 8-row M-tiles per CTA, so each Q0 fragment feeds
// MTL DMMAs and Q0 is read ceil(In / (8 MTL)) times instead of ceil(In / 8).  Same k-slices, warp
// and slice sums in the same fixed orders as k_q0_apply_tc; counters / Wp indexed by row group.
template <int NT, int MTL>
__global__ void __launch_bounds__(256)
k_q0_apply_big(const double* __restrict__ Y, int64_t Aa, int In, int64_t Bb, const double* __restrict__ Q0, int R,
               int kpc, int KS, double* __restrict__ Wp, unsigned* __restrict__ counters, double* __restrict__ W,
               const __grid_constant__ PeerPush pp) {
  __shared__ double red[8][64 * NT];
  __shared__ int last;
  pdl_wait();
  const unsigned long long pe = pp.np ? ld_relaxed_sys(pp.epoch) : 0ull;
  const int64_t poff = (pe & 1ull) ? pp.parity_stride : 0;
  const int64_t J = Aa * Bb, KT = (J + 3) / 4;
  const int ib = blockIdx.x, ks = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[MTL][NT][2];
#pragma unroll
  for (int m = 0; m < MTL; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  const int64_t kb = (int64_t)ks * kpc, ke = min(KT, kb + kpc);
#pragma unroll 2
  for (int64_t kk = kb + warp; kk < ke; kk += 8) {
    const int64_t j = 4 * kk + t;
    const bool jin = j < J;
    const int64_t bq = jin ? j / Aa : 0, aa = jin ? j - bq * Aa : 0;
    double bv[NT], av[MTL];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int c = 8 * n + g;
      bv[n] = (jin && c < R) ? __ldg(Q0 + j + J * c) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < MTL; ++m) {
      const int i = (ib * MTL + m) * 8 + g;
      av[m] = (jin && i < In) ? __ldg(Y + aa + Aa * (i + (int64_t)In * bq)) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < MTL; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma(acc[m][n][0], acc[m][n][1], av[m], bv[n]);
  }
#pragma unroll
  for (int m = 0; m < MTL; ++m) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      red[warp][g * 8 * NT + 8 * n + 2 * t] = acc[m][n][0];
      red[warp][g * 8 * NT + 8 * n + 2 * t + 1] = acc[m][n][1];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * NT; e += blockDim.x) {
      const int r = e / (8 * NT), c = e % (8 * NT), ii = (ib * MTL + m) * 8 + r;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w][e];
      if (ii < In && c < R) {
        if (KS == 1) {
          W[(int64_t)ii * R + c] = s;
          for (int q = 0; q < pp.np; ++q) pp.dst[q][poff + (int64_t)ii * R + c] = s;
        } else {
          Wp[((int64_t)ks * In + ii) * R + c] = s;
        }
      }
    }
    __syncthreads();
  }
  if (KS == 1) {
    if (pp.np) peer_push_done(pp, pe, gridDim.x);
    return;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&counters[ib], 1u) == (unsigned)(KS - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int e = threadIdx.x; e < MTL * 8 * R; e += blockDim.x) {
    const int ii = ib * MTL * 8 + e / R, c = e % R;
    if (ii < In) {
      double s = 0.0;
      for (int k = 0; k < KS; ++k) s += __ldcg(Wp + ((int64_t)k * In + ii) * R + c);
      W[(int64_t)ii * R + c] = s;
      for (int q = 0; q < pp.np; ++q) pp.dst[q][poff + (int64_t)ii * R + c] = s;
    }
  }
  if (threadIdx.x == 0) counters[ib] = 0u;  // re-armed for the next launch (graph replay)
  if (pp.np) peer_push_done(pp, pe, gridDim.x);
}

// ------------------------------------------------------------- one-sided Jacobi SVD of R0
// B = R0 V with orthogonal columns (cyclic round-robin pairs, one warp per pair); returns
// M = U S^+ V^T = sum_{kept j} b_j v_j^T / sigma_j^2 in Ms (R x R, column-major) and the number
// of truncated sigma_j (sigma_j <= tau * sigma_max, reading 15).  Bs, Vs: smem R x (R+1) col-major.
__device__ int jacobi_pinv(const double* R0, int R, double tau, double* Bs, double* Vs, double* Ms,
                           int* sflag) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int n = (R & 1) ? R + 1 : R;  // padded even count (dummy zero column)
  for (int e = tid; e < R * n; e += blockDim.x) {
    const int r = e % R, c = e / R;
    Bs[e] = (c < R) ? R0[r + R * c] : 0.0;
    Vs[e] = (c < R && r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) *sflag = 0;
    __syncthreads();
    for (int s = 0; s < n - 1; ++s) {
      for (int k = wid; k < n / 2; k += nw) {
        int p, q;
        if (k == 0) { p = 0; q = 1 + s; }
        else { p = 1 + (s + k) % (n - 1); q = 1 + (s - k + n - 1) % (n - 1); }
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        if (q >= R) continue;  // dummy column
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < R; r += 32) {
          const double bp = Bs[r + R * p], bq = Bs[r + R * q];
          al += bp * bp; be += bq * bq; ga += bp * bq;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        // |ga| > R eps sqrt(al be), compared squared, and cs = rsqrt(1 + t^2): one square root and
        // one division fewer on the round's dependent chain (the rounds are latency-bound)
        const double thr = (double)R * kEps;
        if (ga * ga > thr * thr * (al * be) && ga != 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = rsqrt(1.0 + tt * tt), sn = cs * tt;
          for (int r = lane; r < R; r += 32) {
            const double bp = Bs[r + R * p], bq = Bs[r + R * q];
            Bs[r + R * p] = cs * bp - sn * bq;
            Bs[r + R * q] = sn * bp + cs * bq;
            const double vp = Vs[r + R * p], vq = Vs[r + R * q];
            Vs[r + R * p] = cs * vp - sn * vq;
            Vs[r + R * q] = sn * vp + cs * vq;
          }
          if (lane == 0) *sflag = 1;
        }
      }
      __syncthreads();
    }
    const int rot = *sflag;
    __syncthreads();
    if (!rot) break;
  }
  // sigma_j = ||b_j||; M = sum_kept b_j v_j^T / sigma_j^2
  __shared__ double sig[64];
  for (int c = wid; c < R; c += nw) {
    double s = 0.0;
    for (int r = lane; r < R; r += 32) s += Bs[r + R * c] * Bs[r + R * c];
    s = warp_sum(s);
    if (lane == 0) sig[c] = sqrt(s);
  }
  __syncthreads();
  double smax = 0.0;
  for (int c = 0; c < R; ++c) smax = fmax(smax, sig[c]);
  int ntr = 0;
  for (int c = 0; c < R; ++c) ntr += (sig[c] > tau * smax) ? 0 : 1;
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int r = e % R, c = e / R;  // M(r, c) = sum_j B(r, j) V(c, j) / sig_j^2
    double s = 0.0;
    for (int j = 0; j < R; ++j)
      if (sig[j] > tau * smax) s += Bs[r + R * j] * Vs[c + R * j] / (sig[j] * sig[j]);
    Ms[r + R * c] = s;
  }
  __syncthreads();
  return ntr;
}

// --------------------------------------------------------------------------- K7: CP-ALS (NE)
// out(idx) = sum_i T(... i@k ...) A_k(i, r) with r the index of mode rm (size R) of T:
// the Khatri-Rao-diagonal contraction that finishes an MTTKRP after its first (dense) TTM.
struct DiagArgs {
  const double* T;
  int nd;
  int64_t dims[kMaxModes];
  int k, rm;
  const double* Ak;
  int64_t lda;
  double* out;  // dims without mode k, column-major
};
// out(o) = sum_i T(.., i at dim k, ..) A_k(i, r(o)): 32 consecutive outputs per CTA on the lanes
// (coalesced along the fastest remaining dimension), the i range split over the 8 warps and the
// warp partials summed in warp order (fixed order, deterministic).  A CTA per 32 outputs keeps
// enough warps in flight when there are few outputs (C2: 4000 outputs, I_k = 400).
__global__ void __launch_bounds__(256) k_diag_contract(DiagArgs a) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t tot = 1;
  for (int d = 0; d < a.nd; ++d) if (d != a.k) tot *= a.dims[d];
  int64_t stride_k = 1;
  for (int d = 0; d < a.k; ++d) stride_k *= a.dims[d];
  const int64_t Ik = a.dims[a.k];
  const int64_t o = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (o < tot) {
    int64_t rem = o, base = 0, st = 1;
    int r = 0;
    for (int d = 0; d < a.nd; ++d) {
      if (d == a.k) { st *= a.dims[d]; continue; }
      const int64_t id = rem % a.dims[d];
      rem /= a.dims[d];
      base += id * st;
      if (d == a.rm) r = (int)id;
      st *= a.dims[d];
    }
    const int64_t chunk = (Ik + 7) / 8, i0 = w * chunk, i1 = min(Ik, i0 + chunk);
    const double* Tp = a.T + base;
    const double* Ap = a.Ak + a.lda * r;
    double s1 = 0.0;
    int64_t i = i0;
    // 8 loads of T (and A) in flight per thread before the FMAs, which keep the pairwise order
    // (even i into s, odd i into s1): the latency-bound 2-deep loop ran at ~0.45 TB/s
    for (; i + 8 <= i1; i += 8) {
      double tv[8], av[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        tv[q] = Tp[(i + q) * stride_k];
        av[q] = __ldg(Ap + i + q);
      }
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        s = fma(tv[q], av[q], s);
        s1 = fma(tv[q + 1], av[q + 1], s1);
      }
    }
    for (; i + 1 < i1; i += 2) {
      s = fma(Tp[i * stride_k], __ldg(Ap + i), s);
      s1 = fma(Tp[(i + 1) * stride_k], __ldg(Ap + i + 1), s1);
    }
    if (i < i1) s = fma(Tp[i * stride_k], __ldg(Ap + i), s);
    s += s1;
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && o < tot) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += part[q][lane];
    a.out[o] = v;
  }
}

// NE tail: S = Hadamard of the other Grams; Ahat S = M by Cholesky (LU with partial pivoting on a
// non-positive pivot, reading 18); normalise; G_n = A_n^T A_n; fast fit.
struct TailNeArgs {
  const double* M;        // In x R, layout given by m_rowmajor
  int m_rowmajor;
  const double* G[kMaxModes];  // Grams (R x R), index k; G[n] ignored
  int N, n, In, R;
  double* A;              // out: normalised factor (column-major)
  double* Gn;             // out: new Gram of mode n
  double* lam;
  unsigned* flags;
  int do_fit;
  const double* nX2;
  double* fit;
  double* Ahat;           // scratch In x R column-major
  int force_lu;           // testing: take the LU path even when S is positive definite
  const double* Spinv;    // CP-ALS-PINV: S_n^+ (R x R, k_ne_pinv): Ahat = M S_n^+ instead of the solve
};
// One CTA of kNeThreads threads; RB = 8/16/32 >= R.  Rows of M are solved kNeThreads at a time on
// a shared-memory row panel with the blocked register solves of cholqr.cuh:
// x S = m, S = L L^T  <=>  y U = m (forward, U = L^T) then x U^T = y (backward).
constexpr int kNeThreads = 512;
constexpr int kNeLd = kNeThreads + 4;
template <int RB>
__global__ void __launch_bounds__(kNeThreads) k_tail_ne(TailNeArgs a) {
  extern __shared__ double smne[];
  double* S = smne;            // RB x RB, zero padded
  double* L = S + RB * RB;     // Cholesky factor (lower) or packed LU, ld RB
  double* U = L + RB * RB;     // L^T, zero padded
  double* P = U + RB * RB;     // row panel, ld kNeLd
  __shared__ double red[32], lam[RB], invd[RB];
  __shared__ int piv[RB];
  __shared__ int use_lu;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int R = a.R, In = a.In;
  for (int e = tid; e < RB * RB; e += nt) {
    const int r = e % RB, c = e / RB;
    double v = 0.0;
    if (r < R && c < R) {
      v = 1.0;
      for (int k = a.N - 1; k >= 0; --k)
        if (k != a.n) v *= a.G[k][r + R * c];
    }
    S[e] = v;
    L[e] = v;
  }
  if (tid == 0) use_lu = a.force_lu;
  if (a.Spinv)  // PINV: the pseudo-inverse in U (zero padded), no factorisation
    for (int e = tid; e < RB * RB; e += nt) {
      const int r = e % RB, c = e / RB;
      U[e] = (r < R && c < R) ? a.Spinv[r + R * c] : 0.0;
    }
  __syncthreads();
  // Cholesky S = L L^T (lower, column-major in L), by warp 0
  if (wid == 0 && !use_lu && !a.Spinv) {
    for (int j = 0; j < R; ++j) {
      double d = L[j + RB * j];
      for (int k = 0; k < j; ++k) d -= L[j + RB * k] * L[j + RB * k];
      if (!(d > 0.0)) { if (lane == 0) use_lu = 1; break; }
      d = sqrt(d);
      for (int i = j + 1 + lane; i < R; i += 32) {
        double v = L[i + RB * j];
        for (int k = 0; k < j; ++k) v -= L[i + RB * k] * L[j + RB * k];
        L[i + RB * j] = v / d;
      }
      __syncwarp();
      if (lane == 0) L[j + RB * j] = d;
      __syncwarp();
    }
    if (!use_lu && lane == 0) {  // ill-conditioning estimate (robust-policy hook)
      double dmax = 0.0, dmin = 1e308;
      for (int j = 0; j < R; ++j) { dmax = fmax(dmax, L[j + RB * j]); dmin = fmin(dmin, L[j + RB * j]); }
      if (!(dmin > 0.0) || (dmax / dmin) * (dmax / dmin) > kNeKappaMax) atomicOr(a.flags, FLAG_NE_ILLCOND);
    }
  }
  __syncthreads();
  if (a.Spinv) {
  } else if (use_lu) {
    if (tid == 0) {
      atomicOr(a.flags, FLAG_NE_CHOL_FALLBACK);
      for (int e = 0; e < RB * RB; ++e) L[e] = S[e];
      for (int j = 0; j < R; ++j) {  // LU with partial pivoting, L and U packed in L
        int p = j;
        for (int i = j + 1; i < R; ++i) if (fabs(L[i + RB * j]) > fabs(L[p + RB * j])) p = i;
        piv[j] = p;
        if (p != j) for (int c = 0; c < R; ++c) { double t = L[j + RB * c]; L[j + RB * c] = L[p + RB * c]; L[p + RB * c] = t; }
        for (int i = j + 1; i < R; ++i) {
          L[i + RB * j] /= L[j + RB * j];
          for (int c = j + 1; c < R; ++c) L[i + RB * c] -= L[i + RB * j] * L[j + RB * c];
        }
      }
    }
  } else {
    for (int e = tid; e < RB * RB; e += nt) {  // U = L^T (upper), invd = 1 / L_jj
      const int r = e % RB, c = e / RB;
      U[e] = (r <= c && c < R) ? L[c + RB * r] : 0.0;
    }
    if (tid < RB) invd[tid] = (tid < R) ? 1.0 / L[tid + RB * tid] : 0.0;
  }
  __syncthreads();
  // rows: Ahat(i,:) S = M(i,:)  (S symmetric)
  double* row = P + tid;
  for (int i0 = 0; i0 < In; i0 += nt) {
    const int i = i0 + tid;
    const bool own = i < In;
#pragma unroll 4
    for (int c = 0; c < RB; ++c)
      row[kNeLd * c] = (own && c < R) ? (a.m_rowmajor ? a.M[(int64_t)i * R + c] : a.M[i + (int64_t)In * c]) : 0.0;
    if (a.Spinv) {  // x = m S^+ 
      double m[RB];
#pragma unroll
      for (int c = 0; c < RB; ++c) m[c] = row[kNeLd * c];
#pragma unroll 4
      for (int c = 0; c < RB; ++c) {
        double x = 0.0;
#pragma unroll
        for (int r = 0; r < RB; ++r) x = fma(m[r], U[r + RB * c], x);
        row[kNeLd * c] = x;
      }
    } else if (!use_lu) {
      cq_row_trsv<RB, false>(row, kNeLd, U, invd);  // y U = m
      cq_row_trsv<RB, true>(row, kNeLd, U, invd);   // x U^T = y
    } else {
      for (int j = 0; j < R; ++j) {
        const int p = piv[j];
        if (p != j) { const double t = row[kNeLd * j]; row[kNeLd * j] = row[kNeLd * p]; row[kNeLd * p] = t; }
      }
      for (int j = 0; j < R; ++j) {
        double v = row[kNeLd * j];
        for (int k = 0; k < j; ++k) v -= L[j + RB * k] * row[kNeLd * k];
        row[kNeLd * j] = v;
      }
      for (int j = R - 1; j >= 0; --j) {
        double v = row[kNeLd * j];
        for (int k = j + 1; k < R; ++k) v -= L[j + RB * k] * row[kNeLd * k];
        row[kNeLd * j] = v / L[j + RB * j];
      }
    }
    if (own)
#pragma unroll 4
      for (int c = 0; c < R; ++c) a.Ahat[i + (int64_t)In * c] = row[kNeLd * c];
  }
  __syncthreads();
  for (int c = wid; c < R; c += nw) {
    const double* col = a.Ahat + (int64_t)In * c;
    double s = 0.0;
    for (int i = lane; i < In; i += 32) s += col[i] * col[i];
    s = warp_sum(s);
    if (lane == 0) lam[c] = sqrt(s);
  }
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < R; ++c) if (!isfinite(lam[c])) atomicOr(a.flags, FLAG_NONFINITE);
  for (int64_t e = tid; e < (int64_t)In * R; e += nt) {
    const int c = (int)(e / In), i = (int)(e % In);
    a.A[e] = (lam[c] > 0.0) ? a.Ahat[e] / lam[c] : (i == 0 ? 1.0 : 0.0);
  }
  if (tid < R) a.lam[tid] = lam[tid];
  __syncthreads();
  // G_n = A_n^T A_n (warp per entry, fixed order)
  for (int e = wid; e < R * R; e += nw) {
    const int x = e % R, y = e / R;
    const double* cx = a.A + (int64_t)In * x;
    const double* cy = a.A + (int64_t)In * y;
    double s = 0.0;
    for (int i = lane; i < In; i += 32) s += cx[i] * cy[i];
    s = warp_sum(s);
    if (lane == 0) a.Gn[e] = s;
  }
  __syncthreads();
  if (a.do_fit) {
    double s = 0.0;  // <M_N, Ahat_N>
    for (int64_t e = tid; e < (int64_t)In * R; e += nt) {
      const int c = (int)(e / In), i = (int)(e % In);
      const double m = a.m_rowmajor ? a.M[(int64_t)i * R + c] : a.M[e];
      s = fma(m, a.Ahat[e], s);
    }
    const double inner = block_sum(s, red);
    double q = 0.0;  // <S_N, diag(lam) G_N diag(lam)>
    for (int e = tid; e < R * R; e += nt) q += S[(e % R) + RB * (e / R)] * lam[e % R] * lam[e / R] * a.Gn[e];
    const double nxh2 = block_sum(q, red);
    if (tid == 0) {
      const double nx2 = *a.nX2;
      *a.fit = 1.0 - sqrt(fmax(0.0, nx2 - 2.0 * inner + nxh2)) / sqrt(nx2);
    }
  }
}

// Gram G = A^T A (warp per entry) for set_factors in the NE variant.
// C = A B for upper-triangular R x R A, B (column-major; one CTA): the shifted CholeskyQR3's
// R0 = R' R_s (short modes, launch_kr_qr).
__global__ void k_tri_mul(const double* __restrict__ A, const double* __restrict__ B, int R, double* __restrict__ C) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int r = e % R, c = e / R;
    double s = 0.0;
    for (int k = r; k <= c; ++k) s = fma(A[r + R * k], B[k + R * c], s);
    C[e] = (r <= c) ? s : 0.0;
  }
}

__global__ void __launch_bounds__(1024) k_gram(const double* __restrict__ A, int In, int R, double* __restrict__ G) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = wid; e < R * R; e += nw) {
    const int x = e % R, y = e / R;
    double s = 0.0;
    for (int i = lane; i < In; i += 32) s += A[i + (int64_t)In * x] * A[i + (int64_t)In * y];
    s = warp_sum(s);
    if (lane == 0) G[e] = s;
  }
}

// Direct residual ||X - Xh||^2: Xh(i) = sum_r lam_r prod_k A_k(i_k, r), over the
// local slab (last-mode offset `off`).  Deterministic block partials.
struct ResidArgs {
  const double* X;
  int64_t n;           // local numel
  int N;
  int64_t dims[kMaxModes];     // local dims
  int64_t off_last;    // global offset of the slab on the last mode
  const double* A[kMaxModes];  // global factors (column-major, lda = global I_k)
  int64_t lda[kMaxModes];
  const double* lam;
  int R;
  double* part;
};
__global__ void k_resid_partial(ResidArgs a) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx[kMaxModes];
    int64_t rem = e;
    for (int k = 0; k < a.N; ++k) { idx[k] = rem % a.dims[k]; rem /= a.dims[k]; }
    idx[a.N - 1] += a.off_last;
    double xh = 0.0;
    for (int r = 0; r < a.R; ++r) {
      double p = a.lam[r];
      for (int k = 0; k < a.N; ++k) p *= a.A[k][idx[k] + a.lda[k] * r];
      xh += p;
    }
    const double d = a.X[e] - xh;
    s = fma(d, d, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) a.part[blockIdx.x] = s;
}
__global__ void k_fit_from_resid(const double* res2, const double* nX2, double* fit) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *fit = 1.0 - sqrt(fmax(0.0, *res2)) / sqrt(*nX2);
}

}  // namespace cpqr
