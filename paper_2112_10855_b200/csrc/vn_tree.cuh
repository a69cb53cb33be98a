// Tree QR of V_n across the Khatri-Rao factors, sm_100a fp64.
//
// V_n = R_N (.) ... (.) R_{n+1} (.) R_{n-1} (.) ... (.) R_1 (Alg. 2 line 6) is never formed.  With
// (A C) (.) (B D) = (A (x) B)(C (.) D) (Eq. (2.1)) a Khatri-Rao product of
// triangular factors is reduced by QRs of R^2 x R pairs: a group [R_a, ..., R_z] (slowest first)
// starts from P = I, S = R_z, and for each next-slower R_k, QR(R_k (.) S) = Q S' gives
// R_k (.) (P S) = (I (x) P) Q S', so P <- (I (x) P) Q, S <- S'.  The retained modes split into two
// groups at h = ceil(N/2) (reading 36, the dimension tree's split): for n < h the
// modes >= h ("hi") do not change between modes 0..h-1 of a sweep, for n >= h the modes < h ("lo")
// do not change between modes h..N-1 -- that group is factored once per half sweep (`fresh`) and
// cached, the other one per mode.  Root: QR(S_hi (.) S_lo) = Q_r R0 and Q0 = (P_hi (x) P_lo) Q_r,
// formed explicitly (T = (I (x) P_lo) Q_r, then Q0 = (P_hi (x) I) T) so the dense DMMA Q0 apply
// (K4) is unchanged.  Every node is the packed-staircase Householder of K2 (R_a (.) R_b has column
// c nonzero on the (c+1)^2 rows of level max(i_a, i_b) <= c, no fill-in), so the
// node QRs cost O(R^4) each instead of K2's one QR of R^{N-1} x R; the result is the same unique
// thin QR (diag R0 > 0) up to rounding, and Q0 keeps V_n's support exactly (the skipped products
// are exact zeros).  One CTA (it runs on the side stream beside the stream pass).
#pragma once
#include "qr_kernels.cuh"

namespace cpqr {

struct VnTreeArgs {
  const double* Rk[kMaxModes];  // every mode's R_k (R x R column-major, upper triangular)
  int N, n, R, h;
  int fresh;          // factor the shared group (first mode of its half in a sweep, or a standalone call)
  double* Psh[2];     // shared-group P (R^{|g|} x R column-major): [0] the hi group (n < h), [1] the lo group
  double* Ssh[2];     // shared-group S (R x R column-major)
  double* Pa;         // own-group chain buffers (ping-pong), R^{|g|} x R
  double* Pb;
  double* T;          // formation intermediate, R^{N-1} x R
  double* Qg;         // dense node Q for R > 16 (R^3 doubles; shared memory below)
  double* Q0;         // out: R^{N-1} x R column-major, Kolda-Bader row order
  double* R0;         // out: R x R column-major, diag >= 0
  unsigned* flags;
};

// packed staircase of a node R_a (.) R_b: column c holds the (c+1)^2 rows of level <= c, level L
// at positions [L^2, (L+1)^2), in increasing Kolda-Bader row i_a R + i_b: position q < L is
// (i_a, i_b) = (q, L), position q >= L is (L, q - L).
__device__ __forceinline__ void node_row(int p, int& ia, int& ib) {
  int L = (int)sqrt((double)p);
  while (L * L > p) --L;
  while ((L + 1) * (L + 1) <= p) ++L;
  const int q = p - L * L;
  if (q < L) { ia = q; ib = L; } else { ia = L; ib = q - L; }
}
__device__ __forceinline__ int node_pos(int ia, int ib) {  // inverse of node_row
  const int L = max(ia, ib);
  return L * L + (ia < L ? ia : L + ib);
}

struct NodeSmem {
  double* V;      // packed staircase, sum_c (c+1)^2 doubles
  double* S;      // R x R: the node's triangular factor (signed: diag >= 0)
  double* sg;     // R: column signs of the node's Q
  double* Qd;     // dense node Q, R^2 x R column-major (shared memory for R <= 16, else global)
  double* Us;     // triangle tree (R <= 16): R slots of RB x RB row-major (leaf triangles / reflectors)
  double* Ys;     //   R slots of RB x RB row-major (down-sweep blocks of Q)
  double* tt;     //   R x RB Householder tau per merge (indexed by the right child's slot)
  int64_t* off;   // R + 1
  int* cnt;       // R
  double *tau, *beta, *w, *np;
};

// QR(A (.) B) for upper-triangular R x R A (slower index) and B: S and the packed, unsigned Q stay
// in shared memory (Q(ia R + ib, c) = sg[c] V[off[c] + node_pos(ia, ib)] for max(ia, ib) <= c).
__device__ void node_qr(const NodeSmem& s, const double* A, const double* B, int R) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int c = 0; c < R; ++c)
    for (int p = tid; p < s.cnt[c]; p += nt) {
      int ia, ib;
      node_row(p, ia, ib);
      s.V[s.off[c] + p] = A[ia + R * c] * B[ib + R * c];
    }
  __syncthreads();
  HHCols M{s.V, s.off, s.cnt};
  hh_factor(M, R, s.tau, s.beta, s.w, s.np);
  for (int e = tid; e < R * R; e += nt) {
    const int r = e % R, c = e / R;
    double v = (r < c) ? s.V[s.off[c] + r] : ((r == c) ? s.beta[r] : 0.0);
    if (s.beta[r] < 0.0) v = -v;
    s.S[e] = v;
  }
  for (int c = tid; c < R; c += nt) s.sg[c] = (s.beta[c] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  hh_formq(M, R, s.tau, s.w);
  // dense, signed copy of the node's Q for the formation products (zeros off the staircase)
  for (int e = tid; e < R * R * R; e += nt) {
    const int c = e / (R * R), row = e - c * R * R;
    const int ia = row / R, ib = row - ia * R;
    s.Qd[e] = (max(ia, ib) <= c) ? s.sg[c] * s.V[s.off[c] + node_pos(ia, ib)] : 0.0;
  }
  __syncthreads();
}


// ------------------------------------------------------------------ node QR by a triangle tree
// R_a (.) R_b stacks R upper-triangular blocks: rows [iR, iR+R) are T_i = R_b diag(R_a(i, :))
// (Khatri-Rao column rule).  QR of a stack of triangles is a binary tree of merges
// QR([U; L]) (both R x R upper triangular; the TSQR tree): merge (p, p+s) runs on one warp with
// lane c owning column c of U and L in registers; reflector j has a 1 at U's row j and entries at
// L's rows 0..j only, so its vector (and tau) overwrite L's slot, which the up-sweep never reads
// again.  The down-sweep applies each merge's reflectors in reverse to [Y; 0] (Y = the parent's
// block, I at the root with the sign fix diag(S) >= 0) and hands the top half to the left child
// and the bottom half to the right child; the leaves' blocks are Q's row blocks.  Merges of one
// tree level run on different warps: ceil(log2 R) levels of R-step warp-local loops instead of R
// block-wide Householder steps over the packed (c+1)^2-row staircase (no block barrier inside a
// merge).  Same unique thin QR (diag S > 0) up to rounding.
template <int RB>
__device__ void tt_merge_up(double* U, double* L, double* tau, int R) {
  const int c = threadIdx.x & 31;
  double u[RB], l[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    u[r] = (c < R) ? U[r * RB + c] : 0.0;
    l[r] = (c < R) ? L[r * RB + c] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    if (j < R) {
      if (c == j) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int r = 0; r <= j; r += 2) {
          s0 = fma(l[r], l[r], s0);
          if (r + 1 <= j) s1 = fma(l[r + 1], l[r + 1], s1);
        }
        const double sig = s0 + s1, x0 = u[j];
        double tj = 0.0, bj = x0, sc = 0.0;
        if (sig != 0.0) {
          const double nrm = sqrt(x0 * x0 + sig);
          bj = (x0 >= 0.0) ? -nrm : nrm;
          tj = (bj - x0) / bj;
          sc = 1.0 / (x0 - bj);
        }
#pragma unroll
        for (int r = 0; r <= j; ++r) L[r * RB + j] = l[r] * sc;
        tau[j] = tj;
        u[j] = bj;
      }
      __syncwarp();
      if (c > j && c < R) {
        const double tj = tau[j];
        double d0 = u[j], d1 = 0.0;
#pragma unroll
        for (int r = 0; r <= j; r += 2) {
          d0 = fma(L[r * RB + j], l[r], d0);
          if (r + 1 <= j) d1 = fma(L[(r + 1) * RB + j], l[r + 1], d1);
        }
        const double d = tj * (d0 + d1);
        u[j] -= d;
#pragma unroll
        for (int r = 0; r <= j; ++r) l[r] = fma(-d, L[r * RB + j], l[r]);
      }
    }
  }
  if (c < R) {
#pragma unroll
    for (int r = 0; r < RB; ++r) U[r * RB + c] = u[r];
  }
  __syncwarp();
}

// [Ytop; Ybot] = H_0 ... H_{R-1} [Y; 0] with the merge's reflectors (vectors in V, tau)
template <int RB>
__device__ void tt_merge_down(double* Y, double* Ybot, const double* V, const double* tau, int R) {
  const int c = threadIdx.x & 31;
  double y[RB], z[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) { y[r] = (c < R) ? Y[r * RB + c] : 0.0; z[r] = 0.0; }
#pragma unroll
  for (int j = RB - 1; j >= 0; --j) {
    if (j < R) {
      const double tj = tau[j];
      double d0 = y[j], d1 = 0.0;
#pragma unroll
      for (int r = 0; r <= j; r += 2) {
        d0 = fma(V[r * RB + j], z[r], d0);
        if (r + 1 <= j) d1 = fma(V[(r + 1) * RB + j], z[r + 1], d1);
      }
      const double d = tj * (d0 + d1);
      y[j] -= d;
#pragma unroll
      for (int r = 0; r <= j; ++r) z[r] = fma(-d, V[r * RB + j], z[r]);
    }
  }
  __syncwarp();
  if (c < R) {
#pragma unroll
    for (int r = 0; r < RB; ++r) { Y[r * RB + c] = y[r]; Ybot[r * RB + c] = z[r]; }
  }
  __syncwarp();
}

// QR(A (.) B) -> s.S (signed, diag >= 0) and the dense s.Qd (R^2 x R column-major), R <= RB <= 16
template <int RB>
__device__ void tt_qr(const NodeSmem& s, const double* A, const double* B, int R) {
  const int tid = threadIdx.x, nt = blockDim.x, wid = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < R * RB * RB; e += nt) {  // leaves T_i(r, c) = B(r, c) A(i, c), r <= c
    const int i = e / (RB * RB), rc = e - i * RB * RB, r = rc / RB, c = rc - r * RB;
    s.Us[e] = (c < R && r <= c) ? B[r + R * c] * A[i + R * c] : 0.0;
  }
  __syncthreads();
  for (int st = 1; st < R; st *= 2) {  // up-sweep: merges (p, p + st), p a multiple of 2 st
    const int nm = (R - st + 2 * st - 1) / (2 * st);
    for (int m = wid; m < nm; m += nw) {
      const int p = 2 * st * m;
      tt_merge_up<RB>(s.Us + p * RB * RB, s.Us + (p + st) * RB * RB, s.tt + (p + st) * RB, R);
    }
    __syncthreads();
  }
  for (int e = tid; e < R * R; e += nt) {  // S = the root's triangle, rows sign-fixed
    const int r = e % R, c = e / R;
    const double d = s.Us[r * RB + r];
    const double v = s.Us[r * RB + c];
    s.S[e] = (r <= c) ? ((d < 0.0) ? -v : v) : 0.0;
  }
  for (int e = tid; e < RB * RB; e += nt) {  // Y_root = diag(sign S(c, c))
    const int r = e / RB, c = e - r * RB;
    s.Ys[e] = (r == c && r < R) ? ((s.Us[r * RB + r] < 0.0) ? -1.0 : 1.0) : 0.0;
  }
  __syncthreads();
  int top = 1;
  while (top < R) top *= 2;
  for (int st = top / 2; st >= 1; st /= 2) {  // down-sweep
    const int nm = (R - st + 2 * st - 1) / (2 * st);
    for (int m = wid; m < nm; m += nw) {
      const int p = 2 * st * m;
      tt_merge_down<RB>(s.Ys + p * RB * RB, s.Ys + (p + st) * RB * RB, s.Us + (p + st) * RB * RB,
                        s.tt + (p + st) * RB, R);
    }
    __syncthreads();
  }
  for (int e = tid; e < R * R * R; e += nt) {  // Q(i R + ib, c) = Y_i(ib, c)
    const int c = e / (R * R), row = e - c * R * R, i = row / R, ib = row - i * R;
    s.Qd[e] = s.Ys[i * RB * RB + ib * RB + c];
  }
  __syncthreads();
}

// out((ia, j), c) = sum_{b <= c} P(j, b) Q_node((ia, b), c), i.e. out = (I_R (x) P) Q_node with
// P: J x R (column-major, global or shared) -- a chain step P <- (I (x) P) Q and the first
// formation step T = (I (x) P_lo) Q_r.  P == nullptr: the identity (out = Q_node densely, J = R).
// One thread per output row: its R entries of P are loaded once into registers, the node's Q comes
// from shared memory, the R outputs are written coalesced across threads (consecutive rows).
template <int RB>
__device__ void kron_node(const NodeSmem& s, const double* P, int64_t J, int R, double* out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t rows = (int64_t)R * J;
  if (!P) {  // identity: out = Q_node
    for (int64_t e = tid; e < rows * R; e += nt) out[e] = s.Qd[e];
    __syncthreads();
    return;
  }
  for (int64_t row = tid; row < rows; row += nt) {
    const int ia = (int)(row / J);  // uniform across a warp when J >= 32
    const int64_t j = row - (int64_t)ia * J;
    double p[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) p[b] = (b < R) ? P[j + J * b] : 0.0;
    const double* q = s.Qd + ia * R;
    for (int c = 0; c < R; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < RB; ++b)
        if (b <= c) acc = fma(p[b], q[b + R * R * c], acc);
      out[row + rows * c] = acc;
    }
  }
  __syncthreads();
}

// Q0((ih, il), c) = sum_{q <= c} P_hi(ih, q) T((q, il), c), rows ih Jlo + il: Q0 = (P_hi (x) I) T.
// T: (R Jlo) x R column-major (the root's dense Q_r itself when there is no P_lo, Jlo = R).
template <int RB>
__device__ void kron_hi(const double* Phi, int64_t Jhi, const double* T, int64_t Jlo, int R, double* Q0) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t J = Jhi * Jlo, JT = (int64_t)R * Jlo;
  for (int64_t row = tid; row < J; row += nt) {
    const int64_t ih = row / Jlo, il = row - ih * Jlo;
    double p[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) p[q] = (q < R) ? Phi[ih + Jhi * q] : 0.0;
    for (int c = 0; c < R; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < RB; ++q)
        if (q <= c) acc = fma(p[q], T[q * Jlo + il + JT * c], acc);
      Q0[row + J * c] = acc;
    }
  }
  __syncthreads();
}

// Factor a group g[0..m) (slowest first): P and S.  S is written to `Sout` (R x R); P into Pout
// (when m >= 2; chain steps ping-pong through Pout / Pscr so that the final P lands in Pout).
// Returns false when P is the identity (m == 1).
template <int RB>
__device__ __forceinline__ void node_qr_rb(const NodeSmem& s, const double* A, const double* B, int R) {
  if (RB <= 16) tt_qr<(RB <= 16 ? RB : 16)>(s, A, B, R);
  else node_qr(s, A, B, R);
}

template <int RB>
__device__ bool group_qr(const NodeSmem& s, const double* const* Rk, const int* g, int m, int R, double* Sout,
                         double* Pout, double* Pscr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (m == 1) {
    for (int e = tid; e < R * R; e += nt) Sout[e] = Rk[g[0]][e];
    __syncthreads();
    return false;
  }
  const int steps = m - 1;  // chain steps k = g[m-2], ..., g[0]
  double* cur = nullptr;
  const double* Sprev = Rk[g[m - 1]];
  int64_t J = R;  // rows of the current P (the identity: R)
  for (int t = 0; t < steps; ++t) {
    node_qr_rb<RB>(s, Rk[g[m - 2 - t]], Sprev, R);
    double* dst = ((steps - 1 - t) % 2 == 0) ? Pout : Pscr;
    kron_node<RB>(s, cur, J, R, dst);
    J *= R;
    cur = dst;
    for (int e = tid; e < R * R; e += nt) Sout[e] = s.S[e];
    __syncthreads();
    Sprev = Sout;
  }
  return true;
}

constexpr int kVnTreeTSmem = 12288;
// node work area (doubles): the triangle tree's 2 R RB^2 + R RB (R <= 16) or the packed staircase
__host__ __device__ inline int vn_tree_node_area(int R) {
  const int rb = R <= 8 ? 8 : 16;
  return R <= 16 ? 2 * R * rb * rb + R * rb : R * (R + 1) * (2 * R + 1) / 6;
}  // doubles of shared memory for the formation intermediate T

template <int RB>
__global__ void __launch_bounds__(RB == 16 ? 512 : 256) k_vn_tree(VnTreeArgs a) {
  extern __shared__ double smv[];
  __shared__ double tau[64], beta[64], w[64], np[64], sg[64];
  __shared__ int64_t off[65];
  __shared__ int cnt[64];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int R = a.R, N = a.N, n = a.n, h = a.h;
  if (tid == 0) {
    int64_t o = 0;
    for (int c = 0; c < R; ++c) { cnt[c] = (c + 1) * (c + 1); off[c] = o; o += cnt[c]; }
    off[R] = o;
  }
  NodeSmem s;
  s.V = smv;
  s.Us = smv;  // R <= 16: the triangle tree's slots instead of the packed staircase
  s.Ys = smv + R * RB * RB;
  s.tt = s.Ys + R * RB * RB;
  s.S = smv + vn_tree_node_area(R);
  double* Sown = s.S + R * R;
  double* Sroot = Sown + R * R;
  double* Ts = Sroot + R * R;  // kVnTreeTSmem doubles
  s.Qd = (R <= 16) ? Ts + kVnTreeTSmem : a.Qg;
  s.sg = sg; s.off = off; s.cnt = cnt; s.tau = tau; s.beta = beta; s.w = w; s.np = np;
  // groups (decreasing mode order): hi = modes >= h, lo = modes < h, without n
  int hi[kMaxModes], lo[kMaxModes], mh = 0, ml = 0;
  for (int k = N - 1; k >= h; --k) if (k != n) hi[mh++] = k;
  for (int k = h - 1; k >= 0; --k) if (k != n) lo[ml++] = k;
  const int side = (n < h) ? 0 : 1;  // which group is shared: hi for n < h, lo for n >= h
  const int* gs = side ? lo : hi;
  const int* go = side ? hi : lo;
  const int ms = side ? ml : mh, mo = side ? mh : ml;
  __syncthreads();
  // shared group: factored once per half sweep, cached in Psh / Ssh
  const bool psh_dense = ms >= 2;
  if (a.fresh) group_qr<RB>(s, a.Rk, gs, ms, R, a.Ssh[side], a.Psh[side], a.Pa);
  // own group
  bool pown_dense = false;
  if (mo > 0) pown_dense = group_qr<RB>(s, a.Rk, go, mo, R, Sown, a.Pb, a.Pa);
  int64_t Jhi = 1, Jlo = 1;
  for (int i = 0; i < mh; ++i) Jhi *= R;
  for (int i = 0; i < ml; ++i) Jlo *= R;
  const int64_t J = Jhi * Jlo;
  if (mo == 0) {  // V_n is the shared group alone (n is the only mode of its half): Q0 = P, R0 = S
    const double* P = a.Psh[side];
    for (int64_t e = tid; e < J * R; e += nt) {
      const int c = (int)(e / J);
      const int64_t row = e % J;
      a.Q0[e] = psh_dense ? P[e] : (row == c ? 1.0 : 0.0);
    }
    for (int e = tid; e < R * R; e += nt) Sroot[e] = a.Ssh[side][e];
    __syncthreads();
  } else {
    const double* Shi = side ? Sown : a.Ssh[0];
    const double* Slo = side ? a.Ssh[1] : Sown;
    const double* Phi = side ? (pown_dense ? a.Pb : nullptr) : (psh_dense ? a.Psh[0] : nullptr);
    const double* Plo = side ? (psh_dense ? a.Psh[1] : nullptr) : (pown_dense ? a.Pb : nullptr);
    node_qr_rb<RB>(s, Shi, Slo, R);  // root: S_hi (.) S_lo = Q_r R0
    for (int e = tid; e < R * R; e += nt) Sroot[e] = s.S[e];
    if (!Phi) {
      kron_node<RB>(s, Plo, Plo ? Jlo : R, R, a.Q0);  // Q0 = (I (x) P_lo) Q_r
    } else if (!Plo) {
      kron_hi<RB>(Phi, Jhi, s.Qd, R, R, a.Q0);  // Q0 = (P_hi (x) I) Q_r
    } else {
      // T = (I (x) P_lo) Q_r, in shared memory when it fits, then Q0 = (P_hi (x) I) T
      double* T = ((int64_t)R * Jlo * R <= kVnTreeTSmem) ? Ts : a.T;
      kron_node<RB>(s, Plo, Jlo, R, T);
      kron_hi<RB>(Phi, Jhi, T, Jlo, R, a.Q0);
    }
  }
  for (int e = tid; e < R * R; e += nt) a.R0[e] = Sroot[e];
  if (tid == 0) {  // ILLCOND_R0 (reading 17): min diag <= rows(V_n) eps max diag
    double mx = 0.0, mn = 1e308;
    for (int c = 0; c < R; ++c) { mx = fmax(mx, fabs(Sroot[c + R * c])); mn = fmin(mn, fabs(Sroot[c + R * c])); }
    if (mn <= (double)J * kEps * mx) atomicOr(a.flags, FLAG_ILLCOND_R0);
  }
}

inline size_t vn_tree_smem(int R) {
  return sizeof(double) * ((size_t)vn_tree_node_area(R) + 3 * (size_t)R * R + kVnTreeTSmem +
                            (R <= 16 ? (size_t)R * R * R : 0));
}

}  // namespace cpqr
