// libcpqr: C-ABI entry points and the host-side sweep driver (streams, CUDA graph, NCCL).
// The per-mode sequence is Alg. 2 lines 6-12 for CP-ALS-QR / QR-SVD and
// Alg. 1 lines 6-11 for CP-ALS.  See DESIGN.md for the kernel map.
#include "../../include/cpqr.h"
#include "qr_kernels.cuh"
#include "rowqr.cuh"
#include "cholqr.cuh"
#include "small_kernels.cuh"
#include "tma_kernels.cuh"
#include "ttm_kernels.cuh"
#include "ktensor_kernels.cuh"
#include "batched_kernels.cuh"
#include "small_ttm.cuh"
#include "vn_tree.cuh"

#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#define CPQR_API extern "C" __attribute__((visibility("default")))

using namespace cpqr;

namespace {

constexpr int kMaxN = kMaxModes;
constexpr int kMaxR = 32;
constexpr int kMaxWorld = kMaxRanks;      // ranks (NCCL) or virtual ranks (CPQR_COMM_LOCAL)
constexpr size_t kQSmemMax = 96 * 1024;   // Q panel budget per CTA (2 CTAs / SM)
constexpr int64_t kQ0MaxSlices = 64;      // k-step slices of k_q0_apply_tc (partials buffer)

struct TtmStep {
  int kind;  // 0 strided, 1 fiber, 2 slice, 3 slice-reduce, 4 strided TMA, 5 fiber TMA, 6 slice TMA, 7 slice fix-up,
            // 8 small slice TMA, 9 small (L2-resident) TTM
  alignas(64) CUtensorMap mx;
  alignas(64) CUtensorMap mq;
  int S = 0, nslots = 1, nfb = 1;
  int64_t G = 1;
  double* P = nullptr;
  const double* in;
  double* out;
  int64_t A, B, F, L;
  int I, I1, I2;
  const double* Q;
  int64_t ldq;
  const double* Q2;
  int64_t ldq2;
  int gps, nseg;
  int cw = 8;  // slice TMA: consumer warps per CTA (4: two CTAs per SM)
  unsigned modes = 0;  // contracted modes (bit k = mode k of the global tensor)
  int skm = -1;        // strided TMA: stream-K split -1 auto (ragged waves), 0 off, 1 always
  int cw1 = 0;         // 1: one CTA per SM (8 consumer warps) so reserved SMs stay free (overlap)
  unsigned* cnt = nullptr;  // strided TMA stream-K: per-CTA arrival counters of the fused fix-up
  int wk = 1, kc = 1;       // k_ttm_small (kind 9): contraction split over WK warps x KC CTAs
  const double* Qt = nullptr;  // k_ttm_small: the transposed zero-padded panel (I x rq row-major)
  int rq = 0;
};

struct DiagStep {
  const double* in;
  double* out;
  int nd;
  int64_t dims[kMaxN];
  int k, rm;
  const double* Ak;
  int64_t lda;
  int mode;  // global mode contracted
};

struct Plan {
  std::vector<TtmStep> steps;
  std::vector<DiagStep> diags;  // NE only
  const double* Y = nullptr;    // final result (device)
  int nd = 0;
  int64_t ydims[kMaxN];
  int64_t Aa = 1, In = 1, Bb = 1;
  int m_rowmajor = 1;  // NE: layout of the MTTKRP result
  size_t max_buf = 0;
  size_t part = 0;
  size_t tree_elems = 0;  // dimension tree: size of the half intermediate this plan writes
  // Z fusion (k_zform, small_kernels.cuh): the last step (a TTM over mode zk) is skipped and the Q0
  // apply reads its input T = zT, viewed (zAa, In, zBb), against Z = (Q_zk (x) I) Q0
  bool zf = false;
  int zk = -1;
  const double* zT = nullptr;
  int64_t zAa = 1, zBb = 1;
  int64_t zcur[kMaxN];    // T's dims
};

// One rank's slab of the tensor (slab data parallelism over the last mode): the
// global range [b, e) of mode N, the local dims, the tensor pointer, the per-mode plans (their TMA
// maps encode this slab's X and the matching rows of Q_N), the dimension-tree buffer and the
// partial W_n (modes n < N) or local rows of W_N.  A context holds one slab (single GPU, or one
// NCCL rank) or, with CPQR_COMM_LOCAL, all p slabs of p virtual ranks run in rank order.
struct Slab {
  int64_t b = 0, e = 0;
  int64_t ldims[kMaxN] = {0};
  int64_t numel = 0;
  const double* X = nullptr;
  double* Xown = nullptr;
  size_t Xown_elems = 0;
  bool have = false;
  Plan plans[kMaxN];
  double* dTree = nullptr;
  size_t tree_alloc = 0;
  double* dWloc = nullptr;
};

}  // namespace

struct cpqr_ctx {
  int N = 0, R = 0, variant = 1;
  int64_t dims[kMaxN] = {0};
  int nslab = 1;            // slabs this context runs: 1, or world with CPQR_COMM_LOCAL
  bool local = false;       // CPQR_COMM_LOCAL: p virtual ranks on one device, combined in rank order
  Slab slabs[kMaxWorld];
  cpqr_options opt;
  int sms = 148;
  cudaStream_t st = nullptr;
  cudaStream_t user = nullptr;
  ncclComm_t comm = nullptr;
  // exchange of the slabs' results: NCCL collectives, the virtual ranks' sum kernel,
  // or the peer push-reduce (CPQR_COMM_PEER / CPQR_COMM_LOCAL_PEER; small_kernels.cuh): receive
  // windows win_base[r] -- this rank's own (cudaMalloc) and its peers' (CUDA IPC), or all p of the
  // virtual ranks -- laid out [2 parities][p slots][slot_elems] doubles, kMaxRanks flags, epoch
  bool exchange = false;      // world > 1, or a one-rank NCCL / PEER exchange (hardware check of the path)
  bool peer = false, peers_connected = false;
  void* win_base[kMaxWorld] = {nullptr};
  bool win_mapped[kMaxWorld] = {false};
  int64_t slot_elems = 0;
  size_t win_data_bytes = 0, win_bytes = 0;
  unsigned* dpushcnt = nullptr;
  unsigned long long peer_timeout_ns = 20000000000ull;
  bool have_tensor = false, have_factors = false;
  double *dA[kMaxN] = {0}, *dQ[kMaxN] = {0}, *dRk[kMaxN] = {0}, *dG[kMaxN] = {0};
  double *dQt[kMaxN] = {0}, *dAt[kMaxN] = {0};  // transposed, zero-padded (I_k x RQ) TMA panels
  int RQ = 16;
  bool use_tma = true;
  bool fuse_slice = true;  // see plan_mode
  bool pinv_ready = false; // M = pinv(R0) already launched for this mode (side stream, after K2)
  bool kt = false;         // Kruskal-tensor input (cpqr_set_ktensor): X never formed
  // short modes (I_k < R, the 10-way sine of sums): the factors are stored with
  // D_k = max(I_k, R) rows (zero rows below I_k) and dims[] holds D_k; tdims[] the true I_k.  The
  // zero rows change nothing in CP-ALS (their rows of X are zero), their QR rows of R_k are exact
  // zeros, and V_n keeps only its prod_{k != n} min(I_k, R) nonzero rows (mixed radix vq).
  bool short_modes = false;
  // odd I_1: mode 1 is stored padded to the next even size (a zero row in X and in A_1, the same
  // exact-zero argument as above), because TMA needs 16-byte global strides: with an odd I_1 every
  // A = prod_{j<k} I_j is odd and all stream passes would fall back to the register-staged kernels
  // (the paper's 75^5 shape: 5x slower).  CPQR_PAD_ODD=0 keeps the unpadded layout.
  bool pad1 = false;
  int64_t tdims[kMaxModes] = {0};
  int vq[kMaxModes] = {0};  // min(I_k, R): the V_n / Q0 row radix of mode k
  double* dVrs = nullptr;   // short modes: the shifted CholeskyQR factor R_s of V_n
  double* dGp2 = nullptr;   // first-level sums of the Gram partials (multi-kernel CholeskyQR, nb > 1024)
  double* dVrp = nullptr;   // short modes: R' of the CholeskyQR2 of V_n R_s^{-1}
  int ktS = 0;
  double* dKtLam = nullptr;
  double* dKtB[kMaxN] = {nullptr};
  double* dKtC = nullptr;  // cross products C_k (N blocks of up to max(R,S)^2)
  double* dKtM = nullptr;  // S x R
  double* dKtP = nullptr;  // k_kt_m chunk partials (large V_n)
  size_t ktP_elems = 0;
  size_t ktC_elems = 0;
  bool vn_cq = false;      // CholeskyQR2 V_n buffers allocated (some mode may use that path)
  bool vn_cq_always = false, vn_cq_tree = false, vn_mode_cq = false;  // per-mode choice (launch_kr_qr)
  int64_t vnJ = 0;         // R^{N-1}
  // tree QR of V_n across the Khatri-Rao factors (NEXT-2; vn_tree.cuh)
  bool vn_krtree = false;
  bool kr_standalone = false;  // a debug call: factor the shared group afresh
  double *dTrP[2] = {nullptr, nullptr}, *dTrS[2] = {nullptr, nullptr}, *dTrPa = nullptr, *dTrPb = nullptr,
         *dTrT = nullptr, *dTrQ = nullptr;
  double *dVn = nullptr, *dVq1 = nullptr, *dVgp = nullptr, *dVr1 = nullptr, *dVr2 = nullptr;
  bool tree = false;       // dimension-tree Multi-TTM (opt.mttm_tree, QR/SVD, N >= 3)
  int tree_h = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t evf = nullptr, evj = nullptr;
  double *dRstack = nullptr, *dV = nullptr, *dtauv = nullptr, *dQtop = nullptr, *dinner = nullptr;
  double* dMpinv = nullptr;
  double *dQ1 = nullptr, *dGp = nullptr, *dinnerp = nullptr, *dR1 = nullptr, *dR2 = nullptr;
  int factor_qr_mode = 0;  // 0 auto (CholeskyQR2, Householder fallback), 1 Householder only
  int nparts = 0;
  int stream_sms = 148;  // CTAs of the stream-X kernels (one SM left to the concurrent V_n QR)
  double *dlam = nullptr, *dQ0 = nullptr, *dR0 = nullptr, *dW = nullptr, *dWp = nullptr,
         *dAhat = nullptr;
  double* dnX2p = nullptr;   // per-slab partial ||X||^2 (CPQR_COMM_LOCAL), summed in rank order
  double* dSk = nullptr;     // stream-K partial slots: 2 per CTA x (256-row unit x R)
  unsigned* dSkCnt = nullptr;  // stream-K fused fix-up: arrival counter per CTA (self re-arming)
  int streamk = -1;          // CPQR_STREAMK: -1 auto, 0 off, 1 always (strided stream kernel)
  // programmatic dependent launch along the per-mode chain (CPQR_PDL=1).  Off by default: measured
  // slower in every config (interleaved A/B, 30 sweeps x 2: C2 -3 %, C3 -1 %, C5 -1 %; with early
  // launch_dependents triggers in the persistent stream kernels C2 -7 %, C3 tree -9 %)
  bool pdl = false;
  bool q0_stair = false;     // staircase Q0 apply (CPQR_Q0_STAIR=1, k_q0_apply_tc<NT, true>)
  // overlap schedule: the tail of mode n (Q0 apply, solve, factor QR) runs on stream
  // tl beside the stream-X pass of mode n+1 whenever that pass does not contract mode n
  bool overlap = false, tail_single = false;
  // CP-ALS (NE), N = 3, one GPU: the one-CTA NE tail of mode n on stream tl beside the MTTKRP's first
  // TTM of mode n+1, which contracts mode (n+2) mod 3 -- not the factor that tail is updating
  bool overlap_ne = false;
  int overlap_reserve = 4;   // SMs the stream passes leave free for the tail / V_n QR
  // stream passes one CTA per SM so the reserved SMs stay free (CPQR_OVERLAP_CW1=1).  Off: the
  // two-CTA-per-SM passes (R <= 12) lose more than the freed SMs gain (interleaved A/B, 40 sweeps
  // x 2: C2 2575 vs 2680, C3 524 vs 560; C4 488 vs 484)
  bool ov_cw1 = false;
  cudaStream_t tl = nullptr;
  cudaEvent_t evY[kMaxN] = {}, evQ[kMaxN] = {}, evK[kMaxN] = {};
  double* dY = nullptr;      // Y_(n) of the overlap schedule (read by the tail while the next pass runs)
  size_t dY_elems = 0;
  // CPQR_TRACE=1 (debugging, eager sweeps only): timing events around the overlap schedule's
  // launches on each stream, printed to stderr after every sweep as a timeline
  bool trace = false;
  std::vector<std::pair<cudaEvent_t, std::string>> tev;
  size_t ntev = 0;
  unsigned* dq0cnt = nullptr;  // per-row-block arrival counters of k_q0_apply_tc (self re-arming)
  double* dZ = nullptr;        // Z fusion: Z = (Q_k (x) I) Q0 of the current mode (k_zform)
  size_t dZ_elems = 0;
  double* buf[2] = {nullptr, nullptr};
  size_t buf_elems = 0;
  double* dPart = nullptr;
  size_t part_elems = 0;
  int* dperm = nullptr;
  double* dKrWork = nullptr;
  double *dnX2 = nullptr, *dfit = nullptr, *dfits = nullptr, *dred = nullptr;
  size_t dred_elems = 0;
  int fits_cap = 0;
  unsigned* dflags = nullptr;
  double* hpin = nullptr;  // pinned: [0] fit, [1] flags
  bool plans_valid = false;
  cudaGraphExec_t gexec = nullptr;   // one sweep
  cudaGraphExec_t gexecG = nullptr;  // gsw sweeps in one graph (the tails overlap across sweeps)
  // sweeps per multi-sweep graph (CPQR_GRAPH_SWEEPS).  Default 1: measured slower with more
  // (interleaved, 40 sweeps x 2: C2 2537 / 2450 / 2285 sweeps/s at 1 / 2 / 4, C4 480 / 466 / 454)
  int gsw = 1;
  int64_t launches_G = 0;
  bool graph_valid = false;
  unsigned* dfitc = nullptr;         // device counter: next slot of dfits (k_store_fit)
  bool ov_first = true, ov_join = true;  // overlap schedule: first / last sweep of a capture
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // profiling (opt.profile): events recorded at phase boundaries; the time since the previous
  // mark is attributed to the mark's phase (cpqr_get_profile ms[0..6])
  std::vector<cudaEvent_t> evp;
  std::vector<int> evphase;
  std::vector<int64_t> evlaunch;
  int nmarks = 0;
  cpqr_profile prof;
  int64_t launch_count = 0;
  int64_t launches_per_sweep = -1;
  double last_fit = NAN;
  unsigned flags = 0;
  std::string err;
  int kr_smem = 0;
  size_t wp_elems = 0;
};

namespace {

cpqr_status fail(cpqr_ctx* c, cpqr_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(c, CPQR_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                \
  } while (0)
#define CKL()                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, CPQR_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                  \
    c->launch_count++;                                                                        \
  } while (0)
#define CN(call)                                                                               \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return fail(c, CPQR_ENCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)
#define TRY(x)                       \
  do {                               \
    cpqr_status s_ = (x);            \
    if (s_ != CPQR_OK) return s_;    \
  } while (0)

int64_t prod(const int64_t* d, int a, int b) {  // prod d[a..b)
  int64_t p = 1;
  for (int i = a; i < b; ++i) p *= d[i];
  return p;
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

bool ne_family(int v) { return v == CPQR_NE || v == CPQR_PINV; }  // Alg. 1 (normal equations)

int choose_kc(int I, int ld) {
  const size_t row = (size_t)ld * sizeof(double);
  const int full = round_up(I, 16);
  if ((size_t)full * row <= kQSmemMax) return full;
  int kc = (int)(kQSmemMax / row) / 16 * 16;
  return std::max(16, kc);
}

template <typename K>
int grid_for(K kernel, int64_t units, size_t smem, int sms) {
  static bool dummy = false;
  (void)dummy;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, smem);
  if (nb < 1) nb = 1;
  int64_t g = std::min<int64_t>(units, (int64_t)sms * nb);
  return (int)std::max<int64_t>(1, g);
}

// ----------------------------------------------------------------------- kernel dispatch
template <int MT, int NT, bool VEC>
void run_strided(const TtmStep& s, int R, cudaStream_t st, int sms) {
  constexpr int LD = 8 * NT + 4;
  const int KC = choose_kc(s.I, LD);
  const size_t smem = (size_t)KC * LD * sizeof(double);
  const int64_t BMc = (int64_t)kWarps * 8 * MT;
  const int64_t units = ((s.A + BMc - 1) / BMc) * s.B;
  auto k = k_ttm_strided<MT, NT, VEC>;
  const int grid = grid_for(k, units, smem, sms);
  k<<<grid, kThreads, smem, st>>>(s.in, s.A, s.I, s.B, s.Q, s.ldq, R, s.out, KC);
}
void launch_strided(const TtmStep& s, int R, cudaStream_t st, int sms) {
  const bool vec = (s.A % 2 == 0) && (((uintptr_t)s.in & 15) == 0);
  switch ((R + 7) / 8) {
    case 1: vec ? run_strided<4, 1, true>(s, R, st, sms) : run_strided<4, 1, false>(s, R, st, sms); break;
    case 2: vec ? run_strided<4, 2, true>(s, R, st, sms) : run_strided<4, 2, false>(s, R, st, sms); break;
    case 3: vec ? run_strided<4, 3, true>(s, R, st, sms) : run_strided<4, 3, false>(s, R, st, sms); break;
    default: vec ? run_strided<4, 4, true>(s, R, st, sms) : run_strided<4, 4, false>(s, R, st, sms); break;
  }
}

template <int MT, int NF, bool VEC>
void run_fiber(const TtmStep& s, int R, cudaStream_t st, int sms) {
  constexpr int LD = 8 * MT + (VEC ? 2 : 4);
  const int KC = choose_kc(s.I, LD);
  const size_t smem = (size_t)KC * LD * sizeof(double);
  const int64_t BF = (int64_t)kWarps * 8 * NF;
  const int64_t units = (s.F + BF - 1) / BF;
  auto k = k_ttm_fiber<MT, NF, VEC>;
  const int grid = grid_for(k, units, smem, sms);
  k<<<grid, kThreads, smem, st>>>(s.in, s.I, s.F, s.Q, s.ldq, R, s.out, KC);
}
void launch_fiber(const TtmStep& s, int R, cudaStream_t st, int sms) {
  const bool vec = (s.I % 2 == 0) && (((uintptr_t)s.in & 15) == 0);
  switch ((R + 7) / 8) {
    case 1: vec ? run_fiber<1, 4, true>(s, R, st, sms) : run_fiber<1, 4, false>(s, R, st, sms); break;
    case 2: vec ? run_fiber<2, 2, true>(s, R, st, sms) : run_fiber<2, 2, false>(s, R, st, sms); break;
    case 3: vec ? run_fiber<3, 2, true>(s, R, st, sms) : run_fiber<3, 2, false>(s, R, st, sms); break;
    default: vec ? run_fiber<4, 2, true>(s, R, st, sms) : run_fiber<4, 2, false>(s, R, st, sms); break;
  }
}

int slice_fw(int R) { return ((R + 7) / 8 == 1) ? 32 : 16; }  // 8 * NF

template <int MT, int NF, bool VEC>
void run_slice(const TtmStep& s, int R, cudaStream_t st, int sms) {
  constexpr int LD = 8 * MT + (VEC ? 2 : 4);
  const int KC = choose_kc(s.I1, LD);
  const size_t smem = (size_t)KC * LD * sizeof(double);
  const int64_t wunits = (int64_t)s.nseg * s.L;
  const int64_t cunits = (wunits + kWarps - 1) / kWarps;
  auto k = k_mttm_slice<MT, NF, VEC>;
  const int grid = grid_for(k, cunits, smem, sms);
  k<<<grid, kThreads, smem, st>>>(s.in, s.I1, s.I2, s.L, s.Q, s.ldq, s.Q2, s.ldq2, R, s.gps, s.out, KC);
}
void launch_slice(const TtmStep& s, int R, cudaStream_t st, int sms) {
  const bool vec = (s.I1 % 2 == 0) && (((uintptr_t)s.in & 15) == 0);
  switch ((R + 7) / 8) {
    case 1: vec ? run_slice<1, 4, true>(s, R, st, sms) : run_slice<1, 4, false>(s, R, st, sms); break;
    case 2: vec ? run_slice<2, 2, true>(s, R, st, sms) : run_slice<2, 2, false>(s, R, st, sms); break;
    case 3: vec ? run_slice<3, 2, true>(s, R, st, sms) : run_slice<3, 2, false>(s, R, st, sms); break;
    default: vec ? run_slice<4, 2, true>(s, R, st, sms) : run_slice<4, 2, false>(s, R, st, sms); break;
  }
}

// ------------------------------------------------------------------------- plan building
// Multi-TTM Y = X x_{k != n} Q_k^T (Alg. 2 line 8).  Stream-X pass: modes 1 and 2 together
// (k_mttm_slice) when n >= 3, else the last mode (k_ttm_strided, the largest contiguous GEMM);
// the remaining TTMs run on the (R/I)-smaller intermediate in decreasing-dimension order
// (ties by decreasing mode, reading 5).
struct PlanIn {
  const double* X;
  const int64_t* ld;  // local dims
  int N, R, n;
  const double* Q[kMaxN];   // per-mode operand (Q_k for QR, A_k for NE); mode N-1 already slab-offset
  int64_t ldq[kMaxN];
  const double* Qt[kMaxN];  // transposed padded panels (TMA), slab-offset for mode N-1
  int RQ;
  bool ne;
  bool tma;
  bool fuse;  // fused two-mode slice kernel allowed for n >= 3
  int pad0 = 0;  // 1: mode 1 is stored padded by one row (odd I_1): orders compare the true dimension
  bool zf_ok = false;  // Z fusion allowed (one slab, no exchange, QR / SVD, dense apply)
  bool ne_ov = false;  // NE overlap schedule: first TTM over mode (n+1) mod 3
  int sms;
  bool tree = false;        // dimension-tree Multi-TTM (QR/SVD variants)
  int h = 0;                // tree split: halves [0, h) and [h, N)
  bool tree_fresh = false;  // this mode computes its half's intermediate from X
  double* tbuf = nullptr;   // the tree buffer
  double* sk = nullptr;     // stream-K partial slots of the strided stream kernel
  unsigned* skcnt = nullptr;  // their arrival counters (zeroed, self re-arming)
  int skm = -1;             // stream-K mode (CPQR_STREAMK)
  bool overlap = false;     // overlap schedule: N = 3 first contraction (n+1) mod 3
  bool ov_cw1 = true;       // overlap schedule: one CTA per SM in the stream passes (CPQR_OVERLAP_CW1)
  double* ybuf = nullptr;   // overlap schedule: the final step writes Y here
};

// Device allocations.  Debugging switches (compute-sanitizer is unavailable on this pool):
//  * CPQR_POISON=1 fills every block with 0xFF bytes (NaN as fp64): a kernel reading memory before
//    it was written shows up as NaN in the parity tests (initcheck's job);
//  * CPQR_CANARY=1 surrounds every block with 4 KB guard bands of a byte pattern, and every
//    cpqr_sweep / cpqr_destroy verifies all of them: a kernel writing out of bounds (before or past
//    its buffer) fails the call with ECUDA and names the allocation (memcheck's job for writes).
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5;
struct Guarded {
  char* base;
  size_t bytes;
};
std::vector<Guarded>& guard_registry() {
  static std::vector<Guarded> g;
  return g;
}
std::mutex& guard_mutex() {
  static std::mutex m;
  return m;
}
bool canary_on() {
  static const bool on = getenv("CPQR_CANARY") && atoi(getenv("CPQR_CANARY")) == 1;
  return on;
}

template <typename T>
cudaError_t dmalloc(T** p, size_t bytes) {
  cudaError_t e;
  if (canary_on()) {
    char* base = nullptr;
    e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuard);
    if (e != cudaSuccess) return e;
    e = cudaMemset(base, kGuardByte, bytes + 2 * kGuard);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(guard_mutex());
    guard_registry().push_back({base, bytes});
    *p = reinterpret_cast<T*>(base + kGuard);
  } else {
    e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  }
  static const bool poison = getenv("CPQR_POISON") != nullptr;
  if (e == cudaSuccess && poison) {
    e = cudaMemset(*p, 0xff, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  return e;
}

// cudaFree for blocks from dmalloc (the guarded base under CPQR_CANARY)
void dfree(void* p) {
  if (!p) return;
  if (canary_on()) {
    std::lock_guard<std::mutex> lk(guard_mutex());
    auto& g = guard_registry();
    for (size_t i = 0; i < g.size(); ++i)
      if (g[i].base + kGuard == p) {
        cudaFree(g[i].base);
        g.erase(g.begin() + i);
        return;
      }
  }
  cudaFree(p);
}

// CPQR_CANARY: the number of guard bytes changed in all live blocks (0 = clean); *which = the first
// offending block's size for the error message
size_t canary_violations(size_t* which) {
  if (!canary_on()) return 0;
  cudaDeviceSynchronize();
  size_t bad = 0;
  std::vector<unsigned char> h(kGuard);
  std::lock_guard<std::mutex> lk(guard_mutex());
  for (const Guarded& g : guard_registry()) {
    for (int side = 0; side < 2; ++side) {
      const char* src = side ? g.base + kGuard + g.bytes : g.base;
      if (cudaMemcpy(h.data(), src, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return (size_t)-1;
      size_t nb = 0;
      for (unsigned char b : h) nb += (b != kGuardByte);
      if (nb && !bad && which) *which = g.bytes;
      bad += nb;
    }
  }
  return bad;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// fp64 tiled map, SWIZZLE_128B (inner box = 16 doubles = 128 B), zero OOB fill.
bool make_tmap(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
               const uint32_t* box) {
  auto enc = get_encode();
  if (!enc) return false;
  if (((uintptr_t)base & 15) != 0) return false;
  for (int i = 0; i < rank - 1; ++i)
    if (strides_bytes[i] % 16 != 0 || strides_bytes[i] >= (1ull << 40)) return false;
  for (int i = 0; i < rank; ++i)
    if (dims[i] == 0 || dims[i] >= (1ull << 31)) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void*>(base),
                   (const cuuint64_t*)dims, (const cuuint64_t*)strides_bytes, (const cuuint32_t*)box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

constexpr size_t kSmemOptin = 227 * 1024;

// Ring depth: as many stages as fit, capped.  Deeper is not better for the HBM-bound passes: a
// compute-free replica of the strided ring (tools/ubench/tma_bench.cu) streams C3's X at 7.2 TB/s
// with 3-4 stages of 32 KB per SM but 6.4 TB/s with 6 (more requests in flight than the memory
// system serves well), and the interleaved sweeps of tools/ab_stages.sh set the defaults:
// strided 4 (3 when a unit has <= 3 k-steps), small slice 3, the rest 8 (C3 +2.5 %, C4 +9 %).
// Env: CPQR_STAGES caps every ring, then CPQR_ST_<KIND> the one kernel kind.
int stages_for(size_t stage, size_t extra, const char* kind_env, int cap = 8) {
  const size_t avail = kSmemOptin - 1024 - 2048 - extra;
  if (const char* v = getenv("CPQR_STAGES")) cap = std::max(2, atoi(v));
  if (const char* v = getenv(kind_env)) cap = std::max(2, atoi(v));
  return (int)std::min<size_t>(cap, avail / stage);
}

// Multi-TTM Y = X x_{k != n} Q_k^T (Alg. 2 line 8).  Stream-X pass: modes 1 and 2 together
// (fused slice kernel) when n >= 3 and the pass is HBM-bound (R < 24: R/4 flop per byte is below
// the FP64-DMMA : HBM balance of ~5.7); when it is FP64-bound (R >= 24) one mode alone, no second
// contraction on the critical DMMA loop: for N = 3 the middle mode (strided kernel), for N >= 4 the
// largest dimension, ties to the highest mode (the strided kernel's slices then have the most
// rows); for n < 3 the last mode (strided kernel, the largest contiguous GEMM).  The remaining TTMs run on the (R/I)-smaller intermediate in decreasing-dimension order
// (ties by decreasing mode, reading 5).  TMA kernels whenever the layout allows
// (even leading dimension, 16-B aligned base), else the register-staged kernels.
// N-tiles of 8 fibres per consumer warp in the fused slice kernel (box height kCW * 8 * NF)
static int slice_nf(int I2) { return I2 >= 256 ? 4 : 2; }

// k_ttm_small (small_ttm.cuh) for a TTM on an intermediate of A I B <= kSmallTtmMax elements (the
// stream pass's output: L2 resident): WK warps x KC CTAs split the contraction so that ~2 CTAs x
// 8 warps per SM have work.  False when the CTA's Q rows exceed the shared-memory budget or the
// row blocks exceed the arrival counters (then the TMA / register-staged kernels run).
constexpr int64_t kSmallTtmMax = 8ll << 20;
bool small_split(int64_t A, int I, int64_t B, int R, int sms, int& WK, int& KC, size_t& smem) {
  const int64_t M = A * B, rt = (M + 15) / 16;
  int64_t KT = ((int64_t)sms * 16 + rt - 1) / rt;
  KT = std::max<int64_t>(1, std::min<int64_t>(KT, std::max(1, I / 16)));
  WK = KT >= 8 ? 8 : KT >= 4 ? 4 : KT >= 2 ? 2 : 1;
  KC = (int)((KT + WK - 1) / WK);
  const int NT = (R + 7) / 8;
  smem = (size_t)WK * 16 * (8 / WK) * (8 * NT + 1) * sizeof(double);  // the warp partials
  const int64_t rcs = (M + 16 * (8 / WK) - 1) / (16 * (8 / WK));
  return KC == 1 || rcs <= 2 * sms;
}

void plan_mode(const PlanIn& in, Plan& p, double* const bufs[2], double* part) {
  p.steps.clear();
  p.diags.clear();
  const int N = in.N, R = in.R, n = in.n;
  const int NT = (R + 7) / 8, NQB = (NT + 1) / 2;
  int64_t cur[kMaxN];
  for (int k = 0; k < N; ++k) cur[k] = in.ld[k];
  const double* src = in.X;
  int nb = 0;
  p.max_buf = 0;
  p.part = 0;
  std::vector<int> todo;
  auto qmap = [&](TtmStep& s, int k, int64_t I) {
    const uint64_t d[2] = {(uint64_t)in.RQ, (uint64_t)I};
    const uint64_t st[1] = {(uint64_t)in.RQ * 8};
    const uint32_t box[2] = {16, 16};
    return in.Qt[k] && make_tmap(&s.mq, in.Qt[k], 2, d, st, box);
  };
  // dimension of mode k for the contraction orders: the pad row of an odd I_1 is not
  // a reason to contract mode 1 first
  auto dim_of = [&](int k) { return (k == 0 && cur[0] == in.ld[0]) ? cur[0] - in.pad0 : cur[k]; };
  double* out_override = nullptr;  // tree plans: the last step of a half pass writes the tree buffer
  auto advance = [&](double* out) {  // the next step reads `out`
    src = out;
    if (!out_override) nb ^= 1;
  };
  auto emit_ttm = [&](int k) {
    TtmStep s{};
    s.modes = 1u << k;
    s.in = src;
    s.out = out_override ? out_override : bufs[nb];
    s.Q = in.Q[k];
    s.ldq = in.ldq[k];
    if (k == 0) {
      s.kind = 1;
      s.I = (int)cur[0];
      s.F = prod(cur, 1, N);
      if (in.tma && s.I % 2 == 0 && s.F < (1ll << 31) && bufs[0]) {
        const uint64_t d[2] = {(uint64_t)s.I, (uint64_t)s.F};
        const uint64_t st[1] = {(uint64_t)s.I * 8};
        const uint32_t box[2] = {16, 128};
        if (make_tmap(&s.mx, src, 2, d, st, box) && qmap(s, k, s.I)) {
          s.kind = 5;
          s.S = stages_for(128 * 128 + NQB * kBoxBytes, 0, "CPQR_ST_FIBER");
        }
      }
    } else {
      s.kind = 0;
      s.A = prod(cur, 0, k);
      s.I = (int)cur[k];
      s.B = prod(cur, k + 1, N);
      if (in.tma && s.A % 2 == 0 && s.A < (1ll << 31) && s.B < (1ll << 31) && bufs[0]) {
        const uint64_t d[3] = {(uint64_t)s.A, (uint64_t)s.I, (uint64_t)s.B};
        const uint64_t st[2] = {(uint64_t)s.A * 8, (uint64_t)s.A * s.I * 8};
        const uint32_t box[3] = {16, 16, 1};
        if (make_tmap(&s.mx, src, 3, d, st, box) && qmap(s, k, s.I)) {
          s.kind = 4;
          s.P = in.sk;
          s.cnt = in.skcnt;
          s.skm = in.skm;
          s.cw1 = (in.overlap && in.ov_cw1) ? 1 : 0;
          s.S = stages_for(16 * kBoxBytes + NQB * kBoxBytes, 0, "CPQR_ST_STRIDED", (s.I + kBK - 1) / kBK <= 3 ? 3 : 4);
        }
      }
    }
    // an intermediate (not X) small enough to sit in L2: the latency-bound small-TTM kernel
    const bool small_off = getenv("CPQR_TTM_SMALL") && atoi(getenv("CPQR_TTM_SMALL")) == 0;  // per plan build (tests)
    {
      const int64_t A = prod(cur, 0, k), B = prod(cur, k + 1, N);
      const int I = (int)cur[k];
      int wk, kc;
      size_t smem;
      // where the TMA kernels are starved: units of 32 CW rows (CW = 4 for R <= 12, else 8) or of
      // 128 fibres fewer than half the SMs, or rows of A < 32 filling few of a unit's rows (C2's
      // intermediates); on C3 / C4's the TMA kernels measured faster (A/B)
      const int64_t ur = (k == 0) ? 128 : (R <= 12 ? 128 : 256);
      const int64_t tunits = (k == 0) ? (B + ur - 1) / ur : ((A + ur - 1) / ur) * B;
      const bool starved = tunits < in.sms / 2 || (k != 0 && A < 32);
      const bool force = getenv("CPQR_TTM_SMALL") && atoi(getenv("CPQR_TTM_SMALL")) == 2;  // tests
      if (!small_off && (starved || force) && src != in.X && (A * I * B <= kSmallTtmMax || (force && A * I * B < (1ll << 30))) && in.Qt[k] &&
          small_split(A, I, B, R, in.sms, wk, kc, smem)) {
        s.kind = 9;
        s.A = A; s.I = I; s.B = B;
        s.Qt = in.Qt[k];
        s.rq = in.RQ;
        s.wk = wk; s.kc = kc;
        s.P = part;
        s.cnt = in.skcnt;
        s.S = (int)smem;
        if (kc > 1) p.part = std::max(p.part, (size_t)((A * B + 16 * (8 / wk) - 1) / (16 * (8 / wk))) * kc * 16 * (8 / wk) * R);
      }
    }
    cur[k] = R;
    p.max_buf = std::max(p.max_buf, (size_t)prod(cur, 0, N));
    p.steps.push_back(s);
    advance(s.out);
  };
  // fused contraction of the two slowest modes f2 = f - 1 and f = N - 1 of src in one pass
  // (k_strided2_tma, R <= 8): false if the layout does not allow it (the caller then emits two TTMs)
  auto emit_ttm2 = [&](int f2, int f) {
    const bool off = getenv("CPQR_STR_FUSE2") && atoi(getenv("CPQR_STR_FUSE2")) == 0;  // per plan build (tests)
    if (off || !in.tma || R > 8 || f != N - 1 || f2 != f - 1 || f2 < 1 || !in.Qt[f] || !bufs[0]) return false;
    TtmStep s{};
    s.modes = (1u << f2) | (1u << f);
    s.in = src;
    s.out = out_override ? out_override : bufs[nb];
    s.A = prod(cur, 0, f2);
    s.I = (int)cur[f2];
    s.B = cur[f];
    if (s.A % 2 != 0 || s.A < 128 || s.A >= (1ll << 31) || s.B >= (1ll << 31)) return false;
    const uint64_t d[3] = {(uint64_t)s.A, (uint64_t)s.I, (uint64_t)s.B};
    const uint64_t st[2] = {(uint64_t)s.A * 8, (uint64_t)s.A * s.I * 8};
    const uint32_t box[3] = {16, 16, 1};
    if (!make_tmap(&s.mx, src, 3, d, st, box) || !qmap(s, f2, s.I)) return false;
    s.kind = 10;
    s.Q = in.Q[f2];
    s.ldq = in.ldq[f2];
    s.Qt = in.Qt[f];
    s.rq = in.RQ;
    s.S = stages_for(9 * kBoxBytes, 0, "CPQR_ST_STRIDED2", 8);
    cur[f2] = R;
    cur[f] = R;
    p.max_buf = std::max(p.max_buf, (size_t)prod(cur, 0, N));
    p.steps.push_back(s);
    advance(s.out);
    return true;
  };
  // fused contraction of modes 0 and 1 of src (fused slice kernels, Alg. 2 line 8)
  auto emit_slice = [&]() {
      TtmStep s{};
      s.modes = 3u;
      s.kind = 2;
      s.in = src;
      s.I1 = (int)cur[0];
      s.I2 = (int)cur[1];
      s.L = prod(cur, 2, N);
      s.Q = in.Q[0];
      s.ldq = in.ldq[0];
      s.Q2 = in.Q[1];
      s.ldq2 = in.ldq[1];
      bool tma = false;
      if (in.tma && s.I1 % 2 == 0 && s.L < (1ll << 31) && bufs[0]) {
        const uint64_t d[3] = {(uint64_t)s.I1, (uint64_t)s.I2, (uint64_t)s.L};
        const uint64_t st[2] = {(uint64_t)s.I1 * 8, (uint64_t)s.I1 * s.I2 * 8};
        // slice TMA decomposition: 128-fibre boxes run CW = 4 warps of NF = 4 fibre tiles, two CTAs
        // per SM (C3 per-mode 524 -> 565 sweeps/s, tree 895 -> 947; CPQR_SLICE_CW=8 restores 8 warps
        // of NF = 2); wider slices keep 256-fibre boxes of 8 warps x NF = 4 unless CPQR_SLICE_WIDE4=1
        static const int scw_env = getenv("CPQR_SLICE_CW") ? atoi(getenv("CPQR_SLICE_CW")) : 0;
        static const bool wide4 = getenv("CPQR_SLICE_WIDE4") && atoi(getenv("CPQR_SLICE_WIDE4")) == 1;
        s.gps = slice_nf(s.I2);
        // 256-fibre boxes waste their second block when I_2 is just above 256 (300^4: 300 of 512
        // fibre slots, and the pass turns DMMA-bound): 128-fibre boxes when they fill >= 10 % better
        auto fillf = [&](int bn) { return (double)s.I2 / ((double)bn * (double)((s.I2 + bn - 1) / bn)); };
        const bool narrow = s.gps == 4 && fillf(128) > 1.10 * fillf(256);
        if (scw_env != 8 && !(in.overlap && in.ov_cw1) && (s.gps == 2 || wide4 || narrow)) { s.cw = 4; s.gps = 4; }
        const uint32_t box[3] = {16, (uint32_t)(s.cw * 8 * s.gps), 1};
        tma = make_tmap(&s.mx, src, 3, d, st, box) && qmap(s, 0, s.I1);
      }
      const bool small = tma && s.I2 <= 64 && s.I2 % 8 == 0 && NT <= 2;
      if (small) {
        const uint64_t d[3] = {(uint64_t)s.I1, (uint64_t)s.I2, (uint64_t)s.L};
        const uint64_t st[2] = {(uint64_t)s.I1 * 8, (uint64_t)s.I1 * s.I2 * 8};
        const uint32_t box[3] = {16, (uint32_t)s.I2, 8};
        if (make_tmap(&s.mx, src, 3, d, st, box)) {
          s.kind = 8;
          s.S = stages_for((size_t)s.I2 * 8 * 128 + NQB * kBoxBytes, 0, "CPQR_ST_SMALL", 3);
          s.out = out_override ? out_override : bufs[nb];
          p.steps.push_back(s);
        } else {
          tma = false;
        }
      }
      if (small && s.kind == 8) {
        // done
      } else if (tma) {
        s.kind = 6;
        const int MT = NT;
        const int BN = s.cw * 8 * s.gps;
        if (s.cw == 4) {
          const size_t stage = (size_t)BN * 128 + NQB * kBoxBytes, extra = (size_t)4 * slice_ldy(R) * R * 8;
          s.S = std::min<int>(stages_for(stage, extra, "CPQR_ST_SLICE", 4), (int)((110 * 1024 - 3072 - extra) / stage));
        } else {
          s.S = stages_for((size_t)BN * 128 + NQB * kBoxBytes, (size_t)kCW * slice_ldy(R) * R * 8, "CPQR_ST_SLICE");
        }
        s.nfb = (s.I2 + BN - 1) / BN;
        const int64_t U = s.L * s.nfb;
        s.G = std::min<int64_t>(U, (int64_t)in.sms * (s.cw == 4 ? 2 : 1));
        int ns = 1;
        for (int64_t l = 0; l < s.L; ++l) {
          const int64_t c0 = ((l * s.nfb + 1) * s.G - 1) / U, c1 = ((l * s.nfb + s.nfb) * s.G - 1) / U;
          ns = std::max<int>(ns, (int)(c1 - c0 + 1));
        }
        s.nslots = ns;
        s.out = out_override ? out_override : bufs[nb];
        s.P = part;
        if (ns > 1) p.part = std::max(p.part, (size_t)s.L * ns * R * R);
        (void)MT;
        p.steps.push_back(s);
        if (ns > 1) {
          TtmStep f = s;
          f.kind = 7;
          p.steps.push_back(f);
        }
      } else {
        const int fw = slice_fw(R);
        const int ngr = (s.I2 + fw - 1) / fw;
        const int64_t target = (int64_t)in.sms * 2 * kWarps * 4;
        int gps = 1;
        if ((int64_t)ngr * s.L > target) gps = (int)std::min<int64_t>(ngr, ((int64_t)ngr * s.L + target - 1) / target);
        s.gps = gps;
        s.nseg = (ngr + gps - 1) / gps;
        if (s.nseg > 1) {
          s.out = part;
          p.part = std::max(p.part, (size_t)s.nseg * s.L * R * R);
        } else {
          s.out = out_override ? out_override : bufs[nb];
        }
        TtmStep sr = s;
        p.steps.push_back(s);
        if (s.nseg > 1) {
          sr.kind = 3;  // reduce partials
          sr.in = part;
          sr.out = out_override ? out_override : bufs[nb];
          p.steps.push_back(sr);
        }
      }
      cur[0] = R;
      cur[1] = R;
      p.max_buf = std::max(p.max_buf, (size_t)prod(cur, 0, N));
      advance(out_override ? out_override : bufs[nb]);
  };
  if (in.ne) {
    // MTTKRP M_n = X_(n) Z_n: one dense TTM with A_k over the largest local dimension (
    // ties: mode 1 for n >= 1, else the last mode -- with slabs the last mode is the smallest), then
    // Khatri-Rao-diagonal contractions.
    int rmode = (n >= 1) ? 0 : N - 1;
    for (int k = N - 1; k >= 0; --k)
      if (k != n && cur[k] > cur[rmode]) rmode = k;
    if (in.ne_ov && N == 3) rmode = (n + 1) % 3;  // never mode n-1, whose factor the previous tail updates
    emit_ttm(rmode);
    int nd = N;
    int64_t dd[kMaxN];
    int orig[kMaxN];
    for (int k = 0; k < N; ++k) { dd[k] = cur[k]; orig[k] = k; }
    for (int k = N - 1; k >= 0; --k) {
      if (k == n || k == rmode) continue;
      int pos = -1, rpos = -1;
      for (int d = 0; d < nd; ++d) {
        if (orig[d] == k) pos = d;
        if (orig[d] == rmode) rpos = d;
      }
      DiagStep ds{};
      ds.in = src;
      ds.out = bufs[nb];
      ds.nd = nd;
      for (int d = 0; d < nd; ++d) ds.dims[d] = dd[d];
      ds.k = pos;
      ds.rm = rpos;
      ds.Ak = in.Q[k];
      ds.lda = in.ldq[k];
      ds.mode = k;
      p.diags.push_back(ds);
      for (int d = pos; d < nd - 1; ++d) { dd[d] = dd[d + 1]; orig[d] = orig[d + 1]; }
      --nd;
      src = bufs[nb];
      nb ^= 1;
    }
    p.Y = src;
    p.nd = nd;
    for (int d = 0; d < nd; ++d) p.ydims[d] = dd[d];
    p.m_rowmajor = (rmode < n) ? 1 : 0;  // (R, I_n) column-major == row-major I_n x R
    return;
  }
  if (in.tree && N >= 3) {
    // Dimension tree: modes [0, h) share T_L = X x_{k >= h} Q_k^T, modes
    // [h, N) share T_R = X x_{k < h} Q_k^T.  The first mode of each half streams X once into the
    // tree buffer; the others start from it.  Same Y_(n) as the per-mode Multi-TTM up to rounding.
    const int h = in.h;
    const bool left = n < h;
    const int o0 = left ? h : 0, o1 = left ? N : h;  // the other half [o0, o1)
    if (in.tree_fresh) {
      std::vector<int> ord;
      if (left) {
        // the right half's modes by decreasing LOCAL dimension, ties last mode first
        // (strided, B = 1): with slabs the slab mode is the smallest and goes last
        for (int k = N - 1; k >= h; --k) ord.push_back(k);
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return dim_of(a) > dim_of(b); });
        size_t q0 = 0;
        if (ord.size() >= 2 && ord[0] == N - 1 && ord[1] == N - 2 && in.fuse && R <= 8) {
          // the two slowest modes in one pass (k_strided2_tma), straight into the tree buffer if
          // they are the whole right half
          if (ord.size() == 2) out_override = in.tbuf;
          if (emit_ttm2(N - 2, N - 1)) q0 = 2;
          else out_override = nullptr;
        }
        for (size_t q = q0; q < ord.size(); ++q) {
          if (q + 1 == ord.size()) out_override = in.tbuf;
          emit_ttm(ord[q]);
        }
      } else if (h >= 2 && in.fuse) {
        if (h == 2) out_override = in.tbuf;
        emit_slice();
        for (int k = 2; k < h; ++k) {
          if (k == h - 1) out_override = in.tbuf;
          emit_ttm(k);
        }
      } else {
        // the left half's modes by decreasing dimension, ties highest mode first (the strided kernel
        // with the most rows A per slice; mode 0, the fibre kernel, last): h = 2 gives (1, 0)
        for (int k = h - 1; k >= 0; --k) ord.push_back(k);
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return dim_of(a) > dim_of(b); });
        for (size_t q = 0; q < ord.size(); ++q) {
          if (q + 1 == ord.size()) out_override = in.tbuf;
          emit_ttm(ord[q]);
        }
      }
      out_override = nullptr;
      p.tree_elems = (size_t)prod(cur, 0, N);
    } else {
      src = in.tbuf;
      for (int k = o0; k < o1; ++k) cur[k] = R;
    }
    for (int k = left ? 0 : h; k < (left ? h : N); ++k) if (k != n) todo.push_back(k);
  } else if (N == 3 && n == 2 && !in.fuse && !in.overlap) {
    emit_ttm(1);  // stream pass over the middle mode (strided kernel), then mode 0 on the intermediate
    todo.push_back(0);
  } else if (N >= 3 && n >= 2 && in.fuse && !(N == 3 && in.overlap)) {
    emit_slice();
    for (int k = 2; k < N; ++k) if (k != n) todo.push_back(k);
  } else if (N == 3 && in.overlap) {
    // overlap schedule: mode n's pass contracts mode (n+1) mod 3, never the mode n-1 whose factor
    // the previous tail is still updating (the fibre kernel on X for n = 2)
    const int f = (n + 1) % 3;
    emit_ttm(f);
    todo.push_back(3 - n - f);
  } else if (N >= 3) {
    // n < 2: the stream pass contracts the largest LOCAL dimension first; ties go to
    // the last mode (strided kernel, B = 1, the largest contiguous GEMM).  With p > 1 slabs the last
    // mode is the smallest local one and is contracted last, so every intermediate scales as 1/p.
    // (Also n >= 2 without the fused slice pass, N >= 4: contracting mode 1 first there gave the
    // strided kernel slices of only A = I_1 rows -- 75^5 R = 32: 16.4 ms per pass against 5.7.)
    int f = (n == N - 1) ? N - 2 : N - 1;
    for (int k = f - 1; k >= 0; --k)
      if (k != n && dim_of(k) > dim_of(f)) f = k;
    // HBM-bound low rank, N >= 4: when the next mode in the order is f - 1, both go in one pass
    // (the R / I-sized intermediate of the first contraction stays on chip)
    int f2 = -1;
    if (N >= 4 && in.fuse && R <= 8 && f == N - 1 && f - 1 != n && f - 1 >= 1) {
      f2 = f - 1;
      for (int k = 0; k < N; ++k)
        if (k != n && k != f && k != f2 && dim_of(k) > dim_of(f2)) f2 = -1;
    }
    if (f2 < 0 || !emit_ttm2(f2, f)) {
      f2 = -1;
      emit_ttm(f);
    }
    for (int k = 0; k < N; ++k) if (k != n && k != f && k != f2) todo.push_back(k);
  } else {
    todo.push_back(1 - n);
  }
  std::sort(todo.begin(), todo.end(), [&](int a, int b) {
    if (dim_of(a) != dim_of(b)) return dim_of(a) > dim_of(b);
    return a > b;
  });
  p.zf = false;
  for (size_t q = 0; q < todo.size(); ++q) {
    if (q + 1 == todo.size() && in.zf_ok && src != in.X && !p.steps.empty()) {
      // Z fusion: skip this last TTM and let the apply kernel take its flops.  Opt-in (CPQR_ZFUSE=1;
      // =2: only where T has <= CPQR_ZFUSE_MAX elements, default 2M): measured C2 per mode +1 to
      // +4 % (2590-2640 -> 2670-2710 sweeps/s) but C2 tree -3.5 %, C3 -1.5 %, C4 -1 % -- the
      // latency-bound apply kernel over J_T = I_k R^{N-2} rows costs what the launch it saves does
      const char* ze = getenv("CPQR_ZFUSE");
      const int zmode = ze ? atoi(ze) : 0;
      static const int64_t zmax = getenv("CPQR_ZFUSE_MAX") ? atoll(getenv("CPQR_ZFUSE_MAX")) : (2ll << 20);
      const int64_t tel = prod(cur, 0, N);
      if (zmode == 1 || (zmode == 2 && tel <= zmax)) {
        p.zf = true;
        p.zk = todo[q];
        p.zT = src;
        for (int k = 0; k < N; ++k) p.zcur[k] = cur[k];
        p.zAa = prod(cur, 0, n);
        p.zBb = prod(cur, n + 1, N);
      }
    }
    emit_ttm(todo[q]);
  }
  if (in.ybuf && p.steps.size() >= 2) {  // overlap schedule: Y goes to its own buffer
    size_t last = p.steps.size() - 1;
    p.steps[last].out = in.ybuf;
    if ((p.steps[last].kind == 7 || p.steps[last].kind == 3) && last > 0) {
      if (p.steps[last].kind == 7) p.steps[last - 1].out = in.ybuf;  // whole slices of the TMA slice pass
    }
    src = in.ybuf;
  }
  p.Y = src;
  p.nd = N;
  for (int k = 0; k < N; ++k) p.ydims[k] = cur[k];
  p.Aa = prod(cur, 0, n);
  p.In = cur[n];
  p.Bb = prod(cur, n + 1, N);
}

template <typename K>
void set_smem(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Launch with the optional programmatic-dependent-launch attribute (the kernel may begin while its
// stream predecessor drains; it calls pdl_wait() before touching global memory, common.cuh) and an
// optional cluster shape.  Captured into the sweep's CUDA graph as programmatic edges.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                      int cluster, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

int launch_tma(const TtmStep& s, int R, cudaStream_t st, int sms, bool pdl) {  // returns #launches
  const int NT = (R + 7) / 8, NQB = (NT + 1) / 2;
  if (s.kind == 4) {
    // CW consumer warps per CTA over 32 CW-row units.  CW = 4 runs two CTAs per SM, each with its
    // own ring, so one computes while the other waits for data: measured C2 +1..5 %, C4 tree +3 %,
    // but C3 -0.8 % and C5 -1.1 % (interleaved A/B), hence only for R <= 12.  Env CPQR_STR_CW=4/8.
    static const int cw_env = getenv("CPQR_STR_CW") ? atoi(getenv("CPQR_STR_CW")) : 0;
    const int cw = s.cw1 ? 8 : cw_env == 4 ? 4 : cw_env == 8 ? 8 : (R <= 12 ? 4 : 8);
    const size_t stage = (size_t)(2 * cw + NQB) * kBoxBytes;
    const int S = cw == 4 ? std::min<int>(s.S, (int)((110 * 1024 - 3072) / stage)) : s.S;
    const size_t smem = 3072 + (size_t)S * stage;
    // rows of a slice per unit: 32 wa, with wb = cw / wa consecutive slices per unit (k_strided_tma).
    // wa = cw unless a shorter unit fills its M-tiles at least 10 % better (short slices: A = R or a
    // small I_1 after the leading modes are contracted; 75^5 R = 32: A = 32 ran at 1/8 of the tiles)
    static const int wa_env = getenv("CPQR_STR_WA") ? atoi(getenv("CPQR_STR_WA")) : 0;
    auto fill = [&](int wa) {
      const int wb = cw / wa;
      const double fa = (double)s.A / (32.0 * wa * (double)((s.A + 32 * wa - 1) / (32 * wa)));
      const double fb = (double)s.B / ((double)wb * (double)((s.B + wb - 1) / wb));
      return fa * fb;
    };
    int wa = cw;
    for (int w = cw / 2; w >= 1; w /= 2)
      if (fill(w) > 1.10 * fill(wa)) wa = w;
    if (wa_env >= 1 && wa_env <= cw && (cw % wa_env) == 0) wa = wa_env;
    const int wbs = cw / wa;
    const int64_t units = ((s.A + 32 * wa - 1) / (32 * wa)) * ((s.B + wbs - 1) / wbs);
    const int grid = (int)std::min<int64_t>(units, (int64_t)sms * (cw == 4 ? 2 : 1));
    // stream-K split (k_strided_tma) when the round-robin waves are ragged by > 2 %: e.g. C5 at 8
    // slabs, 500 units on 147 CTAs.  CPQR_STREAMK=0/1 forces it off / on.
    const double waves = (double)units / grid;
    const bool sk = wa == cw && s.P && grid > 1 && units > grid &&
                    (s.skm == 1 || (s.skm != 0 && std::ceil(waves) / waves > 1.02));
    double* P = sk ? s.P : nullptr;
    // the fix-up is fused into the kernel (last-arriving CTA per cut unit); CPQR_SK_FIXUP=1 keeps the
    // separate k_strided_fixup launch (same sums, same order)
    static const bool sep_fixup = getenv("CPQR_SK_FIXUP") && atoi(getenv("CPQR_SK_FIXUP")) == 1;
    unsigned* skc = (sk && !sep_fixup) ? s.cnt : nullptr;
#define STR(NTV, NPV)                                                                                  \
  {                                                                                                     \
    if (cw == 4) {                                                                                      \
      set_smem(k_strided_tma<NTV, NPV, 4>, smem);                                                       \
      launch_ex(k_strided_tma<NTV, NPV, 4>, grid, (4 + NPV) * 32, smem, st, pdl, 1, s.mx, s.mq, s.A, s.I, s.B, R, s.out, S, P, skc, wa); \
    } else {                                                                                            \
      set_smem(k_strided_tma<NTV, NPV>, smem);                                                          \
      launch_ex(k_strided_tma<NTV, NPV>, grid, (kCW + NPV) * 32, smem, st, pdl, 1, s.mx, s.mq, s.A, s.I, s.B, R, s.out, S, P, skc, wa); \
    }                                                                                                   \
  }
    // producer warps issuing the 16 X boxes of a stage in parallel: a single issuing thread bounds
    // the HBM-bound passes (C2 +16 %); 4 for the FP64-bound R >= 24 passes (+1.5 % on C5, -1.5 % C4)
    static const int np_env = getenv("CPQR_NPROD") ? atoi(getenv("CPQR_NPROD")) : 0;
    const int np = np_env ? np_env : (R >= 24 ? 4 : 2);
    if (np == 4) {
      switch (NT) { case 1: STR(1, 4) break; case 2: STR(2, 4) break; case 3: STR(3, 4) break; default: STR(4, 4) break; }
    } else if (np == 2) {
      switch (NT) { case 1: STR(1, 2) break; case 2: STR(2, 2) break; case 3: STR(3, 2) break; default: STR(4, 2) break; }
    } else {
      switch (NT) { case 1: STR(1, 1) break; case 2: STR(2, 1) break; case 3: STR(3, 1) break; default: STR(4, 1) break; }
    }
#undef STR
    if (sk && !skc) {
      launch_ex(k_strided_fixup, grid - 1, 1024, 0, st, pdl, 1, (const double*)P, s.A, R, s.B, (s.I + kBK - 1) / kBK,
                32 * cw, grid, s.out);
      return 2;
    }
    return 1;
  } else if (s.kind == 5) {
    // 8 warps of 2 fibre tiles; CPQR_FIB_CW=4 runs 4 warps of 4 tiles, two CTAs per SM (parity-
    // tested, but measured slower: C2 NE 2698 -> 2660 sweeps/s, neutral on C2 / C5 intermediates)
    static const int fcw_env = getenv("CPQR_FIB_CW") ? atoi(getenv("CPQR_FIB_CW")) : 0;
    const int cw = fcw_env == 4 ? 4 : 8;
    const size_t stage = 128 * 128 + NQB * kBoxBytes;
    const int S = cw == 4 ? std::min<int>(s.S, (int)((110 * 1024 - 3072) / stage)) : s.S;
    const size_t smem = 3072 + (size_t)S * stage;
    const int64_t units = (s.F + 127) / 128;
    const int grid = (int)std::min<int64_t>(units, (int64_t)sms * (cw == 4 ? 2 : 1));
#define FIB(MTV)                                                                                   \
  {                                                                                                \
    if (cw == 4) {                                                                                 \
      set_smem(k_fiber_tma<MTV, 4>, smem);                                                         \
      launch_ex(k_fiber_tma<MTV, 4>, grid, 5 * 32, smem, st, pdl, 1, s.mx, s.mq, s.I, s.F, R, s.out, S); \
    } else {                                                                                       \
      set_smem(k_fiber_tma<MTV>, smem);                                                            \
      launch_ex(k_fiber_tma<MTV>, grid, kTmaThreads, smem, st, pdl, 1, s.mx, s.mq, s.I, s.F, R, s.out, S); \
    }                                                                                              \
  }
    switch (NT) { case 1: FIB(1) break; case 2: FIB(2) break; case 3: FIB(3) break; default: FIB(4) break; }
#undef FIB
  } else if (s.kind == 6) {
    const int BN = s.cw * 8 * s.gps;
    const size_t smem = 3072 + (size_t)s.S * ((size_t)BN * 128 + NQB * kBoxBytes) + (size_t)s.cw * slice_ldy(R) * R * 8;
#define SLC(MTV, NFV)                                                                                      \
  {                                                                                                        \
    set_smem(k_slice_tma<MTV, NFV>, smem);                                                                 \
    launch_ex(k_slice_tma<MTV, NFV>, (int)s.G, kTmaThreads, smem, st, pdl, 1, s.mx, s.mq, s.I1, s.I2, s.L, s.Q2, \
              s.ldq2, R, s.out, s.P, s.nslots, s.S);                                                       \
  }
#define SLC4(MTV)                                                                                          \
  {                                                                                                        \
    set_smem(k_slice_tma<MTV, 4, 4>, smem);                                                                \
    launch_ex(k_slice_tma<MTV, 4, 4>, (int)s.G, 5 * 32, smem, st, pdl, 1, s.mx, s.mq, s.I1, s.I2, s.L, s.Q2, \
              s.ldq2, R, s.out, s.P, s.nslots, s.S);                                                       \
  }
    if (s.cw == 4) {
      switch (NT) { case 1: SLC4(1) break; case 2: SLC4(2) break; case 3: SLC4(3) break; default: SLC4(4) break; }
    } else if (s.gps == 4) {
      switch (NT) { case 1: SLC(1, 4) break; case 2: SLC(2, 4) break; case 3: SLC(3, 4) break; default: SLC(4, 4) break; }
    } else {
      switch (NT) { case 1: SLC(1, 2) break; case 2: SLC(2, 2) break; case 3: SLC(3, 2) break; default: SLC(4, 2) break; }
    }
#undef SLC
#undef SLC4
  } else if (s.kind == 8) {
    const size_t smem = 3072 + (size_t)s.S * ((size_t)s.I2 * 8 * 128 + NQB * kBoxBytes);
    const int64_t units = (s.L + 7) / 8;
    const int grid = (int)std::min<int64_t>(units, sms);
#define SSM(MTV)                                                                                             \
  {                                                                                                          \
    set_smem(k_slice_small_tma<MTV>, smem);                                                                  \
    launch_ex(k_slice_small_tma<MTV>, grid, kTmaThreads, smem, st, pdl, 1, s.mx, s.mq, s.I1, s.I2, s.L, s.Q2, s.ldq2, \
              R, s.out, s.S);                                                                                  \
  }
    switch (NT) { case 1: SSM(1) break; case 2: SSM(2) break; case 3: SSM(3) break; default: SSM(4) break; }
#undef SSM
  } else if (s.kind == 10) {
    const size_t smem = 3072 + (size_t)s.S * 9 * kBoxBytes;
    const int64_t units = (s.A + 127) / 128;
    const int grid = (int)std::min<int64_t>(units, sms);
    set_smem(k_strided2_tma<2>, smem);
    launch_ex(k_strided2_tma<2>, grid, 10 * 32, smem, st, pdl, 1, s.mx, s.mq, s.A, s.I, (int)s.B, R, s.Qt, s.rq, s.out, s.S);
  } else if (s.kind == 7) {
    const int grid = (int)std::min<int64_t>(s.L, (int64_t)sms * 4);
    launch_ex(k_slice_fixup, grid, 256, 0, st, pdl, 1, (const double*)s.P, s.nslots, s.L, s.nfb, s.G, R * R, s.out);
  }
  return 1;
}

cpqr_status run_plan(cpqr_ctx* c, const Plan& p) {
  for (const TtmStep& s : p.steps) {
    switch (s.kind) {
      case 0: launch_strided(s, c->R, c->st, c->stream_sms); break;
      case 1: launch_fiber(s, c->R, c->st, c->stream_sms); break;
      case 2: launch_slice(s, c->R, c->st, c->stream_sms); break;
      case 3: {
        const int64_t n = s.L * c->R * c->R;
        const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sms * 8);
        k_reduce_slices<<<grid, 256, 0, c->st>>>(s.in, s.nseg, s.L, c->R * c->R, s.out);
        break;
      }
      case 9: {
        const int64_t rcs = (s.A * s.B + 16 * (8 / s.wk) - 1) / (16 * (8 / s.wk));
        const dim3 grid((unsigned)(rcs * s.kc));
        switch ((c->R + 7) / 8) {
#define SML(NTV)                                                                                              \
  case NTV:                                                                                                   \
    set_smem(k_ttm_small<NTV>, s.S);                                                                          \
    launch_ex(k_ttm_small<NTV>, grid, 256, s.S, c->st, c->pdl, 1, s.in, s.A, s.I, s.B, s.Qt, s.rq, c->R, s.out, \
              s.wk, s.kc, s.P, s.cnt);                                                                        \
    break;
          SML(1) SML(2) SML(3) SML(4)
#undef SML
        }
        break;
      }
      default: c->launch_count += launch_tma(s, c->R, c->st, c->stream_sms, c->pdl) - 1; break;
    }
    CKL();
  }
  for (const DiagStep& d : p.diags) {
    DiagArgs a{};
    a.T = d.in;
    a.nd = d.nd;
    for (int i = 0; i < d.nd; ++i) a.dims[i] = d.dims[i];
    a.k = d.k;
    a.rm = d.rm;
    a.Ak = d.Ak;
    a.lda = d.lda;
    a.out = d.out;
    int64_t tot = 1;
    for (int i = 0; i < d.nd; ++i) if (i != d.k) tot *= d.dims[i];
    const int grid = (int)std::max<int64_t>(1, (tot + 31) / 32);
    k_diag_contract<<<grid, 256, 0, c->st>>>(a);
    CKL();
  }
  return CPQR_OK;
}

void fill_plan_in(cpqr_ctx* c, const Slab& sl, PlanIn& in, int n, const double* const* Qover = nullptr,
                  const double* const* Qtover = nullptr) {
  const bool ne = ne_family(c->variant);
  in.X = sl.X;
  in.ld = sl.ldims;
  in.N = c->N;
  in.R = c->R;
  in.n = n;
  in.ne = ne;
  in.tma = c->use_tma;
  in.fuse = c->fuse_slice;
  in.pad0 = c->pad1 ? 1 : 0;
  in.ne_ov = c->overlap_ne;
  in.zf_ok = c->nslab == 1 && !c->exchange && !ne && !c->q0_stair;
  in.sms = c->stream_sms;
  in.tree = c->tree && !ne;
  in.h = c->tree_h;
  in.tree_fresh = (n == 0 || n == c->tree_h);
  in.tbuf = sl.dTree;
  in.sk = c->dSk;
  in.skcnt = c->dSkCnt;
  in.skm = c->streamk;
  in.overlap = c->overlap;
  in.ov_cw1 = c->ov_cw1;
  in.ybuf = c->overlap ? c->dY : nullptr;
  in.RQ = c->RQ;
  for (int k = 0; k < c->N; ++k) {
    const double* base = ne ? c->dA[k] : c->dQ[k];
    const double* bt = ne ? c->dAt[k] : c->dQt[k];
    if (Qover && Qover[k]) base = Qover[k];
    if (Qtover && Qtover[k]) bt = Qtover[k];
    const bool last = (k == c->N - 1);
    in.Q[k] = last ? base + sl.b : base;
    in.Qt[k] = last ? bt + sl.b * c->RQ : bt;
    in.ldq[k] = c->dims[k];
  }
}

cpqr_status build_plans(cpqr_ctx* c) {
  size_t mb = 0, mp = 0, mt = 0;
  for (int q = 0; q < c->nslab; ++q) {
    const Slab& sl = c->slabs[q];
    for (int n = 0; n < c->N; ++n) {
      PlanIn in{};
      fill_plan_in(c, sl, in, n);
      in.tma = false;  // sizing pass (no maps)
      Plan tmp;
      double* nob[2] = {nullptr, nullptr};
      plan_mode(in, tmp, nob, nullptr);
      mb = std::max(mb, tmp.max_buf);
      mp = std::max(mp, tmp.part);
      mt = std::max(mt, tmp.tree_elems);
      // TMA slice partials: L * nslots * R^2 with nslots <= ceil(nfb*G/U)+1 <= 2 + nfb
      if (c->N >= 3 && n >= 2) {
        const int64_t L = prod(sl.ldims, 2, c->N);
        const int nfb = (int)((sl.ldims[1] + 127) / 128);
        mp = std::max(mp, (size_t)L * (size_t)(nfb + 2) * c->R * c->R);
      }
    }
  }
  if (c->overlap) {  // Y_(n) of every mode: I_n R^{N-1} (local) elements
    size_t ye = 0;
    for (int n = 0; n < c->N; ++n) {
      size_t e = (size_t)c->slabs[0].ldims[n];
      for (int k = 0; k < c->N - 1; ++k) e *= (size_t)c->R;
      ye = std::max(ye, e);
    }
    if (ye > c->dY_elems) {
      if (c->dY) dfree(c->dY);
      c->dY = nullptr;
      if (dmalloc(&c->dY, ye * sizeof(double)) != cudaSuccess) return fail(c, CPQR_ENOMEM, "Y buffer");
      c->dY_elems = ye;
    }
  }
  // the ping-pong intermediates and slice partials are shared by the slabs (run in turn on one
  // stream); each slab keeps its own dimension-tree buffer (it lives across modes)
  if (mb > c->buf_elems) {
    for (int i = 0; i < 2; ++i) { if (c->buf[i]) dfree(c->buf[i]); c->buf[i] = nullptr; }
    for (int i = 0; i < 2; ++i)
      if (dmalloc(&c->buf[i], mb * sizeof(double)) != cudaSuccess)
        return fail(c, CPQR_ENOMEM, "intermediate buffers (%zu doubles)", mb);
    c->buf_elems = mb;
  }
  for (int q = 0; q < c->nslab; ++q) {
    Slab& sl = c->slabs[q];
    if (mt > sl.tree_alloc) {
      if (sl.dTree) dfree(sl.dTree);
      sl.dTree = nullptr;
      if (dmalloc(&sl.dTree, mt * sizeof(double)) != cudaSuccess)
        return fail(c, CPQR_ENOMEM, "dimension-tree buffer (%zu doubles)", mt);
      sl.tree_alloc = mt;
    }
  }
  if (mp > c->part_elems) {
    if (c->dPart) dfree(c->dPart);
    c->dPart = nullptr;
    if (dmalloc(&c->dPart, mp * sizeof(double)) != cudaSuccess)
      return fail(c, CPQR_ENOMEM, "slice partials (%zu doubles)", mp);
    c->part_elems = mp;
  }
  for (int q = 0; q < c->nslab; ++q) {
    Slab& sl = c->slabs[q];
    for (int n = 0; n < c->N; ++n) {
      PlanIn in{};
      fill_plan_in(c, sl, in, n);
      plan_mode(in, sl.plans[n], c->buf, c->dPart);
    }
  }
  {  // Z fusion buffer: the largest J_T x R over the modes that use it
    size_t ze = 0;
    for (int q = 0; q < c->nslab; ++q)
      for (int n = 0; n < c->N; ++n) {
        const Plan& p = c->slabs[q].plans[n];
        if (p.zf) ze = std::max(ze, (size_t)(p.zAa * p.zBb) * (size_t)c->R);
      }
    if (ze > c->dZ_elems) {
      if (c->dZ) dfree(c->dZ);
      c->dZ = nullptr;
      if (dmalloc(&c->dZ, ze * sizeof(double)) != cudaSuccess) return fail(c, CPQR_ENOMEM, "Z buffer");
      c->dZ_elems = ze;
    }
  }
  c->plans_valid = true;
  return CPQR_OK;
}

// ----------------------------------------------------------------------------- helpers
// phase marks (opt.profile only; never inside graph capture): the device time since the previous
// mark is attributed to `phase` (cpqr_profile.ms index); phase -1 starts a new interval
void prof_mark(cpqr_ctx* c, int phase) {
  if (!c->opt.profile) return;
  if (c->nmarks == (int)c->evp.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    c->evp.push_back(e);
    c->evphase.push_back(-1);
    c->evlaunch.push_back(0);
  }
  cudaEventRecord(c->evp[c->nmarks], c->st);
  c->evphase[c->nmarks] = phase;
  c->evlaunch[c->nmarks] = c->launch_count;
  ++c->nmarks;
}

int rb_for(int R) { return R <= 8 ? 8 : (R <= 16 ? 16 : 32); }

// Ahat = W R0^{-T} (substitution) or W (R0^T)^+ (SVD) into c->dAhat, per-CTA partials in c->dred.
// M = U S^+ V^T of R0 (QR-SVD): one-sided Jacobi, depends on R0 only
cpqr_status launch_pinv(cpqr_ctx* c, cudaStream_t st, int* ntrunc) {
  const int R = c->R;
  const double tau = (c->opt.svd_tau < 0) ? R * 2.220446049250313e-16 : c->opt.svd_tau;
  const size_t smem = (size_t)(2 * R * R + 2 * R * (R + 1)) * sizeof(double);
  k_svd_pinv<<<1, 512, smem, st>>>(c->dR0, R, tau, c->dMpinv, c->dflags, ntrunc);
  CKL();
  return CPQR_OK;
}

cpqr_status launch_solve(cpqr_ctx* c, const double* W, int In, bool fit, int* ntrunc) {
  const int R = c->R, RB = rb_for(R);
  const double* Rm = c->dR0;
  if (c->variant == CPQR_SVD) {
    if (!c->pinv_ready || ntrunc) TRY(launch_pinv(c, c->st, ntrunc));
    Rm = c->dMpinv;
  }
  const int BT = (RB > 16) ? 64 : 128;
  const int grid = (In + BT - 1) / BT;
  c->nparts = grid;
  switch (RB) {
    case 8: k_solve_rows<8><<<grid, 128, 0, c->st>>>(W, Rm, c->dR0, In, R, c->variant, c->dAhat, c->dred, fit); break;
    case 16: k_solve_rows<16><<<grid, 128, 0, c->st>>>(W, Rm, c->dR0, In, R, c->variant, c->dAhat, c->dred, fit); break;
    default: k_solve_rows<32><<<grid, 64, 0, c->st>>>(W, Rm, c->dR0, In, R, c->variant, c->dAhat, c->dred, fit); break;
  }
  CKL();
  return CPQR_OK;
}


// TSQR launcher.  solve = false: thin QR of the m x R column-major A -> Q, Qt, Rn.
// solve = true: the fused per-mode tail -- Ahat from W (and R0 / M), lambda, A_n = Ahat/lambda into
// Aout, and the QR of A_n (Q, Qt, Rn), plus the fast fit when do_fit.
void cq_multi_attrs() {  // dynamic shared memory of the multi-kernel CholeskyQR2 (once)
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_cq_gram1<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_cq_gram1<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_cq_gram1<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_cq_apply<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_cq_apply<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_cq_apply<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  done = true;
}

// one cluster launch of k_cq_compact: nb CTAs (<= 8) of tb threads, one panel row per thread
cpqr_status launch_cq_compact(cpqr_ctx* c, const CqArgs& q, int RB, int tb, cudaStream_t st) {
  const int ld = ((tb + 15) & ~15) + 4;
  const size_t smem = (size_t)(8 * RB * RB + 2 * ld * RB) * sizeof(double);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(q.nb);
  cfg.blockDim = dim3(tb);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = q.nb;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (c->pdl && st == c->st) ? 2 : 1;
  cudaError_t e = cudaSuccess;
#ifdef CPQR_DEBUG_TIMING
  const int reps = getenv("CPQR_CQ_TWICE") ? 2 : 1;  // warm-vs-cold instruction-fetch experiment
#else
  const int reps = 1;
#endif
#define CQL(RBV)                                                                                    \
  {                                                                                                 \
    cudaFuncSetAttribute(k_cq_compact<RBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    e = cudaLaunchKernelEx(&cfg, k_cq_compact<RBV>, q);                                             \
  }
  for (int rep = 0; rep < reps && e == cudaSuccess; ++rep) {
    switch (RB) { case 8: CQL(8) break; case 16: CQL(16) break; default: CQL(32) break; }
  }
#undef CQL
  if (e != cudaSuccess) return fail(c, CPQR_ECUDA, "k_cq_compact launch: %s", cudaGetErrorString(e));
  CKL();
  return CPQR_OK;
}

// Multi-kernel CholeskyQR2 of the m x R column-major q.A (row blocks of 256 rows) on stream st.
// The Cholesky kernels' view of the nb Gram partials: beyond 1024 row blocks a first level sums
// groups of 512 blocks (k_reduce_gp) into c->dGp2, so the one-CTA Cholesky adds <= 1024 partials
CqArgs cq_reduced(cpqr_ctx* c, const CqArgs& q, cudaStream_t st) {
  if (q.nb <= 1024) return q;
  CqArgs r = q;
  // groups of >= 32 blocks, at most 1024 of them (c->dGp2): 4096 blocks -> 128 CTAs (8 CTAs of 512
  // blocks each took 0.65 ms of the 1M-row V_n QR, twice per mode)
  const int per = std::max(32, (q.nb + 1023) / 1024), ng = (q.nb + per - 1) / per;
  k_reduce_gp<<<ng, 128, 0, st>>>(q.Gp, q.nb, q.R * q.R, per, c->dGp2);
  r.Gp = c->dGp2;
  r.nb = ng;
  return r;
}

cpqr_status launch_cq_multi(cpqr_ctx* c, const CqArgs& q, cudaStream_t st) {
  const int RB = rb_for(c->R);
  const int tb = 32 * ((q.mb + 31) / 32);
  const size_t psm = (size_t)(q.mb | 1) * c->R * 8;
  cq_multi_attrs();
#define CQM(RBV)                                                   \
  {                                                                \
    k_cq_gram1<RBV><<<q.nb, tb, psm, st>>>(q); CKL();              \
    k_cq_chol1<<<1, 256, 0, st>>>(cq_reduced(c, q, st)); CKL();    \
    k_cq_apply<RBV><<<q.nb, tb, psm, st>>>(q, 1); CKL();           \
    k_cq_chol2<<<1, 256, 0, st>>>(cq_reduced(c, q, st), nullptr); CKL(); \
    k_cq_apply<RBV><<<q.nb, tb, psm, st>>>(q, 2); CKL();           \
  }
  switch (RB) { case 8: CQM(8) break; case 16: CQM(16) break; default: CQM(32) break; }
#undef CQM
  return CPQR_OK;
}

cpqr_status launch_tsqr(cpqr_ctx* c, int m, const double* A, bool solve, const double* W, double* Q,
                        double* Qt, double* Rn, double* Aout, bool do_fit) {
  const int R = c->R, RB = rb_for(R);
  if (solve && c->variant == CPQR_SVD && !c->pinv_ready) TRY(launch_pinv(c, c->st, nullptr));
  auto cq_args = [&](int nb) {
    CqArgs q{};
    q.A = A; q.m = m; q.R = R; q.nb = nb; q.mb = (m + nb - 1) / nb; q.solve = solve ? 1 : 0; q.W = W;
    q.Rm = (c->variant == CPQR_SVD) ? c->dMpinv : c->dR0; q.R0 = c->dR0; q.variant = c->variant;
    q.Ahat = c->dAhat; q.Q1 = c->dQ1; q.Gp = c->dGp; q.innerp = c->dinnerp; q.R1 = c->dR1; q.R2 = c->dR2;
    q.Q = Q; q.Qt = Qt; q.RQ = c->RQ; q.Rn = Rn; q.Aout = Aout; q.lam = c->dlam; q.flags = c->dflags;
    q.do_fit = do_fit ? 1 : 0; q.nX2 = c->dnX2; q.fit = c->dfit;
    return q;
  };
  // fast path: CholeskyQR2 (cholqr.cuh), any m; the Householder fallback below then runs gated
  // (only when the device-side kappa / orthogonality guard rejected the CholeskyQR2 result)
  bool gated = false;
  int cq_nb = 0;
  int nbq = (m + 255) / 256;
  // overlap schedule: the tail runs beside the next stream pass on the few SMs it leaves free, so
  // it must not need a co-scheduled cluster: one CTA of up to 512 rows when its panels fit
  if (c->tail_single && m <= 512 && (8 * RB * RB + 2 * (((32 * ((m + 31) / 32) + 15) & ~15) + 4) * RB) * 8 <= 220 * 1024)
    nbq = 1;
  if (c->factor_qr_mode == 0 && nbq <= 8 && !getenv("CPQR_CQ_MULTI")) {  // single cluster launch
    const CqArgs q = cq_args(nbq);
    // >= 8 warps even for short factors: the 2-D Cholesky maps its columns to 8 warps (the rolled
    // fallback for fewer warps cost ~680 vs ~440 cycles per column); spare threads own no row
    TRY(launch_cq_compact(c, q, RB, std::max(256, 32 * ((q.mb + 31) / 32)), c->st));
    gated = true;
    cq_nb = nbq;
  } else if (c->factor_qr_mode == 0) {  // multi-kernel CholeskyQR2, row blocks of <= 256 rows
    TRY(launch_cq_multi(c, cq_args(nbq), c->st));
    gated = true;
    cq_nb = nbq;
  }
  // Householder fallback 1: register-resident TSQR (one thread per row), leaves and root <= 256 rows
  {
    int nl = std::max(1, (m + 255) / 256);
    int mbr = (m + nl - 1) / nl;
    while (nl > 1 && m - (nl - 1) * mbr < R) { --nl; mbr = (m + nl - 1) / nl; }
    if (nl <= 8 && mbr <= 256 && nl * R <= 256 && !getenv("CPQR_SMEM_QR")) {
      RqArgs q{};
      q.A = A; q.m = m; q.R = R; q.nleaf = nl; q.mb = mbr;
      q.Rstack = c->dRstack; q.V = c->dV; q.tauv = c->dtauv; q.Qtop = c->dQtop;
      q.Q = Q; q.Qt = Qt; q.RQ = c->RQ; q.Rn = Rn;
      q.solve = solve ? 1 : 0; q.W = W; q.R0 = c->dR0;
      q.Rm = (c->variant == CPQR_SVD) ? c->dMpinv : c->dR0;
      q.variant = c->variant;
      q.Ahat = c->dAhat; q.part = c->dred; q.Aout = Aout; q.lam = c->dlam; q.flags = c->dflags;
      q.do_fit = do_fit ? 1 : 0; q.nX2 = c->dnX2; q.fit = c->dfit;
      q.gated = gated ? 1 : 0;
      const int tl = 32 * ((mbr + 31) / 32), tr = 32 * ((nl * R + 31) / 32);
      static const bool rq_split_env = getenv("CPQR_RQ_SPLIT") && atoi(getenv("CPQR_RQ_SPLIT")) == 1;
      const bool rq_split = rq_split_env || c->tail_single;  // overlap: no cluster co-scheduling
      static const bool rq_serial_off = getenv("CPQR_RQ_SERIAL") && atoi(getenv("CPQR_RQ_SERIAL")) == 0;
      if (c->tail_single && !rq_split_env && !rq_serial_off) {  // one CTA, the phases in turn (k_rq_serial)
        const int tb = std::max(tl, tr);
        switch (RB) {
          case 8: k_rq_serial<8><<<1, tb, 0, c->st>>>(q); break;
          case 16: k_rq_serial<16><<<1, tb, 0, c->st>>>(q); break;
          default: k_rq_serial<32><<<1, tb, 0, c->st>>>(q); break;
        }
        CKL();
      } else if (!rq_split) {  // one cluster launch of the three phases (k_rq_fused)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nl);
        cfg.blockDim = dim3(std::max(tl, tr));
        cfg.dynamicSmemBytes = 0;
        cfg.stream = c->st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = nl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = c->pdl ? 2 : 1;
        cudaError_t e;
        switch (RB) {
          case 8: e = cudaLaunchKernelEx(&cfg, k_rq_fused<8>, q); break;
          case 16: e = cudaLaunchKernelEx(&cfg, k_rq_fused<16>, q); break;
          default: e = cudaLaunchKernelEx(&cfg, k_rq_fused<32>, q); break;
        }
        if (e != cudaSuccess) return fail(c, CPQR_ECUDA, "k_rq_fused launch: %s", cudaGetErrorString(e));
        CKL();
      } else {
        switch (RB) {
          case 8:
            k_rq_leaf<8><<<nl, tl, 0, c->st>>>(q); CKL();
            k_rq_root<8><<<1, tr, 0, c->st>>>(q); CKL();
            k_rq_qform<8><<<nl, tl, 0, c->st>>>(q); CKL();
            break;
          case 16:
            k_rq_leaf<16><<<nl, tl, 0, c->st>>>(q); CKL();
            k_rq_root<16><<<1, tr, 0, c->st>>>(q); CKL();
            k_rq_qform<16><<<nl, tl, 0, c->st>>>(q); CKL();
            break;
          default:
            k_rq_leaf<32><<<nl, tl, 0, c->st>>>(q); CKL();
            k_rq_root<32><<<1, tr, 0, c->st>>>(q); CKL();
            k_rq_qform<32><<<nl, tl, 0, c->st>>>(q); CKL();
            break;
        }
      }
      return CPQR_OK;
    }
  }
  // Householder fallback 2: shared-memory TSQR, <= 8 leaves of mb rows (2 mb R doubles per leaf)
  int nleaf = std::max(1, std::min(8, (m + 127) / 128));
  int mb = (m + nleaf - 1) / nleaf;
  while (nleaf > 1 && m - (nleaf - 1) * mb < R) { --nleaf; mb = (m + nleaf - 1) / nleaf; }
  const size_t leaf_smem = (size_t)mb * R * 8, qf_smem = 2 * leaf_smem,
               root_smem = (size_t)std::max(nleaf, 2) * R * R * 8;
  if (qf_smem <= 200 * 1024) {
    TsqrArgs a{};
    a.A = A; a.m = m; a.R = R; a.nleaf = nleaf; a.mb = mb;
    a.Rstack = c->dRstack; a.V = c->dV; a.tauv = c->dtauv; a.Qtop = c->dQtop;
    a.Q = Q; a.Qt = Qt; a.RQ = c->RQ; a.Rn = Rn;
    a.solve = solve ? 1 : 0;
    a.W = W;
    a.R0 = c->dR0;
    a.Rm = (c->variant == CPQR_SVD) ? c->dMpinv : c->dR0;
    a.variant = c->variant;
    a.Ahat = c->dAhat; a.part = c->dred; a.Aout = Aout; a.lam = c->dlam; a.flags = c->dflags;
    a.do_fit = do_fit ? 1 : 0; a.nX2 = c->dnX2; a.fit = c->dfit;
    a.gated = gated ? 1 : 0;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_tsqr_leaf<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_tsqr_leaf<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_tsqr_leaf<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_tsqr_root, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_tsqr_qform, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
      attr = true;
    }
    switch (RB) {
      case 8: k_tsqr_leaf<8><<<nleaf, 256, leaf_smem, c->st>>>(a); break;
      case 16: k_tsqr_leaf<16><<<nleaf, 256, leaf_smem, c->st>>>(a); break;
      default: k_tsqr_leaf<32><<<nleaf, 256, leaf_smem, c->st>>>(a); break;
    }
    CKL();
    k_tsqr_root<<<1, 512, root_smem, c->st>>>(a);
    CKL();
    k_tsqr_qform<<<nleaf, 512, qf_smem, c->st>>>(a);
    CKL();
    return CPQR_OK;
  }
  // Householder fallback 3 (very tall factors, e.g. I_n > 3200 at R = 32): one CTA over global
  // memory.  Behind CholeskyQR2 it starts from the Ahat and <W, Ahat R0^T> partials k_cq_gram1
  // already wrote; with Householder forced, k_solve_rows forms them first.
  TallArgs t{};
  t.A = A; t.Ahat = c->dAhat; t.m = m; t.R = R; t.RQ = c->RQ; t.solve = solve ? 1 : 0;
  t.Q = Q; t.Qt = Qt; t.Rn = Rn; t.Aout = Aout; t.lam = c->dlam; t.flags = c->dflags;
  t.gate_bit = gated ? FLAG_USE_HOUSEHOLDER : 0u;
  t.do_fit = do_fit ? 1 : 0;
  t.R0 = c->dR0; t.nX2 = c->dnX2; t.fit = c->dfit;
  if (gated) {
    t.innerp = c->dinnerp; t.ninner = cq_nb; t.istride = 1;
  } else {
    if (solve) TRY(launch_solve(c, W, m, do_fit, nullptr));
    t.innerp = c->dred + RB; t.ninner = solve ? c->nparts : 0; t.istride = RB + 1;
  }
  k_tall_fallback<<<1, 1024, 0, c->st>>>(t);
  CKL();
  return CPQR_OK;
}

cpqr_status launch_factor_qr(cpqr_ctx* c, const double* A, int m, double* Q, double* Qt, double* Rn, bool do_fit) {
  return launch_tsqr(c, m, A, false, nullptr, Q, Qt, Rn, nullptr, do_fit);
}

// Alg. 2 lines 6-7: V_n and its QR -> Q0, R0.  Default: k_kr_qr2, one CTA, Householder on the
// packed staircase.  High rank (R^{N-1} R large): V_n is
// formed densely and factored by the multi-CTA CholeskyQR2 under the same kappa guard as the
// factor QR; k_kr_qr2 then runs only if the guard rejected V_n (device flag FLAG_VN_HOUSEHOLDER).
cpqr_status launch_kr_qr(cpqr_ctx* c, int n) {
  KrQrArgs a{};
  int m = 0;
  for (int k = 0; k < c->N; ++k)
    if (k != n) a.Rk[m++] = c->dRk[k];
  a.N1 = c->N - 1;
  a.R = c->R;
  a.perm = c->dperm;
  a.Q0 = c->dQ0;
  a.R0 = c->dR0;
  a.work_global = c->dKrWork;
  a.use_smem = c->kr_smem > 0;
  a.flags = c->dflags;
  cudaStream_t st = c->side ? c->side : c->st;
  if (c->vn_krtree) {
    // tree QR across the Khatri-Rao factors (one CTA): the group of the other half is factored at
    // the first mode of each half (n == 0, n == h) and reused by the rest of that half
    VnTreeArgs t{};
    for (int k = 0; k < c->N; ++k) t.Rk[k] = c->dRk[k];
    t.N = c->N; t.n = n; t.R = c->R; t.h = c->tree_h;
    t.fresh = (c->kr_standalone || n == 0 || n == c->tree_h) ? 1 : 0;
    for (int i = 0; i < 2; ++i) { t.Psh[i] = c->dTrP[i]; t.Ssh[i] = c->dTrS[i]; }
    t.Pa = c->dTrPa; t.Pb = c->dTrPb; t.T = c->dTrT; t.Qg = c->dTrQ;
    t.Q0 = c->dQ0; t.R0 = c->dR0; t.flags = c->dflags;
    const size_t sm = vn_tree_smem(c->R);
    if (c->R <= 8) k_vn_tree<8><<<1, 256, sm, st>>>(t);
    else if (c->R <= 16) k_vn_tree<16><<<1, 512, sm, st>>>(t);
    else k_vn_tree<32><<<1, 256, sm, st>>>(t);
    CKL();
    return CPQR_OK;
  }
  if (c->short_modes) {
    // short modes (I_k < R): V_n keeps its prod_{k != n} min(I_k, R) nonzero rows (mixed radix); no
    // staircase K2 for them, so the QR is the shifted CholeskyQR3 (Fukaya et al.), stable up to
    // kappa(V_n) ~ 1/eps: a shifted pass G + s I (s = 11 (J R + R (R+1)) eps ||V||_F^2) gives
    // V = Q_s R_s with kappa(Q_s) ~ sqrt(kappa), then CholeskyQR2 of Q_s: Q0 and R0 = R' R_s.
    int64_t J = 1;
    for (int k = 0, m = 0; k < c->N; ++k)
      if (k != n) { a.rad[m++] = c->vq[k]; J *= c->vq[k]; }
    const int grid = (int)std::min<int64_t>((J * c->R + 255) / 256, (int64_t)c->sms * 8);
    k_form_v<<<grid, 256, 0, st>>>(a, J, c->dVn);
    CKL();
    CqArgs q{};
    q.A = c->dVn; q.m = (int)J; q.R = c->R; q.nb = (int)((J + 255) / 256); q.mb = (int)((J + q.nb - 1) / q.nb);
    q.solve = 0; q.Q1 = c->dVq1; q.Gp = c->dVgp; q.innerp = c->dinnerp; q.R1 = c->dVr1; q.R2 = c->dVr2;
    q.Q = c->dQ0; q.Qt = nullptr; q.RQ = c->RQ; q.Rn = c->dVrp; q.flags = c->dflags; q.do_fit = 0;
    q.nX2 = c->dnX2; q.fit = c->dfit; q.hh_bit = FLAG_VN_HOUSEHOLDER;
    q.shift_c = 11.0 * ((double)J * c->R + (double)c->R * (c->R + 1)) * 2.220446049250313e-16;
    const int RB = rb_for(c->R), tb = 32 * ((q.mb + 31) / 32);
    const size_t psm = (size_t)(q.mb | 1) * c->R * 8;
    cq_multi_attrs();
#define SHP(RBV)                                                        \
  {                                                                     \
    k_cq_gram1<RBV><<<q.nb, tb, psm, st>>>(q); CKL();                   \
    k_cq_chol1<<<1, 256, 0, st>>>(cq_reduced(c, q, st)); CKL();         \
    k_cq_apply<RBV><<<q.nb, tb, psm, st>>>(q, 1); CKL();                \
  }
    switch (RB) { case 8: SHP(8) break; case 16: SHP(16) break; default: SHP(32) break; }
#undef SHP
    CK(cudaMemcpyAsync(c->dVrs, c->dVr1, sizeof(double) * c->R * c->R, cudaMemcpyDeviceToDevice, st));
    CqArgs q2 = q;  // CholeskyQR2 of Q_s (in dVq1); V's buffer is free scratch now
    q2.A = c->dVq1; q2.Q1 = c->dVn; q2.shift_c = 0.0;
    TRY(launch_cq_multi(c, q2, st));
    k_tri_mul<<<1, 256, 0, st>>>(c->dVrp, c->dVrs, c->R, c->dR0);  // R0 = R' R_s
    CKL();
    return CPQR_OK;
  }
  if (c->vn_mode_cq) {
    const int64_t J = c->vnJ;
    const int grid = (int)std::min<int64_t>((J * c->R + 255) / 256, (int64_t)c->sms * 8);
    k_form_v<<<grid, 256, 0, st>>>(a, J, c->dVn);
    CKL();
    CqArgs q{};
    q.A = c->dVn; q.m = (int)J; q.R = c->R; q.nb = (int)((J + 255) / 256); q.mb = (int)((J + q.nb - 1) / q.nb);
    q.solve = 0; q.Q1 = c->dVq1; q.Gp = c->dVgp; q.innerp = c->dinnerp; q.R1 = c->dVr1; q.R2 = c->dVr2;
    q.Q = c->dQ0; q.Qt = nullptr; q.RQ = c->RQ; q.Rn = c->dR0; q.flags = c->dflags; q.do_fit = 0;
    q.nX2 = c->dnX2; q.fit = c->dfit; q.hh_bit = FLAG_VN_HOUSEHOLDER;
    // one cluster launch when the rows fit 8 CTAs of <= 512 (R <= 16) or 256 (R <= 32) threads
    const int rb = c->R <= 8 ? 8 : c->R <= 16 ? 16 : 32, tmax = rb <= 16 ? 512 : 256;  // (see create)
    const bool no_compact = getenv("CPQR_VN_COMPACT") && atoi(getenv("CPQR_VN_COMPACT")) == 0;
    if (J <= 8 * tmax && !no_compact) {
      q.nb = (int)std::min<int64_t>(8, (J + 255) / 256);
      q.mb = (int)((J + q.nb - 1) / q.nb);
      TRY(launch_cq_compact(c, q, rb, std::max(256, 32 * ((q.mb + 31) / 32)), st));
    } else {
      TRY(launch_cq_multi(c, q, st));
    }
    a.gate_bit = FLAG_VN_HOUSEHOLDER;
  }
  k_kr_qr2<<<1, 1024, c->kr_smem, st>>>(a);
  CKL();
  return CPQR_OK;
}

// pp: the peer push of this slab's W (np = 0: none), fused into the apply's final sum
// Qm: the J x R matrix applied (default Q0; Z of the Z fusion, with p describing T instead of Y)
cpqr_status launch_q0_apply(cpqr_ctx* c, const Plan& p, double* Wout, const PeerPush& pp = PeerPush{},
                            const double* Qm = nullptr) {
  if (!Qm) Qm = c->dQ0;
  const int64_t J = p.Aa * p.Bb, KT = (J + 3) / 4;
  const int In = (int)p.In;
  // a large V_n: 4 M-tiles per CTA so that Q0 is read once per 32 rows of Y_(n) (k_q0_apply_big)
  const char* big_s = getenv("CPQR_Q0_BIG");  // 0 / 1: never / always (tests); read per launch
  const int big_env = big_s ? atoi(big_s) : -1;
  if (!c->q0_stair && In > 8 && (big_env == 1 || (big_env != 0 && J >= 32768))) {
    constexpr int MTL = 4;
    const int groups = (In + 8 * MTL - 1) / (8 * MTL);
    int64_t KS = std::max<int64_t>(1, std::min<int64_t>((2 * c->sms + groups - 1) / groups, (KT + 7) / 8));
    KS = std::min<int64_t>(KS, kQ0MaxSlices);
    const int kpc = (int)((KT + KS - 1) / KS);
    KS = (KT + kpc - 1) / kpc;
    dim3 grid(groups, (unsigned)KS);
#define Q0B(NTV)                                                                                          \
  launch_ex(k_q0_apply_big<NTV, MTL>, grid, 256, 0, c->st, c->pdl, 1, p.Y, p.Aa, In, p.Bb, Qm, \
            c->R, kpc, (int)KS, c->dWp, c->dq0cnt, Wout, pp)
    switch ((c->R + 7) / 8) { case 1: Q0B(1); break; case 2: Q0B(2); break; case 3: Q0B(3); break; default: Q0B(4); break; }
#undef Q0B
    CKL();
    return CPQR_OK;
  }
  const int iblocks = (In + 7) / 8;
  // slices of Q0's k-steps so that ~2 CTAs per SM run, each with >= 1 k-step per warp
  int64_t KS = std::max<int64_t>(1, std::min<int64_t>((2 * c->sms + iblocks - 1) / iblocks, (KT + 7) / 8));
  KS = std::min<int64_t>(KS, kQ0MaxSlices);
  static const int ks_env = getenv("CPQR_Q0_KS") ? atoi(getenv("CPQR_Q0_KS")) : 0;  // experiments
  if (ks_env > 0) KS = std::min<int64_t>(ks_env, std::min<int64_t>(kQ0MaxSlices, KT));
  const int kpc = (int)((KT + KS - 1) / KS);
  KS = (KT + kpc - 1) / kpc;
  dim3 grid(iblocks, (unsigned)KS);
  const int NT = (c->R + 7) / 8;
#define Q0A(NTV)                                                                                                 \
  (c->q0_stair ? launch_ex(k_q0_apply_tc<NTV, true>, grid, 256, 0, c->st, c->pdl, 1, p.Y, p.Aa, In, p.Bb,           \
                           Qm, c->R, kpc, (int)KS, c->dWp, c->dq0cnt, Wout, (const int*)c->dperm,                     \
                           c->N - 1, pp)                                                                             \
               : launch_ex(k_q0_apply_tc<NTV, false>, grid, 256, 0, c->st, c->pdl, 1, p.Y, p.Aa, In, p.Bb,          \
                           Qm, c->R, kpc, (int)KS, c->dWp, c->dq0cnt, Wout, (const int*)nullptr, 0, pp))
  switch (NT) { case 1: Q0A(1); break; case 2: Q0A(2); break; case 3: Q0A(3); break; default: Q0A(4); break; }
#undef Q0A
  CKL();
  return CPQR_OK;
}

// Z fusion (k_zform): Z = (Q_zk (x) I) Q0 of mode n on stream st (behind the V_n QR), and the
// pseudo-plan under which the apply kernel reads T instead of Y
cpqr_status launch_zform(cpqr_ctx* c, int n, const Plan& p, cudaStream_t st) {
  ZArgs a{};
  a.Qk = c->dQ[p.zk];
  a.ldq = c->dims[p.zk];
  a.Q0 = c->dQ0;
  a.Z = c->dZ;
  a.R = c->R;
  int64_t ystride = 1;
  a.JT = 1;
  for (int k = 0; k < c->N; ++k) {
    if (k == n) continue;
    if (k == p.zk) a.kpos = a.nm;
    a.td[a.nm] = p.zcur[k];
    a.ys[a.nm] = ystride;
    ystride *= c->R;
    a.JT *= p.zcur[k];
    ++a.nm;
  }
  a.JY = ystride;
  if ((size_t)(a.JT * c->R) > c->dZ_elems) return fail(c, CPQR_ECUDA, "Z buffer undersized");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((a.JT * c->R + 255) / 256, (int64_t)c->sms * 4));
  k_zform<<<grid, 256, 0, st>>>(a);
  CKL();
  return CPQR_OK;
}
Plan zf_view(const Plan& p) {
  Plan v;
  v.Y = p.zT;
  v.Aa = p.zAa;
  v.In = p.In;
  v.Bb = p.zBb;
  return v;
}

// where slab q's partial W_n (or its rows of W_N) is written: straight into W without an exchange
double* wloc(cpqr_ctx* c, int q) { return c->exchange ? c->slabs[q].dWloc : c->dW; }

// ---- peer push-reduce (small_kernels.cuh): window accessors and the two halves of an exchange
double* win_data(const cpqr_ctx* c, int r) { return static_cast<double*>(c->win_base[r]); }
unsigned long long* win_flags(const cpqr_ctx* c, int r) {
  return reinterpret_cast<unsigned long long*>(static_cast<char*>(c->win_base[r]) + c->win_data_bytes);
}
unsigned long long* win_epoch(const cpqr_ctx* c, int r) { return win_flags(c, r) + kMaxRanks; }
// this context's own window: virtual rank 0's, or this rank's
int own_win(const cpqr_ctx* c) { return c->local ? 0 : c->opt.rank; }

// the push of slab q: source rank s = q (virtual ranks) or this rank; np = 0 without peer exchange
PeerPush make_push(const cpqr_ctx* c, int q) {
  PeerPush pp{};
  if (!c->peer) return pp;
  const int s = c->local ? q : c->opt.rank;
  pp.np = c->opt.world;
  for (int r = 0; r < pp.np; ++r) {
    pp.dst[r] = win_data(c, r) + (int64_t)s * c->slot_elems;
    pp.flag[r] = win_flags(c, r) + s;
  }
  pp.epoch = win_epoch(c, s);
  pp.gcount = c->dpushcnt;
  pp.parity_stride = (int64_t)pp.np * c->slot_elems;
  static const bool sysf = getenv("CPQR_PEER_FENCE") && std::strcmp(getenv("CPQR_PEER_FENCE"), "sys") == 0;
  pp.sysfence = sysf ? 1 : 0;
  return pp;
}

// this rank's combine of the exchange its own push just started
cpqr_status peer_combine(cpqr_ctx* c, int64_t cnt, int gather, double* out) {
  if (cnt > c->slot_elems) return fail(c, CPQR_EINVAL, "peer exchange of %lld elements exceeds the window slot", (long long)cnt);
  const int o = own_win(c);
  const int64_t tot = gather ? cnt * c->opt.world : cnt;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, (int64_t)c->sms * 4));
  launch_ex(k_peer_combine, grid, 256, 0, c->st, c->pdl, 1, (const double*)win_data(c, o),
            (const unsigned long long*)win_flags(c, o), (const unsigned long long*)win_epoch(c, o), c->opt.world,
            c->slot_elems, cnt, gather, out, c->dflags, (unsigned)FLAG_PEER_TIMEOUT, c->peer_timeout_ns);
  CKL();
  return CPQR_OK;
}

// stand-alone push of every slab's n doubles, then the combine (sum in rank order, or gather)
cpqr_status peer_exchange(cpqr_ctx* c, const double* const* src, int64_t n, int gather, double* out) {
  if (n > c->slot_elems) return fail(c, CPQR_EINVAL, "peer exchange of %lld elements exceeds the window slot", (long long)n);
  for (int q = 0; q < c->nslab; ++q) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)c->sms));
    launch_ex(k_peer_push, grid, 256, 0, c->st, c->pdl, 1, src[q], n, make_push(c, q));
    CKL();
  }
  return peer_combine(c, n, gather, out);
}

// Combine the slabs' results of mode n into the full row-major W_n (or NE's M_n) in c->dW
// (DESIGN.md §8): the sum over ranks for n < N-1 (W_p = Y_p Q0 is linear in the slab, so Q0 is
// applied before the reduction), the ranks' rows in rank order for n == N-1.  Across processes:
// ncclAllReduce / ncclAllGather, or the peer push-reduce.  Virtual ranks (CPQR_COMM_LOCAL): a
// fixed-order sum kernel over the p partials, or one device copy per rank.  src[q]: slab q's local
// result; pushed: the producing kernel already pushed it into the peer windows (the Q0 apply).
cpqr_status combine_w(cpqr_ctx* c, int n, const double* const* src, bool pushed = false) {
  const int64_t R = c->R;
  if (!c->exchange) {
    if (src[0] != c->dW)
      CK(cudaMemcpyAsync(c->dW, src[0], sizeof(double) * c->dims[n] * R, cudaMemcpyDeviceToDevice, c->st));
    return CPQR_OK;
  }
  if (c->peer) {
    const int gather = (n == c->N - 1) ? 1 : 0;
    const int64_t cnt = (gather ? c->slabs[0].ldims[n] : c->dims[n]) * R;
    return pushed ? peer_combine(c, cnt, gather, c->dW) : peer_exchange(c, src, cnt, gather, c->dW);
  }
  if (!c->local) {
    if (n < c->N - 1) {
      CN(ncclAllReduce(src[0], c->dW, (size_t)(c->dims[n] * R), ncclDouble, ncclSum, c->comm, c->st));
    } else {
      CN(ncclAllGather(src[0], c->dW, (size_t)(c->slabs[0].ldims[n] * R), ncclDouble, c->comm, c->st));
    }
    return CPQR_OK;
  }
  if (n < c->N - 1) {
    RankPtrs rp{};
    for (int q = 0; q < c->nslab; ++q) rp.p[q] = src[q];
    const int64_t cnt = c->dims[n] * R;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, (int64_t)c->sms * 4));
    launch_ex(k_sum_ranks, grid, 256, 0, c->st, c->pdl, 1, rp, c->nslab, cnt, c->dW);
    CKL();
  } else {
    for (int q = 0; q < c->nslab; ++q)
      CK(cudaMemcpyAsync(c->dW + c->slabs[q].b * R, src[q], sizeof(double) * c->slabs[q].ldims[n] * R,
                         cudaMemcpyDeviceToDevice, c->st));
  }
  return CPQR_OK;
}

// out_k = P_k^T B_k for the listed modes (k_kt_cross)
cpqr_status kt_cross(cpqr_ctx* c, const int* modes, int K, const double* const* P, int np,
                            const double* const* B, int nb, double* out) {
  KtCrossArgs a{};
  for (int i = 0; i < K; ++i) {
    a.P[i] = P[modes[i]];
    a.B[i] = B[modes[i]];
    a.I[i] = c->dims[modes[i]];
  }
  a.K = K;
  a.np = np;
  a.nb = nb;
  a.out = out;
  const int64_t warps = (int64_t)K * np * nb;
  k_kt_cross<<<(int)((warps * 32 + 255) / 256), 256, 0, c->st>>>(a);
  CKL();
  return CPQR_OK;
}

// Overlap schedule of one mode update (QR / QR-SVD, one slab).  Streams: st runs the
// Multi-TTM (the stream-X pass on all but overlap_reserve SMs, then the remaining TTMs into dY), tl
// the tail (Q0 apply, solve, normalise, factor QR, fit), side the V_n QR.  The pass of mode n waits
// for the tail of mode n-1 only if it contracts mode n-1 (or writes dY itself); otherwise it runs
// beside that tail, and the remaining TTMs -- which do contract mode n-1 -- wait for it.  Same
// arithmetic as mode_update, only the launch order changes.
void trace_mark(cpqr_ctx* c, cudaStream_t st, const char* what, int n) {
  if (!c->trace) return;
  if (c->ntev == c->tev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->tev.push_back({e, ""});
  }
  char buf[64];
  snprintf(buf, sizeof buf, "%s %d %s", st == c->st ? "st" : st == c->tl ? "tl" : "side", n, what);
  c->tev[c->ntev].second = buf;
  cudaEventRecord(c->tev[c->ntev].first, st);
  ++c->ntev;
}

void trace_dump(cpqr_ctx* c) {
  if (!c->trace || c->ntev == 0) return;
  cudaDeviceSynchronize();
  for (size_t i = 0; i < c->ntev; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->tev[0].first, c->tev[i].first);
    fprintf(stderr, "trace %9.1f us  %s\n", 1e3 * ms, c->tev[i].second.c_str());
  }
  c->ntev = 0;
}

// k_kt_m: V_n beyond 64K rows splits its rows over chunks so ~4 CTAs per SM work
int kt_m_chunks(const cpqr_ctx* c, int64_t J, int S) {
  const int tiles = (S + (c->R <= 16 ? 4 : 2) - 1) / (c->R <= 16 ? 4 : 2);
  return (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)c->sms * 4 + tiles - 1) / tiles, J / 65536));
}

cpqr_status mode_update_overlap(cpqr_ctx* c, int n, bool fit_here) {
  const int N = c->N;
  const int In = (int)c->dims[n];
  const int prev = (n + N - 1) % N;
  const Plan& p = c->slabs[0].plans[n];
  // V_n QR (+ SVD of R0) on the side stream once R_{n-1} is final.  The first mode of the first
  // sweep of a capture has no tail before it in the graph (the previous launch completed).
  const bool inflight = !(n == 0 && c->ov_first);  // a tail of mode prev is in this capture
  if (!inflight) {
    CK(cudaEventRecord(c->evf, c->st));
    CK(cudaStreamWaitEvent(c->side, c->evf, 0));
  } else {
    CK(cudaStreamWaitEvent(c->side, c->evQ[prev], 0));
  }
  // small V_n (R^{N-1} <= 512 rows): the one-CTA CholeskyQR2 (k_cq_compact, nb = 1) instead of the
  // one-CTA staircase Householder, which is on this schedule's critical path (C2: 49 us -> ~15 us)
  c->vn_mode_cq = c->vn_cq_always || c->vnJ <= 512;
  trace_mark(c, c->side, "K2 start", n);
  TRY(launch_kr_qr(c, n));
  if (c->variant == CPQR_SVD) {
    TRY(launch_pinv(c, c->side, nullptr));
    c->pinv_ready = true;
  }
  if (p.zf) TRY(launch_zform(c, n, p, c->side));
  trace_mark(c, c->side, "K2 end", n);
  CK(cudaEventRecord(c->evK[n], c->side));
  // the stream-X pass; its dependence on the previous tail
  const Slab& sl = c->slabs[0];
  const size_t nx = (!p.steps.empty() && p.steps[0].in == sl.X) ? 1 : 0;
  bool dep = false;
  for (size_t i = 0; i < p.steps.size(); ++i) {
    const bool pass = i < nx || ((p.steps[i].kind == 7 || p.steps[i].kind == 3) && i == nx);
    if (pass && ((p.steps[i].modes >> prev) & 1u)) dep = true;
    if (pass && p.steps[i].out == c->dY) dep = true;
  }
  if (inflight && dep) CK(cudaStreamWaitEvent(c->st, c->evQ[prev], 0));
  trace_mark(c, c->st, dep ? "pass start (after tail n-1)" : "pass start", n);
  Plan first, rest;
  size_t nf = nx;
  if (nf < p.steps.size() && (p.steps[nf].kind == 7 || p.steps[nf].kind == 3)) ++nf;  // the pass's fix-up
  first.steps.assign(p.steps.begin(), p.steps.begin() + nf);
  rest.steps.assign(p.steps.begin() + nf, p.steps.end() - ((p.zf && nf < p.steps.size()) ? 1 : 0));
  TRY(run_plan(c, first));
  trace_mark(c, c->st, "pass end", n);
  if (inflight && !dep) CK(cudaStreamWaitEvent(c->st, c->evQ[prev], 0));
  trace_mark(c, c->st, "rest start", n);
  TRY(run_plan(c, rest));
  trace_mark(c, c->st, "rest end", n);
  // W_n = Y_(n) Q0 on st with the whole GPU (on the reserved SMs beside the next pass it took 4x
  // longer), once the V_n QR is done
  CK(cudaStreamWaitEvent(c->st, c->evK[n], 0));
  if (p.zf && nf < p.steps.size()) TRY(launch_q0_apply(c, zf_view(p), c->dW, PeerPush{}, c->dZ));
  else TRY(launch_q0_apply(c, p, c->dW));
  trace_mark(c, c->st, "q0 end", n);
  CK(cudaEventRecord(c->evY[n], c->st));
  // the tail on tl: the fused solve / normalise / factor QR (/ fast fit)
  CK(cudaStreamWaitEvent(c->tl, c->evY[n], 0));
  trace_mark(c, c->tl, "tail start", n);
  std::swap(c->st, c->tl);
  cpqr_status st = CPQR_OK;
  {
    c->tail_single = true;
    const bool fit = fit_here && c->opt.fit_mode == CPQR_FIT_FAST;
    st = launch_tsqr(c, In, nullptr, true, c->dW, c->dQ[n], c->dQt[n], c->dRk[n], c->dA[n], fit);
    c->tail_single = false;
  }
  std::swap(c->st, c->tl);
  trace_mark(c, c->tl, "tail end", n);
  c->pinv_ready = false;
  TRY(st);
  if (n == N - 1 && c->opt.fit_mode == CPQR_FIT_FAST) {  // the sweep's fit (computed by this tail)
    k_store_fit<<<1, 32, 0, c->tl>>>(c->dfit, c->dfits, c->dfitc, c->fits_cap);
    CKL();
  }
  CK(cudaEventRecord(c->evQ[n], c->tl));
  // join at the end of the capture (or every sweep with the DIRECT fit, which reads all factors)
  if (n == N - 1 && (c->ov_join || c->opt.fit_mode == CPQR_FIT_DIRECT))
    CK(cudaStreamWaitEvent(c->st, c->evQ[n], 0));
  return CPQR_OK;
}

// The NE tail of mode n on c->st (Alg. 1 lines 7-10 + the fast fit):
// Cholesky (LU fallback) or S_n^+ solve of Ahat S_n = M, lambda, normalise, Gram; then the TMA panel
cpqr_status launch_tail_ne(cpqr_ctx* c, int n, const double* Mfull, int m_rowmajor, bool fit_here) {
  const int N = c->N, In = (int)c->dims[n];
  TailNeArgs a{};
  a.Spinv = c->variant == CPQR_PINV ? c->dMpinv : nullptr;
  a.M = Mfull;
  a.m_rowmajor = m_rowmajor;
  for (int k = 0; k < N; ++k) a.G[k] = c->dG[k];
  a.N = N;
  a.n = n;
  a.In = In;
  a.R = c->R;
  a.A = c->dA[n];
  a.Gn = c->dG[n];
  a.lam = c->dlam;
  a.flags = c->dflags;
  a.do_fit = fit_here && c->opt.fit_mode == CPQR_FIT_FAST;
  a.nX2 = c->dnX2;
  a.fit = c->dfit;
  a.Ahat = c->dAhat;
  a.force_lu = getenv("CPQR_NE_FORCE_LU") ? 1 : 0;
  const int RB = rb_for(c->R);
  const size_t smem = (size_t)(3 * RB * RB + kNeLd * RB) * sizeof(double);
  switch (RB) {
    case 8: set_smem(k_tail_ne<8>, smem); k_tail_ne<8><<<1, kNeThreads, smem, c->st>>>(a); break;
    case 16: set_smem(k_tail_ne<16>, smem); k_tail_ne<16><<<1, kNeThreads, smem, c->st>>>(a); break;
    default: set_smem(k_tail_ne<32>, smem); k_tail_ne<32><<<1, kNeThreads, smem, c->st>>>(a); break;
  }
  CKL();
  k_transpose_pad<<<64, 256, 0, c->st>>>(c->dA[n], c->dims[n], In, c->R, c->RQ, c->dAt[n]);
  CKL();
  return CPQR_OK;
}

// Overlap schedule of one CP-ALS (NE) mode update, N = 3, one slab.  st: the MTTKRP -- its first TTM
// contracts mode (n+1) mod 3 with A_{n+1}, which the tail of mode n-1 (still running on tl) does not
// write; the Khatri-Rao diagonal contraction with A_{n-1} waits for that tail.  tl: the one-CTA tail
// (it also needs G_{n-1}).  M_n is copied out of the ping-pong buffers (the next pass writes them
// while the tail reads M_n).  Same arithmetic as the serial schedule up to the contraction order.
cpqr_status mode_update_ne_overlap(cpqr_ctx* c, int n, bool fit_here) {
  const int N = c->N;
  const int prev = (n + N - 1) % N;
  const Plan& p = c->slabs[0].plans[n];
  const bool inflight = !(n == 0 && c->ov_first);
  Plan first, second;
  first.steps = p.steps;
  second.diags = p.diags;
  bool dep = false;  // the dense TTM must not touch mode prev (plan_mode: ne_ov)
  for (const TtmStep& s : p.steps) dep = dep || ((s.modes >> prev) & 1u);
  if (inflight && dep) CK(cudaStreamWaitEvent(c->st, c->evQ[prev], 0));
  TRY(run_plan(c, first));
  if (inflight && !dep) CK(cudaStreamWaitEvent(c->st, c->evQ[prev], 0));
  TRY(run_plan(c, second));
  const int64_t mel = c->dims[n] * c->R;
  CK(cudaMemcpyAsync(c->dW, p.Y, sizeof(double) * mel, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaEventRecord(c->evY[n], c->st));
  CK(cudaStreamWaitEvent(c->tl, c->evY[n], 0));
  std::swap(c->st, c->tl);
  cpqr_status st = launch_tail_ne(c, n, c->dW, p.m_rowmajor, fit_here);
  if (st == CPQR_OK && n == N - 1 && c->opt.fit_mode == CPQR_FIT_FAST) {
    k_store_fit<<<1, 32, 0, c->st>>>(c->dfit, c->dfits, c->dfitc, c->fits_cap);
    if (cudaGetLastError() != cudaSuccess) st = CPQR_ECUDA;
    else c->launch_count++;
  }
  std::swap(c->st, c->tl);
  TRY(st);
  CK(cudaEventRecord(c->evQ[n], c->tl));
  if (n == N - 1 && (c->ov_join || c->opt.fit_mode == CPQR_FIT_DIRECT)) CK(cudaStreamWaitEvent(c->st, c->evQ[n], 0));
  return CPQR_OK;
}

cpqr_status mode_update(cpqr_ctx* c, int n, bool fit_here) {
  const int N = c->N;
  const int In = (int)c->dims[n];
  if (c->overlap && !c->kt && !c->opt.profile) return mode_update_overlap(c, n, fit_here);
  if (c->overlap_ne && !c->kt && !c->opt.profile) return mode_update_ne_overlap(c, n, fit_here);
  prof_mark(c, -1);
  if (ne_family(c->variant)) {
    const double* Mfull = nullptr;
    int m_rowmajor = c->slabs[0].plans[n].m_rowmajor;
    // CP-ALS-PINV: S_n^+ from the Grams (k_ne_pinv) on the side stream beside the MTTKRP
    const bool pinv = c->variant == CPQR_PINV;
    static const bool no_fork_ne = getenv("CPQR_NO_FORK") != nullptr;
    const bool pfork = pinv && !c->opt.profile && !no_fork_ne;
    if (pinv) {
      if (pfork) {
        CK(cudaEventRecord(c->evf, c->st));
        CK(cudaStreamWaitEvent(c->side, c->evf, 0));
      }
      NePinvArgs q{};
      for (int k = 0; k < N; ++k) q.G[k] = c->dG[k];
      q.N = N; q.n = n; q.R = c->R;
      q.tau = (c->opt.svd_tau < 0) ? c->R * 2.220446049250313e-16 : c->opt.svd_tau;
      q.Mout = c->dMpinv; q.flags = c->dflags;
      const size_t smem = (size_t)(2 * c->R * c->R + 2 * c->R * (c->R + 1)) * sizeof(double);
      k_ne_pinv<<<1, 512, smem, pfork ? c->side : c->st>>>(q);
      CKL();
      if (pfork) CK(cudaEventRecord(c->evj, c->side));
      prof_mark(c, 5);
    }
    if (c->kt) {  // Kruskal input: M_n = B_n diag(lam_x) (*)_{k != n} B_k^T A_k
      int modes[kMaxN], K = 0;
      for (int k = 0; k < N; ++k) if (k != n) modes[K++] = k;
      const double* Ac[kMaxN];
      const double* Bc[kMaxN];
      for (int k = 0; k < N; ++k) { Ac[k] = c->dA[k]; Bc[k] = c->dKtB[k]; }
      TRY(kt_cross(c, modes, K, Bc, c->ktS, Ac, c->R, c->dKtC));
      const int grid = (int)std::min<int64_t>(((int64_t)In * c->R + 255) / 256, (int64_t)c->sms * 8);
      k_kt_mttkrp<<<grid, 256, 0, c->st>>>(c->dKtB[n], In, c->ktS, c->dKtLam, c->dKtC, K, c->R, c->dW);
      CKL();
      Mfull = c->dW;
      m_rowmajor = 1;
      prof_mark(c, 0);
    } else {
      // MTTKRP of each slab (the partial M_n, or M_N's local rows); the virtual ranks copy theirs
      // out of the shared intermediate buffers before the next slab runs
      const double* src[kMaxWorld];
      for (int q = 0; q < c->nslab; ++q) {
        const Plan& p = c->slabs[q].plans[n];
        TRY(run_plan(c, p));
        src[q] = p.Y;
        if (c->local) {
          const int64_t rows = (n == N - 1) ? c->slabs[q].ldims[n] : c->dims[n];
          CK(cudaMemcpyAsync(c->slabs[q].dWloc, p.Y, sizeof(double) * rows * c->R, cudaMemcpyDeviceToDevice, c->st));
          src[q] = c->slabs[q].dWloc;
        }
        prof_mark(c, 0);
      }
      Mfull = src[0];
      if (c->exchange) {
        // the rows of M_N are gathered: its layout must be row-major (rmode < n, plan_mode)
        if (n == N - 1 && !m_rowmajor) return fail(c, CPQR_EINVAL, "NE: column-major M_N cannot be gathered");
        TRY(combine_w(c, n, src));
        Mfull = c->dW;
        prof_mark(c, 6);
      }
    }
    if (pfork) CK(cudaStreamWaitEvent(c->st, c->evj, 0));
    TRY(launch_tail_ne(c, n, Mfull, m_rowmajor, fit_here));
    prof_mark(c, 5);
    return CPQR_OK;
  }
  // Alg. 2 lines 6-7: V_n and its QR (K2), on the side stream: it depends only on the R_k and
  // overlaps the Multi-TTM (joined before the Q0 apply).  With profiling on it runs in line.
  static const bool no_fork = getenv("CPQR_NO_FORK") != nullptr;  // debugging: V_n QR inline
  // dimension-tree modes without an X pass have no long kernel to hide K2 behind, and a side-stream
  // multi-CTA QR would find no free SMs: there the CholeskyQR2 V_n QR runs inline (vn_inline)
  const bool tree_nofresh = c->tree && !(n == 0 || n == c->tree_h) && !ne_family(c->variant) && !c->kt;
  c->vn_mode_cq = c->vn_cq_always || (c->vn_cq_tree && tree_nofresh);
  const bool fork = !c->opt.profile && !no_fork && !(c->vn_mode_cq && tree_nofresh);
  // there the V_n QR runs inline, but the one-CTA SVD of R0 (QR-SVD) still forks to the side
  // stream (the stream grids leave it an SM) and is joined only before the solve
  const bool pinv_fork = !fork && c->variant == CPQR_SVD && !c->opt.profile && !no_fork;
  if (fork) {
    CK(cudaEventRecord(c->evf, c->st));
    CK(cudaStreamWaitEvent(c->side, c->evf, 0));
  }
  {
    cudaStream_t keep = c->side;
    if (!fork) c->side = nullptr;
    cpqr_status st = launch_kr_qr(c, n);
    if (st == CPQR_OK && !c->kt && c->slabs[0].plans[n].zf)
      st = launch_zform(c, n, c->slabs[0].plans[n], fork ? keep : c->st);
    if (st == CPQR_OK && pinv_fork) {
      CK(cudaEventRecord(c->evf, c->st));
      CK(cudaStreamWaitEvent(keep, c->evf, 0));
      c->side = keep;
    }
    if (st == CPQR_OK && c->variant == CPQR_SVD) {  // SVD of R0 right behind its QR, off the critical path
      st = launch_pinv(c, c->side ? c->side : c->st, nullptr);
      c->pinv_ready = (st == CPQR_OK);
    }
    c->side = keep;
    TRY(st);
  }
  if (fork || pinv_fork) CK(cudaEventRecord(c->evj, c->side));
  prof_mark(c, 3);
  if (c->kt) {
    // Kruskal input: C_k = Q_k^T B_k, then W_n = B_n diag(lam_x) [((.)_k C_k)^T Q0]
    int modes[kMaxN], K = 0;
    for (int k = 0; k < N; ++k) if (k != n) modes[K++] = k;
    const double* Qc[kMaxN];
    const double* Bc[kMaxN];
    for (int k = 0; k < N; ++k) { Qc[k] = c->dQ[k]; Bc[k] = c->dKtB[k]; }
    TRY(kt_cross(c, modes, K, Qc, c->R, Bc, c->ktS, c->dKtC));
    prof_mark(c, 0);
    if (fork) CK(cudaStreamWaitEvent(c->st, c->evj, 0));
    KtMArgs ma{};
    ma.C = c->dKtC; ma.N1 = N - 1; ma.R = c->R; ma.S = c->ktS; ma.Q0 = c->dQ0; ma.M = c->dKtM;
    ma.J = 1;
    for (int k = 0, m = 0; k < N; ++k)
      if (k != n) { ma.rad[m] = c->vq[k]; ma.J *= c->vq[k]; ++m; }
    // V_n beyond 64K rows: split the rows over chunks so ~4 CTAs per SM work (partials in c->dPart...)
    ma.nc = kt_m_chunks(c, ma.J, ma.S);
    ma.P = c->dKtP;  // sized by cpqr_set_ktensor (kt_m_chunks)
    if (ma.nc > 1 && (size_t)ma.S * ma.nc * c->R > c->ktP_elems) return fail(c, CPQR_ECUDA, "k_kt_m partials undersized");
    // terms per CTA: kt_m_st when V_n is chunked (Q0 re-read S / st times), else one term per CTA
    // (a small V_n: more CTAs beat fewer passes)
    ma.st = ma.nc > 1 ? (c->R <= 16 ? 4 : 2) : 1;
    const dim3 kg((unsigned)((ma.S + ma.st - 1) / ma.st), (unsigned)ma.nc);
    switch (rb_for(c->R)) {
      case 8: k_kt_m<8><<<kg, 256, 0, c->st>>>(ma); break;
      case 16: k_kt_m<16><<<kg, 256, 0, c->st>>>(ma); break;
      default: k_kt_m<32><<<kg, 256, 0, c->st>>>(ma); break;
    }
    CKL();
    if (ma.nc > 1) {
      k_kt_m_reduce<<<(ma.S * c->R + 255) / 256, 256, 0, c->st>>>(c->dKtP, ma.S, c->R, ma.nc, c->dKtM);
      CKL();
    }
    const int grid = (int)std::min<int64_t>(((int64_t)In * c->R + 255) / 256, (int64_t)c->sms * 8);
    k_kt_w<<<grid, 256, 0, c->st>>>(c->dKtB[n], In, c->ktS, c->dKtLam, c->dKtM, c->R, c->dW);
    CKL();
    prof_mark(c, 4);
  } else {
    // line 8, per slab: the Multi-TTM (first step = the stream-X pass; with the dimension tree only
    // the first mode of each half has one), then line 9: W_p = Y_(n) Q0 of the slab (local rows)
    const double* src[kMaxWorld];
    for (int q = 0; q < c->nslab; ++q) {
      const Slab& sl = c->slabs[q];
      const Plan& p = sl.plans[n];
      const size_t nx = (!p.steps.empty() && p.steps[0].in == sl.X) ? 1 : 0;
      Plan first;
      first.steps.assign(p.steps.begin(), p.steps.begin() + nx);
      TRY(run_plan(c, first));
      prof_mark(c, 0);
      Plan rest;
      rest.steps.assign(p.steps.begin() + nx, p.steps.end() - (p.zf ? 1 : 0));  // Z fusion: no last TTM
      TRY(run_plan(c, rest));
      prof_mark(c, 1);
      if (fork && q == 0) CK(cudaStreamWaitEvent(c->st, c->evj, 0));
      if (p.zf) TRY(launch_q0_apply(c, zf_view(p), wloc(c, q), make_push(c, q), c->dZ));
      else TRY(launch_q0_apply(c, p, wloc(c, q), make_push(c, q)));
      src[q] = wloc(c, q);
      prof_mark(c, 4);
    }
    TRY(combine_w(c, n, src, c->peer));
    prof_mark(c, 6);
  }
  if (pinv_fork) CK(cudaStreamWaitEvent(c->st, c->evj, 0));
  prof_mark(c, 5);
  // lines 10-12: solve (substitution / SVD), lambda, normalise, factor QR (+ fast fit after mode N),
  // one fused launch (k_cq_compact): timed as the factor-QR phase
  const bool fit = fit_here && c->opt.fit_mode == CPQR_FIT_FAST;
  const cpqr_status tst = launch_tsqr(c, In, nullptr, true, c->dW, c->dQ[n], c->dQt[n], c->dRk[n], c->dA[n], fit);
  c->pinv_ready = false;
  TRY(tst);
  prof_mark(c, 2);
  return CPQR_OK;
}

// DIRECT fit: ||X - [[lambda; A]]||^2 over each slab (fixed-order partials), summed
// over the ranks, then fit = 1 - ||X - Xh|| / ||X||.
cpqr_status direct_fit(cpqr_ctx* c) {
  prof_mark(c, -1);
  double* res = c->dred + 4096;
  if (c->kt) {  // Kruskal input: the residual entry by entry from the factors (k_kt_resid)
    KtResidArgs a{};
    for (int k = 0; k < c->N; ++k) { a.B[k] = c->dKtB[k]; a.A[k] = c->dA[k]; a.I[k] = c->tdims[k]; a.ld[k] = c->dims[k]; }
    a.N = c->N; a.S = c->ktS; a.R = c->R; a.lamx = c->dKtLam; a.lam = c->dlam; a.part = c->dred;
    const int grid = c->sms * 4;
    k_kt_resid<<<grid, 256, 0, c->st>>>(a);
    CKL();
    k_sum_final<<<1, 256, 0, c->st>>>(c->dred, grid, res);
    CKL();
    k_fit_from_resid<<<1, 32, 0, c->st>>>(res, c->dnX2, c->dfit);
    CKL();
    prof_mark(c, 5);
    return CPQR_OK;
  }
  for (int q = 0; q < c->nslab; ++q) {
    const Slab& sl = c->slabs[q];
    ResidArgs a{};
    a.X = sl.X;
    a.n = sl.numel;
    a.N = c->N;
    for (int k = 0; k < c->N; ++k) { a.dims[k] = sl.ldims[k]; a.A[k] = c->dA[k]; a.lda[k] = c->dims[k]; }
    a.off_last = sl.b;
    a.lam = c->dlam;
    a.R = c->R;
    a.part = c->dred;
    const int grid = c->sms * 4;
    k_resid_partial<<<grid, 256, 0, c->st>>>(a);
    CKL();
    k_sum_final<<<1, 256, 0, c->st>>>(c->dred, grid, c->nslab > 1 ? res + 8 + q : res);
    CKL();
  }
  prof_mark(c, 5);
  if (c->peer) {  // rank-order sum of the slab residuals through the peer windows
    const double* src[kMaxWorld];
    for (int q = 0; q < c->nslab; ++q) src[q] = c->nslab > 1 ? res + 8 + q : res;
    TRY(peer_exchange(c, src, 1, 0, res));
  } else if (c->nslab > 1) {  // virtual ranks: rank-order sum of the slab residuals
    k_sum_final<<<1, 256, 0, c->st>>>(res + 8, c->nslab, res);
    CKL();
  } else if (c->comm) {
    CN(ncclAllReduce(res, res, 1, ncclDouble, ncclSum, c->comm, c->st));
  }
  prof_mark(c, 6);
  k_fit_from_resid<<<1, 32, 0, c->st>>>(res, c->dnX2, c->dfit);
  CKL();
  prof_mark(c, 5);
  return CPQR_OK;
}

// fold the recorded phase marks into c->prof (after they completed)
void prof_accumulate(cpqr_ctx* c) {
  if (c->nmarks > 0) cudaEventSynchronize(c->evp[c->nmarks - 1]);
  for (int i = 1; i < c->nmarks; ++i) {
    const int ph = c->evphase[i];
    float ms;
    if (ph >= 0 && cudaEventElapsedTime(&ms, c->evp[i - 1], c->evp[i]) == cudaSuccess) {
      c->prof.ms[ph] += ms;
      c->prof.launches[ph] += c->evlaunch[i] - c->evlaunch[i - 1];
    }
  }
  c->nmarks = 0;
}

// One sweep of mode updates, then the fit into the next dfits slot (k_store_fit; in the overlap
// schedule with the fast fit the last tail stores it on its own stream).
cpqr_status one_sweep(cpqr_ctx* c) {
  const bool ov = (c->overlap || c->overlap_ne) && !c->kt && !c->opt.profile;
  for (int n = 0; n < c->N; ++n) {
    TRY(mode_update(c, n, n == c->N - 1));
    if (c->opt.profile) prof_accumulate(c);
  }
  if (c->opt.fit_mode == CPQR_FIT_DIRECT) TRY(direct_fit(c));
  if (!ov || c->opt.fit_mode == CPQR_FIT_DIRECT) {
    k_store_fit<<<1, 32, 0, c->st>>>(c->dfit, c->dfits, c->dfitc, c->fits_cap);
    CKL();
  }
  if (c->opt.profile) prof_accumulate(c);
  return CPQR_OK;
}

// capture `ns` sweeps into a graph; the overlap schedule's tails cross the sweep boundaries inside
cpqr_status capture_sweeps(cpqr_ctx* c, int ns, cudaGraphExec_t* out, int64_t* launches) {
  const int64_t before = c->launch_count;
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  cpqr_status st = CPQR_OK;
  for (int s = 0; s < ns && st == CPQR_OK; ++s) {
    c->ov_first = (s == 0);
    c->ov_join = (s == ns - 1);
    st = one_sweep(c);
  }
  c->ov_first = c->ov_join = true;
  cudaError_t ce = cudaStreamEndCapture(c->st, &g);
  if (st != CPQR_OK) {
    if (ce == cudaSuccess) cudaGraphDestroy(g);
    return st;
  }
  CK(ce);
  if (*out) cudaGraphExecDestroy(*out);
  *out = nullptr;
  CK(cudaGraphInstantiate(out, g, 0));
  cudaGraphDestroy(g);
  *launches = c->launch_count - before;
  return CPQR_OK;
}


cpqr_status ensure_fits(cpqr_ctx* c, int n) {
  if (n <= c->fits_cap) return CPQR_OK;
  if (c->dfits) dfree(c->dfits);
  c->dfits = nullptr;
  if (dmalloc(&c->dfits, sizeof(double) * n) != cudaSuccess) return fail(c, CPQR_ENOMEM, "fits");
  c->fits_cap = n;
  c->graph_valid = false;  // the captured k_store_fit launches hold the old buffer and capacity
  return CPQR_OK;
}

// splitmix64 + Box-Muller: counter-based N(0,1) (cpqr_init_factors)
uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
double normal_at(uint64_t seed, uint64_t i) {
  const uint64_t a = splitmix64(seed * 0x2545F4914F6CDD1Dull + 2 * (i / 2));
  const uint64_t b = splitmix64(seed * 0x2545F4914F6CDD1Dull + 2 * (i / 2) + 1);
  const double u1 = ((a >> 11) + 1.0) * (1.0 / 9007199254740993.0);
  const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
  const double r = std::sqrt(-2.0 * std::log(u1));
  return (i & 1) ? r * std::sin(2.0 * M_PI * u2) : r * std::cos(2.0 * M_PI * u2);
}

cpqr_status begin_call(cpqr_ctx* c) {
  CK(cudaSetDevice(c->opt.device));
  if (c->user) {
    CK(cudaEventRecord(c->ev0, c->user));
    CK(cudaStreamWaitEvent(c->st, c->ev0, 0));
  }
  return CPQR_OK;
}
cpqr_status end_call(cpqr_ctx* c) {
  if (c->user) {
    CK(cudaEventRecord(c->ev1, c->st));
    CK(cudaStreamWaitEvent(c->user, c->ev1, 0));
  }
  CK(cudaStreamSynchronize(c->st));
  return CPQR_OK;
}

}  // namespace

// =============================================================================== C ABI
CPQR_API void cpqr_default_options(cpqr_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->struct_size = sizeof(cpqr_options);
  o->svd_tau = -1.0;
  o->fit_mode = CPQR_FIT_FAST;
  o->device = 0;
  o->stream = nullptr;
  o->rank = 0;
  o->world = 1;
  o->use_graph = 1;
  o->profile = 0;
  o->mttm_tree = 0;
}

CPQR_API const char* cpqr_version(void) { return "cpqr 0.1.0 sm_100a fp64"; }

CPQR_API const char* cpqr_status_string(cpqr_status s) {
  switch (s) {
    case CPQR_OK: return "ok";
    case CPQR_EINVAL: return "invalid argument";
    case CPQR_ENOMEM: return "out of device memory";
    case CPQR_ECUDA: return "CUDA error";
    case CPQR_ENCCL: return "NCCL error";
    case CPQR_ESTATE: return "invalid state (tensor or factors not set)";
    case CPQR_EDIVERGED: return "non-finite factor (diverged)";
    default: return "unknown status";
  }
}

CPQR_API const char* cpqr_last_error(const cpqr_ctx* c) { return c ? c->err.c_str() : "null context"; }

CPQR_API cpqr_status cpqr_nccl_unique_id(uint8_t id[128]) {
  if (!id) return CPQR_EINVAL;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return CPQR_ENCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return CPQR_OK;
}

static int64_t max_dim(const cpqr_ctx* c);
// ---- peer push-reduce: window exchange between processes (CUDA IPC) and its debug hooks
CPQR_API cpqr_status cpqr_peer_handle(cpqr_ctx* c, uint8_t handle[64]) {
  if (!c || !handle) return CPQR_EINVAL;
  if (!c->peer || c->local) return fail(c, CPQR_EINVAL, "cpqr_peer_handle needs comm = CPQR_COMM_PEER");
  CK(cudaSetDevice(c->opt.device));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  CK(cudaIpcGetMemHandle(&h, c->win_base[c->opt.rank]));
  std::memcpy(handle, &h, 64);
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_peer_connect(cpqr_ctx* c, const uint8_t* handles) {
  if (!c || !handles) return CPQR_EINVAL;
  if (!c->peer || c->local) return fail(c, CPQR_EINVAL, "cpqr_peer_connect needs comm = CPQR_COMM_PEER");
  if (c->peers_connected) return c->opt.world == 1 ? CPQR_OK : fail(c, CPQR_ESTATE, "peers already connected");
  CK(cudaSetDevice(c->opt.device));
  for (int r = 0; r < c->opt.world; ++r) {
    if (r == c->opt.rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * (size_t)r, 64);
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->win_base[r] = p;
    c->win_mapped[r] = true;
  }
  c->peers_connected = true;
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_debug_peer(cpqr_ctx* c, int64_t info[4]) {
  if (!c || !info) return CPQR_EINVAL;
  if (!c->peer) return fail(c, CPQR_EINVAL, "no peer windows (comm)");
  TRY(begin_call(c));
  CK(cudaStreamSynchronize(c->st));
  const int o = own_win(c);
  std::vector<unsigned char> w0(c->win_bytes), wr(c->win_bytes);
  CK(cudaMemcpy(w0.data(), c->win_base[o], c->win_bytes, cudaMemcpyDeviceToHost));
  unsigned long long ep = 0, fmin = ~0ull;
  std::memcpy(&ep, w0.data() + c->win_data_bytes + sizeof(unsigned long long) * kMaxRanks, sizeof ep);
  for (int q = 0; q < c->opt.world; ++q) {
    unsigned long long f;
    std::memcpy(&f, w0.data() + c->win_data_bytes + sizeof(unsigned long long) * q, sizeof f);
    fmin = std::min(fmin, f);
  }
  int64_t differ = 0;
  if (c->local)  // every virtual rank received the same slots and flags (the epoch word aside)
    for (int r = 1; r < c->opt.world; ++r) {
      CK(cudaMemcpy(wr.data(), c->win_base[r], c->win_bytes, cudaMemcpyDeviceToHost));
      const size_t cmp = c->win_data_bytes + sizeof(unsigned long long) * kMaxRanks;
      if (std::memcmp(w0.data(), wr.data(), cmp) != 0) ++differ;
      unsigned long long er;
      std::memcpy(&er, wr.data() + cmp, sizeof er);
      if (er != ep) ++differ;
    }
  info[0] = (int64_t)ep;
  info[1] = differ;
  info[2] = (int64_t)c->win_bytes;
  info[3] = (int64_t)fmin;
  return end_call(c);
}

CPQR_API cpqr_status cpqr_debug_peer_put(cpqr_ctx* c, const double* src, int64_t n) {
  if (!c || !src || n < 1) return CPQR_EINVAL;
  if (!c->peer || c->local) return fail(c, CPQR_EINVAL, "cpqr_debug_peer_put needs comm = CPQR_COMM_PEER");
  if (!c->peers_connected) return fail(c, CPQR_ESTATE, "cpqr_peer_connect first");
  if (n > max_dim(c) * c->R) return fail(c, CPQR_EINVAL, "n exceeds max(I_k) R = %lld", (long long)(max_dim(c) * c->R));
  TRY(begin_call(c));
  CK(cudaMemcpyAsync(c->slabs[0].dWloc, src, sizeof(double) * n, cudaMemcpyHostToDevice, c->st));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)c->sms));
  launch_ex(k_peer_push, grid, 256, 0, c->st, false, 1, (const double*)c->slabs[0].dWloc, n, make_push(c, 0));
  CKL();
  return end_call(c);
}

CPQR_API cpqr_status cpqr_debug_peer_get(cpqr_ctx* c, double* out, int64_t n, int gather) {
  if (!c || !out || n < 1) return CPQR_EINVAL;
  if (!c->peer || c->local) return fail(c, CPQR_EINVAL, "cpqr_debug_peer_get needs comm = CPQR_COMM_PEER");
  if (!c->peers_connected) return fail(c, CPQR_ESTATE, "cpqr_peer_connect first");
  const int64_t tot = gather ? n * c->opt.world : n;
  if (n > c->slot_elems || tot > max_dim(c) * c->R) return fail(c, CPQR_EINVAL, "n too large");
  TRY(begin_call(c));
  TRY(peer_combine(c, n, gather ? 1 : 0, c->dW));
  unsigned fl = 0;
  CK(cudaMemcpyAsync(out, c->dW, sizeof(double) * tot, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(&fl, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->st));
  TRY(end_call(c));
  if (fl & FLAG_PEER_TIMEOUT) return fail(c, CPQR_ENCCL, "peer exchange: a rank did not arrive in time");
  return CPQR_OK;
}

static cpqr_status create_impl(cpqr_ctx* c, int N, const int64_t* dims, int R);

CPQR_API cpqr_status cpqr_create(int N, const int64_t* dims, int R, int variant,
                                 const cpqr_options* opt, cpqr_ctx** out) {
  if (!out || !dims) return CPQR_EINVAL;
  *out = nullptr;
  if (N < 2 || N > kMaxN || R < 1 || R > kMaxR) return CPQR_EINVAL;
  if (variant < CPQR_NE || variant > CPQR_PINV) return CPQR_EINVAL;
  for (int k = 0; k < N; ++k)
    if (dims[k] < 1 || dims[k] > (1ll << 31) - 1) return CPQR_EINVAL;
  cpqr_ctx* c = new cpqr_ctx();
  int64_t pdims[kMaxModes];  // short modes (I_k < R) are stored padded to R rows
  for (int k = 0; k < N; ++k) {
    c->tdims[k] = dims[k];
    c->vq[k] = (int)std::min<int64_t>(dims[k], R);
    pdims[k] = std::max<int64_t>(dims[k], R);
    c->short_modes = c->short_modes || dims[k] < R;
  }
  cpqr_default_options(&c->opt);
  if (opt) {
    if (opt->struct_size < sizeof(uint32_t) || opt->struct_size > sizeof(cpqr_options)) { delete c; return CPQR_EINVAL; }
    std::memcpy(&c->opt, opt, opt->struct_size);
    c->opt.struct_size = sizeof(cpqr_options);
  }
  if (c->opt.world < 1 || c->opt.world > kMaxWorld || c->opt.rank < 0 || c->opt.rank >= c->opt.world) {
    delete c;
    return CPQR_EINVAL;
  }
  if (c->opt.comm < CPQR_COMM_NCCL || c->opt.comm > CPQR_COMM_LOCAL_PEER) { delete c; return CPQR_EINVAL; }
  if (c->opt.world > 1 && (dims[N - 1] % c->opt.world) != 0) { delete c; return CPQR_EINVAL; }
  c->variant = variant;
  if (c->short_modes && c->opt.world > 1) { delete c; return CPQR_EINVAL; }  // Kruskal input only
  {
    const char* po = getenv("CPQR_PAD_ODD");
    if (!c->short_modes && (pdims[0] & 1) && !(po && atoi(po) == 0)) {
      pdims[0] += 1;
      c->pad1 = true;
    }
  }
  cpqr_status st = create_impl(c, N, pdims, R);
  if (st != CPQR_OK) {
    fprintf(stderr, "cpqr_create: %s: %s\n", cpqr_status_string(st), c->err.c_str());
    cpqr_destroy(c);
    return st;
  }
  *out = c;
  return CPQR_OK;
}

static cpqr_status create_impl(cpqr_ctx* c, int N, const int64_t* dims, int R) {
  c->N = N;
  c->R = R;
  c->RQ = 16 * ((R + 15) / 16);
  c->use_tma = getenv("CPQR_NO_TMA") == nullptr;
  c->streamk = getenv("CPQR_STREAMK") ? atoi(getenv("CPQR_STREAMK")) : -1;
  c->pdl = getenv("CPQR_PDL") && atoi(getenv("CPQR_PDL")) == 1;
  c->q0_stair = getenv("CPQR_Q0_STAIR") && atoi(getenv("CPQR_Q0_STAIR")) == 1;
  c->gsw = getenv("CPQR_GRAPH_SWEEPS") ? std::max(1, atoi(getenv("CPQR_GRAPH_SWEEPS"))) : 1;
  c->trace = getenv("CPQR_TRACE") && atoi(getenv("CPQR_TRACE")) == 1 && !c->opt.use_graph;
  c->tree = c->opt.mttm_tree != 0 && N >= 3 && !ne_family(c->variant);
  c->tree_h = (N + 1) / 2;
  {
    const char* f = getenv("CPQR_SLICE");  // "1" / "0" force the fused slice kernel on / off
    c->fuse_slice = f ? (f[0] == '1') : (R < 24);
  }
  for (int k = 0; k < N; ++k) c->dims[k] = dims[k];
  // slabs of the last mode: this rank's, or all p of the virtual ranks
  c->local = (c->opt.comm == CPQR_COMM_LOCAL || c->opt.comm == CPQR_COMM_LOCAL_PEER) && c->opt.world > 1;
  c->nslab = c->local ? c->opt.world : 1;
  c->peer = c->opt.comm == CPQR_COMM_PEER || (c->opt.comm == CPQR_COMM_LOCAL_PEER && c->opt.world > 1);
  // a one-rank communicator (world = 1, comm = NCCL, an id given) runs the in-graph collectives on
  // one GPU; so does a one-rank peer window (comm = PEER): hardware checks of the exchange paths
  bool have_id = false;
  for (int i = 0; i < 128; ++i) have_id = have_id || c->opt.nccl_id[i] != 0;
  const bool nccl1 = c->opt.world == 1 && c->opt.comm == CPQR_COMM_NCCL && have_id;
  c->exchange = c->opt.world > 1 || c->peer || nccl1;
  if (const char* t = getenv("CPQR_PEER_TIMEOUT_MS")) c->peer_timeout_ns = 1000000ull * (unsigned long long)std::max(1, atoi(t));
  const int64_t per = dims[N - 1] / c->opt.world;
  for (int q = 0; q < c->nslab; ++q) {
    Slab& sl = c->slabs[q];
    const int r = c->local ? q : c->opt.rank;
    for (int k = 0; k < N; ++k) sl.ldims[k] = dims[k];
    sl.b = per * r;
    sl.e = sl.b + per;
    sl.ldims[N - 1] = per;
    sl.numel = prod(sl.ldims, 0, N);
  }
  std::memset(&c->prof, 0, sizeof c->prof);
  if (cudaSetDevice(c->opt.device) != cudaSuccess) return fail(c, CPQR_ECUDA, "cudaSetDevice(%d)", c->opt.device);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->opt.device);
  // one SM left to the side-stream kernel beside the stream pass (V_n QR, or S_n^+ for PINV)
  c->stream_sms = (c->variant == CPQR_NE || getenv("CPQR_ALL_SMS")) ? c->sms : std::max(1, c->sms - 1);
  {  // overlap schedule (mode_update_overlap): HBM-bound QR / QR-SVD sweeps on one GPU by default
     // (measured vs the serial schedule, 40 sweeps x 2: C2 2615 -> 2680, C3 555 -> 560, C4 465 -> 484)
    const char* ov = getenv("CPQR_OVERLAP");
    const bool elig = !ne_family(c->variant) && !c->tree && !c->exchange && N >= 3 && !c->opt.profile;
    c->overlap = elig && (ov ? atoi(ov) == 1 : R <= 16);
    if (const char* r = getenv("CPQR_OVERLAP_SMS")) c->overlap_reserve = std::max(0, atoi(r));
    if (const char* r = getenv("CPQR_OVERLAP_CW1")) c->ov_cw1 = atoi(r) != 0;
    if (c->overlap) c->stream_sms = std::max(1, c->sms - c->overlap_reserve);
    // NE overlap schedule (mode_update_ne_overlap): 3-way CP-ALS on one GPU; the stream grids leave
    // one SM to the one-CTA tail.  Default where it measured faster: tensors up to 1.2 GB, whose
    // 21-26 us tail is a large share of the pass (C2 400^3 R = 10: 2810 -> 3150 sweeps/s), and
    // R >= 24 (700^3 R = 32: 2.66 -> 2.46 ms per iteration); at 700^3 R = 4..8 its contraction order
    // (mode (n+1) mod 3 first instead of the last mode) costs 8 %.  CPQR_OVERLAP_NE=0/1 off / on
    const char* ovn = getenv("CPQR_OVERLAP_NE");
    const double xbytes = 8.0 * (double)prod(dims, 0, N);
    const bool ne_elig = c->variant == CPQR_NE && N == 3 && !c->exchange && !c->opt.profile;
    c->overlap_ne = ne_elig && (ovn ? atoi(ovn) == 1 : (xbytes <= 1.2e9 || R >= 24));
    if (c->overlap_ne) c->stream_sms = std::max(1, c->sms - 1);
  }
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  c->user = (cudaStream_t)c->opt.stream;
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->tl, cudaStreamNonBlocking));
  for (int k = 0; k < kMaxN; ++k) {
    CK(cudaEventCreateWithFlags(&c->evY[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->evQ[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->evK[k], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&c->evf, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->evj, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev0, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev1, cudaEventDisableTiming));
  int64_t imax = 0;
  for (int k = 0; k < N; ++k) {
    imax = std::max(imax, dims[k]);
    CK(dmalloc(&c->dA[k], sizeof(double) * dims[k] * R));
    CK(dmalloc(&c->dQ[k], sizeof(double) * dims[k] * R));
    CK(dmalloc(&c->dRk[k], sizeof(double) * R * R));
    CK(dmalloc(&c->dG[k], sizeof(double) * R * R));
    CK(dmalloc(&c->dQt[k], sizeof(double) * dims[k] * c->RQ));
    CK(dmalloc(&c->dAt[k], sizeof(double) * dims[k] * c->RQ));
    CK(cudaMemset(c->dRk[k], 0, sizeof(double) * R * R));
    CK(cudaMemset(c->dG[k], 0, sizeof(double) * R * R));
  }
  int64_t J = 1;
  for (int k = 0; k < N - 1; ++k) J *= R;
  if (c->short_modes) {  // V_n rows: prod_{k != n} min(I_k, R), the largest over the modes
    J = 0;
    for (int n = 0; n < N; ++n) {
      int64_t j = 1;
      for (int k = 0; k < N; ++k) if (k != n) j *= c->vq[k];
      J = std::max(J, j);
    }
  }
  if ((double)J * R * 8.0 * 3.0 > 120e9) return fail(c, CPQR_ENOMEM, "V_n of %lld x %d rows: Q0 and the V_n QR buffers exceed 120 GB", (long long)J, R);
  CK(dmalloc(&c->dlam, sizeof(double) * R));
  CK(dmalloc(&c->dQ0, sizeof(double) * J * R));
  CK(dmalloc(&c->dR0, sizeof(double) * R * R));
  CK(dmalloc(&c->dW, sizeof(double) * imax * R));
  if (c->exchange)
    for (int q = 0; q < c->nslab; ++q) CK(dmalloc(&c->slabs[q].dWloc, sizeof(double) * imax * R));
  if (c->peer) {
    // receive windows (plain cudaMalloc: exported through CUDA IPC): this rank's, or all virtual ranks'
    const int np = c->opt.world;
    c->slot_elems = std::max<int64_t>(imax * R, 64);
    c->win_data_bytes = ((size_t)2 * np * c->slot_elems * sizeof(double) + 127) / 128 * 128;
    c->win_bytes = c->win_data_bytes + sizeof(unsigned long long) * (kMaxRanks + 16);
    for (int r = 0; r < np; ++r) {
      if (!c->local && r != c->opt.rank) continue;
      CK(cudaMalloc(&c->win_base[r], c->win_bytes));
      CK(cudaMemset(c->win_base[r], 0, c->win_bytes));
    }
    CK(dmalloc(&c->dpushcnt, sizeof(unsigned) * 4));
    CK(cudaMemset(c->dpushcnt, 0, sizeof(unsigned) * 4));
    c->peers_connected = c->local || np == 1;
  }
  CK(dmalloc(&c->dnX2p, sizeof(double) * 64));
  CK(dmalloc(&c->dfitc, sizeof(unsigned) * 4));
  CK(dmalloc(&c->dSk, sizeof(double) * 2 * (2 * c->sms) * 256 * R));
  CK(dmalloc(&c->dSkCnt, sizeof(unsigned) * (2 * c->sms + 1)));
  CK(cudaMemset(c->dSkCnt, 0, sizeof(unsigned) * (2 * c->sms + 1)));
  CK(dmalloc(&c->dAhat, sizeof(double) * imax * R));
  CK(dmalloc(&c->dRstack, sizeof(double) * 8 * R * R));
  CK(dmalloc(&c->dQtop, sizeof(double) * 8 * R * R));
  CK(dmalloc(&c->dV, sizeof(double) * (imax + 8) * R));
  CK(dmalloc(&c->dtauv, sizeof(double) * 8 * R));
  CK(dmalloc(&c->dinner, sizeof(double) * 4));
  CK(dmalloc(&c->dMpinv, sizeof(double) * R * R));
  CK(dmalloc(&c->dQ1, sizeof(double) * imax * R));
  CK(dmalloc(&c->dGp, sizeof(double) * ((imax + 255) / 256 + 1) * R * R));
  CK(dmalloc(&c->dinnerp, sizeof(double) * ((imax + 255) / 256 + 1)));
  CK(dmalloc(&c->dR1, sizeof(double) * R * R));
  CK(dmalloc(&c->dR2, sizeof(double) * R * R));
  {
    const char* f = getenv("CPQR_FACTOR_QR");
    c->factor_qr_mode = (f && std::string(f) == "householder") ? 1 : 0;
  }
  c->wp_elems = (size_t)imax * R * kQ0MaxSlices;
  CK(dmalloc(&c->dWp, sizeof(double) * c->wp_elems));
  CK(dmalloc(&c->dq0cnt, sizeof(unsigned) * ((imax + 7) / 8 + 1)));
  CK(cudaMemset(c->dq0cnt, 0, sizeof(unsigned) * ((imax + 7) / 8 + 1)));
  CK(dmalloc(&c->dnX2, sizeof(double) * 4));
  CK(dmalloc(&c->dfit, sizeof(double) * 4));
  {  // reduction scratch: k_solve_rows writes ceil(I_n / BT) x (RB + 1) partials (any I_n <= imax);
     // k_sumsq / k_resid use the first sms * 4 slots and dred[4096] (never concurrently)
    const int RB = rb_for(R), BT = RB > 16 ? 64 : 128;
    c->dred_elems = std::max<size_t>(8192, (size_t)((imax + BT - 1) / BT) * (RB + 1) + 64);
    CK(dmalloc(&c->dred, sizeof(double) * c->dred_elems));
  }
  CK(dmalloc(&c->dflags, sizeof(unsigned) * 4));
  CK(cudaMemset(c->dflags, 0, sizeof(unsigned) * 4));
  CK(cudaMallocHost(&c->hpin, sizeof(double) * 64));
  // staircase row order for K2: sort KB rows of R^{N-1} by (level, index).  Short modes (mixed-radix
  // V_n) and V_n beyond 2^28 rows use the CholeskyQR path only: no K2.
  if (!c->short_modes && J <= (1ll << 28)) {
    std::vector<int> perm(J);
    std::vector<int> lvl(J);
    for (int64_t j = 0; j < J; ++j) {
      int64_t x = j;
      int l = 0;
      for (int m = 0; m < N - 1; ++m) { l = std::max<int>(l, (int)(x % R)); x /= R; }
      lvl[j] = l;
      perm[j] = (int)j;
    }
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return lvl[a] < lvl[b]; });
    CK(dmalloc(&c->dperm, sizeof(int) * J));
    CK(cudaMemcpy(c->dperm, perm.data(), sizeof(int) * J, cudaMemcpyHostToDevice));
    int64_t packed = 0;
    for (int cc = 1; cc <= R; ++cc) {
      int64_t p = 1;
      for (int m = 0; m < N - 1; ++m) p *= cc;
      packed += p;
    }
    const size_t bytes = packed * sizeof(double);
    if (bytes <= 200 * 1024) {
      c->kr_smem = (int)bytes;
      CK(cudaFuncSetAttribute(k_kr_qr2, cudaFuncAttributeMaxDynamicSharedMemorySize, c->kr_smem));
    } else {
      c->kr_smem = 0;
      CK(dmalloc(&c->dKrWork, bytes));
    }
  }
  {  // high rank: V_n QR by the multi-CTA CholeskyQR2 (see launch_kr_qr)
    const char* v = getenv("CPQR_VN_QR");  // "cq" / "householder" force the choice
    // every mode above R^{N-1} R = 2e5 (the one-CTA K2 dominates the sweep); from 5e4, inline, in the
    // dimension tree's modes without an X pass, which cannot hide K2 (see mode_update)
    // (at world > 1 the V_n QR is replicated and must hide behind a p-times shorter pass: the
    // one-CTA K2 still does on C5 at p = 8, while C3 gains from CPQR_VN_QR=cq -- the multi-CTA
    // CholeskyQR2 cannot co-run with the stream grid and is exposed)
    c->vn_cq_always = c->short_modes || !c->dperm || (v ? std::string(v) == "cq" : (J * R >= 200000));
    {  // tree modes without an X pass run the V_n QR inline (CholeskyQR2); CPQR_VN_TREE=0/1 overrides
      const char* t = getenv("CPQR_VN_TREE");
      // the one-launch cluster CholeskyQR2 (k_cq_compact) takes V_n up to 8 CTAs x 512 rows (R <= 16)
      // or x 256 rows (R <= 32): inline it is cheaper than the exposed K2 in every measured config
      // (C2-C5 tree +2..14 %); larger V_n take the multi-kernel CholeskyQR2 from R^{N-1} R = 5e4
      const bool compact_ok = J <= 8 * (R <= 16 ? 512 : 256);
      c->vn_cq_tree = !v && c->tree && (t ? atoi(t) == 1 : (compact_ok || J * R >= 50000));
    }
    // tree QR of V_n (vn_tree.cuh): CPQR_VN_QR=tree; N >= 3, not with short modes
    c->vn_krtree = !c->short_modes && N >= 3 && v && std::string(v) == "tree";
    if (c->vn_krtree) {
      c->vn_cq_always = c->vn_cq_tree = false;
      const int h = c->tree_h;
      int64_t Jh = 1, Jl = 1;
      for (int i = 0; i < N - h; ++i) Jh *= R;
      for (int i = 0; i < h; ++i) Jl *= R;
      CK(dmalloc(&c->dTrP[0], sizeof(double) * Jh * R));
      CK(dmalloc(&c->dTrP[1], sizeof(double) * Jl * R));
      CK(dmalloc(&c->dTrS[0], sizeof(double) * R * R));
      CK(dmalloc(&c->dTrS[1], sizeof(double) * R * R));
      CK(dmalloc(&c->dTrPa, sizeof(double) * std::max(Jh, Jl) * R));
      CK(dmalloc(&c->dTrPb, sizeof(double) * std::max(Jh, Jl) * R));
      CK(dmalloc(&c->dTrT, sizeof(double) * J * R));
      if (R > 16) CK(dmalloc(&c->dTrQ, sizeof(double) * R * R * R));
      CK(cudaFuncSetAttribute(k_vn_tree<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vn_tree_smem(R)));
      CK(cudaFuncSetAttribute(k_vn_tree<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vn_tree_smem(R)));
      CK(cudaFuncSetAttribute(k_vn_tree<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vn_tree_smem(R)));
    }
    c->vn_cq = c->vn_cq_always || c->vn_cq_tree || (c->overlap && J <= 512);
    c->vnJ = J;
    if (c->vn_cq) {
      CK(dmalloc(&c->dVn, sizeof(double) * J * R));
      CK(dmalloc(&c->dVq1, sizeof(double) * J * R));
      CK(dmalloc(&c->dVgp, sizeof(double) * ((J + 255) / 256 + 1) * R * R));
      CK(dmalloc(&c->dVr1, sizeof(double) * R * R));
      CK(dmalloc(&c->dVr2, sizeof(double) * R * R));
      if (c->short_modes) {
        CK(dmalloc(&c->dVrs, sizeof(double) * R * R));
        CK(dmalloc(&c->dVrp, sizeof(double) * R * R));
      }
    }
  }
  {  // first-level Gram sums of the multi-kernel CholeskyQR beyond 1024 row blocks (cq_reduced)
    const int64_t nbmax = std::max<int64_t>((imax + 255) / 256, c->vn_cq ? (J + 255) / 256 : 0);
    if (nbmax > 1024) CK(dmalloc(&c->dGp2, sizeof(double) * 1025 * R * R));
  }
  // PEER ranks need no communicator; with an id they get one (cpqr_debug_mode's Y collectives)
  if ((c->opt.world > 1 && !c->local && (!c->peer || have_id)) || nccl1) {
    ncclUniqueId id;
    std::memcpy(&id, c->opt.nccl_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&c->comm, c->opt.world, id, c->opt.rank);
    if (r != ncclSuccess) return fail(c, CPQR_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_destroy(cpqr_ctx* c) {
  if (!c) return CPQR_OK;
  cudaSetDevice(c->opt.device);
  if (c->st) cudaStreamSynchronize(c->st);
  {
    size_t which = 0;
    if (const size_t bad = canary_violations(&which))
      fprintf(stderr, "cpqr_destroy: CPQR_CANARY: %zu guard bytes overwritten (first: block of %zu bytes)\n", bad, which);
  }
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->gexecG) cudaGraphExecDestroy(c->gexecG);
  if (c->dfitc) dfree(c->dfitc);
  if (c->comm) ncclCommDestroy(c->comm);
  for (int r = 0; r < kMaxWorld; ++r) {
    if (!c->win_base[r]) continue;
    if (c->win_mapped[r]) cudaIpcCloseMemHandle(c->win_base[r]);
    else cudaFree(c->win_base[r]);
  }
  dfree(c->dpushcnt);
  for (int k = 0; k < kMaxN; ++k) {
    dfree(c->dA[k]); dfree(c->dQ[k]); dfree(c->dRk[k]); dfree(c->dG[k]);
    dfree(c->dQt[k]); dfree(c->dAt[k]);
  }
  if (c->side) cudaStreamDestroy(c->side);
  if (c->tl) cudaStreamDestroy(c->tl);
  for (int k = 0; k < kMaxN; ++k) {
    if (c->evY[k]) cudaEventDestroy(c->evY[k]);
    if (c->evQ[k]) cudaEventDestroy(c->evQ[k]);
    if (c->evK[k]) cudaEventDestroy(c->evK[k]);
  }
  if (c->dY) dfree(c->dY);
  if (c->evf) cudaEventDestroy(c->evf);
  if (c->evj) cudaEventDestroy(c->evj);
  double* ps[] = {c->dQ1, c->dGp, c->dinnerp, c->dR1, c->dR2, c->dMpinv, c->dRstack, c->dQtop, c->dV, c->dtauv, c->dinner, c->dlam, c->dQ0, c->dR0, c->dW, c->dnX2p, c->dSk, c->dWp, c->dAhat, c->buf[0], c->buf[1],
                  c->dPart, c->dKrWork, c->dnX2, c->dfit, c->dfits, c->dred,
                  c->dVn, c->dVq1, c->dVgp, c->dVr1, c->dVr2, c->dVrs, c->dVrp, c->dGp2,
                  c->dTrP[0], c->dTrP[1], c->dTrS[0], c->dTrS[1], c->dTrPa, c->dTrPb, c->dTrT, c->dTrQ};
  for (double* p : ps) if (p) dfree(p);
  if (c->dperm) dfree(c->dperm);
  if (c->dflags) dfree(c->dflags);
  if (c->dq0cnt) dfree(c->dq0cnt);
  if (c->dKtP) dfree(c->dKtP);
  if (c->dSkCnt) dfree(c->dSkCnt);
  if (c->dZ) dfree(c->dZ);
  for (int k = 0; k < kMaxN; ++k) if (c->dKtB[k]) dfree(c->dKtB[k]);
  if (c->dKtLam) dfree(c->dKtLam);
  if (c->dKtM) dfree(c->dKtM);
  if (c->dKtC) dfree(c->dKtC);
  for (int q = 0; q < kMaxWorld; ++q) {
    Slab& sl = c->slabs[q];
    if (sl.Xown) dfree(sl.Xown);
    if (sl.dTree) dfree(sl.dTree);
    if (sl.dWloc) dfree(sl.dWloc);
  }
  if (c->hpin) cudaFreeHost(c->hpin);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (cudaEvent_t e : c->evp) cudaEventDestroy(e);
  for (auto& e : c->tev) cudaEventDestroy(e.first);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
  return CPQR_OK;
}

// one slab's tensor: borrowed in place, or copied into a slab-owned buffer; its partial ||X||^2
static cpqr_status set_slab(cpqr_ctx* c, Slab& sl, const double* x, int mem, double* nx2_out) {
  const size_t bytes = sizeof(double) * sl.numel;
  if (c->pad1) {
    // odd I_1: every kind of input is copied into the slab-owned buffer with mode 1 padded to even
    // (the pad row stays zero: written once here, never touched by the row copies)
    const int64_t I = c->tdims[0], D = c->dims[0], rows = sl.numel / D;
    if (sl.Xown_elems < (size_t)sl.numel) {
      if (sl.Xown) dfree(sl.Xown);
      sl.Xown = nullptr;
      if (dmalloc(&sl.Xown, bytes) != cudaSuccess) return fail(c, CPQR_ENOMEM, "tensor (%zu bytes)", bytes);
      sl.Xown_elems = sl.numel;
    }
    CK(cudaMemsetAsync(sl.Xown, 0, bytes, c->st));
    const double* src = x;
    double* stage = nullptr;
    if (mem == CPQR_MEM_HOST) {  // one contiguous H2D copy, then the padding on the device
      if (dmalloc(&stage, sizeof(double) * I * rows) != cudaSuccess)
        return fail(c, CPQR_ENOMEM, "tensor staging (%zu bytes)", sizeof(double) * (size_t)(I * rows));
      CK(cudaMemcpyAsync(stage, x, sizeof(double) * I * rows, cudaMemcpyHostToDevice, c->st));
      src = stage;
    }
    k_pad_rows<<<c->sms * 8, 256, 0, c->st>>>(src, I, D, rows, sl.Xown);
    CKL();
    if (stage) {
      CK(cudaStreamSynchronize(c->st));
      dfree(stage);
    }
    sl.X = sl.Xown;
  } else if (mem == CPQR_MEM_DEVICE_BORROW) {
    if (sl.Xown) { dfree(sl.Xown); sl.Xown = nullptr; sl.Xown_elems = 0; }
    sl.X = x;
  } else {
    if (sl.Xown_elems < (size_t)sl.numel) {
      if (sl.Xown) dfree(sl.Xown);
      sl.Xown = nullptr;
      if (dmalloc(&sl.Xown, bytes) != cudaSuccess) return fail(c, CPQR_ENOMEM, "tensor (%zu bytes)", bytes);
      sl.Xown_elems = sl.numel;
    }
    CK(cudaMemcpyAsync(sl.Xown, x, bytes, mem == CPQR_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->st));
    sl.X = sl.Xown;
  }
  const int grid = c->sms * 4;
  k_sumsq_partial<<<grid, 256, 0, c->st>>>(sl.X, sl.numel, c->dred);
  CKL();
  k_sum_final<<<1, 256, 0, c->st>>>(c->dred, grid, nx2_out);
  CKL();
  sl.have = true;
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_set_tensor(cpqr_ctx* c, const double* x, int64_t b, int64_t e, int mem) {
  if (!c || !x) return c ? fail(c, CPQR_EINVAL, "null tensor") : CPQR_EINVAL;
  if (mem != CPQR_MEM_HOST && mem != CPQR_MEM_DEVICE_COPY && mem != CPQR_MEM_DEVICE_BORROW)
    return fail(c, CPQR_EINVAL, "bad mem kind %d", mem);
  if (c->short_modes)
    return fail(c, CPQR_EINVAL, "a dense tensor needs I_k >= R in every mode (short modes: Kruskal input only)");
  // which slabs [b, e) covers: this rank's, or (virtual ranks) one rank's or all of them
  int q0 = -1, q1 = -1;
  if (c->local && b == 0 && e == c->dims[c->N - 1]) {
    q0 = 0;
    q1 = c->nslab;
  } else {
    for (int q = 0; q < c->nslab; ++q)
      if (b == c->slabs[q].b && e == c->slabs[q].e) { q0 = q; q1 = q + 1; }
  }
  if (q0 < 0)
    return fail(c, CPQR_EINVAL, "slab [%lld,%lld) is not %s (rank %d/%d%s)", (long long)b, (long long)e,
                c->local ? "[0, I_N) or one virtual rank's slab" : "this rank's slab", c->opt.rank, c->opt.world,
                c->local ? ", virtual ranks" : "");
  TRY(begin_call(c));
  CK(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned) * 4, c->st));
  c->flags = 0;
  const int64_t slice = prod(c->tdims, 0, c->N - 1);  // elements per index of the last mode (caller's layout)
  for (int q = q0; q < q1; ++q) {
    const double* xs = x + (c->slabs[q].b - b) * slice;
    TRY(set_slab(c, c->slabs[q], xs, mem, c->nslab > 1 ? c->dnX2p + q : c->dnX2));
  }
  bool all = true;
  for (int q = 0; q < c->nslab; ++q) all = all && c->slabs[q].have;
  c->kt = false;
  c->graph_valid = false;
  c->have_tensor = all;
  if (all) {
    if (c->peer) {  // ||X||^2 = rank-order sum of the slab partials through the peer windows
      if (!c->peers_connected) return fail(c, CPQR_ESTATE, "CPQR_COMM_PEER: cpqr_peer_connect first");
      const double* src[kMaxWorld];
      for (int q = 0; q < c->nslab; ++q) src[q] = c->nslab > 1 ? c->dnX2p + q : c->dnX2;
      TRY(peer_exchange(c, src, 1, 0, c->dnX2));
    } else if (c->nslab > 1) {  // virtual ranks: ||X||^2 = rank-order sum of the slab partials
      k_sum_final<<<1, 256, 0, c->st>>>(c->dnX2p, c->nslab, c->dnX2);
      CKL();
    } else if (c->comm) {
      CN(ncclAllReduce(c->dnX2, c->dnX2, 1, ncclDouble, ncclSum, c->comm, c->st));
    }
    TRY(build_plans(c));
  }
  if (c->peer && all) {  // a rank missing from the ||X||^2 exchange
    unsigned fl = 0;
    CK(cudaMemcpyAsync(&fl, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->st));
    TRY(end_call(c));
    if (fl & FLAG_PEER_TIMEOUT) {
      c->have_tensor = false;
      return fail(c, CPQR_ENCCL, "peer exchange of ||X||^2: a rank did not arrive within %llu ms",
                  (unsigned long long)(c->peer_timeout_ns / 1000000ull));
    }
    return CPQR_OK;
  }
  return end_call(c);
}

CPQR_API cpqr_status cpqr_batched_qr(int P, const int64_t* dims, int R, const double* X, const double* A0,
                                     int max_iters, double tol, double* A, double* lam, double* fits,
                                     int* iters, void* stream) {
  return cpqr_batched(P, dims, R, CPQR_QR, -1.0, X, A0, max_iters, tol, A, lam, fits, iters, stream);
}

CPQR_API cpqr_status cpqr_batched(int P, const int64_t* dims, int R, int variant, double tau, const double* X,
                                  const double* A0, int max_iters, double tol, double* A, double* lam,
                                  double* fits, int* iters, void* stream) {
  if (P < 0 || !dims || !X || !A0 || !A || !lam || !fits || !iters || max_iters < 1) return CPQR_EINVAL;
  if (variant < CPQR_NE || variant > CPQR_PINV) return CPQR_EINVAL;
  if (R < 1 || R > kBatMaxR) return CPQR_EINVAL;
  for (int k = 0; k < 3; ++k)
    if (dims[k] < R || dims[k] > kBatMaxI) return CPQR_EINVAL;
  if (dims[0] * dims[1] * R > kBatTBuf || dims[1] * dims[2] * R > kBatTBuf || R * R > kBatMaxI) return CPQR_EINVAL;
  if (P == 0) return CPQR_OK;
  BatchedArgs a{};
  a.X = X; a.A0 = A0; a.R = R; a.max_iters = max_iters; a.tol = tol;
  for (int k = 0; k < 3; ++k) a.I[k] = (int)dims[k];
  a.A = A; a.lam = lam; a.fits = fits; a.iters = iters;
  a.variant = variant; a.tau = tau;
  const size_t smem = (size_t)(kBatTBuf + 64 * 64 + 3 * 64 * 8 + 3 * 64 + 64 * 8 + 64 + 2 * 64 * 8 +
                               2 * 64 + 2 * 72 + 2 * 64) * sizeof(double);
  if (cudaFuncSetAttribute(k_batched_cpqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return CPQR_ECUDA;
  k_batched_cpqr<<<P, 256, smem, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? CPQR_OK : CPQR_ECUDA;
}

CPQR_API cpqr_status cpqr_set_ktensor(cpqr_ctx* c, int S, const double* lam, const double* const* B) {
  if (!c || !B || S < 1) return c ? fail(c, CPQR_EINVAL, "Kruskal input: S >= 1 and B required") : CPQR_EINVAL;
  if (c->opt.world > 1) return fail(c, CPQR_EINVAL, "Kruskal input is single-GPU (the factors are replicated)");
  if (c->opt.fit_mode == CPQR_FIT_DIRECT && S + c->R > kKtResidMaxSR)
    return fail(c, CPQR_EINVAL, "Kruskal DIRECT fit: S + R = %d > %d", S + c->R, kKtResidMaxSR);
  for (int k = 0; k < c->N; ++k)
    if (!B[k]) return fail(c, CPQR_EINVAL, "B[%d] is NULL", k);
  TRY(begin_call(c));
  const int N = c->N, R = c->R;
  if (S != c->ktS) {
    for (int k = 0; k < N; ++k) { if (c->dKtB[k]) dfree(c->dKtB[k]); c->dKtB[k] = nullptr; }
    if (c->dKtLam) dfree(c->dKtLam);
    if (c->dKtM) dfree(c->dKtM);
    if (c->dKtC) dfree(c->dKtC);
    c->dKtLam = c->dKtM = c->dKtC = nullptr;
    for (int k = 0; k < N; ++k) CK(dmalloc(&c->dKtB[k], sizeof(double) * c->dims[k] * S));
    CK(dmalloc(&c->dKtLam, sizeof(double) * S));
    CK(dmalloc(&c->dKtM, sizeof(double) * S * R));
    const int mx = std::max(R, S);
    c->ktC_elems = (size_t)N * mx * mx;
    CK(dmalloc(&c->dKtC, sizeof(double) * c->ktC_elems));
    c->ktS = S;
  }
  {  // k_kt_m chunk partials of the largest V_n (never allocated inside a graph capture)
    size_t need = 0;
    for (int n = 0; n < N; ++n) {
      int64_t J = 1;
      for (int k = 0; k < N; ++k) if (k != n) J *= c->vq[k];
      const int nc = kt_m_chunks(c, J, S);
      if (nc > 1) need = std::max(need, (size_t)S * nc * R);
    }
    if (need > c->ktP_elems) {
      if (c->dKtP) dfree(c->dKtP);
      c->dKtP = nullptr;
      CK(dmalloc(&c->dKtP, sizeof(double) * need));
      c->ktP_elems = need;
    }
  }
  for (int k = 0; k < N; ++k) {  // (short modes: I_k rows of the max(I_k, R)-row zero-padded array)
    if (c->tdims[k] != c->dims[k]) CK(cudaMemsetAsync(c->dKtB[k], 0, sizeof(double) * c->dims[k] * S, c->st));
    CK(cudaMemcpy2DAsync(c->dKtB[k], sizeof(double) * c->dims[k], B[k], sizeof(double) * c->tdims[k],
                         sizeof(double) * c->tdims[k], S, cudaMemcpyHostToDevice, c->st));
  }
  std::vector<double> ones(S, 1.0);
  CK(cudaMemcpyAsync(c->dKtLam, lam ? lam : ones.data(), sizeof(double) * S, cudaMemcpyHostToDevice, c->st));
  int modes[kMaxN];
  for (int k = 0; k < N; ++k) modes[k] = k;
  const double* Bc[kMaxN];
  for (int k = 0; k < N; ++k) Bc[k] = c->dKtB[k];
  TRY(kt_cross(c, modes, N, Bc, S, Bc, S, c->dKtC));  // G_k = B_k^T B_k
  k_kt_norm2<<<1, 256, 0, c->st>>>(c->dKtC, N, S, c->dKtLam, c->dnX2);
  CKL();
  CK(cudaStreamSynchronize(c->st));  // the host arrays may go away after return
  c->have_tensor = true;
  c->kt = true;
  c->graph_valid = false;
  return end_call(c);
}

static cpqr_status upload_factors(cpqr_ctx* c, const double* const* A, const double* lam) {
  const int R = c->R;
  // a new run: clear the sticky device flags (FLAG_NONFINITE of a diverged run included) and the
  // host-side OR of the condition flags
  CK(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned) * 4, c->st));
  c->flags = 0;
  for (int k = 0; k < c->N; ++k) {
    if (!A[k]) {
      if (ne_family(c->variant) && k != 0) return fail(c, CPQR_EINVAL, "NE needs A[%d]", k);
      if (k != 0) return fail(c, CPQR_EINVAL, "A[%d] is NULL", k);
      continue;
    }
    if (c->tdims[k] == c->dims[k]) {
      CK(cudaMemcpyAsync(c->dA[k], A[k], sizeof(double) * c->dims[k] * R, cudaMemcpyHostToDevice, c->st));
    } else {  // a short mode: I_k rows into the zero-padded max(I_k, R)-row array
      CK(cudaMemsetAsync(c->dA[k], 0, sizeof(double) * c->dims[k] * R, c->st));
      CK(cudaMemcpy2DAsync(c->dA[k], sizeof(double) * c->dims[k], A[k], sizeof(double) * c->tdims[k],
                           sizeof(double) * c->tdims[k], R, cudaMemcpyHostToDevice, c->st));
    }
    if (ne_family(c->variant)) {
      k_gram<<<1, 1024, 0, c->st>>>(c->dA[k], (int)c->dims[k], R, c->dG[k]);
      CKL();
      k_transpose_pad<<<64, 256, 0, c->st>>>(c->dA[k], c->dims[k], (int)c->dims[k], R, c->RQ, c->dAt[k]);
      CKL();
    } else {
      TRY(launch_factor_qr(c, c->dA[k], (int)c->dims[k], c->dQ[k], c->dQt[k], c->dRk[k], false));
    }
  }
  std::vector<double> l(R, 1.0);
  if (lam) for (int r = 0; r < R; ++r) l[r] = lam[r];
  CK(cudaMemcpyAsync(c->dlam, l.data(), sizeof(double) * R, cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->have_factors = true;
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_set_factors(cpqr_ctx* c, const double* const* A, const double* lam) {
  if (!c || !A) return c ? fail(c, CPQR_EINVAL, "null factors") : CPQR_EINVAL;
  TRY(begin_call(c));
  TRY(upload_factors(c, A, lam));
  return end_call(c);
}

CPQR_API cpqr_status cpqr_init_factors(cpqr_ctx* c, uint64_t seed) {
  if (!c) return CPQR_EINVAL;
  std::vector<std::vector<double>> h(c->N);
  std::vector<const double*> p(c->N);
  uint64_t ctr = 0;
  for (int k = 0; k < c->N; ++k) {
    h[k].resize(c->tdims[k] * c->R);
    for (auto& v : h[k]) v = normal_at(seed, ctr++);
    p[k] = h[k].data();
  }
  return cpqr_set_factors(c, p.data(), nullptr);
}

CPQR_API cpqr_status cpqr_sweep(cpqr_ctx* c, int nsweeps, double* fits) {
  if (!c || nsweeps < 0) return CPQR_EINVAL;
  if (!c->have_tensor || !c->have_factors) return fail(c, CPQR_ESTATE, "tensor/factors not set");
  TRY(begin_call(c));
  TRY(ensure_fits(c, std::max(1, nsweeps)));
  const bool graph = c->opt.use_graph && !c->opt.profile;
  CK(cudaMemsetAsync(c->dfitc, 0, sizeof(unsigned), c->st));
  for (int s = 0; s < nsweeps;) {
    if (graph) {
      if (!c->graph_valid) {
        TRY(capture_sweeps(c, 1, &c->gexec, &c->launches_per_sweep));
        if (c->gsw > 1) TRY(capture_sweeps(c, c->gsw, &c->gexecG, &c->launches_G));
        c->graph_valid = true;
      }
      if (c->gsw > 1 && nsweeps - s >= c->gsw) {
        CK(cudaGraphLaunch(c->gexecG, c->st));
        c->launch_count += c->launches_G;
        s += c->gsw;
      } else {
        CK(cudaGraphLaunch(c->gexec, c->st));
        c->launch_count += c->launches_per_sweep;
        ++s;
      }
    } else {
      const int64_t before = c->launch_count;
      static const bool sync_modes = getenv("CPQR_SYNC_MODES") != nullptr;  // debugging
      if (sync_modes) {
        for (int n = 0; n < c->N; ++n) {
          TRY(mode_update(c, n, n == c->N - 1));
          CK(cudaDeviceSynchronize());
        }
        if (c->opt.fit_mode == CPQR_FIT_DIRECT) TRY(direct_fit(c));
        k_store_fit<<<1, 32, 0, c->st>>>(c->dfit, c->dfits, c->dfitc, c->fits_cap);
        CKL();
      } else {
        TRY(one_sweep(c));
      }
      trace_dump(c);
      c->launches_per_sweep = c->launch_count - before;
      ++s;
    }
  }
  if (nsweeps > 0) {
    std::vector<double> hf(nsweeps);
    CK(cudaMemcpyAsync(hf.data(), c->dfits, sizeof(double) * nsweeps, cudaMemcpyDeviceToHost, c->st));
    unsigned fl = 0;
    CK(cudaMemcpyAsync(&fl, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->st));
    TRY(end_call(c));
    if (c->variant != CPQR_QR) fl &= ~(unsigned)FLAG_ILLCOND_R0;
    c->flags |= fl;
    c->last_fit = hf[nsweeps - 1];
    if (fits) std::memcpy(fits, hf.data(), sizeof(double) * nsweeps);
    if (fl & FLAG_PEER_TIMEOUT)
      return fail(c, CPQR_ENCCL, "peer exchange: a rank did not arrive within %llu ms (CPQR_PEER_TIMEOUT_MS)",
                  (unsigned long long)(c->peer_timeout_ns / 1000000ull));
    if (fl & FLAG_NONFINITE) return fail(c, CPQR_EDIVERGED, "non-finite factor");
    size_t which = 0;
    if (const size_t bad = canary_violations(&which))
      return fail(c, CPQR_ECUDA, "CPQR_CANARY: %zu guard bytes overwritten (first: block of %zu bytes)", bad, which);
    return CPQR_OK;
  }
  return end_call(c);
}

CPQR_API cpqr_status cpqr_get_factors(cpqr_ctx* c, double* const* A_out, double* lam) {
  if (!c) return CPQR_EINVAL;
  if (!c->have_factors) return fail(c, CPQR_ESTATE, "factors not set");
  TRY(begin_call(c));
  if (A_out)
    for (int k = 0; k < c->N; ++k)
      if (A_out[k])
        CK(cudaMemcpy2DAsync(A_out[k], sizeof(double) * c->tdims[k], c->dA[k], sizeof(double) * c->dims[k],
                             sizeof(double) * c->tdims[k], c->R, cudaMemcpyDeviceToHost, c->st));
  if (lam) CK(cudaMemcpyAsync(lam, c->dlam, sizeof(double) * c->R, cudaMemcpyDeviceToHost, c->st));
  return end_call(c);
}

CPQR_API cpqr_status cpqr_get_fit(cpqr_ctx* c, double* fit) {
  if (!c || !fit) return CPQR_EINVAL;
  *fit = c->last_fit;
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_get_flags(cpqr_ctx* c, uint32_t* f) {
  if (!c || !f) return CPQR_EINVAL;
  *f = c->flags & 0xffu;
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_get_profile(cpqr_ctx* c, cpqr_profile* p, int reset) {
  if (!c || !p) return CPQR_EINVAL;
  *p = c->prof;
  // algorithmic bytes / flops of the stream-X passes of one sweep:
  // bytes = passes * 8 * numel (X read once per pass: N passes, or 2 with the dimension tree);
  // flops = the first TTM of each pass (+ the fused second contraction of the slice kernels)
  // (summed over the slabs this context runs)
  double fl = 0.0, by = 0.0;
  for (int q = 0; q < c->nslab && !c->kt && c->plans_valid; ++q) {
    const Slab& sl = c->slabs[q];
    for (int n = 0; n < c->N; ++n) {
      const Plan& pl = sl.plans[n];
      if (pl.steps.empty() || pl.steps[0].in != sl.X) continue;  // passes over X only
      const TtmStep& s = pl.steps[0];
      const double R = c->R, nel = (double)sl.numel;
      by += 8.0 * nel;
      if (s.kind == 2 || s.kind == 6 || s.kind == 8) fl += 2.0 * nel * R + 2.0 * (nel / (double)s.I1) * R * R;
      else if (s.kind == 10) fl += 2.0 * nel * R + 2.0 * (nel / (double)s.I) * R * R;
      else fl += 2.0 * nel * R;
    }
  }
  p->bytes0 = by;
  p->flops0 = fl;
  p->launches_total = c->launch_count;
  if (reset) std::memset(&c->prof, 0, sizeof c->prof);
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_get_timings(cpqr_ctx* c, double* ms) {
  if (!c || !ms) return CPQR_EINVAL;
  for (int i = 0; i < 7; ++i) ms[i] = c->prof.ms[i];
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_launches_per_sweep(cpqr_ctx* c, int64_t* n) {
  if (!c || !n) return CPQR_EINVAL;
  *n = c->launches_per_sweep;
  return CPQR_OK;
}

// device scratch freed on every exit path of the debug entry points
struct DevScratch {
  std::vector<void*> ptrs;
  template <typename T>
  cudaError_t alloc(T** p, size_t bytes) {
    cudaError_t e = dmalloc(p, bytes);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
  ~DevScratch() {
    for (void* p : ptrs) dfree(p);
  }
};

static int64_t max_dim(const cpqr_ctx* c) {
  int64_t m = 0;
  for (int k = 0; k < c->N; ++k) m = std::max(m, c->dims[k]);
  return m;
}

CPQR_API cpqr_status cpqr_debug_mode(cpqr_ctx* c, int n, const double* const* Qo, double* Y_out,
                                     double* Q0_out, double* R0_out, double* W_out) {
  if (!c) return CPQR_EINVAL;
  if (n < 0 || n >= c->N) return fail(c, CPQR_EINVAL, "mode %d", n);
  if (!c->have_tensor || !c->have_factors) return fail(c, CPQR_ESTATE, "tensor/factors not set");
  if (ne_family(c->variant)) return fail(c, CPQR_EINVAL, "debug_mode is for the QR/SVD variants");
  if (c->kt) return fail(c, CPQR_EINVAL, "debug_mode needs a dense tensor (Kruskal input forms no Y)");
  TRY(begin_call(c));
  const int R = c->R, N = c->N;
  DevScratch sc;
  std::vector<double*> tmpQ(N, nullptr), tmpQt(N, nullptr);
  for (int k = 0; k < N; ++k) {
    if (Qo && k != n && Qo[k]) {
      CK(sc.alloc(&tmpQ[k], sizeof(double) * c->dims[k] * R));
      CK(sc.alloc(&tmpQt[k], sizeof(double) * c->dims[k] * c->RQ));
      if (c->tdims[k] != c->dims[k]) CK(cudaMemsetAsync(tmpQ[k], 0, sizeof(double) * c->dims[k] * R, c->st));
      CK(cudaMemcpy2DAsync(tmpQ[k], sizeof(double) * c->dims[k], Qo[k], sizeof(double) * c->tdims[k],
                           sizeof(double) * c->tdims[k], R, cudaMemcpyHostToDevice, c->st));
      k_transpose_pad<<<64, 256, 0, c->st>>>(tmpQ[k], c->dims[k], (int)c->dims[k], R, c->RQ, tmpQt[k]);
      CKL();
    }
  }
  CK(cudaEventRecord(c->evf, c->st));
  CK(cudaStreamWaitEvent(c->side, c->evf, 0));
  c->vn_mode_cq = c->vn_cq_always;
  c->kr_standalone = true;
  const cpqr_status kst = launch_kr_qr(c, n);
  c->kr_standalone = false;
  TRY(kst);
  CK(cudaEventRecord(c->evj, c->side));
  // per slab: Multi-TTM (fresh from X, the tree buffer holds no valid half intermediate outside a
  // sweep), Q0 apply; the debug Y is summed over the ranks (n < N-1) or gathered (n == N-1)
  double* yfull = nullptr;
  int64_t ylocal = 0, ytot = 0;
  const double* src[kMaxWorld];
  for (int q = 0; q < c->nslab; ++q) {
    PlanIn in{};
    fill_plan_in(c, c->slabs[q], in, n, tmpQ.data(), tmpQt.data());
    in.tree_fresh = true;
    Plan p;
    plan_mode(in, p, c->buf, c->dPart);
    TRY(run_plan(c, p));
    if (q == 0) CK(cudaStreamWaitEvent(c->st, c->evj, 0));
    TRY(launch_q0_apply(c, p, wloc(c, q), make_push(c, q)));
    src[q] = wloc(c, q);
    ylocal = (int64_t)p.Aa * p.In * p.Bb;
    if (Y_out) {
      ytot = (c->opt.world > 1 && n == N - 1) ? ylocal * c->opt.world : ylocal;
      if (!yfull) CK(sc.alloc(&yfull, sizeof(double) * ytot));
      if (!c->local) {
        CK(cudaMemcpyAsync(yfull, p.Y, sizeof(double) * ylocal, cudaMemcpyDeviceToDevice, c->st));
      } else if (n == N - 1) {
        CK(cudaMemcpyAsync(yfull + q * ylocal, p.Y, sizeof(double) * ylocal, cudaMemcpyDeviceToDevice, c->st));
      } else if (q == 0) {
        CK(cudaMemcpyAsync(yfull, p.Y, sizeof(double) * ylocal, cudaMemcpyDeviceToDevice, c->st));
      } else {
        RankPtrs rp{};
        rp.p[0] = yfull;
        rp.p[1] = p.Y;
        k_sum_ranks<<<(int)std::min<int64_t>((ylocal + 255) / 256, (int64_t)c->sms * 4), 256, 0, c->st>>>(rp, 2, ylocal, yfull);
        CKL();
      }
    }
  }
  TRY(combine_w(c, n, src, c->peer));
  if (Y_out && c->opt.world > 1 && !c->local && !c->comm)
    return fail(c, CPQR_EINVAL, "debug_mode: Y across CPQR_COMM_PEER ranks needs an NCCL id (pass Y_out = NULL)");
  if (Y_out && c->comm) {
    double* ycoll = nullptr;
    CK(sc.alloc(&ycoll, sizeof(double) * ytot));
    if (n == N - 1) CN(ncclAllGather(yfull, ycoll, (size_t)ylocal, ncclDouble, c->comm, c->st));
    else CN(ncclAllReduce(yfull, ycoll, (size_t)ylocal, ncclDouble, ncclSum, c->comm, c->st));
    yfull = ycoll;
  }
  std::vector<double> w((size_t)c->dims[n] * R);
  CK(cudaMemcpyAsync(w.data(), c->dW, sizeof(double) * w.size(), cudaMemcpyDeviceToHost, c->st));
  if (Y_out && n == 0 && c->tdims[0] != c->dims[0]) {  // mode 1 stored padded: drop the pad row of every fibre
    CK(cudaMemcpy2DAsync(Y_out, sizeof(double) * c->tdims[0], yfull, sizeof(double) * c->dims[0],
                         sizeof(double) * c->tdims[0], (size_t)(ytot / c->dims[0]), cudaMemcpyDeviceToHost, c->st));
  } else if (Y_out) {
    CK(cudaMemcpyAsync(Y_out, yfull, sizeof(double) * ytot, cudaMemcpyDeviceToHost, c->st));
  }
  int64_t J = 1;
  for (int k = 0; k < N - 1; ++k) J *= R;
  if (Q0_out) CK(cudaMemcpyAsync(Q0_out, c->dQ0, sizeof(double) * J * R, cudaMemcpyDeviceToHost, c->st));
  if (R0_out) CK(cudaMemcpyAsync(R0_out, c->dR0, sizeof(double) * R * R, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (W_out)
    for (int64_t i = 0; i < c->tdims[n]; ++i)
      for (int r = 0; r < R; ++r) W_out[i + c->tdims[n] * r] = w[i * R + r];
  return end_call(c);
}

CPQR_API cpqr_status cpqr_debug_plan(cpqr_ctx* c, int n, int slab, int64_t* info, int cap, int* nsteps) {
  if (!c || !info || !nsteps || cap < 0) return CPQR_EINVAL;
  if (n < 0 || n >= c->N || slab < 0 || slab >= c->nslab) return fail(c, CPQR_EINVAL, "mode %d / slab %d", n, slab);
  if (!c->plans_valid || c->kt) return fail(c, CPQR_ESTATE, "no dense tensor set");
  const Slab& sl = c->slabs[slab];
  const Plan& p = sl.plans[n];
  const int64_t R = c->R;
  int cnt = 0;
  auto put = [&](int64_t kind, int64_t modes, int64_t in, int64_t out, int64_t flops, int64_t xp) {
    if (cnt < cap) {
      int64_t* r = info + 6 * cnt;
      r[0] = kind; r[1] = modes; r[2] = in; r[3] = out; r[4] = flops; r[5] = xp;
    }
    ++cnt;
  };
  for (const TtmStep& s : p.steps) {
    const int64_t xp = (s.in == sl.X) ? 1 : 0;
    switch (s.kind) {
      case 0: case 4: case 9: put(s.kind, s.modes, s.A * s.I * s.B, s.A * R * s.B, 2 * s.A * s.I * s.B * R, xp); break;
      case 10:  // both contractions of the fused pass: over I (all B slices), then over B
        put(s.kind, s.modes, s.A * s.I * s.B, s.A * R * R, 2 * s.A * s.I * s.B * R + 2 * s.A * R * s.B * R, xp);
        break;
      case 1: case 5: put(s.kind, s.modes, (int64_t)s.I * s.F, R * s.F, 2 * (int64_t)s.I * s.F * R, xp); break;
      case 2: case 6: case 8:
        put(s.kind, s.modes, (int64_t)s.I1 * s.I2 * s.L, R * R * s.L,
            2 * (int64_t)s.I1 * s.I2 * s.L * R + 2 * R * (int64_t)s.I2 * s.L * R, xp);
        break;
      default: put(s.kind, 0, 0, 0, 0, 0); break;  // partial-sum fix-ups
    }
  }
  for (const DiagStep& d : p.diags) {
    int64_t tot = 1;
    for (int i = 0; i < d.nd; ++i) tot *= d.dims[i];
    put(100, 1 << d.mode, tot, tot / d.dims[d.k], 2 * tot, 0);
  }
  *nsteps = cnt;
  return CPQR_OK;
}

CPQR_API cpqr_status cpqr_debug_qr(cpqr_ctx* c, const double* A, int64_t m, double* Q, double* Rf) {
  if (!c || !A) return CPQR_EINVAL;
  if (m < c->R || m > max_dim(c))
    return fail(c, CPQR_EINVAL, "debug_qr: m = %lld outside [R, max(dims)] (context workspaces)", (long long)m);
  TRY(begin_call(c));
  const int R = c->R;
  DevScratch sc;
  double *dA = nullptr, *dQ = nullptr, *dR = nullptr, *dQt = nullptr;
  CK(sc.alloc(&dA, sizeof(double) * m * R));
  CK(sc.alloc(&dQ, sizeof(double) * m * R));
  CK(sc.alloc(&dR, sizeof(double) * R * R));
  CK(sc.alloc(&dQt, sizeof(double) * m * c->RQ));
  CK(cudaMemcpyAsync(dA, A, sizeof(double) * m * R, cudaMemcpyHostToDevice, c->st));
  TRY(launch_factor_qr(c, dA, (int)m, dQ, dQt, dR, false));
  if (Q) CK(cudaMemcpyAsync(Q, dQ, sizeof(double) * m * R, cudaMemcpyDeviceToHost, c->st));
  if (Rf) CK(cudaMemcpyAsync(Rf, dR, sizeof(double) * R * R, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return end_call(c);
}

CPQR_API cpqr_status cpqr_debug_svd_solve(cpqr_ctx* c, const double* R0, const double* W, int64_t m,
                                          double tau, double* Ahat, int* ntrunc) {
  if (!c || !R0 || !W || !Ahat) return CPQR_EINVAL;
  if (m < 1 || m > max_dim(c))
    return fail(c, CPQR_EINVAL, "debug_svd_solve: m = %lld outside [1, max(dims)]", (long long)m);
  TRY(begin_call(c));
  const int R = c->R;
  DevScratch sc;
  double *dW = nullptr, *dR0keep = nullptr;
  unsigned* dflkeep = nullptr;
  int* dnt = nullptr;
  CK(sc.alloc(&dW, sizeof(double) * m * R));
  CK(sc.alloc(&dR0keep, sizeof(double) * R * R));
  CK(sc.alloc(&dflkeep, sizeof(unsigned) * 4));
  CK(sc.alloc(&dnt, sizeof(int)));
  CK(cudaMemsetAsync(dnt, 0, sizeof(int), c->st));
  // the solve runs on the context's R0 / flag slots: save them and restore them afterwards, so a
  // debug call leaves the solver state untouched
  CK(cudaMemcpyAsync(dR0keep, c->dR0, sizeof(double) * R * R, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(dflkeep, c->dflags, sizeof(unsigned) * 4, cudaMemcpyDeviceToDevice, c->st));
  std::vector<double> wr((size_t)m * R);
  for (int64_t i = 0; i < m; ++i)
    for (int r = 0; r < R; ++r) wr[i * R + r] = W[i + m * r];
  CK(cudaMemcpyAsync(dW, wr.data(), sizeof(double) * m * R, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->dR0, R0, sizeof(double) * R * R, cudaMemcpyHostToDevice, c->st));
  cpqr_status st;
  {
    const double keep = c->opt.svd_tau;
    const int kv = c->variant;
    const bool kr = c->pinv_ready;
    c->opt.svd_tau = tau;
    c->variant = CPQR_SVD;
    st = launch_solve(c, dW, (int)m, false, dnt);
    c->opt.svd_tau = keep;
    c->variant = kv;
    c->pinv_ready = kr;
  }
  if (st == CPQR_OK) {
    CK(cudaMemcpyAsync(Ahat, c->dAhat, sizeof(double) * m * R, cudaMemcpyDeviceToHost, c->st));
    int nt = 0;
    CK(cudaMemcpyAsync(&nt, dnt, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (ntrunc) *ntrunc = nt;
  }
  cudaMemcpyAsync(c->dR0, dR0keep, sizeof(double) * R * R, cudaMemcpyDeviceToDevice, c->st);
  cudaMemcpyAsync(c->dflags, dflkeep, sizeof(unsigned) * 4, cudaMemcpyDeviceToDevice, c->st);
  CK(cudaStreamSynchronize(c->st));
  TRY(st);
  return end_call(c);
}
