/*
 * cpqr.h — C ABI of libcpqr: the per-mode least-squares hot path of QR-based CP-ALS
 * (arXiv 2112.10855, Alg. 2 "CP-ALS-QR"), its QR-SVD variant
 * and normal-equations CP-ALS (Alg. 1), on B200 (sm_100a).
 *
 * Conventions (DESIGN.md §Data layout, §Readings):
 *   - all arithmetic is IEEE fp64;
 *   - the dense tensor X (I_1 x ... x I_N) is column-major, mode 1 fastest (PAPER.md:109,
 *     Kolda-Bader unfolding, reading 1);
 *   - factor matrices A_n (I_n x R) are column-major with leading dimension I_n;
 *   - Khatri-Rao / Kronecker products use A_N (.) ... (.) A_1 (last factor's row fastest,
 *     PAPER.md:93-95), so V_n rows and Y_(n) columns are in Kolda-Bader order;
 *   - every thin QR returns diag(R) >= 0 (reading 6); lambda_r = ||Ahat(:,r)||_2 >= 0.
 *
 * Errors: every entry point returns a cpqr_status (0 = OK, > 0 = error).  No C++ exception
 * crosses the ABI.  cpqr_last_error() gives a human-readable message for the last failure on
 * a context.  A context is not thread-safe; distinct contexts are independent.
 * Ownership: the context owns all device workspaces, its streams and its NCCL communicator;
 * every pointer passed in is borrowed for the duration of the call only, except a tensor
 * given with CPQR_MEM_DEVICE_BORROW (kept until the next cpqr_set_tensor or cpqr_destroy).
 * Synchronisation: every call is synchronous with respect to the host on return (results
 * written to host buffers are valid), unless stated otherwise.  Device inputs must be complete
 * when a call is made: the context runs on its own non-blocking stream (or opt.stream) and does
 * not order itself after work the caller queued on other streams (the Python binding
 * synchronises torch's current stream before passing a CUDA tensor).
 */
#ifndef CPQR_H
#define CPQR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t cpqr_status;
enum {
  CPQR_OK = 0,
  CPQR_EINVAL = 1,     /* bad argument (N, dims, R, variant, NULL pointer, slab range, ...) */
  CPQR_ENOMEM = 2,     /* device allocation failed */
  CPQR_ECUDA = 3,      /* CUDA runtime error (message in cpqr_last_error) */
  CPQR_ENCCL = 4,      /* NCCL error, or a rank missing from a peer exchange (timeout) */
  CPQR_ESTATE = 5,     /* call out of order (no tensor / no factors yet) */
  CPQR_EDIVERGED = 6   /* a non-finite lambda appeared during the sweeps: the factors are then
                          non-finite (the remaining modes of the call ran on them); restore a
                          finite state with cpqr_set_factors / cpqr_init_factors, which clear
                          the condition */
};

/* Variant of the per-mode LS solve (substitution or SVD; Alg. 1: normal eqs):
 *   CPQR_NE   CP-ALS, Alg. 1: Ahat S_n = M_n by Cholesky (LU fallback, reading 18);
 *   CPQR_QR   CP-ALS-QR, Alg. 2: Ahat R0^T = W_n by back substitution;
 *   CPQR_SVD  CP-ALS-QR-SVD: Ahat = W_n (R0^T)^+ by the SVD of R0, svd_tau;
 *   CPQR_PINV CP-ALS-PINV: Alg. 1 with Ahat = M_n S_n^+, the SVD
 *             pseudo-inverse of S_n (one-sided Jacobi), dropping sigma_i <= svd_tau sigma_max. */
typedef enum { CPQR_NE = 0, CPQR_QR = 1, CPQR_SVD = 2, CPQR_PINV = 3 } cpqr_variant;

/* Fit computation: FAST uses the identity ||X-Xh||^2 = ||X||^2 - 2<X,Xh>
 * + ||Xh||^2 with already-computed quantities; DIRECT forms the residual explicitly (one extra
 * pass over X, used for noiseless problems, reading 19/28). */
typedef enum { CPQR_FIT_FAST = 0, CPQR_FIT_DIRECT = 1 } cpqr_fit_mode;

/* Where the tensor passed to cpqr_set_tensor lives. */
typedef enum {
  CPQR_MEM_HOST = 0,          /* host memory; copied to the device (pinned is faster) */
  CPQR_MEM_DEVICE_COPY = 1,   /* device memory; copied into a context-owned buffer */
  CPQR_MEM_DEVICE_BORROW = 2  /* device memory; used in place, caller keeps it alive */
} cpqr_mem;

/* Non-fatal condition flags (cpqr_get_flags), OR-ed over all sweeps run since the last
 * cpqr_set_factors / cpqr_init_factors / cpqr_set_tensor (each of which clears them). */
enum {
  CPQR_FLAG_ILLCOND_R0 = 1u,      /* QR variant: min|R0_jj| <= R^(N-1)*eps*max|R0_jj| (reading 17) */
  CPQR_FLAG_NE_CHOL_FALLBACK = 2u,/* NE: Cholesky met a non-positive pivot; LU used (reading 18) */
  CPQR_FLAG_SVD_TRUNCATED = 4u,   /* SVD / PINV: at least one sigma_i <= tau*sigma_max dropped */
  CPQR_FLAG_NE_ILLCOND = 8u       /* NE: kappa(S_n) estimate (max/min Cholesky pivot)^2 > 1e8: the
                                     normal equations lose > 8 digits; a robust driver switches to
                                     QR / QR-SVD */
};

/* How the ranks of the slab data parallelism (cpqr_options.world > 1) exchange W_n. */
typedef enum {
  CPQR_COMM_NCCL = 0,  /* one process (context) per GPU; ncclAllReduce / ncclAllGather over NVLink */
  CPQR_COMM_LOCAL = 1, /* virtual ranks: ONE context on one device runs all `world` slabs in rank
                          order (each with its own plans, TMA maps and slab of Q_N) and combines
                          them with a fixed-order sum kernel (modes n < N) or one device copy per
                          rank (mode N); `rank` is ignored.  The multi-GPU code path on one GPU, for
                          parity tests and per-rank timing projections. */
  CPQR_COMM_PEER = 2,  /* one process (context) per GPU, no collective library on the data path: the
                          Q0 apply's final sum (Alg. 2 line 9; NE: a copy kernel) stores this rank's
                          W_n partial straight into a slot of EVERY rank's receive window over
                          NVLink peer memory and raises a flag; each rank then sums the p slots in
                          rank order (modes n < N) or places the ranks' rows (mode N), so the
                          factors stay bitwise identical on all ranks (SURVEY.md 8(f) NEXT-2,
                          DESIGN.md §8).  ||X||^2 and the DIRECT residual take the same path.  The
                          windows are exchanged with cpqr_peer_handle / cpqr_peer_connect before
                          cpqr_set_tensor; nccl_id is optional (only cpqr_debug_mode's Y uses it). */
  CPQR_COMM_LOCAL_PEER = 3 /* CPQR_COMM_LOCAL with the exchange of CPQR_COMM_PEER: p receive windows
                          in the one context, every virtual rank pushes into all of them (the same
                          kernels on one GPU, none waiting on another); cpqr_debug_peer checks that
                          all windows received identical bytes. */
} cpqr_comm;

typedef struct cpqr_options {
  uint32_t struct_size;   /* = sizeof(cpqr_options); ABI versioning */
  double svd_tau;         /* SVD / PINV truncation: keep sigma_i > svd_tau*sigma_max; < 0 -> R*eps */
  int32_t fit_mode;       /* cpqr_fit_mode */
  int32_t device;         /* CUDA device ordinal */
  void* stream;           /* borrowed cudaStream_t to run on (e.g. torch's), or NULL: own stream */
  int32_t rank, world;    /* slab data parallelism over the last mode (world = 1: single GPU) */
  uint8_t nccl_id[128];   /* ncclUniqueId from cpqr_nccl_unique_id() on rank 0, broadcast */
  int32_t use_graph;      /* 1: capture one sweep as a CUDA graph and replay it */
  int32_t profile;        /* 1: record CUDA events around each phase (cpqr_get_profile) */
  int32_t mttm_tree;      /* QR/SVD, N >= 3: 1 = dimension-tree Multi-TTM: modes
                             [0, h) share T_L = X x_{k>=h} Q_k^T and modes [h, N) share
                             T_R = X x_{k<h} Q_k^T, h = ceil(N/2), so a sweep streams X twice
                             instead of N times; Y_(n) equals the per-mode Multi-TTM up to
                             rounding.  0 (default) = one pass over X per mode (Alg. 2 line 8). */
  int32_t comm;           /* cpqr_comm: how world > 1 ranks exchange W_n (default CPQR_COMM_NCCL).  With
                             world = 1, CPQR_COMM_NCCL plus a non-zero nccl_id, or CPQR_COMM_PEER, run
                             the same in-graph exchange on one rank (a hardware check of the path). */
} cpqr_options;

/* Fills *opt with defaults: svd_tau = -1, FAST fit, device 0, own stream, world 1,
 * use_graph 1, profile 0, mttm_tree 0, comm NCCL. */
void cpqr_default_options(cpqr_options* opt);

typedef struct cpqr_ctx cpqr_ctx;

/* Create a solver for an N-way tensor of global dims[0..N-1] and CP rank R.
 * Preconditions: 2 <= N <= 10; 1 <= R <= 32; 1 <= dims[k] < 2^31.  A dense tensor needs tall
 * factors, R <= dims[k] for all k (reading 27).  "Short modes" dims[k] < R (the
 * 10-way sine of sums: I_k = 8 < R = 10) are accepted for Kruskal input only
 * (cpqr_set_ktensor; cpqr_set_tensor then returns EINVAL), world = 1: the factors are stored
 * zero-padded to R rows, V_n keeps its prod_{k != n} min(I_k, R) nonzero rows and is factored by the
 * shifted CholeskyQR3; the factor arrays the caller passes and receives stay dims[k] x R.  V_n and
 * its QR buffers must fit: 3 x 8 x R x max_n prod_{k != n} min(dims[k], R) bytes <= 120 GB (ENOMEM).
 * 1 <= world <= 16 and world divides dims[N-1]: with world = p > 1 the
 * last mode is split into p equal slabs (cpqr_set_tensor), every variant (NE, QR, SVD) and both
 * Multi-TTM schedules run slab-parallel, the factors are replicated (identical on every rank).
 * Factor heights: any I_n (CholeskyQR2 for every height; its Householder fallback is the
 * register / shared-memory TSQR up to ~3200 rows at R = 32 and a one-CTA global-memory
 * Householder beyond, slow but exact).
 * Errors: EINVAL, ENOMEM, ECUDA, ENCCL. */
cpqr_status cpqr_create(int N, const int64_t* dims, int R, int variant,
                        const cpqr_options* opt, cpqr_ctx** out);

/* Set the local tensor slab X(:, ..., :, slab_begin:slab_end) (0-based, end exclusive, on the
 * last mode), column-major I_1 x ... x I_{N-1} x (slab_end - slab_begin) = a contiguous block
 * of the global column-major tensor at element offset slab_begin * prod_{k<N} I_k.
 * world = 1 requires [0, I_N); with NCCL ranks, this rank's slab [r I_N/p, (r+1) I_N/p).  With
 * CPQR_COMM_LOCAL either the whole tensor [0, I_N) (split into the p slabs) or one virtual
 * rank's slab (the sweep needs every slab set).  Computes ||X||^2 (summed over the ranks) and
 * clears the condition flags.
 * Odd I_1: TMA needs 16-byte global strides, so the library stores mode 1 padded to I_1 + 1 with a
 * zero row (in X and in A_1; exact: the pad row of every W_1, Ahat_1 and Q_1 stays zero).  The
 * tensor is then COPIED into a context-owned padded buffer whatever `mem` says (a borrowed tensor
 * too; host input is staged once on the device), costing prod(I_k) (1 + 1/I_1) extra doubles; all
 * arrays the caller passes or receives keep I_1 rows.  CPQR_PAD_ODD=0 (environment, at create)
 * keeps the unpadded layout and the slower register-staged stream kernels.
 * Errors: EINVAL (slab range / NULL / mem kind), ENOMEM, ECUDA, ENCCL. */
cpqr_status cpqr_set_tensor(cpqr_ctx* ctx, const double* x, int64_t slab_begin,
                            int64_t slab_end, int mem);

/* Batched CP-ALS-QR of P independent small 3-way problems, one CTA per problem (SURVEY.md 8(f)
 * NEXT-4; the collinear-factor study's regime).  Stateless: all pointers are
 * DEVICE pointers, launched on `stream` (NULL: default stream), asynchronous.
 *   dims[3] = I_1, I_2, I_3 (R <= I_k <= 64), 1 <= R <= 8, I_1 I_2 R <= 16384, I_2 I_3 R <= 16384.
 *   X: P consecutive column-major I_1 x I_2 x I_3 tensors.  A0 / A: P blocks of the three factors
 *   (I_1 x R, I_2 x R, I_3 x R column-major, consecutive); A0[mode 1] is unused (Alg. 2 line 2).
 *   Each CTA runs QR-variant sweeps until the fit changes by less than tol or
 *   max_iters sweeps; fits: P x max_iters (NaN after the last sweep), iters: P, lam: P x R.
 * Errors: EINVAL (shapes / NULL), ECUDA (launch). */
cpqr_status cpqr_batched_qr(int P, const int64_t* dims, int R, const double* X, const double* A0,
                            int max_iters, double tol, double* A, double* lam, double* fits,
                            int* iters, void* stream);

/* cpqr_batched_qr for any of the four solvers of the paper's accuracy study:
 * variant = CPQR_NE (Alg. 1, Cholesky solve with an LU fallback), CPQR_QR, CPQR_SVD (QR-SVD,
 * sigma_i kept iff sigma_i > tau sigma_max of R0) or CPQR_PINV (Alg. 1 with
 * pinv(S_n), same tau rule); tau < 0 means R * eps.  NE / PINV use A0 of modes
 * 2 and 3 (Alg. 1 line 3; A0[mode 1] unused, as for QR).  Same shapes, layouts, outputs and errors
 * as cpqr_batched_qr (which is this call with CPQR_QR). */
cpqr_status cpqr_batched(int P, const int64_t* dims, int R, int variant, double tau, const double* X,
                         const double* A0, int max_iters, double tol, double* A, double* lam,
                         double* fits, int* iters, void* stream);

/* Kruskal-tensor input: X = [[lambda; B_1..B_N]] of rank S is never formed.
 * B[k] is a host pointer to the column-major I_k x S matrix B_k, lambda a host S-vector (NULL:
 * ones).  Each mode then computes W_n = B_n diag(lambda) [((.)_{k != n} Q_k^T B_k)^T Q0]
 * (QR / SVD) or the MTTKRP B_n diag(lambda) (*)_{k != n} B_k^T A_k (NE) in O(R^N S + I_n R S),
 * and ||X||^2 = lambda^T ((*)_k B_k^T B_k) lambda.  Replaces a dense tensor set before (and
 * cpqr_set_tensor replaces this).  The arrays are copied before return.  Single GPU (world = 1);
 * cpqr_debug_mode is unavailable.  The DIRECT fit (opt.fit_mode) evaluates
 * ||X - Xh|| entry by entry from the factors of both Kruskal tensors, never forming either
 * (O(prod I_k (S + R)) flops; S + R <= 512), so relative errors below the fast fit's sqrt(eps)
 * floor are resolved.  Errors: EINVAL, ENOMEM, ECUDA. */
cpqr_status cpqr_set_ktensor(cpqr_ctx* ctx, int S, const double* lambda, const double* const* B);

/* Set the factors: A[k] is a host pointer to the column-major I_k x R matrix A_k (k = 0..N-1;
 * A[0] may be NULL for the QR/SVD variants: Alg. 2 line 2 initialises A_2..A_N only).
 * lambda: host R-vector or NULL (ones).  Must be identical on all ranks.  Recomputes the factor
 * QR cache (Alg. 2 line 3) or the Gram matrices (Alg. 1 line 3).  Errors: EINVAL. */
cpqr_status cpqr_set_factors(cpqr_ctx* ctx, const double* const* A, const double* lambda);

/* Initialise the factors with i.i.d. N(0,1) entries from a counter-based generator
 * (splitmix64 + Box-Muller, seed-determined, identical on every rank), lambda = 1. */
cpqr_status cpqr_init_factors(cpqr_ctx* ctx, uint64_t seed);

/* Run exactly nsweeps sweeps over modes 1..N (Alg. 2 lines 4-13 / Alg. 1 lines 4-12); no early
 * stop (convergence is the caller's policy).  If fits != NULL, fits[s] = fit
 * after sweep s (computed after mode N).  Synchronous.
 * Errors: ESTATE (no tensor/factors), EDIVERGED, ENCCL, ECUDA. */
cpqr_status cpqr_sweep(cpqr_ctx* ctx, int nsweeps, double* fits);

/* Current normalised factors (unit 2-norm columns) into host buffers A_out[k] (column-major
 * I_k x R, NULL entries skipped) and lambda (R, may be NULL).  Identical on all ranks. */
cpqr_status cpqr_get_factors(cpqr_ctx* ctx, double* const* A_out, double* lambda_out);

cpqr_status cpqr_get_fit(cpqr_ctx* ctx, double* fit);      /* fit after the last sweep */
cpqr_status cpqr_get_flags(cpqr_ctx* ctx, uint32_t* flags);

/* Per-phase device time (ms) accumulated since the last reset, Table 3.1 taxonomy
 * (PAPER.md:495-510), only with opt.profile = 1 (eager launches, V_n QR inline):
 *   ms[0] Multi-TTM stream-X pass (the dominant kernel; NE: the whole MTTKRP)
 *   ms[1] Multi-TTM remaining TTMs
 *   ms[2] factor QR: the fused tail launch (solve, normalise, factor QR, fast fit)
 *   ms[3] computing Q0 (QR of V_n)       ms[4] applying Q0
 *   ms[5] other (S_n^+ of PINV, the NE tail, the DIRECT fit)
 *   ms[6] exchange of W_n across the ranks (NCCL, the virtual ranks' combine, or the peer combine)
 * Slab-parallel phases (0, 1, 4 and the NE MTTKRP) are summed over the slabs a context runs.
 * launches[0..6]: kernel launches per phase; bytes0/flops0: algorithmic HBM bytes and flops of
 * phase 0.  reset != 0 zeroes the counters after reading. */
typedef struct cpqr_profile {
  double ms[7];
  int64_t launches[7];
  double bytes0, flops0;
  int64_t launches_total;
} cpqr_profile;
cpqr_status cpqr_get_profile(cpqr_ctx* ctx, cpqr_profile* prof, int reset);
/* cpqr_get_timings: the seven per-phase milliseconds of cpqr_get_profile
 * (ms[0..6] as above: the paper's five-way split, with the Multi-TTM's
 * stream-X pass separated from its remaining TTMs and the exchange separated from "other"),
 * accumulated since the last reset; zeros unless opt.profile = 1.  ms: caller buffer of 7
 * doubles.  Errors: EINVAL (NULL ctx or ms). */
cpqr_status cpqr_get_timings(cpqr_ctx* ctx, double* ms);

/* Kernel launches issued by one cpqr_sweep(ctx, 1, ...) (claims for bench "gpu_launches"). */
cpqr_status cpqr_launches_per_sweep(cpqr_ctx* ctx, int64_t* n);

/* Parity hook: for mode n (0-based) compute Alg. 2 lines 6-9 (V_n, Q0/R0, Multi-TTM Y, W_n)
 * from the current factor QR cache, or from Q_override[k] (host, column-major I_k x R, k != n)
 * if Q_override != NULL (R_k from the cache still define V_n), WITHOUT changing state.
 * Outputs (host, any may be NULL):
 *   Y_out : the Multi-TTM result tensor Y = X x_{k!=n} Q_k^T (dims R..I_n..R, column-major;
 *           its mode-n unfolding is Y_(n) in Kolda-Bader order).  With world > 1 each rank's
 *           partial Y is summed across ranks (debug only).
 *   Q0_out: R^{N-1} x R column-major, rows in Kolda-Bader order;  R0_out: R x R column-major;
 *   W_out : I_n x R column-major (global rows). */
cpqr_status cpqr_debug_mode(cpqr_ctx* ctx, int n, const double* const* Q_override,
                            double* Y_out, double* Q0_out, double* R0_out, double* W_out);

/* The Multi-TTM plan of mode n (0-based) on slab `slab` (0 unless CPQR_COMM_LOCAL), for the
 * plan tables of DESIGN.md §8 and the contraction-order tests: writes
 * min(cap, #steps) rows of 6 int64 to info -- kernel kind (0/4 strided, 1/5 fibre, 2/6/8 fused
 * slice, 3/7 partial-sum fix-up, 9 small TTM, 10 fused last-two-modes strided pass, 100 NE Khatri-Rao
 * diagonal), bitmask of the contracted global
 * modes, input elements, output elements, flops, 1 if the step reads X -- and #steps to *nsteps.
 * Errors: EINVAL, ESTATE (no dense tensor set). */
cpqr_status cpqr_debug_plan(cpqr_ctx* ctx, int n, int slab, int64_t* info, int cap, int* nsteps);

/* Stand-alone kernels exposed for parity tests (host in/out, column-major):
 * thin Householder QR of an m x R matrix (m >= R): Q (m x R), Rf (R x R), diag(Rf) >= 0. */
cpqr_status cpqr_debug_qr(cpqr_ctx* ctx, const double* A, int64_t m, double* Q, double* Rf);
/* One-sided Jacobi SVD pseudo-inverse solve: Ahat = W U S^+ V^T for R0 = U S V^T
 * (PAPER.md:335-339), W m x R; returns the number of truncated singular values in *ntrunc. */
cpqr_status cpqr_debug_svd_solve(cpqr_ctx* ctx, const double* R0, const double* W, int64_t m,
                                 double tau, double* Ahat, int* ntrunc);

cpqr_status cpqr_destroy(cpqr_ctx* ctx);
const char* cpqr_status_string(cpqr_status s);
const char* cpqr_last_error(const cpqr_ctx* ctx);

/* NCCL bootstrap: rank 0 calls this, broadcasts the 128 bytes (e.g. over torch.distributed),
 * every rank passes them in cpqr_options.nccl_id.  Returns ENCCL if NCCL is unavailable. */
cpqr_status cpqr_nccl_unique_id(uint8_t id[128]);

/* CPQR_COMM_PEER bootstrap (one process per GPU; P2P access between the devices required):
 * cpqr_peer_handle writes the 64-byte CUDA IPC handle of this rank's receive window; the caller
 * all-gathers the handles in rank order (e.g. torch.distributed.all_gather) and passes the
 * world x 64 bytes to cpqr_peer_connect on every rank, which maps the peers' windows
 * (cudaIpcOpenMemHandle).  Both before cpqr_set_tensor.  world = 1 needs neither.
 * Errors: EINVAL (other comm modes, NULL), ESTATE (connected twice), ECUDA (IPC / no P2P). */
cpqr_status cpqr_peer_handle(cpqr_ctx* ctx, uint8_t handle[64]);
cpqr_status cpqr_peer_connect(cpqr_ctx* ctx, const uint8_t* handles);

/* State of the peer windows (CPQR_COMM_PEER / CPQR_COMM_LOCAL_PEER), for tests: info[0] =
 * exchanges completed by this rank (its epoch), info[1] = virtual ranks' windows whose received
 * bytes, flags or epoch differ from window 0 (LOCAL_PEER; else 0), info[2] = bytes per window,
 * info[3] = the smallest arrival flag of this rank's window. */
cpqr_status cpqr_debug_peer(cpqr_ctx* ctx, int64_t info[4]);
/* Plumbing check of the IPC windows between processes WITHOUT kernels that wait on each other:
 * cpqr_debug_peer_put pushes n host doubles as one exchange into every rank's window (the
 * k_peer_push kernel; it never waits); after a host-side barrier, cpqr_debug_peer_get runs the
 * combine of that exchange -- the rank-order sum (gather = 0, n doubles) or the ranks' blocks in
 * rank order (gather = 1, world x n doubles) -- into a host buffer.  Every rank must put before
 * any rank gets (else the combine waits up to CPQR_PEER_TIMEOUT_MS, default 20000, then ENCCL). */
cpqr_status cpqr_debug_peer_put(cpqr_ctx* ctx, const double* src, int64_t n);
cpqr_status cpqr_debug_peer_get(cpqr_ctx* ctx, double* out, int64_t n, int gather);

/* Library version string ("cpqr <semver> sm_100a"). */
const char* cpqr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CPQR_H */
