"""Plain, slow, obviously-correct fp64 oracle for the CP-ALS-QR hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

Conventions:
  * tensors are numpy arrays of shape (I_1, ..., I_N) in Fortran (column-major) order,
    mode 1 fastest -- the bytes of the C-order (I_N, ..., I_1) buffer that synth.py makes;
  * modes are 0-based in code (paper mode n == code mode n-1);
  * Kronecker / Khatri-Rao follow PAPER.md:93-95 (second operand's index fastest), so
    Z_n = A_N (.) ... (.) A_1 has A_1's row index fastest (reading 1, Kolda-Bader);
  * every thin QR returns diag(R) >= 0 (reading 6);
  * fp64 throughout.

Pinned by tests/test_oracle_pins.py (closed forms, worked examples, brute force,
library routines, invariants).  No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

EPS = np.finfo(np.float64).eps

FLAG_ILLCOND_R0 = 1
FLAG_NE_CHOL_FALLBACK = 2
FLAG_SVD_TRUNCATED = 4

__all__ = [
    "EPS", "FLAG_ILLCOND_R0", "FLAG_NE_CHOL_FALLBACK", "FLAG_SVD_TRUNCATED",
    "as_tensor", "kron", "khatri_rao", "hadamard", "matricize", "tensorize", "ttm",
    "multi_ttm", "ttm_order", "qr_pos", "kr_of_triangular", "structured_qr", "kr_group_qr",
    "vn_tree_groups", "tree_qr", "apply_q0",
    "solve_qr", "solve_svd", "pinv_svd", "normalize", "full_tensor", "fit_fast_qr", "fit_fast_ne",
    "fit_direct", "mode_update_qr", "mode_update_ne", "cp_als_qr", "cp_als_ne",
    "qr_cost", "ttm_cost", "mttkrp", "ktensor_norm2", "w_ktensor", "mttkrp_ktensor",
    "sine_of_sums_ktensor", "sine_of_sums_rank_n_ktensor", "score",
]


# ----------------------------------------------------------------------------- layout
def as_tensor(Xc: np.ndarray) -> np.ndarray:
    """C-order (I_N..I_1) buffer -> Fortran (I_1..I_N) view of the same bytes."""
    return Xc.T


# ------------------------------------------------------------------ matrix products §2.2
def kron(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Kronecker product: [A (x) B](K(i-1)+k, M(j-1)+l) = A(i,j) B(k,l)."""
    I, J = A.shape
    K, M = B.shape
    return (A[:, None, :, None] * B[None, :, None, :]).reshape(I * K, J * M)


def khatri_rao(mats) -> np.ndarray:
    """Khatri-Rao product: column k is A(:,k) (x) B(:,k); applied left to right,
    so the LAST matrix's row index is fastest."""
    out = mats[0]
    for B in mats[1:]:
        I, R = out.shape
        J, R2 = B.shape
        assert R == R2
        out = (out[:, None, :] * B[None, :, :]).reshape(I * J, R)
    return out


def hadamard(A, B):
    """Elementwise product."""
    return A * B


# ------------------------------------------------------------- tensor operations §2.2
def matricize(X: np.ndarray, n: int) -> np.ndarray:
    """Mode-n unfolding X_(n): columns are mode-n fibers, in Kolda-Bader order
    (reading 1): element (i_1..i_N) -> row i_n, column sum_{k!=n} i_k J_k, J_k = prod_{m<k,m!=n} I_m."""
    return np.reshape(np.moveaxis(X, n, 0), (X.shape[n], -1), order="F")


def tensorize(M: np.ndarray, dims, n: int) -> np.ndarray:
    """Inverse of matricize (fold back)."""
    dims = tuple(dims)
    rest = dims[:n] + dims[n + 1:]
    T = np.reshape(M, (dims[n],) + rest, order="F")
    return np.moveaxis(T, 0, n)


def ttm(X: np.ndarray, U: np.ndarray, n: int) -> np.ndarray:
    """n-mode product Y = X x_n U:
    Y(i_1..j..i_N) = sum_{i_n} X(i_1..i_n..i_N) U(j, i_n), i.e. Y_(n) = U X_(n).

    Written on the 3-index view X3(a, i_n, b) (a over modes < n, fastest; b over modes > n)
    of the same column-major bytes: Y3(a, j, b) = sum_i U(j, i) X3(a, i, b)."""
    dims = X.shape
    A = int(np.prod(dims[:n], dtype=np.int64))
    B = int(np.prod(dims[n + 1:], dtype=np.int64))
    X3 = np.reshape(X, (A, dims[n], B), order="F")
    # X3.T is the C-order (B, I_n, A) view; U @ (I_n, A) for each b.
    Y3 = np.matmul(U, X3.T).T                       # (A, J, B), Fortran-contiguous
    return np.reshape(Y3, dims[:n] + (U.shape[0],) + dims[n + 1:], order="F")


def ttm_order(dims, skip: int):
    """Order of the N-1 TTMs: decreasing tensor dimension; ties broken by
    decreasing mode index (reading 5)."""
    modes = [k for k in range(len(dims)) if k != skip]
    return sorted(modes, key=lambda k: (-dims[k], -k))


def multi_ttm(X: np.ndarray, Us: dict, order=None) -> np.ndarray:
    """Multi-TTM Y = X x_{k} U_k over the modes in Us (Eq. (2.2)), as a
    sequence of single TTMs, in decreasing-dimension order by default."""
    if order is None:
        modes = sorted(Us.keys(), key=lambda k: (-X.shape[k], -k))
    else:
        modes = list(order)
    Y = X
    for k in modes:
        Y = ttm(Y, Us[k], k)
    return Y


def mttkrp(X: np.ndarray, factors, n: int) -> np.ndarray:
    """MTTKRP M_n = X_(n) Z_n, Z_n = A_N (.) ... (.) A_{n+1} (.) A_{n-1} (.) ... (.) A_1
    (Alg. 1 lines 7-8; Eq. (cp_mat))."""
    N = X.ndim
    Z = khatri_rao([factors[k] for k in range(N - 1, -1, -1) if k != n])
    return matricize(X, n) @ Z


# --------------------------------------------------------------------------- QR / LS
def qr_pos(A: np.ndarray):
    """Compact/thin QR A = QR by LAPACK Householder, then the sign fix
    diag(R) >= 0 (reading 6; a zero diagonal keeps sign +1)."""
    Q, R = np.linalg.qr(A, mode="reduced")
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return Q * s[None, :], R * s[:, None]


def kr_of_triangular(Rs, n: int) -> np.ndarray:
    """V_n = R_N (.) ... (.) R_{n+1} (.) R_{n-1} (.) ... (.) R_1 (Alg. 2 line 6)."""
    N = len(Rs)
    return khatri_rao([Rs[k] for k in range(N - 1, -1, -1) if k != n])


def structured_qr(Rs, n: int):
    """Q0, R0 = QR(V_n), dense (Alg. 2 line 7; PAPER.md:314 treats V_n dense)."""
    return qr_pos(kr_of_triangular(Rs, n))


def kr_group_qr(Rg):
    """QR of the Khatri-Rao product of a group of triangular factors, Rg = [R_a, R_b, ...] in the
    product's order (R_a slowest), by a chain of pairwise QRs (the tree across the Khatri-Rao
    factors of PAPER.md:479).  With (A C) (.) (B D) = (A (x) B)(C (.) D) (Eq. (2.1),
    PAPER.md:97-100): start from P = I, S = (the fastest factor); for each next-slower
    factor R_k, QR(R_k (.) S) = Q S' gives R_k (.) (P S) = (I (x) P) Q S', so P <- (I (x) P) Q,
    S <- S'.  Returns (P, S): the group's product = P S, P orthonormal, S upper triangular with
    diag >= 0.  A one-factor group returns (I, R_k) (R_k is already triangular).  A short mode
    (I_k < R) contributes its min(I_k, R) x R trapezoidal R_k (economy QR, reading 34)."""
    P, S = np.eye(Rg[-1].shape[0]), Rg[-1]
    for Rk in reversed(Rg[:-1]):
        Qm, S = qr_pos(khatri_rao([Rk, S]))
        P = kron(np.eye(Rk.shape[0]), P) @ Qm
    return P, S


def vn_tree_groups(N: int, n: int):
    """The two factor groups of V_n in the tree QR (reading 36): the modes are split at
    h = ceil(N/2) as in the dimension tree; the retained modes of the half that
    does not hold n form a group shared by every mode of the other half (their R_k do not change
    between those modes in a sweep), the rest of n's own half the other group.  Both in decreasing
    mode order (the Khatri-Rao order of V_n).  Returns (hi, lo): V_n = [(.) hi] (.) [(.) lo]."""
    h = (N + 1) // 2
    hi = [k for k in range(N - 1, h - 1, -1) if k != n]
    lo = [k for k in range(h - 1, -1, -1) if k != n]
    return hi, lo


def tree_qr(Rs, n: int):
    """Q0, R0 = QR(V_n) by a tree across the Khatri-Rao factors (SURVEY.md 8(f)
    NEXT-2): each group of vn_tree_groups is reduced by kr_group_qr to (P_g, S_g), then the root
    QR(S_hi (.) S_lo) = Q_r R0 and Q0 = (P_hi (x) P_lo) Q_r, since
    V_n = (P_hi S_hi) (.) (P_lo S_lo) = (P_hi (x) P_lo)(S_hi (.) S_lo) (Eq. (2.1)).  Equal to the
    dense QR of V_n (structured_qr) up to rounding: the thin QR with diag(R0) > 0 is unique."""
    hi, lo = vn_tree_groups(len(Rs), n)
    if not hi or not lo:                      # N = 2: one retained factor
        g = hi or lo
        return kr_group_qr([Rs[k] for k in g])
    P_hi, S_hi = kr_group_qr([Rs[k] for k in hi])
    P_lo, S_lo = kr_group_qr([Rs[k] for k in lo])
    Q_r, R0 = qr_pos(khatri_rao([S_hi, S_lo]))
    return kron(P_hi, P_lo) @ Q_r, R0


def apply_q0(Y: np.ndarray, n: int, Q0: np.ndarray) -> np.ndarray:
    """W_n = Y_(n) Q0 (Alg. 2 line 9)."""
    return matricize(Y, n) @ Q0


def solve_qr(R0: np.ndarray, W: np.ndarray) -> np.ndarray:
    """Solve Ahat R0^T = W by substitution (Alg. 2 line 10; Eq. (ls-qr-q0-step)
    PAPER.md:331).  (Ahat R0^T)(:, j) = sum_{l >= j} Ahat(:, l) R0(j, l) with R0 upper
    triangular, so back substitution over columns j = R..1."""
    R = R0.shape[0]
    Ahat = np.zeros_like(W)
    for j in range(R - 1, -1, -1):
        acc = W[:, j].copy()
        for l in range(j + 1, R):
            acc -= Ahat[:, l] * R0[j, l]
        Ahat[:, j] = acc / R0[j, j]
    return Ahat


def solve_svd(R0: np.ndarray, W: np.ndarray, tau: float = -1.0):
    """CP-ALS-QR-SVD solve: R0 = U S V^T, Ahat = W U S^+ V^T, truncating
    sigma_i <= tau * sigma_max (reading 15; tau < 0 -> R*eps).  Returns (Ahat, n_truncated)."""
    R = R0.shape[0]
    if tau < 0:
        tau = R * EPS
    U, s, Vt = np.linalg.svd(R0)
    keep = s > tau * s[0]
    Ahat = ((W @ U[:, keep]) / s[keep][None, :]) @ Vt[keep, :]
    return Ahat, int(R - keep.sum())


def pinv_svd(S: np.ndarray, tau: float = -1.0):
    """Moore-Penrose pseudo-inverse by the SVD, as MATLAB's pinv: S = U diag(s)
    V^T, S^+ = V diag(1/s_i) U^T over the kept s_i > tau * s_max (reading 32: tau < 0 -> R*eps, the
    max(size(S)) * eps(norm(S)) default up to the ulp rounding of eps(norm)).  Returns
    (S^+, n_truncated)."""
    R = S.shape[0]
    if tau < 0:
        tau = R * EPS
    U, s, Vt = np.linalg.svd(S)
    keep = s > tau * s[0]
    P = (Vt[keep, :].T / s[keep][None, :]) @ U[:, keep].T
    return P, int(R - keep.sum())


def normalize(Ahat: np.ndarray):
    """Normalize columns (Alg. 2 line 11): lam_r = ||Ahat(:,r)||_2, A = Ahat/lam.
    A zero column gives lam_r = 0 and column e_1 (reading 10)."""
    lam = np.sqrt(np.sum(Ahat * Ahat, axis=0))
    A = np.empty_like(Ahat)
    for r in range(Ahat.shape[1]):
        if lam[r] > 0:
            A[:, r] = Ahat[:, r] / lam[r]
        else:
            A[:, r] = 0.0
            A[0, r] = 1.0
    return A, lam


# ------------------------------------------------------------------------------ fits
def full_tensor(lam, factors) -> np.ndarray:
    """X_hat = sum_r lam_r a_r^(1) o ... o a_r^(N) (Eq. (cp)), built from
    Eq. (cp_mat): X_hat_(1) = Ahat_1 Z_1^T."""
    dims = tuple(A.shape[0] for A in factors)
    N = len(factors)
    Ahat1 = factors[0] * np.asarray(lam)[None, :]
    if N == 1:
        return Ahat1.sum(axis=1)
    Z1 = khatri_rao([factors[k] for k in range(N - 1, 0, -1)])
    return tensorize(Ahat1 @ Z1.T, dims, 0)


def fit_direct(X, lam, factors) -> float:
    """fit = 1 - ||X - X_hat||_F / ||X||_F with X_hat formed explicitly."""
    Xh = full_tensor(lam, factors)
    return 1.0 - np.linalg.norm((X - Xh).ravel()) / np.linalg.norm(X.ravel())


def _fit_from_terms(nX2, inner, nXh2):
    """||X - X_hat||^2 = ||X||^2 - 2<X,X_hat> + ||X_hat||^2; clamp (reading 14)."""
    res = np.sqrt(max(0.0, nX2 - 2.0 * inner + nXh2))
    return 1.0 - res / np.sqrt(nX2)


def fit_fast_qr(nX2, W_N, Ahat_N, R0, R_N, lam) -> float:
    """Efficient error for CP-ALS-QR:
    <X,X_hat> = <W_N, Ahat_N R0^T>,  ||X_hat||^2 = <R0^T R0, diag(lam) R_N^T R_N diag(lam)>."""
    inner = float(np.sum(W_N * (Ahat_N @ R0.T)))
    D = np.diag(lam)
    nXh2 = float(np.sum((R0.T @ R0) * (D @ R_N.T @ R_N @ D)))
    return _fit_from_terms(nX2, inner, nXh2)


def fit_fast_ne(nX2, M_N, Ahat_N, S_N, G_N, lam) -> float:
    """Efficient error for CP-ALS:
    <X,X_hat> = <M_N, Ahat_N>,  ||X_hat||^2 = <S_N, diag(lam) G_N diag(lam)>."""
    inner = float(np.sum(M_N * Ahat_N))
    D = np.diag(lam)
    nXh2 = float(np.sum(S_N * (D @ G_N @ D)))
    return _fit_from_terms(nX2, inner, nXh2)


# ----------------------------------------------------------------------- mode updates
def mode_update_qr(X, Qs, Rs, n, variant="QR", tau=-1.0, order=None, kt=None):
    """One CP-ALS-QR(-SVD) mode update, Alg. 2 lines 6-12, in the paper's
    order.  Qs/Rs: factor QR cache (entry n ignored).  kt = (lam_x, B): Kruskal input, X unused
    (lines 8-9 by w_ktensor).  Returns a dict of every intermediate."""
    N = X.ndim if kt is None else len(kt[1])
    V = kr_of_triangular(Rs, n)                                   # line 6
    Q0, R0 = qr_pos(V)                                            # line 7
    if kt is None:
        Y = multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n},  # line 8
                      order=order)
        W = apply_q0(Y, n, Q0)                                    # line 9
    else:
        Y = None
        W = w_ktensor(kt[0], kt[1], Qs, n, Q0)                    # lines 8-9
    ntrunc = 0
    if variant == "QR":                                           # line 10
        Ahat = solve_qr(R0, W)
    elif variant == "SVD":
        Ahat, ntrunc = solve_svd(R0, W, tau)
    else:
        raise ValueError(variant)
    A, lam = normalize(Ahat)                                      # line 11
    Qn, Rn = qr_pos(A)                                            # line 12
    d = np.abs(np.diag(R0))
    # reading 17: numerically rank-deficient R0 when min|R0_jj| <= rows(V_n) * eps * max|R0_jj|
    # (the numpy.linalg.matrix_rank default tolerance, applied to V_n's R factor)
    flags = FLAG_ILLCOND_R0 if (variant == "QR" and d.min() <= V.shape[0] * EPS * d.max()) else 0
    if ntrunc:
        flags |= FLAG_SVD_TRUNCATED
    return dict(V=V, Q0=Q0, R0=R0, Y=Y, Yn=None if Y is None else matricize(Y, n), W=W, Ahat=Ahat,
                A=A, lam=lam, Q=Qn, R=Rn, ntrunc=ntrunc, flags=flags)


def mode_update_ne(X, factors, grams, n, kt=None, solve="chol", tau=-1.0):
    """One CP-ALS mode update, Alg. 1 lines 6-11: S_n = Hadamard of the other
    Grams; M_n = X_(n) Z_n (MTTKRP); solve Ahat S_n = M_n by Cholesky, falling back
    to LU with partial pivoting on a non-positive pivot (reading 18) -- or, solve="pinv"
    (CP-ALS-PINV), Ahat = M_n S_n^+ with the SVD pseudo-inverse (pinv_svd);
    normalize; G_n = A_n^T A_n.  kt = (lam_x, B): Kruskal input (MTTKRP by mttkrp_ktensor,
    PAPER.md:446-450)."""
    N = len(factors)
    S = np.ones_like(grams[0])
    for k in range(N - 1, -1, -1):                                # line 6
        if k != n:
            S = hadamard(S, grams[k])
    M = mttkrp(X, factors, n) if kt is None else mttkrp_ktensor(kt[0], kt[1], factors, n)  # lines 7-8
    flags = 0
    if solve == "pinv":                                           # line 9, CP-ALS-PINV
        P, ntrunc = pinv_svd(S, tau)
        Ahat = M @ P
        if ntrunc:
            flags |= FLAG_SVD_TRUNCATED
    else:
        try:                                                      # line 9
            L = np.linalg.cholesky(S)
            T = scipy.linalg.solve_triangular(L, M.T, lower=True)
            Ahat = scipy.linalg.solve_triangular(L.T, T, lower=False).T
        except np.linalg.LinAlgError:
            Ahat = scipy.linalg.solve(S, M.T, assume_a="gen").T
            flags |= FLAG_NE_CHOL_FALLBACK
    A, lam = normalize(Ahat)                                      # line 10
    G = A.T @ A                                                   # line 11
    return dict(S=S, M=M, Ahat=Ahat, A=A, lam=lam, G=G, flags=flags)


# ------------------------------------------------------------ Kruskal-tensor input (§3.3.2)
def ktensor_norm2(lam_x, B) -> float:
    """||X||^2 of a Kruskal tensor X = [[lam_x; B_1..B_N]]: lam_x^T (B_1^T B_1 * ... * B_N^T B_N)
    lam_x (Hadamard product of the factor Grams; PAPER.md:127-131 with Eq. (cp_mat))."""
    G = np.ones((len(lam_x), len(lam_x)))
    for Bk in B:
        G = hadamard(G, Bk.T @ Bk)
    lam_x = np.asarray(lam_x, dtype=np.float64)
    return float(lam_x @ G @ lam_x)


def w_ktensor(lam_x, B, Qs, n: int, Q0) -> np.ndarray:
    """W_n = Y_(n) Q0 for a Kruskal input without forming X or Y: Y is the
    Kruskal tensor [[lam_x; Q_1^T B_1, .., B_n, .., Q_N^T B_N]], so
    Y_(n) = B_n diag(lam_x) (C_N (.) .. (.) C_{n+1} (.) C_{n-1} (.) .. (.) C_1)^T with C_k = Q_k^T B_k
    (the Khatri-Rao order of the Kolda-Bader unfolding, Eq. (cp_mat)), and
    W_n = B_n diag(lam_x) [ (.)_k C_k )^T Q0 ]."""
    N = len(B)
    Z = khatri_rao([Qs[k].T @ B[k] for k in range(N - 1, -1, -1) if k != n])
    return (B[n] * np.asarray(lam_x)[None, :]) @ (Z.T @ Q0)


def mttkrp_ktensor(lam_x, B, factors, n: int) -> np.ndarray:
    """M_n = X_(n) Z_n for a Kruskal input: B_n diag(lam_x) (*)_{k != n}
    (B_k^T A_k), the Hadamard product of the small cross-Gram matrices."""
    N = len(B)
    H = np.ones((len(lam_x), factors[0].shape[1]))
    for k in range(N - 1, -1, -1):
        if k != n:
            H = hadamard(H, B[k].T @ factors[k])
    return (B[n] * np.asarray(lam_x)[None, :]) @ H


def sine_of_sums_ktensor(N: int, n: int):
    """The N-variable sine of sums sin(x_1 + .. + x_N) on the grid x_j = 2 pi i / n, i < n
    (PAPER.md:597), as its exact rank-2^{N-1} Kruskal representation: expanding
    with sin(a+b) = sin a cos b + cos a sin b, every term is a product over the modes of sin or cos
    with an odd number k of sines and sign (-1)^((k-1)/2)."""
    x = 2.0 * np.pi * np.arange(n) / n
    terms = [t for t in range(1 << N) if bin(t).count("1") % 2 == 1]
    lam = np.array([(-1.0) ** ((bin(t).count("1") - 1) // 2) for t in terms])
    B = [np.stack([np.sin(x) if (t >> j) & 1 else np.cos(x) for t in terms], axis=1) for j in range(N)]
    return lam, B


def sine_of_sums_rank_n_ktensor(N: int, n: int, alpha=None):
    """The rank-N representation of sin(x_1 + .. + x_N) (Eq. (sinsum_rkd)):
    sum_j sin(x_j) prod_{k != j} sin(x_k + alpha_k - alpha_j) / sin(alpha_k - alpha_j), on the grid
    x = 2 pi i / n, with alpha_j = (j - 1) pi / N by default (the paper leaves alpha open; any
    values with sin(alpha_k - alpha_j) != 0 are exact; reading 33).  Used for the 10-way case
    "in rank-10 representation"."""
    x = 2.0 * np.pi * np.arange(n) / n
    a = np.pi * np.arange(N) / N if alpha is None else np.asarray(alpha, dtype=np.float64)
    lam = np.ones(N)
    B = []
    for k in range(N):
        cols = []
        for j in range(N):
            cols.append(np.sin(x) if k == j else np.sin(x + a[k] - a[j]) / np.sin(a[k] - a[j]))
        B.append(np.stack(cols, axis=1))
    return lam, B


# ------------------------------------------------------------------- score (§4.2)
def score(lam_a, A, lam_b, B) -> float:
    """Similarity of two rank-R Kruskal tensors up to scaling and permutation, in [0, 1]
    (the score of the cited Tomasi-Bro comparison; reading 30): columns
    normalised (norms folded into the weights); for a permutation p of the components
    score_p = (1/R) sum_r (1 - |l_r - m_p(r)| / max(l_r, m_p(r))) prod_k |a_r^(k) . b_p(r)^(k)|,
    and the score is the maximum over all permutations (exhaustive; R <= 8)."""
    import itertools
    N = len(A)
    R = A[0].shape[1]
    la = np.abs(np.asarray(lam_a, dtype=np.float64)).copy()
    lb = np.abs(np.asarray(lam_b, dtype=np.float64)).copy()
    An, Bn = [], []
    for k in range(N):
        na = np.linalg.norm(A[k], axis=0)
        nb = np.linalg.norm(B[k], axis=0)
        la *= na
        lb *= nb
        An.append(A[k] / np.where(na > 0, na, 1.0))
        Bn.append(B[k] / np.where(nb > 0, nb, 1.0))
    cong = np.ones((R, R))
    for k in range(N):
        cong *= np.abs(An[k].T @ Bn[k])                  # cong[r, q] = prod_k |a_r . b_q|
    den = np.maximum(la[:, None], lb[None, :])
    pen = 1.0 - np.abs(la[:, None] - lb[None, :]) / np.where(den > 0, den, 1.0)
    S = pen * cong
    return float(max(np.mean(S[np.arange(R), list(p)]) for p in itertools.permutations(range(R))))


# ---------------------------------------------------------------------------- drivers
def cp_als_qr(X, A0, sweeps, variant="QR", tau=-1.0, fit_mode="fast", debug_sweep1=False,
              order=None, kt=None):
    """CP-ALS-QR / CP-ALS-QR-SVD, Alg. 2, exactly `sweeps` sweeps (no early
    stop; reading 12).  X: Fortran (I_1..I_N) array.  A0: initial factors (A0[0] unused,
    PAPER.md:350).  fit after mode N of every sweep (reading 13): fast or
    direct.  kt = (lam_x, B): Kruskal input instead of X (X = None, PAPER.md:440-456;
    the direct fit then forms X = full_tensor(lam_x, B)).  Returns dict(lam, factors,
    fits, flags, debug)."""
    N = X.ndim if kt is None else len(kt[1])
    nX2 = float(np.dot(X.ravel(order="K"), X.ravel(order="K"))) if kt is None else ktensor_norm2(*kt)
    Xd = X if (kt is None or fit_mode == "fast") else full_tensor(*kt)
    factors = [np.array(A, dtype=np.float64, order="F") for A in A0]
    Qs, Rs = [None] * N, [None] * N
    for k in range(1, N):                                         # line 3
        Qs[k], Rs[k] = qr_pos(factors[k])
    lam = np.ones(factors[0].shape[1])
    fits, flags, debug = [], 0, []
    for s in range(sweeps):                                       # line 4
        last = None
        for n in range(N):                                        # line 5
            qs_in = [None if (k == n or Qs[k] is None) else Qs[k].copy() for k in range(N)] if (debug_sweep1 and s == 0) else None
            u = mode_update_qr(X, Qs, Rs, n, variant, tau, order, kt)
            factors[n], lam, Qs[n], Rs[n] = u["A"], u["lam"], u["Q"], u["R"]
            flags |= u["flags"]
            if debug_sweep1 and s == 0:
                d = {k: u[k] for k in ("Yn", "Q0", "R0", "W", "Ahat", "A", "lam")}
                d["Qs_in"] = qs_in  # the Q_k this mode's Multi-TTM used (debug snapshot)
                debug.append(d)
            last = u
        if fit_mode == "fast":
            fits.append(fit_fast_qr(nX2, last["W"], last["Ahat"], last["R0"], Rs[N - 1], lam))
        else:
            fits.append(fit_direct(Xd, lam, factors))
    return dict(lam=lam, factors=factors, fits=fits, flags=flags, debug=debug, Qs=Qs, Rs=Rs,
                nX2=nX2)


def cp_als_ne(X, A0, sweeps, fit_mode="fast", kt=None, solve="chol", tau=-1.0):
    """CP-ALS with normal equations, Alg. 1, exactly `sweeps` sweeps; solve="pinv"
    is CP-ALS-PINV.  Fit: PAPER.md:417-425 (fast) or direct.  kt = (lam_x, B):
    Kruskal input instead of X (a direct fit forms X = full_tensor(lam_x, B))."""
    N = X.ndim if kt is None else len(kt[1])
    nX2 = float(np.dot(X.ravel(order="K"), X.ravel(order="K"))) if kt is None else ktensor_norm2(*kt)
    Xd = X if (kt is None or fit_mode == "fast") else full_tensor(*kt)
    factors = [np.array(A, dtype=np.float64, order="F") for A in A0]
    grams = [A.T @ A for A in factors]                            # line 3
    lam = np.ones(factors[0].shape[1])
    fits, flags = [], 0
    for s in range(sweeps):
        last = None
        for n in range(N):
            u = mode_update_ne(X, factors, grams, n, kt, solve, tau)
            factors[n], lam, grams[n] = u["A"], u["lam"], u["G"]
            flags |= u["flags"]
            last = u
        if fit_mode == "fast":
            fits.append(fit_fast_ne(nX2, last["M"], last["Ahat"], last["S"], grams[N - 1], lam))
        else:
            fits.append(fit_direct(Xd, lam, factors))
    return dict(lam=lam, factors=factors, fits=fits, flags=flags, nX2=nX2)


# ------------------------------------------------------------------ cost model §3.2
def qr_cost(N: int, R: int) -> int:
    """Dense QR of V_n with explicit Q0: 4 R^{N+1} (Eq. (QRcost); leading term)."""
    return 4 * R ** (N + 1)


def ttm_cost(dims, n: int, R: int, order=None) -> int:
    """Multi-TTM flops (Eq. (TTMcost), general form of reading 4): the j-th
    TTM over mode k_j costs 2 * (current tensor size) * R."""
    order = ttm_order(dims, n) if order is None else order
    cur = list(dims)
    total = 0
    for k in order:
        total += 2 * int(np.prod(cur, dtype=np.int64)) * R
        cur[k] = R
    return total
