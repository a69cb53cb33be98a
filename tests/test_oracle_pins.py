"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it pins and is chosen so that a plausible mistake in the oracle
(dropped term, wrong sign or index, transposed operand, wrong Kronecker order, wrong TTM
order, wrong solve side) fails at least one of them.  None of these tests retypes an oracle
formula: the reference values are hand-derived worked examples (tests/golden), brute-force
loops over the paper's index definitions, closed forms, library routines (LAPACK lstsq/pinv/
svd), invariants and textbook special cases.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2112_10855_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
rng = np.random.default_rng(12345)


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def rand_tensor(dims):
    return np.asfortranarray(rng.standard_normal(dims))


# ------------------------------------------------------------------ products (§2.2)
def test_kron_worked_example_and_index_formula():
    g = GOLD["kron"]
    assert np.array_equal(O.kron(np.array(g["A"], float), np.array(g["B"], float)), np.array(g["expected"], float))
    # PAPER.md:93 index formula, 1-based: [A(x)B](K(i-1)+k, M(j-1)+l) = A(i,j) B(k,l)
    A, B = rng.standard_normal((3, 2)), rng.standard_normal((4, 5))
    K, M = B.shape
    out = O.kron(A, B)
    for i, j, k, l in itertools.product(range(1, 4), range(1, 3), range(1, 5), range(1, 6)):
        assert out[K * (i - 1) + k - 1, M * (j - 1) + l - 1] == A[i - 1, j - 1] * B[k - 1, l - 1]


def test_khatri_rao_worked_example_and_columns():
    g = GOLD["khatri_rao"]
    assert np.array_equal(O.khatri_rao([np.array(g["A"], float), np.array(g["B"], float)]),
                          np.array(g["expected"], float))
    A, B, C = rng.standard_normal((3, 4)), rng.standard_normal((2, 4)), rng.standard_normal((5, 4))
    KR = O.khatri_rao([A, B, C])
    for r in range(4):   # column r is A(:,r) (x) B(:,r) (x) C(:,r)
        assert np.array_equal(KR[:, r], O.kron(O.kron(A[:, r:r + 1], B[:, r:r + 1]), C[:, r:r + 1])[:, 0])


def test_mixed_product_identity_eq_2_1():
    # PAPER.md:97-100 Eq. (2.1): (C (x) D)(A (.) B) = (CA) (.) (DB), A: KxJ, B: IxJ, C: IxK, D: JxI
    I, J, K = 3, 4, 5
    A, B = rng.standard_normal((K, J)), rng.standard_normal((I, J))
    C, D = rng.standard_normal((I, K)), rng.standard_normal((J, I))
    lhs = O.kron(C, D) @ O.khatri_rao([A, B])
    rhs = O.khatri_rao([C @ A, D @ B])
    assert rel(lhs, rhs) <= 1e-13


# --------------------------------------------------------- matricization and TTM
def test_matricize_kolda_bader_bruteforce_and_roundtrip():
    dims = (3, 4, 2, 3)
    X = rand_tensor(dims)
    for n in range(4):
        Xn = O.matricize(X, n)
        for idx in itertools.product(*[range(d) for d in dims]):
            col, J = 0, 1
            for k in range(4):       # reading 1: column sum_{k!=n} i_k J_k, J_k = prod_{m<k,m!=n} I_m
                if k == n:
                    continue
                col += idx[k] * J
                J *= dims[k]
            assert Xn[idx[n], col] == X[idx]
        assert np.array_equal(O.tensorize(Xn, dims, n), X)
    # SPEC.md example: dims [2,2,2], mode 3 -> row k = slice X(:,:,k) flattened column-major
    Y = rand_tensor((2, 2, 2))
    Y3 = O.matricize(Y, 2)
    for k in range(2):
        assert np.array_equal(Y3[k], Y[:, :, k].ravel(order="F"))


def test_ttm_bruteforce_definition():
    # Y(i1..j..iN) = sum_{i_n} X(i1..i_n..iN) U(j, i_n)
    dims = (3, 4, 2)
    X = rand_tensor(dims)
    for n in range(3):
        U = rng.standard_normal((5, dims[n]))
        Y = O.ttm(X, U, n)
        out_dims = list(dims)
        out_dims[n] = 5
        assert Y.shape == tuple(out_dims)
        for idx in itertools.product(*[range(d) for d in out_dims]):
            s = 0.0
            for i in range(dims[n]):
                src = list(idx)
                src[n] = i
                s += X[tuple(src)] * U[idx[n], i]
            assert abs(Y[idx] - s) <= 1e-13 * (1 + abs(s))
        assert np.allclose(O.matricize(Y, n), U @ O.matricize(X, n), rtol=0, atol=1e-13)
    assert np.array_equal(O.ttm(X, np.eye(4), 1), X)


def test_multi_ttm_equals_eq_2_2_kronecker_and_is_order_invariant():
    # PAPER.md:118-121 Eq. (2.2): Y_(n) = X_(n) (U_N (x) ... (x) U_{n+1} (x) U_{n-1} ... (x) U_1)^T
    for dims in [(4, 3, 5), (3, 4, 2, 3), (2, 3, 2, 2, 3)]:
        N = len(dims)
        X = rand_tensor(dims)
        Us = {k: rng.standard_normal((2, dims[k])) for k in range(N)}
        for n in range(N):
            sub = {k: Us[k] for k in range(N) if k != n}
            Y = O.multi_ttm(X, sub)
            K = None
            for k in range(N - 1, -1, -1):
                if k == n:
                    continue
                K = Us[k] if K is None else O.kron(K, Us[k])
            assert rel(O.matricize(Y, n), O.matricize(X, n) @ K.T) <= 1e-13
            for perm in itertools.permutations(sub.keys()):
                assert rel(O.multi_ttm(X, sub, order=perm), Y) <= 1e-13


def test_ttm_order_is_decreasing_dimension():
    assert O.ttm_order((30, 40, 50), 0) == [2, 1]
    assert O.ttm_order((50, 40, 30), 1) == [0, 2]
    assert O.ttm_order((8, 8, 8, 8), 1) == [3, 2, 0]      # ties: decreasing mode (reading 5)


# ------------------------------------------------------------------------- QR
def test_qr_pos_properties_and_special_cases():
    A = rng.standard_normal((50, 5))
    Q, R = O.qr_pos(A)
    assert rel(Q @ R, A) <= 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(5)) <= 1e-14
    assert np.allclose(np.tril(R, -1), 0) and np.all(np.diag(R) >= 0)
    Q, R = O.qr_pos(np.diag([3.0, 4.0]))
    assert np.allclose(R, np.diag([3.0, 4.0]), atol=1e-15) and np.allclose(Q, np.eye(2), atol=1e-15)
    Q, R = O.qr_pos(np.diag([-3.0, 4.0]))
    assert np.allclose(R, np.diag([3.0, 4.0]), atol=1e-15) and np.allclose(Q, np.diag([-1.0, 1.0]), atol=1e-15)


def _setup_factors(dims, R):
    A = [rng.standard_normal((d, R)) for d in dims]
    QR = [O.qr_pos(a) for a in A]
    return A, [q for q, _ in QR], [r for _, r in QR]


@pytest.mark.parametrize("dims", [(6, 5, 4), (5, 4, 3, 4), (3, 4, 3, 3, 4)])
def test_structured_qr_eq_Z_qr(dims):
    # Z_n = (Q_N (x)...(x) Q_1 skip n) Q0 R0, Q orthonormal, R0 upper triangular
    R = 3
    N = len(dims)
    A, Qs, Rs = _setup_factors(dims, R)
    for n in range(N):
        Z = O.khatri_rao([A[k] for k in range(N - 1, -1, -1) if k != n])
        Q0, R0 = O.structured_qr(Rs, n)
        K = None
        for k in range(N - 1, -1, -1):
            if k == n:
                continue
            K = Qs[k] if K is None else O.kron(K, Qs[k])
        Qfull = K @ Q0
        assert rel(Qfull @ R0, Z) <= 1e-13
        assert np.linalg.norm(Qfull.T @ Qfull - np.eye(R)) <= 1e-13
        assert np.allclose(np.tril(R0, -1), 0)
        # R0 equals the R of the explicitly formed Z_n (unique under diag >= 0, reading 6)
        _, Rz = O.qr_pos(Z)
        assert rel(R0, Rz) <= 1e-12


def test_vn_tree_groups_partition_and_sharing():
    # reading 36: hi and lo partition the retained modes {k != n}, each in decreasing (Khatri-Rao)
    # order, hi above lo; the group of the other half is the same for every mode of a half
    for N in range(2, 11):
        h = (N + 1) // 2
        for n in range(N):
            hi, lo = O.vn_tree_groups(N, n)
            assert sorted(hi + lo) == [k for k in range(N) if k != n]
            assert hi + lo == sorted(hi + lo, reverse=True)
            if n < h:
                assert hi == list(range(N - 1, h - 1, -1))            # shared by modes 0..h-1
            else:
                assert lo == list(range(h - 1, -1, -1))               # shared by modes h..N-1


@pytest.mark.parametrize("N,R", [(3, 3), (4, 3), (4, 5), (5, 3), (6, 2)])
def test_kr_group_qr_bruteforce_product(N, R):
    # P S = Khatri-Rao of the group, formed here entry by entry from PAPER.md:95's column rule
    # V(j, c) = prod_m R_m(j_m, c) (last factor fastest); P orthonormal, S upper triangular, diag >= 0
    _, _, Rs = _setup_factors((7,) * N, R)
    P, S = O.kr_group_qr(Rs)
    V = np.zeros((R ** N, R))
    for idx in itertools.product(range(R), repeat=N):       # idx[0] slowest
        j = 0
        for i in idx:
            j = j * R + i
        for c in range(R):
            V[j, c] = np.prod([Rs[m][idx[m], c] for m in range(N)])
    assert rel(P @ S, V) <= 1e-13
    assert np.linalg.norm(P.T @ P - np.eye(R)) <= 1e-13
    assert np.allclose(np.tril(S, -1), 0) and np.all(np.diag(S) >= 0)
    P1, S1 = O.kr_group_qr(Rs[:1])                          # one factor: (I, R_k)
    assert np.array_equal(P1, np.eye(R)) and np.array_equal(S1, Rs[0])


@pytest.mark.parametrize("dims,R", [((6, 5), 3), ((6, 5, 4), 3), ((5, 4, 3, 4), 4), ((3, 4, 3, 3, 4), 3),
                                    ((4, 4, 4, 4, 4, 4), 2), ((9, 9, 9, 9), 8)])
def test_tree_qr_equals_lapack_qr_of_vn(dims, R):
    # the tree QR across the Khatri-Rao factors reaches the thin QR of V_n, unique
    # under diag(R0) > 0 (reading 6): equal to LAPACK's QR of the explicitly formed V_n up to rounding
    N = len(dims)
    _, _, Rs = _setup_factors(dims, R)
    for n in range(N):
        V = O.kr_of_triangular(Rs, n)
        Q0, R0 = O.tree_qr(Rs, n)
        Qd, Rd = np.linalg.qr(V, mode="reduced")
        s = np.sign(np.diag(Rd))
        Qd, Rd = Qd * s[None, :], Rd * s[:, None]
        assert rel(R0, Rd) <= 1e-12 and rel(Q0, Qd) <= 1e-11
        assert rel(Q0 @ R0, V) <= 1e-13
        assert np.linalg.norm(Q0.T @ Q0 - np.eye(R)) <= 1e-13
        # Q0 keeps V_n's staircase support: zero where the row level > column
        rad = [Rs[k].shape[0] for k in range(N) if k != n]      # fastest factor first
        for j in range(V.shape[0]):
            lvl, t = 0, j
            for r in rad:
                lvl, t = max(lvl, t % r), t // r
            assert np.all(np.abs(Q0[j, :lvl]) <= 1e-13)


def test_structured_qr_identity_gives_selection_and_staircase_support():
    R, N = 3, 4
    Q0, R0 = O.structured_qr([np.eye(R)] * N, 0)
    assert np.allclose(R0, np.eye(R))
    sel = np.zeros((R ** 3, R))
    for r in range(R):
        sel[r + R * r + R * R * r, r] = 1.0   # selection matrix
    assert np.allclose(Q0, sel)
    # staircase: V_n and Q0 vanish on rows whose level max_k i_k exceeds the column
    R = 4
    _, _, Rs = _setup_factors((6, 6, 6, 6), R)
    V = O.kr_of_triangular(Rs, 2)
    Q0, _ = O.structured_qr(Rs, 2)
    nnz = 0
    for j in range(R ** 3):
        lvl = max(j % R, (j // R) % R, j // (R * R))
        for c in range(R):
            if lvl > c:
                assert V[j, c] == 0.0 and abs(Q0[j, c]) <= 1e-14
            else:
                nnz += 1
    assert nnz == sum(j ** 3 for j in range(1, R + 1))


# ----------------------------------------------------------------------- solves
def test_solve_qr_worked_example_and_lstsq():
    g = GOLD["solve_qr"]
    out = O.solve_qr(np.array(g["R0"], float), np.array(g["W"], float))
    assert np.allclose(out, np.array(g["expected"]), rtol=0, atol=1e-15)
    # the whole mode update equals LAPACK least squares min ||X_(n) - Ahat Z_n^T||
    dims, R = (5, 4, 6), 3
    X = rand_tensor(dims)
    A, Qs, Rs = _setup_factors(dims, R)
    for n in range(3):
        u = O.mode_update_qr(X, Qs, Rs, n)
        Z = O.khatri_rao([A[k] for k in range(2, -1, -1) if k != n])
        ref = np.linalg.lstsq(Z, O.matricize(X, n).T, rcond=None)[0].T
        assert rel(u["Ahat"], ref) <= 1e-13
        # orthogonal invariance: residual of Eq. (ls-qr-step) == residual of Eq. (ls_n)
        r1 = np.linalg.norm(O.matricize(X, n) - u["Ahat"] @ Z.T) ** 2
        r2 = np.linalg.norm(X) ** 2 - np.linalg.norm(u["W"]) ** 2
        assert abs(r1 - r2) <= 1e-12 * np.linalg.norm(X) ** 2


def test_solve_svd_examples_and_pinv():
    g = GOLD["solve_svd_truncate"]
    out, nt = O.solve_svd(np.array(g["R0"], float), np.array(g["W"], float), g["tau"])
    assert np.allclose(out, np.array(g["expected"]), atol=1e-15) and nt == g["ntrunc"]
    R0 = np.triu(rng.standard_normal((5, 5))) + 3 * np.eye(5)
    W = rng.standard_normal((7, 5))
    out, nt = O.solve_svd(R0, W, 0.0)
    assert nt == 0 and rel(out, O.solve_qr(R0, W)) <= 1e-13      # SPEC.md:220 cross-solver
    R0s = R0.copy()
    R0s[4, 4] = 1e-17
    out, nt = O.solve_svd(R0s, W, 1e-12)
    assert nt == 1 and rel(out, W @ np.linalg.pinv(R0s.T, rcond=1e-12)) <= 1e-12


def test_gram_solve_example_and_ne_equals_qr():
    g = GOLD["gram_solve"]
    X = rand_tensor((3, 3, 3))
    # mode_update_ne solves Ahat S = M; check on the worked S/M through the same Cholesky path
    import scipy.linalg
    S, M = np.array(g["S"], float), np.array(g["M"], float)
    L = np.linalg.cholesky(S)
    out = scipy.linalg.cho_solve((L, True), M.T).T
    assert np.allclose(out, g["expected"])
    # NE S_n = Z_n^T Z_n and NE == QR after one sweep on a well-conditioned problem
    conf, Xc, truth, init = synth.small_problem((12, 10, 8), 3, seed=7)
    Xt = O.as_tensor(Xc)
    grams = [a.T @ a for a in init]
    u = O.mode_update_ne(Xt, init, grams, 1)
    Z = O.khatri_rao([init[2], init[0]])
    assert rel(u["S"], Z.T @ Z) <= 1e-13
    a = O.cp_als_qr(Xt, init, 1)
    b = O.cp_als_ne(Xt, init, 1)
    for k in range(3):
        assert rel(a["factors"][k], b["factors"][k]) <= 1e-9
    assert abs(a["fits"][0] - b["fits"][0]) <= 1e-9


def test_ne_cholesky_fallback_flag():
    X = rand_tensor((4, 4, 4))
    f = [rng.standard_normal((4, 2)) for _ in range(3)]
    grams = [a.T @ a for a in f]
    grams[0] = np.array([[1.0, 0.5], [0.5, -1.0]])     # indefinite Hadamard factor
    u = O.mode_update_ne(X, f, grams, 2)
    assert u["flags"] & O.FLAG_NE_CHOL_FALLBACK
    assert rel(u["Ahat"] @ u["S"], u["M"]) <= 1e-12


# ------------------------------------------------------------ normalize / cache / fit
def test_normalize_contract():
    A = rng.standard_normal((6, 3))
    A[:, 1] = 0.0
    An, lam = O.normalize(A)
    assert np.allclose(np.linalg.norm(An[:, [0, 2]], axis=0), 1.0, atol=1e-15)
    assert lam[1] == 0 and np.array_equal(An[:, 1], np.eye(6)[:, 0]) and np.all(lam >= 0)
    assert np.allclose(An * lam, A)


def test_sweep_invariants_fast_vs_direct_and_pythagoras():
    conf, Xc, truth, init = synth.small_problem((10, 9, 8), 3, seed=3, eta=0.05)
    X = O.as_tensor(Xc)
    out = O.cp_als_qr(X, init, 4)
    outd = O.cp_als_qr(X, init, 4, fit_mode="direct")
    for f, fd in zip(out["fits"], outd["fits"]):
        assert abs(f - fd) <= 1e-10                     # PAPER.md:427 sqrt(eps) regime, residual >> 0
    for k in range(3):                                  # cache coherence, normalisation
        assert rel(out["Qs"][k] @ out["Rs"][k], out["factors"][k]) <= 1e-13
        assert np.allclose(np.linalg.norm(out["factors"][k], axis=0), 1.0, atol=1e-14)
    # Pythagoras for the QR variant: ||X||^2 = ||W_N||^2 + res^2 (derived from Eq. Z_qr)
    Qs, Rs = [None] + out["Qs"][1:], out["Rs"]
    u = O.mode_update_qr(X, out["Qs"], out["Rs"], 2)
    res2 = np.linalg.norm(X - O.full_tensor(u["lam"], out["factors"][:2] + [u["A"]])) ** 2
    assert abs(np.linalg.norm(X) ** 2 - np.linalg.norm(u["W"]) ** 2 - res2) <= 1e-12 * np.linalg.norm(X) ** 2


def test_fixed_point_rank1_and_monotone():
    # init = truth on a noiseless planted tensor -> one sweep returns the truth model
    conf, Xc, truth, _ = synth.small_problem((9, 8, 7), 3, seed=11, eta=0.0)
    X = O.as_tensor(Xc)
    out = O.cp_als_qr(X, truth, 1, fit_mode="direct")
    assert 1.0 - out["fits"][0] <= 1e-13
    # rank 1: exact after one sweep
    conf, Xc, truth, init = synth.small_problem((7, 6, 5), 1, seed=12, eta=0.0)
    out = O.cp_als_qr(O.as_tensor(Xc), init, 1, fit_mode="direct")
    assert 1.0 - out["fits"][0] <= 1e-13
    # monotone residual across sweeps (block coordinate descent), direct fit, noisy
    conf, Xc, truth, init = synth.small_problem((10, 9, 8), 3, seed=13, eta=0.1)
    X = O.as_tensor(Xc)
    for variant in ("QR", "SVD"):
        fits = O.cp_als_qr(X, init, 15, variant=variant, fit_mode="direct")["fits"]
        assert all(b >= a - 1e-12 for a, b in zip(fits, fits[1:]))
    fits = O.cp_als_ne(X, init, 15, fit_mode="direct")["fits"]
    assert all(b >= a - 1e-12 for a, b in zip(fits, fits[1:]))


def test_planted_noiseless_recovery():
    conf, Xc, truth, init = synth.small_problem((30, 40, 50), 5, seed=21, eta=0.0)
    X = O.as_tensor(Xc)
    out = O.cp_als_qr(X, init, 120, fit_mode="fast")
    fd = O.fit_direct(X, out["lam"], out["factors"])
    assert 1.0 - fd <= 1e-12


def test_n2_eckart_young():
    # N = 2: V_n = R_k, so CP-ALS-QR is alternating LS for a rank-R matrix factorisation whose
    # limit is the truncated SVD (Eckart-Young); relerr -> sqrt(sum_{i>R} s_i^2)/||X||.
    M = rng.standard_normal((60, 40))
    s = np.linalg.svd(M, compute_uv=False)
    init = [rng.standard_normal((60, 5)), rng.standard_normal((40, 5))]
    out = O.cp_als_qr(np.asfortranarray(M), init, 400, fit_mode="direct")
    target = np.sqrt(np.sum(s[5:] ** 2)) / np.linalg.norm(M)
    assert abs((1 - out["fits"][-1]) - target) <= 1e-9
    Q0, R0 = O.structured_qr([None, np.triu(rng.standard_normal((5, 5)))], 0)
    assert np.allclose(np.abs(Q0), np.eye(5))


def test_svd_exact_duplicate_min_norm_and_qr_illcond_flag():
    # Exact duplicate columns in every init factor except mode 1 -> Z_1 has rank R-1
    conf, Xc, truth, init = synth.small_problem((12, 11, 10), 3, seed=31, eta=0.01)
    X = O.as_tensor(Xc)
    dup = [a.copy() for a in init]
    for k in range(1, 3):
        dup[k][:, 1] = dup[k][:, 0]
    out = O.cp_als_qr(X, dup, 3, variant="SVD", tau=1e-12, fit_mode="direct")
    assert out["flags"] & O.FLAG_SVD_TRUNCATED
    for k in range(3):
        assert rel(out["factors"][k][:, 1], out["factors"][k][:, 0]) <= 1e-10
    assert all(b >= a - 1e-12 for a, b in zip(out["fits"], out["fits"][1:]))
    qr = O.cp_als_qr(X, dup, 1, variant="QR")
    assert qr["flags"] & O.FLAG_ILLCOND_R0


# ------------------------------------------------------------- CP-ALS-PINV
def test_pinv_svd_penrose_conditions_and_known_spectrum():
    # the four Moore-Penrose conditions (the definition of S^+) on a singular symmetric S and a
    # singular non-symmetric matrix, and the exact inverse when S is nonsingular
    B = rng.standard_normal((6, 4))
    for S in (B @ B.T, rng.standard_normal((6, 3)) @ rng.standard_normal((3, 6))):
        P, nt = O.pinv_svd(S)
        assert nt == 6 - np.linalg.matrix_rank(S)
        sc = np.linalg.norm(S)
        assert np.linalg.norm(S @ P @ S - S) <= 1e-12 * sc
        assert np.linalg.norm(P @ S @ P - P) <= 1e-12 * np.linalg.norm(P)
        assert np.linalg.norm((S @ P).T - S @ P) <= 1e-12
        assert np.linalg.norm((P @ S).T - P @ S) <= 1e-12
    G = rng.standard_normal((5, 5))
    S = G @ G.T + 5 * np.eye(5)
    P, nt = O.pinv_svd(S)
    assert nt == 0 and np.linalg.norm(S @ P - np.eye(5)) <= 1e-13
    # known spectrum: Q diag(1, 1e-3, 1e-17) Q^T -> the third value is dropped (<= 3 eps), the
    # second kept, P = Q diag(1, 1e3, 0) Q^T
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    S = Q @ np.diag([1.0, 1e-3, 1e-17]) @ Q.T
    P, nt = O.pinv_svd(S)
    assert nt == 1
    assert rel(P, Q @ np.diag([1.0, 1e3, 0.0]) @ Q.T) <= 1e-10


def test_cp_als_pinv_equals_cholesky_on_well_conditioned():
    conf, Xc, truth, init = synth.small_problem((9, 8, 7), 3, seed=21, eta=0.05)
    X = O.as_tensor(Xc)
    a = O.cp_als_ne(X, init, 3)
    b = O.cp_als_ne(X, init, 3, solve="pinv")
    assert b["flags"] == 0
    for k in range(3):
        assert rel(b["factors"][k], a["factors"][k]) <= 1e-10
    assert np.max(np.abs(np.array(a["fits"]) - np.array(b["fits"]))) <= 1e-12


def test_cp_als_pinv_exact_duplicate_is_the_min_norm_solution():
    # Exact duplicate columns (1, 2) of A_2, A_3: S_1 = Z_1^T Z_1 is singular.  The pseudo-inverse
    # solve gives the minimum-norm LS solution of min ||X_(1) - Ahat Z_1^T||, the same one the
    # QR-SVD route computes through the SVD of R0 -- an independent path --
    # and it keeps the two columns equal.
    conf, Xc, truth, init = synth.small_problem((10, 9, 8), 3, seed=33, eta=0.05)
    X = O.as_tensor(Xc)
    dup = [a.copy() for a in init]
    for k in (1, 2):
        dup[k][:, 1] = dup[k][:, 0]
    grams = [A.T @ A for A in dup]
    u = O.mode_update_ne(X, dup, grams, 0, solve="pinv")
    assert u["flags"] & O.FLAG_SVD_TRUNCATED
    Qs, Rs = [None] * 3, [None] * 3
    for k in (1, 2):
        Qs[k], Rs[k] = O.qr_pos(dup[k])
    v = O.mode_update_qr(X, Qs, Rs, 0, variant="SVD", tau=1e-12)
    assert rel(u["Ahat"], v["Ahat"]) <= 1e-9
    assert rel(u["Ahat"][:, 1], u["Ahat"][:, 0]) <= 1e-12
    Z = O.khatri_rao([dup[2], dup[1]])
    ref = np.linalg.lstsq(Z, O.matricize(X, 0).T, rcond=None)[0].T  # LAPACK min-norm LS
    assert rel(u["Ahat"], ref) <= 1e-9


# ---------------------------------------------------------------- generators / costs
def test_generators_closed_forms():
    c2 = synth.CONFIGS[2]
    small = synth.Config(2, (40, 30, 20), 10, "congruence", 0.9, 0.01, ("QR",), 1)
    A = synth.truth_factors(small)
    C = 0.9 * np.ones((10, 10)) + 0.1 * np.eye(10)
    for a in A:
        assert np.allclose(a.T @ a, C, atol=1e-13)
        ev = np.linalg.eigvalsh(a.T @ a)
        assert abs(ev[-1] / ev[0] - (1 + 9 * 0.9) / (1 - 0.9)) <= 1e-6 * (1 + 9 * 0.9) / 0.1
    p = synth.Config(4, (20, 20, 20), 8, "pair", 0.999, 0.0, ("SVD",), 1)
    for a in synth.truth_factors(p):
        assert abs(a[:, 0] @ a[:, 1] - 0.999) <= 1e-15 and np.allclose(np.linalg.norm(a, axis=0), 1)
    conf, Xc, truth, init = synth.small_problem((8, 7, 6), 2, seed=5, eta=0.01)
    clean = synth.planted_tensor(truth)
    assert abs(np.linalg.norm(Xc - clean) / np.linalg.norm(clean) - 0.01) <= 1e-14
    # planted tensor == Eq. (cp) written as a brute-force sum of outer products
    ref = np.einsum("ir,jr,kr->kji", *truth)
    assert rel(clean, ref) <= 1e-14
    assert c2.dims == (400, 400, 400)
    # chunked normal draws equal one-shot draws (cache / chunking safety)
    g1, g2 = np.random.default_rng(3), np.random.default_rng(3)
    assert np.array_equal(g1.standard_normal(1000), np.concatenate([g2.standard_normal(300), g2.standard_normal(700)]))


def test_cost_model_formulas():
    # Eq. (TTMcost) PAPER.md:389-393 for sorted dims I1 >= ... >= IN, mode n = N (last)
    dims, R = (9, 8, 7, 6), 3
    n = 3
    expect = 2 * 9 * 8 * 7 * 6 * R * (1 + R / 9 + R ** 2 / (9 * 8))
    assert O.ttm_cost(dims, n, R, order=[0, 1, 2]) == pytest.approx(expect, rel=1e-15)
    assert O.qr_cost(3, 32) == 4 * 32 ** 4


def test_survey_dryrun_anchor_c1():
    g = GOLD["dryrun_c1"]
    conf, Xc, truth, init = synth.make_problem(1, cache=False)
    X = O.as_tensor(Xc)
    assert abs(O.fit_direct(X, np.ones(5), truth) - g["fit_truth"]) <= 2e-10
    out = O.cp_als_qr(X, init, g["sweeps"])
    assert abs(out["fits"][0] - g["fit_sweep1"]) <= 2e-10
    assert abs(out["fits"][-1] - g["fit_last"]) <= 2e-10


# ------------------------------------------------------------ Kruskal input
@pytest.mark.parametrize("N,n", [(3, 9), (4, 8), (5, 6)])
def test_sine_of_sums_ktensor_closed_form(N, n):
    """The rank-2^{N-1} representation reproduces sin(x_1 + .. + x_N) on the grid
    x = 2 pi i / n pointwise."""
    lam, B = O.sine_of_sums_ktensor(N, n)
    assert len(lam) == 2 ** (N - 1) and all(b.shape == (n, 2 ** (N - 1)) for b in B)
    X = O.full_tensor(lam, B)
    x = 2 * np.pi * np.arange(n) / n
    grid = np.meshgrid(*([x] * N), indexing="ij")
    assert np.max(np.abs(X - np.sin(sum(grid)))) <= 1e-13


def test_ktensor_direct_fit_resolves_below_the_fast_fit_floor():
    """on the 4-way sine of sums (exact rank N = 4 representation exists,
    PAPER.md:599-602) CP-ALS-QR converges to machine precision; the DIRECT relative error of the
    Kruskal driver equals the residual against the closed form sin(x_1 + .. + x_4) (an
    independent formation of X) and falls below 1e-13, where the fast formula's
    ||X||^2 - 2<X,Xh> + ||Xh||^2 cancellation (relative error ~ sqrt(eps) ~ 1e-8) cannot see it."""
    N, n = 4, 16
    lam_x, B = O.sine_of_sums_ktensor(N, n)
    g = np.random.default_rng(7)
    A0 = [g.standard_normal((n, N)) for _ in range(N)]
    out = O.cp_als_qr(None, A0, 30, fit_mode="direct", kt=(lam_x, B))
    x = 2 * np.pi * np.arange(n) / n
    Xc = np.sin(sum(np.meshgrid(*([x] * N), indexing="ij")))
    Xh = O.full_tensor(out["lam"], out["factors"])
    rel_closed = np.linalg.norm((Xc - Xh).ravel()) / np.linalg.norm(Xc.ravel())
    assert abs((1 - out["fits"][-1]) - rel_closed) <= 1e-14
    assert 1 - out["fits"][-1] <= 1e-13
    fast = O.cp_als_qr(None, A0, 30, kt=(lam_x, B))
    assert np.max(np.abs(np.array(fast["fits"][:5]) - np.array(out["fits"][:5]))) <= 1e-7  # same iterates


@pytest.mark.parametrize("dims,S,R", [((7, 6, 5), 3, 2), ((5, 4, 6, 3), 4, 3)])
def test_ktensor_formulas_match_the_formed_tensor(dims, S, R):
    """||X||^2, W_n = Y_(n) Q0 and M_n = X_(n) Z_n computed from the factors
    equal the dense definitions on the formed tensor [[lam; B]]."""
    rng = np.random.default_rng(13)
    lam = rng.standard_normal(S)
    B = [rng.standard_normal((d, S)) for d in dims]
    X = O.full_tensor(lam, B)
    assert abs(O.ktensor_norm2(lam, B) - float(np.sum(X * X))) <= 1e-12 * float(np.sum(X * X))
    A = [rng.standard_normal((d, R)) for d in dims]
    Qs = [O.qr_pos(a)[0] for a in A]
    Rs = [O.qr_pos(a)[1] for a in A]
    for n in range(len(dims)):
        Q0, R0 = O.structured_qr(Rs, n)
        Wd = O.apply_q0(O.multi_ttm(X, {k: Qs[k].T for k in range(len(dims)) if k != n}), n, Q0)
        Wk = O.w_ktensor(lam, B, Qs, n, Q0)
        assert np.linalg.norm(Wk - Wd) <= 1e-12 * np.linalg.norm(Wd)
        Md = O.mttkrp(X, A, n)
        Mk = O.mttkrp_ktensor(lam, B, A, n)
        assert np.linalg.norm(Mk - Md) <= 1e-12 * np.linalg.norm(Md)


@pytest.mark.parametrize("variant", ["QR", "SVD", "NE"])
def test_ktensor_drivers_match_dense_drivers(variant):
    """CP-ALS(-QR) on a Kruskal input (X never formed) follows the dense-input algorithm on the
    formed tensor: same fits and factors up to rounding."""
    lam, B = O.sine_of_sums_ktensor(4, 10)
    X = O.full_tensor(lam, B)
    rng = np.random.default_rng(3)
    A0 = [rng.standard_normal((10, 4)) for _ in range(4)]
    if variant == "NE":
        a = O.cp_als_ne(None, A0, 3, kt=(lam, B))
        b = O.cp_als_ne(X, A0, 3)
    else:
        a = O.cp_als_qr(None, A0, 3, variant=variant, kt=(lam, B))
        b = O.cp_als_qr(X, A0, 3, variant=variant)
    assert np.max(np.abs(np.array(a["fits"]) - np.array(b["fits"]))) <= 1e-11
    for fa, fb in zip(a["factors"], b["factors"]):
        assert np.linalg.norm(fa - fb) <= 1e-9 * np.linalg.norm(fb)


# ------------------------------------------------------------------- score
def test_score_limits_and_invariances():
    """1 for equal Kruskal tensors, invariant to component permutation, column scaling (folded
    into the weights) and sign flips; 0 when the components are orthogonal in one mode; the
    weight penalty alone for equal directions with weights 1 vs 2."""
    rng = np.random.default_rng(5)
    R = 4
    A = [rng.standard_normal((d, R)) for d in (6, 7, 8)]
    lam = rng.uniform(1, 2, R)
    assert abs(O.score(lam, A, lam, A) - 1.0) <= 1e-14
    p = [2, 0, 3, 1]
    d = np.array([2.0, -1.0, 0.5, -3.0])       # per-component scale (and sign) in every mode
    B = [a[:, p] * d for a in A]
    assert abs(O.score(lam, A, lam[p] / np.abs(d) ** 3, B) - 1.0) <= 1e-12
    E = [np.eye(8)[:6, :R], np.eye(8)[:7, :R], np.eye(8)[:, :R]]
    Fo = [np.vstack([np.zeros((4, R)), np.ones((2, R))]), E[1], E[2]]  # mode-1 columns orthogonal to E's
    assert O.score(np.ones(R), E, np.ones(R), Fo) <= 1e-14
    assert abs(O.score(np.ones(R), E, 2.0 * np.ones(R), E) - 0.5) <= 1e-14


# ---------------------------------------------------- short modes (I_k < R)
def test_short_modes_mode_update_is_the_least_squares_minimizer():
    """I_k < R (the 10-way sine of sums has I_k = 8 < R = 10): qr_pos returns the economy QR
    (Q_k I_k x I_k, R_k I_k x R, trapezoidal), V_n has prod_{k != n} I_k rows, and the QR mode
    update still equals LAPACK least squares min ||X_(n) - Ahat Z_n^T|| whenever Z_n has full
    column rank."""
    dims, R = (2, 3, 7, 6), 4
    X = rand_tensor(dims)
    A, Qs, Rs = _setup_factors(dims, R)
    assert Rs[0].shape == (2, 4) and Qs[1].shape == (3, 3)
    for n in range(4):
        u = O.mode_update_qr(X, Qs, Rs, n)
        Z = O.khatri_rao([A[k] for k in range(3, -1, -1) if k != n])
        assert np.linalg.matrix_rank(Z) == R
        ref = np.linalg.lstsq(Z, O.matricize(X, n).T, rcond=None)[0].T
        assert rel(u["Ahat"], ref) <= 1e-12, n


def test_short_modes_zero_padding_is_exact():
    """The library stores a short mode's factor with max(I_k, R) rows, the extra rows zero, and
    pads the Kruskal input's B_k the same way: CP-ALS-QR on the padded problem follows the
    unpadded one exactly up to rounding (the padded rows of X are zero, so every Ahat keeps them
    zero; their rows of R_k are zero, so V_n's extra rows are zero).  Pinned here on the oracle."""
    rng2 = np.random.default_rng(8)
    dims, R, S = (3, 5, 4, 6), 5, 3
    lam = rng2.standard_normal(S)
    B = [rng2.standard_normal((d, S)) for d in dims]
    A0 = [rng2.standard_normal((d, R)) for d in dims]
    pad = lambda M, d: np.vstack([M, np.zeros((d - M.shape[0], M.shape[1]))])
    pd = [max(d, R) for d in dims]
    a = O.cp_als_qr(None, A0, 3, kt=(lam, B))
    b = O.cp_als_qr(None, [pad(M, d) for M, d in zip(A0, pd)], 3, kt=(lam, [pad(M, d) for M, d in zip(B, pd)]))
    assert np.max(np.abs(np.array(a["fits"]) - np.array(b["fits"]))) <= 1e-12
    for k in range(4):
        assert rel(b["factors"][k][:dims[k]], a["factors"][k]) <= 1e-11, k
        assert np.all(b["factors"][k][dims[k]:] == 0.0)


@pytest.mark.parametrize("N,n", [(3, 7), (5, 6), (10, 3)])
def test_sine_of_sums_rank_n_representation_closed_form(N, n):
    """Eq. (sinsum_rkd): the rank-N Kruskal tensor equals sin(x_1 + .. + x_N)
    entry by entry on the grid x = 2 pi i / n (and so equals the rank-2^{N-1} representation)."""
    lam, B = O.sine_of_sums_rank_n_ktensor(N, n)
    assert len(lam) == N and all(b.shape == (n, N) for b in B)
    X = O.full_tensor(lam, B)
    x = 2.0 * np.pi * np.arange(n) / n
    idx = np.indices((n,) * N)
    ref = np.sin(sum(x[idx[k]] for k in range(N)))
    assert np.max(np.abs(X - ref)) <= 1e-11
