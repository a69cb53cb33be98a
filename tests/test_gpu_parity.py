"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Tolerances (north_star / SURVEY.md §8(c)): Y relative Frobenius <= 1e-11; factors and lambda
after one sweep <= 1e-9; fit within 1e-8.  Small shapes span several tiles and ragged tails
(odd sizes disable the 16-byte load path, exercising the scalar kernels too)."""
import numpy as np
import pytest

import oracle as O
from paper_2112_10855_b200 import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


@pytest.fixture(scope="module")
def cp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_10855_b200 import cpqr
    return cpqr


SHAPES = [
    ((30, 40, 50), 5),        # C1 shape
    ((37, 29, 43), 7),        # odd sizes: scalar (non-VEC) kernels, ragged tiles
    ((64, 48, 40), 16),       # R = 16
    ((70, 66, 34), 32),       # R = 32 (4 M/N tiles), ragged fibres
    ((12, 10, 9, 11), 6),     # N = 4
    ((6, 7, 5, 6, 8), 3),     # N = 5
    ((60, 40), 5),            # N = 2
]


@pytest.mark.parametrize("dims,R", SHAPES)
def test_debug_mode_Y_Q0_W(cp, dims, R):
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=101 + len(dims) + R)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    N = len(dims)
    Qs, Rs = [None] * N, [None] * N
    for k in range(N):
        Qs[k], Rs[k] = O.qr_pos(init[k])
    for n in range(N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
        Q0o, R0o = O.structured_qr(Rs, n)
        assert rel(out["R0"], R0o) <= 1e-11
        assert rel(out["Q0"], Q0o) <= 1e-11
        Wo = O.apply_q0(Yo, n, Q0o)
        assert rel(out["W"], Wo) <= 1e-11
    s.close()


@pytest.mark.parametrize("m,R", [(50, 5), (1000, 32), (37, 7), (128, 16)])
def test_factor_qr(cp, m, R):
    A = np.random.default_rng(m + R).standard_normal((m, R))
    s = cp.CPQR((m, m), R, "QR")
    Q, Rf = s.debug_qr(A)
    Qo, Ro = O.qr_pos(A)
    assert rel(Rf, Ro) <= 1e-13 and rel(Q, Qo) <= 1e-12
    assert np.all(np.diag(Rf) >= 0)
    s.close()


def test_svd_solve_truncation_and_agreement(cp):
    rng = np.random.default_rng(5)
    R = 8
    R0 = np.triu(rng.standard_normal((R, R))) + 4 * np.eye(R)
    W = rng.standard_normal((40, R))
    s = cp.CPQR((40, 40), R, "SVD")
    out, nt = s.debug_svd_solve(R0, W, 0.0)
    ref, _ = O.solve_svd(R0, W, 0.0)
    assert nt == 0 and rel(out, ref) <= 1e-12
    R0[5, 5] = 1e-17 * abs(R0).max()
    R0[5, 6:] = 0.0
    out, nt = s.debug_svd_solve(R0, W, 1e-12)
    ref, ntr = O.solve_svd(R0, W, 1e-12)
    assert nt == ntr == 1 and rel(out, ref) <= 1e-10
    s.close()


@pytest.mark.parametrize("dims,R,variant", [
    ((30, 40, 50), 5, "QR"), ((37, 29, 43), 7, "SVD"), ((30, 40, 50), 5, "NE"),
    ((12, 10, 9, 11), 6, "QR"), ((6, 7, 5, 6, 8), 3, "SVD"), ((70, 66, 34), 32, "QR"), ((60, 40), 5, "QR"),
    ((21, 19, 17), 4, "NE"),
])
def test_sweeps_match_oracle(cp, dims, R, variant):
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=7 + R, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(init)
    fits = s.sweep(1)
    lam, A = s.get_factors()
    ref = O.cp_als_ne(X, init, 1) if variant == "NE" else O.cp_als_qr(X, init, 1, variant=variant)
    for k in range(len(dims)):
        assert rel(A[k], ref["factors"][k]) <= 1e-9, (k, rel(A[k], ref["factors"][k]))
    assert rel(lam, ref["lam"]) <= 1e-9
    assert abs(fits[0] - ref["fits"][0]) <= 1e-8
    more = s.sweep(4)
    ref5 = O.cp_als_ne(X, init, 5) if variant == "NE" else O.cp_als_qr(X, init, 5, variant=variant)
    assert np.max(np.abs(more - np.array(ref5["fits"][1:]))) <= 1e-8
    s.close()


def test_graph_and_eager_paths_agree_bitwise(cp):
    dims, R = (30, 40, 50), 5
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=3)
    outs = []
    for g in (True, False):
        s = cp.CPQR(dims, R, "QR", use_graph=g)
        s.set_tensor(Xc)
        s.set_factors(init)
        f = s.sweep(3)
        outs.append((f, s.get_factors()))
        s.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    for a, b in zip(outs[0][1][1], outs[1][1][1]):
        assert np.array_equal(a, b)


def test_direct_fit_and_torch_borrow(cp):
    import torch
    dims, R = (30, 40, 50), 5
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=8, eta=0.0)
    s = cp.CPQR(dims, R, "QR", fit_mode="direct")
    Xt = torch.from_numpy(Xc).cuda()
    s.set_tensor(Xt)  # borrowed device pointer
    s.set_factors(truth)
    f = s.sweep(1)
    assert 1.0 - f[0] <= 1e-13
    s.close()


def test_errors_are_reported(cp):
    # wide factors (I_k < R, reading 27) are accepted for Kruskal input only (short modes, the
    # 10-way sine of sums): a dense tensor is rejected
    w = cp.CPQR((4, 4, 4), 8, "QR")
    with pytest.raises(cp.CpqrError):
        w.set_tensor(np.zeros((4, 4, 4)))
    w.close()
    with pytest.raises(cp.CpqrError):
        cp.CPQR((4,) * 11, 2, "QR")           # N > 10
    s = cp.CPQR((10, 10, 10), 2, "QR")
    with pytest.raises(cp.CpqrError) as e:
        s.sweep(1)                           # no tensor yet
    assert e.value.status == 5
    s.close()


@pytest.mark.parametrize("dims,R", [((30, 40, 50), 5), ((64, 48, 40), 16), ((12, 10, 9, 11), 6)])
def test_register_staged_fallback_kernels(cp, dims, R, monkeypatch):
    """The non-TMA (register-staged) kernels used for odd/unaligned layouts, forced on even shapes."""
    monkeypatch.setenv("CPQR_NO_TMA", "1")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=55)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    f = s.sweep(2)
    ref = O.cp_als_qr(O.as_tensor(Xc), init, 2)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("dims,R,variant", [((16, 48, 20, 9), 8, "SVD"), ((32, 64, 20), 16, "QR"),
                                            ((24, 40, 12, 10), 5, "QR")])
def test_small_slice_kernel(cp, dims, R, variant):
    """I2 <= 64, I2 % 8 == 0: the whole-slice-per-warp TMA kernel (modes n >= 3)."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=91, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(init)
    N = len(dims)
    Qs = [O.qr_pos(a)[0] for a in init]
    for n in range(2, N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11
    f = s.sweep(2)
    ref = O.cp_als_qr(X, init, 2, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("dims,R,variant", [((30, 40, 50), 5, "QR"), ((70, 66, 34), 32, "QR"),
                                            ((12, 10, 9, 11), 6, "SVD")])
def test_householder_factor_qr_path(cp, dims, R, variant, monkeypatch):
    """Force the Householder TSQR factor QR (the CholeskyQR2 fallback) for whole sweeps."""
    monkeypatch.setenv("CPQR_FACTOR_QR", "householder")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=17, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(init)
    f = s.sweep(2)
    lam, A = s.get_factors()
    ref = O.cp_als_qr(X, init, 2, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    for k in range(len(dims)):
        assert rel(A[k], ref["factors"][k]) <= 1e-9
    s.close()


def test_factor_qr_fallback_on_ill_conditioned_panel(cp):
    """kappa(A) ~ 1e10: CholeskyQR2 must hand over to Householder; Q orthonormal, QR = A."""
    rng = np.random.default_rng(3)
    m, R = 300, 8
    U, _ = np.linalg.qr(rng.standard_normal((m, R)))
    Vt, _ = np.linalg.qr(rng.standard_normal((R, R)))
    A = U @ np.diag(np.logspace(0, -10, R)) @ Vt
    s = cp.CPQR((m, m), R, "QR")
    Q, Rf = s.debug_qr(A)
    assert np.linalg.norm(Q.T @ Q - np.eye(R)) <= 1e-13
    assert rel(Q @ Rf, A) <= 1e-14 and np.all(np.diag(Rf) >= 0)
    Qo, Ro = O.qr_pos(A)
    assert rel(Rf, Ro) <= 1e-12
    s.close()


@pytest.mark.parametrize("dims,R", [((30, 40, 50), 5), ((70, 66, 34), 32)])
def test_multi_kernel_cholqr_path(cp, dims, R, monkeypatch):
    """The 5-launch CholeskyQR2 path (used for factors taller than 8 x 256 rows), forced."""
    monkeypatch.setenv("CPQR_CQ_MULTI", "1")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=23, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    f = s.sweep(2)
    ref = O.cp_als_qr(X, init, 2)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("dims,R,fuse", [((34, 300, 40), 32, "1"), ((70, 66, 34), 32, "1"),
                                         ((64, 48, 40), 16, "0"), ((26, 270, 24, 25), 24, "1"),
                                         ((26, 270, 24, 25), 24, "0"), ((300, 40, 100), 32, "0")])
def test_fused_slice_on_and_off(cp, dims, R, fuse, monkeypatch):
    """Modes n >= 3 with the fused two-mode slice kernel forced on (NF = 4 for I2 >= 256, ragged
    last fibre block, per-warp Y in shared memory) or off (strided pass over the middle mode).
    (300, 40, 100): 200 strided units > the grid, so the stream-K last wave (pieces of 1-2 k-steps
    summed by the last arrival) runs."""
    monkeypatch.setenv("CPQR_SLICE", fuse)
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=73, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    N = len(dims)
    Qs = [O.qr_pos(a)[0] for a in init]
    for n in range(2, N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
    f = s.sweep(2)
    ref = O.cp_als_qr(X, init, 2)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("dims,R,variant,fuse", [((30, 40, 50), 5, "QR", None), ((70, 66, 34), 32, "QR", "0"),
                                                 ((64, 48, 40), 16, "QR", "1"), ((12, 10, 9, 11), 6, "SVD", None),
                                                 ((6, 7, 5, 6, 8), 3, "QR", None), ((300, 40, 100), 32, "QR", "0")])
def test_dimension_tree_multittm(cp, dims, R, variant, fuse, monkeypatch):
    """opt.mttm_tree: two passes over X per sweep, halves [0, h) / [h, N).
    Same mode updates as Alg. 2 up to rounding: factors after one sweep <= 1e-9 and fits within
    1e-8 of the oracle's per-mode CP-ALS-QR; Y of every mode (fresh tree plan) <= 1e-11."""
    if fuse is not None:
        monkeypatch.setenv("CPQR_SLICE", fuse)
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=29, eta=0.05)
    X = O.as_tensor(Xc)
    N = len(dims)
    s = cp.CPQR(dims, R, variant, tree=True)
    s.set_tensor(Xc)
    s.set_factors(init)
    Qs = [O.qr_pos(a)[0] for a in init]
    for n in range(N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(3)])
    ref = O.cp_als_qr(X, init, 4, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


def test_dimension_tree_graph_replay_matches_eager(cp):
    """The tree buffer carries state between the modes of a sweep: CUDA-graph replay and eager
    launches must agree bitwise."""
    dims, R = (40, 36, 30, 28), 8
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5, eta=0.05)
    out = []
    for g in (True, False):
        s = cp.CPQR(dims, R, "QR", tree=True, use_graph=g)
        s.set_tensor(Xc)
        s.set_factors(init)
        f = s.sweep(3)
        lam, A = s.get_factors()
        out.append((f, lam, A))
        s.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert all(np.array_equal(a, b) for a, b in zip(out[0][2], out[1][2]))


@pytest.mark.parametrize("dims,R,variant", [((40, 36, 30, 28), 8, "QR"), ((30, 28, 26, 24, 22), 5, "SVD"),
                                             ((40, 36, 30), 10, "QR")])
def test_dimension_tree_inline_vn_qr(cp, dims, R, variant, monkeypatch):
    """CPQR_VN_TREE=1: the tree's modes without an X pass run the V_n QR inline by the multi-CTA
    CholeskyQR2 (no side-stream fork), the fresh modes by the side-stream Householder K2.  The
    mode updates are Alg. 2's: factors after one sweep <= 1e-9, fits within 1e-8 of the oracle,
    graph replay bitwise equal to eager launches."""
    monkeypatch.setenv("CPQR_VN_TREE", "1")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=31, eta=0.05)
    X = O.as_tensor(Xc)
    out = []
    for g in (True, False):
        s = cp.CPQR(dims, R, variant, tree=True, use_graph=g)
        s.set_tensor(Xc)
        s.set_factors(init)
        f1 = s.sweep(1)
        lam, A = s.get_factors()
        f = np.concatenate([f1, s.sweep(3)])
        out.append((f, lam, A))
        s.close()
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    for k in range(len(dims)):
        assert rel(out[0][2][k], ref1["factors"][k]) <= 1e-9, (k, rel(out[0][2][k], ref1["factors"][k]))
    ref = O.cp_als_qr(X, init, 4, variant=variant)
    assert np.max(np.abs(out[0][0] - np.array(ref["fits"]))) <= 1e-8
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert all(np.array_equal(a, b) for a, b in zip(out[0][2], out[1][2]))


@pytest.mark.parametrize("dims,R,force_lu", [((40, 36, 30), 10, False), ((44, 41, 38), 20, False),
                                              ((12, 10, 9, 11), 6, False), ((40, 36, 30), 10, True)])
def test_ne_variant_tail(cp, dims, R, force_lu, monkeypatch):
    """Normal-equations CP-ALS (Alg. 1) at RB = 16 / 32 and N = 4 (blocked row solves
    y L^T = m, x L = y on the row panel), and the LU-with-partial-pivoting path (reading 18) forced
    on a positive-definite S: fits within 1e-8, factors after one sweep <= 1e-9 of the oracle."""
    if force_lu:
        monkeypatch.setenv("CPQR_NE_FORCE_LU", "1")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=61, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "NE")
    s.set_tensor(Xc)
    s.set_factors(init)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_ne(X, init, 1)
    for k in range(len(dims)):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(3)])
    ref = O.cp_als_ne(X, init, 4)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    if force_lu:
        assert s.flags & 2  # NE_CHOL_FALLBACK reported
    s.close()


def test_run_to_run_determinism(cp):
    """Every reduction is fixed-order, so repeated runs are bitwise identical.  N = 5 with a
    48-row strided step (many TMA boxes partly out of bounds) and back-to-back graph replays vs one
    sweep per call: a race or a TMA misuse shows up as a second distinct result."""
    dims, R = (48, 20, 12, 10, 8), 8
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=97, eta=0.05)
    s = cp.CPQR(dims, R, "SVD")
    s.set_tensor(Xc)
    s.set_factors(init)
    ref = s.debug_mode(0)["Y"]
    for _ in range(150):
        assert np.array_equal(s.debug_mode(0)["Y"], ref)
    fa = s.sweep(12)
    s.close()
    s = cp.CPQR(dims, R, "SVD")
    s.set_tensor(Xc)
    s.set_factors(init)
    fb = np.concatenate([s.sweep(1) for _ in range(12)])
    s.close()
    assert np.array_equal(fa, fb)


def test_householder_fallback_inside_captured_graph(cp):
    """Factors with congruence 1 - 1e-10 (kappa(A_n) > 1e5): CholeskyQR2 fails its guard and the
    device-flag-gated Householder TSQR kernels take over, inside the captured CUDA graph and in
    eager launches alike.  Both must agree bitwise and follow the oracle.  (A conditional graph
    node for this branch measured slower than the three early-exiting kernels: C2 -4 %.)"""
    dims, R = (40, 36, 30), 4
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=83, eta=1e-6, kind="congruence", c=1.0 - 1e-10)
    Xt = O.as_tensor(Xc)
    res = []
    for g in (True, False):
        s = cp.CPQR(dims, R, "QR", use_graph=g)
        s.set_tensor(Xc)
        s.set_factors(truth)  # start at the (ill-conditioned) planted factors
        f = s.sweep(3)
        lam, A = s.get_factors()
        res.append((f, lam, A))
        s.close()
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert all(np.array_equal(a, b) for a, b in zip(res[0][2], res[1][2]))
    ref = O.cp_als_qr(Xt, truth, 3)
    assert np.max(np.abs(res[0][0] - np.array(ref["fits"]))) <= 1e-8


@pytest.mark.parametrize("dims,R,variant", [((30, 40, 50), 1, "QR"), ((12, 10, 9, 11), 1, "QR"),
                                            ((8, 8, 8), 8, "QR"), ((5, 5, 5, 5), 5, "SVD"),
                                            ((3,) * 8, 2, "QR"), ((40, 3), 3, "QR")])
def test_edge_shapes(cp, dims, R, variant):
    """Degenerate and extreme shapes: rank one, square factors (I_k = R), the maximum order N = 8,
    N = 2 with a square factor (exact fit 1).  Fits within 1e-8 and factors <= 1e-9 of the oracle."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5, eta=0.01)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(init)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    for k in range(len(dims)):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(2)])
    ref = O.cp_als_qr(X, init, 3, variant=variant)
    # an exact fit (N = 2, square factor) puts ||X||^2 - 2<X,Xh> + ||Xh||^2 at the rounding level,
    # where the fast fit only resolves sqrt(eps) ~ 1.5e-8: there both sides must sit
    # at fit 1 within that floor (sqrt(8 eps) = 4.2e-8); elsewhere within 1e-8
    rf = np.array(ref["fits"])
    tol = np.where(rf > 1 - 1e-7, 4.3e-8, 1e-8)
    assert np.all(np.abs(f - rf) <= tol), (f, rf)
    s.close()


def test_zero_tensor(cp):
    """X = 0 (degenerate: every W is 0).  QR: the factors collapse to e_1 columns, R0 is singular
    and the oracle's back substitution produces NaN; the library reports EDIVERGED with the
    ILLCOND_R0 flag.  SVD: everything is truncated, lambda = 0, and the fit is 0/0 = NaN in both."""
    import warnings
    dims, R = (6, 5, 4), 2
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5)
    Z = np.zeros_like(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Z)
    s.set_factors(init)
    with pytest.raises(cp.CpqrError) as ei:
        s.sweep(2)
    assert "EDIVERGED" in str(ei.value) and s.flags & 1
    s.close()
    s = cp.CPQR(dims, R, "SVD")
    s.set_tensor(Z)
    s.set_factors(init)
    f = s.sweep(2)
    lam, A = s.get_factors()
    assert np.all(np.isnan(f)) and np.all(lam == 0.0) and s.flags & 4
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = O.cp_als_qr(O.as_tensor(Z), init, 2, variant="SVD")
    assert np.all(ref["lam"] == 0.0) and np.all(np.isnan(ref["fits"]))
    s.close()


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("dims,R,variant,kind,c", [((30, 40, 50), 5, "QR", "normal", 0.0),
                                                   ((12, 10, 9, 11), 6, "QR", "normal", 0.0),
                                                   ((9, 8, 7, 8, 9), 4, "SVD", "normal", 0.0),
                                                   ((40, 36, 30), 4, "QR", "congruence", 1.0 - 1e-10),
                                                   ((12, 11, 9, 10, 13), 8, "QR", "normal", 0.0),
                                                   ((24, 20, 18, 22), 16, "QR", "normal", 0.0)])
def test_vn_qr_by_cholesky_qr2(cp, dims, R, variant, kind, c, compact, monkeypatch):
    """High-rank V_n QR path, forced on small shapes: V_n formed densely and
    factored under the kappa guard by the one-launch cluster CholeskyQR2 (k_cq_compact, up to 8 CTAs
    x 512 rows: the J = 4096 cases fill it) or the multi-kernel CholeskyQR2 (compact=False); with congruence 1 - 1e-10 the
    guard rejects V_n and the staircase Householder K2 runs instead (device flag).  Q0 orthonormal,
    V_n = Q0 R0 with diag(R0) > 0 (the unique thin QR), sweeps follow the oracle."""
    monkeypatch.setenv("CPQR_VN_QR", "cq")
    monkeypatch.setenv("CPQR_VN_COMPACT", "1" if compact else "0")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=67, eta=0.05, kind=kind, c=c)
    X = O.as_tensor(Xc)
    start = truth if kind == "congruence" else init
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(start)
    Rs = [O.qr_pos(a)[1] for a in start]
    for n in range(len(dims)):
        d = s.debug_mode(n)
        Q0o, R0o = O.structured_qr(Rs, n)
        assert np.linalg.norm(d["Q0"].T @ d["Q0"] - np.eye(R)) <= 1e-12
        assert rel(d["R0"], R0o) <= 1e-9, (n, rel(d["R0"], R0o))
        assert rel(d["Q0"], Q0o) <= 1e-9, (n, rel(d["Q0"], Q0o))
    f = s.sweep(3)
    ref = O.cp_als_qr(X, start, 3, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


def test_high_rank_sweeps(cp):
    """A high-rank problem (R^{N-1} R = 1.05e6 >= the 2e5 threshold, so the CholeskyQR2 V_n QR runs
    by default): 40^4, R = 32.  Factors after one sweep <= 1e-9, fits within 1e-8 of the oracle."""
    dims, R = (40, 40, 40, 40), 32
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=71, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, init, 1)
    for k in range(4):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(2)])
    ref = O.cp_als_qr(X, init, 3)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("N,n,R,variant", [(4, 16, 4, "QR"), (4, 16, 4, "SVD"), (4, 16, 4, "NE"),
                                           (5, 8, 5, "QR"), (3, 40, 3, "QR")])
def test_kruskal_input(cp, N, n, R, variant):
    """Kruskal-tensor input: the sine-of-sums tensor
    (rank 2^{N-1}) or a random rank-5 Kruskal tensor (N = 3), never formed on the
    GPU.  Factors after one sweep <= 1e-9 and fits within 1e-8 of the oracle's Kruskal drivers,
    which are pinned to the dense algorithm on the formed tensor; also equal to the GPU's own
    dense path on the formed tensor."""
    if N == 3:
        rng = np.random.default_rng(41)
        lam_x, B = rng.standard_normal(5), [rng.standard_normal((n, 5)) for _ in range(N)]
    else:
        lam_x, B = O.sine_of_sums_ktensor(N, n)
    rng = np.random.default_rng(9)
    A0 = [rng.standard_normal((n, R)) for _ in range(N)]
    dims = (n,) * N
    s = cp.CPQR(dims, R, variant)
    s.set_ktensor(lam_x, B)
    s.set_factors(A0)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    if variant == "NE":
        ref1, ref = O.cp_als_ne(None, A0, 1, kt=(lam_x, B)), O.cp_als_ne(None, A0, 4, kt=(lam_x, B))
    else:
        ref1 = O.cp_als_qr(None, A0, 1, variant=variant, kt=(lam_x, B))
        ref = O.cp_als_qr(None, A0, 4, variant=variant, kt=(lam_x, B))
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(3)])
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()
    # the GPU's dense path on the formed tensor follows the same trajectory
    Xf = O.full_tensor(lam_x, B)
    sd = cp.CPQR(dims, R, variant)
    sd.set_tensor(np.ascontiguousarray(np.transpose(Xf)))
    sd.set_factors(A0)
    fd = sd.sweep(4)
    sd.close()
    assert np.max(np.abs(fd - f)) <= 1e-9


def test_kruskal_input_errors(cp):
    lam_x, B = O.sine_of_sums_ktensor(4, 8)
    s = cp.CPQR((8,) * 4, 3, "QR")
    s.set_ktensor(lam_x, B)
    s.set_factors([np.eye(8)[:, :3]] * 4)
    with pytest.raises(cp.CpqrError):
        s.debug_mode(0)
    s.close()
    s = cp.CPQR((8,) * 4, 3, "QR", fit_mode="direct", world=2, comm="local")
    with pytest.raises(cp.CpqrError):  # Kruskal input is single-GPU
        s.set_ktensor(lam_x, B)
    s.close()


@pytest.mark.parametrize("N,n,variant", [(4, 16, "QR"), (4, 16, "SVD"), (4, 16, "NE"), (4, 16, "PINV"),
                                         (5, 10, "QR"), (5, 10, "PINV")])
def test_kruskal_direct_relative_error(cp, N, n, variant):
    """The DIRECT relative error for Kruskal input: the
    residual is evaluated entry by entry from both Kruskal tensors' factors on the GPU (the
    tensor is never formed).  Per sweep it matches the oracle (which forms X) within 1e-8; on the
    converged sine of sums (rank N fit to the rank-2^{N-1} input) it resolves
    relative errors far below the fast fit's sqrt(eps) floor: QR-based variants
    reach <= 1e-13, as in the paper's Fig. 4.2/4.3 curves."""
    lam_x, B = O.sine_of_sums_ktensor(N, n)
    rng = np.random.default_rng(7)
    A0 = [rng.standard_normal((n, N)) for _ in range(N)]
    s = cp.CPQR((n,) * N, N, variant, fit_mode="direct")
    s.set_ktensor(lam_x, B)
    s.set_factors(A0)
    f = s.sweep(30)
    s.close()
    if variant in ("NE", "PINV"):
        ref = O.cp_als_ne(None, A0, 30, fit_mode="direct", kt=(lam_x, B), solve="pinv" if variant == "PINV" else "chol")
    else:
        ref = O.cp_als_qr(None, A0, 30, variant=variant, fit_mode="direct", kt=(lam_x, B))
    relerr, rref = 1 - f, 1 - np.array(ref["fits"])
    assert np.max(np.abs(relerr - rref)) <= 1e-8, (relerr, rref)
    if variant in ("QR", "SVD"):
        assert relerr[-1] <= 1e-13 and rref[-1] <= 1e-13, (relerr[-1], rref[-1])
    assert abs(relerr[-1] - rref[-1]) <= 1e-12


def _batched_inputs(dims, R, seeds, **kw):
    import torch
    Xs, A0s, truths = [], [], []
    for sd in seeds:
        conf, Xc, truth, init = synth.small_problem(dims, R, seed=sd, **kw)
        Xs.append(Xc)
        A0s.append(init)
        truths.append(truth)
    X = torch.from_numpy(np.stack(Xs)).cuda()
    A0 = [torch.from_numpy(np.stack([np.ascontiguousarray(a[k].T) for a in A0s])).cuda() for k in range(3)]
    return Xs, A0s, X, A0


@pytest.mark.parametrize("dims,R,kw", [((20, 18, 16), 3, dict(eta=0.05)),
                                       ((12, 14, 10), 5, dict(eta=1e-3, kind="congruence", c=0.99))])
def test_batched_one_cta_per_problem(cp, dims, R, kw):
    """cpqr_batched_qr: each CTA runs a whole CP-ALS-QR solve.  With tol = 0
    it runs exactly max_iters sweeps: factors and lambda after 1 sweep <= 1e-9, fits within 1e-8
    of the oracle for every sweep, for every problem of the batch."""
    seeds = [101, 102, 103, 104, 105, 106]
    Xs, A0s, X, A0 = _batched_inputs(dims, R, seeds, **kw)
    for sweeps in (1, 6):
        A, lam, fits, iters = cp.batched_qr(X, A0, R, max_iters=sweeps, tol=0.0)
        A = [a.cpu().numpy() for a in A]
        lam, fits, iters = lam.cpu().numpy(), fits.cpu().numpy(), iters.cpu().numpy()
        assert np.all(iters == sweeps)
        for p in range(len(seeds)):
            ref = O.cp_als_qr(O.as_tensor(Xs[p]), A0s[p], sweeps)
            assert np.max(np.abs(fits[p] - np.array(ref["fits"]))) <= 1e-8, (p, fits[p], ref["fits"])
            if sweeps == 1:
                for k in range(3):
                    assert rel(A[k][p].T, ref["factors"][k]) <= 1e-9, (p, k)
                assert rel(lam[p], ref["lam"]) <= 1e-9


def test_batched_stopping_rule_and_paper_shape(cp):
    """tol > 0: a problem stops at the first sweep whose fit change is below tol (NaN afterwards);
    the paper's 50^3 rank-5 shape runs and matches the oracle's fits."""
    Xs, A0s, X, A0 = _batched_inputs((50, 50, 50), 5, [201, 202], eta=1e-4)
    A, lam, fits, iters = cp.batched_qr(X, A0, 5, max_iters=40, tol=1e-9)
    fits, iters = fits.cpu().numpy(), iters.cpu().numpy()
    for p in range(2):
        k = int(iters[p])
        f = fits[p, :k]
        assert np.all(np.isnan(fits[p, k:]))
        if k < 40:
            assert abs(f[-1] - f[-2]) < 1e-9 and np.all(np.abs(np.diff(f[:-1])) >= 1e-9)
        ref = O.cp_als_qr(O.as_tensor(Xs[p]), A0s[p], k)
        assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8


def test_profile_and_timings(cp, monkeypatch):
    """opt.profile = 1 (the paper's per-phase time breakdown): eager sweeps with
    events around each phase.  cpqr_get_timings returns the same seven per-phase ms as
    cpqr_get_profile; the stream-X pass is timed, the algorithmic bytes equal N passes over X, and
    the fits equal those of the graph path bitwise (profiling changes launch order only)."""
    dims, R = (40, 36, 30), 6
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=13, eta=0.05)
    monkeypatch.setenv("CPQR_OVERLAP", "0")  # profiling runs the serial schedule (same plans)
    fits = []
    for prof in (True, False):
        s = cp.CPQR(dims, R, "QR", profile=prof, use_graph=not prof)
        s.set_tensor(Xc)
        s.set_factors(init)
        fits.append(s.sweep(3))
        if prof:
            t = s.timings()
            p = s.profile(reset=True)
            assert len(t) == 7 and t == p["ms"]
            assert t[0] > 0.0 and all(v >= 0.0 for v in t)
            assert t[2] > 0.0  # the fused factor-QR tail is timed (it was never written in round 1)
            assert p["bytes0"] == len(dims) * 8.0 * np.prod(dims)
            # launches per phase add up to the launches of the profiled sweeps
            assert sum(p["launches"]) > 0 and p["launches"][2] >= 1
            assert s.timings() == [0.0] * 7  # reset by profile(reset=True)
        s.close()
    assert np.array_equal(fits[0], fits[1])


@pytest.mark.parametrize("dims,R", [((24, 200, 6, 5), 4), ((40, 130, 7, 6), 6), ((18, 300, 5, 4), 3)])
def test_slice_kernel_split_slices(cp, dims, R):
    """Fused slice pass (modes 1 and 2 in one TMA pass, k_slice_tma) where a slice spans several
    128- or 256-fibre units (I_2 = 130, 200, 300) and I_1 is ragged against the 16-row k-stage:
    every slice's Y is summed from per-CTA partial slots by the fix-up kernel.  Y of the modes that
    take the slice pass (n >= 2) <= 1e-11 against the oracle's Multi-TTM, and one sweep's factors
    <= 1e-9."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=53, eta=0.05)
    X = O.as_tensor(Xc)
    N = len(dims)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    Qs = [O.qr_pos(a)[0] for a in init]
    for n in range(2, N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
    s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, init, 1)
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    s.close()


@pytest.mark.parametrize("dims,R", [((30, 40, 50), 5), ((12, 10, 9, 11), 4), ((9, 8, 7, 6, 8), 4)])
def test_svd_truncation_exact_duplicate(cp, dims, R):
    """A truncating QR-SVD sweep on the GPU (SURVEY.md 8(c) 'Solve (SVD) (ii)').
    Columns 1 and 2 of every initial factor but the first (unused, Alg. 2 line 2) are equal, so
    Z_1 and R0 have rank R-1: the SVD with tau = 1e-12 drops one singular value and the LS
    solution is the unique minimum-norm one, which keeps the two columns equal.  Both sides must
    set SVD_TRUNCATED and agree (factors <= 1e-9 after one sweep, fits within 1e-8 on every
    sweep); the QR variant flags R0 as numerically singular (ILLCOND_R0) or diverges."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=31 + len(dims), eta=0.01)
    X = O.as_tensor(Xc)
    N = len(dims)
    dup = [a.copy() for a in init]
    for k in range(1, N):
        dup[k][:, 1] = dup[k][:, 0]
    s = cp.CPQR(dims, R, "SVD", svd_tau=1e-12)
    s.set_tensor(Xc)
    s.set_factors(dup)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, dup, 1, variant="SVD", tau=1e-12)
    assert ref1["flags"] & O.FLAG_SVD_TRUNCATED
    assert s.flags & cp.FLAG_SVD_TRUNCATED
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
        assert rel(A[k][:, 1], A[k][:, 0]) <= 1e-10, (k, rel(A[k][:, 1], A[k][:, 0]))
    assert rel(lam, ref1["lam"]) <= 1e-9
    f = np.concatenate([f1, s.sweep(2)])
    ref = O.cp_als_qr(X, dup, 3, variant="SVD", tau=1e-12)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8, (f, ref["fits"])
    lam, A = s.get_factors()
    for k in range(N):
        assert rel(A[k][:, 1], A[k][:, 0]) <= 1e-10
    s.close()
    q = cp.CPQR(dims, R, "QR")
    q.set_tensor(Xc)
    q.set_factors(dup)
    try:
        q.sweep(1)
        assert q.flags & cp.FLAG_ILLCOND_R0, q.flags
    except cp.CpqrError as e:
        assert e.status == 6 and q.flags & cp.FLAG_ILLCOND_R0, e
    q.close()


def test_edivergred_cleared_by_set_factors(cp):
    """After EDIVERGED (X = 0 makes R0 singular) a new tensor and cpqr_set_factors restore a finite
    state: the sticky non-finite condition and the flags are cleared (cpqr.h)."""
    dims, R = (6, 5, 4), 2
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(np.zeros_like(Xc))
    s.set_factors(init)
    with pytest.raises(cp.CpqrError):
        s.sweep(1)
    s.set_tensor(Xc)
    s.set_factors(init)
    assert s.flags == 0
    f = s.sweep(2)
    ref = O.cp_als_qr(O.as_tensor(Xc), init, 2)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("variant", ["QR", "SVD"])
@pytest.mark.parametrize("dims,R", [((20000, 33, 40), 32), ((40, 33, 20000), 32), ((13000, 9, 10), 8)])
def test_tall_factor_mode(cp, dims, R, variant):
    """One factor far taller than the shared-memory tails (I_n > 3200 at R = 32 took an
    unfused path that returned EINVAL with the fast fit and overran a partials buffer): the
    multi-kernel CholeskyQR2 handles it in the first mode and in the last (with the fused fast
    fit)."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=11 + R, eta=0.01)
    A0 = [a.copy() for a in init]
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(A0)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    X = O.as_tensor(Xc)
    ref1 = O.cp_als_qr(X, A0, 1, variant=variant)
    for k in range(3):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(1)])
    ref = O.cp_als_qr(X, A0, 2, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("m,R", [(20000, 32), (13000, 8)])
def test_tall_factor_qr_fallback(cp, m, R):
    """A tall panel with kappa ~ 1e10: the multi-kernel CholeskyQR2 rejects it and the gated
    one-CTA global-memory Householder (k_tall_fallback) factors it (Q orthonormal, QR = A, R as
    LAPACK's up to the column scaling's conditioning)."""
    rng = np.random.default_rng(m)
    U, _ = np.linalg.qr(rng.standard_normal((m, R)))
    Vt, _ = np.linalg.qr(rng.standard_normal((R, R)))
    A = U @ np.diag(np.logspace(0, -10, R)) @ Vt
    s = cp.CPQR((m, m), R, "QR")
    Q, Rf = s.debug_qr(A)
    assert np.linalg.norm(Q.T @ Q - np.eye(R)) <= 1e-13
    assert rel(Q @ Rf, A) <= 1e-14 and np.all(np.diag(Rf) >= 0)
    Qo, Ro = O.qr_pos(A)
    assert rel(Rf, Ro) <= 1e-12
    s.close()


def test_tall_factor_forced_householder(cp, monkeypatch):
    """The very-tall Householder path with CholeskyQR2 disabled (CPQR_FACTOR_QR=householder):
    k_solve_rows forms Ahat and its partials (buffer sized for any I_n), k_tall_fallback the rest."""
    monkeypatch.setenv("CPQR_FACTOR_QR", "householder")
    dims, R = (9000, 33, 64), 32
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=3, eta=0.01)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    f = s.sweep(2)
    lam, A = s.get_factors()
    X = O.as_tensor(Xc)
    ref = O.cp_als_qr(X, init, 2)
    for k in range(3):
        assert rel(A[k], ref["factors"][k]) <= 1e-9, (k, rel(A[k], ref["factors"][k]))
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


def test_debug_calls_leave_state_and_bound_m(cp):
    """cpqr_debug_svd_solve restores R0 and the flags; m > max(dims) is rejected."""
    dims, R = (12, 10, 9), 4
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=8)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    f_a = s.sweep(1)
    g = np.random.default_rng(1)
    R0 = np.triu(g.standard_normal((R, R)))
    R0[3, 3] = 0.0
    W = g.standard_normal((12, R))
    out, nt = s.debug_svd_solve(R0, W, 1e-12)
    assert nt == 1 and s.flags == 0
    with pytest.raises(cp.CpqrError):
        s.debug_svd_solve(R0, g.standard_normal((13, R)), 1e-12)
    with pytest.raises(cp.CpqrError):
        s.debug_qr(g.standard_normal((13, R)))
    f_b = s.sweep(1)
    s.close()
    t = cp.CPQR(dims, R, "QR")
    t.set_tensor(Xc)
    t.set_factors(init)
    f_c = t.sweep(2)
    t.close()
    assert np.array_equal(np.concatenate([f_a, f_b]), f_c)


@pytest.mark.parametrize("dims,R", [((30, 40, 50), 5), ((12, 10, 9, 11), 4)])
def test_pinv_exact_duplicate(cp, dims, R):
    """CP-ALS-PINV on an exactly singular S_n (columns 1 and 2 of the initial
    factors equal): the pseudo-inverse drops one singular value (SVD_TRUNCATED on both sides),
    gives the minimum-norm solution (the two columns stay equal) and matches the oracle."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=61 + len(dims), eta=0.01)
    X = O.as_tensor(Xc)
    N = len(dims)
    dup = [a.copy() for a in init]
    for k in range(N):
        dup[k][:, 1] = dup[k][:, 0]
    s = cp.CPQR(dims, R, "PINV", svd_tau=1e-12)
    s.set_tensor(Xc)
    s.set_factors(dup)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_ne(X, dup, 1, solve="pinv", tau=1e-12)
    assert ref1["flags"] & O.FLAG_SVD_TRUNCATED and s.flags & cp.FLAG_SVD_TRUNCATED
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
        assert rel(A[k][:, 1], A[k][:, 0]) <= 1e-10
    f = np.concatenate([f1, s.sweep(2)])
    ref = O.cp_als_ne(X, dup, 3, solve="pinv", tau=1e-12)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("mode", ["1", "0"])
@pytest.mark.parametrize("dims,R,world", [((70, 66, 34), 32, 1), ((300, 260, 64), 32, 8), ((97, 130, 40), 10, 1),
                                          ((64, 48, 40, 24), 16, 4)])
def test_streamk_strided_split(cp, dims, R, world, mode, monkeypatch):
    """The strided stream kernel's stream-K split (k-step ranges per CTA, partial slots, fixed-order
    fix-up; CPQR_STREAMK=1 forces it) and the round-robin decomposition (0) both match the oracle:
    Y of every mode <= 1e-11, factors <= 1e-9, fits <= 1e-8."""
    monkeypatch.setenv("CPQR_STREAMK", mode)
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=400 + R)
    X = O.as_tensor(Xc)
    N = len(dims)
    s = cp.CPQR(dims, R, "QR", world=world, comm="local")
    s.set_tensor(Xc)
    s.set_factors(init)
    Qs = [O.qr_pos(init[k])[0] for k in range(N)]
    for n in range(N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
        assert np.max(np.abs(out["Y"] - Yo)) <= 1e-11 * np.max(np.abs(Yo))
    f = s.sweep(2)
    ref = O.cp_als_qr(X, init, 2)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    lam, A = s.get_factors()
    for k in range(N):
        assert rel(A[k], ref["factors"][k]) <= 1e-9
    s.close()


@pytest.mark.parametrize("mode", ["1", "0"])
@pytest.mark.parametrize("dims,R,variant", [((70, 66, 34), 10, "QR"), ((37, 29, 43), 7, "SVD"), ((300, 260, 64), 32, "QR"),
                                            ((24, 20, 18, 22), 8, "QR"), ((9, 8, 7, 6, 8), 4, "SVD"),
                                            ((520, 40, 30), 6, "QR")])
def test_overlap_schedule(cp, dims, R, variant, mode, monkeypatch):
    """The overlap schedule (CPQR_OVERLAP=1: the tail of mode n on a second stream beside the
    stream-X pass of mode n+1 when that pass does not contract mode n; N = 3 passes contract mode
    (n+1) mod 3; the tail as one CTA for I_n <= 512) and the serial schedule (0) both match the
    oracle -- factors <= 1e-9 after one sweep, fits <= 1e-8 -- and are run-to-run bitwise
    reproducible (graph replays)."""
    monkeypatch.setenv("CPQR_OVERLAP", mode)
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=500 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    runs = []
    for _ in range(2):
        s = cp.CPQR(dims, R, variant)
        s.set_tensor(Xc)
        s.set_factors(init)
        f1 = s.sweep(1)
        lam, A = s.get_factors()
        f = np.concatenate([f1, s.sweep(3)])
        runs.append((f, A))
        s.close()
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    ref = O.cp_als_qr(X, init, 4, variant=variant)
    f, A = runs[0]
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    assert np.array_equal(runs[0][0], runs[1][0])


@pytest.mark.parametrize("dims,R", [((40, 40, 40, 40), 32), ((64, 64, 64, 64), 24), ((30, 38, 48), 5),
                                    ((9, 8, 7, 6, 8), 4)])
def test_staircase_q0_apply(cp, dims, R, monkeypatch):
    """The staircase Q0 apply (CPQR_Q0_STAIR=1): W_n =
    Y_(n) Q0 over each column's (c+1)^{N-1} staircase rows only (rows in level order) equals the
    oracle's dense product within 1e-11 for every mode, at the high-rank shapes 40^4 R = 32 and
    64^4 R = 24, and the sweep matches the dense apply's."""
    import torch
    monkeypatch.setenv("CPQR_Q0_STAIR", "1")
    g = np.random.default_rng(R)
    N = len(dims)
    Xc = g.standard_normal(tuple(reversed(dims)))
    X = O.as_tensor(Xc)
    init = [g.standard_normal((d, R)) for d in dims]
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(torch.from_numpy(Xc).cuda())
    s.set_factors(init)
    Qs, Rs = [None] * N, [None] * N
    for k in range(N):
        Qs[k], Rs[k] = O.qr_pos(init[k])
    for n in range(N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Wo = O.apply_q0(out["Y"], n, out["Q0"])  # the oracle's dense product of the GPU's Y and Q0
        assert rel(out["W"], Wo) <= 1e-11, (n, rel(out["W"], Wo))
    f_st = s.sweep(2)
    s.close()
    monkeypatch.setenv("CPQR_Q0_STAIR", "0")
    d = cp.CPQR(dims, R, "QR")
    d.set_tensor(torch.from_numpy(Xc).cuda())
    d.set_factors(init)
    f_dn = d.sweep(2)
    d.close()
    assert np.max(np.abs(f_st - f_dn)) <= 1e-10


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("dims,R,variant,fit_mode", [((70, 66, 34), 10, "QR", "fast"), ((24, 20, 18, 22), 8, "SVD", "fast"),
                                                     ((30, 38, 48), 5, "QR", "direct")])
def test_multi_sweep_graph(cp, dims, R, variant, fit_mode, overlap, monkeypatch):
    """CPQR_GRAPH_SWEEPS=3: several sweeps captured in one CUDA graph (the overlap schedule's tails
    cross the sweep boundaries inside it; each sweep's fit goes to its slot through a device
    counter).  Bitwise the same fits and factors as one graph per sweep, for call lengths that mix
    3-sweep and 1-sweep graphs and grow the fits buffer (re-capture)."""
    monkeypatch.setenv("CPQR_OVERLAP", overlap)
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=600 + R)
    out = {}
    for gs in ("1", "3"):
        monkeypatch.setenv("CPQR_GRAPH_SWEEPS", gs)
        s = cp.CPQR(dims, R, variant, fit_mode=fit_mode)
        s.set_tensor(Xc)
        s.set_factors(init)
        f = np.concatenate([s.sweep(2), s.sweep(7), s.sweep(4)])
        lam, A = s.get_factors()
        out[gs] = (f, A)
        s.close()
    assert np.array_equal(out["1"][0], out["3"][0])
    assert all(np.array_equal(a, b) for a, b in zip(out["1"][1], out["3"][1]))
    ref = O.cp_als_qr(O.as_tensor(Xc), init, 13, variant=variant, fit_mode=fit_mode)
    assert np.max(np.abs(out["3"][0] - np.array(ref["fits"]))) <= 1e-8


@pytest.mark.parametrize("small", ["2", "1", "0"])
@pytest.mark.parametrize("dims,R", [((400, 40, 30), 10), ((12, 300, 250), 10), ((30, 40, 50), 5),
                                    ((37, 29, 43), 7), ((24, 20, 18, 22), 16), ((9, 8, 7, 6, 8), 4),
                                    ((70, 66, 34), 32), ((8, 500, 64), 3), ((33, 41, 27, 30), 24)])
def test_small_ttm_kernel(cp, dims, R, small, monkeypatch):
    """The remaining TTMs on L2-resident intermediates (k_ttm_small, plan kind 9: 16-row DMMA tiles,
    the contraction split over warps and CTAs, warp partials summed in warp order and CTA partials by
    the last-arriving CTA in CTA order) against the oracle's Multi-TTM: Y of every
    mode <= 1e-11 (Frobenius) and max|dY| <= 1e-11 max|Y| (element-wise), with the kernel forced on
    every intermediate (CPQR_TTM_SMALL=2), on where the TMA kernels are starved (1, default) and off
    (0: the TMA / register-staged kernels).  Shapes cover A = 1 (fibre
    contraction), A < 8 (rows spanning several b), ragged 16-row tiles, R = 3..32 (NT = 1..4), and
    the cross-CTA split (KC > 1: few rows, long contraction, e.g. 120 rows x I = 250)."""
    monkeypatch.setenv("CPQR_TTM_SMALL", small)
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=700 + R + len(dims))
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    N = len(dims)
    Qs = [O.qr_pos(init[k])[0] for k in range(N)]
    used = 0
    for n in range(N):
        used += sum(st["kind"] == "small-ttm" for st in s.debug_plan(n))
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
        assert np.max(np.abs(out["Y"] - Yo)) <= 1e-11 * np.max(np.abs(Yo)), n
    if small == "2":
        assert used > 0
    if small == "0":
        assert used == 0
    f = s.sweep(2)
    s.close()
    ref = O.cp_als_qr(X, init, 2)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8


@pytest.mark.parametrize("dims,R", [((70, 66, 34), 10), ((520, 40, 30), 6), ((24, 20, 18, 22), 8)])
def test_overlap_schedule_householder_tail(cp, dims, R, monkeypatch):
    """The overlap schedule with the Householder factor QR forced (CPQR_FACTOR_QR=householder): its
    tail runs the whole TSQR (leaves, root, Q formation) in ONE CTA (k_rq_serial) beside the next
    stream pass; factors <= 1e-9 after one sweep and fits <= 1e-8 against the oracle."""
    monkeypatch.setenv("CPQR_OVERLAP", "1")
    monkeypatch.setenv("CPQR_FACTOR_QR", "householder")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=900 + R)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    f = np.concatenate([f1, s.sweep(2)])
    s.close()
    ref1, ref = O.cp_als_qr(X, init, 1), O.cp_als_qr(X, init, 3)
    for k in range(len(dims)):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, k
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8


def _oracle_run(variant, X, A0, sweeps, tau=-1.0):
    if variant in ("QR", "SVD"):
        return O.cp_als_qr(X, A0, sweeps, variant=variant, tau=tau)
    return O.cp_als_ne(X, A0, sweeps, solve="pinv" if variant == "PINV" else "chol", tau=tau)


@pytest.mark.parametrize("variant", ["NE", "SVD", "PINV", "QR"])
@pytest.mark.parametrize("dims,R,kw", [((20, 18, 16), 3, dict(eta=0.05)),
                                       ((12, 14, 10), 5, dict(eta=1e-3, kind="congruence", c=0.99)),
                                       ((50, 50, 50), 5, dict(eta=1e-4)), ((33, 30, 31), 5, dict(eta=1e-4))])
def test_batched_all_variants(cp, dims, R, kw, variant):
    """cpqr_batched: the four solvers of the accuracy study one CTA per problem --
    CP-ALS (Alg. 1, Cholesky), CP-ALS-PINV, CP-ALS-QR and QR-SVD (Alg. 2,
    PAPER.md:335-339) -- against the oracle's drivers: factors and lambda <= 1e-9 after one sweep,
    fits within 1e-8 for every sweep of a 6-sweep run (tol = 0), every problem of the batch."""
    seeds = [301, 302, 303, 304]
    Xs, A0s, X, A0 = _batched_inputs(dims, R, seeds, **kw)
    for sweeps in (1, 6):
        A, lam, fits, iters = cp.batched_qr(X, A0, R, max_iters=sweeps, tol=0.0, variant=variant)
        A = [a.cpu().numpy() for a in A]
        lam, fits, iters = lam.cpu().numpy(), fits.cpu().numpy(), iters.cpu().numpy()
        assert np.all(iters == sweeps)
        for p in range(len(seeds)):
            ref = _oracle_run(variant, O.as_tensor(Xs[p]), A0s[p], sweeps)
            assert np.max(np.abs(fits[p] - np.array(ref["fits"]))) <= 1e-8, (p, fits[p], ref["fits"])
            if sweeps == 1:
                for k in range(3):
                    assert rel(A[k][p].T, ref["factors"][k]) <= 1e-9, (p, k, rel(A[k][p].T, ref["factors"][k]))
                assert rel(lam[p], ref["lam"]) <= 1e-9


@pytest.mark.parametrize("variant", ["SVD", "PINV"])
def test_batched_truncation_exact_duplicate(cp, variant):
    """Exact duplicate columns (A_k(:,2) = A_k(:,1) for the initial factors of modes 2, 3): R0 (QR-SVD)
    and S_n (PINV) are singular, sigma's below tau sigma_max are dropped,
    and the minimum-norm solution is unique: the batched solvers match the oracle's after one sweep
    (factors <= 1e-9) and the duplicated columns of A_1 stay equal."""
    import torch
    dims, R = (16, 14, 12), 4
    Xs, A0s, X, A0 = _batched_inputs(dims, R, [401, 402], eta=0.05)
    for p in range(2):
        for k in (1, 2):
            A0s[p][k][:, 1] = A0s[p][k][:, 0]
    A0 = [torch.from_numpy(np.stack([np.ascontiguousarray(a[k].T) for a in A0s])).cuda() for k in range(3)]
    A, lam, fits, iters = cp.batched_qr(X, A0, R, max_iters=1, tol=0.0, variant=variant, tau=1e-12)
    A = [a.cpu().numpy() for a in A]
    for p in range(2):
        ref = _oracle_run(variant, O.as_tensor(Xs[p]), A0s[p], 1, tau=1e-12)
        assert rel(A[0][p].T, ref["factors"][0]) <= 1e-9, p
        assert np.allclose(A[0][p][0], A[0][p][1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("n", [0, 1])
def test_tma_ring_war_determinism_l2_resident(cp, n):
    """The C3 shape (128^4, R = 16): the Multi-TTM's later strided steps stream an L2-resident
    intermediate, so the TMA refill of a ring stage lands within a few hundred cycles of the
    consumers' release.  Without fence.proxy.async between the consumers' ld.shared reads and the
    release (generic vs async proxy, write-after-read), ~1-2 % of these Multi-TTMs had one 16-row
    box wrong.  100 repeats of mode n's Multi-TTM must be bitwise identical."""
    import torch
    from paper_2112_10855_b200 import synth as S
    conf = S.CONFIGS[3]
    g = torch.Generator(device="cuda").manual_seed(11)
    X = torch.randn(int(np.prod(conf.dims)), dtype=torch.float64, device="cuda", generator=g)
    s = cp.CPQR(conf.dims, conf.R, "QR")
    s.set_tensor(X)
    s.set_factors(S.init_factors(conf))
    ref = s.debug_mode(n)["Y"]
    bad = sum(not np.array_equal(s.debug_mode(n)["Y"], ref) for _ in range(100))
    s.close()
    del X
    torch.cuda.empty_cache()
    assert bad == 0, bad


@pytest.mark.parametrize("dims,R,tree", [((40, 36, 30), 6, False), ((24, 20, 18, 22), 8, False),
                                         ((9, 8, 7, 6, 8), 4, False), ((24, 20, 18, 22), 8, True)])
def test_cost_accounting_matches_oracle_ttm_cost(cp, dims, R, tree):
    """SURVEY.md 8(c) cost accounting: the flops the library attributes to each Multi-TTM step
    (cpqr_debug_plan) follow Eq. (TTMcost): for every mode, in the library's own
    contraction order, the steps' flops sum to the oracle's ttm_cost(dims, n, R, order) (fused slice
    steps count both contractions); and cpqr_get_profile's flops0 / bytes0 equal the stream-X
    passes' first steps and N (or 2 with the dimension tree) reads of X.  The library stores an
    odd I_1 padded to I_1 + 1 (a zero row, cpqr.h cpqr_set_tensor: TMA needs 16-byte strides) and
    counts the work it executes, so the paper's formula is evaluated on the stored dims."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5)
    stored = (dims[0] + (dims[0] & 1),) + tuple(dims[1:])
    s = cp.CPQR(dims, R, "QR", profile=True, use_graph=False, tree=tree)
    s.set_tensor(Xc)
    s.set_factors(init)
    N = len(dims)
    first, passes = 0.0, 0
    for n in range(N):
        pl = [st for st in s.debug_plan(n) if st["kind"] not in ("slice-reduce", "slice-fixup")]
        order = [k for st in pl for k in st["modes"]]
        if not tree:
            assert sorted(order) == [k for k in range(N) if k != n]
            assert sum(st["flops"] for st in pl) == O.ttm_cost(stored, n, R, order=order), (n, pl)
        if pl and pl[0]["x_pass"]:
            first += pl[0]["flops"]
            passes += 1
    p = s.profile()
    s.close()
    assert passes == (2 if tree else N)
    assert p["flops0"] == first and p["bytes0"] == passes * 8.0 * np.prod(stored)


def _kt_oracle(variant, lam, B, A0, sweeps, fit_mode="fast"):
    if variant in ("QR", "SVD"):
        return O.cp_als_qr(None, A0, sweeps, variant=variant, kt=(lam, B), fit_mode=fit_mode)
    return O.cp_als_ne(None, A0, sweeps, solve="pinv" if variant == "PINV" else "chol", kt=(lam, B),
                       fit_mode=fit_mode)


@pytest.mark.parametrize("variant", ["QR", "SVD", "NE", "PINV"])
@pytest.mark.parametrize("dims,R,S", [((3, 5, 4, 6), 5, 6), ((3,) * 10, 4, 5), ((4,) * 10, 5, 3)])
def test_short_modes_kruskal(cp, dims, R, S, variant):
    """Short modes I_k < R with Kruskal input (the 10-way sine of sums has I_k = 8 < R = 10,
    PAPER.md:630-645), N up to 10: the library stores such factors zero-padded to R rows (pinned on
    the oracle: test_short_modes_zero_padding_is_exact), keeps V_n's prod min(I_k, R) nonzero rows
    and factors it by the shifted CholeskyQR3; against the oracle's economy-QR run: factors <= 1e-9
    after one sweep, fits within 1e-8 over three.  (4,)*10 has a 262144-row V_n (chunked M)."""
    g = np.random.default_rng(len(dims) * 100 + R)
    lam = g.standard_normal(S)
    B = [g.standard_normal((d, S)) for d in dims]
    A0 = [g.standard_normal((d, R)) for d in dims]
    s = cp.CPQR(dims, R, variant)
    s.set_ktensor(lam, B)
    s.set_factors(A0)
    f1 = s.sweep(1)
    lam1, A = s.get_factors()
    f = np.concatenate([f1, s.sweep(2)])
    s.close()
    ref1, ref = _kt_oracle(variant, lam, B, A0, 1), _kt_oracle(variant, lam, B, A0, 3)
    for k in range(len(dims)):
        assert A[k].shape == (dims[k], R)
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    assert rel(lam1, ref1["lam"]) <= 1e-9
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8, (f, ref["fits"])


def test_short_modes_direct_fit_and_errors(cp):
    """Short modes: the DIRECT relative error iterates the true I_k (not the padded
    rows) and matches the oracle; a dense tensor is rejected (EINVAL: short modes need Kruskal
    input)."""
    dims, R, S = (3, 6, 4, 5), 5, 4
    g = np.random.default_rng(77)
    lam = g.standard_normal(S)
    B = [g.standard_normal((d, S)) for d in dims]
    A0 = [g.standard_normal((d, R)) for d in dims]
    s = cp.CPQR(dims, R, "QR", fit_mode="direct")
    with pytest.raises(cp.CpqrError):
        s.set_tensor(np.zeros(dims[::-1]))
    s.set_ktensor(lam, B)
    s.set_factors(A0)
    f = s.sweep(3)
    s.close()
    ref = _kt_oracle("QR", lam, B, A0, 3, fit_mode="direct")
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-10, (f, ref["fits"])


@pytest.mark.parametrize("variant,tree,mem", [("QR", False, "host"), ("SVD", True, "borrow"), ("NE", False, "copy"),
                                              ("PINV", False, "host"), ("QR", False, "borrow")])
@pytest.mark.parametrize("dims,R", [((35, 34, 33), 6), ((75, 40, 33), 32), ((15, 14, 13, 12), 5), ((9, 7, 5, 6, 8), 4)])
def test_odd_first_mode_is_padded_for_tma(cp, dims, R, variant, tree, mem):
    """Odd I_1 (the paper's 75^5 shape): mode 1 is stored padded to even so the TMA
    stream kernels run (cpqr.h cpqr_set_tensor); host, copied and borrowed tensors all take the
    padded copy.  The plans must use the TMA kernels on X, Y / W / factors / fits match the oracle
    on the true dims, and CPQR_PAD_ODD=0 (the unpadded fallback kernels) gives the same results."""
    import os
    import torch
    if R > min(dims):
        pytest.skip("tall factors only")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=900 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    ne = variant in ("NE", "PINV")

    def make():
        s = cp.CPQR(dims, R, variant, tree=tree)
        if mem == "host":
            s.set_tensor(Xc)
        else:
            s.set_tensor(torch.from_numpy(np.ascontiguousarray(Xc)).cuda(), copy=(mem == "copy"))
        s.set_factors(init)
        return s
    s = make()
    kinds = [st["kind"] for n in range(N) for st in s.debug_plan(n) if st["x_pass"]]
    assert kinds and all("tma" in k for k in kinds), kinds
    if not ne:
        Qs, Rs = zip(*[O.qr_pos(a) for a in init])
        for n in range(N):
            out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
            Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
            assert out["Y"].shape == Yo.shape and rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
            Q0o, R0o = O.structured_qr(list(Rs), n)
            assert rel(out["W"], O.apply_q0(Yo, n, Q0o)) <= 1e-11
    ref1 = O.cp_als_ne(X, init, 1, solve="pinv" if variant == "PINV" else "chol") if ne else \
        O.cp_als_qr(X, init, 1, variant=variant)
    ref = O.cp_als_ne(X, init, 3, solve="pinv" if variant == "PINV" else "chol") if ne else \
        O.cp_als_qr(X, init, 3, variant=variant)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    assert [a.shape for a in A] == [(d, R) for d in dims]
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(2)])
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    lam3, A3 = s.get_factors()
    s.close()
    os.environ["CPQR_PAD_ODD"] = "0"
    try:
        u = make()
    finally:
        del os.environ["CPQR_PAD_ODD"]
    fu = u.sweep(3)
    lamu, Au = u.get_factors()
    u.close()
    assert np.max(np.abs(fu - f)) <= 1e-9
    for k in range(N):
        assert rel(Au[k], A3[k]) <= 1e-8


@pytest.mark.parametrize("dims,R,variant,world", [((30, 38, 48), 5, "QR", 1), ((70, 66, 32), 32, "QR", 1),
                                                  ((33, 20, 18, 16), 8, "SVD", 1), ((9, 8, 7, 6, 8), 4, "QR", 1),
                                                  ((70, 66, 32), 32, "QR", 4), ((24, 20, 18, 16), 8, "QR", 8)])
def test_q0_apply_big_kernel(cp, dims, R, variant, world):
    """k_q0_apply_big (4 M-tiles per CTA, chosen for V_n of >= 32768 rows) forced on small shapes:
    W of every mode against the oracle's apply_q0 (<= 1e-11, element-wise too), sweeps against the
    oracle, and -- with virtual ranks -- the fused peer push bitwise equal to the sum-kernel exchange."""
    import os
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=1300 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    os.environ["CPQR_Q0_BIG"] = "1"
    try:
        comm = "local_peer" if world > 1 else "local"
        s = cp.CPQR(dims, R, variant, world=world, comm=comm)
        s.set_tensor(Xc)
        s.set_factors(init)
        Qs, Rs = zip(*[O.qr_pos(a) for a in init])
        for n in range(N):
            out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
            Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
            Q0o, R0o = O.structured_qr(list(Rs), n)
            Wo = O.apply_q0(Yo, n, Q0o)
            assert rel(out["W"], Wo) <= 1e-11, (n, rel(out["W"], Wo))
            assert np.max(np.abs(out["W"] - Wo)) <= 1e-11 * np.max(np.abs(Wo))
        f = s.sweep(3)
        lam, A = s.get_factors()
        if world > 1:
            assert s.debug_peer()["windows_differing"] == 0
        s.close()
        if world > 1:
            t = cp.CPQR(dims, R, variant, world=world, comm="local")
            t.set_tensor(Xc)
            t.set_factors(init)
            t.sweep(3)
            lt, At = t.get_factors()
            t.close()
            assert all(np.array_equal(x, y) for x, y in zip(A, At))
    finally:
        del os.environ["CPQR_Q0_BIG"]
    ref = O.cp_als_qr(X, init, 3, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    for k in range(N):
        assert rel(A[k], ref["factors"][k]) <= 1e-8


@pytest.mark.parametrize("variant", ["QR", "SVD"])
@pytest.mark.parametrize("dims,R", [((20, 20, 20, 20), 8), ((14, 13, 13, 13), 5), ((22, 9, 9, 9, 9), 4),
                                    ((16, 12, 12, 12, 12), 8), ((130, 6, 7, 7), 3)])
def test_fused_last_two_modes_pass(cp, dims, R, variant):
    """k_strided2_tma (N >= 4, R <= 8): modes 1 and 2 contract the two slowest modes in ONE pass over
    X when they are next in the decreasing-dimension order.  The plan must show the
    fused step, its flops must be Eq. (TTMcost) for that order, Y / W of every mode, factors and
    fits must match the oracle, and CPQR_STR_FUSE2=0 (two separate TTMs) must agree."""
    import os
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=1500 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    s = cp.CPQR(dims, R, variant)
    s.set_tensor(Xc)
    s.set_factors(init)
    stored = (dims[0] + (dims[0] & 1),) + tuple(dims[1:])
    fused = 0
    for n in range(N):
        pl = [st for st in s.debug_plan(n) if st["kind"] not in ("slice-reduce", "slice-fixup")]
        order = [k for st in pl for k in st["modes"]]
        assert sum(st["flops"] for st in pl) == O.ttm_cost(stored, n, R, order=order), (n, pl)
        fused += sum(1 for st in pl if st["kind"] == "strided2-tma")
    assert fused >= 1, fused  # mode 1, and mode 2 when mode 1 is not the largest
    Qs, Rs = zip(*[O.qr_pos(a) for a in init])
    for n in range(N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
        assert np.max(np.abs(out["Y"] - Yo)) <= 1e-11 * np.max(np.abs(Yo)), n
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    ref = O.cp_als_qr(X, init, 3, variant=variant)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(2)])
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()
    os.environ["CPQR_STR_FUSE2"] = "0"
    try:
        u = cp.CPQR(dims, R, variant)
    finally:
        pass
    u.set_tensor(Xc)
    u.set_factors(init)
    assert not any(st["kind"] == "strided2-tma" for n in range(N) for st in u.debug_plan(n))
    fu = u.sweep(3)
    u.close()
    del os.environ["CPQR_STR_FUSE2"]
    assert np.max(np.abs(fu - f)) <= 1e-10


@pytest.mark.parametrize("dims,R", [((18, 300, 7, 6), 6), ((16, 270, 18, 17), 16), ((16, 520, 12, 11), 10)])
def test_slice_pass_box_width_by_fill(cp, dims, R):
    """The fused slice pass takes 128-fibre boxes instead of 256-fibre ones when I_2 sits just above
    a multiple of 256 (the paper's 300^4: 300 of 512 fibre slots): Y of the modes that use it
    (n >= 3) against the oracle, element-wise, and the sweeps."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=1700 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(Xc)
    s.set_factors(init)
    assert any("slice" in st["kind"] for n in range(2, N) for st in s.debug_plan(n))
    Qs, Rs = zip(*[O.qr_pos(a) for a in init])
    for n in range(2, N):
        out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
        assert np.max(np.abs(out["Y"] - Yo)) <= 1e-11 * np.max(np.abs(Yo)), n
    ref = O.cp_als_qr(X, init, 3)
    f = s.sweep(3)
    s.close()
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8


@pytest.mark.parametrize("world", [1, 4])
def test_odd_first_mode_direct_fit_and_slabs(cp, world):
    """Odd I_1 (stored padded) with the DIRECT fit (the residual pass reads the padded X and A_1) and
    with virtual ranks: fits of every sweep against the oracle's direct fit."""
    dims, R = (21, 18, 16), 4
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=91, eta=0.0)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR", fit_mode="direct", world=world, comm="local")
    s.set_tensor(Xc)
    s.set_factors(init)
    f = s.sweep(4)
    lam, A = s.get_factors()
    s.close()
    ref = O.cp_als_qr(X, init, 4, fit_mode="direct")
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8, (f, ref["fits"])
    for k in range(3):
        assert A[k].shape == (dims[k], R) and rel(A[k], ref["factors"][k]) <= 1e-7


@pytest.mark.parametrize("dims,R,variant,tree", [((30, 38, 48), 5, "QR", False), ((33, 20, 18, 16), 8, "SVD", False),
                                                 ((24, 20, 18, 16), 8, "QR", True), ((9, 8, 7, 6, 8), 4, "QR", False),
                                                 ((70, 66, 32), 32, "QR", False)])
def test_z_fusion(cp, dims, R, variant, tree):
    """CPQR_ZFUSE=1: the last TTM and the Q0 apply as one product W = T_(n) [(Q_k (x) I) Q0] (Z formed
    on the side stream by k_zform): factors after one sweep and fits of three against the oracle,
    in the overlap and the serial schedule, and against the unfused sweep."""
    import os
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=1900 + R + len(dims))
    X = O.as_tensor(Xc)
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    ref = O.cp_als_qr(X, init, 3, variant=variant)
    base = cp.CPQR(dims, R, variant, tree=tree)
    base.set_tensor(Xc)
    base.set_factors(init)
    fb = base.sweep(3)
    base.close()
    for overlap in ("1", "0"):
        os.environ["CPQR_ZFUSE"] = "1"
        os.environ["CPQR_OVERLAP"] = overlap
        try:
            s = cp.CPQR(dims, R, variant, tree=tree)
            s.set_tensor(Xc)
            s.set_factors(init)
            f1 = s.sweep(1)
            lam, A = s.get_factors()
            f = np.concatenate([f1, s.sweep(2)])
            s.close()
        finally:
            del os.environ["CPQR_ZFUSE"]
            del os.environ["CPQR_OVERLAP"]
        for k in range(len(dims)):
            assert rel(A[k], ref1["factors"][k]) <= 1e-9, (overlap, k, rel(A[k], ref1["factors"][k]))
        assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
        assert np.max(np.abs(f - fb)) <= 1e-10


@pytest.mark.parametrize("dims,R,fit_mode", [((30, 38, 48), 5, "fast"), ((41, 36, 24), 6, "direct"), ((70, 66, 32), 32, "fast")])
def test_ne_overlap_schedule(cp, dims, R, fit_mode):
    """CP-ALS (NE), N = 3: the overlap schedule (the one-CTA tail of mode n beside the first TTM of
    mode n+1, which contracts mode (n+2) mod 3) against the oracle and against the serial schedule
    (CPQR_OVERLAP_NE=0; the two contract in different orders, so they agree to rounding only), as a
    CUDA graph and eagerly (bitwise equal)."""
    import os
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=2100 + R)
    X = O.as_tensor(Xc)
    ref1 = O.cp_als_ne(X, init, 1)
    ref = O.cp_als_ne(X, init, 4, fit_mode=fit_mode)
    out = {}
    for key, env, graph in [("ov", None, True), ("ov_eager", None, False), ("serial", "0", True)]:
        if env is not None:
            os.environ["CPQR_OVERLAP_NE"] = env
        try:
            s = cp.CPQR(dims, R, "NE", fit_mode=fit_mode, use_graph=graph)
        finally:
            os.environ.pop("CPQR_OVERLAP_NE", None)
        s.set_tensor(Xc)
        s.set_factors(init)
        f1 = s.sweep(1)
        lam1, A1 = s.get_factors()
        f = np.concatenate([f1, s.sweep(3)])
        out[key] = (f, A1, s.get_factors()[1])
        s.close()
        for k in range(3):
            assert rel(A1[k], ref1["factors"][k]) <= 1e-9, (key, k, rel(A1[k], ref1["factors"][k]))
        assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8, (key, f, ref["fits"])
    assert np.array_equal(out["ov"][0], out["ov_eager"][0])
    assert all(np.array_equal(x, y) for x, y in zip(out["ov"][2], out["ov_eager"][2]))
    assert np.max(np.abs(out["ov"][0] - out["serial"][0])) <= 1e-10
