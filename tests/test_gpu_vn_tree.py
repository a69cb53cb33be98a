"""GPU parity of the tree QR of V_n across the Khatri-Rao factors (CPQR_VN_QR=tree; SURVEY.md 8(f)
NEXT-2; csrc/vn_tree.cuh) against the oracle's `tree_qr` and its dense
`structured_qr` (LAPACK on the formed V_n): Q0, R0 of every mode, one CTA per V_n, the shared
group factored at the first mode of each half sweep and reused (exercised by every sweep below),
sweeps in every schedule (per mode, dimension tree, overlap on/off, virtual ranks)."""
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
    ((30, 40, 50), 5),            # N = 3: one node (the K2 problem)
    ((12, 10, 9, 11), 6),         # N = 4: shared pair + root
    ((24, 20, 18, 22), 16),       # N = 4, R = 16 (C3's rank)
    ((6, 7, 5, 6, 8), 3),         # N = 5: chains of 2 on both sides
    ((9, 8, 10, 9, 8), 8),        # N = 5, R = 8 (C4's rank)
    ((5, 4, 5, 4, 5, 4), 3),      # N = 6
    ((4, 3, 4, 3, 4, 3, 4), 3),   # N = 7
]


@pytest.mark.parametrize("dims,R", SHAPES)
def test_tree_qr_debug_mode_q0_r0(cp, dims, R, monkeypatch):
    """Q0, R0 of every mode (debug_mode: the shared group factored afresh) within 1e-11 of the
    oracle's tree QR and of LAPACK's QR of the formed V_n; Q0 orthonormal; W = Y Q0."""
    monkeypatch.setenv("CPQR_VN_QR", "tree")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=211 + len(dims) + R)
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
        Q0t, R0t = O.tree_qr(Rs, n)
        Q0d, R0d = O.structured_qr(Rs, n)
        assert rel(out["R0"], R0t) <= 1e-11 and rel(out["R0"], R0d) <= 1e-11, n
        assert rel(out["Q0"], Q0t) <= 1e-11 and rel(out["Q0"], Q0d) <= 1e-11, n
        assert np.linalg.norm(out["Q0"].T @ out["Q0"] - np.eye(R)) <= 1e-12
        # element-wise: Q0 keeps V_n's staircase support exactly (zeros where level > column)
        assert np.max(np.abs(out["Q0"] - Q0d)) <= 1e-11 * np.max(np.abs(Q0d))
        Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
        assert rel(out["W"], O.apply_q0(Yo, n, Q0d)) <= 1e-11
    s.close()


@pytest.mark.parametrize("variant", ["QR", "SVD"])
@pytest.mark.parametrize("dims,R", SHAPES[1:6])
@pytest.mark.parametrize("sched", ["permode", "tree", "overlap0"])
def test_tree_qr_sweeps_match_oracle(cp, dims, R, variant, sched, monkeypatch):
    """Sweeps with the tree QR (shared group cached across the modes of each half): factors after
    one sweep <= 1e-9, every fit of three sweeps within 1e-8 of the oracle (dense LAPACK QR of V_n)."""
    monkeypatch.setenv("CPQR_VN_QR", "tree")
    if sched == "overlap0":
        monkeypatch.setenv("CPQR_OVERLAP", "0")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=223 + len(dims) + R, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, variant, tree=(sched == "tree"))
    s.set_tensor(Xc)
    s.set_factors(init)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, init, 1, variant=variant)
    for k in range(len(dims)):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(2)])
    ref = O.cp_als_qr(X, init, 3, variant=variant)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()


@pytest.mark.parametrize("dims,R,world", [((12, 10, 9, 16), 6, 4), ((9, 8, 10, 9, 8), 8, 2), ((24, 20, 18, 24), 16, 8)])
def test_tree_qr_virtual_ranks(cp, dims, R, world, monkeypatch):
    """Slab data parallelism (virtual ranks) with the tree QR: the V_n QR is replicated, the
    factors follow the oracle and are bitwise those of world = 1 up to the W reduction order."""
    monkeypatch.setenv("CPQR_VN_QR", "tree")
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=227 + world, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR", world=world, comm="local")
    s.set_tensor(Xc)
    s.set_factors(init)
    f = s.sweep(3)
    lam, A = s.get_factors()
    ref = O.cp_als_qr(X, init, 3)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    for k in range(len(dims)):
        assert rel(A[k], ref["factors"][k]) <= 1e-7
    s.close()


def test_tree_qr_high_rank(cp, monkeypatch):
    """High rank (40^4, R = 32: V_n is 32768 x 32; nodes 1024 x 32 in 116 KB of shared memory):
    factors after one sweep <= 1e-9 and fits within 1e-8 of the oracle, Q0/R0 of one mode <= 1e-10."""
    import torch
    monkeypatch.setenv("CPQR_VN_QR", "tree")
    dims, R = (40, 40, 40, 40), 32
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=71, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, "QR")
    s.set_tensor(torch.from_numpy(Xc).cuda())
    s.set_factors(init)
    Rs = [O.qr_pos(a)[1] for a in init]
    d = s.debug_mode(2)
    Q0o, R0o = O.structured_qr(Rs, 2)
    assert rel(d["R0"], R0o) <= 1e-10 and rel(d["Q0"], Q0o) <= 1e-10
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    ref1 = O.cp_als_qr(X, init, 1)
    for k in range(4):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    f = np.concatenate([f1, s.sweep(2)])
    ref = O.cp_als_qr(X, init, 3)
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8
    s.close()
