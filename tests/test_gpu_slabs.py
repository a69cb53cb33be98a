"""GPU parity of the slab data-parallel path on ONE B200.

With cpqr_options.comm = CPQR_COMM_LOCAL one context runs the p slabs of p virtual ranks in rank
order: each slab has its own plans (TMA maps over its block of X and its rows of Q_N), its own
dimension-tree buffer and its own partial W_n; the exchange step is a fixed-order sum over the
ranks (modes n < N, NCCL's all-reduce) or one copy per rank (mode N, NCCL's all-gather).  This is
the multi-GPU code path minus the NCCL call, so every world size is checked against the oracle
here (no kernels wait on each other: the ranks run one after another on one stream).

Tolerances (north_star): Y of every mode <= 1e-11, factors and lambda after one sweep <= 1e-9,
fits within 1e-8 on every sweep; Y is also checked element-wise (max |dY| / max |Y| <= 1e-11).
"""
import numpy as np
import pytest

import oracle as O
from paper_2112_10855_b200 import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def maxrel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def cp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_10855_b200 import cpqr
    return cpqr


CASES = [
    # C1-like 3-way, odd dims, last mode divisible by 8
    ((30, 38, 48), 5, "QR", False),
    ((70, 66, 32), 32, "QR", False),          # R = 32: the FP64-bound (C5) stream plans
    ((40, 36, 24), 6, "NE", False),
    # C3-like 4-way (fused slice pass for n >= 2)
    ((24, 20, 18, 16), 8, "QR", False),
    ((24, 20, 18, 16), 8, "SVD", True),       # dimension tree
    ((16, 14, 12, 16), 6, "NE", False),
    ((16, 14, 12, 16), 6, "PINV", False),
    # C4-like 5-way
    ((9, 8, 7, 6, 8), 4, "SVD", False),
    ((9, 8, 7, 6, 8), 4, "QR", True),
]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("dims,R,variant,tree", CASES)
def test_virtual_ranks_match_oracle(cp, dims, R, variant, tree, world):
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=301 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    s = cp.CPQR(dims, R, variant, tree=tree, world=world, comm="local")
    s.set_tensor(Xc)
    s.set_factors(init)
    ne = variant in ("NE", "PINV")
    solve = "pinv" if variant == "PINV" else "chol"
    if not ne:
        Qs, Rs = [None] * N, [None] * N
        for k in range(N):
            Qs[k], Rs[k] = O.qr_pos(init[k])
        for n in range(N):
            out = s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(N)])
            Yo = O.multi_ttm(X, {k: Qs[k].T for k in range(N) if k != n})
            assert rel(out["Y"], Yo) <= 1e-11, (n, rel(out["Y"], Yo))
            assert maxrel(out["Y"], Yo) <= 1e-11, (n, maxrel(out["Y"], Yo))
            Q0o, R0o = O.structured_qr(Rs, n)
            assert rel(out["W"], O.apply_q0(Yo, n, Q0o)) <= 1e-11
        ref = O.cp_als_qr(X, init, 3, variant=variant)
    else:
        ref = O.cp_als_ne(X, init, 3, solve=solve)
    ref1 = O.cp_als_ne(X, init, 1, solve=solve) if ne else O.cp_als_qr(X, init, 1, variant=variant)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    for k in range(N):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    assert rel(lam, ref1["lam"]) <= 1e-9
    f = np.concatenate([f1, s.sweep(2)])
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8, (f, ref["fits"])
    s.close()


@pytest.mark.parametrize("world", [2, 8])
def test_virtual_ranks_direct_fit_and_per_slab_set(cp, world):
    """DIRECT fit summed over the slabs; setting each virtual rank's slab separately (its own
    buffer, like a separate GPU) gives bitwise the same sweep as setting the whole tensor."""
    dims, R = (20, 18, 16), 4
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=77, eta=0.0)
    X = O.as_tensor(Xc)
    a = cp.CPQR(dims, R, "QR", fit_mode="direct", world=world, comm="local")
    a.set_tensor(Xc)
    a.set_factors(init)
    fa = a.sweep(4)
    b = cp.CPQR(dims, R, "QR", fit_mode="direct", world=world, comm="local")
    per = dims[-1] // world
    for q in range(world):
        b.set_tensor(np.ascontiguousarray(Xc[q * per:(q + 1) * per]), slab=(q * per, (q + 1) * per))
    b.set_factors(init)
    fb = b.sweep(4)
    assert np.array_equal(fa, fb)
    la, Aa = a.get_factors()
    lb, Ab = b.get_factors()
    assert all(np.array_equal(x, y) for x, y in zip(Aa, Ab))
    ref = O.cp_als_qr(X, init, 4, fit_mode="direct")
    assert np.max(np.abs(fa - np.array(ref["fits"]))) <= 1e-8, (fa, ref["fits"])
    a.close()
    b.close()


def test_virtual_ranks_reject_bad_slab(cp):
    dims, R = (12, 10, 8), 3
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5)
    s = cp.CPQR(dims, R, "QR", world=4, comm="local")
    with pytest.raises(cp.CpqrError):
        s.set_tensor(np.ascontiguousarray(Xc[:3]), slab=(0, 3))
    s.set_factors(init)
    s.set_tensor(np.ascontiguousarray(Xc[:2]), slab=(0, 2))
    with pytest.raises(cp.CpqrError) as ei:  # the other three slabs are missing
        s.sweep(1)
    assert "ESTATE" in str(ei.value)
    s.close()


@pytest.mark.parametrize("dims,R", [((64, 64, 64), 8), ((1000, 1000, 1000), 32), ((128, 128, 128, 128), 16),
                                    ((48, 48, 48, 48, 48), 8)])
def test_slab_plans_scale_as_one_over_p(cp, dims, R):
    """PAPER.md:387 (decreasing dimension) applied to the LOCAL dims: with p slabs the slab mode is
    the smallest local dimension and is never contracted first (unless it is the only choice), so
    the stream pass's flops and every intermediate shrink as 1/p (the final partial Y does not)."""
    import os
    import torch
    N = len(dims)
    # the one-GPU plan may fuse the last two modes into one pass (k_strided2_tma, R <= 8), which the
    # slab plans cannot (the slab mode is contracted last): compare like with like
    os.environ["CPQR_STR_FUSE2"] = "0"
    X = torch.zeros(int(np.prod(dims)), dtype=torch.float64, device="cuda")
    init = [np.eye(d, R) for d in dims]
    base = None
    for p in [1, 2, 4, 8]:
        s = cp.CPQR(dims, R, "QR", world=p, comm="local")
        s.set_tensor(X)
        s.set_factors(init)
        plans = [s.debug_plan(n) for n in range(N)]
        stats = []
        for n, pl in enumerate(plans):
            main = [st for st in pl if st["kind"] not in ("slice-reduce", "slice-fixup")]
            fl = sum(st["flops"] for st in main)
            inter = sum(st["out_elems"] for st in main[:-1])  # the last step writes the partial Y
            first = main[0]
            assert first["x_pass"]
            if p > 1:
                assert N - 1 not in first["modes"], (p, n, main)  # the slab mode is never first
            stats.append((fl, inter))
        if base is None:
            base = stats
        else:
            for n in range(N):
                assert stats[n][0] <= 1.02 * base[n][0] / p + 1, (p, n, stats[n], base[n])
                assert stats[n][1] <= 1.02 * base[n][1] / p + 1, (p, n, stats[n], base[n])
        s.close()
    del os.environ["CPQR_STR_FUSE2"]
    del X
    torch.cuda.empty_cache()
