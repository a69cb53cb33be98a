"""Seeded randomized parity (GPU vs the CPU oracle) over shapes the hand-picked cases do not pin:
N in {3, 4, 5}, every I_k drawn in [R, 64] (ragged against the 16-row TMA stages and the 8-wide
DMMA tiles; slices of 1-2 fibre units), R in [1, 20], variant QR / SVD / NE, per-mode and
dimension-tree Multi-TTM.  Tolerances are north_star's: factors and lambda after one sweep from
the shared init <= 1e-9 relative, fits of two sweeps within 1e-8."""
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


def cases(n=48, seed=20260):
    g = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        N = int(g.integers(3, 6))
        R = int(g.integers(1, 21))
        cap = {3: 64, 4: 40, 5: 20}[N]
        if R > cap:
            continue
        dims = tuple(int(g.integers(R, cap + 1)) for _ in range(N))
        if np.prod(dims) > 400_000:
            continue
        variant = ["QR", "SVD", "NE"][len(out) % 3]
        tree = variant != "NE" and bool(g.integers(0, 2))
        out.append((dims, R, variant, tree, int(g.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("dims,R,variant,tree,seed", cases())
def test_fuzz_sweep_parity(cp, dims, R, variant, tree, seed):
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=seed % 100000, eta=0.05)
    X = O.as_tensor(Xc)
    s = cp.CPQR(dims, R, variant, tree=tree)
    s.set_tensor(Xc)
    s.set_factors(init)
    f1 = s.sweep(1)
    lam, A = s.get_factors()
    f = np.concatenate([f1, s.sweep(1)])
    s.close()
    if variant == "NE":
        ref1, ref = O.cp_als_ne(X, init, 1), O.cp_als_ne(X, init, 2)
    else:
        ref1, ref = O.cp_als_qr(X, init, 1, variant=variant), O.cp_als_qr(X, init, 2, variant=variant)
    for k in range(len(dims)):
        assert rel(A[k], ref1["factors"][k]) <= 1e-9, (k, rel(A[k], ref1["factors"][k]))
    assert rel(lam, ref1["lam"]) <= 1e-9
    assert np.max(np.abs(f - np.array(ref["fits"]))) <= 1e-8, (f, ref["fits"])
