"""GPU tests of the caller-facing driver (paper_2112_10855_b200/solver.py): the paper's stopping
rule and the robust NE -> QR-SVD policy."""
import numpy as np
import pytest

import oracle as O
from paper_2112_10855_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_10855_b200 import solver
    return solver


def test_stopping_rule_matches_oracle_trajectory(solver):
    """cp_als(QR) stops at the first sweep whose fit change is below tol; its fits are the oracle's
    CP-ALS-QR fits up to that sweep."""
    dims, R = (20, 18, 16), 3
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=19, eta=1e-3)
    out = solver.cp_als(Xc, R, method="QR", init=init, max_iters=60, tol=1e-10, chunk=7)
    ref = O.cp_als_qr(O.as_tensor(Xc), init, len(out["fits"]))
    assert np.max(np.abs(out["fits"] - np.array(ref["fits"]))) <= 1e-8
    d = np.abs(np.diff(out["fits"]))
    k = out["iters"]
    if out["converged"]:
        assert d[k - 2] < 1e-10 and np.all(d[: k - 2] >= 1e-10)


def test_robust_policy_switches_on_ill_conditioning(solver):
    """Congruence 1 - 1e-10 with 1e-10 noise: the normal equations are ill-conditioned, the NE run
    raises CPQR_FLAG_NE_ILLCOND and the robust driver continues with QR-SVD from the current
    factors; a well-conditioned problem stays on NE throughout."""
    R = 4
    conf, Xc, truth, init = synth.small_problem((30, 28, 26), R, seed=23, eta=1e-10, kind="congruence",
                                                c=1.0 - 1e-10)
    out = solver.cp_als(Xc, R, method="robust", init=init, max_iters=40, tol=1e-15, chunk=5)
    assert [m for m, _ in out["trace"]] == ["NE", "SVD"]
    conf, Xc, truth, init = synth.small_problem((30, 28, 26), R, seed=23, eta=1e-2)
    out = solver.cp_als(Xc, R, method="robust", init=init, max_iters=40, tol=1e-15, chunk=5)
    assert [m for m, _ in out["trace"]] == ["NE"]
