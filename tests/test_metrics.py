"""The package's score (paper_2112_10855_b200/metrics.py, used by the collinear-grid workload)
equals the oracle's independent implementation."""
import numpy as np

import oracle as O
from paper_2112_10855_b200 import metrics


def test_score_matches_oracle():
    rng = np.random.default_rng(11)
    for R in (2, 4, 5):
        A = [rng.standard_normal((d, R)) for d in (9, 8, 7)]
        B = [a + 0.3 * rng.standard_normal(a.shape) for a in A]
        la, lb = rng.uniform(0.5, 2, R), rng.uniform(0.5, 2, R)
        p = rng.permutation(R)
        Bp = [b[:, p] for b in B]
        assert abs(metrics.score(la, A, lb[p], Bp) - O.score(la, A, lb[p], Bp)) <= 1e-13
        assert abs(metrics.score(la, A, la, A) - 1.0) <= 1e-13
