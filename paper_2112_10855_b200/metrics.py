"""Evaluation metrics for CP decompositions (host-side numpy; not part of the GPU hot path).

score(): the similarity of two Kruskal tensors up to scaling and permutation used by the paper's
collinear-factor experiments (reading 30).  Independent of the
oracle's implementation (tests/test_metrics.py pins the two against each other).
"""
from __future__ import annotations

import itertools

import numpy as np


def _unit_columns(factors, lam):
    w = np.abs(np.asarray(lam, dtype=np.float64)).copy()
    out = []
    for F in factors:
        F = np.asarray(F, dtype=np.float64)
        nrm = np.sqrt(np.einsum("ij,ij->j", F, F))
        w = w * nrm
        out.append(F / np.where(nrm > 0.0, nrm, 1.0))
    return out, w


def score(lam_true, A_true, lam_est, A_est) -> float:
    """max over component matchings p of mean_r [(1 - |w_r - v_p(r)| / max(w_r, v_p(r)))
    * prod_k |<a_r^(k), b_p(r)^(k)>|] with unit-norm columns and norms folded into the weights
    w, v.  1 for equivalent Kruskal tensors, 0 for unrelated ones."""
    U, w = _unit_columns(A_true, lam_true)
    V, v = _unit_columns(A_est, lam_est)
    R = U[0].shape[1]
    sim = np.ones((R, R))
    for Uk, Vk in zip(U, V):
        sim = sim * np.abs(Uk.T @ Vk)
    big = np.maximum.outer(w, v)
    sim = sim * (1.0 - np.abs(np.subtract.outer(w, v)) / np.where(big > 0.0, big, 1.0))
    best = 0.0
    for perm in itertools.permutations(range(R)):
        best = max(best, float(sim[np.arange(R), perm].mean()))
    return best
