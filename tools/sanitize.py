"""Small cases that launch every kernel of libcpqr, for compute-sanitizer (racecheck, synccheck,
memcheck, initcheck).  Each case runs a context through set_tensor / set_factors / two sweeps
(CUDA graph, and eagerly for the first case) and prints its fits; run it under the sanitizer:

  compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize.py

Coverage: strided TMA pass (8 warps / 4 producers, 4 warps x 2 CTAs per SM, stream-K split and
fix-up), fibre TMA pass, fused slice TMA pass (NF = 2 and 4, slices split across CTAs + fix-up),
small-slice pass, register-staged fallbacks (odd leading dimension), dimension tree, V_n QR
(staircase Householder and CholeskyQR2), Q0 apply, cluster tail (CholeskyQR2) with its gated
Householder TSQR fallback, one-CTA tail of the overlap schedule, QR-SVD pseudo-inverse, NE / PINV
tails and MTTKRP diagonal contraction, virtual ranks, Kruskal input with the DIRECT fit, the tall
factor fallback, batched small problems.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2112_10855_b200 import cpqr, synth  # noqa: E402

CASES = [
    # dims, R, variant, options, env
    ((70, 66, 34), 32, "QR", {}, {"CPQR_STREAMK": "1"}),
    ((70, 66, 34), 32, "QR", {"use_graph": False}, {"CPQR_OVERLAP": "1"}),
    ((37, 29, 43), 7, "SVD", {}, {}),
    ((64, 48, 40), 10, "QR", {}, {"CPQR_OVERLAP": "0"}),
    ((24, 300, 6, 5), 4, "QR", {}, {}),
    ((24, 130, 7, 6), 6, "SVD", {"tree": True}, {}),
    ((9, 8, 8, 6, 8), 4, "SVD", {}, {}),
    ((40, 36, 24), 6, "NE", {}, {}),
    ((16, 14, 12, 16), 6, "PINV", {}, {}),
    ((600, 40, 30), 8, "QR", {}, {"CPQR_OVERLAP": "0"}),
    ((30, 38, 48), 5, "QR", {"world": 4, "comm": "local"}, {}),
    ((40, 36, 24), 6, "NE", {"world": 2, "comm": "local"}, {}),
]


def run_case(dims, R, variant, opts, env, illcond=False):
    for k, v in env.items():
        os.environ[k] = v
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=91, eta=0.05)
    A0 = [a.copy() for a in init]
    if illcond:
        A0[1][:, 1] = A0[1][:, 0] * (1 + 1e-9)  # kappa ~ 1e9: CholeskyQR2 hands over to Householder
    s = cpqr.CPQR(dims, R, variant, **opts)
    s.set_tensor(Xc)
    s.set_factors(A0)
    f = s.sweep(2)
    s.close()
    for k in env:
        del os.environ[k]
    print(dims, R, variant, opts, env, "illcond" if illcond else "", f, flush=True)


def main():
    for c in CASES:
        run_case(*c)
    run_case((300, 40, 30), 8, "QR", {}, {"CPQR_OVERLAP": "0"}, illcond=True)
    # Kruskal input, DIRECT fit
    lam_x = np.array([1.0, -0.5, 0.25])
    g = np.random.default_rng(3)
    B = [g.standard_normal((12, 3)) for _ in range(4)]
    s = cpqr.CPQR((12,) * 4, 3, "QR", fit_mode="direct")
    s.set_ktensor(lam_x, B)
    s.set_factors([g.standard_normal((12, 3)) for _ in range(4)])
    print("ktensor", s.sweep(2), flush=True)
    s.close()
    # tall factor: multi-kernel CholeskyQR2 + the gated one-CTA fallback (debug_qr on kappa 1e10)
    m, R = 4000, 8
    U, _ = np.linalg.qr(g.standard_normal((m, R)))
    A = U @ np.diag(np.logspace(0, -10, R))
    s = cpqr.CPQR((m, m), R, "QR")
    Q, Rf = s.debug_qr(A)
    print("tall qr", float(np.linalg.norm(Q.T @ Q - np.eye(R))), flush=True)
    s.close()
    # batched small problems (one CTA each)
    import torch
    P, dims, R = 4, (12, 10, 9), 3
    Xs = torch.from_numpy(np.stack([synth.small_problem(dims, R, seed=70 + p)[1] for p in range(P)])).cuda()
    A0 = [torch.from_numpy(np.stack([g.standard_normal((R, d)) for _ in range(P)])).cuda() for d in dims]
    out = cpqr.batched_qr(Xs, A0, R, max_iters=5)
    torch.cuda.synchronize()
    print("batched iters", out[3].cpu().numpy(), flush=True)


if __name__ == "__main__":
    main()
