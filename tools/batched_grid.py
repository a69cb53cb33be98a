"""The collinear-factor study (Table 4.1) as FOUR batched
launches -- CP-ALS (NE), CP-ALS-PINV, CP-ALS-QR and CP-ALS-QR-SVD (cpqr_batched, one CTA per
problem, the device-side stopping rule of PAPER.md:532) -- over the 3 x 3 grid of noise
{1e-4, 1e-7, 1e-10} x collinearity {1-1e-4, 1-1e-7, 1-1e-10} plus a benign control column c = 0.5,
`trials` problems per cell (the paper: 100), 50^3 rank 5, shared random init per trial, up to 500
sweeps, tolerance 1e-15 on the change in relative error.  Reports per cell and method the median
score (Tomasi-Bro), sweeps and relative error ||X - Xh|| / ||X|| (computed on the
GPU from the factors), and each method's launch time; with --context also the per-context driver's
QR run (solver.cp_als, 12 solves in flight) for the batched-vs-context throughput ratio.

  python tools/batched_grid.py [trials] [--context]
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2112_10855_b200 import cpqr, metrics, solver, synth  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 100
context = "--context" in sys.argv
dims, R = (50, 50, 50), 5
noises = [1e-4, 1e-7, 1e-10]
colls = [0.5, 1 - 1e-4, 1 - 1e-7, 1 - 1e-10]  # c = 0.5: a benign control column
methods = ["NE", "PINV", "QR", "SVD"]
probs = []
for ci in range(len(colls)):
    for ni in range(3):
        for t in range(trials):
            conf, Xc, truth, init = synth.small_problem(dims, R, seed=7000 + 100 * (3 * ci + ni) + t,
                                                        eta=noises[ni], kind="congruence", c=colls[ci])
            probs.append((ci, ni, Xc, truth, init))
P = len(probs)
X = torch.from_numpy(np.stack([p[2] for p in probs])).cuda()
A0 = [torch.from_numpy(np.stack([np.ascontiguousarray(p[4][k].T) for p in probs])).cuda() for k in range(3)]
nX = torch.linalg.vector_norm(X.reshape(P, -1), dim=1)
res = {}
for m in methods:
    cpqr.batched_qr(X, A0, R, max_iters=2, tol=0.0, variant=m)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    A, lam, fits, iters = cpqr.batched_qr(X, A0, R, max_iters=500, tol=1e-15, variant=m)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    Xh = torch.einsum("pr,pri,prj,prk->pkji", lam, A[0], A[1], A[2])  # C order (I_3, I_2, I_1)
    rel = (torch.linalg.vector_norm((X - Xh).reshape(P, -1), dim=1) / nX).cpu().numpy()
    An = [a.cpu().numpy() for a in A]
    lamn, it = lam.cpu().numpy(), iters.cpu().numpy()
    sc = np.array([metrics.score(np.ones(R), probs[p][3], lamn[p], [An[k][p].T for k in range(3)])
                   if np.all(np.isfinite(lamn[p])) else 0.0 for p in range(P)])
    res[m] = dict(t=t, sweeps=int(it.sum()), iters=it, rel=rel, score=sc)

print(f"# collinear-factor grid, batched (cpqr_batched: one CTA per problem, one launch per method), 1 B200")
print(f"# {P} problems per method (50^3, R = 5; {len(colls)} x 3 cells x {trials} trials), up to 500 sweeps, tol 1e-15")
for m in methods:
    r = res[m]
    print(f"{m:5s}: {r['t']:.3f} s, {r['sweeps']} sweeps -> {r['sweeps'] / r['t']:.0f} sweeps/s")
if context:
    def job(p):
        out = solver.cp_als(probs[p][2], R, method="QR", init=probs[p][4], max_iters=500, tol=1e-15, chunk=10)
        return out["iters"]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(12) as ex:
        ctx = list(ex.map(job, range(P)))
    tc = time.perf_counter() - t0
    print(f"QR per-context driver (12 in flight): {tc:.3f} s, {sum(ctx)} sweeps -> {sum(ctx) / tc:.0f} sweeps/s")
print("# cell (noise, collinearity) | method | median score | median sweeps | median rel.err | converged (< 500)")
for ni in range(3):
    for ci in range(len(colls)):
        idx = [p for p in range(P) if probs[p][0] == ci and probs[p][1] == ni]
        cl = "0.5    " if ci == 0 else f"1-{1 - colls[ci]:.0e}"
        for m in methods:
            r = res[m]
            print(f"eta={noises[ni]:.0e} c={cl} | {m:5s} | {np.median(r['score'][idx]):.6f} | "
                  f"{np.median(r['iters'][idx]):5.0f} | {np.median(r['rel'][idx]):.3e} | "
                  f"{int(np.sum(r['iters'][idx] < 500))}/{len(idx)}")
