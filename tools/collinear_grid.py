"""The paper's collinear-factor experiment (§4.2) on the
GPU: 50^3 rank-5 tensors with factor congruence c in {1-1e-4, 1-1e-7, 1-1e-10} and noise
eta in {1e-4, 1e-7, 1e-10} (synth.py recipe: A = U chol(C)^T, noise scaled to eta ||X||), shared
random init per trial, up to 500 sweeps, tolerance 1e-15 on the change in relative error.  Methods:
CP-ALS (NE), CP-ALS-PINV, CP-ALS-QR, CP-ALS-QR-SVD and the robust NE -> QR-SVD policy
(PAPER.md:660).  A control column c = 0.5 checks that construction + score reach 1 when the
problem is benign.
Reports per cell and method the median score, sweeps and relative error.
Many small independent solves run concurrently (one context + stream each, a thread pool).

  python tools/collinear_grid.py [trials] [workers]
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10855_b200 import metrics, solver, synth  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 5
workers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims, R = (50, 50, 50), 5
noises = [1e-4, 1e-7, 1e-10]
colls = [0.5, 1 - 1e-4, 1 - 1e-7, 1 - 1e-10]  # c = 0.5: a benign control column
methods = ["NE", "PINV", "QR", "SVD", "robust"]


def relerr(Xc, lam, A):
    Xh = np.einsum("r,ir,jr,kr->kji", lam, A[0], A[1], A[2])  # C order (I_3, I_2, I_1)
    return float(np.linalg.norm(Xc - Xh) / np.linalg.norm(Xc))


def job(args):
    ci, ni, t, m = args
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=7000 + 100 * (3 * ci + ni) + t,
                                                eta=noises[ni], kind="congruence", c=colls[ci])
    out = solver.cp_als(Xc, R, method=m, init=init, max_iters=500, tol=1e-15, chunk=10)
    if out["diverged"]:  # plain NE on a numerically singular S (LU on a zero pivot)
        return (ci, ni, m), (0.0, out["iters"], float("nan"), False, "diverged")
    sc = metrics.score(np.ones(R), truth, out["lam"], out["factors"])
    return (ci, ni, m), (sc, out["iters"], relerr(Xc, out["lam"], out["factors"]), out["converged"],
                         out["trace"][-1][0])


tasks = [(ci, ni, t, m) for ci in range(len(colls)) for ni in range(3) for t in range(trials) for m in methods]
t0 = time.perf_counter()
with ThreadPoolExecutor(workers) as ex:
    res = list(ex.map(job, tasks))
dt = time.perf_counter() - t0
agg = {}
for key, val in res:
    agg.setdefault(key, []).append(val)
print(f"# collinear grid: {len(tasks)} solves ({trials} trials x {3 * len(colls)} cells x {len(methods)} methods), "
      f"{workers} concurrent, {dt:.1f} s wall")
print("# cell (noise, congruence) | method | median score | median sweeps | median rel.err | converged | ends in")
for ni in range(3):
    for ci in range(len(colls)):
        for m in methods:
            v = agg[(ci, ni, m)]
            sc, it, re = (np.nanmedian([x[i] for x in v]) if i == 2 and not all(np.isnan([x[2] for x in v]))
                          else np.median([x[i] for x in v]) for i in range(3))
            conv = sum(x[3] for x in v)
            ends = ",".join(sorted({x[4] for x in v}))
            cs = f"c={colls[ci]:.1f}  " if colls[ci] < 0.9 else f"c=1-{1 - colls[ci]:.0e}"
            print(f"eta={noises[ni]:.0e} {cs} | {m:6s} | {sc:.6f} | {it:5.0f} | {re:.3e} | "
                  f"{conv}/{len(v)} | {ends}")
