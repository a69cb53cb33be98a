"""Collinear-factor grid with CP-ALS-QR as ONE batched launch (cpqr_batched_qr,
one CTA per problem, device-side stopping rule) vs the per-context driver (solver.cp_als, 12 solves
in flight).  usage: python tools/batched_grid.py [trials]"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2112_10855_b200 import cpqr, metrics, solver, synth  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dims, R = (50, 50, 50), 5
noises = [1e-4, 1e-7, 1e-10]
colls = [1 - 1e-4, 1 - 1e-7, 1 - 1e-10]
probs = []
for ci in range(3):
    for ni in range(3):
        for t in range(trials):
            conf, Xc, truth, init = synth.small_problem(dims, R, seed=7000 + 100 * (3 * ci + ni) + t,
                                                        eta=noises[ni], kind="congruence", c=colls[ci])
            probs.append((ci, ni, Xc, truth, init))
P = len(probs)
X = torch.from_numpy(np.stack([p[2] for p in probs])).cuda()
A0 = [torch.from_numpy(np.stack([np.ascontiguousarray(p[4][k].T) for p in probs])).cuda() for k in range(3)]
cpqr.batched_qr(X, A0, R, max_iters=2, tol=0.0)  # warm-up
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
A, lam, fits, iters = cpqr.batched_qr(X, A0, R, max_iters=500, tol=1e-15)
e1.record()
torch.cuda.synchronize()
tb = e0.elapsed_time(e1) / 1e3
A = [a.cpu().numpy() for a in A]
lam, iters = lam.cpu().numpy(), iters.cpu().numpy()
sb = [metrics.score(np.ones(R), probs[p][3], lam[p], [A[k][p].T for k in range(3)]) for p in range(P)]


def job(p):
    out = solver.cp_als(probs[p][2], R, method="QR", init=probs[p][4], max_iters=500, tol=1e-15, chunk=10)
    return out["iters"], metrics.score(np.ones(R), probs[p][3], out["lam"], out["factors"])


t0 = time.perf_counter()
with ThreadPoolExecutor(12) as ex:
    ctx = list(ex.map(job, range(P)))
tc = time.perf_counter() - t0
sweeps_b = int(iters.sum())
print(f"# {P} problems (50^3, R = 5; 9 cells x {trials} trials), CP-ALS-QR, up to 500 sweeps, tol 1e-15")
print(f"batched (one CTA per problem, one launch): {tb:.3f} s, {sweeps_b} sweeps -> {sweeps_b / tb:.0f} sweeps/s")
print(f"per-context driver (12 in flight):          {tc:.3f} s, {sum(c[0] for c in ctx)} sweeps -> "
      f"{sum(c[0] for c in ctx) / tc:.0f} sweeps/s")
print("# cell | median score batched / context | median sweeps batched / context")
for ni in range(3):
    for ci in range(3):
        idx = [p for p in range(P) if probs[p][0] == ci and probs[p][1] == ni]
        print(f"eta={noises[ni]:.0e} c=1-{1 - colls[ci]:.0e} | {np.median([sb[p] for p in idx]):.6f} / "
              f"{np.median([ctx[p][1] for p in idx]):.6f} | {np.median(iters[idx]):.0f} / "
              f"{np.median([ctx[p][0] for p in idx]):.0f}")
