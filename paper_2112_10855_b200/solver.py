"""CP-ALS driver with the paper's stopping rule and the robust NE -> QR-SVD policy.

cp_als(X, R, method): the caller-facing solve (SPEC-style cp_als(X, opts, method) -> result) on top
of libcpqr's fixed-count sweeps (cpqr_sweep never stops early, PAPER.md:362 leaves convergence to
the caller).  Sweeps run in chunks; the solve stops at the first sweep whose change in relative
error 1 - fit is below `tol` (tolerance on the change in relative error), or after
`max_iters` sweeps.  The reported iteration count is that sweep; the returned factors are those
at the end of its chunk (reading 31: at most chunk - 1 further sweeps of a converged iteration).

method = "robust": normal-equations CP-ALS by default, switching to CP-ALS-QR-SVD from the current
factors once the NE solve flags ill-conditioning (CPQR_FLAG_NE_ILLCOND: kappa(S_n) estimate above
1e8, or the LU fallback) -- the policy the paper proposes.
"""
from __future__ import annotations

import numpy as np

from . import cpqr


def cp_als(X, R, method="QR", init=None, max_iters=500, tol=1e-15, chunk=10, svd_tau=-1.0, seed=0,
           device=0, use_graph=True):
    """X: C-ordered (I_N..I_1) numpy array or torch tensor (the library's layout).  init: list of
    I_k x R host arrays (default: N(0,1) from `seed`).  Returns dict(lam, factors, fits, iters,
    converged, trace) with trace the list of (method, first sweep) segments."""
    dims = tuple(int(d) for d in np.shape(X)[::-1])
    if init is None:
        rng = np.random.default_rng(seed)
        init = [rng.standard_normal((d, R)) for d in dims]
    methods = ["NE", "SVD"] if method == "robust" else [method]
    factors, lam = init, None
    fits, trace, it, converged, diverged = [], [], 0, False, False
    for mi, m in enumerate(methods):
        s = cpqr.CPQR(dims, R, m, svd_tau=svd_tau, device=device, use_graph=use_graph)
        s.set_tensor(X)
        s.set_factors(factors, lam)
        trace.append((m, it))
        prev = fits[-1] if fits else None
        switch = False
        robust_ne = mi + 1 < len(methods)  # the NE phase of the robust policy: check every sweep
        good = (lam, factors)
        while it < max_iters and not converged:
            k = 1 if robust_ne else min(chunk, max_iters - it)
            try:
                f = s.sweep(k)
            except cpqr.CpqrError as e:
                if "EDIVERGED" not in str(e):
                    raise
                if not robust_ne:
                    diverged = True
                    break
                switch = True  # restart from the last finite factors
                break
            for j, v in enumerate(f):
                fits.append(float(v))
                if prev is not None and abs(v - prev) < tol:
                    converged = True
                    it += j + 1
                    break
                prev = float(v)
            else:
                it += k
            if robust_ne and not converged:
                if s.flags & (cpqr.FLAG_NE_ILLCOND | cpqr.FLAG_NE_CHOL_FALLBACK):
                    switch = True
                    break
                good = s.get_factors()
        if switch:
            lam, factors = good
        else:
            lam, factors = s.get_factors()
        s.close()
        if converged or not switch:
            break
    return dict(lam=lam, factors=factors, fits=np.array(fits), iters=it, converged=converged,
                diverged=diverged, trace=trace)
