"""Relative-error curves of §4.3 on the GPU: the sine-of-sums tensor in its
rank-2^{N-1} Kruskal representation (never formed), a rank-N CP fit by CP-ALS (NE), CP-ALS-PINV,
CP-ALS-QR and CP-ALS-QR-SVD from the same random init, tolerance 0, 40 iterations, the relative
error ||X - Xh|| / ||X|| computed DIRECTLY (entry by entry from the factors) after
every iteration.  The paper's figures are not available, so this prints the curves (every 5th
iteration and the minimum) for the paper's cases N = 4 (n = 64, 128) and N = 5 (n = 32, 64), and
the 10-way case (n = 8, "rank-10 representation" read as the rank-N input of
Eq. (sinsum_rkd), alpha_j = (j-1) pi / N, reading 33; model rank 10 > I_k = 8, the short-mode path)
from several random initializations (the paper shows two).

  python tools/sine_curves.py [--iters 40] [--seed 1] [--cases 4:64,4:128,5:32,5:64,10:8r]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2112_10855_b200 import cpqr  # noqa: E402


def sine_of_sums(N, n):
    """Rank-2^{N-1} representation of sin(x_1 + .. + x_N), x = 2 pi i / n."""
    x = 2.0 * np.pi * np.arange(n) / n
    terms = [t for t in range(1 << N) if bin(t).count("1") % 2 == 1]
    lam = np.array([(-1.0) ** ((bin(t).count("1") - 1) // 2) for t in terms])
    B = [np.stack([np.sin(x) if (t >> j) & 1 else np.cos(x) for t in terms], axis=1) for j in range(N)]
    return lam, B


def sine_of_sums_rank_n(N, n):
    """The rank-N representation (Eq. (sinsum_rkd)), alpha_j = (j-1) pi / N."""
    x = 2.0 * np.pi * np.arange(n) / n
    a = np.pi * np.arange(N) / N
    B = [np.stack([np.sin(x) if k == j else np.sin(x + a[k] - a[j]) / np.sin(a[k] - a[j]) for j in range(N)], axis=1)
         for k in range(N)]
    return np.ones(N), B


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cases", default="4:64,4:128,5:32,5:64,10:8r")
    ap.add_argument("--seeds10", default="1,2,3")
    args = ap.parse_args()
    for case in args.cases.split(","):
        rank_n = case.endswith("r")
        N, n = (int(v) for v in case.rstrip("r").split(":"))
        lam_x, B = sine_of_sums_rank_n(N, n) if rank_n else sine_of_sums(N, n)
        for seed in ([int(v) for v in args.seeds10.split(",")] if N == 10 else [args.seed]):
            run_case(N, n, lam_x, B, seed, args.iters)


def run_case(N, n, lam_x, B, seed, iters):
    g = np.random.default_rng(seed)
    A0 = [g.standard_normal((n, N)) for _ in range(N)]
    print(f"\n# sine of sums N={N} n={n}: input rank {len(lam_x)}, model rank R={N}, {iters} iterations,"
          f" init seed {seed}, direct relative error (every 5th iteration; min)", flush=True)
    for variant, label in (("NE", "CP-ALS"), ("PINV", "CP-ALS-PINV"), ("QR", "CP-ALS-QR"), ("SVD", "CP-ALS-QR-SVD")):
        s = cpqr.CPQR((n,) * N, N, variant, fit_mode="direct")
        s.set_ktensor(lam_x, B)
        s.set_factors(A0)
        t0 = time.perf_counter()
        try:
            f = s.sweep(iters)
            err = 1.0 - f
            note = ""
        except cpqr.CpqrError as e:
            err, note = np.full(iters, np.nan), f" ({e})"
        dt = time.perf_counter() - t0
        s.close()
        pts = " ".join(f"{e:.1e}" for e in err[4::5])
        print(f"{label:14s} {pts}   min {np.nanmin(err) if np.any(np.isfinite(err)) else float('nan'):.2e}"
              f"   [{dt * 1e3 / iters:.2f} ms/iter]{note}", flush=True)


if __name__ == "__main__":
    main()
