"""Relative-error curves of §4.3 on the GPU: the sine-of-sums tensor in its
rank-2^{N-1} Kruskal representation (never formed), a rank-N CP fit by CP-ALS (NE), CP-ALS-PINV,
CP-ALS-QR and CP-ALS-QR-SVD from the same random init, tolerance 0, 40 iterations, the relative
error ||X - Xh|| / ||X|| computed DIRECTLY (entry by entry from the factors) after
every iteration.  The paper's figures are not available, so this prints the curves (every 5th
iteration and the minimum) for the paper's cases N = 4 (n = 64, 128) and N = 5 (n = 32, 64).

  python tools/sine_curves.py [--iters 40] [--seed 1]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cases", default="4:64,4:128,5:32,5:64")
    args = ap.parse_args()
    for case in args.cases.split(","):
        N, n = (int(v) for v in case.split(":"))
        lam_x, B = sine_of_sums(N, n)
        g = np.random.default_rng(args.seed)
        A0 = [g.standard_normal((n, N)) for _ in range(N)]
        print(f"\n# sine of sums N={N} n={n}: input rank {len(lam_x)}, model rank R={N}, {args.iters} iterations,"
              f" direct relative error (every 5th iteration; min)")
        for variant, label in (("NE", "CP-ALS"), ("PINV", "CP-ALS-PINV"), ("QR", "CP-ALS-QR"), ("SVD", "CP-ALS-QR-SVD")):
            s = cpqr.CPQR((n,) * N, N, variant, fit_mode="direct")
            s.set_ktensor(lam_x, B)
            s.set_factors(A0)
            t0 = time.perf_counter()
            try:
                f = s.sweep(args.iters)
                err = 1.0 - f
                note = ""
            except cpqr.CpqrError as e:
                err, note = np.full(args.iters, np.nan), f" ({e})"
            dt = time.perf_counter() - t0
            s.close()
            pts = " ".join(f"{e:.1e}" for e in err[4::5])
            print(f"{label:14s} {pts}   min {np.nanmin(err) if np.any(np.isfinite(err)) else float('nan'):.2e}"
                  f"   [{dt * 1e3 / args.iters:.2f} ms/iter]{note}")


if __name__ == "__main__":
    main()
