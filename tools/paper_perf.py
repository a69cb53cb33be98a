#!/usr/bin/env python
"""The paper's performance experiment on one B200 (Fig. "its", Table 3.1).

"Randomly generated cubical tensors of three, four, and five modes" of dimension 700, 300 and 75,
increasing rank, "the average iteration time over 10 iterations (omitting the first iteration)",
for CP-ALS, CP-ALS-PINV, CP-ALS-QR and CP-ALS-QR-SVD, broken down into the components of Table 3.1
(PAPER.md:495-510), with the slowdown ratio QR / CP-ALS per rank.  The ranks are only in the
paper's figure, not in its text: R in {4, 8, 16, 32} here (R <= 32 is the
library's limit).  Entries are U[0,1) from torch's device generator (seeded); the tensor is never
on the host.  No oracle run at these sizes: every cell checks instead that the four solvers, which
share no Multi-TTM / MTTKRP code path choice (NE and PINV stream X against A_k and contract the
Khatri-Rao diagonal, QR and SVD against Q_k and apply Q0), reach the same fit after the same
sweeps from the same init to 1e-8 -- for a well-conditioned random tensor they are the same
iteration in exact arithmetic.

Per cell: `iter_ms` = CUDA-graph sweeps timed with CUDA events (10 sweeps after 1 warm-up);
the breakdown = cpqr_get_timings of eager sweeps (profile = 1; the phases then include launch gaps
and the V_n QR runs inline instead of hidden on the side stream, so they sum to more than iter_ms).

  python tools/paper_perf.py [--shapes 3 4 5] [--ranks 4 8 16 32] [--n4 300] [--iters 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2112_10855_b200 import cpqr

PHASES = ["stream_pass", "rest_ttm", "factor_qr_tail", "q0_compute", "q0_apply", "other", "exchange"]


def device_uniform(numel, seed):
    """U[0,1) fp64 on the device, generated in chunks (the generator state carries across them)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    X = torch.empty(numel, dtype=torch.float64, device="cuda")
    step = 1 << 28
    for o in range(0, numel, step):
        X[o:o + step].uniform_(0.0, 1.0, generator=g)
    return X


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", type=int, nargs="+", default=[3, 4, 5])
    ap.add_argument("--ranks", type=int, nargs="+", default=[4, 8, 16, 32])
    ap.add_argument("--n3", type=int, default=700)
    ap.add_argument("--n4", type=int, default=300)
    ap.add_argument("--n5", type=int, default=75)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    side = {3: a.n3, 4: a.n4, 5: a.n5}
    rows = []
    for N in a.shapes:
        dims = (side[N],) * N
        numel = int(np.prod(dims))
        X = device_uniform(numel, 1000 + N)
        for R in a.ranks:
            cell = {}
            for variant in ["NE", "PINV", "QR", "SVD"]:
                # timed: CUDA-graph sweeps, the first iteration omitted
                s = cpqr.CPQR(dims, R, variant)
                s.set_tensor(X)
                s.init_factors(7 + R)
                s.sweep(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                fits = s.sweep(a.iters)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                flags = s.flags
                s.close()
                # breakdown: eager sweeps with events around each phase
                p = cpqr.CPQR(dims, R, variant, profile=True, use_graph=False)
                p.set_tensor(X)
                p.init_factors(7 + R)
                p.sweep(1)
                p.profile(reset=True)
                p.sweep(2)
                pr = p.profile(reset=True)
                p.close()
                ph = {k: v / 2 for k, v in zip(PHASES, pr["ms"])}
                cell[variant] = dict(iter_ms=ms, fit=float(fits[-1]), flags=int(flags), phases=ph)
            f = [cell[v]["fit"] for v in cell]
            agree = max(f) - min(f)
            row = dict(dims=list(dims), R=R, cells=cell, fit_spread=agree,
                       slowdown_qr_over_ne=cell["QR"]["iter_ms"] / cell["NE"]["iter_ms"],
                       slowdown_svd_over_pinv=cell["SVD"]["iter_ms"] / cell["PINV"]["iter_ms"])
            rows.append(row)
            print(json.dumps(row), flush=True)
            if agree > 1e-8:
                print("CHECK FAILED: the four solvers disagree", dims, R, f, flush=True)
        del X
        torch.cuda.empty_cache()
    print("\n| tensor | R | CP-ALS | CP-ALS-PINV | CP-ALS-QR | CP-ALS-QR-SVD | QR / CP-ALS | fit spread | "
          "QR breakdown: Multi-TTM (pass + rest) / QR of factors + solve (tail) / computing Q0 / applying Q0 / other |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        c = r["cells"]
        q = c["QR"]["phases"]
        print(f"| {r['dims'][0]}^{len(r['dims'])} | {r['R']} | {c['NE']['iter_ms']:.3f} | {c['PINV']['iter_ms']:.3f} | "
              f"{c['QR']['iter_ms']:.3f} | {c['SVD']['iter_ms']:.3f} | {r['slowdown_qr_over_ne']:.2f}x | "
              f"{r['fit_spread']:.1e} | {q['stream_pass'] + q['rest_ttm']:.3f} / {q['factor_qr_tail']:.3f} / "
              f"{q['q0_compute']:.3f} / {q['q0_apply']:.3f} / {q['other']:.3f} |")


if __name__ == "__main__":
    main()
