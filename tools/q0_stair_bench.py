"""Staircase vs dense Q0 apply: per-mode time of the Q0
apply phase (cpqr_get_profile ms[4], eager sweeps with CUDA events around each phase) and the
graph sweep time, CPQR_Q0_STAIR=0/1 interleaved, on the BASELINE configs and high-rank shapes.

  python tools/q0_stair_bench.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2112_10855_b200 import cpqr
    cases = [((400, 400, 400), 10), ((128, 128, 128, 128), 16), ((48, 48, 48, 48, 48), 8), ((1000, 1000, 1000), 32),
             ((40, 40, 40, 40), 32), ((64, 64, 64, 64), 24), ((24, 24, 24, 24, 24), 12)]
    print("| dims | R | Q0 apply dense (us/mode) | staircase | flop ratio | sweep dense (ms) | sweep staircase (ms) |")
    print("|---|---|---|---|---|---|---|")
    for dims, R in cases:
        N = len(dims)
        X = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda")
        rng = np.random.default_rng(0)
        init = [rng.standard_normal((d, R)) for d in dims]
        res = {}
        for stair in ("0", "1", "0", "1"):
            os.environ["CPQR_Q0_STAIR"] = stair
            s = cpqr.CPQR(dims, R, "QR", profile=True, use_graph=False)
            s.set_tensor(X)
            s.set_factors(init)
            s.sweep(1)
            s.profile(reset=True)
            s.sweep(3)
            q0 = s.profile()["ms"][4] / 3 / N * 1e3
            s.close()
            g = cpqr.CPQR(dims, R, "QR")
            g.set_tensor(X)
            g.set_factors(init)
            g.sweep(2)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g.sweep(10)
            torch.cuda.synchronize()
            sw = (time.perf_counter() - t0) / 10 * 1e3
            g.close()
            r = res.setdefault(stair, [1e30, 1e30])
            r[0], r[1] = min(r[0], q0), min(r[1], sw)
        nnz = sum((c + 1) ** (N - 1) for c in range(R))
        print(f"| {dims} | {R} | {res['0'][0]:.1f} | {res['1'][0]:.1f} | {nnz / (R ** N):.2f} | "
              f"{res['0'][1]:.3f} | {res['1'][1]:.3f} |", flush=True)
        del X
        torch.cuda.empty_cache()
    os.environ.pop("CPQR_Q0_STAIR", None)


if __name__ == "__main__":
    main()
