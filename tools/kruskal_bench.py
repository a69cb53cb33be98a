"""Sine-of-sums sweeps/s: Kruskal input (X never formed) vs the dense path on the
formed tensor, same factors, CUDA graph, CUDA-event timing.  usage: python tools/kruskal_bench.py N n R [variant]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle as O
from paper_2112_10855_b200 import cpqr
N, n, R = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
variant = sys.argv[4] if len(sys.argv) > 4 else "QR"
lam_x, B = O.sine_of_sums_ktensor(N, n)
rng = np.random.default_rng(1)
A0 = [rng.standard_normal((n, R)) for _ in range(N)]
dims = (n,) * N
out = {}
for mode in ("kruskal", "dense"):
    s = cpqr.CPQR(dims, R, variant)
    if mode == "kruskal":
        s.set_ktensor(lam_x, B)
    else:
        # the formed tensor, built on the GPU from the factors (C order (I_N..I_1) = column-major)
        Bt = [torch.from_numpy(b).cuda() for b in B]
        X = torch.zeros(dims, dtype=torch.float64, device="cuda")
        for t in range(len(lam_x)):
            v = Bt[N - 1][:, t] * lam_x[t]
            for k in range(N - 2, -1, -1):
                v = torch.einsum("...,i->...i", v, Bt[k][:, t])
            X += v
        s.set_tensor(X.contiguous())
    s.set_factors(A0)
    s.sweep(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); f = s.sweep(20); e1.record(); torch.cuda.synchronize()
    out[mode] = (20 / (e0.elapsed_time(e1) / 1e3), f[-1])
    s.close()
print(f"sine-of-sums N={N} n={n} rank-{len(lam_x)} input, R={R} {variant}: "
      f"Kruskal {out['kruskal'][0]:.1f} sweeps/s (fit {out['kruskal'][1]:.10f}), "
      f"dense {out['dense'][0]:.1f} sweeps/s (fit {out['dense'][1]:.10f}), "
      f"speedup {out['kruskal'][0] / out['dense'][0]:.1f}x")
