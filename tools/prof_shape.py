"""Profiling driver for an arbitrary cubical shape (perf only): python tools/prof_shape.py --n 75 --N 5 --R 32
[--variant QR] [--plans]; used under ncu for launch lists of the paper's shapes (tools/paper_perf.py)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2112_10855_b200 import cpqr

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=75)
ap.add_argument("--N", type=int, default=5)
ap.add_argument("--R", type=int, default=32)
ap.add_argument("--variant", default="QR")
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--plans", action="store_true")
a = ap.parse_args()
dims = (a.n,) * a.N
X = torch.rand(a.n ** a.N, dtype=torch.float64, device="cuda")
s = cpqr.CPQR(dims, a.R, a.variant, use_graph=False)
s.set_tensor(X)
s.init_factors(3)
if a.plans:
    for n in range(a.N):
        for st in s.debug_plan(n):
            print(n, st["kind"], st["modes"], "in %.3g out %.3g GF %.3g" % (st["in_elems"], st["out_elems"], st["flops"] / 1e9))
s.sweep(a.sweeps)
torch.cuda.synchronize()
print("fit", s.fit)
