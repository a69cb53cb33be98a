"""Profiling driver: one eager CP-ALS-QR sweep of the 10-way sine of sums (N = 10, n = 8, R = 10,
short modes) for an ncu launch list."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
sys.argv = ["x"]
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import sine_curves as sc
from paper_2112_10855_b200 import cpqr
lam, B = sc.sine_of_sums_rank_n(10, 8)
g = np.random.default_rng(1)
A0 = [g.standard_normal((8, 10)) for _ in range(10)]
s = cpqr.CPQR((8,) * 10, 10, "QR", fit_mode="direct", use_graph=False)
s.set_ktensor(lam, B); s.set_factors(A0)
s.sweep(1)
