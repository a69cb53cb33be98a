"""Profiling driver (perf only, no parity): a BASELINE config with a device-random tensor, a few
sweeps through the C-ABI.  Used under ncu:  python tools/prof_case.py --config 5 --sweeps 1"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2112_10855_b200 import cpqr, synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--variant", default=None)
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--graph", type=int, default=0)
ap.add_argument("--profile", type=int, default=1)
ap.add_argument("--tree", type=int, default=0)
ap.add_argument("--world", type=int, default=1, help="virtual ranks (CPQR_COMM_LOCAL)")
a = ap.parse_args()
conf = synth.CONFIGS[a.config]
variant = a.variant or conf.variants[0]
torch.manual_seed(0)
X = torch.randn(int(np.prod(conf.dims)), dtype=torch.float64, device="cuda")
init = synth.init_factors(conf)
s = cpqr.CPQR(conf.dims, conf.R, variant, svd_tau=conf.svd_tau, use_graph=bool(a.graph), profile=bool(a.profile),
               tree=bool(a.tree), world=a.world, comm="local")
s.set_tensor(X)
s.set_factors(init)
s.sweep(a.warm)
s.profile(reset=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
f = s.sweep(a.sweeps)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
p = s.profile()
names = ["stream_pass", "rest_ttm", "factor_qr_tail", "q0_compute", "q0_apply", "other", "exchange"]
print(conf.name, variant, "ms/sweep %.3f" % (1e3 * dt / a.sweeps),
      {n: round(v / a.sweeps, 4) for n, v in zip(names, p["ms"])}, "launches/sweep", s.launches_per_sweep())
