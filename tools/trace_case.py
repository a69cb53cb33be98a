import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2112_10855_b200 import cpqr, synth
cfg = int(sys.argv[1])
conf = synth.CONFIGS[cfg]
X = torch.randn(int(np.prod(conf.dims)), dtype=torch.float64, device="cuda")
init = synth.init_factors(conf)
s = cpqr.CPQR(conf.dims, conf.R, conf.variants[0], svd_tau=conf.svd_tau, use_graph=False)
s.set_tensor(X); s.set_factors(init)
s.sweep(3)
