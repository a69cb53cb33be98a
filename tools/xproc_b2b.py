"""Warm-up configs, then C4 SVD: 1 sweep, then 19 back-to-back sweeps; print the fits (full precision)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
graph = sys.argv[1] == "1"
warm = sys.argv[2] == "1"
if warm:
    for cfg, var in [(1, "QR"), (2, "QR"), (2, "NE"), (3, "QR"), (3, "SVD")]:
        conf, Xc, truth, init = synth.make_problem(cfg)
        s = cpqr.CPQR(conf.dims, conf.R, var, svd_tau=conf.svd_tau)
        Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
        s.set_tensor(Xd); s.set_factors(init); s.sweep(conf.sweeps); s.close()
        del Xd; torch.cuda.empty_cache()
conf, Xc, truth, init = synth.make_problem(4)
s = cpqr.CPQR(conf.dims, conf.R, "SVD", svd_tau=conf.svd_tau, fit_mode="direct", use_graph=graph)
Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
s.set_tensor(Xd); s.set_factors(init)
f = np.concatenate([s.sweep(1), s.sweep(19)])
print(" ".join("%.17g" % v for v in f[[1, 3, 5, 9, 19]]))
