"""Run the full-size test file's earlier configs in this process, then the C4 hash sequence."""
import os, sys, runpy
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
for cfg, var in [(1, "QR"), (2, "QR"), (2, "NE"), (3, "QR"), (3, "SVD")]:
    conf, Xc, truth, init = synth.make_problem(cfg)
    s = cpqr.CPQR(conf.dims, conf.R, var, svd_tau=conf.svd_tau)
    Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
    s.set_tensor(Xd)
    s.set_factors(init)
    if var != "NE":
        for n in range(conf.N):
            s.debug_mode(n)
    s.sweep(conf.sweeps)
    s.close()
    del Xd
    torch.cuda.empty_cache()
sys.argv = ["xproc_hash.py", "4"]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "xproc_hash.py"), run_name="__main__")
