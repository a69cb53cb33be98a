"""Compare one sweep's factors / lambda / fit bitwise between two builds of libcpqr (run twice with
CPQR_LIB set, hashes printed): python tools/xlib_bitwise.py CFG[,CFG..] [tree]"""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:10]
for cfg in [int(c) for c in sys.argv[1].split(",")]:
    conf, Xc, truth, init = synth.make_problem(cfg)
    s = cpqr.CPQR(conf.dims, conf.R, conf.variants[0], svd_tau=conf.svd_tau, tree=len(sys.argv) > 2)
    s.set_tensor(torch.from_numpy(np.ascontiguousarray(Xc)).cuda())
    s.set_factors(init)
    f = s.sweep(2)
    lam, A = s.get_factors()
    print(cfg, h(f) + h(lam) + "".join(h(a) for a in A), flush=True)
    s.close()
