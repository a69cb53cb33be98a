"""Per-sweep factor hashes (one graph replay per call) after running the earlier full-size configs."""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
warm = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if warm:
    for cfg, var in [(1, "QR"), (2, "QR"), (2, "NE"), (3, "QR"), (3, "SVD")]:
        conf, Xc, truth, init = synth.make_problem(cfg)
        s = cpqr.CPQR(conf.dims, conf.R, var, svd_tau=conf.svd_tau)
        Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
        s.set_tensor(Xd); s.set_factors(init); s.sweep(conf.sweeps); s.close()
        del Xd; torch.cuda.empty_cache()
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
conf, Xc, truth, init = synth.make_problem(4)
s = cpqr.CPQR(conf.dims, conf.R, "SVD", svd_tau=conf.svd_tau, fit_mode="direct")
Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
s.set_tensor(Xd); s.set_factors(init)
out = []
for it in range(8):
    f = s.sweep(1)
    lam, A = s.get_factors()
    out.append(h(lam) + ":" + ",".join(h(a) for a in A))
print(" | ".join(out))
