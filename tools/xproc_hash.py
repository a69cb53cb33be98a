"""Cross-process determinism probe: the full-size test's sequence for one config, hashed per stage."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import oracle as O
from paper_2112_10855_b200 import cpqr, synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
conf, Xc, truth, init = synth.make_problem(cfg)
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:10]
print("inputs", h(Xc), [h(a) for a in init])
variant = conf.variants[-1]
s = cpqr.CPQR(conf.dims, conf.R, variant, svd_tau=conf.svd_tau, fit_mode="direct" if cfg == 4 else "fast")
Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
s.set_tensor(Xd)
s.set_factors(init)
Qs = [O.qr_pos(a)[0] for a in init]
dbg = [s.debug_mode(n, Q_override=[Qs[k] if k != n else None for k in range(conf.N)]) for n in range(conf.N)]
print("debug", [(h(d["Y"]), h(d["W"]), h(d["R0"])) for d in dbg])
f1 = s.sweep(1)
lam, A = s.get_factors()
print("sweep1", h(f1), h(lam), [h(a) for a in A])
f = s.sweep(conf.sweeps - 1)
print("fits", h(f), f[:4])
