"""Stress determinism: repeat debug_mode of every mode and the tail pieces many times on C4."""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
conf, Xc, truth, init = synth.make_problem(cfg)
var = conf.variants[-1]
s = cpqr.CPQR(conf.dims, conf.R, var, svd_tau=conf.svd_tau)
s.set_tensor(torch.from_numpy(np.ascontiguousarray(Xc)).cuda())
s.set_factors(init)
for n in range(conf.N):
    seen = {k: set() for k in ("Y", "W", "Q0", "R0")}
    for r in range(reps):
        d = s.debug_mode(n)
        for k in seen:
            seen[k].add(h(d[k]))
    print("mode", n, {k: len(v) for k, v in seen.items()}, flush=True)
d = s.debug_mode(0)
sv = set(); qr = set()
for r in range(reps * 5):
    out, nt = s.debug_svd_solve(d["R0"], d["W"], conf.svd_tau)
    sv.add(h(out))
    Q, Rf = s.debug_qr(init[1] + 0.0)
    qr.add(h(Q) + h(Rf))
print("svd_solve variants", len(sv), "qr variants", len(qr))
