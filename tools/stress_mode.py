"""Repeat debug_mode(n) many times on a config; report the number of distinct Y results."""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
cfg, n, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
conf, Xc, truth, init = synth.make_problem(cfg)
s = cpqr.CPQR(conf.dims, conf.R, "SVD" if "SVD" in conf.variants else "QR", svd_tau=conf.svd_tau)
s.set_tensor(torch.from_numpy(np.ascontiguousarray(Xc)).cuda())
s.set_factors(init)
seen = {}
ref = None
for r in range(reps):
    y = s.debug_mode(n)["Y"]
    k = h(y)
    seen[k] = seen.get(k, 0) + 1
    if ref is None:
        ref = y
    elif k != h(ref) and seen[k] == 1:
        d = np.abs(y - ref)
        idx = np.argwhere(d > 0)
        print("  diff at", len(idx), "entries, max", d.max(), "first idx", idx[:3].tolist(), "shape", y.shape)
print("cfg", cfg, "mode", n, "variants", sorted(seen.values(), reverse=True))
