"""Stress run-to-run determinism of whole sweeps (CUDA-graph replay, default options): the same
init, one sweep, hashed factors / lambda / fit, `reps` times per (config, variant, tree).  Any
second hash is a race.  Usage: python tools/stress_sweep.py CFG[,CFG..] REPS [tree|per_mode|both]"""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3,4").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
which = sys.argv[3] if len(sys.argv) > 3 else "both"
trees = {"tree": [True], "per_mode": [False]}.get(which, [False, True])
bad = 0
for cfg in cfgs:
    conf, Xc, truth, init = synth.make_problem(cfg)
    Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
    for var in conf.variants:
        for tree in trees:
            s = cpqr.CPQR(conf.dims, conf.R, var, svd_tau=conf.svd_tau, tree=tree)
            s.set_tensor(Xd)
            seen = {}
            for r in range(reps):
                s.set_factors(init)
                f = s.sweep(2)
                lam, A = s.get_factors()
                key = h(f) + h(lam) + "".join(h(a) for a in A)
                seen.setdefault(key, []).append(r)
            s.close()
            bad += len(seen) > 1
            print(cfg, var, "tree" if tree else "per_mode", "distinct", len(seen),
                  {k: v[:5] for k, v in seen.items()} if len(seen) > 1 else "", flush=True)
    del Xd
    torch.cuda.empty_cache()
print("NONDETERMINISTIC" if bad else "deterministic")
