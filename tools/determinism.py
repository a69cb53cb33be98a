"""Bitwise run-to-run determinism probe: debug_mode (Y, W, Q0, R0) of every mode and whole sweeps,
repeated in one process on a BASELINE config (default C4).  usage: python tools/determinism.py [cfg] [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2112_10855_b200 import cpqr, synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
warm_cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if warm_cfg:  # run another config first in this process (as the full-size test file does)
    c2, X2, _, i2 = synth.make_problem(warm_cfg)
    s = cpqr.CPQR(c2.dims, c2.R, c2.variants[0], svd_tau=c2.svd_tau)
    s.set_tensor(torch.from_numpy(np.ascontiguousarray(X2)).cuda())
    s.set_factors(i2)
    s.sweep(3)
    s.close()
conf, Xc, truth, init = synth.make_problem(cfg)
variant = conf.variants[-1]
Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
N = conf.N
base = None
for rep in range(reps):
    s = cpqr.CPQR(conf.dims, conf.R, variant, svd_tau=conf.svd_tau)
    s.set_tensor(Xd)
    s.set_factors(init)
    outs = [s.debug_mode(n) for n in range(N)]
    fits = s.sweep(conf.sweeps)
    lam, A = s.get_factors()
    s.close()
    cur = (outs, fits, lam, A)
    if base is None:
        base = cur
        continue
    diffs = []
    for n in range(N):
        for key in ("Y", "W", "Q0", "R0"):
            if not np.array_equal(base[0][n][key], outs[n][key]):
                diffs.append(f"mode {n} {key} max|d|={np.max(np.abs(base[0][n][key] - outs[n][key])):.3e}")
    if not np.array_equal(base[1], fits):
        diffs.append(f"fits max|d|={np.max(np.abs(base[1] - fits)):.3e} first idx={int(np.argmax(base[1] != fits))}")
    print(f"rep {rep}:", "bitwise identical" if not diffs else "; ".join(diffs), flush=True)
