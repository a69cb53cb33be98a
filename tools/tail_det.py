"""Determinism of the tail pieces on C4-like inputs: debug_svd_solve (Jacobi pinv + solve) and
debug_qr (CholeskyQR2 / Householder factor QR), repeated in-process; hashes printed for cross-process."""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr, synth
h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
conf, Xc, truth, init = synth.make_problem(4)
s = cpqr.CPQR(conf.dims, conf.R, "SVD", svd_tau=conf.svd_tau)
s.set_tensor(torch.from_numpy(np.ascontiguousarray(Xc)).cuda())
s.set_factors(init)
d = s.debug_mode(0)
R0, W = d["R0"], d["W"]
svd = set(); qr = set()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    out, nt = s.debug_svd_solve(R0, W, conf.svd_tau)
    svd.add(h(out))
    Q, Rf = s.debug_qr(init[1])
    qr.add(h(Q) + h(Rf))
print("R0", h(R0), "W", h(W), "svd_solve", sorted(svd), "qr", sorted(qr))
