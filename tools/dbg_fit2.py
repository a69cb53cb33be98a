import numpy as np, oracle as O
from paper_2112_10855_b200 import synth, cpqr
dims,R=(30,40,50),5
conf, Xc, truth, init = synth.small_problem(dims, R, seed=7 + R, eta=0.05)
X=O.as_tensor(Xc)
for v in ("QR","SVD"):
    s=cpqr.CPQR(dims,R,v,use_graph=False); s.set_tensor(Xc); s.set_factors(init); f=s.sweep(1)
    import ctypes; ctypes.CDLL(None)
    ref=O.cp_als_qr(X,init,1,variant=v,debug_sweep1=True); d=ref["debug"][-1]
    W=d["W"]; Ah=d["Ahat"]; R0=d["R0"]
    print(v, "oracle inner", np.sum(W*(Ah@R0.T)), "|W|^2", np.sum(W*W), "nx2", ref["nX2"])
