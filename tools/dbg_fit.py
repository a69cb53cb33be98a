import numpy as np, oracle as O
from paper_2112_10855_b200 import synth, cpqr
for dims,R in [((37,29,43),7),((38,30,44),7),((37,29,43),8),((30,40,50),5)]:
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=7 + R, eta=0.05)
    X=O.as_tensor(Xc)
    for v in ("QR","SVD"):
        s=cpqr.CPQR(dims,R,v); s.set_tensor(Xc); s.set_factors(init); f=s.sweep(1); lam,A=s.get_factors()
        ref=O.cp_als_qr(X,init,1,variant=v)
        print(dims,R,v,"gpu fit",f[0],"oracle",ref["fits"][0],"direct(gpu factors)",O.fit_direct(X,lam,A), "fac err", max(np.linalg.norm(a-b)/np.linalg.norm(b) for a,b in zip(A,ref["factors"])))
        s.close()
