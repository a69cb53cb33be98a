import numpy as np, sys
sys.path.insert(0, '.')
import oracle as O
from paper_2112_10855_b200 import cpqr, synth
def run(dims, R, var, X=None, sweeps=3, seed=5):
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=seed, eta=0.01)
    if X is not None: Xc = X
    s = cpqr.CPQR(dims, R, var)
    s.set_tensor(Xc); s.set_factors(init)
    try:
        f = s.sweep(sweeps); lam, A = s.get_factors(); st = "ok"
    except Exception as e:
        f, lam, A, st = None, None, None, str(e)[:80]
    fl = s.flags
    s.close()
    ref = O.cp_als_qr(O.as_tensor(Xc), init, sweeps, variant=var) if var != "NE" else O.cp_als_ne(O.as_tensor(Xc), init, sweeps)
    print(dims, R, var, st, "flags", fl, "gpu fits", None if f is None else np.round(f, 12), "ref fits", np.round(ref["fits"], 12), "lam", None if lam is None else lam[:3], "reflam", ref["lam"][:3])
import warnings; warnings.simplefilter("ignore")
run((30, 40, 50), 1, "QR"); run((12, 10, 9, 11), 1, "QR"); run((8, 8, 8), 8, "QR"); run((5, 5, 5, 5), 5, "SVD")
run((3,)*8, 2, "QR"); run((40, 3), 3, "QR")
run((6, 5, 4), 2, "QR", X=np.zeros((4, 5, 6))); run((6, 5, 4), 2, "SVD", X=np.zeros((4, 5, 6)))
