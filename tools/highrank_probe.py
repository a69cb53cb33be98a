"""Phase profile of one CP-ALS-QR sweep on an ad-hoc high-rank problem (R^(N-1) large)."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10855_b200 import cpqr
dims = eval(sys.argv[1]); R = int(sys.argv[2]); var = sys.argv[3] if len(sys.argv) > 3 else "QR"
torch.manual_seed(0)
X = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda")
rng = np.random.default_rng(0)
init = [rng.standard_normal((d, R)) for d in dims]
for graph in (False, True):
    s = cpqr.CPQR(dims, R, var, profile=not graph, use_graph=graph)
    s.set_tensor(X); s.set_factors(init); s.sweep(1)
    s.profile(reset=True); torch.cuda.synchronize(); t0 = time.perf_counter()
    s.sweep(2); torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 2
    p = s.profile()
    names = ["stream_pass", "rest_ttm", "factor_qr", "q0_compute", "q0_apply", "other"]
    print(dims, R, var, "graph" if graph else "eager", "ms/sweep %.3f" % (1e3 * dt),
          {n: round(v / 2, 3) for n, v in zip(names, p["ms"])} if not graph else "")
    s.close()
