import sys, numpy as np
sys.path.insert(0, '.')
from paper_2112_10855_b200 import cpqr, synth
dims, R, variant = eval(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
conf, Xc, truth, init = synth.small_problem(dims, R, seed=91, eta=0.05)
s = cpqr.CPQR(dims, R, variant, use_graph=False)
s.set_tensor(Xc); s.set_factors(init)
print(s.sweep(2))
s.close()
