"""Per-rank Multi-TTM plans of the slab data parallelism: for C3, C4 and C5 at p =
1/2/4/8 slabs, every mode's steps as cpqr_debug_plan reports them (kernel, contracted modes,
output elements, flops), the stream pass's flops and the intermediates per rank, and their ratio
to p = 1 (1/p scaling, PAPER.md:387 applied to the local dimensions).  Runs on one GPU with
virtual ranks (CPQR_COMM_LOCAL): the plans are the ones the NCCL ranks build.

  python tools/plan_table.py [--configs 3 4 5]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2112_10855_b200 import cpqr, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4, 5])
    args = ap.parse_args()
    for cfg in args.configs:
        conf = synth.CONFIGS[cfg]
        dims, R, N = conf.dims, conf.R, conf.N
        X = torch.zeros(int(np.prod(dims)), dtype=torch.float64, device="cuda")
        init = [np.eye(d, R) for d in dims]
        print(f"\n### {conf.name} ({conf.variants[0]}), per rank; flops and elements in units of 1e6\n")
        print("| p | mode | steps: kernel [contracted modes] -> output elems | stream-pass flops | "
              "intermediate elems | total flops | vs p=1 (flops, interm.) |")
        print("|---|---|---|---|---|---|---|")
        base = {}
        for p in [1, 2, 4, 8]:
            s = cpqr.CPQR(dims, R, conf.variants[0], world=p, comm="local")
            s.set_tensor(X)
            s.set_factors(init)
            for n in range(N):
                pl = [st for st in s.debug_plan(n) if st["kind"] not in ("slice-reduce", "slice-fixup")]
                desc = "; ".join(f"{st['kind']} {[m + 1 for m in st['modes']]} -> {st['out_elems'] / 1e6:.3g}" for st in pl)
                fl0 = pl[0]["flops"]
                inter = sum(st["out_elems"] for st in pl[:-1])
                tot = sum(st["flops"] for st in pl)
                if p == 1:
                    base[n] = (tot, inter)
                rat = f"{base[n][0] / tot:.2f}x, " + (f"{base[n][1] / inter:.2f}x" if inter else "-")
                print(f"| {p} | {n + 1} | {desc} | {fl0 / 1e6:.4g} | {inter / 1e6:.4g} | {tot / 1e6:.4g} | {rat} |")
            s.close()
        del X
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
