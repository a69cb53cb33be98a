#!/usr/bin/env python
"""Per-rank timing projection of the slab data parallelism on ONE B200.

A CPQR_COMM_LOCAL context with world = p runs the p slabs of p virtual ranks in turn on one GPU
(the multi-GPU code path minus the NCCL call).  With opt.profile the library records device time
per phase (cpqr_get_profile): the slab-parallel phases (stream-X pass, remaining TTMs, Q0 apply)
summed over the p slabs, and the replicated phases (V_n QR, the fused factor-QR tail, other) once.
The projected time of one rank on its own GPU is

    T_rank(p) = (stream + rest + q0_apply) / p + tail + other + max(0, vn_qr - stream / p) + comm(p)

(the one-CTA Householder V_n QR hides behind the stream pass on the side stream as on one GPU,
as far as the pass is long enough; the multi-CTA CholeskyQR2 V_n QR (high rank, or CPQR_VN_QR=cq)
cannot co-run with the stream grid and is counted in full; the virtual ranks' combine kernel is
excluded; comm(p) is NOT measured here -- no multi-GPU box -- and is an
assumed per-mode NCCL latency).  Also printed: the measured sweep time of the LOCAL context (all slabs in sequence, CUDA
graph), which is p times the slab work plus the tails.  A projection, not a measurement.

  python tools/slab_projection.py [--configs 3 4 5] [--ps 1 2 4 8] [--comm-us 15]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2112_10855_b200 import cpqr, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4, 5])
    ap.add_argument("--ps", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--comm-us", type=float, default=15.0, help="assumed NCCL latency per mode (not measured)")
    ap.add_argument("--sweeps", type=int, default=3)
    ap.add_argument("--tree", action="store_true")
    ap.add_argument("--comm", default="local", choices=["local", "local_peer"],
                    help="virtual ranks' exchange: the sum kernel, or the fused peer push-reduce (push fused "
                         "into the Q0 apply + combine kernel; its cost then shows in q0_apply and local_combine)")
    args = ap.parse_args()
    rows = []
    for cfg in args.configs:
        conf, Xc, truth, init = synth.make_problem(cfg)
        variant = conf.variants[0]
        Xd = torch.from_numpy(np.ascontiguousarray(Xc)).cuda()
        del Xc
        base = None
        for p in args.ps:
            kw = dict(svd_tau=conf.svd_tau, tree=args.tree, world=p, comm=args.comm if p > 1 else "local")
            s = cpqr.CPQR(conf.dims, conf.R, variant, profile=True, use_graph=False, **kw)
            s.set_tensor(Xd)
            s.set_factors(init)
            s.sweep(1)
            s.profile(reset=True)
            s.sweep(args.sweeps)
            pr = s.profile(reset=True)
            s.close()
            ms = [v / args.sweeps for v in pr["ms"]]
            stream, rest, fqr, vn, q0a, other, exch = ms
            slab = (stream + rest + q0a) / p
            # the one-CTA Householder V_n QR (p = 1, low rank) runs on the SM the stream grids leave
            # free and hides behind the pass; the CholeskyQR2 V_n QR (p > 1, or R^{N-1} R >= 2e5) is
            # a multi-CTA launch that cannot co-run with a 147-CTA stream grid: counted in full
            J = conf.R ** (conf.N - 1)
            vq = os.environ.get("CPQR_VN_QR")  # "tree": one CTA like K2 (hides behind the pass)
            cq = vq == "cq" or (vq != "tree" and J * conf.R >= 200000)
            vn_exposed = vn if cq else max(0.0, vn - stream / p)
            t_rank = slab + fqr + other + vn_exposed + conf.N * args.comm_us / 1e3 * (p > 1)
            # the LOCAL context's own sweep time (graph, all p slabs in sequence)
            g = cpqr.CPQR(conf.dims, conf.R, variant, **kw)
            g.set_tensor(Xd)
            g.set_factors(init)
            g.sweep(2)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            g.sweep(args.sweeps)
            e1.record()
            torch.cuda.synchronize()
            t_local = e0.elapsed_time(e1) / args.sweeps
            g.close()
            if base is None:
                base = t_rank
            row = dict(config=conf.name, variant=variant, tree=args.tree, p=p, comm=args.comm,
                       per_sweep_ms=dict(stream_pass=stream, rest_ttm=rest, q0_apply=q0a, vn_qr=vn,
                                         factor_qr_tail=fqr, other=other, local_combine=exch),
                       slab_work_per_rank_ms=slab, projected_rank_ms=t_rank,
                       projected_sweeps_s=1e3 / t_rank, projected_aggregate_speedup=base / t_rank,
                       projected_efficiency=base / t_rank / p, local_context_sweep_ms=t_local,
                       comm_us_per_mode_assumed=args.comm_us if p > 1 else 0.0)
            rows.append(row)
            print(json.dumps(row), flush=True)
        del Xd
        torch.cuda.empty_cache()
    print("\n| config | p | stream/p | rest/p | Q0 apply/p | tail | other | V_n QR | projected ms | sweeps/s | eff |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        m = r["per_sweep_ms"]
        p = r["p"]
        print(f"| {r['config']} {r['variant']} | {p} | {m['stream_pass'] / p:.3f} | {m['rest_ttm'] / p:.3f} | "
              f"{m['q0_apply'] / p:.3f} | {m['factor_qr_tail']:.3f} | {m['other']:.3f} | {m['vn_qr']:.3f} | "
              f"{r['projected_rank_ms']:.3f} | {r['projected_sweeps_s']:.0f} | {r['projected_efficiency']:.2f} |")


if __name__ == "__main__":
    main()
