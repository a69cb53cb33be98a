#!/usr/bin/env python
"""Benchmark: CP-ALS-QR sweeps/s and Multi-TTM HBM GB/s (fp64) on 1..8 B200 (BASELINE.json metric).

A "step" is one CP-ALS-QR sweep (Alg. 2 lines 5-13): all N mode updates over
the whole (slab of the) tensor, i.e. every row of SURVEY.md §8(a).  Default workload: C5
(1000^3, R = 32, QR variant, 8 GB fp64), sharded in 1000/p slabs on mode 3; --config selects
another BASELINE config.  Inputs are the seeded synthetic tensors of synth.py (DESIGN.md
§Inputs); X (8 GB) is far larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--variant QR] [--tree]
  python bench.py --impl reference ...     # the CPU oracle (oracle/) on the host cores

The headline `value` times the paper's schedule (one Multi-TTM pass over X per mode, Alg. 2
line 8).  The same line carries "dimension_tree": the dimension-tree Multi-TTM (PAPER.md:472-478,
SURVEY.md §8(f) NEXT-1; two passes over X per sweep, identical mode updates up to rounding) timed
the same way on the same resident tensor.  --tree swaps the two.

Multi-GPU: one process per GPU under torch.distributed.run (`--gpus N` without WORLD_SIZE in
the environment re-launches itself that way); the NCCL id (or, with --comm peer, the CUDA IPC
handles of the peer windows) travels over a gloo group; timing =
CUDA events on the stream the library runs on, max over ranks.  The same slab path on one GPU
(virtual ranks, parity tests and per-rank projections): tests/test_gpu_slabs.py,
tools/slab_projection.py.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2112_10855_b200 import synth  # noqa: E402

P64_DMMA_TFLOPS = 37.08        # measured, profiles/ubench_r01.log (mma.sync m8n8k4 f64, 148 SMs)
HBM_READ_GBS = 7243.3          # measured read-only stream, profiles/ubench_r01.log


def peaks():
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(m["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    def __init__(self, index=0, period=0.005):
        self.index, self.period, self.samples, self.stop = index, period, [], False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop = True
        if self.nv:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        nv = self.nv
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        reasons = sorted({n for _, r in self.samples for n, bit in names.items() if r & bit})
        return {"sm_mhz": float(np.median([s for s, _ in self.samples])), "sm_max_mhz": float(self.max_sm),
                "reasons": reasons, "samples": len(self.samples), "source": "NVML, 5 ms"}


METRIC = "CP-ALS-QR sweeps/s & Multi-TTM HBM GB/s (fp64)"


def bench_config(conf, variant, world, tree):
    """The `config` object of both arms (identical keys and values)."""
    numel_local = int(np.prod(conf.dims)) // world
    return {"workload": conf.name, "variant": variant, "dims": list(conf.dims), "R": conf.R,
            "global_batch": 1, "parallelism": f"slab-dp{world} on mode {conf.N}",
            "multittm": "dimension tree (2 passes over X per sweep)" if tree else
                        "per mode (one pass over X per mode, Alg. 2 line 8)",
            "l2": ("inputs larger than L2 (X = %.2f GB/GPU vs 126 MB L2), no flush needed" % (8.0 * numel_local / 1e9))
                  if 8.0 * numel_local > 126e6 else
                  ("X = %.2f MB/GPU fits in L2: a launch-latency-bound config, timed warm" % (8.0 * numel_local / 1e6))}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def load_input(conf, rank, world):
    """Full X on the host (cached .npy, memory-mapped) and this rank's contiguous slab."""
    cdir = synth._cache_dir()
    if world > 1:
        import torch.distributed as dist
        if rank == 0:
            synth.make_problem(conf.cfg)  # generate + cache once
        dist.barrier()
    conf, Xc, truth, init = synth.make_problem(conf.cfg)
    per = conf.dims[-1] // world
    slab = Xc[rank * per:(rank + 1) * per]
    return conf, Xc, slab, truth, init, cdir


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(conf, Xc, init, variant, sweeps=2):
    """The oracle as it stands, on this host's cores, on a bounded sample: one untimed warm-up
    sweep (PAPER.md:520 excludes the first iteration), then `sweeps` timed full sweeps."""
    import oracle as O
    X = O.as_tensor(Xc)
    cores = len(os.sched_getaffinity(0))
    run = (lambda A0, k: O.cp_als_ne(X, A0, k)) if variant == "NE" else \
        (lambda A0, k: O.cp_als_qr(X, A0, k, variant=variant, tau=conf.svd_tau))
    A1 = run(init, 1)["factors"]
    t0 = time.perf_counter()
    run(A1, sweeps)
    dt = time.perf_counter() - t0
    return {"value": sweeps / dt, "unit": "sweeps/s", "cores": cores, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"{sweeps} full CP-ALS-{variant} sweeps of {conf.name} after 1 untimed sweep from the "
                      f"shared init, numpy/OpenBLAS fp64, wall clock"}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    conf = synth.CONFIGS[args.config]
    variant = args.variant or conf.variants[0]
    conf, Xc, truth, init = synth.make_problem(conf.cfg)
    import oracle as O
    X = O.as_tensor(Xc)
    cores = len(os.sched_getaffinity(0))
    run = (lambda A0, s: O.cp_als_ne(X, A0, s)) if variant == "NE" else \
        (lambda A0, s: O.cp_als_qr(X, A0, s, variant=variant, tau=conf.svd_tau))
    state = run(init, max(1, args.warmup))   # warm-up sweeps (untimed)
    A0 = state["factors"]
    t0 = time.perf_counter()
    run(A0, args.steps)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "sweeps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (synth.py seeded recipe of BASELINE.json config; no dataset)",
            "config": bench_config(conf, variant, world, bool(args.tree and variant != "NE" and conf.N >= 3)),
            "cpu_baseline": {"value": v, "unit": "sweeps/s", "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"{args.steps} full sweeps of {conf.name} after {args.warmup} warm-up"},
            "e2e": {"value": v, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def relaunch(n):
    """`--gpus N` outside torch.distributed.run: re-launch this command as N ranks, one per GPU."""
    import socket
    import torch
    if args_impl_is_gpu() and torch.cuda.device_count() < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {torch.cuda.device_count()} "
              f"(the one-GPU slab path is tools/slab_projection.py)", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def args_impl_is_gpu():
    return "reference" not in sys.argv[1:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--variant", default=None)
    ap.add_argument("--impl", default="cpqr", choices=["cpqr", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--tree", action="store_true", help="headline = dimension-tree Multi-TTM")
    ap.add_argument("--comm", default="auto", choices=["auto", "nccl", "peer"],
                    help="exchange of W_n across ranks: NCCL collectives or the fused peer push-reduce "
                         "(CPQR_COMM_PEER); auto = NCCL at world > 1, none at world 1 (nccl / peer at world 1 "
                         "run the in-graph exchange on one rank)")
    args = ap.parse_args()
    # NCCL's version banner (NCCL_DEBUG=VERSION) goes to stdout by default: keep stdout to the JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    from paper_2112_10855_b200 import cpqr
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")

    comm = args.comm if args.comm != "auto" else "nccl"

    def new_nccl_id():
        """A fresh ncclUniqueId for every context (one NCCL communicator each), broadcast from
        rank 0 over the gloo group; all ranks create contexts in the same order."""
        if comm != "nccl" or (world == 1 and args.comm == "auto"):
            return None
        if world == 1:
            return cpqr.nccl_unique_id()
        import torch.distributed as dist
        obj = [cpqr.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def new_ctx(**kw):
        """One context of this rank; CPQR_COMM_PEER ranks exchange their window handles (gloo)."""
        s = cpqr.CPQR(conf.dims, conf.R, variant, svd_tau=conf.svd_tau, device=local, stream=stream.cuda_stream,
                      rank=rank, world=world, nccl_id=new_nccl_id(), comm=comm, **kw)
        if comm == "peer" and world > 1:
            s.connect_peers_torch()
        return s
    conf = synth.CONFIGS[args.config]
    variant = args.variant or conf.variants[0]
    conf, Xc, slab, truth, init, _ = load_input(conf, rank, world)

    stream = torch.cuda.current_stream()
    tree_ok = variant != "NE" and conf.N >= 3
    tree = bool(args.tree and tree_ok)
    Xd = torch.from_numpy(np.ascontiguousarray(slab)).to(f"cuda:{local}")

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def timed_arm(use_tree, sample_clocks):
        """W warm-up sweeps (CUDA-graph capture), then exactly K sweeps between CUDA events on
        the library's stream, barrier + synchronize on both sides, max over ranks."""
        s = new_ctx(tree=use_tree)
        s.set_tensor(Xd)                     # device-resident input (borrowed)
        s.set_factors(init)
        s.sweep(args.warmup)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = s.profile(reset=False)["launches_total"]
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            e0.record(stream)
            s.sweep(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        launches = s.profile(reset=False)["launches_total"] - launches0
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        s.close()
        return ms, launches, (clk.summary() if sample_clocks else None)

    ms, launches, clocks = timed_arm(tree, True)
    sweeps_s = args.steps / (ms / 1e3)
    other = None
    if tree_ok:
        ms2, l2, _ = timed_arm(not tree, False)
        other = {"value": args.steps / (ms2 / 1e3), "unit": "sweeps/s", "ms_per_step": ms2 / args.steps,
                 "gpu_launches": int(l2)}

    # phase profile (separate short run; events around each phase on the library stream)
    sp = new_ctx(profile=True, use_graph=False, tree=tree)
    prof = None
    if sp is not None:
        sp.set_tensor(Xd)
        sp.set_factors(init)
        sp.sweep(1)
        sp.profile(reset=True)
        nprof = 2
        sp.sweep(nprof)
        prof = sp.profile(reset=True)
        prof["sweeps"] = nprof
        sp.close()

    # end-to-end through the public API with HOST buffers: H2D of X (pinned), set_factors,
    # the config's sweep count, D2H of factors + fits -- per step = one solve
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(np.ascontiguousarray(slab)).pin_memory()
        se = new_ctx(tree=tree)
        se.set_tensor(Xh)
        se.set_factors(init)
        se.sweep(1)
        barrier()
        torch.cuda.synchronize()
        nrep = 2
        t0 = time.perf_counter()
        f1 = f2 = None
        for _ in range(nrep):
            se.set_tensor(Xh)
            se.set_factors(init)
            fits = se.sweep(conf.sweeps)
            lam, A = se.get_factors()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        barrier()
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([dt], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = Xh.numel() * 8 + sum(int(np.prod(a.shape)) * 8 for a in init)
        d2h = sum(int(np.prod(a.shape)) * 8 for a in A) + conf.R * 8 + conf.sweeps * 8
        e2e = {"value": nrep * conf.sweeps / dt, "unit": "sweeps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "step": f"one solve through the C-ABI from host buffers: H2D X slab (pinned) + set_factors + "
                       f"{conf.sweeps} sweeps + D2H factors/fits; wall clock, max over ranks"}
        se.close()
    if rank != 0:
        return 0
    hbm_peak, hbm_src = peaks()
    numel_local = int(np.prod(conf.dims)) // world
    # X read once per mode; twice per sweep with the dimension tree
    mt_bytes_sweep = (2 if tree else conf.N) * 8.0 * numel_local
    line = {
        "metric": METRIC,
        "value": sweeps_s * 1.0, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth.py seeded recipe of BASELINE.json config; no dataset)",
        "config": bench_config(conf, variant, world, tree),
        "exchange": comm if (world > 1 or args.comm != "auto") else "none (one GPU)",
        "gpu_launches": int(launches),
    }
    if prof:
        nsw = prof["sweeps"]
        n_launch0 = (2 if tree else conf.N) * nsw
        t0_avg_ms = prof["ms"][0] / n_launch0
        bytes_launch = prof["bytes0"] / (2 if tree else conf.N)
        flops_launch = prof["flops0"] / (2 if tree else conf.N)
        gbs = bytes_launch / (t0_avg_ms / 1e3) / 1e9
        tfl = flops_launch / (t0_avg_ms / 1e3) / 1e12
        t_hbm, t_fp = bytes_launch / (hbm_peak * 1e9), flops_launch / (P64_DMMA_TFLOPS * 1e12)
        if t_fp > t_hbm:
            roof = {"bound": "tensor", "achieved": tfl, "peak": P64_DMMA_TFLOPS, "unit": "TFLOP/s",
                    "frac": tfl / P64_DMMA_TFLOPS, "peak_source": "measured FP64 DMMA (profiles/ubench_r01.log)"}
        else:
            roof = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                    "peak_source": hbm_src}
        roof["kernel"] = ("Multi-TTM stream-X pass (k_strided_tma / k_strided2_tma / k_slice_tma / k_slice_small_tma), "
                          "avg over %d passes" % n_launch0)
        roof["traffic"] = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            roof["traffic"] = json.load(open(tfile)).get(conf.name)
        roof["hbm_gbs"] = gbs
        roof["hbm_frac"] = gbs / hbm_peak
        roof["fp64_tflops"] = tfl
        roof["roofline_frac"] = max(t_hbm, t_fp) / (t0_avg_ms / 1e3)
        line["roofline"] = roof
        line["multi_ttm_gbs"] = mt_bytes_sweep / ((prof["ms"][0] + prof["ms"][1]) / nsw / 1e3) / 1e9
        line["phase_ms_per_sweep"] = {k: v / nsw for k, v in zip(
            ["stream_pass", "rest_ttm", "factor_qr_tail", "q0_compute", "q0_apply", "other", "exchange"],
            prof["ms"])}
    line["clocks"] = clocks
    if other:
        line["per_mode" if tree else "dimension_tree"] = dict(other, note=(
            "the other Multi-TTM schedule, same config/inputs/timing; dimension tree = PAPER.md:472-478, "
            "SURVEY.md 8(f) NEXT-1, mode updates identical up to rounding (tests/test_gpu_parity.py)"))
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(conf, Xc, init, variant)
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
