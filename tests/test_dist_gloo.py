"""Multi-process (world size 2, gloo, CPU) tests of the slab data-parallel decomposition that
libcpqr implements with NCCL: X is split into contiguous slabs of the last mode;
for modes n < N each rank's partial W_p = Y_p Q0 (from its slab and the matching rows of Q_N)
all-reduces to the full W_n; for mode N the ranks own disjoint rows of W_N, all-gathered in rank
order.  Uses the oracle for the arithmetic, torch.distributed (gloo) for the exchange.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, dims, R, results):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2112_10855_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        conf, Xc, truth, init = synth.small_problem(dims, R, seed=41, eta=0.05)
        N = len(dims)
        per = dims[-1] // world
        b, e = rank * per, (rank + 1) * per
        Xfull = O.as_tensor(Xc)
        Xslab = O.as_tensor(np.ascontiguousarray(Xc[b:e]))       # contiguous block of the buffer
        assert np.array_equal(Xslab, Xfull[..., b:e])
        Qs, Rs = [None] * N, [None] * N
        for k in range(N):
            Qs[k], Rs[k] = O.qr_pos(init[k])
        ok = True
        for n in range(N):
            Q0, R0 = O.structured_qr(Rs, n)
            Us = {k: Qs[k].T for k in range(N) if k != n}
            if n < N - 1:
                Us[N - 1] = Qs[N - 1][b:e].T                        # the slab's rows of Q_N
            Yp = O.multi_ttm(Xslab, Us)
            Wp = O.apply_q0(Yp, n, Q0)
            if n < N - 1:
                t = torch.from_numpy(np.ascontiguousarray(Wp))
                dist.all_reduce(t)                                   # NCCL all-reduce in libcpqr
                W = t.numpy()
            else:
                parts = [torch.zeros(per, R, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(Wp)))
                W = torch.cat(parts).numpy()                          # rows in rank order
            Wref = O.apply_q0(O.multi_ttm(Xfull, {k: Qs[k].T for k in range(N) if k != n}), n, Q0)
            err = np.linalg.norm(W - Wref) / np.linalg.norm(Wref)
            ok = ok and err <= 1e-13
            # replicated tail on identical inputs gives identical factors on every rank
            A, lam = O.normalize(O.solve_qr(R0, W))
            g = torch.from_numpy(A.copy())
            gl = [torch.zeros_like(g) for _ in range(world)]
            dist.all_gather(gl, g)
            ok = ok and all(torch.equal(gl[0], x) for x in gl)
        # ||X||^2 all-reduced from the slabs
        t = torch.tensor([float(np.sum(Xslab ** 2))], dtype=torch.float64)
        dist.all_reduce(t)
        ok = ok and abs(t.item() - float(np.sum(Xfull ** 2))) <= 1e-12 * t.item()
        # NCCL id bootstrap: 128 bytes broadcast from rank 0 (bench.py uses the same call)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ok = ok and obj[0] == bytes(range(128))
        results[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,R", [((12, 10, 8), 4), ((6, 5, 7, 8), 3)])
def test_slab_decomposition_world2(dims, R):
    world = 2
    port = 29500 + (sum(dims) * 7 + R) % 1000
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, dims, R, results), nprocs=world, join=True)
    assert results.get(0) and results.get(1), dict(results)


def test_slab_bounds_match_library_convention():
    # cpqr_create: per = I_N // world, rank q owns [q per, (q+1) per); I_N % world == 0 required
    from paper_2112_10855_b200 import synth  # noqa: F401
    for IN, world in [(1000, 8), (128, 4), (48, 2)]:
        per = IN // world
        spans = [(q * per, (q + 1) * per) for q in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == IN
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _tree_worker(rank, world, port, dims, R, results):
    """Dimension-tree Multi-TTM over slabs: T_L = X_slab x_{k>=h} Q_k^T (Q_N's slab rows) is a
    rank-partial of the left-half intermediate, so W_n (n < h) all-reduces as in the per-mode
    schedule; T_R = X_slab x_{k<h} Q_k^T keeps the slab's i_N, so modes h..N-2 all-reduce and mode
    N all-gathers rows.  Checked against the full-tensor per-mode W of every mode."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2112_10855_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        conf, Xc, truth, init = synth.small_problem(dims, R, seed=43, eta=0.05)
        N = len(dims)
        h = (N + 1) // 2
        per = dims[-1] // world
        b, e = rank * per, (rank + 1) * per
        Xfull = O.as_tensor(Xc)
        Xslab = O.as_tensor(np.ascontiguousarray(Xc[b:e]))
        Qs = [O.qr_pos(a)[0] for a in init]
        Rs = [O.qr_pos(a)[1] for a in init]

        def slabQ(k):
            return Qs[k][b:e] if k == N - 1 else Qs[k]
        TL = O.multi_ttm(Xslab, {k: slabQ(k).T for k in range(h, N)})
        TR = O.multi_ttm(Xslab, {k: Qs[k].T for k in range(h)})
        ok = True
        for n in range(N):
            Q0, R0 = O.structured_qr(Rs, n)
            if n < h:
                Yp = O.multi_ttm(TL, {k: Qs[k].T for k in range(h) if k != n})
            else:
                Yp = O.multi_ttm(TR, {k: slabQ(k).T for k in range(h, N) if k != n})
            Wp = O.apply_q0(Yp, n, Q0)
            if n < N - 1:
                t = torch.from_numpy(np.ascontiguousarray(Wp))
                dist.all_reduce(t)
                W = t.numpy()
            else:
                parts = [torch.zeros(per, R, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(Wp)))
                W = torch.cat(parts).numpy()
            Wref = O.apply_q0(O.multi_ttm(Xfull, {k: Qs[k].T for k in range(N) if k != n}), n, Q0)
            ok = ok and np.linalg.norm(W - Wref) <= 1e-13 * np.linalg.norm(Wref)
        results[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,R", [((12, 10, 8), 4), ((6, 5, 7, 8), 3), ((5, 4, 6, 3, 4), 2)])
def test_dimension_tree_slab_decomposition_world2(dims, R):
    world = 2
    port = 30500 + (sum(dims) * 11 + R) % 1000
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_tree_worker, args=(world, port, dims, R, results), nprocs=world, join=True)
    assert results.get(0) and results.get(1), dict(results)


def test_bench_reference_arm_under_torchrun_world2():
    """bench.py's launch contract on CPU: under torch.distributed.run with 2 ranks the reference arm
    (the oracle) runs on rank 0 alone and prints exactly ONE JSON line; the other rank exits 0."""
    import json
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", f"--master-port={port}", os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
           "--config", "1", "--steps", "2", "--warmup", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2 and d["unit"] == "sweeps/s"
    assert d["config"]["workload"].startswith("C1") and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


@pytest.mark.parametrize("p", [2, 3, 8])
def test_peer_window_protocol_model(p):
    """Host-side model of the peer push-reduce protocol (small_kernels.cuh): p ranks,
    each with a receive window of [2 parities][p slots] and p arrival flags, run exchanges
    e = 1..E as push (store into slot `rank`, parity (e-1) & 1, of EVERY window -- one micro-step per
    destination, in any order -- then, after all of them, raise flag[rank] = e on every window, again
    one micro-step per destination) and combine (wait for all p flags >= e, then read the p slots of
    that parity).  Under random interleavings of the ranks' micro-steps, every combine must read
    exactly the values pushed for ITS exchange (no slot overwritten early, none stale) and no rank
    may deadlock -- the claim behind "flags only grow, two parities, no reset, no second barrier"."""
    import random
    E = 7
    for seed in range(200):
        rng = random.Random(1000 * p + seed)
        slot = [[[None] * p for _ in range(2)] for _ in range(p)]   # slot[dst][parity][src]
        flag = [[0] * p for _ in range(p)]                          # flag[dst][src]
        # per-rank program counter: (exchange e, phase, pending micro-steps)
        state = [dict(e=1, phase="data", todo=list(range(p))) for _ in range(p)]
        done = [False] * p
        steps = 0
        while not all(done):
            steps += 1
            assert steps < 100000, "no progress"
            ready = []
            for r in range(p):
                if done[r]:
                    continue
                st = state[r]
                if st["phase"] in ("data", "flag") or all(flag[r][q] >= st["e"] for q in range(p)):
                    ready.append(r)
            assert ready, ("deadlock", seed, [(s["e"], s["phase"]) for s in state])
            r = rng.choice(ready)
            st = state[r]
            e = st["e"]
            if st["phase"] == "data":
                d = st["todo"].pop(rng.randrange(len(st["todo"])))
                slot[d][(e - 1) & 1][r] = (r, e)
                if not st["todo"]:
                    st["phase"], st["todo"] = "flag", list(range(p))
            elif st["phase"] == "flag":
                d = st["todo"].pop(rng.randrange(len(st["todo"])))
                assert flag[d][r] == e - 1   # flags only grow, one exchange at a time
                flag[d][r] = e
                if not st["todo"]:
                    st["phase"] = "combine"
            else:  # combine: all p flags have reached e
                got = [slot[r][(e - 1) & 1][q] for q in range(p)]
                assert got == [(q, e) for q in range(p)], (seed, r, e, got)
                if e == E:
                    done[r] = True
                else:
                    state[r] = dict(e=e + 1, phase="data", todo=list(range(p)))
