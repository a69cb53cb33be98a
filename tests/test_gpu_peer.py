"""GPU tests of the peer push-reduce exchange on ONE B200.

CPQR_COMM_PEER replaces the NCCL all-reduce / all-gather of W_n by stores into every rank's receive
window issued by the Q0 apply's final sum (NE: a copy kernel), a flag per source rank, and a
rank-order combine.  What one GPU can check without kernels that wait on each other:
  * virtual ranks (CPQR_COMM_LOCAL_PEER): the same push / flag / combine kernels with p windows in
    one context, the ranks one after another on one stream -- bitwise equal to the sum-kernel
    exchange of CPQR_COMM_LOCAL (same rank order), which tests/test_gpu_slabs.py checks against the
    oracle; every window must have received identical bytes; oracle parity is re-checked here too;
  * one rank (world = 1, CPQR_COMM_PEER): the in-graph push to its own window;
  * one rank NCCL (world = 1, an NCCL id): ncclAllReduce / ncclAllGather captured in the sweep graph;
  * two processes on the one GPU: CUDA IPC window exchange, push, flags and combine, sequenced by
    host barriers (cpqr_debug_peer_put / _get) so that no kernel waits on another process.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_2112_10855_b200 import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


@pytest.fixture(scope="module")
def cp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_10855_b200 import cpqr
    return cpqr


CASES = [
    ((30, 38, 48), 5, "QR", False),
    ((70, 66, 32), 32, "QR", False),
    ((40, 36, 24), 6, "NE", False),
    ((24, 20, 18, 16), 8, "SVD", True),
    ((16, 14, 12, 16), 6, "PINV", False),
    ((9, 8, 7, 6, 8), 4, "QR", False),
]


def exchanges_per_sweep(N, direct=False):
    return N + (1 if direct else 0)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("dims,R,variant,tree", CASES)
def test_peer_push_virtual_ranks(cp, dims, R, variant, tree, world):
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=511 + R + len(dims))
    X = O.as_tensor(Xc)
    N = len(dims)
    ne = variant in ("NE", "PINV")
    a = cp.CPQR(dims, R, variant, tree=tree, world=world, comm="local")
    b = cp.CPQR(dims, R, variant, tree=tree, world=world, comm="local_peer")
    for s in (a, b):
        s.set_tensor(Xc)
        s.set_factors(init)
    st = b.debug_peer()
    assert st["epoch"] == 1 and st["min_flag"] == 1 and st["windows_differing"] == 0, st  # ||X||^2
    if not ne:
        for n in range(N):
            wa, wb = a.debug_mode(n)["W"], b.debug_mode(n)["W"]
            assert np.array_equal(wa, wb), n
    fa, fb = a.sweep(3), b.sweep(3)
    # the factors never see ||X||^2: bitwise; the fits do, and the two modes sum the p slab norms in
    # different orders (a block reduction vs rank order): equal to a few ulp
    assert np.max(np.abs(fa - fb)) <= 1e-13, (fa, fb)
    la, Aa = a.get_factors()
    lb, Ab = b.get_factors()
    assert np.array_equal(la, lb) and all(np.array_equal(x, y) for x, y in zip(Aa, Ab))
    st = b.debug_peer()
    want = 1 + (0 if ne else N) + 3 * exchanges_per_sweep(N)
    assert st["epoch"] == want and st["min_flag"] == want and st["windows_differing"] == 0, (st, want)
    assert b.flags == a.flags
    ref = O.cp_als_ne(X, init, 3, solve="pinv" if variant == "PINV" else "chol") if ne else \
        O.cp_als_qr(X, init, 3, variant=variant)
    assert np.max(np.abs(fb - np.array(ref["fits"]))) <= 1e-8
    a.close()
    b.close()


@pytest.mark.parametrize("world", [2, 8])
def test_peer_push_direct_fit_eager_and_graph(cp, world):
    dims, R = (20, 18, 16), 4
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=78, eta=0.0)
    X = O.as_tensor(Xc)
    out = []
    for graph in (True, False):
        s = cp.CPQR(dims, R, "QR", fit_mode="direct", world=world, comm="local_peer", use_graph=graph)
        s.set_tensor(Xc)
        s.set_factors(init)
        f = s.sweep(4)
        st = s.debug_peer()
        assert st["epoch"] == 1 + 4 * exchanges_per_sweep(3, direct=True) and st["windows_differing"] == 0, st
        out.append((f, s.get_factors()))
        s.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert all(np.array_equal(x, y) for x, y in zip(out[0][1][1], out[1][1][1]))
    ref = O.cp_als_qr(X, init, 4, fit_mode="direct")
    assert np.max(np.abs(out[0][0] - np.array(ref["fits"]))) <= 1e-8


@pytest.mark.parametrize("comm", ["peer", "nccl"])
@pytest.mark.parametrize("dims,R,variant,tree", CASES)
def test_one_rank_exchange_in_graph(cp, dims, R, variant, tree, comm):
    """world = 1 through the exchange path: the push to the rank's own window, or a one-rank NCCL
    communicator whose collectives are captured in the sweep graph -- bitwise the plain sweep."""
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=611 + R)
    # the plain context runs the serial schedules the exchange paths use (the switches are read at create)
    os.environ["CPQR_OVERLAP"] = "0"
    os.environ["CPQR_OVERLAP_NE"] = "0"
    try:
        a = cp.CPQR(dims, R, variant, tree=tree)
    finally:
        del os.environ["CPQR_OVERLAP"]
        del os.environ["CPQR_OVERLAP_NE"]
    kw = dict(nccl_id=cp.nccl_unique_id()) if comm == "nccl" else {}
    b = cp.CPQR(dims, R, variant, tree=tree, world=1, comm=comm, **kw)
    for s in (a, b):
        s.set_tensor(Xc)
        s.set_factors(init)
    fa, fb = a.sweep(3), b.sweep(3)
    assert np.array_equal(fa, fb), (fa, fb)
    la, Aa = a.get_factors()
    lb, Ab = b.get_factors()
    assert np.array_equal(la, lb) and all(np.array_equal(x, y) for x, y in zip(Aa, Ab))
    if comm == "peer":
        st = b.debug_peer()
        assert st["epoch"] == 1 + 3 * len(dims) and st["min_flag"] == st["epoch"], st
    a.close()
    b.close()


def test_peer_requires_connect_and_rejects_misuse(cp):
    dims, R = (12, 10, 8), 3
    conf, Xc, truth, init = synth.small_problem(dims, R, seed=5)
    s = cp.CPQR(dims, R, "QR", world=2, rank=0, comm="peer")
    assert len(s.peer_handle()) == 64
    with pytest.raises(cp.CpqrError) as ei:  # windows not exchanged yet
        s.set_tensor(np.ascontiguousarray(Xc[:4]))
    assert "ESTATE" in str(ei.value)
    s.close()
    t = cp.CPQR(dims, R, "QR", world=2, comm="local_peer")
    with pytest.raises(cp.CpqrError):
        t.peer_handle()
    t.close()


def test_peer_connect_rejects_a_handle_of_the_same_process(cp):
    """CUDA IPC cannot map a window of the calling process: connect fails cleanly (ECUDA), nothing
    hangs, and the contexts can still be destroyed."""
    dims, R = (12, 10, 8), 3
    s = cp.CPQR(dims, R, "QR", world=2, rank=0, comm="peer")
    t = cp.CPQR(dims, R, "QR", world=2, rank=1, comm="peer")
    with pytest.raises(cp.CpqrError):
        s.peer_connect([s.peer_handle(), t.peer_handle()])
    t.close()
    s.close()


def _ipc_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["CPQR_PEER_TIMEOUT_MS"] = "200"
    import torch
    import torch.distributed as dist
    from paper_2112_10855_b200 import cpqr
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dims, R = (40, 30, 8 * world), 4
        s = cpqr.CPQR(dims, R, "QR", world=world, rank=rank, comm="peer", device=0)
        s.connect_peers_torch()
        n = 40  # gathered: world x n doubles must fit W (max I x R = 160)
        res = {}
        for it, gather in enumerate([False, True, False]):
            src = np.arange(n, dtype=np.float64) * (rank + 1) + 1000.0 * it + 0.25 * rank
            s.debug_peer_put(src)
            dist.barrier()  # every rank has pushed before any rank combines: no kernel ever waits
            got = s.debug_peer_get(n, gather=gather)
            dist.barrier()
            parts = [np.arange(n, dtype=np.float64) * (r + 1) + 1000.0 * it + 0.25 * r for r in range(world)]
            if gather:
                want = np.concatenate(parts)
            else:
                want = parts[0].copy()
                for p in parts[1:]:
                    want = want + p
            res[it] = bool(np.array_equal(got, want))
        st = s.debug_peer()
        res["epoch"] = st["epoch"]
        res["min_flag"] = st["min_flag"]
        # a rank whose peers never push gives up after CPQR_PEER_TIMEOUT_MS and reports ENCCL
        res["timeout"] = None
        if rank == 0:
            s.debug_peer_put(np.ones(n))
            try:
                s.debug_peer_get(n)
                res["timeout"] = "no error"
            except cpqr.CpqrError as e:
                res["timeout"] = str(e)
        dist.barrier()
        s.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_windows_across_processes(cp, world):
    """CUDA IPC plumbing of CPQR_COMM_PEER between `world` processes sharing the one GPU: window
    handles all-gathered over gloo, every rank pushes into every window (k_peer_push), a host
    barrier, then every rank combines (k_peer_combine, flags already raised)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650 + world + (os.getpid() % 200)
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=240)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert out[r][0] and out[r][1] and out[r][2], (r, out[r])
        assert out[r]["epoch"] == 3 and out[r]["min_flag"] == 3, out[r]
    assert "ENCCL" in out[0]["timeout"], out[0]
