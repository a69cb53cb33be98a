"""Thin ctypes binding of libcpqr (include/cpqr.h).  Argument marshalling only: every step of
the CP-ALS(-QR) path runs in the library's sm_100a kernels.  There is no CPU fallback: if
libcpqr.so is missing or fails to load, importing this module raises.

Tensors follow the library convention: X is the column-major I_1 x ... x I_N buffer, i.e. a
C-contiguous numpy array / torch tensor of shape (I_N, ..., I_1).  Factors are (I_k, R) arrays,
passed column-major (numpy arrays are converted with np.asfortranarray).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPQR_LIB", os.path.join(_HERE, "libcpqr.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libcpqr.so not built ({LIB_PATH}); run `python -m paper_2112_10855_b200.build`")
_lib = C.CDLL(LIB_PATH)

NE, QR, SVD, PINV = 0, 1, 2, 3
VARIANTS = {"NE": NE, "QR": QR, "SVD": SVD, "PINV": PINV}
FIT_FAST, FIT_DIRECT = 0, 1
MEM_HOST, MEM_DEVICE_COPY, MEM_DEVICE_BORROW = 0, 1, 2
COMM_NCCL, COMM_LOCAL, COMM_PEER, COMM_LOCAL_PEER = 0, 1, 2, 3
FLAG_ILLCOND_R0, FLAG_NE_CHOL_FALLBACK, FLAG_SVD_TRUNCATED, FLAG_NE_ILLCOND = 1, 2, 4, 8
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "ESTATE", 6: "EDIVERGED"}

EXPORTS = [
    "cpqr_default_options", "cpqr_create", "cpqr_set_tensor", "cpqr_set_factors", "cpqr_init_factors",
    "cpqr_set_ktensor", "cpqr_batched_qr", "cpqr_batched", "cpqr_sweep", "cpqr_get_factors", "cpqr_get_fit", "cpqr_get_flags", "cpqr_get_profile", "cpqr_get_timings",
    "cpqr_launches_per_sweep", "cpqr_debug_mode", "cpqr_debug_plan", "cpqr_debug_qr", "cpqr_debug_svd_solve",
    "cpqr_destroy", "cpqr_status_string", "cpqr_last_error", "cpqr_nccl_unique_id", "cpqr_version",
    "cpqr_peer_handle", "cpqr_peer_connect", "cpqr_debug_peer", "cpqr_debug_peer_put", "cpqr_debug_peer_get",
]


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("svd_tau", C.c_double), ("fit_mode", C.c_int32),
                ("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_id", C.c_uint8 * 128), ("use_graph", C.c_int32), ("profile", C.c_int32),
                ("mttm_tree", C.c_int32), ("comm", C.c_int32)]


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 7), ("launches", C.c_int64 * 7), ("bytes0", C.c_double),
                ("flops0", C.c_double), ("launches_total", C.c_int64)]


_P = C.c_void_p
_DP = C.POINTER(C.c_double)
_sig = {
    "cpqr_default_options": (None, [C.POINTER(Options)]),
    "cpqr_create": (C.c_int32, [C.c_int, C.POINTER(C.c_int64), C.c_int, C.c_int, C.POINTER(Options), C.POINTER(_P)]),
    "cpqr_set_tensor": (C.c_int32, [_P, C.c_void_p, C.c_int64, C.c_int64, C.c_int]),
    "cpqr_set_ktensor": (C.c_int32, [_P, C.c_int, _DP, C.POINTER(_DP)]),
    "cpqr_batched_qr": (C.c_int32, [C.c_int, C.POINTER(C.c_int64), C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                    C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cpqr_batched": (C.c_int32, [C.c_int, C.POINTER(C.c_int64), C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                 C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cpqr_set_factors": (C.c_int32, [_P, C.POINTER(_DP), _DP]),
    "cpqr_init_factors": (C.c_int32, [_P, C.c_uint64]),
    "cpqr_sweep": (C.c_int32, [_P, C.c_int, _DP]),
    "cpqr_get_factors": (C.c_int32, [_P, C.POINTER(_DP), _DP]),
    "cpqr_get_fit": (C.c_int32, [_P, _DP]),
    "cpqr_get_flags": (C.c_int32, [_P, C.POINTER(C.c_uint32)]),
    "cpqr_get_profile": (C.c_int32, [_P, C.POINTER(Profile), C.c_int]),
    "cpqr_get_timings": (C.c_int32, [_P, C.POINTER(C.c_double)]),
    "cpqr_launches_per_sweep": (C.c_int32, [_P, C.POINTER(C.c_int64)]),
    "cpqr_debug_mode": (C.c_int32, [_P, C.c_int, C.POINTER(_DP), _DP, _DP, _DP, _DP]),
    "cpqr_debug_qr": (C.c_int32, [_P, _DP, C.c_int64, _DP, _DP]),
    "cpqr_debug_svd_solve": (C.c_int32, [_P, _DP, _DP, C.c_int64, C.c_double, _DP, C.POINTER(C.c_int)]),
    "cpqr_debug_plan": (C.c_int32, [_P, C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int)]),
    "cpqr_destroy": (C.c_int32, [_P]),
    "cpqr_status_string": (C.c_char_p, [C.c_int32]),
    "cpqr_last_error": (C.c_char_p, [_P]),
    "cpqr_nccl_unique_id": (C.c_int32, [C.POINTER(C.c_uint8)]),
    "cpqr_version": (C.c_char_p, []),
    "cpqr_peer_handle": (C.c_int32, [_P, C.POINTER(C.c_uint8)]),
    "cpqr_peer_connect": (C.c_int32, [_P, C.POINTER(C.c_uint8)]),
    "cpqr_debug_peer": (C.c_int32, [_P, C.POINTER(C.c_int64)]),
    "cpqr_debug_peer_put": (C.c_int32, [_P, _DP, C.c_int64]),
    "cpqr_debug_peer_get": (C.c_int32, [_P, _DP, C.c_int64, C.c_int]),
}
for _name, (_res, _args) in _sig.items():
    if "CPQR_LIB" in os.environ and not hasattr(_lib, _name):
        continue  # an alternate (older / instrumented A-B) build may lack newer entry points
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class CpqrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def version() -> str:
    return _lib.cpqr_version().decode()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    st = _lib.cpqr_nccl_unique_id(buf)
    if st:
        raise CpqrError(st, "ncclGetUniqueId failed")
    return bytes(buf)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def batched_qr(X, A0, R, max_iters=500, tol=1e-15, stream=None, variant="QR", tau=-1.0):
    """Batched CP-ALS, one CTA per problem (cpqr_batched; variant "QR" is cpqr_batched_qr, also
    "NE", "SVD", "PINV" with the truncation tau for SVD / PINV).  X: CUDA float64 tensor
    (P, I_3, I_2, I_1) C-contiguous (= P column-major tensors); A0: list of three CUDA float64
    tensors (P, R, I_k) C-contiguous (= column-major I_k x R per problem).  Returns (A, lam, fits,
    iters) as CUDA tensors: A a list of (P, R, I_k), lam (P, R), fits (P, max_iters), iters (P,)."""
    import torch
    P, I3, I2, I1 = X.shape
    dims = (C.c_int64 * 3)(I1, I2, I3)
    dev = X.device
    A0cat = torch.cat([a.reshape(P, -1) for a in A0], dim=1).contiguous()
    Aout = torch.empty_like(A0cat)
    lam = torch.empty((P, R), dtype=torch.float64, device=dev)
    fits = torch.empty((P, max_iters), dtype=torch.float64, device=dev)
    iters = torch.empty((P,), dtype=torch.int32, device=dev)
    if stream is None:  # run in order with the torch work that produced X / A0 and reads the outputs
        stream = torch.cuda.current_stream(dev).cuda_stream
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    st = _lib.cpqr_batched(P, dims, int(R), v, float(tau), C.c_void_p(X.data_ptr()), C.c_void_p(A0cat.data_ptr()),
                           int(max_iters), float(tol), C.c_void_p(Aout.data_ptr()), C.c_void_p(lam.data_ptr()),
                           C.c_void_p(fits.data_ptr()), C.c_void_p(iters.data_ptr()),
                           C.c_void_p(int(stream)) if stream else None)
    if st:
        raise CpqrError(st, "cpqr_batched failed")
    out, o = [], 0
    for I in (I1, I2, I3):
        out.append(Aout[:, o:o + I * R].reshape(P, R, I))
        o += I * R
    return out, lam, fits, iters


class CPQR:
    """One CP-ALS(-QR) solver over a (slab of a) dense fp64 tensor on one GPU."""

    def __init__(self, dims, R, variant="QR", svd_tau=-1.0, fit_mode="fast", device=0, stream=None,
                 rank=0, world=1, nccl_id=None, use_graph=True, profile=False, tree=False, comm="nccl"):
        """world > 1 with comm="nccl": this process is rank `rank` of `world` (one GPU each, slab
        of the last mode, NCCL id from nccl_unique_id() on rank 0).  comm="local": ONE context on
        this device runs all `world` slabs as virtual ranks (cpqr.h CPQR_COMM_LOCAL); set_tensor
        then takes the whole tensor.  comm="peer": one process per GPU with the fused push-reduce over
        peer windows (CPQR_COMM_PEER; call peer_connect() with the all-gathered peer_handle()s, or
        connect_peers_torch(), before set_tensor); comm="local_peer": its virtual-rank form."""
        self.dims = tuple(int(d) for d in dims)
        self.N, self.R = len(self.dims), int(R)
        self.variant = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        opt = Options()
        _lib.cpqr_default_options(C.byref(opt))
        opt.svd_tau = float(svd_tau)
        opt.fit_mode = FIT_DIRECT if fit_mode == "direct" else FIT_FAST
        opt.device = int(device)
        opt.stream = C.c_void_p(int(stream)) if stream else None
        opt.rank, opt.world = int(rank), int(world)
        if nccl_id is not None:
            C.memmove(opt.nccl_id, bytes(nccl_id), 128)
        opt.use_graph = 1 if use_graph else 0
        opt.profile = 1 if profile else 0
        opt.mttm_tree = 1 if tree else 0  # dimension-tree Multi-TTM (QR/SVD, N >= 3)
        opt.comm = {"nccl": COMM_NCCL, "local": COMM_LOCAL, "peer": COMM_PEER, "local_peer": COMM_LOCAL_PEER}[comm]
        self.rank, self.world, self.comm = int(rank), int(world), comm
        per = self.dims[-1] // self.world
        virt = comm in ("local", "local_peer")
        self.slab = (0, self.dims[-1]) if virt else (per * self.rank, per * (self.rank + 1))
        d = (C.c_int64 * self.N)(*self.dims)
        h = _P()
        st = _lib.cpqr_create(self.N, d, self.R, self.variant, C.byref(opt), C.byref(h))
        if st:
            raise CpqrError(st, "cpqr_create failed (see stderr)")
        self._h = h
        self._x_ref = None

    # ------------------------------------------------------------------ helpers
    def _check(self, st):
        if st:
            raise CpqrError(st, _lib.cpqr_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            _lib.cpqr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------------- API
    def set_tensor(self, X, copy=False, slab=None):
        """X: numpy array (host) or torch tensor (host or CUDA), C-contiguous (I_N_local..I_1).
        slab=(b, e): the range of the last mode X holds (default: this rank's slab; comm="local":
        the whole tensor, or one virtual rank's slab)."""
        b, e = slab if slab is not None else self.slab
        try:
            import torch
            is_torch = isinstance(X, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_torch = False
        if is_torch:
            assert X.dtype == torch.float64 and X.is_contiguous()
            if X.is_cuda:
                mem = MEM_DEVICE_COPY if copy else MEM_DEVICE_BORROW
                # the context reads X on its own stream: finish the torch work that produced X first
                torch.cuda.current_stream(X.device).synchronize()
            else:
                mem = MEM_HOST
            ptr = C.c_void_p(X.data_ptr())
        else:
            X = np.ascontiguousarray(X, dtype=np.float64)
            mem, ptr = MEM_HOST, C.c_void_p(X.ctypes.data)
        self._check(_lib.cpqr_set_tensor(self._h, ptr, b, e, mem))
        self._x_ref = X if mem == MEM_DEVICE_BORROW else None

    def set_ktensor(self, lam, B):
        """Kruskal-tensor input X = [[lam; B_1..B_N]]: B[k] is I_k x S."""
        arrs = [np.asfortranarray(np.asarray(b, dtype=np.float64)) for b in B]
        S = arrs[0].shape[1]
        ptrs = (_DP * self.N)(*[_dptr(a) for a in arrs])
        lam = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
        self._check(_lib.cpqr_set_ktensor(self._h, int(S), _dptr(lam) if lam is not None else _DP(), ptrs))

    def set_factors(self, factors, lam=None):
        arrs = [None if A is None else np.asfortranarray(np.asarray(A, dtype=np.float64)) for A in factors]
        ptrs = (_DP * self.N)(*[(_dptr(a) if a is not None else _DP()) for a in arrs])
        lp = _dptr(np.ascontiguousarray(lam, dtype=np.float64)) if lam is not None else _DP()
        self._check(_lib.cpqr_set_factors(self._h, ptrs, lp))

    def init_factors(self, seed):
        self._check(_lib.cpqr_init_factors(self._h, int(seed)))

    def sweep(self, nsweeps=1) -> np.ndarray:
        fits = np.zeros(max(1, nsweeps))
        self._check(_lib.cpqr_sweep(self._h, int(nsweeps), _dptr(fits)))
        return fits[:nsweeps]

    def get_factors(self):
        outs = [np.zeros((d, self.R), order="F") for d in self.dims]
        lam = np.zeros(self.R)
        ptrs = (_DP * self.N)(*[_dptr(a) for a in outs])
        self._check(_lib.cpqr_get_factors(self._h, ptrs, _dptr(lam)))
        return lam, outs

    @property
    def fit(self):
        f = C.c_double()
        self._check(_lib.cpqr_get_fit(self._h, C.byref(f)))
        return f.value

    @property
    def flags(self):
        f = C.c_uint32()
        self._check(_lib.cpqr_get_flags(self._h, C.byref(f)))
        return f.value

    # -------------------------------------------------------- peer windows (CPQR_COMM_PEER)
    def peer_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        self._check(_lib.cpqr_peer_handle(self._h, buf))
        return bytes(buf)

    def peer_connect(self, handles):
        """handles: the ranks' peer_handle() bytes in rank order."""
        blob = b"".join(bytes(h) for h in handles)
        assert len(blob) == 64 * self.world
        self._check(_lib.cpqr_peer_connect(self._h, (C.c_uint8 * len(blob)).from_buffer_copy(blob)))

    def connect_peers_torch(self, group=None):
        """All-gather the window handles over a torch.distributed process group and connect."""
        import torch
        import torch.distributed as dist
        mine = torch.frombuffer(bytearray(self.peer_handle()), dtype=torch.uint8).clone()
        if dist.get_backend(group) == "nccl":
            mine = mine.cuda()
        outs = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(outs, mine, group=group)
        self.peer_connect([bytes(o.cpu().numpy().tobytes()) for o in outs])

    def debug_peer(self):
        info = (C.c_int64 * 4)()
        self._check(_lib.cpqr_debug_peer(self._h, info))
        return dict(epoch=info[0], windows_differing=info[1], window_bytes=info[2], min_flag=info[3])

    def debug_peer_put(self, src):
        src = np.ascontiguousarray(src, dtype=np.float64)
        self._check(_lib.cpqr_debug_peer_put(self._h, _dptr(src), src.size))

    def debug_peer_get(self, n, gather=False):
        out = np.zeros(n * (self.world if gather else 1))
        self._check(_lib.cpqr_debug_peer_get(self._h, _dptr(out), int(n), 1 if gather else 0))
        return out

    def profile(self, reset=True):
        p = Profile()
        self._check(_lib.cpqr_get_profile(self._h, C.byref(p), 1 if reset else 0))
        return dict(ms=list(p.ms), launches=list(p.launches), bytes0=p.bytes0, flops0=p.flops0,
                    launches_total=p.launches_total)

    def timings(self):
        """cpqr_get_timings: per-phase ms since the last profile reset (needs profile=True):
        stream-X pass, remaining TTMs, factor QR (fused tail), Q0 compute, Q0 apply, other,
        exchange."""
        ms = (C.c_double * 7)()
        self._check(_lib.cpqr_get_timings(self._h, ms))
        return list(ms)

    def launches_per_sweep(self):
        n = C.c_int64()
        self._check(_lib.cpqr_launches_per_sweep(self._h, C.byref(n)))
        return n.value

    def debug_mode(self, n, Q_override=None):
        """Alg. 2 lines 6-9 for mode n without changing state: dict(Y, Q0, R0, W) (host arrays;
        Y is the column-major Multi-TTM tensor returned as a Fortran array of its dims)."""
        R, N = self.R, self.N
        ydims = [R] * N
        ydims[n] = self.dims[n]
        Y = np.zeros(ydims, order="F")
        J = R ** (N - 1)
        Q0 = np.zeros((J, R), order="F")
        R0 = np.zeros((R, R), order="F")
        W = np.zeros((self.dims[n], R), order="F")
        qp = None
        keep = []
        if Q_override is not None:
            arr = []
            for k in range(N):
                if k == n or Q_override[k] is None:
                    arr.append(_DP())
                else:
                    a = np.asfortranarray(Q_override[k], dtype=np.float64)
                    keep.append(a)
                    arr.append(_dptr(a))
            qp = (_DP * N)(*arr)
        self._check(_lib.cpqr_debug_mode(self._h, int(n), qp, Y.ctypes.data_as(_DP), Q0.ctypes.data_as(_DP),
                                         R0.ctypes.data_as(_DP), W.ctypes.data_as(_DP)))
        return dict(Y=Y, Q0=Q0, R0=R0, W=W)

    PLAN_KINDS = {0: "strided", 1: "fiber", 2: "slice", 3: "slice-reduce", 4: "strided-tma", 5: "fiber-tma",
                  6: "slice-tma", 7: "slice-fixup", 8: "slice-small-tma", 9: "small-ttm", 10: "strided2-tma",
                  100: "ne-diag"}

    def debug_plan(self, n, slab=0):
        """The Multi-TTM plan of mode n on one slab (cpqr_debug_plan): a list of dicts with the
        kernel kind, the contracted modes, input / output elements and flops of every step."""
        cap = 64
        buf = (C.c_int64 * (6 * cap))()
        cnt = C.c_int()
        self._check(_lib.cpqr_debug_plan(self._h, int(n), int(slab), buf, cap, C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            kind, mask, ni, no, fl, xp = (int(v) for v in buf[6 * i:6 * i + 6])
            out.append(dict(kind=self.PLAN_KINDS.get(kind, kind), modes=[k for k in range(self.N) if mask >> k & 1],
                            in_elems=ni, out_elems=no, flops=fl, x_pass=bool(xp)))
        return out

    def debug_qr(self, A):
        A = np.asfortranarray(A, dtype=np.float64)
        m = A.shape[0]
        Q = np.zeros((m, self.R), order="F")
        Rf = np.zeros((self.R, self.R), order="F")
        self._check(_lib.cpqr_debug_qr(self._h, _dptr(A), m, Q.ctypes.data_as(_DP), Rf.ctypes.data_as(_DP)))
        return Q, Rf

    def debug_svd_solve(self, R0, W, tau):
        R0 = np.asfortranarray(R0, dtype=np.float64)
        W = np.asfortranarray(W, dtype=np.float64)
        m = W.shape[0]
        out = np.zeros((m, self.R), order="F")
        nt = C.c_int()
        self._check(_lib.cpqr_debug_svd_solve(self._h, _dptr(R0), _dptr(W), m, float(tau),
                                              out.ctypes.data_as(_DP), C.byref(nt)))
        return out, nt.value
