"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is the ONLY code shared by the oracle side (tests, bench's cpu_baseline)
and the CUDA side.  It holds none of the CP-ALS-QR arithmetic: it draws random numbers
and builds the planted tensor X = [[lambda; A_1..A_N]] + noise (Eq. (cp)),
written out here with its own plain einsum/matmul so it shares no helper with either side.

Recipe (SURVEY.md §8(c) "Generator recipe, exact draw order"):
  rng_s = numpy.random.default_rng(211210855 + 10*cfg + s)
  s = 0  truth factors, drawn for k = 1..N as C-order (I_k, R) arrays
         kind 'normal'     : A_k ~ N(0,1)                                  (C1)
         kind 'congruence' : G ~ N(0,1); U = Q of numpy.linalg.qr(G) (no sign fix);
                             C = c*11^T + (1-c)I; A_k = U @ cholesky(C).T  (C2, C3, C5;
                             reading 21: A_k^T A_k = C exactly)
         kind 'pair'       : G ~ N(0,1), columns normalised; u = g2 - (g2.g1) g1, normalised;
                             g2 <- c g1 + sqrt(1-c^2) u                     (C4; reading 22)
         lambda = 1
  s = 1  noise E ~ N(0,1) of C-order shape (I_N, ..., I_1) (= column-major X's memory order);
         X = X_clean + eta*||X_clean||/||E|| * E   (reading 20); eta = 0 draws nothing
  s = 2  init factors A0_k ~ N(0,1), C-order (I_k, R), k = 1..N (A0_1 drawn though unused)
  s = 3  exact-duplicate test stream (tests only)

All tensors are returned as the flat column-major buffer (a C-order ndarray of shape
(I_N, ..., I_1), which has exactly the bytes of column-major X with mode 1 fastest).
Factors are returned as Fortran-ordered (I_k, R) float64 arrays (column-major, the layout
the C-ABI takes).
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 211210855


@dataclass(frozen=True)
class Config:
    cfg: int
    dims: tuple
    R: int
    kind: str          # 'normal' | 'congruence' | 'pair'
    c: float           # congruence (unused for 'normal')
    eta: float         # relative noise level
    variants: tuple    # variants BASELINE.json runs on this config
    sweeps: int
    gpus: tuple = (1,)
    svd_tau: float = -1.0   # SVD truncation tau (<0: library default R*eps)
    name: str = ""

    @property
    def N(self):
        return len(self.dims)

    @property
    def numel(self):
        return int(np.prod(self.dims, dtype=np.int64))


# BASELINE.json "configs" (C1..C5), transcribed; SURVEY.md §8 config key.
CONFIGS = {
    1: Config(1, (30, 40, 50), 5, "normal", 0.0, 0.01, ("QR",), 5, (1,), name="C1 30x40x50 R5"),
    2: Config(2, (400, 400, 400), 10, "congruence", 0.9, 0.01, ("QR", "NE"), 20, (1,), name="C2 400^3 R10"),
    3: Config(3, (128, 128, 128, 128), 16, "congruence", 0.99, 0.001, ("QR", "SVD"), 20, (1, 2, 4, 8),
              name="C3 128^4 R16"),
    4: Config(4, (48, 48, 48, 48, 48), 8, "pair", 0.999, 0.0, ("SVD",), 20, (1, 2, 4, 8), svd_tau=1e-12,
              name="C4 48^5 R8"),
    5: Config(5, (1000, 1000, 1000), 32, "congruence", 0.5, 0.01, ("QR",), 10, (1, 2, 4, 8),
              name="C5 1000^3 R32"),
}


def rng(cfg: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(SEED_BASE + 10 * cfg + stream)


def truth_factors(conf: Config):
    g = rng(conf.cfg, 0)
    out = []
    for I in conf.dims:
        G = g.standard_normal((I, conf.R))
        if conf.kind == "normal":
            A = G
        elif conf.kind == "congruence":
            U, _ = np.linalg.qr(G)
            C = conf.c * np.ones((conf.R, conf.R)) + (1.0 - conf.c) * np.eye(conf.R)
            A = U @ np.linalg.cholesky(C).T
        elif conf.kind == "pair":
            A = G / np.linalg.norm(G, axis=0)
            g1 = A[:, 0].copy()
            u = A[:, 1] - (A[:, 1] @ g1) * g1
            u /= np.linalg.norm(u)
            A[:, 1] = conf.c * g1 + np.sqrt(1.0 - conf.c ** 2) * u
        else:
            raise ValueError(conf.kind)
        out.append(np.asfortranarray(A))
    return out


def init_factors(conf: Config, stream: int = 2):
    g = rng(conf.cfg, stream)
    return [np.asfortranarray(g.standard_normal((I, conf.R))) for I in conf.dims]


def _kr_rows(mats):
    """Rows of mats[0] (x) mats[1] (x) ... column-wise, LAST matrix's row index fastest."""
    out = mats[0]
    for M in mats[1:]:
        out = (out[:, None, :] * M[None, :, :]).reshape(-1, out.shape[1])
    return out


def planted_tensor(factors, weights=None, chunk_rows: int = 1 << 14):
    """X_clean as a C-order (I_N, ..., I_1) array: X(i_1..i_N) = sum_r lam_r prod_k A_k(i_k, r)."""
    dims = tuple(A.shape[0] for A in factors)
    R = factors[0].shape[1]
    lam = np.ones(R) if weights is None else np.asarray(weights, dtype=np.float64)
    A1 = factors[0] * lam[None, :]
    rest = [np.ascontiguousarray(A) for A in factors[1:][::-1]]  # A_N, ..., A_2 (A_2 fastest)
    J = int(np.prod(dims[1:], dtype=np.int64))
    X = np.empty((J, dims[0]), dtype=np.float64)
    if len(rest) == 0:
        X[:] = A1.sum(axis=1)[None, :]
    else:
        # chunk over the slowest factor so the Khatri-Rao rows never exceed ~chunk_rows*R
        slow = rest[0]
        inner = _kr_rows(rest[1:]) if len(rest) > 1 else np.ones((1, R))
        per = inner.shape[0]
        step = max(1, chunk_rows // max(1, per))
        for s0 in range(0, slow.shape[0], step):
            s1 = min(slow.shape[0], s0 + step)
            K = (slow[s0:s1, None, :] * inner[None, :, :]).reshape(-1, R)
            X[s0 * per:s1 * per] = K @ A1.T
    return X.reshape(dims[::-1])


def add_noise(Xc: np.ndarray, eta: float, g: np.random.Generator, chunk: int = 1 << 26):
    """In place: X <- X + eta*||X||/||E|| * E, E ~ N(0,1) drawn in memory order."""
    if eta == 0.0:
        return Xc
    flat = Xc.reshape(-1)
    nx2 = float(np.dot(flat, flat)) if flat.size <= chunk else sum(
        float(np.dot(flat[i:i + chunk], flat[i:i + chunk])) for i in range(0, flat.size, chunk))
    E = g.standard_normal(flat.size)
    ne2 = sum(float(np.dot(E[i:i + chunk], E[i:i + chunk])) for i in range(0, E.size, chunk))
    scale = eta * np.sqrt(nx2) / np.sqrt(ne2)
    for i in range(0, flat.size, chunk):
        flat[i:i + chunk] += scale * E[i:i + chunk]
    del E
    return Xc


def _cache_dir():
    return os.environ.get("CPQR_CACHE", "/tmp/cpqr_cache")


def make_problem(cfg, cache: bool = True):
    """Return (conf, Xc, truth_factors, init_factors) for config cfg (int or Config).

    Xc is the C-order (I_N..I_1) float64 array = column-major X.  Large tensors are cached
    as .npy under $CPQR_CACHE (content-addressed by the recipe; a cache is only an
    accelerator: a missing or mismatched file is regenerated)."""
    conf = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    truth = truth_factors(conf)
    init = init_factors(conf)
    key = hashlib.sha1(repr((conf.cfg, conf.dims, conf.R, conf.kind, conf.c, conf.eta, "v1")).encode()).hexdigest()[:12]
    path = os.path.join(_cache_dir(), f"X_c{conf.cfg}_{key}.npy")
    if cache and conf.numel >= (1 << 24) and os.path.exists(path):
        try:
            Xc = np.load(path, mmap_mode="r")
            if Xc.shape == tuple(conf.dims[::-1]) and Xc.dtype == np.float64:
                return conf, np.asarray(Xc), truth, init
        except Exception:
            pass
    Xc = planted_tensor(truth)
    add_noise(Xc, conf.eta, rng(conf.cfg, 1))
    if cache and conf.numel >= (1 << 24):
        try:
            os.makedirs(_cache_dir(), exist_ok=True)
            tmp = path + f".tmp{os.getpid()}"
            np.save(tmp, Xc)
            os.replace(tmp + ".npy" if not tmp.endswith(".npy") else tmp, path)
        except Exception:
            pass
    return conf, Xc, truth, init


def small_problem(dims, R, seed, eta=0.01, kind="normal", c=0.0):
    """Ad-hoc seeded problem for tests (not a BASELINE config): cfg id derived from seed."""
    conf = Config(1000 + seed, tuple(dims), R, kind, c, eta, ("QR",), 1, name=f"adhoc{seed}")
    truth = truth_factors(conf)
    Xc = planted_tensor(truth)
    add_noise(Xc, eta, rng(conf.cfg, 1))
    return conf, Xc, truth, init_factors(conf)
