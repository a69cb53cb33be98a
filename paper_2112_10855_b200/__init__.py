"""paper_2112_10855_b200: B200-native (sm_100a, fp64) hot path of QR-based CP-ALS (arXiv 2112.10855).

`cpqr` is the thin ctypes binding of libcpqr.so (include/cpqr.h); `synth` holds the seeded
input generators shared with the tests.  Import `paper_2112_10855_b200.cpqr` explicitly: it
raises if the CUDA library is not built (no CPU fallback).
"""
__all__ = ["cpqr", "synth", "build"]
