"""Build libcpqr.so in-tree for sm_100a (nvcc, no JIT cache): `python -m paper_2112_10855_b200.build`."""
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcpqr.so")
SRC = [os.path.join(HERE, "csrc", "cpqr.cu")]
DEPS = SRC + sorted(os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
                    if f.endswith(".cuh")) + [os.path.join(ROOT, "include", "cpqr.h")]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=True, out=None):
    """out: another path for an instrumented build (e.g. CPQR_DEBUG_TIMING=1 ... --out libcpqr_dbg.so,
    loaded with CPQR_LIB=...); the default in-tree libcpqr.so is the product library."""
    LIB = out or globals()["LIB"]
    if not force and out is None and up_to_date():
        return LIB
    inc, lib = nccl_dirs()
    # link against libnccl.so.2 by soname (the pip package ships no unversioned symlink)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v" if verbose == "ptxas" else "-O3", *(["-DCPQR_DEBUG_FIT"] if os.environ.get("CPQR_DEBUG_FIT") else []), *(["-DCPQR_DEBUG_TIMING"] if os.environ.get("CPQR_DEBUG_TIMING") else []), *(["-DCPQR_DEBUG_HANG"] if os.environ.get("CPQR_DEBUG_HANG") else []),
           *([f"-DCPQR_RELEASE_MODE={int(os.environ['CPQR_RELEASE_MODE'])}"] if os.environ.get("CPQR_RELEASE_MODE") else []),
           *([f"-DCPQR_CQ_CLOSED_FORM={int(os.environ['CPQR_CQ_CLOSED_FORM'])}"] if os.environ.get("CPQR_CQ_CLOSED_FORM") else []),
           "-I", inc, "-I", os.path.join(ROOT, "include"),
           *SRC, "-o", LIB + ".tmp",
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    if os.path.exists(LIB + ".tmp"):
        os.remove(LIB + ".tmp")
    r = subprocess.run(cmd)
    if r.returncode != 0 or not os.path.exists(LIB + ".tmp"):
        raise RuntimeError(f"nvcc failed (rc={r.returncode}); libcpqr.so NOT rebuilt")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    build(force="--force" in sys.argv, verbose="ptxas" if "--ptxas" in sys.argv else True,
          out=os.path.join(HERE, o) if o and not os.path.isabs(o) else o)
