"""Build libpotr_b200.so in-tree with nvcc for sm_100a.

The library is plain CUDA C++ behind an extern "C" ABI (include/potr_b200.h);
it is loaded with ctypes, so it does not depend on torch's C++ ABI.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_lib", "libpotr_b200.so")
SOURCES = ["capi.cu", "raster.cu", "sh.cu", "metrics.cu", "codec.cu", "sort.cu", "controller.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # float64 parity: never contract a*b+c into FMA (the reference's numpy /
    # numba arithmetic does not); explicit fma() calls are kept.
    "--fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-lgomp", "-shared", "-cudart", "static",
]


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "potr_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    """Compile if any source is newer than the library; returns its path.
    Process-safe: concurrent callers (ranks of one job) serialize on a lock
    file and the library is replaced atomically."""
    import fcntl
    if not force and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    with open(LIB + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not needs_build():  # another process built it meanwhile
            return LIB
        tmp = f"{LIB}.{os.getpid()}.tmp"
        flags = list(NVCC_FLAGS) + (["-Xptxas", "-v"] if verbose else [])
        cmd = [nvcc(), *flags, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building libpotr_b200.so")
        if verbose:
            sys.stderr.write(res.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
