"""Build the in-tree CUDA shared library libgrpo_async.so for sm_100a.

    python paper_2604_26256_b200/build.py [--force]     # or __graft_entry__.build()

nvcc cross-compiles here without a GPU; the .so travels to the GPU box with
the gpurun snapshot.  cudart is linked statically so the library does not
depend on which libcudart torch ships.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libgrpo_async.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-cudart", "static",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]
LINK = []  # no cuBLAS: every GEMM of the path is a hand-written tcgen05 kernel


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *NVCC_FLAGS, "-I", INCLUDE, "-shared", "-o", tmp, *sources(), *LINK]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(ROOT, "build", "ptxas_grpo_async.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-6000:])
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stdout.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
