"""Device twin of synth/gen.py's LogitsSpec (TEST/BENCH INPUT GENERATOR).

Builds and loads synth/libgrpo_synth.so; fills bf16 logits on the GPU with the
same counter-based generator the host uses, bit for bit.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "synth_fill.cu")
LIB = os.path.join(HERE, "libgrpo_synth.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-cudart", "static", "-shared",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.synth_fill_logits.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                           C.c_int64, C.c_uint64, C.c_void_p, C.c_float, C.c_void_p]
        _lib.synth_fill_logits.restype = C.c_int
    return _lib


def fill_logits(out, spec, row_begin, n_rows, V, base_dev=None, stream=None):
    """out: 16-bit CUDA tensor [>= n_rows, ld]; fills rows row_begin.. of the spec."""
    import torch
    if base_dev is None:
        base_dev = torch.from_numpy(np.ascontiguousarray(spec.base, np.float32)).to(out.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = lib().synth_fill_logits(out.data_ptr(), n_rows, row_begin, spec.period, V, out.shape[1],
                                 int(spec.key), base_dev.data_ptr(), float(spec.scale), s.cuda_stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill_logits failed: cuda error {rc}")
    return base_dev
