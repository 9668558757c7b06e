"""GPU side of the input generator (workload/csrc/gen.cu -> workload/libwlgen.so).

Input plumbing for tests and bench.py only: fills tables / upstream gradients in HBM with
the same counter-based values as workload/gen.py (bit-identical, pinned by the tests).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libwlgen.so")
SRC = os.path.join(HERE, "csrc", "gen.cu")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                               "-shared", "-cudart", "static", SRC, "-o", LIB])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.wl_fill_table.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int64,
                                    C.c_int, C.c_void_p]
        L.wl_fill_grad.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int64, C.c_int64,
                                   C.c_int, C.c_void_p]
        L.wl_flush.argtypes = [C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p]
        _lib = L
    return _lib


def fill_table(dst_tensor, nrows, dim, pitch, seed, table, row0=0, shift=26, stream=None):
    """dst_tensor: CUDA fp32 tensor holding [nrows][pitch] (view or slice)."""
    import torch
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    rc = lib().wl_fill_table(C.c_void_p(dst_tensor.data_ptr()), int(nrows), int(dim), int(pitch),
                             int(seed) & 0xFFFFFFFFFFFFFFFF, int(table), int(row0), int(shift), C.c_void_p(s))
    assert rc == 0, rc


def fill_grad(dst_tensor, batch, F, dim, seed, step, shift, sample0=0, stream=None):
    import torch
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    rc = lib().wl_fill_grad(C.c_void_p(dst_tensor.data_ptr()), int(batch), int(F), int(dim),
                            int(seed) & 0xFFFFFFFFFFFFFFFF, int(step), int(sample0), int(shift), C.c_void_p(s))
    assert rc == 0, rc


def flush_l2(buf, stream=None):
    import torch
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    rc = lib().wl_flush(C.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(), 0x3F800000, C.c_void_p(s))
    assert rc == 0, rc
