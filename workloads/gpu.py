"""GPU fill of the counter-Gaussian workload matrix (workloads/csrc/gen.cu -> libihtgen.so).

Input generation only (no method arithmetic); bit-identical to
workloads.gen.gaussian_block, so config 4's 64 GiB Phi can be produced block-wise
on the device instead of crossing PCIe.
"""
import ctypes
import os

import torch

from .gen import gauss_scale32

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libihtgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError("libihtgen.so not built; run python -m paper_1802_04907_b200.build")
        lib = ctypes.CDLL(_LIB)
        lib.ihtgen_gauss_fill.restype = ctypes.c_int
        lib.ihtgen_gauss_fill.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                          ctypes.c_float, ctypes.c_void_p]
        _lib = lib
    return _lib


def gauss_fill(out, key, n_total, row0, col0, sd, stream=None):
    """Fill the CUDA float32 matrix `out` (rows x cols, row-major) with
    Phi[row0:row0+rows, col0:col0+cols] of the counter-Gaussian matrix."""
    assert out.is_cuda and out.dtype == torch.float32 and out.stride(1) == 1
    rows, cols = out.shape
    st = (stream or torch.cuda.current_stream()).cuda_stream
    rc = _load().ihtgen_gauss_fill(ctypes.c_void_p(out.data_ptr()), rows, cols, out.stride(0), row0, col0,
                                   n_total, key, float(gauss_scale32(sd)), ctypes.c_void_p(st))
    if rc != 0:
        raise RuntimeError("ihtgen_gauss_fill failed")
    return out
