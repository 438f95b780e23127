"""Test helper: copy between host numpy arrays and raw device pointers
returned by the C ABI (paro_buffer), via the CUDA runtime torch ships."""
import ctypes
import glob
import os

import numpy as np

_rt = None


def _cudart():
    global _rt
    if _rt is None:
        import nvidia.cuda_runtime as cr
        path = glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))[0]
        _rt = ctypes.CDLL(path)
        _rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _rt.cudaMemcpy.restype = ctypes.c_int
        _rt.cudaDeviceSynchronize.restype = ctypes.c_int
    return _rt


def d2h(ptr, n, dtype):
    out = np.empty(n, dtype=dtype)
    rt = _cudart()
    assert rt.cudaDeviceSynchronize() == 0
    assert rt.cudaMemcpy(out.ctypes.data, ctypes.c_void_p(ptr), out.nbytes, 2) == 0
    return out


def h2d(ptr, arr):
    arr = np.ascontiguousarray(arr)
    rt = _cudart()
    assert rt.cudaMemcpy(ctypes.c_void_p(ptr), arr.ctypes.data, arr.nbytes, 1) == 0
