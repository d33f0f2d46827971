"""Loader for the in-tree CUDA library (paper_2504_12471_b200/libd2ft_b200.so).

There is no CPU fallback: if the library is missing or cannot reach a GPU the
calls fail loudly with an Error."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# D2FT_B200_LIB lets profiling experiments load an alternative build of the
# same library (never a CPU path: every build is the sm_100a library).
LIB_PATH = os.environ.get("D2FT_B200_LIB", os.path.join(HERE, "libd2ft_b200.so"))

# d2ft::errc (error.hpp:12-19) + cuda
ERRC = {1: "config", 2: "input", 3: "dimension", 4: "state", 5: "numeric", 6: "size", 7: "cuda"}


class Error(RuntimeError):
    """Mirror of d2ft::Error (error.hpp:21-28): message + category `kind`."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = ERRC.get(code, "unknown")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Error(4, f"d2ft_b200: CUDA library not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.d2ft_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise Error(rc, lib().d2ft_last_error().decode())


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def i32(x, n=None):
    a = np.ascontiguousarray(x, dtype=np.int32)
    if n is not None and a.shape != (n,):
        a = np.ascontiguousarray(np.broadcast_to(a, (n,)), dtype=np.int32)
    return a


def f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def u8(x):
    return np.ascontiguousarray(x, dtype=np.uint8)
