"""GPU: the tcgen05/TMEM/TMA GEMM core (single CTA, B-multicast CTA pairs bn < 0, and pair UMMA with
cta_group::2, bn = -2208) against a plain fp32 reference of the same op (bf16-rounded operands, fp64
accumulation on the host)."""
import ctypes as C

import numpy as np
import pytest

from paper_2504_12471_b200 import _lib

pytestmark = pytest.mark.gpu


def bf16(x):
    """round-to-nearest-even bf16 bits and the rounded fp32 values"""
    f = np.ascontiguousarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    back = (r.astype(np.uint32) << 16).view(np.float32)
    return r, back


_TESTING = None


def _testing():
    """The GEMM self-test hooks live in libd2ft_b200_testing.so (not in the
    product library); errors come back through the product's d2ft_last_error."""
    global _TESTING
    if _TESTING is None:
        import os
        _lib.lib()  # the product library first (the hooks link against it)
        _TESTING = C.CDLL(os.path.join(os.path.dirname(_lib.LIB_PATH), "libd2ft_b200_testing.so"))
    return _TESTING


def _call(name, *args):
    fn = getattr(_testing(), name)
    _lib.check(fn(*args))


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (256, 512, 768, 256), (200, 300, 320, 208),
                                      (384, 320, 448, 160), (1000, 700, 1024, 256),
                                      (640, 416, 768, -208), (384, 320, 448, -160), (130, 500, 128, -208),
                                      (640, 416, 768, -2208), (256, 208, 64, -2208), (130, 500, 128, -2208),
                                      (1000, 700, 1024, -2208)])
def test_dense(M, N, K, bn):
    rng = np.random.default_rng(M + N + K)
    A, Af = bf16(rng.standard_normal((M, K)))
    B, Bf = bf16(rng.standard_normal((N, K)))
    D = np.zeros((M, N), np.float32)
    _call("d2ft_test_gemm_dense", _lib.ptr(A), _lib.ptr(B), C.c_int(M), C.c_int(N), C.c_int(K), C.c_int(bn),
          _lib.ptr(D))
    ref = Af.astype(np.float64) @ Bf.astype(np.float64).T
    err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err


@pytest.mark.parametrize("M,N,K,bn", [(128, 64, 64, 64), (256, 208, 448, 208), (384, 416, 320, 208),
                                      (200, 200, 768, 208), (512, 624, 320, -208), (384, 128, 192, -64),
                                      (130, 96, 128, 64), (512, 624, 320, -2208), (256, 208, 768, -2208),
                                      (130, 200, 128, -2208)])
def test_mn_major_b(M, N, K, bn):
    """B stored [K][N] (N contiguous) and read by UMMA as an MN-major operand."""
    rng = np.random.default_rng(M * 3 + N + K)
    A, Af = bf16(rng.standard_normal((M, K)))
    BT, BTf = bf16(rng.standard_normal((K, N)))
    D = np.zeros((M, N), np.float32)
    _call("d2ft_test_gemm_mn", _lib.ptr(A), _lib.ptr(BT), C.c_int(M), C.c_int(N), C.c_int(K), C.c_int(bn),
          _lib.ptr(D))
    ref = Af.astype(np.float64) @ BTf.astype(np.float64)
    err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err


@pytest.mark.parametrize("M,N,K", [(128, 208, 64), (384, 416, 448), (264, 200, 320)])
def test_mn_major_a_and_b(M, N, K):
    """A stored [K][M] and B stored [K][N], both read MN-major."""
    rng = np.random.default_rng(M + 7 * N + K)
    AT, ATf = bf16(rng.standard_normal((K, M)))
    BT, BTf = bf16(rng.standard_normal((K, N)))
    D = np.zeros((M, N), np.float32)
    _call("d2ft_test_gemm_mn_ab", _lib.ptr(AT), _lib.ptr(BT), C.c_int(M), C.c_int(N), C.c_int(K), _lib.ptr(D))
    ref = ATf.astype(np.float64).T @ BTf.astype(np.float64)
    err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err


def test_planes_tokens_as_n():
    M, T, K, P = 448, 197, 768, 5
    rng = np.random.default_rng(1)
    A, Af = bf16(rng.standard_normal((M, K)))
    X, Xf = bf16(rng.standard_normal((P, T, K)))
    D = np.zeros((P, M, T), np.float32)
    _call("d2ft_test_gemm_planes", _lib.ptr(A), _lib.ptr(X), C.c_int(M), C.c_int(T), C.c_int(K), C.c_int(P),
          _lib.ptr(D))
    ref = np.einsum("mk,ptk->pmt", Af.astype(np.float64), Xf.astype(np.float64))
    err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err


def test_tokens_as_k_zero_fill():
    M, N, T, TP, P = 320, 768, 197, 208, 6
    rng = np.random.default_rng(2)
    XT, XTf = bf16(rng.standard_normal((P, M, TP)))
    YT, YTf = bf16(rng.standard_normal((P, N, TP)))
    D = np.zeros((M, N), np.float32)
    _call("d2ft_test_gemm_tokenk", _lib.ptr(XT), _lib.ptr(YT), C.c_int(M), C.c_int(N), C.c_int(T), C.c_int(TP),
          C.c_int(P), _lib.ptr(D))
    ref = np.einsum("pmt,pnt->mn", XTf[:, :, :T].astype(np.float64), YTf[:, :, :T].astype(np.float64))
    err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err


def test_dense_throughput_reported():
    ms = C.c_double()
    M = N = K = 8192
    _call("d2ft_test_gemm_bench", C.c_int(M), C.c_int(N), C.c_int(K), C.c_int(10), C.byref(ms))
    tflops = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
    print(f"dense 8192^3 bf16 tcgen05: {ms.value:.3f} ms = {tflops:.0f} TFLOP/s")
    assert tflops > 100
