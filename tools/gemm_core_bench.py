"""Dense GEMM core throughput at the step's tile shapes (CTA pairs): B
multicast vs pair UMMA, with / without output stores, MN-major A or B."""
import ctypes as C
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2504_12471_b200 import _lib
_lib.lib()
lib = C.CDLL(os.path.join(os.path.dirname(_lib.LIB_PATH), "libd2ft_b200_testing.so"))  # the GEMM self-test hooks
names = ["multicast N208", "pair N208", "multicast N208 nostore", "pair N208 nostore", "pair A-MN N208 nostore",
         "pair B-MN N208 nostore", "pair B-MN N256 nostore", "pair B-MN N128 nostore", "multicast B-MN N208 nostore"]
nn = [208, 208, 208, 208, 208, 208, 256, 128, 208]
for K in (768,):
    M = 148 * 2 * 128 * 12
    for var in range(9):
        ms = C.c_double()
        _lib.check(lib.d2ft_test_gemm_bench_pair(C.c_int(M), C.c_int(K), C.c_int(var), C.c_int(20), C.byref(ms)))
        tf = 2.0 * M * nn[var] * K / (ms.value * 1e-3) / 1e12
        print(f"M={M} K={K} {names[var]}: {ms.value*1e3:.1f} us, {tf:.0f} TFLOP/s")
