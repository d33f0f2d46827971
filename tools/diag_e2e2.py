"""Diagnostic: e2e leg timing with and without a preceding profiled (eager) pass."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_2504_12471_b200 import _lib, engine as E, scheduler as S
lib = _lib.lib()
B = 64; K = 144
x, y, bwd, fwd, capf, capo = bench.workload(B)
m = E.SubnetModel(E.VIT_B16, B)
m.stage(x, y, S.ScoreTable(K, B, fwd, bwd), S.CostModel(), S.Capacities(capf.tolist(), capo.tolist()))
lib.d2ft_host_alloc.restype = C.c_void_p
hx = lib.d2ft_host_alloc(C.c_size_t(x.nbytes))
px = np.frombuffer((C.c_char * x.nbytes).from_address(hx), np.float32).reshape(x.shape); px[...] = x
pc = np.zeros((4, K), np.int32); pc[0], pc[1], pc[2], pc[3] = 2, 3, capf, capo
yy = np.ascontiguousarray(y.astype(np.int32)); bw = np.ascontiguousarray(bwd); fw = np.ascontiguousarray(fwd)
loss = C.c_double()
def e2e(tag, steps=10):
    ms = C.c_double()
    _lib.check(lib.d2ft_engine_bench_e2e(m._h, _lib.ptr(px), _lib.ptr(yy), _lib.ptr(bw), _lib.ptr(fw), _lib.ptr(pc[0]), _lib.ptr(pc[1]),
               _lib.ptr(pc[2]), _lib.ptr(pc[3]), C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9),
               C.c_int(1), C.c_int(steps), C.byref(ms), C.byref(loss)))
    print(tag, "e2e ms/step", ms.value / steps)
def dev(tag, steps=10):
    ms = C.c_double()
    _lib.check(lib.d2ft_engine_bench_device(m._h, C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9), C.c_int(3), C.c_int(steps), C.byref(ms), C.byref(loss)))
    print(tag, "device ms/step", ms.value / steps)
dev("a"); e2e("a")
m.set_profiling(True); dev("prof"); m.set_profiling(False)
e2e("b"); dev("c"); e2e("c"); e2e("d", 30)
