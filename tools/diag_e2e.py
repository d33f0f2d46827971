import ctypes as C, time, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_2504_12471_b200 import _lib, engine as E, scheduler as S
lib=_lib.lib()
B=64; K=144
x,y,bwd,fwd,capf,capo=bench.workload(B)
m=E.SubnetModel(E.VIT_B16,B)
m.stage(x,y,S.ScoreTable(K,B,fwd,bwd),S.CostModel(),S.Capacities(capf.tolist(),capo.tolist()))
lib.d2ft_host_alloc.restype=C.c_void_p
hx=lib.d2ft_host_alloc(C.c_size_t(x.nbytes))
px=np.frombuffer((C.c_char*x.nbytes).from_address(hx),np.float32).reshape(x.shape); px[...]=x
cf=np.full(K,2,np.int32); cb=np.full(K,3,np.int32)
loss=C.c_double()
bw=np.ascontiguousarray(bwd); fw=np.ascontiguousarray(fwd); yy=np.ascontiguousarray(y.astype(np.int32))
def step(nxt):
    _lib.check(lib.d2ft_engine_step_pipelined(m._h, _lib.ptr(px) if nxt else None, _lib.ptr(yy), _lib.ptr(bw), _lib.ptr(fw), _lib.ptr(cf), _lib.ptr(cb), _lib.ptr(capf), _lib.ptr(capo), C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9), C.byref(loss), None))
_lib.check(lib.d2ft_engine_prefetch(m._h, _lib.ptr(px), C.c_int(B)))
for i in range(3): step(True)
ts=[]
for i in range(10):
    t0=time.perf_counter(); step(True); ts.append((time.perf_counter()-t0)*1e3)
print("pipelined step ms", [round(t,3) for t in ts])
ms=C.c_double()
_lib.check(lib.d2ft_engine_bench_device(m._h, C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9), C.c_int(2), C.c_int(10), C.byref(ms), C.byref(loss)))
print("device ms/step", ms.value/10)
t0=time.perf_counter(); _lib.check(lib.d2ft_engine_step_resident(m._h, C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9))); t1=time.perf_counter()
_lib.check(lib.d2ft_engine_sync(m._h, C.byref(loss))); t2=time.perf_counter()
print("resident enqueue ms", (t1-t0)*1e3, "sync ms", (t2-t1)*1e3)
pc = np.zeros((4, K), np.int32); pc[0], pc[1], pc[2], pc[3] = 2, 3, capf, capo
for steps in (10, 30):
    ms_e2e = C.c_double()
    _lib.check(lib.d2ft_engine_bench_e2e(m._h, _lib.ptr(px), _lib.ptr(yy), _lib.ptr(bw), _lib.ptr(fw), _lib.ptr(pc[0]), _lib.ptr(pc[1]),
            _lib.ptr(pc[2]), _lib.ptr(pc[3]), C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9),
            C.c_int(1), C.c_int(steps), C.byref(ms_e2e), C.byref(loss)))
    print("bench_e2e ms/step", steps, ms_e2e.value / steps)
