"""Scheduler latency on the GPU at the bench's shapes (bench.sched_shapes):
device time of the fused schedule launch and the host round trip."""
import sys, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
import bench
from paper_2504_12471_b200 import _lib, scheduler as S
lib = _lib.lib()
for tag, K, N, cf_, co_ in bench.sched_shapes():
    u = np.empty(2 * K * N); _lib.check(lib.d2ft_uniform_stream(C.c_uint64(1), C.c_uint64(0), C.c_int(u.size), _lib.ptr(u)))
    u = u.reshape(K, N, 2) * 10.0
    H = 16 if K == 384 else 12
    sc = S.Scheduler(K, N, H, S.max_cols_for(2, 3, cf_, co_, N))
    d, e, _ = sc.bench(u[:, :, 1], u[:, :, 0], 2, 3, cf_, co_, warmup=3, iters=20)
    print(tag, "us_device", round(d, 2), "us_e2e", round(e, 2), flush=True)
    sc.close()
