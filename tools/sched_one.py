"""One shape of the scheduler sweep (for ncu): python tools/sched_one.py r iters"""
import sys, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2504_12471_b200 import _lib, scheduler as S
lib = _lib.lib()
r, iters = float(sys.argv[1]), int(sys.argv[2])
K, N = 144, 1024
u = np.empty(2 * K * N); _lib.check(lib.d2ft_uniform_stream(C.c_uint64(1), C.c_uint64(0), C.c_int(u.size), _lib.ptr(u)))
u = u.reshape(K, N, 2) * 10.0
nb = int(r * N)
cf_, co_ = np.full(K, nb * 5, np.int32), np.full(K, nb * 2, np.int32)
sc = S.Scheduler(K, N, 12, S.max_cols_for(2, 3, cf_, co_, N))
d, e, _ = sc.bench(u[:, :, 1], u[:, :, 0], 2, 3, cf_, co_, warmup=1, iters=iters)
print(r, "us_device", round(d, 2))
