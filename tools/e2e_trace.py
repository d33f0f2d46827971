"""Per-step host enqueue / sync split of the e2e Dataset path (D2FT_E2E_TRACE)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["D2FT_E2E_TRACE"] = "1"
import bench
from paper_2504_12471_b200 import _lib, engine as E
lib = _lib.lib()
B, K = 64, 144
x, y, bwd, fwd, capf, capo = bench.workload(B)
m = E.SubnetModel(E.VIT_B16, B)
n_units = 4 * B
dset = E.make_synthetic_dataset_f64(n_units, bench.NCLS, bench.D, bench.T, 0.5, 7)
uu = np.empty(2 * K * n_units)
_lib.check(lib.d2ft_uniform_stream(C.c_uint64(1), C.c_uint64(0), C.c_int(uu.size), _lib.ptr(uu)))
uu = uu.reshape(K, n_units, 2) * 10.0
tfwd, tbwd = np.ascontiguousarray(uu[:, :, 0]), np.ascontiguousarray(uu[:, :, 1])
steps = 8
order = np.ascontiguousarray(np.concatenate([np.random.default_rng(3).permutation(n_units) for _ in range(3)])[:(steps + 2) * B], np.int32)
pc = np.zeros((4, K), np.int32); pc[0], pc[1], pc[2], pc[3] = 2, 3, capf, capo
ms, loss = C.c_double(), C.c_double()
_lib.check(lib.d2ft_engine_bench_e2e_units(m._h, dset.handle(), _lib.ptr(order), C.c_int(B), C.c_int(1), _lib.ptr(tbwd),
           _lib.ptr(tfwd), C.c_int(n_units), _lib.ptr(pc[0]), _lib.ptr(pc[1]), _lib.ptr(pc[2]), _lib.ptr(pc[3]),
           C.c_double(0.05), C.c_double(0.9), C.c_int(2), C.c_int(steps), C.byref(ms), C.byref(loss)))
print("ms/step", ms.value / steps)
