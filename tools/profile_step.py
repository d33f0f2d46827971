"""Short ViT-B/16 D2FT run for ncu captures: one warm-up step + N timed steps
on device-resident inputs (same workload as bench.py)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2504_12471_b200 import _lib  # noqa: E402
from paper_2504_12471_b200 import engine as E  # noqa: E402
from paper_2504_12471_b200 import scheduler as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
B = 64
K = 144
x, y, bwd, fwd, capf, capo = bench.workload(B)
m = E.SubnetModel(E.VIT_B16, B)
m.stage(x, y, S.ScoreTable(K, B, fwd, bwd), S.CostModel(), S.Capacities(capf.tolist(), capo.tolist()))
ms, loss = C.c_double(), C.c_double()
_lib.check(_lib.lib().d2ft_engine_bench_device(m._h, C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9),
                                               C.c_int(1), C.c_int(steps), C.byref(ms), C.byref(loss)))
print("ms/step", ms.value / steps, "loss", loss.value)
