"""Per-phase device times of the bench workload (ViT-B/16, batch 64) for the
library named by D2FT_B200_LIB (default: the in-tree build).  Used to compare
experiment builds (tools/build_variants.sh); prints one JSON line."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2504_12471_b200 import _lib  # noqa: E402
from paper_2504_12471_b200 import engine as E  # noqa: E402
from paper_2504_12471_b200 import scheduler as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
B = 64
K = 144
x, y, bwd, fwd, capf, capo = bench.workload(B)
m = E.SubnetModel(E.VIT_B16, B)
m.stage(x, y, S.ScoreTable(K, B, fwd, bwd), S.CostModel(), S.Capacities(capf.tolist(), capo.tolist()))
ms, loss = C.c_double(), C.c_double()
lib = _lib.lib()
_lib.check(lib.d2ft_engine_bench_device(m._h, C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9),
                                        C.c_int(3), C.c_int(steps), C.byref(ms), C.byref(loss)))
plain = ms.value / steps
m.set_profiling(True)
_lib.check(lib.d2ft_engine_bench_device(m._h, C.c_int(B), C.c_int(1), C.c_double(0.05), C.c_double(0.9),
                                        C.c_int(1), C.c_int(steps), C.byref(ms), C.byref(loss)))
ph = m.phase_ms()
print(json.dumps({"lib": os.environ.get("D2FT_B200_LIB", "in-tree"), "ms_per_step": round(plain, 4),
                  "phase_ms": {k: round(v, 3) for k, v in ph.items()}}))
