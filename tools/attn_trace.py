"""Phase timeline of the attention kernels (experiment build with
-DD2FT_ATTN_TRACE, loaded through D2FT_B200_LIB): one ViT-B batch-64 step,
layer 6, per-CTA SM-clock stamps of the forward / backward kernels.
Prints per-event-code mean offsets (cycles from the CTA's first stamp) and
per-item durations."""
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2504_12471_b200 import _lib  # noqa: E402
from paper_2504_12471_b200 import engine as E  # noqa: E402
from paper_2504_12471_b200 import scheduler as S  # noqa: E402

B, K = 64, 144
x, y, bwd, fwd, capf, capo = bench.workload(B)
m = E.SubnetModel(E.VIT_B16, B)
m.stage(x, y, S.ScoreTable(K, B, fwd, bwd), S.CostModel(), S.Capacities(capf.tolist(), capo.tolist()))
lib = _lib.lib()
CT, EV = 16, 16 * 64
buf = np.zeros((CT, EV), np.uint64)
cnt = np.zeros(CT, np.int32)
for _ in range(3):
    m.step_resident()
m.sync()
for kind in (0, 1):
    lib.d2ft_debug_attn_trace(C.c_int(kind), _lib.ptr(buf), _lib.ptr(cnt))
m.step_resident()
m.sync()
for kind, name in ((0, "forward"), (1, "backward")):
    lib.d2ft_debug_attn_trace(C.c_int(kind), _lib.ptr(buf), _lib.ptr(cnt))
    print(f"=== {name}: events per CTA {cnt.tolist()}")
    rel = defaultdict(list)
    for b in range(CT):
        ev = [int(v) for v in buf[b] if int(v) != 0]
        if not ev:
            continue
        t0 = min(v & 0xFFFFFFFFFF for v in ev)
        rows = sorted(((v & 0xFFFFFFFFFF) - t0, (v >> 40) & 0xff, v >> 56, (v >> 48) & 0xff) for v in ev)
        if b < 3:
            print(f"-- CTA {b}")
            for t, w, code, item in rows:
                print(f"{t:8d}  warp {w:2d} code {code:3d} item {item}")
        for t, w, code, item in rows:
            rel[(code, item)].append(t)
    print("-- mean offset per (code, item) over CTAs")
    for k in sorted(rel, key=lambda k: (k[1], np.mean(rel[k]))):
        print(f"code {k[0]:3d} item {k[1]:2d}: {np.mean(rel[k]):9.0f}  (n={len(rel[k])})")
m.close()
