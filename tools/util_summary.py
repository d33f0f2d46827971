"""Summarise an ncu --metrics CSV (tools/kernel_util.sh) per kernel name:
launches, mean duration, SM-active fraction, tensor-pipe utilisation, DRAM GB/s."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = None
acc = defaultdict(lambda: defaultdict(list))
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("d2ft_b200::", "")
    if "gemm_sm100_kernel<" in short:
        short = short.split("<")[1].split(",")[0]
    met, val = r[hdr.index("Metric Name")], r[hdr.index("Metric Value")]
    try:
        acc[short][met].append(float(val.replace(",", "")))
    except ValueError:
        pass
print(f"{'kernel':34s} {'n':>4s} {'us':>8s} {'sm_act':>7s} {'tensor%':>8s} {'dram GB/s':>10s}")
for k, m in sorted(acc.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    n = len(t)
    us = sum(t) / n / 1e3 if t and max(t) > 1e3 else sum(t) / max(n, 1)
    act = sum(m["sm__cycles_active.avg"]) / max(sum(m["sm__cycles_elapsed.avg"]), 1)
    tp = sum(m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]) / max(n, 1)
    byt = sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])
    gbs = byt / max(sum(t), 1)  # bytes / ns = GB/s if duration in ns
    print(f"{k[:34]:34s} {n:4d} {us:8.1f} {act:7.2f} {tp:8.1f} {gbs:10.0f}")
