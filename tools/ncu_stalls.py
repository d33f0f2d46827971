"""Summarise an ncu `--page source --csv --print-source sass` export: stall
reasons per SASS range (e.g. producer / MMA / epilogue regions of the GEMM).
usage: ncu_stalls.py export.csv [a:b[:name] ...]   (first kernel in the file)"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
out = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    out.append(r)
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
print(rows[0][1][:100], "instructions:", len(out))
ranges = [a.split(":") for a in sys.argv[2:]] or [["0", str(len(out)), "all"]]
for rg in ranges:
    a, b = int(rg[0]), int(rg[1])
    name = rg[2] if len(rg) > 2 else f"{a}:{b}"
    c = Counter()
    for r in out[a:b]:
        for i in cols:
            if r[i].isdigit():
                c[hdr[i][6:]] += int(r[i])
    tot = sum(c.values())
    print(f"{name:10s} {tot:6d}  " + "  ".join(f"{k}={v}" for k, v in c.most_common(8)))
