"""Top SASS instructions by warp-stall samples from an ncu source export
(`ncu -i X.ncu-rep --page source --csv --print-source sass`), plus every
mbarrier wait with the samples of the spin branch after it.
usage: ncu_src.py export.csv [top_n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 3]
iS = hdr.index("Warp Stall Sampling (All Samples)")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
smp = lambda r: int(r[iS] or 0)
print(rows[0][1][:120], "| samples", sum(smp(r) for r in data))
for r in sorted(data, key=lambda r: -smp(r))[:top_n]:
    st = sorted([(int(r[i]), hdr[i][6:]) for i in cols if r[i].isdigit() and int(r[i]) > 0], reverse=True)[:3]
    print(f"{r[0][-5:]} {smp(r):5d}  {r[1][:70]:70s} {st}")
print("--- waits (spin samples)")
for i, r in enumerate(data):
    if "TRYWAIT" in r[1]:
        print(f"{r[0][-5:]} {smp(r) + smp(data[i + 1]):5d}  {r[1][:80]}")
