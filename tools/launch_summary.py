"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel kind."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def kind(name):
    m = re.search(r"(G1|G3|G4|G5|G7|G8|EmbedFwd|EmbedW|DenseProb|PlanesProb|TokenKProb)<", name)
    if m:
        return m.group(1)
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(anonymous namespace\)::|d2ft_b200::|<unnamed>::|unnamed>::", "", name)
    return name.split("(")[0]


def summarise(path, steps=1):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in load(path):
        v = float(d["Metric Value"])
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
        k = kind(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(t for _, t in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:40s} {c:5d} launches {t / steps:10.1f} us/step {t / c:9.1f} us/launch {100 * t / tot:5.1f}%")
    out.append(f"total {tot / steps:.1f} us/step")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1))
