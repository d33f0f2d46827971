"""Shared helpers for the step parity tests (tolerances stated here).

Tolerances (BASELINE.json north_star; bf16 operands, fp32 accumulation):
  * gradients / weight updates: normwise max relative error per tensor
        max|gpu - ref| / max|ref|  <= 1e-2
  * fp32-path outputs (loss, updated weights): relative error <= 1e-3
The reference's own element metric |a-b|/max(|a|,|b|,1e-6) (oracles.cpp:358-361)
is dominated by near-zero entries after bf16 rounding, so the per-tensor
normwise form is used and stated in DESIGN.md §5.
"""
import numpy as np

GRAD_TOL = 1e-2
FP32_TOL = 1e-3


def tensor_slices(L, H, d, ffn, T, C):
    dh, fs = d // H, ffn // H
    out = []
    off = 0

    def add(name, n):
        nonlocal off
        out.append((name, off, off + n))
        off += n

    add("w_embed", d * d)
    add("b_embed", d)
    add("pos", T * d)
    for l in range(L):
        for h in range(H):
            for nm, n in (("wq", d * dh), ("wk", d * dh), ("wv", d * dh), ("wo", dh * d), ("w1", d * fs), ("b1", fs),
                          ("w2", fs * d), ("b2", d // H)):
                add(f"b{l}h{h}.{nm}", n)
    add("w_cls", d * C)
    add("b_cls", C)
    return out


def normwise(a, b):
    den = np.max(np.abs(b))
    if den == 0.0:
        return float(np.max(np.abs(a)))
    return float(np.max(np.abs(a - b)) / den)


def compare_tensors(got, ref, slices, tol, skip_zero_ref=True):
    """Returns the list of (name, err) above tol."""
    bad = []
    for name, a, b in slices:
        r = ref[a:b]
        if skip_zero_ref and not np.any(r):
            if np.any(got[a:b]):
                bad.append((name, float(np.max(np.abs(got[a:b])))))
            continue
        e = normwise(got[a:b], r)
        if e > tol:
            bad.append((name, e))
    return bad


# Elementwise view beside the normwise one (reported): over
# the entries that carry the tensor (|ref| >= floor * max|ref|), the largest
# |gpu - ref| / |ref| and the reference's own metric
# |a - b| / max(|a|, |b|, 1e-6) (oracles.cpp:358-361).
ELEM_FLOOR = 1e-3


def elementwise(got, ref, floor=ELEM_FLOOR):
    m = float(np.max(np.abs(ref))) if ref.size else 0.0
    if m == 0.0:
        return 0.0, 0.0
    mask = np.abs(ref) >= floor * m
    g, r = got[mask], ref[mask]
    rel = np.abs(g - r) / np.abs(r)
    refm = np.abs(g - r) / np.maximum(np.maximum(np.abs(g), np.abs(r)), 1e-6)
    return float(rel.max()), float(refm.max())


def family(name):
    return name.split(".")[-1] if "." in name else name


def error_report(got, ref, slices):
    """Per tensor family (wq, wk, ..., w_embed, w_cls): the worst normwise and
    elementwise errors over all its tensors, plus the 99.9th percentile of the
    elementwise error over the family's carrying entries."""
    fam = {}
    for name, a, b in slices:
        r = ref[a:b]
        if not np.any(r):
            continue
        g = got[a:b]
        nw = normwise(g, r)
        el, refm = elementwise(g, r)
        m = np.max(np.abs(r))
        mask = np.abs(r) >= ELEM_FLOOR * m
        f = fam.setdefault(family(name), {"normwise": 0.0, "elementwise": 0.0, "ref_metric": 0.0, "_rel": []})
        f["normwise"] = max(f["normwise"], nw)
        f["elementwise"] = max(f["elementwise"], el)
        f["ref_metric"] = max(f["ref_metric"], refm)
        f["_rel"].append(np.abs(g[mask] - r[mask]) / np.abs(r[mask]))
    out = {}
    for k, f in fam.items():
        rel = np.concatenate(f.pop("_rel"))
        f["elementwise_p999"] = float(np.quantile(rel, 0.999))
        out[k] = {kk: float("%.3g" % v) for kk, v in f.items()}
    return out


def write_report(test, report):
    """Print the achieved errors and append them to gpurun_out/parity_report.jsonl
    (collected with the GPU run; summarised in profiles/)."""
    import json
    import os
    line = json.dumps({"test": test, **report})
    print(line)
    root = os.environ.get("GRAFT_REPO_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = os.path.join(root, "gpurun_out")
    try:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "parity_report.jsonl"), "a") as f:
            f.write(line + "\n")
    except OSError:
        pass
