"""Markdown view of a parity report (tests/test_parity_bench_gpu.py writes
gpurun_out/parity_report.jsonl; profiles/r2_parity_report.jsonl collects the
round's runs).  usage: parity_report_md.py report.jsonl > report.md"""
import json
import sys

print("# r2 parity report (tests/test_parity_bench_gpu.py on one B200)\n")
print("Per tensor family, worst over its tensors. normwise = max|gpu-ref|/max|ref| (the asserted bar, 1e-2);")
print("elementwise = max |gpu-ref|/|ref| over entries with |ref| >= 1e-3 max|ref|; ref_metric = the reference's")
print("|a-b|/max(|a|,|b|,1e-6) over the same entries; p999 = 99.9th percentile of elementwise.\n")
for line in open(sys.argv[1]):
    r = json.loads(line)
    print(f"## {r['test']}")
    for k in ("loss_rel", "params_normwise", "cells"):
        if k in r:
            print(f"{k}: {r[k]}")
    for part in ("update", "velocity", "grad"):
        if part not in r:
            continue
        print(f"\n{part}:\n")
        print("| family | normwise | elementwise | ref_metric | p99.9 |")
        print("|---|---|---|---|---|")
        for fam, e in r[part].items():
            print(f"| {fam} | {e['normwise']:.3g} | {e['elementwise']:.3g} | {e['ref_metric']:.3g} | "
                  f"{e['elementwise_p999']:.3g} |")
    print()
