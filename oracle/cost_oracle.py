"""ORACLE / TEST INFRASTRUCTURE ONLY — the checker for the GPU schedule
metrics (csrc/metrics.cu), never called by the product.

Pure-Python restatement of the reference's cost accounting and batch
simulator, /root/reference/proj/core/src/cost_sim.cpp.  Python floats are
IEEE doubles evaluated without FMA, in the reference's order, so the results
are bit-identical to the reference built for baseline x86-64.  Pinned against
the reference's own known answers (tests/test_cost_sim.cpp) in
tests/test_oracle_pins.py and against the compiled reference (oracle/_ref)
where it exists."""
from __future__ import annotations

import math

import numpy as np

# default_timing_table (cost_sim.cpp:9-13): (count, full_ms, fwd_ms)
DEFAULT_TIMING = [(1, 2.01, 0.86), (2, 2.20, 1.01), (3, 2.27, 1.05), (4, 2.74, 1.20), (5, 3.16, 1.48)]


def time_ms(table, count: int, full: bool) -> float:
    """DeviceProfile::time_ms (cost_sim.cpp:40-69)."""
    if count < 0:
        raise ValueError("negative micro-batch count")
    if count == 0:
        return 0.0
    val = (lambda e: e[1]) if full else (lambda e: e[2])
    for e in table:
        if e[0] == count:
            return val(e)
    lo_count, lo_val = 0, 0.0
    for e in table:
        if e[0] < count:
            lo_count, lo_val = e[0], val(e)
        else:
            slope = (val(e) - lo_val) / float(e[0] - lo_count)
            return lo_val + slope * float(count - lo_count)
    last = table[-1]
    prev_count, prev_val = (table[-2][0], val(table[-2])) if len(table) >= 2 else (0, 0.0)
    slope = (val(last) - prev_val) / float(last[0] - prev_count)
    return val(last) + slope * float(count - last[0])


def _row_units(codes: np.ndarray, cf, cb, k: int) -> int:
    """row_cost_units (scheduler.cpp:442-446)."""
    row = codes[k]
    return int((row == 1).sum()) * (cf[k] + cb[k]) + int((row == 2).sum()) * cf[k]


def _pop_var(loads) -> float:
    mean = 0.0
    for v in loads:
        mean += v
    mean /= len(loads)
    var = 0.0
    for v in loads:
        var += (v - mean) * (v - mean)
    return var / len(loads)


def compute_cost_fraction(codes, cf, cb) -> float:
    """cost_sim.cpp:71-81."""
    K, N = codes.shape
    used = sum(_row_units(codes, cf, cb, k) for k in range(K))
    total = sum(N * (cf[k] + cb[k]) for k in range(K))
    return 0.0 if total == 0 else float(used) / float(total)


def comm_cost_fraction(codes) -> float:
    """cost_sim.cpp:83-93 (sequential 1.0 / 0.5 sum: exact)."""
    used = 0.0
    for c in codes.reshape(-1):
        if c == 1:
            used += 1.0
        elif c == 2:
            used += 0.5
    return 0.0 if codes.size == 0 else used / float(codes.size)


def workload_variance(codes, cf, cb) -> float:
    """cost_sim.cpp:95-107: variance over rows of load / full load."""
    K, N = codes.shape
    if K == 0:
        return 0.0
    loads = []
    for k in range(K):
        full_load = float(N) * (cf[k] + cb[k])
        loads.append(_row_units(codes, cf, cb, k) / full_load if full_load > 0.0 else 0.0)
    return _pop_var(loads)


def simulate_batch(codes, cf, cb, memory_units, tables, caps=None, busy_ms=None):
    """cost_sim.cpp:109-172.  tables[p] = [(count, full_ms, fwd_ms), ...];
    busy_ms (measured per-device busy time) replaces the tables when given.
    Returns (compute, comm, variance, makespan, residual, per_device_busy)."""
    K, N = codes.shape
    if sum(memory_units) != K:
        raise ValueError("profiles host a different number of rows")
    compute = compute_cost_fraction(codes, cf, cb)
    comm = comm_cost_fraction(codes)
    loads, busy_out = [], []
    makespan, residual_sq, row = 0.0, 0.0, 0
    for p, mu in enumerate(memory_units):
        n_full = n_fwd = units = full_units = limit = 0
        for _ in range(mu):
            n_full += int((codes[row] == 1).sum())
            n_fwd += int((codes[row] == 2).sum())
            units += _row_units(codes, cf, cb, row)
            full_units += N * (cf[row] + cb[row])
            if caps is not None:
                limit += int(caps[0][row]) + int(caps[1][row])
            row += 1
        busy = float(busy_ms[p]) if busy_ms is not None else (
            time_ms(tables[p], n_full, True) + time_ms(tables[p], n_fwd, False))
        busy_out.append(busy)
        makespan = max(makespan, busy)
        loads.append(float(units) / float(full_units) if full_units > 0 else 0.0)
        if caps is not None:
            diff = float(units) - float(limit)
            residual_sq += diff * diff
    return compute, comm, _pop_var(loads), makespan, math.sqrt(residual_sq), busy_out
