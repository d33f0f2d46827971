"""Host-side mirror of the reference scheduler API (core/include/d2ft/scheduler.hpp).

Same names, argument meaning and error behaviour as the reference; the
arithmetic (every DP, merge and compaction) runs in the sm_100a kernels of
libd2ft_b200.so through the C-ABI (include/d2ft_b200.h).  `threads` arguments
are accepted for signature compatibility and ignored: results never depend on
them (threading.hpp:12-13), exactly like the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import Error, check, f64, i32, lib, ptr, u8

FULL, FORWARD_ONLY, SHORTCUT = 1, 2, 3  # OperationKind, model.hpp:35-39


@dataclass
class CostModel:
    """scheduler.hpp:23-55."""
    forward_cost: int = 2
    backward_cost: int = 3
    comm_forward: int = 1
    comm_backward: int = 1
    forward_cost_per_device: List[int] = field(default_factory=list)
    backward_cost_per_device: List[int] = field(default_factory=list)

    def cf(self, device: int) -> int:
        return self.forward_cost_per_device[device] if self.forward_cost_per_device else self.forward_cost

    def cb(self, device: int) -> int:
        return self.backward_cost_per_device[device] if self.backward_cost_per_device else self.backward_cost

    def full_cost(self, device: int) -> int:
        return self.cf(device) + self.cb(device)

    def op_cost(self, device: int, code: int) -> int:  # scheduler.cpp:15-22
        if code == 1:
            return self.full_cost(device)
        if code == 2:
            return self.cf(device)
        if code == 3:
            return 0
        raise Error(2, f"invalid schedule code {code}")

    def validate(self) -> None:  # scheduler.cpp:24-35
        if self.forward_cost < 0 or self.backward_cost < 0:
            raise Error(1, "cost model: costs must be nonnegative integers")
        if any(v < 0 for v in self.forward_cost_per_device):
            raise Error(1, "cost model: per-device forward cost negative")
        if any(v < 0 for v in self.backward_cost_per_device):
            raise Error(1, "cost model: per-device backward cost negative")
        if self.comm_forward != self.comm_backward:
            raise Error(1, "cost model: forward/backward tensors have equal size, comm units must match")

    def row_arrays(self, devices: int):
        cf = np.array([self.cf(k) for k in range(devices)], np.int32)
        cb = np.array([self.cb(k) for k in range(devices)], np.int32)
        return cf, cb

    @staticmethod
    def full_finetune() -> "CostModel":
        return CostModel()

    @staticmethod
    def lora_finetune() -> "CostModel":
        return CostModel(forward_cost=7, backward_cost=1)


@dataclass
class Capacities:
    """scheduler.hpp:60-66."""
    full: List[int] = field(default_factory=list)
    fwd: List[int] = field(default_factory=list)

    def devices(self) -> int:
        return len(self.full)

    def validate(self) -> None:  # scheduler.cpp:37-43
        if len(self.full) != len(self.fwd):
            raise Error(2, "capacities: pool sizes differ")
        if any(v < 0 for v in self.full):
            raise Error(2, "capacities: negative full capacity")
        if any(v < 0 for v in self.fwd):
            raise Error(2, "capacities: negative forward capacity")


@dataclass
class BudgetOverride:
    device: int = 0
    n_full: int = 0
    n_fwd: int = 0


@dataclass
class BudgetSpec:
    """scheduler.hpp:70-83."""
    n_full: int = 2
    n_fwd: int = 2
    overrides: List[BudgetOverride] = field(default_factory=list)

    def n_full_for(self, device: int) -> int:
        for o in self.overrides:
            if o.device == device:
                return o.n_full
        return self.n_full

    def n_fwd_for(self, device: int) -> int:
        for o in self.overrides:
            if o.device == device:
                return o.n_fwd
        return self.n_fwd

    def validate(self, micro_batches: int) -> None:  # scheduler.cpp:57-68
        def check_pair(nf, no):
            if nf < 0 or no < 0:
                raise Error(2, "budget: counts must be nonnegative")
            if nf + no > micro_batches:
                raise Error(2, f"budget: n_full + n_fwd exceeds micro-batches per batch "
                               f"({nf}+{no} > {micro_batches})")
        check_pair(self.n_full, self.n_fwd)
        for o in self.overrides:
            check_pair(o.n_full, o.n_fwd)


@dataclass
class ScoreTable:
    """scoring.hpp:30-41: K x N forward (A^po) and backward (A^pf) scores."""
    subnets: int
    micro_batches: int
    forward: np.ndarray
    backward: np.ndarray
    fwd_metric: str = "fisher_information"
    bwd_metric: str = "weight_magnitude"

    def __post_init__(self):
        self.forward = f64(self.forward).reshape(self.subnets, self.micro_batches) if np.size(self.forward) \
            else np.zeros((self.subnets, self.micro_batches))
        self.backward = f64(self.backward).reshape(self.subnets, self.micro_batches) if np.size(self.backward) \
            else np.zeros((self.subnets, self.micro_batches))

    def fwd(self, k, i):
        return float(self.forward[k, i])

    def bwd(self, k, i):
        return float(self.backward[k, i])

    def validate(self) -> None:  # scoring.cpp:30-47
        for side in (self.forward, self.backward):
            if not np.all(np.isfinite(side)):
                raise Error(5, "score table contains non-finite entries")
            if np.any(side < 0.0):
                raise Error(5, "score table contains negative entries")


class ScheduleTable:
    """scheduler.hpp:86-116: K x N codes, row-major by device, default 3."""

    def __init__(self, devices: int = 0, micro_batches: int = 0, codes: Optional[np.ndarray] = None):
        self.devices = devices
        self.micro_batches = micro_batches
        if codes is None:
            self.codes = np.full((devices, micro_batches), SHORTCUT, np.uint8)
        else:
            self.codes = u8(codes).reshape(devices, micro_batches)

    def code(self, k, i) -> int:
        return int(self.codes[k, i])

    def set_code(self, k, i, c) -> None:
        self.codes[k, i] = c

    def op(self, k, i) -> int:
        return self.code(k, i)

    def column(self, i) -> np.ndarray:
        return self.codes[:, i].copy()

    def row_counts(self, k):
        row = self.codes[k]
        return dict(n_full=int((row == 1).sum()), n_fwd=int((row == 2).sum()), n_shortcut=int((row == 3).sum()))

    def validate(self) -> None:
        if self.codes.shape != (self.devices, self.micro_batches):
            raise Error(2, "schedule table: dimension mismatch")
        if np.any((self.codes < 1) | (self.codes > 3)):
            raise Error(2, "schedule table: code out of range")

    def __eq__(self, other) -> bool:
        return (isinstance(other, ScheduleTable) and self.devices == other.devices
                and self.micro_batches == other.micro_batches and np.array_equal(self.codes, other.codes))

    def __repr__(self):
        return f"ScheduleTable({self.devices}x{self.micro_batches})"


@dataclass
class ScalerConfig:
    """scheduler.hpp:118-127."""
    mode: str = "constant"  # "max" | "min" | "constant"
    lam: float = 1.0

    def validate(self) -> None:
        if self.mode == "constant" and not (self.lam > 0.0):
            raise Error(1, "scaler: constant lambda must be > 0")

    @staticmethod
    def max() -> "ScalerConfig":
        return ScalerConfig("max", 1.0)

    @staticmethod
    def min() -> "ScalerConfig":
        return ScalerConfig("min", 1.0)

    @staticmethod
    def constant(l: float) -> "ScalerConfig":
        return ScalerConfig("constant", l)


@dataclass
class CostTables:
    w_full: np.ndarray
    w_fwd: np.ndarray


@dataclass
class DpResult:
    selection: np.ndarray  # K x N uint8
    objective: np.ndarray  # K fp64


@dataclass
class ScalerResult:
    table: ScheduleTable
    lambda_used: float = 1.0
    fell_back: bool = False


def build_cost_tables(cost_model: CostModel, devices: int, micro_batches: int) -> CostTables:
    """scheduler.cpp:104-119 (host bookkeeping: constant rows)."""
    if devices < 1 or micro_batches < 1:
        raise Error(2, "cost tables require at least one device and one micro-batch")
    cost_model.validate()
    cf, cb = cost_model.row_arrays(devices)
    return CostTables(np.repeat((cf + cb)[:, None], micro_batches, 1).astype(np.int32),
                      np.repeat(cf[:, None], micro_batches, 1).astype(np.int32))


def dp_search(scores, weights, capacities, threads: int = 1) -> DpResult:
    """scheduler.cpp:121-189 on the GPU (count-compressed kernel for constant rows)."""
    s = f64(scores)
    if s.ndim == 1:
        s = s.reshape(1, -1)
    K = s.shape[0]
    N = s.shape[1] if K else 0
    w = i32(weights).reshape(K, N)
    c = i32(capacities)
    if c.shape != (K,):
        raise Error(2, "dp_search: scores, weights and capacities must agree on device count")
    sel = np.zeros((K, N), np.uint8)
    obj = np.zeros(K, np.float64)
    check(lib().d2ft_dp_search(ptr(s), ptr(w), ptr(c), C.c_int(K), C.c_int(N), ptr(sel), ptr(obj)))
    return DpResult(sel, obj)


def merge_selections(full_selection, fwd_selection) -> ScheduleTable:
    """scheduler.cpp:191-220 on the GPU."""
    a = u8(full_selection)
    b = u8(fwd_selection)
    if a.shape[0] != b.shape[0]:
        raise Error(2, "merge_selections: device counts differ")
    if a.shape != b.shape:
        raise Error(2, "merge_selections: ragged selection rows")
    K, N = a.shape
    codes = np.zeros((K, N), np.uint8)
    check(lib().d2ft_merge_selections(ptr(a), ptr(b), C.c_int(K), C.c_int(N), ptr(codes)))
    return ScheduleTable(K, N, codes)


def knapsack_schedule(scores: ScoreTable, cost_model: CostModel, capacities: Capacities,
                      threads: int = 1) -> ScheduleTable:
    """scheduler.cpp:222-236 on the GPU (one fused launch)."""
    scores.validate()
    capacities.validate()
    K, N = scores.subnets, scores.micro_batches
    if capacities.devices() != K:
        raise Error(2, "knapsack_schedule: capacities device count mismatch")
    if K < 1 or N < 1:
        raise Error(2, "cost tables require at least one device and one micro-batch")
    cost_model.validate()
    cf, cb = cost_model.row_arrays(K)
    codes = np.zeros((K, N), np.uint8)
    check(lib().d2ft_knapsack_schedule(ptr(scores.backward), ptr(scores.forward), ptr(cf), ptr(cb),
                                       ptr(i32(capacities.full)), ptr(i32(capacities.fwd)), C.c_int(K),
                                       C.c_int(N), ptr(codes)))
    return ScheduleTable(K, N, codes)


def scaler_schedule(scores: ScoreTable, cost_model: CostModel, total_capacity: Sequence[int],
                    scaler: ScalerConfig, threads: int = 1) -> ScalerResult:
    """scheduler.cpp:321-426 on the GPU."""
    scores.validate()
    scaler.validate()
    cost_model.validate()
    K, N = scores.subnets, scores.micro_batches
    tc = i32(total_capacity)
    if tc.shape != (K,):
        raise Error(2, "scaler_schedule: capacity count mismatch")
    cf, cb = cost_model.row_arrays(K)
    mode = {"max": 0, "min": 1, "constant": 2}[scaler.mode]
    codes = np.zeros((K, N), np.uint8)
    lu = C.c_double()
    fb = C.c_int()
    check(lib().d2ft_scaler_schedule(ptr(scores.backward), ptr(scores.forward), ptr(cf), ptr(cb), ptr(tc),
                                     C.c_int(K), C.c_int(N), C.c_int(mode), C.c_double(scaler.lam), ptr(codes),
                                     C.byref(lu), C.byref(fb)))
    if fb.value:
        import sys
        print("[d2ft] scaler: degenerate all-zero scores, falling back to lambda=1", file=sys.stderr)
    return ScalerResult(ScheduleTable(K, N, codes), lu.value, bool(fb.value))


def capacities_from_budget(budget: BudgetSpec, cost_model: CostModel, devices: int,
                           micro_batches: int) -> Capacities:
    """scheduler.cpp:428-440."""
    budget.validate(micro_batches)
    cost_model.validate()
    return Capacities([budget.n_full_for(k) * cost_model.full_cost(k) for k in range(devices)],
                      [budget.n_fwd_for(k) * cost_model.cf(k) for k in range(devices)])


def row_cost_units(table: ScheduleTable, cost_model: CostModel, device: int) -> int:
    """scheduler.cpp:442-446."""
    return sum(cost_model.op_cost(device, int(c)) for c in table.codes[device])


@dataclass
class SharedBudgetReport:
    devices: list
    violations: list

    def ok(self) -> bool:
        return not self.violations


def check_shared_budget(table: ScheduleTable, cost_model: CostModel, capacities: Capacities) -> SharedBudgetReport:
    """scheduler.cpp:448-465."""
    table.validate()
    capacities.validate()
    if capacities.devices() != table.devices:
        raise Error(2, "check_shared_budget: capacities device count mismatch")
    devs, viol = [], []
    for k in range(table.devices):
        units = row_cost_units(table, cost_model, k)
        limit = capacities.full[k] + capacities.fwd[k]
        if units > limit:
            viol.append(k)
        devs.append(dict(device=k, cost_units=units, limit=limit))
    return SharedBudgetReport(devs, viol)


def brute_force_schedule(scores: ScoreTable, cost_model: CostModel, capacities: Capacities,
                         threads: int = 1) -> ScheduleTable:
    """scheduler.cpp:248-302 on the GPU (3^N enumeration per row, N <= 14)."""
    scores.validate()
    capacities.validate()
    K, N = scores.subnets, scores.micro_batches
    if capacities.devices() != K:
        raise Error(2, "brute_force_schedule: capacities device count mismatch")
    cf, cb = cost_model.row_arrays(K)
    codes = np.zeros((K, N), np.uint8)
    check(lib().d2ft_brute_force_schedule(ptr(scores.backward), ptr(scores.forward), ptr(cf), ptr(cb),
                                          ptr(i32(capacities.full)), ptr(i32(capacities.fwd)), C.c_int(K),
                                          C.c_int(N), ptr(codes)))
    return ScheduleTable(K, N, codes)


def schedule_objective(table: ScheduleTable, scores: ScoreTable) -> np.ndarray:
    """scheduler.cpp:304-319 (per-row realised value; host accounting)."""
    if table.devices != scores.subnets or table.micro_batches != scores.micro_batches:
        raise Error(2, "schedule_objective: table/score dimensions differ")
    out = np.zeros(table.devices)
    for k in range(table.devices):
        for i in range(table.micro_batches):
            c = table.codes[k, i]
            if c == 1:
                out[k] += scores.backward[k, i] + scores.forward[k, i]
            elif c == 2:
                out[k] += scores.forward[k, i]
    return out


@dataclass
class CompactLists:
    fwd_idx: np.ndarray
    fwd_cnt: np.ndarray
    full_idx: np.ndarray
    full_cnt: np.ndarray
    act_heads: np.ndarray
    act_cnt: np.ndarray
    full_heads: np.ndarray
    full_hcnt: np.ndarray


def compact(table: ScheduleTable, heads_per_block: int) -> CompactLists:
    """Warp-ballot compaction of a code table into per-row micro-batch lists and
    per-(micro-batch, block) head lists (the implicit skips of model.cpp:431-436,
    455-466, 499-508).  Unused tail entries are -1."""
    table.validate()
    K, N, H = table.devices, table.micro_batches, heads_per_block
    if H < 1 or K % H:
        raise Error(2, "compact: K must be a multiple of heads_per_block")
    L = K // H
    out = CompactLists(np.full((K, N), -1, np.int32), np.zeros(K, np.int32), np.full((K, N), -1, np.int32),
                       np.zeros(K, np.int32), np.full((N * L, H), -1, np.int32), np.zeros(N * L, np.int32),
                       np.full((N * L, H), -1, np.int32), np.zeros(N * L, np.int32))
    check(lib().d2ft_compact(ptr(table.codes), C.c_int(K), C.c_int(N), C.c_int(H), ptr(out.fwd_idx),
                             ptr(out.fwd_cnt), ptr(out.full_idx), ptr(out.full_cnt), ptr(out.act_heads),
                             ptr(out.act_cnt), ptr(out.full_heads), ptr(out.full_hcnt)))
    return out


class Scheduler:
    """Reusable device context for repeated schedules of one shape (the step
    engine's and bench.py's path): pre-sized buffers, one fused launch."""

    def __init__(self, K: int, N: int, H: int, max_cols: int):
        self.K, self.N, self.H = K, N, H
        self._h = C.c_void_p()
        check(lib().d2ft_sched_create(C.c_int(K), C.c_int(N), C.c_int(H), C.c_int(max_cols), C.byref(self._h)))

    def close(self):
        if self._h:
            lib().d2ft_sched_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, bwd, fwd, cf, cb, cap_full, cap_fwd) -> np.ndarray:
        codes = np.zeros((self.K, self.N), np.uint8)
        check(lib().d2ft_sched_run_host(self._h, ptr(f64(bwd)), ptr(f64(fwd)), ptr(i32(cf, self.K)),
                                        ptr(i32(cb, self.K)), ptr(i32(cap_full)), ptr(i32(cap_fwd)), ptr(codes)))
        return codes

    def bench(self, bwd, fwd, cf, cb, cap_full, cap_fwd, warmup=3, iters=20):
        codes = np.zeros((self.K, self.N), np.uint8)
        us_dev = C.c_double()
        us_e2e = C.c_double()
        check(lib().d2ft_sched_bench(self._h, ptr(f64(bwd)), ptr(f64(fwd)), ptr(i32(cf, self.K)),
                                     ptr(i32(cb, self.K)), ptr(i32(cap_full)), ptr(i32(cap_fwd)), C.c_int(warmup),
                                     C.c_int(iters), C.byref(us_dev), C.byref(us_e2e), ptr(codes)))
        return us_dev.value, us_e2e.value, codes


def max_cols_for(cf, cb, cap_full, cap_fwd, N) -> int:
    """Largest count-compressed DP width over both pools (see csrc/sched.cu)."""
    def cols(wt, cap):
        return 1 if wt == 0 else min(cap // wt, N) + 1
    mc = 1
    for a, b, f, o in zip(np.broadcast_to(cf, len(cap_full)), np.broadcast_to(cb, len(cap_full)), cap_full, cap_fwd):
        mc = max(mc, cols(int(a) + int(b), int(f)), cols(int(a), int(o)))
    return mc
