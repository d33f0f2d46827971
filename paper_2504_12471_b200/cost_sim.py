"""Host mirror of the reference's cost accounting and device simulator,
core/include/d2ft/cost_sim.hpp (same names, argument meaning and errors).

The metrics run as one CUDA kernel over the code table
(csrc/metrics.cu, d2ft_schedule_metrics): bit-identical to the reference.
`simulate_batch(..., busy_ms=...)` replaces the calibrated timing table with
MEASURED per-device busy times (e.g. the head partition's per-rank busy
time from the step), which is what the simulation stands in for on real
hardware.  There is no CPU fallback: without the library these fail loudly."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional, Sequence

import numpy as np

from ._lib import Error, check, f64, i32, lib, ptr, u8
from .scheduler import BudgetOverride, BudgetSpec, Capacities, CostModel, ScheduleTable


@dataclass
class TimingEntry:
    """cost_sim.hpp:18-22."""
    count: int = 0
    full_ms: float = 0.0
    fwd_ms: float = 0.0


def default_timing_table() -> List[TimingEntry]:
    """cost_sim.cpp:10-14 (the paper's calibrated unit timings)."""
    return [TimingEntry(1, 2.01, 0.86), TimingEntry(2, 2.20, 1.01), TimingEntry(3, 2.27, 1.05),
            TimingEntry(4, 2.74, 1.20), TimingEntry(5, 3.16, 1.48)]


class Speed(Enum):
    Slow = 0
    Fast = 1


@dataclass
class DeviceProfile:
    """cost_sim.hpp:27-41."""
    device_id: int = 0
    memory_units: int = 1
    speed_class: Speed = Speed.Slow
    timing_table: List[TimingEntry] = field(default_factory=list)

    @staticmethod
    def standard(i: int) -> "DeviceProfile":  # cost_sim.cpp:16-21
        return DeviceProfile(device_id=i, timing_table=default_timing_table())

    def validate(self) -> None:  # cost_sim.cpp:23-36
        if self.memory_units < 1:
            raise Error(2, "device profile: memory_units must be >= 1")
        if not self.timing_table:
            raise Error(2, "device profile: empty timing table")
        prev = None
        for e in self.timing_table:
            if e.count < 1 or e.full_ms < 0.0 or e.fwd_ms < 0.0:
                raise Error(2, "device profile: invalid timing entry")
            if prev is not None and (e.count <= prev.count or e.full_ms < prev.full_ms or e.fwd_ms < prev.fwd_ms):
                raise Error(2, "device profile: timing table must be monotone nondecreasing")
            prev = e

    def _arrays(self):
        t = self.timing_table
        return (i32([e.count for e in t]), f64([e.full_ms for e in t]), f64([e.fwd_ms for e in t]))

    def time_ms(self, count: int, full: bool) -> float:  # cost_sim.cpp:38-69 (d2ft_device_time_ms)
        if count < 0:
            raise Error(2, "device profile: negative micro-batch count")
        cnt, fu, fw = self._arrays()
        out = C.c_double()
        check(lib().d2ft_device_time_ms(ptr(cnt), ptr(fu), ptr(fw), C.c_int(len(cnt)), C.c_int(count),
                                        C.c_int(1 if full else 0), C.byref(out)))
        return out.value


@dataclass
class BatchMetrics:
    """cost_sim.hpp:43-50 (+ row_workload_variance = workload_variance())."""
    compute_fraction: float = 0.0
    comm_fraction: float = 0.0
    workload_variance: float = 0.0
    makespan_ms: float = 0.0
    per_device_busy_ms: List[float] = field(default_factory=list)
    imbalance_residual: float = 0.0
    row_workload_variance: float = 0.0
    row_counts: Optional[np.ndarray] = None  # K x 3 (n_full, n_fwd, n_shortcut)


class _CMetrics(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("compute_fraction", "comm_fraction", "workload_variance", "makespan_ms",
                                          "imbalance_residual", "row_workload_variance")]


def _metrics(schedule: ScheduleTable, cost_model: CostModel, profiles: Sequence[DeviceProfile] = (),
             capacities: Optional[Capacities] = None, busy_ms: Optional[Sequence[float]] = None) -> BatchMetrics:
    K, N = schedule.devices, schedule.micro_batches
    codes = u8(schedule.codes).reshape(-1)
    if codes.size != K * N:
        raise Error(2, "schedule table: dimension mismatch")
    cost_model.validate()
    cf, cb = cost_model.row_arrays(K)
    n_dev = len(profiles)
    mu = i32([p.memory_units for p in profiles]) if n_dev else i32([0])
    toff = [0]
    cnt, fu, fw = [], [], []
    for p in profiles:
        cnt += [e.count for e in p.timing_table]
        fu += [e.full_ms for e in p.timing_table]
        fw += [e.fwd_ms for e in p.timing_table]
        toff.append(len(cnt))
    toff, cnt, fu, fw = i32(toff), i32(cnt or [0]), f64(fu or [0.0]), f64(fw or [0.0])
    busy_in = None
    if busy_ms is not None:
        busy_in = f64(busy_ms)
        if busy_in.shape != (n_dev,):
            raise Error(2, "simulate_batch: one measured busy time per device")
    cap_f = cap_o = None
    if capacities is not None:
        capacities.validate()
        if capacities.devices() != K:
            raise Error(2, "simulate_batch: capacities must be per schedule row")
        cap_f, cap_o = i32(capacities.full), i32(capacities.fwd)
    out = _CMetrics()
    busy = np.zeros(max(n_dev, 1))
    rc = np.zeros((max(K, 1), 3), np.int32)
    nul = C.c_void_p(None)
    check(lib().d2ft_schedule_metrics(
        ptr(codes), C.c_int(K), C.c_int(N), ptr(cf), ptr(cb), C.c_int(n_dev), ptr(mu), ptr(toff), ptr(cnt), ptr(fu),
        ptr(fw), ptr(busy_in) if busy_in is not None else nul, ptr(cap_f) if cap_f is not None else nul,
        ptr(cap_o) if cap_o is not None else nul, C.byref(out), ptr(busy), ptr(rc)))
    return BatchMetrics(out.compute_fraction, out.comm_fraction, out.workload_variance, out.makespan_ms,
                        [float(b) for b in busy[:n_dev]], out.imbalance_residual, out.row_workload_variance,
                        rc[:K].copy())


def compute_cost_fraction(schedule: ScheduleTable, cost_model: CostModel) -> float:
    """cost_sim.hpp:52-54, cost_sim.cpp:71-80."""
    return _metrics(schedule, cost_model).compute_fraction


def comm_cost_fraction(schedule: ScheduleTable) -> float:
    """cost_sim.hpp:56-59, cost_sim.cpp:82-92."""
    return _metrics(schedule, CostModel()).comm_fraction


def workload_variance(schedule: ScheduleTable, cost_model: CostModel) -> float:
    """cost_sim.hpp:61-63, cost_sim.cpp:94-110."""
    return _metrics(schedule, cost_model).row_workload_variance


def simulate_batch(schedule: ScheduleTable, profiles: Sequence[DeviceProfile], cost_model: CostModel,
                   capacities: Optional[Capacities] = None,
                   busy_ms: Optional[Sequence[float]] = None) -> BatchMetrics:
    """cost_sim.hpp:65-73, cost_sim.cpp:112-172.  busy_ms: measured per-device
    busy times (replace the timing tables; the profiles still give the
    row-to-device mapping)."""
    if not profiles:
        raise Error(2, "simulate_batch: no device profiles")
    return _metrics(schedule, cost_model, profiles, capacities, busy_ms)


class HeteroMode(Enum):
    Memory = 0
    Compute = 1


@dataclass
class HeteroSetup:
    """cost_sim.hpp:77-80."""
    profiles: List[DeviceProfile] = field(default_factory=list)
    budget: BudgetSpec = field(default_factory=BudgetSpec)


def build_hetero_profiles(mode: HeteroMode, count: int, subnet_units: int) -> HeteroSetup:
    """cost_sim.hpp:82-85, cost_sim.cpp:174-209 (configuration, host side)."""
    if count < 0 or subnet_units < 1:
        raise Error(2, "build_hetero_profiles: bad arguments")
    s = HeteroSetup(budget=BudgetSpec(n_full=2, n_fwd=2))
    if mode == HeteroMode.Memory:
        if 2 * count > subnet_units:
            raise Error(2, f"build_hetero_profiles: {count} large devices cannot host {subnet_units} subnet units")
        for i in range(count):
            p = DeviceProfile.standard(i)
            p.memory_units = 2
            s.profiles.append(p)
        for i in range(subnet_units - 2 * count):
            s.profiles.append(DeviceProfile.standard(count + i))
    else:
        if count > subnet_units:
            raise Error(2, "build_hetero_profiles: more fast devices than subnet units")
        for i in range(subnet_units):
            p = DeviceProfile.standard(i)
            if i < count:
                p.speed_class = Speed.Fast
                s.budget.overrides.append(BudgetOverride(i, 3, 1))
            s.profiles.append(p)
    return s


@dataclass
class ReferencePoint:
    """cost_sim.hpp:87-98."""
    setting: str = ""
    n_full: int = 0
    n_fwd: int = 0
    n_shortcut: int = 0
    computed_pct: float = 0.0
    nominal_pct: float = 0.0
    discrepancy: bool = False


def _point(setting, nf, no, ns, nominal, cm, comm) -> ReferencePoint:  # cost_sim.cpp:212-227
    t = ScheduleTable(1, nf + no + ns)
    t.codes[0, :nf] = 1
    t.codes[0, nf:nf + no] = 2
    m = _metrics(t, cm)
    pct = 100.0 * (m.comm_fraction if comm else m.compute_fraction)
    return ReferencePoint(setting, nf, no, ns, pct, nominal, abs(pct - nominal) > 0.5)


def lora_compute_reference_points() -> List[ReferencePoint]:
    """cost_sim.cpp:231-238."""
    cm = CostModel.lora_finetune()
    return [_point("3pf+2po of 5", 3, 2, 0, 95.0, cm, False), _point("3pf+1po+1ps of 5", 3, 1, 1, 75.0, cm, False),
            _point("3pf+2ps of 5", 3, 0, 2, 60.0, cm, False)]


def lora_comm_reference_points() -> List[ReferencePoint]:
    """cost_sim.cpp:240-247."""
    cm = CostModel.lora_finetune()
    return [_point("3pf+2po of 5", 3, 2, 0, 90.0, cm, True), _point("3pf+1po+1ps of 5", 3, 1, 1, 70.0, cm, True),
            _point("2pf+1po+2ps of 5", 2, 1, 2, 50.0, cm, True)]
