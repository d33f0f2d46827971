"""Host mirror of the reference's artifact formats, core/include/d2ft/
serialize.hpp (same function names, argument meaning and errors), over the
C++ writers/readers in csrc/serialize.cu.  JSON matches the reference's
nlohmann dump(2) layout; CSV doubles are shortest round-trip
(format_double)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._lib import Error, check, f64, i32, lib, ptr, u8
from .cost_sim import BatchMetrics, _CMetrics
from .scheduler import ScheduleTable, ScoreTable

# scoring.hpp:18-23 (Metric enum order), names as scoring.cpp:12-20
METRICS = ["fisher_information", "weight_magnitude", "gradient_magnitude", "taylor_importance"]


@dataclass
class EpochRecord:
    """trainer.hpp:82-88."""
    epoch: int = 0
    loss: float = 0.0
    top1: float = 0.0
    compute_fraction: float = 0.0
    comm_fraction: float = 0.0


@dataclass
class TrainHistory:
    """trainer.hpp:90-92."""
    epochs: List[EpochRecord] = field(default_factory=list)


def _text(fn, *args) -> str:
    """Call a text-producing entry point, growing the buffer on status 6."""
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        n = C.c_size_t()
        rc = fn(*args, buf, C.c_size_t(cap), C.byref(n))
        if rc == 6 and n.value + 1 > cap:
            cap = n.value + 1
            continue
        check(rc)
        return buf.raw[:n.value].decode()


def _metric_id(name: str) -> int:
    if name not in METRICS:
        raise Error(1, f"unknown metric: {name}")
    return METRICS.index(name)


def format_double(v: float) -> str:
    """serialize.hpp:23-24: shortest round-trip decimal."""
    return _text(lib().d2ft_format_double, C.c_double(v))


def atomic_write_file(path: str, contents: str) -> None:
    """serialize.hpp:26 (temp file + rename)."""
    data = contents.encode()
    check(lib().d2ft_atomic_write_file(path.encode(), data, C.c_size_t(len(data))))


def read_file(path: str) -> str:
    """serialize.hpp:27 (input error when missing)."""
    return _text(lib().d2ft_read_file, path.encode())


# --- ScoreTable ----------------------------------------------------------
def score_table_to_json(t: ScoreTable) -> str:
    fo, bo = f64(t.forward).reshape(-1), f64(t.backward).reshape(-1)
    return _text(lib().d2ft_score_table_to_json, ptr(fo), ptr(bo), C.c_int(t.subnets), C.c_int(t.micro_batches),
                 C.c_int(_metric_id(t.fwd_metric)), C.c_int(_metric_id(t.bwd_metric)))


def score_table_from_json(text: str) -> ScoreTable:
    raw = text.encode()
    K, N, fm, bm = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    rc = lib().d2ft_score_table_from_json(raw, C.c_size_t(len(raw)), C.byref(K), C.byref(N), C.byref(fm),
                                          C.byref(bm), None, None, C.c_size_t(0))
    if rc != 6:  # 6 = sized only (no buffers yet)
        check(rc)
    cells = K.value * N.value
    fo, bo = np.zeros(max(cells, 1)), np.zeros(max(cells, 1))
    check(lib().d2ft_score_table_from_json(raw, C.c_size_t(len(raw)), C.byref(K), C.byref(N), C.byref(fm),
                                           C.byref(bm), ptr(fo), ptr(bo), C.c_size_t(fo.size)))
    return ScoreTable(K.value, N.value, fo[:cells], bo[:cells], METRICS[fm.value], METRICS[bm.value])


def score_table_to_csv(t: ScoreTable) -> str:
    fo, bo = f64(t.forward).reshape(-1), f64(t.backward).reshape(-1)
    return _text(lib().d2ft_score_table_to_csv, ptr(fo), ptr(bo), C.c_int(t.subnets), C.c_int(t.micro_batches))


# --- ScheduleTable -------------------------------------------------------
def schedule_table_to_json(t: ScheduleTable) -> str:
    codes = u8(t.codes).reshape(-1)
    return _text(lib().d2ft_schedule_table_to_json, ptr(codes), C.c_int(t.devices), C.c_int(t.micro_batches))


def schedule_table_from_json(text: str) -> ScheduleTable:
    raw = text.encode()
    K, N = C.c_int(), C.c_int()
    rc = lib().d2ft_schedule_table_from_json(raw, C.c_size_t(len(raw)), C.byref(K), C.byref(N), None, C.c_size_t(0))
    if rc != 6:
        check(rc)
    codes = np.zeros(max(K.value * N.value, 1), np.uint8)
    check(lib().d2ft_schedule_table_from_json(raw, C.c_size_t(len(raw)), C.byref(K), C.byref(N), ptr(codes),
                                              C.c_size_t(codes.size)))
    return ScheduleTable(K.value, N.value, codes[:K.value * N.value])


def schedule_table_to_csv(t: ScheduleTable) -> str:
    codes = u8(t.codes).reshape(-1)
    return _text(lib().d2ft_schedule_table_to_csv, ptr(codes), C.c_int(t.devices), C.c_int(t.micro_batches))


# --- BatchMetrics --------------------------------------------------------
def _cm(m: BatchMetrics) -> _CMetrics:
    return _CMetrics(m.compute_fraction, m.comm_fraction, m.workload_variance, m.makespan_ms, m.imbalance_residual,
                     m.row_workload_variance)


def batch_metrics_to_json(m: BatchMetrics, run_id: str, method: str) -> str:
    busy = f64(m.per_device_busy_ms or [0.0])
    return _text(lib().d2ft_batch_metrics_to_json, C.byref(_cm(m)), ptr(busy), C.c_int(len(m.per_device_busy_ms)),
                 run_id.encode(), method.encode())


def batch_metrics_csv_header() -> str:
    return _text(lib().d2ft_batch_metrics_csv_header)


def batch_metrics_to_csv_row(m: BatchMetrics, run_id: str, method: str) -> str:
    return _text(lib().d2ft_batch_metrics_to_csv_row, C.byref(_cm(m)), run_id.encode(), method.encode())


# --- TrainHistory --------------------------------------------------------
def _hist_arrays(h: TrainHistory):
    e = h.epochs
    return (i32([r.epoch for r in e] or [0]), f64([r.loss for r in e] or [0.0]), f64([r.top1 for r in e] or [0.0]),
            f64([r.compute_fraction for r in e] or [0.0]), f64([r.comm_fraction for r in e] or [0.0]))


def history_to_csv(h: TrainHistory) -> str:
    a = _hist_arrays(h)
    return _text(lib().d2ft_history_to_csv, *[ptr(x) for x in a], C.c_int(len(h.epochs)))


def history_to_json(h: TrainHistory) -> str:
    a = _hist_arrays(h)
    return _text(lib().d2ft_history_to_json, *[ptr(x) for x in a], C.c_int(len(h.epochs)))


def history_from_csv(text: str) -> TrainHistory:
    raw = text.encode()
    cap = max(1, raw.count(b"\n") + 1)
    ep = np.zeros(cap, np.int32)
    cols = [np.zeros(cap) for _ in range(4)]
    n = C.c_int()
    check(lib().d2ft_history_from_csv(raw, C.c_size_t(len(raw)), ptr(ep), *[ptr(c) for c in cols], C.c_int(cap),
                                      C.byref(n)))
    return TrainHistory([EpochRecord(int(ep[r]), *(float(c[r]) for c in cols)) for r in range(n.value)])
