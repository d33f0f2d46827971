"""Artifact formats and cost accounting, CPU side.

* serialize: the reference's own test_serialize.cpp cases, restated against
  the C++ writers/readers of csrc/serialize.cu (host code, no GPU), plus the
  nlohmann dump(2) layout on literal expected strings and random round trips.
* cost_sim: the oracle restatement (oracle/cost_oracle.py) pinned to the
  literal expectations of test_cost_sim.cpp and, when it is built here, to the
  unmodified reference (oracle/_ref) on random tables; DeviceProfile.time_ms
  and build_hetero_profiles (host entry points) against both.
The GPU metrics kernel is checked against this oracle in test_metrics_gpu.py."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import cost_oracle as CO
from oracle import lib as O
from paper_2504_12471_b200 import Error, ScheduleTable, ScoreTable
from paper_2504_12471_b200 import cost_sim as CS
from paper_2504_12471_b200 import serialize as S


# ---------------------------------------------------------------- test_serialize.cpp
def test_score_table_json_round_trip():  # test_serialize.cpp:11-30
    t = ScoreTable(2, 3, [[0.5, 1.25, 0.0], [2.0, 3.5, 0.1]], [[1.0, 1.0, 1.0], [4.0, 4.0, 4.0]],
                   "fisher_information", "weight_magnitude")
    back = S.score_table_from_json(S.score_table_to_json(t))
    assert (back.subnets, back.micro_batches) == (2, 3)
    assert (back.fwd_metric, back.bwd_metric) == (t.fwd_metric, t.bwd_metric)
    assert np.array_equal(back.forward, t.forward) and np.array_equal(back.backward, t.backward)
    csv = S.score_table_to_csv(t)
    assert csv[:30] == "subnet_id,micro_batch,fwd,bwd\n"
    assert "1,1,3.5,4" in csv


def test_score_table_json_rejects_malformed_input():  # test_serialize.cpp:32-40
    for bad in ["{nope", "{}",
                '{"subnets":1,"micro_batches":2,"fwd_metric":"fisher_information",'
                '"bwd_metric":"weight_magnitude","forward":[[1.0]],"backward":[[1.0,2.0]]}']:
        with pytest.raises(Error):
            S.score_table_from_json(bad)
    with pytest.raises(Error) as e:
        S.score_table_from_json("{nope")
    assert str(e.value) == "score table: malformed JSON" and e.value.kind == "input"
    with pytest.raises(Error) as e:
        S.score_table_from_json("{}")
    assert str(e.value) == "score table: missing field 'subnets'"
    with pytest.raises(Error) as e:  # metric_from_name: config error
        S.score_table_from_json('{"subnets":0,"micro_batches":0,"fwd_metric":"x","bwd_metric":"x",'
                                '"forward":[],"backward":[]}')
    assert e.value.kind == "config" and str(e.value) == "unknown metric: x"
    with pytest.raises(Error) as e:  # validate: negative score -> numeric
        S.score_table_from_json('{"subnets":1,"micro_batches":1,"fwd_metric":"fisher_information",'
                                '"bwd_metric":"weight_magnitude","forward":[[-1]],"backward":[[1]]}')
    assert e.value.kind == "numeric"
    with pytest.raises(Error) as e:
        S.score_table_from_json('{"subnets":"a","micro_batches":1}')
    assert str(e.value) == "score table: field 'subnets' has the wrong type"


def test_schedule_table_round_trip_and_validation():  # test_serialize.cpp:42-60
    t = ScheduleTable(2, 3)
    t.set_code(0, 0, 1)
    t.set_code(0, 1, 2)
    t.set_code(1, 2, 1)
    assert S.schedule_table_from_json(S.schedule_table_to_json(t)) == t
    csv = S.schedule_table_to_csv(t)
    assert csv[:27] == "subnet_id,micro_batch,code\n"
    assert "0,1,2\n" in csv
    with pytest.raises(Error) as e:
        S.schedule_table_from_json('{"devices":1,"micro_batches":1,"codes":[[9]]}')
    assert str(e.value) == "schedule table: code out of range"
    with pytest.raises(Error) as e:
        S.schedule_table_from_json('{"devices":2,"micro_batches":1,"codes":[[1]]}')
    assert str(e.value) == "schedule table: codes row count mismatch"
    with pytest.raises(Error) as e:
        S.schedule_table_from_json('{"devices":1,"micro_batches":2,"codes":[[1]]}')
    assert str(e.value) == "schedule table: codes column count mismatch"


def test_history_csv_round_trip():  # test_serialize.cpp:62-73
    h = S.TrainHistory([S.EpochRecord(0, 1.5, 0.25, 0.6, 0.7), S.EpochRecord(1, 1.25, 0.5, 0.6, 0.7)])
    back = S.history_from_csv(S.history_to_csv(h))
    assert len(back.epochs) == 2
    assert back.epochs[1].loss == 1.25 and back.epochs[1].top1 == 0.5 and back.epochs[0].compute_fraction == 0.6
    assert back == h
    with pytest.raises(Error):
        S.history_from_csv("")
    with pytest.raises(Error) as e:
        S.history_from_csv("epoch,loss,top1,compute_fraction,comm_fraction\n1,2.0\n")
    assert str(e.value) == "history csv: short row"


def test_format_double_is_shortest_round_trip():  # test_serialize.cpp:75-81
    assert S.format_double(0.5) == "0.5"
    assert S.format_double(0.1) == "0.1"
    assert S.format_double(2.0) == "2"
    tricky = 1.0 / 3.0
    assert float(S.format_double(tricky)) == tricky
    rng = np.random.default_rng(7)
    for v in np.concatenate([rng.standard_normal(200) * 10.0 ** rng.integers(-30, 30, 200), [5e-324, 1.7e308]]):
        assert float(S.format_double(float(v))) == v
        assert len(S.format_double(float(v))) <= len(repr(float(v))) + 1  # repr is shortest too


def test_atomic_file_write_and_read_back(tmp_path):  # test_serialize.cpp:83-89
    path = str(tmp_path / "test_serialize_file.txt")
    S.atomic_write_file(path, "hello\nworld\n")
    assert S.read_file(path) == "hello\nworld\n"
    assert not os.path.exists(path + ".tmp")
    os.remove(path)
    with pytest.raises(Error) as e:
        S.read_file(path)
    assert e.value.kind == "input"


# ---------------------------------------------------------------- nlohmann dump(2) layout
def test_schedule_json_layout_matches_nlohmann_dump2():
    t = ScheduleTable(2, 3, [[1, 2, 3], [3, 3, 1]])
    expect = ('{\n  "codes": [\n    [\n      1,\n      2,\n      3\n    ],\n    [\n      3,\n      3,\n'
              '      1\n    ]\n  ],\n  "devices": 2,\n  "micro_batches": 3\n}\n')
    assert S.schedule_table_to_json(t) == expect
    assert S.schedule_table_to_json(ScheduleTable(0, 0)) == '{\n  "codes": [],\n  "devices": 0,\n  "micro_batches": 0\n}\n'


def test_json_double_layout_matches_nlohmann():
    # nlohmann::detail::to_chars: shortest digits, decimal for 1e-4 <= |x| < 1e15,
    # ".0" on integral values, two-digit signed exponents otherwise
    cases = [(0.5, "0.5"), (2.0, "2.0"), (0.0, "0.0"), (-0.0, "-0.0"), (0.1, "0.1"), (1e-4, "0.0001"),
             (1e-5, "1e-05"), (123456.789, "123456.789"), (1e14, "100000000000000.0"), (1e15, "1e+15"),
             (1.5e20, "1.5e+20"), (-2.5e-7, "-2.5e-07"), (1e100, "1e+100"), (1 / 3, "0.3333333333333333"),
             (5e-324, "5e-324"), (float("nan"), "null"), (float("inf"), "null")]
    for v, s in cases:
        assert S._text(S.lib().d2ft_json_double, C.c_double(v)) == s, v


def test_score_table_json_layout():
    t = ScoreTable(1, 2, [[0.5, 2.0]], [[1e-5, 0.0]], "taylor_importance", "gradient_magnitude")
    expect = ('{\n  "backward": [\n    [\n      1e-05,\n      0.0\n    ]\n  ],\n'
              '  "bwd_metric": "gradient_magnitude",\n  "forward": [\n    [\n      0.5,\n      2.0\n    ]\n  ],\n'
              '  "fwd_metric": "taylor_importance",\n  "micro_batches": 2,\n  "subnets": 1\n}\n')
    assert S.score_table_to_json(t) == expect


def test_batch_metrics_formats():
    m = CS.BatchMetrics(0.52, 0.5, 0.25, 2.74, [2.74, 2.2], 5.0)
    js = S.batch_metrics_to_json(m, 'run "7"', "d2ft")
    assert js == ('{\n  "comm_fraction": 0.5,\n  "compute_fraction": 0.52,\n  "imbalance_residual": 5.0,\n'
                  '  "makespan_ms": 2.74,\n  "method": "d2ft",\n  "per_device_busy_ms": [\n    2.74,\n    2.2\n  ],\n'
                  '  "run_id": "run \\"7\\"",\n  "workload_variance": 0.25\n}\n')
    assert S.batch_metrics_csv_header() == ("run_id,method,compute_fraction,comm_fraction,workload_variance,"
                                            "makespan_ms,imbalance_residual\n")
    assert S.batch_metrics_to_csv_row(m, "r1", "d2ft") == "r1,d2ft,0.52,0.5,0.25,2.74,5\n"


def test_history_json_layout():
    h = S.TrainHistory([S.EpochRecord(0, 1.5, 0.25, 0.6, 0.7)])
    assert S.history_to_json(h) == ('{\n  "epochs": [\n    {\n      "comm_fraction": 0.7,\n'
                                    '      "compute_fraction": 0.6,\n      "epoch": 0,\n      "loss": 1.5,\n'
                                    '      "top1": 0.25\n    }\n  ]\n}\n')
    assert S.history_to_json(S.TrainHistory()) == '{\n  "epochs": []\n}\n'


def test_random_round_trips():
    rng = np.random.default_rng(11)
    for trial in range(20):
        K, N = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        f = np.abs(rng.standard_normal((K, N))) * 10.0 ** rng.integers(-8, 8, (K, N))
        b = np.abs(rng.standard_normal((K, N)))
        t = ScoreTable(K, N, f, b, S.METRICS[trial % 4], S.METRICS[(trial + 1) % 4])
        back = S.score_table_from_json(S.score_table_to_json(t))
        assert np.array_equal(back.forward, t.forward) and np.array_equal(back.backward, t.backward)
        st = ScheduleTable(K, N, rng.integers(1, 4, (K, N)))
        assert S.schedule_table_from_json(S.schedule_table_to_json(st)) == st


# ---------------------------------------------------------------- cost_sim oracle pins
def _row(nf, no, ns):
    return np.array([[1] * nf + [2] * no + [3] * ns], np.uint8)


def test_oracle_cost_fractions_known_answers():  # test_cost_sim.cpp:24-42
    for n_po, exp in enumerate([0.20, 0.28, 0.36, 0.44, 0.52]):
        assert CO.compute_cost_fraction(_row(1, n_po, 4 - n_po), [2], [3]) == exp
    assert CO.compute_cost_fraction(_row(5, 0, 0), [2], [3]) == 1.0
    for (nf, no, ns), exp in {(2, 1, 2): 0.5, (3, 1, 1): 0.7, (3, 2, 0): 0.8, (0, 0, 5): 0.0, (5, 0, 0): 1.0}.items():
        assert CO.comm_cost_fraction(_row(nf, no, ns)) == exp


def test_oracle_workload_variance_known_answers():  # test_cost_sim.cpp:44-98
    t = np.full((4, 5), 3, np.uint8)
    t[:, :3] = 1
    assert CO.workload_variance(t, [2] * 4, [3] * 4) == 0.0
    t = np.full((2, 5), 3, np.uint8)
    t[0, :] = 1
    assert CO.workload_variance(t, [2] * 2, [3] * 2) == 0.25
    rng = np.random.default_rng(31337)
    for _ in range(20):
        t = rng.integers(1, 4, (3, 6)).astype(np.uint8)
        loads = [sum(5 if c == 1 else 2 if c == 2 else 0 for c in row) / 30.0 for row in t]
        mean = (loads[0] + loads[1] + loads[2]) / 3.0
        ref = 0.0
        for l in loads:  # a plain loop: Python >= 3.12 sum() of floats is compensated
            ref += (l - mean) * (l - mean)
        ref /= 3.0
        assert CO.workload_variance(t, [2] * 3, [3] * 3) == ref


def test_oracle_timing_table_known_answers():  # test_cost_sim.cpp:100-131
    T = CO.DEFAULT_TIMING
    for c, full, exp in [(1, True, 2.01), (1, False, 0.86), (2, True, 2.20), (3, True, 2.27), (4, False, 1.20),
                         (5, True, 3.16), (5, False, 1.48), (0, True, 0.0)]:
        assert CO.time_ms(T, c, full) == exp
    sparse = [(2, 2.0, 1.0), (4, 3.0, 2.0)]
    assert CO.time_ms(sparse, 3, True) == pytest.approx(2.5)
    assert CO.time_ms(sparse, 3, False) == pytest.approx(1.5)
    assert CO.time_ms(sparse, 1, True) == pytest.approx(1.0)
    assert CO.time_ms(T, 7, True) == pytest.approx(3.16 + 2 * (3.16 - 2.74))


def test_oracle_simulate_batch_known_answers():  # test_cost_sim.cpp:133-199
    T = CO.DEFAULT_TIMING
    assert CO.simulate_batch(_row(1, 0, 4), [2], [3], [1], [T])[3] == 2.01
    assert CO.simulate_batch(_row(0, 1, 4), [2], [3], [1], [T])[3] == 0.86
    t = np.full((3, 5), 3, np.uint8)
    t[:, :2] = 1
    r = CO.simulate_batch(t, [2] * 3, [3] * 3, [2, 1], [T, T])
    assert r[5] == [2.74, 2.20] and r[3] == 2.74
    assert CO.simulate_batch(_row(2, 2, 1), [2], [3], [1], [T], caps=([10], [4]))[4] == 0.0
    assert CO.simulate_batch(_row(2, 2, 1), [2], [3], [1], [T], caps=([15], [4]))[4] == 5.0


def _ref_metrics(codes, cf, cb, mu, tables, caps=None):
    R = O.ref_lib()
    K, N = codes.shape
    toff = np.cumsum([0] + [len(t) for t in tables]).astype(np.int32)
    flat = [e for t in tables for e in t] or [(1, 0.0, 0.0)]
    cnt = np.array([e[0] for e in flat], np.int32)
    fu = np.array([e[1] for e in flat])
    fw = np.array([e[2] for e in flat])
    out = np.zeros(6)
    busy = np.zeros(max(1, len(mu)))
    cfa, cba = np.array(cf, np.int32), np.array(cb, np.int32)
    mua = np.array(mu or [0], np.int32)
    cf_ = np.ascontiguousarray(caps[0], np.int32) if caps else None
    co_ = np.ascontiguousarray(caps[1], np.int32) if caps else None
    p = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
    rc = R.ref_schedule_metrics(p(np.ascontiguousarray(codes)), K, N, 0, 0, p(cfa), p(cba), len(mu), p(mua), p(toff),
                                p(cnt), p(fu), p(fw), p(cf_), p(co_), p(out), p(busy))
    assert rc == 0, R.ref_last_error()
    return out, busy[:len(mu)]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_oracle_matches_reference_cost_sim_bitwise():
    rng = np.random.default_rng(99)
    for trial in range(60):
        K, N = int(rng.integers(1, 40)), int(rng.integers(1, 30))
        codes = rng.integers(1, 4, (K, N)).astype(np.uint8)
        cf = rng.integers(0, 8, K).tolist()
        cb = rng.integers(0, 8, K).tolist()
        mu = []
        while sum(mu) < K:
            mu.append(int(min(rng.integers(1, 4), K - sum(mu))))
        tables = []
        for _ in mu:
            n = int(rng.integers(1, 6))
            counts = np.sort(rng.choice(np.arange(1, 12), n, replace=False))
            tables.append([(int(c), float(a), float(b)) for c, a, b in
                           zip(counts, np.sort(rng.random(n) * 5), np.sort(rng.random(n) * 2))])
        caps = (rng.integers(0, 100, K), rng.integers(0, 50, K)) if trial % 2 else None
        ref, ref_busy = _ref_metrics(codes, cf, cb, mu, tables, caps)
        o = CO.simulate_batch(codes, cf, cb, mu, tables, caps=caps)
        assert list(o[:5]) == ref[:5].tolist()
        assert o[5] == ref_busy.tolist()
        assert CO.workload_variance(codes, cf, cb) == ref[5]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_time_ms_host_entry_matches_reference():
    R = O.ref_lib()
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(1, 6))
        counts = np.sort(rng.choice(np.arange(1, 12), n, replace=False))
        prof = CS.DeviceProfile(timing_table=[CS.TimingEntry(int(c), float(a), float(b)) for c, a, b in
                                              zip(counts, np.sort(rng.random(n) * 5), np.sort(rng.random(n) * 2))])
        cnt, fu, fw = prof._arrays()
        for count in range(0, 15):
            for full in (True, False):
                out = C.c_double()
                assert R.ref_time_ms(cnt.ctypes.data_as(C.c_void_p), fu.ctypes.data_as(C.c_void_p),
                                     fw.ctypes.data_as(C.c_void_p), n, count, int(full), C.byref(out)) == 0
                assert prof.time_ms(count, full) == out.value
                assert CO.time_ms([(e.count, e.full_ms, e.fwd_ms) for e in prof.timing_table], count, full) == out.value


def test_device_profile_validation_and_defaults():  # test_cost_sim.cpp:100-131
    p = CS.DeviceProfile.standard(0)
    assert p.time_ms(1, True) == 2.01 and p.time_ms(5, False) == 1.48 and p.time_ms(0, True) == 0.0
    assert p.time_ms(7, True) == pytest.approx(3.16 + 2 * (3.16 - 2.74))
    bad = CS.DeviceProfile.standard(0)
    bad.timing_table = [CS.TimingEntry(1, 2.0, 1.0), CS.TimingEntry(2, 1.5, 1.2)]
    with pytest.raises(Error):
        bad.validate()
    with pytest.raises(Error):
        p.time_ms(-1, True)


def test_build_hetero_profiles():  # test_cost_sim.cpp:201-255
    s = CS.build_hetero_profiles(CS.HeteroMode.Memory, 9, 74)
    assert len(s.profiles) == 65 and sum(p.memory_units for p in s.profiles) == 74
    assert sum(p.memory_units == 2 for p in s.profiles) == 9
    assert (s.budget.n_full, s.budget.n_fwd, s.budget.overrides) == (2, 2, [])
    for count in (9, 14, 19):
        s = CS.build_hetero_profiles(CS.HeteroMode.Memory, count, 74)
        assert sum(p.memory_units for p in s.profiles) == 74 and len(s.profiles) == 74 - count
    s = CS.build_hetero_profiles(CS.HeteroMode.Compute, 2, 6)
    assert len(s.profiles) == 6 and s.profiles[0].speed_class == CS.Speed.Fast
    assert s.profiles[2].speed_class == CS.Speed.Slow
    assert [(o.n_full, o.n_fwd) for o in s.budget.overrides] == [(3, 1), (3, 1)]
    assert s.budget.n_full_for(0) == 3 and s.budget.n_full_for(3) == 2
    s = CS.build_hetero_profiles(CS.HeteroMode.Compute, 0, 4)
    assert all(p.speed_class == CS.Speed.Slow for p in s.profiles) and not s.budget.overrides
    with pytest.raises(Error):
        CS.build_hetero_profiles(CS.HeteroMode.Memory, 40, 74)
    with pytest.raises(Error):
        CS.build_hetero_profiles(CS.HeteroMode.Compute, 10, 6)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_build_hetero_profiles_matches_reference():
    R = O.ref_lib()
    for mode in (0, 1):
        for count in range(0, 12):
            for units in (1, 6, 20, 74):
                np_, no = C.c_int(), C.c_int()
                mu, fast, ovr, b2 = (np.zeros(200, np.int32), np.zeros(200, np.int32), np.zeros(600, np.int32),
                                     np.zeros(2, np.int32))
                rc = R.ref_build_hetero_profiles(mode, count, units, 200, C.byref(np_), mu.ctypes.data_as(C.c_void_p),
                                                 fast.ctypes.data_as(C.c_void_p), ovr.ctypes.data_as(C.c_void_p),
                                                 C.byref(no), b2.ctypes.data_as(C.c_void_p))
                try:
                    s = CS.build_hetero_profiles(CS.HeteroMode(mode), count, units)
                except Error as e:
                    assert rc == e.code
                    continue
                assert rc == 0
                assert [p.memory_units for p in s.profiles] == mu[:np_.value].tolist()
                assert [int(p.speed_class == CS.Speed.Fast) for p in s.profiles] == fast[:np_.value].tolist()
                assert [(o.device, o.n_full, o.n_fwd) for o in s.budget.overrides] == \
                    [tuple(ovr[3 * i:3 * i + 3]) for i in range(no.value)]
                assert [s.budget.n_full, s.budget.n_fwd] == b2.tolist()
