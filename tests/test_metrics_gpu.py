"""GPU schedule metrics (csrc/metrics.cu) against the pinned oracle
(oracle/cost_oracle.py, see test_artifacts_cpu.py) and the literal
expectations of the reference's test_cost_sim.cpp: bit-exact."""
import ctypes as C

import numpy as np
import pytest

from oracle import cost_oracle as CO
from paper_2504_12471_b200 import Capacities, CostModel, Error, ScheduleTable
from paper_2504_12471_b200 import cost_sim as CS

pytestmark = pytest.mark.gpu


def _row(nf, no, ns):
    return ScheduleTable(1, nf + no + ns, [[1] * nf + [2] * no + [3] * ns])


def test_cost_fractions_known_answers():  # test_cost_sim.cpp:24-42
    cm = CostModel()
    for n_po, exp in enumerate([0.20, 0.28, 0.36, 0.44, 0.52]):
        assert CS.compute_cost_fraction(_row(1, n_po, 4 - n_po), cm) == exp
    assert CS.compute_cost_fraction(_row(5, 0, 0), cm) == 1.0
    for (nf, no, ns), exp in {(2, 1, 2): 0.5, (3, 1, 1): 0.7, (3, 2, 0): 0.8, (0, 0, 5): 0.0, (5, 0, 0): 1.0}.items():
        assert CS.comm_cost_fraction(_row(nf, no, ns)) == exp


def test_workload_variance_known_answers():  # test_cost_sim.cpp:44-98
    cm = CostModel()
    t = ScheduleTable(4, 5)
    t.codes[:, :3] = 1
    assert CS.workload_variance(t, cm) == 0.0
    t = ScheduleTable(2, 5)
    t.codes[0, :] = 1
    assert CS.workload_variance(t, cm) == 0.25
    rng = np.random.default_rng(555)
    t = ScheduleTable(4, 5)
    for k in range(4):
        perm = rng.permutation(5)
        t.codes[k, perm[:2]] = 1
        t.codes[k, perm[2]] = 2
    assert CS.workload_variance(t, cm) == 0.0


def test_simulate_batch_known_answers():  # test_cost_sim.cpp:133-199
    cm = CostModel()
    std = CS.DeviceProfile.standard
    assert CS.simulate_batch(_row(1, 0, 4), [std(0)], cm).makespan_ms == 2.01
    assert CS.simulate_batch(_row(0, 1, 4), [std(0)], cm).makespan_ms == 0.86
    t = ScheduleTable(2, 5)
    t.codes[:, :2] = 1
    m = CS.simulate_batch(t, [std(0), std(1)], cm)
    assert m.per_device_busy_ms[0] == m.per_device_busy_ms[1] == m.makespan_ms and m.workload_variance == 0.0
    t = ScheduleTable(3, 5)
    t.codes[:, :2] = 1
    large = std(0)
    large.memory_units = 2
    m = CS.simulate_batch(t, [large, std(1)], cm)
    assert m.per_device_busy_ms == [2.74, 2.20] and m.makespan_ms == 2.74
    rng = np.random.default_rng(4711)
    t = ScheduleTable(4, 5, rng.integers(1, 4, (4, 5)))
    m = CS.simulate_batch(t, [std(k) for k in range(4)], cm)
    assert m.makespan_ms >= sum(m.per_device_busy_ms) / 4
    t = _row(2, 2, 1)
    assert CS.simulate_batch(t, [std(0)], cm, Capacities([10], [4])).imbalance_residual == 0.0
    assert CS.simulate_batch(t, [std(0)], cm, Capacities([15], [4])).imbalance_residual == 5.0
    with pytest.raises(Error) as e:
        CS.simulate_batch(ScheduleTable(3, 5), [std(0), std(1)], cm)
    assert e.value.kind == "input" and "host 2 subnet units but the schedule has 3 rows" in str(e.value)
    with pytest.raises(Error) as e:
        CS.simulate_batch(ScheduleTable(1, 2, [[1, 7]]), [std(0)], cm)
    assert str(e.value) == "schedule table: code out of range"


def _random_case(rng, K, N):
    codes = rng.integers(1, 4, (K, N)).astype(np.uint8)
    cf = rng.integers(0, 8, K).tolist()
    cb = rng.integers(0, 8, K).tolist()
    mu = []
    while sum(mu) < K:
        mu.append(int(min(rng.integers(1, 5), K - sum(mu))))
    tables = []
    for _ in mu:
        n = int(rng.integers(1, 6))
        counts = np.sort(rng.choice(np.arange(1, 4 * N + 2), n, replace=False))
        tables.append([(int(c), float(a), float(b)) for c, a, b in
                       zip(counts, np.sort(rng.random(n) * 5), np.sort(rng.random(n) * 2))])
    return codes, cf, cb, mu, tables


def test_random_tables_bit_exact_vs_oracle():
    rng = np.random.default_rng(2026)
    for trial in range(40):
        K, N = int(rng.integers(1, 60)), int(rng.integers(1, 40))
        codes, cf, cb, mu, tables = _random_case(rng, K, N)
        caps = (rng.integers(0, 200, K), rng.integers(0, 100, K)) if trial % 2 else None
        cm = CostModel(forward_cost_per_device=cf, backward_cost_per_device=cb)
        profiles = [CS.DeviceProfile(p, m, timing_table=[CS.TimingEntry(*e) for e in t])
                    for p, (m, t) in enumerate(zip(mu, tables))]
        m = CS.simulate_batch(ScheduleTable(K, N, codes), profiles, cm,
                              Capacities(list(caps[0]), list(caps[1])) if caps else None)
        o = CO.simulate_batch(codes, cf, cb, mu, tables, caps=caps)
        assert (m.compute_fraction, m.comm_fraction, m.workload_variance, m.makespan_ms, m.imbalance_residual) == o[:5]
        assert m.per_device_busy_ms == o[5]
        assert m.row_workload_variance == CO.workload_variance(codes, cf, cb)
        assert np.array_equal(m.row_counts, np.stack([(codes == c).sum(1) for c in (1, 2, 3)], 1))


def test_measured_busy_times_replace_the_table():
    rng = np.random.default_rng(3)
    codes, cf, cb, mu, tables = _random_case(rng, 144, 64)
    busy = rng.random(len(mu)) * 4.0
    cm = CostModel(forward_cost_per_device=cf, backward_cost_per_device=cb)
    profiles = [CS.DeviceProfile(p, m, timing_table=[CS.TimingEntry(*e) for e in t])
                for p, (m, t) in enumerate(zip(mu, tables))]
    m = CS.simulate_batch(ScheduleTable(144, 64, codes), profiles, cm, busy_ms=busy)
    o = CO.simulate_batch(codes, cf, cb, mu, tables, busy_ms=busy)
    assert m.per_device_busy_ms == busy.tolist() and m.makespan_ms == busy.max()
    assert (m.compute_fraction, m.comm_fraction, m.workload_variance) == o[:3]


def test_scheduler_sweep_size_table():
    # BASELINE.json configs[4]: batch 1024 x 144 subnets, 8 devices of 18 rows
    rng = np.random.default_rng(8)
    K, N = 144, 1024
    codes = rng.integers(1, 4, (K, N)).astype(np.uint8)
    T = CO.DEFAULT_TIMING
    profiles = [CS.DeviceProfile.standard(p) for p in range(8)]
    for p in profiles:
        p.memory_units = 18
    m = CS.simulate_batch(ScheduleTable(K, N, codes), profiles, CostModel())
    o = CO.simulate_batch(codes, [2] * K, [3] * K, [18] * 8, [T] * 8)
    assert (m.compute_fraction, m.comm_fraction, m.workload_variance, m.makespan_ms) == o[:4]
    assert m.per_device_busy_ms == o[5]


def test_lora_reference_points():  # test_cost_sim.cpp:257-279
    pts = CS.lora_compute_reference_points()
    assert [p.computed_pct for p in pts] == [95.0, 77.5, 60.0]
    assert abs(pts[0].computed_pct - pts[0].nominal_pct) <= 3.0 and abs(pts[1].computed_pct - pts[1].nominal_pct) <= 3.0
    assert pts[2].computed_pct == pts[2].nominal_pct
    pts = CS.lora_comm_reference_points()
    assert [p.computed_pct for p in pts] == [80.0, 70.0, 50.0]
    assert [p.discrepancy for p in pts] == [True, False, False]


def test_device_entry_matches_host_entry():
    import torch
    from paper_2504_12471_b200._lib import check, lib

    rng = np.random.default_rng(12)
    K, N = 36, 48
    codes, cf, cb, mu, tables = _random_case(rng, K, N)
    cm = CostModel(forward_cost_per_device=cf, backward_cost_per_device=cb)
    profiles = [CS.DeviceProfile(p, m, timing_table=[CS.TimingEntry(*e) for e in t])
                for p, (m, t) in enumerate(zip(mu, tables))]
    host = CS.simulate_batch(ScheduleTable(K, N, codes), profiles, cm)
    dev = torch.device("cuda:0")
    t_codes = torch.from_numpy(codes.reshape(-1)).to(dev)
    i = lambda a: torch.tensor(a, dtype=torch.int32, device=dev)
    d = lambda a: torch.tensor(a, dtype=torch.float64, device=dev)
    toff = np.cumsum([0] + [len(t) for t in tables]).tolist()
    flat = [e for t in tables for e in t]
    out6, busy = torch.zeros(6, dtype=torch.float64, device=dev), torch.zeros(len(mu), dtype=torch.float64, device=dev)
    rc, err = torch.zeros(3 * K, dtype=torch.int32, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)
    args = [i(cf), i(cb), i(mu), i(toff), i([e[0] for e in flat]), d([e[1] for e in flat]), d([e[2] for e in flat])]
    P = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None
    check(lib().d2ft_schedule_metrics_device(
        P(t_codes), K, N, P(args[0]), P(args[1]), len(mu), P(args[2]), P(args[3]), P(args[4]), P(args[5]),
        P(args[6]), None, None, None, P(out6), P(busy), P(rc), P(err), None))
    torch.cuda.synchronize()
    o = out6.cpu().numpy()
    assert err.item() == 0
    assert o.tolist() == [host.compute_fraction, host.comm_fraction, host.workload_variance, host.makespan_ms,
                          host.imbalance_residual, host.row_workload_variance]
    assert busy.cpu().numpy().tolist() == host.per_device_busy_ms


def test_empty_tables():  # cost_sim.cpp: zero cells -> 0 fractions, zero rows -> 0 variance
    cm = CostModel()
    m = CS._metrics(ScheduleTable(0, 0), cm)
    assert (m.compute_fraction, m.comm_fraction, m.row_workload_variance) == (0.0, 0.0, 0.0)
    m = CS._metrics(ScheduleTable(3, 0), cm)
    assert (m.compute_fraction, m.comm_fraction, m.row_workload_variance) == (0.0, 0.0, 0.0)
    assert m.row_counts.tolist() == [[0, 0, 0]] * 3
    zero = CostModel(forward_cost=0, backward_cost=0)
    t = ScheduleTable(2, 4, [[1, 2, 3, 1], [3, 3, 3, 3]])
    assert CS.compute_cost_fraction(t, zero) == CO.compute_cost_fraction(t.codes, [0, 0], [0, 0]) == 0.0
    assert CS.workload_variance(t, zero) == 0.0
