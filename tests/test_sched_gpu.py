"""GPU parity: the sm_100a scheduler/compaction kernels against the oracle.

Bar: bit-exact (selections, objectives, codes, lists) — SURVEY.md §8c."""
import os

import numpy as np
import pytest

import paper_2504_12471_b200 as P
from oracle import lib as O

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _table(b, f):
    K, N = b.shape
    return P.ScoreTable(K, N, f, b)


def test_dp_search_known_answers():
    # test_scheduler.cpp:62-87
    r = P.dp_search([[5.0, 4.0]], [[2, 2]], [0])
    assert r.objective[0] == 0.0 and r.selection[0].tolist() == [0, 0]
    r = P.dp_search([[5.0, 4.0, 3.0]], [[2, 2, 2]], [4])
    assert r.objective[0] == 9.0 and r.selection[0].tolist() == [1, 1, 0]
    with pytest.raises(P.Error) as e:
        P.dp_search([[1.0]], [[1]], [-1])
    assert e.value.kind == "input"
    with pytest.raises(P.Error) as e:
        P.dp_search([[float("nan")]], [[1]], [1])
    assert e.value.kind == "numeric"
    r = P.dp_search([[2.0] * 5], [[5] * 5], [15])
    assert r.selection[0].tolist() == [1, 1, 1, 0, 0]


def test_dp_search_acceptance_crit1_style():
    # acceptance_main.cpp:67-103: 100 instances, K<=6, N<=12, w in [1,7], cap < 40
    rng = np.random.default_rng(0xACCE97)
    for trial in range(100):
        K = int(rng.integers(1, 7))
        N = int(rng.integers(1, 13))
        s = rng.random((K, N)) * 10.0
        w = rng.integers(1, 8, (K, N)).astype(np.int32)
        if trial % 3 == 0:
            w[:] = w[:, :1]  # constant rows -> count-compressed kernel
        caps = rng.integers(0, 40, K).astype(np.int32)
        got = P.dp_search(s, w, caps)
        sel, obj = O.dp_search(s, w, caps)
        assert np.array_equal(got.selection, sel), trial
        assert np.array_equal(got.objective, obj), trial


def test_dp_search_zero_weights_and_large_caps():
    rng = np.random.default_rng(3)
    for trial in range(30):
        K, N = int(rng.integers(1, 9)), int(rng.integers(1, 200))
        s = rng.random((K, N)) * 10.0
        s[rng.random((K, N)) < 0.2] = 0.0
        wt = rng.integers(0, 4, K)
        w = np.repeat(wt[:, None], N, 1).astype(np.int32)
        caps = rng.integers(0, 6 * N + 10, K).astype(np.int32)
        got = P.dp_search(s, w, caps)
        sel, obj = O.dp_search(s, w, caps)
        assert np.array_equal(got.selection, sel) and np.array_equal(got.objective, obj), trial


def test_knapsack_literal_cases():
    cm = P.CostModel()
    t = P.ScoreTable(1, 2, [[9.0, 1.0]], [[5.0, 1.0]])
    assert P.knapsack_schedule(t, cm, P.Capacities([5], [2])).codes.tolist() == [[1, 3]]
    t = P.ScoreTable(1, 3, [[0.0, 8.0, 1.0]], [[9.0, 1.0, 1.0]])
    assert P.knapsack_schedule(t, cm, P.Capacities([5], [2])).codes.tolist() == [[1, 2, 3]]
    t = P.ScoreTable(2, 5, np.zeros((2, 5)), [[7.0] * 5, [1.5] * 5])
    caps = P.capacities_from_budget(P.BudgetSpec(3, 0), cm, 2, 5)
    assert P.knapsack_schedule(t, cm, caps).codes.tolist() == [[1, 1, 1, 3, 3]] * 2


def test_knapsack_errors_mirror_reference():
    cm = P.CostModel()
    t = P.ScoreTable(1, 2, [[1.0, -1.0]], [[1.0, 1.0]])
    with pytest.raises(P.Error) as e:
        P.knapsack_schedule(t, cm, P.Capacities([5], [2]))
    assert e.value.kind == "numeric"
    t = P.ScoreTable(1, 2, [[1.0, 1.0]], [[1.0, 1.0]])
    with pytest.raises(P.Error) as e:
        P.knapsack_schedule(t, cm, P.Capacities([-1], [2]))
    assert e.value.kind == "input"
    with pytest.raises(P.Error) as e:
        P.knapsack_schedule(t, P.CostModel(forward_cost=-1), P.Capacities([1], [2]))
    assert e.value.kind == "config"


def test_knapsack_random_vs_oracle():
    rng = np.random.default_rng(11)
    for trial in range(60):
        K = int(rng.integers(1, 20))
        N = int(rng.integers(1, 300))
        b, f = O.random_score_table(K, N, 500 + trial, zero_prob=0.15 if trial % 2 else 0.0)
        cf = rng.integers(0, 4, K).astype(np.int32)
        cb = rng.integers(0, 4, K).astype(np.int32)
        capf = rng.integers(0, 5 * N + 3, K).astype(np.int32)
        capo = rng.integers(0, 3 * N + 3, K).astype(np.int32)
        cm = P.CostModel(forward_cost_per_device=cf.tolist(), backward_cost_per_device=cb.tolist())
        got = P.knapsack_schedule(_table(b, f), cm, P.Capacities(capf.tolist(), capo.tolist()))
        assert np.array_equal(got.codes, O.knapsack_schedule(b, f, cf, cb, capf, capo)), trial


def test_golden_schedules_bit_exact():
    """Training shapes (tiny, ViT-B 144x64, ViT-L 384x256), the 144x1024 sweep at
    r = 0.25/0.5/0.75/1.0, and heterogeneous costs — against codes produced by
    the unmodified reference (tests/golden/make_golden.py)."""
    g = np.load(os.path.join(GOLDEN, "schedules.npz"))
    for key in [k for k in g.files if k.startswith("codes_")]:
        tag = key[len("codes_"):]
        K, N, seed = (int(v) for v in g["shape_" + tag])
        b, f = O.bench_scores(K, N, seed)
        cm = P.CostModel(forward_cost_per_device=g["cf_" + tag].tolist(),
                         backward_cost_per_device=g["cb_" + tag].tolist())
        caps = P.Capacities(g["capf_" + tag].tolist(), g["capo_" + tag].tolist())
        got = P.knapsack_schedule(_table(b, f), cm, caps)
        assert np.array_equal(got.codes, g[key]), tag


def test_scheduler_context_matches_and_is_deterministic():
    K, N = 144, 64
    b, f = O.bench_scores(K, N, 1)
    nb = (2 * N) // 5
    capf, capo = np.full(K, nb * 5, np.int32), np.full(K, nb * 2, np.int32)
    s = P.Scheduler(K, N, 12, P.scheduler.max_cols_for(2, 3, capf, capo, N))
    ref = O.knapsack_schedule(b, f, 2, 3, capf, capo)
    for _ in range(5):
        assert np.array_equal(s.run(b, f, 2, 3, capf, capo), ref)
    us_dev, us_e2e, codes = s.bench(b, f, 2, 3, capf, capo, warmup=2, iters=10)
    assert np.array_equal(codes, ref) and us_dev > 0 and us_e2e >= us_dev * 0.5


def test_compaction_vs_oracle():
    rng = np.random.default_rng(5)
    for H, L, N in ((4, 2, 16), (12, 12, 64), (16, 3, 256), (12, 12, 1024)):
        codes = rng.integers(1, 4, (H * L, N)).astype(np.uint8)
        got = P.compact(P.ScheduleTable(H * L, N, codes), H)
        ref = O.compact(codes, H)
        for name in ("fwd_cnt", "full_cnt", "act_cnt", "full_hcnt", "fwd_idx", "full_idx", "act_heads",
                     "full_heads"):
            assert np.array_equal(getattr(got, name), ref[name]), (H, L, N, name)


def test_scaler_vs_oracle():
    rng = np.random.default_rng(9)
    cm = P.CostModel()
    for trial in range(30):
        K, N = int(rng.integers(1, 6)), int(rng.integers(1, 40))
        b, f = O.random_score_table(K, N, 900 + trial, zero_prob=0.1)
        tot = rng.integers(0, 6 * N, K).astype(np.int32)
        for mode, sc in ((0, P.ScalerConfig.max()), (1, P.ScalerConfig.min()),
                         (2, P.ScalerConfig.constant(0.05 + trial / 30))):
            got = P.scaler_schedule(_table(b, f), cm, tot, sc)
            codes, lam, fb = O.scaler_schedule(b, f, 2, 3, tot, mode, sc.lam)
            assert np.array_equal(got.table.codes, codes) and got.lambda_used == lam and got.fell_back == fb


def test_merge_exhaustive():
    for n in range(1, 6):
        a = np.array([[(m >> i) & 1 for i in range(n)] for m in range(1 << n)], np.uint8)
        for fb in range(1 << n):
            b = np.array([[(fb >> i) & 1 for i in range(n)]] * (1 << n), np.uint8)
            got = P.merge_selections(a, b).codes
            assert np.array_equal(got, np.where(a == 1, 1, np.where(b == 1, 2, 3)))


def test_brute_force_vs_oracle_and_dominance():
    # test_scheduler.cpp:201-250: exhaustive optimum dominates the bi-level result
    rng = np.random.default_rng(21)
    cm = P.CostModel()
    for trial in range(12):
        K, N = int(rng.integers(1, 4)), int(rng.integers(1, 9))
        b, f = O.random_score_table(K, N, 500 + trial)
        capf = rng.integers(0, 18, K).astype(np.int32)
        capo = rng.integers(0, 7, K).astype(np.int32)
        t = _table(b, f)
        caps = P.Capacities(capf.tolist(), capo.tolist())
        got = P.brute_force_schedule(t, cm, caps)
        assert np.array_equal(got.codes, O.brute_force_schedule(b, f, 2, 3, capf, capo)), trial
        heur = P.knapsack_schedule(t, cm, caps)
        assert np.all(P.schedule_objective(got, t) >= P.schedule_objective(heur, t))
    with pytest.raises(P.Error) as e:
        P.brute_force_schedule(P.ScoreTable(1, 15, np.ones((1, 15)), np.ones((1, 15))), cm, P.Capacities([10], [2]))
    assert e.value.kind == "size"


def test_device_capacities_beyond_context_width_are_refused():
    """device-resident capacities bypass the host width check; a row
    needing more DP columns than the context's max_cols must come back as a
    size error with an all-shortcut row (not a hang or a wrong schedule), and
    the reference's category order must win when several checks fail."""
    import ctypes as C
    import torch
    from paper_2504_12471_b200._lib import lib
    K, N, H = 4, 1600, 4
    h = C.c_void_p()
    assert lib().d2ft_sched_create(K, N, H, 32, C.byref(h)) == 0
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(1)
    b = torch.tensor(rng.uniform(0, 10, (K, N)), device=dev, dtype=torch.float64)
    f = torch.tensor(rng.uniform(0, 10, (K, N)), device=dev, dtype=torch.float64)
    cf = torch.full((K,), 2, device=dev, dtype=torch.int32)
    cb = torch.full((K,), 3, device=dev, dtype=torch.int32)
    capf = torch.tensor([5 * 10, 5 * 1500, 5 * 10, 5 * 10], device=dev, dtype=torch.int32)  # row 1: 1501 columns
    capo = torch.full((K,), 2 * 10, device=dev, dtype=torch.int32)
    codes = torch.zeros((K, N), device=dev, dtype=torch.uint8)
    err = torch.zeros(1, device=dev, dtype=torch.int32)

    def run():
        err.zero_()
        rc = lib().d2ft_sched_run_device(h, C.c_void_p(b.data_ptr()), C.c_void_p(f.data_ptr()),
                                         C.c_void_p(cf.data_ptr()), C.c_void_p(cb.data_ptr()),
                                         C.c_void_p(capf.data_ptr()), C.c_void_p(capo.data_ptr()),
                                         C.c_void_p(codes.data_ptr()), 0, C.c_void_p(err.data_ptr()), None)
        assert rc == 0
        torch.cuda.synchronize()
        return int(err.item()), codes.cpu().numpy()

    e, c = run()
    assert e == 6 and np.all(c[1] == 3)  # kSize, row refused
    ref = O.knapsack_schedule(b.cpu().numpy(), f.cpu().numpy(), 2, 3, capf.cpu().numpy(), capo.cpu().numpy())
    for k in (0, 2, 3):
        assert np.array_equal(c[k], ref[k])
    # several failures in one row: numeric (scores) is reported before input (capacities)
    capf[1] = -5
    b[1, 7] = float("nan")
    e, c = run()
    assert e == 5 and np.all(c[1] == 3)
    b[1, 7] = 1.0
    cf[1] = -1
    e, _ = run()
    assert e == 2  # input (negative capacity) before config (negative cost)
    lib().d2ft_sched_destroy(h)
