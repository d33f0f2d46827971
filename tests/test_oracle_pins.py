"""Pin the CPU oracle (oracle/sched_oracle.c, oracle/model_oracle.py) before
trusting it: the literal expectations of the reference's own tests, the
committed golden vectors made from the unmodified reference, and (when it is
built here) oracle/_ref byte-for-byte.  CPU only."""
import itertools
import os

import numpy as np
import pytest

from oracle import lib as O
from oracle import model_oracle as MO

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- test_scheduler.cpp literals
def test_dp_search_known_answers():
    # test_scheduler.cpp:62-87
    sel, obj = O.dp_search([[5.0, 4.0]], [[2, 2]], [0])
    assert obj[0] == 0.0 and sel[0].tolist() == [0, 0]
    sel, obj = O.dp_search([[5.0, 4.0, 3.0]], [[2, 2, 2]], [4])
    assert obj[0] == 9.0 and sel[0].tolist() == [1, 1, 0]
    with pytest.raises(O.OracleError) as e:
        O.dp_search([[1.0]], [[1]], [-1])
    assert e.value.code == 2
    with pytest.raises(O.OracleError) as e:
        O.dp_search([[np.nan]], [[1]], [1])
    assert e.value.code == 5
    sel, _ = O.dp_search([[2.0] * 5], [[5] * 5], [15])
    assert sel[0].tolist() == [1, 1, 1, 0, 0]


def _subset_best(scores, weights, cap):  # oracles.cpp:491-507
    best = 0.0
    n = len(scores)
    for mask in range(1 << n):
        w = 0
        v = 0.0
        for i in range(n):
            if mask >> i & 1:
                w += weights[i]
                v += scores[i]
        if w <= cap and v > best:
            best = v
    return best


def test_dp_search_exact_vs_enumeration():
    # test_scheduler.cpp:89-115 style: random instances, exact objective
    rng = np.random.default_rng(2024)
    for _ in range(60):
        n = int(rng.integers(1, 12))
        s = rng.random(n) * 9.0
        w = rng.integers(1, 8, n)
        cap = int(rng.integers(0, 25))
        sel, obj = O.dp_search([s], [w], [cap])
        assert obj[0] == _subset_best(list(s), list(w), cap)
        assert float(np.sum(s[sel[0] == 1])) == obj[0] or abs(float(np.sum(s[sel[0] == 1])) - obj[0]) < 1e-12
        assert int(np.sum(w[sel[0] == 1])) <= cap


def test_merge_rules_exhaustive():
    # acceptance crit. 7 (acceptance_main.cpp:304-330), N <= 4 here
    for n in range(1, 5):
        for fa, fb in itertools.product(range(1 << n), repeat=2):
            a = np.array([[(fa >> i) & 1 for i in range(n)]], np.uint8)
            b = np.array([[(fb >> i) & 1 for i in range(n)]], np.uint8)
            c = O.merge_selections(a, b)
            exp = np.where(a == 1, 1, np.where(b == 1, 2, 3))
            assert np.array_equal(c, exp)


def test_knapsack_merge_cases():
    # test_scheduler.cpp:133-164
    c = O.knapsack_schedule([[5.0, 1.0]], [[9.0, 1.0]], 2, 3, [5], [2])
    assert c.tolist() == [[1, 3]]
    c = O.knapsack_schedule([[9.0, 1.0, 1.0]], [[0.0, 8.0, 1.0]], 2, 3, [5], [2])
    assert c.tolist() == [[1, 2, 3]]
    b, f = O.random_score_table(3, 5, 1)
    c = O.knapsack_schedule(b, f, 2, 3, [0, 0, 0], [0, 0, 0])
    assert np.all(c == 3)


def test_constant_scores_lowest_index_fill():
    # test_scheduler.cpp:385-403
    b = np.array([[7.0] * 5, [1.5] * 5])
    f = np.zeros((2, 5))
    c = O.knapsack_schedule(b, f, 2, 3, [15, 15], [0, 0])
    assert c.tolist() == [[1, 1, 1, 3, 3]] * 2


def test_scaler_lambda_zero_counts():
    # test_scheduler.cpp:276-283: 12 units fit two full ops plus one forward-only
    b, f = O.random_score_table(1, 5, 42)
    c, lam, fb = O.scaler_schedule(b, f, 2, 3, [12], 2, 1e-12)
    assert (c == 1).sum() == 2 and (c == 2).sum() == 1 and not fb


def test_scaler_all_zero_fallback():
    c, lam, fb = O.scaler_schedule(np.zeros((1, 3)), np.zeros((1, 3)), 2, 3, [10], 0)
    assert fb and lam == 1.0


def test_shared_budget_accounting():
    # test_scheduler.cpp:405-418
    codes = np.array([[1, 1, 1, 1], [3, 3, 3, 3]], np.uint8)
    assert O.oracle_lib().or_row_cost_units(O._ptr(np.ascontiguousarray(codes[0])), 4, 2, 3) == 20


# ---------------------------------------------------------------- golden vectors (made from oracle/_ref)
def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing")
    return np.load(path)


def test_golden_schedules():
    g = _golden("schedules.npz")
    for key in [k for k in g.files if k.startswith("codes_")]:
        tag = key[len("codes_"):]
        K, N, seed = (int(v) for v in g["shape_" + tag])
        b, f = O.bench_scores(K, N, seed)
        c = O.knapsack_schedule(b, f, g["cf_" + tag], g["cb_" + tag], g["capf_" + tag], g["capo_" + tag])
        assert np.array_equal(c, g[key]), tag


def test_golden_dp():
    g = _golden("dp_search.npz")
    sel, obj = O.dp_search(g["scores"], g["weights"], g["caps"])
    assert np.array_equal(sel, g["sel"])
    assert np.array_equal(obj, g["obj"])


def test_golden_rng_and_init():
    g = _golden("rng_init.npz")
    assert np.array_equal(O.uniform_stream(1, 0, 64), g["uniform_1_0"])
    assert np.array_equal(O.shuffle_iota(3, 0xE000, 40), g["shuffle_3_E000"])
    p = O.partition_model(2, 4, 32, 64, 16, 4, 1)
    assert np.array_equal(p, g["params_tiny32"])
    x, lab = O.make_dataset(8, 4, 32, 16, 0.5, 7)
    assert np.array_equal(x, g["data_x"]) and np.array_equal(lab, g["data_y"])


def test_golden_model_step():
    g = _golden("model_step.npz")
    cfg = MO.Config(*[int(v) for v in g["cfg"]])
    p = g["params"].copy()
    v = np.zeros_like(p)
    loss, _ = MO.train_batch(cfg, p, v, g["x"], g["y"], g["codes"], 1, 0.05, 0.9)
    assert abs(loss - float(g["loss"])) <= 1e-12 * max(1.0, abs(float(g["loss"])))
    assert np.max(np.abs(p - g["params_after"])) <= 1e-12
    loss1, gr, eng = MO.forward_backward(cfg, g["params"], g["x"][:2], g["y"][:2], g["codes"][:, 0])
    assert np.max(np.abs(gr - g["fb_grads"])) <= 1e-12 * max(1.0, np.max(np.abs(g["fb_grads"])))
    assert np.array_equal(eng, g["fb_engaged"])


# ---------------------------------------------------------------- against oracle/_ref (built here)
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built on this host")


@needs_ref
def test_oracle_matches_reference_scheduler_random():
    rng = np.random.default_rng(7)
    for trial in range(40):
        K = int(rng.integers(1, 7))
        N = int(rng.integers(1, 40))
        b, f = O.random_score_table(K, N, 100 + trial, zero_prob=0.2 if trial % 2 else 0.0)
        cf, cb = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        capf = rng.integers(0, 5 * N, K).astype(np.int32)
        capo = rng.integers(0, 3 * N, K).astype(np.int32)
        assert np.array_equal(O.knapsack_schedule(b, f, cf, cb, capf, capo),
                              O.ref_knapsack_schedule(b, f, cf, cb, capf, capo))
        w = rng.integers(0, 8, (K, N)).astype(np.int32)
        s1, o1 = O.dp_search(b, w, capf)
        s2, o2 = O.ref_dp_search(b, w, capf)
        assert np.array_equal(s1, s2) and np.array_equal(o1, o2)
        tot = (capf + capo).astype(np.int32)
        for mode in (0, 1, 2):
            c1 = O.scaler_schedule(b, f, cf, cb, tot, mode, 0.37)
            c2 = O.ref_scaler_schedule(b, f, cf, cb, tot, mode, 0.37)
            assert np.array_equal(c1[0], c2[0]) and c1[1] == c2[1] and c1[2] == c2[2]
        if N <= 7:
            assert np.array_equal(O.brute_force_schedule(b, f, cf, cb, capf, capo),
                                  O.ref_brute_force_schedule(b, f, cf, cb, capf, capo))


@needs_ref
def test_oracle_matches_reference_model():
    cfg = MO.Config(2, 4, 32, 64, 16, 4)
    r = O.RefModel(2, 4, 32, 64, 16, 4, 1)
    p = O.partition_model(2, 4, 32, 64, 16, 4, 1)
    assert np.array_equal(p, r.params())
    rng = np.random.default_rng(0)
    p = p + 0.05 * rng.standard_normal(p.size)
    r.set_params(p)
    x, y = O.make_dataset(4, 4, 32, 16, 0.5, 7)
    col = np.array([1, 2, 3, 1, 1, 1, 2, 3], np.uint8)
    l1, g1, e1 = MO.forward_backward(cfg, p, x[:2], y[:2], col)
    l2, g2, e2 = r.forward_backward(x[:2], y[:2], col)
    assert abs(l1 - l2) < 1e-12 and np.max(np.abs(g1 - g2)) < 1e-12 and np.array_equal(e1, e2)


@needs_ref
@pytest.mark.parametrize("mbs", [1, 2])
def test_oracle_prepass_matches_reference(mbs):
    """The numpy restatement of prepass_scores / metric_value (model_oracle.py)
    against the unmodified reference's prepass_scores (scoring.cpp:108-151),
    all four metrics, on a perturbed model."""
    cfg = MO.Config(2, 4, 32, 64, 16, 4)
    r = O.RefModel(2, 4, 32, 64, 16, 4, 1)
    p = O.partition_model(2, 4, 32, 64, 16, 4, 1) + 0.05 * np.random.default_rng(1).standard_normal(r.n)
    r.set_params(p)
    x, y = O.make_dataset(4, 4, 32, 16, 0.5, 7)
    for fi, bi in ((0, 1), (2, 3)):
        rf, rb = r.prepass_scores(x, y, mbs, fi, bi, threads=2)
        of, ob = MO.prepass_scores(cfg, p, x, y, mbs, MO.METRICS[fi], MO.METRICS[bi])
        assert np.allclose(of, rf, rtol=1e-10, atol=0) and np.allclose(ob, rb, rtol=1e-10, atol=0)
    assert np.array_equal(r.params(), p)  # no update


def _split_lora(cfg, rank, flat):
    """The reference's canonical vector with adapters (visit_tensors: each
    block's base tensors, then its six adapter matrices) -> (base, adapters)."""
    sl = MO.subnet_slices(cfg)
    lb = MO.lora_block_size(cfg, rank)
    base, ad, off = [], [], 0
    for si, (a, b) in enumerate(sl):
        n = b - a
        base.append(flat[off:off + n])
        off += n
        if 1 <= si <= cfg.K:
            ad.append(flat[off:off + lb])
            off += lb
    assert off == flat.size
    return np.concatenate(base), np.concatenate(ad)


def _join_lora(cfg, rank, base, ad):
    sl = MO.subnet_slices(cfg)
    lb = MO.lora_block_size(cfg, rank)
    parts = []
    for si, (a, b) in enumerate(sl):
        parts.append(base[a:b])
        if 1 <= si <= cfg.K:
            parts.append(ad[(si - 1) * lb:si * lb])
    return np.concatenate(parts)


@needs_ref
def test_oracle_lora_matches_reference():
    """LoRA: attach_lora's init (model.cpp:165-195), the
    adapter forward/backward (model.cpp:204-211, 273-302) and the LoRA trainer
    step (adapters only, trainer.cpp:124-133) of the numpy restatement against
    the unmodified reference."""
    cfg = MO.Config(2, 4, 32, 64, 16, 4)
    rank, scaling = 4, 0.5
    r = O.RefModel(2, 4, 32, 64, 16, 4, 1)
    p = O.partition_model(2, 4, 32, 64, 16, 4, 1) + 0.05 * np.random.default_rng(2).standard_normal(r.n)
    r.set_params(p)
    r.attach_lora(rank, scaling)
    base, ad = _split_lora(cfg, rank, r.params())
    assert np.array_equal(base, p)
    assert np.array_equal(ad, MO.lora_init(cfg, rank, 1))  # down = 0, up ~ N(0, 1/rank), same streams
    ad = ad + 0.05 * np.random.default_rng(3).standard_normal(ad.size)  # nonzero down: every term live
    r.set_params(_join_lora(cfg, rank, p, ad))
    x, y = O.make_dataset(4, 4, 32, 16, 0.5, 7)
    col = np.array([1, 2, 3, 1, 1, 1, 2, 3], np.uint8)
    l1, ga, e1 = MO.forward_backward(cfg, p, x[:2], y[:2], col, lora=(rank, scaling, ad))
    l2, g2, e2 = r.forward_backward(x[:2], y[:2], col)
    gb2, ga2 = _split_lora(cfg, rank, g2)
    assert abs(l1 - l2) < 1e-12 and np.array_equal(e1, e2)
    assert np.max(np.abs(ga - ga2)) < 1e-12
    assert not np.any(gb2)  # base tensors frozen: no gradient
    codes = np.array([[1, 2], [3, 1], [1, 1], [2, 3], [3, 3], [1, 3], [2, 2], [1, 1]], np.uint8)
    a_o, v_o = ad.copy(), np.zeros_like(ad)
    for _ in range(2):
        lr_ = r.train_batch(x, y, codes, 2, 0.05, 0.9)
        lo, _ = MO.train_batch_lora(cfg, p, rank, scaling, a_o, v_o, x, y, codes, 2, 0.05, 0.9)
        assert abs(lo - lr_) < 1e-12
    b3, a3 = _split_lora(cfg, rank, r.params())
    assert np.array_equal(b3, p)  # base frozen
    assert np.max(np.abs(a3 - a_o)) < 1e-12
    _, v3 = _split_lora(cfg, rank, r.velocity())
    assert np.max(np.abs(v3 - v_o)) < 1e-12


@needs_ref
def test_oracle_lora_prepass_matches_reference():
    """prepass_scores in LoRA mode (scoring.cpp:108-151 with lora_enabled():
    the metrics walk the adapter tensors only) of the numpy restatement
    against the unmodified reference, every metric pair."""
    cfg = MO.Config(2, 4, 32, 64, 16, 4)
    rank, scaling = 4, 0.5
    r = O.RefModel(2, 4, 32, 64, 16, 4, 1)
    p = O.partition_model(2, 4, 32, 64, 16, 4, 1) + 0.05 * np.random.default_rng(2).standard_normal(r.n)
    r.set_params(p)
    r.attach_lora(rank, scaling)
    _, ad = _split_lora(cfg, rank, r.params())
    ad = ad + 0.05 * np.random.default_rng(4).standard_normal(ad.size)
    r.set_params(_join_lora(cfg, rank, p, ad))
    x, y = O.make_dataset(4, 4, 32, 16, 0.5, 7)
    for mbs in (1, 2):
        for fi, bi in ((0, 1), (2, 3)):
            rf, rb = r.prepass_scores(x, y, mbs, fi, bi)
            of, ob = MO.prepass_scores_lora(cfg, p, rank, scaling, ad, x, y, mbs, MO.METRICS[fi], MO.METRICS[bi])
            assert np.allclose(of, rf, rtol=1e-10, atol=0) and np.allclose(ob, rb, rtol=1e-10, atol=0)


def test_parallel_trainer_matches_serial():
    """train_batch_parallel (the forked-worker oracle of the batch-64 ViT-B
    parity test) equals the serial trainer body up to fp64 re-association."""
    cfg = MO.Config(2, 2, 16, 32, 8, 4)
    rng = np.random.default_rng(5)
    flat = rng.standard_normal(MO.param_count(cfg)) * 0.3
    x = rng.standard_normal((12, cfg.T, cfg.d))
    y = np.arange(12) % cfg.C
    codes = rng.integers(1, 4, (cfg.K, 6)).astype(np.uint8)
    codes[1, :] = 3
    p1, v1 = flat.copy(), np.zeros_like(flat)
    p2, v2 = flat.copy(), np.zeros_like(flat)
    for _ in range(2):
        l1, t1 = MO.train_batch(cfg, p1, v1, x, y, codes, 2, 0.05, 0.9)
        l2, t2 = MO.train_batch_parallel(cfg, p2, v2, x, y, codes, 2, 0.05, 0.9, workers=3)
        assert l1 == l2 and np.array_equal(t1, t2)
    assert np.max(np.abs(p1 - p2)) <= 1e-13 and np.max(np.abs(v1 - v2)) <= 1e-13
