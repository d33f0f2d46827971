"""GPU parity of the D2FT step against the fp64 oracle (oracle/model_oracle.py,
itself pinned to the unmodified reference).  Tolerances: tests/step_util.py."""
import numpy as np
import pytest

import paper_2504_12471_b200 as P
from paper_2504_12471_b200 import engine as E
from oracle import lib as O
from oracle import model_oracle as MO

from step_util import FP32_TOL, GRAD_TOL, compare_tensors, normwise, tensor_slices

pytestmark = pytest.mark.gpu


def _cfgs(cfg):
    oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len, cfg.num_classes)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    return oc, sl


def _perturbed_params(cfg, seed=3, scale=0.02):
    """Reference init plus small noise so every bias is nonzero (exercises b1/b2 paths)."""
    p = E.partition_model(cfg)
    return p + scale * np.random.default_rng(seed).standard_normal(p.size)


SMALL = E.ModelConfig(2, 4, 128, 256, 64, 4, 1)      # dh = 32
SMALL64 = E.ModelConfig(2, 2, 128, 256, 50, 4, 5)    # dh = 64, ragged T


@pytest.mark.parametrize("cfg", [SMALL, SMALL64], ids=["dh32", "dh64"])
@pytest.mark.parametrize("colkind", ["full", "mixed", "shortcut"])
def test_forward_backward_parity(cfg, colkind):
    oc, sl = _cfgs(cfg)
    p = _perturbed_params(cfg)
    n = 3
    x, y = E.make_synthetic_dataset(4, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:n], y[:n]
    K = cfg.scheduled_subnet_count()
    if colkind == "full":
        col = np.ones(K, np.uint8)
    elif colkind == "shortcut":
        col = np.full(K, 3, np.uint8)
    else:
        col = np.array([(1, 2, 3)[k % 3] for k in range(K)], np.uint8)
    m = E.SubnetModel(cfg, 4, p)
    loss, g, eng = m.forward_backward(x, y, col)
    rl, rg, reng = MO.forward_backward(oc, p, x.astype(np.float64), y, col)
    assert np.array_equal(eng, reng)
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    bad = compare_tensors(g, rg, sl, GRAD_TOL)
    assert not bad, bad[:8]


@pytest.mark.parametrize("T", [1, 8, 16, 24])
@pytest.mark.parametrize("H", [2, 4], ids=["dh64", "dh32"])
def test_short_sequences_vs_oracle(T, H):
    """Sequences shorter than one 128-row UMMA tile (the tcgen05 attention
    reads its K / V tiles as M = 128 operands): forward/backward parity."""
    cfg = E.ModelConfig(2, H, 128, 256, T, 4, 17)
    oc, sl = _cfgs(cfg)
    p = _perturbed_params(cfg)
    x, y = E.make_synthetic_dataset(4, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    col = np.array([(1, 2, 1, 3)[k % 4] for k in range(K)], np.uint8)
    m = E.SubnetModel(cfg, 4, p)
    loss, g, eng = m.forward_backward(x[:3], y[:3], col)
    rl, rg, reng = MO.forward_backward(oc, p, x[:3].astype(np.float64), y[:3], col)
    assert np.array_equal(eng, reng)
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    # T = 1: softmax over one key is constant, dWq / dWk are exactly 0 in the
    # reference and fp32 cancellation residue (~1e-8) here: absolute check
    bad = compare_tensors(g, rg, sl, GRAD_TOL, skip_zero_ref=False)
    assert not bad, bad[:8]
    m.close()


def test_forward_only_keeps_loss_and_drops_grads():
    # test_model.cpp:326-369: p_o changes no loss vs p_f; grads only for Full
    cfg = SMALL
    p = _perturbed_params(cfg)
    x, y = E.make_synthetic_dataset(4, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    m = E.SubnetModel(cfg, 4, p)
    l_full, _, _ = m.forward_backward(x[:1], y[:1], np.ones(K, np.uint8))
    col = np.ones(K, np.uint8)
    col[1] = 2
    l_mixed, g, eng = m.forward_backward(x[:1], y[:1], col)
    assert l_full == l_mixed  # identical activations, bitwise
    assert eng[2] == 0 and not np.any(g[slice(*E.subnet_slices(cfg)[2])])


@pytest.mark.parametrize("mbs", [1, 2])
def test_step_codes_vs_oracle_trainer(mbs):
    cfg = SMALL
    oc, sl = _cfgs(cfg)
    p = _perturbed_params(cfg)
    n_mb = 4
    B = n_mb * mbs
    x, y = E.make_synthetic_dataset(8, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:B], y[:B]
    K = cfg.scheduled_subnet_count()
    rng = np.random.default_rng(mbs)
    codes = rng.integers(1, 4, (K, n_mb)).astype(np.uint8)
    codes[0, :] = 3  # one subnet never runs Full -> no update, momentum untouched
    m = E.SubnetModel(cfg, B, p)
    for step in range(2):  # two steps exercise the momentum recurrence
        loss = m.step_codes(x, y, codes, mbs, 0.05, 0.9)
        if step == 0:
            pr, vr = p.copy(), np.zeros_like(p)
        rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, codes, mbs, 0.05, 0.9)
        assert abs(loss - rl) <= FP32_TOL * abs(rl), (step, loss, rl)
    pg = m.params()
    p32 = p.astype(np.float32).astype(np.float64)  # the engine keeps fp32 masters
    assert normwise(pg, pr) <= FP32_TOL
    bad = compare_tensors(pg - p32, pr - p, sl, GRAD_TOL)
    assert not bad, bad[:8]
    bad = compare_tensors(m.velocity(), vr, sl, GRAD_TOL)
    assert not bad, bad[:8]
    a, b = E.subnet_slices(cfg)[1]
    assert np.array_equal(pg[a:b], p[a:b].astype(np.float32).astype(np.float64))  # untouched subnet bytes


def test_d2ft_step_schedule_and_numerics():
    """Full D2FT batch at the BASELINE tiny config (2x4, d=128, T=64, B=16):
    bit-exact schedule + in-tolerance numerics vs the oracle trainer."""
    cfg = E.TINY
    oc, sl = _cfgs(cfg)
    p = _perturbed_params(cfg)
    B = 16
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 1)
    nb = (2 * B) // 5
    caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
    m = E.SubnetModel(cfg, B, p)
    loss, table = m.d2ft_step(x, y, P.ScoreTable(K, B, f, b), P.CostModel(), caps, 1, 0.05, 0.9)
    ref_codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
    assert np.array_equal(table.codes, ref_codes)
    pr, vr = p.copy(), np.zeros_like(p)
    rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, ref_codes, 1, 0.05, 0.9)
    assert abs(loss - rl) <= FP32_TOL * abs(rl)
    p32 = p.astype(np.float32).astype(np.float64)
    bad = compare_tensors(m.params() - p32, pr - p, sl, GRAD_TOL)
    assert not bad, bad[:8]


def test_vitb_forward_backward_few_samples():
    """ViT-B/16 dims (12x12, d=768, ffn=3072, T=197), 2 samples, mixed column."""
    cfg = E.VIT_B16
    oc, sl = _cfgs(cfg)
    p = E.partition_model(cfg)
    x, y = E.make_synthetic_dataset(8, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:2], y[:2]
    K = cfg.scheduled_subnet_count()
    col = np.array([(1, 2, 3, 1, 2)[k % 5] for k in range(K)], np.uint8)
    m = E.SubnetModel(cfg, 2, p)
    loss, g, eng = m.forward_backward(x, y, col)
    rl, rg, reng = MO.forward_backward(oc, p, x.astype(np.float64), y, col)
    assert np.array_equal(eng, reng)
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    bad = compare_tensors(g, rg, sl, GRAD_TOL)
    assert not bad, bad[:8]


def test_vitb_full_batch_step_properties():
    """ViT-B/16 batch 64 (BASELINE configs[1]) with ragged random scores: the
    schedule is bit-exact vs the oracle, the step is finite and deterministic
    (two fresh engines give identical bytes)."""
    cfg = E.VIT_B16
    B = 64
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 1)
    nb = (2 * B) // 5
    caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
    st = P.ScoreTable(K, B, f, b)
    outs = []
    for _ in range(2):
        m = E.SubnetModel(cfg, B)
        loss, table = m.d2ft_step(x, y, st, P.CostModel(), caps)
        outs.append((loss, table.codes.copy(), m.params()))
        m.close()
    assert np.array_equal(outs[0][1], O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd))
    assert np.isfinite(outs[0][0]) and outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][2], outs[1][2])


def test_vitl_forward_backward_one_sample():
    """ViT-L/16 dims (BASELINE configs[3]: 24x16, d=1024, ffn=4096, T=197; 16
    heads = the widest head list of the GEMM tile caches), 1 sample, mixed
    column, against the fp64 oracle."""
    cfg = E.VIT_L16
    oc, sl = _cfgs(cfg)
    p = E.partition_model(cfg)
    x, y = E.make_synthetic_dataset(8, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:1], y[:1]
    K = cfg.scheduled_subnet_count()
    col = np.array([(1, 2, 3, 1, 2, 1, 3)[k % 7] for k in range(K)], np.uint8)
    m = E.SubnetModel(cfg, 1, p)
    loss, g, eng = m.forward_backward(x, y, col)
    m.close()
    rl, rg, reng = MO.forward_backward(oc, p, x.astype(np.float64), y, col)
    assert np.array_equal(eng, reng)
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    bad = compare_tensors(g, rg, sl, GRAD_TOL)
    assert not bad, bad[:8]


def test_vitl_batch_step_properties():
    """ViT-L/16 batch 32 with ragged random scores (384 scheduled rows): the
    schedule is bit-exact vs the oracle and the step is finite and
    deterministic across two fresh engines."""
    cfg = E.VIT_L16
    B = 32
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 1)
    nb = (2 * B) // 5
    caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
    st = P.ScoreTable(K, B, f, b)
    outs = []
    for _ in range(2):
        m = E.SubnetModel(cfg, B)
        loss, table = m.d2ft_step(x, y, st, P.CostModel(), caps)
        outs.append((loss, table.codes.copy(), m.params()))
        m.close()
    assert np.array_equal(outs[0][1], O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd))
    assert np.isfinite(outs[0][0]) and outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][2], outs[1][2])


def test_side_stream_schedule_is_bitwise_neutral(monkeypatch):
    """The weight-gradient GEMMs and per-block SGD on the side stream
    (engine default) change only the execution order: two ViT-B D2FT steps
    give bitwise the same weights, momentum and losses as the single-stream
    engine (D2FT_NO_SIDE)."""
    cfg = E.VIT_B16
    B = 16
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 1)
    nb = (2 * B) // 5
    caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("D2FT_NO_SIDE", env)
        else:
            monkeypatch.delenv("D2FT_NO_SIDE", raising=False)
        m = E.SubnetModel(cfg, B)
        losses = [m.d2ft_step(x, y, P.ScoreTable(K, B, f, b), P.CostModel(), caps, 1, 0.05, 0.9)[0] for _ in range(2)]
        out.append((losses, m.params(), m.velocity()))
        m.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])


@pytest.mark.parametrize("cfg", [SMALL, SMALL64], ids=["dh32", "dh64"])
def test_nonfinite_gradient_is_numeric_error(cfg):
    """trainer.cpp:118: a non-finite gradient makes the step fail with a
    numeric error (the reference throws from sgd_momentum_step; its model is
    then partially updated, here every finite element is — in both cases the
    caller restores the parameters).  After set_params the engine steps
    exactly like a fresh one."""
    K = cfg.scheduled_subnet_count()
    B = 4
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    b, f = O.bench_scores(K, B, 2)
    st = P.ScoreTable(K, B, f, b)
    caps = P.Capacities([10] * K, [4] * K)
    m = E.SubnetModel(cfg, B)
    p0 = m.params()
    bad = x.copy()
    bad[1, 3, 5] = np.nan
    with pytest.raises(E.Error) as e:
        m.d2ft_step(bad, y, st, P.CostModel(), caps)
    assert e.value.kind == "numeric"
    bad[1, 3, 5] = np.inf
    with pytest.raises(E.Error) as e:
        m.step_codes(bad, y, np.ones((K, B), np.uint8), 1)
    assert e.value.kind == "numeric"
    m.set_params(p0)
    fresh = E.SubnetModel(cfg, B)
    la, ta = m.d2ft_step(x, y, st, P.CostModel(), caps)
    lb, tb = fresh.d2ft_step(x, y, st, P.CostModel(), caps)
    assert la == lb and np.array_equal(ta.codes, tb.codes) and np.array_equal(m.params(), fresh.params())
    m.close()
    fresh.close()
