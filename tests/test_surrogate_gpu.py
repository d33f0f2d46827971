"""GPU: the opt-in p_s surrogate (BASELINE north_star "skip-with-linear-
surrogate ... surrogate heads run as one small dense GEMM"; csrc
step_gemms.cuh Sur1 / Sur2) against the fp64 oracle extended with the same
definition (oracle/model_oracle.forward_backward(surrogate=...)).  The
reference's p_s is a pure bypass (model.cpp:326-328, 458); rank 0 — the
default — must keep it bit for bit."""
import numpy as np
import pytest

import paper_2504_12471_b200 as P
from paper_2504_12471_b200 import engine as E
from oracle import lib as O
from oracle import model_oracle as MO

from step_util import FP32_TOL, GRAD_TOL, compare_tensors, tensor_slices

pytestmark = pytest.mark.gpu

SMALL = E.ModelConfig(2, 4, 128, 256, 64, 4, 1)      # dh = 32
SMALL64 = E.ModelConfig(2, 2, 128, 256, 50, 4, 5)    # dh = 64, ragged T


def _oc(cfg):
    return MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                     cfg.num_classes)


def _factors(cfg, rank, seed=9, scale=0.05):
    return scale * np.random.default_rng(seed).standard_normal(cfg.scheduled_subnet_count() * 2 * cfg.model_dim * rank)


@pytest.mark.parametrize("cfg", [SMALL, SMALL64], ids=["dh32", "dh64"])
@pytest.mark.parametrize("rank", [8, 16])
def test_surrogate_forward_backward_vs_oracle(cfg, rank):
    oc = _oc(cfg)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    p = E.partition_model(cfg) + 0.02 * np.random.default_rng(3).standard_normal(E.param_count(cfg))
    x, y = E.make_synthetic_dataset(4, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    col = np.array([(3, 1, 2, 3)[k % 4] for k in range(K)], np.uint8)
    fac = _factors(cfg, rank)
    m = E.SubnetModel(cfg, 4, p)
    m.set_surrogate(rank, fac)
    loss, g, eng = m.forward_backward(x[:3], y[:3], col)
    rl, rg, reng = MO.forward_backward(oc, p, x[:3].astype(np.float64), y[:3], col, surrogate=(rank, fac))
    rl0, _, _ = MO.forward_backward(oc, p, x[:3].astype(np.float64), y[:3], col)
    assert abs(rl - rl0) > 1e-3 * abs(rl0)  # the surrogate changes the loss measurably
    assert np.array_equal(eng, reng)
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    bad = compare_tensors(g, rg, sl, GRAD_TOL)
    assert not bad, bad[:8]
    # rank 0: the reference's bypass again, bit for bit
    m.set_surrogate(0)
    l0, g0, _ = m.forward_backward(x[:3], y[:3], col)
    fresh = E.SubnetModel(cfg, 4, p)
    l1, g1, _ = fresh.forward_backward(x[:3], y[:3], col)
    assert l0 == l1 and np.array_equal(g0, g1)
    m.close()
    fresh.close()


def test_surrogate_d2ft_step_vs_oracle_trainer():
    """The batch body with the surrogate on: per-sample ragged schedule from
    the GPU knapsack, 4 micro-batches, SGD — against the oracle trainer."""
    cfg = SMALL64
    oc = _oc(cfg)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    rank = 16
    fac = _factors(cfg, rank, seed=12)
    B = 4
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 5)
    caps = P.Capacities([5] * K, [2] * K)  # 1 Full + 1 forward-only + 2 p_s per row
    m = E.SubnetModel(cfg, B)
    m.set_surrogate(rank, fac)
    p0 = m.params()
    loss, table = m.d2ft_step(x, y, P.ScoreTable(K, B, f, b), P.CostModel(), caps, 1, 0.05, 0.9)
    codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
    assert np.array_equal(table.codes, codes) and np.any(codes == 3)
    pr, vr = p0.copy(), np.zeros_like(p0)
    rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, codes, 1, 0.05, 0.9, surrogate=(rank, fac))
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    bad = compare_tensors(m.params() - p0, pr - p0, sl, GRAD_TOL)
    assert not bad, bad[:8]
    m.close()


def test_surrogate_errors():
    cfg = SMALL64
    m = E.SubnetModel(cfg, 2)
    for r in (4, 12, 72):
        with pytest.raises(E.Error) as e:
            m.set_surrogate(r, _factors(cfg, r))
        assert e.value.kind == "config"
    with pytest.raises(E.Error) as e:
        m.set_surrogate(8, np.zeros(5))
    assert e.value.kind == "dimension"
    m.close()
