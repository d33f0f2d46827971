"""GPU scoring pre-pass (prepass_scores, scoring.cpp:108-151) against the fp64
oracle restatement (oracle/model_oracle.prepass_scores): every metric of every
scheduled head-subnet and unit.  Tolerance: 1e-2 relative per entry for the
gradient metrics (north_star's gradient bar; fp16 GEMM operands, per-unit
gradients — not averaged over a batch; achieved <= 1.7e-3, LoRA Fisher the
largest, profiles/r2_prepass_errors.jsonl), 1e-5 for WeightMagnitude (fp32
masters)."""
import json
import os

import numpy as np
import pytest

from paper_2504_12471_b200 import engine as E
from oracle import model_oracle as MO

pytestmark = pytest.mark.gpu

SMALL = E.ModelConfig(2, 4, 128, 256, 64, 4, 1)      # dh = 32 (mma.sync attention)
SMALL64 = E.ModelConfig(2, 2, 128, 256, 50, 4, 5)    # dh = 64 (tcgen05 attention), ragged T


def _report(case, metric, rel):
    """Achieved error beside the assertion (gpurun_out/prepass_errors.jsonl)."""
    rec = {"case": case, "metric": metric, "max_rel": float(rel.max()), "p99": float(np.percentile(rel, 99))}
    print(json.dumps(rec))
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "prepass_errors.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")


def _oc(cfg):
    return MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                     cfg.num_classes)


def _check(cfg, n, mbs, nsamp_data=8):
    p = E.partition_model(cfg) + 0.02 * np.random.default_rng(5).standard_normal(E.param_count(cfg))
    x, y = E.make_synthetic_dataset(nsamp_data, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:n], y[:n]
    m = E.SubnetModel(cfg, n, p)
    before = m.params()
    for fm, bm in (("fisher_information", "weight_magnitude"), ("gradient_magnitude", "taylor_importance")):
        t = m.prepass_scores(x, y, mbs, fm, bm)
        rf, rb = MO.prepass_scores(_oc(cfg), p, x.astype(np.float64), y, mbs, fm, bm)
        for got, ref, metric in ((t.forward, rf, fm), (t.backward, rb, bm)):
            tol = 1e-5 if metric == "weight_magnitude" else 1e-2
            rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)
            _report(f"L{cfg.num_blocks}H{cfg.heads_per_block}d{cfg.model_dim}T{cfg.seq_len} n{n} mbs{mbs}", metric, rel)
            assert rel.max() <= tol, (metric, rel.max(), np.unravel_index(rel.argmax(), rel.shape))
    assert np.array_equal(m.params(), before)  # no update (scoring.hpp:46-47)
    m.close()


@pytest.mark.parametrize("cfg", [SMALL, SMALL64], ids=["dh32", "dh64"])
@pytest.mark.parametrize("n,mbs", [(4, 1), (4, 2)])
def test_prepass_matches_oracle(cfg, n, mbs):
    _check(cfg, n, mbs)


def test_prepass_vitb_two_samples():
    _check(E.VIT_B16, 2, 1)


def test_prepass_feeds_the_step():
    """The pre-pass table drives a D2FT step end to end (scores -> knapsack -> step)."""
    from paper_2504_12471_b200 import scheduler as S
    cfg = SMALL64
    x, y = E.make_synthetic_dataset(8, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    m = E.SubnetModel(cfg, 8)
    t = m.prepass_scores(x, y, 1)
    K = cfg.scheduled_subnet_count()
    caps = S.Capacities([3 * 5] * K, [3 * 2] * K)
    loss, table = m.d2ft_step(x, y, t, S.CostModel(), caps)
    assert np.isfinite(loss)
    assert np.array_equal(table.codes, S.knapsack_schedule(t, S.CostModel(), caps).codes)
    m.close()


@pytest.mark.parametrize("cfg", [SMALL, SMALL64], ids=["dh32", "dh64"])
@pytest.mark.parametrize("mbs", [1, 2])
def test_prepass_lora_matches_oracle(cfg, mbs):
    """LoRA-mode pre-pass (scoring.cpp:108-151 with lora_enabled(): metrics
    over the adapter tensors, oracle pinned to the reference in
    test_oracle_pins.py::test_oracle_lora_prepass_matches_reference)."""
    rank, scaling = 4, 0.5
    p = E.partition_model(cfg) + 0.02 * np.random.default_rng(5).standard_normal(E.param_count(cfg))
    ad = E.lora_init(cfg, rank) + 0.05 * np.random.default_rng(6).standard_normal(
        E.lora_init(cfg, rank).size)
    n = 4
    x, y = E.make_synthetic_dataset(8, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:n], y[:n]
    m = E.SubnetModel(cfg, n, p)
    m.attach_lora(rank, scaling, ad)
    before, abefore = m.params(), m.lora_params()
    for fm, bm in (("fisher_information", "weight_magnitude"), ("gradient_magnitude", "taylor_importance")):
        t = m.prepass_scores(x, y, mbs, fm, bm)
        rf, rb = MO.prepass_scores_lora(_oc(cfg), p, rank, scaling, ad, x.astype(np.float64), y, mbs, fm, bm)
        for got, ref, metric in ((t.forward, rf, fm), (t.backward, rb, bm)):
            tol = 1e-5 if metric == "weight_magnitude" else 1e-2
            rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)
            _report(f"lora L{cfg.num_blocks}H{cfg.heads_per_block}d{cfg.model_dim} mbs{mbs}", metric, rel)
            assert rel.max() <= tol, (metric, rel.max(), np.unravel_index(rel.argmax(), rel.shape))
    assert np.array_equal(m.params(), before) and np.array_equal(m.lora_params(), abefore)
    m.close()
