"""Oracle parity of the path bench.py times: ViT-B/16 D2FT steps through
`SubnetModel.d2ft_step` (d2ft_engine_step: the captured CUDA graph with the
side stream, tcgen05 attention at dh = 64, ragged per-head sample lists from
U[0,10) scores) against the fp64 trainer body (oracle/model_oracle.py, pinned
to the unmodified reference), plus dh = 64 trainer bodies with random
per-sample codes at mbs 1 and 2.

Bars (tests/step_util.py): gradients / weight updates / momentum normwise
<= 1e-2 per tensor, loss and updated weights <= 1e-3.  The elementwise errors
(entries with |ref| >= 1e-3 max|ref|) are reported beside them
(gpurun_out/parity_report.jsonl)."""
import os

import numpy as np
import pytest

import paper_2504_12471_b200 as P
from paper_2504_12471_b200 import engine as E
from oracle import lib as O
from oracle import model_oracle as MO

from step_util import FP32_TOL, GRAD_TOL, compare_tensors, error_report, normwise, tensor_slices, write_report

pytestmark = pytest.mark.gpu


def _cfgs(cfg):
    oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len, cfg.num_classes)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    return oc, sl


def _workers():
    n = os.cpu_count() or 1
    try:  # ~2.5 GB of fp64 gradient buffers per ViT-B worker
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        n = min(n, max(1, int(avail // (2.5 * 2**30))))
    except (ValueError, OSError):
        pass
    return max(1, min(n, 32))


def _bench_inputs(cfg, B):
    """bench.py's workload(): make_synthetic_dataset(noise 0.5, seed 7), scores
    U[0,10) from make_rng(1, 0) (bench_scheduler.cpp:13-27), budget
    floor(2B/5) p_f + floor(2B/5) p_o per row, cf = 2, cb = 3."""
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 1)
    nb = (2 * B) // 5
    caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
    return x, y, b, f, caps


@pytest.mark.parametrize("B", [64])
def test_vitb_bench_step_vs_oracle(B):
    """BASELINE configs[1] exactly as bench.py runs it (ViT-B/16, batch 64,
    per-sample schedule, reference init): two steps through the graph path,
    each compared with the oracle trainer body on the oracle's own schedule."""
    cfg = E.VIT_B16
    oc, sl = _cfgs(cfg)
    x, y, b, f, caps = _bench_inputs(cfg, B)
    K = cfg.scheduled_subnet_count()
    p0 = E.partition_model(cfg)
    ref_codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
    # oracle first (forked workers, before this process drives the engine)
    pr, vr = p0.copy(), np.zeros_like(p0)
    ref_losses = []
    for _ in range(2):
        rl, _ = MO.train_batch_parallel(oc, pr, vr, x.astype(np.float64), y, ref_codes, 1, 0.05, 0.9,
                                        workers=_workers())
        ref_losses.append(rl)
    m = E.SubnetModel(cfg, B)
    st = P.ScoreTable(K, B, f, b)
    losses = []
    for _ in range(2):
        loss, table = m.d2ft_step(x, y, st, P.CostModel(), caps, 1, 0.05, 0.9)
        assert np.array_equal(table.codes, ref_codes)
        losses.append(loss)
    pg, vg = m.params(), m.velocity()
    m.close()
    for s in range(2):
        assert abs(losses[s] - ref_losses[s]) <= FP32_TOL * abs(ref_losses[s]), (s, losses, ref_losses)
    p32 = p0.astype(np.float32).astype(np.float64)  # the engine keeps fp32 masters
    rep = {"loss_rel": [abs(losses[s] - ref_losses[s]) / abs(ref_losses[s]) for s in range(2)],
           "params_normwise": normwise(pg, pr),
           "update": error_report(pg - p32, pr - p0, sl), "velocity": error_report(vg, vr, sl),
           "cells": {"full": int((ref_codes == 1).sum()), "fwd": int((ref_codes == 2).sum())}}
    write_report(f"vitb_bench_step_B{B}", rep)
    assert normwise(pg, pr) <= FP32_TOL
    bad = compare_tensors(pg - p32, pr - p0, sl, GRAD_TOL)
    assert not bad, bad[:8]
    bad = compare_tensors(vg, vr, sl, GRAD_TOL)
    assert not bad, bad[:8]


def test_vitl_step_vs_oracle():
    """BASELINE configs[3]'s model (ViT-L/16: 24 blocks x 16 heads, d = 1024,
    ffn 4096, T = 197) through the graph path with a ragged bench-style
    schedule (U[0,10) scores, floor(2B/5) p_f + p_o per row), batch 8, one
    step against the oracle trainer body."""
    cfg = E.VIT_L16
    oc, sl = _cfgs(cfg)
    B = 8
    x, y, b, f, caps = _bench_inputs(cfg, B)
    K = cfg.scheduled_subnet_count()
    p0 = E.partition_model(cfg)
    ref_codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
    assert (ref_codes == 1).any() and (ref_codes == 2).any() and (ref_codes == 3).any()
    pr, vr = p0.copy(), np.zeros_like(p0)
    workers = max(1, min(B, _workers() * 2 // 7))  # ~9 GB of fp64 buffers per ViT-L worker
    rl, _ = MO.train_batch_parallel(oc, pr, vr, x.astype(np.float64), y, ref_codes, 1, 0.05, 0.9, workers=workers)
    m = E.SubnetModel(cfg, B)
    loss, table = m.d2ft_step(x, y, P.ScoreTable(K, B, f, b), P.CostModel(), caps, 1, 0.05, 0.9)
    assert np.array_equal(table.codes, ref_codes)
    pg, vg = m.params(), m.velocity()
    m.close()
    assert abs(loss - rl) <= FP32_TOL * abs(rl), (loss, rl)
    p32 = p0.astype(np.float32).astype(np.float64)
    rep = {"loss_rel": abs(loss - rl) / abs(rl), "params_normwise": normwise(pg, pr),
           "update": error_report(pg - p32, pr - p0, sl), "velocity": error_report(vg, vr, sl),
           "cells": {"full": int((ref_codes == 1).sum()), "fwd": int((ref_codes == 2).sum())}}
    write_report("vitl_step_B8", rep)
    assert normwise(pg, pr) <= FP32_TOL
    bad = compare_tensors(pg - p32, pr - p0, sl, GRAD_TOL)
    assert not bad, bad[:8]
    bad = compare_tensors(vg, vr, sl, GRAD_TOL)
    assert not bad, bad[:8]


SMALL64 = E.ModelConfig(2, 2, 128, 256, 50, 4, 5)    # dh = 64 (tcgen05 attention), ragged T
MID64 = E.ModelConfig(3, 4, 256, 1024, 197, 8, 9)    # dh = 64, T = 197 as ViT-B


def _perturbed(cfg, seed=3, scale=0.02):
    p = E.partition_model(cfg)
    return p + scale * np.random.default_rng(seed).standard_normal(p.size)


@pytest.mark.parametrize("cfg", [SMALL64, MID64], ids=["small64", "mid64"])
@pytest.mark.parametrize("mbs", [1, 2])
def test_dh64_trainer_random_codes(cfg, mbs):
    """Trainer body (step_codes: eager, side stream) at dh = 64 with random
    per-micro-batch codes (ragged per-head sample lists through the tcgen05
    attention and the K-gather GEMMs), 1/n_mb accumulation and two SGD steps;
    row 0 never runs Full, so its parameters and momentum must stay untouched."""
    oc, sl = _cfgs(cfg)
    p = _perturbed(cfg)
    n_mb = 6
    B = n_mb * mbs
    x, y = E.make_synthetic_dataset(8 * ((B + 7) // 8), cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:B], y[:B]
    K = cfg.scheduled_subnet_count()
    rng = np.random.default_rng(17 + mbs)
    codes = rng.integers(1, 4, (K, n_mb)).astype(np.uint8)
    codes[0, :] = np.where(codes[0, :] == 1, 2, codes[0, :])  # row 0: forward-only or skipped, never Full
    m = E.SubnetModel(cfg, B, p)
    pr, vr = p.copy(), np.zeros_like(p)
    for step in range(2):
        loss = m.step_codes(x, y, codes, mbs, 0.05, 0.9)
        rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, codes, mbs, 0.05, 0.9)
        assert abs(loss - rl) <= FP32_TOL * abs(rl), (step, loss, rl)
    pg, vg = m.params(), m.velocity()
    m.close()
    p32 = p.astype(np.float32).astype(np.float64)
    write_report(f"dh64_trainer_{cfg.model_dim}_mbs{mbs}",
                 {"update": error_report(pg - p32, pr - p, sl), "velocity": error_report(vg, vr, sl)})
    assert normwise(pg, pr) <= FP32_TOL
    bad = compare_tensors(pg - p32, pr - p, sl, GRAD_TOL)
    assert not bad, bad[:8]
    bad = compare_tensors(vg, vr, sl, GRAD_TOL)
    assert not bad, bad[:8]
    a, b = E.subnet_slices(cfg)[1]
    assert np.array_equal(pg[a:b], p32[a:b]) and not np.any(vg[a:b])  # untouched subnet: p and v keep their bytes


@pytest.mark.parametrize("mbs", [1, 2])
def test_dh64_d2ft_step_graph(mbs):
    """d2ft_step (the graph path with the GPU knapsack) at dh = 64, T = 197,
    mbs 1 and 2, two steps: bit-exact schedule, trainer-body numerics."""
    cfg = MID64
    oc, sl = _cfgs(cfg)
    p = _perturbed(cfg)
    n_mb = 10
    B = n_mb * mbs
    x, y = E.make_synthetic_dataset(8 * ((B + 7) // 8), cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    x, y = x[:B], y[:B]
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, n_mb, 5)
    nb = (2 * n_mb) // 5
    caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
    ref_codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
    m = E.SubnetModel(cfg, B, p)
    pr, vr = p.copy(), np.zeros_like(p)
    for step in range(2):
        loss, table = m.d2ft_step(x, y, P.ScoreTable(K, n_mb, f, b), P.CostModel(), caps, mbs, 0.05, 0.9)
        assert np.array_equal(table.codes, ref_codes)
        rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, ref_codes, mbs, 0.05, 0.9)
        assert abs(loss - rl) <= FP32_TOL * abs(rl), (step, loss, rl)
    pg, vg = m.params(), m.velocity()
    m.close()
    p32 = p.astype(np.float32).astype(np.float64)
    write_report(f"dh64_d2ft_step_mbs{mbs}",
                 {"update": error_report(pg - p32, pr - p, sl), "velocity": error_report(vg, vr, sl)})
    bad = compare_tensors(pg - p32, pr - p, sl, GRAD_TOL)
    assert not bad, bad[:8]
    bad = compare_tensors(vg, vr, sl, GRAD_TOL)
    assert not bad, bad[:8]

