"""GPU: the head-partitioned step on one B200.

`world` engines form an in-process head partition (partition.LocalGroup, the
exchange is a fixed-order device sum) and step the same batch from host
threads.  The owner-merged parameters, the velocity and the loss must match
the whole-model engine and the fp64 oracle trainer to the step tolerances
(tests/step_util.py); the schedule each rank derives is bit-identical to the
oracle's.  The NCCL exchange is exercised at world 1 (the driver's boxes have
one GPU); its multi-rank path shares every line but the all-reduce call."""
import os
import socket

import numpy as np
import pytest

from paper_2504_12471_b200 import engine as E
from paper_2504_12471_b200 import partition as PT
from paper_2504_12471_b200.scheduler import Capacities, CostModel, ScoreTable
from oracle import lib as O
from oracle import model_oracle as MO

from step_util import FP32_TOL, GRAD_TOL, compare_tensors, normwise, tensor_slices

pytestmark = pytest.mark.gpu

SMALL = E.ModelConfig(2, 4, 128, 256, 64, 4, 1)  # dh = 32


def _setup(cfg, B, seed=3):
    p = E.partition_model(cfg)
    p = p + 0.02 * np.random.default_rng(seed).standard_normal(p.size)
    x, y = E.make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    return p, x, y


@pytest.mark.parametrize("world", [2, 3])
def test_local_partition_step_codes_matches_oracle(world):
    cfg = SMALL
    oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len, cfg.num_classes)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    n_mb, mbs = 4, 1
    B = n_mb * mbs
    p, x, y = _setup(cfg, B)
    K = cfg.scheduled_subnet_count()
    codes = np.random.default_rng(world).integers(1, 4, (K, n_mb)).astype(np.uint8)
    g = PT.LocalGroup([E.SubnetModel(cfg, B, p) for _ in range(world)])
    try:
        losses = []
        pr, vr = p.copy(), np.zeros_like(p)
        for step in range(2):
            ls = g.run(lambda r, m: m.step_codes(x, y, codes, mbs, 0.05, 0.9))
            rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, codes, mbs, 0.05, 0.9)
            assert len(set(ls)) == 1, ls  # every rank sees the same exchanged activations
            assert abs(ls[0] - rl) <= FP32_TOL * abs(rl), (step, ls[0], rl)
            losses.append(ls[0])
        merged = PT.merge_owned(cfg, [m.params() for m in g.models])
        vel = PT.merge_owned(cfg, [m.velocity() for m in g.models])
        p32 = p.astype(np.float32).astype(np.float64)
        assert normwise(merged, pr) <= FP32_TOL
        bad = compare_tensors(merged - p32, pr - p, sl, GRAD_TOL)
        assert not bad, bad[:8]
        bad = compare_tensors(vel, vr, sl, GRAD_TOL)
        assert not bad, bad[:8]
    finally:
        g.close()


def test_local_partition_matches_whole_model_engine():
    """world 2 vs one engine on the BASELINE tiny config with the GPU schedule:
    same codes, and parameters equal to fp32 summation-order noise."""
    cfg = E.TINY
    B = 16
    p, x, y = _setup(cfg, B, 5)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 1)
    nb = (2 * B) // 5
    caps = Capacities([nb * 5] * K, [nb * 2] * K)
    st = ScoreTable(K, B, f, b)
    whole = E.SubnetModel(cfg, B, p)
    lw, tw = whole.d2ft_step(x, y, st, CostModel(), caps, 1, 0.05, 0.9)
    g = PT.LocalGroup([E.SubnetModel(cfg, B, p) for _ in range(2)])
    try:
        res = g.run(lambda r, m: m.d2ft_step(x, y, st, CostModel(), caps, 1, 0.05, 0.9))
        for lr_, tr in res:
            assert np.array_equal(tr.codes, tw.codes)  # every rank derives the global table
            assert abs(lr_ - lw) <= 1e-5 * abs(lw)
        merged = PT.merge_owned(cfg, [m.params() for m in g.models])
        pw = whole.params()
        p32 = p.astype(np.float32).astype(np.float64)
        assert normwise(merged - p32, pw - p32) <= 1e-3
        busy, ratio = PT.busy_units(tw.codes, cfg.heads_per_block, 2)
        assert busy.sum() > 0 and ratio >= 1.0
    finally:
        g.close()
        whole.close()


def test_nccl_partition_world1_is_the_whole_model():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        cfg = SMALL
        B = 4
        p, x, y = _setup(cfg, B)
        K = cfg.scheduled_subnet_count()
        codes = np.random.default_rng(9).integers(1, 4, (K, B)).astype(np.uint8)
        a = E.SubnetModel(cfg, B, p)
        m = E.SubnetModel(cfg, B, p)
        PT.join_nccl(m, PT.HeadPartition(cfg.heads_per_block, 0, 1))
        la = a.step_codes(x, y, codes, 1, 0.05, 0.9)
        lm = m.step_codes(x, y, codes, 1, 0.05, 0.9)
        assert la == lm
        assert np.array_equal(a.params(), m.params())
        assert np.array_equal(PT.gather_params(m, m.partition), m.params())
        a.close()
        m.close()
    finally:
        dist.destroy_process_group()
