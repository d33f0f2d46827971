"""GPU: the head-partitioned step on one B200.

`world` engines form an in-process head partition (partition.LocalGroup, the
exchange is a fixed-order device sum) and step the same batch from host
threads.  The owner-merged parameters, the velocity and the loss must match
the whole-model engine and the fp64 oracle trainer to the step tolerances
(tests/step_util.py); the schedule each rank derives is bit-identical to the
oracle's — for both row mappings (head-interleaved, SPEC-contiguous) and 1-3
exchange chunks.  The NCCL exchange runs at world 1 (the driver's boxes have
one GPU): the partitioned data path (owner mask, fp32 partial sums, one
ncclAllReduce per block, direction and chunk on the exchange stream, captured
in the step's CUDA graph) executes and is compared with the whole-model
engine and the oracle."""
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


@pytest.mark.parametrize("world,mapping,chunks", [(2, "heads", 1), (2, "heads", 2), (3, "heads", 3),
                                                  (2, "contiguous", 2), (3, "contiguous", 1)])
def test_local_partition_step_codes_matches_oracle(world, mapping, chunks):
    cfg = SMALL
    oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len, cfg.num_classes)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    n_mb, mbs = 4, 1
    B = n_mb * mbs
    p, x, y = _setup(cfg, B)
    K = cfg.scheduled_subnet_count()
    codes = np.random.default_rng(world).integers(1, 4, (K, n_mb)).astype(np.uint8)
    g = PT.LocalGroup([E.SubnetModel(cfg, B, p) for _ in range(world)], mapping, chunks)
    try:
        losses = []
        pr, vr = p.copy(), np.zeros_like(p)
        for step in range(2):
            ls = g.run(lambda r, m: m.step_codes(x, y, codes, mbs, 0.05, 0.9))
            rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, codes, mbs, 0.05, 0.9)
            assert len(set(ls)) == 1, ls  # every rank sees the same exchanged activations
            assert abs(ls[0] - rl) <= FP32_TOL * abs(rl), (step, ls[0], rl)
            losses.append(ls[0])
        merged = PT.merge_owned(cfg, [m.params() for m in g.models], g.partition)
        vel = PT.merge_owned(cfg, [m.velocity() for m in g.models], g.partition)
        # 2 steps x L blocks x 2 directions x the non-empty chunks
        calls, nbytes = PT.exchange_stats(g.models[0])
        assert calls == 2 * cfg.num_blocks * 2 * min(chunks, B)
        assert nbytes == 2 * cfg.num_blocks * 2 * B * cfg.seq_len * cfg.model_dim * 4
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


def test_nccl_partition_world1_runs_the_exchange():
    """An NCCL partition of one rank: every block's partial output and dxn go
    through ncclAllReduce (eager step_codes, then d2ft_step, whose CUDA graph
    captures the all-reduces and replays them).  Results agree with the
    whole-model engine to fp32 summation-order noise (the partitioned path
    keeps dxn in fp32) and with the fp64 oracle trainer at the step
    tolerances."""
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        cfg = SMALL
        oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
        sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                           cfg.num_classes)
        B = 4
        p, x, y = _setup(cfg, B)
        K = cfg.scheduled_subnet_count()
        codes = np.random.default_rng(9).integers(1, 4, (K, B)).astype(np.uint8)
        a = E.SubnetModel(cfg, B, p)
        m = E.SubnetModel(cfg, B, p)
        part = PT.HeadPartition(cfg.heads_per_block, 0, 1)
        PT.join_nccl(m, part, chunks=2)
        la = a.step_codes(x, y, codes, 1, 0.05, 0.9)
        lm = m.step_codes(x, y, codes, 1, 0.05, 0.9)
        calls, nbytes = PT.exchange_stats(m)
        assert calls == cfg.num_blocks * 2 * 2 and nbytes == cfg.num_blocks * 2 * B * cfg.seq_len * cfg.model_dim * 4
        assert abs(la - lm) <= 1e-6 * abs(la)
        p32 = p.astype(np.float32).astype(np.float64)
        assert normwise(m.params() - p32, a.params() - p32) <= 1e-3
        rl, _ = MO.train_batch(oc, p.copy(), np.zeros_like(p), x.astype(np.float64), y, codes, 1, 0.05, 0.9)
        assert abs(lm - rl) <= FP32_TOL * abs(rl)
        assert np.array_equal(PT.gather_params(m, m.partition), m.params())
        # graph path: the knapsack schedule + step captured once, replayed
        b, f = O.bench_scores(K, B, 1)
        nb = (2 * B) // 5
        caps = Capacities([nb * 5] * K, [nb * 2] * K)
        st = ScoreTable(K, B, f, b)
        for i in range(3):
            lw, tw = a.d2ft_step(x, y, st, CostModel(), caps, 1, 0.05, 0.9)
            lp, tp = m.d2ft_step(x, y, st, CostModel(), caps, 1, 0.05, 0.9)
            assert np.array_equal(tw.codes, tp.codes)
            assert abs(lw - lp) <= 1e-4 * abs(lw), (i, lw, lp)
        calls2, _ = PT.exchange_stats(m)
        assert calls2 == calls + 3 * cfg.num_blocks * 2 * 2
        assert normwise(m.params() - p32, a.params() - p32) <= 1e-3
        a.close()
        m.close()
    finally:
        dist.destroy_process_group()


def test_local_partition_graphless_chunks_match_single_chunk():
    """Exchange chunking only reorders when the sums run, never what they
    add: chunks 1 and 3 give bit-identical parameters (ViT-shaped dh 64)."""
    cfg = E.ModelConfig(2, 4, 256, 512, 197, 4, 1)
    B = 8
    p, x, y = _setup(cfg, B, 13)
    K = cfg.scheduled_subnet_count()
    codes = np.random.default_rng(4).integers(1, 4, (K, B)).astype(np.uint8)
    res = []
    for chunks in (1, 3):
        g = PT.LocalGroup([E.SubnetModel(cfg, B, p) for _ in range(2)], "heads", chunks)
        try:
            ls = g.run(lambda r, m: m.step_codes(x, y, codes, 1, 0.05, 0.9))
            res.append((ls[0], PT.merge_owned(cfg, [m.params() for m in g.models], g.partition)))
        finally:
            g.close()
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])
