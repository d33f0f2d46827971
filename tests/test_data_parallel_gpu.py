"""GPU: data parallelism over the global batch (d2ft_engine_data_parallel_*).

`world` engines on one device form an in-process data-parallel group
(partition.LocalGroup(data_parallel=True); the gradient all-reduce is a
fixed-order device sum); each steps its slice of the batch
(partition.dp_slice) with the GLOBAL score table.  Every rank must end with the
same bytes, equal to one engine stepping the whole batch up to the all-reduce's
summation order, and to the fp64 oracle trainer on the whole batch at the step
tolerances.  The NCCL path runs at world 1 (one GPU per box): it must give the
single engine's bytes exactly (the all-reduce of one rank is the identity)."""
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

SMALL = E.ModelConfig(2, 4, 128, 256, 64, 4, 1)      # dh = 32
SMALL64 = E.ModelConfig(2, 2, 128, 256, 50, 4, 5)    # dh = 64


def _setup(cfg, B, seed=3):
    p = E.partition_model(cfg)
    p = p + 0.02 * np.random.default_rng(seed).standard_normal(p.size)
    n = -(-B // cfg.num_classes) * cfg.num_classes  # the generator wants whole classes
    x, y = E.make_synthetic_dataset(n, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
    return p, x[:B], y[:B]


@pytest.mark.parametrize("cfg,world,mbs", [(SMALL, 2, 1), (SMALL64, 3, 1), (SMALL64, 2, 2)],
                         ids=["dh32-w2", "dh64-w3", "dh64-w2-mbs2"])
def test_local_data_parallel_d2ft_step(cfg, world, mbs):
    oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len, cfg.num_classes)
    sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
    n_mb = 6
    B = n_mb * mbs
    p, x, y = _setup(cfg, B)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, n_mb, 7)
    st = ScoreTable(K, n_mb, f, b)
    caps = Capacities([2 * 5] * K, [2 * 2] * K)
    whole = E.SubnetModel(cfg, B, p)
    g = PT.LocalGroup([E.SubnetModel(cfg, B // world, p) for _ in range(world)], data_parallel=True)
    try:
        pr, vr = p.copy(), np.zeros_like(p)
        for step in range(2):
            def body(r, m):
                lo, hi = PT.dp_slice(n_mb, mbs, r, world)
                return m.d2ft_step(x[lo:hi], y[lo:hi], st, CostModel(), caps, mbs, 0.05, 0.9)
            outs = g.run(body)
            lw, tw = whole.d2ft_step(x, y, st, CostModel(), caps, mbs, 0.05, 0.9)
            codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
            for _, t in outs:
                assert np.array_equal(t.codes, codes) and np.array_equal(tw.codes, codes)
            loss = sum(l for l, _ in outs)  # each rank returns its share of the batch loss
            assert abs(loss - lw) <= 1e-5 * abs(lw), (loss, lw)
            rl, _ = MO.train_batch(oc, pr, vr, x.astype(np.float64), y, codes, mbs, 0.05, 0.9)
            assert abs(loss - rl) <= FP32_TOL * abs(rl), (step, loss, rl)
        ps = [m.params() for m in g.models]
        for q in ps[1:]:
            assert np.array_equal(q, ps[0])  # one all-reduced gradient, one SGD: identical on every rank
        assert np.array_equal(g.models[0].velocity(), g.models[-1].velocity())
        p32 = p.astype(np.float32).astype(np.float64)
        bad_w = compare_tensors(whole.params() - p32, pr - p, sl, GRAD_TOL)
        bad_d = compare_tensors(ps[0] - p32, pr - p, sl, GRAD_TOL)
        assert not bad_w and not bad_d, ("whole vs oracle", bad_w[:4], "dp vs oracle", bad_d[:4])
        # vs one engine on the whole batch: each rank's fp16 gradient operands
        # carry its own power-of-two scale (its samples' max |dX|) and the
        # all-reduce sums in another order; the wq / wk updates amplify such
        # rounding differences to ~2e-4
        bad = compare_tensors(ps[0] - p32, whole.params() - p32, sl, 2e-3)
        assert not bad, bad[:8]
        bad = compare_tensors(ps[0] - p32, pr - p, sl, GRAD_TOL)
        assert not bad, bad[:8]
        calls, nbytes = PT.exchange_stats(g.models[0])
        # per step: block l's two weight matrices as soon as its G5 / G7 are
        # done (overlapping the backward of block l-1), then the rest
        assert calls == 2 * (2 * cfg.num_blocks + 2) and nbytes > 0 and nbytes % (2 * 4) == 0
    finally:
        g.close()
        whole.close()


def test_local_data_parallel_untouched_rows_and_errors():
    """A row whose Full cells all sit on one rank: the other rank's stale
    gradient rows must not leak into the all-reduce (zeroed), and rows with no
    Full cell anywhere keep params and velocity (trainer.cpp:264-268)."""
    cfg = SMALL
    n_mb, world = 4, 2
    p, x, y = _setup(cfg, n_mb)
    K = cfg.scheduled_subnet_count()
    codes = np.full((K, n_mb), 2, np.uint8)
    codes[0, 0] = 1          # row 0: Full only in rank 0's half
    codes[1, 3] = 1          # row 1: Full only in rank 1's half
    codes[2, :] = 3          # row 2: never touched
    codes[3, :] = 1
    whole = E.SubnetModel(cfg, n_mb, p)
    g = PT.LocalGroup([E.SubnetModel(cfg, n_mb // world, p) for _ in range(world)], data_parallel=True)
    try:
        for _ in range(2):  # a second step: stale rows of step 1 would show up here
            g.run(lambda r, m: m.step_codes(x[2 * r:2 * r + 2], y[2 * r:2 * r + 2], codes, 1, 0.05, 0.9))
            whole.step_codes(x, y, codes, 1, 0.05, 0.9)
        sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                           cfg.num_classes)
        p32 = p.astype(np.float32).astype(np.float64)
        got = g.models[0].params()
        bad = compare_tensors(got - p32, whole.params() - p32, sl, 2e-3)
        assert not bad, bad[:8]
        a, b_ = E.subnet_slices(cfg)[1 + 2]
        assert np.array_equal(got[a:b_], p32[a:b_]) and not np.any(g.models[1].velocity()[a:b_])
        with pytest.raises(E.Error) as e:  # 5 micro-batches do not split over 2 ranks
            g.run(lambda r, m: m.step_codes(x[:2], y[:2], np.ones((K, 5), np.uint8), 1))
        assert e.value.kind in ("config", "input")
        with pytest.raises(E.Error) as e:
            g.models[0].attach_lora(2, 1.0)
        assert e.value.kind == "state"
    finally:
        g.close()
        whole.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_nccl_data_parallel_world1_matches_single_engine():
    """The NCCL all-reduce path, captured in the step's CUDA graph, at world 1:
    bit-identical to the single engine."""
    import torch
    import torch.distributed as dist
    cfg = SMALL64
    B = 6
    p, x, y = _setup(cfg, B)
    K = cfg.scheduled_subnet_count()
    b, f = O.bench_scores(K, B, 9)
    st = ScoreTable(K, B, f, b)
    caps = Capacities([2 * 5] * K, [2 * 2] * K)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        m = E.SubnetModel(cfg, B, p)
        PT.join_nccl_dp(m, 0, 1)
        ref = E.SubnetModel(cfg, B, p)
        for _ in range(3):
            l1, t1 = m.d2ft_step(x, y, st, CostModel(), caps)
            l2, t2 = ref.d2ft_step(x, y, st, CostModel(), caps)
            assert l1 == l2 and np.array_equal(t1.codes, t2.codes)
        assert np.array_equal(m.params(), ref.params()) and np.array_equal(m.velocity(), ref.velocity())
        calls, _ = PT.exchange_stats(m)
        assert calls == 3 * (2 * cfg.num_blocks + 2)
        m.close()
        ref.close()
    finally:
        dist.destroy_process_group()
