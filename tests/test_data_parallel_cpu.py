"""CPU: host logic of the data-parallel multi-GPU path, world_size 2 over
torch.distributed gloo, on the fp64 oracle.

Every rank takes its micro-batches of the global batch (partition.dp_slice,
the same function bench.py and the GPU tests use), accumulates their
gradients with the GLOBAL 1/n_mb weight (trainer.cpp:247-260), the ranks
all-reduce the sums, and the SGD touches the subnets with a Full cell anywhere
in the global table (trainer.cpp:264-268).  The result must be the
reference trainer's step on the whole batch (loss and updated parameters)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import model_oracle as MO
from paper_2504_12471_b200 import partition as PT


def test_dp_slices_tile_the_batch():
    for n_mb, mbs, world in ((6, 1, 2), (6, 2, 3), (8, 4, 8), (64, 1, 8)):
        spans = [PT.dp_slice(n_mb, mbs, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n_mb * mbs
        assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
        assert all((b - a) % mbs == 0 for a, b in spans)
    try:
        PT.dp_slice(5, 1, 0, 2)
        raise AssertionError("expected a config error")
    except PT.Error as e:
        assert e.kind == "config"


def _dp_step(cfg, flat, vel, inputs, labels, codes, mbs, lr, mom, rank, world):
    n_mb = codes.shape[1]
    lo, hi = PT.dp_slice(n_mb, mbs, rank, world)
    inv = 1.0 / n_mb
    accum = np.zeros_like(flat)
    loss = 0.0
    for j in range(lo // mbs, hi // mbs):
        l, g, _ = MO.forward_backward(cfg, flat, inputs[j * mbs:(j + 1) * mbs], labels[j * mbs:(j + 1) * mbs],
                                      codes[:, j])
        loss += l * inv
        accum += g * inv
    t = torch.from_numpy(np.concatenate([accum, [loss]]))
    dist.all_reduce(t)  # the engine's gradient all-reduce (and the callers' loss sum)
    accum, loss = t.numpy()[:-1], float(t.numpy()[-1])
    touched = np.zeros(cfg.K + 2, bool)
    touched[0] = touched[-1] = True
    touched[1:-1] = (codes == 1).any(axis=1)  # global Full counts
    for si, (a, b) in enumerate(MO.subnet_slices(cfg)):
        if touched[si]:
            vel[a:b] = mom * vel[a:b] + accum[a:b]
            flat[a:b] -= lr * vel[a:b]
    return loss


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = MO.Config(2, 4, 16, 32, 6, 3)
        rng = np.random.default_rng(11)
        flat0 = rng.standard_normal(MO.param_count(cfg)) * 0.2
        out = []
        for mbs in (1, 2):
            n_mb = 4
            inputs = rng.standard_normal((n_mb * mbs, cfg.T, cfg.d))
            labels = np.arange(n_mb * mbs) % cfg.C
            codes = rng.integers(1, 4, size=(cfg.K, n_mb)).astype(np.uint8)
            codes[0, :] = 3  # untouched everywhere
            codes[1, :] = 2
            codes[1, 0] = 1  # Full only in rank 0's half
            f_ref, v_ref = flat0.copy(), np.zeros_like(flat0)
            f_dp, v_dp = flat0.copy(), np.zeros_like(flat0)
            errs = []
            for _ in range(2):
                rl, _ = MO.train_batch(cfg, f_ref, v_ref, inputs, labels, codes, mbs, 0.05, 0.9)
                dl = _dp_step(cfg, f_dp, v_dp, inputs, labels, codes, mbs, 0.05, 0.9, rank, world)
                errs.append((abs(dl - rl) / abs(rl), np.max(np.abs(f_dp - f_ref)) / np.max(np.abs(f_ref - flat0))))
            out.append((mbs, errs, np.array_equal(f_dp[MO.subnet_slices(cfg)[1][0]:MO.subnet_slices(cfg)[1][1]],
                                                  flat0[MO.subnet_slices(cfg)[1][0]:MO.subnet_slices(cfg)[1][1]])))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_data_parallel_step_matches_whole_batch_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in res:
        assert len(out) == 2
        for mbs, errs, untouched_same in out:
            for le, pe in errs:
                assert le < 1e-12 and pe < 1e-10, (rank, mbs, le, pe)
            assert untouched_same
