"""CPU: host logic of the head-partitioned multi-GPU path,
world_size 2 over torch.distributed gloo.

The partitioned algorithm is checked end to end on the fp64 oracle: each rank
computes only its own rows' block contributions (rank 0 adds the residual),
the ranks all-reduce the partial block outputs and the partial dxn per sample
chunk (asynchronously, in the engine's issue order), and the result must equal
the unpartitioned reference step (loss, owned-subnet and replicated
gradients), for both row mappings and 1-3 exchange chunks.  The same
HeadPartition / owner_slices / merge code the GPU path uses decides
ownership."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import model_oracle as MO
from paper_2504_12471_b200 import partition as PT
from paper_2504_12471_b200.engine import ModelConfig


def test_every_head_has_one_owner():
    for H in (2, 4, 12, 16):
        for world in (1, 2, 3, 8):
            owned = [PT.HeadPartition(H, r, world).owned_heads() for r in range(world)]
            flat = sorted(h for o in owned for h in o)
            assert flat == list(range(H))
            sizes = [len(o) for o in owned]
            assert max(sizes) - min(sizes) <= 1


def test_local_codes_union_is_global():
    rng = np.random.default_rng(3)
    L, H, n = 3, 4, 5
    codes = rng.integers(1, 4, size=(L * H, n)).astype(np.uint8)
    world = 3
    views = [PT.HeadPartition(H, r, world).local_codes(codes) for r in range(world)]
    for k in range(L * H):
        owner = (k % H) % world
        for r in range(world):
            expect = codes[k] if r == owner else np.full(n, 3, np.uint8)
            assert np.array_equal(views[r][k], expect)


def test_owner_slices_cover_flat_vector():
    cfg = ModelConfig(2, 4, 16, 32, 8, 4, 1)
    from paper_2504_12471_b200.engine import param_count
    sl = PT.owner_slices(cfg, 3)
    cov = np.zeros(param_count(cfg), int)
    for _, a, b in sl:
        cov[a:b] += 1
    assert np.all(cov == 1)
    flats = [np.full(param_count(cfg), float(r)) for r in range(3)]
    m = PT.merge_owned(cfg, flats)
    for r, a, b in sl:
        assert np.all(m[a:b] == r)


def test_busy_units_imbalance():
    codes = np.array([[1, 1], [2, 3], [1, 2], [3, 3]], np.uint8)  # L=1, H=4
    busy, ratio = PT.busy_units(codes, 4, 2)
    assert busy.tolist() == [(5 + 5) + (5 + 2), 2]  # rows 0, 2 -> rank 0; rows 1, 3 -> rank 1
    assert math.isclose(ratio, busy.max() / busy.mean())


def test_contiguous_mapping_is_spec_literal():
    """cost_sim.cpp:138-152: device r hosts memory_units[r] consecutive rows."""
    for L, H, world in ((12, 12, 8), (2, 4, 3), (24, 16, 8), (1, 4, 4)):
        K = L * H
        owners = [PT.HeadPartition(H, r, world, "contiguous", L).row_owners() for r in range(world)]
        assert all(np.array_equal(o, owners[0]) for o in owners)
        o = owners[0]
        assert np.all(np.diff(o) >= 0) and o[0] == 0 and o[-1] == world - 1
        units = PT.HeadPartition(H, 0, world, "contiguous", L).memory_units()
        assert units == np.bincount(o, minlength=world).tolist() and sum(units) == K
        assert max(units) - min(units) <= 1


def test_rank_capacities_balance_uneven_mapping():
    """ViT-B heads on 8 ranks: 24 vs 12 rows.  The BudgetSpec overrides give
    the light ranks a larger per-row budget; every row's capacity is its
    owner's budget x the row's cost (capacities_from_budget)."""
    from paper_2504_12471_b200.scheduler import CostModel
    part = PT.HeadPartition(12, 0, 8)
    N = 512
    spec, caps = PT.rank_capacities(part, 12, N, (2 * N) // 5, (2 * N) // 5)
    owners = part.row_owners(12)
    rows = np.bincount(owners)
    assert rows.tolist() == [24] * 4 + [12] * 4
    for k in range(owners.size):
        nf, no = spec.n_full_for(k), spec.n_fwd_for(k)
        assert nf + no <= N
        assert caps.full[k] == nf * CostModel().full_cost(k) and caps.fwd[k] == no * CostModel().cf(k)
    units = [sum(caps.full[k] + caps.fwd[k] for k in range(owners.size) if owners[k] == r) for r in range(8)]
    uniform = [rows[r] * ((2 * N) // 5) * 7 for r in range(8)]
    assert max(units) / min(units) < max(uniform) / min(uniform)
    _, flat = PT.rank_capacities(part, 12, N, (2 * N) // 5, (2 * N) // 5, balance=False)
    assert len(set(flat.full)) == 1


# ---------------------------------------------------------------- gloo, world 2
def _partitioned_step(cfg, flat, inputs, labels, column, part, chunks):
    """Oracle forward/backward of one micro-batch of n samples computed the
    way the partitioned engine does it: own rows only, the partial block
    outputs / dxn of every sample chunk [c*n/C, (c+1)*n/C) all-reduced
    asynchronously (gloo, issued in chunk order like the engine's exchange
    stream), each chunk's LayerNorm waiting for its own sum."""
    p = MO.unpack(cfg, flat)
    grads = np.zeros_like(flat)
    g = MO.unpack(cfg, grads)
    L, H = cfg.L, cfg.H
    local = part.local_codes(np.asarray(column, np.uint8).reshape(-1, 1))[:, 0]
    n = len(inputs)
    bounds = [(c * n // chunks, (c + 1) * n // chunks) for c in range(chunks)]

    def exchange(a):
        """Chunked async all-reduce of a [n][T][d] array; returns the waits."""
        t = torch.from_numpy(np.ascontiguousarray(a))
        works = [(lo, hi, dist.all_reduce(t[lo:hi], async_op=True)) for lo, hi in bounds if hi > lo]
        return t, works

    inp = np.asarray(inputs, np.float64)
    x = inp @ p["w_embed"] + p["b_embed"] + p["pos"]
    xs = [x]
    caches = [[None] * cfg.K for _ in range(n)]
    for l in range(L):
        xin = xs[-1]
        xn = np.stack([MO.layer_norm(xin[si]) for si in range(n)])
        partial = xin.copy() if part.rank == 0 else np.zeros_like(xin)
        for si in range(n):
            for h in range(H):
                r = l * H + h
                if local[r] == 3:
                    continue
                cache = {} if local[r] == 1 else None
                partial[si] += MO.block_contribution(cfg, p["blocks"][r], h, xn[si], cache)
                caches[si][r] = cache
        t, works = exchange(partial)
        for lo, hi, w in works:  # the next block's LN of a chunk waits for that chunk only
            w.wait()
        xs.append(t.numpy())
    loss = 0.0
    dx = np.zeros_like(x)
    for si in range(n):
        fx = xs[-1][si]
        xn_h = MO.layer_norm(fx)
        pooled = xn_h.mean(axis=0)
        logits = pooled @ p["w_cls"] + p["b_cls"]
        e = np.exp(logits - logits.max())
        lab = int(labels[si])
        loss += (math.log(e.sum()) - (logits[lab] - logits.max())) / n
        dlog = e / e.sum()
        dlog[lab] -= 1.0
        dlog /= n
        g["w_cls"] += np.outer(pooled, dlog)
        g["b_cls"] += dlog
        dx[si] = MO.layer_norm_backward(fx, np.broadcast_to((dlog @ p["w_cls"].T) / cfg.T, fx.shape))
    for l in range(L - 1, -1, -1):
        dxn = np.zeros_like(xs[l])
        for si in range(n):
            for h in range(H):
                r = l * H + h
                if local[r] == 1:
                    MO.contribution_backward(cfg, p["blocks"][r], h, caches[si][r], dx[si], dxn[si], g["blocks"][r])
        # LN-backward gate: any Full head in the block on ANY rank (global codes)
        anyf = any(column[l * H + h] == 1 for h in range(H))
        t, works = exchange(dxn)
        for lo, hi, w in works:
            w.wait()
            if anyf:
                for si in range(lo, hi):
                    dx[si] = dx[si] + MO.layer_norm_backward(xs[l][si], t.numpy()[si])
    for si in range(n):
        g["w_embed"] += inp[si].T @ dx[si]
        g["b_embed"] += dx[si].sum(axis=0)
        g["pos"] += dx[si]
    return loss, grads


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = MO.Config(2, 4, 16, 32, 6, 3)
        mc = ModelConfig(2, 4, 16, 32, 6, 3, 1)
        rng = np.random.default_rng(11)
        flat = rng.standard_normal(MO.param_count(cfg)) * 0.2
        inputs = rng.standard_normal((3, cfg.T, cfg.d))
        labels = np.array([0, 2, 1])
        column = np.array([1, 2, 3, 1, 3, 1, 2, 2], np.uint8)  # K = 8 rows
        ref_loss, ref_grads, _ = MO.forward_backward(cfg, flat, inputs, labels, column)
        out = []
        for mapping in ("heads", "contiguous"):
            part = PT.HeadPartition(cfg.H, rank, world, mapping, cfg.L)
            for chunks in (1, 2, 3):
                loss, grads = _partitioned_step(cfg, flat, inputs, labels, column, part, chunks)
                # owned subnets (and the replicated embed/head) match the whole-model step
                ok = abs(loss - ref_loss) <= 1e-12 * abs(ref_loss)
                err = 0.0
                for r, a, b in PT.owner_slices(mc, world, part):
                    if r == rank or (a == 0) or b == len(flat):
                        err = max(err, np.max(np.abs(grads[a:b] - ref_grads[a:b])) /
                                  (np.max(np.abs(ref_grads)) + 1e-300))
                # gathered ownership-merge across ranks reproduces the whole-model gradient
                t = torch.from_numpy(grads)
                parts = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                merged = PT.merge_owned(mc, [x.numpy() for x in parts], part)
                merr = np.max(np.abs(merged - ref_grads)) / np.max(np.abs(ref_grads))
                out.append((mapping, chunks, ok, err, merr))
        # NCCL id bootstrap travels through the (gloo) group
        uid = PT.share_unique_id(rank)
        uids = [None] * world
        dist.all_gather_object(uids, uid)
        q.put((rank, out, len(uid) == 128 and uids[0] == uids[1]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partitioned_step_matches_whole_model_gloo():
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
    for rank, out, uid_ok in res:
        assert len(out) == 6
        for mapping, chunks, ok, err, merr in out:
            assert ok, (rank, mapping, chunks)
            assert err < 1e-12, (rank, mapping, chunks, err)
            assert merr < 1e-12, (rank, mapping, chunks, merr)
        assert uid_ok
