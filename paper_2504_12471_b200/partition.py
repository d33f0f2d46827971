"""Head partition of the D2FT step across GPUs.

The reference runs every subnet in one process (no communication anywhere);
this is the multi-GPU executor around the same step.  Rank r of `world` owns
the heads h with h % world == r of every block (head-interleaved tensor
parallelism, SURVEY.md §8e option ii):

* scheduling — rows are independent (scheduler.cpp:148), so every rank runs
  the same knapsack over all rows and keeps the rows of its heads
  (`local_codes`); no communication;
* forward — each rank's G3 produces the PARTIAL block output over its active
  heads (rank 0 adds the residual), and the ranks sum the partials: the one
  exchange per block (model.cpp:454-468 is that sum);
* backward — each rank's G8 produces the dxn partial over its Full heads and
  the ranks sum them before the replicated LayerNorm backward
  (model.cpp:497-508); the LN gate uses the global Full count;
* parameters — a head's weights and gradients are authoritative on its owner;
  embedding and classifier are replicated (identical inputs, identical math),
  so no gradient all-reduce exists.

The exchange is an NCCL all-reduce (one process per GPU, `join_nccl`) or, for
testing the partitioned math on a single GPU, an in-process group of engines
stepped from host threads (`LocalGroup`).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from ._lib import Error, check, lib, ptr


@dataclass(frozen=True)
class HeadPartition:
    heads_per_block: int
    rank: int
    world: int

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise Error(1, "partition: rank out of range")

    def owner(self, head: int) -> int:
        return head % self.world

    def owned_heads(self) -> list[int]:
        return [h for h in range(self.heads_per_block) if self.owner(h) == self.rank]

    def owned_rows(self, num_blocks: int) -> list[int]:
        """Scheduled rows k = l*H + h (scheduler row order) this rank computes."""
        H = self.heads_per_block
        return [l * H + h for l in range(num_blocks) for h in self.owned_heads()]

    def row_mask(self, num_blocks: int) -> np.ndarray:
        m = np.zeros(num_blocks * self.heads_per_block, bool)
        m[self.owned_rows(num_blocks)] = True
        return m

    def local_codes(self, codes: np.ndarray) -> np.ndarray:
        """The rank's view of a K x n schedule table: other ranks' rows -> p_s (3)."""
        c = np.array(codes, np.uint8, copy=True)
        K = c.shape[0]
        c[~self.row_mask(K // self.heads_per_block)] = 3
        return c


def owner_slices(cfg, world: int):
    """[(rank, start, stop)] of every subnet slice of the canonical flat vector:
    block subnet k = l*H + h belongs to h % world; embed and head to rank 0."""
    from .engine import subnet_slices
    sl = subnet_slices(cfg)
    H = cfg.heads_per_block
    out = [(0,) + sl[0]]
    for k in range(cfg.num_blocks * H):
        out.append(((k % H) % world,) + sl[1 + k])
    out.append((0,) + sl[-1])
    return out


def merge_owned(cfg, flats_by_rank) -> np.ndarray:
    """Canonical flat vector assembled from each subnet's owner."""
    world = len(flats_by_rank)
    out = np.array(flats_by_rank[0], np.float64, copy=True)
    for r, a, b in owner_slices(cfg, world):
        out[a:b] = flats_by_rank[r][a:b]
    return out


def gather_params(model, part: HeadPartition, group=None) -> np.ndarray:
    """All ranks: the merged (owner-authoritative) parameters of a partitioned
    model, gathered with torch.distributed (any backend)."""
    import torch
    import torch.distributed as dist
    mine = torch.from_numpy(model.params())
    parts = [torch.empty_like(mine) for _ in range(part.world)]
    dist.all_gather(parts, mine, group=group)
    return merge_owned(model.config, [p.numpy() for p in parts])


def share_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id; every rank returns it."""
    import torch.distributed as dist
    obj = [None]
    if rank == 0:
        buf = (C.c_uint8 * 128)()
        check(lib().d2ft_nccl_unique_id(buf))
        obj[0] = bytes(buf)
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def join_nccl(model, part: HeadPartition, group=None) -> None:
    """Make `model` (a SubnetModel on this rank's GPU) rank `part.rank` of an
    NCCL head partition; collective over the torch.distributed group."""
    uid = share_unique_id(part.rank, group)
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    check(lib().d2ft_engine_partition_nccl(model._h, C.c_int(part.rank), C.c_int(part.world), buf))
    model.partition = part


class LocalGroup:
    """`world` engines on one device forming a head partition (single-GPU test
    harness; the exchange is a fixed-order device sum).  `run(fn)` calls
    fn(rank, model) on one host thread per rank and returns the results."""

    def __init__(self, models):
        self.models = list(models)
        self.world = len(self.models)
        self._g = C.c_void_p()
        check(lib().d2ft_local_group_create(C.c_int(self.world), C.byref(self._g)))
        for r, m in enumerate(self.models):
            check(lib().d2ft_engine_partition_local(m._h, self._g, C.c_int(r)))
            m.partition = HeadPartition(m.config.heads_per_block, r, self.world)

    def run(self, fn):
        out = [None] * self.world
        err = [None] * self.world

        def body(r):
            try:
                out[r] = fn(r, self.models[r])
            except BaseException as e:  # re-raised on the caller's thread
                err[r] = e

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        for m in self.models:
            m.close()
        if self._g:
            lib().d2ft_local_group_destroy(self._g)
            self._g = C.c_void_p()


def busy_units(codes: np.ndarray, heads_per_block: int, world: int, cf: float = 2.0, cb: float = 3.0):
    """Per-rank busy time in cost units of one batch (cost_model: a Full cell
    costs cf + cb, a forward-only cell cf, model.hpp cost units) and the
    max/mean imbalance the partition incurs."""
    c = np.asarray(codes)
    K = c.shape[0]
    per_row = (c == 1).sum(axis=1) * (cf + cb) + (c == 2).sum(axis=1) * cf
    busy = np.zeros(world)
    for k in range(K):
        busy[(k % heads_per_block) % world] += per_row[k]
    mean = busy.mean()
    return busy, (busy.max() / mean if mean > 0 else 1.0)
