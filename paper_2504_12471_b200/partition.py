"""Head partition of the D2FT step across GPUs.

The reference runs every subnet in one process (no communication anywhere);
this is the multi-GPU executor around the same step.  Every scheduled row
(subnet k = l*H + h) has one owning rank: by default rank h % world owns head
h of every block (head-interleaved tensor parallelism, SURVEY.md §8e option
ii); the SPEC-literal contiguous mapping (cost_sim.cpp:138-152) is the
alternative (`HeadPartition.mapping`).

* scheduling — rows are independent (scheduler.cpp:148), so every rank runs
  the same knapsack over all rows and keeps the rows it owns
  (`local_codes`); no communication.  Per-rank budgets enter as BudgetSpec
  overrides (`rank_capacities`), which is how an uneven mapping is balanced;
* forward — each rank's G3 produces the PARTIAL block output over its active
  heads (rank 0 adds the residual), and the ranks sum the partials: the one
  exchange per block (model.cpp:454-468 is that sum);
* backward — each rank's G8 produces the dxn partial over its Full heads and
  the ranks sum them before the replicated LayerNorm backward
  (model.cpp:497-508); the LN gate uses the global Full count;
* parameters — a head's weights and gradients are authoritative on its owner;
  embedding and classifier are replicated (identical inputs, identical math),
  so no gradient all-reduce exists.

The exchange is an NCCL all-reduce (one process per GPU, `join_nccl`; captured
in the step's CUDA graph) or, for testing the partitioned math on a single
GPU, an in-process group of engines stepped from host threads (`LocalGroup`).
Either way it runs per sample chunk on an exchange stream: the sum of chunk c
overlaps G3 / G8 of chunk c+1 and feeds that chunk's LayerNorm alone.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from ._lib import Error, check, lib, ptr


MAPPINGS = ("heads", "contiguous")


@dataclass(frozen=True)
class HeadPartition:
    """Row -> rank mapping of the scheduled subnets (row k = l*H + h).

    mapping "heads" (default, the executor SURVEY §8e recommends): rank
    h % world owns head h of every block — tensor parallelism over heads, every
    rank busy in every block.  mapping "contiguous" (the SPEC-literal one,
    cost_sim.cpp:138-152 / cost_sim.hpp:65-69): device r hosts memory_units[r]
    consecutive rows, K // world each and one more on the first K % world
    devices; a block's heads then live on one or two ranks."""
    heads_per_block: int
    rank: int
    world: int
    mapping: str = "heads"
    num_blocks: int = 0  # required by "contiguous"

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise Error(1, "partition: rank out of range")
        if self.mapping not in MAPPINGS:
            raise Error(1, f"partition: mapping must be one of {MAPPINGS}")
        if self.mapping == "contiguous" and self.num_blocks < 1:
            raise Error(1, "partition: the contiguous mapping needs num_blocks")

    def owner(self, head: int) -> int:
        """Owner of head `head` under the head-interleaved mapping."""
        return head % self.world

    def memory_units(self, num_blocks: int | None = None) -> list[int]:
        """Rows hosted per rank (DeviceProfile::memory_units)."""
        K = (num_blocks or self.num_blocks) * self.heads_per_block
        return [len(self.rows_of(r, num_blocks or self.num_blocks)) for r in range(self.world)] \
            if self.mapping == "heads" else [K // self.world + (r < K % self.world) for r in range(self.world)]

    def row_owners(self, num_blocks: int | None = None) -> np.ndarray:
        """owner[k] for every scheduled row k = l*H + h."""
        L = num_blocks or self.num_blocks
        H = self.heads_per_block
        K = L * H
        if self.mapping == "heads":
            return np.array([(k % H) % self.world for k in range(K)], np.int32)
        units = [K // self.world + (r < K % self.world) for r in range(self.world)]
        return np.repeat(np.arange(self.world, dtype=np.int32), units)

    def rows_of(self, rank: int, num_blocks: int) -> list[int]:
        return [int(k) for k in np.flatnonzero(self.row_owners(num_blocks) == rank)]

    def owned_heads(self) -> list[int]:
        """Heads of every block this rank owns (head-interleaved mapping)."""
        if self.mapping != "heads":
            raise Error(1, "partition: owned_heads is defined for the head-interleaved mapping")
        return [h for h in range(self.heads_per_block) if self.owner(h) == self.rank]

    def owned_rows(self, num_blocks: int) -> list[int]:
        """Scheduled rows k = l*H + h (scheduler row order) this rank computes."""
        return self.rows_of(self.rank, num_blocks)

    def row_mask(self, num_blocks: int) -> np.ndarray:
        return self.row_owners(num_blocks) == self.rank

    def local_codes(self, codes: np.ndarray) -> np.ndarray:
        """The rank's view of a K x n schedule table: other ranks' rows -> p_s (3)."""
        c = np.array(codes, np.uint8, copy=True)
        K = c.shape[0]
        c[~self.row_mask(K // self.heads_per_block)] = 3
        return c


def owner_slices(cfg, world: int, part: HeadPartition | None = None):
    """[(rank, start, stop)] of every subnet slice of the canonical flat vector:
    block subnet k = l*H + h belongs to its row's owner (h % world by
    default); embed and head to rank 0."""
    from .engine import subnet_slices
    sl = subnet_slices(cfg)
    H = cfg.heads_per_block
    owners = part.row_owners(cfg.num_blocks) if part is not None else \
        np.array([(k % H) % world for k in range(cfg.num_blocks * H)])
    out = [(0,) + sl[0]]
    for k in range(cfg.num_blocks * H):
        out.append((int(owners[k]),) + sl[1 + k])
    out.append((0,) + sl[-1])
    return out


def merge_owned(cfg, flats_by_rank, part: HeadPartition | None = None) -> np.ndarray:
    """Canonical flat vector assembled from each subnet's owner."""
    world = len(flats_by_rank)
    out = np.array(flats_by_rank[0], np.float64, copy=True)
    for r, a, b in owner_slices(cfg, world, part):
        out[a:b] = flats_by_rank[r][a:b]
    return out


def merge_owned_lora(cfg, rank: int, flats_by_rank, part: HeadPartition) -> np.ndarray:
    """LoRA adapters (d2ft_engine_attach_lora layout: per block subnet k, in
    scheduled order) assembled from each subnet's owner — under a head
    partition only the owner trains a head's adapters (its Full cells)."""
    per = 3 * (cfg.model_dim * rank + rank * cfg.head_dim())
    owners = part.row_owners(cfg.num_blocks)
    out = np.array(flats_by_rank[0], np.float64, copy=True)
    for k, r in enumerate(owners):
        out[k * per:(k + 1) * per] = flats_by_rank[int(r)][k * per:(k + 1) * per]
    return out


def rank_capacities(part: HeadPartition, num_blocks: int, micro_batches: int, n_full: int, n_fwd: int,
                    cost_model=None, balance: bool = True):
    """Per-rank knapsack capacities through BudgetSpec overrides
    (scheduler.cpp:45-55, 428-440): every row of rank r gets the budget
    (n_full_r, n_fwd_r).  balance=True scales the base budget by
    mean_rows / rows_r so each rank's budgeted cost units (rows_r x budget)
    match — D2FT's load balancing of an uneven mapping (ViT-B's 12 heads on 8
    GPUs: 24 vs 12 rows per rank) — and clips n_full_r + n_fwd_r to the
    micro-batch count, shrinking both in proportion.  Returns
    (BudgetSpec, Capacities)."""
    from .scheduler import BudgetOverride, BudgetSpec, CostModel, capacities_from_budget
    cost_model = cost_model or CostModel()
    owners = part.row_owners(num_blocks)
    K = owners.size
    rows = np.bincount(owners, minlength=part.world)
    per_rank = []
    for r in range(part.world):
        f = (K / part.world) / rows[r] if (balance and rows[r]) else 1.0
        nf, no = int(n_full * f), int(n_fwd * f)
        if nf + no > micro_batches:
            sh = micro_batches / (nf + no)
            nf = int(nf * sh)
            no = min(int(no * sh), micro_batches - nf)
        per_rank.append((nf, no))
    spec = BudgetSpec(n_full, n_fwd, [BudgetOverride(int(k), *per_rank[int(owners[k])]) for k in range(K)])
    return spec, capacities_from_budget(spec, cost_model, K, micro_batches)


def gather_params(model, part: HeadPartition, group=None) -> np.ndarray:
    """All ranks: the merged (owner-authoritative) parameters of a partitioned
    model, gathered with torch.distributed (any backend)."""
    import torch
    import torch.distributed as dist
    mine = torch.from_numpy(model.params())
    parts = [torch.empty_like(mine) for _ in range(part.world)]
    dist.all_gather(parts, mine, group=group)
    return merge_owned(model.config, [p.numpy() for p in parts], part)


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


def _apply_mapping(model, part: HeadPartition) -> None:
    owners = part.row_owners(model.config.num_blocks)
    check(lib().d2ft_engine_set_row_owner(model._h, ptr(owners), C.c_int(owners.size)))
    model.partition = part


def join_nccl(model, part: HeadPartition, group=None, chunks: int | None = None) -> None:
    """Make `model` (a SubnetModel on this rank's GPU) rank `part.rank` of an
    NCCL head partition; collective over the torch.distributed group.
    `chunks`: sample chunks of the per-block exchange (engine default 2)."""
    uid = share_unique_id(part.rank, group)
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    check(lib().d2ft_engine_partition_nccl(model._h, C.c_int(part.rank), C.c_int(part.world), buf))
    _apply_mapping(model, part)
    if chunks is not None:
        check(lib().d2ft_engine_set_exchange_chunks(model._h, C.c_int(chunks)))


def exchange_stats(model) -> tuple[int, int]:
    """(all-reduce calls, payload bytes) this rank issued so far."""
    calls, nbytes = C.c_ulonglong(), C.c_ulonglong()
    check(lib().d2ft_engine_exchange_stats(model._h, C.byref(calls), C.byref(nbytes)))
    return calls.value, nbytes.value


# ---------------------------------------------------------------- data parallel
def dp_slice(n_mb: int, mbs: int, rank: int, world: int) -> tuple[int, int]:
    """Samples [lo, hi) of the global batch rank `rank` holds under data
    parallelism: micro-batches [rank*n_mb/world, (rank+1)*n_mb/world)."""
    if n_mb % world:
        raise Error(1, "data parallel: the micro-batches of a batch must divide evenly over the ranks")
    per = n_mb // world
    return rank * per * mbs, (rank + 1) * per * mbs


def join_nccl_dp(model, rank: int, world: int, group=None) -> None:
    """Make `model` rank `rank` of an NCCL data-parallel group (collective
    over the torch.distributed group): afterwards its steps take the global
    score table and this rank's slice of the batch (`dp_slice`)."""
    uid = share_unique_id(rank, group)
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    check(lib().d2ft_engine_data_parallel_nccl(model._h, C.c_int(rank), C.c_int(world), buf))
    model.data_parallel = (rank, world)


class LocalGroup:
    """`world` engines on one device forming a head partition (single-GPU test
    harness; the exchange is a fixed-order device sum).  `run(fn)` calls
    fn(rank, model) on one host thread per rank and returns the results."""

    def __init__(self, models, mapping: str = "heads", chunks: int | None = None, data_parallel: bool = False):
        self.models = list(models)
        self.world = len(self.models)
        self._g = C.c_void_p()
        check(lib().d2ft_local_group_create(C.c_int(self.world), C.byref(self._g)))
        if data_parallel:  # engines of one data-parallel group (gradient all-reduce)
            for r, m in enumerate(self.models):
                check(lib().d2ft_engine_data_parallel_local(m._h, self._g, C.c_int(r)))
                m.data_parallel = (r, self.world)
            self.partition = None
            return
        for r, m in enumerate(self.models):
            check(lib().d2ft_engine_partition_local(m._h, self._g, C.c_int(r)))
            _apply_mapping(m, HeadPartition(m.config.heads_per_block, r, self.world, mapping,
                                            m.config.num_blocks))
            if chunks is not None:
                check(lib().d2ft_engine_set_exchange_chunks(m._h, C.c_int(chunks)))
        self.partition = self.models[0].partition

    def run(self, fn):
        out = [None] * self.world
        err = [None] * self.world

        def body(r):
            try:
                out[r] = fn(r, self.models[r])
            except BaseException as e:  # re-raised on the caller's thread
                err[r] = e
                lib().d2ft_local_group_abort(self._g)  # peers waiting in the exchange fail instead of hanging

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        first = next((e for e in err if e is not None and "aborted by a failing rank" not in str(e)), None)
        first = first or next((e for e in err if e is not None), None)
        if first is not None:  # the root cause, not a peer's abort
            raise first
        return out

    def close(self):
        for m in self.models:
            m.close()
        if self._g:
            lib().d2ft_local_group_destroy(self._g)
            self._g = C.c_void_p()


def busy_units(codes: np.ndarray, heads_per_block: int, world: int, cf: float = 2.0, cb: float = 3.0,
               owners: np.ndarray | None = None):
    """Per-rank busy time in cost units of one batch (cost_model: a Full cell
    costs cf + cb, a forward-only cell cf, model.hpp cost units) and the
    max/mean imbalance the partition incurs (owners: row -> rank, default
    head-interleaved)."""
    c = np.asarray(codes)
    K = c.shape[0]
    per_row = (c == 1).sum(axis=1) * (cf + cb) + (c == 2).sum(axis=1) * cf
    busy = np.zeros(world)
    for k in range(K):
        busy[int(owners[k]) if owners is not None else (k % heads_per_block) % world] += per_row[k]
    mean = busy.mean()
    return busy, (busy.max() / mean if mean > 0 else 1.0)
