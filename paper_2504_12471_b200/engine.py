"""Host mirror of the reference model/trainer interface for the D2FT step.

Names follow the reference: ModelConfig (model.hpp:43-57), partition_model
(model.cpp:140-156), SubnetModel.forward_backward (model.cpp:416-520),
make_synthetic_dataset (trainer.cpp:83-111), and `d2ft_step`, the batch body
of train() for the D2FT policy (trainer.cpp:214-292).  All compute runs in the
sm_100a kernels behind include/d2ft_b200_engine.h; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import Error, check, f64, i32, lib, ptr, u8
from .scheduler import Capacities, CostModel, ScheduleTable, ScoreTable


class _Cfg(C.Structure):
    _fields_ = [("num_blocks", C.c_int), ("heads_per_block", C.c_int), ("model_dim", C.c_int),
                ("ffn_hidden", C.c_int), ("seq_len", C.c_int), ("num_classes", C.c_int), ("seed", C.c_uint64)]


@dataclass
class ModelConfig:
    """model.hpp:43-57 (defaults as the reference)."""
    num_blocks: int = 2
    heads_per_block: int = 2
    model_dim: int = 16
    ffn_hidden: int = 32
    seq_len: int = 8
    num_classes: int = 4
    seed: int = 1

    def head_dim(self) -> int:
        return self.model_dim // self.heads_per_block

    def ffn_slice_dim(self) -> int:
        return self.ffn_hidden // self.heads_per_block

    def subnet_count(self) -> int:
        return self.num_blocks * self.heads_per_block + 2

    def scheduled_subnet_count(self) -> int:
        return self.num_blocks * self.heads_per_block

    def _c(self) -> _Cfg:
        return _Cfg(self.num_blocks, self.heads_per_block, self.model_dim, self.ffn_hidden, self.seq_len,
                    self.num_classes, self.seed)


# scoring.hpp:19-24 (Metric enum order; names as metric_name, scoring.cpp)
METRICS = ("fisher_information", "weight_magnitude", "gradient_magnitude", "taylor_importance")

# presets of BASELINE.json
TINY = ModelConfig(2, 4, 128, 512, 64, 4, 1)
VIT_B16 = ModelConfig(12, 12, 768, 3072, 197, 8, 1)
VIT_L16 = ModelConfig(24, 16, 1024, 4096, 197, 8, 1)


def param_count(cfg: ModelConfig) -> int:
    d, H, dh, fs = cfg.model_dim, cfg.heads_per_block, cfg.head_dim(), cfg.ffn_slice_dim()
    block = 3 * d * dh + dh * d + d * fs + fs + fs * d + d // H
    return d * d + d + cfg.seq_len * d + cfg.num_blocks * H * block + d * cfg.num_classes + cfg.num_classes


def subnet_slices(cfg: ModelConfig):
    """[(start, stop)] of embed, the L*H block subnets, head in the canonical flat vector."""
    d, H, dh, fs = cfg.model_dim, cfg.heads_per_block, cfg.head_dim(), cfg.ffn_slice_dim()
    e = d * d + d + cfg.seq_len * d
    b = 3 * d * dh + dh * d + d * fs + fs + fs * d + d // H
    out = [(0, e)] + [(e + k * b, e + (k + 1) * b) for k in range(cfg.num_blocks * H)]
    out.append((e + cfg.num_blocks * H * b, e + cfg.num_blocks * H * b + d * cfg.num_classes + cfg.num_classes))
    return out


def partition_model(cfg: ModelConfig) -> np.ndarray:
    """Canonical fp64 initial parameters (model.cpp:140-156), bit-identical to the reference."""
    out = np.empty(param_count(cfg), np.float64)
    c = cfg._c()
    check(lib().d2ft_partition_model(C.byref(c), ptr(out)))
    return out


def lora_init(cfg: ModelConfig, rank: int) -> np.ndarray:
    """attach_lora's initial adapters (model.cpp:174-192), bit-identical to the
    reference: per block subnet down_q[d][r] = 0, up_q[r][dh] ~ N(0, 1/r), k, v."""
    n = cfg.num_blocks * cfg.heads_per_block * 3 * (cfg.model_dim * rank + rank * cfg.head_dim())
    out = np.empty(n, np.float64)
    c = cfg._c()
    check(lib().d2ft_lora_init(C.byref(c), C.c_int(rank), ptr(out)))
    return out


def make_synthetic_dataset(num_samples, num_classes, token_dim, seq_len, noise_level=0.5, seed=7):
    """trainer.cpp:83-111; samples as fp32 [n][T][d], labels int32."""
    x = np.empty((num_samples, seq_len, token_dim), np.float32)
    y = np.empty(num_samples, np.int32)
    check(lib().d2ft_make_synthetic_dataset(C.c_int(num_samples), C.c_int(num_classes), C.c_int(token_dim),
                                            C.c_int(seq_len), C.c_double(noise_level), C.c_uint64(seed), ptr(x),
                                            ptr(y)))
    return x, y


def _aligned_f64(shape) -> np.ndarray:
    """A fresh page-aligned fp64 array (one Matrix allocation of the reference's
    vector<Matrix>; page alignment lets d2ft_dataset_create page-lock each
    sample on its own)."""
    n = int(np.prod(shape))
    # 8 KB of slack: the aligned start (<= 4 KB in) plus the page-rounded end
    # the registration covers both stay inside this allocation
    raw = np.empty(n + 1024, np.float64)
    off = (-raw.ctypes.data % 4096) // 8
    return raw[off:off + n].reshape(shape)


class Dataset:
    """data.hpp:18-42: `samples` is a list of fp64 [seq_len][token_dim] arrays
    (one per sample, as vector<Matrix>), `labels` ints, `num_classes`.  The
    device handle (d2ft_dataset_create) borrows the arrays and page-locks them
    for the per-batch gather of d2ft_engine_step_units."""

    def __init__(self, samples, labels, num_classes: int):
        self.samples = [np.ascontiguousarray(s, np.float64) for s in samples]
        self.labels = i32(labels)
        self.num_classes = int(num_classes)
        if len(self.samples) != self.labels.size:
            raise Error(2, "dataset: samples and labels must align")
        self._h = None

    def size(self) -> int:
        return len(self.samples)

    def micro_batch_count(self, micro_batch_size: int) -> int:
        if micro_batch_size < 1 or self.size() % micro_batch_size:
            raise Error(2, "dataset size must be a multiple of the micro-batch size")  # data.hpp:26-28
        return self.size() // micro_batch_size

    def unit_inputs(self, unit: int, micro_batch_size: int):
        return self.samples[unit * micro_batch_size:(unit + 1) * micro_batch_size]

    def unit_labels(self, unit: int, micro_batch_size: int):
        return self.labels[unit * micro_batch_size:(unit + 1) * micro_batch_size]

    def handle(self, pin: bool = True):
        if self._h is None:
            T, d = self.samples[0].shape
            if any(s.shape != (T, d) for s in self.samples):
                raise Error(2, "dataset: samples must share one shape")
            ptrs = (C.c_void_p * self.size())(*[s.ctypes.data for s in self.samples])
            h = C.c_void_p()
            check(lib().d2ft_dataset_create(ptrs, ptr(self.labels), C.c_int(self.size()), C.c_int(self.num_classes),
                                            C.c_int(T), C.c_int(d), C.c_int(1 if pin else 0), C.byref(h)))
            self._h = h
        return self._h

    def close(self):
        if self._h is not None:
            lib().d2ft_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_synthetic_dataset_f64(num_samples, num_classes, token_dim, seq_len, noise_level=0.5, seed=7) -> Dataset:
    """trainer.cpp:83-111 as the reference's fp64 Dataset (bit-identical samples)."""
    flat = np.empty((num_samples, seq_len, token_dim), np.float64)
    y = np.empty(num_samples, np.int32)
    check(lib().d2ft_make_synthetic_dataset_f64(C.c_int(num_samples), C.c_int(num_classes), C.c_int(token_dim),
                                                C.c_int(seq_len), C.c_double(noise_level), C.c_uint64(seed),
                                                ptr(flat), ptr(y)))
    samples = []
    for i in range(num_samples):
        a = _aligned_f64((seq_len, token_dim))
        a[...] = flat[i]
        samples.append(a)
    return Dataset(samples, y, num_classes)


class SubnetModel:
    """Device-resident subnet model + optimizer state on one B200."""

    def __init__(self, config: ModelConfig, max_batch: int, params: np.ndarray | None = None):
        self.config = config
        self.max_batch = max_batch
        self.partition = None  # partition.HeadPartition once joined to a head partition
        self.data_parallel = None  # (rank, world) once joined to a data-parallel group
        self._h = C.c_void_p()
        c = config._c()
        L = lib()
        L.d2ft_engine_param_count.restype = C.c_int64
        L.d2ft_engine_stream.restype = C.c_void_p
        check(L.d2ft_engine_create(C.byref(c), C.c_int(max_batch), C.byref(self._h)))
        self.n = int(L.d2ft_engine_param_count(self._h))
        self.set_params(partition_model(config) if params is None else params)

    def close(self):
        if self._h:
            lib().d2ft_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def scheduled_count(self) -> int:
        return self.config.scheduled_subnet_count()

    def parameter_count(self) -> int:
        return self.n

    def set_params(self, flat) -> None:
        a = f64(flat)
        if a.size != self.n:
            raise Error(3, f"set_params: expected {self.n} values, got {a.size}")
        check(lib().d2ft_engine_set_params(self._h, ptr(a)))

    def params(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        check(lib().d2ft_engine_get_params(self._h, ptr(out)))
        return out

    def velocity(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        check(lib().d2ft_engine_get_velocity(self._h, ptr(out)))
        return out

    def grads(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        check(lib().d2ft_engine_get_grads(self._h, ptr(out)))
        return out

    # ---- opt-in p_s surrogate (d2ft_engine_set_surrogate) ------------------
    def set_surrogate(self, rank: int, factors=None) -> None:
        """p_s as "skip with a linear surrogate" (BASELINE north_star): a
        shortcut cell adds LN(x)_s . down . up; factors per block subnet in
        scheduled order, down [d][rank] then up [rank][d].  rank 0 restores the
        reference's pure bypass (the default; every parity run)."""
        cfg = self.config
        n = cfg.scheduled_subnet_count() * 2 * cfg.model_dim * rank
        a = None
        if rank:
            a = f64(factors)
            if a.size != n:
                raise Error(3, f"set_surrogate: expected {n} values, got {a.size}")
        check(lib().d2ft_engine_set_surrogate(self._h, C.c_int(rank), ptr(a) if a is not None else None))
        self.surrogate_rank = rank

    # ---- LoRA (model.cpp:165-195; csrc/lora.cu) ----------------------------
    def attach_lora(self, rank: int, scaling: float, adapters: np.ndarray | None = None) -> None:
        """SubnetModel::attach_lora: rank-r adapters on Q/K/V, base frozen.
        adapters default to the reference's initial values (lora_init)."""
        a = lora_init(self.config, rank) if adapters is None else f64(adapters)
        check(lib().d2ft_engine_attach_lora(self._h, C.c_int(rank), C.c_double(scaling), ptr(a)))
        self.lora_rank, self.lora_scaling = rank, scaling

    def lora_enabled(self) -> bool:
        return bool(getattr(self, "lora_rank", 0))

    def _lora_n(self) -> int:
        lib().d2ft_engine_lora_count.restype = C.c_int64
        return int(lib().d2ft_engine_lora_count(self._h))

    def set_lora(self, adapters) -> None:
        a = f64(adapters)
        if a.size != self._lora_n():
            raise Error(3, f"set_lora: expected {self._lora_n()} values, got {a.size}")
        check(lib().d2ft_engine_set_lora(self._h, ptr(a)))

    def _get_lora(self, which: int) -> np.ndarray:
        out = np.empty(self._lora_n(), np.float64)
        check(lib().d2ft_engine_get_lora(self._h, C.c_int(which), ptr(out)))
        return out

    def lora_params(self) -> np.ndarray:
        return self._get_lora(0)

    def lora_velocity(self) -> np.ndarray:
        return self._get_lora(1)

    def lora_grads(self) -> np.ndarray:
        return self._get_lora(2)

    def forward_backward(self, inputs, labels, schedule_column):
        """model.cpp:416-520: returns (loss, grads_flat, engaged).  Gradients of
        subnets that are not engaged are zeroed here, mirroring the reference's
        disengaged optionals."""
        col = u8(schedule_column)
        if col.size != self.scheduled_count():
            raise Error(2, "schedule column must have one operation per scheduled subnet")
        if len(inputs) == 0 or len(inputs) != len(labels):
            raise Error(2, "micro-batch inputs and labels must be non-empty and aligned")  # model.cpp:424
        x, y = self._batch(inputs, labels, len(labels), global_batch=False)
        loss = C.c_double()
        check(lib().d2ft_engine_forward_backward(self._h, ptr(x), ptr(y), C.c_int(len(y)), ptr(col), C.byref(loss)))
        g = self.grads()
        engaged = np.zeros(self.scheduled_count() + 2, np.uint8)
        engaged[0] = engaged[-1] = 1
        engaged[1:-1] = (col == 1)
        for si, (a, b) in enumerate(subnet_slices(self.config)):
            if not engaged[si]:
                g[a:b] = 0.0
        return loss.value, g, engaged

    def step_codes(self, samples, labels, codes, mbs=1, lr=0.05, momentum=0.9) -> float:
        """Trainer batch with an explicit K x n_mb schedule table."""
        c = u8(codes.codes if isinstance(codes, ScheduleTable) else codes)
        if c.ndim != 2 or c.shape[0] != self.scheduled_count():
            raise Error(2, f"step_codes: schedule table must be {self.scheduled_count()} x n_mb, got {c.shape}")
        n_mb = c.shape[1]
        x, y = self._batch(samples, labels, n_mb * mbs)
        loss = C.c_double()
        check(lib().d2ft_engine_step_codes(self._h, ptr(x), ptr(y), ptr(c), C.c_int(n_mb), C.c_int(mbs),
                                           C.c_double(lr), C.c_double(momentum), C.byref(loss)))
        return loss.value

    def _batch(self, samples, labels, B, global_batch=True):
        """Samples [B][T][d] fp32 and B labels of one batch (the C entry
        points read exactly B of each); on a data-parallel engine a batch
        step's B is the global batch and the caller passes this rank's slice."""
        x = np.ascontiguousarray(samples, np.float32)
        y = i32(labels)
        cfg = self.config
        if global_batch and self.data_parallel is not None:  # this rank holds its slice of the global batch
            B //= self.data_parallel[1]
        if y.ndim != 1 or y.size != B:
            raise Error(2, f"batch of {B} units needs {B} labels, got {y.size}")
        if x.shape != (B, cfg.seq_len, cfg.model_dim):
            raise Error(2, f"batch of {B} units needs samples of shape {(B, cfg.seq_len, cfg.model_dim)}, "
                           f"got {x.shape}")
        if B > self.max_batch:
            raise Error(6, f"batch of {B} units exceeds the engine capacity {self.max_batch}")
        return x, y

    def d2ft_step(self, samples, labels, scores: ScoreTable, cost_model: CostModel, capacities: Capacities,
                  mbs=1, lr=0.05, momentum=0.9):
        """One D2FT batch (trainer.cpp:214-292): GPU knapsack schedule from the
        batch's score slice, forward/backward of the active heads, SGD.
        Returns (batch_loss, ScheduleTable)."""
        K, n_mb = scores.subnets, scores.micro_batches
        if K != self.scheduled_count():
            raise Error(2, f"d2ft_step: score table has {K} rows, the model schedules {self.scheduled_count()} subnets")
        scores.validate()
        capacities.validate()
        if len(capacities.full) != K or len(capacities.fwd) != K:
            raise Error(2, "knapsack_schedule: capacities device count mismatch")
        cost_model.validate()
        cf, cb = cost_model.row_arrays(K)
        x, y = self._batch(samples, labels, n_mb * mbs)
        codes = np.zeros((K, n_mb), np.uint8)
        loss = C.c_double()
        check(lib().d2ft_engine_step(self._h, ptr(x), ptr(y), ptr(scores.backward), ptr(scores.forward), ptr(cf),
                                     ptr(cb), ptr(i32(capacities.full)), ptr(i32(capacities.fwd)), C.c_int(n_mb),
                                     C.c_int(mbs), C.c_double(lr), C.c_double(momentum), C.byref(loss), ptr(codes)))
        return loss.value, ScheduleTable(K, n_mb, codes)

    def step_units(self, dataset: Dataset, units, scores: ScoreTable, cost_model: CostModel,
                   capacities: Capacities, mbs=1, lr=0.05, momentum=0.9, units_next=None):
        """trainer.cpp:214-268 over dataset units: the batch is `units` (unit u =
        samples [u*mbs, (u+1)*mbs)), `scores` the whole pre-pass table
        (K x micro_batch_count), sliced per batch (slice_scores,
        trainer.cpp:139-154).  The fp64 samples are gathered on the device;
        `units_next` prefetches the next batch (pass it as `units` next call).
        Returns (batch_loss, ScheduleTable)."""
        K = self.scheduled_count()
        u = i32(units)
        n_mb = u.size
        total = dataset.micro_batch_count(mbs)
        if scores.subnets != K or scores.micro_batches != total:
            raise Error(2, f"step_units: score table must be {K} x {total}, got {scores.subnets} x {scores.micro_batches}")
        if len(capacities.full) != K or len(capacities.fwd) != K:
            raise Error(2, "knapsack_schedule: capacities device count mismatch")
        if n_mb * mbs > self.max_batch:
            raise Error(6, f"batch of {n_mb * mbs} units exceeds the engine capacity {self.max_batch}")
        un = None
        if units_next is not None:
            un = i32(units_next)
            if un.size != n_mb:
                raise Error(2, "step_units: the next batch must have as many units")
        cost_model.validate()
        cf, cb = cost_model.row_arrays(K)
        codes = np.zeros((K, n_mb), np.uint8)
        loss = C.c_double()
        check(lib().d2ft_engine_step_units(self._h, dataset.handle(), ptr(u), C.c_int(n_mb), C.c_int(mbs),
                                           ptr(un) if un is not None else None, ptr(scores.backward),
                                           ptr(scores.forward), C.c_int(total), ptr(cf), ptr(cb),
                                           ptr(i32(capacities.full)), ptr(i32(capacities.fwd)), C.c_double(lr),
                                           C.c_double(momentum), C.byref(loss), ptr(codes)))
        # the engine staged the next batch's labels / score slice from these
        # tables and recognises them by address: keep them alive until then
        self._staged = (dataset, scores.backward, scores.forward) if un is not None else None
        return loss.value, ScheduleTable(K, n_mb, codes)

    def prepass_scores(self, samples, labels, micro_batch_size=1, fwd_metric="fisher_information",
                       bwd_metric="weight_magnitude") -> ScoreTable:
        """prepass_scores (scoring.cpp:108-151): every micro-batch forward and
        backward with all scheduled subnets Full and no update; the chosen
        metric of each head-subnet's unit gradient (scoring.cpp:57-96)."""
        x = np.ascontiguousarray(samples, np.float32)
        y = i32(labels)
        n = len(y)
        if n == 0:
            raise Error(2, "prepass_scores: empty dataset")
        if micro_batch_size < 1 or n % micro_batch_size:
            raise Error(2, "dataset size must be a multiple of the micro-batch size")
        units = n // micro_batch_size
        K = self.scheduled_count()
        fo = np.zeros((K, units), np.float64)
        bo = np.zeros((K, units), np.float64)
        check(lib().d2ft_engine_prepass_scores(self._h, ptr(x), ptr(y), C.c_int(n), C.c_int(micro_batch_size),
                                               C.c_int(METRICS.index(fwd_metric)), C.c_int(METRICS.index(bwd_metric)),
                                               ptr(fo), ptr(bo)))
        t = ScoreTable(K, units, fo, bo, fwd_metric, bwd_metric)
        t.validate()
        return t

    # -- bench path -------------------------------------------------------
    def stage(self, samples, labels, scores: ScoreTable, cost_model: CostModel, capacities: Capacities, mbs=1):
        K, n_mb = scores.subnets, scores.micro_batches
        if K != self.scheduled_count() or len(capacities.full) != K or len(capacities.fwd) != K:
            raise Error(2, "knapsack_schedule: capacities device count mismatch")
        cf, cb = cost_model.row_arrays(K)
        x, y = self._batch(samples, labels, n_mb * mbs)
        check(lib().d2ft_engine_stage_device(self._h, ptr(x), ptr(y), ptr(scores.backward),
                                             ptr(scores.forward), ptr(cf), ptr(cb), ptr(i32(capacities.full)),
                                             ptr(i32(capacities.fwd)), C.c_int(n_mb), C.c_int(mbs)))
        self._staged = (n_mb, mbs)

    def step_resident(self, lr=0.05, momentum=0.9):
        n_mb, mbs = self._staged
        check(lib().d2ft_engine_step_resident(self._h, C.c_int(n_mb), C.c_int(mbs), C.c_double(lr),
                                              C.c_double(momentum)))

    def sync(self) -> float:
        loss = C.c_double()
        check(lib().d2ft_engine_sync(self._h, C.byref(loss)))
        return loss.value

    def stream(self) -> int:
        return lib().d2ft_engine_stream(self._h)

    def set_profiling(self, on: bool):
        check(lib().d2ft_engine_set_profiling(self._h, C.c_int(1 if on else 0)))

    PHASES = ("sched", "embed", "ln", "G1", "attn_fwd", "G3", "head", "G4", "attn_bwd", "G5", "G7", "G8", "bias",
              "ln_bwd", "embed_wgrad", "sgd", "exchange")

    def phase_ms(self):
        out = np.zeros(len(self.PHASES))
        steps = C.c_int()
        check(lib().d2ft_engine_phase_ms(self._h, ptr(out), C.c_int(len(out)), C.byref(steps)))
        n = max(1, steps.value)
        return {k: float(v) / n for k, v in zip(self.PHASES, out)}


def smoke_step() -> None:
    """__graft_entry__.smoke(): one tiny D2FT step on cuda:0 vs the fp64 oracle,
    at the BASELINE tiny shape (dh = 32, mma.sync attention) and at dh = 64
    (the tcgen05 attention kernels the ViT configs run)."""
    from oracle import lib as O
    from oracle import model_oracle as MO
    for cfg in (ModelConfig(2, 4, 128, 256, 64, 4, 1), ModelConfig(2, 2, 128, 256, 64, 4, 1)):
        B = 8
        x, y = make_synthetic_dataset(B, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
        K = cfg.scheduled_subnet_count()
        b, f = O.bench_scores(K, B, 3)
        caps = Capacities([(2 * B // 5) * 5] * K, [(2 * B // 5) * 2] * K)
        m = SubnetModel(cfg, B)
        p0 = m.params()
        loss, table = m.d2ft_step(x, y, ScoreTable(K, B, f, b), CostModel(), caps, 1, 0.05, 0.9)
        ref_codes = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
        assert np.array_equal(table.codes, ref_codes), "smoke: GPU schedule differs from the oracle"
        oc = MO.Config(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                       cfg.num_classes)
        pr = p0.copy()
        v = np.zeros_like(pr)
        ref_loss, _ = MO.train_batch(oc, pr, v, x.astype(np.float64), y, ref_codes, 1, 0.05, 0.9)
        assert abs(loss - ref_loss) <= 1e-3 * abs(ref_loss), (loss, ref_loss)
        dp, dr = m.params() - p0.astype(np.float32).astype(np.float64), pr - p0
        rel = np.max(np.abs(dp - dr)) / np.max(np.abs(dr))
        assert rel <= 1e-2, rel
        m.close()
