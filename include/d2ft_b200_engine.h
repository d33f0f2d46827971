/* d2ft_b200 — C-ABI of the D2FT step engine (one B200).
 *
 * Replaces, for the D2FT policy, the batch body of
 *   d2ft::train()                     core/src/trainer.cpp:214-292
 * i.e. knapsack_schedule (scheduler.cpp:222-236) -> per micro-batch
 *   SubnetModel::forward_backward     core/src/model.cpp:416-520
 * -> 1/n_mb accumulation (trainer.cpp:247-260) -> sgd_momentum_step on the
 * subnets that received gradients (trainer.cpp:113-134, 264-268).
 * Status codes as in d2ft_b200.h.  Parameters cross the boundary in the
 * reference's canonical fp64 order (model.hpp:117-153, the order of
 * SubnetModel::parameter_bytes / the checkpoint); the engine keeps fp32
 * masters + velocity and bf16 operand copies on the device.
 */
#ifndef D2FT_B200_ENGINE_H
#define D2FT_B200_ENGINE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ModelConfig (model.hpp:43-57).  The B200 engine requires model_dim % 128 == 0,
 * model_dim <= 1024, head_dim (d/H) in {32, 64}, seq_len <= 256, <= 64 classes. */
typedef struct {
  int num_blocks, heads_per_block, model_dim, ffn_hidden, seq_len, num_classes;
  uint64_t seed;
} d2ft_model_config;

typedef struct d2ft_engine d2ft_engine;

int d2ft_engine_create(const d2ft_model_config* cfg, int max_batch, d2ft_engine** out);
int d2ft_engine_destroy(d2ft_engine* e);
/* number of fp64 values in the canonical flat parameter vector */
int64_t d2ft_engine_param_count(d2ft_engine* e);
/* load parameters (canonical fp64 order); resets the momentum to zero */
int d2ft_engine_set_params(d2ft_engine* e, const double* flat);
int d2ft_engine_get_params(d2ft_engine* e, double* flat);
/* momentum buffers, canonical order (the trainer's `velocity`, trainer.cpp:194-196) */
int d2ft_engine_get_velocity(d2ft_engine* e, double* flat);
/* gradients of the last forward_backward / step, canonical order; subnets
 * without a Full cell hold stale values (check the schedule) */
int d2ft_engine_get_grads(d2ft_engine* e, double* flat);

/* ---- LoRA: SubnetModel::attach_lora (model.cpp:165-195).
 * Rank-r adapters on Q/K/V of every head-subnet; afterwards the step trains
 * only the adapters (visit_trainable, model.hpp:155-172; trainer.cpp:124-133)
 * and the base weights stay frozen.  Adapters are a flat fp64 array in
 * visit_tensors order per block subnet (l, h): down_q [d][r], up_q [r][dh],
 * down_k, up_k, down_v, up_v (model.hpp:139-146); initial values from
 * d2ft_lora_init.  Errors: state (already attached), config (rank < 1 or
 * rank > min(d, d/H)), as the reference. */
int d2ft_engine_attach_lora(d2ft_engine* e, int rank, double scaling, const double* adapters);
int64_t d2ft_engine_lora_count(d2ft_engine* e); /* adapter doubles (0 = none attached) */
int d2ft_engine_set_lora(d2ft_engine* e, const double* adapters); /* also zeroes their velocity */
/* which: 0 adapters, 1 velocity, 2 gradients of the last forward_backward / step */
int d2ft_engine_get_lora(d2ft_engine* e, int which, double* adapters);

/* Opt-in p_s surrogate ("skip with a linear surrogate", BASELINE north_star /
 * PAPER.md:25-26; the reference's p_s is a pure bypass, model.cpp:326-328,
 * 458, which rank 0 — the default — keeps bit for bit).  With rank R > 0 a
 * shortcut cell (sample s, head-subnet (l,h)) adds LN(x_l)_s . down . up to
 * the block output: factors per block subnet in scheduled order (l-major,
 * h-minor), down [d][R] then up [R][d], fp64 (stored fp16).  Frozen: no
 * gradient flows through a surrogate (as p_o, model.cpp:501).  R a multiple
 * of 8 in [8, 64]; state error on a head-partitioned engine. */
int d2ft_engine_set_surrogate(d2ft_engine* e, int rank, const double* factors);

/* SubnetModel::forward_backward (model.cpp:416-520) for n samples of one
 * micro-batch under one schedule column (K = L*H codes).  Loss = mean CE;
 * gradients (scaled 1/n) readable with d2ft_engine_get_grads. */
int d2ft_engine_forward_backward(d2ft_engine* e, const float* samples, const int32_t* labels, int n,
                                 const uint8_t* column, double* loss_out);

/* SubnetModel::logits (model.cpp logits, every subnet active) for n <= max
 * batch samples: logits_out n x num_classes.  No parameter changes; the
 * gradient buffers are clobbered.  evaluate() (trainer.cpp:307-319) is the
 * argmax over these. */
int d2ft_engine_logits(d2ft_engine* e, const float* samples, int n, double* logits_out);

/* One trainer batch with an explicit K x n_mb schedule table (Standard policy
 * = all 1).  samples: (n_mb*mbs) x T x d fp32 in micro-batch order; loss_out
 * = batch loss as trainer.cpp:254. */
int d2ft_engine_step_codes(d2ft_engine* e, const float* samples, const int32_t* labels, const uint8_t* codes,
                           int n_mb, int mbs, double lr, double momentum, double* loss_out);

/* One D2FT batch: schedule from the batch's score slice (K x n_mb fp64,
 * ScoreTable::backward / forward of trainer.cpp:139-154) with per-row costs
 * cf/cb and capacities, then forward/backward/SGD.  codes_out (K x n_mb,
 * may be NULL) receives the schedule.  Host buffers; synchronous. */
int d2ft_engine_step(d2ft_engine* e, const float* samples, const int32_t* labels, const double* bwd_scores,
                     const double* fwd_scores, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                     const int32_t* cap_fwd, int n_mb, int mbs, double lr, double momentum, double* loss_out,
                     uint8_t* codes_out);

/* Scoring pre-pass, prepass_scores (scoring.hpp:48-54, scoring.cpp:108-151):
 * every micro-batch of micro_batch_size samples runs forward + backward with
 * all scheduled subnets Full and no weight update; fwd_out / bwd_out (K x
 * num_samples/micro_batch_size, row-major = ScoreTable::forward / backward)
 * receive the chosen metric of each head-subnet's unit gradient: 0
 * FisherInformation (sum g^2), 1 WeightMagnitude (sum |w|), 2
 * GradientMagnitude (sum |g|), 3 TaylorImportance (sum |w g|) — the Metric
 * enum order.  Parameters are unchanged. */
int d2ft_engine_prepass_scores(d2ft_engine* e, const float* samples, const int32_t* labels, int num_samples,
                               int micro_batch_size, int fwd_metric, int bwd_metric, double* fwd_out,
                               double* bwd_out);

/* Input pipeline (a data loader's double buffering; no reference counterpart:
 * trainer.cpp:214-292 reads batches from host memory).  d2ft_engine_prefetch
 * starts the H2D copy of a batch's samples (pinned host memory) on the
 * engine's copy stream; d2ft_engine_step_pipelined then runs the step on the
 * prefetched samples (as d2ft_engine_step) and, if samples_next != NULL,
 * prefetches the next batch while this one computes. */
int d2ft_engine_prefetch(d2ft_engine* e, const float* samples, int batch);
int d2ft_engine_step_pipelined(d2ft_engine* e, const float* samples_next, const int32_t* labels,
                               const double* bwd_scores, const double* fwd_scores, const int32_t* cf,
                               const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, int n_mb, int mbs,
                               double lr, double momentum, double* loss_out, uint8_t* codes_out);

/* The reference's Dataset (data.hpp:18-42): num_samples fp64 seq_len x
 * token_dim row-major matrices (Matrix::data of dataset.samples[i]) and their
 * labels.  The sample pointers are borrowed — the caller's vector<Matrix>
 * stays the owner and must outlive the handle; labels are copied.  pin != 0
 * page-locks every sample (cudaHostRegister; undone by destroy) so the
 * per-batch gather runs at DMA speed. */
typedef struct d2ft_dataset d2ft_dataset;
int d2ft_dataset_create(const double* const* samples, const int32_t* labels, int num_samples, int num_classes,
                        int seq_len, int token_dim, int pin, d2ft_dataset** out);
int d2ft_dataset_destroy(d2ft_dataset* ds);

/* The D2FT batch body of train() over dataset units (trainer.cpp:214-268):
 * the batch is units[0..n_mb) (unit u = samples [u*mbs, (u+1)*mbs),
 * Dataset::unit_inputs / unit_labels), scores are the whole pre-pass
 * ScoreTable (K x total_units row-major backward / forward) sliced per batch
 * as slice_scores (trainer.cpp:139-154).  The fp64 samples are gathered H2D
 * and converted on the device; units_next != NULL gathers the next batch on
 * the copy stream while this one computes (the next call must pass those
 * units) and stages its labels and score slice on the host (the next call
 * must pass the same dataset and unmodified score table; other arguments are
 * re-checked).  loss_out = batch loss (trainer.cpp:254); codes_out (K x n_mb,
 * may be NULL) = the schedule. */
int d2ft_engine_step_units(d2ft_engine* e, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs,
                           const int32_t* units_next, const double* bwd_scores, const double* fwd_scores,
                           int total_units, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                           const int32_t* cap_fwd, double lr, double momentum, double* loss_out, uint8_t* codes_out);
/* The same batch body under an explicit K x n_mb schedule table (codes
 * {1,2,3}; the Standard / Random / Scaler / pruning policies of
 * trainer.cpp:220-243). */
int d2ft_engine_step_units_codes(d2ft_engine* e, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs,
                                 const int32_t* units_next, const uint8_t* codes, double lr, double momentum,
                                 double* loss_out);
/* bench.py's end-to-end leg over the Dataset path: warmup + steps batches,
 * batch i = order[i*n_mb .. (i+1)*n_mb); ms_out = CUDA-event time of the
 * timed steps (fp64 gather, score slicing, schedule, step, loss/codes D2H and
 * host sync of every step inside). */
int d2ft_engine_bench_e2e_units(d2ft_engine* e, const d2ft_dataset* ds, const int32_t* order, int n_mb, int mbs,
                                const double* bwd_scores, const double* fwd_scores, int total_units,
                                const int32_t* cf, const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd,
                                double lr, double momentum, int warmup, int steps, double* ms_out, double* loss_out);

/* Benchmark path: stage inputs once on the device, then run device-resident
 * steps (asynchronous on d2ft_engine_stream) and d2ft_engine_sync. */
int d2ft_engine_stage_device(d2ft_engine* e, const float* samples, const int32_t* labels, const double* bwd_scores,
                             const double* fwd_scores, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                             const int32_t* cap_fwd, int n_mb, int mbs);
int d2ft_engine_step_resident(d2ft_engine* e, int n_mb, int mbs, double lr, double momentum);
int d2ft_engine_sync(d2ft_engine* e, double* loss_out);
/* Timed loops for bench.py: device-resident steps on the staged inputs, and
 * end-to-end host-buffer steps (H2D of samples/labels/scores + D2H of loss and
 * codes + host sync inside every step).  CUDA events on the engine stream;
 * ms_out = total ms over `steps`. */
int d2ft_engine_bench_device(d2ft_engine* e, int n_mb, int mbs, double lr, double momentum, int warmup, int steps,
                             double* ms_out, double* loss_out);
int d2ft_engine_bench_e2e(d2ft_engine* e, const float* samples, const int32_t* labels, const double* bwd_scores,
                          const double* fwd_scores, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                          const int32_t* cap_fwd, int n_mb, int mbs, double lr, double momentum, int warmup,
                          int steps, double* ms_out, double* loss_out);
void* d2ft_engine_stream(d2ft_engine* e);

/* Per-phase device time (CUDA events between phases) accumulated while
 * profiling is on: sched, embed, ln, G1, attn_fwd, G3, head, G4, attn_bwd,
 * G5, G7, G8, bias, ln_bwd, embed_wgrad, sgd. */
int d2ft_engine_set_profiling(d2ft_engine* e, int on);
int d2ft_engine_phase_ms(d2ft_engine* e, double* ms_out, int n, int* steps);
/* per-sample schedule codes of the last step, K x max_batch */
int d2ft_engine_codes(d2ft_engine* e, uint8_t* codes_exp_out);

/* n draws of uniform_double(make_rng(seed, stream)) (rng.hpp:24-31) */
int d2ft_uniform_stream(uint64_t seed, uint64_t stream, int n, double* out);
/* ---- head partition across GPUs (no reference counterpart:
 * the reference runs every subnet in one process).  Rank r of `world` owns
 * heads h with h % world == r of every block: it schedules every row (rows
 * are independent, so all ranks derive the same table), keeps its own rows,
 * and after each block's forward (partial block outputs) and backward (dxn
 * partials) the ranks sum their partials, the one data-path exchange.  The
 * embedding and classifier are replicated.  Parameters and gradients of a
 * head are authoritative on its owner only. */
typedef struct d2ft_local_group d2ft_local_group;
/* 128-byte NCCL unique id (rank 0 creates it, all ranks pass it below) */
int d2ft_nccl_unique_id(uint8_t* id_out);
/* join an NCCL group: one process per GPU, exchange = ncclAllReduce(sum) */
int d2ft_engine_partition_nccl(d2ft_engine* e, int rank, int world, const uint8_t* id);
/* in-process group of `world` engines on one device, stepped from `world`
 * host threads; exchange = fixed-order device sum (single-GPU test harness) */
int d2ft_local_group_create(int world, d2ft_local_group** out);
int d2ft_local_group_destroy(d2ft_local_group* g);
/* a rank failed: every rank waiting in the group's exchange returns a state error */
int d2ft_local_group_abort(d2ft_local_group* g);
int d2ft_engine_partition_local(d2ft_engine* e, d2ft_local_group* g, int rank);
/* Data parallelism over the GLOBAL batch (an alternative to the head
 * partition): rank r of `world` holds micro-batches [r*n_mb/world,
 * (r+1)*n_mb/world) of every batch.  After joining, the step entry points
 * (d2ft_engine_step, _step_pipelined, _step_codes, _stage_device /
 * _step_resident / _bench_device / _bench_e2e) take n_mb = the global
 * micro-batch count, the global K x n_mb score (or code) table, and THIS
 * rank's samples and labels only; every rank runs the same knapsack over the
 * global table, computes its samples' forward/backward with the global 1/B
 * loss weight, and the weight gradients are all-reduced (NCCL, captured in
 * the step graph) before the SGD, whose touched-subnet rule uses the global
 * Full counts — trainer.cpp:247-268 for the global batch.  loss_out is this
 * rank's share of the batch loss (sum over ranks = the batch loss).  State
 * errors: an engine already partitioned / data parallel, LoRA adapters,
 * the Dataset path.  n_mb must divide evenly over the ranks (config). */
int d2ft_engine_data_parallel_nccl(d2ft_engine* e, int rank, int world, const uint8_t* id);
int d2ft_engine_data_parallel_local(d2ft_engine* e, d2ft_local_group* g, int rank);

/* row -> rank mapping of a partitioned engine: owner[k] for every scheduled
 * subnet row k = l*H + h (default after joining: h % world, head-interleaved;
 * partition.py also builds the SPEC-literal contiguous mapping of
 * cost_sim.cpp:138-152, memory_units consecutive rows per device) */
int d2ft_engine_set_row_owner(d2ft_engine* e, const int32_t* owner, int K);
/* the per-block exchanges run per sample chunk (1..8, default 2 or
 * $D2FT_EXCH_CHUNKS) on an exchange stream, overlapping the next chunk's
 * G3 / G8 and the previous chunk's LayerNorm */
int d2ft_engine_set_exchange_chunks(d2ft_engine* e, int chunks);
/* all-reduce calls issued by this rank so far and their payload bytes
 * (graph replays included) */
int d2ft_engine_exchange_stats(d2ft_engine* e, unsigned long long* calls, unsigned long long* bytes);

/* select the CUDA device for subsequent engine/scheduler creation on this thread */
int d2ft_set_device(int device);
/* partition_model (model.cpp:140-156): canonical fp64 flat initial
 * parameters, bit-identical to the reference for the same config/seed. */
int d2ft_partition_model(const d2ft_model_config* cfg, double* out);
/* attach_lora's initial adapters (model.cpp:174-192): down = 0, up_q/k/v
 * ~ N(0, 1/rank) from make_rng(seed, 0x10000 + subnet index); layout as
 * d2ft_engine_attach_lora, L*H*3*(d*r + r*dh) doubles. */
int d2ft_lora_init(const d2ft_model_config* cfg, int rank, double* out);
/* make_synthetic_dataset (trainer.cpp:83-111), samples returned as fp32
 * (the engine's input precision; the fp64 draws are rounded once). */
int d2ft_make_synthetic_dataset(int num_samples, int num_classes, int token_dim, int seq_len, double noise,
                                uint64_t seed, float* samples, int32_t* labels);
/* the same draws kept in fp64: Dataset::samples of the reference bit for bit */
int d2ft_make_synthetic_dataset_f64(int num_samples, int num_classes, int token_dim, int seq_len, double noise,
                                    uint64_t seed, double* samples, int32_t* labels);

#ifdef __cplusplus
}
#endif
#endif
