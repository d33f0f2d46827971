/* d2ft_b200 — C-ABI of the B200-native D2FT hot path.
 *
 * This header is the drop-in boundary.  Every entry point
 * replaces one reference interface, cited per function as
 * /root/reference/proj/<file>:<line>.  Plain pointers and sizes only; no
 * torch or C++ types.  All functions return a status:
 *     0 OK
 *     1 config  2 input  3 dimension  4 state  5 numeric  6 size
 *       (the reference's d2ft::errc, core/include/d2ft/error.hpp:12-19)
 *     7 cuda    (device/runtime failure; no CPU fallback exists)
 * and d2ft_last_error() returns a thread-local message for the last failure.
 * Inputs are validated BEFORE any launch, mirroring the reference's
 * "worker threads must not throw" pre-validation (core/src/scheduler.cpp:131-142).
 *
 * Memory conventions: "host" entry points take host pointers and copy;
 * "_device" entry points take device pointers and a cudaStream_t (as void*),
 * never allocate and never synchronise.  Tables are row-major K x N with
 * K = scheduled subnets (L*H) and N = micro-batches, exactly the layout of
 * ScheduleTable::codes (core/include/d2ft/scheduler.hpp:86-96).
 */
#ifndef D2FT_B200_H
#define D2FT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define D2FT_OK 0
#define D2FT_ERR_CONFIG 1
#define D2FT_ERR_INPUT 2
#define D2FT_ERR_DIMENSION 3
#define D2FT_ERR_STATE 4
#define D2FT_ERR_NUMERIC 5
#define D2FT_ERR_SIZE 6
#define D2FT_ERR_CUDA 7

const char* d2ft_last_error(void);
/* kernels launched by this library so far (bench.py's gpu_launches) */
unsigned long long d2ft_launch_count(void);
/* page-locked host buffers (full-speed H2D for the end-to-end path) */
void* d2ft_host_alloc(size_t bytes);
void d2ft_host_free(void* p);
/* Library build tag and the sm arch the kernels were built for (100 = sm_100a). */
int d2ft_build_info(int* sm_arch, int* abi_version);

/* ------------------------------------------------------------------ scheduler
 * Cost model per row: cf[k] = CostModel::cf(k), cb[k] = CostModel::cb(k)
 * (scheduler.hpp:23-55; uniform models pass K equal entries). */

/* dp_search — scheduler.hpp:141-147, scheduler.cpp:121-189.
 * scores K x N fp64, weights K x N int32, caps K.  sel_out K x N (0/1),
 * obj_out K.  Bit-identical selections and objectives. */
int d2ft_dp_search(const double* scores, const int32_t* weights, const int32_t* caps, int K, int N,
                   uint8_t* sel_out, double* obj_out);

/* merge_selections — scheduler.hpp:151-152, scheduler.cpp:191-220. */
int d2ft_merge_selections(const uint8_t* full_sel, const uint8_t* fwd_sel, int K, int N, uint8_t* codes_out);

/* knapsack_schedule — scheduler.hpp:157-158, scheduler.cpp:222-236
 * (validate -> build_cost_tables -> dp_search x2 -> merge_selections).
 * bwd/fwd = ScoreTable::backward/forward (scoring.hpp:30-41). */
int d2ft_knapsack_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                           const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes_out);

/* scaler_schedule — scheduler.hpp:177-184, scheduler.cpp:321-426.
 * mode 0 = Max, 1 = Min, 2 = Constant(lambda). */
int d2ft_scaler_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                         const int32_t* total_cap, int K, int N, int mode, double lambda, uint8_t* codes_out,
                         double* lambda_used, int* fell_back);

/* brute_force_schedule — scheduler.hpp:162-163, scheduler.cpp:248-302:
 * exhaustive per-row optimum over 3^N assignments (N <= 14, else status 6). */
int d2ft_brute_force_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                              const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes_out);

/* Compaction of a code table (the implicit skips of model.cpp:431-436,
 * 455-466, 499-508 made explicit).  H = heads per block (K % H == 0),
 * L = K / H.  Outputs (host):
 *   fwd_idx  K x N  ascending micro-batches with code 1|2, fwd_cnt  K
 *   full_idx K x N  ascending micro-batches with code 1,   full_cnt K
 *   act_heads  (N*L) x H ascending heads with code 1|2 per (micro-batch, block), act_cnt  N*L
 *   full_heads (N*L) x H ascending heads with code 1,                        full_hcnt N*L
 * Unused tail entries are left untouched. */
int d2ft_compact(const uint8_t* codes, int K, int N, int H, int32_t* fwd_idx, int32_t* fwd_cnt,
                 int32_t* full_idx, int32_t* full_cnt, int32_t* act_heads, int32_t* act_cnt,
                 int32_t* full_heads, int32_t* full_hcnt);

/* Reusable scheduler context: pre-sized device buffers, pinned staging,
 * one fused schedule+merge+compaction launch per call. */
typedef struct d2ft_sched d2ft_sched;
int d2ft_sched_create(int K, int N, int H, int max_cols, d2ft_sched** out);
int d2ft_sched_destroy(d2ft_sched* s);
/* Device pointers; lists may be NULL.  err_dev (int32, may be NULL) receives
 * the first validation failure seen on the device: per row, in the
 * reference's order numeric (scores) > input (capacities) > config (costs),
 * then size (a row needing more DP columns than max_cols of the context; the
 * row is written as all-shortcut instead of being solved). */
int d2ft_sched_run_device(d2ft_sched* s, const double* bwd, const double* fwd, const int32_t* cf,
                          const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, uint8_t* codes,
                          int with_lists, int32_t* err_dev, void* stream);
/* Host buffers end to end: validate, H2D, schedule, D2H; synchronous. */
int d2ft_sched_run_host(d2ft_sched* s, const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                        const int32_t* cap_full, const int32_t* cap_fwd, uint8_t* codes_out);
/* Timing helper for bench.py: uploads once, then times `iters` fused launches
 * with CUDA events on the launching stream (us_device) and `iters` host
 * round trips (us_e2e, H2D of the scores + D2H of the codes included). */
int d2ft_sched_bench(d2ft_sched* s, const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                     const int32_t* cap_full, const int32_t* cap_fwd, int warmup, int iters, double* us_device,
                     double* us_e2e, uint8_t* codes_out);
/* Device views of the context's compaction lists (for the step engine). */
int d2ft_sched_lists(d2ft_sched* s, int32_t** fwd_idx, int32_t** fwd_cnt, int32_t** full_idx, int32_t** full_cnt,
                     int32_t** act_heads, int32_t** act_cnt, int32_t** full_heads, int32_t** full_hcnt);


/* ------------------------------------------------------------------ schedule metrics
 * cost_sim.hpp:57-90 (BatchMetrics, compute_cost_fraction, comm_cost_fraction,
 * workload_variance, simulate_batch), evaluated by one CUDA kernel over the
 * code table; bit-identical to the reference built without FMA contraction.
 * Field order is the order of the d2ft_schedule_metrics_device out6 array. */
typedef struct d2ft_batch_metrics {
  double compute_fraction;      /* compute_cost_fraction (cost_sim.cpp:71-81) */
  double comm_fraction;         /* comm_cost_fraction (cost_sim.cpp:83-93) */
  double workload_variance;     /* simulate_batch: over devices (cost_sim.cpp:159-166); 0 without devices */
  double makespan_ms;           /* max per-device busy time */
  double imbalance_residual;    /* || units_p - sum(cap_full + cap_fwd) || over devices (0 without capacities) */
  double row_workload_variance; /* workload_variance(): over schedule rows (cost_sim.cpp:95-107) */
} d2ft_batch_metrics;

/* DeviceProfile::time_ms (cost_sim.cpp:40-69): table of n entries (counts
 * strictly increasing), exact / interpolated / extrapolated busy ms. */
int d2ft_device_time_ms(const int32_t* counts, const double* full_ms, const double* fwd_ms, int n, int count,
                        int full, double* out);

/* simulate_batch (cost_sim.hpp:86-89, cost_sim.cpp:109-172) and the three
 * standalone metrics in one launch.  Host pointers; synchronous.
 *   codes K x N; cf/cb per row (CostModel::cf/cb).
 *   n_dev devices (0: fractions and row variance only), memory_units[n_dev]
 *   consecutive rows each (the reference's in-order row-to-device mapping).
 *   Busy time per device: busy_ms[n_dev] MEASURED (e.g. the head partition's
 *   per-rank busy time) when non-NULL, else the timing table of device p:
 *   entries [table_off[p], table_off[p+1]) of table_count / table_full_ms /
 *   table_fwd_ms (DeviceProfile::timing_table).
 *   cap_full/cap_fwd (K, may be NULL): Capacities for the imbalance residual.
 * Outputs: out; per_device_busy_ms[n_dev] and row_counts[K x 3] (n_full,
 * n_fwd, n_shortcut per row; ScheduleTable::row_counts) may be NULL. */
int d2ft_schedule_metrics(const uint8_t* codes, int K, int N, const int32_t* cf, const int32_t* cb, int n_dev,
                          const int32_t* memory_units, const int32_t* table_off, const int32_t* table_count,
                          const double* table_full_ms, const double* table_fwd_ms, const double* busy_ms,
                          const int32_t* cap_full, const int32_t* cap_fwd, d2ft_batch_metrics* out,
                          double* per_device_busy_ms, int32_t* row_counts);
/* Same on device pointers (e.g. the scheduler context's codes), no
 * allocation, no synchronisation: out6 = the six d2ft_batch_metrics fields
 * in order; err_dev (zeroed by the caller) receives 2 on an invalid code.
 * The caller validates profiles/capacities (d2ft_schedule_metrics does). */
int d2ft_schedule_metrics_device(const uint8_t* codes, int K, int N, const int32_t* cf, const int32_t* cb, int n_dev,
                                 const int32_t* memory_units, const int32_t* table_off, const int32_t* table_count,
                                 const double* table_full_ms, const double* table_fwd_ms, const double* busy_ms,
                                 const int32_t* cap_full, const int32_t* cap_fwd, double* out6,
                                 double* per_device_busy_ms, int32_t* row_counts, int32_t* err_dev, void* stream);


/* ------------------------------------------------------------------ artifact formats
 * serialize.hpp:21-53 / serialize.cpp:17-222: the reference pipeline's JSON
 * and CSV wire formats (host code; no GPU).  Text outputs go to a caller
 * buffer of `cap` bytes, NUL-terminated; *len = text length; status 6 (size)
 * with *len set when cap <= *len, so callers can size and retry.  JSON
 * layout is nlohmann::json::dump(2) (sorted keys, 2-space indent, shortest
 * round-trip doubles); metric ids are the Metric enum order of
 * scoring.hpp:18-23 (0 fisher_information .. 3 taylor_importance).
 * Readers take (text, n) and fail with the reference's messages. */
int d2ft_format_double(double v, char* buf, size_t cap, size_t* len);                       /* serialize.cpp:17-21 */
int d2ft_json_double(double v, char* buf, size_t cap, size_t* len);                         /* nlohmann layout */
int d2ft_score_table_to_json(const double* fwd, const double* bwd, int K, int N, int fwd_metric, int bwd_metric,
                             char* buf, size_t cap, size_t* len);                          /* serialize.cpp:66-75 */
/* fills K, N and the metric ids, then the K x N tables if cap_cells >= K*N (else status 6) */
int d2ft_score_table_from_json(const char* text, size_t n, int* K, int* N, int* fwd_metric, int* bwd_metric,
                               double* fwd, double* bwd, size_t cap_cells);                /* serialize.cpp:77-88 */
int d2ft_score_table_to_csv(const double* fwd, const double* bwd, int K, int N, char* buf, size_t cap,
                            size_t* len);                                                  /* serialize.cpp:90-99 */
int d2ft_schedule_table_to_json(const uint8_t* codes, int K, int N, char* buf, size_t cap,
                                size_t* len);                                              /* serialize.cpp:101-113 */
int d2ft_schedule_table_from_json(const char* text, size_t n, int* K, int* N, uint8_t* codes,
                                  size_t cap_cells);                                       /* serialize.cpp:115-135 */
int d2ft_schedule_table_to_csv(const uint8_t* codes, int K, int N, char* buf, size_t cap,
                               size_t* len);                                               /* serialize.cpp:137-146 */
int d2ft_batch_metrics_to_json(const d2ft_batch_metrics* m, const double* per_device_busy_ms, int n_dev,
                               const char* run_id, const char* method, char* buf, size_t cap,
                               size_t* len);                                               /* serialize.cpp:148-160 */
int d2ft_batch_metrics_csv_header(char* buf, size_t cap, size_t* len);                      /* serialize.cpp:162-165 */
int d2ft_batch_metrics_to_csv_row(const d2ft_batch_metrics* m, const char* run_id, const char* method, char* buf,
                                  size_t cap, size_t* len);                                /* serialize.cpp:167-173 */
/* TrainHistory (trainer.hpp:82-92) as parallel arrays of n epochs */
int d2ft_history_to_csv(const int32_t* epoch, const double* loss, const double* top1, const double* compute_fraction,
                        const double* comm_fraction, int n, char* buf, size_t cap, size_t* len); /* serialize.cpp:175-182 */
int d2ft_history_to_json(const int32_t* epoch, const double* loss, const double* top1, const double* compute_fraction,
                         const double* comm_fraction, int n, char* buf, size_t cap, size_t* len); /* serialize.cpp:184-198 */
int d2ft_history_from_csv(const char* text, size_t n_text, int32_t* epoch, double* loss, double* top1,
                          double* compute_fraction, double* comm_fraction, int cap, int* n); /* serialize.cpp:200-222 */
int d2ft_atomic_write_file(const char* path, const char* data, size_t n);                  /* serialize.cpp:23-34 */
int d2ft_read_file(const char* path, char* buf, size_t cap, size_t* len);                   /* serialize.cpp:36-42 */

#ifdef __cplusplus
}
#endif
#endif /* D2FT_B200_H */
