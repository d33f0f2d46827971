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
 * the first validation failure (numeric/input/config) seen on the device. */
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

#ifdef __cplusplus
}
#endif
#endif /* D2FT_B200_H */
