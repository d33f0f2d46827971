/* ORACLE / TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference's scheduler path, its RNG, its model
 * initialisation and synthetic data.
 * Each function cites the reference file:line it follows.  Pinned against
 *   (1) the literal expectations in proj/tests/test_scheduler.cpp (tests/
 *       test_oracle_pins.py) and
 *   (2) the unmodified reference built by oracle/Makefile (oracle/_ref),
 *       byte-for-byte on random instances (tests/test_oracle_vs_ref.py) and
 *       via committed golden vectors (tests/golden/).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 */
#ifndef D2FT_SCHED_ORACLE_H
#define D2FT_SCHED_ORACLE_H
#include <stdint.h>

/* rng.hpp:16-59 */
uint64_t or_splitmix64(uint64_t x);
void or_uniform_stream(uint64_t seed, uint64_t stream, int n, double* out);
void or_gaussian_stream(uint64_t seed, uint64_t stream, int n, double* out);
void or_shuffle_iota(uint64_t seed, uint64_t stream, int n, int32_t* out);

/* scheduler.cpp:121-189 (full (N+1)x(cap+1) table, strict >, != backtrack). */
int or_dp_search(const double* scores, const int32_t* weights, const int32_t* caps, int K, int N,
                 uint8_t* sel_out, double* obj_out);
/* scheduler.cpp:191-220 */
void or_merge_selections(const uint8_t* full_sel, const uint8_t* fwd_sel, int K, int N, uint8_t* codes);
/* scheduler.cpp:222-236 with build_cost_tables (scheduler.cpp:104-119).
 * cf/cb are per-row arrays (uniform models pass K copies). */
int or_knapsack_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                         const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes);
/* scheduler.cpp:321-426; mode 0 Max, 1 Min, 2 Constant */
int or_scaler_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                       const int32_t* total_cap, int K, int N, int mode, double lambda, uint8_t* codes,
                       double* lambda_used, int* fell_back);
/* scheduler.cpp:248-302 */
int or_brute_force_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                            const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes);
/* scheduler.cpp:442-446 */
int or_row_cost_units(const uint8_t* codes, int N, int cf, int cb);

/* Compaction restated from the implicit skips in model.cpp:431-436, 455-466,
 * 499-508: per scheduled row k the ascending micro-batch list with code 1|2
 * (forward set) and code 1 (Full set); per (micro-batch i, block l) the
 * ascending head list with code 1|2 and code 1.  H = heads per block,
 * L = K / H.  Arrays: fwd_idx/full_idx K x N, fwd_cnt/full_cnt K,
 * act_heads/full_heads (N*L) x H, act_cnt/full_hcnt N*L. */
void or_compact(const uint8_t* codes, int K, int N, int H, int32_t* fwd_idx, int32_t* fwd_cnt,
                int32_t* full_idx, int32_t* full_cnt, int32_t* act_heads, int32_t* act_cnt,
                int32_t* full_heads, int32_t* full_hcnt);

/* model.cpp:91-156: canonical flat fp64 parameter vector of partition_model. */
int64_t or_param_count(int L, int H, int d, int ffn, int T, int C);
void or_partition_model(int L, int H, int d, int ffn, int T, int C, uint64_t seed, double* out);
/* trainer.cpp:83-111 */
int or_make_dataset(int num_samples, int C, int d, int T, double noise, uint64_t seed, double* samples,
                    int32_t* labels);
#endif
