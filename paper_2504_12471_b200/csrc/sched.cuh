// Scheduler + compaction kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace d2ft_b200 {

// Device-resident outputs of the schedule/compaction launch for a K x N
// schedule with H heads per block (L = K / H blocks).
struct CompactLists {
  int32_t* fwd_idx;     // K x N   ascending micro-batches with code 1|2 per row
  int32_t* fwd_cnt;     // K
  int32_t* full_idx;    // K x N   ascending micro-batches with code 1 per row
  int32_t* full_cnt;    // K
  int32_t* act_heads;   // (N*L) x H  ascending heads with code 1|2 per (micro-batch, block)
  int32_t* act_cnt;     // N*L
  int32_t* full_heads;  // (N*L) x H  ascending heads with code 1
  int32_t* full_hcnt;   // N*L
};

struct SchedWorkspace {
  uint32_t* bits_global;      // decision bits when they do not fit shared memory (may be null)
  size_t bits_global_words;   // capacity of bits_global in 32-bit words
  unsigned int* done_counter; // one zero-initialised counter (last-block column compaction)
  int32_t* err_flag;          // device error slot (first non-OK status wins), may be null
};

// Bytes of dynamic shared memory the knapsack launch needs for N items and
// at most max_cols DP columns per pool; 0 if the decision bits must spill to
// global memory (then the launch uses SchedWorkspace::bits_global).
size_t knapsack_smem_bytes(int N, int max_cols, bool* bits_in_smem);
size_t knapsack_global_bits_words(int K, int N, int max_cols);

// knapsack_schedule (scheduler.cpp:222-236) fused with merge_selections and
// compaction: one CTA per row runs the count-compressed fp64 0/1 knapsack
// for the Full pool (weight cf+cb, capacity cap_full) then the Forward pool
// (weight cf, capacity cap_fwd), merges into codes, writes the row's lists;
// the last CTA to finish writes the per-(micro-batch, block) head lists.
// lists may be null (schedule only).  validate=true makes the kernel reject
// non-finite / negative scores into ws.err_flag (device-pointer API).
void launch_knapsack_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                              const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, int H,
                              int max_cols, uint8_t* codes, const CompactLists* lists,
                              const SchedWorkspace& ws, bool validate, cudaStream_t stream);

// dp_search rows (scheduler.cpp:121-189).  Rows whose weights are constant
// use the count-compressed kernel; the rest use the general kernel.
void launch_dp_const(const double* scores, const int32_t* row_wt, const int32_t* caps, const int32_t* rows,
                     int nrows, int N, int max_cols, uint8_t* sel, double* obj, const SchedWorkspace& ws,
                     cudaStream_t stream);
void launch_dp_general(const double* scores, const int32_t* weights, const int32_t* caps, const int32_t* rows,
                       int nrows, int N, int max_cap, uint8_t* sel, double* obj, uint32_t* bits_global,
                       double* vals_global, cudaStream_t stream);

// merge_selections (scheduler.cpp:191-220)
void launch_merge(const uint8_t* full_sel, const uint8_t* fwd_sel, size_t n, uint8_t* codes, cudaStream_t s);

// compaction only, from an existing code table
void launch_compact(const uint8_t* codes, int K, int N, int H, const CompactLists& lists, cudaStream_t s);

// scaler_schedule DP (scheduler.cpp:379-424): multiple-choice knapsack per row
// given lambda (computed on the host or by launch_scaler_lambda).
void launch_scaler(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                   const int32_t* total_cap, int K, int N, const double* lambda_dev, int max_cap,
                   uint8_t* codes, uint8_t* choice_global, double* vals_global, cudaStream_t s);

// brute_force_schedule (scheduler.cpp:248-302), N <= 14
void launch_brute_force(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                        const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes,
                        cudaStream_t s);

}  // namespace d2ft_b200
