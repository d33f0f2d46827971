// Schedule metrics on the GPU: the reference's cost
// accounting and batch simulator (core/src/cost_sim.cpp:71-172) evaluated
// straight on a device-resident code table, so a step that schedules on the
// GPU reports its compute / communication fractions, workload variance and
// per-device busy time without copying the K x N codes back.
//
// One CTA: the per-row operation counts (the only O(K N) part) are warp
// reductions over the codes; the fp64 arithmetic that follows is O(K) and is
// done by one thread in the reference's summation order with no FMA
// contraction (__dadd_rn / __dmul_rn), so every output is bit-identical to
// compute_cost_fraction / comm_cost_fraction / workload_variance /
// simulate_batch compiled without FMA (the x86-64 baseline the reference
// builds for).
//
// Busy time: either the reference's calibrated timing table per device
// (DeviceProfile::time_ms, cost_sim.cpp:40-69, interpolation and
// extrapolation included) or MEASURED per-device busy milliseconds from the
// step (the head partition's per-rank busy time), which is what replaces the
// simulation on real hardware.
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/d2ft_b200.h"
#include "common.cuh"

namespace d2ft_b200 {
namespace {

constexpr int kMetricsThreads = 1024;

struct MetricsArgs {
  const uint8_t* codes;  // K x N
  int K, N;
  const int32_t* cf;  // K
  const int32_t* cb;  // K
  int n_dev;
  const int32_t* memory_units;  // n_dev (rows per device, in order)
  const int32_t* table_off;     // n_dev + 1 (device p: entries [off[p], off[p+1]))
  const int32_t* table_count;
  const double* table_full;
  const double* table_fwd;
  const double* busy_in;    // n_dev measured busy ms, or null (timing tables)
  const int32_t* cap_full;  // K or null
  const int32_t* cap_fwd;
  int32_t* row_counts;  // K x 3 (n_full, n_fwd, n_shortcut)
  double* busy_out;     // n_dev
  double* out;          // 6 doubles (d2ft_batch_metrics order)
  int32_t* err;         // first invalid code -> kInput
};

// DeviceProfile::time_ms (cost_sim.cpp:40-69) for one device's table.
__host__ __device__ double time_ms(const int32_t* cnt, const double* full_ms, const double* fwd_ms, int n, int count,
                                   bool full) {
  if (count == 0) return 0.0;
  const double* val = full ? full_ms : fwd_ms;
  for (int j = 0; j < n; ++j)
    if (cnt[j] == count) return val[j];
  int lo_count = 0;
  double lo_val = 0.0;
#ifdef __CUDA_ARCH__
#define D2FT_ADD(a, b) __dadd_rn((a), (b))
#define D2FT_MUL(a, b) __dmul_rn((a), (b))
#else
#define D2FT_ADD(a, b) ((a) + (b))
#define D2FT_MUL(a, b) ((a) * (b))
#endif
  for (int j = 0; j < n; ++j) {
    if (cnt[j] < count) {
      lo_count = cnt[j];
      lo_val = val[j];
    } else {
      const double slope = (val[j] - lo_val) / (double)(cnt[j] - lo_count);
      return D2FT_ADD(lo_val, D2FT_MUL(slope, (double)(count - lo_count)));
    }
  }
  int prev_count = 0;
  double prev_val = 0.0;
  if (n >= 2) {
    prev_count = cnt[n - 2];
    prev_val = val[n - 2];
  }
  const double slope = (val[n - 1] - prev_val) / (double)(cnt[n - 1] - prev_count);
  return D2FT_ADD(val[n - 1], D2FT_MUL(slope, (double)(count - cnt[n - 1])));
}

// population variance of v[0..n) in the reference's order (cost_sim.cpp:98-104, 159-165)
__device__ double pop_variance(const double* v, int n) {
  double mean = 0.0;
  for (int i = 0; i < n; ++i) mean = __dadd_rn(mean, v[i]);
  mean = mean / (double)n;
  double var = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = __dadd_rn(v[i], -mean);
    var = __dadd_rn(var, __dmul_rn(d, d));
  }
  return var / (double)n;
}

__global__ void __launch_bounds__(kMetricsThreads) schedule_metrics_kernel(MetricsArgs a) {
  extern __shared__ double loads[];  // max(K, n_dev)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ScheduleTable::row_counts (scheduler.cpp:76-86) per row; invalid codes
  // fail ScheduleTable::validate (scheduler.cpp:88-96)
  for (int k = warp; k < a.K; k += kMetricsThreads / 32) {
    const uint8_t* row = a.codes + (size_t)k * a.N;
    int nf = 0, no = 0, ns = 0, bad = 0;
    for (int i = lane; i < a.N; i += 32) {
      const uint8_t c = row[i];
      nf += c == 1;
      no += c == 2;
      ns += c == 3;
      bad |= (c < 1 || c > 3);
    }
    nf = __reduce_add_sync(0xffffffffu, nf);
    no = __reduce_add_sync(0xffffffffu, no);
    ns = __reduce_add_sync(0xffffffffu, ns);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) {
      a.row_counts[3 * k] = nf;
      a.row_counts[3 * k + 1] = no;
      a.row_counts[3 * k + 2] = ns;
      if (bad) atomicCAS(a.err, 0, (int)kInput);
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (*a.err) return;
  const int K = a.K, N = a.N;
  auto units_of = [&](int k) {  // row_cost_units (scheduler.cpp:442-446)
    const int full = a.cf[k] + a.cb[k];
    return a.row_counts[3 * k] * full + a.row_counts[3 * k + 1] * a.cf[k];
  };
  // compute_cost_fraction (cost_sim.cpp:71-81)
  long long used = 0, total = 0;
  for (int k = 0; k < K; ++k) {
    used += units_of(k);
    total += (long long)N * (a.cf[k] + a.cb[k]);
  }
  a.out[0] = total == 0 ? 0.0 : (double)used / (double)total;
  // comm_cost_fraction (cost_sim.cpp:83-93): p_f 1, p_o 1/2, exact in fp64
  long long twice = 0;
  for (int k = 0; k < K; ++k) twice += 2LL * a.row_counts[3 * k] + a.row_counts[3 * k + 1];
  const long long cells = (long long)K * N;
  a.out[1] = cells == 0 ? 0.0 : ((double)twice * 0.5) / (double)cells;
  // workload_variance per row (cost_sim.cpp:95-107)
  if (K == 0) {
    a.out[5] = 0.0;
  } else {
    for (int k = 0; k < K; ++k) {
      const double full_load = (double)N * (double)(a.cf[k] + a.cb[k]);
      loads[k] = full_load > 0.0 ? (double)units_of(k) / full_load : 0.0;
    }
    a.out[5] = pop_variance(loads, K);
  }
  // simulate_batch per device (cost_sim.cpp:109-172)
  double makespan = 0.0, residual_sq = 0.0;
  int row = 0;
  for (int p = 0; p < a.n_dev; ++p) {
    int n_full = 0, n_fwd = 0;
    long long units = 0, full_units = 0, limit_units = 0;
    for (int u = 0; u < a.memory_units[p]; ++u, ++row) {
      n_full += a.row_counts[3 * row];
      n_fwd += a.row_counts[3 * row + 1];
      units += units_of(row);
      full_units += (long long)N * (a.cf[row] + a.cb[row]);
      if (a.cap_full) limit_units += a.cap_full[row] + a.cap_fwd[row];
    }
    double busy;
    if (a.busy_in) {
      busy = a.busy_in[p];
    } else {
      const int o = a.table_off[p], n = a.table_off[p + 1] - o;
      busy = __dadd_rn(time_ms(a.table_count + o, a.table_full + o, a.table_fwd + o, n, n_full, true),
                       time_ms(a.table_count + o, a.table_full + o, a.table_fwd + o, n, n_fwd, false));
    }
    a.busy_out[p] = busy;
    makespan = makespan < busy ? busy : makespan;  // std::max
    loads[p] = full_units > 0 ? (double)units / (double)full_units : 0.0;
    if (a.cap_full) {
      const double diff = (double)units - (double)limit_units;
      residual_sq = __dadd_rn(residual_sq, __dmul_rn(diff, diff));
    }
  }
  a.out[2] = a.n_dev > 0 ? pop_variance(loads, a.n_dev) : 0.0;
  a.out[3] = makespan;
  a.out[4] = __dsqrt_rn(residual_sq);
}

// Host-side validation, in the reference's order: schedule (codes are
// checked on the device), DeviceProfile::validate per profile
// (cost_sim.cpp:22-38), hosted-unit count, capacity shape (cost_sim.cpp:113-131).
void validate_metrics(int K, int N, const int32_t* cf, const int32_t* cb, int n_dev, const int32_t* mu,
                      const int32_t* toff, const int32_t* tcnt, const double* tfull, const double* tfwd,
                      const double* busy, const int32_t* cap_full, const int32_t* cap_fwd) {
  D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "schedule table: dimension mismatch");
  for (int k = 0; k < K; ++k)
    D2FT_REQUIRE(cf[k] >= 0 && cb[k] >= 0, kConfig, "cost model: costs must be nonnegative integers");
  D2FT_REQUIRE(n_dev >= 0, kInput, "simulate_batch: negative device count");
  if (n_dev == 0) return;
  int hosted = 0;
  for (int p = 0; p < n_dev; ++p) {
    D2FT_REQUIRE(mu[p] >= 1, kInput, "device profile: memory_units must be >= 1");
    if (!busy) {
      const int o = toff[p], n = toff[p + 1] - o;
      D2FT_REQUIRE(n >= 1, kInput, "device profile: empty timing table");
      for (int j = 0; j < n; ++j) {
        D2FT_REQUIRE(tcnt[o + j] >= 1 && tfull[o + j] >= 0.0 && tfwd[o + j] >= 0.0, kInput,
                     "device profile: invalid timing entry");
        if (j > 0)
          D2FT_REQUIRE(tcnt[o + j] > tcnt[o + j - 1] && tfull[o + j] >= tfull[o + j - 1] &&
                           tfwd[o + j] >= tfwd[o + j - 1],
                       kInput, "device profile: timing table must be monotone nondecreasing");
      }
    } else {
      D2FT_REQUIRE(std::isfinite(busy[p]) && busy[p] >= 0.0, kNumeric, "simulate_batch: invalid measured busy time");
    }
    hosted += mu[p];
  }
  D2FT_REQUIRE(hosted == K, kInput,
               "simulate_batch: profiles host " + std::to_string(hosted) + " subnet units but the schedule has " +
                   std::to_string(K) + " rows");
  (void)cap_fwd;
  (void)cap_full;
}

void launch_metrics(const MetricsArgs& a, cudaStream_t st) {
  const int smem = (int)sizeof(double) * std::max(1, std::max(a.K, a.n_dev));
  D2FT_REQUIRE(smem <= 200 * 1024, kSize, "schedule metrics: more than 25600 rows or devices");
  if (smem > 48 * 1024)
    D2FT_CUDA(cudaFuncSetAttribute(schedule_metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  schedule_metrics_kernel<<<1, kMetricsThreads, smem, st>>>(a);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace
}  // namespace d2ft_b200

using namespace d2ft_b200;

extern "C" {

int d2ft_device_time_ms(const int32_t* counts, const double* full_ms, const double* fwd_ms, int n, int count,
                        int full, double* out) {
  return guarded([&] {
    D2FT_REQUIRE(count >= 0, kInput, "device profile: negative micro-batch count");
    D2FT_REQUIRE(n >= 1, kInput, "device profile: empty timing table");
    *out = time_ms(counts, full_ms, fwd_ms, n, count, full != 0);
  });
}

int d2ft_schedule_metrics_device(const uint8_t* codes, int K, int N, const int32_t* cf, const int32_t* cb, int n_dev,
                                 const int32_t* memory_units, const int32_t* table_off, const int32_t* table_count,
                                 const double* table_full_ms, const double* table_fwd_ms, const double* busy_ms,
                                 const int32_t* cap_full, const int32_t* cap_fwd, double* out6,
                                 double* per_device_busy_ms, int32_t* row_counts, int32_t* err_dev, void* stream) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0 && n_dev >= 0, kInput, "schedule metrics: negative dimensions");
    D2FT_REQUIRE(err_dev && out6 && row_counts, kInput, "schedule metrics: null output");
    MetricsArgs a{codes,       K,        N,       cf,         cb,      n_dev,      memory_units,
                  table_off,   table_count, table_full_ms, table_fwd_ms, busy_ms, cap_full,  cap_fwd,
                  row_counts,  per_device_busy_ms, out6, err_dev};
    launch_metrics(a, (cudaStream_t)stream);
  });
}

int d2ft_schedule_metrics(const uint8_t* codes, int K, int N, const int32_t* cf, const int32_t* cb, int n_dev,
                          const int32_t* memory_units, const int32_t* table_off, const int32_t* table_count,
                          const double* table_full_ms, const double* table_fwd_ms, const double* busy_ms,
                          const int32_t* cap_full, const int32_t* cap_fwd, d2ft_batch_metrics* out,
                          double* per_device_busy_ms, int32_t* row_counts) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "schedule table: dimension mismatch");
    for (size_t c = 0; c < (size_t)K * N; ++c)  // ScheduleTable::validate first (cost_sim.cpp:113)
      D2FT_REQUIRE(codes[c] >= 1 && codes[c] <= 3, kInput, "schedule table: code out of range");
    validate_metrics(K, N, cf, cb, n_dev, memory_units, table_off, table_count, table_full_ms, table_fwd_ms, busy_ms,
                     cap_full, cap_fwd);
    const int n_tab = (n_dev > 0 && !busy_ms) ? table_off[n_dev] : 0;
    // one device arena: codes | ints | doubles
    const size_t cells = (size_t)K * N;
    const size_t n_int = 2 * (size_t)K + (size_t)n_dev + (n_dev + 1) + n_tab + (cap_full ? 2 * (size_t)K : 0) +
                         3 * (size_t)K + 1;
    const size_t n_dbl = 2 * (size_t)n_tab + (busy_ms ? n_dev : 0) + n_dev + 6;
    const size_t off_int = (cells + 15) / 16 * 16, off_dbl = off_int + (n_int * 4 + 15) / 16 * 16;
    std::vector<uint8_t> h(off_dbl + n_dbl * 8, 0);
    std::memcpy(h.data(), codes, cells);
    int32_t* hi = reinterpret_cast<int32_t*>(h.data() + off_int);
    double* hd = reinterpret_cast<double*>(h.data() + off_dbl);
    size_t pi = 0, pd = 0;
    auto put_i = [&](const int32_t* s, size_t n) {
      size_t at = pi;
      if (s && n) std::memcpy(hi + pi, s, n * 4);
      pi += n;
      return at;
    };
    auto put_d = [&](const double* s, size_t n) {
      size_t at = pd;
      if (s && n) std::memcpy(hd + pd, s, n * 8);
      pd += n;
      return at;
    };
    const size_t i_cf = put_i(cf, K), i_cb = put_i(cb, K), i_mu = put_i(memory_units, n_dev);
    std::vector<int32_t> toff(n_dev + 1, 0);
    if (n_tab) for (int p = 0; p <= n_dev; ++p) toff[p] = table_off[p] - table_off[0];
    const size_t i_toff = put_i(toff.data(), n_dev + 1), i_tcnt = put_i(n_tab ? table_count + table_off[0] : nullptr, n_tab);
    size_t i_cfull = 0, i_cfwd = 0;
    if (cap_full) {
      i_cfull = put_i(cap_full, K);
      i_cfwd = put_i(cap_fwd, K);
    }
    const size_t i_rc = put_i(nullptr, 3 * (size_t)K), i_err = put_i(nullptr, 1);
    const size_t d_tfull = put_d(n_tab ? table_full_ms + table_off[0] : nullptr, n_tab),
                 d_tfwd = put_d(n_tab ? table_fwd_ms + table_off[0] : nullptr, n_tab);
    const size_t d_busy_in = put_d(busy_ms, busy_ms ? n_dev : 0);
    const size_t d_busy = put_d(nullptr, n_dev), d_out = put_d(nullptr, 6);
    uint8_t* dbase = nullptr;
    D2FT_CUDA(cudaMalloc(&dbase, h.size()));
    struct Free {
      uint8_t* p;
      ~Free() { cudaFree(p); }
    } guard{dbase};
    D2FT_CUDA(cudaMemcpy(dbase, h.data(), h.size(), cudaMemcpyHostToDevice));
    int32_t* di = reinterpret_cast<int32_t*>(dbase + off_int);
    double* dd = reinterpret_cast<double*>(dbase + off_dbl);
    MetricsArgs a{dbase,
                  K,
                  N,
                  di + i_cf,
                  di + i_cb,
                  n_dev,
                  di + i_mu,
                  di + i_toff,
                  di + i_tcnt,
                  dd + d_tfull,
                  dd + d_tfwd,
                  busy_ms ? dd + d_busy_in : nullptr,
                  cap_full ? di + i_cfull : nullptr,
                  cap_full ? di + i_cfwd : nullptr,
                  di + i_rc,
                  dd + d_busy,
                  dd + d_out,
                  di + i_err};
    launch_metrics(a, 0);
    D2FT_CUDA(cudaMemcpy(h.data(), dbase, h.size(), cudaMemcpyDeviceToHost));
    D2FT_REQUIRE(hi[i_err] == 0, kInput, "schedule table: code out of range");
    if (row_counts) std::memcpy(row_counts, hi + i_rc, 3 * (size_t)K * 4);
    if (per_device_busy_ms) std::memcpy(per_device_busy_ms, hd + d_busy, (size_t)n_dev * 8);
    const double* o = hd + d_out;
    out->compute_fraction = o[0];
    out->comm_fraction = o[1];
    out->workload_variance = o[2];
    out->makespan_ms = o[3];
    out->imbalance_residual = o[4];
    out->row_workload_variance = o[5];
  });
}

}  // extern "C"
