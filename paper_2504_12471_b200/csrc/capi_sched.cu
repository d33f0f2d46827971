// C-ABI: scheduler and compaction entry points (include/d2ft_b200.h).
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/d2ft_b200.h"
#include "common.cuh"
#include "sched.cuh"

namespace d2ft_b200 {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
std::atomic<unsigned long long> g_launches{0};

namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) D2FT_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void upload(const T* h, size_t count) {
    if (!count) return;
    D2FT_CUDA(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
    // from pageable memory cudaMemcpy returns once the bytes are staged, not
    // landed; the kernels run on non-blocking streams, so wait for the DMA
    D2FT_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  }
  void download(T* h, size_t count) const {
    if (count) D2FT_CUDA(cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost));
  }
};

// ScoreTable::validate (scoring.cpp:30-47): forward side first, then backward;
// every element finite then non-negative.
void validate_scores(const double* bwd, const double* fwd, size_t n) {
  const double* sides[2] = {fwd, bwd};
  for (int s = 0; s < 2; ++s)
    for (size_t c = 0; c < n; ++c) {
      D2FT_REQUIRE(std::isfinite(sides[s][c]), kNumeric, "score table contains non-finite entries");
      D2FT_REQUIRE(sides[s][c] >= 0.0, kNumeric, "score table contains negative entries");
    }
}

// Capacities::validate (scheduler.cpp:37-43), build_cost_tables dims
// (scheduler.cpp:105-107), CostModel::validate (scheduler.cpp:24-35).
void validate_knapsack(const int32_t* cf, const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd,
                       int K, int N) {
  for (int k = 0; k < K; ++k) D2FT_REQUIRE(cap_full[k] >= 0, kInput, "capacities: negative full capacity");
  for (int k = 0; k < K; ++k) D2FT_REQUIRE(cap_fwd[k] >= 0, kInput, "capacities: negative forward capacity");
  D2FT_REQUIRE(K >= 1 && N >= 1, kInput, "cost tables require at least one device and one micro-batch");
  for (int k = 0; k < K; ++k)
    D2FT_REQUIRE(cf[k] >= 0 && cb[k] >= 0, kConfig, "cost model: costs must be nonnegative integers");
}

int row_cols(int wt, int cap, int N) { return wt == 0 ? 1 : (cap / wt < N ? cap / wt : N) + 1; }

int knapsack_max_cols(const int32_t* cf, const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, int K,
                      int N) {
  int mc = 1;
  for (int k = 0; k < K; ++k) {
    mc = std::max(mc, row_cols(cf[k] + cb[k], cap_full[k], N));
    mc = std::max(mc, row_cols(cf[k], cap_fwd[k], N));
  }
  return mc;
}

}  // namespace

struct SchedCtx {
  int K, N, H, max_cols;
  DevBuf<double> bwd, fwd;
  DevBuf<int32_t> cf, cb, cap_full, cap_fwd;
  DevBuf<uint8_t> codes;
  DevBuf<int32_t> lists_mem;
  DevBuf<uint32_t> bits;
  DevBuf<unsigned int> counter;
  DevBuf<int32_t> err;
  CompactLists lists{};
  SchedWorkspace ws{};
  cudaStream_t stream = nullptr;
  double* h_bwd = nullptr;  // pinned staging
  double* h_fwd = nullptr;
  uint8_t* h_codes = nullptr;

  SchedCtx(int K_, int N_, int H_, int mc) : K(K_), N(N_), H(H_), max_cols(mc) {
    const size_t KN = (size_t)K * N;
    const int L = K / H;
    bwd.alloc(KN);
    fwd.alloc(KN);
    cf.alloc(K);
    cb.alloc(K);
    cap_full.alloc(K);
    cap_fwd.alloc(K);
    codes.alloc(KN);
    const size_t nl = 2 * KN + 2 * (size_t)K + 2 * (size_t)N * L * H + 2 * (size_t)N * L;
    lists_mem.alloc(nl);
    int32_t* p = lists_mem.p;
    lists.fwd_idx = p;
    p += KN;
    lists.full_idx = p;
    p += KN;
    lists.fwd_cnt = p;
    p += K;
    lists.full_cnt = p;
    p += K;
    lists.act_heads = p;
    p += (size_t)N * L * H;
    lists.full_heads = p;
    p += (size_t)N * L * H;
    lists.act_cnt = p;
    p += (size_t)N * L;
    lists.full_hcnt = p;
    bool in_smem = true;
    knapsack_smem_bytes(N, max_cols, &in_smem);
    if (!in_smem) {
      bits.alloc(knapsack_global_bits_words(K, N, max_cols));
      ws.bits_global = bits.p;
      ws.bits_global_words = bits.n;
    }
    counter.alloc(1);
    D2FT_CUDA(cudaMemset(counter.p, 0, sizeof(unsigned int)));
    err.alloc(1);
    D2FT_CUDA(cudaMemset(err.p, 0, sizeof(int32_t)));
    ws.done_counter = counter.p;
    ws.err_flag = err.p;
    D2FT_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    D2FT_CUDA(cudaMallocHost(&h_bwd, KN * sizeof(double)));
    D2FT_CUDA(cudaMallocHost(&h_fwd, KN * sizeof(double)));
    D2FT_CUDA(cudaMallocHost(&h_codes, KN));
  }
  ~SchedCtx() {
    if (stream) cudaStreamDestroy(stream);
    if (h_bwd) cudaFreeHost(h_bwd);
    if (h_fwd) cudaFreeHost(h_fwd);
    if (h_codes) cudaFreeHost(h_codes);
  }

  void upload_costs(const int32_t* cf_h, const int32_t* cb_h, const int32_t* capf_h, const int32_t* capo_h) {
    D2FT_REQUIRE(knapsack_max_cols(cf_h, cb_h, capf_h, capo_h, K, N) <= max_cols, kSize,
                 "scheduler context: capacities exceed the max_cols the context was created for");
    cf.upload(cf_h, K);
    cb.upload(cb_h, K);
    cap_full.upload(capf_h, K);
    cap_fwd.upload(capo_h, K);
  }

  void launch(const double* b, const double* f, const int32_t* cf_d, const int32_t* cb_d, const int32_t* cfull,
              const int32_t* cfwd, uint8_t* out, bool with_lists, int32_t* err_dev, bool validate, cudaStream_t s) {
    SchedWorkspace w = ws;
    if (err_dev) w.err_flag = err_dev;
    launch_knapsack_schedule(b, f, cf_d, cb_d, cfull, cfwd, K, N, H, max_cols, out, with_lists ? &lists : nullptr,
                             w, validate, s);
  }
};

}  // namespace d2ft_b200

using namespace d2ft_b200;

struct d2ft_sched {
  SchedCtx* ctx;
};

extern "C" {

const char* d2ft_last_error(void) { return g_last_error.c_str(); }

unsigned long long d2ft_launch_count(void) { return g_launches.load(); }

void* d2ft_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}
void d2ft_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int d2ft_build_info(int* sm_arch, int* abi_version) {
  if (sm_arch) *sm_arch = 100;
  if (abi_version) *abi_version = 1;
  return 0;
}

int d2ft_dp_search(const double* scores, const int32_t* weights, const int32_t* caps, int K, int N, uint8_t* sel_out,
                   double* obj_out) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "dp_search: negative dimensions");
    for (int k = 0; k < K; ++k) D2FT_REQUIRE(caps[k] >= 0, kInput, "dp_search: negative capacity");
    for (int k = 0; k < K; ++k) {  // scheduler.cpp:132-142, row by row
      for (int i = 0; i < N; ++i)
        D2FT_REQUIRE(std::isfinite(scores[(size_t)k * N + i]), kNumeric, "dp_search: non-finite score");
      for (int i = 0; i < N; ++i)
        D2FT_REQUIRE(weights[(size_t)k * N + i] >= 0, kInput, "dp_search: negative weight");
    }
    if (K == 0) return;
    if (N == 0) {
      for (int k = 0; k < K; ++k) obj_out[k] = 0.0;
      return;
    }
    std::vector<int32_t> const_rows, gen_rows, row_wt(K, 0);
    int max_cols = 1, max_cap = 0;
    for (int k = 0; k < K; ++k) {
      const int32_t* w = weights + (size_t)k * N;
      bool same = true;
      for (int i = 1; i < N && same; ++i) same = w[i] == w[0];
      if (same) {
        const_rows.push_back(k);
        row_wt[k] = w[0];
        max_cols = std::max(max_cols, row_cols(w[0], caps[k], N));
      } else {
        gen_rows.push_back(k);
        max_cap = std::max(max_cap, caps[k]);
      }
    }
    const size_t KN = (size_t)K * N;
    DevBuf<double> d_s(KN), d_obj(K);
    DevBuf<int32_t> d_w(KN), d_caps(K), d_rwt(K), d_rows(K);
    DevBuf<uint8_t> d_sel(KN);
    d_s.upload(scores, KN);
    d_w.upload(weights, KN);
    d_caps.upload(caps, K);
    d_rwt.upload(row_wt.data(), K);
    if (!const_rows.empty()) {
      d_rows.upload(const_rows.data(), const_rows.size());
      SchedWorkspace ws{};
      DevBuf<uint32_t> bits;
      bool in_smem = true;
      knapsack_smem_bytes(N, max_cols, &in_smem);
      if (!in_smem) {
        bits.alloc(knapsack_global_bits_words((int)const_rows.size(), N, max_cols));
        ws.bits_global = bits.p;
        ws.bits_global_words = bits.n;
      }
      launch_dp_const(d_s.p, d_rwt.p, d_caps.p, d_rows.p, (int)const_rows.size(), N, max_cols, d_sel.p, d_obj.p, ws,
                      nullptr);
      D2FT_CUDA(cudaDeviceSynchronize());
    }
    if (!gen_rows.empty()) {
      const size_t wordsW = (size_t)(max_cap + 1 + 31) / 32;
      const size_t nbits = gen_rows.size() * (size_t)N * wordsW;
      const size_t nvals = gen_rows.size() * 2 * (size_t)(max_cap + 1);
      D2FT_REQUIRE(nbits * 4 + nvals * 8 < (size_t)16 << 30, kSize, "dp_search: DP table exceeds 16 GiB");
      DevBuf<uint32_t> bits(nbits);
      DevBuf<double> vals(nvals);
      DevBuf<int32_t> d_grows(gen_rows.size());
      d_grows.upload(gen_rows.data(), gen_rows.size());
      launch_dp_general(d_s.p, d_w.p, d_caps.p, d_grows.p, (int)gen_rows.size(), N, max_cap, d_sel.p, d_obj.p,
                        bits.p, vals.p, nullptr);
      D2FT_CUDA(cudaDeviceSynchronize());
    }
    d_sel.download(sel_out, KN);
    d_obj.download(obj_out, K);
  });
}

int d2ft_merge_selections(const uint8_t* full_sel, const uint8_t* fwd_sel, int K, int N, uint8_t* codes_out) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "merge_selections: negative dimensions");
    const size_t n = (size_t)K * N;
    if (n == 0) return;
    DevBuf<uint8_t> a(n), b(n), c(n);
    a.upload(full_sel, n);
    b.upload(fwd_sel, n);
    launch_merge(a.p, b.p, n, c.p, nullptr);
    c.download(codes_out, n);
  });
}

int d2ft_knapsack_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                           const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes_out) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "knapsack_schedule: negative dimensions");
    validate_scores(bwd, fwd, (size_t)K * N);
    validate_knapsack(cf, cb, cap_full, cap_fwd, K, N);
    const int mc = knapsack_max_cols(cf, cb, cap_full, cap_fwd, K, N);
    SchedCtx ctx(K, N, 1, mc);
    ctx.upload_costs(cf, cb, cap_full, cap_fwd);
    ctx.bwd.upload(bwd, (size_t)K * N);
    ctx.fwd.upload(fwd, (size_t)K * N);
    ctx.launch(ctx.bwd.p, ctx.fwd.p, ctx.cf.p, ctx.cb.p, ctx.cap_full.p, ctx.cap_fwd.p, ctx.codes.p, false, nullptr,
               false, ctx.stream);
    D2FT_CUDA(cudaStreamSynchronize(ctx.stream));
    ctx.codes.download(codes_out, (size_t)K * N);
  });
}

int d2ft_scaler_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                         const int32_t* total_cap, int K, int N, int mode, double lambda, uint8_t* codes_out,
                         double* lambda_used, int* fell_back) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "scaler_schedule: negative dimensions");
    const size_t KN = (size_t)K * N;
    validate_scores(bwd, fwd, KN);                                     // scheduler.cpp:324
    D2FT_REQUIRE(mode >= 0 && mode <= 2, kConfig, "scaler: unknown mode");
    if (mode == 2) D2FT_REQUIRE(lambda > 0.0, kConfig, "scaler: constant lambda must be > 0");  // :98-102
    for (int k = 0; k < K; ++k)
      D2FT_REQUIRE(cf[k] >= 0 && cb[k] >= 0, kConfig, "cost model: costs must be nonnegative integers");
    for (int k = 0; k < K; ++k) D2FT_REQUIRE(total_cap[k] >= 0, kInput, "scaler_schedule: negative capacity");
    // lambda selection, scheduler.cpp:336-376 (a handful of scalar reductions)
    double max_fwd = 0.0, max_bwd = 0.0, min_pos_fwd = 0.0, min_pos_bwd = 0.0;
    bool have_f = false, have_b = false;
    for (size_t c = 0; c < KN; ++c) {
      const double f = fwd[c], b = bwd[c];
      max_fwd = std::max(max_fwd, f);
      max_bwd = std::max(max_bwd, b);
      if (f > 0.0 && (!have_f || f < min_pos_fwd)) min_pos_fwd = f, have_f = true;
      if (b > 0.0 && (!have_b || b < min_pos_bwd)) min_pos_bwd = b, have_b = true;
    }
    double lam = 1.0;
    int fb = 0;
    if (mode == 0) {
      if (max_fwd > 0.0 && have_b) lam = 0.5 * min_pos_bwd / max_fwd;
      else fb = 1;
    } else if (mode == 1) {
      if (have_f) lam = max_bwd > 0.0 ? 2.0 * max_bwd / min_pos_fwd : 1.0;
      else fb = 1;
    } else {
      lam = lambda;
    }
    *lambda_used = lam;
    *fell_back = fb;
    if (KN == 0) return;
    int max_cap = 0;
    for (int k = 0; k < K; ++k) max_cap = std::max(max_cap, total_cap[k]);
    const size_t nchoice = KN * (size_t)(max_cap + 1);
    D2FT_REQUIRE(nchoice + (size_t)K * 2 * (max_cap + 1) * 8 < (size_t)16 << 30, kSize,
                 "scaler_schedule: choice table exceeds 16 GiB");
    DevBuf<double> d_b(KN), d_f(KN), d_lam(1), vals((size_t)K * 2 * (max_cap + 1));
    DevBuf<int32_t> d_cf(K), d_cb(K), d_cap(K);
    DevBuf<uint8_t> d_codes(KN), choice(nchoice);
    d_b.upload(bwd, KN);
    d_f.upload(fwd, KN);
    d_lam.upload(&lam, 1);
    d_cf.upload(cf, K);
    d_cb.upload(cb, K);
    d_cap.upload(total_cap, K);
    launch_scaler(d_b.p, d_f.p, d_cf.p, d_cb.p, d_cap.p, K, N, d_lam.p, max_cap, d_codes.p, choice.p, vals.p,
                  nullptr);
    D2FT_CUDA(cudaDeviceSynchronize());
    d_codes.download(codes_out, KN);
  });
}

int d2ft_brute_force_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                              const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes_out) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "brute_force_schedule: negative dimensions");
    const size_t KN = (size_t)K * N;
    validate_scores(bwd, fwd, KN);  // scheduler.cpp:250
    for (int k = 0; k < K; ++k) D2FT_REQUIRE(cap_full[k] >= 0, kInput, "capacities: negative full capacity");
    for (int k = 0; k < K; ++k) D2FT_REQUIRE(cap_fwd[k] >= 0, kInput, "capacities: negative forward capacity");
    D2FT_REQUIRE(N <= 14, kSize,
                 "brute_force_schedule: " + std::to_string(N) + " micro-batches exceeds the 3^N enumeration bound (N <= 14)");
    if (K == 0) return;
    DevBuf<double> d_b(KN ? KN : 1), d_f(KN ? KN : 1);
    DevBuf<int32_t> d_cf(K), d_cb(K), d_cfu(K), d_cfw(K);
    DevBuf<uint8_t> d_codes(KN ? KN : 1);
    d_b.upload(bwd, KN);
    d_f.upload(fwd, KN);
    d_cf.upload(cf, K);
    d_cb.upload(cb, K);
    d_cfu.upload(cap_full, K);
    d_cfw.upload(cap_fwd, K);
    launch_brute_force(d_b.p, d_f.p, d_cf.p, d_cb.p, d_cfu.p, d_cfw.p, K, N, d_codes.p, nullptr);
    D2FT_CUDA(cudaDeviceSynchronize());
    d_codes.download(codes_out, KN);
  });
}

int d2ft_compact(const uint8_t* codes, int K, int N, int H, int32_t* fwd_idx, int32_t* fwd_cnt, int32_t* full_idx,
                 int32_t* full_cnt, int32_t* act_heads, int32_t* act_cnt, int32_t* full_heads, int32_t* full_hcnt) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 1 && N >= 1 && H >= 1 && K % H == 0, kInput, "compact: need K >= 1, N >= 1, K % H == 0");
    for (size_t c = 0; c < (size_t)K * N; ++c)
      D2FT_REQUIRE(codes[c] >= 1 && codes[c] <= 3, kInput, "schedule table: code out of range");
    SchedCtx ctx(K, N, H, 1);
    ctx.codes.upload(codes, (size_t)K * N);
    launch_compact(ctx.codes.p, K, N, H, ctx.lists, ctx.stream);
    D2FT_CUDA(cudaStreamSynchronize(ctx.stream));
    const int L = K / H;
    const size_t KN = (size_t)K * N, cells = (size_t)N * L;
    std::vector<int32_t> buf(ctx.lists_mem.n);
    ctx.lists_mem.download(buf.data(), buf.size());
    const int32_t* base = ctx.lists_mem.p;
    auto off = [&](const int32_t* p) { return (size_t)(p - base); };
    std::vector<int32_t> fc(K), uc(K), ac(cells), hc(cells);
    std::memcpy(fwd_cnt, buf.data() + off(ctx.lists.fwd_cnt), K * 4);
    std::memcpy(full_cnt, buf.data() + off(ctx.lists.full_cnt), K * 4);
    std::memcpy(act_cnt, buf.data() + off(ctx.lists.act_cnt), cells * 4);
    std::memcpy(full_hcnt, buf.data() + off(ctx.lists.full_hcnt), cells * 4);
    for (int k = 0; k < K; ++k) {
      std::memcpy(fwd_idx + (size_t)k * N, buf.data() + off(ctx.lists.fwd_idx) + (size_t)k * N, fwd_cnt[k] * 4);
      std::memcpy(full_idx + (size_t)k * N, buf.data() + off(ctx.lists.full_idx) + (size_t)k * N, full_cnt[k] * 4);
    }
    for (size_t c = 0; c < cells; ++c) {
      std::memcpy(act_heads + c * H, buf.data() + off(ctx.lists.act_heads) + c * H, act_cnt[c] * 4);
      std::memcpy(full_heads + c * H, buf.data() + off(ctx.lists.full_heads) + c * H, full_hcnt[c] * 4);
    }
    (void)KN;
  });
}

int d2ft_sched_create(int K, int N, int H, int max_cols, d2ft_sched** out) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 1 && N >= 1 && H >= 1 && K % H == 0, kInput, "sched_create: need K,N,H >= 1 and K % H == 0");
    D2FT_REQUIRE(max_cols >= 1 && max_cols <= 2048, kSize, "sched_create: max_cols must be in [1, 2048]");
    *out = new d2ft_sched{new SchedCtx(K, N, H, max_cols)};
  });
}

int d2ft_sched_destroy(d2ft_sched* s) {
  return guarded([&] {
    if (s) {
      delete s->ctx;
      delete s;
    }
  });
}

int d2ft_sched_run_device(d2ft_sched* s, const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                          const int32_t* cap_full, const int32_t* cap_fwd, uint8_t* codes, int with_lists,
                          int32_t* err_dev, void* stream) {
  return guarded([&] {
    D2FT_REQUIRE(s && s->ctx, kState, "sched_run_device: null context");
    s->ctx->launch(bwd, fwd, cf, cb, cap_full, cap_fwd, codes, with_lists != 0, err_dev, true,
                   static_cast<cudaStream_t>(stream));
  });
}

int d2ft_sched_run_host(d2ft_sched* s, const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                        const int32_t* cap_full, const int32_t* cap_fwd, uint8_t* codes_out) {
  return guarded([&] {
    D2FT_REQUIRE(s && s->ctx, kState, "sched_run_host: null context");
    SchedCtx& c = *s->ctx;
    const size_t KN = (size_t)c.K * c.N;
    validate_scores(bwd, fwd, KN);
    validate_knapsack(cf, cb, cap_full, cap_fwd, c.K, c.N);
    c.upload_costs(cf, cb, cap_full, cap_fwd);
    D2FT_CUDA(cudaMemcpyAsync(c.bwd.p, bwd, KN * 8, cudaMemcpyHostToDevice, c.stream));
    D2FT_CUDA(cudaMemcpyAsync(c.fwd.p, fwd, KN * 8, cudaMemcpyHostToDevice, c.stream));
    c.launch(c.bwd.p, c.fwd.p, c.cf.p, c.cb.p, c.cap_full.p, c.cap_fwd.p, c.codes.p, true, nullptr, false, c.stream);
    D2FT_CUDA(cudaMemcpyAsync(codes_out, c.codes.p, KN, cudaMemcpyDeviceToHost, c.stream));
    D2FT_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int d2ft_sched_bench(d2ft_sched* s, const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                     const int32_t* cap_full, const int32_t* cap_fwd, int warmup, int iters, double* us_device,
                     double* us_e2e, uint8_t* codes_out) {
  return guarded([&] {
    D2FT_REQUIRE(s && s->ctx && iters >= 1, kState, "sched_bench: bad arguments");
    SchedCtx& c = *s->ctx;
    const size_t KN = (size_t)c.K * c.N;
    validate_scores(bwd, fwd, KN);
    validate_knapsack(cf, cb, cap_full, cap_fwd, c.K, c.N);
    c.upload_costs(cf, cb, cap_full, cap_fwd);
    std::memcpy(c.h_bwd, bwd, KN * 8);
    std::memcpy(c.h_fwd, fwd, KN * 8);
    c.bwd.upload(bwd, KN);
    c.fwd.upload(fwd, KN);
    cudaEvent_t e0, e1;
    D2FT_CUDA(cudaEventCreate(&e0));
    D2FT_CUDA(cudaEventCreate(&e1));
    for (int i = 0; i < warmup; ++i)
      c.launch(c.bwd.p, c.fwd.p, c.cf.p, c.cb.p, c.cap_full.p, c.cap_fwd.p, c.codes.p, true, nullptr, false, c.stream);
    D2FT_CUDA(cudaStreamSynchronize(c.stream));
    D2FT_CUDA(cudaEventRecord(e0, c.stream));
    for (int i = 0; i < iters; ++i)
      c.launch(c.bwd.p, c.fwd.p, c.cf.p, c.cb.p, c.cap_full.p, c.cap_fwd.p, c.codes.p, true, nullptr, false, c.stream);
    D2FT_CUDA(cudaEventRecord(e1, c.stream));
    D2FT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *us_device = 1000.0 * ms / iters;
    // end to end from pinned host buffers: H2D scores, schedule, D2H codes
    D2FT_CUDA(cudaEventRecord(e0, c.stream));
    for (int i = 0; i < iters; ++i) {
      D2FT_CUDA(cudaMemcpyAsync(c.bwd.p, c.h_bwd, KN * 8, cudaMemcpyHostToDevice, c.stream));
      D2FT_CUDA(cudaMemcpyAsync(c.fwd.p, c.h_fwd, KN * 8, cudaMemcpyHostToDevice, c.stream));
      c.launch(c.bwd.p, c.fwd.p, c.cf.p, c.cb.p, c.cap_full.p, c.cap_fwd.p, c.codes.p, true, nullptr, false, c.stream);
      D2FT_CUDA(cudaMemcpyAsync(c.h_codes, c.codes.p, KN, cudaMemcpyDeviceToHost, c.stream));
      D2FT_CUDA(cudaStreamSynchronize(c.stream));
    }
    D2FT_CUDA(cudaEventRecord(e1, c.stream));
    D2FT_CUDA(cudaEventSynchronize(e1));
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *us_e2e = 1000.0 * ms / iters;
    std::memcpy(codes_out, c.h_codes, KN);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int d2ft_sched_lists(d2ft_sched* s, int32_t** fwd_idx, int32_t** fwd_cnt, int32_t** full_idx, int32_t** full_cnt,
                     int32_t** act_heads, int32_t** act_cnt, int32_t** full_heads, int32_t** full_hcnt) {
  return guarded([&] {
    D2FT_REQUIRE(s && s->ctx, kState, "sched_lists: null context");
    const CompactLists& l = s->ctx->lists;
    *fwd_idx = l.fwd_idx;
    *fwd_cnt = l.fwd_cnt;
    *full_idx = l.full_idx;
    *full_cnt = l.full_cnt;
    *act_heads = l.act_heads;
    *act_cnt = l.act_cnt;
    *full_heads = l.full_heads;
    *full_hcnt = l.full_hcnt;
  });
}

}  // extern "C"
