// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference C++ library, compiled
// from the sources where they lie under /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libd2ft_ref.so.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.
//
// Every entry point calls the reference's own public API:
//   scheduler   proj/core/include/d2ft/scheduler.hpp:135-207
//   model       proj/core/include/d2ft/model.hpp:216-265
//   trainer     proj/core/include/d2ft/trainer.hpp:71-98, body of train()
//               at proj/core/src/trainer.cpp:247-268 (composed here with the
//               same public calls, in the same order)
//   rng         proj/core/include/d2ft/rng.hpp:16-59
//   cost_sim    proj/core/include/d2ft/cost_sim.hpp:18-103
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "d2ft/cost_sim.hpp"
#include "d2ft/data.hpp"
#include "d2ft/model.hpp"
#include "d2ft/rng.hpp"
#include "d2ft/scheduler.hpp"
#include "d2ft/scoring.hpp"
#include "d2ft/scoring.hpp"
#include "d2ft/trainer.hpp"

using namespace d2ft;

namespace {

thread_local std::string g_err;

int code_of(const Error& e) {
  switch (e.kind()) {
    case errc::config: return 1;
    case errc::input: return 2;
    case errc::dimension: return 3;
    case errc::state: return 4;
    case errc::numeric: return 5;
    case errc::size: return 6;
  }
  return 99;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

std::vector<std::vector<double>> rows_d(const double* p, int K, int N) {
  std::vector<std::vector<double>> r(static_cast<std::size_t>(K));
  for (int k = 0; k < K; ++k) r[k].assign(p + static_cast<std::size_t>(k) * N, p + static_cast<std::size_t>(k + 1) * N);
  return r;
}
std::vector<std::vector<int>> rows_i(const int32_t* p, int K, int N) {
  std::vector<std::vector<int>> r(static_cast<std::size_t>(K));
  for (int k = 0; k < K; ++k) r[k].assign(p + static_cast<std::size_t>(k) * N, p + static_cast<std::size_t>(k + 1) * N);
  return r;
}

ScoreTable make_table(const double* bwd, const double* fwd, int K, int N) {
  ScoreTable t;
  t.subnets = K;
  t.micro_batches = N;
  t.backward = rows_d(bwd, K, N);
  t.forward = rows_d(fwd, K, N);
  return t;
}

CostModel make_cost(int cf, int cb, const int32_t* cf_dev, const int32_t* cb_dev, int K) {
  CostModel cm;
  cm.forward_cost = cf;
  cm.backward_cost = cb;
  if (cf_dev) cm.forward_cost_per_device.assign(cf_dev, cf_dev + K);
  if (cb_dev) cm.backward_cost_per_device.assign(cb_dev, cb_dev + K);
  return cm;
}

struct RefModel {
  SubnetModel model;
  std::vector<Subnet> velocity;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- rng
// n draws of uniform_double from make_rng(seed, stream) (rng.hpp:24-31).
void ref_uniform_stream(uint64_t seed, uint64_t stream, int n, double* out) {
  auto rng = make_rng(seed, stream);
  for (int i = 0; i < n; ++i) out[i] = uniform_double(rng);
}
void ref_gaussian_stream(uint64_t seed, uint64_t stream, int n, double* out) {
  auto rng = make_rng(seed, stream);
  for (int i = 0; i < n; ++i) out[i] = gaussian(rng);
}
void ref_shuffle_iota(uint64_t seed, uint64_t stream, int n, int32_t* out) {
  auto rng = make_rng(seed, stream);
  std::vector<int> v(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = i;
  shuffle(v, rng);
  for (int i = 0; i < n; ++i) out[i] = v[i];
}

// ---------------------------------------------------------------- scheduler
int ref_dp_search(const double* scores, const int32_t* weights, const int32_t* caps, int K, int N,
                  int threads, uint8_t* sel_out, double* obj_out) {
  return guarded([&] {
    std::vector<int> c(caps, caps + K);
    DpResult r = dp_search(rows_d(scores, K, N), rows_i(weights, K, N), c, threads);
    for (int k = 0; k < K; ++k) {
      obj_out[k] = r.objective[k];
      std::memcpy(sel_out + static_cast<std::size_t>(k) * N, r.selection[k].data(), N);
    }
  });
}

int ref_merge_selections(const uint8_t* full_sel, const uint8_t* fwd_sel, int K, int N, uint8_t* codes) {
  return guarded([&] {
    std::vector<std::vector<uint8_t>> a(K), b(K);
    for (int k = 0; k < K; ++k) {
      a[k].assign(full_sel + static_cast<std::size_t>(k) * N, full_sel + static_cast<std::size_t>(k + 1) * N);
      b[k].assign(fwd_sel + static_cast<std::size_t>(k) * N, fwd_sel + static_cast<std::size_t>(k + 1) * N);
    }
    ScheduleTable t = merge_selections(a, b);
    std::memcpy(codes, t.codes.data(), t.codes.size());
  });
}

int ref_knapsack_schedule(const double* bwd, const double* fwd, int cf, int cb, const int32_t* cf_dev,
                          const int32_t* cb_dev, const int32_t* cap_full, const int32_t* cap_fwd, int K,
                          int N, int threads, uint8_t* codes) {
  return guarded([&] {
    Capacities caps;
    caps.full.assign(cap_full, cap_full + K);
    caps.fwd.assign(cap_fwd, cap_fwd + K);
    ScheduleTable t = knapsack_schedule(make_table(bwd, fwd, K, N), make_cost(cf, cb, cf_dev, cb_dev, K), caps, threads);
    std::memcpy(codes, t.codes.data(), t.codes.size());
  });
}

int ref_brute_force_schedule(const double* bwd, const double* fwd, int cf, int cb, const int32_t* cap_full,
                             const int32_t* cap_fwd, int K, int N, uint8_t* codes) {
  return guarded([&] {
    Capacities caps;
    caps.full.assign(cap_full, cap_full + K);
    caps.fwd.assign(cap_fwd, cap_fwd + K);
    ScheduleTable t = brute_force_schedule(make_table(bwd, fwd, K, N), make_cost(cf, cb, nullptr, nullptr, K), caps);
    std::memcpy(codes, t.codes.data(), t.codes.size());
  });
}

// mode: 0 Max, 1 Min, 2 Constant (scheduler.hpp:118-127)
int ref_scaler_schedule(const double* bwd, const double* fwd, int cf, int cb, const int32_t* total_cap, int K,
                        int N, int mode, double lambda, int threads, uint8_t* codes, double* lambda_used,
                        int* fell_back) {
  return guarded([&] {
    ScalerConfig sc;
    sc.mode = mode == 0 ? ScalerConfig::Mode::Max : mode == 1 ? ScalerConfig::Mode::Min : ScalerConfig::Mode::Constant;
    sc.lambda = lambda;
    std::vector<int> tc(total_cap, total_cap + K);
    ScalerResult r = scaler_schedule(make_table(bwd, fwd, K, N), make_cost(cf, cb, nullptr, nullptr, K), tc, sc, threads);
    std::memcpy(codes, r.table.codes.data(), r.table.codes.size());
    *lambda_used = r.lambda_used;
    *fell_back = r.fell_back ? 1 : 0;
  });
}

int ref_capacities_from_budget(int n_full, int n_fwd, const int32_t* ovr, int n_ovr, int cf, int cb, int K, int N,
                               int32_t* cap_full, int32_t* cap_fwd) {
  return guarded([&] {
    BudgetSpec b;
    b.n_full = n_full;
    b.n_fwd = n_fwd;
    for (int i = 0; i < n_ovr; ++i) b.overrides.push_back({ovr[3 * i], ovr[3 * i + 1], ovr[3 * i + 2]});
    Capacities c = capacities_from_budget(b, make_cost(cf, cb, nullptr, nullptr, K), K, N);
    for (int k = 0; k < K; ++k) {
      cap_full[k] = c.full[k];
      cap_fwd[k] = c.fwd[k];
    }
  });
}

// ---------------------------------------------------------------- model
void* ref_model_create(int L, int H, int d, int ffn, int T, int C, uint64_t seed) {
  try {
    ModelConfig cfg;
    cfg.num_blocks = L;
    cfg.heads_per_block = H;
    cfg.model_dim = d;
    cfg.ffn_hidden = ffn;
    cfg.seq_len = T;
    cfg.num_classes = C;
    cfg.seed = seed;
    auto* m = new RefModel{SubnetModel(cfg), {}};
    for (const Subnet& s : m->model.subnets()) m->velocity.push_back(zeros_like(s));
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

uint64_t ref_model_param_count(void* h) { return static_cast<RefModel*>(h)->model.parameter_count(); }

// attach_lora (model.cpp:165-195); velocities are re-made so they carry the
// adapter slots sgd_momentum_step visits in LoRA mode
int ref_model_attach_lora(void* h, int rank, double scaling) {
  return guarded([&] {
    auto* m = static_cast<RefModel*>(h);
    m->model.attach_lora(rank, scaling);
    m->velocity.clear();
    for (const Subnet& s : m->model.subnets()) m->velocity.push_back(zeros_like(s));
  });
}

// doubles in the canonical flat vector, adapters included (parameter_bytes(true))
int64_t ref_model_flat_count(void* h) {
  return static_cast<int64_t>(static_cast<RefModel*>(h)->model.parameter_bytes(true).size() / sizeof(double));
}

// canonical order (model.hpp:117-153), identical to parameter_bytes()
void ref_model_get_params(void* h, double* out) {
  auto* m = static_cast<RefModel*>(h);
  std::vector<uint8_t> b = m->model.parameter_bytes(true);
  std::memcpy(out, b.data(), b.size());
}

void ref_model_set_params(void* h, const double* in) {
  auto* m = static_cast<RefModel*>(h);
  std::size_t off = 0;
  for (Subnet& s : m->model.subnets()) {
    visit_tensors(s, [&](const char*, Matrix& mat) {
      std::memcpy(mat.data.data(), in + off, mat.data.size() * sizeof(double));
      off += mat.data.size();
    });
  }
}

void ref_model_get_velocity(void* h, double* out) {
  auto* m = static_cast<RefModel*>(h);
  std::size_t off = 0;
  for (Subnet& s : m->velocity) {
    visit_tensors(s, [&](const char*, Matrix& mat) {
      std::memcpy(out + off, mat.data.data(), mat.data.size() * sizeof(double));
      off += mat.data.size();
    });
  }
}

static void fill_inputs(const RefModel* m, const double* inputs, int n, std::vector<Matrix>& xs) {
  const ModelConfig& c = m->model.config();
  for (int i = 0; i < n; ++i) {
    Matrix x(c.seq_len, c.model_dim);
    std::memcpy(x.data.data(), inputs + static_cast<std::size_t>(i) * c.seq_len * c.model_dim,
                x.data.size() * sizeof(double));
    xs.push_back(std::move(x));
  }
}

// SubnetModel::forward_backward (model.cpp:416-520). grads_flat receives the
// canonical-order gradient of every subnet (zeros where not engaged).
int ref_forward_backward(void* h, const double* inputs, const int32_t* labels, int n, const uint8_t* column,
                         double* loss, double* grads_flat, uint8_t* engaged) {
  return guarded([&] {
    auto* m = static_cast<RefModel*>(h);
    std::vector<Matrix> xs;
    fill_inputs(m, inputs, n, xs);
    std::vector<int> lab(labels, labels + n);
    std::vector<OperationKind> col(static_cast<std::size_t>(m->model.scheduled_count()));
    for (std::size_t r = 0; r < col.size(); ++r) col[r] = static_cast<OperationKind>(column[r]);
    ForwardBackwardResult fb = m->model.forward_backward(xs, lab, col);
    *loss = fb.loss;
    std::size_t off = 0;
    for (std::size_t si = 0; si < fb.grads.size(); ++si) {
      const Subnet& s = m->model.subnets()[si];
      engaged[si] = fb.grads[si].has_value() ? 1 : 0;
      visit_tensors(s, [&](const char* name, const Matrix& mat) {
        if (fb.grads[si]) {
          visit_tensors(*fb.grads[si], [&](const char* gname, const Matrix& g) {
            if (std::strcmp(name, gname) == 0) std::memcpy(grads_flat + off, g.data.data(), g.data.size() * sizeof(double));
          });
        } else {
          std::memset(grads_flat + off, 0, mat.data.size() * sizeof(double));
        }
        off += mat.data.size();
      });
    }
  });
}

// prepass_scores (scoring.cpp:108-151) of the unmodified reference on a
// dataset of n samples; fwd / bwd receive ScoreTable::forward / backward
// (K x n/mbs, row-major).  Metrics: scoring.hpp Metric enum order.
int ref_prepass_scores(void* h, const double* inputs, const int32_t* labels, int n, int mbs, int fwd_metric,
                       int bwd_metric, int threads, double* fwd, double* bwd) {
  return guarded([&] {
    auto* m = static_cast<RefModel*>(h);
    Dataset ds;
    fill_inputs(m, inputs, n, ds.samples);
    ds.labels.assign(labels, labels + n);
    ds.num_classes = m->model.config().num_classes;
    ScoreTable t = prepass_scores(m->model, ds, mbs, static_cast<Metric>(fwd_metric), static_cast<Metric>(bwd_metric),
                                  threads);
    for (int k = 0; k < t.subnets; ++k)
      for (int u = 0; u < t.micro_batches; ++u) {
        fwd[static_cast<std::size_t>(k) * t.micro_batches + u] = t.fwd(k, u);
        bwd[static_cast<std::size_t>(k) * t.micro_batches + u] = t.bwd(k, u);
      }
  });
}

// One D2FT batch exactly as the body of train() (trainer.cpp:247-268):
// forward_backward per micro-batch under table.column(j), accumulate with
// 1/n_mb in micro-batch order, sgd_momentum_step on subnets with accum.
// `inputs` holds the n_mb*mbs samples in unit order; codes is K x n_mb.
int ref_train_batch(void* h, const double* inputs, const int32_t* labels, int n_mb, int mbs, const uint8_t* codes,
                    double lr, double momentum, double* batch_loss) {
  return guarded([&] {
    auto* m = static_cast<RefModel*>(h);
    SubnetModel& model = m->model;
    const int K = model.scheduled_count();
    ScheduleTable table(K, n_mb);
    std::memcpy(table.codes.data(), codes, table.codes.size());
    table.validate();
    const ModelConfig& c = model.config();
    const double inv_mb = 1.0 / static_cast<double>(n_mb);
    std::vector<std::optional<Subnet>> accum(model.subnets().size());
    double loss = 0.0;
    for (int j = 0; j < n_mb; ++j) {
      std::vector<Matrix> xs;
      fill_inputs(m, inputs + static_cast<std::size_t>(j) * mbs * c.seq_len * c.model_dim, mbs, xs);
      std::vector<int> lab(labels + static_cast<std::size_t>(j) * mbs, labels + static_cast<std::size_t>(j + 1) * mbs);
      ForwardBackwardResult fb = model.forward_backward(xs, lab, table.column(j));
      loss += fb.loss * inv_mb;
      for (std::size_t si = 0; si < fb.grads.size(); ++si) {
        if (!fb.grads[si]) continue;
        if (!accum[si]) accum[si].emplace(zeros_like(model.subnet(static_cast<int>(si))));
        accumulate(*accum[si], *fb.grads[si], inv_mb);
      }
    }
    for (std::size_t si = 0; si < accum.size(); ++si) {
      if (!accum[si]) continue;
      sgd_momentum_step(model.subnet(static_cast<int>(si)), *accum[si], m->velocity[si], lr, momentum,
                        model.lora_enabled());
    }
    *batch_loss = loss;
  });
}

// Same batch body, with the per-micro-batch forward_backward calls (const,
// independent) spread over `threads` host threads; accumulation and the SGD
// step stay sequential in micro-batch order, so results are identical to
// ref_train_batch (the harness-level parallel loop SURVEY.md §7 names).
int ref_train_batch_parallel(void* h, const double* inputs, const int32_t* labels, int n_mb, int mbs,
                             const uint8_t* codes, double lr, double momentum, int threads, double* batch_loss) {
  return guarded([&] {
    auto* m = static_cast<RefModel*>(h);
    SubnetModel& model = m->model;
    const int K = model.scheduled_count();
    ScheduleTable table(K, n_mb);
    std::memcpy(table.codes.data(), codes, table.codes.size());
    table.validate();
    const ModelConfig& c = model.config();
    std::vector<ForwardBackwardResult> res(static_cast<std::size_t>(n_mb));
    std::vector<std::string> errs(static_cast<std::size_t>(n_mb));
    auto work = [&](int t) {
      for (int j = t; j < n_mb; j += threads) {
        try {
          std::vector<Matrix> xs;
          fill_inputs(m, inputs + static_cast<std::size_t>(j) * mbs * c.seq_len * c.model_dim, mbs, xs);
          std::vector<int> lab(labels + static_cast<std::size_t>(j) * mbs, labels + static_cast<std::size_t>(j + 1) * mbs);
          res[j] = model.forward_backward(xs, lab, table.column(j));
        } catch (const std::exception& e) {
          errs[j] = e.what();
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw input_error(e);
    const double inv_mb = 1.0 / static_cast<double>(n_mb);
    std::vector<std::optional<Subnet>> accum(model.subnets().size());
    double loss = 0.0;
    for (int j = 0; j < n_mb; ++j) {
      loss += res[j].loss * inv_mb;
      for (std::size_t si = 0; si < res[j].grads.size(); ++si) {
        if (!res[j].grads[si]) continue;
        if (!accum[si]) accum[si].emplace(zeros_like(model.subnet(static_cast<int>(si))));
        accumulate(*accum[si], *res[j].grads[si], inv_mb);
      }
    }
    for (std::size_t si = 0; si < accum.size(); ++si) {
      if (!accum[si]) continue;
      sgd_momentum_step(model.subnet(static_cast<int>(si)), *accum[si], m->velocity[si], lr, momentum,
                        model.lora_enabled());
    }
    *batch_loss = loss;
  });
}

int ref_logits(void* h, const double* input, double* out) {
  return guarded([&] {
    auto* m = static_cast<RefModel*>(h);
    std::vector<Matrix> xs;
    fill_inputs(m, input, 1, xs);
    Matrix lg = m->model.logits(xs[0]);
    std::memcpy(out, lg.data.data(), lg.data.size() * sizeof(double));
  });
}

// make_synthetic_dataset (trainer.cpp:83-111)
int ref_make_dataset(int num_samples, int C, int d, int T, double noise, uint64_t seed, double* samples,
                     int32_t* labels) {
  return guarded([&] {
    SynthDatasetSpec spec;
    spec.num_samples = num_samples;
    spec.num_classes = C;
    spec.token_dim = d;
    spec.seq_len = T;
    spec.noise_level = noise;
    spec.seed = seed;
    Dataset ds = make_synthetic_dataset(spec);
    for (int i = 0; i < num_samples; ++i) {
      std::memcpy(samples + static_cast<std::size_t>(i) * T * d, ds.samples[i].data.data(),
                  static_cast<std::size_t>(T) * d * sizeof(double));
      labels[i] = ds.labels[i];
    }
  });
}

// ---------------------------------------------------------------- cost_sim
int ref_time_ms(const int32_t* cnt, const double* full_ms, const double* fwd_ms, int n, int count, int full,
                double* out) {
  return guarded([&] {
    DeviceProfile p;
    for (int j = 0; j < n; ++j) p.timing_table.push_back({cnt[j], full_ms[j], fwd_ms[j]});
    p.validate();
    *out = p.time_ms(count, full != 0);
  });
}

// out6 = compute_fraction, comm_fraction, workload_variance (devices),
// makespan_ms, imbalance_residual, workload_variance() over rows.
// n_dev == 0: only the three standalone metrics.
int ref_schedule_metrics(const uint8_t* codes, int K, int N, int cf, int cb, const int32_t* cf_dev,
                         const int32_t* cb_dev, int n_dev, const int32_t* mu, const int32_t* toff, const int32_t* tcnt,
                         const double* tfull, const double* tfwd, const int32_t* cap_full, const int32_t* cap_fwd,
                         double* out6, double* busy) {
  return guarded([&] {
    ScheduleTable t(K, N);
    for (size_t c = 0; c < static_cast<size_t>(K) * N; ++c) t.codes[c] = codes[c];
    CostModel cm = make_cost(cf, cb, cf_dev, cb_dev, K);
    out6[0] = compute_cost_fraction(t, cm);
    out6[1] = comm_cost_fraction(t);
    out6[5] = workload_variance(t, cm);
    out6[2] = out6[3] = out6[4] = 0.0;
    if (n_dev == 0) return;
    std::vector<DeviceProfile> profiles;
    for (int p = 0; p < n_dev; ++p) {
      DeviceProfile d;
      d.device_id = p;
      d.memory_units = mu[p];
      for (int j = toff[p]; j < toff[p + 1]; ++j) d.timing_table.push_back({tcnt[j], tfull[j], tfwd[j]});
      profiles.push_back(std::move(d));
    }
    Capacities caps;
    if (cap_full) {
      caps.full.assign(cap_full, cap_full + K);
      caps.fwd.assign(cap_fwd, cap_fwd + K);
    }
    BatchMetrics m = simulate_batch(t, profiles, cm, cap_full ? &caps : nullptr);
    out6[0] = m.compute_fraction;
    out6[1] = m.comm_fraction;
    out6[2] = m.workload_variance;
    out6[3] = m.makespan_ms;
    out6[4] = m.imbalance_residual;
    for (int p = 0; p < n_dev; ++p) busy[p] = m.per_device_busy_ms[p];
  });
}

// build_hetero_profiles (cost_sim.hpp:79-81): profiles as (memory_units,
// fast) pairs, budget overrides as (device, n_full, n_fwd) triples.
int ref_build_hetero_profiles(int mode, int count, int units, int max_prof, int* n_prof, int32_t* mu, int32_t* fast,
                              int32_t* ovr, int* n_ovr, int32_t* budget2) {
  return guarded([&] {
    HeteroSetup s = build_hetero_profiles(mode == 0 ? HeteroMode::Memory : HeteroMode::Compute, count, units);
    *n_prof = static_cast<int>(s.profiles.size());
    if (*n_prof > max_prof) throw size_error("too many profiles");
    for (int p = 0; p < *n_prof; ++p) {
      mu[p] = s.profiles[p].memory_units;
      fast[p] = s.profiles[p].speed_class == DeviceProfile::Speed::Fast;
    }
    *n_ovr = static_cast<int>(s.budget.overrides.size());
    for (int i = 0; i < *n_ovr && i < max_prof; ++i) {
      ovr[3 * i] = s.budget.overrides[i].device;
      ovr[3 * i + 1] = s.budget.overrides[i].n_full;
      ovr[3 * i + 2] = s.budget.overrides[i].n_fwd;
    }
    budget2[0] = s.budget.n_full;
    budget2[1] = s.budget.n_fwd;
  });
}

// lora_{compute,comm}_reference_points (cost_sim.hpp:96-101): 3 rows of
// (n_full, n_fwd, n_shortcut, computed_pct, nominal_pct, discrepancy).
int ref_lora_reference_points(int comm, int32_t* counts9, double* pct6, int32_t* disc3) {
  return guarded([&] {
    std::vector<ReferencePoint> pts = comm ? lora_comm_reference_points() : lora_compute_reference_points();
    for (int i = 0; i < 3; ++i) {
      counts9[3 * i] = pts[i].n_full;
      counts9[3 * i + 1] = pts[i].n_fwd;
      counts9[3 * i + 2] = pts[i].n_shortcut;
      pct6[2 * i] = pts[i].computed_pct;
      pct6[2 * i + 1] = pts[i].nominal_pct;
      disc3[i] = pts[i].discrepancy ? 1 : 0;
    }
  });
}

}  // extern "C"
