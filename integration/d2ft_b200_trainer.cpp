// Operator / trainer binding over the B200 engine (see d2ft_b200_trainer.hpp).
// Host bookkeeping only: parameter layout conversion between the reference's
// Subnet tensors and the engine's canonical fp64 vector (model.hpp:117-153),
// the epoch / batch loop of train() (trainer.cpp:158-305) and its cost
// accounting.  Every forward, backward, schedule and update runs in the
// engine's sm_100a kernels.
#include "d2ft_b200_trainer.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <optional>
#include <string>

#include "d2ft/baselines.hpp"
#include "d2ft/linalg.hpp"
#include "d2ft/rng.hpp"
#include "d2ft/scheduler.hpp"
#include "d2ft/scoring.hpp"

namespace d2ft::b200 {

namespace {

void rethrow(int rc) {
  if (rc == D2FT_OK) return;
  const std::string msg = d2ft_last_error();
  switch (rc) {
    case D2FT_ERR_CONFIG: throw config_error(msg);
    case D2FT_ERR_INPUT: throw input_error(msg);
    case D2FT_ERR_DIMENSION: throw dimension_error(msg);
    case D2FT_ERR_STATE: throw state_error(msg);
    case D2FT_ERR_NUMERIC: throw numeric_error(msg);
    case D2FT_ERR_SIZE: throw size_error(msg);
    default: throw state_error("d2ft_b200 device failure: " + msg);
  }
}

bool is_adapter(const char* name) { return std::strncmp(name, "lora.", 5) == 0; }

// base tensors of every subnet in canonical order <-> flat fp64
std::vector<double> base_flat(const SubnetModel& m) {
  std::vector<double> out;
  out.reserve(m.parameter_count());
  for (const Subnet& s : m.subnets())
    visit_tensors(s, [&](const char* name, const Matrix& t) {
      if (!is_adapter(name)) out.insert(out.end(), t.data.begin(), t.data.end());
    });
  return out;
}

// adapters of the block subnets in visit_tensors order (d2ft_engine_attach_lora layout)
std::vector<double> adapter_flat(const SubnetModel& m) {
  std::vector<double> out;
  for (const Subnet& s : m.subnets())
    visit_tensors(s, [&](const char* name, const Matrix& t) {
      if (is_adapter(name)) out.insert(out.end(), t.data.begin(), t.data.end());
    });
  return out;
}

// flat (base) -> tensors of `subnets` selected by `take(si)`; adapters from `ad` when non-null
template <typename Take>
void scatter(std::vector<Subnet>& subnets, const std::vector<double>& flat, const std::vector<double>* ad,
             Take take) {
  size_t o = 0, oa = 0;
  for (size_t si = 0; si < subnets.size(); ++si) {
    const bool t = take(si);
    visit_tensors(subnets[si], [&](const char* name, Matrix& m) {
      const size_t n = m.data.size();
      if (is_adapter(name)) {
        if (ad && t) std::copy(ad->begin() + oa, ad->begin() + oa + n, m.data.begin());
        oa += n;
      } else {
        if (t) std::copy(flat.begin() + o, flat.begin() + o + n, m.data.begin());
        o += n;
      }
    });
  }
}

std::vector<float> to_f32(std::span<const Matrix> xs, int T, int d) {
  std::vector<float> out;
  out.reserve(xs.size() * (size_t)T * d);
  for (const Matrix& x : xs) {
    check_shape(x, T, d, "micro-batch input");
    for (double v : x.data) out.push_back(static_cast<float>(v));
  }
  return out;
}

// RAII dataset handle (borrows the samples; page-locks them)
struct DeviceDataset {
  d2ft_dataset* h = nullptr;
  DeviceDataset(const Dataset& ds, int num_classes) {
    std::vector<const double*> ptrs;
    for (const Matrix& m : ds.samples) ptrs.push_back(m.data.data());
    std::vector<int32_t> labels(ds.labels.begin(), ds.labels.end());
    const Matrix& s0 = ds.samples.front();
    rethrow(d2ft_dataset_create(ptrs.data(), labels.data(), ds.size(), num_classes, s0.rows, s0.cols, 1, &h));
  }
  ~DeviceDataset() { d2ft_dataset_destroy(h); }
};

}  // namespace

// ----------------------------------------------------------------- DeviceModel
DeviceModel::DeviceModel(const SubnetModel& host, int max_batch) : shape_(host), max_batch_(max_batch) {
  const ModelConfig& c = host.config();
  d2ft_model_config mc{c.num_blocks, c.heads_per_block, c.model_dim, c.ffn_hidden, c.seq_len, c.num_classes, c.seed};
  rethrow(d2ft_engine_create(&mc, max_batch, &eng_));
  try {
    upload(host);
  } catch (...) {
    d2ft_engine_destroy(eng_);
    throw;
  }
}

DeviceModel::~DeviceModel() { d2ft_engine_destroy(eng_); }

void DeviceModel::upload(const SubnetModel& host) {
  const std::vector<double> flat = base_flat(host);
  if ((int64_t)flat.size() != d2ft_engine_param_count(eng_)) throw dimension_error("upload: parameter count mismatch");
  rethrow(d2ft_engine_set_params(eng_, flat.data()));
  if (host.lora_enabled()) {
    const std::vector<double> ad = adapter_flat(host);
    const LoraAdapter& a = *host.subnet(1).lora;
    if (!lora_) {
      rethrow(d2ft_engine_attach_lora(eng_, a.rank, a.scaling, ad.data()));
      lora_ = true;
    } else {
      rethrow(d2ft_engine_set_lora(eng_, ad.data()));
    }
  } else if (lora_) {
    throw state_error("upload: the device model has adapters, the host model has none");
  }
}

void DeviceModel::download(SubnetModel& host, const std::vector<char>* touched) const {
  auto take = [&](size_t si) { return !touched || (*touched)[si] != 0; };
  if (lora_) {  // base tensors are frozen: only the adapters move (trainer.cpp:124-133)
    std::vector<double> ad((size_t)d2ft_engine_lora_count(eng_));
    rethrow(d2ft_engine_get_lora(eng_, 0, ad.data()));
    size_t oa = 0;
    for (size_t si = 0; si < host.subnets().size(); ++si)
      visit_tensors(host.subnet((int)si), [&](const char* name, Matrix& m) {
        if (!is_adapter(name)) return;
        if (take(si)) std::copy(ad.begin() + oa, ad.begin() + oa + m.data.size(), m.data.begin());
        oa += m.data.size();
      });
    return;
  }
  std::vector<double> flat((size_t)d2ft_engine_param_count(eng_));
  rethrow(d2ft_engine_get_params(eng_, flat.data()));
  scatter(host.subnets(), flat, nullptr, take);
}

ForwardBackwardResult DeviceModel::forward_backward(std::span<const Matrix> inputs, std::span<const int> labels,
                                                    std::span<const OperationKind> schedule_column) const {
  const ModelConfig& c = shape_.config();
  const int K = shape_.scheduled_count();
  if ((int)schedule_column.size() != K)
    throw input_error("schedule column must have one operation per scheduled subnet");  // model.cpp:420-422
  if (inputs.size() != labels.size() || inputs.empty())
    throw input_error("micro-batch inputs and labels must be non-empty and aligned");  // model.cpp:423-425
  if ((int)inputs.size() > max_batch_) throw size_error("forward_backward: micro-batch exceeds the device batch");
  const std::vector<float> x = to_f32(inputs, c.seq_len, c.model_dim);
  std::vector<int32_t> y(labels.begin(), labels.end());
  std::vector<uint8_t> col(K);
  for (int k = 0; k < K; ++k) col[k] = static_cast<uint8_t>(schedule_column[k]);
  ForwardBackwardResult out;
  rethrow(d2ft_engine_forward_backward(eng_, x.data(), y.data(), (int)y.size(), col.data(), &out.loss));
  // engaged: embed, head, Full block subnets (model.cpp:427-436)
  const size_t S = shape_.subnets().size();
  std::vector<char> take(S, 0);
  take.front() = take.back() = 1;
  for (int k = 0; k < K; ++k) take[shape_.subnet_index_of_scheduled(k)] = col[k] == 1;
  std::vector<Subnet> g;
  g.reserve(S);
  for (const Subnet& s : shape_.subnets()) g.push_back(zeros_like(s));
  if (!lora_) {
    std::vector<double> flat((size_t)d2ft_engine_param_count(eng_));
    rethrow(d2ft_engine_get_grads(eng_, flat.data()));
    scatter(g, flat, nullptr, [&](size_t si) { return take[si] != 0; });
  } else {  // LoRA: only adapter gradients (base tensors frozen, model.cpp:512-517)
    std::vector<double> ad((size_t)d2ft_engine_lora_count(eng_));
    rethrow(d2ft_engine_get_lora(eng_, 2, ad.data()));
    size_t oa = 0;
    for (size_t si = 0; si < S; ++si)
      visit_tensors(g[si], [&](const char* name, Matrix& m) {
        if (!is_adapter(name)) return;
        if (take[si]) std::copy(ad.begin() + oa, ad.begin() + oa + m.data.size(), m.data.begin());
        oa += m.data.size();
      });
  }
  out.grads.resize(S);
  for (size_t si = 0; si < S; ++si)
    if (take[si]) out.grads[si].emplace(std::move(g[si]));
  return out;
}

Matrix DeviceModel::logits(const Matrix& input) const {
  const ModelConfig& c = shape_.config();
  check_shape(input, c.seq_len, c.model_dim, "logits input");
  const std::vector<float> x = to_f32(std::span<const Matrix>(&input, 1), c.seq_len, c.model_dim);
  Matrix out(1, c.num_classes);
  rethrow(d2ft_engine_logits(eng_, x.data(), 1, out.data.data()));
  return out;
}

double evaluate(const DeviceModel& model, const Dataset& dataset) {
  if (dataset.size() == 0) return 0.0;
  const int C = model.config().num_classes;
  const int T = dataset.samples.front().rows, d = dataset.samples.front().cols;
  const int chunk = model.max_batch();
  int correct = 0;
  std::vector<double> lg((size_t)chunk * C);
  for (int i0 = 0; i0 < dataset.size(); i0 += chunk) {
    const int n = std::min(chunk, dataset.size() - i0);
    const std::vector<float> x = to_f32(std::span<const Matrix>(dataset.samples).subspan(i0, n), T, d);
    rethrow(d2ft_engine_logits(model.engine(), x.data(), n, lg.data()));
    for (int i = 0; i < n; ++i) {  // trainer.cpp:311-316: first maximum wins
      int best = 0;
      for (int j = 1; j < C; ++j)
        if (lg[(size_t)i * C + j] > lg[(size_t)i * C + best]) best = j;
      if (best == dataset.labels[i0 + i]) ++correct;
    }
  }
  return static_cast<double>(correct) / dataset.size();
}

// ----------------------------------------------------------------- train
TrainHistory train(SubnetModel& model, const Dataset& dataset, const TrainConfig& config) {
  config.validate(dataset.size());  // trainer.cpp:159-163: fails before touching the model
  for (const Matrix& sample : dataset.samples)
    check_shape(sample, model.config().seq_len, model.config().model_dim, "train sample");

  const int mbs = config.micro_batch_size;
  const int n_mb = config.micro_batches_per_batch();
  const int total_units = dataset.micro_batch_count(mbs);
  const int batches_per_epoch = total_units / n_mb;
  const int K = model.scheduled_count();
  const bool lora = model.lora_enabled();

  DeviceModel dev(model, config.batch_size);
  DeviceDataset dds(dataset, model.config().num_classes);

  // one-time scoring pre-pass on the device, in chunks of the device batch
  ScoreTable scores;
  const bool needs_scores = config.policy.kind == PolicyKind::D2FT || config.policy.kind == PolicyKind::Scaler;
  std::vector<double> s_fwd, s_bwd;  // K x total_units row-major
  if (needs_scores) {
    s_fwd.assign((size_t)K * total_units, 0.0);
    s_bwd.assign((size_t)K * total_units, 0.0);
    const int chunk_units = std::max(1, config.batch_size / mbs);
    std::vector<double> fo, bo;
    for (int u0 = 0; u0 < total_units; u0 += chunk_units) {
      const int nu = std::min(chunk_units, total_units - u0);
      const std::vector<float> x = to_f32(std::span<const Matrix>(dataset.samples).subspan((size_t)u0 * mbs,
                                                                                          (size_t)nu * mbs),
                                          model.config().seq_len, model.config().model_dim);
      std::vector<int32_t> y(dataset.labels.begin() + (size_t)u0 * mbs, dataset.labels.begin() + (size_t)(u0 + nu) * mbs);
      fo.assign((size_t)K * nu, 0.0);
      bo.assign((size_t)K * nu, 0.0);
      rethrow(d2ft_engine_prepass_scores(dev.engine(), x.data(), y.data(), nu * mbs, mbs,
                                         static_cast<int>(config.fwd_metric), static_cast<int>(config.bwd_metric),
                                         fo.data(), bo.data()));
      for (int k = 0; k < K; ++k)
        for (int u = 0; u < nu; ++u) {
          s_fwd[(size_t)k * total_units + u0 + u] = fo[(size_t)k * nu + u];
          s_bwd[(size_t)k * total_units + u0 + u] = bo[(size_t)k * nu + u];
        }
    }
    scores.subnets = K;
    scores.micro_batches = total_units;
    scores.fwd_metric = config.fwd_metric;
    scores.bwd_metric = config.bwd_metric;
    scores.forward.assign(K, std::vector<double>(total_units));
    scores.backward.assign(K, std::vector<double>(total_units));
    for (int k = 0; k < K; ++k)
      for (int u = 0; u < total_units; ++u) {
        scores.forward[k][u] = s_fwd[(size_t)k * total_units + u];
        scores.backward[k][u] = s_bwd[(size_t)k * total_units + u];
      }
    scores.validate();
  }

  const Capacities capacities = capacities_from_budget(config.budget, config.cost_model, K, n_mb);
  std::vector<int> total_capacity(K);
  for (int k = 0; k < K; ++k) total_capacity[k] = capacities.full[k] + capacities.fwd[k];
  std::vector<int32_t> cf(K), cb(K), capf(capacities.full.begin(), capacities.full.end()),
      capo(capacities.fwd.begin(), capacities.fwd.end());
  for (int k = 0; k < K; ++k) {
    cf[k] = config.cost_model.cf(k);
    cb[k] = config.cost_model.cb(k);
  }

  std::optional<DynamicPruningPolicy> pruning;
  if (config.policy.kind == PolicyKind::DPruningM)
    pruning.emplace(BaselineKind::dpruning_m(config.policy.refresh_interval));
  else if (config.policy.kind == PolicyKind::DPruningMG)
    pruning.emplace(BaselineKind::dpruning_mg(config.policy.refresh_interval));
  std::vector<double> last_grad_magnitudes;

  std::vector<int> unit_order(total_units);
  std::iota(unit_order.begin(), unit_order.end(), 0);
  // subnets the device has updated (trainer.cpp:264-268: embed / head every
  // batch outside LoRA mode, a block subnet when its row held a Full cell)
  std::vector<char> touched(model.subnets().size(), 0);
  TrainHistory history;
  int iteration = 0;
  std::vector<uint8_t> codes((size_t)K * n_mb);

  for (int epoch = 0; epoch < config.epochs; ++epoch) {
    auto erng = make_rng(config.seed, 0xE000u + static_cast<std::uint64_t>(epoch));
    shuffle(unit_order, erng);
    double epoch_loss = 0.0;
    long long used_units = 0, full_units = 0, comm_cells = 0;
    double used_comm = 0.0;

    for (int b = 0; b < batches_per_epoch; ++b) {
      std::vector<int32_t> units(unit_order.begin() + (size_t)b * n_mb, unit_order.begin() + (size_t)(b + 1) * n_mb);
      std::vector<int32_t> next;
      if (b + 1 < batches_per_epoch)
        next.assign(unit_order.begin() + (size_t)(b + 1) * n_mb, unit_order.begin() + (size_t)(b + 2) * n_mb);
      const int32_t* nx = next.empty() ? nullptr : next.data();
      double batch_loss = 0.0;
      ScheduleTable table(K, n_mb);
      if (config.policy.kind == PolicyKind::D2FT) {
        // knapsack_schedule(slice_scores(scores, units), ...) inside the step (trainer.cpp:224-227)
        rethrow(d2ft_engine_step_units(dev.engine(), dds.h, units.data(), n_mb, mbs, nx, s_bwd.data(), s_fwd.data(),
                                       total_units, cf.data(), cb.data(), capf.data(), capo.data(),
                                       config.learning_rate, config.momentum, &batch_loss, codes.data()));
        std::copy(codes.begin(), codes.end(), table.codes.begin());
      } else {
        switch (config.policy.kind) {  // trainer.cpp:220-243
          case PolicyKind::Standard:
            std::fill(table.codes.begin(), table.codes.end(), 1);
            break;
          case PolicyKind::Scaler: {
            ScoreTable s;  // slice_scores, trainer.cpp:139-154
            s.subnets = K;
            s.micro_batches = n_mb;
            s.fwd_metric = scores.fwd_metric;
            s.bwd_metric = scores.bwd_metric;
            s.forward.assign(K, {});
            s.backward.assign(K, {});
            for (int k = 0; k < K; ++k)
              for (int u : units) {
                s.forward[k].push_back(scores.fwd(k, u));
                s.backward[k].push_back(scores.bwd(k, u));
              }
            table = scaler_schedule(s, config.cost_model, total_capacity, config.policy.scaler, config.threads).table;
            break;
          }
          case PolicyKind::Random:
            table = random_schedule(config.budget, K, n_mb,
                                    splitmix64(config.seed ^ (0xB000u + static_cast<std::uint64_t>(iteration))));
            break;
          case PolicyKind::DPruningM:
          case PolicyKind::DPruningMG:
            dev.download(model, &touched);  // the policy ranks the current weights
            table = pruning->schedule(model, last_grad_magnitudes, config.budget, config.cost_model, n_mb, iteration);
            break;
          default:
            throw config_error("train: unknown policy");
        }
        rethrow(d2ft_engine_step_units_codes(dev.engine(), dds.h, units.data(), n_mb, mbs, nx, table.codes.data(),
                                             config.learning_rate, config.momentum, &batch_loss));
      }
      epoch_loss += batch_loss / batches_per_epoch;
      if (!lora) touched.front() = touched.back() = 1;
      for (int r = 0; r < K; ++r)
        for (int j = 0; j < n_mb; ++j)
          if (table.code(r, j) == 1) touched[model.subnet_index_of_scheduled(r)] = 1;

      for (int k = 0; k < K; ++k) {  // trainer.cpp:270-279
        used_units += row_cost_units(table, config.cost_model, k);
        full_units += static_cast<long long>(n_mb) * config.cost_model.full_cost(k);
      }
      for (std::uint8_t c : table.codes) {
        if (c == 1) used_comm += 1.0;
        else if (c == 2) used_comm += 0.5;
      }
      comm_cells += static_cast<long long>(K) * n_mb;

      if (pruning) {  // trainer.cpp:281-289: gradient magnitude of each touched row's batch gradient
        last_grad_magnitudes.assign(K, 0.0);
        std::vector<double> gflat((size_t)d2ft_engine_param_count(dev.engine()));
        std::vector<double> gad;
        if (lora) {
          gad.resize((size_t)d2ft_engine_lora_count(dev.engine()));
          rethrow(d2ft_engine_get_lora(dev.engine(), 2, gad.data()));
        } else {
          rethrow(d2ft_engine_get_grads(dev.engine(), gflat.data()));
        }
        std::vector<Subnet> g;
        for (const Subnet& s : model.subnets()) g.push_back(zeros_like(s));
        scatter(g, gflat, lora ? &gad : nullptr, [](size_t) { return true; });
        for (int r = 0; r < K; ++r) {
          bool touched = false;
          for (int j = 0; j < n_mb; ++j) touched |= table.code(r, j) == 1;
          if (touched)
            last_grad_magnitudes[r] = gradient_magnitude(g[model.subnet_index_of_scheduled(r)], lora);
        }
      }
      ++iteration;
    }

    dev.download(model, &touched);
    EpochRecord rec;
    rec.epoch = epoch;
    rec.loss = epoch_loss;
    rec.top1 = evaluate(dev, dataset);
    rec.compute_fraction = full_units > 0 ? static_cast<double>(used_units) / static_cast<double>(full_units) : 0.0;
    rec.comm_fraction = comm_cells > 0 ? used_comm / static_cast<double>(comm_cells) : 0.0;
    history.epochs.push_back(rec);
  }
  return history;
}

}  // namespace d2ft::b200
