// Reference-side binding: the d2ft scheduler API (core/include/d2ft/scheduler.hpp)
// implemented over the B200 C-ABI (include/d2ft_b200.h).
//
// A reference maintainer builds this file INSTEAD of core/src/scheduler.cpp and
// links libd2ft_b200.so: every caller of knapsack_schedule / dp_search /
// merge_selections / scaler_schedule / brute_force_schedule (trainer.cpp:226,
// cli.cpp:364, baselines, the tests) then runs the sm_100a kernels.  The small
// value-type methods and budget arithmetic are host bookkeeping, restated
// here; every DP, merge and enumeration goes through the C-ABI.  Errors come
// back as the reference's d2ft::Error with the same errc category.
#include <cmath>
#include <cstdio>
#include <optional>
#include <string>
#include <vector>

#include "d2ft/scheduler.hpp"
#include "d2ft_b200.h"

namespace d2ft {

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

std::vector<double> flatten(const std::vector<std::vector<double>>& rows, int n) {
  std::vector<double> out;
  out.reserve(rows.size() * static_cast<std::size_t>(n));
  for (const auto& r : rows) out.insert(out.end(), r.begin(), r.end());
  return out;
}

void row_costs(const CostModel& cm, int K, std::vector<int32_t>& cf, std::vector<int32_t>& cb) {
  cf.resize(static_cast<std::size_t>(K));
  cb.resize(static_cast<std::size_t>(K));
  for (int k = 0; k < K; ++k) {
    cf[static_cast<std::size_t>(k)] = cm.cf(k);
    cb[static_cast<std::size_t>(k)] = cm.cb(k);
  }
}

}  // namespace

// ----------------------------------------------------------- value types
int CostModel::op_cost(int device, std::uint8_t code) const {
  if (code == 1) return full_cost(device);
  if (code == 2) return cf(device);
  if (code == 3) return 0;
  throw input_error("invalid schedule code " + std::to_string(code));
}

void CostModel::validate() const {
  bool neg = forward_cost < 0 || backward_cost < 0;
  if (neg) throw config_error("cost model: costs must be nonnegative integers");
  for (int v : forward_cost_per_device)
    if (v < 0) throw config_error("cost model: per-device forward cost negative");
  for (int v : backward_cost_per_device)
    if (v < 0) throw config_error("cost model: per-device backward cost negative");
  if (comm_forward != comm_backward) throw config_error("cost model: comm units must match");
}

void Capacities::validate() const {
  if (full.size() != fwd.size()) throw input_error("capacities: pool sizes differ");
  for (int v : full)
    if (v < 0) throw input_error("capacities: negative full capacity");
  for (int v : fwd)
    if (v < 0) throw input_error("capacities: negative forward capacity");
}

int BudgetSpec::n_full_for(int device) const {
  for (const Override& o : overrides)
    if (o.device == device) return o.n_full;
  return n_full;
}

int BudgetSpec::n_fwd_for(int device) const {
  for (const Override& o : overrides)
    if (o.device == device) return o.n_fwd;
  return n_fwd;
}

void BudgetSpec::validate(int micro_batches) const {
  auto one = [&](int nf, int no) {
    if (nf < 0 || no < 0) throw input_error("budget: counts must be nonnegative");
    if (nf + no > micro_batches) throw input_error("budget: n_full + n_fwd exceeds micro-batches per batch");
  };
  one(n_full, n_fwd);
  for (const Override& o : overrides) one(o.n_full, o.n_fwd);
}

std::vector<OperationKind> ScheduleTable::column(int i) const {
  std::vector<OperationKind> out(static_cast<std::size_t>(devices));
  for (int k = 0; k < devices; ++k) out[static_cast<std::size_t>(k)] = op(k, i);
  return out;
}

ScheduleTable::Counts ScheduleTable::row_counts(int k) const {
  Counts c;
  for (int i = 0; i < micro_batches; ++i) {
    const std::uint8_t v = code(k, i);
    c.n_full += v == 1;
    c.n_fwd += v == 2;
    c.n_shortcut += v == 3;
  }
  return c;
}

void ScheduleTable::validate() const {
  if (devices < 0 || micro_batches < 0 ||
      codes.size() != static_cast<std::size_t>(devices) * static_cast<std::size_t>(micro_batches))
    throw input_error("schedule table: dimension mismatch");
  for (std::uint8_t c : codes)
    if (c < 1 || c > 3) throw input_error("schedule table: code out of range");
}

void ScalerConfig::validate() const {
  if (mode == Mode::Constant && !(lambda > 0.0)) throw config_error("scaler: constant lambda must be > 0");
}

// ----------------------------------------------------------- scheduling (GPU)
CostTables build_cost_tables(const CostModel& cost_model, int devices, int micro_batches) {
  if (devices < 1 || micro_batches < 1) throw input_error("cost tables require at least one device and one micro-batch");
  cost_model.validate();
  CostTables t;
  for (int k = 0; k < devices; ++k) {
    t.w_full.emplace_back(static_cast<std::size_t>(micro_batches), cost_model.full_cost(k));
    t.w_fwd.emplace_back(static_cast<std::size_t>(micro_batches), cost_model.cf(k));
  }
  return t;
}

DpResult dp_search(const std::vector<std::vector<double>>& scores, const std::vector<std::vector<int>>& weights,
                   const std::vector<int>& capacities, int /*threads: results never depend on it*/) {
  const int K = static_cast<int>(scores.size());
  if (weights.size() != scores.size() || capacities.size() != scores.size())
    throw input_error("dp_search: scores, weights and capacities must agree on device count");
  for (int cap : capacities)
    if (cap < 0) throw input_error("dp_search: negative capacity");
  for (int k = 0; k < K; ++k)
    if (scores[static_cast<std::size_t>(k)].size() != weights[static_cast<std::size_t>(k)].size())
      throw input_error("dp_search: score/weight row length mismatch");
  DpResult r;
  r.selection.resize(static_cast<std::size_t>(K));
  r.objective.assign(static_cast<std::size_t>(K), 0.0);
  bool rect = true;
  for (int k = 1; k < K; ++k) rect = rect && scores[static_cast<std::size_t>(k)].size() == scores[0].size();
  auto run = [&](int k0, int nk, int n) {
    std::vector<double> s;
    std::vector<int32_t> w, c;
    for (int k = k0; k < k0 + nk; ++k) {
      s.insert(s.end(), scores[static_cast<std::size_t>(k)].begin(), scores[static_cast<std::size_t>(k)].end());
      w.insert(w.end(), weights[static_cast<std::size_t>(k)].begin(), weights[static_cast<std::size_t>(k)].end());
      c.push_back(capacities[static_cast<std::size_t>(k)]);
    }
    std::vector<std::uint8_t> sel(static_cast<std::size_t>(nk) * n);
    std::vector<double> obj(static_cast<std::size_t>(nk));
    rethrow(d2ft_dp_search(s.data(), w.data(), c.data(), nk, n, sel.data(), obj.data()));
    for (int k = 0; k < nk; ++k) {
      r.selection[static_cast<std::size_t>(k0 + k)].assign(sel.begin() + static_cast<std::ptrdiff_t>(k) * n,
                                                           sel.begin() + static_cast<std::ptrdiff_t>(k + 1) * n);
      r.objective[static_cast<std::size_t>(k0 + k)] = obj[static_cast<std::size_t>(k)];
    }
  };
  if (K == 0) return r;
  if (rect) run(0, K, static_cast<int>(scores[0].size()));
  else
    for (int k = 0; k < K; ++k) run(k, 1, static_cast<int>(scores[static_cast<std::size_t>(k)].size()));
  return r;
}

ScheduleTable merge_selections(const std::vector<std::vector<std::uint8_t>>& full_selection,
                               const std::vector<std::vector<std::uint8_t>>& fwd_selection) {
  if (full_selection.size() != fwd_selection.size()) throw input_error("merge_selections: device counts differ");
  const int K = static_cast<int>(full_selection.size());
  const int n = K > 0 ? static_cast<int>(full_selection.front().size()) : 0;
  std::vector<std::uint8_t> a, b;
  for (int k = 0; k < K; ++k) {
    if (static_cast<int>(full_selection[static_cast<std::size_t>(k)].size()) != n ||
        static_cast<int>(fwd_selection[static_cast<std::size_t>(k)].size()) != n)
      throw input_error("merge_selections: ragged selection rows");
    a.insert(a.end(), full_selection[static_cast<std::size_t>(k)].begin(), full_selection[static_cast<std::size_t>(k)].end());
    b.insert(b.end(), fwd_selection[static_cast<std::size_t>(k)].begin(), fwd_selection[static_cast<std::size_t>(k)].end());
  }
  ScheduleTable out(K, n);
  if (K * n) rethrow(d2ft_merge_selections(a.data(), b.data(), K, n, out.codes.data()));
  return out;
}

ScheduleTable knapsack_schedule(const ScoreTable& scores, const CostModel& cost_model, const Capacities& capacities,
                                int /*threads*/) {
  scores.validate();
  capacities.validate();
  const int K = scores.subnets, n = scores.micro_batches;
  if (capacities.devices() != K) throw input_error("knapsack_schedule: capacities device count mismatch");
  if (K < 1 || n < 1) throw input_error("cost tables require at least one device and one micro-batch");
  cost_model.validate();
  std::vector<int32_t> cf, cb;
  row_costs(cost_model, K, cf, cb);
  const std::vector<double> b = flatten(scores.backward, n), f = flatten(scores.forward, n);
  ScheduleTable out(K, n);
  rethrow(d2ft_knapsack_schedule(b.data(), f.data(), cf.data(), cb.data(), capacities.full.data(),
                                 capacities.fwd.data(), K, n, out.codes.data()));
  return out;
}

ScheduleTable brute_force_schedule(const ScoreTable& scores, const CostModel& cost_model, const Capacities& capacities,
                                   int /*threads*/) {
  scores.validate();
  capacities.validate();
  const int K = scores.subnets, n = scores.micro_batches;
  if (capacities.devices() != K) throw input_error("brute_force_schedule: capacities device count mismatch");
  std::vector<int32_t> cf, cb;
  row_costs(cost_model, K, cf, cb);
  const std::vector<double> b = flatten(scores.backward, n), f = flatten(scores.forward, n);
  ScheduleTable out(K, n);
  rethrow(d2ft_brute_force_schedule(b.data(), f.data(), cf.data(), cb.data(), capacities.full.data(),
                                    capacities.fwd.data(), K, n, out.codes.data()));
  return out;
}

std::vector<double> schedule_objective(const ScheduleTable& table, const ScoreTable& scores) {
  if (table.devices != scores.subnets || table.micro_batches != scores.micro_batches)
    throw input_error("schedule_objective: table/score dimensions differ");
  std::vector<double> obj(static_cast<std::size_t>(table.devices), 0.0);
  for (int k = 0; k < table.devices; ++k)
    for (int i = 0; i < table.micro_batches; ++i) {
      const std::uint8_t c = table.code(k, i);
      if (c == 1) obj[static_cast<std::size_t>(k)] += scores.bwd(k, i) + scores.fwd(k, i);
      else if (c == 2) obj[static_cast<std::size_t>(k)] += scores.fwd(k, i);
    }
  return obj;
}

ScalerResult scaler_schedule(const ScoreTable& scores, const CostModel& cost_model,
                             const std::vector<int>& total_capacity, const ScalerConfig& scaler, int /*threads*/) {
  scores.validate();
  scaler.validate();
  cost_model.validate();
  const int K = scores.subnets, n = scores.micro_batches;
  if (static_cast<int>(total_capacity.size()) != K) throw input_error("scaler_schedule: capacity count mismatch");
  std::vector<int32_t> cf, cb;
  row_costs(cost_model, K, cf, cb);
  const std::vector<double> b = flatten(scores.backward, n), f = flatten(scores.forward, n);
  const int mode = scaler.mode == ScalerConfig::Mode::Max ? 0 : scaler.mode == ScalerConfig::Mode::Min ? 1 : 2;
  ScalerResult r;
  r.table = ScheduleTable(K, n);
  int fell = 0;
  rethrow(d2ft_scaler_schedule(b.data(), f.data(), cf.data(), cb.data(), total_capacity.data(), K, n, mode,
                               scaler.lambda, r.table.codes.data(), &r.lambda_used, &fell));
  r.fell_back = fell != 0;
  if (r.fell_back) std::fprintf(stderr, "[d2ft] scaler: degenerate all-zero scores, falling back to lambda=1\n");
  return r;
}

Capacities capacities_from_budget(const BudgetSpec& budget, const CostModel& cost_model, int devices,
                                  int micro_batches) {
  budget.validate(micro_batches);
  cost_model.validate();
  Capacities caps;
  for (int k = 0; k < devices; ++k) {
    caps.full.push_back(budget.n_full_for(k) * cost_model.full_cost(k));
    caps.fwd.push_back(budget.n_fwd_for(k) * cost_model.cf(k));
  }
  return caps;
}

int row_cost_units(const ScheduleTable& table, const CostModel& cost_model, int device) {
  int units = 0;
  for (int i = 0; i < table.micro_batches; ++i) units += cost_model.op_cost(device, table.code(device, i));
  return units;
}

SharedBudgetReport check_shared_budget(const ScheduleTable& table, const CostModel& cost_model,
                                       const Capacities& capacities) {
  table.validate();
  capacities.validate();
  if (capacities.devices() != table.devices) throw input_error("check_shared_budget: capacities device count mismatch");
  SharedBudgetReport rep;
  for (int k = 0; k < table.devices; ++k) {
    SharedBudgetReport::Entry e;
    e.device = k;
    e.cost_units = row_cost_units(table, cost_model, k);
    e.limit = capacities.full[static_cast<std::size_t>(k)] + capacities.fwd[static_cast<std::size_t>(k)];
    if (e.cost_units > e.limit) rep.violations.push_back(k);
    rep.devices.push_back(e);
  }
  return rep;
}

}  // namespace d2ft
