// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference artifact writers and
// readers (proj/core/src/serialize.cpp, compiled where it lies against the
// image's nlohmann json 3.11.3 by oracle/Makefile) so the tests can byte-
// compare this repo's writers (csrc/serialize.cu) with the reference's.
// Text results go to (buf, cap); *n = length; status 6 when cap is too small
// (the same convention as the product's text entry points).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "d2ft/error.hpp"
#include "d2ft/serialize.hpp"

using namespace d2ft;

namespace {

thread_local std::string g_ser_err;

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
int text_out(char* buf, size_t cap, size_t* n, F&& f) {
  std::string s;
  try {
    s = f();
  } catch (const Error& e) {
    g_ser_err = e.what();
    return code_of(e);
  } catch (const std::exception& e) {
    g_ser_err = e.what();
    return 99;
  }
  *n = s.size();
  if (s.size() + 1 > cap) return 6;
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return 0;
}

ScoreTable score_table(int K, int N, const double* fwd, const double* bwd, int fm, int bm) {
  ScoreTable t;
  t.subnets = K;
  t.micro_batches = N;
  t.fwd_metric = static_cast<Metric>(fm);
  t.bwd_metric = static_cast<Metric>(bm);
  t.forward.resize(K);
  t.backward.resize(K);
  for (int k = 0; k < K; ++k) {
    t.forward[k].assign(fwd + (size_t)k * N, fwd + (size_t)(k + 1) * N);
    t.backward[k].assign(bwd + (size_t)k * N, bwd + (size_t)(k + 1) * N);
  }
  return t;
}

TrainHistory history(int n, const int32_t* epoch, const double* loss, const double* top1, const double* cf,
                     const double* comm) {
  TrainHistory h;
  for (int i = 0; i < n; ++i) h.epochs.push_back(EpochRecord{epoch[i], loss[i], top1[i], cf[i], comm[i]});
  return h;
}

}  // namespace

extern "C" {

const char* ref_ser_last_error() { return g_ser_err.c_str(); }

int ref_ser_format_double(double v, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] { return format_double(v); });
}

// fmt 0 = JSON, 1 = CSV
int ref_ser_score_table(int K, int N, const double* fwd, const double* bwd, int fm, int bm, int fmt, char* buf,
                        size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] {
    const ScoreTable t = score_table(K, N, fwd, bwd, fm, bm);
    return fmt == 0 ? score_table_to_json(t) : score_table_to_csv(t);
  });
}

int ref_ser_schedule_table(int K, int N, const uint8_t* codes, int fmt, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] {
    ScheduleTable t(K, N);
    t.codes.assign(codes, codes + (size_t)K * N);
    return fmt == 0 ? schedule_table_to_json(t) : schedule_table_to_csv(t);
  });
}

// m = {compute_fraction, comm_fraction, workload_variance, makespan_ms,
// imbalance_residual}; fmt 0 = JSON, 1 = CSV row, 2 = CSV header
int ref_ser_batch_metrics(const double* m, const double* busy, int nbusy, const char* run_id, const char* method,
                          int fmt, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] {
    BatchMetrics b;
    b.compute_fraction = m[0];
    b.comm_fraction = m[1];
    b.workload_variance = m[2];
    b.makespan_ms = m[3];
    b.imbalance_residual = m[4];
    b.per_device_busy_ms.assign(busy, busy + nbusy);
    if (fmt == 2) return batch_metrics_csv_header();
    return fmt == 0 ? batch_metrics_to_json(b, run_id, method) : batch_metrics_to_csv_row(b, run_id, method);
  });
}

// fmt 0 = JSON, 1 = CSV
int ref_ser_history(int nep, const int32_t* epoch, const double* loss, const double* top1, const double* cf,
                    const double* comm, int fmt, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] {
    const TrainHistory h = history(nep, epoch, loss, top1, cf, comm);
    return fmt == 0 ? history_to_json(h) : history_to_csv(h);
  });
}

// Readers: parse with the reference, then re-emit with the reference's JSON
// (or CSV for the history) writer; a rejected input returns its errc status
// and message (ref_ser_last_error).
int ref_ser_score_table_reparse(const char* text, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] { return score_table_to_json(score_table_from_json(text)); });
}

int ref_ser_schedule_table_reparse(const char* text, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] { return schedule_table_to_json(schedule_table_from_json(text)); });
}

int ref_ser_history_reparse(const char* text, char* buf, size_t cap, size_t* n) {
  return text_out(buf, cap, n, [&] { return history_to_csv(history_from_csv(text)); });
}

}  // extern "C"
