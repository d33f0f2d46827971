// Host-side model initialisation and synthetic data of the product (SURVEY
// §8a rows a12, a21): the same deterministic streams as the reference so a
// B200 run starts from the reference's exact weights and inputs.
//   partition_model         model.cpp:91-156 (per-subnet streams make_rng(seed, index))
//   make_synthetic_dataset  trainer.cpp:61-111
//   make_rng / gaussian     rng.hpp:16-50 (std::mt19937_64 is fully specified by the standard)
#include <algorithm>
#include <cmath>
#include <string>
#include <cstring>
#include <random>

#include "../../include/d2ft_b200_engine.h"
#include "common.cuh"

namespace d2ft_b200 {
namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
std::mt19937_64 stream_rng(uint64_t seed, uint64_t stream) { return std::mt19937_64(splitmix64(seed ^ splitmix64(stream))); }
double unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
double normal(std::mt19937_64& g) {
  double u1 = unit(g);
  const double u2 = unit(g);
  while (u1 <= 0.0) u1 = unit(g);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}
double* fill(double* p, size_t n, std::mt19937_64& g, double sd) {
  for (size_t i = 0; i < n; ++i) p[i] = sd * normal(g);
  return p + n;
}
double* zeros(double* p, size_t n) {
  std::memset(p, 0, n * sizeof(double));
  return p + n;
}

}  // namespace
}  // namespace d2ft_b200

using namespace d2ft_b200;

extern "C" {

int d2ft_lora_init(const d2ft_model_config* c, int rank, double* out) {
  return guarded([&] {
    D2FT_REQUIRE(c && out, kInput, "lora_init: null argument");
    const int L = c->num_blocks, H = c->heads_per_block, d = c->model_dim;
    D2FT_REQUIRE(L >= 1 && H >= 1 && d >= 1 && d % H == 0, kConfig, "model config: invalid dimensions");
    const int dh = d / H;
    D2FT_REQUIRE(rank >= 1, kConfig, "lora rank must be >= 1");
    D2FT_REQUIRE(rank <= std::min(d, dh), kConfig,
                 "lora rank " + std::to_string(rank) + " exceeds min(d, d/H) = " + std::to_string(std::min(d, dh)));
    double* p = out;
    const double sd = 1.0 / std::sqrt(rank);
    for (int k = 0; k < L * H; ++k) {
      auto g = stream_rng(c->seed, 0x10000u + 1u + (uint64_t)k);  // subnet index 1 + l*H + h
      double* blk = p;
      for (int x = 0; x < 3; ++x) {
        p = zeros(p, (size_t)d * rank);   // down_x
        p += (size_t)rank * dh;           // up_x, filled below in q, k, v order
      }
      for (int x = 0; x < 3; ++x)
        fill(blk + (size_t)x * ((size_t)d * rank + (size_t)rank * dh) + (size_t)d * rank, (size_t)rank * dh, g, sd);
    }
  });
}

int d2ft_partition_model(const d2ft_model_config* c, double* out) {
  return guarded([&] {
    D2FT_REQUIRE(c && out, kInput, "partition_model: null argument");
    const int L = c->num_blocks, H = c->heads_per_block, d = c->model_dim, ffn = c->ffn_hidden, T = c->seq_len,
              C = c->num_classes;
    D2FT_REQUIRE(L >= 1 && H >= 1 && d >= 1 && ffn >= 1 && T >= 1 && C >= 1, kConfig,
                 "model config: all dimensions must be >= 1");
    D2FT_REQUIRE(d % H == 0, kConfig, "model config: model_dim must be divisible by heads_per_block");
    D2FT_REQUIRE(ffn % H == 0, kConfig, "model config: ffn_hidden must be divisible by heads_per_block");
    const size_t dh = d / H, fs = ffn / H;
    double* p = out;
    uint64_t index = 0;
    auto g = stream_rng(c->seed, index++);
    p = fill(p, (size_t)d * d, g, 1.0 / std::sqrt(d));
    p = zeros(p, d);
    p = fill(p, (size_t)T * d, g, 0.02);
    for (int l = 0; l < L; ++l)
      for (int h = 0; h < H; ++h) {
        auto b = stream_rng(c->seed, index++);
        const double isd = 1.0 / std::sqrt(d);
        p = fill(p, (size_t)d * dh, b, isd);  // wq
        p = fill(p, (size_t)d * dh, b, isd);  // wk
        p = fill(p, (size_t)d * dh, b, isd);  // wv
        p = fill(p, dh * d, b, isd);          // wo
        p = fill(p, (size_t)d * fs, b, isd);  // w1
        p = zeros(p, fs);                     // b1
        p = fill(p, fs * d, b, 1.0 / std::sqrt(ffn));  // w2
        p = zeros(p, d / H);                           // b2
      }
    auto hg = stream_rng(c->seed, index++);
    p = fill(p, (size_t)d * C, hg, 1.0 / std::sqrt(d));
    zeros(p, C);
  });
}

// rng.hpp:29-31: n draws of uniform_double from make_rng(seed, stream)
// (bench_scheduler.cpp:13-27 draws the synthetic score tables this way).
int d2ft_uniform_stream(uint64_t seed, uint64_t stream, int n, double* out) {
  return guarded([&] {
    auto g = stream_rng(seed, stream);
    for (int i = 0; i < n; ++i) out[i] = unit(g);
  });
}

int d2ft_set_device(int device) {
  return guarded([&] { D2FT_CUDA(cudaSetDevice(device)); });
}

}  // extern "C"

namespace {
template <typename T>
void synth(int num_samples, int num_classes, int token_dim, int seq_len, double noise, uint64_t seed, T* samples,
           int32_t* labels) {
  D2FT_REQUIRE(num_samples >= 1 && num_classes >= 1 && token_dim >= 1 && seq_len >= 1, kInput,
               "dataset spec: degenerate dimensions");
  D2FT_REQUIRE(noise >= 0.0 && std::isfinite(noise), kInput, "dataset spec: noise_level must be nonnegative and finite");
  D2FT_REQUIRE(num_samples % num_classes == 0, kInput, "dataset spec: num_samples must be a multiple of num_classes");
  std::vector<double> means((size_t)num_classes * token_dim);
  auto mg = stream_rng(seed, 0);
  for (double& v : means) v = normal(mg);
  for (int i = 0; i < num_samples; ++i) {
    const int label = i % num_classes;
    auto g = stream_rng(seed, 1 + (uint64_t)i);
    T* x = samples + (size_t)i * seq_len * token_dim;
    for (int t = 0; t < seq_len; ++t)
      for (int j = 0; j < token_dim; ++j)
        x[(size_t)t * token_dim + j] = (T)(means[(size_t)label * token_dim + j] + noise * normal(g));
    labels[i] = label;
  }
}
}  // namespace

extern "C" {

int d2ft_make_synthetic_dataset(int num_samples, int num_classes, int token_dim, int seq_len, double noise,
                                uint64_t seed, float* samples, int32_t* labels) {
  return guarded([&] { synth(num_samples, num_classes, token_dim, seq_len, noise, seed, samples, labels); });
}

int d2ft_make_synthetic_dataset_f64(int num_samples, int num_classes, int token_dim, int seq_len, double noise,
                                    uint64_t seed, double* samples, int32_t* labels) {
  return guarded([&] { synth(num_samples, num_classes, token_dim, seq_len, noise, seed, samples, labels); });
}

}  // extern "C"
