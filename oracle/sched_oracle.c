/* ORACLE / TEST INFRASTRUCTURE ONLY — see sched_oracle.h.
 * Plain C, compiled with -ffp-contract=off (no FMA) so every fp64 add and
 * compare happens exactly as in the reference's C++ loops. */
#include "sched_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { E_OK = 0, E_CONFIG = 1, E_INPUT = 2, E_DIM = 3, E_STATE = 4, E_NUMERIC = 5, E_SIZE = 6 };

/* ------------------------------------------------------------------ rng */
/* rng.hpp:16-21 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* std::mt19937_64 as specified by the C++ standard ([rand.predef]). */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->mti >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:24-26 */
static void make_rng(mt64* g, uint64_t seed, uint64_t stream) {
  mt64_seed(g, or_splitmix64(seed ^ or_splitmix64(stream)));
}
/* rng.hpp:29-31 */
static double uniform_double(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
/* rng.hpp:34-42 */
static uint64_t uniform_below(mt64* g, uint64_t n) {
  const uint64_t limit = ~(uint64_t)0 - (~(uint64_t)0 % n);
  uint64_t x;
  do {
    x = mt64_next(g);
  } while (x >= limit);
  return x % n;
}
/* rng.hpp:45-50 */
static double gaussian(mt64* g) {
  double u1 = uniform_double(g);
  double u2 = uniform_double(g);
  while (u1 <= 0.0) u1 = uniform_double(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

void or_uniform_stream(uint64_t seed, uint64_t stream, int n, double* out) {
  mt64 g;
  make_rng(&g, seed, stream);
  for (int i = 0; i < n; ++i) out[i] = uniform_double(&g);
}
void or_gaussian_stream(uint64_t seed, uint64_t stream, int n, double* out) {
  mt64 g;
  make_rng(&g, seed, stream);
  for (int i = 0; i < n; ++i) out[i] = gaussian(&g);
}
/* rng.hpp:53-59 */
void or_shuffle_iota(uint64_t seed, uint64_t stream, int n, int32_t* out) {
  mt64 g;
  make_rng(&g, seed, stream);
  for (int i = 0; i < n; ++i) out[i] = i;
  for (size_t i = (size_t)n; i > 1; --i) {
    size_t j = (size_t)uniform_below(&g, i);
    int32_t t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

/* ------------------------------------------------------------ scheduler */
/* One row of dp_search, scheduler.cpp:149-186: phase 1 fills the full
 * (n+1) x (cap+1) table with `take > skip` (ties keep skip); phase 2
 * backtracks with `table[i][w] != table[i-1][w]`. */
static double dp_row(const double* s, const int32_t* wt, int n, int cap, uint8_t* sel) {
  size_t W = (size_t)cap + 1;
  double* t = (double*)calloc((size_t)(n + 1) * W, sizeof(double));
  for (int i = 1; i <= n; ++i) {
    const int w_i = wt[i - 1];
    const double val = s[i - 1];
    const double* prev = t + (size_t)(i - 1) * W;
    double* cur = t + (size_t)i * W;
    for (int w = 0; w <= cap; ++w) {
      double skip = prev[w];
      if (w >= w_i) {
        double take = prev[w - w_i] + val;
        cur[w] = take > skip ? take : skip;
      } else {
        cur[w] = skip;
      }
    }
  }
  int w = cap;
  for (int i = 0; i < n; ++i) sel[i] = 0;
  for (int i = n; i > 0; --i) {
    if (t[(size_t)i * W + w] != t[(size_t)(i - 1) * W + w]) {
      sel[i - 1] = 1;
      w -= wt[i - 1];
    }
  }
  double obj = t[(size_t)n * W + cap];
  free(t);
  return obj;
}

/* scheduler.cpp:121-189 (validation order :128-142 preserved) */
int or_dp_search(const double* scores, const int32_t* weights, const int32_t* caps, int K, int N,
                 uint8_t* sel_out, double* obj_out) {
  for (int k = 0; k < K; ++k)
    if (caps[k] < 0) return E_INPUT;
  for (int k = 0; k < K; ++k) {
    for (int i = 0; i < N; ++i)
      if (!isfinite(scores[(size_t)k * N + i])) return E_NUMERIC;
    for (int i = 0; i < N; ++i)
      if (weights[(size_t)k * N + i] < 0) return E_INPUT;
  }
  for (int k = 0; k < K; ++k)
    obj_out[k] = dp_row(scores + (size_t)k * N, weights + (size_t)k * N, N, caps[k], sel_out + (size_t)k * N);
  return E_OK;
}

/* scheduler.cpp:191-220 */
void or_merge_selections(const uint8_t* full_sel, const uint8_t* fwd_sel, int K, int N, uint8_t* codes) {
  for (size_t c = 0; c < (size_t)K * N; ++c) codes[c] = full_sel[c] ? 1 : (fwd_sel[c] ? 2 : 3);
}

/* ScoreTable::validate, scoring.cpp:30-47: forward side first, then backward;
 * per element finite-check then sign-check. */
static int validate_scores(const double* bwd, const double* fwd, int K, int N) {
  const double* sides[2] = {fwd, bwd};
  for (int s = 0; s < 2; ++s)
    for (size_t c = 0; c < (size_t)K * N; ++c) {
      double v = sides[s][c];
      if (!isfinite(v)) return E_NUMERIC;
      if (v < 0.0) return E_NUMERIC;
    }
  return E_OK;
}

/* scheduler.cpp:222-236 */
int or_knapsack_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                         const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes) {
  int e = validate_scores(bwd, fwd, K, N);
  if (e) return e;
  for (int k = 0; k < K; ++k) /* Capacities::validate, scheduler.cpp:37-43 */
    if (cap_full[k] < 0) return E_INPUT;
  for (int k = 0; k < K; ++k)
    if (cap_fwd[k] < 0) return E_INPUT;
  if (K < 1 || N < 1) return E_INPUT; /* build_cost_tables, scheduler.cpp:105-107 */
  for (int k = 0; k < K; ++k)         /* CostModel::validate, scheduler.cpp:24-35 */
    if (cf[k] < 0 || cb[k] < 0) return E_CONFIG;
  size_t KN = (size_t)K * N;
  int32_t* w_full = (int32_t*)malloc(KN * sizeof(int32_t));
  int32_t* w_fwd = (int32_t*)malloc(KN * sizeof(int32_t));
  for (int k = 0; k < K; ++k) /* scheduler.cpp:112-117: constant along the row */
    for (int i = 0; i < N; ++i) {
      w_full[(size_t)k * N + i] = cf[k] + cb[k];
      w_fwd[(size_t)k * N + i] = cf[k];
    }
  uint8_t* sf = (uint8_t*)malloc(KN);
  uint8_t* so = (uint8_t*)malloc(KN);
  double* obj = (double*)malloc((size_t)K * sizeof(double));
  e = or_dp_search(bwd, w_full, cap_full, K, N, sf, obj);
  if (!e) e = or_dp_search(fwd, w_fwd, cap_fwd, K, N, so, obj);
  if (!e) or_merge_selections(sf, so, K, N, codes);
  free(w_full);
  free(w_fwd);
  free(sf);
  free(so);
  free(obj);
  return e;
}

/* scheduler.cpp:321-426 */
int or_scaler_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                       const int32_t* total_cap, int K, int N, int mode, double lambda, uint8_t* codes,
                       double* lambda_used, int* fell_back) {
  int e = validate_scores(bwd, fwd, K, N);
  if (e) return e;
  if (mode == 2 && !(lambda > 0.0)) return E_CONFIG;
  for (int k = 0; k < K; ++k)
    if (cf[k] < 0 || cb[k] < 0) return E_CONFIG;
  for (int k = 0; k < K; ++k)
    if (total_cap[k] < 0) return E_INPUT;
  double max_fwd = 0.0, max_bwd = 0.0, min_pos_fwd = 0.0, min_pos_bwd = 0.0;
  int have_f = 0, have_b = 0;
  for (size_t c = 0; c < (size_t)K * N; ++c) {
    double f = fwd[c], b = bwd[c];
    max_fwd = max_fwd > f ? max_fwd : f; /* std::max(a,b) = (a<b)?b:a */
    max_bwd = max_bwd > b ? max_bwd : b;
    if (f > 0.0 && (!have_f || f < min_pos_fwd)) { min_pos_fwd = f; have_f = 1; }
    if (b > 0.0 && (!have_b || b < min_pos_bwd)) { min_pos_bwd = b; have_b = 1; }
  }
  *fell_back = 0;
  if (mode == 0) {
    if (max_fwd > 0.0 && have_b) *lambda_used = 0.5 * min_pos_bwd / max_fwd;
    else { *lambda_used = 1.0; *fell_back = 1; }
  } else if (mode == 1) {
    if (have_f) *lambda_used = max_bwd > 0.0 ? 2.0 * max_bwd / min_pos_fwd : 1.0;
    else { *lambda_used = 1.0; *fell_back = 1; }
  } else {
    *lambda_used = lambda;
  }
  const double lam = *lambda_used;
  for (int k = 0; k < K; ++k) {
    const int cap = total_cap[k];
    const int w_full = cf[k] + cb[k], w_fwd = cf[k];
    size_t W = (size_t)cap + 1;
    double* val = (double*)calloc((size_t)(N + 1) * W, sizeof(double));
    uint8_t* ch = (uint8_t*)malloc((size_t)(N + 1) * W);
    memset(ch, 3, (size_t)(N + 1) * W);
    for (int i = 1; i <= N; ++i) {
      const double v_fwd = lam * fwd[(size_t)k * N + i - 1];
      const double v_full = bwd[(size_t)k * N + i - 1];
      const double* prev = val + (size_t)(i - 1) * W;
      for (int w = 0; w <= cap; ++w) {
        double best = prev[w];
        uint8_t bc = 3;
        if (w >= w_fwd) {
          double cand = prev[w - w_fwd] + v_fwd;
          if (cand > best) { best = cand; bc = 2; }
        }
        if (w >= w_full) {
          double cand = prev[w - w_full] + v_full;
          if (cand > best) { best = cand; bc = 1; }
        }
        val[(size_t)i * W + w] = best;
        ch[(size_t)i * W + w] = bc;
      }
    }
    int w = cap;
    for (int i = N; i > 0; --i) {
      uint8_t c = ch[(size_t)i * W + w];
      codes[(size_t)k * N + i - 1] = c;
      if (c == 1) w -= w_full;
      else if (c == 2) w -= w_fwd;
    }
    free(val);
    free(ch);
  }
  return E_OK;
}

/* scheduler.cpp:248-302 */
int or_brute_force_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                            const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes) {
  int e = validate_scores(bwd, fwd, K, N);
  if (e) return e;
  for (int k = 0; k < K; ++k)
    if (cap_full[k] < 0 || cap_fwd[k] < 0) return E_INPUT;
  if (N > 14) return E_SIZE;
  int total = 1;
  for (int i = 0; i < N; ++i) total *= 3;
  for (int k = 0; k < K; ++k) {
    const int cap = cap_full[k] + cap_fwd[k];
    const int c_full = cf[k] + cb[k], c_fwd = cf[k];
    double best = -1.0;
    int best_assign = 0;
    for (int assign = 0; assign < total; ++assign) {
      int cost = 0;
      double value = 0.0;
      int rest = assign;
      for (int i = 0; i < N && cost <= cap; ++i) {
        int digit = rest % 3;
        rest /= 3;
        if (digit == 2) {
          cost += c_full;
          value += bwd[(size_t)k * N + i] + fwd[(size_t)k * N + i];
        } else if (digit == 1) {
          cost += c_fwd;
          value += fwd[(size_t)k * N + i];
        }
      }
      if (cost <= cap && value > best) {
        best = value;
        best_assign = assign;
      }
    }
    int rest = best_assign;
    for (int i = 0; i < N; ++i) {
      int digit = rest % 3;
      rest /= 3;
      codes[(size_t)k * N + i] = digit == 2 ? 1 : digit == 1 ? 2 : 3;
    }
  }
  return E_OK;
}

/* scheduler.cpp:442-446 with CostModel::op_cost (scheduler.cpp:15-22) */
int or_row_cost_units(const uint8_t* codes, int N, int cf, int cb) {
  int u = 0;
  for (int i = 0; i < N; ++i) u += codes[i] == 1 ? cf + cb : codes[i] == 2 ? cf : 0;
  return u;
}

/* ------------------------------------------------------------ compaction */
void or_compact(const uint8_t* codes, int K, int N, int H, int32_t* fwd_idx, int32_t* fwd_cnt,
                int32_t* full_idx, int32_t* full_cnt, int32_t* act_heads, int32_t* act_cnt,
                int32_t* full_heads, int32_t* full_hcnt) {
  const int L = K / H;
  for (int k = 0; k < K; ++k) {
    int a = 0, f = 0;
    for (int i = 0; i < N; ++i) {
      uint8_t c = codes[(size_t)k * N + i];
      if (c == 1 || c == 2) fwd_idx[(size_t)k * N + a++] = i;  /* model.cpp:457-458 */
      if (c == 1) full_idx[(size_t)k * N + f++] = i;            /* model.cpp:431-436, 501 */
    }
    fwd_cnt[k] = a;
    full_cnt[k] = f;
  }
  for (int i = 0; i < N; ++i)
    for (int l = 0; l < L; ++l) {
      int a = 0, f = 0;
      size_t cell = (size_t)i * L + l;
      for (int h = 0; h < H; ++h) { /* model.cpp:455-466 head order */
        uint8_t c = codes[(size_t)(l * H + h) * N + i];
        if (c == 1 || c == 2) act_heads[cell * H + a++] = h;
        if (c == 1) full_heads[cell * H + f++] = h;
      }
      act_cnt[cell] = a;
      full_hcnt[cell] = f;
    }
}

/* ---------------------------------------------------------------- model */
int64_t or_param_count(int L, int H, int d, int ffn, int T, int C) {
  int64_t dh = d / H, fs = ffn / H;
  int64_t embed = (int64_t)d * d + d + (int64_t)T * d;
  int64_t block = 3 * (int64_t)d * dh + dh * d + (int64_t)d * fs + fs + fs * d + d / H;
  int64_t head = (int64_t)d * C + C;
  return embed + (int64_t)L * H * block + head;
}

static double* fill_gauss(double* p, int64_t n, mt64* g, double stddev) {
  for (int64_t i = 0; i < n; ++i) p[i] = stddev * gaussian(g); /* model.cpp:91-93 */
  return p + n;
}

/* model.cpp:95-156 in the canonical tensor order of model.hpp:117-153 */
void or_partition_model(int L, int H, int d, int ffn, int T, int C, uint64_t seed, double* out) {
  const int64_t dh = d / H, fs = ffn / H;
  double* p = out;
  mt64 g;
  uint64_t index = 0;
  make_rng(&g, seed, index++);
  p = fill_gauss(p, (int64_t)d * d, &g, 1.0 / sqrt((double)d)); /* w_embed */
  memset(p, 0, sizeof(double) * d);                              /* b_embed */
  p += d;
  p = fill_gauss(p, (int64_t)T * d, &g, 0.02); /* pos */
  for (int l = 1; l <= L; ++l)
    for (int h = 1; h <= H; ++h) {
      make_rng(&g, seed, index++);
      const double isd = 1.0 / sqrt((double)d);
      p = fill_gauss(p, (int64_t)d * dh, &g, isd); /* wq */
      p = fill_gauss(p, (int64_t)d * dh, &g, isd); /* wk */
      p = fill_gauss(p, (int64_t)d * dh, &g, isd); /* wv */
      p = fill_gauss(p, dh * d, &g, isd);          /* wo */
      p = fill_gauss(p, (int64_t)d * fs, &g, isd); /* w1 */
      memset(p, 0, sizeof(double) * fs);           /* b1 */
      p += fs;
      p = fill_gauss(p, fs * d, &g, 1.0 / sqrt((double)ffn)); /* w2 */
      memset(p, 0, sizeof(double) * (d / H));                /* b2 */
      p += d / H;
    }
  make_rng(&g, seed, index++);
  p = fill_gauss(p, (int64_t)d * C, &g, 1.0 / sqrt((double)d)); /* w_cls */
  memset(p, 0, sizeof(double) * C);                             /* b_cls */
}

/* trainer.cpp:61-111 */
int or_make_dataset(int num_samples, int C, int d, int T, double noise, uint64_t seed, double* samples,
                    int32_t* labels) {
  if (num_samples < 1 || C < 1 || d < 1 || T < 1) return E_INPUT;
  if (noise < 0.0 || !isfinite(noise)) return E_INPUT;
  if (num_samples % C != 0) return E_INPUT;
  double* means = (double*)malloc(sizeof(double) * (size_t)C * d);
  mt64 g;
  make_rng(&g, seed, 0);
  for (int c = 0; c < C; ++c)
    for (int j = 0; j < d; ++j) means[(size_t)c * d + j] = gaussian(&g);
  for (int i = 0; i < num_samples; ++i) {
    int label = i % C;
    make_rng(&g, seed, 1 + (uint64_t)i);
    double* x = samples + (size_t)i * T * d;
    for (int t = 0; t < T; ++t)
      for (int j = 0; j < d; ++j) x[(size_t)t * d + j] = means[(size_t)label * d + j] + noise * gaussian(&g);
    labels[i] = label;
  }
  free(means);
  return E_OK;
}
