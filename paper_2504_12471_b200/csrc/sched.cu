// D2FT scheduler and compaction kernels for sm_100a.
//
// Bit-exactness contract (SURVEY.md §7 "Hard parts" 1): the reference's
// dp_search (scheduler.cpp:121-189) fills T[i][w] = max(T[i-1][w],
// T[i-1][w-wt] + s) with a STRICT `take > skip` and backtracks with
// `T[i][w] != T[i-1][w]`.  Two exact rewrites make it GPU-shaped:
//  (1) decision bits: select(i,w) == (take > skip) at (i,w), so the backtrack
//      needs one bit per cell instead of the fp64 table;
//  (2) count compression: build_cost_tables (scheduler.cpp:104-119) gives every
//      item of a row the same weight wt, so T[i][w] == U[i][floor(w/wt)] with
//      the same fp64 operations in the same order; columns beyond i are equal
//      to column i, so only min(cap/wt, N)+1 columns are needed.
// Every fp64 operation is an add (__dadd_rn) or a compare: no contraction.
#include <type_traits>

#include "common.cuh"
#include "sched.cuh"

namespace d2ft_b200 {

namespace {

constexpr int kThreads = 256;  // 8 warps: the maximum warps one row uses
constexpr int kCMax = 8;       // DP values per thread: up to 2048 columns in registers
constexpr size_t kSmemCap = 220 * 1024;

__device__ __forceinline__ void named_sync(int nthreads) {
  if (nthreads == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
  }
}

__host__ __device__ inline void row_geometry(int ncols, int* nw, int* C) {
  int w = (ncols + 127) / 128;
  w = w < 1 ? 1 : (w > 8 ? 8 : w);
  *nw = w;
  *C = (ncols + 32 * w - 1) / (32 * w);
}

__host__ __device__ inline int row_words(int ncols) {
  int nw, C;
  row_geometry(ncols, &nw, &C);
  return nw * C;
}

__device__ inline void set_err(int32_t* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

// Backtrack of one row (scheduler.cpp:176-183): from item N down, the column
// is min(cap/wt - taken so far, i) and the decision bit says take.  Serial by
// nature; the bit read of step i decides the address of step i-1.  Bits in
// shared memory: one thread walks them.  Bits in global memory (large N): the
// walk would pay a dependent L2 round trip per item (~0.4 ms for 2 x 1024
// items), so warp 0 stages the decision words of the next 32 items (whole
// rows, coalesced) into shared memory `stage` and lane 0 walks those.
// bit_of(row_words, col) reads a column's bit in the path's word layout.
template <class BitOf>
__device__ void backtrack_row(const uint32_t* bits, int words, int N, int wt, int cap, uint8_t* sel,
                              uint32_t* stage, BitOf bit_of) {
  // called by one whole warp
  const int lane = threadIdx.x & 31;
  if (!stage) {
    if (lane == 0) {
      long long mm = (wt == 0) ? 0 : (long long)(cap / wt);
      for (int i = N; i > 0; --i) {
        const int col = (wt == 0) ? 0 : (int)(mm < i ? mm : i);
        const unsigned b = bit_of(bits + (size_t)(i - 1) * words, col);
        sel[i - 1] = (uint8_t)b;
        if (b && wt > 0) mm -= 1;
      }
    }
    __syncwarp();
    return;
  }
  long long mm = (wt == 0) ? 0 : (long long)(cap / wt);
  for (int i1 = N; i1 > 0; i1 -= 32) {
    const int i0 = i1 > 32 ? i1 - 32 : 0;
    const int n = (i1 - i0) * words;
    const uint32_t* src = bits + (size_t)i0 * words;
    // L2-direct loads: 1.8x faster than L1-allocating ones for this
    // write-once / read-once stream (sweep r = 0.25: 181 vs 324 us)
    for (int q = lane; q < n; q += 32) stage[q] = __ldcg(src + q);
    __syncwarp();
    if (lane == 0) {
      for (int i = i1; i > i0; --i) {
        const int col = (wt == 0) ? 0 : (int)(mm < i ? mm : i);
        const unsigned b = bit_of(stage + (size_t)(i - 1 - i0) * words, col);
        sel[i - 1] = (uint8_t)b;
        if (b && wt > 0) mm -= 1;
      }
    }
    mm = __shfl_sync(0xffffffffu, mm, 0);
    __syncwarp();
  }
}

struct BitOfWords {  // column c -> word c / 32, bit c % 32 (warp and block paths)
  __device__ unsigned operator()(const uint32_t* row, int col) const { return (row[col >> 5] >> (col & 31)) & 1u; }
};

// One warp (the training shapes: ViT-B 25 p_f of 64 -> 26 columns, ViT-L 102
// of 256 -> 103): lane holds columns m = 32 j + lane, j < CW.  Column m-1
// comes from the lane below (shuffle up) or, for lane 0, from lane 31 of the
// previous 32-column group — registers only, no shared-memory exchange or
// barrier per item.  Same fp64 adds in the same order and the same
// decision-bit words (word j = columns 32 j .. 32 j + 31) as the block path.
// All threads of the block call it (block-uniform arguments).
// Run by warp `wsel` alone (no block barrier): DP, objective, backtrack.
template <int CW>
__device__ void dp_row_warp(const double* s_scores, int N, int wt, int cap, int Mp, uint32_t* bits, uint8_t* sel,
                            double* s_obj, uint32_t* stage, int wsel) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == wsel) {
    double v[CW];
    bool okc[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int m = 32 * j + lane;
      v[j] = 0.0;
      okc[j] = (wt == 0) ? (m == 0) : (m >= 1 && m <= Mp);
    }
    for (int i = 0; i < N; ++i) {
      const double s = s_scores[i];
      double prev[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const double up = __shfl_up_sync(0xffffffffu, v[j], 1);
        double wrap = 0.0;
        if (j > 0) wrap = __shfl_sync(0xffffffffu, v[j - 1], 31);
        prev[j] = lane > 0 ? up : wrap;
        if (wt == 0) prev[j] = v[j];  // zero weight: take reads the same column
      }
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const double take = __dadd_rn(prev[j], s);
        const bool d = okc[j] && (take > v[j]);  // scheduler.cpp:167 strict >
        if (d) v[j] = take;
        const unsigned ball = __ballot_sync(0xffffffffu, d);
        if (lane == 0) bits[(size_t)i * CW + j] = ball;
      }
    }
#pragma unroll
    for (int j = 0; j < CW; ++j)
      if (32 * j + lane == Mp) *s_obj = v[j];
    __threadfence_block();  // every lane's decision words (shared or global) before lane 0 reads them
    __syncwarp();
    backtrack_row(bits, CW, N, wt, cap, sel, stage, BitOfWords{});
  }
}

// Block path (more than 256 columns, up to 8 warps): columns m = j * nthr +
// warp * 32 + lane; the boundary column of each warp crosses through a
// double-buffered shared exchange and one named barrier per item.
template <int CC>
__device__ void dp_row_block(const double* s_scores, int N, int wt, int cap, int Mp, int nw, uint32_t* bits,
                             double* xch, uint8_t* sel, double* s_obj, uint32_t* stage) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = nw * 32;
  const int words = nw * CC;
  const bool active = tid < nthr;
  double v[kCMax];
#pragma unroll
  for (int j = 0; j < kCMax; ++j) v[j] = 0.0;
  if (active && lane == 31) {
#pragma unroll
    for (int j = 0; j < kCMax; ++j) xch[warp * kCMax + j] = 0.0;  // parity 0
  }
  __syncthreads();
  int p = 0;
  if (active) {
    for (int i = 0; i < N; ++i) {
      const double s = s_scores[i];
      const double* xin = xch + p * (8 * kCMax);
      double* xout = xch + (p ^ 1) * (8 * kCMax);
#pragma unroll
      for (int j = 0; j < CC; ++j) {
        {
          const int m = j * nthr + warp * 32 + lane;
          double prev = __shfl_up_sync(0xffffffffu, v[j], 1);
          if (lane == 0) {
            if (warp > 0) prev = xin[(warp - 1) * kCMax + j];
            else prev = (j > 0) ? xin[(nw - 1) * kCMax + (j - 1)] : 0.0;
          }
          bool ok;
          if (wt == 0) {  // zero weight: take reads the same column
            prev = v[j];
            ok = (m == 0);
          } else {
            ok = (m >= 1) && (m <= Mp);
          }
          const double take = __dadd_rn(prev, s);
          const bool d = ok && (take > v[j]);  // scheduler.cpp:167 strict >
          if (d) v[j] = take;
          const unsigned ball = __ballot_sync(0xffffffffu, d);
          if (lane == 0) bits[(size_t)i * words + j * nw + warp] = ball;
          if (lane == 31) xout[warp * kCMax + j] = v[j];
        }
      }
      p ^= 1;
      named_sync(nthr);
    }
    // objective = U[N][Mp]
#pragma unroll
    for (int j = 0; j < CC; ++j) {
      if (j * nthr + warp * 32 + lane == Mp) *s_obj = v[j];
    }
  }
  __syncthreads();
  if (warp == 0) backtrack_row(bits, words, N, wt, cap, sel, stage, BitOfWords{});
  __syncthreads();
}

// Single warp, contiguous columns per lane (rows of up to 32 * 40 columns:
// the training shapes and the 1024-item sweep): lane l holds columns
// m = l * CL + j.  Column m-1 is the lane's own previous register except for
// j = 0 (one shuffle per item), so an item costs one shuffle plus CL
// independent add / compare / select — no shared-memory exchange, no barrier.
// The same fp64 adds in the same order as the reference; decision bits are a
// CL-bit mask per (item, lane): one 32-bit word (CL <= 32: rows of up to
// 1024 columns, 128 B per item, so the 1024-item sweep keeps its bits in
// shared memory) or a word pair (CL > 32), at (32 i + l).
constexpr int kLaneColsMax = 40;
template <int CL>
struct BitOfLane {  // column c -> lane c / CL, bit c % CL
  __device__ unsigned operator()(const uint32_t* row, int col) const {
    if constexpr (CL <= 32) return (row[col / CL] >> (col % CL)) & 1u;
    else return (unsigned)((reinterpret_cast<const uint64_t*>(row)[col / CL] >> (col % CL)) & 1u);
  }
};
template <int CL>
__device__ void dp_row_lane(const double* s_scores, int N, int wt, int cap, int Mp, uint32_t* bits, uint8_t* sel,
                            double* s_obj, uint32_t* stage, int wsel) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWords = CL <= 32 ? 32 : 64;  // decision words per item
  if (warp == wsel) {
    double v[CL];
    bool okc[CL];
#pragma unroll
    for (int j = 0; j < CL; ++j) {
      const int m = lane * CL + j;
      v[j] = 0.0;
      okc[j] = (wt == 0) ? (m == 0) : (m >= 1 && m <= Mp);
    }
    for (int i = 0; i < N; ++i) {
      const double s = s_scores[i];
      double left = __shfl_up_sync(0xffffffffu, v[CL - 1], 1);  // column l*CL - 1, before this item
      if (lane == 0) left = 0.0;
      // decision bits into 4 independent accumulators (short OR chains)
      using MaskT = std::conditional_t<(CL <= 32), uint32_t, uint64_t>;  // one decision bit per column
      MaskT acc4[4] = {0, 0, 0, 0};
      if (wt == 0) {  // zero weight: take reads the same column (only m == 0 may take)
#pragma unroll
        for (int j = 0; j < CL; ++j) {
          const double take = __dadd_rn(v[j], s);
          const bool d = okc[j] && (take > v[j]);
          if (d) v[j] = take;
          acc4[j & 3] |= (MaskT)d << j;
        }
      } else {
        // all takes from the previous item's values first, then the compares,
        // then the updates: CL independent chains the scheduler can interleave
        // (the fused per-column form issued DADD -> DSETP -> FSEL serially,
        // ~25 cycles a column).  Columns past Mp may update freely (nothing at
        // or below Mp reads them, the backtrack never visits them); column 0
        // (lane 0) never takes: its left neighbour is -inf.
        double t[CL];
        t[0] = __dadd_rn(lane == 0 ? -INFINITY : left, s);
#pragma unroll
        for (int j = 1; j < CL; ++j) t[j] = __dadd_rn(v[j - 1], s);
        bool d[CL];
#pragma unroll
        for (int j = 0; j < CL; ++j) d[j] = t[j] > v[j];  // scheduler.cpp:167 strict >
#pragma unroll
        for (int j = 0; j < CL; ++j) {
          acc4[j & 3] |= (MaskT)d[j] << j;
          v[j] = d[j] ? t[j] : v[j];
        }
      }
      const MaskT m = (acc4[0] | acc4[1]) | (acc4[2] | acc4[3]);
      if constexpr (CL <= 32) bits[(size_t)i * 32 + lane] = (uint32_t)m;
      else reinterpret_cast<uint64_t*>(bits)[(size_t)i * 32 + lane] = m;
    }
#pragma unroll
    for (int j = 0; j < CL; ++j)
      if (lane * CL + j == Mp) *s_obj = v[j];
    __threadfence_block();  // every lane's decision words (shared or global) before lane 0 reads them
    __syncwarp();
    backtrack_row(bits, kWords, N, wt, cap, sel, stage, BitOfLane<CL>{});
  }
}

// Rows of up to 32 * kLaneColsMax count-compressed columns run on one warp
// (`wsel`; the other warps of the block are free for the other pool).
__device__ void dp_row_small(const double* s_scores, int N, int wt, int cap, uint32_t* bits, uint8_t* sel,
                             double* s_obj, uint32_t* stage, int wsel) {
  const int Mp = (wt == 0) ? 0 : min(cap / wt, N);  // last stored column
  const int ncols = Mp + 1;
  if (ncols <= 32) return dp_row_warp<1>(s_scores, N, wt, cap, Mp, bits, sel, s_obj, stage, wsel);
  const int c = (ncols + 31) / 32;  // columns per lane, rounded up to an instantiated width
#define D2FT_LANE(W) \
  if (c <= W) return dp_row_lane<W>(s_scores, N, wt, cap, Mp, bits, sel, s_obj, stage, wsel);
  D2FT_LANE(2) D2FT_LANE(4) D2FT_LANE(6) D2FT_LANE(8) D2FT_LANE(10) D2FT_LANE(12) D2FT_LANE(14) D2FT_LANE(16)
  D2FT_LANE(18) D2FT_LANE(20) D2FT_LANE(24) D2FT_LANE(26) D2FT_LANE(28) D2FT_LANE(32)  // 32-bit masks
  D2FT_LANE(33) D2FT_LANE(36)
#undef D2FT_LANE
  return dp_row_lane<kLaneColsMax>(s_scores, N, wt, cap, Mp, bits, sel, s_obj, stage, wsel);
}

// Count-compressed 0/1 knapsack of one row (all threads of the block call it
// with block-uniform arguments).  s_scores: the row's N scores in shared
// memory.  Writes sel[i] in {0,1} (shared or global) and the objective
// T[N][cap] to *s_obj, both visible to the block on return.
__device__ void dp_row_const(const double* s_scores, int N, int wt, int cap, uint32_t* bits, double* xch,
                             uint8_t* sel, double* s_obj, uint32_t* stage) {
  const int Mp = (wt == 0) ? 0 : min(cap / wt, N);  // last stored column
  const int ncols = Mp + 1;
  if (ncols <= 32 * kLaneColsMax) {
    dp_row_small(s_scores, N, wt, cap, bits, sel, s_obj, stage, 0);
    __syncthreads();
    return;
  }
  int nw, C;
  row_geometry(ncols, &nw, &C);
  switch (C) {  // compile-time columns per thread
    case 1: return dp_row_block<1>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    case 2: return dp_row_block<2>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    case 3: return dp_row_block<3>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    case 4: return dp_row_block<4>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    case 5: return dp_row_block<5>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    case 6: return dp_row_block<6>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    case 7: return dp_row_block<7>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
    default: return dp_row_block<8>(s_scores, N, wt, cap, Mp, nw, bits, xch, sel, s_obj, stage);
  }
}

struct KnapsackArgs {
  const double* bwd;
  const double* fwd;
  const int32_t* cf;
  const int32_t* cb;
  const int32_t* cap_full;
  const int32_t* cap_fwd;
  int K, N, H;
  uint8_t* codes;
  CompactLists lists;
  bool have_lists;
  SchedWorkspace ws;
  bool bits_in_smem;
  int words_max;
  int max_cols;  // DP columns per row the launch is sized for
  bool validate;
  int lists_smem_bytes;  // dynamic shared memory of the launch (staging of the table for the column lists)
  bool cols_in_kernel;   // the last CTA builds the column lists (table staged in its shared memory)
  bool two_pools;        // every row fits one warp: the two pools run concurrently (2 warps)
};

// Warp 0 writes the ascending index lists of one row (codes in smem).
__device__ void row_lists(const uint8_t* s_codes, int N, int32_t* fwd_idx, int32_t* fwd_cnt, int32_t* full_idx,
                          int32_t* full_cnt) {
  const int lane = threadIdx.x & 31;
  int a = 0, f = 0;
  for (int base = 0; base < N; base += 32) {
    const int i = base + lane;
    const uint8_t c = i < N ? s_codes[i] : 3;
    const unsigned ma = __ballot_sync(0xffffffffu, c == 1 || c == 2);
    const unsigned mf = __ballot_sync(0xffffffffu, c == 1);
    const unsigned lt = (1u << lane) - 1u;
    if (c == 1 || c == 2) fwd_idx[a + __popc(ma & lt)] = i;
    if (c == 1) full_idx[f + __popc(mf & lt)] = i;
    a += __popc(ma);
    f += __popc(mf);
  }
  if (lane == 0) {
    *fwd_cnt = a;
    *full_cnt = f;
  }
}

// Per-(micro-batch, block) head lists; thread per cell, heads ascending.
// kHoist (the global-memory table of compact_cols_kernel): every head's code
// is loaded before the list stores, which may alias `codes` as far as the
// compiler knows (byte pointer) and otherwise serialise one L2 round trip
// per head.  The knapsack kernel's shared-memory table keeps the plain loop
// (the hoisted form measured slower there: 35 vs 25 us at ViT-B).
template <bool kHoist>
__device__ void column_lists(const uint8_t* codes, int K, int N, int H, const CompactLists& L, int tid0,
                             int stride) {
  const int nb = K / H;
  // consecutive threads take consecutive micro-batches of one block, so each
  // head's code loads of a warp are one contiguous 32-byte segment
  for (int q = tid0; q < N * nb; q += stride) {
    const int l = q / N, i = q % N;
    const int cell = i * nb + l;
    int a = 0, f = 0;
    if (kHoist && H <= 16) {
      uint8_t cc[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) cc[h] = h < H ? __ldg(codes + (size_t)(l * H + h) * N + i) : 0;
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        if (cc[h] == 1 || cc[h] == 2) L.act_heads[(size_t)cell * H + a++] = h;
        if (cc[h] == 1) L.full_heads[(size_t)cell * H + f++] = h;
      }
    } else {
      for (int h = 0; h < H; ++h) {
        const uint8_t c = codes[(size_t)(l * H + h) * N + i];
        if (c == 1 || c == 2) L.act_heads[(size_t)cell * H + a++] = h;
        if (c == 1) L.full_heads[(size_t)cell * H + f++] = h;
      }
    }
    L.act_cnt[cell] = a;
    L.full_hcnt[cell] = f;
  }
}

__global__ void __launch_bounds__(kThreads) knapsack_kernel(KnapsackArgs A) {
  D2FT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem[];
  const int k = blockIdx.x;
  const int N = A.N;
  // layout (sched_smem_layout): scores of the two pools, the block path's
  // exchange, objectives, codes, the two pools' selections, then the two
  // pools' decision bits (shared) or backtrack staging (bits in global)
  const int Np = (N + 15) & ~15;
  double* s_scores = reinterpret_cast<double*>(smem);
  double* s_scores2 = s_scores + N;              // Forward pool (two-pool launches)
  double* xch = s_scores2 + N;                   // 2 x 8 x kCMax
  double* s_obj = xch + 2 * 8 * kCMax;           // [2] (+pad)
  uint8_t* s_codes = reinterpret_cast<uint8_t*>(s_obj + 4);
  uint8_t* s_sel = s_codes + Np;
  uint8_t* s_sel2 = s_sel + Np;
  uint32_t* bits_base = reinterpret_cast<uint32_t*>(s_sel2 + Np);
  const size_t pool_words = A.bits_in_smem ? (size_t)N * A.words_max : (size_t)32 * A.words_max;
  uint32_t* bits = A.bits_in_smem ? bits_base : A.ws.bits_global + (size_t)2 * k * N * A.words_max;
  uint32_t* bits2 = A.bits_in_smem ? bits_base + pool_words : bits + (size_t)N * A.words_max;
  // global bits: the backtrack's staging words sit where the bits would
  uint32_t* stage = A.bits_in_smem ? nullptr : bits_base;
  uint32_t* stage2 = A.bits_in_smem ? nullptr : bits_base + pool_words;
  // validation outcome: one bit per category, resolved after the barrier in
  // the reference's order (ScoreTable::validate -> numeric, Capacities ->
  // input, CostModel -> config; scheduler.cpp:24-43, scoring.cpp:30-47), then
  // this launch's own column limit (size)
  __shared__ int s_flags, s_bad;
  if (threadIdx.x == 0) s_flags = 0;
  __syncthreads();

  const int cfk = A.cf[k], cbk = A.cb[k];
  if (A.validate) {
    bool bad = false;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double b = A.bwd[(size_t)k * N + i], f = A.fwd[(size_t)k * N + i];
      bad |= !isfinite(b) || !isfinite(f) || b < 0.0 || f < 0.0;  // scoring.cpp:38-41
    }
    if (bad) atomicOr(&s_flags, 1);
    if (threadIdx.x == 0 && (A.cap_full[k] < 0 || A.cap_fwd[k] < 0)) atomicOr(&s_flags, 2);
    if (threadIdx.x == 0 && (cfk < 0 || cbk < 0)) atomicOr(&s_flags, 4);
  }
  if (threadIdx.x == 0) {
    // device-resident capacities are not seen by the host: a row whose
    // count-compressed DP needs more columns than this launch was sized for
    // (thread count, decision-bit words) is refused instead of run
    auto cols = [N](int wt, int cap) { return wt <= 0 ? 1 : min(max(cap, 0) / wt, N) + 1; };
    if (cols(cfk + cbk, A.cap_full[k]) > A.max_cols || cols(cfk, A.cap_fwd[k]) > A.max_cols) atomicOr(&s_flags, 8);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int f = s_flags;
    s_bad = (f & 1) ? kNumeric : (f & 2) ? kInput : (f & 4) ? kConfig : (f & 8) ? kSize : 0;
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) set_err(A.ws.err_flag, s_bad);
    for (int i = threadIdx.x; i < N; i += blockDim.x) A.codes[(size_t)k * N + i] = 3;
    // fall through to the compaction epilogue with an all-shortcut row
  }
  if (!s_bad && A.two_pools) {
    // the two pools are independent DPs (scheduler.cpp:233-234): warp 0
    // runs the Full pool on the backward scores (weight cf+cb), warp 1 the
    // Forward pool on the forward scores (weight cf), concurrently
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      s_scores[i] = A.bwd[(size_t)k * N + i];
      s_scores2[i] = A.fwd[(size_t)k * N + i];
    }
    __syncthreads();
    dp_row_small(s_scores, N, cfk + cbk, A.cap_full[k], bits, s_sel, s_obj, stage, 0);
    dp_row_small(s_scores2, N, cfk, A.cap_fwd[k], bits2, s_sel2, s_obj + 1, stage2, 1);
    __syncthreads();
    // merge (scheduler.cpp:205-216): full wins, then forward, else shortcut
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const uint8_t c = s_sel[i] ? 1 : (s_sel2[i] ? 2 : 3);
      s_codes[i] = c;
      A.codes[(size_t)k * N + i] = c;
    }
  } else if (!s_bad) {
    // pass 1: Full pool on backward scores, weight cf+cb (scheduler.cpp:233)
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_scores[i] = A.bwd[(size_t)k * N + i];
    __syncthreads();
    dp_row_const(s_scores, N, cfk + cbk, A.cap_full[k], bits, xch, s_sel, s_obj, stage);
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_codes[i] = s_sel[i] ? 1 : 3;
    // pass 2: Forward pool on forward scores, weight cf (scheduler.cpp:234)
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_scores[i] = A.fwd[(size_t)k * N + i];
    __syncthreads();
    dp_row_const(s_scores, N, cfk, A.cap_fwd[k], bits, xch, s_sel, s_obj, stage);
    // merge (scheduler.cpp:205-216): full wins, then forward, else shortcut
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const uint8_t c = s_codes[i] == 1 ? 1 : (s_sel[i] ? 2 : 3);
      s_codes[i] = c;
      A.codes[(size_t)k * N + i] = c;
    }
  } else {
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_codes[i] = 3;
  }
  __syncthreads();
  if (!A.have_lists) return;
  if (threadIdx.x < 32)
    row_lists(s_codes, N, A.lists.fwd_idx + (size_t)k * N, A.lists.fwd_cnt + k, A.lists.full_idx + (size_t)k * N,
              A.lists.full_cnt + k);
  if (!A.cols_in_kernel) return;  // large tables: compact_cols_kernel after this launch
  // last CTA to finish builds the per-(micro-batch, block) head lists
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(A.ws.done_counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    // the whole K x N table into this CTA's (now free) shared memory with
    // coalesced 16-byte loads when it fits, then every cell scans it there:
    // the per-cell head loops were 12 strided global loads each
    const size_t kn = (size_t)A.K * N;
    if (kn <= (size_t)A.lists_smem_bytes && (kn & 15) == 0) {
      uint8_t* tab = reinterpret_cast<uint8_t*>(smem);
      for (size_t q = threadIdx.x; q < kn / 16; q += blockDim.x)
        reinterpret_cast<uint4*>(tab)[q] = __ldcg(reinterpret_cast<const uint4*>(A.codes) + q);
      __syncthreads();
      column_lists<false>(tab, A.K, N, A.H, A.lists, threadIdx.x, blockDim.x);
    } else {
      column_lists<false>(A.codes, A.K, N, A.H, A.lists, threadIdx.x, blockDim.x);
    }
    if (threadIdx.x == 0) *A.ws.done_counter = 0u;  // re-arm for the next launch
  }
}

struct DpConstArgs {
  const double* scores;
  const int32_t* row_wt;
  const int32_t* caps;
  const int32_t* rows;
  int N;
  uint8_t* sel;
  double* obj;
  SchedWorkspace ws;
  bool bits_in_smem;
  int words_max;
};

__global__ void __launch_bounds__(kThreads) dp_const_kernel(DpConstArgs A) {
  D2FT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem[];
  const int k = A.rows[blockIdx.x];
  const int N = A.N;
  // single-pool layout of sched_smem_layout(pools = 1)
  const int Np = (N + 15) & ~15;
  double* s_scores = reinterpret_cast<double*>(smem);
  double* xch = s_scores + N;
  double* s_obj = xch + 2 * 8 * kCMax;
  uint8_t* s_codes = reinterpret_cast<uint8_t*>(s_obj + 4);
  uint8_t* s_sel = s_codes + Np;
  uint32_t* bits = A.bits_in_smem ? reinterpret_cast<uint32_t*>(s_sel + Np)
                                  : A.ws.bits_global + (size_t)blockIdx.x * N * A.words_max;
  uint32_t* stage = A.bits_in_smem ? nullptr : reinterpret_cast<uint32_t*>(s_sel + Np);
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_scores[i] = A.scores[(size_t)k * N + i];
  __syncthreads();
  dp_row_const(s_scores, N, A.row_wt[k], A.caps[k], bits, xch, s_sel, s_obj, stage);
  const double obj = *s_obj;
  for (int i = threadIdx.x; i < N; i += blockDim.x) A.sel[(size_t)k * N + i] = s_sel[i];
  if (threadIdx.x == 0) A.obj[k] = obj;
}

// General-weight row (dp_search with non-constant weights): values over
// w in [0, cap] double-buffered in global/shared memory, one bit per cell.
__global__ void __launch_bounds__(kThreads) dp_general_kernel(const double* scores, const int32_t* weights,
                                                               const int32_t* caps, const int32_t* rows, int N,
                                                               int max_cap, uint8_t* sel, double* obj,
                                                               uint32_t* bits_global, double* vals_global) {
  D2FT_PDL_ENTRY();
  const int k = rows[blockIdx.x];
  const int cap = caps[k];
  const int W = cap + 1;
  const int wordsW = (max_cap + 1 + 31) / 32;
  uint32_t* bits = bits_global + (size_t)blockIdx.x * N * wordsW;
  double* va = vals_global + (size_t)blockIdx.x * 2 * (max_cap + 1);
  double* vb = va + (max_cap + 1);
  const double* s = scores + (size_t)k * N;
  const int32_t* wt = weights + (size_t)k * N;
  for (int w = threadIdx.x; w < W; w += blockDim.x) va[w] = 0.0;
  __syncthreads();
  for (int i = 0; i < N; ++i) {
    const int wi = wt[i];
    const double si = s[i];
    for (int base = 0; base < W; base += blockDim.x) {
      const int w = base + threadIdx.x;
      bool d = false;
      if (w < W) {
        const double skip = va[w];
        double nv = skip;
        if (w >= wi) {
          const double take = __dadd_rn(va[w - wi], si);
          d = take > skip;
          if (d) nv = take;
        }
        vb[w] = nv;
      }
      const unsigned ball = __ballot_sync(0xffffffffu, d);
      if ((threadIdx.x & 31) == 0 && w < W) bits[(size_t)i * wordsW + (w >> 5)] = ball;
    }
    __syncthreads();
    double* t = va;
    va = vb;
    vb = t;
  }
  if (threadIdx.x == 0) {
    obj[k] = va[cap];
    int w = cap;
    for (int i = N; i > 0; --i) {
      const unsigned b = (__ldcg(bits + (size_t)(i - 1) * wordsW + (w >> 5)) >> (w & 31)) & 1u;
      sel[(size_t)k * N + i - 1] = (uint8_t)b;
      if (b) w -= wt[i - 1];
    }
  }
}

__global__ void merge_kernel(const uint8_t* a, const uint8_t* b, size_t n, uint8_t* codes) {
  D2FT_PDL_ENTRY();
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < n; c += (size_t)gridDim.x * blockDim.x)
    codes[c] = a[c] ? 1 : (b[c] ? 2 : 3);
}

__global__ void compact_rows_kernel(const uint8_t* codes, int N, CompactLists L) {
  D2FT_PDL_ENTRY();
  extern __shared__ uint8_t s_codes[];
  const int k = blockIdx.x;
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_codes[i] = codes[(size_t)k * N + i];
  __syncthreads();
  if (threadIdx.x < 32)
    row_lists(s_codes, N, L.fwd_idx + (size_t)k * N, L.fwd_cnt + k, L.full_idx + (size_t)k * N, L.full_cnt + k);
}

__global__ void compact_cols_kernel(const uint8_t* codes, int K, int N, int H, CompactLists L) {
  D2FT_PDL_ENTRY();
  column_lists<true>(codes, K, N, H, L, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// scaler_schedule row DP (scheduler.cpp:379-424).  Choices p_s, then p_o
// (value lambda*f via __dmul_rn, weight cf), then p_f (value b, weight cf+cb),
// each replacing the incumbent only on strict improvement.
__global__ void __launch_bounds__(kThreads) scaler_kernel(const double* bwd, const double* fwd, const int32_t* cf,
                                                          const int32_t* cb, const int32_t* total_cap, int N,
                                                          const double* lambda_dev, int max_cap, uint8_t* codes,
                                                          uint8_t* choice_global, double* vals_global) {
  D2FT_PDL_ENTRY();
  const int k = blockIdx.x;
  const int cap = total_cap[k];
  const int W = cap + 1;
  const int w_fwd = cf[k], w_full = cf[k] + cb[k];
  const double lam = *lambda_dev;
  uint8_t* ch = choice_global + (size_t)k * N * (max_cap + 1);
  double* va = vals_global + (size_t)k * 2 * (max_cap + 1);
  double* vb = va + (max_cap + 1);
  for (int w = threadIdx.x; w < W; w += blockDim.x) va[w] = 0.0;
  __syncthreads();
  for (int i = 0; i < N; ++i) {
    const double v_fwd = __dmul_rn(lam, fwd[(size_t)k * N + i]);
    const double v_full = bwd[(size_t)k * N + i];
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
      double best = va[w];
      uint8_t c = 3;
      if (w >= w_fwd) {
        const double cand = __dadd_rn(va[w - w_fwd], v_fwd);
        if (cand > best) {
          best = cand;
          c = 2;
        }
      }
      if (w >= w_full) {
        const double cand = __dadd_rn(va[w - w_full], v_full);
        if (cand > best) {
          best = cand;
          c = 1;
        }
      }
      vb[w] = best;
      ch[(size_t)i * (max_cap + 1) + w] = c;
    }
    __syncthreads();
    double* t = va;
    va = vb;
    vb = t;
  }
  if (threadIdx.x == 0) {
    int w = cap;
    for (int i = N; i > 0; --i) {
      const uint8_t c = __ldcg(ch + (size_t)(i - 1) * (max_cap + 1) + w);
      codes[(size_t)k * N + i - 1] = c;
      if (c == 1) w -= w_full;
      else if (c == 2) w -= w_fwd;
    }
  }
}

// brute_force_schedule (scheduler.cpp:248-302): one CTA per row enumerates
// all 3^N assignments (digit 0 = p_s, 1 = p_o, 2 = p_f; value summed in item
// order with the reference's early exit on cost > cap), keeping the maximum
// value and, among equal values, the smallest assignment index — exactly the
// reference's sequential "first found strict maximum".
__global__ void __launch_bounds__(kThreads) brute_kernel(const double* bwd, const double* fwd, const int32_t* cf,
                                                         const int32_t* cb, const int32_t* cap_full,
                                                         const int32_t* cap_fwd, int N, int total, uint8_t* codes) {
  D2FT_PDL_ENTRY();
  const int k = blockIdx.x;
  const int cap = cap_full[k] + cap_fwd[k];
  const int c_full = cf[k] + cb[k], c_fwd = cf[k];
  const double* b = bwd + (size_t)k * N;
  const double* f = fwd + (size_t)k * N;
  double best = -1.0;
  int best_a = 0x7fffffff;
  for (int a = threadIdx.x; a < total; a += blockDim.x) {
    int cost = 0, rest = a;
    double value = 0.0;
    for (int i = 0; i < N && cost <= cap; ++i) {
      const int digit = rest % 3;
      rest /= 3;
      if (digit == 2) {
        cost += c_full;
        value = __dadd_rn(value, __dadd_rn(b[i], f[i]));
      } else if (digit == 1) {
        cost += c_fwd;
        value = __dadd_rn(value, f[i]);
      }
    }
    if (cost <= cap && (value > best || (value == best && a < best_a))) {
      best = value;
      best_a = a;
    }
  }
  __shared__ double sv[kThreads];
  __shared__ int sa[kThreads];
  sv[threadIdx.x] = best;
  sa[threadIdx.x] = best_a;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int a2 = sa[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && a2 < sa[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        sa[threadIdx.x] = a2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int rest = sa[0] == 0x7fffffff ? 0 : sa[0];
    for (int i = 0; i < N; ++i) {
      const int digit = rest % 3;
      rest /= 3;
      codes[(size_t)k * N + i] = digit == 2 ? 1 : digit == 1 ? 2 : 3;
    }
  }
}

}  // namespace

void launch_brute_force(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                        const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, uint8_t* codes,
                        cudaStream_t s) {
  int total = 1;
  for (int i = 0; i < N; ++i) total *= 3;
  brute_kernel<<<K, kThreads, 0, s>>>(bwd, fwd, cf, cb, cap_full, cap_fwd, N, total, codes);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

// decision-bit words per item: the block path's row words, or a 64-bit mask
// per lane for the single-warp lane path
int bits_words_per_item(int max_cols) {
  const int w = (max_cols + 31) / 32 + 8;
  if (max_cols <= 32 * 32) return w > 32 ? w : 32;            // lane path, 32-bit masks
  if (max_cols <= 32 * kLaneColsMax) return w > 64 ? w : 64;  // lane path, 64-bit masks
  return w;
}
// pools = 2: the knapsack launch whose rows all fit one warp (both pools
// concurrently, each with its own scores / selection / bits); 1: one pool at
// a time (dp_search rows, and knapsack rows on the 8-warp block path).
int knapsack_pools(int max_cols) { return max_cols <= 32 * kLaneColsMax ? 2 : 1; }
size_t sched_smem_layout(int N, int max_cols, int pools, bool* bits_in_smem) {
  const int words = bits_words_per_item(max_cols);
  const size_t Np = (size_t)((N + 15) & ~15);
  // scores of both pools always reserved (the kernel's layout is fixed)
  const size_t base = (size_t)2 * N * 8 + 2 * 8 * kCMax * 8 + 32 + 3 * Np;
  const size_t with_bits = base + (size_t)pools * N * words * 4;
  if (with_bits <= kSmemCap) {
    *bits_in_smem = true;
    return with_bits;
  }
  *bits_in_smem = false;
  return base + (size_t)pools * 32 * words * 4;  // the backtrack's staging of 32 items per pool
}
size_t knapsack_smem_bytes(int N, int max_cols, bool* bits_in_smem) {
  return sched_smem_layout(N, max_cols, knapsack_pools(max_cols), bits_in_smem);
}

size_t knapsack_global_bits_words(int K, int N, int max_cols) {
  const int words = bits_words_per_item(max_cols);
  return (size_t)2 * K * N * words;  // both pools of every row
}

void launch_knapsack_schedule(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                              const int32_t* cap_full, const int32_t* cap_fwd, int K, int N, int H, int max_cols,
                              uint8_t* codes, const CompactLists* lists, const SchedWorkspace& ws, bool validate,
                              cudaStream_t stream) {
  D2FT_REQUIRE(max_cols <= kThreads * kCMax, kSize, "knapsack: more than 2048 DP columns per row");
  KnapsackArgs A{};
  A.bwd = bwd;
  A.fwd = fwd;
  A.cf = cf;
  A.cb = cb;
  A.cap_full = cap_full;
  A.cap_fwd = cap_fwd;
  A.K = K;
  A.N = N;
  A.H = H;
  A.codes = codes;
  A.have_lists = lists != nullptr;
  if (lists) A.lists = *lists;
  A.ws = ws;
  A.validate = validate;
  A.words_max = bits_words_per_item(max_cols);
  A.max_cols = max_cols;
  A.two_pools = knapsack_pools(max_cols) == 2;
  size_t smem = knapsack_smem_bytes(N, max_cols, &A.bits_in_smem);
  // room to stage the K x N table for the last CTA's column lists (<= 48 KB)
  const size_t kn = (size_t)K * N;
  if (lists && kn <= 48 * 1024 && kn > smem) smem = (kn + 15) & ~size_t(15);
  A.lists_smem_bytes = (int)smem;
  A.cols_in_kernel = kn <= smem && (kn & 15) == 0;
  if (!A.bits_in_smem)
    D2FT_REQUIRE(ws.bits_global && ws.bits_global_words >= knapsack_global_bits_words(K, N, max_cols), kState,
                 "knapsack: global decision-bit workspace too small");
  static unsigned long long attr_done = 0;
  once_per_device(attr_done, [&] {
    D2FT_CUDA(cudaFuncSetAttribute(knapsack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap));
    D2FT_CUDA(cudaFuncSetAttribute(dp_const_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap));
  });
  // rows that fit the single-warp DP need one warp (more CTAs per SM, the
  // DP's registers only for 32 threads); wider rows use the 8-warp block path
  const int threads = A.two_pools ? 64 : kThreads;
  knapsack_kernel<<<K, threads, smem, stream>>>(A);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
  if (lists && !A.cols_in_kernel) {  // column lists over many CTAs (one thread per cell)
    const int cells = N * (K / H);
    compact_cols_kernel<<<(cells + 127) / 128, 128, 0, stream>>>(codes, K, N, H, *lists);
    count_launch();
    D2FT_CUDA(cudaGetLastError());
  }
}

void launch_dp_const(const double* scores, const int32_t* row_wt, const int32_t* caps, const int32_t* rows,
                     int nrows, int N, int max_cols, uint8_t* sel, double* obj, const SchedWorkspace& ws,
                     cudaStream_t stream) {
  if (nrows == 0) return;
  D2FT_REQUIRE(max_cols <= kThreads * kCMax, kSize, "dp_search: more than 2048 DP columns per row");
  DpConstArgs A{};
  A.scores = scores;
  A.row_wt = row_wt;
  A.caps = caps;
  A.rows = rows;
  A.N = N;
  A.sel = sel;
  A.obj = obj;
  A.ws = ws;
  A.words_max = bits_words_per_item(max_cols);
  const size_t smem = sched_smem_layout(N, max_cols, 1, &A.bits_in_smem);
  if (!A.bits_in_smem)
    D2FT_REQUIRE(ws.bits_global && ws.bits_global_words >= (size_t)nrows * N * A.words_max, kState,
                 "dp_search: global decision-bit workspace too small");
  D2FT_CUDA(cudaFuncSetAttribute(dp_const_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap));
  dp_const_kernel<<<nrows, max_cols <= 32 * kLaneColsMax ? 32 : kThreads, smem, stream>>>(A);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_dp_general(const double* scores, const int32_t* weights, const int32_t* caps, const int32_t* rows,
                       int nrows, int N, int max_cap, uint8_t* sel, double* obj, uint32_t* bits_global,
                       double* vals_global, cudaStream_t stream) {
  if (nrows == 0) return;
  dp_general_kernel<<<nrows, kThreads, 0, stream>>>(scores, weights, caps, rows, N, max_cap, sel, obj, bits_global,
                                                    vals_global);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_merge(const uint8_t* full_sel, const uint8_t* fwd_sel, size_t n, uint8_t* codes, cudaStream_t s) {
  if (n == 0) return;
  const int blocks = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  merge_kernel<<<blocks, 256, 0, s>>>(full_sel, fwd_sel, n, codes);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_compact(const uint8_t* codes, int K, int N, int H, const CompactLists& lists, cudaStream_t s) {
  compact_rows_kernel<<<K, 128, (size_t)N, s>>>(codes, N, lists);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
  const int cells = N * (K / H);
  compact_cols_kernel<<<(cells + 255) / 256, 256, 0, s>>>(codes, K, N, H, lists);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_scaler(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                   const int32_t* total_cap, int K, int N, const double* lambda_dev, int max_cap, uint8_t* codes,
                   uint8_t* choice_global, double* vals_global, cudaStream_t s) {
  scaler_kernel<<<K, kThreads, 0, s>>>(bwd, fwd, cf, cb, total_cap, N, lambda_dev, max_cap, codes, choice_global,
                                       vals_global);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace d2ft_b200
