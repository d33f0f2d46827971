// tcgen05 attention for dh = 64 (softmax(Q K^T / sqrt(dh)) V of
// an active (sample, head) cell, model.cpp:205-213).
//
// Forward, one CTA (4 warps, thread = query row = TMEM lane) per (sample,
// active head), two CTAs per SM:
//   TMA: Q (two 128-row tiles), K (TQ rows) and V (64-key blocks) of the cell
//        from the token-major QKV buffer (128-byte swizzle, rows >= T zero).
//   per query tile:  S = Q K^T        UMMA M=128 N=TQ K=64 -> TMEM cols [0, TQ)
//                    row max / exp2 / row sum straight from TMEM (each thread
//                    owns a whole score row: no shuffles), P (fp16, two per
//                    column) written back over S with tcgen05.st
//                    O = P V          UMMA with A = P from TMEM, B = V read
//                                     MN-major from shared memory -> cols [128, 192)
//                    O / rowsum -> OGT (feature-major, coalesced over tokens),
//                    lse (log2 domain) for the backward.
// The whole key range (T <= 256) fits one score row, so there is no online
// rescaling.
#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "gemm_sm100.cuh"
#include "ptx.cuh"
#include "step_common.cuh"
#include "step_kernels.cuh"

namespace d2ft_b200 {

namespace {

constexpr int kQTile = 128;

// Experiment builds (-DD2FT_ATTN_TRACE): per-CTA event stamps (SM clock) of
// the attention kernels of one layer, read back with d2ft_debug_attn_trace.
#ifdef D2FT_ATTN_TRACE
// stamps go to shared memory (one 64-entry ring per warp, written by lane 0:
// no global round trip inside the timed phases) and are copied out at exit
constexpr int kTrCtas = 16, kTrWarps = 16, kTrPer = 96, kTrLayer = 6;
__device__ unsigned long long g_attn_trace[2][kTrCtas][kTrWarps * kTrPer];
__device__ int g_attn_trace_n[2][kTrCtas];
#define ATR_DECL(nw)                                \
  __shared__ unsigned long long tr_buf[nw][kTrPer]; \
  int tr_n = 0;                                     \
  constexpr int tr_nw = nw;
#define ATR(kind, code, item)                                                                          \
  do {                                                                                                 \
    if ((threadIdx.x & 31) == 0 && tr_n < kTrPer && (threadIdx.x >> 5) < tr_nw)                        \
      tr_buf[threadIdx.x >> 5][tr_n++] = ((unsigned long long)(code) << 56) |                          \
                                         ((unsigned long long)((item) & 255) << 48) |                   \
                                         ((unsigned long long)clock64() & 0xFFFFFFFFFFull);           \
  } while (0)
#define ATR_FLUSH(kind)                                                                                \
  do {                                                                                                 \
    const int b_ = blockIdx.x + blockIdx.y * gridDim.x, w_ = threadIdx.x >> 5;                         \
    if (a.l == kTrLayer && b_ < kTrCtas && (threadIdx.x & 31) == 0 && w_ < tr_nw) {                    \
      for (int i_ = 0; i_ < kTrPer; ++i_)                                                              \
        g_attn_trace[kind][b_][w_ * kTrPer + i_] = i_ < tr_n ? tr_buf[w_][i_] | ((unsigned long long)w_ << 40) : 0ull; \
      atomicAdd(&g_attn_trace_n[kind][b_], tr_n);                                                      \
    }                                                                                                  \
  } while (0)
#define ATR_Q(kind, code, item) \
  do {                          \
    if (q4 == 0) ATR(kind, code, item); \
  } while (0)
#else
#define ATR_DECL(nw)
#define ATR_FLUSH(kind) \
  do {                  \
  } while (0)
#define ATR_Q(kind, code, item) \
  do {                          \
  } while (0)
#define ATR(kind, code, item) \
  do {                        \
  } while (0)
#endif

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp; P is rounded to fp16 right after)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2eF = 1.4426950408889634f;

// 2^x for x <= 0 on the FMA pipe: round-to-nearest split x = j + f
// (|f| <= 1/2) by the 1.5 * 2^23 shifter, 2^f by a degree-4 fit (Chebyshev
// nodes on [-1/2, 1/2], relative error 3.5e-6 — below the fp16 rounding P
// gets next), j added to the exponent field.  x is clamped at -125 (P rounds
// to 0 in fp16 far above that).
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float j = t - 12582912.f;
  const float f = x - j;
  float p = fmaf(0.00966637f, f, 0.05592198f);
  p = fmaf(p, f, 0.24022349f);
  p = fmaf(p, f, 0.69312105f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// Forward softmax variants (experiment builds; defaults = the measured best):
//   D2FT_ATTN_POLY   exponentials per 16 computed by exp2_poly (the rest on the SFU)
//   D2FT_AF_FREE     release the O accumulator's TMEM columns after its last load
//   D2FT_AF_SKIPDEAD warps whose 32 queries all lie past T skip the softmax
//   D2FT_AF_SINGLE   one read of the scores against a running reference max
#ifndef D2FT_ATTN_POLY
#define D2FT_ATTN_POLY 0
#endif
#ifndef D2FT_AF_FREE
#define D2FT_AF_FREE 0
#endif
#ifndef D2FT_AF_SKIPDEAD
#define D2FT_AF_SKIPDEAD 0
#endif
#ifndef D2FT_AF_SINGLE
#define D2FT_AF_SINGLE 0
#endif
constexpr int kPolyExp = D2FT_ATTN_POLY;
constexpr bool kFreeEarly = D2FT_AF_FREE, kSkipDead = D2FT_AF_SKIPDEAD;
constexpr int kFwdSmWarps = 4;  // softmax warps per query tile (one per TMEM lane quarter)
constexpr int kFwdThreads = 128 + 2 * 32 * kFwdSmWarps;
// largest excess of a later chunk's max over the running reference before
// the stored P is rescaled: P <= 2^8, well inside fp16
constexpr float kRescaleGap = 8.f;

struct AttnFwdArgs {
  Dims D;
  int l;
  const int* items;  // block l: (sample << 8 | active slot), plan_kernel
  const int* count;  // block l: number of items
  const int* act_heads;
  act_t* OGT;  // block l
  float* lse;  // block l
  const uint8_t* codes;  // expanded K x Bmax (code 1 = Full)
  float* O32T;           // block l: [Bmax][H][64][TP] fp32 O of Full cells (the backward's D)
  float gap;             // softmax rescale threshold (kRescaleGap; D2FT_ATTN_RESCALE_GAP overrides, tests)
};

__host__ __device__ inline int attn_fwd_stage_bytes(int TQ) {
  const int b = 2 * kQTile * 128 + TQ * 128 + ((TQ + 63) / 64) * 8192;
  return (b + 1023) & ~1023;
}
__host__ __device__ inline int attn_tc_smem(int TQ) { return 2 * attn_fwd_stage_bytes(TQ) + 1024; }

// Persistent, warp-specialised: warp 0 TMA (two item stages), warp 1 MMA,
// warp 2 TMEM allocator, warps 4-7 / 8-11 = softmax+epilogue of query tile
// 0 / 1 (TMEM columns [0,256) / [256,512)), so both tiles of an item run in
// parallel and the next item's operands land during the current one.
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const AttnFwdArgs a) {
  pdl_trigger();
  ATR_DECL(12)
  const Dims& D = a.D;
  const int TQ = D.TQ, T = D.T;
  const int nkv = (TQ + 63) / 64, nqt = (T + kQTile - 1) / kQTile;
  const uint32_t stage = attn_fwd_stage_bytes(TQ);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t load_full[2], load_empty[2], s_full[2], p_full[2], o_full[2], tfree[2];
  __shared__ uint32_t tslot[1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmQ);
    ptx::tma_prefetch(&tmK);
    ptx::tma_prefetch(&tmV);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&load_full[i], 1);
      ptx::mbar_init(&load_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], kFwdSmWarps);
      ptx::mbar_init(&o_full[i], 1);
      ptx::mbar_init(&tfree[i], kFwdSmWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  const int nitems = *a.count;
  auto decode = [&](int i, int& s, int& h) {
    const int it = a.items[i];
    s = it >> 8;
    h = a.act_heads[(s * D.L + a.l) * D.H + (it & 255)];
  };

  if (warp == 0) {
    if (lane == 0) {
      for (int i = blockIdx.x, it = 0; i < nitems; i += gridDim.x, ++it) {
        const int buf = it & 1;
        ptx::mbar_wait(&load_empty[buf], ((it >> 1) & 1) ^ 1);
        ATR(0, 0, it);
        int s, h;
        decode(i, s, h);
        const int plane = (a.l * D.Bmax + s) * D.H + h;
        uint8_t* sQ = smem + buf * stage;
        uint8_t* sK = sQ + 2 * kQTile * 128;
        uint8_t* sV = sK + TQ * 128;
        ptx::mbar_arrive_expect_tx(&load_full[buf], (uint32_t)(nqt * kQTile * 128 + TQ * 128 + nkv * 8192));
        for (int qt = 0; qt < nqt; ++qt)
          ptx::tma_load_3d(sQ + qt * kQTile * 128, &tmQ, &load_full[buf], 0, qt * kQTile, plane);
        ptx::tma_load_3d(sK, &tmK, &load_full[buf], 64, 0, plane);
        for (int j = 0; j < nkv; ++j) ptx::tma_load_3d(sV + j * 8192, &tmV, &load_full[buf], 128, 64 * j, plane);
      }
    }
  } else if (warp == 1) {
    const uint32_t idS = ptx::idesc_f16_m128(TQ, 0);
    const uint32_t idO = ptx::idesc_f16_m128(64, 0) | (1u << 16);  // B = V, MN-major
    for (int i = blockIdx.x, it = 0; i < nitems; i += gridDim.x, ++it) {
      const int buf = it & 1;
      ptx::mbar_wait(&load_full[buf], (it >> 1) & 1);
      if (lane == 0) ATR(0, 1, it);
      ptx::tc_fence_after();
      const uint32_t qb = ptx::smem_u32(smem + buf * stage);
      const uint32_t kb = qb + 2 * kQTile * 128, vb = kb + TQ * 128;
      for (int t = 0; t < nqt; ++t) {
        ptx::mbar_wait(&tfree[t], (it & 1) ^ 1);
        if (lane == 0) ATR(0, 2 + t, it);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint64_t qd = ptx::desc_sw128(qb + t * kQTile * 128), kd = ptx::desc_sw128(kb);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::umma_bf16(tmem + 256 * t, qd + (uint64_t)(kk * 2), kd + (uint64_t)(kk * 2), idS, kk);
          ptx::umma_commit(&s_full[t]);
        }
        __syncwarp();
      }
      for (int t = 0; t < nqt; ++t) {
        ptx::mbar_wait(&p_full[t], it & 1);
        if (lane == 0) ATR(0, 4 + t, it);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          for (int kk = 0; kk < TQ / 16; ++kk)
            ptx::umma_ts(tmem + 256 * t + 128, tmem + 256 * t + kk * 8,
                         ptx::desc_sw128_mn(vb + (kk >> 2) * 8192 + (kk & 3) * 2048, 8192), idO, kk);
          ptx::umma_commit(&o_full[t]);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::umma_commit(&load_empty[buf]);
      __syncwarp();
    }
#if D2FT_AF_SINGLE == 0
  } else if (warp >= 4 && (warp - 4) / 4 < nqt) {
    // One warp per TMEM lane quarter of each query tile; thread = query row:
    // row max, then P = 2^(s*sl2 - max) as fp16 pairs written back over S,
    // then O / rowsum out of TMEM.
    const int t = (warp - 4) / 4, q4 = warp & 3;
    const uint32_t base = tmem + 256 * t + ((uint32_t)(q4 * 32) << 16);
    const float sl2 = kLog2eF * 0.125f;  // log2(e) / sqrt(64)
    const int cfull = T & ~15;           // chunks [0, cfull) hold valid keys only
    const int row = t * kQTile + q4 * 32 + lane;  // query
    // a warp whose 32 queries all lie past T has nothing to compute: its P
    // rows only feed O rows that are never stored (MMA rows are independent)
    const bool live = !kSkipDead || t * kQTile + q4 * 32 < T;
    for (int i = blockIdx.x, it = 0; i < nitems; i += gridDim.x, ++it) {
      int s, h;
      decode(i, s, h);
      const size_t sh = (size_t)s * D.H + h;
      ptx::mbar_wait(&s_full[t], it & 1);
      ATR_Q(0, 10 + 8 * t, it);
      ptx::tc_fence_after();
      float mx = -INFINITY, sum = 0.f;
      if (live) {
        for (int c0 = 0; c0 < TQ; c0 += 16) {
          float v[16];
          ptx::tmem_ld16(base + c0, v);
          if (c0 < cfull) {
#pragma unroll
            for (int j = 0; j < 16; ++j) mx = fmaxf(mx, v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < T) mx = fmaxf(mx, v[j]);
          }
        }
        mx *= sl2;
        ATR_Q(0, 11 + 8 * t, it);
        for (int c0 = 0; c0 < TQ; c0 += 16) {
          float v[16];
          if (it == 1) ATR_Q(0, 30, c0 >> 4);
          ptx::tmem_ld16(base + c0, v);
          if (it == 1) ATR_Q(0, 31, c0 >> 4);
          float p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float x = fmaf(v[j], sl2, -mx);
            p[j] = j < kPolyExp ? exp2_poly(x) : fast_exp2(x);
          }
          if (it == 1) ATR_Q(0, 32, c0 >> 4);
          if (c0 >= cfull) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j >= T) p[j] = 0.f;
          }
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sum += p[2 * j] + p[2 * j + 1];
            __half2 hp = __floats2half2_rn(p[2 * j], p[2 * j + 1]);
            pk[j] = *reinterpret_cast<uint32_t*>(&hp);
          }
          ptx::tmem_st8(base + (c0 >> 1), pk);
          if (it == 1) ATR_Q(0, 33, c0 >> 4);
        }
        ptx::tmem_st_wait();
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[t]);
      ATR_Q(0, 12 + 8 * t, it);
      if (row < T) a.lse[sh * T + row] = mx + log2f(sum);
      ptx::mbar_wait(&o_full[t], it & 1);
      ATR_Q(0, 13 + 8 * t, it);
      ptx::tc_fence_after();
      const float inv = 1.f / sum;
      act_t* o = a.OGT + sh * D.PO * D.TP + row;
      // Full cells also keep O in fp32: the backward's D = rowsum(dO . O) must be
      // consistent with its dP = dO V^T to the fp32 level (the softmax backward
      // dP - D cancels strongly when tokens are alike; an fp16 O costs ~1e-2 on
      // the wq/wk gradients at ViT-L)
      const bool full = a.codes[(size_t)(a.l * D.H + h) * D.Bmax + s] == 1;
      float* o32 = a.O32T + sh * 64 * D.TP + row;
      if (live) {
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          float v[16];
          ptx::tmem_ld16(base + 128 + c0, v);
          if (kFreeEarly && c0 == 48) {  // the accumulator is in registers: release its columns
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tfree[t]);
          }
          if (row < T) {
#pragma unroll
            for (int j = 0; j < 16; ++j) o[(size_t)(c0 + j) * D.TP] = to_act(v[j] * inv);
            if (full) {
#pragma unroll
              for (int j = 0; j < 16; ++j) o32[(size_t)(c0 + j) * D.TP] = v[j] * inv;
            }
          }
        }
      }
      if (!kFreeEarly || !live) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tfree[t]);
      }
      ATR_Q(0, 14 + 8 * t, it);
    }
  }
#else  // D2FT_AF_SINGLE: single read of the scores against a running reference max
  } else if (warp >= 4 && (warp - 4) / 4 < nqt) {
    // One warp per TMEM lane quarter of each query tile; thread = query row.
    // TMEM reads bound this loop, so each score is read once:
    // the row's reference max m comes from its first 64 columns (kept in
    // registers), every later chunk is exponentiated against m, and a chunk
    // whose max exceeds m by more than kRescaleGap (P would leave the fp16
    // range) rescales the P already stored by 2^(m - m') first (rare).
    // lse = m + log2(sum) holds for any m, so no second pass is needed.
    const int t = (warp - 4) / 4, q4 = warp & 3;
    const uint32_t base = tmem + 256 * t + ((uint32_t)(q4 * 32) << 16);
    const float sl2 = kLog2eF * 0.125f;  // log2(e) / sqrt(64)
    const int row = t * kQTile + q4 * 32 + lane;  // query
    // a warp whose 32 queries all lie past T has nothing to compute: its P
    // rows only feed O rows that are never stored (MMA rows are independent)
    const bool live = t * kQTile + q4 * 32 < T;
    const int nch = TQ / 16, npre = nch < 4 ? nch : 4;
    for (int i = blockIdx.x, it = 0; i < nitems; i += gridDim.x, ++it) {
      int s, h;
      decode(i, s, h);
      const size_t sh = (size_t)s * D.H + h;
      // Full cells also keep O in fp32 (the backward's D = rowsum(dO . O) must be
      // consistent with its dP = dO V^T to the fp32 level: the softmax backward
      // dP - D cancels strongly when tokens are alike; an fp16 O costs ~1e-2 on
      // the wq/wk gradients at ViT-L).  Loaded before the waits.
      const bool full = a.codes[(size_t)(a.l * D.H + h) * D.Bmax + s] == 1;
      ptx::mbar_wait(&s_full[t], it & 1);
      ATR_Q(0, 10 + 8 * t, it);
      ptx::tc_fence_after();
      float m = 0.f, sum = 0.f;
      if (live) {
        auto exp_chunk = [&](const uint32_t (&v)[16], int c0) {
          float p[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float x = fmaf(__uint_as_float(v[e]), sl2, -m);
            p[e] = e < kPolyExp ? exp2_poly(x) : fast_exp2(x);
          }
          if (c0 + 16 > T) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c0 + e >= T) p[e] = 0.f;
          }
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            sum += p[2 * e] + p[2 * e + 1];
            __half2 hp = __floats2half2_rn(p[2 * e], p[2 * e + 1]);
            pk[e] = *reinterpret_cast<uint32_t*>(&hp);
          }
          ptx::tmem_st8(base + (c0 >> 1), pk);
        };
        auto chunk_max = [&](const uint32_t (&v)[16], int c0) {
          float x = -INFINITY;
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c0 + e < T) x = fmaxf(x, __uint_as_float(v[e]));
          return x * sl2;
        };
        uint32_t pre[4][16];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < npre) ptx::tmem_ld16_async(base + 16 * j, pre[j]);
        ptx::tmem_ld_wait(pre[0]);
        ptx::tmem_ld_wait(pre[1]);
        ptx::tmem_ld_wait(pre[2]);
        ptx::tmem_ld_wait(pre[3]);
        m = -INFINITY;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < npre) m = fmaxf(m, chunk_max(pre[j], 16 * j));
        uint32_t cur[16], nxt[16];
        if (npre < nch) ptx::tmem_ld16_async(base + 16 * npre, cur);  // in flight during the prologue's math
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < npre) exp_chunk(pre[j], 16 * j);
        ATR_Q(0, 11 + 8 * t, it);
        if (npre < nch) ptx::tmem_ld_wait(cur);
        for (int j = npre; j < nch; ++j) {
          const int c0 = 16 * j;
          if (j + 1 < nch) ptx::tmem_ld16_async(base + c0 + 16, nxt);
          const float cm = chunk_max(cur, c0);
          if (__any_sync(0xffffffffu, cm > m + a.gap)) {
            // rare: P of chunks [0, j) to the new reference (lanes that do not
            // need it scale by 1)
            const float mn = fmaxf(m, cm);
            const float f = fast_exp2(m - mn);
            const __half2 f2 = __float2half2_rn(f);
            ptx::tmem_st_wait();
            for (int jj = 0; jj < j; ++jj) {
              uint32_t q[8];
              ptx::tmem_ld8_async(base + 8 * jj, q);
              ptx::tmem_ld_wait(q);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                __half2 hv = __hmul2(*reinterpret_cast<__half2*>(&q[e]), f2);
                q[e] = *reinterpret_cast<uint32_t*>(&hv);
              }
              ptx::tmem_st8(base + 8 * jj, q);
            }
            sum *= f;
            m = mn;
          }
          exp_chunk(cur, c0);
          if (j + 1 < nch) {
            ptx::tmem_ld_wait(nxt);
#pragma unroll
            for (int e = 0; e < 16; ++e) cur[e] = nxt[e];
          }
        }
        ptx::tmem_st_wait();
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[t]);
      ATR_Q(0, 12 + 8 * t, it);
      if (live && row < T) a.lse[sh * T + row] = m + log2f(sum);
      const float inv = 1.f / sum;
      ptx::mbar_wait(&o_full[t], it & 1);
      ATR_Q(0, 13 + 8 * t, it);
      ptx::tc_fence_after();
      if (live) {
        act_t* og = a.OGT + sh * D.PO * D.TP + row;
        float* o32 = a.O32T + sh * 64 * D.TP + row;
        uint32_t o[16];
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 16) {
          ptx::tmem_ld16_async(base + 128 + c0, o);
          ptx::tmem_ld_wait(o);
          if (c0 == 48) {  // the accumulator is in registers: release the columns
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tfree[t]);
          }
          if (row < T) {
#pragma unroll
            for (int e = 0; e < 16; ++e) og[(size_t)(c0 + e) * D.TP] = to_act(__uint_as_float(o[e]) * inv);
            if (full) {
#pragma unroll
              for (int e = 0; e < 16; ++e) o32[(size_t)(c0 + e) * D.TP] = __uint_as_float(o[e]) * inv;
            }
          }
        }
      } else {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tfree[t]);
      }
      ATR_Q(0, 14 + 8 * t, it);
    }
  }
#endif
  ptx::tc_fence_before();
  __syncthreads();
  ATR_FLUSH(0);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Backward, one CTA (4 warps) per (sample, Full head), keys as M (model.cpp
// 262-271; FA2 order, deterministic):
//   TMA: Q, K, V, dO tiles ([TQ rows][64], 128-byte swizzle).  Each tile is both
//   a K-major operand (rows = M or N) and an MN-major B operand (rows = K,
//   N = dh), so no transposed copies exist.
//   D_q = rowsum(dO . O) (O from OGT), lse in log2 units -> shared vectors.
//   per key tile (128 keys = TMEM lanes):
//     S^T = K Q^T, dP^T = V dO^T          -> TMEM [0, TQ), [256, 256+TQ)
//     P^T = exp2(S^T sl2 - lse), dS^T = P^T (dP^T - D): fp16, written back over
//     the scores (A operands from TMEM) and dS^T also into shared memory
//     dV = P^T dO, dK = dS^T Q / sqrt(dh)  -> TMEM [128,192), [384,448) -> dY1T
//   dQ = dS K / sqrt(dh): A = dS^T from shared memory read MN-major (queries
//   contiguous in 64-wide blocks), B = K  -> TMEM [0,64), [64,128) -> dY1T
struct AttnBwdArgs {
  Dims D;
  int l;
  const int* full_heads;
  const int* full_hcnt;
  const float* O32T;  // block l: [Bmax][H][64][TP] fp32 O (attention forward, Full cells)
  const float* lse;   // block l
  act_t* dY1T;        // [Bmax][H][PQ][TP]
};

// Q, K, V, dO tiles + 4 dS^T query blocks.  The S^T / dP^T UMMAs read K and V
// as M = 128 A operands: with TQ < 128 they read past their tile into the
// following ones (rows past T only feed TMEM lanes of keys >= T, never
// stored), so the allocation must cover sV + 128 rows for short sequences.
__host__ __device__ inline int attn_bwd_tc_smem(int TQ) {
  const int tiles = 8 * TQ * 128, v_extent = 2 * TQ * 128 + kQTile * 128;
  return (tiles > v_extent ? tiles : v_extent) + 1024;
}

// 16 warps: warp w owns TMEM lane quarter w % 4 (its 32 keys / queries) and
// column group w / 4 of every elementwise pass (softmax backward over the
// query columns, dV / dK / dQ drains), so the latency-bound per-element work
// of a cell runs on 4x the warps of one-warp-per-lane-quarter.
constexpr int kBwdWarps = 16;
__global__ void __launch_bounds__(32 * kBwdWarps, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmdO,
                       const AttnBwdArgs a) {
  D2FT_PDL_ENTRY();
  ATR_DECL(1)
  const Dims& D = a.D;
  const int s = blockIdx.y, slot = blockIdx.x;
  if (s >= D.B || slot >= a.full_hcnt[s * D.L + a.l]) return;
  const int h = a.full_heads[(s * D.L + a.l) * D.H + slot];
  const int plane = (a.l * D.Bmax + s) * D.H + h;
  const int TQ = D.TQ, T = D.T;
  const int nkt = (T + kQTile - 1) / kQTile;
  const size_t sh = (size_t)s * D.H + h;
  const uint32_t tile_bytes = (uint32_t)TQ * 128;
  constexpr int NT = 32 * kBwdWarps;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + tile_bytes;
  uint8_t* sV = sK + tile_bytes;
  uint8_t* sdO = sV + tile_bytes;
  uint8_t* sDS = sdO + tile_bytes;  // 4 query blocks x [TQ keys][128 B]
  __shared__ float lse2[256], Dv[256];  // statically shared: LDS, not generic loads
  __shared__ uint64_t bar[4];             // 0 load, 1 S/dP, 2 dV/dK, 3 dQ
  __shared__ uint32_t tslot[1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q4 = warp & 3, cg = warp >> 2;  // TMEM lane quarter, column group
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmQKV);
    ptx::tma_prefetch(&tmdO);
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) ATR(1, 0, slot);
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar[0], 4 * tile_bytes);
    ptx::tma_load_3d(sQ, &tmQKV, &bar[0], 0, 0, plane);
    ptx::tma_load_3d(sK, &tmQKV, &bar[0], 64, 0, plane);
    ptx::tma_load_3d(sV, &tmQKV, &bar[0], 128, 0, plane);
    ptx::tma_load_3d(sdO, &tmdO, &bar[0], 0, 0, (int)sh);
  }
  // lse (log2 units; +inf past T so P = 0) and the O rows for D, loaded while the tiles land
  for (int q = threadIdx.x; q < TQ; q += NT) lse2[q] = q < T ? a.lse[sh * T + q] : INFINITY;
  {
    // D_q = sum_f dO[q][f] O[q][f]: two threads per query, 32 features each
    const int q = threadIdx.x >> 1, hf = threadIdx.x & 1;
    float ov[32];
    if (q < T) {
      const float* o = a.O32T + sh * 64 * D.TP + (size_t)(32 * hf) * D.TP + q;
#pragma unroll
      for (int f = 0; f < 32; ++f) ov[f] = o[(size_t)f * D.TP];
    }
    ptx::mbar_wait(&bar[0], 0);
    float acc = 0.f;
    if (q < T) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cc = 4 * hf + c;
        const uint4 raw = *reinterpret_cast<const uint4*>(sdO + q * 128 + ((cc ^ (q & 7)) << 4));
        const act_t* hv = reinterpret_cast<const act_t*>(&raw);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += __half2float(hv[i]) * ov[c * 8 + i];
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (hf == 0 && q < TQ) Dv[q] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) ATR(1, 1, slot);

  const float sl2 = kLog2eF * 0.125f;
  const float scale = 0.125f;  // 1 / sqrt(64)
  const uint32_t idS = ptx::idesc_f16_m128(TQ, 0);                 // K-major A and B
  const uint32_t idG = ptx::idesc_f16_m128(64, 0) | (1u << 16);    // B (dh-wide tile) MN-major
  const uint32_t idQ = ptx::idesc_f16_m128(64, 0) | (1u << 15) | (1u << 16);  // A and B MN-major
  const uint32_t lrow = (uint32_t)(q4 * 32) << 16;
  const uint32_t SA = 0, SB = 256;
  act_t* dyt = a.dY1T + sh * D.PQ * D.TP;
  const uint32_t sds = ptx::smem_u32(sDS);
  const int nch = TQ / 16;
  for (int kt = 0; kt < nkt; ++kt) {
    if (threadIdx.x == 0) {
      ptx::tc_fence_after();
      const uint64_t kd = ptx::desc_sw128(ptx::smem_u32(sK + kt * kQTile * 128));
      const uint64_t vd = ptx::desc_sw128(ptx::smem_u32(sV + kt * kQTile * 128));
      const uint64_t qd = ptx::desc_sw128(ptx::smem_u32(sQ));
      const uint64_t od = ptx::desc_sw128(ptx::smem_u32(sdO));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        ptx::umma_bf16(tmem + SA, kd + (uint64_t)(kk * 2), qd + (uint64_t)(kk * 2), idS, kk);
        ptx::umma_bf16(tmem + SB, vd + (uint64_t)(kk * 2), od + (uint64_t)(kk * 2), idS, kk);
      }
      ptx::umma_commit(&bar[1]);
    }
    ptx::mbar_wait(&bar[1], kt & 1);
    if (threadIdx.x == 0) ATR(1, 2 + 4 * kt, slot);
    ptx::tc_fence_after();
    const int k = kt * kQTile + q4 * 32 + lane;  // this thread's key (TMEM lane)
    const bool kv = k < T;
    for (int j = cg; j < nch; j += 4) {
      const int c0 = 16 * j;
      float sv[16], dp[16];
      ptx::tmem_ld16(tmem + lrow + SA + c0, sv);
      ptx::tmem_ld16(tmem + lrow + SB + c0, dp);
      float p[16], ds[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        p[i] = kv ? fast_exp2(fmaf(sv[i], sl2, -lse2[c0 + i])) : 0.f;
        ds[i] = p[i] * (dp[i] - Dv[c0 + i]);
      }
      uint32_t pp[8], pd[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        __half2 a2 = __floats2half2_rn(p[2 * i], p[2 * i + 1]);
        __half2 b2 = __floats2half2_rn(ds[2 * i], ds[2 * i + 1]);
        pp[i] = *reinterpret_cast<uint32_t*>(&a2);
        pd[i] = *reinterpret_cast<uint32_t*>(&b2);
      }
      ptx::tmem_st8(tmem + lrow + SA + (c0 >> 1), pp);
      ptx::tmem_st8(tmem + lrow + SB + (c0 >> 1), pd);
      // dS^T row k, queries c0..c0+15 -> query block c0/64, 16-byte chunks (c0%64)/8 (+1), swizzled
      if (k < TQ) {  // rows past TQ would run into the next query block
        const uint32_t rb = sds + (uint32_t)(c0 >> 6) * tile_bytes + (uint32_t)k * 128;
        const int ch = (c0 & 63) >> 3;
        ptx::st_shared_v4(rb + ((ch ^ (k & 7)) << 4), pd[0], pd[1], pd[2], pd[3]);
        ptx::st_shared_v4(rb + (((ch + 1) ^ (k & 7)) << 4), pd[4], pd[5], pd[6], pd[7]);
      }
    }
    ptx::tmem_st_wait();
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) ATR(1, 3 + 4 * kt, slot);
    if (threadIdx.x == 0) {
      ptx::tc_fence_after();
      for (int kk = 0; kk < TQ / 16; ++kk) {
        const uint64_t od = ptx::desc_sw128_mn(ptx::smem_u32(sdO) + kk * 2048, 8192);
        const uint64_t qd = ptx::desc_sw128_mn(ptx::smem_u32(sQ) + kk * 2048, 8192);
        ptx::umma_ts(tmem + SA + 128, tmem + SA + kk * 8, od, idG, kk);  // dV += P^T dO
        ptx::umma_ts(tmem + SB + 128, tmem + SB + kk * 8, qd, idG, kk);  // dK += dS^T Q
      }
      ptx::umma_commit(&bar[2]);
    }
    ptx::mbar_wait(&bar[2], kt & 1);
    if (threadIdx.x == 0) ATR(1, 4 + 4 * kt, slot);
    ptx::tc_fence_after();
    {
      const int c0 = 16 * cg;  // this warp's 16 of the 64 dV / dK columns
      float dv[16], dk[16];
      ptx::tmem_ld16(tmem + lrow + SA + 128 + c0, dv);
      ptx::tmem_ld16(tmem + lrow + SB + 128 + c0, dk);
      if (kv) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          dyt[(size_t)(D.dh + c0 + i) * D.TP + k] = to_act(dk[i] * scale);
          dyt[(size_t)(2 * D.dh + c0 + i) * D.TP + k] = to_act(dv[i]);
        }
      }
    }
    ptx::tc_fence_before();
    __syncthreads();  // TMEM regions free for the next key tile
    if (threadIdx.x == 0) ATR(1, 5 + 4 * kt, slot);
  }
  // dQ = dS K: query tiles of 128 (two 64-wide MN-major blocks of dS^T each)
  if (threadIdx.x == 0) {
    ptx::tc_fence_after();
    for (int qt = 0; qt < nkt; ++qt)
      for (int kk = 0; kk < TQ / 16; ++kk) {
        const uint64_t ad = ptx::desc_sw128_mn(sds + (uint32_t)(2 * qt) * tile_bytes + kk * 2048, tile_bytes);
        const uint64_t bd = ptx::desc_sw128_mn(ptx::smem_u32(sK) + kk * 2048, 8192);
        ptx::umma_bf16(tmem + 64 * qt, ad, bd, idQ, kk);
      }
    ptx::umma_commit(&bar[3]);
  }
  ptx::mbar_wait(&bar[3], 0);
  if (threadIdx.x == 0) ATR(1, 20, slot);
  ptx::tc_fence_after();
  for (int qt = 0; qt < nkt; ++qt) {
    const int q = qt * kQTile + q4 * 32 + lane;
    const int c0 = 16 * cg;
    float dq[16];
    ptx::tmem_ld16(tmem + lrow + 64 * qt + c0, dq);
    if (q < T) {
#pragma unroll
      for (int i = 0; i < 16; ++i) dyt[(size_t)(c0 + i) * D.TP + q] = to_act(dq[i] * scale);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ATR(1, 21, slot);
  ATR_FLUSH(1);
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

void launch_attn_bwd_tc(const CUtensorMap& tmQKV, const CUtensorMap& tmdO, const Dims& D, int l, const int* full_heads,
                        const int* full_hcnt, const float* O32T, const float* lse, act_t* dY1T, cudaStream_t st) {
  D2FT_REQUIRE(D.dh == 64 && D.TQ <= 256, kConfig, "tcgen05 attention: head_dim 64, T <= 256");
  const int sm = attn_bwd_tc_smem(D.TQ);
  D2FT_REQUIRE(attn_bwd_tc_fits(D.TQ), kConfig, "tcgen05 attention backward: shared memory");
  static unsigned long long attr = 0;
  once_per_device(attr, [&] {
    D2FT_CUDA(cudaFuncSetAttribute(attn_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 223 * 1024));
  });
  dim3 grid(D.H, D.B);
  attn_bwd_tc_kernel<<<grid, 32 * kBwdWarps, sm, st>>>(tmQKV, tmdO, AttnBwdArgs{D, l, full_heads, full_hcnt, O32T, lse, dY1T});
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_attn_fwd_tc(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV, const Dims& D, int l,
                        const int* items, const int* count, const int* act_heads, act_t* OGT, float* lse,
                        const uint8_t* codes, float* O32T, cudaStream_t st) {
  D2FT_REQUIRE(D.dh == 64 && D.TQ <= 256, kConfig, "tcgen05 attention: head_dim 64, T <= 256");
  const int sm = attn_tc_smem(D.TQ);
  static unsigned long long attr = 0;
  once_per_device(attr, [&] {
    D2FT_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_max_attn()));
  });
  const char* g = getenv("D2FT_ATTN_RESCALE_GAP");  // tests force the rescale path with a small gap
  const float gap = g ? (float)atof(g) : kRescaleGap;
  attn_fwd_tc_kernel<<<num_sms(), kFwdThreads, sm, st>>>(
      tmQ, tmK, tmV, AttnFwdArgs{D, l, items, count, act_heads, OGT, lse, codes, O32T, gap});
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

int sm_max_attn() { return attn_tc_smem(256); }

}  // namespace d2ft_b200

#ifdef D2FT_ATTN_TRACE
// experiment builds: copy the trace (kind 0 forward, 1 backward) of one launch
// of layer kTrLayer; out = [kTrCtas][kTrWarps * kTrPer] u64 stamps
// (code << 56 | item << 48 | warp << 40 | 40-bit SM clock), counts = [kTrCtas]; clears it
extern "C" int d2ft_debug_attn_trace(int kind, unsigned long long* out, int* counts) {
  using namespace d2ft_b200;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(g_attn_trace[0]), kind * sizeof(g_attn_trace[0]));
  static unsigned long long zt[kTrCtas][kTrWarps * kTrPer] = {};
  cudaMemcpyToSymbol(g_attn_trace, zt, sizeof(zt), kind * sizeof(zt));
  cudaMemcpyFromSymbol(counts, g_attn_trace_n, sizeof(g_attn_trace_n[0]), kind * sizeof(g_attn_trace_n[0]));
  static int zero[kTrCtas] = {};
  cudaMemcpyToSymbol(g_attn_trace_n, zero, sizeof(zero), kind * sizeof(zero));
  return (int)cudaGetLastError();
}
#endif

namespace d2ft_b200 {
bool attn_bwd_tc_fits(int TQ) { return attn_bwd_tc_smem(TQ) + 4096 <= 227 * 1024; }  // + static shared

}  // namespace d2ft_b200
