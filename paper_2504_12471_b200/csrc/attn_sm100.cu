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

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp; P is rounded to fp16 right after)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2eF = 1.4426950408889634f;

struct AttnFwdArgs {
  Dims D;
  int l;
  const int* act_heads;
  const int* act_cnt;
  act_t* OGT;  // block l
  float* lse;  // block l
};

__host__ __device__ inline int attn_tc_smem(int TQ) {
  const int nkv = (TQ + 63) / 64;
  return 2 * kQTile * 128 + TQ * 128 + nkv * 8192 + 1024 + 64;
}

__global__ void __launch_bounds__(128, 2)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const AttnFwdArgs a) {
  const Dims& D = a.D;
  const int s = blockIdx.y, slot = blockIdx.x;
  if (s >= D.B || slot >= a.act_cnt[s * D.L + a.l]) return;
  const int h = a.act_heads[(s * D.L + a.l) * D.H + slot];
  const int plane = (a.l * D.Bmax + s) * D.H + h;
  const int TQ = D.TQ, T = D.T;
  const int nkv = (TQ + 63) / 64, nqt = (T + kQTile - 1) / kQTile;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // nqt x [128 rows][128 B]
  uint8_t* sK = sQ + 2 * kQTile * 128;  // [TQ rows][128 B]
  uint8_t* sV = sK + TQ * 128;          // nkv x [64 keys][128 B]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + nkv * 8192);  // 0 load, 1 S done, 2 O done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmQ);
    ptx::tma_prefetch(&tmK);
    ptx::tma_prefetch(&tmV);
    for (int i = 0; i < 3; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc(tslot, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar[0], (uint32_t)(nqt * kQTile * 128 + TQ * 128 + nkv * 8192));
    for (int qt = 0; qt < nqt; ++qt) ptx::tma_load_3d(sQ + qt * kQTile * 128, &tmQ, &bar[0], 0, qt * kQTile, plane);
    ptx::tma_load_3d(sK, &tmK, &bar[0], 64, 0, plane);
    for (int j = 0; j < nkv; ++j) ptx::tma_load_3d(sV + j * 8192, &tmV, &bar[0], 128, 64 * j, plane);
    ptx::mbar_wait(&bar[0], 0);
  }
  const float sl2 = kLog2eF * 0.125f;  // log2(e) / sqrt(64)
  const uint32_t idS = ptx::idesc_f16_m128(TQ, 0);
  const uint32_t idO = ptx::idesc_f16_m128(64, 0) | (1u << 16);  // B = V, MN-major
  const uint32_t lrow = (uint32_t)(warp * 32) << 16;               // this warp's TMEM lane quarter
  const size_t sh = (size_t)s * D.H + h;
  for (int qt = 0; qt < nqt; ++qt) {
    if (threadIdx.x == 0) {
      ptx::tc_fence_after();
      const uint64_t qd = ptx::desc_sw128(ptx::smem_u32(sQ + qt * kQTile * 128));
      const uint64_t kd = ptx::desc_sw128(ptx::smem_u32(sK));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) ptx::umma_bf16(tmem, qd + (uint64_t)(kk * 2), kd + (uint64_t)(kk * 2), idS, kk);
      ptx::umma_commit(&bar[1]);
    }
    ptx::mbar_wait(&bar[1], qt & 1);
    ptx::tc_fence_after();
    // row max over the valid keys (scores in log2 units); only the chunk that
    // straddles T needs the key mask
    const int cfull = T & ~15;  // chunks [0, cfull) hold valid keys only
    float mx = -INFINITY;
    for (int c0 = 0; c0 < TQ; c0 += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + lrow + c0, v);
      if (c0 < cfull) {
#pragma unroll
        for (int i = 0; i < 16; ++i) mx = fmaxf(mx, v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < T) mx = fmaxf(mx, v[i]);
      }
    }
    mx *= sl2;
    // P = exp2(S * sl2 - max), fp16 pairs written back over the scores
    float sum = 0.f;
    for (int c0 = 0; c0 < TQ; c0 += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + lrow + c0, v);
      float p[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) p[i] = fast_exp2(fmaf(v[i], sl2, -mx));
      if (c0 >= cfull) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i >= T) p[i] = 0.f;
      }
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        sum += p[2 * i] + p[2 * i + 1];
        __half2 hp = __floats2half2_rn(p[2 * i], p[2 * i + 1]);
        pk[i] = *reinterpret_cast<uint32_t*>(&hp);
      }
      ptx::tmem_st8(tmem + lrow + (c0 >> 1), pk);
    }
    ptx::tmem_st_wait();
    const int t = qt * kQTile + threadIdx.x;
    if (t < T) a.lse[sh * T + t] = mx + log2f(sum);
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      ptx::tc_fence_after();
      for (int kk = 0; kk < TQ / 16; ++kk) {
        const uint32_t vb = ptx::smem_u32(sV + (kk >> 2) * 8192) + (kk & 3) * 2048;
        ptx::umma_ts(tmem + 128, tmem + kk * 8, ptx::desc_sw128_mn(vb, 8192), idO, kk);
      }
      ptx::umma_commit(&bar[2]);
    }
    ptx::mbar_wait(&bar[2], qt & 1);
    ptx::tc_fence_after();
    const float inv = 1.f / sum;
    act_t* o = a.OGT + sh * D.PO * D.TP + t;
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + lrow + 128 + c0, v);
      if (t < T) {
#pragma unroll
        for (int i = 0; i < 16; ++i) o[(size_t)(c0 + i) * D.TP] = to_act(v[i] * inv);
      }
    }
    ptx::tc_fence_before();
    __syncthreads();  // O and P read before the next tile's S overwrites the columns
  }
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

}  // namespace

void launch_attn_fwd_tc(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV, const Dims& D, int l,
                        const int* act_heads, const int* act_cnt, act_t* OGT, float* lse, cudaStream_t st) {
  D2FT_REQUIRE(D.dh == 64 && D.TQ <= 256, kConfig, "tcgen05 attention: head_dim 64, T <= 256");
  const int sm = attn_tc_smem(D.TQ);
  static bool attr = false;
  if (!attr) {
    D2FT_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_max_attn()));
    attr = true;
  }
  dim3 grid(D.H, D.B);
  attn_fwd_tc_kernel<<<grid, 128, sm, st>>>(tmQ, tmK, tmV, AttnFwdArgs{D, l, act_heads, act_cnt, OGT, lse});
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

int sm_max_attn() { return attn_tc_smem(256); }

}  // namespace d2ft_b200
