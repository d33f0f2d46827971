// Shared dimensions and device helpers of the D2FT step engine.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace d2ft_b200 {

using bf16 = __nv_bfloat16;

// Model/step geometry (ModelConfig, model.hpp:43-57, plus the B200 layout).
struct Dims {
  int L, H, d, ffn, T, C;  // reference config
  int dh, fs;              // head dim d/H, FFN slice ffn/H
  int PQ, PO;              // rows per head of [Wq|Wk|Wv|W1]^T (3dh+fs) and of [Wo;W2] (dh+fs)
  int UQ, UO;              // 64-row units per head: ceil(PQ/64), ceil(PO/64)
  int TP;                  // token pitch of token-innermost (transposed) buffers: T rounded to 8
  int TQ;                  // T rounded to 16 (attention row padding)
  int TB;                  // 64-token K-blocks per sample: ceil(T/64)
  int Bmax;                // batch capacity of the buffers
  int B;                   // samples in this step
  int K() const { return L * H; }
};

__device__ __forceinline__ float gelu_f(float z) { return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float z) {
  return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) + z * 0.39894228040143268f * __expf(-0.5f * z * z);
}

__device__ __forceinline__ void st_bf16x8(bf16* dst, const float* v) {
  __align__(16) __nv_bfloat162 h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(h);
}

}  // namespace d2ft_b200
