// Shared dimensions and device helpers of the D2FT step engine.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace d2ft_b200 {

using bf16 = __nv_bfloat16;
// GEMM / attention operand type of the step.  fp16 (10-bit mantissa): the same
// tcgen05 rate as bf16, 4x finer rounding (the wq/wk gradients are
// ill-conditioned on token-similar inputs).  Gradient operands
// carry a per-step power-of-two scale so they stay inside the fp16 range.
using act_t = __half;
__device__ __forceinline__ act_t to_act(float v) { return __float2half_rn(v); }
__device__ __forceinline__ float act_to_f(act_t v) { return __half2float(v); }
// Power-of-two gradient scale S (max|S*dX_L| in (1/2, 1]) from the running max
// written by the head kernel; every consumer derives the identical S.
__device__ __forceinline__ float grad_scale(const float* gmax) {
  const float m = *gmax;
  return m > 0.f ? exp2f(-ceilf(log2f(m))) : 1.f;
}

// epilogue warpgroups of the step GEMMs (GemmShape::EPI) — G4's db1 partials
constexpr int kEpiGroups = 4;

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
// GELU and its derivative (linalg.cpp:182-188, exact-erf form) sharing one
// exp: Phi(z) = 0.5 (1 + erf(z/sqrt2)) with erf from Abramowitz & Stegun
// 7.1.26, |error| <= 3e-7 on Phi over all z (checked against scipy's erf;
// far below the fp16 rounding of the stored g / GELU').  ~14 instructions
// against ~35 for erff + expf.
__device__ __forceinline__ void gelu_and_grad(float z, float& g, float& gp) {
  const float x = fabsf(z) * 0.70710678118654752f;
  const float t = __fdividef(1.0f, fmaf(0.3275911f, x, 1.0f));
  const float ex = __expf(-0.5f * z * z);  // e^{-x^2}
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f), 0.254829592f);
  const float erf_abs = 1.0f - poly * ex;
  const float cdf = 0.5f + copysignf(0.5f * erf_abs, z);
  g = z * cdf;
  gp = cdf + z * 0.39894228040143268f * ex;
}
__device__ __forceinline__ float gelu_grad_f(float z) {
  return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) + z * 0.39894228040143268f * __expf(-0.5f * z * z);
}

__device__ __forceinline__ void st_act_x8(act_t* dst, const float* v) {
  __align__(16) __half2 h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(h);
}

}  // namespace d2ft_b200
