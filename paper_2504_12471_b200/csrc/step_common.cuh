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
// Epilogue warpgroups of G3 and G4 (their prefetch strides and G4's db1
// partial-sum slots depend on them; engine.cu instantiates the GEMMs with the
// same values).  G4 with 2: 0.515 vs 0.64 ms per step at 4 (ViT-B).
#ifndef D2FT_G3_EPI
#define D2FT_G3_EPI 4
#endif
#ifndef D2FT_G4_EPI
#define D2FT_G4_EPI 2
#endif
constexpr int kG3Epi = D2FT_G3_EPI;
constexpr int kG4Epi = D2FT_G4_EPI;
// scoring pre-pass: GEMM tiles per (unit, head) partial slot (>= m-tiles (d/128 <= 8) x n-tiles (2))
constexpr int kScoreTiles = 16;

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
// Two elements at once with sm_100 packed fp32 arithmetic (FFMA2 / FMUL2):
// the same A&S 7.1.26 evaluation as gelu_and_grad (the 0.5 of Phi folded into
// the polynomial coefficients), ~12 instructions per element instead of ~24.
// This is the G1 epilogue's inner loop (4/7 of its rows are GELU rows).
struct f32x2 {
  unsigned long long v;
};
__device__ __forceinline__ f32x2 f2_make(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_split(f32x2 x, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
}
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ void gelu_and_grad2(float z0, float z1, float& g0, float& g1, float& gp0, float& gp1) {
  const f32x2 z = f2_make(z0, z1);
  const f32x2 one = f2_make(1.f, 1.f);
  // t = 1 / (1 + p |z| / sqrt2)
  const float kp = 0.3275911f * 0.70710678118654752f;
  const f32x2 den = f2_fma(f2_make(fabsf(z0), fabsf(z1)), f2_make(kp, kp), one);
  float d0, d1;
  f2_split(den, d0, d1);
  const f32x2 t = f2_make(__fdividef(1.f, d0), __fdividef(1.f, d1));
  // e^{-z^2/2} = 2^{-z^2 log2(e) / 2}
  const float ke = -0.5f * 1.4426950408889634f;
  float a0, a1;
  f2_split(f2_mul(f2_mul(z, z), f2_make(ke, ke)), a0, a1);
  float ex0, ex1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex0) : "f"(a0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex1) : "f"(a1));
  const f32x2 ex = f2_make(ex0, ex1);
  // q = 0.5 * poly(t) * ex = 0.5 (1 - erf(|z|/sqrt2)) = Phi(-|z|)
  f32x2 poly = f2_fma(t, f2_make(0.5f * 1.061405429f, 0.5f * 1.061405429f),
                      f2_make(0.5f * -1.453152027f, 0.5f * -1.453152027f));
  poly = f2_fma(t, poly, f2_make(0.5f * 1.421413741f, 0.5f * 1.421413741f));
  poly = f2_fma(t, poly, f2_make(0.5f * -0.284496736f, 0.5f * -0.284496736f));
  poly = f2_fma(t, poly, f2_make(0.5f * 0.254829592f, 0.5f * 0.254829592f));
  const f32x2 q = f2_mul(f2_mul(poly, t), ex);
  float q0, q1;
  f2_split(q, q0, q1);
  const f32x2 cdf = f2_make(z0 >= 0.f ? 1.f - q0 : q0, z1 >= 0.f ? 1.f - q1 : q1);
  f2_split(f2_mul(z, cdf), g0, g1);
  const float kc = 0.39894228040143268f;  // 1/sqrt(2 pi)
  f2_split(f2_fma(f2_mul(z, ex), f2_make(kc, kc), cdf), gp0, gp1);
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
