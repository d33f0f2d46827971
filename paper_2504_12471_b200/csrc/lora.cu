// LoRA variant of the step: rank-r adapters on Q/K/V of
// every head-subnet, base weights frozen (model.cpp:165-195, 204-211,
// 273-302; trainer visit_trainable, model.hpp:155-172).
//
// The step reuses the base path unchanged by linearity:
//   forward   q = xn Wq + s (xn D) U        = xn W_eff,   W_eff = Wq + s D U
//   dxn       dq Wq^T + s (dq U^T) D^T     = dq W_eff^T
//   gU        s Σ_samples (xn D)^T dq      = s D^T gW,   gW = Σ xn^T dq
//   gD        s Σ_samples xn^T (dq U^T)    = s gW U^T
// so the fp16 operand rows of [Wq|Wk|Wv] hold W_eff (lora_merge, after every
// adapter update), G1 / G8 run as before, G7 still produces gW (the base
// weight gradient of q/k/v, never applied), and lora_grad turns it into the
// adapter gradients — two (d x dh) x (dh x r)-sized products per projection
// instead of per-sample low-rank GEMMs.  G5, the bias reductions and the
// embed / classifier weight gradients are skipped (frozen tensors).
//
// Adapter arena (fp32): [L][H][ down_q d x r | up_q r x dh | down_k | up_k |
// down_v | up_v ] = visit_tensors order of the LoRA tensors (model.hpp:139-146).
#include "common.cuh"
#include "step_common.cuh"
#include "step_kernels.cuh"

namespace d2ft_b200 {
namespace {

constexpr int kLoraI = 64;  // feature rows per tile

// W1T_bf rows q*dh + j of head (l,h):  fp16(W[i][j] + s * sum_r D[i][r] U[r][j])
__global__ void __launch_bounds__(256) lora_merge_kernel(Dims D, int rank, float s, const float* W1T, const float* A,
                                                         act_t* W1T_bf) {
  D2FT_PDL_ENTRY();
  extern __shared__ float sm[];
  const int dh = D.dh, d = D.d;
  const int lhq = blockIdx.y, q = lhq % 3, lh = lhq / 3;
  const int i0 = blockIdx.x * kLoraI;
  const size_t per = 3 * ((size_t)d * rank + (size_t)rank * dh);
  const float* down = A + lh * per + q * ((size_t)d * rank + (size_t)rank * dh);
  const float* up = down + (size_t)d * rank;
  float* sD = sm;                  // [kLoraI][rank]
  float* sU = sm + kLoraI * rank;  // [rank][dh]
  for (int x = threadIdx.x; x < kLoraI * rank; x += blockDim.x) {
    const int i = i0 + x / rank;
    sD[x] = i < d ? down[(size_t)i * rank + x % rank] : 0.f;
  }
  for (int x = threadIdx.x; x < rank * dh; x += blockDim.x) sU[x] = up[x];
  __syncthreads();
  const size_t row0 = ((size_t)lh * D.PQ + (size_t)q * dh) * d;
  for (int x = threadIdx.x; x < kLoraI * dh; x += blockDim.x) {
    const int j = x / kLoraI, ii = x % kLoraI, i = i0 + ii;  // consecutive threads: consecutive features
    if (i >= d) continue;
    float acc = 0.f;
    for (int r = 0; r < rank; ++r) acc = fmaf(sD[ii * rank + r], sU[r * dh + j], acc);
    const size_t o = row0 + (size_t)j * d + i;
    W1T_bf[o] = to_act(W1T[o] + s * acc);
  }
}

// gD[i][r] = s sum_j gW[i][j] U[r][j],  gU[r][j] = s sum_i D[i][r] gW[i][j],
// gW[i][j] = G7's gradient row q*dh + j, column i (W1T layout).  One CTA per
// (l, h, q) with Full cells; feature tiles of 64 in a fixed order
// (deterministic).
__global__ void __launch_bounds__(256) lora_grad_kernel(Dims D, int rank, float s, const float* G1T, const float* A,
                                                        float* AG, const int* full_cnt) {
  D2FT_PDL_ENTRY();
  extern __shared__ float sm[];
  const int dh = D.dh, d = D.d;
  const int lhq = blockIdx.x, q = lhq % 3, lh = lhq / 3;
  if (full_cnt[lh] == 0) return;  // untouched subnet: its gradient is never applied
  const size_t blk = (size_t)d * rank + (size_t)rank * dh;
  const size_t per = 3 * blk;
  const float* down = A + lh * per + q * blk;
  const float* up = down + (size_t)d * rank;
  float* gdown = AG + lh * per + q * blk;
  float* gup = gdown + (size_t)d * rank;
  float* sU = sm;                       // [rank][dh]
  float* sG = sU + rank * dh;           // [kLoraI][dh + 1]
  float* sD = sG + kLoraI * (dh + 1);   // [kLoraI][rank]
  for (int x = threadIdx.x; x < rank * dh; x += blockDim.x) sU[x] = up[x];
  const float* g = G1T + ((size_t)lh * D.PQ + (size_t)q * dh) * d;
  // gU accumulators: output o = threadIdx.x + k*256 of the rank x dh tile
  constexpr int kAcc = 16;  // rank * dh <= 64 * 64 = 4096 = 16 x 256
  float acc[kAcc];
#pragma unroll
  for (int k = 0; k < kAcc; ++k) acc[k] = 0.f;
  for (int i0 = 0; i0 < d; i0 += kLoraI) {
    __syncthreads();
    for (int x = threadIdx.x; x < kLoraI * dh; x += blockDim.x) {
      const int j = x / kLoraI, ii = x % kLoraI, i = i0 + ii;
      sG[ii * (dh + 1) + j] = i < d ? g[(size_t)j * d + i] : 0.f;
    }
    for (int x = threadIdx.x; x < kLoraI * rank; x += blockDim.x) {
      const int i = i0 + x / rank;
      sD[x] = i < d ? down[(size_t)i * rank + x % rank] : 0.f;
    }
    __syncthreads();
    // gD rows of this tile (complete here)
    for (int x = threadIdx.x; x < kLoraI * rank; x += blockDim.x) {
      const int ii = x / rank, r = x % rank, i = i0 + ii;
      if (i >= d) continue;
      float a = 0.f;
      for (int j = 0; j < dh; ++j) a = fmaf(sG[ii * (dh + 1) + j], sU[r * dh + j], a);
      gdown[(size_t)i * rank + r] = s * a;
    }
#pragma unroll
    for (int k = 0; k < kAcc; ++k) {
      const int o = threadIdx.x + k * 256;
      if (o < rank * dh) {
        const int r = o / dh, j = o % dh;
        float a = acc[k];
        for (int ii = 0; ii < kLoraI; ++ii) a = fmaf(sD[ii * rank + r], sG[ii * (dh + 1) + j], a);
        acc[k] = a;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kAcc; ++k) {
    const int o = threadIdx.x + k * 256;
    if (o < rank * dh) gup[o] = s * acc[k];
  }
}

// LoRA-mode pre-pass scores (scoring.cpp:57-96 with lora_mode: visit_trainable
// walks only the six adapter tensors of a block subnet): one CTA per (l, h),
// fp64 sums in a fixed order (per-thread strided partials, then a tree), the
// chosen metric of the unit's adapter gradient -> fo / bo [K][n_units].
__global__ void __launch_bounds__(256) lora_score_kernel(Dims D, int rank, const float* A, const float* AG, int fm,
                                                         int bm, int unit, int n_units, double* fo, double* bo) {
  const int lh = blockIdx.x;
  const size_t per = 3 * ((size_t)D.d * rank + (size_t)rank * D.dh);
  const float* w = A + lh * per;
  const float* g = AG + lh * per;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // fisher, |w|, |g|, |w g| (Metric enum order)
  for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
    const double gv = g[i], wv = w[i];
    acc[0] += gv * gv;
    acc[1] += fabs(wv);
    acc[2] += fabs(gv);
    acc[3] += fabs(wv * gv);
  }
  __shared__ double red[4][256];
  for (int m = 0; m < 4; ++m) red[m][threadIdx.x] = acc[m];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int m = 0; m < 4; ++m) red[m][threadIdx.x] += red[m][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    fo[(size_t)lh * n_units + unit] = red[fm][0];
    bo[(size_t)lh * n_units + unit] = red[bm][0];
  }
}

}  // namespace

void launch_lora_score(const Dims& D, int rank, const float* A, const float* AG, int fwd_metric, int bwd_metric,
                       int unit, int n_units, double* fo, double* bo, cudaStream_t st) {
  lora_score_kernel<<<D.L * D.H, 256, 0, st>>>(D, rank, A, AG, fwd_metric, bwd_metric, unit, n_units, fo, bo);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_lora_merge(const Dims& D, int rank, float scaling, const float* W1T, const float* A, act_t* W1T_bf,
                       cudaStream_t st) {
  const int smem = (kLoraI * rank + rank * D.dh) * 4;
  dim3 grid((D.d + kLoraI - 1) / kLoraI, D.L * D.H * 3);
  lora_merge_kernel<<<grid, 256, smem, st>>>(D, rank, scaling, W1T, A, W1T_bf);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_lora_grad(const Dims& D, int rank, float scaling, const float* G1T, const float* A, float* AG,
                      const int* full_cnt, cudaStream_t st) {
  const int smem = (rank * D.dh + kLoraI * (D.dh + 1) + kLoraI * rank) * 4;
  static unsigned long long attr = 0;
  once_per_device(attr, [&] {
    D2FT_CUDA(cudaFuncSetAttribute(lora_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  });
  lora_grad_kernel<<<D.L * D.H * 3, 256, smem, st>>>(D, rank, scaling, G1T, A, AG, full_cnt);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace d2ft_b200
