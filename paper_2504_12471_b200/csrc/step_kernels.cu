// Non-GEMM kernels of the D2FT step for sm_100a.
#include "common.cuh"
#include "step_kernels.cuh"

namespace d2ft_b200 {

namespace {

constexpr float kLnEps = 1e-5f;  // model.hpp:32

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ codes / plan
__global__ void expand_codes_kernel(const uint8_t* codes, int K, int n_mb, int mbs, int B, int Bmax, uint8_t* out,
                                    int mb0) {
  D2FT_PDL_ENTRY();
  const size_t n = (size_t)K * Bmax;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / Bmax), s = (int)(i % Bmax);
    out[i] = s < B ? codes[(size_t)k * n_mb + mb0 + s / mbs] : (uint8_t)3;
  }
}

// data parallel: Full cells per row over the whole batch's table (K x n_mb)
__global__ void row_full_count_kernel(const uint8_t* codes, int n_mb, int* out) {
  const int k = blockIdx.x;
  int c = 0;
  for (int i = threadIdx.x; i < n_mb; i += blockDim.x) c += codes[(size_t)k * n_mb + i] == 1;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    out[k] = t;
  }
}

// data parallel: a head-subnet with no Full cell among THIS rank's samples
// gets no gradient writes from this rank's GEMMs (its rows keep old values);
// zero them so the all-reduce sums only real contributions.  Row k = (l, h):
// [Wq|Wk|Wv|W1]^T rows (contiguous), b1 slice, [Wo;W2]^T columns h*PO.. of
// every output row (strided), b2 slice.
__global__ void zero_untouched_kernel(Dims D, const int* full_cnt, float* G, size_t o_w1, size_t o_b1, size_t o_w2,
                                      size_t o_b2) {
  const int k = blockIdx.x;
  if (full_cnt[k] != 0) return;
  const int l = k / D.H, h = k % D.H;
  float* w1 = G + o_w1 + (size_t)k * D.PQ * D.d;
  for (size_t i = threadIdx.x; i < (size_t)D.PQ * D.d; i += blockDim.x) w1[i] = 0.f;
  for (int i = threadIdx.x; i < D.fs; i += blockDim.x) G[o_b1 + (size_t)k * D.fs + i] = 0.f;
  float* w2 = G + o_w2 + (size_t)l * D.d * D.H * D.PO + (size_t)h * D.PO;
  for (size_t i = threadIdx.x; i < (size_t)D.d * D.PO; i += blockDim.x)
    w2[(i / D.PO) * D.H * D.PO + i % D.PO] = 0.f;
  for (int i = threadIdx.x; i < D.d / D.H; i += blockDim.x) G[o_b2 + (size_t)l * D.d + h * (D.d / D.H) + i] = 0.f;
}

// rank of v[i] in decreasing order, ties by index (a stable counting rank)
__device__ __forceinline__ int desc_rank(const int* v, int n, int i) {
  const int x = v[i];
  int r = 0;
  for (int j = 0; j < n; ++j) r += (v[j] > x) | ((v[j] == x) & (j < i));
  return r;
}
// the same within i's sample chunk [c*n/C, (c+1)*n/C) (exchange chunks of a
// head partition): position = chunk start + rank in the chunk
__device__ __forceinline__ int desc_rank_chunked(const int* v, int n, int chunks, int i) {
  if (chunks <= 1) return desc_rank(v, n, i);
  int lo = 0, hi = n;
  for (int c = 0; c < chunks; ++c) {
    const int a = (int)((long long)c * n / chunks), b = (int)((long long)(c + 1) * n / chunks);
    if (i >= a && i < b) lo = a, hi = b;
  }
  return lo + desc_rank(v + lo, hi - lo, i - lo);
}

__global__ void plan_kernel(Dims D, const int* act_cnt, const int* full_hcnt, const int* full_cnt, Plan pl) {
  D2FT_PDL_ENTRY();
  const int l = blockIdx.x;
  __shared__ int s1[1024], s4[1024], va[1024], vf[1024], sa[1024], sf[1024], vh[64];
  int c1 = 0, c4 = 0;
  const int s = threadIdx.x;
  if (s < D.B) {
    va[s] = act_cnt[s * D.L + l];
    vf[s] = full_hcnt[s * D.L + l];
    c1 = (D.UQ * va[s] + 3) / 4;  // slots of 4 units (2 per CTA of the pair)
    c4 = (D.UO * vf[s] + 3) / 4;
  }
  if (s < D.H) vh[s] = full_cnt[l * D.H + s];
  s1[threadIdx.x] = c1;
  s4[threadIdx.x] = c4;
  sa[threadIdx.x] = s < D.B ? va[s] : 0;
  sf[threadIdx.x] = s < D.B ? vf[s] : 0;
  __syncthreads();
  // cost orders of the dynamically scheduled GEMMs: samples by active / Full
  // head count (G3, G8), heads by Full sample count (G5, G7), largest first
  if (s < D.B) {
    pl.ord_act[l * D.Bmax + desc_rank_chunked(va, D.B, pl.chunks, s)] = s;
    pl.ord_full[l * D.Bmax + desc_rank_chunked(vf, D.B, pl.chunks, s)] = s;
  }
  if (s < D.H) pl.ord_head[l * D.H + desc_rank(vh, D.H, s)] = s;
  for (int o = 1; o < blockDim.x; o <<= 1) {  // inclusive Hillis-Steele scans
    int a1 = 0, a4 = 0, aa = 0, af = 0;
    if ((int)threadIdx.x >= o) {
      a1 = s1[threadIdx.x - o];
      a4 = s4[threadIdx.x - o];
      aa = sa[threadIdx.x - o];
      af = sf[threadIdx.x - o];
    }
    __syncthreads();
    s1[threadIdx.x] += a1;
    s4[threadIdx.x] += a4;
    sa[threadIdx.x] += aa;
    sf[threadIdx.x] += af;
    __syncthreads();
  }
  const size_t cap = (size_t)D.Bmax * ((D.UQ * D.H + 1) / 2);
  const size_t cap4 = (size_t)D.Bmax * ((D.UO * D.H + 1) / 2);
  if (s < D.B) {
    const int b1 = s1[s] - c1, b4 = s4[s] - c4;
    for (int i = 0; i < c1; ++i) pl.g1_tiles[l * cap + b1 + i] = (s << 16) | (4 * i);
    for (int i = 0; i < c4; ++i) pl.g4_tiles[l * cap4 + b4 + i] = (s << 16) | (4 * i);
    // attention work items (sample, active / Full head slot) in sample order
    const size_t capa = (size_t)D.Bmax * D.H;
    for (int a = 0, b = sa[s] - va[s]; a < va[s]; ++a) pl.af_items[l * capa + b + a] = (s << 8) | a;
    for (int a = 0, b = sf[s] - vf[s]; a < vf[s]; ++a) pl.ab_items[l * capa + b + a] = (s << 8) | a;
  }
  if (threadIdx.x == blockDim.x - 1) {
    pl.g1_count[l] = s1[threadIdx.x];
    pl.g4_count[l] = s4[threadIdx.x];
    pl.af_count[l] = sa[threadIdx.x];
    pl.ab_count[l] = sf[threadIdx.x];
  }
}

// ------------------------------------------------------------------ row-tile kernels
// One CTA = 32 tokens of one sample, 8 warps, warp per row.  Shared tile
// [32][d+2] act_t (odd word pitch: conflict-free transposed reads).

__device__ __forceinline__ void write_transposed(const act_t* tile, int pitch, int d, int t0, int TP, act_t* outT) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (t0 + lane >= TP) return;
  for (int m = warp; m < d; m += 8) outT[(size_t)m * TP + t0 + lane] = tile[lane * pitch + m];
}

template <int NV>
__global__ void prep_input_kernel(Dims D, const float* x, act_t* inp, act_t* inpT) {
  D2FT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem[];
  act_t* tile = reinterpret_cast<act_t*>(smem);
  const int pitch = D.d + 2;
  const int s = blockIdx.y, t0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < 32; r += 8) {
    const int t = t0 + r;
    float v[NV];  // the row's loads all in flight before any use
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = t < D.T ? x[((size_t)s * D.T + t) * D.d + lane + 32 * j] : 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const act_t b = to_act(v[j]);
      tile[r * pitch + lane + 32 * j] = b;
      if (t < D.T) inp[((size_t)s * D.T + t) * D.d + lane + 32 * j] = b;
    }
  }
  __syncthreads();
  write_transposed(tile, pitch, D.d, t0, D.TP, inpT + (size_t)s * D.d * D.TP);
}

// Vectorised row access: lane handles elements 4*lane + 128*q + e (q < NV/4,
// e < 4): 16-byte fp32 / 8-byte fp16 accesses, 512 contiguous bytes per warp
// instruction.
__device__ __forceinline__ void ld4(const float* p, float* v) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
}
__device__ __forceinline__ void ld4h(const act_t* p, float* v) {
  const uint2 t = *reinterpret_cast<const uint2*>(p);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&t.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&t.y));
  v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}
__device__ __forceinline__ void st4h(act_t* p, float a, float b, float c, float d) {
  const __half2 x = __floats2half2_rn(a, b), y = __floats2half2_rn(c, d);
  uint2 t;
  t.x = *reinterpret_cast<const uint32_t*>(&x);
  t.y = *reinterpret_cast<const uint32_t*>(&y);
  *reinterpret_cast<uint2*>(p) = t;
}

template <int NV>
__global__ void __launch_bounds__(512) ln_fwd_kernel(Dims D, const float* x, act_t* xn, float* stats, int s0) {
  D2FT_PDL_ENTRY();
  const int s = s0 + blockIdx.y, t0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NQ = NV / 4;
  for (int r = warp; r < 32; r += blockDim.x >> 5) {
    const int t = t0 + r;
    if (t >= D.T) continue;
    const size_t ro = ((size_t)s * D.T + t) * D.d + 4 * lane;
    float v[NV];
#pragma unroll
    for (int q = 0; q < NQ; ++q) ld4(x + ro + 128 * q, v + 4 * q);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) sum += v[j];
    const float mean = warp_sum(sum) / D.d;  // linalg.cpp:136-139, two-pass
    float sq = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float dv = v[j] - mean;
      sq += dv * dv;
    }
    const float var = warp_sum(sq) / D.d;
    const float rstd = 1.0f / sqrtf(var + kLnEps);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      st4h(xn + ro + 128 * q, (v[4 * q] - mean) * rstd, (v[4 * q + 1] - mean) * rstd, (v[4 * q + 2] - mean) * rstd,
           (v[4 * q + 3] - mean) * rstd);
    if (lane == 0) {
      stats[((size_t)s * D.T + t) * 2] = mean;
      stats[((size_t)s * D.T + t) * 2 + 1] = rstd;
    }
  }
}

constexpr int kLnbWarps = 16;  // LN backward: 32 tokens per CTA, 2 rows per warp
template <int NV>
__global__ void __launch_bounds__(32 * kLnbWarps) ln_bwd_prep_kernel(Dims D, int l, const int* full_hcnt, const float* x_l, const act_t* xn_l,
                                   const float* stats_l, const float* dxn, const act_t* dxn_h, float* dX, act_t* dC,
                                   float* part_cs, const float* gmax, int s0) {
  D2FT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem[];
  float* cs = reinterpret_cast<float*>(smem);  // [kLnbWarps][d] per-warp column sums
  const int s = s0 + blockIdx.y, t0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NQ = NV / 4;
  const bool do_ln = l >= 0 && full_hcnt[s * D.L + l] > 0;  // model.cpp:508
  const float S = grad_scale(gmax);  // fp16 gradient operands carry S
  const float iS = 1.f / S;
  float* csw = cs + warp * D.d + 4 * lane;
#pragma unroll
  for (int q = 0; q < NQ; ++q) *reinterpret_cast<float4*>(csw + 128 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int r = warp; r < 32; r += kLnbWarps) {
    const int t = t0 + r;
    if (t >= D.T) continue;
    const size_t ro = ((size_t)s * D.T + t) * D.d + 4 * lane;
    float v[NV];
#pragma unroll
    for (int q = 0; q < NQ; ++q) ld4(dX + ro + 128 * q, v + 4 * q);
    if (do_ln) {  // linalg.cpp:153-180
      const float mean = stats_l[((size_t)s * D.T + t) * 2], rstd = stats_l[((size_t)s * D.T + t) * 2 + 1];
      float y[NV], dy[NV];
      // fp16 inputs (single engine): y = the stored LN output, dxn in S units
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (xn_l) {
          ld4h(xn_l + ro + 128 * q, y + 4 * q);
        } else {
          ld4(x_l + ro + 128 * q, y + 4 * q);
#pragma unroll
          for (int e = 0; e < 4; ++e) y[4 * q + e] = (y[4 * q + e] - mean) * rstd;
        }
        if (dxn_h) {
          ld4h(dxn_h + ro + 128 * q, dy + 4 * q);
#pragma unroll
          for (int e = 0; e < 4; ++e) dy[4 * q + e] *= iS;
        } else {
          ld4(dxn + ro + 128 * q, dy + 4 * q);
        }
      }
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        s1 += dy[j];
        s2 += dy[j] * y[j];
      }
      const float dmean = warp_sum(s1) / D.d, ddot = warp_sum(s2) / D.d;
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] += (dy[j] - dmean - y[j] * ddot) * rstd;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        *reinterpret_cast<float4*>(dX + ro + 128 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      st4h(dC + ro + 128 * q, v[4 * q] * S, v[4 * q + 1] * S, v[4 * q + 2] * S, v[4 * q + 3] * S);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float4 c = *reinterpret_cast<float4*>(csw + 128 * q);
      c.x += v[4 * q], c.y += v[4 * q + 1], c.z += v[4 * q + 2], c.w += v[4 * q + 3];
      *reinterpret_cast<float4*>(csw + 128 * q) = c;
    }
  }
  __syncthreads();
  const int ntile = (D.T + 31) / 32;
  for (int m = threadIdx.x; m < D.d; m += blockDim.x) {
    float c = 0.f;
    for (int w = 0; w < kLnbWarps; ++w) c += cs[w * D.d + m];
    part_cs[((size_t)s * ntile + blockIdx.x) * D.d + m] = c;
  }
}

// ------------------------------------------------------------------ head
// LN -> mean over tokens -> linear -> cross-entropy (model.cpp:342-355,
// 400-414, 470-492); backward to dX = dL/dx_L.  One CTA per sample.
// 4-CTA cluster per sample: each CTA takes a quarter of the tokens; the
// partial pooled sums meet over DSMEM (fixed rank order, identical in every
// CTA), every CTA redoes the tiny classifier + CE, and backpropagates its own
// tokens.  One CTA per sample kept only 64 of 148 SMs busy.
constexpr int kHeadCluster = 4;
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int NV>
__global__ void __launch_bounds__(256, 2) head_kernel(Dims D, const float* xL, const int* labels, const float* Wc,
                                                   const float* bc, float scale, double* loss_s, float* pooled_out,
                                                   float* dlog_out, float* dX, float* gmax, float* logits_out) {
  D2FT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem[];
  const int nw = blockDim.x >> 5;
  float* part = reinterpret_cast<float*>(smem);  // [nw][d]
  float* ppart = part + nw * D.d;                // [d] this CTA's pooled partial (read by the peers)
  float* pooled = ppart + D.d;                   // [d]
  float* dpooled = pooled + D.d;                 // [d]
  float* rowstat = dpooled + D.d;                // [T][2]
  __shared__ float logits[64], dlog[64];
  __shared__ double ex[64];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int s = blockIdx.x / kHeadCluster;
  const int tq = (D.T + kHeadCluster - 1) / kHeadCluster;
  const int ta = rank * tq, tb = min(D.T, ta + tq);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nv = NV;
  float acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.f;
  for (int t = ta + warp; t < tb; t += nw) {
    const float* row = xL + ((size_t)s * D.T + t) * D.d;
    float v[NV];
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (j < nv) {
        v[j] = row[lane + 32 * j];
        sum += v[j];
      }
    const float mean = warp_sum(sum) / D.d;
    float sq = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (j < nv) sq += (v[j] - mean) * (v[j] - mean);
    const float rstd = 1.0f / sqrtf(warp_sum(sq) / D.d + kLnEps);
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (j < nv) acc[j] += (v[j] - mean) * rstd;
    if (lane == 0) {
      rowstat[2 * t] = mean;
      rowstat[2 * t + 1] = rstd;
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (j < nv) part[warp * D.d + lane + 32 * j] = acc[j];
  __syncthreads();
  for (int m = threadIdx.x; m < D.d; m += blockDim.x) {
    float p = 0.f;
    for (int w = 0; w < nw; ++w) p += part[w * D.d + m];
    ppart[m] = p;
  }
  cluster_barrier();  // every CTA's partial is complete
  for (int m = threadIdx.x; m < D.d; m += blockDim.x) {
    float p = 0.f;
    for (int r = 0; r < kHeadCluster; ++r) p += ld_cluster_f32(cluster_addr(ppart + m, r));
    pooled[m] = p / D.T;  // row_mean (linalg.cpp:101-105)
    if (rank == 0) pooled_out[(size_t)s * D.d + m] = pooled[m];
  }
  cluster_barrier();  // peers' partials read: they may proceed (and exit)
  for (int c = warp; c < D.C; c += nw) {
    float z = 0.f;
    for (int m = lane; m < D.d; m += 32) z += pooled[m] * Wc[(size_t)m * D.C + c];
    z = warp_sum(z);
    if (lane == 0) {
      logits[c] = z + bc[c];
      if (rank == 0) logits_out[(size_t)s * D.C + c] = logits[c];  // SubnetModel::logits (evaluate)
    }
  }
  __syncthreads();
  if (warp == 0) {  // cross_entropy, model.cpp:400-414 (fp64 reduction)
    // the exps on the lanes, the sum serially in class order (lane 0)
    double mx = -INFINITY;
    for (int c = lane; c < D.C; c += 32) mx = fmax(mx, (double)logits[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int c = lane; c < D.C; c += 32) ex[c] = exp((double)logits[c] - mx);
    __syncwarp();
    double sum = 0.0;
    if (lane == 0) {
      for (int c = 0; c < D.C; ++c) sum += ex[c];
      if (rank == 0) loss_s[s] = log(sum) - ((double)logits[labels[s]] - mx);
    }
    sum = __shfl_sync(0xffffffffu, sum, 0);
    const int lab = labels[s];
    for (int c = lane; c < D.C; c += 32) {
      double p = ex[c] / sum;
      if (c == lab) p -= 1.0;
      dlog[c] = (float)(p * scale);
      if (rank == 0) dlog_out[(size_t)s * D.C + c] = dlog[c];
    }
  }
  __syncthreads();
  for (int m = threadIdx.x; m < D.d; m += blockDim.x) {
    float z = 0.f;
    for (int c = 0; c < D.C; ++c) z += dlog[c] * Wc[(size_t)m * D.C + c];
    dpooled[m] = z / D.T;  // dxn_h = dpooled / T (model.cpp:489-491)
  }
  __syncthreads();
  float dmean_l = 0.f;
  for (int m = lane; m < D.d; m += 32) dmean_l += dpooled[m];
  const float dmean = warp_sum(dmean_l) / D.d;
  for (int t = ta + warp; t < tb; t += nw) {
    const size_t ro = ((size_t)s * D.T + t) * D.d;
    const float mean = rowstat[2 * t], rstd = rowstat[2 * t + 1];
    float y[NV];
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (j < nv) {
        y[j] = (xL[ro + lane + 32 * j] - mean) * rstd;
        s2 += dpooled[lane + 32 * j] * y[j];
      }
    const float ddot = warp_sum(s2) / D.d;
    float amax = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (j < nv) {
        const float g = (dpooled[lane + 32 * j] - dmean - y[j] * ddot) * rstd;
        dX[ro + lane + 32 * j] = g;
        amax = fmaxf(amax, fabsf(g));
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) atomicMax(reinterpret_cast<unsigned int*>(gmax), __float_as_uint(amax));  // >= 0: int order
  }
}

// warp per output: lanes split the samples (fixed order: lane partials, then
// a shuffle tree), so the B-long reductions run 32-wide
__global__ void head_reduce_kernel(Dims D, const double* loss_s, const float* pooled, const float* dlog, float* dWc,
                                   float* dbc, double* loss, int loss_div) {
  D2FT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i < D.d * D.C) {
    const int m = i / D.C, c = i % D.C;
    float a = 0.f;
    for (int s = lane; s < D.B; s += 32) a += pooled[(size_t)s * D.d + m] * dlog[(size_t)s * D.C + c];
    a = warp_sum(a);
    if (lane == 0) dWc[i] = a;
  } else if (i < D.d * D.C + D.C) {
    const int c = i - D.d * D.C;
    float a = 0.f;
    for (int s = lane; s < D.B; s += 32) a += dlog[(size_t)s * D.C + c];
    a = warp_sum(a);
    if (lane == 0) dbc[c] = a;
  } else if (i == D.d * D.C + D.C && lane == 0) {
    double a = 0.0;
    for (int s = 0; s < D.B; ++s) a += loss_s[s];
    *loss = a / loss_div;  // batch loss = sum of CE / B (this rank's share under data parallelism)
  }
}

// ------------------------------------------------------------------ bias / embed reductions
// db2 (model.cpp:250-252) and db1 (model.cpp:257) of block l: sums over the
// Full samples of each head.  32 outputs per CTA (lane), samples split over
// the 8 warps, warp partials combined in fixed order (deterministic).
// 32 outputs per CTA, 32 warps striding over the samples (fixed order: warp
// partials then lanes' sum over warps), so the per-layer reduction runs at
// full memory parallelism despite only (d + H*fs)/32 CTAs.
// db2 / db1 of every block in one launch (blockIdx.y = block): fixed-order
// sums over the Full samples of each head of the per-tile column sums of the
// incoming gradient (model.cpp:250-252) and of G4's per-column-group db1
// partials (model.cpp:257).
__global__ void __launch_bounds__(1024) bias_reduce_kernel(Dims D, const uint8_t* codes, const float* part_cs,
                                                           const float* part_db1, float* db1, float* db2) {
  D2FT_PDL_ENTRY();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = blockIdx.y;
  const int i = blockIdx.x * 32 + lane;
  const int ntile = (D.T + 31) / 32;
  const int nout = D.d + D.H * D.fs;
  const float* pcs = part_cs + (size_t)l * D.Bmax * ntile * D.d;
  const float* pdb = part_db1 + (size_t)l * kG4Epi * D.Bmax * D.H * D.fs;
  float a = 0.f;
  if (i < nout) {
    if (i < D.d) {
      const int m = i, h = m / (D.d / D.H);
      const uint8_t* row = codes + (size_t)(l * D.H + h) * D.Bmax;
      for (int s = warp; s < D.B; s += 32)
        if (row[s] == 1) {
#pragma unroll 4
          for (int tt = 0; tt < ntile; ++tt) a += pcs[((size_t)s * ntile + tt) * D.d + m];
        }
    } else {
      const int q = i - D.d, h = q / D.fs, j = q % D.fs;
      const uint8_t* row = codes + (size_t)(l * D.H + h) * D.Bmax;
      for (int s = warp; s < D.B; s += 32)
        if (row[s] == 1)
#pragma unroll
          for (int e = 0; e < kG4Epi; ++e) a += pdb[(((size_t)e * D.Bmax + s) * D.H + h) * D.fs + j];
    }
  }
  red[warp][lane] = a;
  __syncthreads();
  if (warp == 0 && i < nout) {
    float t = 0.f;
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    if (i < D.d) db2[(size_t)l * D.d + i] = t;
    else db1[(size_t)l * D.H * D.fs + (i - D.d)] = t;
  }
}

__global__ void embed_reduce_kernel(Dims D, int KS, const float* part, const float* part_cs, const float* dX,
                                    float* dWeT, float* dbe, float* dpos) {
  D2FT_PDL_ENTRY();
  const size_t dd = (size_t)D.d * D.d;
  const size_t td = (size_t)D.T * D.d;
  const int ntile = (D.T + 31) / 32;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < dd + td;
       i += (size_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    if (i < dd) {  // dW_embed (model.cpp:514), sum of the split-K partials
#pragma unroll 8
      for (int k = 0; k < KS; ++k) a += part[k * dd + i];
      dWeT[i] = a;
    } else if (i < dd + td) {  // dpos (model.cpp:516)
      const size_t q = i - dd;
#pragma unroll 8
      for (int s = 0; s < D.B; ++s) a += dX[(size_t)s * td + q];
      dpos[q] = a;
    }
  }
}

// out[c] = sum_r in[r][c]: 32 columns per CTA, 32 warps striding the rows,
// fixed-order combine (deterministic).  db_embed (model.cpp:515) from the
// per-tile column sums of the LN-backward kernel.
__global__ void __launch_bounds__(1024) colsum_kernel(const float* in, int rows, int cols, float* out) {
  D2FT_PDL_ENTRY();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float a = 0.f;
  if (c < cols)
    for (int r = warp; r < rows; r += 32) a += in[(size_t)r * cols + c];
  red[warp][lane] = a;
  __syncthreads();
  if (warp == 0 && c < cols) {
    float t = 0.f;
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    out[c] = t;
  }
}

// ------------------------------------------------------------------ SGD / copies
__global__ void sgd_kernel(float* p, float* v, const float* g, act_t* pbf, size_t n, long long outer, long long inner,
                           int H, const int* full_cnt, float lr, float mom, int* err) {
  D2FT_PDL_ENTRY();
  // 4 consecutive elements per thread (every segment's `inner` is a multiple of 4)
  const size_t n4 = n / 4;
  for (size_t i4 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i4 < n4 + (n % 4 ? 1 : 0);
       i4 += (size_t)gridDim.x * blockDim.x) {
    const size_t i = i4 * 4;
    if (outer > 0 && full_cnt) {
      const long long k = ((long long)i / outer) * H + ((long long)i / inner) % H;
      if (full_cnt[k] == 0) continue;  // trainer.cpp:264-268: untouched subnets keep p and v
    }
    if (i + 4 <= n) {
      const float4 gi = *reinterpret_cast<const float4*>(g + i);
      float4 vi = *reinterpret_cast<const float4*>(v + i);
      float4 pi = *reinterpret_cast<const float4*>(p + i);
      if (!isfinite(gi.x) || !isfinite(gi.y) || !isfinite(gi.z) || !isfinite(gi.w)) {
        atomicCAS(err, 0, (int)kNumeric);  // trainer.cpp:118
        continue;
      }
      vi.x = mom * vi.x + gi.x;  // trainer.cpp:119-120
      vi.y = mom * vi.y + gi.y;
      vi.z = mom * vi.z + gi.z;
      vi.w = mom * vi.w + gi.w;
      pi.x -= lr * vi.x;
      pi.y -= lr * vi.y;
      pi.z -= lr * vi.z;
      pi.w -= lr * vi.w;
      *reinterpret_cast<float4*>(v + i) = vi;
      *reinterpret_cast<float4*>(p + i) = pi;
      if (pbf) {
        __align__(8) __half2 h[2] = {__floats2half2_rn(pi.x, pi.y), __floats2half2_rn(pi.z, pi.w)};
        *reinterpret_cast<uint2*>(pbf + i) = *reinterpret_cast<const uint2*>(h);
      }
    } else {
      for (size_t j = i; j < n; ++j) {
        const float gi = g[j];
        if (!isfinite(gi)) {
          atomicCAS(err, 0, (int)kNumeric);
          continue;
        }
        const float vi = mom * v[j] + gi;
        v[j] = vi;
        p[j] -= lr * vi;
        if (pbf) pbf[j] = to_act(p[j]);
      }
    }
  }
}

// Dataset::samples (fp64 Matrix, data.hpp:18-20) -> the engine's fp32 input:
// the batch's samples arrive H2D as fp64 in batch order; two doubles per thread
// per iteration (n is even: every sample is T x d with d a multiple of 128).
__global__ void f64_to_f32_kernel(const double2* __restrict__ in, float2* __restrict__ out, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(in + i);
    out[i] = make_float2((float)v.x, (float)v.y);
  }
}

__global__ void f32_to_bf16_kernel(const float* in, act_t* out, size_t n) {
  D2FT_PDL_ENTRY();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = to_act(in[i]);
}

// ------------------------------------------------------------------ attention (mma.sync, FA2 style)
// One CTA per (sample, head) slot, one warp per 16-row strip.  q, k, v, dO are
// fp16 (G1 / G4 epilogues), staged with cp.async (zero-filled past T) into
// row-major shared tiles with a 16-byte pad (conflict-free ldmatrix); A and B
// fragments come from ldmatrix / ldmatrix.trans, so no transposed copies.
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
// A (16x16) at (r0, k0) of row-major X[row][k], pitch P halves
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const act_t* X, int P, int r0, int k0, int lane) {
  ldsm_x4(a, X + (size_t)(r0 + (lane & 15)) * P + k0 + (lane >> 4) * 8);
}
// B for two n8 tiles (n0, n0+8) x k16 from n-major Y[n][k]: {b0,b1} of n0, {b0,b1} of n0+8
__device__ __forceinline__ void frag_b_n(uint32_t (&b)[4], const act_t* Y, int P, int n0, int k0, int lane) {
  ldsm_x4(b, Y + (size_t)(n0 + (lane & 7) + ((lane >> 4) << 3)) * P + k0 + ((lane >> 3) & 1) * 8);
}
// B for two n8 tiles x k16 from k-major X[k][n] (transposed load)
__device__ __forceinline__ void frag_b_k(uint32_t (&b)[4], const act_t* X, int P, int n0, int k0, int lane) {
  ldsm_x4_t(b, X + (size_t)(k0 + (lane & 7) + (((lane >> 3) & 1) << 3)) * P + n0 + (lane >> 4) * 8);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// rows [0,TQ) of cols [off, off+DH) of a [T][pitch] fp16 slice -> smem [TQ][DH+8]
template <int DH>
__device__ void stage_rows(const act_t* g, int pitch, int off, int T, int TQ, act_t* dst) {
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < TQ * CH; i += blockDim.x) {
    const int t = i / CH, c = i % CH;
    const bool v = t < T;
    cp_async16(dst + t * (DH + 8) + c * 8, g + (size_t)(v ? t : 0) * pitch + off + c * 8, v);
  }
}
// Scalar feature-major stores of a 16 x DH fragment block: outT[f][t0 + row]
template <int DH>
__device__ __forceinline__ void store_frag_T(const float (&o)[DH / 8][4], float sc, act_t* outT, int TP, int t0,
                                             int T, int g, int c) {
  const int ta = t0 + g, tb = t0 + g + 8;
#pragma unroll
  for (int nf = 0; nf < DH / 8; ++nf) {
    const int f = nf * 8 + 2 * c;
    if (ta < T) {
      outT[(size_t)f * TP + ta] = __float2half_rn(o[nf][0] * sc);
      outT[(size_t)(f + 1) * TP + ta] = __float2half_rn(o[nf][1] * sc);
    }
    if (tb < T) {
      outT[(size_t)f * TP + tb] = __float2half_rn(o[nf][2] * sc);
      outT[(size_t)(f + 1) * TP + tb] = __float2half_rn(o[nf][3] * sc);
    }
  }
}

// Forward: one warp per 16-query strip (blockDim = 32 * TQ/16), online softmax
// over 32-key chunks.
// MINB = 2: two CTAs per SM (T <= 208, 416 threads, <= 72 registers)
template <int DH, int MINB>
__global__ void __launch_bounds__(MINB == 2 ? 416 : 512, MINB) attn_fwd_kernel(Dims D, int l, const int* act_heads, const int* act_cnt,
                                                       const act_t* QKV, act_t* OGT, float* lse) {
  D2FT_PDL_ENTRY();
  const int s = blockIdx.y, a = blockIdx.x;
  if (s >= D.B || a >= act_cnt[s * D.L + l]) return;
  const int h = act_heads[(s * D.L + l) * D.H + a];
  extern __shared__ __align__(16) unsigned char smem[];
  const int TQ = D.TQ;
  constexpr int P = DH + 8;
  act_t* Qs = reinterpret_cast<act_t*>(smem);  // [TQ][P]
  act_t* Ks = Qs + TQ * P;
  act_t* Vs = Ks + TQ * P;
  const size_t sh = (size_t)s * D.H + h;
  const act_t* y = QKV + sh * D.T * (3 * DH);
  stage_rows<DH>(y, 3 * DH, 0, D.T, TQ, Qs);
  stage_rows<DH>(y, 3 * DH, DH, D.T, TQ, Ks);
  stage_rows<DH>(y, 3 * DH, 2 * DH, D.T, TQ, Vs);
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, c = lane & 3;
  const float sl2 = kLog2e / sqrtf((float)DH);  // 1/sqrt(dh) (model.cpp:213) in log2 units
  const int r0 = warp * 16;
  uint32_t qa[DH / 16][4];
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) frag_a(qa[ks], Qs, P, r0, ks * 16, lane);
  float o[DH / 8][4];
#pragma unroll
  for (int nf = 0; nf < DH / 8; ++nf) o[nf][0] = o[nf][1] = o[nf][2] = o[nf][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  for (int kc = 0; kc < TQ; kc += 32) {
    float sc[4][4];
#pragma unroll
    for (int np = 0; np < 2; ++np) {
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[2 * np][e] = sc[2 * np + 1][e] = 0.f;
      if (kc + np * 16 < TQ) {
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) {
          uint32_t b[4];
          frag_b_n(b, Ks, P, kc + np * 16, ks * 16, lane);
          mma16816(sc[2 * np], qa[ks], b[0], b[1]);
          mma16816(sc[2 * np + 1], qa[ks], b[2], b[3]);
        }
      }
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int key = kc + nt * 8 + 2 * c;
      sc[nt][0] = key < D.T ? sc[nt][0] * sl2 : -INFINITY;
      sc[nt][1] = key + 1 < D.T ? sc[nt][1] * sl2 : -INFINITY;
      sc[nt][2] = key < D.T ? sc[nt][2] * sl2 : -INFINITY;
      sc[nt][3] = key + 1 < D.T ? sc[nt][3] * sl2 : -INFINITY;
    }
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float cr0 = m0 == -INFINITY ? 0.f : exp2f(m0 - mx0);
    const float cr1 = m1 == -INFINITY ? 0.f : exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    l0 *= cr0;
    l1 *= cr1;
#pragma unroll
    for (int nf = 0; nf < DH / 8; ++nf) {
      o[nf][0] *= cr0;
      o[nf][1] *= cr0;
      o[nf][2] *= cr1;
      o[nf][3] *= cr1;
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      sc[nt][0] = exp2f(sc[nt][0] - m0);
      sc[nt][1] = exp2f(sc[nt][1] - m0);
      sc[nt][2] = exp2f(sc[nt][2] - m1);
      sc[nt][3] = exp2f(sc[nt][3] - m1);
      l0 += sc[nt][0] + sc[nt][1];
      l1 += sc[nt][2] + sc[nt][3];
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (kc + j * 16 < TQ) {
        uint32_t pa[4] = {pack2(sc[2 * j][0], sc[2 * j][1]), pack2(sc[2 * j][2], sc[2 * j][3]),
                          pack2(sc[2 * j + 1][0], sc[2 * j + 1][1]), pack2(sc[2 * j + 1][2], sc[2 * j + 1][3])};
#pragma unroll
        for (int nf = 0; nf < DH / 8; nf += 2) {
          uint32_t b[4];
          frag_b_k(b, Vs, P, nf * 8, kc + j * 16, lane);
          mma16816(o[nf], pa, b[0], b[1]);
          mma16816(o[nf + 1], pa, b[2], b[3]);
        }
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
  for (int nf = 0; nf < DH / 8; ++nf) {
    o[nf][0] *= i0;
    o[nf][1] *= i0;
    o[nf][2] *= i1;
    o[nf][3] *= i1;
  }
  store_frag_T<DH>(o, 1.f, OGT + sh * D.PO * D.TP, D.TP, r0, D.T, g, c);
  if (c == 0) {  // log2-domain log-sum-exp of the scaled scores
    if (r0 + g < D.T) lse[sh * D.T + r0 + g] = m0 + log2f(l0);
    if (r0 + g + 8 < D.T) lse[sh * D.T + r0 + g + 8] = m1 + log2f(l1);
  }
}

// A fragment (16x16 at (i0, k0)) of A[i][k] held transposed as X[k][i]
__device__ __forceinline__ void frag_a_t(uint32_t (&a)[4], const act_t* X, int P, int i0, int k0, int lane) {
  ldsm_x4_t(a, X + (size_t)(k0 + (lane & 7) + ((lane >> 4) << 3)) * P + i0 + ((lane >> 3) & 1) * 8);
}

// Backward (model.cpp:262-271), FA2 order, deterministic.  D_i = rowsum(dO.O)
// (fp16 O; == rowdot(P, dP) of softmax_rows_backward, linalg.cpp:118-128).
// Phase 1, one warp per 16-key strip: S^T, P^T, dP^T, dS^T -> dV, dK, and
// dS^T kept in shared memory; phase 2, one warp per 16-query strip: dQ = dS.K.
template <int DH>
__global__ void __launch_bounds__(512) attn_bwd_kernel(Dims D, int l, const int* full_heads, const int* full_hcnt,
                                                       const act_t* QKV, const act_t* OGT, const act_t* dO,
                                                       const float* lse, act_t* dY1T) {
  D2FT_PDL_ENTRY();
  const int s = blockIdx.y, a = blockIdx.x;
  if (s >= D.B || a >= full_hcnt[s * D.L + l]) return;
  const int h = full_heads[(s * D.L + l) * D.H + a];
  extern __shared__ __align__(16) unsigned char smem[];
  const int TQ = D.TQ;
  constexpr int P = DH + 8;
  const int PS = TQ + 8;
  act_t* Qs = reinterpret_cast<act_t*>(smem);
  act_t* Ks = Qs + TQ * P;
  act_t* Vs = Ks + TQ * P;
  act_t* dOs = Vs + TQ * P;
  act_t* dST = dOs + TQ * P;  // [TQ keys][TQ+8 queries]
  float* Dv = reinterpret_cast<float*>(dST + TQ * PS);
  float* L2 = Dv + TQ;
  const size_t sh = (size_t)s * D.H + h;
  const act_t* y = QKV + sh * D.T * (3 * DH);
  stage_rows<DH>(y, 3 * DH, 0, D.T, TQ, Qs);
  stage_rows<DH>(y, 3 * DH, DH, D.T, TQ, Ks);
  stage_rows<DH>(y, 3 * DH, 2 * DH, D.T, TQ, Vs);
  stage_rows<DH>(dO + sh * D.T * D.dh, D.dh, 0, D.T, TQ, dOs);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, c = lane & 3;
  // D_i and L2_i per query row (rows >= T: D = 0, L2 = +inf -> P = 0); O is
  // read feature-major from OGT (coalesced over t), dO row-wise (16-byte loads)
  for (int t = threadIdx.x; t < TQ; t += blockDim.x) {
    float acc = 0.f;
    if (t < D.T) {
      const act_t* o = OGT + sh * D.PO * D.TP + t;
      const act_t* dor = dO + (sh * D.T + t) * D.dh;
#pragma unroll
      for (int f0 = 0; f0 < DH; f0 += 8) {
        __align__(16) act_t v[8];
        *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(dor + f0);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += __half2float(v[i]) * __half2float(o[(size_t)(f0 + i) * D.TP]);
      }
    }
    Dv[t] = acc;
    L2[t] = t < D.T ? lse[sh * D.T + t] : INFINITY;
  }
  cp_async_wait_all();
  __syncthreads();
  const float sl2 = kLog2e / sqrtf((float)DH);
  const float scale = 1.0f / sqrtf((float)DH);
  act_t* dyt = dY1T + sh * D.PQ * D.TP;

  {  // ---- phase 1: key strip -> dK, dV, dS^T
    const int k0 = warp * 16;
    uint32_t ka_[DH / 16][4], va[DH / 16][4];
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      frag_a(ka_[ks], Ks, P, k0, ks * 16, lane);
      frag_a(va[ks], Vs, P, k0, ks * 16, lane);
    }
    float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
    for (int nf = 0; nf < DH / 8; ++nf)
#pragma unroll
      for (int e = 0; e < 4; ++e) dk[nf][e] = dv[nf][e] = 0.f;
    const bool key0 = k0 + g < D.T, key1 = k0 + g + 8 < D.T;
    for (int qc = 0; qc < TQ; qc += 16) {
      float st[2][4] = {}, dp[2][4] = {};
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        uint32_t b[4];
        frag_b_n(b, Qs, P, qc, ks * 16, lane);
        mma16816(st[0], ka_[ks], b[0], b[1]);
        mma16816(st[1], ka_[ks], b[2], b[3]);
        frag_b_n(b, dOs, P, qc, ks * 16, lane);
        mma16816(dp[0], va[ks], b[0], b[1]);
        mma16816(dp[1], va[ks], b[2], b[3]);
      }
      float pt[2][4], ds[2][4];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int q = qc + hh * 8 + 2 * c;
        const float l2a = L2[q], l2b = L2[q + 1], da = Dv[q], db = Dv[q + 1];
        pt[hh][0] = key0 ? exp2f(st[hh][0] * sl2 - l2a) : 0.f;
        pt[hh][1] = key0 ? exp2f(st[hh][1] * sl2 - l2b) : 0.f;
        pt[hh][2] = key1 ? exp2f(st[hh][2] * sl2 - l2a) : 0.f;
        pt[hh][3] = key1 ? exp2f(st[hh][3] * sl2 - l2b) : 0.f;
        ds[hh][0] = pt[hh][0] * (dp[hh][0] - da);
        ds[hh][1] = pt[hh][1] * (dp[hh][1] - db);
        ds[hh][2] = pt[hh][2] * (dp[hh][2] - da);
        ds[hh][3] = pt[hh][3] * (dp[hh][3] - db);
        *reinterpret_cast<uint32_t*>(dST + (size_t)(k0 + g) * PS + q) = pack2(ds[hh][0], ds[hh][1]);
        *reinterpret_cast<uint32_t*>(dST + (size_t)(k0 + g + 8) * PS + q) = pack2(ds[hh][2], ds[hh][3]);
      }
      const uint32_t pa[4] = {pack2(pt[0][0], pt[0][1]), pack2(pt[0][2], pt[0][3]), pack2(pt[1][0], pt[1][1]),
                              pack2(pt[1][2], pt[1][3])};
      const uint32_t sa[4] = {pack2(ds[0][0], ds[0][1]), pack2(ds[0][2], ds[0][3]), pack2(ds[1][0], ds[1][1]),
                              pack2(ds[1][2], ds[1][3])};
#pragma unroll
      for (int nf = 0; nf < DH / 8; nf += 2) {
        uint32_t b[4];
        frag_b_k(b, dOs, P, nf * 8, qc, lane);
        mma16816(dv[nf], pa, b[0], b[1]);
        mma16816(dv[nf + 1], pa, b[2], b[3]);
        frag_b_k(b, Qs, P, nf * 8, qc, lane);
        mma16816(dk[nf], sa, b[0], b[1]);
        mma16816(dk[nf + 1], sa, b[2], b[3]);
      }
    }
    store_frag_T<DH>(dk, scale, dyt + (size_t)DH * D.TP, D.TP, k0, D.T, g, c);
    store_frag_T<DH>(dv, 1.f, dyt + (size_t)2 * DH * D.TP, D.TP, k0, D.T, g, c);
  }
  __syncthreads();
  {  // ---- phase 2: query strip -> dQ = dS . K
    const int i0 = warp * 16;
    float dq[DH / 8][4];
#pragma unroll
    for (int nf = 0; nf < DH / 8; ++nf) dq[nf][0] = dq[nf][1] = dq[nf][2] = dq[nf][3] = 0.f;
    for (int kc = 0; kc < TQ; kc += 16) {
      uint32_t sa[4];
      frag_a_t(sa, dST, PS, i0, kc, lane);
#pragma unroll
      for (int nf = 0; nf < DH / 8; nf += 2) {
        uint32_t b[4];
        frag_b_k(b, Ks, P, nf * 8, kc, lane);
        mma16816(dq[nf], sa, b[0], b[1]);
        mma16816(dq[nf + 1], sa, b[2], b[3]);
      }
    }
    store_frag_T<DH>(dq, scale, dyt, D.TP, i0, D.T, g, c);
  }
}

size_t attn_fwd_smem(int DH, int TQ) { return (size_t)(3 * TQ * (DH + 8)) * 2; }
size_t attn_bwd_smem(int DH, int TQ) {
  return (size_t)(4 * TQ * (DH + 8) + TQ * (TQ + 8)) * 2 + (size_t)2 * TQ * 4;
}

// d = 32 * NV: instantiate the row kernels for the supported model widths
#define D2FT_NV_DISPATCH(d, ...)                                                     \
  do {                                                                              \
    switch ((d) / 32) {                                                             \
      case 4: { constexpr int NV = 4; __VA_ARGS__ } break;                          \
      case 8: { constexpr int NV = 8; __VA_ARGS__ } break;                          \
      case 16: { constexpr int NV = 16; __VA_ARGS__ } break;                        \
      case 24: { constexpr int NV = 24; __VA_ARGS__ } break;                        \
      case 32: { constexpr int NV = 32; __VA_ARGS__ } break;                        \
      default: throw Fail{kConfig, "row kernels: model_dim must be 128, 256, 512, 768 or 1024"}; \
    }                                                                               \
  } while (0)

int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

void launch_expand_codes(const uint8_t* codes, int K, int n_mb, int mbs, int B, int Bmax, uint8_t* out,
                         cudaStream_t st, int mb0) {
  expand_codes_kernel<<<grid_for((size_t)K * Bmax, 256), 256, 0, st>>>(codes, K, n_mb, mbs, B, Bmax, out, mb0);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_row_full_count(const uint8_t* codes, int K, int n_mb, int* out, cudaStream_t st) {
  row_full_count_kernel<<<K, 128, 0, st>>>(codes, n_mb, out);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_zero_untouched(const Dims& D, const int* full_cnt, float* G, size_t o_w1, size_t o_b1, size_t o_w2,
                           size_t o_b2, cudaStream_t st) {
  zero_untouched_kernel<<<D.K(), 256, 0, st>>>(D, full_cnt, G, o_w1, o_b1, o_w2, o_b2);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_plan(const Dims& D, const int* act_cnt, const int* full_hcnt, const int* full_cnt, const Plan& pl,
                 cudaStream_t st) {
  int threads = 32;
  while (threads < D.B) threads <<= 1;
  D2FT_REQUIRE(threads <= 1024, kSize, "plan: batch above 1024 samples");
  D2FT_REQUIRE(D.H <= 64, kSize, "plan: at most 64 heads");
  plan_kernel<<<D.L, threads, 0, st>>>(D, act_cnt, full_hcnt, full_cnt, pl);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

static size_t tile_smem(const Dims& D) { return (size_t)32 * (D.d + 2) * 2 + 16; }

void launch_prep_input(const Dims& D, const float* x, act_t* inp, act_t* inpT, cudaStream_t st) {
  dim3 grid((D.T + 31) / 32, D.B);
  const size_t sm = tile_smem(D);
  D2FT_NV_DISPATCH(D.d, {
    D2FT_CUDA(cudaFuncSetAttribute(prep_input_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    prep_input_kernel<NV><<<grid, 256, sm, st>>>(D, x, inp, inpT);
  });
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_ln_fwd(const Dims& D, const float* x, act_t* xn, float* stats, cudaStream_t st, int s0, int ns) {
  if (ns < 0) ns = D.B;
  if (ns == 0) return;
  dim3 grid((D.T + 31) / 32, ns);
  D2FT_NV_DISPATCH(D.d, { ln_fwd_kernel<NV><<<grid, 512, 0, st>>>(D, x, xn, stats, s0); });  // 2 rows per warp
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_ln_bwd_prep(const Dims& D, int l, const int* full_hcnt, const float* x_l, const act_t* xn_l,
                        const float* stats_l, const float* dxn, const act_t* dxn_h, float* dX, act_t* dC,
                        float* part_cs, const float* gmax, cudaStream_t st, int s0, int ns) {
  if (ns < 0) ns = D.B;
  if (ns == 0) return;
  dim3 grid((D.T + 31) / 32, ns);
  const size_t sm = (size_t)kLnbWarps * D.d * 4;
  D2FT_NV_DISPATCH(D.d, {
    D2FT_CUDA(cudaFuncSetAttribute(ln_bwd_prep_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    ln_bwd_prep_kernel<NV><<<grid, 32 * kLnbWarps, sm, st>>>(D, l, full_hcnt, x_l, xn_l, stats_l, dxn, dxn_h, dX, dC,
                                                              part_cs, gmax, s0);
  });
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_attn_fwd(const Dims& D, int l, const int* act_heads, const int* act_cnt, const act_t* Y1, act_t* OGT,
                     float* lse, cudaStream_t st) {
  dim3 grid(D.H, D.B);
  auto go = [&](auto kern, int dh) {
    const size_t sm = attn_fwd_smem(dh, D.TQ);
    D2FT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, D.TQ * 2, sm, st>>>(D, l, act_heads, act_cnt, Y1, OGT, lse);
    count_launch();
  };
  const bool two = D.TQ * 2 <= 416;
  if (D.dh == 64) {
    if (two) go(attn_fwd_kernel<64, 2>, 64);
    else go(attn_fwd_kernel<64, 1>, 64);
  } else if (D.dh == 32) {
    if (two) go(attn_fwd_kernel<32, 2>, 32);
    else go(attn_fwd_kernel<32, 1>, 32);
  } else {
    throw Fail{kConfig, "attention: head_dim must be 32 or 64"};
  }
  D2FT_CUDA(cudaGetLastError());
}

void launch_attn_bwd(const Dims& D, int l, const int* full_heads, const int* full_hcnt, const act_t* Y1,
                     const act_t* OGT, const act_t* dO, const float* lse, act_t* dY1T, cudaStream_t st) {
  dim3 grid(D.H, D.B);
  if (D.dh == 64) {
    const size_t sm = attn_bwd_smem(64, D.TQ);
    D2FT_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attn_bwd_kernel<64><<<grid, D.TQ * 2, sm, st>>>(D, l, full_heads, full_hcnt, Y1, OGT, dO, lse, dY1T);
    count_launch();
  } else if (D.dh == 32) {
    const size_t sm = attn_bwd_smem(32, D.TQ);
    D2FT_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attn_bwd_kernel<32><<<grid, D.TQ * 2, sm, st>>>(D, l, full_heads, full_hcnt, Y1, OGT, dO, lse, dY1T);
    count_launch();
  } else {
    throw Fail{kConfig, "attention: head_dim must be 32 or 64"};
  }
  D2FT_CUDA(cudaGetLastError());
}

void launch_head(const Dims& D, const float* xL, const int* labels, const float* Wc, const float* bc, float scale,
                 double* loss_s, float* pooled, float* dlog, float* dX, float* gmax, float* logits, cudaStream_t st) {
  D2FT_REQUIRE(D.C <= 64, kConfig, "head: at most 64 classes");
  // 8 warps: two CTAs per SM (registers), so the B x 4 CTAs of ViT-B run as
  // one wave (512-thread CTAs ran one per SM, 1.94 waves)
  const int threads = 256;
  const size_t sm = (size_t)((threads / 32 + 3) * D.d + 2 * D.T) * 4;
  D2FT_NV_DISPATCH(D.d, {
    D2FT_CUDA(cudaFuncSetAttribute(head_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(D.B * kHeadCluster);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kHeadCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    D2FT_CUDA(cudaLaunchKernelEx(&cfg, head_kernel<NV>, D, xL, labels, Wc, bc, scale, loss_s, pooled, dlog, dX, gmax,
                                 logits));
  });
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_head_reduce(const Dims& D, const double* loss_s, const float* pooled, const float* dlog, float* dWc,
                        float* dbc, double* loss, cudaStream_t st, int loss_div) {
  const int n = (D.d * D.C + D.C + 1) * 32;  // a warp per output
  head_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(D, loss_s, pooled, dlog, dWc, dbc, loss,
                                                      loss_div > 0 ? loss_div : D.B);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_bias_reduce(const Dims& D, const uint8_t* codes, const float* part_cs, const float* part_db1, float* db1,
                        float* db2, cudaStream_t st) {
  const int n = D.d + D.H * D.fs;
  bias_reduce_kernel<<<dim3((n + 31) / 32, D.L), 1024, 0, st>>>(D, codes, part_cs, part_db1, db1, db2);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_embed_reduce(const Dims& D, int KS, const float* part, const float* part_cs, const float* dX, float* dWeT,
                         float* dbe, float* dpos, cudaStream_t st) {
  const size_t n = (size_t)D.d * D.d + (size_t)D.T * D.d;
  embed_reduce_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(D, KS, part, part_cs, dX, dWeT, dbe, dpos);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
  colsum_kernel<<<(D.d + 31) / 32, 1024, 0, st>>>(part_cs, D.B * ((D.T + 31) / 32), D.d, dbe);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_sgd(float* p, float* v, const float* g, act_t* pbf, size_t n, long long outer, long long inner, int H,
                const int* full_cnt, float lr, float mom, int* err, cudaStream_t st) {
  if (!n) return;
  sgd_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, st>>>(p, v, g, pbf, n, outer, inner, H, full_cnt, lr, mom, err);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}


void launch_f64_to_f32(const double* in, float* out, size_t n, cudaStream_t st) {
  f64_to_f32_kernel<<<grid_for(n / 2, 256), 256, 0, st>>>(reinterpret_cast<const double2*>(in),
                                                           reinterpret_cast<float2*>(out), n / 2);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

void launch_f32_to_act(const float* in, act_t* out, size_t n, cudaStream_t st) {
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace d2ft_b200

namespace d2ft_b200 {

// ---------------------------------------------------------------- scoring pre-pass
// Bias parts of the unit gradients (b1 from G4's per-sample partials, b2 from
// the LN backward's per-tile column sums of the gradient entering the block),
// for every block: part[((l * n_units + u) * H + h) * 3 + {f2, fa, ft}].
__global__ void score_bias_kernel(Dims D, int mbs, int n_units, const float* part_db1, const float* part_cs,
                                  const float* b1, const float* b2, float* part) {
  D2FT_PDL_ENTRY();
  const int u = blockIdx.x, h = blockIdx.y, l = blockIdx.z;
  const int ntile = (D.T + 31) / 32, w = D.d / D.H;
  const float* pdb = part_db1 + (size_t)l * kG4Epi * D.Bmax * D.H * D.fs;
  const float* pcs = part_cs + (size_t)l * D.Bmax * ntile * D.d;
  float f2 = 0.f, fa = 0.f, ft = 0.f;
  for (int j = threadIdx.x; j < D.fs + w; j += blockDim.x) {
    float g = 0.f, wt;
    if (j < D.fs) {
      for (int s = u * mbs; s < (u + 1) * mbs; ++s)
        for (int e = 0; e < kG4Epi; ++e) g += pdb[(((size_t)e * D.Bmax + s) * D.H + h) * D.fs + j];
      wt = b1[((size_t)l * D.H + h) * D.fs + j];
    } else {
      const int m = h * w + (j - D.fs);
      for (int s = u * mbs; s < (u + 1) * mbs; ++s)
        for (int tt = 0; tt < ntile; ++tt) g += pcs[((size_t)s * ntile + tt) * D.d + m];
      wt = b2[(size_t)l * D.d + m];
    }
    f2 = fmaf(g, g, f2);
    fa += fabsf(g);
    ft += fabsf(g * wt);
  }
  __shared__ float red[3][32];
  f2 = warp_sum(f2);
  fa = warp_sum(fa);
  ft = warp_sum(ft);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = f2;
    red[1][warp] = fa;
    red[2][warp] = ft;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    float a = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a += red[threadIdx.x][i];
    part[(((size_t)l * n_units + u) * D.H + h) * 3 + threadIdx.x] = a;
  }
}

// WeightMagnitude per scheduled head-subnet (scoring.cpp:66-72): sum |w| over
// wq, wk, wv, wo, w1, b1, w2, b2 (fp32 masters, fp64 sum per thread).
__global__ void score_weight_kernel(Dims D, const float* W1T, const float* W2T, const float* b1, const float* b2,
                                    double* wm) {
  D2FT_PDL_ENTRY();
  const int h = blockIdx.x, l = blockIdx.y, w = D.d / D.H;
  const float* a = W1T + ((size_t)l * D.H + h) * D.PQ * D.d;
  const float* c = W2T + (size_t)l * D.d * D.H * D.PO + h * D.PO;
  double s = 0.0;
  for (size_t i = threadIdx.x; i < (size_t)D.PQ * D.d; i += blockDim.x) s += fabsf(a[i]);
  for (size_t i = threadIdx.x; i < (size_t)D.d * D.PO; i += blockDim.x) s += fabsf(c[(i / D.PO) * D.H * D.PO + i % D.PO]);
  for (int i = threadIdx.x; i < D.fs; i += blockDim.x) s += fabsf(b1[((size_t)l * D.H + h) * D.fs + i]);
  for (int i = threadIdx.x; i < w; i += blockDim.x) s += fabsf(b2[(size_t)l * D.d + h * w + i]);
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    wm[l * D.H + h] = t;
  }
}

// table[k][u] of a metric (0 Fisher, 1 WeightMagnitude, 2 GradientMagnitude,
// 3 Taylor; scoring.hpp:19-24) from the fixed-order sum of the GEMM partials
// (S7 then S5, tile then warp) and the bias part.
__global__ void score_reduce_kernel(Dims D, int n_units, const float* p7, const float* p5, const float* pb,
                                    const double* wm, int fwd_metric, int bwd_metric, double* fwd_out,
                                    double* bwd_out) {
  D2FT_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int K = D.L * D.H;
  if (i >= K * n_units) return;
  const int k = i / n_units, u = i % n_units, l = k / D.H, h = k % D.H;
  double acc[3] = {0.0, 0.0, 0.0};
  const size_t per = (size_t)n_units * D.H * kScoreTiles * 16 * 3;  // one block's partials
  for (int which = 0; which < 2; ++which) {
    const float* p = (which ? p5 : p7) + l * per + (((size_t)u * D.H + h) * kScoreTiles) * 16 * 3;
    for (int e = 0; e < kScoreTiles * 16; ++e)
      for (int q = 0; q < 3; ++q) acc[q] += p[e * 3 + q];
  }
  for (int q = 0; q < 3; ++q) acc[q] += pb[(((size_t)l * n_units + u) * D.H + h) * 3 + q];
  auto pick = [&](int metric) {
    switch (metric) {
      case 0: return acc[0];
      case 1: return wm[k];
      case 2: return acc[1];
      default: return acc[2];
    }
  };
  fwd_out[(size_t)k * n_units + u] = pick(fwd_metric);
  bwd_out[(size_t)k * n_units + u] = pick(bwd_metric);
}

void launch_score_bias(const Dims& D, int mbs, int n_units, const float* part_db1, const float* part_cs,
                       const float* b1, const float* b2, float* part, cudaStream_t st) {
  score_bias_kernel<<<dim3(n_units, D.H, D.L), 256, 0, st>>>(D, mbs, n_units, part_db1, part_cs, b1, b2, part);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}
void launch_score_weight(const Dims& D, const float* W1T, const float* W2T, const float* b1, const float* b2,
                         double* wm, cudaStream_t st) {
  score_weight_kernel<<<dim3(D.H, D.L), 512, 0, st>>>(D, W1T, W2T, b1, b2, wm);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}
void launch_score_reduce(const Dims& D, int n_units, const float* p7, const float* p5, const float* pb,
                         const double* wm, int fwd_metric, int bwd_metric, double* fwd_out, double* bwd_out,
                         cudaStream_t st) {
  const int n = D.L * D.H * n_units;
  score_reduce_kernel<<<(n + 127) / 128, 128, 0, st>>>(D, n_units, p7, p5, pb, wm, fwd_metric, bwd_metric, fwd_out,
                                                       bwd_out);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace d2ft_b200
