// GEMM problem policies of the D2FT step (GEMM table G1-G8).
// Orientation: "tokens as N" — a sample's T tokens are the UMMA N dimension
// (one TMA box of BN token rows, zero-filled past T), weight features are M
// in 64-row units gathered per active head, so no tile ever straddles two
// samples.  Weight gradients use "tokens as K" over the Full micro-batches of
// a head.  All operands are K-major fp16 (act_t); accumulation is fp32 in TMEM;
// gradient operands carry the step's power-of-two scale S (step_common.cuh).
#pragma once
#include "gemm_sm100.cuh"
#include <cuda_fp16.h>

#include "step_common.cuh"

namespace d2ft_b200 {

struct NoRow {};

// The step GEMMs run as CTA pairs (GemmShape CLUSTER = 2): a tile slot holds
// two tiles that share the B operand; `rank` selects the CTA's tile.
__host__ __device__ inline int mpairs(int mtiles) { return (mtiles + 1) / 2; }
constexpr int kUnitsPerSlot = 4;  // G1/G4: 2 x 64-row units per CTA

// ---------------------------------------------------------------- embed fwd
// x0[s][t][m] = sum_j inp[s][t][j] w_embed[j][m] + b_embed[m] + pos[t][m]
// (model.cpp:313-317).  A = WeT (d x d), B = inp (plane s).
template <int BN>
struct EmbedFwd {
  Dims D;
  const float* be;
  const float* pos;
  float* x0;
  struct Tile {
    int nkb, s, mt;
  };
  using Row = NoRow;
  // slot = (sample, pair of 128-row m-tiles); both CTAs share the sample's tokens (B)
  __device__ int ntiles() const { return D.B * mpairs(D.d / 128); }
  __device__ void tile(int t, int rank, Tile& c) const {
    c.s = t / mpairs(D.d / 128);
    c.mt = 2 * (t % mpairs(D.d / 128)) + rank;
    c.nkb = D.d / 64;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, 0, kb * 64, 0, c.s};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    const float b = be[m];
    float p[16];  // all loads first: the stores below may alias as far as the compiler knows
#pragma unroll
    for (int i = 0; i < 16; ++i) p[i] = col0 + i < D.T ? __ldg(pos + (size_t)(col0 + i) * D.d + m) : 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int t = col0 + i;
      if (t < D.T) x0[((size_t)c.s * D.T + t) * D.d + m] = v[i] + b + p[i];
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// ---------------------------------------------------------------- G1
// [q|k|v|z] = xn . [Wq|Wk|Wv|W1]  per (sample, active head)  (model.cpp:200-202, 218-220)
// A = W1T (plane l, rows h*PQ + f), B = xn (plane l*Bmax + s).  Epilogue:
// q,k,v -> QKV (token-major, attention operands); g = gelu(z + b1) -> OGT
// (feature-major: G3's MN-major B and G5's B); GELU'(z + b1) -> ZT (G4; only
// for Full cells — p_o cells never run backward, model.cpp:501).
//
// Every output leaves through shared memory and bulk tensor stores, 32 tokens
// per chunk: a warp's 32 accumulator rows (one feature each; the q / k / v /
// z section is warp-uniform since dh and fs are multiples of 32) x 32 tokens
// are staged and written by one TMA store per destination.  Per-lane global
// stores (32 rows per instruction) made the LSU the limiter of this epilogue;
// the GELU pair runs on packed fp32 (gelu_and_grad2).
#ifndef D2FT_G1_CW
#define D2FT_G1_CW 32  // tokens per epilogue chunk (16 or 32)
#endif
#ifndef D2FT_G1_BUFS
#define D2FT_G1_BUFS 1  // staging buffers per epilogue warp
#endif
template <int BN>
struct G1 {
  Dims D;
  int l;
  const int* tiles;
  const int* count;
  const int* act_heads;
  const int* act_cnt;
  const uint8_t* codes;  // expanded K x Bmax (code 1 = Full)
  const float* b1;  // block l: [H][fs]
  // bulk-store maps: [0] ZT, [1] OGT (CW tokens x 32 rows, CW*2-byte swizzle), [2] QKV (32 features x CW tokens)
  const CUtensorMap* maps;
  static constexpr int kChunk = D2FT_G1_CW;
  static constexpr int kNC = kChunk / 8;  // 16-byte chunks per staged row
  static constexpr bool kNonEmpty = true;
  static constexpr int kBufs = D2FT_G1_BUFS;
  static constexpr int kBufBytes = 2 * 32 * kChunk * 2;  // g tile + GELU' tile (or the QKV tile)
  static constexpr int kEpiStageBytes = kBufs * kBufBytes;
  struct Tile {
    int nkb, s, u0, nu, r0, r1;  // r0/r1: weight rows of the two 64-row units (fixed per tile)
  };
  struct Row {
    int valid, h, f, full, buf;
    float bias;
    uint8_t* stage;  // this warp's staging (kEpiStageBytes)
  };
  __device__ int ntiles() const { return *count; }
  __device__ int unit_row(int s, int u) const {
    const int h = act_heads[(s * D.L + l) * D.H + u / D.UQ];
    return h * D.PQ + (u % D.UQ) * 64;
  }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int p = tiles[t];
    c.s = p >> 16;
    c.u0 = (p & 0xffff) + 2 * rank;
    c.nu = D.UQ * act_cnt[c.s * D.L + l];
    c.nkb = D.d / 64;
    c.r0 = unit_row(c.s, c.u0 < c.nu ? c.u0 : c.nu - 1);  // units past nu: valid rows, ignored rows
    c.r1 = unit_row(c.s, c.u0 + 1 < c.nu ? c.u0 + 1 : c.nu - 1);
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.r0, c.r1, l, kb * 64, 0, l * D.Bmax + c.s};
  }
  __device__ void row_begin(const Tile& c, int row, Row& r) const {
    if (kBufs > 1) {  // buffer parity restarts: the previous tile's stores must have read both buffers
      if ((threadIdx.x & 31) == 0) ptx::bulk_wait_read<0>();
      r.buf = 0;
    }
    const int u = c.u0 + (row >> 6);
    r.valid = u < c.nu;
    if (!r.valid) return;
    r.h = act_heads[(c.s * D.L + l) * D.H + u / D.UQ];
    r.f = (u % D.UQ) * 64 + (row & 63);
    r.valid = r.f < D.PQ;
    r.full = codes[(size_t)(l * D.H + r.h) * D.Bmax + c.s] == 1;
    r.bias = (r.valid && r.f >= 3 * D.dh) ? b1[r.h * D.fs + (r.f - 3 * D.dh)] : 0.f;
  }
  __device__ void chunk(const Tile& c, int, int col0, const float (&v)[kChunk], Row& r) const {
    if (!r.valid || col0 >= D.T) return;  // warp-uniform
    const int lane = threadIdx.x & 31;
    // the store that last used this buffer must have read it; the wait comes
    // after this chunk's math, which hides it
    auto staging_free = [&]() {
      if (lane == 0) ptx::bulk_wait_read<kBufs - 1>();
      __syncwarp();
    };
    const int buf = kBufs > 1 ? r.buf : 0;
    uint8_t* stp = r.stage + buf * kBufBytes;
    const uint32_t sb = ptx::smem_u32(stp);
    const int plane = (l * D.Bmax + c.s) * D.H + r.h;
    const int f0 = r.f - lane;  // the warp's first feature row
    if (kBufs > 1) r.buf ^= 1;
    if (r.f < 3 * D.dh) {  // q, k, v: staged [kChunk tokens][32 features]
      uint32_t hv[kChunk / 2];
#pragma unroll
      for (int i = 0; i < kChunk / 2; ++i) {
        const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        hv[i] = *reinterpret_cast<const uint32_t*>(&h);
      }
      staging_free();
#pragma unroll
      for (int i = 0; i < kChunk / 2; ++i) {
        ptx::st_shared_u16(sb + (2 * i) * 64 + lane * 2, (unsigned short)(hv[i] & 0xffffu));
        ptx::st_shared_u16(sb + (2 * i + 1) * 64 + lane * 2, (unsigned short)(hv[i] >> 16));
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
#ifndef D2FT_EXP_G1_NOSTORE
        ptx::tma_store_3d(maps + 2, stp, f0, col0, plane);
#endif
        ptx::bulk_commit();
      }
      return;
    }
    const int j0 = f0 - 3 * D.dh;
    uint32_t hg[kChunk / 2], hz[kChunk / 2];  // half2 pairs of g = GELU(z) and GELU'(z), tokens 2i, 2i+1
#pragma unroll
    for (int i = 0; i < kChunk / 2; ++i) {
      float g0, g1, d0, d1;
#ifndef D2FT_EXP_G1_NOMATH
      gelu_and_grad2(v[2 * i] + r.bias, v[2 * i + 1] + r.bias, g0, g1, d0, d1);
#else
      g0 = v[2 * i] + r.bias, g1 = v[2 * i + 1] + r.bias, d0 = g1, d1 = g0;  // experiment: no GELU math
#endif
      const __half2 a = __floats2half2_rn(g0, g1), b = __floats2half2_rn(d0, d1);
      hg[i] = *reinterpret_cast<const uint32_t*>(&a);
      hz[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
    // row `lane` of a [32][kChunk] fp16 tile is kNC 16-byte chunks; the
    // (kChunk*2)-byte swizzle keeps the 8 lanes of each store phase on
    // distinct banks
    const uint32_t rb = sb + lane * (kChunk * 2), sw = ((lane * kNC) >> 3) & (kNC - 1);
    staging_free();
#pragma unroll
    for (int q = 0; q < kNC; ++q) {
      const uint32_t o = ((q ^ sw) << 4);
      ptx::st_shared_v4(rb + o, hg[4 * q], hg[4 * q + 1], hg[4 * q + 2], hg[4 * q + 3]);
      if (r.full)
        ptx::st_shared_v4(rb + kBufBytes / 2 + o, hz[4 * q], hz[4 * q + 1], hz[4 * q + 2], hz[4 * q + 3]);
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
#ifndef D2FT_EXP_G1_NOSTORE
      ptx::tma_store_3d(maps + 1, stp, col0, D.dh + j0, plane);
      if (r.full) ptx::tma_store_3d(maps + 0, stp + kBufBytes / 2, col0, j0, plane);
#endif
      ptx::bulk_commit();
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// ---------------------------------------------------------------- G3
// x_{l+1} = x_l + sum_{active h} ( [O_h|g_h] . [Wo_h;W2_h] + b2_h on its slice )
// (model.cpp:216, 221-225, 454-468).  A = W2T (plane l, K offset h*PO),
// B = OGT read MN-major (plane (l*Bmax+s)*H+h, rows = K features, tokens
// contiguous).  K = concatenation over the sample's active heads; the sum over
// heads happens inside TMEM in head order.
template <int BN>
struct G3 {
  Dims D;
  int l;
  const int* act_heads;
  const int* act_cnt;
  const uint8_t* codes;  // expanded K x Bmax
  const float* b2;       // block l: [d]
  const float* xin;
  float* xout;
  const int* order;  // block l: samples by decreasing active-head count (slot order)
  int* ctr;          // dynamic tile counter (gemm_sm100.cuh): K varies by sample
  struct Tile {
    int nkb, s, mt;
    int heads[16];  // the sample's active heads in block l (cached once per tile)
  };
  struct Row {
    float bias;
    float xi[16];  // residual of the warp's next chunk (prefetched one chunk ahead)
  };
  __device__ int ntiles() const { return D.B * mpairs(D.d / 128); }
  __device__ int ncols(const Tile&) const { return D.T; }
  __device__ void tile(int t, int rank, Tile& c) const {
    c.s = order[t / mpairs(D.d / 128)];
    c.mt = 2 * (t % mpairs(D.d / 128)) + rank;
    const int n = act_cnt[c.s * D.L + l];
    c.nkb = D.UO * n;
    const int* hp = act_heads + (c.s * D.L + l) * D.H;
#pragma unroll
    for (int a = 0; a < 16; ++a) c.heads[a] = a < n ? hp[a] : 0;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int a = kb / D.UO, kk = kb % D.UO;
    const int h = c.heads[a];
    return KCoord{h * D.PO + kk * 64, c.mt * 128, c.mt * 128 + 64, l, 0, kk * 64, (l * D.Bmax + c.s) * D.H + h};
  }
  __device__ void row_begin(const Tile& c, int row, Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    const int hm = m / (D.d / D.H);
    const uint8_t code = codes[(size_t)(l * D.H + hm) * D.Bmax + c.s];
    r.bias = (code == 1 || code == 2) ? b2[m] : 0.f;  // p_s adds nothing (model.cpp:458)
  }
  // xin == nullptr: partial block output of a head partition (the residual is
  // added by partition rank 0 only, so the exchange sum carries it once)
  __device__ void prefetch(const Tile& c, int row, int col0, Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d || col0 >= D.T) return;
    const size_t o0 = ((size_t)c.s * D.T + col0) * D.d + m;
#pragma unroll
    for (int i = 0; i < 16; ++i) r.xi[i] = (xin && col0 + i < D.T) ? __ldg(xin + o0 + (size_t)i * D.d) : 0.f;
  }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d || col0 >= D.T) return;
    const size_t o0 = ((size_t)c.s * D.T + col0) * D.d + m;
    float xi[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) xi[i] = r.xi[i];
    prefetch(c, row, col0 + 16 * kG3Epi, r);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (col0 + i < D.T) xout[o0 + (size_t)i * D.d] = xi[i] + v[i] + r.bias;
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// ---------------------------------------------------------------- G4
// d[O|g] = dC . [Wo;W2]^T per (sample, Full head)  (model.cpp:247, 262);
// epilogue dz = dg * gelu'(z) (model.cpp:254), db1 row sums (model.cpp:257).
// A = W2 (plane l, rows h*PO + f), B = dC (plane s).  Outputs leave through
// shared-memory staging and bulk tensor stores, 32 tokens per chunk (as G1).
template <int BN>
struct G4 {
  Dims D;
  int l;
  const int* tiles;
  const int* count;
  const int* full_heads;
  const int* full_hcnt;
  const act_t* ZT;  // block l: [Bmax][H][fs][TP]  GELU'(z), written by G1
  float* part_db1; // [EPI][Bmax][H][fs]
  const float* gmax;
  const CUtensorMap* maps;  // bulk-store maps: [3] dO (32 features x 32 tokens), [4] dY1T (32 tokens x 32 rows, 64B swizzle)
  int* ctr;                 // non-null: dynamic tile claiming (gemm_sm100.cuh); null: static striding
  static constexpr int kChunk = 32;
  static constexpr bool kNonEmpty = true;
  static constexpr int kEpiStageBytes = 2048;
  struct Tile {
    int nkb, s, u0, nu, r0, r1;
  };
  struct Row {
    int valid, h, f;
    float db;
    uint4 gp[4];  // GELU'(z) of the warp's next chunk (prefetched one chunk ahead)
    uint8_t* stage;
  };
  __device__ int ntiles() const { return *count; }
  __device__ int unit_row(int s, int u) const {
    const int h = full_heads[(s * D.L + l) * D.H + u / D.UO];
    return h * D.PO + (u % D.UO) * 64;
  }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int p = tiles[t];
    c.s = p >> 16;
    c.u0 = (p & 0xffff) + 2 * rank;
    c.nu = D.UO * full_hcnt[c.s * D.L + l];
    c.nkb = D.d / 64;
    c.r0 = unit_row(c.s, c.u0 < c.nu ? c.u0 : c.nu - 1);
    c.r1 = unit_row(c.s, c.u0 + 1 < c.nu ? c.u0 + 1 : c.nu - 1);
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.r0, c.r1, l, kb * 64, 0, c.s};
  }
  __device__ void row_begin(const Tile& c, int row, Row& r) const {
    const int u = c.u0 + (row >> 6);
    r.valid = u < c.nu;
    r.db = 0.f;
    if (!r.valid) return;
    r.h = full_heads[(c.s * D.L + l) * D.H + u / D.UO];
    r.f = (u % D.UO) * 64 + (row & 63);
    r.valid = r.f < D.PO;
  }
  // GELU' row of this feature, 32 contiguous tokens from col0 (four 16-byte
  // loads), issued a chunk ahead so their latency hides behind the MMA wait.
  __device__ void prefetch(const Tile& c, int, int col0, Row& r) const {
    if (!r.valid || r.f < D.dh || col0 >= D.T) return;
    const act_t* z = ZT + (((size_t)c.s * D.H + r.h) * D.fs + (r.f - D.dh)) * D.TP + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      r.gp[q] = col0 + 8 * q + 8 <= D.TP ? *reinterpret_cast<const uint4*>(z + 8 * q) : make_uint4(0, 0, 0, 0);
  }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[32], Row& r) const {
    if (!r.valid || col0 >= D.T) return;  // warp-uniform
    const int lane = threadIdx.x & 31;
    auto staging_free = [&]() {  // the previous chunk's store has read the staging (after this chunk's math)
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
    };
    const uint32_t sb = ptx::smem_u32(r.stage);
    const int plane = c.s * D.H + r.h;
    const int f0 = r.f - lane;
    if (r.f < D.dh) {  // dO: staged [32 tokens][32 features]
      uint32_t hv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        hv[i] = *reinterpret_cast<const uint32_t*>(&h);
      }
      staging_free();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        ptx::st_shared_u16(sb + (2 * i) * 64 + lane * 2, (unsigned short)(hv[i] & 0xffffu));
        ptx::st_shared_u16(sb + (2 * i + 1) * 64 + lane * 2, (unsigned short)(hv[i] >> 16));
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_3d(maps + 3, r.stage, f0, col0, plane);
        ptx::bulk_commit();
      }
      return;
    }
    uint32_t gz[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      gz[4 * q] = r.gp[q].x;
      gz[4 * q + 1] = r.gp[q].y;
      gz[4 * q + 2] = r.gp[q].z;
      gz[4 * q + 3] = r.gp[q].w;
    }
    prefetch(c, row, col0 + 32 * kG4Epi, r);
    uint32_t hz[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 gp = __half22float2(*reinterpret_cast<const __half2*>(&gz[i]));
      const float d0 = col0 + 2 * i < D.T ? v[2 * i] * gp.x : 0.f;
      const float d1 = col0 + 2 * i + 1 < D.T ? v[2 * i + 1] * gp.y : 0.f;
      r.db += d0 + d1;
      const __half2 h = __floats2half2_rn(d0, d1);
      hz[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    const uint32_t rb = sb + lane * 64, sw = (lane >> 1) & 3;
    staging_free();
#pragma unroll
    for (int q = 0; q < 4; ++q)
      ptx::st_shared_v4(rb + ((q ^ sw) << 4), hz[4 * q], hz[4 * q + 1], hz[4 * q + 2], hz[4 * q + 3]);
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_3d(maps + 4, r.stage, col0, 3 * D.dh + (f0 - D.dh), plane);
      ptx::bulk_commit();
    }
  }
  // one partial per column group (summed in fixed order by bias_reduce)
  __device__ void row_end(const Tile& c, int, int group, Row& r) const {
    if (r.valid && r.f >= D.dh)
      part_db1[(((size_t)group * D.Bmax + c.s) * D.H + r.h) * D.fs + (r.f - D.dh)] = r.db / grad_scale(gmax);
  }
};

// ---------------------------------------------------------------- fused SGD
// sgd_momentum_step (trainer.cpp:114-121) applied in the G5 / G7 epilogues
// when a training step follows: the weight gradient never reaches HBM and the
// separate SGD pass skips [Wq|Wk|Wv|W1]^T and [Wo;W2]^T (the bulk of the
// parameters).  Same arithmetic as sgd_kernel (bitwise).  Tiles of heads
// without Full samples (nkb == 0) leave p and v untouched (trainer.cpp:264-268).
// P == nullptr: write the gradient (forward_backward API, pre-pass, LoRA).
struct FusedSgd {
  float* P;     // master weights of block l's segment, gradient indexing
  float* V;     // momentum
  act_t* Pbf;   // fp16 operand copy
  float lr, mom;
  int* err;
  __device__ __forceinline__ void apply(size_t i, float g) const {
    if (!isfinite(g)) {
      atomicCAS(err, 0, 5);  // kNumeric (trainer.cpp:118)
      return;
    }
    const float v = mom * V[i] + g;
    const float p = P[i] - lr * v;
    V[i] = v;
    P[i] = p;
    Pbf[i] = to_act(p);
  }
};

// ---------------------------------------------------------------- G5
// dW2T[l][m][h*PO + f] = sum_{s in Full(h)} sum_t dC[s][t][m] [O|g][s][h][t][f]
// (model.cpp:249, 263).  A = dC read MN-major (plane s, [t][m] as [K][M]),
// B = OGT (plane (l*Bmax+s)*H+h).
// Epilogue: per-lane 16-byte stores (16 contiguous fp32 of the thread's row).
// D2FT_G5_TMA=1 (opt-in): each warp stages its 32 rows x 16 fp32 (64-byte
// swizzle) and writes them with one bulk tensor store ([5] of the store maps)
// — G5 0.526 -> 0.496 ms per step, but the G7 that follows it 0.563 -> 0.608
// (same box, two runs), the step neutral; not adopted.
#ifndef D2FT_G5_TMA
#define D2FT_G5_TMA 0
#endif
template <int BN>
struct G5 {
  Dims D;
  int l;
  const int* full_idx;  // row k: Bmax entries
  const int* full_cnt;
  float* dW2T;  // block l: [d][H*PO]
  const float* gmax;
  const int* order;  // block l: heads by decreasing Full-sample count
  int* ctr;
  FusedSgd sgd;
  const CUtensorMap* maps;  // [5]: dW2T bulk-store map (fp32, 16 x 32 box, 64B swizzle)
  static constexpr int kEpiStageBytes = D2FT_G5_TMA ? 32 * 16 * 4 : 0;
  struct Tile {
    int nkb, h, mt, nt;
  };
  struct Row {
    float inv;
    uint8_t* stage;
  };
  __device__ int ntn() const { return (D.PO + BN - 1) / BN; }
  // slot = (head, m-tile pair, n-tile): the pair shares B = [O|g]^T of (s, h)
  __device__ int ntiles() const { return D.H * mpairs(D.d / 128) * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int per = mpairs(D.d / 128) * ntn();
    c.h = order[t / per];
    const int r = t % per;
    c.mt = 2 * (r / ntn()) + rank;
    c.nt = r % ntn();
    c.nkb = D.TB * full_cnt[l * D.H + c.h];
  }
  // the last 64-token block of a sample carries T - 64*(TB-1) tokens
  __device__ int ksteps(const Tile&, int kb) const {
    return kb % D.TB == D.TB - 1 ? (D.T - 64 * (D.TB - 1) + 15) / 16 : 4;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int s = full_idx[(size_t)(l * D.H + c.h) * D.Bmax + kb / D.TB];
    const int t0 = (kb % D.TB) * 64;
    return KCoord{t0, c.mt * 128, c.mt * 128 + 64, s, t0, c.nt * BN, (l * D.Bmax + s) * D.H + c.h};
  }
  __device__ void row_begin(const Tile&, int, Row& r) const { r.inv = 1.f / grad_scale(gmax); }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    const int f0 = c.nt * BN + col0;
    if (sgd.P) {
      if (c.nkb == 0) return;
      const size_t o = (size_t)m * D.H * D.PO + c.h * D.PO + f0;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (f0 + i < D.PO) sgd.apply(o + i, v[i] * r.inv);
      return;
    }
    if constexpr (D2FT_G5_TMA > 0) {
      if (f0 + 16 <= D.PO && (m - (int)(threadIdx.x & 31)) + 32 <= D.d) {  // warp-uniform
        const int lane = threadIdx.x & 31;
        const uint32_t sb = ptx::smem_u32(r.stage), rb = sb + lane * 64, sw = (lane >> 1) & 3;
        if (lane == 0) ptx::bulk_wait_read<0>();  // the previous chunk's store has read the staging
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ptx::st_shared_v4(rb + ((q ^ sw) << 4), __float_as_uint(v[4 * q] * r.inv),
                            __float_as_uint(v[4 * q + 1] * r.inv), __float_as_uint(v[4 * q + 2] * r.inv),
                            __float_as_uint(v[4 * q + 3] * r.inv));
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_3d(maps + 5, r.stage, c.h * D.PO + f0, m - lane, l);
          ptx::bulk_commit();
        }
        return;
      }
    }
    float* out = dW2T + (size_t)m * D.H * D.PO + c.h * D.PO;
    if (f0 + 16 <= D.PO) {  // 16 contiguous fp32 of this row: four 16-byte stores
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4*>(out + f0 + i) =
            make_float4(v[i] * r.inv, v[i + 1] * r.inv, v[i + 2] * r.inv, v[i + 3] * r.inv);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (f0 + i < D.PO) out[f0 + i] = v[i] * r.inv;
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// ---------------------------------------------------------------- G7
// dW1T[l][h][f][m] = sum_{s in Full(h)} sum_t xn[s][t][m] d[q|k|v|z][s][h][f][t]
// (model.cpp:256, 286).  M = model features m (d = 6 x 128: no padded rows),
// N = the head's PQ = 2 x 224 features, K = tokens of the head's Full samples.
// A = xn read MN-major (token-major [t][m] as [K][M]), B = dY1T (K-major).
template <int BN>
struct G7 {
  Dims D;
  int l;
  const int* full_idx;
  const int* full_cnt;
  float* dW1T;  // block l: [H][PQ][d]
  const float* gmax;
  const int* order;  // block l: heads by decreasing Full-sample count
  int* ctr;
  FusedSgd sgd;
  struct Tile {
    int nkb, h, mt, nt;
  };
  struct Row {
    float inv;
  };
  __device__ int ntm() const { return (D.d + 127) / 128; }
  __device__ int ntn() const { return (D.PQ + BN - 1) / BN; }
  // slot = (head, m-tile pair, n-tile): the pair shares B = dY1T rows of (s, h)
  __device__ int ntiles() const { return D.H * mpairs(ntm()) * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int per = mpairs(ntm()) * ntn();
    c.h = order[t / per];
    const int r = t % per;
    c.mt = 2 * (r / ntn()) + rank;
    c.nt = r % ntn();
    c.nkb = D.TB * full_cnt[l * D.H + c.h];
  }
  // the last 64-token block of a sample carries T - 64*(TB-1) tokens
  __device__ int ksteps(const Tile&, int kb) const {
    return kb % D.TB == D.TB - 1 ? (D.T - 64 * (D.TB - 1) + 15) / 16 : 4;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int s = full_idx[(size_t)(l * D.H + c.h) * D.Bmax + kb / D.TB];
    const int t0 = (kb % D.TB) * 64;
    return KCoord{t0, c.mt * 128, c.mt * 128 + 64, l * D.Bmax + s, t0, c.nt * BN, s * D.H + c.h};
  }
  __device__ void row_begin(const Tile&, int, Row& r) const { r.inv = 1.f / grad_scale(gmax); }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    const int f0 = c.nt * BN + col0;
    if (sgd.P) {
      if (c.nkb == 0) return;
      const size_t o = ((size_t)c.h * D.PQ + f0) * D.d + m;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (f0 + i < D.PQ) sgd.apply(o + (size_t)i * D.d, v[i] * r.inv);
      return;
    }
    // lanes hold consecutive m: each store instruction writes 128 contiguous bytes
    float* out = dW1T + ((size_t)c.h * D.PQ + f0) * D.d + m;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (f0 + i < D.PQ) out[(size_t)i * D.d] = v[i] * r.inv;
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// ---------------------------------------------------------------- G8
// dxn[s] = sum_{Full h} d[q|k|v|z]_h . [Wq|Wk|Wv|W1]_h^T  (model.cpp:259, 288)
// A = W1 (plane l, K offset h*PQ), B = dY1T read MN-major (plane s*H+h).
template <int BN>
struct G8 {
  Dims D;
  int l;
  const int* full_heads;
  const int* full_hcnt;
  float* dxn;     // [Bmax][T][d] fp32 (head partition: the exchange sums it), or
  act_t* dxn_h;   // [Bmax][T][d] fp16 in gradient-scale units (single engine; LN backward undoes S)
  const float* gmax;
  const int* order;  // block l: samples by decreasing Full-head count
  int* ctr;
  struct Tile {
    int nkb, s, mt;
    int heads[16];
  };
  struct Row {
    float inv;
  };
  __device__ int ntiles() const { return D.B * mpairs(D.d / 128); }
  __device__ int ncols(const Tile&) const { return D.T; }
  __device__ void tile(int t, int rank, Tile& c) const {
    c.s = order[t / mpairs(D.d / 128)];
    c.mt = 2 * (t % mpairs(D.d / 128)) + rank;
    const int n = full_hcnt[c.s * D.L + l];
    c.nkb = D.UQ * n;
    const int* hp = full_heads + (c.s * D.L + l) * D.H;
#pragma unroll
    for (int a = 0; a < 16; ++a) c.heads[a] = a < n ? hp[a] : 0;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int a = kb / D.UQ, kk = kb % D.UQ;
    const int h = c.heads[a];
    return KCoord{h * D.PQ + kk * 64, c.mt * 128, c.mt * 128 + 64, l, 0, kk * 64, c.s * D.H + h};
  }
  __device__ void row_begin(const Tile&, int, Row& r) const { r.inv = 1.f / grad_scale(gmax); }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int t = col0 + i;
      if (t < D.T) {
        if (dxn_h) dxn_h[((size_t)c.s * D.T + t) * D.d + m] = to_act(v[i]);
        else dxn[((size_t)c.s * D.T + t) * D.d + m] = v[i] * r.inv;
      }
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// ---------------------------------------------------------------- embed wgrad
// dWeT[m][j] = sum_s sum_t dx0[s][t][m] inp[s][t][j]  (model.cpp:514), split
// over KS sample groups into partial sums (reduced deterministically later).
// A = dC read MN-major, B = inpT.
template <int BN>
struct EmbedW {
  Dims D;
  int KS;
  float* part;  // [KS][d][d]
  const float* gmax;
  struct Tile {
    int nkb, ks, mt, nt, s0;
  };
  struct Row {
    float inv;
  };
  __device__ int ntn() const { return (D.d + BN - 1) / BN; }
  __device__ int ntiles() const { return KS * mpairs(D.d / 128) * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int per = mpairs(D.d / 128) * ntn();
    c.ks = t / per;
    const int r = t % per;
    c.mt = 2 * (r / ntn()) + rank;
    c.nt = r % ntn();
    c.s0 = c.ks * D.B / KS;
    c.nkb = D.TB * ((c.ks + 1) * D.B / KS - c.s0);
  }
  // the last 64-token block of a sample carries T - 64*(TB-1) tokens
  __device__ int ksteps(const Tile&, int kb) const {
    return kb % D.TB == D.TB - 1 ? (D.T - 64 * (D.TB - 1) + 15) / 16 : 4;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int s = c.s0 + kb / D.TB;
    const int t0 = (kb % D.TB) * 64;
    return KCoord{t0, c.mt * 128, c.mt * 128 + 64, s, t0, c.nt * BN, s};
  }
  __device__ void row_begin(const Tile&, int, Row& r) const { r.inv = 1.f / grad_scale(gmax); }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    float* out = part + ((size_t)c.ks * D.d + m) * D.d;
    const int n0 = c.nt * BN + col0;
    if (n0 + 16 <= D.d) {  // the row's 16 contiguous floats as four 16-byte stores (scalar stores: LSU-throttled)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(out + n0 + 4 * q) =
            make_float4(v[4 * q] * r.inv, v[4 * q + 1] * r.inv, v[4 * q + 2] * r.inv, v[4 * q + 3] * r.inv);
      return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (n0 + i < D.d) out[n0 + i] = v[i] * r.inv;
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

}  // namespace d2ft_b200

namespace d2ft_b200 {

// ---------------------------------------------------------------- scoring pre-pass
// prepass_scores (scoring.cpp:108-151): every micro-batch ("unit") runs
// forward + backward with all subnets Full and no update; each scheduled
// head-subnet's unit gradient is reduced to sum(g^2) (FisherInformation),
// sum|g| (GradientMagnitude) and sum|w g| (TaylorImportance), scoring.cpp:57-96.
// The unit gradients of the weight matrices are the G7 / G5 products with K
// restricted to the unit's tokens; nothing is stored — the epilogue folds the
// three sums per thread and one lane per warp writes the warp's partials:
//   part[((u * H + h) * kScoreTiles + tile) * 16 + warp][3],  tile = mt * 2 + nt
// (fixed-order reduction in score_reduce_kernel).

struct ScoreRow {
  float f2, fa, ft;  // sum g^2, sum |g|, sum |w g|
  float inv;
};
__device__ __forceinline__ void score_row_end(float* part, size_t base, int warp, ScoreRow& r) {
  float a = r.f2, b = r.fa, c = r.ft;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    float* p = part + (base * 16 + warp) * 3;
    p[0] = a;
    p[1] = b;
    p[2] = c;
  }
}

// unit gradients of [Wq|Wk|Wv|W1] (G7 with K = the unit's tokens): M = d, N = PQ
template <int BN>
struct S7 {
  Dims D;
  int l, mbs, n_units;
  const float* W1T;  // block l master: [H][PQ][d]
  const float* gmax;
  float* part;
  struct Tile {
    int nkb, u, h, mt, nt;
  };
  using Row = ScoreRow;
  __device__ int ntm() const { return (D.d + 127) / 128; }
  __device__ int ntn() const { return (D.PQ + BN - 1) / BN; }
  __device__ int ntiles() const { return n_units * D.H * mpairs(ntm()) * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int per = mpairs(ntm()) * ntn();
    c.u = t / (D.H * per);
    c.h = (t / per) % D.H;
    const int r = t % per;
    c.mt = 2 * (r / ntn()) + rank;
    c.nt = r % ntn();
    c.nkb = D.TB * mbs;
  }
  __device__ int ksteps(const Tile&, int kb) const {
    return kb % D.TB == D.TB - 1 ? (D.T - 64 * (D.TB - 1) + 15) / 16 : 4;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int s = c.u * mbs + kb / D.TB;
    const int t0 = (kb % D.TB) * 64;
    return KCoord{t0, c.mt * 128, c.mt * 128 + 64, l * D.Bmax + s, t0, c.nt * BN, s * D.H + c.h};
  }
  __device__ void row_begin(const Tile&, int, Row& r) const {
    r.f2 = r.fa = r.ft = 0.f;
    r.inv = 1.f / grad_scale(gmax);
  }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    const int f0 = c.nt * BN + col0;
    const float* w = W1T + ((size_t)c.h * D.PQ + f0) * D.d + m;  // lanes: consecutive m
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (f0 + i < D.PQ) {
        const float g = v[i] * r.inv;
        r.f2 = fmaf(g, g, r.f2);
        r.fa += fabsf(g);
        r.ft += fabsf(g * __ldg(w + (size_t)i * D.d));
      }
  }
  __device__ void row_end(const Tile& c, int, int, Row& r) const {
    const int warp = (threadIdx.x >> 5) - 4;
    score_row_end(part, ((size_t)c.u * D.H + c.h) * kScoreTiles + c.mt * ntn() + c.nt, warp, r);
  }
};

// unit gradients of [Wo;W2] (G5 with K = the unit's tokens): M = d, N = PO
template <int BN>
struct S5 {
  Dims D;
  int l, mbs, n_units;
  const float* W2T;  // block l master: [d][H*PO]
  const float* gmax;
  float* part;
  struct Tile {
    int nkb, u, h, mt, nt;
  };
  using Row = ScoreRow;
  __device__ int ntn() const { return (D.PO + BN - 1) / BN; }
  __device__ int ntiles() const { return n_units * D.H * mpairs(D.d / 128) * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int per = mpairs(D.d / 128) * ntn();
    c.u = t / (D.H * per);
    c.h = (t / per) % D.H;
    const int r = t % per;
    c.mt = 2 * (r / ntn()) + rank;
    c.nt = r % ntn();
    c.nkb = D.TB * mbs;
  }
  __device__ int ksteps(const Tile&, int kb) const {
    return kb % D.TB == D.TB - 1 ? (D.T - 64 * (D.TB - 1) + 15) / 16 : 4;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int s = c.u * mbs + kb / D.TB;
    const int t0 = (kb % D.TB) * 64;
    return KCoord{t0, c.mt * 128, c.mt * 128 + 64, s, t0, c.nt * BN, (l * D.Bmax + s) * D.H + c.h};
  }
  __device__ void row_begin(const Tile&, int, Row& r) const {
    r.f2 = r.fa = r.ft = 0.f;
    r.inv = 1.f / grad_scale(gmax);
  }
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row& r) const {
    const int m = c.mt * 128 + row;
    if (m >= D.d) return;
    const int f0 = c.nt * BN + col0;
    const float* w = W2T + (size_t)m * D.H * D.PO + c.h * D.PO + f0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (f0 + i < D.PO) {
        const float g = v[i] * r.inv;
        r.f2 = fmaf(g, g, r.f2);
        r.fa += fabsf(g);
        r.ft += fabsf(g * __ldg(w + i));
      }
  }
  __device__ void row_end(const Tile& c, int, int, Row& r) const {
    const int warp = (threadIdx.x >> 5) - 4;
    score_row_end(part, ((size_t)c.u * D.H + c.h) * kScoreTiles + c.mt * ntn() + c.nt, warp, r);
  }
};

// ---------------------------------------------------------------- surrogate (opt-in p_s)
// p_s as "skip with a linear surrogate" (north_star) instead
// of the reference's pure bypass (model.cpp:326-328, 458): a shortcut cell
// (s, l, h) adds xn_s . A_{l,h} . B_{l,h} (rank-R factors, frozen, no
// gradient — like p_o it never runs backward, model.cpp:501).  Off (rank 0)
// in every parity run; two small dense GEMMs per block when on:
//   Sur1: U[s] = xn_s . [A_{l,1} .. A_{l,H}]   (M = H*R features, N = tokens, K = d)
//         epilogue keeps a head's R columns only where the cell is p_s -> U [Bmax][H*R][TP] fp16
//   Sur2: x_{l+1}[s] += U[s] . [B_{l,1}; ..; B_{l,H}]   (M = d, N = tokens, K = H*R, B read MN-major)
// A operands: SurA [L][H*R][d] (A^T), SurB [L][d][H*R] (B^T), fp16.  Samples
// without a p_s cell in the block skip both (nkb = 0).
template <int BN>
struct Sur1 {
  Dims D;
  int l, HR, R;
  const int* act_cnt;    // [Bmax][L]
  const uint8_t* codes;  // expanded K x Bmax
  act_t* U;              // [Bmax][HR][TP]
  struct Tile {
    int nkb, s, mt;
  };
  using Row = NoRow;
  __device__ int ntiles() const { return D.B * mpairs((HR + 127) / 128); }
  __device__ void tile(int t, int rank, Tile& c) const {
    const int mp = mpairs((HR + 127) / 128);
    c.s = t / mp;
    c.mt = 2 * (t % mp) + rank;
    c.nkb = act_cnt[c.s * D.L + l] < D.H ? D.d / 64 : 0;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, l, kb * 64, 0, l * D.Bmax + c.s};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    const int f = c.mt * 128 + row;
    if (c.nkb == 0 || f >= HR || col0 >= D.T) return;
    const bool ps = codes[(size_t)(l * D.H + f / R) * D.Bmax + c.s] == 3;
    act_t* u = U + ((size_t)c.s * HR + f) * D.TP + col0;
#pragma unroll
    for (int i = 0; i < 16; i += 2)
      if (col0 + i < D.TP)
        *reinterpret_cast<__half2*>(u + i) = __floats2half2_rn(ps ? v[i] : 0.f, ps ? v[i + 1] : 0.f);
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

template <int BN>
struct Sur2 {
  Dims D;
  int l, HR;
  const int* act_cnt;
  float* xout;  // x_{l+1}, already holding x_l + the active heads (G3)
  struct Tile {
    int nkb, s, mt;
  };
  using Row = NoRow;
  __device__ int ntiles() const { return D.B * mpairs(D.d / 128); }
  __device__ int ncols(const Tile&) const { return D.T; }
  __device__ void tile(int t, int rank, Tile& c) const {
    c.s = t / mpairs(D.d / 128);
    c.mt = 2 * (t % mpairs(D.d / 128)) + rank;
    c.nkb = act_cnt[c.s * D.L + l] < D.H ? (HR + 63) / 64 : 0;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, l, 0, kb * 64, c.s};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    const int m = c.mt * 128 + row;
    if (c.nkb == 0 || m >= D.d || col0 >= D.T) return;
    float* x = xout + ((size_t)c.s * D.T + col0) * D.d + m;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (col0 + i < D.T) x[(size_t)i * D.d] += v[i];
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

}  // namespace d2ft_b200
