// Non-GEMM kernels of the D2FT step (launch wrappers).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "step_common.cuh"

namespace d2ft_b200 {

// codes [K][n_mb] -> per-sample codes [K][Bmax] (sample s uses column s / mbs; s >= B -> 3)
// codes_exp[k][s] = codes[k][mb0 + s / mbs] for the B samples (mb0: first
// micro-batch of this data-parallel rank), 3 past B
void launch_expand_codes(const uint8_t* codes, int K, int n_mb, int mbs, int B, int Bmax, uint8_t* out,
                         cudaStream_t st, int mb0 = 0);
void launch_row_full_count(const uint8_t* codes, int K, int n_mb, int* out, cudaStream_t st);
void launch_zero_untouched(const Dims& D, const int* full_cnt, float* G, size_t o_w1, size_t o_b1, size_t o_w2,
                           size_t o_b2, cudaStream_t st);
// Per-block GEMM plan of one batch: G1 / G4 tile lists over (sample, 64-row
// unit pair) and the cost orders of the dynamically scheduled GEMMs.
struct Plan {
  int *g1_tiles, *g1_count, *g4_tiles, *g4_count;
  int* ord_act;   // [L][Bmax] samples by decreasing active-head count (G3)
  int* ord_full;  // [L][Bmax] samples by decreasing Full-head count (G8)
  int* ord_head;  // [L][H] heads by decreasing Full-sample count (G5, G7)
  int *af_items, *af_count;  // [L][Bmax*H] (sample << 8 | active slot) of the attention forward
  int *ab_items, *ab_count;  // [L][Bmax*H] (sample << 8 | Full slot) of the attention backward
  int chunks = 1;  // ord_act / ord_full sorted within sample chunks [c*B/C, (c+1)*B/C) (head-partition exchange)
};
void launch_plan(const Dims& D, const int* act_cnt, const int* full_hcnt, const int* full_cnt, const Plan& pl,
                 cudaStream_t st);
// fp32 samples [B][T][d] -> act_t token-major + feature-major copies
void launch_prep_input(const Dims& D, const float* x, act_t* inp, act_t* inpT, cudaStream_t st);
// LayerNorm (no affine, eps 1e-5) of x -> xn (token-major fp16), stats (mean, rstd);
// samples [s0, s0 + ns) (ns < 0: the whole batch D.B)
void launch_ln_fwd(const Dims& D, const float* x, act_t* xn, float* stats, cudaStream_t st, int s0 = 0, int ns = -1);
// attention forward / backward (one CTA per (sample, active|Full head) slot)
// (O feature-major into OGT rows 0..dh-1; dq|dk|dv feature-major into dY1T rows 0..3dh-1)
void launch_attn_fwd(const Dims& D, int l, const int* act_heads, const int* act_cnt, const act_t* Y1, act_t* OGT,
                     float* lse, cudaStream_t st);
void launch_attn_bwd(const Dims& D, int l, const int* full_heads, const int* full_hcnt, const act_t* Y1,
                     const act_t* OGT, const act_t* dO, const float* lse, act_t* dY1T, cudaStream_t st);
// tcgen05 attention forward (attn_sm100.cu), dh = 64: tensor maps over the
// whole QKV buffer [L][Bmax][H][T][3dh] with boxes of 64 x 128 (Q), 64 x TQ
// (K), 64 x 64 (V) rows; planes (l*Bmax + s)*H + h
void launch_attn_fwd_tc(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV, const Dims& D, int l,
                        const int* items, const int* count, const int* act_heads, act_t* OGT, float* lse,
                        const uint8_t* codes, float* O32T, cudaStream_t st);
int sm_max_attn();
// tcgen05 attention backward (attn_sm100.cu), dh = 64: tmQKV = the K map above
// (box 64 x TQ), tmdO over dO [Bmax][H][T][dh] with box 64 x TQ
void launch_attn_bwd_tc(const CUtensorMap& tmQKV, const CUtensorMap& tmdO, const Dims& D, int l, const int* full_heads,
                        const int* full_hcnt, const float* O32T, const float* lse, act_t* dY1T, cudaStream_t st);
bool attn_bwd_tc_fits(int TQ);
// head: LN -> mean-pool -> linear -> CE; writes loss_s, pooled, logits, dlogits, and dX = dL/dx_L
void launch_head(const Dims& D, const float* xL, const int* labels, const float* Wc, const float* bc, float scale,
                 double* loss_s, float* pooled, float* dlog, float* dX, float* gmax, float* logits, cudaStream_t st);
void launch_head_reduce(const Dims& D, const double* loss_s, const float* pooled, const float* dlog, float* dWc,
                        float* dbc, double* loss, cudaStream_t st,
                        int loss_div = 0);
// dX += LN_bwd(x_l, dxn) for samples with a Full head in block l (if l >= 0), then
// emit dC (act_t token-major) and per-tile column sums.
// x_l (fp32) or xn_l (the stored fp16 LN output) for y; dxn (fp32) or dxn_h (fp16, gradient-scale units)
void launch_ln_bwd_prep(const Dims& D, int l, const int* full_hcnt, const float* x_l, const act_t* xn_l,
                        const float* stats_l, const float* dxn, const act_t* dxn_h, float* dX, act_t* dC,
                        float* part_cs, const float* gmax, cudaStream_t st, int s0 = 0, int ns = -1);
void launch_bias_reduce(const Dims& D, const uint8_t* codes, const float* part_cs, const float* part_db1, float* db1,
                        float* db2, cudaStream_t st);
void launch_embed_reduce(const Dims& D, int KS, const float* part, const float* part_cs, const float* dX, float* dWeT,
                         float* dbe, float* dpos, cudaStream_t st);
// SGD with momentum (trainer.cpp:113-134) on one tensor; elements whose
// scheduled row k = (i/outer)*H + (i/inner)%H has full_cnt[k] == 0 are skipped
// (outer == 0: always touched).  pbf (may be null) receives the act_t copy.
void launch_sgd(float* p, float* v, const float* g, act_t* pbf, size_t n, long long outer, long long inner, int H,
                const int* full_cnt, float lr, float mom, int* err, cudaStream_t st);
void launch_f32_to_act(const float* in, act_t* out, size_t n, cudaStream_t st);
void launch_f64_to_f32(const double* in, float* out, size_t n, cudaStream_t st);
// LoRA (lora.cu): W_eff = W + s D U into the fp16 q/k/v operand rows; adapter
// gradients from G7's q/k/v weight gradient
void launch_lora_merge(const Dims& D, int rank, float scaling, const float* W1T, const float* A, act_t* W1T_bf,
                       cudaStream_t st);
void launch_lora_score(const Dims& D, int rank, const float* A, const float* AG, int fwd_metric, int bwd_metric,
                       int unit, int n_units, double* fo, double* bo, cudaStream_t st);
void launch_lora_grad(const Dims& D, int rank, float scaling, const float* G1T, const float* A, float* AG,
                      const int* full_cnt, cudaStream_t st);

// scoring pre-pass (step_gemms.cuh S5 / S7 + these): bias parts of the unit
// gradients, WeightMagnitude per head-subnet, and the K x n_units tables
void launch_score_bias(const Dims& D, int mbs, int n_units, const float* part_db1, const float* part_cs,
                       const float* b1, const float* b2, float* part, cudaStream_t st);
void launch_score_weight(const Dims& D, const float* W1T, const float* W2T, const float* b1, const float* b2,
                         double* wm, cudaStream_t st);
void launch_score_reduce(const Dims& D, int n_units, const float* p7, const float* p5, const float* pb,
                         const double* wm, int fwd_metric, int bwd_metric, double* fwd_out, double* bwd_out,
                         cudaStream_t st);

}  // namespace d2ft_b200
