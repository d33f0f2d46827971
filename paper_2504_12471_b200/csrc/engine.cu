// D2FT step engine: one fine-tuning step of the subnet-partitioned model on
// one B200 (trainer.cpp:214-292 for the D2FT policy), device resident.
//
//   schedule (fused knapsack kernel) -> expand to per-sample codes -> compaction
//   -> embed GEMM -> L x [LN, G1, attention, G3] -> head/CE
//   -> L x [G4, attention bwd, G5, G7, G8, bias sums, LN bwd]
//   -> embed wgrad -> SGD-momentum on touched subnets (+ act_t operand copies)
//
// Parameters live as fp32 masters in an arena laid out for the GEMMs (see
// DESIGN.md §3); the canonical fp64 flat vector of the reference
// (model.hpp:117-153) is the interchange format at the C-ABI.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <chrono>

#include "../../include/d2ft_b200.h"
#include "../../include/d2ft_b200_engine.h"
#include "common.cuh"
#include "exchange.cuh"
#include "gemm_sm100.cuh"
#include "sched.cuh"
#include "step_common.cuh"
#include "step_gemms.cuh"
#include "step_kernels.cuh"

constexpr int kG7BN = 224;  // G7 N tile: PQ = 448 = 2 x 224 (ViT-B/L)
#ifndef D2FT_CG2
#define D2FT_CG2 1  // pair UMMA (cta_group::2) for the K-major-B GEMMs; 0 = B multicast (experiment builds)
#endif
constexpr int kCG2 = D2FT_CG2;
#ifndef D2FT_CG2_BMN
#define D2FT_CG2_BMN 1  // pair UMMA also for the MN-major-B GEMMs (G3, G8)
#endif
constexpr int kCG2Bmn = D2FT_CG2_BMN;
#ifndef D2FT_CG_STAGES_208
#define D2FT_CG_STAGES_208 6  // pipeline stages of the pair-UMMA N = 208 GEMMs (G3, G4, G8)
#endif
constexpr int kCGStages208 = D2FT_CG_STAGES_208;
#ifndef D2FT_BMN_ROUND
#define D2FT_BMN_ROUND 0
#endif
constexpr int kBmnRound = D2FT_BMN_ROUND;
#ifndef D2FT_EPI_WIDE_STAGES
#define D2FT_EPI_WIDE_STAGES 3  // pipeline stages of a staged-epilogue GEMM with > 2 epilogue warpgroups
#endif
constexpr int kEpiWideStages = D2FT_EPI_WIDE_STAGES;
// SGD in the G5 / G7 epilogues: opt-in.  Correct (the GPU suite passes with
// it on) but measured slower on the ViT-B step: 7.89 vs 5.59 ms — G5's
// row-per-thread epilogue turns the p / v read-modify-write into
// uncoalesced scalar traffic (0.52 -> 2.87 ms) and G7's coalesced one still
// does not hide 18 B / weight under its MMAs (0.59 -> 0.99 ms), against a
// separate streaming SGD pass of 0.30 ms for those weights.
#ifndef D2FT_FUSE_SGD
#define D2FT_FUSE_SGD 0
#endif
constexpr bool kFuseSgd = D2FT_FUSE_SGD;
#ifndef D2FT_G5_EPI
#define D2FT_G5_EPI 4
#endif
#ifndef D2FT_G7_EPI
#define D2FT_G7_EPI 4
#endif
#ifndef D2FT_G4_PAIR
#define D2FT_G4_PAIR 1
#endif
#ifndef D2FT_G8_EPI
#define D2FT_G8_EPI 4
#endif
#ifndef D2FT_G1_EPI
#define D2FT_G1_EPI 2  // epilogue warpgroups of the G1 GEMM (experiment builds vary it)
#endif
// G1 with the sample's xn resident in shared memory across its unit groups
// (GemmShape RES, pair UMMA): d = 768 (12 k-blocks) and T <= 208 only.
// Opt-in: correct (step parity suite) but slower — 156 KB of resident B
// leaves room for only 2 weight stages (G1 1.16 vs 0.95 ms per step) or 3
// with 16-token epilogue chunks (0.99), DESIGN.md §10.
#ifndef D2FT_G1_RESB
#define D2FT_G1_RESB 0
#endif
#ifndef D2FT_G1_RES_STAGES
#define D2FT_G1_RES_STAGES 2
#endif
// G1 on pair UMMA (B split between the pair instead of multicast, 6 stages
// instead of 4) at T <= 208: G1 0.875-0.885 vs 0.906-0.909 ms per step on one
// box (two A/B runs), step -0.4%.  0 = the multicast pair of gemm_tokN.
#ifndef D2FT_G1_PAIR
#define D2FT_G1_PAIR 1
#endif
// G4 in the resident-B mode (the sample's dC half kept in shared memory
// across its unit groups, static contiguous tile ranges): opt-in; correct on
// the step parity suite, but 3 stages fit: G4 0.634 vs 0.546 ms per step
#ifndef D2FT_G4_RESB
#define D2FT_G4_RESB 0
#endif
#ifndef D2FT_G1_PAIR_STAGES
#define D2FT_G1_PAIR_STAGES 6
#endif

namespace d2ft_b200 {

namespace {

template <typename T>
T* dalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  if (n == 0) n = 1;
  D2FT_CUDA(cudaMalloc(&p, n * sizeof(T) + 256));
  D2FT_CUDA(cudaMemset(p, 0, n * sizeof(T) + 256));
  owned.push_back(p);
  return static_cast<T*>(p);
}

// Phases timed when profiling is on (d2ft_engine_phase_ms).
enum Phase {
  PH_SCHED,
  PH_EMBED,
  PH_LN,
  PH_G1,
  PH_ATTN_F,
  PH_G3,
  PH_HEAD,
  PH_G4,
  PH_ATTN_B,
  PH_G5,
  PH_G7,
  PH_G8,
  PH_BIAS,
  PH_LN_BWD,
  PH_EMBED_W,
  PH_SGD,
  PH_EXCH,  // head-partition exchange (partitioned engines only)
  PH_COUNT
};

}  // namespace

struct Engine {
  Dims D{};
  int Kmax_mb;  // scheduler items capacity (= Bmax)
  int KS = 8;   // embed wgrad split
  int BNt;      // token tile (UMMA N) of the tokens-as-N GEMMs
  std::vector<void*> owned;
  cudaStream_t st = nullptr;

  // parameter arena segments (fp32 masters, velocity, gradient share offsets)
  struct Seg {
    size_t off, n;
    long long outer, inner;
  };
  enum { S_W1T, S_B1, S_W2T, S_B2, S_WET, S_BE, S_POS, S_WC, S_BC, S_N };
  Seg seg[S_N];
  size_t nparam = 0;
  float *P = nullptr, *V = nullptr, *G = nullptr;
  // LoRA (lora.cu): adapter arena [L][H][down_q|up_q|down_k|up_k|down_v|up_v],
  // velocity and gradient; rank 0 = no adapters attached
  int lora_rank = 0;
  float lora_scaling = 0.f;
  float *LA = nullptr, *LV = nullptr, *LG = nullptr;
  size_t lora_per() const { return 3 * ((size_t)D.d * lora_rank + (size_t)lora_rank * D.dh); }
  size_t lora_count() const { return (size_t)D.L * D.H * lora_per(); }
  act_t *W1T_bf, *W2T_bf, *WeT_bf;  // fp16 operand copies (G4 / G8 read W2T / W1T MN-major)
  // opt-in p_s surrogate (step_gemms.cuh Sur1 / Sur2): rank 0 = the
  // reference's pure bypass; SurA [L][H*R][d], SurB [L][d][H*R], U [Bmax][H*R][TP]
  int sur_rank = 0;
  act_t *SurA = nullptr, *SurB = nullptr, *SurU = nullptr;
  CUtensorMap tm_SA, tm_SB, tm_U64;

  // activations
  float* x;       // [L+1][Bmax][T][d]
  float* stats;   // [L][Bmax][T][2]
  act_t* xn;  // [L][Bmax][T][d] (G1's B; G7's A read MN-major)
  act_t *QKV, *ZT, *OGT;
  float* lse;     // [L][Bmax][H][T]
  float* O32T = nullptr;  // [L][Bmax][H][64][TP] fp32 attention output of Full cells (tcgen05 path)
  act_t *inp, *inpT;
  float* samples_dev;
  // input pipeline: the next batch's samples are copied H2D on a copy stream
  // into samples_stage while the current batch computes (d2ft_engine_prefetch)
  float* samples_stage = nullptr;
  double* stage64 = nullptr;  // fp64 Dataset samples of the next batch, gathered H2D (prefetch_units)
  cudaStream_t cst = nullptr;
  // side stream: G5 (dW of [Wo;W2]) only needs the incoming gradient dC and
  // the forward's [O|g], so it runs beside G4 / attention backward / G7 / G8
  // and joins before the LN backward overwrites dC
  cudaStream_t st2 = nullptr;
  std::vector<cudaEvent_t> side_ev;  // [5L+1]: G5 fork / join, G7 fork / join, G8 done per block; final join
  // G7 (dW of [Wq|Wk|Wv|W1]) also runs on the side stream, forked after the
  // attention backward and joined before the next block's G4 overwrites dY1T.
  // The weight-gradient GEMMs then fill the critical path's tails (the
  // attention backward's last round, G4 / G8 ramps), and each block's weight
  // SGD follows its G7 there instead of ending the step: ViT-B 5.25 vs
  // 5.47 ms per step (5.49 before the per-block SGD; G5 alone 5.46; same box,
  // tools/ab_side.sh).
  // D2FT_NO_SIDE / D2FT_NO_SIDE_G7 turn them off; D2FT_SIDE_CTAS caps the side
  // kernels' grids (64: 5.66 ms — fewer SMs, same long tiles).  Default cap:
  // all SMs but 20 (128 of 148), which stay free for the critical path's
  // kernels: −0.05 ms per step on average over six paired same-box runs of
  // the final build, every pair in its favour (112 and 96 in between, 0 =
  // uncapped the slowest; 120-144 within run-to-run noise of 128).
  bool use_side = getenv("D2FT_NO_SIDE") == nullptr;
  int side_ctas = getenv("D2FT_SIDE_CTAS") ? atoi(getenv("D2FT_SIDE_CTAS")) : -1;  // -1: num_sms() - 20
  bool side_g7 = getenv("D2FT_NO_SIDE_G7") == nullptr;
  // grid cap of a side-stream GEMM (launch_gemm's max_ctas: > 0 caps, 0 = all SMs)
  int side_cap() const { return side_ctas >= 0 ? side_ctas : (num_sms() > 40 ? num_sms() - 20 : 0); }
  cudaEvent_t ev_copied = nullptr, ev_stage_free = nullptr;
  bool have_prefetch = false;
  int prefetch_B = 0;
  std::vector<int32_t> prefetched_units;  // the units of a Dataset prefetch (empty: a host-buffer prefetch)
  int* labels_dev;
  float* logits_dev;  // [Bmax][C] head logits of the last forward (d2ft_engine_logits)
  // backward scratch
  float *dX, *dxn, *part_cs, *part_db1, *part_ew;
  act_t *dC, *dO, *dY1T;  // dC: G4's B, G5's / EmbedW's A (read MN-major)
  double *loss_s, *loss;
  float *pooled, *dlog;
  // schedule / compaction
  double *bwd_dev, *fwd_dev;
  int32_t *cf_dev, *cb_dev, *capf_dev, *capo_dev;
  uint8_t *codes_mb, *codes_exp;
  int32_t* lists_mem;
  CompactLists lists{};
  int *g1_tiles, *g1_count, *g4_tiles, *g4_count;
  int *ord_act, *ord_full, *ord_head;  // cost orders (plan_kernel)
  int *af_items, *af_count, *ab_items, *ab_count;  // attention work lists (plan_kernel)
  // head partition (exchange.cuh): null = the whole model on this GPU
  std::unique_ptr<Exchange> ex;
  CUtensorMap* store_maps;  // device copies of the epilogue bulk-store maps: [0] ZT, [1] OGT, [2] QKV (G1), [3] dO, [4] dY1T (G4)
  int* full_any;  // [B][L] Full heads of the sample in the block over ALL ranks (LN-backward gate)
  // Partitioned whenever an exchange is attached, world 1 included: the
  // partition's data path (owner mask, fp32 partial sums, the all-reduce
  // call) then runs on a one-GPU box as well.
  bool partitioned() const { return ex != nullptr; }
  // data parallelism (d2ft_engine_data_parallel_*): rank r of W holds micro-
  // batches [r*n_mb/W, (r+1)*n_mb/W) of the GLOBAL batch, every rank runs the
  // same knapsack over the global score table, and the weight gradients are
  // all-reduced before the SGD — the global batch's trainer step
  // (trainer.cpp:247-268) with the per-sample work split across GPUs.
  std::unique_ptr<Exchange> dpx;
  int dp_mb0 = 0;      // first global micro-batch of this rank (current step)
  int B_glob = 0;      // samples of the global batch (the 1/B loss weight)
  int Nmax = 0;        // micro-batch columns the score / code tables hold (Bmax; world x Bmax when data parallel)
  // (re)size the K x Nmax score and code tables (device and pinned host)
  void size_tables(int nmax) {
    D2FT_CUDA(cudaStreamSynchronize(st));
    const size_t K = (size_t)D.K();
    for (void* q : {(void*)bwd_dev, (void*)codes_mb})
      if (q) {
        owned.erase(std::find(owned.begin(), owned.end(), q));
        cudaFree(q);
      }
    if (h_scores) cudaFreeHost(h_scores);
    if (h_codes) cudaFreeHost(h_codes);
    bwd_dev = dalloc<double>(2 * K * nmax, owned);
    fwd_dev = bwd_dev + K * nmax;
    codes_mb = dalloc<uint8_t>(K * nmax, owned);
    D2FT_CUDA(cudaMallocHost(&h_scores, 2 * K * nmax * sizeof(double)));
    D2FT_CUDA(cudaMallocHost(&h_codes, K * nmax));
    Nmax = nmax;
    sched_max_cols = 0;  // decision-bit workspace sized again for the new tables
    drop_graph();
  }
  int* full_cnt_glob = nullptr;  // [K] Full cells per row over the global batch (SGD touch rule)
  std::vector<cudaEvent_t> dp_ev;  // [L] block l's weight gradients complete, [L] the step's gradients all-reduced
  cudaEvent_t dp_event(int i) {
    if (dp_ev.empty()) {
      dp_ev.resize(D.L + 1);
      for (auto& e : dp_ev) D2FT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return dp_ev[i];
  }
  bool data_parallel() const { return dpx != nullptr; }
  // samples this rank holds for a global batch of n_mb micro-batches of mbs
  int local_B(int n_mb, int mbs) {
    D2FT_REQUIRE(n_mb >= 1 && mbs >= 1, kConfig, "train: batch_size must be a positive multiple of micro_batch_size");
    B_glob = n_mb * mbs;
    if (!dpx) {
      dp_mb0 = 0;
      return n_mb * mbs;
    }
    D2FT_REQUIRE(n_mb % dpx->world == 0, kConfig,
                 "data parallel: the micro-batches of a batch must divide evenly over the ranks");
    dp_mb0 = dpx->rank * (n_mb / dpx->world);
    return n_mb / dpx->world * mbs;
  }
  int* row_owner = nullptr;  // [K] rank owning scheduled row k (partition mapping, partition.py)
  // Exchange stream and chunks: G3 / G8 run per sample chunk [c*B/C, (c+1)*B/C)
  // and each chunk's all-reduce runs on xst while the next chunk computes;
  // the LayerNorm of a chunk waits only for that chunk's sum.
  static constexpr int kMaxXChunks = 8;
  cudaStream_t xst = nullptr;
  int xchunks = getenv("D2FT_EXCH_CHUNKS") ? atoi(getenv("D2FT_EXCH_CHUNKS")) : 2;
  std::vector<cudaEvent_t> xev;  // [dir][L][chunk][ready, done]
  int active_chunks() const {
    if (!partitioned() || profiling) return 1;
    return std::max(1, std::min(std::min(xchunks, kMaxXChunks), D.B));
  }
  int chunk_lo(int c, int C) const { return (int)((long long)c * D.B / C); }
  bool async_exchange() const { return partitioned() && !profiling; }
  cudaEvent_t xevent(int dir, int l, int c, int kind) {
    if (xev.empty()) {
      xev.resize((size_t)2 * D.L * kMaxXChunks * 2);
      for (auto& e : xev) D2FT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return xev[(((size_t)dir * D.L + l) * kMaxXChunks + c) * 2 + kind];
  }
  // exchange of rows [lo, lo+n) of a [B][T][d] fp32 buffer after the producer
  // (on st) finished them: on xst with events, or inline when profiling
  void exchange_chunk(int dir, int l, int c, float* buf, int lo, int n) {
    const size_t row = (size_t)D.T * D.d;
    if (!async_exchange()) {
      mark(PH_EXCH);
      ex->allreduce_sum(buf + (size_t)lo * row, (size_t)n * row, st);
      return;
    }
    D2FT_CUDA(cudaEventRecord(xevent(dir, l, c, 0), st));
    D2FT_CUDA(cudaStreamWaitEvent(xst, xevent(dir, l, c, 0), 0));
    ex->allreduce_sum(buf + (size_t)lo * row, (size_t)n * row, xst);
    D2FT_CUDA(cudaEventRecord(xevent(dir, l, c, 1), xst));
  }
  void wait_exchange(int dir, int l, int c) {
    if (async_exchange()) D2FT_CUDA(cudaStreamWaitEvent(st, xevent(dir, l, c, 1), 0));
  }
  int* ctrs;                           // dynamic tile counters: [L][8] + 8, zeroed per pass
                                       // (the variable-K GEMMs; uniform ones stay static),
                                       // then [L][2][kMaxXChunks] for the chunked G3 / G8
  enum { C_G3, C_G5, C_G7, C_G8, C_G4 };
  int* ctr(int l, int kind) { return ctrs + (l < 0 ? (size_t)D.L * 8 : (size_t)l * 8) + kind; }
  int* xctr(int l, int dir, int c) { return ctrs + (size_t)(D.L + 1) * 8 + ((size_t)l * 2 + dir) * kMaxXChunks + c; }
  size_t ctr_count() const { return (size_t)(D.L + 1) * 8 + (size_t)D.L * 2 * kMaxXChunks; }
  uint32_t* sched_bits = nullptr;
  size_t sched_bits_words = 0;
  unsigned int* sched_counter;
  int* err;
  float* gmax;  // running max |dX_L| -> gradient scale S
  int sched_max_cols = 0;
  // pinned staging
  float* h_samples = nullptr;
  int* h_labels = nullptr;
  double* h_scores = nullptr;
  // Dataset-path staging, double-buffered: batch i+1's labels, score slice
  // (bwd at 0, fwd at K * Nmax, as on the device) and cost / capacity rows
  // are gathered and validated while batch i computes (units_step)
  int* u_lab[2] = {nullptr, nullptr};
  double* u_sc[2] = {nullptr, nullptr};
  int32_t* u_caps[2] = {nullptr, nullptr};
  struct UnitsPrep {
    bool valid = false;
    int buf = 0, n_mb = 0, mbs = 0, total_units = 0;
    const void* ds = nullptr;
    const double *bwd = nullptr, *fwd = nullptr;
    std::vector<int32_t> units;
  } prep;
  int ubuf = 0;
  void ensure_units_staging() {
    if (u_lab[0]) return;
    const size_t K = (size_t)D.K();
    for (int b = 0; b < 2; ++b) {
      D2FT_CUDA(cudaMallocHost(&u_lab[b], (size_t)D.Bmax * sizeof(int)));
      D2FT_CUDA(cudaMallocHost(&u_sc[b], 2 * K * Nmax * sizeof(double)));
      D2FT_CUDA(cudaMallocHost(&u_caps[b], 4 * K * sizeof(int32_t)));
    }
  }
  double* h_loss = nullptr;
  int* h_err = nullptr;
  uint8_t* h_codes = nullptr;

  // tensor maps
  CUtensorMap tm_WeT, tm_inp, tm_W1T, tm_xn, tm_xn64, tm_W2T, tm_dC, tm_dC64, tm_OGT, tm_OGT64, tm_dY1T, tm_dY1Tb,
      tm_Q, tm_K, tm_V, tm_dO, tm_inpT;

  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_phase;
  double phase_ms[PH_COUNT] = {};
  int profiled_steps = 0;

  // CUDA graph of one compute step (schedule + forward/backward + SGD) for a
  // fixed (batch, micro-batch size, lr, momentum): the ~150 launches of a
  // step replay without host launch overhead or inter-kernel gaps.  Eager
  // when profiling (per-phase events) or partitioned (host-side exchange).
  cudaGraphExec_t gexec = nullptr;
  int g_nmb = -1, g_mbs = -1;
  float g_lr = 0.f, g_mom = 0.f;
  unsigned long long g_kernels = 0;  // kernels per replay (for d2ft_launch_count)
  unsigned long long g_xcalls = 0, g_xbytes = 0;  // exchange calls / bytes per replay (partitioned)
  bool use_graphs = getenv("D2FT_NO_GRAPH") == nullptr;
  // opt-in (D2FT_PDL=1): measured slower on the ViT-B step (6.13 / 5.96 ms with
  // early / implicit trigger vs 5.88 ms plain graph edges)
  bool use_pdl = getenv("D2FT_PDL") != nullptr;

  // kernel -> kernel edges of the captured step become programmatic
  // (programmatic dependent launch): the successor launches as soon as every
  // CTA of its predecessor has started (pdl_trigger at kernel entry) and runs
  // its prologue (barrier init, TMEM allocation, descriptor prefetch) on the
  // SMs the predecessor's tail leaves idle; pdl_wait orders the data.
  static void make_edges_programmatic(cudaGraph_t g) {
    size_t n = 0;
    D2FT_CUDA(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &n));
    std::vector<cudaGraphNode_t> from(n), to(n);
    std::vector<cudaGraphEdgeData> ed(n);
    D2FT_CUDA(cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &n));
    for (size_t i = 0; i < n; ++i) {
      cudaGraphNodeType a, b;
      D2FT_CUDA(cudaGraphNodeGetType(from[i], &a));
      D2FT_CUDA(cudaGraphNodeGetType(to[i], &b));
      if (a != cudaGraphNodeTypeKernel || b != cudaGraphNodeTypeKernel || ed[i].type != cudaGraphDependencyTypeDefault)
        continue;
      D2FT_CUDA(cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &ed[i], 1));
      cudaGraphEdgeData e{};
      e.from_port = cudaGraphKernelNodePortProgrammatic;
      e.type = cudaGraphDependencyTypeProgrammatic;
      D2FT_CUDA(cudaGraphAddDependencies_v2(g, &from[i], &to[i], &e, 1));
    }
  }

  std::vector<cudaEvent_t> pool;
  void mark(int ph) {
    if (!profiling) return;
    if (ev.size() >= pool.size()) {
      cudaEvent_t e;
      D2FT_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    cudaEvent_t e = pool[ev.size()];
    D2FT_CUDA(cudaEventRecord(e, st));
    ev.push_back(e);
    ev_phase.push_back(ph);
  }
  void collect() {
    if (!profiling || ev.empty()) return;
    D2FT_CUDA(cudaEventSynchronize(ev.back()));
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      D2FT_CUDA(cudaEventElapsedTime(&ms, ev[i - 1], ev[i]));
      if (ev_phase[i - 1] < PH_COUNT) phase_ms[ev_phase[i - 1]] += ms;
    }
    ev.clear();
    ev_phase.clear();
  }

  Engine(const d2ft_model_config& c, int Bmax) {
    D2FT_REQUIRE(c.num_blocks >= 1 && c.heads_per_block >= 1 && c.model_dim >= 1 && c.ffn_hidden >= 1 &&
                     c.seq_len >= 1 && c.num_classes >= 1,
                 kConfig, "model config: all dimensions must be >= 1");
    D2FT_REQUIRE(c.model_dim % c.heads_per_block == 0, kConfig,
                 "model config: model_dim must be divisible by heads_per_block");
    D2FT_REQUIRE(c.ffn_hidden % c.heads_per_block == 0, kConfig,
                 "model config: ffn_hidden must be divisible by heads_per_block");
    D.L = c.num_blocks;
    D.H = c.heads_per_block;
    D.d = c.model_dim;
    D.ffn = c.ffn_hidden;
    D.T = c.seq_len;
    D.C = c.num_classes;
    D.dh = D.d / D.H;
    D.fs = D.ffn / D.H;
    D2FT_REQUIRE(D.d % 128 == 0 && D.d <= 1024, kConfig, "b200 engine: model_dim must be a multiple of 128, <= 1024");
    D2FT_REQUIRE(D.dh == 32 || D.dh == 64, kConfig, "b200 engine: head_dim (d/H) must be 32 or 64");
    D2FT_REQUIRE(D.fs % 32 == 0, kConfig, "b200 engine: ffn slice (ffn/H) must be a multiple of 32");
    D2FT_REQUIRE(D.T <= 256, kConfig, "b200 engine: seq_len must be <= 256");
    D2FT_REQUIRE(D.H <= 16, kConfig, "b200 engine: at most 16 heads per block");
    D2FT_REQUIRE(D.C <= 64, kConfig, "b200 engine: at most 64 classes");
    D2FT_REQUIRE(Bmax >= 1 && Bmax <= 1024, kConfig, "b200 engine: batch capacity must be in [1, 1024]");
    D.PQ = 3 * D.dh + D.fs;
    D.PO = D.dh + D.fs;
    D.UQ = (D.PQ + 63) / 64;
    D.UO = (D.PO + 63) / 64;
    D.TP = (D.T + 7) / 8 * 8;
    D.TQ = (D.T + 15) / 16 * 16;
    D.TB = (D.T + 63) / 64;
    D.Bmax = Bmax;
    D.B = Bmax;
    Kmax_mb = Bmax;
    BNt = D.T <= 64 ? 64 : D.T <= 128 ? 128 : D.T <= 208 ? 208 : 256;
    KS = std::min(8, Bmax);
    {
      int least = 0, greatest = 0;
      D2FT_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      // the step's critical path runs at the highest priority; the off-path
      // weight-gradient GEMMs (side stream) fill the SMs it leaves idle
      D2FT_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, greatest));
      D2FT_CUDA(cudaStreamCreateWithPriority(&st2, cudaStreamNonBlocking, least));
    }
    D2FT_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
    D2FT_CUDA(cudaEventCreateWithFlags(&ev_copied, cudaEventDisableTiming));
    D2FT_CUDA(cudaEventCreateWithFlags(&ev_stage_free, cudaEventDisableTiming));
    alloc_all();
    make_maps();
  }

  ~Engine() {
    for (auto e : pool) cudaEventDestroy(e);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (st) cudaStreamSynchronize(st);
    for (void* p : owned) cudaFree(p);
    if (h_samples) cudaFreeHost(h_samples);
    if (h_labels) cudaFreeHost(h_labels);
    if (h_scores) cudaFreeHost(h_scores);
    for (int b = 0; b < 2; ++b) {
      if (u_lab[b]) cudaFreeHost(u_lab[b]);
      if (u_sc[b]) cudaFreeHost(u_sc[b]);
      if (u_caps[b]) cudaFreeHost(u_caps[b]);
    }
    if (h_loss) cudaFreeHost(h_loss);
    if (h_err) cudaFreeHost(h_err);
    if (h_codes) cudaFreeHost(h_codes);
    if (cst) cudaStreamSynchronize(cst);
    if (ev_copied) cudaEventDestroy(ev_copied);
    if (ev_stage_free) cudaEventDestroy(ev_stage_free);
    if (cst) cudaStreamDestroy(cst);
    for (auto e : side_ev) cudaEventDestroy(e);
    for (auto e : xev) cudaEventDestroy(e);
    for (auto e : dp_ev) cudaEventDestroy(e);
    ex.reset();  // the communicators before their stream
    dpx.reset();
    if (xst) cudaStreamDestroy(xst);
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }

  void alloc_all() {
    const size_t L = D.L, H = D.H, d = D.d, T = D.T, Bm = D.Bmax, PQ = D.PQ, PO = D.PO, TP = D.TP, fs = D.fs;
    size_t off = 0;
    auto add = [&](int id, size_t n, long long outer, long long inner) {
      seg[id] = Seg{off, n, outer, inner};
      off += (n + 63) / 64 * 64;
    };
    add(S_W1T, L * H * PQ * d, (long long)(H * PQ * d), (long long)(PQ * d));
    add(S_B1, L * H * fs, (long long)(H * fs), (long long)fs);
    add(S_W2T, L * d * H * PO, (long long)(d * H * PO), (long long)PO);
    add(S_B2, L * d, (long long)d, (long long)(d / H));
    add(S_WET, d * d, 0, 1);
    add(S_BE, d, 0, 1);
    add(S_POS, T * d, 0, 1);
    add(S_WC, d * D.C, 0, 1);
    add(S_BC, D.C, 0, 1);
    nparam = off;
    P = dalloc<float>(nparam, owned);
    V = dalloc<float>(nparam, owned);
    G = dalloc<float>(nparam, owned);
    W1T_bf = dalloc<act_t>(L * H * PQ * d, owned);
    W2T_bf = dalloc<act_t>(L * d * H * PO, owned);
    WeT_bf = dalloc<act_t>(d * d, owned);

    x = dalloc<float>((L + 1) * Bm * T * d, owned);
    stats = dalloc<float>(L * Bm * T * 2, owned);
    xn = dalloc<act_t>(L * Bm * T * d, owned);
    QKV = dalloc<act_t>(L * Bm * H * T * 3 * D.dh, owned);
    ZT = dalloc<act_t>(L * Bm * H * fs * TP, owned);
    OGT = dalloc<act_t>(L * Bm * H * PO * TP, owned);
    lse = dalloc<float>(L * Bm * H * T, owned);
    if (D.dh == 64) O32T = dalloc<float>(L * Bm * H * 64 * TP, owned);
    inp = dalloc<act_t>(Bm * T * d, owned);
    inpT = dalloc<act_t>(Bm * d * TP, owned);
    samples_dev = dalloc<float>(Bm * T * d, owned);
    samples_stage = dalloc<float>(Bm * T * d, owned);
    labels_dev = dalloc<int>(Bm, owned);

    dX = dalloc<float>(Bm * T * d, owned);
    dxn = dalloc<float>(Bm * T * d, owned);
    const size_t ntile = (T + 31) / 32;
    // per-slot partial sums, reduced for all blocks in one launch after the
    // backward loop: part_cs slot l = column sums of the gradient entering
    // block l (slot L: entering the embedding), part_db1 slot l = G4 partials
    part_cs = dalloc<float>((L + 1) * Bm * ntile * d, owned);
    part_db1 = dalloc<float>(L * (size_t)kG4Epi * Bm * H * fs, owned);
    part_ew = dalloc<float>((size_t)KS * d * d, owned);
    dC = dalloc<act_t>(Bm * T * d, owned);
    dO = dalloc<act_t>(Bm * H * T * D.dh, owned);
    dY1T = dalloc<act_t>(Bm * H * PQ * TP, owned);
    loss_s = dalloc<double>(Bm, owned);
    loss = dalloc<double>(1, owned);
    pooled = dalloc<float>(Bm * d, owned);
    dlog = dalloc<float>(Bm * D.C, owned);
    logits_dev = dalloc<float>(Bm * D.C, owned);

    const size_t K = (size_t)D.K();
    // the two score tables and the four per-row cost / capacity vectors are
    // one allocation each, so a staged batch reaches the device in two copies
    bwd_dev = dalloc<double>(2 * K * Bm, owned);
    fwd_dev = bwd_dev + K * Bm;
    Nmax = (int)Bm;
    cf_dev = dalloc<int32_t>(4 * K, owned);
    cb_dev = cf_dev + K;
    capf_dev = cf_dev + 2 * K;
    capo_dev = cf_dev + 3 * K;
    codes_mb = dalloc<uint8_t>(K * Bm, owned);
    codes_exp = dalloc<uint8_t>(K * Bm, owned);
    const size_t cells = Bm * L;
    lists_mem = dalloc<int32_t>(2 * K * Bm + 2 * K + 2 * cells * H + 2 * cells, owned);
    int32_t* p = lists_mem;
    lists.fwd_idx = p;
    p += K * Bm;
    lists.full_idx = p;
    p += K * Bm;
    lists.fwd_cnt = p;
    p += K;
    lists.full_cnt = p;
    p += K;
    lists.act_heads = p;
    p += cells * H;
    lists.full_heads = p;
    p += cells * H;
    lists.act_cnt = p;
    p += cells;
    lists.full_hcnt = p;
    g1_tiles = dalloc<int>(L * Bm * ((D.UQ * H + 1) / 2), owned);
    g4_tiles = dalloc<int>(L * Bm * ((D.UO * H + 1) / 2), owned);
    g1_count = dalloc<int>(L, owned);
    g4_count = dalloc<int>(L, owned);
    ord_act = dalloc<int>(L * Bm, owned);
    ord_full = dalloc<int>(L * Bm, owned);
    ord_head = dalloc<int>(L * H, owned);
    ctrs = dalloc<int>(ctr_count(), owned);
    row_owner = dalloc<int>(L * H, owned);
    full_any = dalloc<int>(L * Bm, owned);
    store_maps = dalloc<CUtensorMap>(8, owned);
    af_items = dalloc<int>(L * Bm * H, owned);
    ab_items = dalloc<int>(L * Bm * H, owned);
    af_count = dalloc<int>(L, owned);
    ab_count = dalloc<int>(L, owned);
    sched_counter = dalloc<unsigned int>(1, owned);
    err = dalloc<int>(1, owned);
    gmax = dalloc<float>(1, owned);

    D2FT_CUDA(cudaMallocHost(&h_samples, Bm * T * d * sizeof(float)));
    D2FT_CUDA(cudaMallocHost(&h_labels, Bm * sizeof(int)));
    D2FT_CUDA(cudaMallocHost(&h_scores, 2 * K * Bm * sizeof(double)));
    D2FT_CUDA(cudaMallocHost(&h_loss, sizeof(double)));
    D2FT_CUDA(cudaMallocHost(&h_err, sizeof(int)));
    D2FT_CUDA(cudaMallocHost(&h_codes, K * Bm));
  }

  void make_maps() {
    const uint64_t L = D.L, H = D.H, d = D.d, T = D.T, Bm = D.Bmax, PQ = D.PQ, PO = D.PO, TP = D.TP;
    // A operands (box 64 rows)
    tm_WeT = make_tmap_f16_3d(WeT_bf, d, d, 1, d * 2, d * d * 2, 64);
    tm_W1T = make_tmap_f16_3d(W1T_bf, d, H * PQ, L, d * 2, H * PQ * d * 2, 64);
    tm_W2T = make_tmap_f16_3d(W2T_bf, H * PO, d, L, H * PO * 2, d * H * PO * 2, 64);
    // MN-major A (64 M x 64 K boxes): dC for G5 / EmbedW, xn for G7
    tm_dC64 = make_tmap_f16_3d(dC, d, T, Bm, d * 2, T * d * 2, 64);
    tm_xn64 = make_tmap_f16_3d(xn, d, T, L * Bm, d * 2, T * d * 2, 64);
    tm_dY1T = make_tmap_f16_3d(dY1T, T, PQ, Bm * H, TP * 2, PQ * TP * 2, 64);
    // B operands, tokens as N (box BNt/2: each CTA of a pair loads half, multicast)
    tm_inp = make_tmap_f16_3d(inp, d, T, Bm, d * 2, T * d * 2, BNt / 2);
    tm_xn = make_tmap_f16_3d(xn, d, T, L * Bm, d * 2, T * d * 2, BNt / 2);
    tm_dC = make_tmap_f16_3d(dC, d, T, Bm, d * 2, T * d * 2, BNt / 2);
    // attention operands (tcgen05 path, dh = 64): Q / K / V column blocks of the QKV rows
    if (D.dh == 64) {
      const uint64_t W = 3 * D.dh;
      tm_Q = make_tmap_f16_3d(QKV, W, T, L * Bm * H, W * 2, T * W * 2, 128);
      tm_K = make_tmap_f16_3d(QKV, W, T, L * Bm * H, W * 2, T * W * 2, D.TQ);
      tm_V = make_tmap_f16_3d(QKV, W, T, L * Bm * H, W * 2, T * W * 2, 64);
      tm_dO = make_tmap_f16_3d(dO, D.dh, T, Bm * H, D.dh * 2, T * D.dh * 2, D.TQ);
    }
    {  // G1 epilogue bulk stores: 32 tokens x 32 feature rows (feature-major) or
       // 32 features x 32 tokens (token-major QKV), clipped at T
      CUtensorMap sm[6];
      constexpr int cw = G1<208>::kChunk;
#ifndef D2FT_EXP_G1_HALFBOX
      sm[0] = make_tmap_store_f16_3d(ZT, T, D.fs, L * Bm * H, TP * 2, D.fs * TP * 2, cw, 32, cw * 2);
      sm[1] = make_tmap_store_f16_3d(OGT, T, PO, L * Bm * H, TP * 2, PO * TP * 2, cw, 32, cw * 2);
      sm[2] = make_tmap_store_f16_3d(QKV, 3 * D.dh, T, L * Bm * H, 3 * D.dh * 2, T * 3 * D.dh * 2, 32, cw);
#else  // experiment: same store count, half the bytes (results wrong; timing only)
      sm[0] = make_tmap_store_f16_3d(ZT, T, D.fs, L * Bm * H, TP * 2, D.fs * TP * 2, cw / 2, 32, cw);
      sm[1] = make_tmap_store_f16_3d(OGT, T, PO, L * Bm * H, TP * 2, PO * TP * 2, cw / 2, 32, cw);
      sm[2] = make_tmap_store_f16_3d(QKV, 3 * D.dh, T, L * Bm * H, 3 * D.dh * 2, T * 3 * D.dh * 2, 32, cw / 2);
#endif
      // G4 epilogue: dO (token-major) and the dz rows of dY1T (feature-major)
      sm[3] = make_tmap_store_f16_3d(dO, D.dh, T, Bm * H, D.dh * 2, T * D.dh * 2, 32, 32);
      sm[4] = make_tmap_store_f16_3d(dY1T, T, PQ, Bm * H, TP * 2, PQ * TP * 2, 32, 32, 64);
      // G5 epilogue: the [Wo;W2] weight-gradient rows (fp32, [L][d][H*PO])
      sm[5] = make_tmap_store_f32_3d(G + seg[S_W2T].off, (uint64_t)H * PO, d, L, (uint64_t)H * PO * 4,
                                     (uint64_t)d * H * PO * 4, 16, 32, 64);
      D2FT_CUDA(cudaMemcpy(store_maps, sm, sizeof(sm), cudaMemcpyHostToDevice));
    }
    // B operands, tokens as N read MN-major from feature-major buffers (64 x 64 boxes)
    tm_OGT64 = make_tmap_f16_3d(OGT, T, PO, L * Bm * H, TP * 2, PO * TP * 2, 64);
    // (tm_dY1T above doubles as G8's MN-major B)
    // B operands, tokens as K (half boxes, multicast)
    tm_OGT = make_tmap_f16_3d(OGT, T, PO, L * Bm * H, TP * 2, PO * TP * 2, 80);
    tm_dY1Tb = make_tmap_f16_3d(dY1T, T, PQ, Bm * H, TP * 2, PQ * TP * 2, kG7BN / 2);  // G7's B (half per CTA)
    tm_inpT = make_tmap_f16_3d(inpT, T, d, Bm, TP * 2, d * TP * 2, 128);
  }

  // ---------------------------------------------------------------- params
  // canonical flat (model.hpp:117-153) <-> arena
  template <bool kToArena>
  void convert(double* flat, std::vector<float>& a) const {
    const int L = D.L, H = D.H, d = D.d, dh = D.dh, fs = D.fs, T = D.T, C = D.C, PQ = D.PQ, PO = D.PO;
    size_t o = 0;
    auto mv = [&](size_t ai) {
      if (kToArena) a[ai] = (float)flat[o++];
      else flat[o++] = a[ai];
    };
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) mv(seg[S_WET].off + (size_t)j * d + i);  // w_embed[i][j] -> WeT[j][i]
    for (int j = 0; j < d; ++j) mv(seg[S_BE].off + j);
    for (int t = 0; t < T; ++t)
      for (int j = 0; j < d; ++j) mv(seg[S_POS].off + (size_t)t * d + j);
    for (int l = 0; l < L; ++l)
      for (int h = 0; h < H; ++h) {
        const size_t w1 = seg[S_W1T].off + ((size_t)(l * H + h) * PQ) * d;
        const size_t w2 = seg[S_W2T].off + (size_t)l * d * H * PO + (size_t)h * PO;
        for (int q = 0; q < 3; ++q)  // wq, wk, wv [d][dh] -> W1T rows q*dh + j
          for (int i = 0; i < d; ++i)
            for (int j = 0; j < dh; ++j) mv(w1 + (size_t)(q * dh + j) * d + i);
        for (int j = 0; j < dh; ++j)  // wo [dh][d] -> W2T[m][h*PO + j]
          for (int m = 0; m < d; ++m) mv(w2 + (size_t)m * H * PO + j);
        for (int i = 0; i < d; ++i)  // w1 [d][fs] -> W1T rows 3dh + j
          for (int j = 0; j < fs; ++j) mv(w1 + (size_t)(3 * dh + j) * d + i);
        for (int j = 0; j < fs; ++j) mv(seg[S_B1].off + (size_t)(l * H + h) * fs + j);
        for (int j = 0; j < fs; ++j)  // w2 [fs][d] -> W2T[m][h*PO + dh + j]
          for (int m = 0; m < d; ++m) mv(w2 + (size_t)m * H * PO + dh + j);
        for (int j = 0; j < d / H; ++j) mv(seg[S_B2].off + (size_t)l * d + h * (d / H) + j);
      }
    for (int i = 0; i < d; ++i)
      for (int c = 0; c < C; ++c) mv(seg[S_WC].off + (size_t)i * C + c);
    for (int c = 0; c < C; ++c) mv(seg[S_BC].off + c);
  }

  size_t canonical_count() const {
    const size_t d = D.d, dh = D.dh, fs = D.fs, H = D.H;
    return d * d + d + (size_t)D.T * d + (size_t)D.L * H * (3 * d * dh + dh * d + d * fs + fs + fs * d + d / H) +
           d * D.C + D.C;
  }

  // attach_lora (model.cpp:165-195) with the caller's initial adapters
  void attach_lora(int rank, double scaling, const double* init) {
    D2FT_REQUIRE(!lora_rank, kState, "lora adapters already attached");
    D2FT_REQUIRE(!data_parallel(), kState, "lora: not available on a data-parallel engine");
    D2FT_REQUIRE(rank >= 1, kConfig, "lora rank must be >= 1");
    const int cap = std::min(D.d, D.dh);
    D2FT_REQUIRE(rank <= cap, kConfig,
                 "lora rank " + std::to_string(rank) + " exceeds min(d, d/H) = " + std::to_string(cap));
    D2FT_REQUIRE(rank * D.dh <= 4096, kConfig, "lora: rank x head_dim above 4096 is not supported");
    D2FT_CUDA(cudaStreamSynchronize(st));
    lora_rank = rank;
    lora_scaling = (float)scaling;
    LA = dalloc<float>(lora_count(), owned);
    LV = dalloc<float>(lora_count(), owned);
    LG = dalloc<float>(lora_count(), owned);
    D2FT_CUDA(cudaMemsetAsync(LV, 0, lora_count() * 4, st));
    D2FT_CUDA(cudaMemsetAsync(LG, 0, lora_count() * 4, st));
    set_lora(init);
    if (gexec) {  // the captured step has no adapter work
      D2FT_CUDA(cudaGraphExecDestroy(gexec));
      gexec = nullptr;
    }
  }
  void set_lora(const double* flat) {
    std::vector<float> a(lora_count());
    for (size_t i = 0; i < a.size(); ++i) a[i] = (float)flat[i];
    D2FT_CUDA(cudaMemcpyAsync(LA, a.data(), a.size() * 4, cudaMemcpyHostToDevice, st));
    launch_lora_merge(D, lora_rank, lora_scaling, P + seg[S_W1T].off, LA, W1T_bf, st);
    D2FT_CUDA(cudaStreamSynchronize(st));
  }
  void get_lora(const float* src, double* flat) {
    std::vector<float> a(lora_count());
    D2FT_CUDA(cudaStreamSynchronize(st));
    D2FT_CUDA(cudaMemcpy(a.data(), src, a.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < a.size(); ++i) flat[i] = a[i];
  }

  void refresh_bf16_all() {
    launch_f32_to_act(P + seg[S_W1T].off, W1T_bf, seg[S_W1T].n, st);
    launch_f32_to_act(P + seg[S_W2T].off, W2T_bf, seg[S_W2T].n, st);
    launch_f32_to_act(P + seg[S_WET].off, WeT_bf, seg[S_WET].n, st);
  }

  // factors per block subnet (l, h) in scheduled order: down [d][R], up [R][d]
  void set_surrogate(int rank, const double* factors) {
    D2FT_REQUIRE(!partitioned(), kState, "surrogate: not available on a head-partitioned engine");
    D2FT_REQUIRE(rank == 0 || (rank >= 8 && rank <= 64 && rank % 8 == 0), kConfig,
                 "surrogate rank must be 0 (off) or a multiple of 8 in [8, 64]");
    D2FT_REQUIRE(rank == 0 || factors, kInput, "surrogate: null factors");
    drop_graph();
    D2FT_CUDA(cudaStreamSynchronize(st));
    if (rank == 0) {
      sur_rank = 0;
      return;
    }
    const size_t L = D.L, H = D.H, d = D.d, R = rank, HR = H * R;
    if (rank != sur_rank) {
      for (act_t* q : {SurA, SurB, SurU})
        if (q) {
          owned.erase(std::find(owned.begin(), owned.end(), (void*)q));
          cudaFree(q);
        }
      SurA = dalloc<act_t>(L * HR * d, owned);
      SurB = dalloc<act_t>(L * d * HR, owned);
      SurU = dalloc<act_t>((size_t)D.Bmax * HR * D.TP, owned);
      D2FT_CUDA(cudaMemset(SurU, 0, (size_t)D.Bmax * HR * D.TP * sizeof(act_t)));
      tm_SA = make_tmap_f16_3d(SurA, d, HR, L, d * 2, HR * d * 2, 64);
      tm_SB = make_tmap_f16_3d(SurB, HR, d, L, HR * 2, d * HR * 2, 64);
      tm_U64 = make_tmap_f16_3d(SurU, D.T, HR, D.Bmax, (uint64_t)D.TP * 2, HR * D.TP * 2, 64);
    }
    std::vector<act_t> a(L * HR * d), b(L * d * HR);
    for (size_t l = 0; l < L; ++l)
      for (size_t h = 0; h < H; ++h) {
        const double* down = factors + (l * H + h) * 2 * d * R;
        const double* up = down + d * R;
        for (size_t i = 0; i < d; ++i)
          for (size_t r = 0; r < R; ++r) {
            a[(l * HR + h * R + r) * d + i] = __float2half_rn((float)down[i * R + r]);
            b[(l * d + i) * HR + h * R + r] = __float2half_rn((float)up[r * d + i]);
          }
      }
    D2FT_CUDA(cudaMemcpy(SurA, a.data(), a.size() * sizeof(act_t), cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(SurB, b.data(), b.size() * sizeof(act_t), cudaMemcpyHostToDevice));
    sur_rank = rank;
  }

  void set_params(const double* flat) {
    std::vector<float> a(nparam, 0.f);
    convert<true>(const_cast<double*>(flat), a);
    D2FT_CUDA(cudaMemcpyAsync(P, a.data(), nparam * 4, cudaMemcpyHostToDevice, st));
    refresh_bf16_all();
    if (lora_rank) launch_lora_merge(D, lora_rank, lora_scaling, P + seg[S_W1T].off, LA, W1T_bf, st);
    D2FT_CUDA(cudaStreamSynchronize(st));
  }
  void get_arena(float* src, double* flat) {
    std::vector<float> a(nparam);
    D2FT_CUDA(cudaStreamSynchronize(st));
    D2FT_CUDA(cudaMemcpy(a.data(), src, nparam * 4, cudaMemcpyDeviceToHost));
    convert<false>(flat, a);
  }

  // ---------------------------------------------------------------- GEMM dispatch
  // Tokens-as-N GEMMs on CTA pairs; BMN = 1: B is a feature-major buffer
  // read MN-major (its 64-token blocks cost more shared memory per stage).
  // AMN = 1: A (weights) read MN-major from the other GEMM's copy.
  template <template <int> class Prob, int BMN = 0, int AMN = 0, int EPI = 4, int PAIR_UMMA = 1, class... Args>
  void gemm_tokN(const CUtensorMap& a, const CUtensorMap& b, Args... args) {
    // K-major B: pair UMMA (cta_group::2, B split across the pair, deeper
    // pipeline); MN-major B: B multicast to both CTAs of the pair.  (G1 at
    // T <= 208 launches its pair-UMMA shape directly, D2FT_G1_PAIR; other
    // token tiles keep multicast here.)
    constexpr int CG = !PAIR_UMMA ? 0 : (BMN ? kCG2Bmn : kCG2);
    // Pair UMMA with MN-major B: each CTA holds BN/2 token columns of B as
    // 64-wide swizzle blocks; a partial last block (208/2 = 104) costs a third
    // of the mainloop rate (dense core bench), so D2FT_BMN_ROUND=1 rounds the
    // tile up to whole blocks (the epilogue skips the columns past T).
    int bn = BNt;
    if (BMN && CG && kBmnRound) bn = (BNt + 127) / 128 * 128;
    switch (bn) {
      case 64:
        launch_gemm<Prob<64>, GemmShape<64, (!CG && EPI > 2 && epi_stage_bytes<Prob<64>>::value) ? kEpiWideStages : 8, 0, EPI, 2, BMN, AMN, CG>>(a, b, Prob<64>{args...}, 0, st);
        break;
      case 128:
        launch_gemm<Prob<128>, GemmShape<128, (!CG && EPI > 2 && epi_stage_bytes<Prob<128>>::value) ? kEpiWideStages : (CG ? 8 : 6), 0, EPI, 2, BMN, AMN, CG>>(a, b, Prob<128>{args...}, 0, st);
        break;
      case 208:
        // multicast B: 4 stages when the B blocks are MN-major or the epilogue stages bulk stores
        launch_gemm<Prob<208>, GemmShape<208, CG ? kCGStages208 : ((BMN || epi_stage_bytes<Prob<208>>::value) ? (EPI > 2 ? kEpiWideStages : 4) : 5), 0, EPI, 2,
                                         BMN, AMN, CG>>(a, b, Prob<208>{args...}, 0, st);
        break;
      default:
        launch_gemm<Prob<256>, GemmShape<256, (!CG && EPI > 2 && epi_stage_bytes<Prob<256>>::value) ? kEpiWideStages : (CG ? 5 : 4), 0, EPI, 2, BMN, AMN, CG>>(a, b, Prob<256>{args...}, 0, st);
        break;
    }
  }

  // ---------------------------------------------------------------- the step
  // Requires codes_exp + compaction lists + plan for this batch.
  // scoring pre-pass mode of run_forward_backward: unit-mean loss, the weight
  // gradient GEMMs replaced by per-unit score reductions, no embedding wgrad
  struct ScoreMode {
    int n_units, mbs;
    float *p7, *p5;  // [L][n_units][H][kScoreTiles][16][3]
  };
  void run_forward_backward(const ScoreMode* sm = nullptr) {
    const size_t L = D.L, Bm = D.Bmax, T = D.T, d = D.d, H = D.H;
    const size_t xs = Bm * T * d;
    mark(PH_EMBED);
    D2FT_CUDA(cudaMemsetAsync(ctrs, 0, ctr_count() * sizeof(int), st));
    launch_prep_input(D, samples_dev, inp, inpT, st);
    gemm_tokN<EmbedFwd>(tm_WeT, tm_inp, D, P + seg[S_BE].off, P + seg[S_POS].off, x);
    const int XC = active_chunks();
    for (int l = 0; l < D.L; ++l) {
      mark(PH_LN);
      if (l == 0 || !partitioned()) {
        launch_ln_fwd(D, x + l * xs, xn + l * xs, stats + (size_t)l * Bm * T * 2, st);
      } else {  // chunk c of x_l as soon as its exchange is done
        for (int c = 0; c < XC; ++c) {
          const int lo = chunk_lo(c, XC), n = chunk_lo(c + 1, XC) - lo;
          if (!n) continue;
          wait_exchange(0, l - 1, c);
          launch_ln_fwd(D, x + l * xs, xn + l * xs, stats + (size_t)l * Bm * T * 2, st, lo, n);
        }
      }
      mark(PH_G1);
      act_t* QKVl = QKV + (size_t)l * Bm * H * T * 3 * D.dh;
      act_t* ZTl = ZT + (size_t)l * Bm * H * D.fs * D.TP;
      act_t* OGTl = OGT + (size_t)l * Bm * H * D.PO * D.TP;
      const size_t g1cap = Bm * ((D.UQ * H + 1) / 2);
      if (D2FT_G1_RESB && BNt == 208 && D.d == 12 * 64)
        launch_gemm<G1<208>, GemmShape<208, D2FT_G1_RES_STAGES, 0, D2FT_G1_EPI, 2, 0, 0, 1, 12>>(
            tm_W1T, tm_xn,
            G1<208>{D, l, g1_tiles + l * g1cap, g1_count + l, lists.act_heads, lists.act_cnt, (const uint8_t*)codes_exp,
                    P + seg[S_B1].off + (size_t)l * H * D.fs, (const CUtensorMap*)store_maps},
            0, st);
      else if (D2FT_G1_PAIR && BNt == 208)
        launch_gemm<G1<208>, GemmShape<208, D2FT_G1_PAIR_STAGES, 0, D2FT_G1_EPI, 2, 0, 0, 1>>(
            tm_W1T, tm_xn,
            G1<208>{D, l, g1_tiles + l * g1cap, g1_count + l, lists.act_heads, lists.act_cnt, (const uint8_t*)codes_exp,
                    P + seg[S_B1].off + (size_t)l * H * D.fs, (const CUtensorMap*)store_maps},
            0, st);
      else
        gemm_tokN<G1, 0, 0, D2FT_G1_EPI, 0>(tm_W1T, tm_xn, D, l, g1_tiles + l * g1cap, g1_count + l, lists.act_heads,
                                         lists.act_cnt, (const uint8_t*)codes_exp, P + seg[S_B1].off + (size_t)l * H * D.fs,
                                         (const CUtensorMap*)store_maps);
      mark(PH_ATTN_F);
      if (D.dh == 64 && D.TQ <= 256)
        launch_attn_fwd_tc(tm_Q, tm_K, tm_V, D, l, af_items + l * Bm * H, af_count + l, lists.act_heads, OGTl,
                           lse + (size_t)l * Bm * H * T, codes_exp, O32T + (size_t)l * Bm * H * 64 * D.TP, st);
      else
        launch_attn_fwd(D, l, lists.act_heads, lists.act_cnt, QKVl, OGTl, lse + (size_t)l * Bm * H * T, st);
      mark(PH_G3);
      // partitioned: partial block output, residual added once (rank 0), then
      // summed across ranks chunk by chunk (the sum of chunk c overlaps G3 of c+1)
      const float* xres = partitioned() && ex->rank != 0 ? nullptr : x + l * xs;
      for (int c = 0; c < XC; ++c) {
        const int lo = chunk_lo(c, XC), n = chunk_lo(c + 1, XC) - lo;
        if (!n) continue;
        Dims Dc = D;
        Dc.B = n;  // G3's tiles: the chunk's samples in ord_act[lo, lo+n)
        gemm_tokN<G3, 1, 0, kG3Epi>(tm_W2T, tm_OGT64, Dc, l, lists.act_heads, lists.act_cnt, codes_exp,
                         P + seg[S_B2].off + (size_t)l * d, xres, x + (l + 1) * xs, ord_act + l * Bm + lo,
                         XC > 1 ? xctr(l, 0, c) : ctr(l, C_G3));
        if (partitioned()) exchange_chunk(0, l, c, x + (l + 1) * xs, lo, n);
      }
      if (sur_rank) {  // p_s cells add their linear surrogate (off in parity mode)
        const int HR = D.H * sur_rank;
        gemm_tokN<Sur1>(tm_SA, tm_xn, D, l, HR, sur_rank, (const int*)lists.act_cnt, (const uint8_t*)codes_exp, SurU);
        gemm_tokN<Sur2, 1>(tm_SB, tm_U64, D, l, HR, (const int*)lists.act_cnt, x + (l + 1) * xs);
      }
    }
    if (partitioned())
      for (int c = 0; c < XC; ++c)
        if (chunk_lo(c + 1, XC) > chunk_lo(c, XC)) wait_exchange(0, (int)L - 1, c);
    mark(PH_HEAD);
    D2FT_CUDA(cudaMemsetAsync(gmax, 0, sizeof(float), st));
    launch_head(D, x + L * xs, labels_dev, P + seg[S_WC].off, P + seg[S_BC].off,
                sm ? 1.0f / (float)sm->mbs : 1.0f / (float)(data_parallel() ? B_glob : D.B), loss_s, pooled,
                dlog, dX, gmax, logits_dev, st);
    launch_head_reduce(D, loss_s, pooled, dlog, G + seg[S_WC].off, G + seg[S_BC].off, loss, st,
                       data_parallel() ? B_glob : 0);
    mark(PH_LN_BWD);
    launch_ln_bwd_prep(D, -1, lists.full_hcnt, nullptr, nullptr, nullptr, nullptr, nullptr, dX, dC, cs_slot(L - 1),
                       gmax, st);
    const bool side = use_side && !profiling && !sm;  // LoRA: G7 only ([Wo;W2] frozen)
    bool forked = false;  // work went to the side stream in this pass
    // SGD in the G5 / G7 epilogues (FusedSgd) when a training step follows;
    // G8 runs before G7 so the layer's fp16 W1 operand is updated after its
    // last reader; not with the side stream (G5 would overlap G4's W2 reads)
    sgd_fused = sgd_fuse_req && !side && !sm && !lora_rank;
    // training step with both weight-gradient GEMMs on the side stream: each
    // block's weight SGD follows its G7 there (after G8, the block's last
    // reader of the fp16 operands), overlapping the lower blocks' backward
    sgd_layer = step_train && side && side_g7 && !sm && !lora_rank && !sgd_fused && !data_parallel();
    auto g5 = [&](int l, cudaStream_t s5) {
      // the bulk-store staging of the G5 epilogue (16 warps x 2 KB) costs one stage
      launch_gemm<G5<160>, GemmShape<160, kCG2 ? (D2FT_G5_TMA ? 7 : 8) : 6, 0, D2FT_G5_EPI, 2, 0, 1, kCG2>>(
          tm_dC64, tm_OGT, G5<160>{D, l, lists.full_idx, lists.full_cnt, G + seg[S_W2T].off + (size_t)l * d * H * D.PO, gmax,
                  ord_head + l * H, ctr(l, C_G5), fsgd(S_W2T, W2T_bf, (size_t)l * d * H * D.PO),
                  (const CUtensorMap*)store_maps},
          s5 == st ? 0 : side_cap(), s5);
    };
    for (int l = D.L - 1; l >= 0; --l) {
      act_t* QKVl = QKV + (size_t)l * Bm * H * T * 3 * D.dh;
      act_t* ZTl = ZT + (size_t)l * Bm * H * D.fs * D.TP;
      const act_t* OGTl = OGT + (size_t)l * Bm * H * D.PO * D.TP;
      if (side && !lora_rank) {
        D2FT_CUDA(cudaEventRecord(side_event(5 * l), st));
        D2FT_CUDA(cudaStreamWaitEvent(st2, side_event(5 * l), 0));
        forked = true;
        g5(l, st2);
        D2FT_CUDA(cudaEventRecord(side_event(5 * l + 1), st2));
      }
      if (side && side_g7 && l + 1 < (int)L)  // G7(l+1) read dY1T
        D2FT_CUDA(cudaStreamWaitEvent(st, side_event(5 * (l + 1) + 3), 0));
      mark(PH_G4);
      const size_t g4cap = Bm * ((D.UO * H + 1) / 2);
      if (D2FT_G4_RESB && BNt == 208 && D.d == 12 * 64)
        launch_gemm<G4<208>, GemmShape<208, 3, 0, kG4Epi, 2, 0, 1, 1, 12>>(
            tm_W2T, tm_dC,
            G4<208>{D, l, g4_tiles + l * g4cap, g4_count + l, lists.full_heads, lists.full_hcnt, (const act_t*)ZTl,
                    db1_slot(l), (const float*)gmax, (const CUtensorMap*)store_maps, (int*)nullptr},
            0, st);
      else
        gemm_tokN<G4, 0, 1, kG4Epi, D2FT_G4_PAIR>(tm_W2T, tm_dC, D, l, g4_tiles + l * g4cap, g4_count + l, lists.full_heads,
                                                 lists.full_hcnt, (const act_t*)ZTl, db1_slot(l), (const float*)gmax,
                                                 (const CUtensorMap*)store_maps, side ? ctr(l, C_G4) : (int*)nullptr);
      mark(PH_ATTN_B);
      if (D.dh == 64 && attn_bwd_tc_fits(D.TQ))
        launch_attn_bwd_tc(tm_K, tm_dO, D, l, lists.full_heads, lists.full_hcnt, O32T + (size_t)l * Bm * H * 64 * D.TP,
                           lse + (size_t)l * Bm * H * T,
                           dY1T, st);
      else
        launch_attn_bwd(D, l, lists.full_heads, lists.full_hcnt, QKVl, OGTl, dO, lse + (size_t)l * Bm * H * T, dY1T,
                        st);
      if (side && side_g7) D2FT_CUDA(cudaEventRecord(side_event(5 * l + 2), st));
      mark(PH_G5);
      const size_t sper = sm ? (size_t)sm->n_units * H * kScoreTiles * 16 * 3 : 0;
      if (sm) {
        launch_gemm<S5<160>, GemmShape<160, kCG2 ? 8 : 6, 0, 4, 2, 0, 1, kCG2>>(
            tm_dC64, tm_OGT,
            S5<160>{D, l, sm->mbs, sm->n_units, P + seg[S_W2T].off + (size_t)l * d * H * D.PO, gmax, sm->p5 + l * sper},
            0, st);
      } else if (!side && !lora_rank) {  // LoRA: [Wo;W2] frozen
        g5(l, st);
      }
      mark(PH_G8);
      // single engine: dxn leaves G8 as fp16 in gradient-scale units (half the
      // bytes of G8's stores and the LN backward's reads); partitioned: fp32
      // for the cross-rank sum
      act_t* dxn_h = partitioned() ? nullptr : reinterpret_cast<act_t*>(dxn);
      for (int c = 0; c < XC; ++c) {  // per exchange chunk, as G3
        const int lo = chunk_lo(c, XC), n = chunk_lo(c + 1, XC) - lo;
        if (!n) continue;
        Dims Dc = D;
        Dc.B = n;
        gemm_tokN<G8, 1, 1, D2FT_G8_EPI>(tm_W1T, tm_dY1T, Dc, l, lists.full_heads, lists.full_hcnt, dxn, dxn_h,
                                         (const float*)gmax, ord_full + l * Bm + lo,
                                         XC > 1 ? xctr(l, 1, c) : ctr(l, C_G8));
        if (partitioned()) exchange_chunk(1, l, c, dxn, lo, n);
      }
      if (sgd_layer) D2FT_CUDA(cudaEventRecord(side_event(5 * l + 4), st));  // last reader of W1T_bf[l] / W2T_bf[l]
      mark(PH_G7);
      if (sm)
        launch_gemm<S7<kG7BN>, GemmShape<kG7BN, kCG2 ? 7 : 5, 0, 4, 2, 0, 1, kCG2>>(
            tm_xn64, tm_dY1Tb,
            S7<kG7BN>{D, l, sm->mbs, sm->n_units, P + seg[S_W1T].off + (size_t)l * H * D.PQ * d, gmax,
                      sm->p7 + l * sper},
            0, st);
      else {
        const bool s7 = side && side_g7;
        cudaStream_t g7s = st;
        if (s7) {
          D2FT_CUDA(cudaStreamWaitEvent(st2, side_event(5 * l + 2), 0));  // dY1T of block l complete
          forked = true;
          g7s = st2;
        }
        launch_gemm<G7<kG7BN>, GemmShape<kG7BN, kCG2 ? 7 : 5, 0, D2FT_G7_EPI, 2, 0, 1, kCG2>>(
            tm_xn64, tm_dY1Tb,
            G7<kG7BN>{D, l, lists.full_idx, lists.full_cnt, G + seg[S_W1T].off + (size_t)l * H * D.PQ * d, gmax,
                      ord_head + l * H, ctr(l, C_G7), fsgd(S_W1T, W1T_bf, (size_t)l * H * D.PQ * d)},
            s7 ? side_cap() : 0, g7s);
        if (s7) D2FT_CUDA(cudaEventRecord(side_event(5 * l + 3), st2));
        if (data_parallel() && step_train) {
          // data parallel: block l's [Wq|Wk|Wv|W1]^T and [Wo;W2]^T gradients
          // are final (G7 after G5 on the side stream, or both on st): sum
          // them over the ranks on the exchange stream while the backward
          // goes on with block l-1
          D2FT_CUDA(cudaEventRecord(dp_event(l), side ? st2 : st));
          D2FT_CUDA(cudaStreamWaitEvent(xst, dp_event(l), 0));
          dpx->allreduce_sum(G + seg[S_W1T].off + (size_t)l * H * D.PQ * d, (size_t)H * D.PQ * d, xst);
          dpx->allreduce_sum(G + seg[S_W2T].off + (size_t)l * d * H * D.PO, (size_t)d * H * D.PO, xst);
        }
        if (sgd_layer) {  // this block's [Wq|Wk|Wv|W1]^T and [Wo;W2]^T SGD, off the critical path
          D2FT_CUDA(cudaStreamWaitEvent(st2, side_event(5 * l + 4), 0));
          sgd_block(S_W1T, W1T_bf, l, st2);
          sgd_block(S_W2T, W2T_bf, l, st2);
        }
      }
      if (side && !lora_rank) D2FT_CUDA(cudaStreamWaitEvent(st, side_event(5 * l + 1), 0));  // G5 read dC
      mark(PH_LN_BWD);
      for (int c = 0; c < XC; ++c) {
        const int lo = chunk_lo(c, XC), n = chunk_lo(c + 1, XC) - lo;
        if (!n) continue;
        if (partitioned()) wait_exchange(1, l, c);
        launch_ln_bwd_prep(D, l, partitioned() ? full_any : lists.full_hcnt, x + l * xs,
                           partitioned() ? nullptr : xn + l * xs, stats + (size_t)l * Bm * T * 2,
                           partitioned() ? dxn : nullptr, dxn_h, dX, dC, cs_slot(l == 0 ? (int)L : l - 1), gmax, st,
                           lo, n);
      }
    }
    // everything on the side stream (G5, G7, per-block SGD) joins here, or —
    // in a training step — after the remaining SGD (train_body), so the embed
    // / bias gradients and the small SGD segments overlap the side stream's
    // last G7 and block SGD (they touch none of its buffers)
    // join only a side stream that received work in this pass (LoRA with G7
    // on the main stream forks nothing: joining an empty side stream inside
    // a graph capture is an error)
    side_pending = forked;
    if (forked && (!step_train || lora_rank)) join_side();  // lora_grad reads G7's output
    if (sm) return;  // the pre-pass scores only the scheduled head-subnets
    if (lora_rank) {  // only the adapters train (model.hpp:155-172)
      mark(PH_BIAS);
      launch_lora_grad(D, lora_rank, lora_scaling, G + seg[S_W1T].off, LA, LG, lists.full_cnt, st);
      return;
    }
    mark(PH_EMBED_W);
    launch_gemm<EmbedW<256>, GemmShape<256, kCG2 ? 6 : 4, 0, 4, 2, 0, 1, kCG2>>(tm_dC64, tm_inpT, EmbedW<256>{D, KS, part_ew, gmax}, 0, st);
    launch_embed_reduce(D, KS, part_ew, cs_slot(L), dX, G + seg[S_WET].off, G + seg[S_BE].off, G + seg[S_POS].off, st);
    mark(PH_BIAS);
    launch_bias_reduce(D, codes_exp, part_cs, part_db1, G + seg[S_B1].off, G + seg[S_B2].off, st);
  }

  cudaEvent_t side_event(int i) {
    if (side_ev.empty()) {
      side_ev.resize(5 * D.L + 1);
      for (auto& e : side_ev) D2FT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return side_ev[i];
  }
  // prepass_scores (scoring.cpp:108-151) on the staged samples/labels:
  // n_units micro-batches of mbs samples, all head-subnets Full, no update.
  void prepass(int n_units, int mbs, int fwd_metric, int bwd_metric, double* fwd_host, double* bwd_host) {
    D2FT_REQUIRE(!partitioned(), kState, "prepass: not available on a head-partitioned engine");
    if (lora_rank) return prepass_lora(n_units, mbs, fwd_metric, bwd_metric, fwd_host, bwd_host);
    const int B = n_units * mbs;
    begin_step(B);
    const int K = D.K();
    const size_t per = (size_t)D.L * n_units * D.H * kScoreTiles * 16 * 3;
    if (score_cap < per) {
      D2FT_CUDA(cudaStreamSynchronize(st));
      float* p = nullptr;
      D2FT_CUDA(cudaMalloc(&p, (2 * per + (size_t)D.L * n_units * D.H * 3) * sizeof(float)));
      owned.push_back(p);
      score_buf = p;
      score_cap = per;
      double* q = nullptr;
      D2FT_CUDA(cudaMalloc(&q, ((size_t)K + 2 * (size_t)K * D.Bmax) * sizeof(double)));
      owned.push_back(q);
      score_dbl = q;
    }
    float *p7 = score_buf, *p5 = score_buf + per, *pb = score_buf + 2 * per;
    double *wm = score_dbl, *fo = score_dbl + K, *bo = fo + (size_t)K * D.Bmax;
    D2FT_CUDA(cudaMemsetAsync(codes_exp, 1, (size_t)K * D.Bmax, st));  // every cell Full
    D2FT_CUDA(cudaMemsetAsync(score_buf, 0, 2 * per * sizeof(float), st));  // unused tile slots sum as 0
    compact_and_plan();
    ScoreMode m{n_units, mbs, p7, p5};
    run_forward_backward(&m);
    launch_score_bias(D, mbs, n_units, part_db1, part_cs, P + seg[S_B1].off, P + seg[S_B2].off, pb, st);
    launch_score_weight(D, P + seg[S_W1T].off, P + seg[S_W2T].off, P + seg[S_B1].off, P + seg[S_B2].off, wm, st);
    launch_score_reduce(D, n_units, p7, p5, pb, wm, fwd_metric, bwd_metric, fo, bo, st);
    D2FT_CUDA(cudaMemcpyAsync(fwd_host, fo, (size_t)K * n_units * 8, cudaMemcpyDeviceToHost, st));
    D2FT_CUDA(cudaMemcpyAsync(bwd_host, bo, (size_t)K * n_units * 8, cudaMemcpyDeviceToHost, st));
  }
  // LoRA mode (scoring.cpp:129-148 with lora_enabled): the metric runs over
  // the adapter gradients of each unit's own forward/backward (all Full), so
  // the units run one after another on the staged samples; the weight sums
  // use the adapters (visit_trainable).  Parameters and velocities untouched.
  void prepass_lora(int n_units, int mbs, int fwd_metric, int bwd_metric, double* fwd_host, double* bwd_host) {
    const int B = n_units * mbs, K = D.K();
    const size_t per = (size_t)D.T * D.d;
    if (!lab_stage) lab_stage = dalloc<int>(D.Bmax, owned);
    if (!lora_scores) lora_scores = dalloc<double>(2 * (size_t)K * D.Bmax, owned);
    double *fo = lora_scores, *bo = lora_scores + (size_t)K * n_units;
    D2FT_CUDA(cudaMemcpyAsync(samples_stage, samples_dev, (size_t)B * per * 4, cudaMemcpyDeviceToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(lab_stage, labels_dev, (size_t)B * 4, cudaMemcpyDeviceToDevice, st));
    for (int u = 0; u < n_units; ++u) {
      begin_step(mbs);
      D2FT_CUDA(cudaMemcpyAsync(samples_dev, samples_stage + (size_t)u * mbs * per, (size_t)mbs * per * 4,
                                cudaMemcpyDeviceToDevice, st));
      D2FT_CUDA(cudaMemcpyAsync(labels_dev, lab_stage + (size_t)u * mbs, (size_t)mbs * 4, cudaMemcpyDeviceToDevice, st));
      D2FT_CUDA(cudaMemsetAsync(codes_exp, 1, (size_t)K * D.Bmax, st));  // every cell Full
      compact_and_plan();
      run_forward_backward();
      launch_lora_score(D, lora_rank, LA, LG, fwd_metric, bwd_metric, u, n_units, fo, bo, st);
    }
    D2FT_CUDA(cudaMemcpyAsync(fwd_host, fo, (size_t)K * n_units * 8, cudaMemcpyDeviceToHost, st));
    D2FT_CUDA(cudaMemcpyAsync(bwd_host, bo, (size_t)K * n_units * 8, cudaMemcpyDeviceToHost, st));
  }
  int* lab_stage = nullptr;
  double* lora_scores = nullptr;
  float* score_buf = nullptr;
  double* score_dbl = nullptr;
  size_t score_cap = 0;

  float* cs_slot(int k) { return part_cs + (size_t)k * D.Bmax * ((D.T + 31) / 32) * D.d; }
  float* db1_slot(int l) { return part_db1 + (size_t)l * kG4Epi * D.Bmax * D.H * D.fs; }

  // fused SGD (step_gemms.cuh FusedSgd): requested by train_body for the next
  // run_forward_backward; sgd_fused records whether the GEMMs applied it
  bool sgd_fuse_req = false, sgd_fused = false;
  bool step_train = false, sgd_layer = false;  // train_body in progress / per-block side-stream SGD applied
  float sgd_lr = 0.f, sgd_mom = 0.f;
  FusedSgd fsgd(int id, act_t* pbf, size_t off) const {
    if (!sgd_fused) return FusedSgd{nullptr, nullptr, nullptr, 0.f, 0.f, nullptr};
    return FusedSgd{P + seg[id].off + off, V + seg[id].off + off, pbf + off, sgd_lr, sgd_mom, err};
  }
  // forward/backward + SGD of one training step (the trainer's batch body)
  void train_body(float lr, float mom) {
    sgd_fuse_req = kFuseSgd && !data_parallel();
    step_train = true;
    sgd_lr = lr;
    sgd_mom = mom;
    run_forward_backward();
    sgd_fuse_req = false;
    step_train = false;
    if (data_parallel()) {  // the global batch's gradient: sum of every rank's (already 1/B_glob-weighted) share
      if (side_pending) join_side();
      mark(PH_EXCH);
      // the block weight matrices went per block during the backward; the
      // biases, embedding, positions and classifier now, then the SGD waits
      D2FT_CUDA(cudaEventRecord(dp_event(D.L), st));
      D2FT_CUDA(cudaStreamWaitEvent(xst, dp_event(D.L), 0));
      dpx->allreduce_sum(G + seg[S_B1].off, seg[S_B1].n, xst);
      dpx->allreduce_sum(G + seg[S_B2].off, nparam - seg[S_B2].off, xst);
      D2FT_CUDA(cudaEventRecord(dp_event(D.L), xst));
      D2FT_CUDA(cudaStreamWaitEvent(st, dp_event(D.L), 0));
    }
    // the remaining SGD may overlap the side stream only when the side
    // stream already updated (and alone writes) the block weight matrices'
    // gradients; otherwise run_sgd reads what G5 / G7 there still write
    if (side_pending && !sgd_layer) join_side();
    run_sgd(lr, mom);
    if (side_pending) join_side();
    sgd_fused = false;
    sgd_layer = false;
  }
  bool side_pending = false;
  void join_side() {
    D2FT_CUDA(cudaEventRecord(side_event(5 * D.L), st2));
    D2FT_CUDA(cudaStreamWaitEvent(st, side_event(5 * D.L), 0));
    side_pending = false;
  }
  // sgd_momentum_step on block l's part of a per-block segment
  void sgd_block(int id, act_t* pbf, int l, cudaStream_t s) {
    const Seg& g = seg[id];
    const size_t o = g.off + (size_t)l * g.outer;
    launch_sgd(P + o, V + o, G + o, pbf + (size_t)l * g.outer, (size_t)g.outer, g.outer, g.inner, D.H,
               lists.full_cnt + l * D.H, sgd_lr, sgd_mom, err, s);
  }

  void run_sgd(float lr, float mom) {
    mark(PH_SGD);
    const int* fc = data_parallel() ? full_cnt_glob : lists.full_cnt;
    if (lora_rank) {  // adapters of subnets with Full cells, then W_eff for the next step
      const long long per = (long long)lora_per();
      launch_sgd(LA, LV, LG, nullptr, lora_count(), (long long)D.H * per, per, D.H, fc, lr, mom, err, st);
      launch_lora_merge(D, lora_rank, lora_scaling, P + seg[S_W1T].off, LA, W1T_bf, st);
      return;
    }
    auto sgd = [&](int id, act_t* pbf, const int* touch) {
      const Seg& s = seg[id];
      launch_sgd(P + s.off, V + s.off, G + s.off, pbf, s.n, s.outer, s.inner, D.H, touch, lr, mom, err, st);
    };
    if (!sgd_fused && !sgd_layer) sgd(S_W1T, W1T_bf, fc);
    sgd(S_B1, nullptr, fc);
    if (!sgd_fused && !sgd_layer) sgd(S_W2T, W2T_bf, fc);
    sgd(S_B2, nullptr, fc);
    sgd(S_WET, WeT_bf, nullptr);
    sgd(S_BE, nullptr, nullptr);
    sgd(S_POS, nullptr, nullptr);
    sgd(S_WC, nullptr, nullptr);
    sgd(S_BC, nullptr, nullptr);
  }

  // per-sample codes already in codes_exp: compaction + plan
  void compact_and_plan() {
    if (partitioned()) {  // keep the global Full counts, then drop the heads other ranks own
      launch_compact(codes_exp, D.K(), D.Bmax, D.H, lists, st);
      D2FT_CUDA(cudaMemcpyAsync(full_any, lists.full_hcnt, (size_t)D.L * D.Bmax * sizeof(int),
                                cudaMemcpyDeviceToDevice, st));
      launch_mask_rows(codes_exp, D.K(), D.Bmax, row_owner, ex->rank, st);
    }
    launch_compact(codes_exp, D.K(), D.Bmax, D.H, lists, st);
    launch_plan(D, lists.act_cnt, lists.full_hcnt, lists.full_cnt,
                Plan{g1_tiles, g1_count, g4_tiles, g4_count, ord_act, ord_full, ord_head, af_items, af_count, ab_items,
                     ab_count, active_chunks()}, st);
  }

  void ensure_sched(int max_cols) {
    if (max_cols <= sched_max_cols) return;
    sched_max_cols = max_cols;
    // the captured step baked in the knapsack launch's geometry (threads,
    // shared memory, decision-bit buffer): capture again
    drop_graph();
    bool in_smem = true;
    knapsack_smem_bytes(Nmax, max_cols, &in_smem);
    if (!in_smem) {
      const size_t w = knapsack_global_bits_words(D.K(), Nmax, max_cols);
      if (w > sched_bits_words) {
        D2FT_CUDA(cudaStreamSynchronize(st));
        void* p = nullptr;
        D2FT_CUDA(cudaMalloc(&p, w * 4));
        owned.push_back(p);
        sched_bits = static_cast<uint32_t*>(p);
        sched_bits_words = w;
      }
    }
  }

  // D2FT schedule of n_mb micro-batches from device scores/costs.
  void schedule_device(int n_mb, int mbs) {
    mark(PH_SCHED);
    SchedWorkspace ws{};
    ws.bits_global = sched_bits;
    ws.bits_global_words = sched_bits_words;
    ws.done_counter = sched_counter;
    ws.err_flag = err;
    launch_knapsack_schedule(bwd_dev, fwd_dev, cf_dev, cb_dev, capf_dev, capo_dev, D.K(), n_mb, D.H, sched_max_cols,
                             codes_mb, nullptr, ws, true, st);
    expand_and_plan(n_mb, mbs);
  }
  // codes_mb (K x n_mb, the whole batch) -> this rank's per-sample codes,
  // compaction, plan; data parallel: the global Full counts and zeroed
  // gradient rows this rank does not touch (their all-reduce input)
  void expand_and_plan(int n_mb, int mbs) {
    launch_expand_codes(codes_mb, D.K(), n_mb, mbs, D.B, D.Bmax, codes_exp, st, dp_mb0);
    compact_and_plan();
    if (data_parallel()) {
      launch_row_full_count(codes_mb, D.K(), n_mb, full_cnt_glob, st);
      launch_zero_untouched(D, lists.full_cnt, G, seg[S_W1T].off, seg[S_B1].off, seg[S_W2T].off, seg[S_B2].off, st);
    }
  }

  // One D2FT batch from host buffers (pinned for full-speed DMA): H2D of the
  // samples, labels and score slice, schedule, step, D2H of loss and codes.
  void host_step(const float* samples, const int32_t* labels, const double* bwd_scores, const double* fwd_scores,
                 const int32_t* cf, const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, int n_mb,
                 int mbs, double lr, double momentum, const float* samples_next = nullptr) {
    const int K = D.K();
    const int B = local_B(n_mb, mbs);
    begin_step(B);
    const size_t KN = (size_t)K * n_mb;
    // the small H2D copies go first: the host->device copy engine serves
    // transfers in submission order, so behind a prefetch of the next batch's
    // samples (released by consume_prefetch below) they would wait ~0.7 ms
    D2FT_CUDA(cudaMemcpyAsync(labels_dev, labels, B * 4, cudaMemcpyHostToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(bwd_dev, bwd_scores, KN * 8, cudaMemcpyHostToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(fwd_dev, fwd_scores, KN * 8, cudaMemcpyHostToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(cf_dev, cf, K * 4, cudaMemcpyHostToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(cb_dev, cb, K * 4, cudaMemcpyHostToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(capf_dev, cap_full, K * 4, cudaMemcpyHostToDevice, st));
    D2FT_CUDA(cudaMemcpyAsync(capo_dev, cap_fwd, K * 4, cudaMemcpyHostToDevice, st));
    if (samples) D2FT_CUDA(cudaMemcpyAsync(samples_dev, samples, (size_t)B * D.T * D.d * 4, cudaMemcpyHostToDevice, st));
    else consume_prefetch(B);  // samples == nullptr: the batch prefetched by d2ft_engine_prefetch
    compute_step(n_mb, mbs, lr, momentum);
    if (samples_next) prefetch(samples_next, B);  // overlaps this batch's compute
    D2FT_CUDA(cudaMemcpyAsync(h_codes, codes_mb, KN, cudaMemcpyDeviceToHost, st));
  }

  // Next batch's samples (pinned host memory for an asynchronous copy) ->
  // samples_stage on the copy stream, overlapping whatever the engine stream
  // is computing; the stage is reused only after the previous batch left it.
  void prefetch(const float* samples, int B) {
    D2FT_REQUIRE(B >= 1 && B <= D.Bmax, kSize, "prefetch: batch exceeds the engine capacity");
    D2FT_CUDA(cudaStreamWaitEvent(cst, ev_stage_free, 0));
    D2FT_CUDA(cudaMemcpyAsync(samples_stage, samples, (size_t)B * D.T * D.d * 4, cudaMemcpyHostToDevice, cst));
    D2FT_CUDA(cudaEventRecord(ev_copied, cst));
    have_prefetch = true;
    prefetch_B = B;
    prefetched_units.clear();
  }
  // The data.hpp Dataset path (trainer.cpp:247-253 reads
  // dataset.unit_inputs(units[j], mbs), fp64 Matrix samples): the batch's
  // samples are gathered H2D as fp64 in batch order on the copy stream (one
  // DMA per sample; page-locked by d2ft_dataset_create for full speed), then
  // converted to fp32 into samples_stage on the same stream.  Overlaps the
  // engine stream's current step; consume_prefetch picks it up.
  void prefetch_units(const double* const* samples, const int32_t* units, int n_mb, int mbs) {
    const int B = n_mb * mbs;
    D2FT_REQUIRE(B >= 1 && B <= D.Bmax, kSize, "prefetch: batch exceeds the engine capacity");
    const size_t per = (size_t)D.T * D.d;
    if (!stage64) stage64 = dalloc<double>((size_t)D.Bmax * per, owned);
    D2FT_CUDA(cudaStreamWaitEvent(cst, ev_stage_free, 0));
    for (int j = 0; j < n_mb; ++j)
      for (int i = 0; i < mbs; ++i) {
        const size_t s = (size_t)units[j] * mbs + i;
        D2FT_CUDA(cudaMemcpyAsync(stage64 + ((size_t)j * mbs + i) * per, samples[s], per * 8,
                                  cudaMemcpyHostToDevice, cst));
      }
    launch_f64_to_f32(stage64, samples_stage, (size_t)B * per, cst);
    D2FT_CUDA(cudaEventRecord(ev_copied, cst));
    have_prefetch = true;
    prefetch_B = B;
    prefetched_units.assign(units, units + n_mb);
  }
  // prefetched samples -> samples_dev on the engine stream (device copy, ~12 us at ViT-B)
  void consume_prefetch(int B) {
    D2FT_REQUIRE(have_prefetch && prefetch_B == B, kState, "step: no prefetched batch of this size");
    D2FT_CUDA(cudaStreamWaitEvent(st, ev_copied, 0));
    D2FT_CUDA(cudaMemcpyAsync(samples_dev, samples_stage, (size_t)B * D.T * D.d * 4, cudaMemcpyDeviceToDevice, st));
    D2FT_CUDA(cudaEventRecord(ev_stage_free, st));
    have_prefetch = false;
  }

  // schedule + forward/backward + SGD on the staged device inputs (after begin_step)
  void compute_step(int n_mb, int mbs, double lr, double momentum) {
    if (profiling || (partitioned() && !ex->capturable()) || (data_parallel() && !dpx->capturable()) || !use_graphs) {
      schedule_device(n_mb, mbs);
      train_body((float)lr, (float)momentum);
      return;
    }
    if (!gexec || g_nmb != n_mb || g_mbs != mbs || g_lr != (float)lr || g_mom != (float)momentum) {
      if (gexec) {
        D2FT_CUDA(cudaGraphExecDestroy(gexec));
        gexec = nullptr;
      }
      cudaGraph_t g = nullptr;
      const unsigned long long n0 = d2ft_b200::launch_count();
      Exchange* xx = ex ? ex.get() : dpx.get();  // the engine's collective (partition or data parallel)
      const unsigned long long xc0 = xx ? xx->calls : 0, xb0 = xx ? xx->bytes : 0;
      D2FT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      schedule_device(n_mb, mbs);
      train_body((float)lr, (float)momentum);
      D2FT_CUDA(cudaStreamEndCapture(st, &g));
      g_kernels = d2ft_b200::launch_count() - n0;
      g_xcalls = xx ? xx->calls - xc0 : 0;
      g_xbytes = xx ? xx->bytes - xb0 : 0;
      if (use_pdl) make_edges_programmatic(g);
      D2FT_CUDA(cudaGraphInstantiate(&gexec, g, 0));
      D2FT_CUDA(cudaGraphDestroy(g));
      g_nmb = n_mb;
      g_mbs = mbs;
      g_lr = (float)lr;
      g_mom = (float)momentum;
    } else {
      d2ft_b200::add_launches(g_kernels);
      if (Exchange* xx = ex ? ex.get() : dpx.get()) {  // the replay issues the captured all-reduces again
        xx->calls += g_xcalls;
        xx->bytes += g_xbytes;
      }
    }
    D2FT_CUDA(cudaGraphLaunch(gexec, st));
  }

  // a partition was attached: exchange stream, default head-interleaved
  // mapping (row k = l*H + h -> rank h % world), the captured step is stale
  void on_partition() {
    drop_graph();
    if (!xst) {
      int least = 0, greatest = 0;
      D2FT_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      D2FT_CUDA(cudaStreamCreateWithPriority(&xst, cudaStreamNonBlocking, greatest));
    }
    std::vector<int> own(D.K());
    for (int k = 0; k < D.K(); ++k) own[k] = (k % D.H) % ex->world;
    set_row_owner(own.data());
  }
  void set_row_owner(const int* owner) {
    D2FT_REQUIRE(ex, kState, "row owner: the engine is not partitioned");
    for (int k = 0; k < D.K(); ++k)
      D2FT_REQUIRE(owner[k] >= 0 && owner[k] < ex->world, kConfig, "row owner: rank out of range");
    drop_graph();
    D2FT_CUDA(cudaMemcpy(row_owner, owner, (size_t)D.K() * sizeof(int), cudaMemcpyHostToDevice));
  }

  void drop_graph() {
    if (gexec) {
      D2FT_CUDA(cudaStreamSynchronize(st));
      D2FT_CUDA(cudaGraphExecDestroy(gexec));
      gexec = nullptr;
    }
  }

  void begin_step(int B) {
    D2FT_REQUIRE(B >= 1 && B <= D.Bmax, kSize, "step: batch exceeds the engine capacity");
    if (profiling) ++profiled_steps;
    D.B = B;
    D2FT_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  }

  int finish_and_check() {
    mark(PH_COUNT);
    D2FT_CUDA(cudaMemcpyAsync(h_loss, loss, sizeof(double), cudaMemcpyDeviceToHost, st));
    D2FT_CUDA(cudaMemcpyAsync(h_err, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    D2FT_CUDA(cudaStreamSynchronize(st));
    collect();
    return *h_err;
  }
};

}  // namespace d2ft_b200

using namespace d2ft_b200;

struct d2ft_engine {
  Engine* e;
};

// data.hpp:18-42 Dataset: borrowed fp64 sample pointers (the caller's
// vector<Matrix> owns them), labels, optionally page-locked.
struct d2ft_dataset {
  std::vector<const double*> samples;
  std::vector<int32_t> labels;
  std::vector<void*> pinned;  // cudaHostRegister'ed sample buffers (unregistered on destroy)
  int num_classes = 0, T = 0, d = 0;
};

namespace {

void validate_labels(const int32_t* labels, int B, int C) {
  for (int i = 0; i < B; ++i) D2FT_REQUIRE(labels[i] >= 0 && labels[i] < C, kInput, "label out of range");
}

void validate_sched_inputs(const double* bwd, const double* fwd, const int32_t* cf, const int32_t* cb,
                           const int32_t* cap_full, const int32_t* cap_fwd, int K, int N) {
  const double* sides[2] = {fwd, bwd};
  for (int s = 0; s < 2; ++s)
    for (size_t c = 0; c < (size_t)K * N; ++c) {
      D2FT_REQUIRE(std::isfinite(sides[s][c]), kNumeric, "score table contains non-finite entries");
      D2FT_REQUIRE(sides[s][c] >= 0.0, kNumeric, "score table contains negative entries");
    }
  for (int k = 0; k < K; ++k) D2FT_REQUIRE(cap_full[k] >= 0, kInput, "capacities: negative full capacity");
  for (int k = 0; k < K; ++k) D2FT_REQUIRE(cap_fwd[k] >= 0, kInput, "capacities: negative forward capacity");
  for (int k = 0; k < K; ++k)
    D2FT_REQUIRE(cf[k] >= 0 && cb[k] >= 0, kConfig, "cost model: costs must be nonnegative integers");
}

int max_cols_of(const int32_t* cf, const int32_t* cb, const int32_t* capf, const int32_t* capo, int K, int N) {
  auto cols = [N](int wt, int cap) { return wt == 0 ? 1 : std::min(cap / wt, N) + 1; };
  int mc = 1;
  for (int k = 0; k < K; ++k) mc = std::max(mc, std::max(cols(cf[k] + cb[k], capf[k]), cols(cf[k], capo[k])));
  return mc;
}

void check_status(int e) {
  if (e) throw Fail{e, e == kNumeric ? "non-finite score or gradient detected on the device"
                                     : "device-side validation failed"};
}

}  // namespace

extern "C" {

int d2ft_engine_create(const d2ft_model_config* cfg, int max_batch, d2ft_engine** out) {
  return guarded([&] {
    D2FT_REQUIRE(cfg && out, kInput, "engine_create: null argument");
    *out = new d2ft_engine{new Engine(*cfg, max_batch)};
  });
}

int d2ft_engine_destroy(d2ft_engine* e) {
  return guarded([&] {
    if (e) {
      delete e->e;
      delete e;
    }
  });
}

int64_t d2ft_engine_param_count(d2ft_engine* e) { return e && e->e ? (int64_t)e->e->canonical_count() : -1; }

int d2ft_engine_set_params(d2ft_engine* e, const double* flat) {
  return guarded([&] {
    D2FT_REQUIRE(e && e->e && flat, kInput, "set_params: null argument");
    e->e->set_params(flat);
    D2FT_CUDA(cudaMemsetAsync(e->e->V, 0, e->e->nparam * 4, e->e->st));
    D2FT_CUDA(cudaStreamSynchronize(e->e->st));
  });
}

int d2ft_engine_get_params(d2ft_engine* e, double* flat) {
  return guarded([&] { e->e->get_arena(e->e->P, flat); });
}

int d2ft_engine_get_velocity(d2ft_engine* e, double* flat) {
  return guarded([&] { e->e->get_arena(e->e->V, flat); });
}

int d2ft_engine_get_grads(d2ft_engine* e, double* flat) {
  return guarded([&] { e->e->get_arena(e->e->G, flat); });
}

int d2ft_engine_set_surrogate(d2ft_engine* e, int rank, const double* factors) {
  return guarded([&] {
    D2FT_REQUIRE(e && e->e, kInput, "set_surrogate: null engine");
    e->e->set_surrogate(rank, factors);
  });
}

int d2ft_engine_attach_lora(d2ft_engine* e, int rank, double scaling, const double* adapters) {
  return guarded([&] {
    D2FT_REQUIRE(e && e->e && adapters, kInput, "attach_lora: null argument");
    e->e->attach_lora(rank, scaling, adapters);
  });
}

int64_t d2ft_engine_lora_count(d2ft_engine* e) {
  return e && e->e && e->e->lora_rank ? (int64_t)e->e->lora_count() : 0;
}

int d2ft_engine_set_lora(d2ft_engine* e, const double* adapters) {
  return guarded([&] {
    D2FT_REQUIRE(e && e->e && adapters, kInput, "set_lora: null argument");
    D2FT_REQUIRE(e->e->lora_rank, kState, "set_lora: no adapters attached");
    e->e->set_lora(adapters);
    D2FT_CUDA(cudaMemsetAsync(e->e->LV, 0, e->e->lora_count() * 4, e->e->st));
    D2FT_CUDA(cudaStreamSynchronize(e->e->st));
  });
}

int d2ft_engine_get_lora(d2ft_engine* e, int which, double* adapters) {
  return guarded([&] {
    D2FT_REQUIRE(e && e->e && adapters, kInput, "get_lora: null argument");
    D2FT_REQUIRE(e->e->lora_rank, kState, "get_lora: no adapters attached");
    D2FT_REQUIRE(which >= 0 && which <= 2, kInput, "get_lora: which is 0 (params), 1 (velocity) or 2 (grads)");
    e->e->get_lora(which == 0 ? e->e->LA : which == 1 ? e->e->LV : e->e->LG, adapters);
  });
}

int d2ft_nccl_unique_id(uint8_t* id_out) {
  return guarded([&] {
    D2FT_REQUIRE(id_out, kInput, "nccl_unique_id: null argument");
    nccl_unique_id(id_out);
  });
}

int d2ft_engine_partition_nccl(d2ft_engine* h, int rank, int world, const uint8_t* id) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && id, kInput, "partition: null argument");
    D2FT_REQUIRE(world >= 1 && rank >= 0 && rank < world, kConfig, "partition: rank out of range");
    Engine& E = *h->e;
    D2FT_REQUIRE(!E.data_parallel(), kState, "partition: the engine is data parallel");
    D2FT_CUDA(cudaStreamSynchronize(E.st));
    E.ex = make_nccl_exchange(rank, world, id);
    E.on_partition();
  });
}

struct d2ft_local_group {
  LocalGroup* g;
};

int d2ft_local_group_create(int world, d2ft_local_group** out) {
  return guarded([&] {
    D2FT_REQUIRE(out, kInput, "local_group_create: null argument");
    *out = new d2ft_local_group{local_group_create(world)};
  });
}

int d2ft_local_group_destroy(d2ft_local_group* g) {
  return guarded([&] {
    if (g) {
      local_group_destroy(g->g);
      delete g;
    }
  });
}

int d2ft_local_group_abort(d2ft_local_group* g) {
  return guarded([&] {
    D2FT_REQUIRE(g, kInput, "local_group_abort: null argument");
    local_group_abort(g->g);
  });
}

int d2ft_engine_partition_local(d2ft_engine* h, d2ft_local_group* g, int rank) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && g, kInput, "partition: null argument");
    Engine& E = *h->e;
    D2FT_REQUIRE(!E.data_parallel(), kState, "partition: the engine is data parallel");
    D2FT_CUDA(cudaStreamSynchronize(E.st));
    E.ex = make_local_exchange(g->g, rank);
    E.on_partition();
  });
}

namespace {
void join_data_parallel(Engine& E, std::unique_ptr<Exchange> x) {
  D2FT_REQUIRE(!E.partitioned() && !E.data_parallel(), kState, "data parallel: the engine already joined a group");
  D2FT_REQUIRE(!E.lora_rank, kState, "data parallel: not available with LoRA adapters attached");
  D2FT_CUDA(cudaStreamSynchronize(E.st));
  E.drop_graph();
  if (!E.full_cnt_glob) E.full_cnt_glob = dalloc<int>(E.D.K(), E.owned);
  if (!E.xst) {  // the gradient all-reduces run on the exchange stream, overlapping the backward
    int least = 0, greatest = 0;
    D2FT_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    D2FT_CUDA(cudaStreamCreateWithPriority(&E.xst, cudaStreamNonBlocking, greatest));
  }
  E.size_tables(x->world * E.D.Bmax);  // the global batch's table: up to world x Bmax micro-batches
  E.dpx = std::move(x);
}
}  // namespace

int d2ft_engine_data_parallel_nccl(d2ft_engine* h, int rank, int world, const uint8_t* id) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && id, kInput, "data parallel: null argument");
    D2FT_REQUIRE(world >= 1 && rank >= 0 && rank < world, kConfig, "data parallel: rank out of range");
    join_data_parallel(*h->e, make_nccl_exchange(rank, world, id));
  });
}

int d2ft_engine_data_parallel_local(d2ft_engine* h, d2ft_local_group* g, int rank) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && g, kInput, "data parallel: null argument");
    join_data_parallel(*h->e, make_local_exchange(g->g, rank));
  });
}

int d2ft_engine_forward_backward(d2ft_engine* h, const float* samples, const int32_t* labels, int n,
                                 const uint8_t* column, double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    D2FT_REQUIRE(n >= 1, kInput, "micro-batch inputs and labels must be non-empty and aligned");
    for (int k = 0; k < E.D.K(); ++k)
      D2FT_REQUIRE(column[k] >= 1 && column[k] <= 3, kInput, "schedule table: code out of range");
    validate_labels(labels, n, E.D.C);
    E.begin_step(n);
    const size_t xs = (size_t)n * E.D.T * E.D.d;
    D2FT_CUDA(cudaMemcpyAsync(E.samples_dev, samples, xs * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.labels_dev, labels, n * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.codes_mb, column, E.D.K(), cudaMemcpyHostToDevice, E.st));
    launch_expand_codes(E.codes_mb, E.D.K(), 1, n, n, E.D.Bmax, E.codes_exp, E.st);
    E.compact_and_plan();
    E.run_forward_backward();
    check_status(E.finish_and_check());
    *loss_out = *E.h_loss;
  });
}

int d2ft_engine_logits(d2ft_engine* h, const float* samples, int n, double* logits_out) {
  return guarded([&] {
    Engine& E = *h->e;
    D2FT_REQUIRE(samples && logits_out, kInput, "logits: null argument");
    D2FT_REQUIRE(n >= 1 && n <= E.D.Bmax, kSize, "logits: batch exceeds the engine capacity");
    // every subnet active (model.cpp logits): a forward-only column runs the
    // identical forward; no block backward, no update
    std::vector<uint8_t> col(E.D.K(), 2);
    std::vector<int32_t> lab(n, 0);
    E.begin_step(n);
    const size_t xs = (size_t)n * E.D.T * E.D.d;
    D2FT_CUDA(cudaMemcpyAsync(E.samples_dev, samples, xs * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.labels_dev, lab.data(), n * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.codes_mb, col.data(), E.D.K(), cudaMemcpyHostToDevice, E.st));
    launch_expand_codes(E.codes_mb, E.D.K(), 1, n, n, E.D.Bmax, E.codes_exp, E.st);
    E.compact_and_plan();
    E.run_forward_backward();
    std::vector<float> lg((size_t)n * E.D.C);
    D2FT_CUDA(cudaMemcpyAsync(lg.data(), E.logits_dev, lg.size() * 4, cudaMemcpyDeviceToHost, E.st));
    check_status(E.finish_and_check());
    for (size_t i = 0; i < lg.size(); ++i) logits_out[i] = lg[i];
  });
}

int d2ft_engine_prepass_scores(d2ft_engine* h, const float* samples, const int32_t* labels, int num_samples,
                               int micro_batch_size, int fwd_metric, int bwd_metric, double* fwd_out,
                               double* bwd_out) {
  return guarded([&] {
    Engine& E = *h->e;
    D2FT_REQUIRE(num_samples >= 1, kInput, "prepass_scores: empty dataset");
    D2FT_REQUIRE(micro_batch_size >= 1 && num_samples % micro_batch_size == 0, kInput,
                 "dataset size must be a multiple of the micro-batch size");
    D2FT_REQUIRE(num_samples <= E.D.Bmax, kSize, "prepass_scores: more samples than the engine's batch capacity");
    D2FT_REQUIRE(fwd_metric >= 0 && fwd_metric <= 3 && bwd_metric >= 0 && bwd_metric <= 3, kConfig,
                 "unknown metric");
    D2FT_REQUIRE(fwd_out && bwd_out, kInput, "prepass_scores: null output");
    validate_labels(labels, num_samples, E.D.C);
    D2FT_CUDA(cudaMemcpyAsync(E.samples_dev, samples, (size_t)num_samples * E.D.T * E.D.d * 4, cudaMemcpyHostToDevice,
                              E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.labels_dev, labels, num_samples * 4, cudaMemcpyHostToDevice, E.st));
    E.prepass(num_samples / micro_batch_size, micro_batch_size, fwd_metric, bwd_metric, fwd_out, bwd_out);
    check_status(E.finish_and_check());
    for (size_t i = 0; i < (size_t)E.D.K() * (num_samples / micro_batch_size); ++i)
      D2FT_REQUIRE(std::isfinite(fwd_out[i]) && std::isfinite(bwd_out[i]), kNumeric,
                   "prepass_scores produced a non-finite score");
  });
}

int d2ft_engine_step_codes(d2ft_engine* h, const float* samples, const int32_t* labels, const uint8_t* codes,
                           int n_mb, int mbs, double lr, double momentum, double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    const int B = E.local_B(n_mb, mbs);  // data parallel: n_mb and codes cover the global batch
    for (size_t c = 0; c < (size_t)E.D.K() * n_mb; ++c)
      D2FT_REQUIRE(codes[c] >= 1 && codes[c] <= 3, kInput, "schedule table: code out of range");
    validate_labels(labels, B, E.D.C);
    E.begin_step(B);
    D2FT_CUDA(cudaMemcpyAsync(E.samples_dev, samples, (size_t)B * E.D.T * E.D.d * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.labels_dev, labels, B * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.codes_mb, codes, (size_t)E.D.K() * n_mb, cudaMemcpyHostToDevice, E.st));
    E.expand_and_plan(n_mb, mbs);
    E.train_body((float)lr, (float)momentum);
    check_status(E.finish_and_check());
    *loss_out = *E.h_loss;
  });
}

int d2ft_engine_step(d2ft_engine* h, const float* samples, const int32_t* labels, const double* bwd_scores,
                     const double* fwd_scores, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                     const int32_t* cap_fwd, int n_mb, int mbs, double lr, double momentum, double* loss_out,
                     uint8_t* codes_out) {
  return guarded([&] {
    Engine& E = *h->e;
    const int K = E.D.K();
    D2FT_REQUIRE(n_mb >= 1 && mbs >= 1, kConfig, "train: batch_size must be a positive multiple of micro_batch_size");
    validate_sched_inputs(bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, K, n_mb);
    validate_labels(labels, E.local_B(n_mb, mbs), E.D.C);
    E.ensure_sched(max_cols_of(cf, cb, cap_full, cap_fwd, K, n_mb));
    E.host_step(samples, labels, bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, n_mb, mbs, lr, momentum);
    check_status(E.finish_and_check());
    *loss_out = *E.h_loss;
    if (codes_out) std::memcpy(codes_out, E.h_codes, (size_t)K * n_mb);
  });
}

int d2ft_engine_prefetch(d2ft_engine* h, const float* samples, int batch) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && samples, kInput, "prefetch: null argument");
    h->e->prefetch(samples, batch);
  });
}

int d2ft_engine_step_pipelined(d2ft_engine* h, const float* samples_next, const int32_t* labels,
                               const double* bwd_scores, const double* fwd_scores, const int32_t* cf,
                               const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, int n_mb, int mbs,
                               double lr, double momentum, double* loss_out, uint8_t* codes_out) {
  return guarded([&] {
    Engine& E = *h->e;
    const int K = E.D.K();
    D2FT_REQUIRE(n_mb >= 1 && mbs >= 1, kConfig, "train: batch_size must be a positive multiple of micro_batch_size");
    validate_sched_inputs(bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, K, n_mb);
    validate_labels(labels, E.local_B(n_mb, mbs), E.D.C);
    E.ensure_sched(max_cols_of(cf, cb, cap_full, cap_fwd, K, n_mb));
    E.host_step(nullptr, labels, bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, n_mb, mbs, lr, momentum,
                samples_next);
    check_status(E.finish_and_check());
    *loss_out = *E.h_loss;
    if (codes_out) std::memcpy(codes_out, E.h_codes, (size_t)K * n_mb);
  });
}

int d2ft_dataset_create(const double* const* samples, const int32_t* labels, int num_samples, int num_classes,
                        int seq_len, int token_dim, int pin, d2ft_dataset** out) {
  return guarded([&] {
    D2FT_REQUIRE(samples && labels && out, kInput, "dataset: null argument");
    D2FT_REQUIRE(num_samples >= 1 && num_classes >= 1 && seq_len >= 1 && token_dim >= 1, kInput,
                 "dataset: sizes must be positive");
    for (int i = 0; i < num_samples; ++i) {
      D2FT_REQUIRE(samples[i], kInput, "dataset: null sample");
      D2FT_REQUIRE(labels[i] >= 0 && labels[i] < num_classes, kInput, "dataset: label out of range");
    }
    auto ds = std::make_unique<d2ft_dataset>();
    ds->samples.assign(samples, samples + num_samples);
    ds->labels.assign(labels, labels + num_samples);
    ds->num_classes = num_classes;
    ds->T = seq_len;
    ds->d = token_dim;
    if (pin) {
      // Page-lock only samples that start on a page boundary (the caller
      // allocated them page-aligned, so the pages they touch are theirs): a
      // registration that covers pages shared with other allocations — heap
      // neighbours of small matrices — makes later copies of those
      // neighbours straddle a registered range (the driver then refuses them
      // or DMAs unlocked bytes).  Every other sample stays pageable: its copy
      // is staged by the driver (slower, same bytes).
      const size_t bytes = (size_t)seq_len * token_dim * sizeof(double);
      const size_t pg = 4096;
      for (int i = 0; i < num_samples; ++i) {
        void* p = const_cast<double*>(samples[i]);
        if (reinterpret_cast<uintptr_t>(p) % pg) continue;
        if (cudaHostRegister(p, (bytes + pg - 1) / pg * pg, cudaHostRegisterDefault) == cudaSuccess)
          ds->pinned.push_back(p);
        else
          cudaGetLastError();
      }
    }
    *out = ds.release();
  });
}

int d2ft_dataset_destroy(d2ft_dataset* ds) {
  return guarded([&] {
    if (!ds) return;
    for (void* p : ds->pinned) cudaHostUnregister(p);
    delete ds;
  });
}

namespace {
// the units of one batch: in range, the dataset matches the engine
void validate_units(const Engine& E, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs) {
  D2FT_REQUIRE(ds && units, kInput, "step_units: null argument");
  D2FT_REQUIRE(!E.data_parallel(), kState, "step_units: not available on a data-parallel engine");
  D2FT_REQUIRE(n_mb >= 1 && mbs >= 1, kConfig, "train: batch_size must be a positive multiple of micro_batch_size");
  D2FT_REQUIRE(ds->T == E.D.T && ds->d == E.D.d, kInput, "train sample: shape does not match the model");
  const int total = (int)ds->samples.size() / mbs;
  D2FT_REQUIRE((int)ds->samples.size() % mbs == 0, kInput, "dataset size must be a multiple of the micro-batch size");
  for (int j = 0; j < n_mb; ++j) D2FT_REQUIRE(units[j] >= 0 && units[j] < total, kInput, "step_units: unit out of range");
}

// One batch of the Dataset path (trainer.cpp:214-268), gathered into pinned
// staging set `buf`: labels as dataset.unit_labels, the score slice as
// slice_scores (trainer.cpp:139-154) from the full K x total_units table, the
// cost / capacity rows; validated in the reference's order.
void units_prepare(Engine& E, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs,
                   const double* bwd_scores, const double* fwd_scores, int total_units, const int32_t* cf,
                   const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, int buf) {
  E.prep.valid = false;
  E.ensure_units_staging();
  const int K = E.D.K();
  const int B = n_mb * mbs;
  int* lab = E.u_lab[buf];
  for (int j = 0; j < n_mb; ++j)
    for (int i = 0; i < mbs; ++i) lab[j * mbs + i] = ds->labels[(size_t)units[j] * mbs + i];
  validate_labels(lab, B, E.D.C);
  double* sb = E.u_sc[buf];
  double* sf = sb + (size_t)K * E.Nmax;
  for (int k = 0; k < K; ++k)
    for (int j = 0; j < n_mb; ++j) {
      sb[(size_t)k * n_mb + j] = bwd_scores[(size_t)k * total_units + units[j]];
      sf[(size_t)k * n_mb + j] = fwd_scores[(size_t)k * total_units + units[j]];
    }
  validate_sched_inputs(sb, sf, cf, cb, cap_full, cap_fwd, K, n_mb);
  int32_t* caps = E.u_caps[buf];
  std::memcpy(caps, cf, (size_t)K * 4);
  std::memcpy(caps + K, cb, (size_t)K * 4);
  std::memcpy(caps + 2 * K, cap_full, (size_t)K * 4);
  std::memcpy(caps + 3 * K, cap_fwd, (size_t)K * 4);
  E.prep.buf = buf;
  E.prep.n_mb = n_mb;
  E.prep.mbs = mbs;
  E.prep.total_units = total_units;
  E.prep.ds = ds;
  E.prep.bwd = bwd_scores;
  E.prep.fwd = fwd_scores;
  E.prep.units.assign(units, units + n_mb);
  E.prep.valid = true;
}

// One batch of the Dataset path: the staged batch (prepared while the
// previous one computed, or now) goes up in three copies (labels, both score
// slices, the cost / capacity rows), then the step; the next batch's fp64
// samples are prefetched and its host inputs staged behind this step.  A
// validation error of the next batch is raised by its own step.
void units_step(Engine& E, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs, const int32_t* units_next,
                const double* bwd_scores, const double* fwd_scores, int total_units, const int32_t* cf,
                const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd, double lr, double momentum) {
  const int K = E.D.K();
  const int B = n_mb * mbs;
  const size_t KN = (size_t)K * n_mb;
  // the staged batch is used when it is this one: same units, dataset and
  // score table (which the caller keeps unmodified, as for the prefetched
  // samples) and the same cost / capacity rows (compared here)
  const auto same_rows = [&](int buf) {
    const int32_t* c = E.u_caps[buf];
    return !std::memcmp(c, cf, (size_t)K * 4) && !std::memcmp(c + K, cb, (size_t)K * 4) &&
           !std::memcmp(c + 2 * K, cap_full, (size_t)K * 4) && !std::memcmp(c + 3 * K, cap_fwd, (size_t)K * 4);
  };
  if (!(E.prep.valid && E.prep.n_mb == n_mb && E.prep.mbs == mbs && E.prep.ds == ds && E.prep.bwd == bwd_scores &&
        E.prep.fwd == fwd_scores && E.prep.total_units == total_units &&
        std::equal(units, units + n_mb, E.prep.units.begin(), E.prep.units.end()) && same_rows(E.prep.buf)))
    units_prepare(E, ds, units, n_mb, mbs, bwd_scores, fwd_scores, total_units, cf, cb, cap_full, cap_fwd, E.ubuf);
  const int buf = E.prep.buf;
  E.prep.valid = false;
  E.ensure_sched(max_cols_of(cf, cb, cap_full, cap_fwd, K, n_mb));
  if (!E.have_prefetch) E.prefetch_units(ds->samples.data(), units, n_mb, mbs);
  E.begin_step(B);
  D2FT_CUDA(cudaMemcpyAsync(E.labels_dev, E.u_lab[buf], (size_t)B * 4, cudaMemcpyHostToDevice, E.st));
  D2FT_CUDA(cudaMemcpyAsync(E.bwd_dev, E.u_sc[buf], ((size_t)K * E.Nmax + KN) * 8, cudaMemcpyHostToDevice, E.st));
  D2FT_CUDA(cudaMemcpyAsync(E.cf_dev, E.u_caps[buf], (size_t)K * 16, cudaMemcpyHostToDevice, E.st));
  E.consume_prefetch(B);
  E.compute_step(n_mb, mbs, lr, momentum);
  D2FT_CUDA(cudaMemcpyAsync(E.h_codes, E.codes_mb, KN, cudaMemcpyDeviceToHost, E.st));
  E.ubuf = buf ^ 1;
  if (units_next) {
    E.prefetch_units(ds->samples.data(), units_next, n_mb, mbs);
    try {
      units_prepare(E, ds, units_next, n_mb, mbs, bwd_scores, fwd_scores, total_units, cf, cb, cap_full, cap_fwd,
                    buf ^ 1);
    } catch (...) {
      E.prep.valid = false;  // prepared again (and the error raised) by the next batch's step
    }
  }
}
}  // namespace

int d2ft_engine_step_units(d2ft_engine* h, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs,
                           const int32_t* units_next, const double* bwd_scores, const double* fwd_scores,
                           int total_units, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                           const int32_t* cap_fwd, double lr, double momentum, double* loss_out, uint8_t* codes_out) {
  return guarded([&] {
    Engine& E = *h->e;
    validate_units(E, ds, units, n_mb, mbs);
    if (units_next) validate_units(E, ds, units_next, n_mb, mbs);
    D2FT_REQUIRE(bwd_scores && fwd_scores && cf && cb && cap_full && cap_fwd && loss_out, kInput,
                 "step_units: null argument");
    D2FT_REQUIRE(total_units == (int)ds->samples.size() / mbs, kInput,
                 "step_units: score table columns must equal the dataset's micro-batch units");
    D2FT_REQUIRE(!E.have_prefetch || (E.prefetch_B == n_mb * mbs &&
                                      std::equal(units, units + n_mb, E.prefetched_units.begin(),
                                                 E.prefetched_units.end())),
                 kState, "step_units: the prefetched batch holds other units");
    units_step(E, ds, units, n_mb, mbs, units_next, bwd_scores, fwd_scores, total_units, cf, cb, cap_full, cap_fwd, lr,
               momentum);
    check_status(E.finish_and_check());
    *loss_out = *E.h_loss;
    if (codes_out) std::memcpy(codes_out, E.h_codes, (size_t)E.D.K() * n_mb);
  });
}

// The batch body for a given schedule table (Standard / Random / Scaler /
// pruning policies, trainer.cpp:220-243 then :247-268) over dataset units.
int d2ft_engine_step_units_codes(d2ft_engine* h, const d2ft_dataset* ds, const int32_t* units, int n_mb, int mbs,
                                 const int32_t* units_next, const uint8_t* codes, double lr, double momentum,
                                 double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    validate_units(E, ds, units, n_mb, mbs);
    if (units_next) validate_units(E, ds, units_next, n_mb, mbs);
    D2FT_REQUIRE(codes && loss_out, kInput, "step_units: null argument");
    const int B = n_mb * mbs;
    D2FT_REQUIRE(B <= E.D.Bmax, kSize, "step: batch exceeds the engine capacity");
    for (size_t c = 0; c < (size_t)E.D.K() * n_mb; ++c)
      D2FT_REQUIRE(codes[c] >= 1 && codes[c] <= 3, kInput, "schedule table: code out of range");
    D2FT_REQUIRE(!E.have_prefetch || (E.prefetch_B == B && std::equal(units, units + n_mb, E.prefetched_units.begin(),
                                                                      E.prefetched_units.end())),
                 kState, "step_units: the prefetched batch holds other units");
    for (int j = 0; j < n_mb; ++j)
      for (int i = 0; i < mbs; ++i) E.h_labels[j * mbs + i] = ds->labels[(size_t)units[j] * mbs + i];
    validate_labels(E.h_labels, B, E.D.C);
    std::memcpy(E.h_codes, codes, (size_t)E.D.K() * n_mb);
    if (!E.have_prefetch) E.prefetch_units(ds->samples.data(), units, n_mb, mbs);
    E.begin_step(B);
    D2FT_CUDA(cudaMemcpyAsync(E.labels_dev, E.h_labels, B * 4, cudaMemcpyHostToDevice, E.st));
    D2FT_CUDA(cudaMemcpyAsync(E.codes_mb, E.h_codes, (size_t)E.D.K() * n_mb, cudaMemcpyHostToDevice, E.st));
    E.consume_prefetch(B);
    launch_expand_codes(E.codes_mb, E.D.K(), n_mb, mbs, B, E.D.Bmax, E.codes_exp, E.st);
    E.compact_and_plan();
    E.train_body((float)lr, (float)momentum);
    if (units_next) E.prefetch_units(ds->samples.data(), units_next, n_mb, mbs);
    check_status(E.finish_and_check());
    *loss_out = *E.h_loss;
  });
}

// bench.py's e2e leg through the Dataset path: `steps` batches whose units
// are order[i*n_mb .. (i+1)*n_mb) (the trainer's shuffled unit order), every
// step gathering its fp64 samples H2D (prefetched while the previous batch
// computes), slicing its scores, and reading loss + codes back with a host
// sync.  CUDA events on the engine stream; the first gather is inside.
int d2ft_engine_bench_e2e_units(d2ft_engine* h, const d2ft_dataset* ds, const int32_t* order, int n_mb, int mbs,
                                const double* bwd_scores, const double* fwd_scores, int total_units,
                                const int32_t* cf, const int32_t* cb, const int32_t* cap_full, const int32_t* cap_fwd,
                                double lr, double momentum, int warmup, int steps, double* ms_out, double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    D2FT_REQUIRE(warmup >= 0 && steps >= 1, kInput, "bench: steps must be positive");
    D2FT_REQUIRE(total_units == (int)ds->samples.size() / mbs, kInput,
                 "step_units: score table columns must equal the dataset's micro-batch units");
    for (int i = 0; i < warmup + steps; ++i) validate_units(E, ds, order + (size_t)i * n_mb, n_mb, mbs);
    D2FT_REQUIRE(!E.have_prefetch, kState, "bench: a prefetched batch is pending");
    for (int i = 0; i < warmup; ++i) {
      units_step(E, ds, order + (size_t)i * n_mb, n_mb, mbs, nullptr, bwd_scores, fwd_scores, total_units, cf, cb,
                 cap_full, cap_fwd, lr, momentum);
      check_status(E.finish_and_check());
    }
    cudaEvent_t e0, e1;
    D2FT_CUDA(cudaEventCreate(&e0));
    D2FT_CUDA(cudaEventCreate(&e1));
    D2FT_CUDA(cudaEventRecord(e0, E.st));
    D2FT_CUDA(cudaStreamWaitEvent(E.cst, e0, 0));  // the first gather is inside the timed region
    const int32_t* ord = order + (size_t)warmup * n_mb;
    const bool trace = getenv("D2FT_E2E_TRACE") != nullptr;  // host enqueue / sync split per step (stderr)
    for (int i = 0; i < steps; ++i) {
      const auto h0 = std::chrono::steady_clock::now();
      units_step(E, ds, ord + (size_t)i * n_mb, n_mb, mbs, i + 1 < steps ? ord + (size_t)(i + 1) * n_mb : nullptr,
                 bwd_scores, fwd_scores, total_units, cf, cb, cap_full, cap_fwd, lr, momentum);
      const auto h1 = std::chrono::steady_clock::now();
      check_status(E.finish_and_check());
      const auto h2 = std::chrono::steady_clock::now();
      if (trace)
        fprintf(stderr, "e2e units step %d: enqueue %.3f ms, sync %.3f ms\n", i,
                std::chrono::duration<double, std::milli>(h1 - h0).count(),
                std::chrono::duration<double, std::milli>(h2 - h1).count());
    }
    D2FT_CUDA(cudaEventRecord(e1, E.st));
    D2FT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = ms;
    if (loss_out) *loss_out = *E.h_loss;
  });
}

// bench.py's e2e leg: `steps` host-buffer steps (after `warmup`), each with its
// H2D copies and the loss/codes D2H and a host sync, CUDA-event timed on the
// engine stream.  ms_out = total milliseconds of the timed steps.
int d2ft_engine_bench_e2e(d2ft_engine* h, const float* samples, const int32_t* labels, const double* bwd_scores,
                          const double* fwd_scores, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                          const int32_t* cap_fwd, int n_mb, int mbs, double lr, double momentum, int warmup,
                          int steps, double* ms_out, double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    const int K = E.D.K();
    validate_sched_inputs(bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, K, n_mb);
    validate_labels(labels, E.local_B(n_mb, mbs), E.D.C);
    E.ensure_sched(max_cols_of(cf, cb, cap_full, cap_fwd, K, n_mb));
    // Every step copies its own samples H2D; the copy of batch i+1 runs on the
    // copy stream while batch i computes (the data-loader pipeline of
    // d2ft_engine_prefetch + d2ft_engine_step(samples = NULL, samples_next)).
    const int B = E.local_B(n_mb, mbs);
    for (int i = 0; i < warmup; ++i) {
      E.host_step(samples, labels, bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, n_mb, mbs, lr, momentum);
      check_status(E.finish_and_check());
    }
    cudaEvent_t e0, e1;
    D2FT_CUDA(cudaEventCreate(&e0));
    D2FT_CUDA(cudaEventCreate(&e1));
    D2FT_CUDA(cudaEventRecord(e0, E.st));
    D2FT_CUDA(cudaStreamWaitEvent(E.cst, e0, 0));  // the first copy is inside the timed region
    E.prefetch(samples, B);
    const bool trace = getenv("D2FT_E2E_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    for (int i = 0; i < steps; ++i) {
      const auto h0 = std::chrono::steady_clock::now();
      if (trace) {
        tev.emplace_back();
        D2FT_CUDA(cudaEventCreate(&tev.back()));
        D2FT_CUDA(cudaEventRecord(tev.back(), E.st));
      }
      E.host_step(nullptr, labels, bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, n_mb, mbs, lr, momentum,
                  i + 1 < steps ? samples : nullptr);
      const auto h1 = std::chrono::steady_clock::now();
      check_status(E.finish_and_check());
      const auto h2 = std::chrono::steady_clock::now();
      if (trace)
        fprintf(stderr, "e2e step %d: enqueue %.3f ms, sync %.3f ms\n", i,
                std::chrono::duration<double, std::milli>(h1 - h0).count(),
                std::chrono::duration<double, std::milli>(h2 - h1).count());
    }
    if (trace) {
      for (size_t i = 1; i < tev.size(); ++i) {
        float ms = 0.f;
        D2FT_CUDA(cudaEventElapsedTime(&ms, tev[i - 1], tev[i]));
        fprintf(stderr, "e2e gpu step %zu: %.3f ms\n", i - 1, ms);
      }
      for (auto e : tev) cudaEventDestroy(e);
    }
    D2FT_CUDA(cudaEventRecord(e1, E.st));
    D2FT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = ms;
    if (loss_out) *loss_out = *E.h_loss;
  });
}

// bench.py's device leg: `steps` device-resident steps on the staged inputs,
// CUDA-event timed on the engine stream (inputs already in HBM).
int d2ft_engine_bench_device(d2ft_engine* h, int n_mb, int mbs, double lr, double momentum, int warmup, int steps,
                             double* ms_out, double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    for (int i = 0; i < warmup; ++i) {
      E.begin_step(E.local_B(n_mb, mbs));
      E.compute_step(n_mb, mbs, lr, momentum);
    }
    check_status(E.finish_and_check());
    cudaEvent_t e0, e1;
    D2FT_CUDA(cudaEventCreate(&e0));
    D2FT_CUDA(cudaEventCreate(&e1));
    D2FT_CUDA(cudaEventRecord(e0, E.st));
    for (int i = 0; i < steps; ++i) {
      E.begin_step(E.local_B(n_mb, mbs));
      E.compute_step(n_mb, mbs, lr, momentum);
    }
    D2FT_CUDA(cudaEventRecord(e1, E.st));
    D2FT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = ms;
    check_status(E.finish_and_check());
    if (loss_out) *loss_out = *E.h_loss;
  });
}

int d2ft_engine_stage_device(d2ft_engine* h, const float* samples, const int32_t* labels, const double* bwd_scores,
                             const double* fwd_scores, const int32_t* cf, const int32_t* cb, const int32_t* cap_full,
                             const int32_t* cap_fwd, int n_mb, int mbs) {
  return guarded([&] {
    Engine& E = *h->e;
    const int K = E.D.K();
    const int B = E.local_B(n_mb, mbs);
    D2FT_REQUIRE(B >= 1 && B <= E.D.Bmax, kSize, "stage: batch exceeds the engine capacity");
    validate_sched_inputs(bwd_scores, fwd_scores, cf, cb, cap_full, cap_fwd, K, n_mb);
    validate_labels(labels, B, E.D.C);
    E.ensure_sched(max_cols_of(cf, cb, cap_full, cap_fwd, K, n_mb));
    const size_t KN = (size_t)K * n_mb;
    D2FT_CUDA(cudaMemcpy(E.samples_dev, samples, (size_t)B * E.D.T * E.D.d * 4, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.labels_dev, labels, B * 4, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.bwd_dev, bwd_scores, KN * 8, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.fwd_dev, fwd_scores, KN * 8, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.cf_dev, cf, K * 4, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.cb_dev, cb, K * 4, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.capf_dev, cap_full, K * 4, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(E.capo_dev, cap_fwd, K * 4, cudaMemcpyHostToDevice));
  });
}

// Device-resident step on the staged inputs: no host copies, no sync.
int d2ft_engine_step_resident(d2ft_engine* h, int n_mb, int mbs, double lr, double momentum) {
  return guarded([&] {
    Engine& E = *h->e;
    E.begin_step(E.local_B(n_mb, mbs));
    E.compute_step(n_mb, mbs, lr, momentum);
  });
}

int d2ft_engine_sync(d2ft_engine* h, double* loss_out) {
  return guarded([&] {
    Engine& E = *h->e;
    check_status(E.finish_and_check());
    if (loss_out) *loss_out = *E.h_loss;
  });
}

void* d2ft_engine_stream(d2ft_engine* h) { return h && h->e ? (void*)h->e->st : nullptr; }

int d2ft_engine_set_row_owner(d2ft_engine* h, const int32_t* owner, int K) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && owner, kInput, "set_row_owner: null argument");
    D2FT_REQUIRE(K == h->e->D.K(), kInput, "set_row_owner: one owner per scheduled subnet");
    D2FT_CUDA(cudaStreamSynchronize(h->e->st));
    h->e->set_row_owner(owner);
  });
}

int d2ft_engine_set_exchange_chunks(d2ft_engine* h, int chunks) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e, kInput, "set_exchange_chunks: null argument");
    D2FT_REQUIRE(chunks >= 1 && chunks <= Engine::kMaxXChunks, kConfig, "exchange chunks: 1..8");
    h->e->drop_graph();
    h->e->xchunks = chunks;
  });
}

int d2ft_engine_exchange_stats(d2ft_engine* h, unsigned long long* calls, unsigned long long* bytes) {
  return guarded([&] {
    D2FT_REQUIRE(h && h->e && calls && bytes, kInput, "exchange_stats: null argument");
    D2FT_CUDA(cudaStreamSynchronize(h->e->st));
    const Exchange* xx = h->e->ex ? h->e->ex.get() : h->e->dpx.get();
    *calls = xx ? xx->calls : 0;
    *bytes = xx ? xx->bytes : 0;
  });
}

int d2ft_engine_set_profiling(d2ft_engine* h, int on) {
  return guarded([&] {
    Engine& E = *h->e;
    E.profiling = on != 0;
    for (double& v : E.phase_ms) v = 0.0;
    E.profiled_steps = 0;
  });
}

int d2ft_engine_phase_ms(d2ft_engine* h, double* ms_out, int n, int* steps) {
  return guarded([&] {
    Engine& E = *h->e;
    for (int i = 0; i < n && i < PH_COUNT; ++i) ms_out[i] = E.phase_ms[i];
    if (steps) *steps = E.profiled_steps;
  });
}

int d2ft_engine_codes(d2ft_engine* h, uint8_t* codes_exp_out) {
  return guarded([&] {
    Engine& E = *h->e;
    D2FT_CUDA(cudaStreamSynchronize(E.st));
    D2FT_CUDA(cudaMemcpy(codes_exp_out, E.codes_exp, (size_t)E.D.K() * E.D.Bmax, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
