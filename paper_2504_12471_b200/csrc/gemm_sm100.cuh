// Persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   D[m][n] = sum_k A[m][k] * B[n][k]     (fp16/bf16 operands, fp32 accumulate in TMEM)
//
// Both operands are K-major and arrive by TMA (128-byte swizzle) from 3-D
// tensor maps, so a problem can gather rows from anywhere (per-head weight
// units, per-sample token planes) and K can be a concatenation of segments
// (active heads of a sample, Full micro-batches of a head).  Out-of-range rows
// or tokens are zero-filled by TMA.  A problem policy P supplies the tile list,
// the per-k-block TMA coordinates and a fused epilogue:
//
//   struct P {
//     struct Tile { int nkb; ... };                 // nkb == 0: accumulator is zero
//     struct Row { ... };                            // per-thread epilogue state
//     __device__ int ntiles() const;                 // tile slots (pairs when CLUSTER == 2)
//     __device__ void tile(int t, int rank, Tile&) const;
//     __device__ KCoord kcoord(const Tile&, int kb) const;
//     __device__ void row_begin(const Tile&, int row, Row&) const;
//     __device__ void chunk(const Tile&, int row, int col0, const float (&v)[16], Row&) const;
//     __device__ void row_end(const Tile&, int row, int group, Row&) const;
//   };
//
// CLUSTER == 2: the two CTAs of a cluster work on the two tiles of a slot,
// which share the B operand (same sample / plane) and the k-block count.  Each
// CTA loads its own A and HALF of B, multicast to both CTAs; MMA completion is
// committed to both CTAs' empty barriers.  Per CTA this cuts the TMA operand
// traffic from A+B to A+B/2 per k-block (the single-CTA kernel is L2->SM
// operand-feed bound).
//
// Roles: warp 0 = TMA producer, warp 1 = MMA issuer (one thread), warp 2 =
// TMEM allocator, warps 4.. = EPI epilogue warpgroups (TMEM lane quarter =
// warp % 4, column group = (warp - 4) / 4).  Tile M = 128 (two 64-row A
// boxes), N = BN, K-block = 64.  Two TMEM accumulators (columns 0 and 256) let
// the epilogue of tile i overlap the MMAs of tile i+1.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "ptx.cuh"
#include <type_traits>
#include <utility>

namespace d2ft_b200 {

struct KCoord {
  int ax, ay0, ay1, az;  // A: k offset, row of the first/second 64-row half, plane
  int bx, by, bz;        // B: k offset, first row of the (full) B tile, plane
};

// FMT: operand format, 0 = fp16 (the step), 1 = bf16 (self-tests).
// EPI: epilogue warpgroups; group e drains column chunks e, e+EPI, ... of the
// accumulator, so EPI x more epilogue loads/stores are in flight per SM.
// CLUSTER: 1, or 2 for the B-sharing CTA pair.
// Optional epilogue hook P::prefetch(tile, row, col0, row_state): issued for
// the warp's first chunk right after the tile's accumulator wait (before the
// TMEM load), so a problem that reads a per-element operand in its epilogue
// can keep that load one chunk ahead.
template <class P, class = void>
struct has_prefetch : std::false_type {};
template <class P>
struct has_prefetch<P, std::void_t<decltype(&P::prefetch)>> : std::true_type {};

// BMN: B operand layout.  0 = K-major (rows of B are the N index, K
// contiguous; one TMA box of BK x BN, or BK x BN/2 per CTA of a pair).
// 1 = MN-major (B stored as [K][N] with N contiguous, e.g. a feature-major
// activation whose N is tokens): the stage holds ceil(BN/64) blocks of
// 64 K-rows x 64 N-elements (one 8 KB TMA box of 64 N x 64 K each, 128-byte
// swizzle), read by UMMA with LBO = 8 KB (next 64-element N block) and
// SBO = 1 KB (next 8 K-rows); the CTAs of a pair load alternate blocks.
// Optional P::ksteps(tile, kb): number of 16-wide K steps of k-block kb that
// carry data (1..4); the MMA skips the rest (tokens-as-K problems whose last
// 64-token block of a sample holds T % 64 tokens).
template <class P, class = void>
struct has_ksteps : std::false_type {};
template <class P>
struct has_ksteps<P, std::void_t<decltype(&P::ksteps)>> : std::true_type {};

// Optional member `int* ctr` (zeroed before the launch): dynamic tile
// scheduling instead of the static slot0 + i*nslots striding.
template <class P, class = void>
struct has_counter : std::false_type {};
template <class P>
struct has_counter<P, std::void_t<decltype(std::declval<P>().ctr)>> : std::true_type {};
constexpr int kTileQ = 4;

// Optional `static constexpr int kEpiStageBytes` (> 0): that many bytes of
// shared memory per epilogue warp, handed to the problem as Row::stage before
// row_begin (staging for bulk tensor stores); the kernel drains the warp's
// bulk stores before exiting.
template <class P, class = void>
struct epi_stage_bytes : std::integral_constant<int, 0> {};
template <class P>
struct epi_stage_bytes<P, std::void_t<decltype(P::kEpiStageBytes)>> : std::integral_constant<int, P::kEpiStageBytes> {};
// Optional `static constexpr int kChunk` (16 or 32): accumulator columns per
// epilogue chunk (TMEM load + P::chunk call); default 16.  Optional
// `static constexpr bool kNonEmpty = true`: no tile has nkb == 0 (skips the
// zero-accumulator selects).
template <class P, class = void>
struct chunk_cols : std::integral_constant<int, 16> {};
template <class P>
struct chunk_cols<P, std::void_t<decltype(P::kChunk)>> : std::integral_constant<int, P::kChunk> {};
// Optional P::ncols(tile): accumulator columns that carry data (e.g. T tokens
// of a BN-wide tile); the epilogue neither loads nor drains chunks past it.
template <class P, class = void>
struct has_ncols : std::false_type {};
template <class P>
struct has_ncols<P, std::void_t<decltype(&P::ncols)>> : std::true_type {};
template <class P, class = void>
struct non_empty : std::false_type {};
template <class P>
struct non_empty<P, std::void_t<decltype(P::kNonEmpty)>> : std::integral_constant<bool, P::kNonEmpty> {};

// Tile ring and k-block queue, both filled by warp 3 (the scheduler warp):
// it resolves each tile's coordinates (prob.tile: the dependent global loads
// of tile lists and head lists) up to kRing tiles ahead into the ring, and
// every k-block's TMA coordinates (prob.kcoord, incl. its integer divisions
// and list lookups) into the kKQ-deep k-block queue.  The producer then only
// pops ready coordinates and issues TMA: ncu showed the producer thread busy
// ~80% of G3 computing coordinates, with the MMA waiting on data ~60%.
constexpr int kRing = 4;
constexpr int kKQ = 16;
template <class P>
struct alignas(16) RingEntry {
  int t;
  int flags;  // resident-B mode: kNewB (first tile of its B plane) | kLastB (last one)
  typename P::Tile c;
};
constexpr int kNewB = 1, kLastB = 2;
struct alignas(16) KRec {
  KCoord k;
  int nk;  // 16-wide K steps of the k-block that carry data (P::ksteps)
};
template <class P>
struct SchedSmem {
  RingEntry<P> ring[kRing];
  KRec kq[kKQ];
  uint64_t ring_full[kRing], ring_empty[kRing], kq_full[kKQ], kq_empty[kKQ];
};
template <class P, class S>
constexpr int gemm_sched_offset() {  // after the epilogue staging
  return S::MAIN_BYTES + 512 + 4 * S::EPI * epi_stage_bytes<P>::value;
}

template <class P, class S>
constexpr int gemm_smem_bytes() {
  return S::SMEM_BYTES + 4 * S::EPI * epi_stage_bytes<P>::value + (int)sizeof(SchedSmem<P>);
}

// AMN: A operand layout.  0 = K-major; 1 = MN-major (A stored [K][M] with M
// contiguous, e.g. a weight matrix kept in the other GEMM's orientation): the
// two 64-row halves of the tile are two 64(M) x 64(K) boxes, LBO = 8 KB.
// CG2: pair UMMA (`tcgen05.mma.cta_group::2`, M = 256 across the CTA pair):
// each CTA holds its own 128 A rows and HALF of B (N/2 rows) — B is split, not
// multicast, so a stage is A + B/2 bytes per CTA and more stages fit; the even
// CTA issues the MMAs for both, its mbarriers count both CTAs' TMA bytes, and
// its commits arrive on both CTAs' barriers.  K-major B only.
// RES > 0: resident B (pair UMMA, K-major B, static tile ranges only).  The
// CTA's half of B for all RES k-blocks of a plane stays in shared memory
// across the consecutive tiles that share the plane (a sample's unit groups
// in G1), so only A streams through the STAGES ring.  Per k-block barriers:
// the MMA of the first tile of a plane waits bfull[kb]; the MMA of the last
// tile commits bempty[kb] after its k-block kb, and the producer of the next
// plane reloads block kb behind it.
template <int BN_, int STAGES_, int FMT_ = 0, int EPI_ = 4, int CLUSTER_ = 1, int BMN_ = 0, int AMN_ = 0,
          int CG2_ = 0, int RES_ = 0>
struct GemmShape {
  static constexpr int BM = 128, BK = 64, BN = BN_, STAGES = STAGES_, FMT = FMT_, EPI = EPI_, CLUSTER = CLUSTER_;
  static constexpr int BMN = BMN_, AMN = AMN_, CG2 = CG2_, RES = RES_;
  static_assert(!CG2 || CLUSTER == 2, "pair UMMA needs a CTA pair");
  static_assert(!RES || (CG2 && !BMN && RES <= 16), "resident B: pair UMMA, K-major B, <= 16 k-blocks");
  // MN-major B: 64-wide N blocks held per CTA (pair UMMA: of this CTA's N/2)
  static constexpr int NBLK = CG2 ? (BN / 2 + 63) / 64 : (BN + 63) / 64;
  static constexpr int THREADS = 128 + 128 * EPI;
  static constexpr int A_BYTES = BM * BK * 2;
  // B bytes held per CTA and stage (CG2: this CTA's N/2 rows)
  static constexpr int B_BYTES = BMN ? NBLK * 64 * BK * 2 : (CG2 ? BN * BK : BN * BK * 2);
  static constexpr int B_PART = CG2 ? B_BYTES : B_BYTES / CLUSTER;  // bytes of B each CTA loads (K-major)
  static constexpr int STAGE_BYTES = RES ? A_BYTES : A_BYTES + B_BYTES;  // bytes a stage's TMA brings per CTA
  static constexpr int B_SLOTS = RES ? RES : STAGES;  // B blocks held: resident plane or one per stage
  static constexpr int MAIN_BYTES = STAGES * A_BYTES + B_SLOTS * B_BYTES;
  static constexpr int SMEM_BYTES = MAIN_BYTES + 1024 + 512;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N");
  static_assert(BMN || (B_BYTES % 1024 == 0 && B_PART % 1024 == 0),
                "B stage parts must keep 1024-byte swizzle alignment");
  static_assert(CLUSTER == 1 || CLUSTER == 2, "cluster of 1 or 2");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};

template <class P, class S>
__global__ void __launch_bounds__(S::THREADS, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const P prob) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S::B_SLOTS * S::B_BYTES);
  uint64_t* empty = full + S::STAGES;
  uint64_t* tfull = empty + S::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* tq_full = tempty + 2;        // rank 0 -> rank 1 tile-id queue (dynamic scheduling)
  uint64_t* tq_empty = tq_full + kTileQ;
  uint64_t* bfull = tq_empty + kTileQ;   // resident B, per k-block (RES)
  uint64_t* bempty = bfull + S::RES;
  int* tq = reinterpret_cast<int*>(bempty + S::RES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kTileQ);
  // per-epilogue-warp staging (epi_stage_bytes), 128-byte aligned, after the barriers
  uint8_t* epi_stage = sB + S::B_SLOTS * S::B_BYTES + 512;
  SchedSmem<P>& sch = *reinterpret_cast<SchedSmem<P>*>(smem + gemm_sched_offset<P, S>());
  RingEntry<P>* ring = sch.ring;
  uint64_t* ring_full = sch.ring_full;
  uint64_t* ring_empty = sch.ring_empty;
  KRec* kq = sch.kq;
  uint64_t* kq_full = sch.kq_full;
  uint64_t* kq_empty = sch.kq_empty;

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = S::CLUSTER == 2 ? (int)ptx::cluster_rank() : 0;
  const int slot0 = blockIdx.x / S::CLUSTER, nslots = gridDim.x / S::CLUSTER;
  constexpr uint16_t kPair = 0x3;
  constexpr bool kDyn = has_counter<P>::value;
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int i = 0; i < S::STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      // multicast B: both CTAs' MMAs read the stage; pair UMMA: the even CTA's commit
      ptx::mbar_init(&empty[i], S::CG2 ? 1 : S::CLUSTER);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4 * S::EPI * (S::CG2 ? 2 : 1));  // pair UMMA: both CTAs' epilogues
    }
    for (int i = 0; i < S::RES; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bempty[i], 1);  // the even CTA's commit, multicast to both
    }
    for (int i = 0; i < kTileQ; ++i) {
      ptx::mbar_init(&tq_full[i], 1);
      ptx::mbar_init(&tq_empty[i], 1);  // rank 1's scheduler
    }
    for (int i = 0; i < kRing; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 2 + 4 * S::EPI);  // producer, MMA warp, epilogue warps
    }
    for (int i = 0; i < kKQ; ++i) {
      ptx::mbar_init(&kq_full[i], 1);
      ptx::mbar_init(&kq_empty[i], has_ksteps<P>::value ? 2 : 1);  // producer (+ MMA warp for ksteps)
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (S::CG2) ptx::tmem_alloc_cg2(tmem_slot, 512);
    else ptx::tmem_alloc(tmem_slot, 512);
  }
  ptx::tc_fence_before();
  if (S::CLUSTER == 2) ptx::cluster_sync();  // peers' barriers exist before any multicast
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the prologue above overlapped the previous kernel's tail
  const int ntiles = prob.ntiles();

  // Tile sequence, produced by warp 3 into the ring.  Static: slot0, slot0 +
  // nslots, ...  Dynamic (P has `ctr`): rank 0's scheduler claims slots with
  // atomicAdd on prob.ctr (the problem orders its slots by decreasing cost)
  // and hands each id to rank 1's scheduler through the kTileQ-deep queue;
  // ids >= ntiles end every role's loop.
  auto for_each_tile = [&](bool leader, auto&& body) {
    for (int i = 0;; ++i) {
      const int q = i % kRing;
      ptx::mbar_wait(&ring_full[q], (i / kRing) & 1);
      if (ring[q].t >= ntiles) break;
      body(static_cast<const typename P::Tile&>(ring[q].c), ring[q].flags);
      __syncwarp(__activemask());
      if (leader) ptx::mbar_arrive(&ring_empty[q]);
    }
  };

  if (warp == 3) {
    if (lane == 0) {
      int kqi = 0;
      auto push = [&](int i, int t, int flags = 0) {
        const int q = i % kRing;
        typename P::Tile c{};
        if (t < ntiles) prob.tile(t, rank, c);  // global loads resolve before the slot is needed
        ptx::mbar_wait(&ring_empty[q], ((i / kRing) & 1) ^ 1);
        ring[q].t = t;
        ring[q].flags = flags;
        ring[q].c = c;
        ptx::mbar_arrive(&ring_full[q]);
        if (t >= ntiles) return;
        for (int kb = 0; kb < c.nkb; ++kb, ++kqi) {
          KRec rec;
          rec.k = prob.kcoord(c, kb);
          rec.nk = S::BK / 16;
          if constexpr (has_ksteps<P>::value) rec.nk = prob.ksteps(c, kb);
          const int j = kqi % kKQ;
          ptx::mbar_wait(&kq_empty[j], ((kqi / kKQ) & 1) ^ 1);
          kq[j] = rec;
          ptx::mbar_arrive(&kq_full[j]);
        }
      };
      bool dyn = false;
      if constexpr (kDyn) dyn = prob.ctr != nullptr;  // a null counter selects static striding
      if (dyn) {
        for (int i = 0;; ++i) {
          int t;
          if (rank == 0) {
            // claim only once the ring slot is free: claiming further ahead
            // than the pipeline needs unbalances the end of the launch
            ptx::mbar_wait(&ring_empty[i % kRing], ((i / kRing) & 1) ^ 1);
            if constexpr (kDyn) t = atomicAdd(prob.ctr, 1);
            if (S::CLUSTER == 2) {
              const int q = i % kTileQ;
              ptx::mbar_wait_cluster(&tq_empty[q], ((i / kTileQ) & 1) ^ 1);
              ptx::st_cluster_u32(ptx::mapa(&tq[q], 1), (uint32_t)t);
              ptx::mbar_arrive_cluster(ptx::mapa(&tq_full[q], 1));
            }
          } else {
            const int q = i % kTileQ;
            ptx::mbar_wait_cluster(&tq_full[q], (i / kTileQ) & 1);
            t = *reinterpret_cast<volatile int*>(&tq[q]);
            ptx::mbar_arrive_cluster(ptx::mapa(&tq_empty[q], 0));
          }
          push(i, t);
          if (t >= ntiles) break;
        }
      } else if (S::RES) {
        // contiguous tile range per slot; a tile's B plane = its k-block 0 coordinate
        const int t0 = (int)((long long)slot0 * ntiles / nslots), t1 = (int)((long long)(slot0 + 1) * ntiles / nslots);
        auto plane = [&](int t) {
          typename P::Tile c{};
          prob.tile(t, rank, c);
          return prob.kcoord(c, 0).bz;
        };
        int cur = t0 < t1 ? plane(t0) : -1, prev = -1;
        for (int i = 0;; ++i) {
          const int t = t0 + i;
          if (t >= t1) {
            push(i, ntiles);
            break;
          }
          const int nxt = t + 1 < t1 ? plane(t + 1) : -1;
          push(i, t, (cur != prev ? kNewB : 0) | (nxt != cur ? kLastB : 0));
          prev = cur;
          cur = nxt;
        }
      } else {
        for (int i = 0;; ++i) {
          const int t = slot0 + i * nslots;
          push(i, t < ntiles ? t : ntiles);
          if (t >= ntiles) break;
        }
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int kqi = 0;
      uint32_t bph = 0;  // resident B: loads of the plane so far (parity)
      for_each_tile(true, [&](const typename P::Tile& c, int flags) {
        const int nkb = c.nkb;
        for (int kb = 0; kb < nkb; ++kb, ++kqi) {
          const int j = kqi % kKQ;
          ptx::mbar_wait(&kq_full[j], (kqi / kKQ) & 1);
          const KCoord k = kq[j].k;
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * S::A_BYTES;
          if constexpr (S::CG2) {
            // both CTAs' bytes complete on the even CTA's full barrier
            const uint32_t fb = ptx::mapa(&full[stage], 0);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE_BYTES);
            if constexpr (S::RES) {
              if (flags & kNewB) {  // block kb of the new plane, once the last tile of the old one read it
                ptx::mbar_wait(&bempty[kb], bph ^ 1);
                if (rank == 0) ptx::mbar_arrive_expect_tx(&bfull[kb], 2 * S::B_BYTES);
                ptx::tma_load_3d_cg2(sB + kb * S::B_BYTES, &tmB, ptx::mapa(&bfull[kb], 0), k.bx,
                                     k.by + rank * (S::BN / 2), k.bz);
              }
            }
            if constexpr (S::AMN) {
              ptx::tma_load_3d_cg2(a, &tmA, fb, k.ay0, k.ax, k.az);
              ptx::tma_load_3d_cg2(a + S::A_BYTES / 2, &tmA, fb, k.ay1, k.ax, k.az);
            } else {
              ptx::tma_load_3d_cg2(a, &tmA, fb, k.ax, k.ay0, k.az);
              ptx::tma_load_3d_cg2(a + S::A_BYTES / 2, &tmA, fb, k.ax, k.ay1, k.az);
            }
            if constexpr (S::RES) {
            } else if constexpr (S::BMN) {  // this CTA's N/2 tokens from k.bx + rank * BN/2, 64 per box
              for (int j2 = 0; j2 < S::NBLK; ++j2)
                ptx::tma_load_3d_cg2(sB + stage * S::B_BYTES + j2 * (64 * S::BK * 2), &tmB, fb,
                                     k.bx + rank * (S::BN / 2) + 64 * j2, k.by, k.bz);
            } else {
              ptx::tma_load_3d_cg2(sB + stage * S::B_BYTES, &tmB, fb, k.bx, k.by + rank * (S::BN / 2), k.bz);
            }
            ptx::mbar_arrive(&kq_empty[j]);
            if (++stage == S::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          ptx::mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
          if constexpr (S::AMN) {  // boxes of 64 M (inner) x 64 K rows
            ptx::tma_load_3d(a, &tmA, &full[stage], k.ay0, k.ax, k.az);
            ptx::tma_load_3d(a + S::A_BYTES / 2, &tmA, &full[stage], k.ay1, k.ax, k.az);
          } else {
            ptx::tma_load_3d(a, &tmA, &full[stage], k.ax, k.ay0, k.az);
            ptx::tma_load_3d(a + S::A_BYTES / 2, &tmA, &full[stage], k.ax, k.ay1, k.az);
          }
          if constexpr (S::BMN) {  // k.bx = first N element, k.by = first K row
            for (int j = rank; j < S::NBLK; j += S::CLUSTER) {
              uint8_t* b = sB + stage * S::B_BYTES + j * (64 * S::BK * 2);
              if (S::CLUSTER == 2) ptx::tma_load_3d_mc(b, &tmB, &full[stage], k.bx + 64 * j, k.by, k.bz, kPair);
              else ptx::tma_load_3d(b, &tmB, &full[stage], k.bx + 64 * j, k.by, k.bz);
            }
          } else if (S::CLUSTER == 2) {
            ptx::tma_load_3d_mc(sB + stage * S::B_BYTES + rank * S::B_PART, &tmB, &full[stage], k.bx,
                                k.by + rank * (S::BN / 2), k.bz, kPair);
          } else {
            ptx::tma_load_3d(sB + stage * S::B_BYTES, &tmB, &full[stage], k.bx, k.by, k.bz);
          }
          ptx::mbar_arrive(&kq_empty[j]);
          if (++stage == S::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (S::RES && (flags & kNewB)) bph ^= 1;
      });
    }
  } else if (warp == 1) {
    // The whole warp runs the MMA loop (warp-uniform control flow keeps the
    // descriptors in uniform registers); one elected lane issues the UMMAs
    // and commits.
    constexpr uint32_t idesc = ptx::idesc_f16(S::CG2 ? 256 : 128, S::BN, S::FMT) | (S::AMN ? (1u << 15) : 0u) |
                               (S::BMN ? (1u << 16) : 0u);
    // pair UMMA: the odd CTA's MMA warp only keeps the ring / k-block queue flowing
    const bool issuer = !S::CG2 || rank == 0;
    int stage = 0, acc = 0, kqm = 0;
    uint32_t phase = 0, acc_phase = 0, bph = 0;
    for_each_tile(lane == 0, [&](const typename P::Tile& cref, int flags) {
      const typename P::Tile c = cref;  // registers (smem reads would be re-done around every store)
      if (!issuer) {
        if constexpr (has_ksteps<P>::value) {
          for (int kb = 0; kb < c.nkb; ++kb, ++kqm) {
            const int j = kqm % kKQ;
            ptx::mbar_wait(&kq_full[j], (kqm / kKQ) & 1);
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&kq_empty[j]);
          }
        }
        return;
      }
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem + acc * 256;
      for (int kb = 0; kb < c.nkb; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t as = ptx::smem_u32(sA + stage * S::A_BYTES);
        const uint64_t ad = S::AMN ? ptx::desc_sw128_mn(as, S::A_BYTES / 2) : ptx::desc_sw128(as);
        if (S::RES && (flags & kNewB)) {
          ptx::mbar_wait(&bfull[kb], bph);
          ptx::tc_fence_after();
        }
        const uint32_t bs = ptx::smem_u32(sB + (S::RES ? kb : stage) * S::B_BYTES);
        const uint64_t bd = S::BMN ? ptx::desc_sw128_mn(bs, 64 * S::BK * 2) : ptx::desc_sw128(bs);
        // K step of 16: +32 B along a K-major row, or +16 rows (2 KB) of an MN-major block
        constexpr uint64_t astep = S::AMN ? (16 * 128) >> 4 : 2;
        constexpr uint64_t bstep = S::BMN ? (16 * 128) >> 4 : 2;
        int nk = S::BK / 16;
        if constexpr (has_ksteps<P>::value) {
          const int j = kqm % kKQ;
          ptx::mbar_wait(&kq_full[j], (kqm / kKQ) & 1);
          nk = kq[j].nk;
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&kq_empty[j]);
          ++kqm;
        }
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < S::BK / 16; ++kk)
            if (kk < nk) {
              if constexpr (S::CG2)
                ptx::umma_f16_cg2(d, ad + (uint64_t)kk * astep, bd + (uint64_t)kk * bstep, idesc, (kb | kk) != 0);
              else
                ptx::umma_bf16(d, ad + (uint64_t)kk * astep, bd + (uint64_t)kk * bstep, idesc, (kb | kk) != 0);
            }
          if constexpr (S::CG2) ptx::umma_commit_cg2_mc(&empty[stage], kPair);
          else if (S::CLUSTER == 2) ptx::umma_commit_mc(&empty[stage], kPair);
          else ptx::umma_commit(&empty[stage]);
          // the plane's last tile has read B block kb: both producers may reload it
          if (S::RES && (flags & kLastB)) ptx::umma_commit_cg2_mc(&bempty[kb], kPair);
        }
        __syncwarp();
        if (++stage == S::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (S::RES && (flags & kNewB)) bph ^= 1;
      if (ptx::elect_one()) {
        if constexpr (S::CG2) ptx::umma_commit_cg2_mc(&tfull[acc], kPair);  // both CTAs' epilogues
        else ptx::umma_commit(&tfull[acc]);
      }
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
  } else if (warp >= 4) {
    const int q = warp & 3;         // TMEM lane quarter
    const int e = (warp - 4) >> 2;  // column group
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for_each_tile(lane == 0, [&](const typename P::Tile& cref, int) {
      const typename P::Tile c = cref;
      // Chunks of this warp: 16*e + i*16*EPI.  Row state and the first
      // chunk's epilogue operands are loaded before the accumulator wait (they
      // do not depend on it), and the accumulator is released to the MMA warp
      // as soon as the warp's last TMEM load has landed.
      constexpr int CW = chunk_cols<P>::value;
      const bool have = non_empty<P>::value || c.nkb > 0;
      int ncol = S::BN;
      if constexpr (has_ncols<P>::value) ncol = min(ncol, prob.ncols(c));
      const int nch = ncol > CW * e ? (ncol - CW * e + CW * S::EPI - 1) / (CW * S::EPI) : 0;
      auto col_of = [&](int i) { return CW * e + i * CW * S::EPI; };
      typename P::Row st;
      if constexpr (epi_stage_bytes<P>::value > 0) st.stage = epi_stage + (warp - 4) * epi_stage_bytes<P>::value;
      prob.row_begin(c, row, st);
      if constexpr (has_prefetch<P>::value) {
        if (nch > 0) prob.prefetch(c, row, col_of(0), st);
      }
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t base = tmem + acc * 256 + ((uint32_t)(q * 32) << 16);
      auto release = [&]() {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (S::CG2 && rank != 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(&tempty[acc], 0));  // the issuing CTA's
          else ptx::mbar_arrive(&tempty[acc]);
        }
      };
#pragma unroll 1
      for (int i = 0; i < nch; ++i) {
        uint32_t b0[CW];
        if (have) {
          if constexpr (CW == 32) {
            ptx::tmem_ld16_async(base + col_of(i), *reinterpret_cast<uint32_t(*)[16]>(&b0[0]));
            ptx::tmem_ld16_async(base + col_of(i) + 16, *reinterpret_cast<uint32_t(*)[16]>(&b0[16]));
          } else {
            ptx::tmem_ld16_async(base + col_of(i), b0);
          }
          ptx::tmem_ld_wait(b0);
        }
        if (i + 1 == nch) release();
        float v[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) v[j] = have ? __uint_as_float(b0[j]) : 0.f;
#ifndef D2FT_EXP_NOEPI
        prob.chunk(c, row, col_of(i), v, st);
#else
        if (v[0] == 12345.f) prob.chunk(c, row, col_of(i), v, st);  // experiment: epilogue stores off
#endif
      }
      if (nch == 0) release();
      prob.row_end(c, row, e, st);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
    if constexpr (epi_stage_bytes<P>::value > 0) {
      if (lane == 0) ptx::bulk_wait0();
    }
  }
  ptx::tc_fence_before();
  // the peer may still commit into our empty barriers / multicast into our smem
  if (S::CLUSTER == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if constexpr (S::CG2) ptx::tmem_dealloc_cg2(tmem, 512);
    else ptx::tmem_dealloc(tmem, 512);
  }
}

// Host side -----------------------------------------------------------------
// 3-D 16-bit tensor map: dim0 contiguous (elements), dim1 rows, dim2 planes;
// strides in bytes (multiples of 16); box = 64 x box_rows x 1, 128-byte
// swizzle, zero fill out of bounds.  fp16 (step operands) or bf16.
CUtensorMap make_tmap_16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                            uint64_t stride2_bytes, uint32_t box_rows, bool bf16);
inline CUtensorMap make_tmap_bf16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                                     uint64_t s2, uint32_t box_rows) {
  return make_tmap_16_3d(base, d0, d1, d2, s1, s2, box_rows, true);
}
inline CUtensorMap make_tmap_f16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                                    uint64_t s2, uint32_t box_rows) {
  return make_tmap_16_3d(base, d0, d1, d2, s1, s2, box_rows, false);
}
// fp16 map for bulk tensor STORES: box = box0 x box1 x 1; the staging tile is
// row-major [box1][box0], plain or swizzled with swizzle_bytes == box0 * 2
// (32 or 64); writes past d0/d1 are clipped.
CUtensorMap make_tmap_store_f16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                                   uint32_t box0, uint32_t box1, int swizzle_bytes = 0);
// fp32 variant (box0 fp32 elements per row; swizzle_bytes == box0 * 4)
CUtensorMap make_tmap_store_f32_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                                   uint32_t box0, uint32_t box1, int swizzle_bytes = 0);

int num_sms();

// Launch: persistent grid of ~one CTA (CLUSTER == 2: one CTA pair per two
// SMs) per SM.  The B tensor map's box must be BN / CLUSTER rows.
template <class P, class S>
void launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const P& prob, int max_ctas, cudaStream_t stream) {
  static_assert(gemm_smem_bytes<P, S>() <= 227 * 1024, "shared memory (stages + epilogue staging)");
  static unsigned long long attr = 0;
  once_per_device(attr, [&] {
    D2FT_CUDA(cudaFuncSetAttribute(gemm_sm100_kernel<P, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   gemm_smem_bytes<P, S>()));
  });
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (max_ctas < 0) grid = -max_ctas;  // explicit grid (may exceed the SM count: non-persistent)
  grid -= grid % S::CLUSTER;
  if (grid < S::CLUSTER) grid = S::CLUSTER;
  if (S::CLUSTER == 1) {
    gemm_sm100_kernel<P, S><<<grid, S::THREADS, gemm_smem_bytes<P, S>(), stream>>>(a, b, prob);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(S::THREADS);
    cfg.dynamicSmemBytes = gemm_smem_bytes<P, S>();
    cfg.stream = stream;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = S::CLUSTER;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    D2FT_CUDA(cudaLaunchKernelEx(&cfg, gemm_sm100_kernel<P, S>, a, b, prob));
  }
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace d2ft_b200
