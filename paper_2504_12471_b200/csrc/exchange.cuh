// Head-partitioned D2FT across ranks: rank r of `world` owns
// the heads h with h % world == r of every block, so each rank computes a
// PARTIAL block output (sum over its active heads) and a partial dxn (sum
// over its Full heads).  The one data-path exchange per block and direction
// is a sum of those partials, identical on every rank.  Exchange is that sum:
// NCCL all-reduce between processes (one GPU each), or an in-process group of
// engines on one device (deterministic fixed-order sum; test harness for the
// partitioned path on a single GPU).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>

namespace d2ft_b200 {

struct Exchange {
  int rank = 0, world = 1;
  unsigned long long calls = 0, bytes = 0;  // all-reduces issued and their payload bytes (this rank)
  virtual ~Exchange() = default;
  // in place: buf[i] <- sum over ranks of buf[i]; stream-ordered on `st`.
  // Every call is issued, world 1 included (the NCCL data path runs on a
  // one-GPU box too).
  virtual void allreduce_sum(float* buf, size_t n, cudaStream_t st) = 0;
  // stream-ordered without host synchronisation (can be captured in a CUDA graph)
  virtual bool capturable() const = 0;
};

void nccl_unique_id(uint8_t out[128]);
std::unique_ptr<Exchange> make_nccl_exchange(int rank, int world, const uint8_t id[128]);

struct LocalGroup;
LocalGroup* local_group_create(int world);
void local_group_destroy(LocalGroup* g);
// wake every rank waiting in the group's exchange with a state error (a peer failed)
void local_group_abort(LocalGroup* g);
std::unique_ptr<Exchange> make_local_exchange(LocalGroup* g, int rank);

// codes[k][s] = 3 (skip) for the scheduled rows k another rank owns (owner[k] != rank)
void launch_mask_rows(uint8_t* codes, int K, int Bmax, const int* owner, int rank, cudaStream_t st);

}  // namespace d2ft_b200
