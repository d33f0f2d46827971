// Exchange implementations (exchange.cuh).  NCCL is resolved with dlopen at
// the first partitioned engine, so single-GPU use never needs it; a process
// that already loaded NCCL (torch) shares that copy (same SONAME).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "exchange.cuh"

namespace d2ft_b200 {

// ------------------------------------------------------------------ NCCL
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = dlerror() ? dlerror() : "dlopen failed";
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
  });
  D2FT_REQUIRE(api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string,
               kCuda, "NCCL unavailable (libnccl.so.2): " + why);
  return api;
}

#define D2FT_NCCL(call)                                                                              \
  do {                                                                                               \
    ncclResult_t r__ = (call);                                                                       \
    if (r__ != ncclSuccess) throw Fail{kCuda, std::string(#call) + ": " + nccl().error_string(r__)}; \
  } while (0)

struct NcclExchange final : Exchange {
  ncclComm_t comm = nullptr;
  ~NcclExchange() override {
    if (comm) nccl().comm_destroy(comm);
  }
  void allreduce_sum(float* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    D2FT_NCCL(nccl().all_reduce(buf, buf, n, ncclFloat32, ncclSum, comm, st));
    ++calls;
    bytes += n * sizeof(float);
  }
  bool capturable() const override { return true; }
};
}  // namespace

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  D2FT_NCCL(nccl().get_unique_id(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
}

std::unique_ptr<Exchange> make_nccl_exchange(int rank, int world, const uint8_t id[128]) {
  auto x = std::make_unique<NcclExchange>();
  x->rank = rank;
  x->world = world;
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  D2FT_NCCL(nccl().comm_init_rank(&x->comm, world, uid, rank));
  return x;
}

// ------------------------------------------------------------------ in-process group
namespace {
constexpr int kMaxLocal = 8;
struct Ptrs {
  const float* p[kMaxLocal];
};
__global__ void sum_ranks_kernel(Ptrs in, int world, size_t n, float* out) {
  D2FT_PDL_ENTRY();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float acc = in.p[0][i];
    for (int r = 1; r < world; ++r) acc += in.p[r][i];  // fixed rank order on every rank
    out[i] = acc;
  }
}
}  // namespace

struct LocalGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned gen = 0;
  bool aborted = false;  // a rank failed outside the exchange: the others must not wait for it
  std::vector<float*> bufs;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    D2FT_REQUIRE(!aborted, kState, "local group: aborted by a failing rank");
    const unsigned g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      D2FT_REQUIRE(gen != g, kState, "local group: aborted by a failing rank");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

LocalGroup* local_group_create(int world) {
  D2FT_REQUIRE(world >= 1 && world <= kMaxLocal, kConfig, "local group: 1..8 ranks");
  auto* g = new LocalGroup;
  g->world = world;
  g->bufs.assign(world, nullptr);
  return g;
}
void local_group_destroy(LocalGroup* g) { delete g; }
void local_group_abort(LocalGroup* g) { g->abort(); }

namespace {
struct LocalExchange final : Exchange {
  LocalGroup* g;
  float* tmp = nullptr;
  size_t cap = 0;
  ~LocalExchange() override {
    if (tmp) cudaFree(tmp);
  }
  bool capturable() const override { return false; }  // host-side barrier between the ranks
  void allreduce_sum(float* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    ++calls;
    bytes += n * sizeof(float);
    if (world == 1) return;  // the sum over one rank is the buffer itself
    if (n > cap) {
      if (tmp) D2FT_CUDA(cudaFree(tmp));
      D2FT_CUDA(cudaMalloc(&tmp, n * sizeof(float)));
      cap = n;
    }
    D2FT_CUDA(cudaStreamSynchronize(st));  // this rank's partial is complete
    g->bufs[rank] = buf;
    g->barrier();
    Ptrs p{};
    for (int r = 0; r < world; ++r) p.p[r] = g->bufs[r];
    sum_ranks_kernel<<<148 * 4, 256, 0, st>>>(p, world, n, tmp);
    count_launch();
    D2FT_CUDA(cudaGetLastError());
    D2FT_CUDA(cudaStreamSynchronize(st));
    g->barrier();  // every rank has read every partial
    D2FT_CUDA(cudaMemcpyAsync(buf, tmp, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
};

__global__ void mask_rows_kernel(uint8_t* codes, int K, int Bmax, const int* owner, int rank) {
  D2FT_PDL_ENTRY();
  const size_t n = (size_t)K * Bmax;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / Bmax);
    if (owner[k] != rank) codes[i] = 3;
  }
}
}  // namespace

std::unique_ptr<Exchange> make_local_exchange(LocalGroup* g, int rank) {
  D2FT_REQUIRE(rank >= 0 && rank < g->world, kConfig, "local group: rank out of range");
  auto x = std::make_unique<LocalExchange>();
  x->g = g;
  x->rank = rank;
  x->world = g->world;
  return x;
}

void launch_mask_rows(uint8_t* codes, int K, int Bmax, const int* owner, int rank, cudaStream_t st) {
  const size_t n = (size_t)K * Bmax;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  mask_rows_kernel<<<blocks, 256, 0, st>>>(codes, K, Bmax, owner, rank);
  count_launch();
  D2FT_CUDA(cudaGetLastError());
}

}  // namespace d2ft_b200
