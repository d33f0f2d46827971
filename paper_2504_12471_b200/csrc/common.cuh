// Shared helpers for the d2ft B200 library (sm_100a only).
#pragma once
#include <mutex>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

namespace d2ft_b200 {

// Status codes of the C-ABI (include/d2ft_b200.h).  1..6 mirror the
// reference's errc categories in declaration order (error.hpp:12-19).
enum Status : int {
  kOk = 0,
  kConfig = 1,
  kInput = 2,
  kDimension = 3,
  kState = 4,
  kNumeric = 5,
  kSize = 6,
  kCuda = 7,
};

void set_error(const std::string& msg);

// Count of kernels this library launched (bench.py's gpu_launches).
// (atomic: engines of an in-process partition group step on separate threads)
extern std::atomic<unsigned long long> g_launches;
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
inline unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
// a CUDA graph replay launches the kernels it captured
inline void add_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Programmatic dependent launch (the step's CUDA graph links consecutive
// kernels with programmatic edges, Engine::compute_step): every kernel lets
// its successor launch right away (pdl_trigger) and waits for its
// predecessor's completion and memory (pdl_wait) before touching data the
// predecessor may write.  Both are no-ops for an ordinary launch.
#ifndef D2FT_NO_PDL_TRIGGER
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_trigger() {}
#endif
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define D2FT_PDL_ENTRY() \
  do {                   \
    ::d2ft_b200::pdl_trigger(); \
    ::d2ft_b200::pdl_wait();    \
  } while (0)

struct Fail {
  int code;
  std::string msg;
};

#define D2FT_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e__ = (call);                                                            \
    if (e__ != cudaSuccess)                                                              \
      throw ::d2ft_b200::Fail{::d2ft_b200::kCuda,                                        \
                              std::string(#call) + ": " + cudaGetErrorString(e__)};      \
  } while (0)

#define D2FT_REQUIRE(cond, code, msg)                     \
  do {                                                    \
    if (!(cond)) throw ::d2ft_b200::Fail{(code), (msg)}; \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Fail& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return kInput;
  }
}

// cudaFuncSetAttribute is per device: a call site keeps one bit per device
// it has configured (`static unsigned long long mask; once_per_device(mask,
// [&] { cudaFuncSetAttribute(...); })`).  Thread-safe: the bit is published
// only after `set` ran, under one process-wide mutex, so a second host thread
// (the engines of an in-process partition, or two engines stepped
// concurrently) never launches a kernel before its shared-memory limit took
// effect (it used to see the bit first and fail the launch).
inline std::mutex& func_attr_mutex() {
  static std::mutex m;
  return m;
}
template <class F>
inline void once_per_device(unsigned long long& mask, F&& set) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit) return;
  std::lock_guard<std::mutex> lk(func_attr_mutex());
  if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit) return;
  set();
  __atomic_fetch_or(&mask, bit, __ATOMIC_RELEASE);
}

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace d2ft_b200
