// Internal plumbing of the B200 FiGaRo library: context, stream-ordered
// device buffers, error propagation and the launch counter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "figaro_cuda.h"

namespace fg {

// Thrown inside the library, turned into an fg_status at the C boundary.
struct Failure {
  fg_status code;
  std::string msg;
};

[[noreturn]] inline void fail(fg_status code, std::string msg) {
  throw Failure{code, std::move(msg)};
}

inline void cuda_check(cudaError_t e, const char* what, const char* file,
                       int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    fail(FG_E_CUDA, buf);
  }
}
#define FG_CUDA(x) ::fg::cuda_check((x), #x, __FILE__, __LINE__)

// Status word written by device kernels (integrity / overflow flags).
enum : unsigned {
  ST_MISSING_CHILD = 1u << 0,   // counts.hpp:143-148 / figaro.hpp:204-209
  ST_OVERFLOW = 1u << 1,        // counts.hpp:47-62
  ST_CIRC_INEXACT = 1u << 2,    // counts.hpp:203-204 (exact_div)
  ST_UP_UNMATCHED = 1u << 3,    // counts.hpp:211-214
  ST_UP_INEXACT = 1u << 4,      // counts.hpp:215-217
  ST_ZERO_COUNT = 1u << 5,      // figaro.hpp:97-104
};

struct Context;

// Caching device allocator owned by a context.  All device work of a context
// is ordered on its one stream, so a block freed by an earlier stage can be
// handed to a later stage without synchronisation.  Steady-state calls with
// the same shapes never reach cudaMalloc.
class BlockCache {
 public:
  void* get(size_t bytes) {
    if (exact()) {  // sanitizer runs: every buffer its own exact allocation
      void* p = nullptr;
      FG_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
      live_[p] = bytes;
      return p;
    }
    bytes = round(bytes);
    auto it = free_.lower_bound(bytes);
    if (it != free_.end() && it->first <= bytes + bytes / 2) {
      void* p = it->second;
      size_t b = it->first;
      free_.erase(it);
      live_[p] = b;
      return p;
    }
    void* p = nullptr;
    ++mallocs_;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      trim();
      FG_CUDA(cudaMalloc(&p, bytes));
    }
    live_[p] = bytes;
    reserved_ += bytes;
    return p;
  }
  void put(void* p) {
    auto it = live_.find(p);
    if (it == live_.end()) return;
    if (exact()) {  // cudaFree waits for the device, so in-flight users finish first
      live_.erase(it);
      cudaFree(p);
      return;
    }
    free_.emplace(it->second, p);
    live_.erase(it);
  }
  // Returns cached blocks to the driver (synchronises the device).
  void trim() {
    if (free_.empty()) return;
    cudaDeviceSynchronize();
    for (auto& kv : free_) {
      cudaFree(kv.second);
      reserved_ -= kv.first;
    }
    free_.clear();
  }
  size_t reserved() const { return reserved_; }
  int64_t mallocs() const { return mallocs_; }
  // FG_EXACT_ALLOC=1: no caching or rounding, so compute-sanitizer memcheck
  // sees every out-of-bounds access.
  static bool exact() {
    static const bool e = getenv("FG_EXACT_ALLOC") != nullptr;
    return e;
  }

 private:
  // Size classes: 512 B steps below 1 MB, then four classes per power of
  // two (x1, x1.25, x1.5, x1.75), so the same request shapes map to the same
  // classes every call and steady-state calls find their blocks again.
  static size_t round(size_t b) {
    if (b < (1 << 20)) return (b + 511) & ~size_t(511);
    size_t p = size_t(1) << 20;
    while (p * 2 <= b) p *= 2;
    const size_t q = p / 4;
    return (b + q - 1) / q * q;
  }
  std::multimap<size_t, void*> free_;
  std::map<void*, size_t> live_;
  size_t reserved_ = 0;
  int64_t mallocs_ = 0;
};

// The cache of the context currently running on this thread (set by the C
// entry points); DevArray allocates from it.
BlockCache*& current_cache();

// Device buffer drawn from the current context's BlockCache.
template <class T>
class DevArray {
 public:
  DevArray() = default;
  DevArray(size_t n, cudaStream_t s) { alloc(n, s); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept { swap(o); }
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  ~DevArray() { release(); }

  void alloc(size_t n, cudaStream_t s) {
    release();
    stream_ = s;
    n_ = n;
    if (n) {
      cache_ = current_cache();
      if (!cache_) fail(FG_E_ARG, "device allocation outside a context");
      p_ = static_cast<T*>(cache_->get(n * sizeof(T)));
    }
  }
  void release() {
    if (p_ && cache_) cache_->put(p_);
    p_ = nullptr;
    n_ = 0;
  }
  void zero() {
    if (n_) FG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), stream_));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

 private:
  void swap(DevArray& o) {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(stream_, o.stream_);
    std::swap(cache_, o.cache_);
  }
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t stream_ = nullptr;
  BlockCache* cache_ = nullptr;
};

struct LaunchCounter {
  int64_t count = 0;
};

// Per-node device state of one pipeline run (see pipeline.cu).
struct NodeState;

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;  // where all work of the context is ordered
  cudaStream_t own = nullptr;     // the context's own stream (fg_ctx_create)
  cudaStream_t copy_stream = nullptr;  // host -> device uploads (run_pipeline)
  int sm_count = 148;
  size_t smem_optin = 0;
  std::string last_error = "ok";
  int64_t launches = 0;
  int64_t syncs = 0;          // host waits on the context stream
  void* nccl = nullptr;       // ncclComm_t of this rank (fg_ctx_set_nccl)
  BlockCache cache;           // declared before every DevArray member
  DevArray<unsigned> status;  // device status word
  // Results of the last pipeline run, kept for fg_get_* inspection.
  struct Saved;
  Saved* saved = nullptr;
};

#define FG_LAUNCHED(ctx) (++(ctx).launches)

// The one way the library waits for its stream (counted in fg_result).
inline void sync_stream(Context& ctx) {
  ++ctx.syncs;
  FG_CUDA(cudaStreamSynchronize(ctx.stream));
}
#define FG_KERNEL_CHECK() FG_CUDA(cudaPeekAtLastError())

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace fg
