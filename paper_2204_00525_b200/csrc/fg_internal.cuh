// Internal plumbing of the B200 FiGaRo library: context, stream-ordered
// device buffers, error propagation and the launch counter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
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

// Stream-ordered device buffer (cudaMallocAsync from the device pool, which
// is configured to keep memory, so steady-state calls do not hit the OS).
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
    if (n) FG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
  }
  void release() {
    if (p_) cudaFreeAsync(p_, stream_);
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
  }
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t stream_ = nullptr;
};

struct LaunchCounter {
  int64_t count = 0;
};

// Per-node device state of one pipeline run (see pipeline.cu).
struct NodeState;

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  int sm_count = 148;
  size_t smem_optin = 0;
  std::string last_error = "ok";
  int64_t launches = 0;
  DevArray<unsigned> status;  // device status word
  // Results of the last pipeline run, kept for fg_get_* inspection.
  struct Saved;
  Saved* saved = nullptr;
};

#define FG_LAUNCHED(ctx) (++(ctx).launches)
#define FG_KERNEL_CHECK() FG_CUDA(cudaPeekAtLastError())

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace fg
