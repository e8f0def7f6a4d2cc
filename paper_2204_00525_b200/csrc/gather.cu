// Multi-GPU R gather over NCCL: every rank's n x n factor is
// all-gathered over NVLink and merged into the global R by one more device
// TSQR.  The reference is single-process; this is the collective a C++
// host uses after fg_run_pipeline on its shard (fg_ctx_set_nccl, fg_gather_r
// in include/figaro_cuda.h).
//
// NCCL is resolved at run time from the process that created the
// communicator (dlsym on the already-loaded libnccl, else dlopen
// libnccl.so.2), so the library has no link-time NCCL dependency and uses the
// caller's NCCL build (e.g. the one torch.distributed loaded).
#include <dlfcn.h>
#include <nccl.h>

#include <vector>

#include "launchers.cuh"

namespace fg {
namespace {

struct NcclApi {
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*count)(const ncclComm_t, int*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = RTLD_DEFAULT;
    if (!dlsym(h, "ncclAllGather")) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
      a.count = reinterpret_cast<decltype(a.count)>(dlsym(h, "ncclCommCount"));
      a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    }
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const auto& api = nccl_api();
    fail(FG_E_NCCL, std::string(what) + ": " +
                        (api.error_string ? api.error_string(r) : "NCCL error"));
  }
}

}  // namespace

void set_nccl(Context& ctx, void* comm) {
  if (comm && !nccl_api().all_gather)
    fail(FG_E_NCCL, "NCCL is not loaded in this process (libnccl.so.2 not found)");
  ctx.nccl = comm;
}

void gather_r(Context& ctx, const double* R_local, int n, int memory, double* R_out) {
  if (!ctx.nccl) fail(FG_E_ARG, "fg_gather_r: no NCCL communicator (fg_ctx_set_nccl)");
  if (n < 0) fail(FG_E_ARG, "fg_gather_r: negative size");
  const auto& api = nccl_api();
  auto comm = static_cast<ncclComm_t>(ctx.nccl);
  int P = 0;
  nccl_check(api.count(comm, &P), "ncclCommCount");
  const size_t nn = (size_t)n * n;
  cudaStream_t st = ctx.stream;
  DevArray<double> local, all((size_t)P * nn, st), R;
  const double* src = R_local;
  if (memory == FG_MEM_HOST) {
    local.alloc(nn, st);
    if (nn) FG_CUDA(cudaMemcpyAsync(local.get(), R_local, nn * sizeof(double),
                                    cudaMemcpyHostToDevice, st));
    src = local.get();
  }
  if (nn) nccl_check(api.all_gather(src, all.get(), nn, ncclDouble, comm, st), "ncclAllGather");
  std::vector<Span> parts;
  for (int p = 0; p < P; ++p) parts.push_back({all.get() + (size_t)p * nn, n, n, n, 0});
  double* dst = R_out;
  if (memory == FG_MEM_HOST) {
    R.alloc(nn, st);
    dst = R.get();
  }
  tsqr(ctx, parts, n, dst);
  if (memory == FG_MEM_HOST && nn)
    FG_CUDA(cudaMemcpyAsync(R_out, dst, nn * sizeof(double), cudaMemcpyDeviceToHost, st));
  sync_stream(ctx);
}

}  // namespace fg
