// K2: count aggregates along the join tree as integer segmented reductions.
//
// Restates compute_counts (counts.hpp:92-224) over dense arrays aligned with
// the sorted key segments instead of std::map<KeyTuple,u64>:
//   bottom-up  theta[k] = rows[k] * prod_c phi_down_c[lidx_c[k]]
//              phi_down[pidx[k]] += theta[k]                (counts.hpp:137-155)
//   top-down   fjs[k] = theta[k] * phi_up[pidx[k]]  (1 at the root)
//              phi_up_c[lidx_c[k]] += fjs[k]; circ[k] = fjs[k] / rows[k]
//              phi_up_c[q] /= phi_down_c[q]                 (counts.hpp:190-219)
// u64 arithmetic with overflow detection (checked_mul / checked_atomic_add,
// counts.hpp:47-62) and exact-division checks (exact_div, counts.hpp:64-71)
// raise bits in the device status word instead of throwing.  Integer adds
// commute, so the tables are bit-identical for any launch shape.
#include "launchers.cuh"

namespace fg {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint64_t mul_chk(uint64_t a, uint64_t b,
                                            unsigned* status) {
  if (__umul64hi(a, b) != 0) {
    atomicOr(status, ST_OVERFLOW);
    return ~0ull;
  }
  return a * b;
}

__device__ __forceinline__ void add_chk(uint64_t* slot, uint64_t d,
                                        unsigned* status) {
  const unsigned long long old =
      atomicAdd(reinterpret_cast<unsigned long long*>(slot),
                static_cast<unsigned long long>(d));
  if (old + d < old) atomicOr(status, ST_OVERFLOW);
}

__global__ void k_theta(const uint64_t* __restrict__ sizes, int64_t G,
                        ChildLinks ch, const int* __restrict__ pidx,
                        uint64_t* phi_down, uint64_t* __restrict__ theta,
                        unsigned* status) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < G;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t t = sizes[k];
    for (int c = 0; c < ch.n; ++c) {
      const int q = ch.lidx[c][k];
      if (q < 0) {
        atomicOr(status, ST_MISSING_CHILD);
        t = 0;
        continue;
      }
      t = mul_chk(t, ch.phi_down[c][q], status);
    }
    theta[k] = t;
    if (pidx) add_chk(&phi_down[pidx[k]], t, status);
  }
}

__global__ void k_fjs(const uint64_t* __restrict__ sizes,
                      const uint64_t* __restrict__ theta, int64_t G,
                      const int* __restrict__ pidx,
                      const uint64_t* __restrict__ phi_up, ChildLinks ch,
                      uint64_t* __restrict__ fjs, uint64_t* __restrict__ circ,
                      unsigned* status) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < G;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t up = pidx ? phi_up[pidx[k]] : 1ull;
    const uint64_t f = mul_chk(theta[k], up, status);
    fjs[k] = f;
    for (int c = 0; c < ch.n; ++c) {
      const int q = ch.lidx[c][k];
      if (q >= 0) add_chk(&ch.phi_up[c][q], f, status);
    }
    const uint64_t m = sizes[k];
    if (m == 0 || f % m != 0) {
      atomicOr(status, ST_CIRC_INEXACT);
      circ[k] = 0;
    } else {
      circ[k] = f / m;
    }
  }
}

__global__ void k_up_div(uint64_t* __restrict__ phi_up,
                         const uint64_t* __restrict__ phi_down, int64_t P,
                         unsigned* status) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = phi_up[q];
    const uint64_t d = phi_down[q];
    if (u == 0) {
      // The parent never produced this key: counts.hpp:211-214.
      atomicOr(status, ST_UP_UNMATCHED);
      continue;
    }
    if (d == 0 || u % d != 0) {
      atomicOr(status, ST_UP_INEXACT);
      phi_up[q] = 0;
      continue;
    }
    phi_up[q] = u / d;
  }
}

inline int grid_for(const Context& ctx, int64_t n) {
  int64_t g = ceil_div(n, kThreads);
  const int64_t cap = static_cast<int64_t>(ctx.sm_count) * 8;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void launch_theta(Context& ctx, const uint64_t* sizes, int64_t G,
                  const ChildLinks& ch, const int* pidx, uint64_t* phi_down,
                  uint64_t* theta, unsigned* status) {
  if (G == 0) return;
  k_theta<<<grid_for(ctx, G), kThreads, 0, ctx.stream>>>(sizes, G, ch, pidx,
                                                         phi_down, theta, status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_fjs(Context& ctx, const uint64_t* sizes, const uint64_t* theta,
                int64_t G, const int* pidx, const uint64_t* phi_up,
                const ChildLinks& ch, uint64_t* fjs, uint64_t* circ,
                unsigned* status) {
  if (G == 0) return;
  k_fjs<<<grid_for(ctx, G), kThreads, 0, ctx.stream>>>(sizes, theta, G, pidx,
                                                       phi_up, ch, fjs, circ,
                                                       status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_up_div(Context& ctx, uint64_t* phi_up, const uint64_t* phi_down,
                   int64_t P, unsigned* status) {
  if (P == 0) return;
  k_up_div<<<grid_for(ctx, P), kThreads, 0, ctx.stream>>>(phi_up, phi_down, P,
                                                          status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

}  // namespace fg
