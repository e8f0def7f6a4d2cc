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
// counts.hpp:47-62; sums through split low/high-word tables, add_split) and exact-division checks (exact_div, counts.hpp:64-71)
// raise bits in the device status word instead of throwing.  Integer adds
// commute, so the tables are bit-identical for any launch shape.
#include <cstdlib>
#include <string>
#include <vector>

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

// Global count tables are accumulated exactly without returning atomics:
// table[0, P) collects the low 32 bits of every addend and table[P, 2P) the
// high 32 bits (neither can wrap for < 2^31 addends), both with
// fire-and-forget reductions (RED); k_finalize / k_up_div then form
// lo + hi * 2^32 in 128-bit arithmetic and flag sums >= 2^64
// (checked_atomic_add, counts.hpp:54-62).
__device__ __forceinline__ void add_split(uint64_t* table, int64_t P, int64_t slot,
                                          uint64_t d) {
  atomicAdd(reinterpret_cast<unsigned long long*>(table + slot), d & 0xffffffffull);
  const unsigned long long h = d >> 32;
  if (h) atomicAdd(reinterpret_cast<unsigned long long*>(table + P + slot), h);
}

// lo + hi * 2^32, or ~0 with ST_OVERFLOW when it does not fit 64 bits.
__device__ __forceinline__ uint64_t combine_split(uint64_t lo, uint64_t hi, unsigned* status) {
  const uint64_t sum = lo + (hi << 32);
  if ((hi >> 32) != 0 || sum < lo) {
    atomicOr(status, ST_OVERFLOW);
    return ~0ull;
  }
  return sum;
}

// Per-block shared-memory cache in front of a split global table: slot
// claimed by atomicCAS on the table index (direct-mapped); a collision goes
// straight to the global table.  Flushed once per block (cache_flush).
constexpr int kCache = 2048;
struct SmemCache {
  int* key;
  unsigned long long* val;
  unsigned* st;
  int lg = 11;  // log2 of the slot count (kCache by default)
};
__device__ __forceinline__ void cache_add(const SmemCache& c, uint64_t* table, int64_t P,
                                          int64_t q, unsigned long long x) {
  const int slot = (int)(((unsigned)q * 2654435761u) >> (32 - c.lg));
  const int old = atomicCAS(&c.key[slot], -1, (int)q);
  if (old == -1 || old == (int)q) {
    const unsigned long long o = atomicAdd(&c.val[slot], x);
    if (o + x < o) atomicOr(c.st, ST_OVERFLOW);
  } else {
    add_split(table, P, q, x);
  }
}

// Warp-aggregated checked add: lanes whose `slot` equals the previous
// lane's form runs (a segmented shuffle scan sums them); the last lane of a
// run issues one atomic.  Segments are sorted by own key, so targets keyed by
// a prefix of it arrive in runs.  Integer sums commute: the table values do
// not depend on the aggregation.
__device__ __forceinline__ void add_runs(uint64_t* table, int64_t P, int64_t slot, uint64_t v,
                                         bool live, unsigned* status,
                                         const SmemCache* cache = nullptr) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t prev = __shfl_up_sync(full, slot, 1);
  const bool prev_live = __shfl_up_sync(full, (int)live, 1) != 0;
  int head = (lane == 0 || !prev_live || prev != slot || !live) ? 1 : 0;
  unsigned long long acc = live ? v : 0ull;
  int ovf = 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(full, acc, o);
    const int hy = __shfl_up_sync(full, head, o);
    const int oy = __shfl_up_sync(full, ovf, o);
    if (lane >= o && !head) {
      const unsigned long long s2 = acc + y;
      if (s2 < acc) ovf = 1;
      acc = s2;
      ovf |= oy;
    }
    if (lane >= o) head |= hy;
  }
  const int64_t next = __shfl_down_sync(full, slot, 1);
  const bool next_live = __shfl_down_sync(full, (int)live, 1) != 0;
  const bool tail = live && (lane == 31 || !next_live || next != slot);
  if (tail) {
    if (ovf) atomicOr(status, ST_OVERFLOW);
    if (cache) cache_add(*cache, table, P, slot, acc);
    else add_split(table, P, slot, acc);
  }
}

// Warp-aggregated checked add for unsorted targets: lanes with equal `slot`
// (__match_any_sync) are summed by a log-depth peer reduction and the lowest
// lane of each peer set issues one atomic.  Zipf-distributed child keys make
// many lanes of a warp hit the same hot entry.
__device__ __forceinline__ void add_peers(uint64_t* table, int64_t P, int slot, uint64_t v,
                                          bool live, unsigned* status, bool shared_table = false) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned peers0 = __match_any_sync(full, live ? slot : -1);
  unsigned long long x = live ? v : 0ull;
  int ovf = 0;
  int rel = __popc(peers0 & ((1u << lane) - 1u));  // peers below this lane
  unsigned peers = peers0 & ~((2u << lane) - 1u);  // peers above this lane
  if (lane == 31) peers = 0;
  while (__any_sync(full, peers != 0)) {
    const int next = __ffs(peers);
    const unsigned long long t = __shfl_sync(full, x, next ? next - 1 : lane);
    const int to = __shfl_sync(full, ovf, next ? next - 1 : lane);
    if ((rel & 1) == 0 && next) {
      const unsigned long long s2 = x + t;
      if (s2 < x) ovf = 1;
      x = s2;
      ovf |= to;
    }
    const unsigned done = __ballot_sync(full, rel & 1);
    peers &= ~done;
    rel >>= 1;
  }
  if (live && lane == __ffs(peers0) - 1) {
    if (ovf) atomicOr(status, ST_OVERFLOW);
    if (shared_table) {
      const unsigned long long old =
          atomicAdd(reinterpret_cast<unsigned long long*>(table + slot), x);
      if (old + x < old) atomicOr(status, ST_OVERFLOW);
    } else {
      add_split(table, P, slot, x);
    }
  }
}

__global__ void k_theta(const uint64_t* __restrict__ sizes, int64_t G,
                        ChildLinks ch, const int* __restrict__ pidx,
                        uint64_t* phi_down, int64_t P, uint64_t* __restrict__ theta,
                        unsigned* status) {
  // Run sums of phi_down go through a per-block cache: a long parent-key
  // run (C3's most frequent k1 covers 5M F segments) costs one global add
  // per block instead of one per warp.
  __shared__ int ckey[kCache];
  __shared__ unsigned long long cval[kCache];
  __shared__ unsigned sst;
  const SmemCache cache{ckey, cval, &sst};
  if (pidx) {
    for (int i = threadIdx.x; i < kCache; i += blockDim.x) {
      ckey[i] = -1;
      cval[i] = 0ull;
    }
    if (threadIdx.x == 0) sst = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t Gw = (G + 31) & ~int64_t(31);  // warp-uniform trip count
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < Gw; k += stride) {
    const bool live = k < G;
    uint64_t t = 0;
    if (live) {
      t = sizes[k];
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
    }
    if (pidx) add_runs(phi_down, P, live ? pidx[k] : -1, t, live, status, &cache);
  }
  if (pidx) {
    __syncthreads();
    if (threadIdx.x == 0 && sst) atomicOr(status, sst);
    for (int i = threadIdx.x; i < kCache; i += blockDim.x)
      if (ckey[i] >= 0 && cval[i]) add_split(phi_down, P, ckey[i], cval[i]);
  }
}

__global__ void k_fjs(const uint64_t* __restrict__ sizes,
                      const uint64_t* __restrict__ theta, int64_t G,
                      const int* __restrict__ pidx,
                      const uint64_t* __restrict__ phi_up, ChildLinks ch,
                      uint64_t* __restrict__ fjs, uint64_t* __restrict__ circ,
                      unsigned* status) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t Gw = (G + 31) & ~int64_t(31);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < Gw; k += stride) {
    const bool live = k < G;
    uint64_t f = 0;
    if (live) {
      const uint64_t up = pidx ? phi_up[pidx[k]] : 1ull;
      f = mul_chk(theta[k], up, status);
      fjs[k] = f;
      const uint64_t m = sizes[k];
      // exact_div (counts.hpp:64-71): 32-bit hardware path when both fit.
      uint64_t q, r;
      if (((f | m) >> 32) == 0) {
        const unsigned q32 = (unsigned)f / (unsigned)m;
        q = q32;
        r = (unsigned)f - q32 * (unsigned)m;
      } else {
        q = m ? f / m : 0;
        r = m ? f - q * m : 1;
      }
      if (m == 0 || r != 0) {
        atomicOr(status, ST_CIRC_INEXACT);
        circ[k] = 0;
      } else {
        circ[k] = q;
      }
    }
    for (int c = 0; c < ch.n; ++c) {
      const int q = live ? ch.lidx[c][k] : -1;
      add_peers(ch.phi_up[c], ch.P[c], q, f, live && q >= 0, status);
    }
  }
}

// Scatter-add of fjs into ONE small child table (P <= kPrivMax) through a
// per-block shared-memory copy: contention stays on-chip (C3's D3 has 1,000
// keys for 54M F segments).
constexpr int kPrivMax = 4096;  // 32 KB of static shared memory
// Scatter-add of fjs into a child table through shared memory.  PRIV: the
// whole table (P <= kPrivMax) is privatised per block; otherwise a
// direct-mapped cache of kCache slots claimed by atomicCAS, collisions going
// to the split global table.  PEERS: warp-aggregate equal targets first
// (__match_any_sync + log-depth peer sums); without it every element is one
// shared-memory atomic (hardware-serialised on equal addresses) -- cheaper
// when a warp's targets repeat only a few times.  Four elements per thread
// are loaded before the atomics.
template <bool PRIV, bool PEERS>
__global__ void __launch_bounds__(256) k_scatter_smem(const uint64_t* __restrict__ fjs, int64_t G,
                                                      const int* __restrict__ lidx,
                                                      uint64_t* table, int64_t P,
                                                      unsigned* status, int lg_slots) {
  // Dynamic shared memory: slot values, then (cache form) the slot keys.
  extern __shared__ __align__(16) unsigned char scatter_smem[];
  const int kSlots = PRIV ? kPrivMax : (1 << lg_slots);
  unsigned long long* cval = reinterpret_cast<unsigned long long*>(scatter_smem);
  int* ckey = reinterpret_cast<int*>(cval + kSlots);
  __shared__ unsigned sst;
  const SmemCache cache{ckey, cval, &sst, lg_slots};
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) {
    if (!PRIV) ckey[i] = -1;
    cval[i] = 0ull;
  }
  if (threadIdx.x == 0) sst = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t Gw = (G + 31) & ~int64_t(31);  // warp-uniform trip count
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k0 < Gw; k0 += 4 * stride) {
    int q[4];
    uint64_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u * stride;
      q[u] = k < G ? lidx[k] : -1;
      v[u] = q[u] >= 0 ? fjs[k] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (PEERS) {
        if (k0 + u * stride >= Gw) continue;  // warp-uniform
        if (PRIV) add_peers(reinterpret_cast<uint64_t*>(cval), 0, q[u], v[u], q[u] >= 0, &sst, true);
        else {
          const unsigned full = 0xffffffffu;
          const int lane = threadIdx.x & 31;
          const unsigned peers0 = __match_any_sync(full, q[u]);
          unsigned long long x = v[u];
          int ovf = 0;
          int rel = __popc(peers0 & ((1u << lane) - 1u));
          unsigned peers = lane == 31 ? 0u : peers0 & ~((2u << lane) - 1u);
          while (__any_sync(full, peers != 0)) {
            const int nx = __ffs(peers);
            const unsigned long long t = __shfl_sync(full, x, nx ? nx - 1 : lane);
            const int to = __shfl_sync(full, ovf, nx ? nx - 1 : lane);
            if ((rel & 1) == 0 && nx) {
              const unsigned long long s2 = x + t;
              if (s2 < x) ovf = 1;
              x = s2;
              ovf |= to;
            }
            peers &= ~__ballot_sync(full, rel & 1);
            rel >>= 1;
          }
          if (q[u] >= 0 && lane == __ffs(peers0) - 1) {
            if (ovf) atomicOr(&sst, ST_OVERFLOW);
            cache_add(cache, table, P, q[u], x);
          }
        }
      } else if (q[u] >= 0) {
        if (PRIV) {
          const unsigned long long o = atomicAdd(&cval[q[u]], v[u]);
          if (o + v[u] < o) atomicOr(&sst, ST_OVERFLOW);
        } else {
          cache_add(cache, table, P, q[u], v[u]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && sst) atomicOr(status, sst);
  for (int i = threadIdx.x; i < (PRIV ? (int)P : kSlots); i += blockDim.x) {
    if (PRIV) {
      if (cval[i]) add_split(table, P, i, cval[i]);
    } else if (ckey[i] >= 0 && cval[i]) {
      add_split(table, P, ckey[i], cval[i]);
    }
  }
}

__global__ void k_up_div(uint64_t* __restrict__ phi_up,
                         const uint64_t* __restrict__ phi_down, int64_t P,
                         unsigned* status) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = combine_split(phi_up[q], phi_up[P + q], status);
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

// Final values of a split table (see add_split).
__global__ void k_finalize(uint64_t* __restrict__ table, int64_t P, unsigned* status) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P;
       q += (int64_t)gridDim.x * blockDim.x)
    table[q] = combine_split(table[q], table[P + q], status);
}

inline int grid_for(const Context& ctx, int64_t n) {
  int64_t g = ceil_div(n, kThreads);
  const int64_t cap = static_cast<int64_t>(ctx.sm_count) * 8;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void launch_theta(Context& ctx, const uint64_t* sizes, int64_t G,
                  const ChildLinks& ch, const int* pidx, uint64_t* phi_down, int64_t P,
                  uint64_t* theta, unsigned* status) {
  if (G == 0) return;
  k_theta<<<grid_for(ctx, G), kThreads, 0, ctx.stream>>>(sizes, G, ch, pidx,
                                                         phi_down, P, theta, status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  if (pidx && P > 0) {
    k_finalize<<<grid_for(ctx, P), kThreads, 0, ctx.stream>>>(phi_down, P, status);
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
  }
}

void launch_fjs(Context& ctx, const uint64_t* sizes, const uint64_t* theta,
                int64_t G, const int* pidx, const uint64_t* phi_up,
                const ChildLinks& ch, const int64_t* child_P, uint64_t* fjs,
                uint64_t* circ, unsigned* status) {
  if (G == 0) return;
  // Children whose table fits shared memory: full privatisation; children
  // with many more segments than keys: the shared-memory cache; others
  // (few segments per key, little contention): warp-aggregated atomics
  // inside k_fjs.
  ChildLinks big{};
  std::vector<int> small, cached;
  for (int c = 0; c < ch.n; ++c) {
    if (child_P[c] <= kPrivMax && G > 4 * child_P[c]) {
      small.push_back(c);
    } else if (G > 16 * child_P[c] && getenv("FG_NO_COUNT_CACHE") == nullptr) {
      cached.push_back(c);
    } else {
      big.lidx[big.n] = ch.lidx[c];
      big.phi_down[big.n] = ch.phi_down[c];
      big.phi_up[big.n] = ch.phi_up[c];
      big.P[big.n] = ch.P[c];
      ++big.n;
    }
  }
  k_fjs<<<grid_for(ctx, G), kThreads, 0, ctx.stream>>>(sizes, theta, G, pidx,
                                                       phi_up, big, fjs, circ,
                                                       status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  // Measured on C3 (54M F segments): the privatised D3 table (1k keys) is
  // fastest with plain shared-memory atomics (0.56 vs 0.88 ms), the cached
  // D2 table (100k Zipf keys) needs the warp aggregation (1.9 vs 6.7 ms).
  // FG_COUNT_SCATTER=peers|direct forces one form for both.
  static const int mode = [] {
    const char* e = getenv("FG_COUNT_SCATTER");
    if (!e) return 0;
    return std::string(e) == "peers" ? 1 : 2;
  }();
  auto launch = [&](auto kern, int c, bool priv) {
    static const int per_sm = [] {
      const char* e = getenv("FG_SCATTER_GRID");
      return e ? std::max(1, atoi(e)) : 4;
    }();
    // Cache slots (log2): FG_SCATTER_SLOTS, default 2^13 (96 KB, two blocks per
    // SM; measured on C3: counts 3.53 ms with 2^11, 3.33 with 2^12, 3.02 with 2^13).
    static const int lg = [] {
      const char* e = getenv("FG_SCATTER_SLOTS");
      return e ? std::min(13, std::max(8, atoi(e))) : 13;
    }();
    const size_t smem = priv ? (size_t)kPrivMax * 8 : ((size_t)12 << lg);
    FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<int64_t>((int64_t)ctx.sm_count * per_sm, ceil_div(G, kThreads));
    kern<<<std::max(grid, 1), kThreads, smem, ctx.stream>>>(fjs, G, ch.lidx[c], ch.phi_up[c],
                                                             child_P[c], status, lg);
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
  };
  for (int c : cached)
    mode != 2 ? launch(k_scatter_smem<false, true>, c, false)
              : launch(k_scatter_smem<false, false>, c, false);
  for (int c : small)
    mode == 1 ? launch(k_scatter_smem<true, true>, c, true)
              : launch(k_scatter_smem<true, false>, c, true);
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
