// K1: key packing, stable radix grouping and key projections.
//
// Replaces the reference's canonicalize sort (relation.hpp:127-167), the
// contiguous key groups (relation.hpp:56-66, counts.hpp:80-88) and the
// per-call KeyTuple projections (join_tree.hpp:57-70) with:
//   * an order-preserving packing of each int64 key tuple into one u64
//     (per-attribute offset encoding, fields in declaration order, most
//     significant first) -- lexicographic tuple order == integer order;
//   * a stable LSD radix sort over only the significant bits carrying the
//     row permutation, and segment-offset extraction (radix.cu);
//   * field re-packing for projections onto parent-shared attributes, and
//     binary search of projected keys in the child's sorted key table.
#include "launchers.cuh"

namespace fg {

namespace {

constexpr int kThreads = 256;

inline int grid_for(const Context& ctx, int64_t n, int per_sm = 8) {
  int64_t g = ceil_div(n, kThreads);
  int64_t cap = static_cast<int64_t>(ctx.sm_count) * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// Min/max of every key column in one pass over the row-major key tuples
// (grid-stride over rows, NK columns known at compile time for the common
// widths, four rows in flight per thread; per-column warp reduction, then
// atomics).  NK = 0: any width up to kMaxKeyCols, one row at a time.
template <int NK>
__global__ void k_key_minmax(const int64_t* __restrict__ keys, int64_t rows,
                             int n_key, const int* __restrict__ attr_of_col,
                             long long* mins, long long* maxs) {
  constexpr int C = NK ? NK : kMaxKeyCols;
  constexpr int U = NK ? 4 : 1;
  long long lo[C], hi[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    lo[c] = LLONG_MAX;
    hi[c] = LLONG_MIN;
  }
  const int nk = NK ? NK : n_key;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < rows; i0 += U * stride) {
    long long v[U][C];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        v[u][c] = 0;
        if (c < nk && i < rows) v[u][c] = keys[i * nk + c];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * stride >= rows) continue;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (c >= nk) continue;
        lo[c] = v[u][c] < lo[c] ? v[u][c] : lo[c];
        hi[c] = v[u][c] > hi[c] ? v[u][c] : hi[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (c >= nk) break;
    long long a = lo[c], b = hi[c];
    for (int o = 16; o; o >>= 1) {
      const long long x = __shfl_xor_sync(0xffffffffu, a, o);
      const long long y = __shfl_xor_sync(0xffffffffu, b, o);
      a = x < a ? x : a;
      b = y > b ? y : b;
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&mins[attr_of_col[c]], a);
      atomicMax(&maxs[attr_of_col[c]], b);
    }
  }
}

template <class KeyT>
__global__ void k_pack_keys(const int64_t* __restrict__ keys, int64_t rows,
                            int n_key, PackSpec spec, KeyT* __restrict__ out,
                            int* __restrict__ iota) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = 0;
#pragma unroll 4
    for (int f = 0; f < spec.n; ++f) {
      const long long v = keys[i * n_key + spec.col[f]];
      const uint64_t enc = (uint64_t)v - (uint64_t)spec.min[f];
      if (spec.bits[f]) k |= enc << spec.shift[f];
    }
    out[i] = static_cast<KeyT>(k);
    if (iota) iota[i] = static_cast<int>(i);
  }
}

__device__ __forceinline__ uint64_t project_one(uint64_t k,
                                                const PackSpec& s) {
  // s.col[f] holds the source shift of field f; s.shift[f] the target one.
  uint64_t o = 0;
  for (int f = 0; f < s.n; ++f) {
    const int b = s.bits[f];
    if (!b) continue;
    const uint64_t mask = b == 64 ? ~0ull : ((1ull << b) - 1);
    o |= ((k >> s.col[f]) & mask) << s.shift[f];
  }
  return o;
}

__global__ void k_project(const uint64_t* __restrict__ in, int64_t n,
                          PackSpec s, uint64_t* __restrict__ out,
                          const int64_t* __restrict__ n_dev) {
  if (n_dev) n = *n_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = project_one(in[i], s);
}

__global__ void k_lookup(const uint64_t* __restrict__ own, int64_t n,
                         PackSpec s, const uint64_t* __restrict__ table,
                         int64_t m, int* __restrict__ out, unsigned* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = project_one(own[i], s);
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (table[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo < m && table[lo] == key) {
      out[i] = static_cast<int>(lo);
    } else {
      out[i] = -1;
      atomicOr(status, ST_MISSING_CHILD);
    }
  }
}

// Dense variant for narrow keys: table index by direct addressing.
__global__ void k_dense_fill(const uint64_t* __restrict__ table, int64_t m,
                             int* __restrict__ dense) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x)
    dense[table[j]] = static_cast<int>(j);
}

__global__ void k_lookup_dense(const uint64_t* __restrict__ own, int64_t n, PackSpec s,
                               const int* __restrict__ dense, int* __restrict__ out,
                               unsigned* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = dense[project_one(own[i], s)];
    out[i] = j;
    if (j < 0) atomicOr(status, ST_MISSING_CHILD);
  }
}

__global__ void k_unpack(const uint64_t* __restrict__ in, int64_t n,
                         PackSpec s, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = in[i];
    for (int f = 0; f < s.n; ++f) {
      const int b = s.bits[f];
      const uint64_t mask = b == 64 ? ~0ull : ((1ull << b) - 1);
      const uint64_t enc = b ? (k >> s.shift[f]) & mask : 0;
      out[i * s.n + f] = (int64_t)(enc + (uint64_t)s.min[f]);
    }
  }
}

__global__ void k_narrow(const uint64_t* __restrict__ in, int64_t n,
                         uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<uint32_t>(in[i]);
}

__global__ void k_iota(int* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<int>(i);
}

__global__ void k_seg_sizes(const int* __restrict__ begins, int64_t G,
                            uint64_t* __restrict__ sizes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G;
       i += (int64_t)gridDim.x * blockDim.x)
    sizes[i] = (uint64_t)(begins[i + 1] - begins[i]);
}

}  // namespace

void launch_key_minmax(Context& ctx, const int64_t* keys, int64_t rows,
                       int n_key, const int* attr_of_col_dev, long long* mins,
                       long long* maxs) {
  if (rows == 0 || n_key == 0) return;
  if (n_key > kMaxKeyCols) fail(FG_E_UNSUPPORTED, "more than 16 key columns");
  const int grid = grid_for(ctx, rows, 8);
  auto kern = n_key == 1 ? k_key_minmax<1>
            : n_key == 2 ? k_key_minmax<2>
            : n_key == 3 ? k_key_minmax<3>
            : n_key == 4 ? k_key_minmax<4> : k_key_minmax<0>;
  kern<<<grid, kThreads, 0, ctx.stream>>>(keys, rows, n_key, attr_of_col_dev, mins, maxs);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

template <class KeyT>
void launch_pack_keys(Context& ctx, const int64_t* keys, int64_t rows,
                      int n_key, const PackSpec& spec, KeyT* out, int* iota) {
  if (rows == 0) return;
  k_pack_keys<KeyT><<<grid_for(ctx, rows), kThreads, 0, ctx.stream>>>(
      keys, rows, n_key, spec, out, iota);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_project(Context& ctx, const uint64_t* in, int64_t n,
                    const PackSpec& s, uint64_t* out, const int64_t* n_dev) {
  if (n == 0) return;
  k_project<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(in, n, s, out, n_dev);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_lookup(Context& ctx, const uint64_t* own_keys, int64_t n,
                   const PackSpec& proj, const uint64_t* table, int64_t m,
                   int* out, unsigned* status) {
  if (n == 0) return;
  k_lookup<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(own_keys, n, proj,
                                                          table, m, out, status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_lookup_bits(Context& ctx, const uint64_t* own_keys, int64_t n,
                        const PackSpec& proj, const uint64_t* table, int64_t m,
                        int bits, int* out, unsigned* status) {
  if (n == 0) return;
  if (bits > 24 || m == 0) {
    launch_lookup(ctx, own_keys, n, proj, table, m, out, status);
    return;
  }
  DevArray<int> dense(size_t(1) << bits, ctx.stream);
  FG_CUDA(cudaMemsetAsync(dense.get(), 0xff, dense.bytes(), ctx.stream));  // -1
  k_dense_fill<<<grid_for(ctx, m), kThreads, 0, ctx.stream>>>(table, m, dense.get());
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  k_lookup_dense<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(own_keys, n, proj,
                                                                dense.get(), out, status);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_unpack(Context& ctx, const uint64_t* in, int64_t n,
                   const PackSpec& spec, int64_t* out) {
  if (n == 0 || spec.n == 0) return;
  k_unpack<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(in, n, spec, out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_narrow(Context& ctx, const uint64_t* in, int64_t n, uint32_t* out) {
  if (n == 0) return;
  k_narrow<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(in, n, out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_iota(Context& ctx, int* out, int64_t n) {
  if (n == 0) return;
  k_iota<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(out, n);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_seg_sizes(Context& ctx, const int* begins, int64_t G,
                      uint64_t* sizes) {
  if (G == 0) return;
  k_seg_sizes<<<grid_for(ctx, G), kThreads, 0, ctx.stream>>>(begins, G, sizes);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void exclusive_sum_int(Context& ctx, const int* in, int* out, int64_t n) {
  scan_int(ctx, in, out, n, false);
}

void inclusive_sum_int(Context& ctx, const int* in, int* out, int64_t n) {
  scan_int(ctx, in, out, n, true);
}

// Grouping is split so several relations can be sorted before one host
// synchronisation reads all the group counts: begin = radix sort (radix.cu)
// + segment extraction into upper-bound (n-row) buffers; finish = adopt them
// once G is known.
template <class KeyT>
void group_begin_t(Context& ctx, const KeyT* keys, int64_t n, int bits,
                   const int* perm_in, GroupOut& out, GroupPending& pend,
                   const uint32_t* hist, int* pidx) {
  cudaStream_t st = ctx.stream;
  out.perm.alloc(n, st);
  pend.n = n;
  pend.begins.alloc(n + 1, st);
  pend.uniq.alloc(n, st);
  pend.nr.alloc(1, st);
  DevArray<KeyT> sorted(n, st);
  radix_sort_pairs<KeyT>(ctx, keys, sorted.get(), perm_in, out.perm.get(), n, bits, hist);
  launch_segments<KeyT>(ctx, sorted.get(), n, pend.begins.get(), pend.uniq.get(),
                        pend.nr.get(), out.perm.get(), pidx);
}

void group_finish(Context& ctx, int64_t G, GroupOut& out, GroupPending& pend) {
  (void)ctx;
  out.G = G;
  out.begins = std::move(pend.begins);
  out.uniq = std::move(pend.uniq);
  pend = GroupPending();
}

void group_begin(Context& ctx, const uint64_t* keys, int64_t n, int bits,
                 const int* perm_in, GroupOut& out, GroupPending& pend,
                 const uint32_t* hist, int* pidx) {
  group_begin_t<uint64_t>(ctx, keys, n, bits, perm_in, out, pend, hist, pidx);
}
void group_begin32(Context& ctx, const uint32_t* keys, int64_t n, int bits,
                   const int* perm_in, GroupOut& out, GroupPending& pend,
                   const uint32_t* hist, int* pidx) {
  group_begin_t<uint32_t>(ctx, keys, n, bits, perm_in, out, pend, hist, pidx);
}

void group_begin_presorted(Context& ctx, const uint64_t* keys, int64_t n,
                           const int* perm_in, GroupOut& out, GroupPending& pend,
                           int* pidx, const int64_t* n_dev, bool want_perm) {
  cudaStream_t st = ctx.stream;
  if (want_perm) out.perm.alloc(n, st);
  pend.n = n;
  pend.begins.alloc(n + 1, st);
  pend.uniq.alloc(n, st);
  pend.nr.alloc(1, st);
  if (n && want_perm) {
    if (perm_in)
      FG_CUDA(cudaMemcpyAsync(out.perm.get(), perm_in, n * sizeof(int),
                              cudaMemcpyDeviceToDevice, st));
    else
      launch_iota(ctx, out.perm.get(), n);
  }
  launch_segments<uint64_t>(ctx, keys, n, pend.begins.get(), pend.uniq.get(), pend.nr.get(),
                            perm_in, pidx, n_dev);
}

template <class KeyT>
void group_sorted_t(Context& ctx, const KeyT* keys, int64_t n, int bits,
                    const int* perm_in, GroupOut& out) {
  GroupPending pend;
  group_begin_t<KeyT>(ctx, keys, n, bits, perm_in, out, pend, nullptr, nullptr);
  int64_t G = 0;
  FG_CUDA(cudaMemcpyAsync(&G, pend.nr.get(), sizeof G, cudaMemcpyDeviceToHost,
                          ctx.stream));
  sync_stream(ctx);
  group_finish(ctx, G, out, pend);
}

void group_sorted(Context& ctx, const uint64_t* keys, int64_t n, int bits,
                  const int* perm_in, GroupOut& out) {
  group_sorted_t<uint64_t>(ctx, keys, n, bits, perm_in, out);
}

void group_sorted32(Context& ctx, const uint32_t* keys, int64_t n, int bits,
                    const int* perm_in, GroupOut& out) {
  group_sorted_t<uint32_t>(ctx, keys, n, bits, perm_in, out);
}

template void launch_pack_keys<uint64_t>(Context&, const int64_t*, int64_t, int,
                                         const PackSpec&, uint64_t*, int*);
template void launch_pack_keys<uint32_t>(Context&, const int64_t*, int64_t, int,
                                         const PackSpec&, uint32_t*, int*);

}  // namespace fg
