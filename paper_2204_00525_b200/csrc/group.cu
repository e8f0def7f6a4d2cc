// K1: key packing, stable radix grouping and key projections.
//
// Replaces the reference's canonicalize sort (relation.hpp:127-167), the
// contiguous key groups (relation.hpp:56-66, counts.hpp:80-88) and the
// per-call KeyTuple projections (join_tree.hpp:57-70) with:
//   * an order-preserving packing of each int64 key tuple into one u64
//     (per-attribute offset encoding, fields in declaration order, most
//     significant first) -- lexicographic tuple order == integer order;
//   * a stable LSD radix sort over only the significant bits (CUB onesweep
//     templates instantiated for sm_100a) carrying the row permutation;
//   * run-length extraction of the segment offsets;
//   * field re-packing for projections onto parent-shared attributes, and
//     binary search of projected keys in the child's sorted key table.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

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

__global__ void k_key_minmax(const int64_t* __restrict__ keys, int64_t rows,
                             int n_key, const int* __restrict__ attr_of_col,
                             long long* mins, long long* maxs) {
  // One column at a time through blockIdx.y; grid-stride over rows.
  const int c = blockIdx.y;
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long v = keys[i * n_key + c];
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
  }
  for (int o = 16; o; o >>= 1) {
    long long a = __shfl_xor_sync(0xffffffffu, lo, o);
    long long b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mins[attr_of_col[c]], lo);
    atomicMax(&maxs[attr_of_col[c]], hi);
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
                          PackSpec s, uint64_t* __restrict__ out) {
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

__global__ void k_iota(int* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<int>(i);
}

__global__ void k_head_flags(const uint64_t* __restrict__ sorted, int64_t n,
                             int* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || sorted[i] != sorted[i - 1]) ? 1 : 0;
}

__global__ void k_scatter_runs(const int* __restrict__ scan,
                               const int* __restrict__ perm, int64_t n,
                               int* __restrict__ pidx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pidx[perm[i]] = scan[i] - 1;
}

__global__ void k_seg_sizes(const int* __restrict__ begins, int64_t G,
                            uint64_t* __restrict__ sizes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G;
       i += (int64_t)gridDim.x * blockDim.x)
    sizes[i] = (uint64_t)(begins[i + 1] - begins[i]);
}

__global__ void k_set_last(int* begins, int64_t G, int n) { begins[G] = n; }

__global__ void k_widen(const uint32_t* __restrict__ in, int64_t n,
                        uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace

void launch_key_minmax(Context& ctx, const int64_t* keys, int64_t rows,
                       int n_key, const int* attr_of_col_dev, long long* mins,
                       long long* maxs) {
  if (rows == 0 || n_key == 0) return;
  dim3 grid(grid_for(ctx, rows, 4), n_key);
  k_key_minmax<<<grid, kThreads, 0, ctx.stream>>>(keys, rows, n_key,
                                                  attr_of_col_dev, mins, maxs);
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
                    const PackSpec& s, uint64_t* out) {
  if (n == 0) return;
  k_project<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(in, n, s, out);
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

template <class KeyT>
void sort_pairs(Context& ctx, const KeyT* keys_in, KeyT* keys_out,
                const int* vals_in, int* vals_out, int64_t n, int bits) {
  if (n == 0) return;
  if (bits == 0) {
    FG_CUDA(cudaMemcpyAsync(keys_out, keys_in, n * sizeof(KeyT),
                            cudaMemcpyDeviceToDevice, ctx.stream));
    FG_CUDA(cudaMemcpyAsync(vals_out, vals_in, n * sizeof(int),
                            cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  size_t temp = 0;
  FG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys_in, keys_out,
                                          vals_in, vals_out, n, 0, bits,
                                          ctx.stream));
  DevArray<unsigned char> tmp(temp, ctx.stream);
  FG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), temp, keys_in, keys_out,
                                          vals_in, vals_out, n, 0, bits,
                                          ctx.stream));
  ctx.launches += (bits + 7) / 8 + 1;
}

template <class KeyT>
void run_length(Context& ctx, const KeyT* sorted, int64_t n,
                KeyT* uniq, int* counts, int64_t* num_runs_dev) {
  size_t temp = 0;
  FG_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, temp, sorted, uniq,
                                             counts, num_runs_dev, n,
                                             ctx.stream));
  DevArray<unsigned char> tmp(temp, ctx.stream);
  FG_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), temp, sorted, uniq,
                                             counts, num_runs_dev, n,
                                             ctx.stream));
  ctx.launches += 2;
}

void exclusive_sum_int(Context& ctx, const int* in, int* out, int64_t n) {
  if (n == 0) return;
  size_t temp = 0;
  FG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, in, out, n, ctx.stream));
  DevArray<unsigned char> tmp(temp, ctx.stream);
  FG_CUDA(
      cub::DeviceScan::ExclusiveSum(tmp.get(), temp, in, out, n, ctx.stream));
  ctx.launches += 2;
}

void inclusive_sum_int(Context& ctx, const int* in, int* out, int64_t n) {
  if (n == 0) return;
  size_t temp = 0;
  FG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, in, out, n, ctx.stream));
  DevArray<unsigned char> tmp(temp, ctx.stream);
  FG_CUDA(
      cub::DeviceScan::InclusiveSum(tmp.get(), temp, in, out, n, ctx.stream));
  ctx.launches += 2;
}

void launch_run_ids(Context& ctx, const uint64_t* sorted, const int* perm,
                    int64_t n, int* flags, int* scan, int* pidx) {
  if (n == 0) return;
  k_head_flags<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(sorted, n, flags);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  inclusive_sum_int(ctx, flags, scan, n);
  k_scatter_runs<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(scan, perm, n,
                                                                pidx);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

// Two-phase grouping so several relations can be sorted before one host
// synchronisation reads all the group counts.
template <class KeyT>
void group_begin_t(Context& ctx, const KeyT* keys, int64_t n, int bits,
                   const int* perm_in, GroupOut& out, GroupPending& pend) {
  out.perm.alloc(n, ctx.stream);
  pend.n = n;
  pend.wide = sizeof(KeyT) == 8;
  DevArray<KeyT>& sorted = *reinterpret_cast<DevArray<KeyT>*>(
      pend.wide ? (void*)&pend.sorted64 : (void*)&pend.sorted32);
  DevArray<KeyT>& uniq = *reinterpret_cast<DevArray<KeyT>*>(
      pend.wide ? (void*)&pend.uniq64 : (void*)&pend.uniq32);
  sorted.alloc(n, ctx.stream);
  sort_pairs<KeyT>(ctx, keys, sorted.get(), perm_in, out.perm.get(), n, bits);
  uniq.alloc(n, ctx.stream);
  pend.counts.alloc(n + 1, ctx.stream);
  pend.nr.alloc(1, ctx.stream);
  if (n) run_length<KeyT>(ctx, sorted.get(), n, uniq.get(), pend.counts.get(), pend.nr.get());
  else pend.nr.zero();
}

void group_finish(Context& ctx, int64_t G, GroupOut& out, GroupPending& pend) {
  const int64_t n = pend.n;
  out.G = G;
  out.begins.alloc(G + 1, ctx.stream);
  exclusive_sum_int(ctx, pend.counts.get(), out.begins.get(), G);
  k_set_last<<<1, 1, 0, ctx.stream>>>(out.begins.get(), G, static_cast<int>(n));
  FG_LAUNCHED(ctx);
  out.uniq.alloc(G, ctx.stream);
  if (G) {
    if (pend.wide) {
      FG_CUDA(cudaMemcpyAsync(out.uniq.get(), pend.uniq64.get(), G * sizeof(uint64_t),
                              cudaMemcpyDeviceToDevice, ctx.stream));
    } else {
      k_widen<<<grid_for(ctx, G), kThreads, 0, ctx.stream>>>(pend.uniq32.get(), G,
                                                            out.uniq.get());
      FG_LAUNCHED(ctx);
      FG_KERNEL_CHECK();
    }
  }
  if (pend.keep_sorted) {
    if (pend.wide) {
      out.sorted = std::move(pend.sorted64);
    } else {
      out.sorted.alloc(n, ctx.stream);
      k_widen<<<grid_for(ctx, n), kThreads, 0, ctx.stream>>>(pend.sorted32.get(), n,
                                                            out.sorted.get());
      FG_LAUNCHED(ctx);
      FG_KERNEL_CHECK();
    }
  }
  pend = GroupPending();
}

void group_begin(Context& ctx, const uint64_t* keys, int64_t n, int bits,
                 const int* perm_in, GroupOut& out, GroupPending& pend) {
  group_begin_t<uint64_t>(ctx, keys, n, bits, perm_in, out, pend);
}
void group_begin32(Context& ctx, const uint32_t* keys, int64_t n, int bits,
                   const int* perm_in, GroupOut& out, GroupPending& pend) {
  group_begin_t<uint32_t>(ctx, keys, n, bits, perm_in, out, pend);
}

void group_begin_presorted(Context& ctx, const uint64_t* keys, int64_t n,
                           const int* perm_in, GroupOut& out, GroupPending& pend) {
  out.perm.alloc(n, ctx.stream);
  pend.n = n;
  pend.wide = true;
  pend.sorted64.alloc(n, ctx.stream);
  if (n) {
    FG_CUDA(cudaMemcpyAsync(out.perm.get(), perm_in, n * sizeof(int),
                            cudaMemcpyDeviceToDevice, ctx.stream));
    FG_CUDA(cudaMemcpyAsync(pend.sorted64.get(), keys, n * sizeof(uint64_t),
                            cudaMemcpyDeviceToDevice, ctx.stream));
  }
  pend.uniq64.alloc(n, ctx.stream);
  pend.counts.alloc(n + 1, ctx.stream);
  pend.nr.alloc(1, ctx.stream);
  if (n) run_length<uint64_t>(ctx, pend.sorted64.get(), n, pend.uniq64.get(),
                              pend.counts.get(), pend.nr.get());
  else pend.nr.zero();
}

template <class KeyT>
void group_sorted_t(Context& ctx, const KeyT* keys, int64_t n, int bits,
                    const int* perm_in, GroupOut& out, bool keep_sorted) {
  GroupPending pend;
  pend.keep_sorted = keep_sorted;
  group_begin_t<KeyT>(ctx, keys, n, bits, perm_in, out, pend);
  int64_t G = 0;
  FG_CUDA(cudaMemcpyAsync(&G, pend.nr.get(), sizeof G, cudaMemcpyDeviceToHost,
                          ctx.stream));
  sync_stream(ctx);
  group_finish(ctx, G, out, pend);
}

void group_sorted(Context& ctx, const uint64_t* keys, int64_t n, int bits,
                  const int* perm_in, GroupOut& out, bool keep_sorted) {
  group_sorted_t<uint64_t>(ctx, keys, n, bits, perm_in, out, keep_sorted);
}

void group_sorted32(Context& ctx, const uint32_t* keys, int64_t n, int bits,
                    const int* perm_in, GroupOut& out, bool keep_sorted) {
  group_sorted_t<uint32_t>(ctx, keys, n, bits, perm_in, out, keep_sorted);
}

template void launch_pack_keys<uint64_t>(Context&, const int64_t*, int64_t, int,
                                         const PackSpec&, uint64_t*, int*);
template void launch_pack_keys<uint32_t>(Context&, const int64_t*, int64_t, int,
                                         const PackSpec&, uint32_t*, int*);

}  // namespace fg
