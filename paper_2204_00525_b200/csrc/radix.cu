// K1 core: hand-written stable LSD radix sort (onesweep with decoupled
// look-back) and segment extraction, for sm_100a.
//
// Replaces the sort of the reference's canonicalize (relation.hpp:127-167)
// and the contiguous key groups it produces (relation.hpp:56-66,
// counts.hpp:80-88).  Keys are the order-preserving packed u32/u64 keys of
// group.cu; only the significant bits are sorted, in passes of <= 8 bits
// whose widths are balanced (C2's 20-bit keys: 7+7+6, C3's 47-bit fact key:
// 8+8+8+8+8+7).
//
// One sort = one histogram launch (every pass's digit histogram in a single
// read of the keys; fused into key packing when the keys are packed here) +
// one memset of the look-back state + one launch per pass.  A pass kernel
// takes tiles of kTile keys in launch order (atomic tile ticket, so every
// earlier tile is resident and look-back always progresses):
//   1. warp-striped coalesced loads (lane l of warp w holds keys
//      w*IPT*32 + i*32 + l of the tile -- i-major, so the warp's items are in
//      input order);
//   2. stable in-warp ranking with __match_any_sync + per-warp 16-bit digit
//      counters in shared memory;
//   3. per-digit tile counts published to the look-back array, then each
//      thread resolves its digits' tile-exclusive prefix by walking back
//      (aggregate / inclusive-prefix flags in one 32-bit word);
//   4. the tile is reordered in shared memory by (digit, rank) and written
//      out with consecutive threads on consecutive output positions of each
//      digit run.
// The first pass may generate the row-id payload itself (vals_in == null),
// so the identity permutation is never written or read.
//
// Segment extraction (k_segments) reads the sorted keys once: head flags,
// a block scan + single-value look-back for the run index, and writes
// begins[run] (int32), uniq[run] (u64), the run count, and optionally
// pidx[perm[pos]] = run (the run id of every input element).
#include <cstdlib>
#include <string>

#include "launchers.cuh"

namespace fg {

namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kMaxPasses = 8;
constexpr uint32_t kPrefixFlag = 0x80000000u;
constexpr unsigned long long kSegPrefix = 1ull << 63;

template <class KeyT>
struct SortCfg;
#ifndef FG_SORT_IPT64
#define FG_SORT_IPT64 16
#endif
template <>
struct SortCfg<uint64_t> {
  static constexpr int kIpt = FG_SORT_IPT64;  // 16: 4096 keys per tile, 48 KB staged
};
#ifndef FG_SORT_IPT32
#define FG_SORT_IPT32 24
#endif
template <>
struct SortCfg<uint32_t> {
  static constexpr int kIpt = FG_SORT_IPT32;  // 24: 6144 keys per tile, 48 KB staged
};

struct PassPlan {
  int n;
  int shift[kMaxPasses];
  int width[kMaxPasses];
};

PassPlan plan_passes(int bits) {
  PassPlan p{};
  if (bits <= 0) return p;
  p.n = (bits + kRadixBits - 1) / kRadixBits;
  int s = 0;
  for (int i = 0; i < p.n; ++i) {
    const int w = bits / p.n + (i < bits % p.n ? 1 : 0);
    p.shift[i] = s;
    p.width[i] = w;
    s += w;
  }
  return p;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive sum of one value per thread (kSortThreads threads).
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* s_warp,
                                                   uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // s_warp may still be read by a previous call
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < kSortWarps ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < kSortWarps; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kSortWarps) s_warp[lane] = t;  // inclusive
  }
  __syncthreads();
  const uint32_t before = warp ? s_warp[warp - 1] : 0;
  if (total) *total = s_warp[kSortWarps - 1];
  return before + x - v;
}

// ---------------------------------------------------------------- histogram

struct HistPlan {
  int n;
  int shift[kMaxPasses];
  uint32_t mask[kMaxPasses];
};

HistPlan hist_plan(const PassPlan& p) {
  HistPlan h{};
  h.n = p.n;
  for (int i = 0; i < p.n; ++i) {
    h.shift[i] = p.shift[i];
    h.mask[i] = (1u << p.width[i]) - 1;
  }
  return h;
}

// Per-warp privatised digit histograms of every pass, one read of the keys.
template <class KeyT>
__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const KeyT* __restrict__ keys,
                                                             int64_t n, HistPlan hp,
                                                             uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t s_hist[];  // [warps][passes][kBins]
  const int warp = threadIdx.x >> 5;
  const int per = hp.n * kBins;
  for (int i = threadIdx.x; i < kSortWarps * per; i += kSortThreads) s_hist[i] = 0;
  __syncthreads();
  uint32_t* my = s_hist + warp * per;
  const int64_t stride = (int64_t)gridDim.x * kSortThreads;
  for (int64_t i = blockIdx.x * (int64_t)kSortThreads + threadIdx.x; i < n; i += stride) {
    const KeyT k = keys[i];
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p)
      if (p < hp.n)
        atomicAdd(&my[p * kBins + (uint32_t)((k >> hp.shift[p]) & hp.mask[p])], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < per; i += kSortThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) s += s_hist[w * per + i];
    if (s) atomicAdd(&hist[i], s);
  }
}

// Key packing (group.cu's per-attribute offset encoding) fused with the
// digit histograms of the sort that follows.
template <class KeyT>
__global__ void __launch_bounds__(kSortThreads) k_pack_hist(
    const int64_t* __restrict__ keys, int64_t rows, int n_key, PackSpec spec,
    KeyT* __restrict__ out, HistPlan hp, uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t s_hist[];
  const int warp = threadIdx.x >> 5;
  const int per = hp.n * kBins;
  for (int i = threadIdx.x; i < kSortWarps * per; i += kSortThreads) s_hist[i] = 0;
  __syncthreads();
  uint32_t* my = s_hist + warp * per;
  const int64_t stride = (int64_t)gridDim.x * kSortThreads;
  for (int64_t i = blockIdx.x * (int64_t)kSortThreads + threadIdx.x; i < rows; i += stride) {
    uint64_t k = 0;
    for (int f = 0; f < spec.n; ++f) {
      const long long v = keys[i * n_key + spec.col[f]];
      const uint64_t enc = (uint64_t)v - (uint64_t)spec.min[f];
      if (spec.bits[f]) k |= enc << spec.shift[f];
    }
    const KeyT kk = static_cast<KeyT>(k);
    out[i] = kk;
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p)
      if (p < hp.n)
        atomicAdd(&my[p * kBins + (uint32_t)((kk >> hp.shift[p]) & hp.mask[p])], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < per; i += kSortThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) s += s_hist[w * per + i];
    if (s) atomicAdd(&hist[i], s);
  }
}

// ------------------------------------------------------------- onesweep pass

template <class KeyT>
struct PassSmem {
  static constexpr int kIpt = SortCfg<KeyT>::kIpt;
  static constexpr int kTile = kSortThreads * kIpt;
  KeyT k[kTile];  // the tile: input order, then (digit, rank) order
  int v[kTile];
  uint16_t warp_cnt[kSortWarps][kBins];
  int glob[kBins];       // output position of tile-local sorted slot 0 of digit d
  uint32_t excl[kBins];  // tile-local exclusive start of digit d
  uint32_t scan_tmp[kSortWarps];
  uint32_t tile;
  unsigned long long bar;  // mbarrier of the tile's bulk copies
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (TMA engine, no tensor map), completing on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

// Tile-exclusive prefix of digit b for `tile` by decoupled look-back over
// the per-tile words of `look` (row stride kBins): LB predecessors are loaded
// per round trip.
template <int LB>
__device__ __forceinline__ uint32_t look_back(const uint32_t* look, int tile, int b) {
  uint32_t pre = 0;
  int t = tile - 1;
  while (true) {
    uint32_t x[LB];
#pragma unroll
    for (int j = 0; j < LB; ++j)
      x[j] = t - j >= 0 ? ld_acquire_u32(&look[(int64_t)(t - j) * kBins + b]) : kPrefixFlag;
    int used = 0;
    bool done = false, stall = false;
#pragma unroll
    for (int j = 0; j < LB; ++j) {
      if (done || stall) continue;
      if (x[j] == 0) {
        stall = true;
      } else if (x[j] & kPrefixFlag) {
        pre += x[j] & ~kPrefixFlag;
        done = true;
      } else {
        pre += x[j] - 1;
        ++used;
      }
    }
    if (done) return pre;
    t -= used;
  }
}

// One LSD pass.  The tile (keys, and the payload unless it is the row id)
// arrives in shared memory by bulk copy; ranking reads it from there, so
// registers hold only the ranks and occupancy is 3 CTAs per SM.
// 4 CTAs per SM for 64-bit keys (measured 7.0 vs 7.3 ms on 100M 47-bit keys),
// 3 for 32-bit keys (their 24-item tiles spill at the 64-register cap).
template <class KeyT, int LB>
__global__ void __launch_bounds__(kSortThreads, sizeof(KeyT) == 8 ? 4 : 3) k_onesweep(
    const KeyT* __restrict__ keys_in, KeyT* __restrict__ keys_out,
    const int* __restrict__ vals_in, int* __restrict__ vals_out, int n, int shift,
    uint32_t mask, const uint32_t* __restrict__ hist, uint32_t* __restrict__ look,
    uint32_t* __restrict__ ticket, int bulk_ok) {
  constexpr int kIpt = SortCfg<KeyT>::kIpt;
  constexpr int kTile = PassSmem<KeyT>::kTile;
  constexpr int kBinsPerThread = kBins / kSortThreads;
  static_assert(kBins % kSortThreads == 0, "bins per thread");
  extern __shared__ __align__(128) unsigned char s_raw[];
  PassSmem<KeyT>& s = *reinterpret_cast<PassSmem<KeyT>*>(s_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    s.tile = atomicAdd(ticket, 1u);
    mbar_init(&s.bar, 1);
  }
  for (int i = tid; i < kSortWarps * kBins; i += kSortThreads)
    (&s.warp_cnt[0][0])[i] = 0;
  __syncthreads();
  const int tile = (int)s.tile;
  const int64_t base = (int64_t)tile * kTile;
  const int tile_n = (int)((int64_t)n - base < kTile ? (int64_t)n - base : kTile);
  const bool full = tile_n == kTile;
  if (full && bulk_ok) {
    if (tid == 0) {
      const unsigned kb = kTile * sizeof(KeyT), vb = vals_in ? kTile * sizeof(int) : 0;
      mbar_expect_tx(&s.bar, kb + vb);
      bulk_g2s(s.k, keys_in + base, kb, &s.bar);
      if (vals_in) bulk_g2s(s.v, vals_in + base, vb, &s.bar);
    }
    mbar_wait(&s.bar, 0);
  } else {
    for (int p = tid; p < tile_n; p += kSortThreads) {
      s.k[p] = keys_in[base + p];
      if (vals_in) s.v[p] = vals_in[base + p];
    }
    __syncthreads();
  }
  const int wb = warp * kIpt * 32;  // this warp's items: wb + i*32 + lane
  constexpr uint32_t kNone = 0xffffffffu;
  auto digit = [&](int i) -> uint32_t {
    const int p = wb + i * 32 + lane;
    return (full || p < tile_n) ? (uint32_t)(s.k[p] >> shift) & mask : kNone;
  };
  // Stable in-warp ranks (items in i-major order = input order); peers of
  // equal digit from one ballot per digit bit.
  uint16_t r[kIpt];
  uint16_t* wc = s.warp_cnt[warp];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint32_t d = digit(i);
    const bool valid = d != kNone;
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int bb = 0; bb < kRadixBits; ++bb) {
      const bool bit = (d >> bb) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
    if (!full) {
      const uint32_t bal = __ballot_sync(0xffffffffu, valid);
      peers &= valid ? bal : ~bal;
    }
    uint32_t before = 0;
    if (valid) before = wc[d];
    __syncwarp();
    if (valid) {
      r[i] = (uint16_t)(before + __popc(peers & lt));
      if ((peers & lt) == 0) wc[d] = (uint16_t)(before + __popc(peers));
    }
    __syncwarp();
  }
  __syncthreads();

  // Per digit: warp offsets, tile count; publish; block scan over digits.
  uint32_t cnt[kBinsPerThread];
  uint32_t local = 0;
#pragma unroll
  for (int j = 0; j < kBinsPerThread; ++j) {
    const int b = tid * kBinsPerThread + j;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = s.warp_cnt[w][b];
      s.warp_cnt[w][b] = (uint16_t)run;
      run += c;
    }
    cnt[j] = run;
    local += run;
    st_release_u32(&look[(int64_t)tile * kBins + b],
                   tile == 0 ? (kPrefixFlag | run) : run + 1);
  }
  // Global digit starts: exclusive scan of the pass histogram.
  uint32_t hsum = 0, hv[kBinsPerThread];
#pragma unroll
  for (int j = 0; j < kBinsPerThread; ++j) {
    hv[j] = hist[tid * kBinsPerThread + j];
    hsum += hv[j];
  }
  uint32_t texcl = block_excl_sum(local, s.scan_tmp, nullptr);
  uint32_t hexcl = block_excl_sum(hsum, s.scan_tmp, nullptr);
#pragma unroll
  for (int j = 0; j < kBinsPerThread; ++j) {
    const int b = tid * kBinsPerThread + j;
    uint32_t pre = 0;
    if (tile > 0) {
      pre = look_back<LB>(look, tile, b);
      st_release_u32(&look[(int64_t)tile * kBins + b], kPrefixFlag | (pre + cnt[j]));
    }
    s.excl[b] = texcl;
    s.glob[b] = (int)(hexcl + pre) - (int)texcl;
    texcl += cnt[j];
    hexcl += hv[j];
  }
  __syncthreads();
  // Reorder the tile in place by (digit, rank): read every owned item, then
  // write it to its sorted slot.
  // (the slot is recomputed from the key in the write loop: no position
  // array, so the kernel fits 4 CTAs per SM)
  KeyT kk[kIpt];
  int vv[kIpt];
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const int p = wb + i * 32 + lane;
    if (full || p < tile_n) {
      kk[i] = s.k[p];
      vv[i] = vals_in ? s.v[p] : (int)(base + p);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const int p = wb + i * 32 + lane;
    if (full || p < tile_n) {
      const uint32_t d = (uint32_t)(kk[i] >> shift) & mask;
      const int q = (int)s.excl[d] + s.warp_cnt[warp][d] + r[i];
      s.k[q] = kk[i];
      s.v[q] = vv[i];
    }
  }
  __syncthreads();
  for (int p = tid; p < tile_n; p += kSortThreads) {
    const KeyT key = s.k[p];
    const int o = s.glob[(uint32_t)(key >> shift) & mask] + p;
    keys_out[o] = key;
    vals_out[o] = s.v[p];
  }
}

// Single-value decoupled look-back by one warp: publishes `total` for
// `tile`, resolves the tile's exclusive prefix 32 predecessors per round trip
// and publishes the inclusive prefix.  Called by all lanes of one warp.
__device__ __forceinline__ unsigned long long warp_look_back(unsigned long long* look,
                                                             int64_t tile,
                                                             unsigned long long total,
                                                             int lane) {
  if (tile == 0) {
    if (lane == 0) st_release_u64(&look[0], kSegPrefix | total);
    return 0;
  }
  if (lane == 0) st_release_u64(&look[tile], total + 1);
  unsigned long long pre = 0;
  int64_t t = tile - 1;
  while (true) {
    const int64_t tt = t - lane;
    unsigned long long x = kSegPrefix;  // before tile 0: a zero prefix
    if (tt >= 0) {
      do {
        x = ld_acquire_u64(&look[tt]);
      } while (x == 0);
    }
    // Nearest predecessor holding an inclusive prefix (lowest lane).
    const uint32_t pm = __ballot_sync(0xffffffffu, (x & kSegPrefix) != 0);
    const int stop = pm ? __ffs(pm) - 1 : 32;
    unsigned long long v = lane < stop ? x - 1 : (lane == stop ? x & ~kSegPrefix : 0);
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    pre += v;
    if (pm) break;
    t -= 32;
  }
  if (lane == 0) st_release_u64(&look[tile], kSegPrefix | (pre + total));
  return pre;
}

// ------------------------------------------------------- segment extraction

#ifndef FG_SEG_IPT
#define FG_SEG_IPT 8
#endif
constexpr int kSegIpt = FG_SEG_IPT;
constexpr int kSegTile = kSortThreads * kSegIpt;

template <class KeyT>
__global__ void __launch_bounds__(kSortThreads) k_segments(
    const KeyT* __restrict__ sorted, int64_t n, int* __restrict__ begins,
    uint64_t* __restrict__ uniq, int64_t* __restrict__ n_runs,
    const int* __restrict__ perm, int* __restrict__ pidx,
    unsigned long long* __restrict__ look, uint32_t* __restrict__ ticket,
    const int64_t* __restrict__ n_dev) {
  __shared__ uint32_t s_tile, s_scan[kSortWarps], s_total;
  __shared__ unsigned long long s_pre;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // n_dev: the element count lives on the device (a group count not yet read
  // by the host); the grid covers the host's upper bound and the tiles past
  // the real end retire at once (nothing looks back at them).
  if (n_dev) n = *n_dev;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  if (tile * kSegTile >= n) return;
  const int64_t wbase = tile * kSegTile + (int64_t)warp * kSegIpt * 32;
  KeyT k[kSegIpt];
  uint32_t flags[kSegIpt];
  uint32_t mine = 0;
#pragma unroll
  for (int i = 0; i < kSegIpt; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    bool head = false;
    if (idx < n) {
      k[i] = sorted[idx];
      head = idx == 0 || sorted[idx - 1] != k[i];
    }
    flags[i] = __ballot_sync(0xffffffffu, head);
    mine += __popc(flags[i]);
  }
  // mine = heads in this warp's chunk (same in every lane).
  uint32_t total;
  const uint32_t wexcl = block_excl_sum(lane == 0 ? mine : 0, s_scan, &total);
  const uint32_t warp_excl = __shfl_sync(0xffffffffu, wexcl, 0);
  if (warp == 0) {
    const unsigned long long pre = warp_look_back(look, tile, total, lane);
    if (lane == 0) {
      s_pre = pre;
      s_total = total;
      if ((tile + 1) * kSegTile >= n) {  // last tile
        *n_runs = (int64_t)(pre + total);
        begins[pre + total] = (int)n;
      }
    }
  }
  __syncthreads();
  const unsigned long long pre = s_pre;
  // Run index of item (i, lane) = heads at or before it - 1.
  uint32_t seen = warp_excl;
#pragma unroll
  for (int i = 0; i < kSegIpt; ++i) {
    const int64_t idx = wbase + i * 32 + lane;
    const uint32_t f = flags[i];
    const uint32_t at = seen + __popc(f & lanemask_lt());
    if (idx < n) {
      const bool head = (f >> lane) & 1u;
      const int64_t run = (int64_t)pre + at + (head ? 1 : 0) - 1;
      if (head) {
        begins[run] = (int)idx;
        uniq[run] = (uint64_t)k[i];
      }
      if (pidx) pidx[perm ? perm[idx] : idx] = (int)run;
    }
    seen += __popc(f);
  }
}

// ------------------------------------------------------------ int scan

constexpr int kScanIpt = 16;
constexpr int kScanTile = kSortThreads * kScanIpt;

// Exclusive or inclusive sum of int32 (single-pass, decoupled look-back).
__global__ void __launch_bounds__(kSortThreads) k_scan_int(
    const int* __restrict__ in, int* __restrict__ out, int64_t n, bool inclusive,
    unsigned long long* __restrict__ look, uint32_t* __restrict__ ticket) {
  __shared__ uint32_t s_tile, s_scan[kSortWarps];
  __shared__ unsigned long long s_pre;
  __shared__ int s_vals[kScanTile];
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile, base = tile * kScanTile;
  for (int i = tid; i < kScanTile; i += kSortThreads)
    s_vals[i] = base + i < n ? in[base + i] : 0;
  __syncthreads();
  int x[kScanIpt];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kScanIpt; ++j) {
    x[j] = s_vals[tid * kScanIpt + j];
    sum += (uint32_t)x[j];
  }
  uint32_t total;
  uint32_t excl = block_excl_sum(sum, s_scan, &total);
  if (tid < 32) {
    const unsigned long long pre = warp_look_back(look, tile, total, tid);
    if (tid == 0) s_pre = pre;
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_pre + excl;
#pragma unroll
  for (int j = 0; j < kScanIpt; ++j) {
    if (!inclusive) s_vals[tid * kScanIpt + j] = (int)run;
    run += (uint32_t)x[j];
    if (inclusive) s_vals[tid * kScanIpt + j] = (int)run;
  }
  __syncthreads();
  for (int i = tid; i < kScanTile; i += kSortThreads)
    if (base + i < n) out[base + i] = s_vals[i];
}

__global__ void k_flags_to_int(const char* __restrict__ keep, int64_t n, int* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    f[i] = keep[i] ? 1 : 0;
}

__global__ void k_compact(const int* __restrict__ in, const char* __restrict__ keep,
                          const int* __restrict__ pos, int64_t n, int* __restrict__ out,
                          int64_t* __restrict__ count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (keep[i]) out[pos[i]] = in[i];
    if (i == n - 1) *count = (int64_t)pos[i] + (keep[i] ? 1 : 0);
  }
}

int hist_grid(const Context& ctx, int64_t n) {
  const int64_t g = std::min<int64_t>(ceil_div(n, kSortThreads * 4), (int64_t)ctx.sm_count * 4);
  return (int)std::max<int64_t>(g, 1);
}

}  // namespace

// Digit histograms of every pass of a `bits`-bit sort (hist: passes x kBins,
// zeroed here).
template <class KeyT>
static void digit_hist(Context& ctx, const KeyT* keys, int64_t n, const PassPlan& pp,
                       uint32_t* hist) {
  FG_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * pp.n * kBins, ctx.stream));
  const size_t smem = sizeof(uint32_t) * kSortWarps * pp.n * kBins;
  FG_CUDA(cudaFuncSetAttribute(k_digit_hist<KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  k_digit_hist<KeyT><<<hist_grid(ctx, n), kSortThreads, smem, ctx.stream>>>(
      keys, n, hist_plan(pp), hist);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

int radix_passes(int bits) { return plan_passes(bits).n; }
size_t radix_hist_size(int bits) { return (size_t)std::max(plan_passes(bits).n, 1) * kBins; }

template <class KeyT>
void launch_pack_hist(Context& ctx, const int64_t* keys, int64_t rows, int n_key,
                      const PackSpec& spec, int bits, KeyT* out, uint32_t* hist) {
  const PassPlan pp = plan_passes(bits);
  FG_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * radix_hist_size(bits), ctx.stream));
  if (rows == 0) return;
  const size_t smem = sizeof(uint32_t) * kSortWarps * std::max(pp.n, 1) * kBins;
  FG_CUDA(cudaFuncSetAttribute(k_pack_hist<KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  k_pack_hist<KeyT><<<hist_grid(ctx, rows), kSortThreads, smem, ctx.stream>>>(
      keys, rows, n_key, spec, out, hist_plan(pp), hist);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

template <class KeyT>
void radix_sort_pairs(Context& ctx, const KeyT* keys_in, KeyT* keys_out, const int* vals_in,
                      int* vals_out, int64_t n, int bits, const uint32_t* hist_in) {
  if (n == 0) return;
  if (n > INT_MAX) fail(FG_E_UNSUPPORTED, "radix sort of more than 2^31-1 keys");
  const PassPlan pp = plan_passes(bits);
  cudaStream_t st = ctx.stream;
  if (pp.n == 0) {  // every key equal: the stable order is the input order
    FG_CUDA(cudaMemcpyAsync(keys_out, keys_in, n * sizeof(KeyT), cudaMemcpyDeviceToDevice, st));
    if (vals_in)
      FG_CUDA(cudaMemcpyAsync(vals_out, vals_in, n * sizeof(int), cudaMemcpyDeviceToDevice, st));
    else
      launch_iota(ctx, vals_out, n);
    return;
  }
  constexpr int kTile = PassSmem<KeyT>::kTile;
  const int64_t tiles = ceil_div(n, kTile);
  // Look-back words of every pass + one tile ticket per pass, one memset.
  DevArray<uint32_t> look((size_t)pp.n * (tiles * kBins + 32), st);
  FG_CUDA(cudaMemsetAsync(look.get(), 0, look.bytes(), st));
  DevArray<uint32_t> hist_own;
  const uint32_t* hist = hist_in;
  if (!hist) {
    hist_own.alloc((size_t)pp.n * kBins, st);
    digit_hist<KeyT>(ctx, keys_in, n, pp, hist_own.get());
    hist = hist_own.get();
  }
  DevArray<KeyT> tk;
  DevArray<int> tv;
  if (pp.n > 1) {
    tk.alloc(n, st);
    tv.alloc(n, st);
  }
  const size_t smem = sizeof(PassSmem<KeyT>);
  // FG_SORT_LB=1|4: look-back predecessors per round trip (experiments).
  static const int lb = [] {
    const char* e = getenv("FG_SORT_LB");
    return e && std::string(e) == "1" ? 1 : 4;
  }();
  // (A persistent two-buffer variant that prefetched its next ticket was
  // measured 10x slower: tiles prefetched but not yet ranked stall every
  // later tile's look-back.)
  auto kern = lb == 1 ? k_onesweep<KeyT, 1> : k_onesweep<KeyT, 4>;
  FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const KeyT* ki = keys_in;
  const int* vi = vals_in;
  for (int p = 0; p < pp.n; ++p) {
    const bool to_out = ((pp.n - 1 - p) & 1) == 0;
    KeyT* ko = to_out ? keys_out : tk.get();
    int* vo = to_out ? vals_out : tv.get();
    uint32_t* lk = look.get() + (size_t)p * (tiles * kBins + 32);
    const int bulk = aligned(ki) && (!vi || aligned(vi)) && !getenv("FG_SORT_NO_BULK");
    kern<<<(unsigned)tiles, kSortThreads, smem, st>>>(
        ki, ko, vi, vo, (int)n, pp.shift[p], (1u << pp.width[p]) - 1, hist + p * kBins,
        lk + 32, lk, bulk);
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    ki = ko;
    vi = vo;
  }
}

template <class KeyT>
void launch_segments(Context& ctx, const KeyT* sorted, int64_t n, int* begins, uint64_t* uniq,
                     int64_t* n_runs, const int* perm, int* pidx, const int64_t* n_dev) {
  cudaStream_t st = ctx.stream;
  if (n == 0) {
    FG_CUDA(cudaMemsetAsync(n_runs, 0, sizeof(int64_t), st));
    FG_CUDA(cudaMemsetAsync(begins, 0, sizeof(int), st));
    return;
  }
  const int64_t tiles = ceil_div(n, kSegTile);
  DevArray<unsigned long long> look(tiles + 2, st);
  FG_CUDA(cudaMemsetAsync(look.get(), 0, look.bytes(), st));
  k_segments<KeyT><<<(unsigned)tiles, kSortThreads, 0, st>>>(
      sorted, n, begins, uniq, n_runs, perm, pidx, look.get() + 2,
      reinterpret_cast<uint32_t*>(look.get()), n_dev);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void scan_int(Context& ctx, const int* in, int* out, int64_t n, bool inclusive) {
  if (n == 0) return;
  cudaStream_t st = ctx.stream;
  const int64_t tiles = ceil_div(n, kScanTile);
  DevArray<unsigned long long> look(tiles + 2, st);
  FG_CUDA(cudaMemsetAsync(look.get(), 0, look.bytes(), st));
  k_scan_int<<<(unsigned)tiles, kSortThreads, 0, st>>>(
      in, out, n, inclusive, look.get() + 2, reinterpret_cast<uint32_t*>(look.get()));
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void compact_flagged(Context& ctx, const int* in, const char* keep, int* out, int64_t n,
                     int64_t* count) {
  cudaStream_t st = ctx.stream;
  if (n == 0) {
    FG_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return;
  }
  DevArray<int> f(n, st), pos(n, st);
  const int grid = hist_grid(ctx, n);
  k_flags_to_int<<<grid, kSortThreads, 0, st>>>(keep, n, f.get());
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  scan_int(ctx, f.get(), pos.get(), n, false);
  k_compact<<<grid, kSortThreads, 0, st>>>(in, keep, pos.get(), n, out, count);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

template void launch_pack_hist<uint64_t>(Context&, const int64_t*, int64_t, int, const PackSpec&,
                                         int, uint64_t*, uint32_t*);
template void launch_pack_hist<uint32_t>(Context&, const int64_t*, int64_t, int, const PackSpec&,
                                         int, uint32_t*, uint32_t*);
template void radix_sort_pairs<uint64_t>(Context&, const uint64_t*, uint64_t*, const int*, int*,
                                         int64_t, int, const uint32_t*);
template void radix_sort_pairs<uint32_t>(Context&, const uint32_t*, uint32_t*, const int*, int*,
                                         int64_t, int, const uint32_t*);
template void launch_segments<uint64_t>(Context&, const uint64_t*, int64_t, int*, uint64_t*,
                                        int64_t*, const int*, int*, const int64_t*);
template void launch_segments<uint32_t>(Context&, const uint32_t*, int64_t, int*, uint64_t*,
                                        int64_t*, const int*, int*, const int64_t*);

}  // namespace fg
