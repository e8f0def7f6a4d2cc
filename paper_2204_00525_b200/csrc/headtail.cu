// K3/K5: segmented heads and tails (plain and generalized) and K4 join.
//
// Reference: head/tail (givens.hpp:59-92), generalized_head/_tail
// (givens.hpp:106-148), heads_and_tails (figaro.hpp:109-159),
// project_away_join_attributes (figaro.hpp:232-294) and
// process_and_join_children (figaro.hpp:179-230).
//
// The reference copies every key group into a fresh Matrix and walks it with
// one thread per group, so a 2M-row group runs on one core.  Here the sorted
// row order is cut into fixed units of kUnit rows, independent of the group
// sizes.  One warp owns a unit at a time (dynamic ticket) and streams it
// through shared memory in batches with cp.async (LDGSTS); rows are gathered
// through the sort permutation, so the input is never physically permuted.
// Each lane owns columns; it carries the running prefix S_j (and, for the
// generalized transform, the weighted prefix) across batches and resets it at
// group starts.  Row coefficients
//     tail_j = (sqrt(j) a_j - S_j / sqrt(j)) / sqrt(j+1) * sqrt(phi)
//            = a_j * alpha_j - S_j * beta_j
// are computed once per row by one lane and broadcast through shared memory.
//
// Groups crossing a unit boundary need the prefix of their earlier rows.
// Short groups (<= kLight rows) re-read those rows (at most kLight, mostly L2
// hits).  Long groups get it from a deterministic pre-pass: per unit the
// partial sum of its continuing group, then a per-group scan over units.
// All results are run-to-run deterministic.
#include <cuda_pipeline.h>

#include "launchers.cuh"

namespace fg {

namespace {

constexpr int kWarps = 8;            // warps per CTA
constexpr int kUnit = 256;           // rows per work unit
constexpr int kLight = 256;          // groups up to this size recompute carries
constexpr int kSmemDoubles = 512;    // per-warp row buffer (4 KB)
constexpr int kMaxRB = 64;           // max rows per batch

struct HtDev {
  const double* data;
  int64_t ld;
  int w;
  const int* perm;
  const int* begins;
  int64_t n_seg;
  int64_t n_rows;
  const double* weights;
  const uint64_t* tail_count;
  const uint64_t* scale_count;
  const int* head_index;
  double* heads;
  int64_t ldh;
  double* tails;
  int64_t ldt;
  double* scales;
  int rb;            // rows per batch
  int64_t n_units;
  // heavy-group carries
  const int* cont;       // per unit: continuing long group or -1
  const double* carry;   // per unit: incoming carry (V values), valid when
                         // cont[u-1] == first group of u
  int* ticket;
};

__device__ __forceinline__ int64_t src_row(const HtDev& a, int64_t p) {
  return a.perm ? (int64_t)a.perm[p] : p;
}

// Last group index g with begins[g] <= p, searching g in [lo, hi).
__device__ __forceinline__ int64_t seg_of(const int* __restrict__ begins,
                                          int64_t p, int64_t lo, int64_t hi) {
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (begins[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

struct WarpSmem {
  double buf[kSmemDoubles];
  double alpha[kMaxRB];
  double beta[kMaxRB];
  double hco[kMaxRB];   // head coefficient at a group's last row
  double wt[kMaxRB];
  int seg[kMaxRB];
  int flags[kMaxRB];    // bit0 start, bit1 last
};

// Copies rows [p, p+nb) of the sorted order (w doubles each) into buf.
__device__ __forceinline__ void stage_rows(const HtDev& a, WarpSmem& sm,
                                           int64_t p, int nb, int lane) {
  const int w = a.w;
  const int total = nb * w;
  for (int e = lane; e < total; e += 32) {
    const int r = e / w;
    const int c = e - r * w;
    const double* src = a.data + src_row(a, p + r) * a.ld + c;
    __pipeline_memcpy_async(&sm.buf[e], src, sizeof(double));
  }
  __pipeline_commit();
}

template <int SLOTS>
__device__ void process_unit(const HtDev& a, WarpSmem& sm, int64_t u,
                             int lane) {
  const int w = a.w;
  const bool weighted = a.weights != nullptr;
  const int64_t p0 = u * kUnit;
  const int64_t p1 = min(p0 + kUnit, a.n_rows);
  int64_t g = seg_of(a.begins, p0, 0, a.n_seg);

  double S[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) S[s] = 0.0;
  double N = 0.0;  // weighted: running sum of squared weights (lane-uniform)

  const int64_t gb = a.begins[g];
  if (gb < p0) {
    // The first group started in an earlier unit: get its prefix.
    if (u > 0 && a.cont && a.cont[u - 1] == (int)g) {
      const int V = w + (weighted ? 1 : 0);
      const double* cr = a.carry + u * (int64_t)V;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int c = lane + 32 * s;
        if (c < w) S[s] = cr[c];
      }
      if (weighted) N = cr[w];
    } else {
      for (int64_t q = gb; q < p0; ++q) {
        const int64_t r = src_row(a, q);
        const double v = weighted ? a.weights[r] : 1.0;
        const double* row = a.data + r * a.ld;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
          const int c = lane + 32 * s;
          if (c < w) S[s] += weighted ? v * row[c] : row[c];
        }
        if (weighted) N += v * v;
      }
    }
  }

  for (int64_t pb = p0; pb < p1; pb += a.rb) {
    const int nb = (int)(p1 - pb < (int64_t)a.rb ? p1 - pb : (int64_t)a.rb);
    if (w > 0) stage_rows(a, sm, pb, nb, lane);
    // Row metadata and coefficients, one row per lane.
    const int64_t g_hi = (g + nb + 1 < a.n_seg) ? g + nb + 1 : a.n_seg;
    for (int base = 0; base < nb; base += 32) {
      const int rr = base + lane;
      const bool live = rr < nb;
      int64_t sg = g;
      int64_t jj = 0, m = 1;
      double v = 1.0;
      int fl = 0;
      if (live) {
        const int64_t p = pb + rr;
        sg = seg_of(a.begins, p, g, g_hi);
        const int64_t b0 = a.begins[sg];
        const int64_t b1 = a.begins[sg + 1];
        jj = p - b0;
        m = b1 - b0;
        fl = (jj == 0 ? 1 : 0) | (p == b1 - 1 ? 2 : 0);
        if (weighted) v = a.weights[src_row(a, p)];
      }
      double ts = 1.0;
      if (live && a.tail_count) ts = sqrt((double)a.tail_count[sg]);
      double al = 0.0, be = 0.0, hc = 0.0, sc = 0.0;
      if (!weighted) {
        if (live && jj >= 1) {
          const double sj = sqrt((double)jj);
          const double sj1 = sqrt((double)(jj + 1));
          al = sj / sj1 * ts;
          be = ts / (sj * sj1);
        }
        if (live && (fl & 2)) {
          const double sm_ = sqrt((double)m);
          hc = 1.0 / sm_;
          sc = sm_;
        }
      } else {
        // Segmented inclusive scan of v^2 over the 32 rows of this chunk.
        double x = live ? v * v : 0.0;
        int st = live ? (fl & 1) : 0;
        // Carry N into the first row unless it starts a group.
        if (lane == 0 && !st) x += N;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, x, o);
          const int sy = __shfl_up_sync(0xffffffffu, st, o);
          if (lane >= o && !st) x += y;
          if (lane >= o) st |= sy;
        }
        // x = inclusive norm^2 through this row; the exclusive value is the
        // previous row's inclusive one (or the carry), 0 at a group start.
        const double incl = x;
        const double prev = __shfl_up_sync(0xffffffffu, incl, 1);
        const double excl = (fl & 1) ? 0.0 : (lane == 0 ? N : prev);
        if (live && jj >= 1) {
          const double np_ = sqrt(excl);
          const double nn = sqrt(incl);
          al = np_ / nn * ts;
          be = v / (np_ * nn) * ts;
        }
        if (live && (fl & 2)) {
          const double nrm = sqrt(incl);
          hc = 1.0 / nrm;
          sc = nrm;
        }
        // New running N = inclusive value of the last row in this chunk.
        const int last_lane = min(31, nb - base - 1);
        N = __shfl_sync(0xffffffffu, incl, last_lane);
      }
      if (live) {
        sm.alpha[rr] = al;
        sm.beta[rr] = be;
        sm.hco[rr] = hc;
        sm.wt[rr] = v;
        sm.seg[rr] = (int)sg;
        sm.flags[rr] = fl;
        if ((fl & 2) && a.scales) {
          const int64_t hi = a.head_index ? a.head_index[sg] : sg;
          a.scales[hi] = a.scale_count ? sqrt((double)a.scale_count[sg]) : sc;
        }
      }
    }
    if (w > 0) __pipeline_wait_prior(0);
    __syncwarp();
    // Column phase: each lane walks the batch rows for its columns.
    for (int rr = 0; rr < nb; ++rr) {
      const int fl = sm.flags[rr];
      const int64_t sg = sm.seg[rr];
      const double al = sm.alpha[rr];
      const double be = sm.beta[rr];
      const double vw = sm.wt[rr];
      const int64_t p = pb + rr;
      double* trow = (a.tails && !(fl & 1)) ? a.tails + (p - sg - 1) * a.ldt
                                            : nullptr;
      double* hrow = nullptr;
      if ((fl & 2) && a.heads) {
        const int64_t hi = a.head_index ? a.head_index[sg] : sg;
        hrow = a.heads + hi * a.ldh;
      }
      const double hc = sm.hco[rr];
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int c = lane + 32 * s;
        if (c < w) {
          if (fl & 1) S[s] = 0.0;
          const double x = sm.buf[rr * w + c];
          if (trow) trow[c] = x * al - S[s] * be;
          S[s] = weighted ? fma(vw, x, S[s]) : S[s] + x;
          if (hrow) hrow[c] = S[s] * hc;
        }
      }
    }
    g = sm.seg[nb - 1];
    __syncwarp();
  }
}

template <int SLOTS>
__global__ void __launch_bounds__(kWarps * 32)
    k_heads_tails(HtDev a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem* all = reinterpret_cast<WarpSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  WarpSmem& sm = all[warp];
  while (true) {
    int64_t u = 0;
    if (lane == 0) u = atomicAdd(a.ticket, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= a.n_units) break;
    process_unit<SLOTS>(a, sm, u, lane);
  }
}

// Pre-pass: per unit, the partial sums of its last group if that group is
// longer than kLight and continues into the next unit.
__global__ void k_unit_tail_sums(HtDev a, int* __restrict__ cont,
                                 double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool weighted = a.weights != nullptr;
  const int V = a.w + (weighted ? 1 : 0);
  for (int64_t u = warp; u < a.n_units; u += nw) {
    const int64_t p0 = u * kUnit;
    const int64_t p1 = min(p0 + kUnit, a.n_rows);
    const int64_t g = seg_of(a.begins, p1 - 1, 0, a.n_seg);
    const int64_t b0 = a.begins[g], b1 = a.begins[g + 1];
    const bool c = (b1 > p1) && (b1 - b0 > kLight);
    if (lane == 0) cont[u] = c ? (int)g : -1;
    if (!c) continue;
    const int64_t q0 = max(b0, p0);
    for (int cb = 0; cb < V; cb += 32) {
      const int col = cb + lane;
      double s = 0.0;
      if (col < V) {
        for (int64_t q = q0; q < p1; ++q) {
          const int64_t r = src_row(a, q);
          const double v = weighted ? a.weights[r] : 1.0;
          if (col < a.w)
            s = weighted ? fma(v, a.data[r * a.ld + col], s)
                         : s + a.data[r * a.ld + col];
          else
            s = fma(v, v, s);
        }
        val[u * (int64_t)V + col] = s;
      }
    }
  }
}

// Per long group: exclusive scan of unit partial sums over its unit chain;
// carry[u] receives the prefix of the group's rows before unit u.
__global__ void k_carry_chain(int64_t n_units, int V, const int* __restrict__ cont,
                              const double* __restrict__ val,
                              double* __restrict__ carry) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n_units; u += nw) {
    const int g = cont[u];
    if (g < 0 || (u > 0 && cont[u - 1] == g)) continue;  // not a chain start
    for (int cb = 0; cb < V; cb += 32) {
      const int col = cb + lane;
      if (col >= V) continue;
      double run = 0.0;
      int64_t x = u;
      while (x < n_units && cont[x] == g) {
        run += val[x * (int64_t)V + col];
        carry[(x + 1) * (int64_t)V + col] = run;
        ++x;
      }
    }
  }
}

// K4: joins child summaries into the node's summary rows.
__global__ void k_join(JoinArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp; k < a.G; k += nw) {
    double cs[kMaxChildren];
    int idx[kMaxChildren];
    double all = 1.0;
    for (int c = 0; c < a.n_children; ++c) {
      idx[c] = a.lidx[c][k];
      cs[c] = idx[c] >= 0 ? a.child_scale[c][idx[c]] : 0.0;
      all *= cs[c];
    }
    double* dst = a.S + k * a.width;
    const double sk = a.scale[k];
    for (int c = 0; c < a.n_children; ++c) {
      if (idx[c] < 0) continue;
      double factor = sk;
      for (int d = 0; d < a.n_children; ++d)
        if (d != c) factor *= cs[d];
      const double* src = a.child_S[c] + (int64_t)idx[c] * a.child_w[c];
      for (int j = lane; j < a.child_w[c]; j += 32)
        dst[a.child_off[c] + j] = src[j] * factor;
    }
    for (int j = lane; j < a.own_w; j += 32) dst[j] *= all;
    __syncwarp();
    if (lane == 0) a.scale[k] = sk * all;
  }
}

template <int SLOTS>
void launch_main(Context& ctx, const HtDev& d) {
  const size_t smem = sizeof(WarpSmem) * kWarps;
  static bool configured = false;
  if (!configured) {
    FG_CUDA(cudaFuncSetAttribute(k_heads_tails<SLOTS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    configured = true;
  }
  int per_sm = 0;
  FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, k_heads_tails<SLOTS>, kWarps * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)ctx.sm_count * per_sm;
  const int64_t need = ceil_div(d.n_units, kWarps);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  k_heads_tails<SLOTS><<<(int)grid, kWarps * 32, smem, ctx.stream>>>(d);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

}  // namespace

void run_heads_tails(Context& ctx, const HeadTailArgs& in) {
  if (in.n_seg == 0 || in.n_rows == 0) return;
  if (in.w > 1024) fail(FG_E_UNSUPPORTED, "heads/tails: more than 1024 columns");
  HtDev d{};
  d.data = in.data;
  d.ld = in.ld;
  d.w = in.w;
  d.perm = in.perm;
  d.begins = in.begins;
  d.n_seg = in.n_seg;
  d.n_rows = in.n_rows;
  d.weights = in.weights;
  d.tail_count = in.tail_count;
  d.scale_count = in.scale_count;
  d.head_index = in.head_index;
  d.heads = in.heads;
  d.ldh = in.ldh;
  d.tails = in.tails;
  d.ldt = in.ldt;
  d.scales = in.scales;
  d.rb = in.w > 0 ? std::max(1, std::min(kMaxRB, kSmemDoubles / in.w)) : kMaxRB;
  d.n_units = ceil_div(in.n_rows, kUnit);

  const int V = in.w + (in.weights ? 1 : 0);
  DevArray<int> cont(d.n_units, ctx.stream);
  DevArray<double> val, carry;
  DevArray<int> ticket(1, ctx.stream);
  ticket.zero();
  d.ticket = ticket.get();
  if (d.n_units > 1) {
    val.alloc(d.n_units * (size_t)V, ctx.stream);
    carry.alloc((d.n_units + 1) * (size_t)V, ctx.stream);
    const int threads = 256;
    int64_t grid = ceil_div(d.n_units * 32, threads);
    grid = std::min<int64_t>(grid, (int64_t)ctx.sm_count * 16);
    k_unit_tail_sums<<<(int)std::max<int64_t>(grid, 1), threads, 0,
                       ctx.stream>>>(d, cont.get(), val.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    k_carry_chain<<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(
        d.n_units, V, cont.get(), val.get(), carry.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    d.cont = cont.get();
    d.carry = carry.get();
  }
  const int slots = (in.w + 31) / 32;
  if (slots <= 1) launch_main<1>(ctx, d);
  else if (slots <= 2) launch_main<2>(ctx, d);
  else if (slots <= 4) launch_main<4>(ctx, d);
  else if (slots <= 8) launch_main<8>(ctx, d);
  else launch_main<32>(ctx, d);
}

void launch_join(Context& ctx, const JoinArgs& a) {
  if (a.G == 0) return;
  const int threads = 256;
  int64_t grid = ceil_div(a.G * 32, threads);
  grid = std::min<int64_t>(grid, (int64_t)ctx.sm_count * 16);
  k_join<<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(a);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

}  // namespace fg
