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
// Groups crossing a unit boundary: a short group (<= kLight rows) is
// finished by the unit it starts in (units snap to its end), so every row is
// read once.  Long groups get the prefix of their earlier rows from a
// deterministic pre-pass: per unit the partial sum of its continuing group,
// then a per-group scan over units.
// All results are run-to-run deterministic: the fused kernel assigns units
// to warps statically (unit u to warp u mod #warps), so each warp's TSQR
// accumulator absorbs the same rows in the same order on every run.
#include <cuda_pipeline.h>

#include <cub/block/block_scan.cuh>

#include <type_traits>

#include <string>

#include "launchers.cuh"
#include "tsqr_warp.cuh"

namespace fg {

namespace {

constexpr int kWarps = 8;            // warps per CTA
#ifndef FG_FUSED_WARPS
#define FG_FUSED_WARPS 8
#endif
constexpr int kFusedWarps = FG_FUSED_WARPS;  // warps per CTA of the fused kernel
constexpr int kUnit = 256;           // rows per work unit
constexpr int kLight = 256;          // groups up to this size recompute carries
#ifndef FG_HT_SMEM
#define FG_HT_SMEM 640
#endif
// Per-warp row buffer (3.75 KB): with the batch metadata 56 KB per 8-warp
// CTA, so 4 CTAs fit an SM (512 doubles: 3; C3 figaro -1.2 ms).
constexpr int kSmemDoubles = FG_HT_SMEM;
#ifndef FG_HT_MINB
#define FG_HT_MINB 3
#endif
constexpr int kMaxRB = 64;           // max rows per batch
constexpr int kVJMax = 4;            // children of a join-on-read node
constexpr int kVJRows = 32;          // max rows per batch with join-on-read

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
  const int* ufirst;     // per unit: group of its first row (or null)
  const int64_t* qb;     // per unit: its first row (n_units + 1 entries, or null)
  const double* head_mul;  // per group: heads *= head_mul[g] (or null)
  int l2hint;              // 1: L2::64B fetch hint for permuted short rows (cp_async)
  int bulk_ok;             // 1: rows contiguous and 16-byte aligned: batches by one bulk copy
  int rowbulk_ok;          // 1: rows 16-byte aligned and long enough: one bulk copy per row
  // Join-on-read (K4 folded into K5; process_and_join_children,
  // figaro.hpp:196-230): with nj >= 0 the data row x is never materialised;
  // it is [jhead[x, :own_w] * all | jS[c][jlidx[c][x]] * f_c ...] with
  // sc_c = jscale[c][jlidx[c][x]] (0 for a missing child), all = prod_c sc_c,
  // f_c = weights[x] * prod_{d != c} sc_d, and its weight is weights[x] * all
  // -- the values and product order of k_join_rows / k_join_elems.
  int nj;
  int own_w;
  const double* jhead;
  int64_t jld;
  const int* jlidx[kVJMax];
  const double* jS[kVJMax];
  const double* jscale[kVJMax];
  int jw[kVJMax];
  int joff[kVJMax];
  // Join-on-write: with wj >= 0 the head emission writes joined summary
  // rows (own head * prod s_c | child summaries * s_own * prod_{d != c} s_d)
  // of total width wwidth, and the joined scale into `scales`.
  int wj;
  int wwidth;
  const int* wlidx[kVJMax];
  const double* wS[kVJMax];
  const double* wsc[kVJMax];
  int wcw[kVJMax];
  int woff[kVJMax];
};

__device__ __forceinline__ int64_t src_row(const HtDev& a, int64_t p) {
  return a.perm ? (int64_t)a.perm[p] : p;
}

// Join-on-read factors of summary row x: f[c] for child c's columns, f[nj]
// for the own columns, idx[c] = child row (-1 missing); returns the weight.
__device__ __forceinline__ double vj_row(const HtDev& a, int64_t x, double* f, int* idx) {
  double sc[kVJMax];
  double all = 1.0;
#pragma unroll
  for (int c = 0; c < kVJMax; ++c) {
    sc[c] = 0.0;
    idx[c] = -1;
    if (c < a.nj) {
      idx[c] = a.jlidx[c][x];
      sc[c] = idx[c] >= 0 ? a.jscale[c][idx[c]] : 0.0;
      all *= sc[c];
    }
  }
  const double sk = a.weights[x];
#pragma unroll
  for (int c = 0; c < kVJMax; ++c) {
    if (c >= a.nj) break;
    double y = sk;
#pragma unroll
    for (int d = 0; d < kVJMax; ++d)
      if (d != c && d < a.nj) y *= sc[d];
    f[c] = y;
  }
  f[a.nj] = all;
  return sk * all;
}

// Which block of the joined row column `col` belongs to: child c, or nj
// for the own columns; `rel` = column within that block.
__device__ __forceinline__ int vj_span(const HtDev& a, int col, int& rel) {
  if (col < a.own_w) {
    rel = col;
    return a.nj;
  }
  int c = 0;
  while (c + 1 < a.nj && col >= a.joff[c + 1]) ++c;
  rel = col - a.joff[c];
  return c;
}

// VEC adjacent values of joined row x starting at column col (one block).
template <int VEC>
__device__ __forceinline__ void vj_load(const HtDev& a, int64_t x, int col, double* out,
                                        double& wgt) {
  double f[kVJMax + 1];
  int idx[kVJMax];
  wgt = vj_row(a, x, f, idx);
  int rel = 0;
  const int c = vj_span(a, col, rel);
  const double* src = nullptr;
  if (c == a.nj) src = a.jhead + x * a.jld + rel;
  else if (idx[c] >= 0) src = a.jS[c] + (int64_t)idx[c] * a.jw[c] + rel;
#pragma unroll
  for (int e = 0; e < VEC; ++e) out[e] = src ? src[e] * f[c] : 0.0;
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

struct NoFuse {};

// Row-groups work on contiguous chunks of a batch at the same time; with
// power-of-two chunk strides their shared-memory reads fall on the same banks
// (ncu on C3's width-8 own pass: 387 M of 835 M shared wavefronts were bank
// conflicts).  The unfused kernels therefore index row metadata by
// rr + rr / chunk (one padding entry per chunk) and shift the staged rows of
// chunk g by g * px rows; kPadRows covers up to 8 row-groups (widths >= 8).
constexpr int kPadRows = 8;
template <int CAP, int VJR = 1, int PAD = 0>
struct WarpSmemT {
  static constexpr int kPad = PAD;
  double buf[CAP];
  double2 coef[kMaxRB + PAD];   // {alpha, beta}: tail = a*alpha - S*beta
  double hco[kMaxRB + PAD];     // head coefficient at a group's last row
  double wt[kMaxRB + PAD];      // generalized weights (plain: the group's scale)
  int2 segfl[kMaxRB + PAD];     // {group, flags}: bit0 start, bit1 last
  unsigned char startf[kMaxRB];  // 1 where a group starts inside the batch
  const double* rowptr[kMaxRB + PAD];  // staging: source row; afterwards: the row's tail slot (or null)
  double* hrowp[kMaxRB + PAD];         // head row of a group's last row (or null)
  unsigned long long bar;              // mbarrier of the bulk-copied batches
  double vjf[VJR][kVJMax + 1];   // join-on-read factors per staged row
  int vjidx[VJR][kVJMax];        // join-on-read child rows per staged row
};
using WarpSmem = WarpSmemT<kSmemDoubles, 1, kPadRows>;
using WarpSmemVJ = WarpSmemT<kSmemDoubles, kVJRows>;
constexpr int kFusedDoubles = 1280;  // one TSQR tile of tails (B x ls)

__device__ __forceinline__ double fast_rsqrt_d(double q) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  const double hq = 0.5 * q;
  r = r * fma(-hq * r, r, 1.5);
  r = r * fma(-hq * r, r, 1.5);
  return r;
}

// sqrt(q) for q >= 0 finite: q * rsqrt(q) plus one correction step (exact
// for perfect squares up to 2^52, <= 1 ulp otherwise); 0 for q = 0.
__device__ __forceinline__ double fast_sqrt_d(double q) {
  if (!(q > 1e-250 && q < 1e250)) return sqrt(q);
  const double r = fast_rsqrt_d(q);
  const double s0 = q * r;
  return fma(0.5 * r, fma(-s0, s0, q), s0);
}

// Lane geometry: the warp is split into G row-groups of L lanes; lane cl of
// a group owns column packets cl + L*s (s < SLOTS) of VEC doubles each.
// ls: row stride of the staged batch in shared memory (doubles).
struct Geo {
  int vec, np, L, G, ls;
};

// Compile-time geometry of the hot unfused shapes (width CW, double2
// packets, row-groups of exactly CW/2 lanes): the index arithmetic of the
// batch loops folds into constants.  kW = 0 marks the run-time Geo.
template <int CW>
struct GeoC {
  static constexpr int kW = CW;
  static constexpr int vec = 2, np = CW / 2, L = CW / 2, G = 32 / (CW / 2), ls = CW;
};
template <class GEO> struct GeoW { static constexpr int value = GEO::kW; };
template <> struct GeoW<Geo> { static constexpr int value = 0; };

// Asynchronous copy of one packet into shared memory with the L2::64B
// fetch hint: without it a miss fills the whole 128-byte line, so gathering
// 64-byte rows through the sort permutation reads every row twice from HBM
// (scripts/gather_probe.cu: 6.53 GB vs 3.41 GB of DRAM reads for 3.2 GB of
// rows).  Only for permuted rows shorter than a line (`narrow`): on
// contiguous or long rows the hint costs the line's second half a second
// request (measured: C3 project-away and C5 own rows slower with it).
template <int VEC>
__device__ __forceinline__ void cp_async(double* dst, const double* src, bool narrow = false) {
  if (narrow) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if (VEC == 2)
      asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(d), "l"(src));
    else
      asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], 8;" ::"r"(d), "l"(src));
  } else {
    __pipeline_memcpy_async(dst, src, VEC * sizeof(double));
  }
}

// mbarrier + 1-D bulk copy (TMA engine, no tensor map) for batches whose rows
// are contiguous in memory (project-away in identity order): one lane issues
// one copy for the whole batch instead of every lane issuing LDGSTS packets,
// which takes the staging off the LSU data pipe (18 % of its wavefronts on
// C3's project-away, which runs that pipe at 86 %).
__device__ __forceinline__ uint32_t ht_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ht_mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ht_smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void ht_bulk_g2s(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
  // earlier generic-proxy reads of the buffer are ordered before the async write
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ht_smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(ht_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(ht_smem_u32(bar))
      : "memory");
}
// The same in two steps, for batches copied row by row: one lane announces
// the batch's bytes, every lane copies the rows it owns.
__device__ __forceinline__ void ht_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ht_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ht_bulk_row(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(ht_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(ht_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ht_mbar_wait(unsigned long long* bar, unsigned phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(ht_smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

// Copies rows [p, p+nb) of the sorted order (w doubles each) into buf.
// pv (KP > 0): the batch's permutation entries, row lane + 32 k in pv[k],
// loaded one batch ahead by the caller so the row gathers do not wait on a
// dependent index load.
// ch > 0: padded indexing (see kPadRows) with chunks of ch rows and a row
// shift of px per chunk; ch = 0: plain indexing.
template <int SLOTS, int VEC, bool VJ, class SM, class GEO, int KP = 0>
__device__ __forceinline__ void stage_rows(const HtDev& a, const GEO& geo,
                                           SM& sm, int64_t p, int nb,
                                           int lane, const int* pv = nullptr,
                                           int ch = 0, int px = 0, int bulk = 0) {
  if constexpr (VJ) {
    // Join-on-read: own head columns and child summary rows are copied into
    // the row buffer; the row factors are applied when the buffer is read.
    for (int rr = lane; rr < nb; rr += 32) {
      const int64_t x = src_row(a, p + rr);
      sm.wt[rr] = vj_row(a, x, sm.vjf[rr], sm.vjidx[rr]);
      sm.rowptr[rr] = a.jhead + x * a.jld;
    }
    __syncwarp();
    const int g = lane / geo.L, cl = lane % geo.L;
    for (int rr = g < geo.G ? g : nb; rr < nb; rr += geo.G) {
      double* dst = sm.buf + rr * geo.ls;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int pk = cl + geo.L * s;
        if (pk >= geo.np) continue;
        int rel = 0;
        const int c = vj_span(a, VEC * pk, rel);
        if (c == a.nj) {
          cp_async<VEC>(dst + VEC * pk, sm.rowptr[rr] + rel);
        } else {
          const int idx = sm.vjidx[rr][c];
          if (idx >= 0) {
            cp_async<VEC>(dst + VEC * pk, a.jS[c] + (int64_t)idx * a.jw[c] + rel);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) dst[VEC * pk + e] = 0.0;
          }
        }
      }
    }
    __pipeline_commit();
    return;
  }
  if (bulk == 2) {
    // one bulk copy per row, issued by the lane that owns the row
    if (lane == 0) ht_expect_tx(&sm.bar, (unsigned)(nb * a.w * sizeof(double)));
    const unsigned rbytes = (unsigned)(a.w * sizeof(double));
    auto row_copy = [&](int rr, int64_t x) {
      const int gq = ch ? rr / ch : 0;
      ht_bulk_row(sm.buf + (rr + gq * px) * geo.ls, a.data + x * a.ld, rbytes, &sm.bar);
      if (a.weights) sm.wt[rr + gq] = a.weights[x];
    };
    if constexpr (KP > 0) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int rr = lane + 32 * k;
        if (rr < nb) row_copy(rr, a.perm ? (int64_t)pv[k] : p + rr);
      }
    } else {
      for (int rr = lane; rr < nb; rr += 32) row_copy(rr, src_row(a, p + rr));
    }
    __syncwarp();
    return;
  }
  if (bulk == 1) {
    // contiguous rows (identity order, ld == w, px == 0): one bulk copy
    if (lane == 0)
      ht_bulk_g2s(sm.buf, a.data + p * a.ld, (unsigned)(nb * a.w * sizeof(double)), &sm.bar);
    if (a.weights) {
      for (int rr = lane; rr < nb; rr += 32) sm.wt[ch ? rr + rr / ch : rr] = a.weights[p + rr];
    }
    __syncwarp();
    return;
  }
  if constexpr (KP > 0) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int rr = lane + 32 * k;
      if (rr < nb) {
        const int64_t x = a.perm ? (int64_t)pv[k] : p + rr;
        const int m = ch ? rr + rr / ch : rr;
        sm.rowptr[m] = a.data + x * a.ld;
        if (a.weights) sm.wt[m] = a.weights[x];
      }
    }
  } else {
    for (int rr = lane; rr < nb; rr += 32) {
      const int64_t x = src_row(a, p + rr);
      const int m = ch ? rr + rr / ch : rr;
      sm.rowptr[m] = a.data + x * a.ld;
      if (a.weights) sm.wt[m] = a.weights[x];
    }
  }
  __syncwarp();
  const int g = lane / geo.L, cl = lane % geo.L;
  const bool narrow = a.perm != nullptr && a.w < 16 && a.l2hint;
  if (ch) {
    // each row-group copies its own chunk (the rows it will scan)
    const int r_lo = min(nb, g * ch), r_hi = g < geo.G ? min(nb, r_lo + ch) : r_lo;
    for (int rr = r_lo; rr < r_hi; ++rr) {
      const double* src = sm.rowptr[rr + g];
      double* dst = sm.buf + (rr + g * px) * geo.ls;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int pk = cl + geo.L * s;
        if (pk < geo.np) cp_async<VEC>(dst + VEC * pk, src + VEC * pk, narrow);
      }
    }
  } else {
    for (int rr = g < geo.G ? g : nb; rr < nb; rr += geo.G) {
      const double* src = sm.rowptr[rr];
      double* dst = sm.buf + rr * geo.ls;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int pk = cl + geo.L * s;
        if (pk < geo.np) cp_async<VEC>(dst + VEC * pk, src + VEC * pk, narrow);
      }
    }
  }
  __pipeline_commit();
}

// F = NoFuse: tails are written to a.tails.  F = WCfg<...>: each batch of
// tails is written in place into the staged rows (group starts become zero
// rows) and absorbed into the warp's TSQR accumulator Racc.
template <int SLOTS, int VEC, class F, bool VJ, class SM, class RA, bool JW = false,
          class GEO = Geo>
__device__ void process_unit(const HtDev& a, const GEO& geo, SM& sm,
                             int64_t u, int lane, RA& Racc, unsigned& bphase) {
  constexpr bool FUSED = !std::is_same<F, NoFuse>::value;
  constexpr int CW = GeoW<GEO>::value;
  const int w = CW ? CW : a.w;
  const bool weighted = a.weights != nullptr;
  const int64_t p0 = u * kUnit;
  // Short groups (<= kLight rows) are never split: the unit a short group
  // starts in finishes it (k_unit_cont moves the next unit's first row,
  // qb[u + 1], to the group's end), so every row is read once.  Long groups
  // keep the unit boundaries and take their prefix from the deterministic
  // pre-pass (chained carries).
  const int64_t q0 = a.qb ? a.qb[u] : p0;
  const int64_t q1 = a.qb ? a.qb[u + 1] : min(p0 + kUnit, a.n_rows);
  int64_t g = a.ufirst ? (int64_t)a.ufirst[u] : seg_of(a.begins, p0, 0, a.n_seg);
  const int grp = lane / geo.L, cl = lane % geo.L;
  // Join-on-read: the block (child or own) of each owned column packet.
  int cs[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    int rel = 0;
    cs[s] = VJ ? vj_span(a, VEC * (cl + geo.L * s), rel) : 0;
  }

  // Running prefix (per owned column) carried into the next batch.
  double S[SLOTS][VEC];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int e = 0; e < VEC; ++e) S[s][e] = 0.0;
  double N = 0.0;  // weighted: running sum of squared weights (lane-uniform)

  const int64_t gb = a.begins[g];
  if (gb < q0) {
    // A long group started in an earlier unit: its prefix from the pre-pass.
    const bool chained = u > 0 && a.cont && a.cont[u - 1] == (int)g;
    const int V = w + (weighted ? 1 : 0);
    const double* cr = chained ? a.carry + u * (int64_t)V : nullptr;
    if (chained && weighted) N = cr[w];
    if (chained) {
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int pk = cl + geo.L * s;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int col = VEC * pk + e;
          if (pk < geo.np && col < w) S[s][e] = cr[col];
        }
      }
    }
  }

  // Rows per batch: a compile-time constant for the specialised shapes (the
  // host computes the same value, prepare()); KS = 32-entry slices of the
  // per-group registers (begins / tail scales / head factors) a batch needs.
  constexpr int kRbC = CW ? ((kMaxRB < kSmemDoubles / (CW ? CW : 1) ? kMaxRB : kSmemDoubles / (CW ? CW : 1)) /
                             (CW ? 32 / (CW / 2) : 1)) * (CW ? 32 / (CW / 2) : 1)
                          : 0;
  constexpr int KS = (CW && !FUSED) ? (kRbC + 1) / 32 + 1 : 3;
  const int rbv = (CW && !FUSED) ? kRbC : a.rb;
  // Permutation entries of the next batch, loaded one batch ahead.
  constexpr int KP = (CW && !FUSED && !VJ) ? (kRbC + 31) / 32 : 0;
  int pnext[KP > 0 ? KP : 1];
  if constexpr (KP > 0) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int64_t pr = q0 + lane + 32 * k;
      pnext[k] = (a.perm && pr < q1) ? a.perm[pr] : 0;
    }
  }
  for (int64_t pb = q0; pb < q1; pb += rbv) {
    const int nb = (int)(q1 - pb < (int64_t)rbv ? q1 - pb : (int64_t)rbv);
    int pcur[KP > 0 ? KP : 1];
    if constexpr (KP > 0) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        pcur[k] = pnext[k];
        const int64_t pr = pb + rbv + lane + 32 * k;
        pnext[k] = (a.perm && lane + 32 * k < rbv && pr < q1) ? a.perm[pr] : 0;
      }
    }
    // The batch's rows lie in groups g .. g+nb: their offsets begins[g ..
    // g+nb+1] and tail scales sqrt(tail_count[g .. g+nb]) are loaded now,
    // three per lane in registers, so their latency overlaps the row
    // gathers below instead of following them (read back by shuffles).
    // (The counts stay raw here: converting them now would make the warp
    // wait for these loads before it has issued the row gathers -- 44 % of
    // the stall samples of C3's own pass; the square root is taken per row
    // in the metadata pass.)
    int bgv[KS];
    unsigned long long tcv[KS];
    double hmv[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int i = lane + 32 * k;
      const int64_t gi = g + i;
      bgv[k] = (i <= nb + 1 && gi <= a.n_seg) ? a.begins[gi] : INT_MAX;
      tcv[k] = (a.tail_count && i <= nb && gi < a.n_seg) ? a.tail_count[gi] : 1ull;
      hmv[k] = (a.head_mul && i <= nb && gi < a.n_seg) ? a.head_mul[gi] : 1.0;
    }
    // Chunk of rows per row-group, and the padded indexing of the unfused
    // kernels (kPadRows): metadata of row rr at rr + rr / ch, its staged data
    // px rows further per chunk when the chunk stride would alias the banks.
    const int ch = (nb + geo.G - 1) / geo.G;
    const bool padded = !FUSED && !VJ && SM::kPad > 0 && geo.G > 1 && geo.G <= SM::kPad;
    const int cap_rows = w > 0 ? kSmemDoubles / w : 0;
    const int px = (padded && geo.L < 8 && (ch * w * 8) % 128 == 0 && nb + geo.G <= cap_rows) ? 1 : 0;
    auto mi = [&](int rr) { return padded ? rr + rr / ch : rr; };
    const int bulk = (FUSED || VJ || w <= 0) ? 0
                     : (a.bulk_ok && px == 0)   ? 1
                     : a.rowbulk_ok             ? 2
                                                : 0;
    if (w > 0)
      stage_rows<SLOTS, VEC, VJ, SM, GEO, KP>(a, geo, sm, pb, nb, lane, pcur, padded ? ch : 0, px,
                                              bulk);
    else if (VJ) __syncwarp();
    // Group starts inside the batch (groups g+1 .. g+nb can start here):
    // flagged in shared memory, then each row's group is g plus a ballot
    // prefix count.
    for (int i = lane; i < (CW && !FUSED ? kRbC : kMaxRB); i += 32) sm.startf[i] = 0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int i = lane + 32 * k - 1;  // group g + 1 + i starts at bgv[k]
      if (i >= 0 && i < nb && g + 1 + i < a.n_seg) {
        const int64_t b = bgv[k];
        if (b < pb + nb) sm.startf[b - pb] = 1;
      }
    }
    __syncwarp();
    // begins[g + i] and the tail scale of group g + i from the registers.
    auto bg_at = [&](int i) -> int64_t {
      int v = __shfl_sync(0xffffffffu, bgv[0], i & 31);
#pragma unroll
      for (int k = 1; k < KS; ++k) {
        const int vk = __shfl_sync(0xffffffffu, bgv[k], i & 31);
        if ((i >> 5) == k) v = vk;
      }
      return v;
    };
    auto ts_at = [&](int i) -> double {
      unsigned long long v = __shfl_sync(0xffffffffu, tcv[0], i & 31);
#pragma unroll
      for (int k = 1; k < KS; ++k) {
        const unsigned long long vk = __shfl_sync(0xffffffffu, tcv[k], i & 31);
        if ((i >> 5) == k) v = vk;
      }
      return fast_sqrt_d((double)v);  // exact for perfect squares
    };
    auto hm_at = [&](int i) -> double {
      double v = __shfl_sync(0xffffffffu, hmv[0], i & 31);
#pragma unroll
      for (int k = 1; k < KS; ++k) {
        const double vk = __shfl_sync(0xffffffffu, hmv[k], i & 31);
        if ((i >> 5) == k) v = vk;
      }
      return v;
    };
    int64_t gcur = g;
    // Row metadata and coefficients, one row per lane.
    for (int base = 0; base < nb; base += 32) {
      const int rr = base + lane;
      const bool live = rr < nb;
      const unsigned smask = __ballot_sync(0xffffffffu, live && sm.startf[rr]);
      int64_t sg = gcur + __popc(smask & ((2u << lane) - 1u));
      gcur += __popc(smask);
      int64_t jj = 0, m = 1;
      double v = 1.0;
      int fl = 0;
      const int li = live ? (int)(sg - g) : 0;  // <= nb
      const int64_t b0 = bg_at(li);
      const int64_t b1 = bg_at(li + 1);
      const double tsr = ts_at(li);
      const double hmr = a.head_mul ? hm_at(li) : 1.0;
      if (live) {
        const int64_t p = pb + rr;
        jj = p - b0;
        m = b1 - b0;
        fl = (jj == 0 ? 1 : 0) | (p == b1 - 1 ? 2 : 0);
        if (VJ || (weighted && w > 0)) v = sm.wt[mi(rr)];  // staged with the row (stage_rows)
        else if (weighted) v = a.weights[src_row(a, p)];
      }
      double ts = 1.0;
      if (live && a.tail_count) ts = tsr;  // sqrt is exact for squares
      double al = 0.0, be = 0.0, hc = 0.0, sc = 0.0;
      if (!weighted) {
        if (live && jj >= 1) {
          // sqrt(j)/sqrt(j+1) and 1/(sqrt(j) sqrt(j+1)) from one rsqrt.
          const double q = (double)jj * (double)(jj + 1);
          const double rq = fast_rsqrt_d(q);
          al = (double)jj * rq * ts;
          be = ts * rq;
        }
        if (live && (fl & 2)) {
          const double rm = fast_rsqrt_d((double)m);
          hc = rm;
          sc = (double)m * rm;
        }
      } else {
        // Segmented inclusive scan of v^2 over the 32 rows of this chunk.
        double x = live ? v * v : 0.0;
        int st = live ? (fl & 1) : 0;
        if (lane == 0 && !st) x += N;  // carry unless the row starts a group
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
        // sqrt(excl)/sqrt(incl) and 1/(sqrt(excl) sqrt(incl)) from one
        // rsqrt of the product (MUFU + two Newton steps, ~1e-16) inside a
        // range where neither the product nor the .ftz approximation can
        // flush; the IEEE sqrt/div sequences (about 6 x 35 instructions per
        // row) only outside it.
        const double pq = excl * incl;
        const bool fast = pq > 1e-250 && pq < 1e250 && incl > 1e-250 && incl < 1e250;
        if (live && jj >= 1) {
          if (fast) {
            const double rq = fast_rsqrt_d(pq);
            al = excl * rq * ts;
            be = v * rq * ts;
          } else {
            const double np_ = sqrt(excl);
            const double nn = sqrt(incl);
            al = np_ / nn * ts;
            be = v / (np_ * nn) * ts;
          }
        }
        if (live && (fl & 2)) {
          if (incl > 1e-250 && incl < 1e250) {
            hc = fast_rsqrt_d(incl);
            sc = incl * hc;
          } else {
            const double nrm = sqrt(incl);
            hc = 1.0 / nrm;
            sc = nrm;
          }
        }
        const int last_lane = min(31, nb - base - 1);
        N = __shfl_sync(0xffffffffu, incl, last_lane);
      }
      if (live) {
        const int mx = mi(rr);
        sm.coef[mx] = make_double2(al, be);
        // head_mul: the join's own-column factor prod_c s_c folded into the
        // head coefficient (figaro.hpp:226, `dst[j] *= all`)
        sm.hco[mx] = hc * hmr;
        sm.wt[mx] = weighted ? v : sc;  // plain rows never read their weight
        sm.segfl[mx] = make_int2((int)sg, fl);
        // Output rows of the emission pass, computed once per row here
        // instead of once per lane there (64-bit index arithmetic).
        const int64_t p = pb + rr;
        sm.rowptr[mx] = (a.tails && !(fl & 1)) ? a.tails + (p - sg - 1) * a.ldt : nullptr;
        double* hp = nullptr;
        if (fl & 2) {
          const int64_t hi = a.head_index ? a.head_index[sg] : sg;
          if (a.heads) hp = a.heads + hi * a.ldh;
          if (a.scales && a.wj < 0)
            a.scales[hi] = a.scale_count ? sqrt((double)a.scale_count[sg]) : sc;
        }
        sm.hrowp[mx] = hp;
      }
    }
    if (bulk) {
      ht_mbar_wait(&sm.bar, bphase);
      bphase ^= 1u;
    } else if (w > 0) {
      __pipeline_wait_prior(0);
    }
    __syncwarp();
    if (w > 0) {
      // Rows of this batch are split into G contiguous chunks, one per
      // row-group.  Pass 1: chunk-local sums since the last group start.
      const int r_lo = min(nb, grp * ch), r_hi = min(nb, r_lo + ch);
      // this row-group's offsets into the metadata arrays / the staged rows
      const int mo = padded ? grp : 0, xo = grp * px;
      double loc[SLOTS][VEC];
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
#pragma unroll
        for (int e = 0; e < VEC; ++e) loc[s][e] = 0.0;
      int has_start = 0;
      for (int rr = r_lo; rr < r_hi; ++rr) {
        const int fl = sm.segfl[rr + mo].y;
        const double vw = sm.wt[rr + mo];
        if (fl & 1) has_start = 1;
        const double* row = sm.buf + (rr + xo) * geo.ls;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
          const int pk = cl + geo.L * s;
          if (pk >= geo.np) continue;
          double x[VEC];
          if (VEC == 2) {
            const double2 t = *reinterpret_cast<const double2*>(row + 2 * pk);
            x[0] = t.x;
            x[VEC - 1] = t.y;
          } else {
            x[0] = row[pk];
          }
          if (VJ) {
            const double fc = sm.vjf[rr][cs[s]];
#pragma unroll
            for (int e = 0; e < VEC; ++e) x[e] *= fc;
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const double base_ = (fl & 1) ? 0.0 : loc[s][e];
            loc[s][e] = weighted ? fma(vw, x[e], base_) : base_ + x[e];
          }
        }
      }
      // Pass 2: segmented scan of the chunk sums across the G groups,
      // seeded with the batch carry S.
      int f = has_start;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (grp == 0 && !f) loc[s][e] += S[s][e];
      for (int o = 1; o < geo.G; o <<= 1) {
        const int fy = __shfl_up_sync(0xffffffffu, f, o * geo.L);
#pragma unroll
        for (int s = 0; s < SLOTS; ++s)
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const double y = __shfl_up_sync(0xffffffffu, loc[s][e], o * geo.L);
            if (grp >= o && !f) loc[s][e] += y;
          }
        if (grp >= o) f |= fy;
      }
      double run[SLOTS][VEC];
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const double ex = __shfl_up_sync(0xffffffffu, loc[s][e], geo.L);
          run[s][e] = grp == 0 ? S[s][e] : ex;
          S[s][e] = __shfl_sync(0xffffffffu, loc[s][e], (geo.G - 1) * geo.L + cl);
        }
      // Pass 3: emit tails (and heads at group ends) for this chunk.
      for (int rr = r_lo; rr < r_hi; ++rr) {
        const int2 sf = sm.segfl[rr + mo];
        const double2 cf = sm.coef[rr + mo];
        const double vw = sm.wt[rr + mo];
        double* trow = const_cast<double*>(sm.rowptr[rr + mo]);
        double* hrow = sm.hrowp[rr + mo];
        const double hc = hrow ? sm.hco[rr + mo] : 0.0;
        const double* row = sm.buf + (rr + xo) * geo.ls;
        // Join-on-write factors of this group (process_and_join_children,
        // figaro.hpp:196-230, in its product order).
        double jsc[kVJMax];
        int jidx[kVJMax];
        double jall = 1.0;
        const bool jwrite = JW && !FUSED && hrow && a.wj >= 0;
        if (jwrite) {
#pragma unroll
          for (int c = 0; c < kVJMax; ++c) {
            jsc[c] = 0.0;
            jidx[c] = -1;
            if (c < a.wj) {
              jidx[c] = a.wlidx[c][sf.x];
              jsc[c] = jidx[c] >= 0 ? a.wsc[c][jidx[c]] : 0.0;
              jall *= jsc[c];
            }
          }
        }
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
          const int pk = cl + geo.L * s;
          if (pk >= geo.np) continue;
          double x[VEC], o[VEC];
          if (VEC == 2) {
            const double2 t = *reinterpret_cast<const double2*>(row + 2 * pk);
            x[0] = t.x;
            x[VEC - 1] = t.y;
          } else {
            x[0] = row[pk];
          }
          if (VJ) {
            const double fc = sm.vjf[rr][cs[s]];
#pragma unroll
            for (int e = 0; e < VEC; ++e) x[e] *= fc;
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            if (sf.y & 1) run[s][e] = 0.0;
            o[e] = x[e] * cf.x - run[s][e] * cf.y;
            run[s][e] = weighted ? fma(vw, x[e], run[s][e]) : run[s][e] + x[e];
          }
          if constexpr (FUSED) {
            double* slot = const_cast<double*>(row) + VEC * pk;
            if (VEC == 2)
              *reinterpret_cast<double2*>(slot) = (sf.y & 1) ? make_double2(0.0, 0.0)
                                                             : make_double2(o[0], o[VEC - 1]);
            else
              slot[0] = (sf.y & 1) ? 0.0 : o[0];
          } else if (trow) {
            if (VEC == 2)
              *reinterpret_cast<double2*>(trow + 2 * pk) = make_double2(o[0], o[VEC - 1]);
            else
              trow[pk] = o[0];
          }
          if (hrow) {
            if (jwrite) {
#pragma unroll
              for (int e = 0; e < VEC; ++e) hrow[VEC * pk + e] = (run[s][e] * hc) * jall;
            } else if (VEC == 2) {
              // one 16-byte store (prepare() checks the alignment of heads / ldh)
              *reinterpret_cast<double2*>(hrow + 2 * pk) =
                  make_double2(run[s][0] * hc, run[s][VEC - 1] * hc);
            } else {
              hrow[pk] = run[s][0] * hc;
            }
          }
        }
        if (jwrite) {
          // The children's summary columns of the joined row, and its scale.
          const double sk = sm.wt[rr + mo];  // plain transform: the group's scale
          for (int col = w + cl; col < a.wwidth; col += geo.L) {
            int c = 0;
            while (c + 1 < a.wj && col >= a.woff[c + 1]) ++c;
            double f = sk;
#pragma unroll
            for (int d = 0; d < kVJMax; ++d)
              if (d != c && d < a.wj) f *= jsc[d];
            hrow[col] = jidx[c] >= 0
                            ? a.wS[c][(int64_t)jidx[c] * a.wcw[c] + (col - a.woff[c])] * f
                            : 0.0;
          }
          if (cl == 0 && a.scales) {
            const int64_t hi = a.head_index ? a.head_index[sf.x] : sf.x;
            a.scales[hi] = sk * jall;
          }
        }
      }
    }
    if constexpr (FUSED) {
      if (w > 0) {
        // The batch (nb <= B rows of tails, zero rows at group starts) is
        // one TSQR tile for this warp's accumulator.
        __syncwarp();
        const int r = lane % F::TR, c = lane / F::TR;
        int cols[F::CPT];
        double X[F::RPT][F::CPT];
#pragma unroll
        for (int q = 0; q < F::CPT; ++q) cols[q] = wcol<F>(q, c);
#pragma unroll
        for (int i = 0; i < F::RPT; ++i) {
          const int rr = i * F::TR + r;
#pragma unroll
          for (int q = 0; q < F::CPT; ++q)
            X[i][q] = (rr < nb && cols[q] < w) ? sm.buf[rr * geo.ls + cols[q]] : 0.0;
        }
        absorb_tile<F>(X, Racc, r, c, cols);
      }
    }
    g = sm.segfl[mi(nb - 1)].x;
    __syncwarp();
  }
}

template <int SLOTS, int VEC, bool VJ, bool JW = false, int CW = 0>
__global__ void __launch_bounds__(kWarps * 32, (VJ || JW || SLOTS > 1) ? 1 : FG_HT_MINB)
    k_heads_tails(HtDev a, Geo geo) {
  using SMT = std::conditional_t<VJ, WarpSmemVJ, WarpSmem>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SMT* all = reinterpret_cast<SMT*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  SMT& sm = all[warp];
  int dummy = 0;
  unsigned bphase = 0;
  if (lane == 0) ht_mbar_init(&sm.bar);
  __syncwarp();
  while (true) {
    int64_t u = 0;
    if (lane == 0) u = atomicAdd(a.ticket, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= a.n_units) break;
    if constexpr (CW > 0) {
      const GeoC<CW> gc{};
      process_unit<SLOTS, VEC, NoFuse, VJ, SMT, int, JW, GeoC<CW>>(a, gc, sm, u, lane, dummy, bphase);
    } else {
      process_unit<SLOTS, VEC, NoFuse, VJ, SMT, int, JW>(a, geo, sm, u, lane, dummy, bphase);
    }
  }
}

// Fused K3 -> K6: heads/tails of own groups with the tails absorbed by a
// per-warp Householder accumulator (never written to HBM).  Writes one
// F::W x F::W partial factor per warp to `partials`.
template <int VEC, class F>
__global__ void __launch_bounds__(kFusedWarps * 32, F::MINB)
    k_heads_tails_tsqr(HtDev a, Geo geo, double* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SM = WarpSmemT<kFusedDoubles>;
  SM* all = reinterpret_cast<SM*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  SM& sm = all[warp];
  double Racc[F::RR][F::CPT];
#pragma unroll
  for (int m = 0; m < F::RR; ++m)
#pragma unroll
    for (int q = 0; q < F::CPT; ++q) Racc[m][q] = 0.0;
  // Static unit -> warp assignment: which rows each accumulator absorbs
  // (and so the rounding of R) depends only on the grid, not on timing.
  unsigned bphase_unused = 0;
  const int64_t nw = (int64_t)gridDim.x * kFusedWarps;
  for (int64_t u = (int64_t)blockIdx.x * kFusedWarps + warp; u < a.n_units; u += nw)
    process_unit<1, VEC, F, false>(a, geo, sm, u, lane, Racc, bphase_unused);
  const int r = lane % F::TR, c = lane / F::TR;
  double* o = partials + ((int64_t)blockIdx.x * kFusedWarps + warp) * F::W * F::W;
#pragma unroll
  for (int m = 0; m < F::RR; ++m)
#pragma unroll
    for (int q = 0; q < F::CPT; ++q)
      if (m * F::TR + r < F::W) o[(m * F::TR + r) * F::W + wcol<F>(q, c)] = Racc[m][q];
}

// Pre-pass part 1: per unit (one thread each), does its last group continue
// into the next unit and is it longer than kLight?  Sets *any if so.
// Also the unit starts: a short group crossing p1 stays with unit u, so
// unit u + 1 starts at its end (qb[u + 1], with ufirst[u + 1] its group).
__global__ void k_unit_cont(HtDev a, int* __restrict__ cont, int* __restrict__ ufirst,
                            int64_t* __restrict__ qb, int* any) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < a.n_units;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = u * kUnit;
    const int64_t p1 = min(p0 + kUnit, a.n_rows);
    const int64_t g = seg_of(a.begins, p1 - 1, 0, a.n_seg);
    const int64_t b0 = a.begins[g], b1 = a.begins[g + 1];
    const bool crosses = b1 > p1;
    const bool c = crosses && (b1 - b0 > kLight);
    cont[u] = c ? (int)g : -1;
    if (c) *any = 1;
    if (u + 1 < a.n_units) {
      // long crossing group: unit u + 1 continues it at p1; otherwise the next
      // unit starts with group g + 1 at p1 or (short crossing group) at b1.
      ufirst[u + 1] = (int)(c ? g : g + 1);
      qb[u + 1] = (crosses && !c) ? b1 : p1;
    } else {
      qb[u + 1] = a.n_rows;
    }
    if (u == 0) {
      ufirst[0] = 0;
      qb[0] = 0;
    }
  }
}

// Pre-pass: per unit, the partial sums of its last group if that group is
// longer than kLight and continues into the next unit.  The warp splits into
// G row-groups of L lanes (L >= column packets of VEC doubles, as in the main
// kernel); group grp sums rows q0+grp, q0+grp+G, ... and the G partial sums
// are combined by a fixed xor-shuffle tree (deterministic).
template <int VEC>
__global__ void k_unit_tail_sums(HtDev a, int* __restrict__ cont,
                                 double* __restrict__ val, Geo geo) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool weighted = a.weights != nullptr;
  const int V = a.w + (weighted ? 1 : 0);
  const int np = geo.np;
  const int grp = lane / geo.L, cl = lane % geo.L;
  for (int64_t u = warp; u < a.n_units; u += nw) {
    const int64_t p0 = u * kUnit;
    const int64_t p1 = min(p0 + kUnit, a.n_rows);
    const int g = cont[u];
    if (g < 0) continue;
    const int64_t q0 = max((int64_t)a.begins[g], p0);
    for (int pb = 0; pb < max(np, 1); pb += geo.L) {
      const int pk = pb + cl;
      double s[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) s[e] = 0.0;
      double nacc = 0.0;
#pragma unroll 4
      for (int64_t p = q0 + grp; p < p1; p += geo.G) {
        const int64_t r = src_row(a, p);
        if (a.nj >= 0) {
          double x[VEC], v = 1.0;
          if (pk < np) {
            vj_load<VEC>(a, r, VEC * pk, x, v);
#pragma unroll
            for (int e = 0; e < VEC; ++e) s[e] = fma(v, x[e], s[e]);
          } else {
            double f[kVJMax + 1];
            int idx[kVJMax];
            v = vj_row(a, r, f, idx);
          }
          nacc = fma(v, v, nacc);
          continue;
        }
        const double v = weighted ? a.weights[r] : 1.0;
        if (pk < np) {
          const double* src = a.data + r * a.ld + VEC * pk;
          if (VEC == 2) {
            const double2 x = *reinterpret_cast<const double2*>(src);
            s[0] = weighted ? fma(v, x.x, s[0]) : s[0] + x.x;
            s[VEC - 1] = weighted ? fma(v, x.y, s[VEC - 1]) : s[VEC - 1] + x.y;
          } else {
            s[0] = weighted ? fma(v, src[0], s[0]) : s[0] + src[0];
          }
        }
        nacc = fma(v, v, nacc);
      }
      for (int o = geo.L; o < 32; o <<= 1) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) s[e] += __shfl_xor_sync(0xffffffffu, s[e], o);
        nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
      }
      if (grp == 0 && pk < np)
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (VEC * pk + e < a.w) val[u * (int64_t)V + VEC * pk + e] = s[e];
      if (weighted && pb == 0 && lane == 0) val[u * (int64_t)V + a.w] = nacc;
    }
  }
}

// Carries of long groups: carry[u+1] = sum of val[u'] over the units u' of
// u's chain (maximal run of equal cont >= 0) up to and including u.  A
// deterministic three-level segmented scan over units (fixed association):
//   k_chain_local: per block of kChainBlk units, per column, the in-block
//                  inclusive run sums (written to carry[u+1]) and the block's
//                  trailing run sum;
//   k_chain_top:   segmented scan over blocks: the carry entering each block;
//   k_chain_fix:   adds the entering carry to units whose chain started in an
//                  earlier block.
constexpr int kChainBlk = 128;

__global__ void k_chain_local(int64_t n_units, int V, const int* __restrict__ cont,
                              const double* __restrict__ val, double* __restrict__ carry,
                              double* __restrict__ tailsum, int* __restrict__ starts_in,
                              const int* any) {
  if (!*any) return;
  const int64_t b = blockIdx.x;
  const int64_t u0 = b * kChainBlk;
  const int64_t u1 = min(u0 + kChainBlk, n_units);
  for (int col = threadIdx.x; col < V; col += blockDim.x) {
    double run = 0.0;
    int started = 0;  // a chain starts inside this block before the current unit
    for (int64_t u = u0; u < u1; ++u) {
      const int g = cont[u];
      if (g < 0) { run = 0.0; started = 1; continue; }
      const bool start = (u == 0) || cont[u - 1] != g;
      if (start) { run = 0.0; started = 1; }
      run += val[u * (int64_t)V + col];
      carry[(u + 1) * (int64_t)V + col] = run;
    }
    tailsum[b * V + col] = run;
    if (col == 0) starts_in[b] = started;
  }
}

// Segmented-sum pair: v is the running sum since the last reset (f = 1).
struct SegPair {
  double v;
  int f;
};
struct SegOp {
  __device__ __forceinline__ SegPair operator()(const SegPair& x, const SegPair& y) const {
    return {y.f ? y.v : x.v + y.v, x.f | y.f};
  }
};
constexpr int kTopThreads = 256, kTopItems = 4;

// One CTA per column: exclusive segmented scan over the blocks' trailing
// sums (reset where a chain starts inside the block), by cub::BlockScan in
// chunks -- a fixed association, so the carries are deterministic.
__global__ void __launch_bounds__(kTopThreads)
    k_chain_top(int64_t n_blocks, int64_t n_units, int V, const int* __restrict__ cont,
                const double* __restrict__ tailsum, const int* __restrict__ starts_in,
                double* __restrict__ cin, const int* any) {
  if (!*any) return;
  using Scan = cub::BlockScan<SegPair, kTopThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int col = blockIdx.x;
  SegPair carry{0.0, 0};
  for (int64_t base = 0; base < n_blocks; base += kTopThreads * kTopItems) {
    SegPair it[kTopItems];
#pragma unroll
    for (int i = 0; i < kTopItems; ++i) {
      const int64_t b = base + threadIdx.x * kTopItems + i;
      it[i] = b < n_blocks ? SegPair{tailsum[b * V + col], starts_in[b]} : SegPair{0.0, 0};
    }
    SegPair agg;
    Scan(tmp).ExclusiveScan(it, it, SegPair{0.0, 0}, SegOp(), agg);
#pragma unroll
    for (int i = 0; i < kTopItems; ++i) {
      const int64_t b = base + threadIdx.x * kTopItems + i;
      if (b >= n_blocks) continue;
      const int64_t u0 = b * kChainBlk;
      const bool cont_in = u0 > 0 && cont[u0] >= 0 && cont[u0 - 1] == cont[u0];
      cin[b * V + col] = cont_in ? SegOp()(carry, it[i]).v : 0.0;
    }
    carry = SegOp()(carry, agg);
    __syncthreads();  // tmp is reused by the next chunk
  }
}

__global__ void k_chain_fix(int64_t n_units, int V, const int* __restrict__ cont,
                            const double* __restrict__ cin, double* __restrict__ carry,
                            const int* any) {
  if (!*any) return;
  const int64_t b = blockIdx.x;
  const int64_t u0 = b * kChainBlk;
  const int64_t u1 = min(u0 + kChainBlk, n_units);
  if (u0 == 0 || cont[u0] < 0 || cont[u0 - 1] != cont[u0]) return;
  const int g = cont[u0];
  for (int col = threadIdx.x; col < V; col += blockDim.x) {
    const double c = cin[b * V + col];
    for (int64_t u = u0; u < u1 && cont[u] == g; ++u)
      carry[(u + 1) * (int64_t)V + col] += c;
  }
}

// K4: joins child summaries into the node's summary rows
// (figaro.hpp:196-230), in two passes.  k_join_rows (thread per row): the
// product of the child scales `all`, the per-child factors
// scale[k] * prod_{d != c} s_d in the reference's product order, and the new
// row scale (scale_out).  k_join_elems (thread per summary element): own
// columns times `all`, child columns = child summary row times its factor.
__global__ void __launch_bounds__(256) k_join_rows(const __grid_constant__ JoinArgs a,
                                                   double* __restrict__ fac) {
  const int nc = a.n_children;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.G;
       k += (int64_t)gridDim.x * blockDim.x) {
    double sc[kMaxChildren];
    double all = 1.0;
#pragma unroll
    for (int c = 0; c < kMaxChildren; ++c) {
      sc[c] = 0.0;
      if (c < nc) {
        const int idx = a.lidx[c][k];
        sc[c] = idx >= 0 ? a.child_scale[c][idx] : 0.0;
        all *= sc[c];
      }
    }
    const double sk = a.scale[k];
    if (a.scale_out) a.scale_out[k] = sk * all;
    double* f = fac + k * (nc + 1);
    f[nc] = all;
#pragma unroll
    for (int c = 0; c < kMaxChildren; ++c) {
      if (c >= nc) break;
      double x = sk;
#pragma unroll
      for (int d = 0; d < kMaxChildren; ++d)
        if (d != c && d < nc) x *= sc[d];
      f[c] = x;
    }
  }
}

constexpr int kJoinTile = 256;  // summary rows per k_join_elems tile

__global__ void __launch_bounds__(256) k_join_elems(const __grid_constant__ JoinArgs a,
                                                    const double* __restrict__ fac) {
  const int nc = a.n_children;
  const unsigned width = (unsigned)a.width;
  // Row tiles keep the element -> (row, column) split in 32-bit arithmetic.
  for (int64_t k0 = blockIdx.x * (int64_t)kJoinTile; k0 < a.G;
       k0 += (int64_t)gridDim.x * kJoinTile) {
    const unsigned rows = (unsigned)(a.G - k0 < kJoinTile ? a.G - k0 : kJoinTile);
    double* S = a.S + k0 * a.width;
    for (unsigned le = threadIdx.x; le < rows * width; le += blockDim.x) {
      const unsigned kk = le / width;
      const int j = (int)(le - kk * width);
      const int64_t k = k0 + kk;
      const double* f = fac + k * (nc + 1);
      if (j < a.own_w) {
        if (!a.own_done) S[le] *= f[nc];
        continue;
      }
      int c = 0;
      while (c + 1 < nc && j >= a.child_off[c + 1]) ++c;
      const int idx = a.lidx[c][k];
      S[le] = idx < 0 ? 0.0
                      : a.child_S[c][(int64_t)idx * a.child_w[c] + (j - a.child_off[c])] * f[c];
    }
  }
}

// The same with two adjacent columns per thread (double2 loads/stores) when
// the width, the own width and every child offset/width are even: half the
// per-element index arithmetic, 16-byte accesses.
__global__ void __launch_bounds__(256) k_join_elems2(const __grid_constant__ JoinArgs a,
                                                     const double* __restrict__ fac) {
  const int nc = a.n_children;
  const unsigned hw = (unsigned)(a.width >> 1);  // double2 per row
  for (int64_t k0 = blockIdx.x * (int64_t)kJoinTile; k0 < a.G;
       k0 += (int64_t)gridDim.x * kJoinTile) {
    const unsigned rows = (unsigned)(a.G - k0 < kJoinTile ? a.G - k0 : kJoinTile);
    double2* S = reinterpret_cast<double2*>(a.S + k0 * a.width);
    for (unsigned le = threadIdx.x; le < rows * hw; le += blockDim.x) {
      const unsigned kk = le / hw;
      const int j = 2 * (int)(le - kk * hw);
      const int64_t k = k0 + kk;
      const double* f = fac + k * (nc + 1);
      if (j < a.own_w) {
        if (a.own_done) continue;
        const double m = f[nc];
        double2 v = S[le];
        v.x *= m;
        v.y *= m;
        S[le] = v;
        continue;
      }
      int c = 0;
      while (c + 1 < nc && j >= a.child_off[c + 1]) ++c;
      const int idx = a.lidx[c][k];
      double2 v = make_double2(0.0, 0.0);
      if (idx >= 0) {
        const double m = f[c];
        v = *reinterpret_cast<const double2*>(
            a.child_S[c] + (int64_t)idx * a.child_w[c] + (j - a.child_off[c]));
        v.x *= m;
        v.y *= m;
      }
      S[le] = v;
    }
  }
}

// K4 in one kernel over tiles of kJoinTile summary rows: thread t first
// computes row t's child scales, factors and joined scale (the reference's
// product order, figaro.hpp:213-228) into shared memory, then the tile's
// double2 elements are written with a fixed (row, packet) split per thread
// -- no factor array in HBM, no per-element division.
constexpr int kJoinMaxC = 4;
#ifndef FG_JOIN_UNROLL
#define FG_JOIN_UNROLL 11
#endif
constexpr int kJoinUnroll = FG_JOIN_UNROLL;
__global__ void __launch_bounds__(kJoinTile) k_join_tile(const __grid_constant__ JoinArgs a) {
  __shared__ double fs[kJoinTile][kJoinMaxC + 1];  // child factors, [nc] = all
  __shared__ int is[kJoinTile][kJoinMaxC];
  const int nc = a.n_children;
  const int hw = (int)(a.width >> 1);
  // Threads cover only the packets this kernel writes: with the own columns
  // already final (own_done) a row's child packets alone, so every lane
  // stores (C3: 6 of 10 packets per row).
  const int pbase = a.own_done ? a.own_w >> 1 : 0;
  const int pw = hw - pbase > 0 ? hw - pbase : 1;
  const int tr = threadIdx.x / pw, tp = pbase + threadIdx.x - (threadIdx.x / pw) * pw;
  const int rpp = kJoinTile / pw;  // rows per pass (>= 1)
  const int j = 2 * tp;
  int c = 0;
  if (j >= a.own_w)
    while (c + 1 < nc && j >= a.child_off[c + 1]) ++c;
  for (int64_t k0 = blockIdx.x * (int64_t)kJoinTile; k0 < a.G;
       k0 += (int64_t)gridDim.x * kJoinTile) {
    const int rows = (int)(a.G - k0 < kJoinTile ? a.G - k0 : kJoinTile);
    if ((int)threadIdx.x < rows) {
      const int64_t k = k0 + threadIdx.x;
      double sc[kJoinMaxC];
      double all = 1.0;
#pragma unroll
      for (int d = 0; d < kJoinMaxC; ++d) {
        sc[d] = 0.0;
        if (d < nc) {
          const int idx = a.lidx[d][k];
          is[threadIdx.x][d] = idx;
          sc[d] = idx >= 0 ? a.child_scale[d][idx] : 0.0;
          all *= sc[d];
        }
      }
      const double sk = a.scale[k];
      if (a.scale_out) a.scale_out[k] = sk * all;
      fs[threadIdx.x][kJoinMaxC] = all;
#pragma unroll
      for (int d = 0; d < kJoinMaxC; ++d) {
        if (d >= nc) break;
        double f = sk;
#pragma unroll
        for (int e = 0; e < kJoinMaxC; ++e)
          if (e != d && e < nc) f *= sc[e];
        fs[threadIdx.x][d] = f;
      }
    }
    __syncthreads();
    if (tr < rpp && j < a.width) {
#pragma unroll kJoinUnroll
      for (int r = tr; r < rows; r += rpp) {
        double2* dst = reinterpret_cast<double2*>(a.S + (k0 + r) * a.width) + tp;
        if (j < a.own_w) {
          if (a.own_done) continue;
          const double m = fs[r][kJoinMaxC];
          double2 v = *dst;
          v.x *= m;
          v.y *= m;
          *dst = v;
        } else {
          const int idx = is[r][c];
          double2 v = make_double2(0.0, 0.0);
          if (idx >= 0) {
            const double m = fs[r][c];
            v = *reinterpret_cast<const double2*>(a.child_S[c] + (int64_t)idx * a.child_w[c] +
                                                  (j - a.child_off[c]));
            v.x *= m;
            v.y *= m;
          }
          *dst = v;
        }
      }
    }
    __syncthreads();
  }
}

template <int SLOTS, int VEC, bool VJ, bool JW = false, int CW = 0>
void launch_main(Context& ctx, const HtDev& d, const Geo& geo) {
  const size_t smem = (VJ ? sizeof(WarpSmemVJ) : sizeof(WarpSmem)) * kWarps;
  auto kern = k_heads_tails<SLOTS, VEC, VJ, JW, CW>;
  FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                        kWarps * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)ctx.sm_count * per_sm;
  const int64_t need = ceil_div(d.n_units, kWarps);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, kWarps * 32, smem, ctx.stream>>>(d, geo);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

template <int VEC>
void launch_slots(Context& ctx, const HtDev& d, const Geo& geo) {
  const int slots = (geo.np + geo.L - 1) / geo.L;
  if (d.nj >= 0) {  // join-on-read: widths up to 4 packets per lane
    if (slots <= 1) launch_main<1, VEC, true>(ctx, d, geo);
    else if (slots <= 2) launch_main<2, VEC, true>(ctx, d, geo);
    else launch_main<4, VEC, true>(ctx, d, geo);
    return;
  }
  if (d.wj >= 0) {  // join-on-write: own widths up to 2 packets per lane
    if (slots > 2) fail(FG_E_UNSUPPORTED, "join-on-write: own width too large");
    if (slots <= 1) launch_main<1, VEC, false, true>(ctx, d, geo);
    else launch_main<2, VEC, false, true>(ctx, d, geo);
    return;
  }
  // Hot shapes with compile-time geometry (C3: own F width 8, project-away
  // width 20; C4: widths 4, 8, 12; 16 for two-relation joins).
  if constexpr (VEC == 2) {
    const bool exact = slots <= 1 && geo.L == geo.np && geo.G == 32 / geo.np &&
                       geo.ls == d.w && d.w == 2 * geo.np && getenv("FG_HT_RUNTIME_GEO") == nullptr;
    if (exact) {
      switch (d.w) {
        case 4: return launch_main<1, 2, false, false, 4>(ctx, d, geo);
        case 8: return launch_main<1, 2, false, false, 8>(ctx, d, geo);
        case 12: return launch_main<1, 2, false, false, 12>(ctx, d, geo);
        case 16: return launch_main<1, 2, false, false, 16>(ctx, d, geo);
        case 20: return launch_main<1, 2, false, false, 20>(ctx, d, geo);
        default: break;
      }
    }
  }
  if (slots <= 1) launch_main<1, VEC, false>(ctx, d, geo);
  else if (slots <= 2) launch_main<2, VEC, false>(ctx, d, geo);
  else if (slots <= 4) launch_main<4, VEC, false>(ctx, d, geo);
  else if (slots <= 8) launch_main<8, VEC, false>(ctx, d, geo);
  else launch_main<16, VEC, false>(ctx, d, geo);
}

}  // namespace

// Shared set-up of the heads/tails launches: device view, carries of long
// groups (pre-pass), lane geometry.  `rb_fixed` forces the batch rows.
struct HtPrep {
  HtDev d{};
  Geo geo{};
  DevArray<int> cont, ticket, ufirst;
  DevArray<int64_t> qb;
  DevArray<double> val, carry;
};

// double2 staging of joined rows: every block starts on an even column and
// every source row on a 16-byte boundary.
static bool vj_vec2_ok(const HeadTailArgs& in) {
  const JoinArgs& j = *in.join;
  bool ok = j.own_w % 2 == 0 && in.join_ldh % 2 == 0 &&
            reinterpret_cast<uintptr_t>(in.join_heads) % 16 == 0;
  for (int c = 0; c < j.n_children; ++c)
    ok = ok && j.child_off[c] % 2 == 0 && j.child_w[c] % 2 == 0 &&
         reinterpret_cast<uintptr_t>(j.child_S[c]) % 16 == 0;
  return ok;
}

static void prepare(Context& ctx, const HeadTailArgs& in, HtPrep& P, int rb_fixed) {
  HtDev& d = P.d;
  if (in.w > 1024) fail(FG_E_UNSUPPORTED, "heads/tails: more than 1024 columns");
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
  d.head_mul = in.head_mul;
  d.l2hint = getenv("FG_NO_L2_HINT") == nullptr;
  d.bulk_ok = !in.perm && !in.join && !in.join_write && in.w > 0 && in.ld == in.w &&
              in.w % 2 == 0 && reinterpret_cast<uintptr_t>(in.data) % 16 == 0 &&
              getenv("FG_NO_BULK") == nullptr;
  {
    // Per-row bulk copies for rows of at least FG_ROW_BULK_MIN doubles
    // (default 16: a 128-byte line) that start on 16-byte boundaries.
    const char* e = getenv("FG_ROW_BULK_MIN");
    const int min_w = e ? atoi(e) : 16;
    d.rowbulk_ok = !in.join && !in.join_write && in.w >= min_w && in.w % 2 == 0 &&
                   in.ld % 2 == 0 && reinterpret_cast<uintptr_t>(in.data) % 16 == 0 &&
                   getenv("FG_NO_BULK") == nullptr;
  }
  d.nj = -1;
  d.wj = -1;
  if (in.join_write) {
    const JoinArgs& j = *in.join_write;
    if (j.n_children > kVJMax) fail(FG_E_ARG, "join-on-write: too many children");
    if (j.own_w != in.w || in.ldh < j.width) fail(FG_E_ARG, "join-on-write: layout");
    d.wj = j.n_children;
    d.wwidth = (int)j.width;
    for (int c = 0; c < j.n_children; ++c) {
      d.wlidx[c] = j.lidx[c];
      d.wS[c] = j.child_S[c];
      d.wsc[c] = j.child_scale[c];
      d.wcw[c] = j.child_w[c];
      d.woff[c] = j.child_off[c];
    }
  }
  if (in.join) {
    const JoinArgs& j = *in.join;
    if (j.n_children > kVJMax) fail(FG_E_ARG, "join-on-read: too many children");
    d.nj = j.n_children;
    d.own_w = j.own_w;
    d.jhead = in.join_heads;
    d.jld = in.join_ldh;
    for (int c = 0; c < j.n_children; ++c) {
      d.jlidx[c] = j.lidx[c];
      d.jS[c] = j.child_S[c];
      d.jscale[c] = j.child_scale[c];
      d.jw[c] = j.child_w[c];
      d.joff[c] = j.child_off[c];
    }
  }
  d.rb = in.w > 0 ? std::max(1, std::min(in.join ? kVJRows : kMaxRB, kSmemDoubles / in.w))
                  : kMaxRB;
  if (in.join && in.w == 0) fail(FG_E_ARG, "join-on-read needs data columns");
  d.n_units = ceil_div(in.n_rows, kUnit);

  const int V = in.w + (in.weights ? 1 : 0);
  DevArray<int>& cont = P.cont;
  DevArray<double>& val = P.val;
  DevArray<double>& carry = P.carry;
  cont.alloc(d.n_units, ctx.stream);
  P.ufirst.alloc(d.n_units, ctx.stream);
  P.qb.alloc(d.n_units + 1, ctx.stream);
  P.ticket.alloc(1, ctx.stream);
  P.ticket.zero();
  d.ticket = P.ticket.get();
  if (d.n_units > 1) {
    val.alloc(d.n_units * (size_t)V, ctx.stream);
    carry.alloc((d.n_units + 1) * (size_t)V, ctx.stream);
    const int threads = 256;
    int64_t grid = ceil_div(d.n_units * 32, threads);
    grid = std::min<int64_t>(grid, (int64_t)ctx.sm_count * 16);
    DevArray<int> any(1, ctx.stream);
    any.zero();
    k_unit_cont<<<(int)std::min<int64_t>(ceil_div(d.n_units, threads), (int64_t)ctx.sm_count * 8),
                  threads, 0, ctx.stream>>>(d, cont.get(), P.ufirst.get(), P.qb.get(),
                                            any.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    const bool vec2 = in.join ? vj_vec2_ok(in)
                              : in.w % 2 == 0 && in.ld % 2 == 0 &&
                                    reinterpret_cast<uintptr_t>(in.data) % 16 == 0;
    Geo tg{};
    tg.vec = vec2 ? 2 : 1;
    tg.np = in.w > 0 ? (in.w + tg.vec - 1) / tg.vec : 1;
    tg.L = 1;
    while (tg.L < tg.np && tg.L < 32) tg.L <<= 1;
    tg.G = 32 / tg.L;
    if (vec2)
      k_unit_tail_sums<2><<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(
          d, cont.get(), val.get(), tg);
    else
      k_unit_tail_sums<1><<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(
          d, cont.get(), val.get(), tg);
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    const int64_t nb = ceil_div(d.n_units, kChainBlk);
    DevArray<double> tailsum(nb * (size_t)V, ctx.stream), cin(nb * (size_t)V, ctx.stream);
    DevArray<int> starts(nb, ctx.stream);
    const int ct = std::min(256, ((V + 31) / 32) * 32);
    k_chain_local<<<(int)nb, ct, 0, ctx.stream>>>(d.n_units, V, cont.get(), val.get(),
                                                  carry.get(), tailsum.get(), starts.get(),
                                                  any.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    k_chain_top<<<V, kTopThreads, 0, ctx.stream>>>(nb, d.n_units, V, cont.get(), tailsum.get(),
                                          starts.get(), cin.get(), any.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    k_chain_fix<<<(int)nb, ct, 0, ctx.stream>>>(d.n_units, V, cont.get(), cin.get(),
                                                carry.get(), any.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    d.cont = cont.get();
    d.carry = carry.get();
    d.ufirst = P.ufirst.get();
    d.qb = P.qb.get();
  }
  // Vector width, lanes per row-group and rows per batch.
  Geo& geo = P.geo;
  const bool src_ok = in.join ? vj_vec2_ok(in)
                              : in.ld % 2 == 0 &&
                                    reinterpret_cast<uintptr_t>(in.data) % 16 == 0;
  const bool aligned = in.w > 0 && in.w % 2 == 0 && src_ok &&
                       (!in.tails || (in.ldt % 2 == 0 &&
                                      reinterpret_cast<uintptr_t>(in.tails) % 16 == 0)) &&
                       (!in.heads || in.join_write ||
                        (in.ldh % 2 == 0 && reinterpret_cast<uintptr_t>(in.heads) % 16 == 0));
  geo.vec = aligned ? 2 : 1;
  geo.np = in.w > 0 ? (in.w + geo.vec - 1) / geo.vec : 1;
  geo.L = 1;
  while (geo.L < geo.np && geo.L < 32) geo.L <<= 1;
  geo.G = 32 / geo.L;
  // Row-groups of exactly np lanes when that packs more rows into the warp
  // (C3's project-away, 10 packets: 3 row-groups / 30 busy lanes instead of
  // 2 / 20); the lanes past G * L idle.  Unfused kernels only.
  if (rb_fixed == 0 && in.w > 0 && !in.join && geo.np < 32 && 32 / geo.np > geo.G &&
      getenv("FG_HT_POW2") == nullptr) {
    geo.L = geo.np;
    geo.G = 32 / geo.np;
  }
  if (in.w > 0) {
    int rb = std::min(in.join ? kVJRows : kMaxRB, kSmemDoubles / in.w);
    if (rb >= geo.G) rb -= rb % geo.G;
    d.rb = std::max(1, rb);
  }
  geo.ls = in.w;
  if (rb_fixed > 0) d.rb = rb_fixed;
}

// Row stride for a fused tile: the TSQR tile load has TR lanes reading TR
// rows of the same TC adjacent columns; ls = TC (mod 2 TC) puts those rows on
// disjoint bank groups (2 wavefronts per 8-byte load instead of TR).
template <class F>
int fused_stride(int w) {
  int ls = w;
  while (ls % (2 * F::TC) != F::TC % (2 * F::TC)) ++ls;
  return ls + (ls & 1);  // double2 staging needs an even stride
}

void run_heads_tails(Context& ctx, const HeadTailArgs& in) {
  if (in.n_seg == 0 || in.n_rows == 0) return;
  if (in.w > 1024) fail(FG_E_UNSUPPORTED, "heads/tails: more than 1024 columns");
  HtPrep P;
  prepare(ctx, in, P, 0);
  if (P.geo.vec == 2) launch_slots<2>(ctx, P.d, P.geo);
  else launch_slots<1>(ctx, P.d, P.geo);
}

namespace {
using FW4 = WCfg<4, 1, 8, 2>;
using FW8 = WCfg<8, 2, 8, 2>;
#ifndef FG_FW16_RPT
#define FG_FW16_RPT 8
#endif
using FW16 = WCfg<16, 4, FG_FW16_RPT, 2>;
using FW16r = WCfg<16, 4, 8, 2, 1>;
using FW32 = WCfg<32, 4, 8, 1>;
using FW12 = WCfg<12, 3, 8, 2>;
using FW20 = WCfg<20, 5, 4, 1>;
using FW24 = WCfg<24, 3, 8, 1>;

template <int VEC, class F>
int launch_fused(Context& ctx, HtPrep& P, DevArray<double>& partials) {
  using SM = WarpSmemT<kFusedDoubles>;
  const size_t smem = sizeof(SM) * kFusedWarps;
  auto kern = k_heads_tails_tsqr<VEC, F>;
  FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                        kFusedWarps * 32, smem));
  int64_t grid = (int64_t)ctx.sm_count * std::max(per_sm, 1);
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, ceil_div(P.d.n_units, kFusedWarps)));
  partials.alloc((size_t)grid * kFusedWarps * F::W * F::W, ctx.stream);
  kern<<<(int)grid, kFusedWarps * 32, smem, ctx.stream>>>(P.d, P.geo, partials.get());
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  return (int)(grid * kFusedWarps);
}

template <class F>
int fused_for(Context& ctx, const HeadTailArgs& in, DevArray<double>& partials) {
  const int ls = fused_stride<F>(in.w);
  if (ls * F::B > kFusedDoubles) return -1;  // caller falls back
  HtPrep P;
  prepare(ctx, in, P, F::B);
  P.geo.ls = ls;
  return P.geo.vec == 2 ? launch_fused<2, F>(ctx, P, partials)
                        : launch_fused<1, F>(ctx, P, partials);
}
}  // namespace

int fused_width(int w) {
  if (w <= 0 || w > 32) return 0;
  for (int b : {4, 8, 12, 16, 20, 24, 32})
    if (w <= b) return b;
  return 0;
}

int run_heads_tails_fused(Context& ctx, const HeadTailArgs& in,
                          DevArray<double>& partials) {
  if (in.n_seg == 0 || in.n_rows == 0) return 0;
  switch (fused_width(in.w)) {
    case 4: return fused_for<FW4>(ctx, in, partials);
    case 8: return fused_for<FW8>(ctx, in, partials);
    case 12: return fused_for<FW12>(ctx, in, partials);
    case 16: {
      const char* e = getenv("FG_FUSED_W16");
      if (e && std::string(e) == "roll") return fused_for<FW16r>(ctx, in, partials);
      return fused_for<FW16>(ctx, in, partials);
    }
    case 20: return fused_for<FW20>(ctx, in, partials);
    case 24: return fused_for<FW24>(ctx, in, partials);
    case 32: return fused_for<FW32>(ctx, in, partials);
    default: fail(FG_E_ARG, "no fused kernel for this width");
  }
}

// all[g] = prod_c s_c of summary row g (figaro.hpp:213-215), for the
// heads/tails kernel to apply to the own columns as it writes them.
__global__ void k_join_all(const __grid_constant__ JoinArgs a, double* __restrict__ all_out) {
  const int nc = a.n_children;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.G;
       k += (int64_t)gridDim.x * blockDim.x) {
    double all = 1.0;
    for (int c = 0; c < nc; ++c) {
      const int idx = a.lidx[c][k];
      all *= idx >= 0 ? a.child_scale[c][idx] : 0.0;
    }
    all_out[k] = all;
  }
}

void launch_join_all(Context& ctx, const JoinArgs& a, double* all_out) {
  if (a.G == 0) return;
  const int64_t grid = std::min<int64_t>(ceil_div(a.G, 256), (int64_t)ctx.sm_count * 16);
  k_join_all<<<(int)std::max<int64_t>(grid, 1), 256, 0, ctx.stream>>>(a, all_out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_join(Context& ctx, const JoinArgs& a) {
  if (a.G == 0) return;
  const int threads = 256;
  bool even = (a.width % 2 == 0) && (a.own_w % 2 == 0) && a.width > 0;
  for (int c = 0; c < a.n_children; ++c)
    even = even && (a.child_off[c] % 2 == 0) && (a.child_w[c] % 2 == 0);
  // (A one-pass variant recomputing the row factors per element was measured
  // 7 ms slower on C3: four dependent loads per element.)
  if (even && a.width / 2 <= kJoinTile && a.n_children <= kJoinMaxC &&
      getenv("FG_JOIN_TWO_PASS") == nullptr) {
    const int64_t grid = std::min<int64_t>(ceil_div(a.G, kJoinTile), (int64_t)ctx.sm_count * 8);
    k_join_tile<<<(int)std::max<int64_t>(grid, 1), kJoinTile, 0, ctx.stream>>>(a);
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    return;
  }
  DevArray<double> fac(a.G * (a.n_children + 1), ctx.stream);
  int64_t grid = std::min<int64_t>(ceil_div(a.G, threads), (int64_t)ctx.sm_count * 16);
  k_join_rows<<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(a, fac.get());
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  const int64_t total = a.G * a.width;
  if (total > 0) {
    grid = std::min<int64_t>(ceil_div(a.G, kJoinTile), (int64_t)ctx.sm_count * 16);
    if (even)
      k_join_elems2<<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(a, fac.get());
    else
      k_join_elems<<<(int)std::max<int64_t>(grid, 1), threads, 0, ctx.stream>>>(a, fac.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
  }
}

}  // namespace fg
