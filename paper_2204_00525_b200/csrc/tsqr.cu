// K6/K7: TSQR post-processing of the R0 spans into the N x N factor R.
//
// Reference: triangularize_block (postprocess.hpp:35-64), the THIN row
// absorb + tournament merge (postprocess.hpp:70-169) and normalize_signs
// (postprocess.hpp:173-190).  The reference rotates row by row with Givens;
// here each CTA owns an upper-triangular accumulator R (shared memory) and
// absorbs B-row tiles with a structured Householder QR of [R; X] (the LAPACK
// tpqrt shape: reflector k touches row k of R and the B tile rows), 2 B W^2
// flops per tile.
//
// Tile pipeline: rows are staged global -> shared with cp.async (LDGSTS,
// coalesced, zero-filled outside the span's column range) one tile ahead of
// the compute, then moved into registers in a column-owner layout: TC column
// groups x TR row lanes, each thread holding RPT rows x CPT columns.  Columns
// are dealt to groups in mirrored pairs (c, 2TC-1-c, ...) so the trailing
// work stays balanced as the active width shrinks.  One CTA barrier per
// column; reductions over the TR lanes of a group are xor-shuffles.
//
// Level 0 factors each span with persistent CTAs; the partial factors are
// then treated as rows of one n-wide matrix (embedded at their column
// offsets) and merged by the same kernel until one CTA remains.  The last R
// is sign-normalised (positive diagonal, strictly-lower entries exactly 0).
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "launchers.cuh"
#include "tsqr_warp.cuh"

namespace fg {

namespace {

struct SegDev {
  const double* data;
  int64_t rows;
  int64_t ld;
  int cols;
  int col_begin;
  int64_t row0;  // first row of this segment in the concatenated row space
};

}  // namespace
}  // namespace fg
#include "tsqr_blk.cuh"
#include "tsqr_la.cuh"
namespace fg {
namespace {

template <int W_, int TC_, int TR_, int RPT_>
struct Cfg {
  static constexpr int W = W_;
  static constexpr int TC = TC_;
  static constexpr int TR = TR_;
  static constexpr int RPT = RPT_;
  static constexpr int CPT = W / TC;
  static constexpr int GPW = 32 / TR;
  static constexpr int NT = TC * TR;
  static constexpr int B = TR * RPT;
  static constexpr int LDS = W + 1;  // padded staging row (bank spread)
  static_assert(W % TC == 0, "W % TC");
  static_assert(TC % GPW == 0, "TC % GPW");
  static constexpr size_t smem_doubles = W * W + 2 * B + 6 + B * LDS;
  static constexpr size_t smem_bytes = smem_doubles * 8 + B * sizeof(int);
};

template <class C>
__device__ __forceinline__ int col_of(int q, int c) {
  return (q & 1) ? (q + 1) * C::TC - 1 - c : q * C::TC + c;
}

template <class C>
__device__ __forceinline__ double group_sum(double x, unsigned mask) {
#pragma unroll
  for (int o = C::TR / 2; o; o >>= 1) x += __shfl_xor_sync(mask, x, o);
  return x;
}

// Issues the cp.async copies of tile `t` (rows t*B .. t*B+B-1 of the
// concatenated segment rows) into `stage`.
template <class C>
__device__ __forceinline__ void stage_tile(const SegDev* __restrict__ segs,
                                           int nseg, int64_t total_rows,
                                           int64_t t, double* stage,
                                           int* rowseg) {
  const int64_t r0 = t * C::B;
  for (int row = threadIdx.x; row < C::B; row += C::NT) {
    const int64_t gr = r0 + row;
    int s = -1;
    if (gr < total_rows) {
      int lo = 0, hi = nseg;  // last segment with row0 <= gr
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (segs[mid].row0 <= gr) lo = mid; else hi = mid;
      }
      s = lo;
    }
    rowseg[row] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < C::B * C::W; e += C::NT) {
    const int row = e / C::W;
    const int col = e - row * C::W;
    double* dst = stage + row * C::LDS + col;
    const int s = rowseg[row];
    if (s >= 0) {
      const SegDev& sg = segs[s];
      const int lc = col - sg.col_begin;
      if (lc >= 0 && lc < sg.cols) {
        __pipeline_memcpy_async(dst, sg.data + (r0 + row - sg.row0) * sg.ld + lc,
                                sizeof(double));
        continue;
      }
    }
    *dst = 0.0;
  }
  __pipeline_commit();
}

template <class C>
__global__ void __launch_bounds__(C::NT)
    k_tsqr(const SegDev* __restrict__ segs, int nseg, int64_t total_rows,
           int64_t total_tiles, int64_t nunits, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  double* R = sm;                         // W x W
  double* vbuf = R + C::W * C::W;         // 2 x B
  double* taus = vbuf + 2 * C::B;         // 2 x {t1, t2}
  double* u0s = taus + 4;                 // 2
  double* stage = u0s + 2;                // B x LDS
  int* rowseg = reinterpret_cast<int*>(stage + C::B * C::LDS);

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int r = lane % C::TR;
  const int gw = lane / C::TR;
  const int c = warp * C::GPW + gw;
  const unsigned gmask =
      C::TR == 32 ? 0xffffffffu : (((1u << C::TR) - 1u) << (gw * C::TR));

  for (int e = threadIdx.x; e < C::W * C::W; e += C::NT) R[e] = 0.0;

  double X[C::RPT][C::CPT];
  int64_t t = blockIdx.x;
  if (t < total_tiles) stage_tile<C>(segs, nseg, total_rows, t, stage, rowseg);

  for (; t < total_tiles; t += nunits) {
    __pipeline_wait_prior(0);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < C::RPT; ++i)
#pragma unroll
      for (int q = 0; q < C::CPT; ++q)
        X[i][q] = stage[(i * C::TR + r) * C::LDS + col_of<C>(q, c)];
    __syncthreads();
    if (t + nunits < total_tiles)
      stage_tile<C>(segs, nseg, total_rows, t + nunits, stage, rowseg);

#pragma unroll
    for (int qb = 0; qb < C::CPT; ++qb) {
      for (int within = 0; within < C::TC; ++within) {
        const int k = qb * C::TC + within;
        const int ck = (qb & 1) ? C::TC - 1 - within : within;
        double* vb = vbuf + (k & 1) * C::B;
        if (c == ck) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int i = 0; i < C::RPT; i += 2) {
            s0 = fma(X[i][qb], X[i][qb], s0);
            if (i + 1 < C::RPT) s1 = fma(X[i + 1][qb], X[i + 1][qb], s1);
          }
          const double sig = group_sum<C>(s0 + s1, gmask);
          const double alpha = R[k * C::W + k];
          const Reflector h = make_reflector(alpha, sig);
          if (h.t1 != 0.0) {
#pragma unroll
            for (int i = 0; i < C::RPT; ++i) vb[i * C::TR + r] = X[i][qb];
          }
          __syncwarp(gmask);
          if (r == 0) {
            R[k * C::W + k] = h.beta;
            taus[2 * (k & 1)] = h.t1;
            taus[2 * (k & 1) + 1] = h.t2;
            u0s[k & 1] = h.u0;
          }
        }
        __syncthreads();
        const double t1 = taus[2 * (k & 1)];
        const double t2 = taus[2 * (k & 1) + 1];
        const double u0 = u0s[k & 1];
        if (t1 == 0.0) continue;
        double v[C::RPT];
#pragma unroll
        for (int i = 0; i < C::RPT; ++i) v[i] = vb[i * C::TR + r];
#pragma unroll
        for (int q = qb; q < C::CPT; ++q) {
          const int j = col_of<C>(q, c);
          if (j <= k) continue;
          const double rkj = R[k * C::W + j];
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int i = 0; i < C::RPT; i += 2) {
            d0 = fma(v[i], X[i][q], d0);
            if (i + 1 < C::RPT) d1 = fma(v[i + 1], X[i + 1][q], d1);
          }
          const double d = group_sum<C>(d0 + d1, gmask);
          const double f = (fma(u0, rkj, d) * t1) * t2;
#pragma unroll
          for (int i = 0; i < C::RPT; ++i) X[i][q] = fma(-f, v[i], X[i][q]);
          __syncwarp(gmask);
          if (r == 0) R[k * C::W + j] = fma(-f, u0, rkj);
        }
      }
    }
  }
  __syncthreads();
  double* o = out + (int64_t)blockIdx.x * C::W * C::W;
  for (int e = threadIdx.x; e < C::W * C::W; e += C::NT) o[e] = R[e];
}

// ---------------------------------------------------------------------------
// Warp-level variant for W <= 32: every warp owns its own accumulator R
// (shared memory, W x W) and absorbs B = TR*RPT-row tiles with warp
// shuffles only -- no CTA barriers.  The column loop is fully unrolled, the
// pivot column is broadcast to all lanes so the reflector is computed
// redundantly without divergence, and each lane forms v for its own rows.
// Partial factors are one per warp.

// Lane (r, c) holds tile rows i*TR + r (i < RPT) of its CPT columns and the
// accumulator entries R[m*TR + r][col] (m < RR) of the same columns, so the
// whole column loop is straight-line register code: pivot broadcast by
// shuffle, reflector computed redundantly by every lane (branch-free, tau = 0
// for an all-zero column), dot products reduced over the TR row lanes.
// bulk = 1 (one dense span of exactly W columns, 16-byte aligned): a warp's
// next tile is fetched by one 1-D bulk copy (TMA engine) into its shared-
// memory slot while the current tile is absorbed -- the slot is free as soon
// as the tile sits in registers -- instead of 8-byte loads whose latency the
// 8 resident warps cannot hide (10 % of the W = 20 kernel's stall samples).
__device__ __forceinline__ uint32_t tw_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tw_bulk_tile(void* dst, const void* src, unsigned bytes,
                                             unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tw_smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(tw_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tw_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tw_mbar_wait(unsigned long long* bar, unsigned phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(tw_smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

template <class C, bool BULK>
__global__ void __launch_bounds__(C::NT, C::MINB)
    k_tsqr_warp(const SegDev* __restrict__ segs, int nseg, int64_t total_rows,
                int64_t total_tiles, int64_t nunits, double* __restrict__ out) {
  constexpr bool bulk = BULK;
  extern __shared__ __align__(16) unsigned char tw_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int r = lane % C::TR;
  const int c = lane / C::TR;
  const int64_t gw = (int64_t)blockIdx.x * C::WARPS + wib;
  if (gw >= nunits) return;
  int cols[C::CPT];
#pragma unroll
  for (int q = 0; q < C::CPT; ++q) cols[q] = wcol<C>(q, c);
  double Racc[C::RR][C::CPT];
#pragma unroll
  for (int m = 0; m < C::RR; ++m)
#pragma unroll
    for (int q = 0; q < C::CPT; ++q) Racc[m][q] = 0.0;

  constexpr unsigned kTileBytes = C::B * C::W * sizeof(double);
  double* tbuf = reinterpret_cast<double*>(tw_raw) + (size_t)wib * C::B * C::W;
  unsigned long long* bar =
      reinterpret_cast<unsigned long long*>(tw_raw + (size_t)C::WARPS * kTileBytes) + wib;
  unsigned phase = 0;
  const double* dense = nullptr;
  if constexpr (bulk) {
    dense = segs[0].data;
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tw_smem_u32(bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if ((gw + 1) * C::B <= total_rows)
        tw_bulk_tile(tbuf, dense + gw * (int64_t)C::B * C::W, kTileBytes, bar);
    }
    __syncwarp();
  }

  for (int64_t t = gw; t < total_tiles; t += nunits) {
    double X[C::RPT][C::CPT];
    if (bulk && (t + 1) * C::B <= total_rows) {  // (compile-time false without BULK)
      // full tiles arrive through the warp's slot (issued one tile ahead)
      tw_mbar_wait(bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int i = 0; i < C::RPT; ++i)
#pragma unroll
        for (int q = 0; q < C::CPT; ++q) X[i][q] = tbuf[(i * C::TR + r) * C::W + cols[q]];
      __syncwarp();
      const int64_t tn = t + nunits;
      if (lane == 0 && tn < total_tiles && (tn + 1) * C::B <= total_rows)
        tw_bulk_tile(tbuf, dense + tn * (int64_t)C::B * C::W, kTileBytes, bar);
      absorb_tile<C>(X, Racc, r, c, cols);
      continue;
    }
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
      const int64_t gr = t * C::B + i * C::TR + r;
      const double* rp = nullptr;
      int lo = 0, hi = 0;
      if (gr < total_rows) {
        int s = 0;
        if (nseg > 1) {
          int a = 0, b = nseg;
          while (b - a > 1) {
            const int mid = (a + b) >> 1;
            if (segs[mid].row0 <= gr) a = mid; else b = mid;
          }
          s = a;
        }
        const SegDev& sg = segs[s];
        rp = sg.data + (gr - sg.row0) * sg.ld - sg.col_begin;
        lo = sg.col_begin;
        hi = sg.col_begin + sg.cols;
      }
#pragma unroll
      for (int q = 0; q < C::CPT; ++q)
        X[i][q] = (rp && cols[q] >= lo && cols[q] < hi) ? __ldg(rp + cols[q]) : 0.0;
    }

    absorb_tile<C>(X, Racc, r, c, cols);
  }
  double* o = out + gw * C::W * C::W;
#pragma unroll
  for (int m = 0; m < C::RR; ++m)
#pragma unroll
    for (int q = 0; q < C::CPT; ++q)
      if (m * C::TR + r < C::W) o[(m * C::TR + r) * C::W + cols[q]] = Racc[m][q];
  // Entries of R below the diagonal are never written by the loop (they
  // stay 0), so the stored factor is upper triangular.
}

__global__ void k_normalize(const double* __restrict__ Rw, int W, int n,
                            double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += gridDim.x * blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;
    double v = j < i ? 0.0 : Rw[i * W + j];
    if (Rw[i * W + i] < 0.0) v = (v == 0.0) ? 0.0 : -v;
    out[e] = v;
  }
}

using W4 = WCfg<4, 1, 8, 2>;
using W8 = WCfg<8, 2, 8, 2>;
using W8c = WCfg<8, 2, 12, 2>;   // 96-row tiles (measured best at W = 8)
using W12 = WCfg<12, 3, 8, 2>;
using W12c = WCfg<12, 3, 12, 2>;  // 96-row tiles (measured best at W = 12)
using W16 = WCfg<16, 2, 8, 2>;
using W16c = WCfg<16, 4, 8, 2>;
using W20 = WCfg<20, 5, 8, 1>;
#ifndef FG_W20_RPT
#define FG_W20_RPT 14
#endif
#ifndef FG_W20_MINB
#define FG_W20_MINB 1
#endif
#ifndef FG_W20_WARPS
#define FG_W20_WARPS 8
#endif
using W20t = WCfg<20, 5, FG_W20_RPT, FG_W20_MINB, 0, FG_W20_WARPS>;  // 112-row tiles (measured best at W = 20)
using W24 = WCfg<24, 3, 8, 2>;
using W32c = WCfg<32, 4, 8, 2>;
using C16 = Cfg<16, 8, 16, 16>;
using C32 = Cfg<32, 16, 16, 8>;
using C40 = Cfg<40, 20, 8, 16>;
using C48 = Cfg<48, 24, 8, 16>;
using C64 = Cfg<64, 32, 8, 16>;
using C128 = Cfg<128, 32, 8, 8>;
// Look-ahead blocked kernels (tsqr_la.cuh): "lab" = single-buffered 64-row
// tiles, full-square R; "lat" = 2-warp CTAs with triangular-block R (more
// CTAs per SM, for large spans).
using L32 = LCfg<32, 64, 2, 6, 1>;
using L40 = LCfg<40, 64, 2, 6, 1>;
using L48 = LCfg<48, 64, 2, 5, 1>;
using L64 = LCfg<64, 64, 4, 3, 1>;
#ifndef FG_L64T_B
#define FG_L64T_B 64
#endif
#ifndef FG_L64T_MINB
#define FG_L64T_MINB 4
#endif
#ifndef FG_L64T_WARPS
#define FG_L64T_WARPS 2
#endif
using L64t = LCfg<64, FG_L64T_B, FG_L64T_WARPS, FG_L64T_MINB, 1, 1>;
using L128 = LCfg<128, 64, 8, 1, 1>;
using L128t = LCfg<128, 32, 4, 2, 1, 1>;

// Kernel per width.  The default is the measured best
// (scripts/tsqr_variants.py, profiles/r1s2/tsqr_variants.txt); FG_TSQR_W<W>
// selects an alternative for experiments: warp | warpc (register warp
// kernels), cta (column-at-a-time CTA kernel), lab | lat (look-ahead).
enum class Kern { Warp, WarpC, Cta, La, LaT };

// Spans of at least this many rows take the 2-warp triangular-R look-ahead
// kernel at W = 64 / 128 (4 / 2 CTAs per SM); smaller ones (merge levels)
// the single-buffered one, whose per-tile latency is lower.
constexpr int64_t kBigSpan = int64_t(1) << 19;

Kern variant(int W, int64_t rows) {
  const std::string key = "FG_TSQR_W" + std::to_string(W);
  const char* e = getenv(key.c_str());
  const std::string v = e ? e : "";
  if (v == "warp") return Kern::Warp;
  if (v == "warpc") return Kern::WarpC;
  if (v == "cta") return Kern::Cta;
  if (v == "lab") return Kern::La;
  if (v == "lat") return Kern::LaT;
  if (W <= 24) return W == 16 ? Kern::WarpC : Kern::Warp;
  if ((W == 64 || W == 128) && rows >= kBigSpan) return Kern::LaT;
  return Kern::La;
}

int bucket(int w) {
  for (int b : {4, 8, 12, 16, 20, 24, 32, 40, 48, 64, 128})
    if (w <= b) return b;
  return 0;
}

// Launch shape of one factorisation kernel: rows per tile, partial factors
// per CTA, and the resident-CTA cap.
struct Plan {
  int B;
  int per_cta;
  int cap;
};

template <class K>
int resident(Context& ctx, K kern, int nt, size_t smem) {
  FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
  return std::max(1, per_sm) * ctx.sm_count;
}

template <class C>
Plan plan_cta(Context& ctx) {
  return {C::B, 1, resident(ctx, k_tsqr<C>, C::NT, C::smem_bytes)};
}
template <class C>
Plan plan_la(Context& ctx) {
  return {C::B, 1, resident(ctx, k_tsqr_la<C, SegDev>, C::NT, C::smem_bytes)};
}
// Shared memory of the warp kernel's bulk-copied tiles (one slot + one
// mbarrier per warp), or 0 when MINB CTAs of it would not fit an SM.
template <class C>
size_t warp_bulk_smem(Context& ctx) {
  const size_t need = (size_t)C::WARPS * (C::B * C::W * sizeof(double) + 8);
  if (getenv("FG_TSQR_NO_BULK")) return 0;
  return (need + 1024) * C::MINB <= 228u * 1024 && need <= ctx.smem_optin ? need : 0;
}
template <class C>
Plan plan_warp(Context& ctx, bool bulk) {
  const size_t smem = bulk ? warp_bulk_smem<C>(ctx) : 0;
  return {C::B, C::WARPS,
          smem ? resident(ctx, k_tsqr_warp<C, true>, C::NT, smem)
               : resident(ctx, k_tsqr_warp<C, false>, C::NT, 0)};
}

// Runs `f` with the config type of width W / kernel k (unsupported
// combinations fall back to the width's default kernel family).
template <class F>
auto with_kernel(int W, Kern k, F&& f) {
  switch (W) {
    case 4: return f(W4{});
    case 8: return k == Kern::WarpC ? f(W8{}) : f(W8c{});
    case 12: return k == Kern::WarpC ? f(W12{}) : f(W12c{});
    case 16: return k == Kern::Cta ? f(C16{}) : k == Kern::Warp ? f(W16{}) : f(W16c{});
    case 20: return k == Kern::WarpC ? f(W20{}) : f(W20t{});
    case 24: return f(W24{});
    case 32: return k == Kern::Cta ? f(C32{}) : (k == Kern::Warp || k == Kern::WarpC) ? f(W32c{}) : f(L32{});
    case 40: return k == Kern::Cta ? f(C40{}) : f(L40{});
    case 48: return k == Kern::Cta ? f(C48{}) : f(L48{});
    case 64: return k == Kern::Cta ? f(C64{}) : k == Kern::LaT ? f(L64t{}) : f(L64{});
    default: return k == Kern::Cta ? f(C128{}) : k == Kern::LaT ? f(L128t{}) : f(L128{});
  }
}

template <class C> struct IsWarp : std::false_type {};
template <int A, int B_, int C_, int D, int E, int F_> struct IsWarp<WCfg<A, B_, C_, D, E, F_>> : std::true_type {};
template <class C> struct IsLa : std::false_type {};
template <int A, int B_, int C_, int D, int E, int G> struct IsLa<LCfg<A, B_, C_, D, E, G>> : std::true_type {};

Plan plan_for(Context& ctx, int W, int64_t rows, bool bulk) {
  return with_kernel(W, variant(W, rows), [&](auto cfg) -> Plan {
    using C = decltype(cfg);
    if constexpr (IsWarp<C>::value) return plan_warp<C>(ctx, bulk);
    else if constexpr (IsLa<C>::value) return plan_la<C>(ctx);
    else return plan_cta<C>(ctx);
  });
}

void launch_for(Context& ctx, int W, const SegDev* segs, int nseg,
                int64_t rows, int64_t tiles, int64_t units, int grid, double* out, bool bulk) {
  cudaStream_t s = ctx.stream;
  with_kernel(W, variant(W, rows), [&](auto cfg) {
    using C = decltype(cfg);
    if constexpr (IsWarp<C>::value) {
      const size_t smem = bulk ? warp_bulk_smem<C>(ctx) : 0;
      if (smem)
        k_tsqr_warp<C, true><<<grid, C::NT, smem, s>>>(segs, nseg, rows, tiles, units, out);
      else
        k_tsqr_warp<C, false><<<grid, C::NT, 0, s>>>(segs, nseg, rows, tiles, units, out);
    }
    else if constexpr (IsLa<C>::value)
      k_tsqr_la<C, SegDev><<<grid, C::NT, C::smem_bytes, s>>>(segs, nseg, rows, tiles, units, out);
    else
      k_tsqr<C><<<grid, C::NT, C::smem_bytes, s>>>(segs, nseg, rows, tiles, units, out);
    return 0;
  });
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

// A batch of W x W partial factors, meaningful width `cols` at `col_begin`.
struct Partial {
  const double* data;
  int count;
  int W;
  int cols;
  int col_begin;
};

// Factors the concatenation of `segs` (bucket W); each factor unit (CTA or
// warp) takes about `tiles_per_unit` tiles.  Returns the number of partial
// factors written to out.
int factor(Context& ctx, int W, std::vector<SegDev> segs, int64_t tiles_per_unit,
           DevArray<double>& out) {
  int64_t all_rows = 0;
  for (auto& s : segs) all_rows += s.rows;
  // One dense span of exactly W columns on 16-byte boundaries: the warp
  // kernels fetch its tiles by bulk copies.
  static const int64_t bulk_min_rows = [] {
    const char* e = getenv("FG_TSQR_BULK_MIN_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)1 << 20;
  }();
  const bool bulk = segs.size() == 1 && segs[0].cols == W && segs[0].ld == W &&
                    segs[0].col_begin == 0 && (W % 2) == 0 && all_rows >= bulk_min_rows &&
                    reinterpret_cast<uintptr_t>(segs[0].data) % 16 == 0;
  const Plan p = plan_for(ctx, W, all_rows, bulk);
  // A unit must absorb more rows than a factor has, or merges cannot shrink.
  tiles_per_unit = std::max<int64_t>(tiles_per_unit, 2 * ceil_div(W, p.B));
  int64_t rows = 0;
  for (auto& s : segs) {
    s.row0 = rows;
    rows += s.rows;
  }
  const int64_t tiles = ceil_div(rows, p.B);
  const int64_t units = std::max<int64_t>(
      1, std::min<int64_t>((int64_t)p.cap * p.per_cta, ceil_div(tiles, tiles_per_unit)));
  const int grid = (int)ceil_div(units, p.per_cta);
  DevArray<SegDev> dsegs(segs.size(), ctx.stream);
  FG_CUDA(cudaMemcpyAsync(dsegs.get(), segs.data(), segs.size() * sizeof(SegDev),
                          cudaMemcpyHostToDevice, ctx.stream));
  out.alloc((size_t)units * W * W, ctx.stream);
  launch_for(ctx, W, dsegs.get(), (int)segs.size(), rows, tiles, units, grid, out.get(), bulk);
  // Pageable host -> device copies are staged before cudaMemcpyAsync
  // returns, so `segs` may go out of scope.  Every unit gets >= 1 tile.
  return (int)units;
}

}  // namespace

void tsqr(Context& ctx, const std::vector<Span>& spans_in, int n,
          double* R_out) {
  if (n <= 0) return;
  const int WN = bucket(n);
  if (!WN) fail(FG_E_UNSUPPORTED, "TSQR: more than 128 data columns");
  std::vector<DevArray<double>> keep;
  std::vector<Partial> parts;

  // Level 0: each span on its own set of persistent CTAs.
  for (const Span& s : spans_in) {
    if (s.partials) {
      if (s.count) parts.push_back({s.partials, s.count, s.W, s.cols, s.col_begin});
      continue;
    }
    if (s.rows == 0 || s.cols == 0) continue;
    const int W = bucket(s.cols);
    DevArray<double> out;
    const int cnt =
        factor(ctx, W, {SegDev{s.data, s.rows, s.ld, s.cols, 0, 0}}, 2, out);
    parts.push_back({out.get(), cnt, W, s.cols, s.col_begin});
    keep.push_back(std::move(out));
  }

  // Merge levels in the n-wide space until a single factor remains.
  while (!parts.empty()) {
    int total = 0;
    for (const Partial& p : parts) total += p.count;
    if (total == 1 && parts[0].W == WN && parts[0].col_begin == 0) break;
    std::vector<SegDev> segs;
    for (const Partial& p : parts)
      for (int k = 0; k < p.count; ++k)
        segs.push_back({p.data + (int64_t)k * p.W * p.W, p.cols, p.W, p.cols,
                        p.col_begin, 0});
    DevArray<double> out;
    const int cnt = factor(ctx, WN, std::move(segs), 4, out);
    if (cnt >= total && total > 1)
      fail(FG_E_CUDA, "TSQR merge level did not reduce the number of factors");
    parts.clear();
    parts.push_back({out.get(), cnt, WN, n, 0});
    keep.push_back(std::move(out));
  }

  if (parts.empty()) {
    FG_CUDA(cudaMemsetAsync(R_out, 0, sizeof(double) * n * n, ctx.stream));
    return;
  }
  const int threads = 256;
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div((int64_t)n * n, threads), 64));
  k_normalize<<<blocks, threads, 0, ctx.stream>>>(parts[0].data, WN, n, R_out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

}  // namespace fg
