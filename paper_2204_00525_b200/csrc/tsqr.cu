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

#include "launchers.cuh"

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
  static constexpr size_t smem_doubles = W * W + 2 * B + 2 + B * LDS;
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
           int64_t total_tiles, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  double* R = sm;                         // W x W
  double* vbuf = R + C::W * C::W;         // 2 x B
  double* taus = vbuf + 2 * C::B;         // 2
  double* stage = taus + 2;               // B x LDS
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

  for (; t < total_tiles; t += gridDim.x) {
    __pipeline_wait_prior(0);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < C::RPT; ++i)
#pragma unroll
      for (int q = 0; q < C::CPT; ++q)
        X[i][q] = stage[(i * C::TR + r) * C::LDS + col_of<C>(q, c)];
    __syncthreads();
    if (t + gridDim.x < total_tiles)
      stage_tile<C>(segs, nseg, total_rows, t + gridDim.x, stage, rowseg);

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
          double tau = 0.0;
          if (sig > 0.0) {
            const double nrm = sqrt(fma(alpha, alpha, sig));
            const double beta = alpha >= 0.0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            const double scal = 1.0 / (alpha - beta);
#pragma unroll
            for (int i = 0; i < C::RPT; ++i) vb[i * C::TR + r] = X[i][qb] * scal;
            __syncwarp(gmask);
            if (r == 0) R[k * C::W + k] = beta;
          }
          if (r == 0) taus[k & 1] = tau;
        }
        __syncthreads();
        const double tau = taus[k & 1];
        if (tau == 0.0) continue;
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
          const double f = tau * (d + rkj);
#pragma unroll
          for (int i = 0; i < C::RPT; ++i) X[i][q] = fma(-f, v[i], X[i][q]);
          __syncwarp(gmask);
          if (r == 0) R[k * C::W + j] = rkj - f;
        }
      }
    }
  }
  __syncthreads();
  double* o = out + (int64_t)blockIdx.x * C::W * C::W;
  for (int e = threadIdx.x; e < C::W * C::W; e += C::NT) o[e] = R[e];
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

using C4 = Cfg<4, 4, 32, 8>;
using C8 = Cfg<8, 4, 32, 8>;
using C16 = Cfg<16, 8, 16, 16>;
using C32 = Cfg<32, 16, 16, 8>;
using C64 = Cfg<64, 32, 8, 16>;
using C128 = Cfg<128, 32, 8, 8>;

int bucket(int w) {
  for (int b : {4, 8, 16, 32, 64, 128})
    if (w <= b) return b;
  return 0;
}

template <class C>
int max_ctas(Context& ctx) {
  FG_CUDA(cudaFuncSetAttribute(k_tsqr<C>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)C::smem_bytes));
  int per_sm = 0;
  FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tsqr<C>,
                                                        C::NT, C::smem_bytes));
  return std::max(1, per_sm) * ctx.sm_count;
}

struct Plan {
  int B;
  int cap;
};

template <class C>
Plan plan_of(Context& ctx) {
  return {C::B, max_ctas<C>(ctx)};
}

Plan plan_for(Context& ctx, int W) {
  switch (W) {
    case 4: return plan_of<C4>(ctx);
    case 8: return plan_of<C8>(ctx);
    case 16: return plan_of<C16>(ctx);
    case 32: return plan_of<C32>(ctx);
    case 64: return plan_of<C64>(ctx);
    default: return plan_of<C128>(ctx);
  }
}

template <class C>
void launch(Context& ctx, const SegDev* segs, int nseg, int64_t rows,
            int64_t tiles, int grid, double* out) {
  k_tsqr<C><<<grid, C::NT, C::smem_bytes, ctx.stream>>>(segs, nseg, rows,
                                                         tiles, out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

void launch_for(Context& ctx, int W, const SegDev* segs, int nseg,
                int64_t rows, int64_t tiles, int grid, double* out) {
  switch (W) {
    case 4: launch<C4>(ctx, segs, nseg, rows, tiles, grid, out); break;
    case 8: launch<C8>(ctx, segs, nseg, rows, tiles, grid, out); break;
    case 16: launch<C16>(ctx, segs, nseg, rows, tiles, grid, out); break;
    case 32: launch<C32>(ctx, segs, nseg, rows, tiles, grid, out); break;
    case 64: launch<C64>(ctx, segs, nseg, rows, tiles, grid, out); break;
    default: launch<C128>(ctx, segs, nseg, rows, tiles, grid, out); break;
  }
}

// A batch of W x W partial factors, meaningful width `cols` at `col_begin`.
struct Partial {
  const double* data;
  int count;
  int W;
  int cols;
  int col_begin;
};

// Factors the concatenation of `segs` (bucket W) with CTAs taking about
// `tiles_per_cta` tiles each; returns the number of partial factors in out.
int factor(Context& ctx, int W, std::vector<SegDev> segs, int64_t tiles_per_cta,
           DevArray<double>& out) {
  const Plan p = plan_for(ctx, W);
  int64_t rows = 0;
  for (auto& s : segs) {
    s.row0 = rows;
    rows += s.rows;
  }
  const int64_t tiles = ceil_div(rows, p.B);
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(p.cap, ceil_div(tiles, tiles_per_cta)));
  DevArray<SegDev> dsegs(segs.size(), ctx.stream);
  FG_CUDA(cudaMemcpyAsync(dsegs.get(), segs.data(), segs.size() * sizeof(SegDev),
                          cudaMemcpyHostToDevice, ctx.stream));
  out.alloc((size_t)grid * W * W, ctx.stream);
  launch_for(ctx, W, dsegs.get(), (int)segs.size(), rows, tiles, grid,
             out.get());
  // Pageable host -> device copies are staged before cudaMemcpyAsync
  // returns, so `segs` may go out of scope.
  return grid;
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
