// K6/K7: TSQR post-processing of the R0 spans into the N x N factor R.
//
// Reference: triangularize_block (postprocess.hpp:35-64), the THIN row
// absorb + tournament merge (postprocess.hpp:70-169) and normalize_signs
// (postprocess.hpp:173-190).  The reference rotates row by row with Givens;
// here each CTA owns an upper-triangular accumulator R (shared memory) and
// absorbs B-row tiles of one span with a structured Householder QR of
// [R; X] (the LAPACK tpqrt shape: reflector k touches row k of R and all B
// rows of the tile), so a tile costs 2 B W^2 flops.  The tile lives in
// registers in a column-owner layout: TC column groups x TR row lanes, each
// thread holding RPT rows x CPT columns.  Columns are dealt to groups in
// mirrored pairs (c, 2TC-1-c, ...), so every group keeps the same amount of
// trailing work as the active width shrinks.  One barrier per column.
//
// Spans are factored in parallel by persistent CTAs (level 0); the partial
// factors are embedded at their column offsets and merged by further
// launches of the same kernel until one CTA remains; its R is
// sign-normalised (positive diagonal, strictly-lower entries exactly zero).
#include <algorithm>

#include "launchers.cuh"

namespace fg {

namespace {

struct TsqrSeg {
  const double* data;
  int64_t rows;
  int64_t ld;
  int cols;
  int col_begin;
  int64_t tile0;  // first global tile of this segment
};

constexpr int kMaxSegs = 64;

struct TsqrParams {
  int nseg;
  int64_t total_tiles;
  TsqrSeg seg[kMaxSegs];
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
  static_assert(W % TC == 0, "W % TC");
  static_assert(TC % GPW == 0, "TC % GPW");
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

template <class C>
__global__ void __launch_bounds__(C::NT)
    k_tsqr(const __grid_constant__ TsqrParams P, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  double* R = sm;                       // W x W
  double* vbuf = sm + C::W * C::W;      // 2 x B
  double* taus = vbuf + 2 * C::B;       // 2

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int r = lane % C::TR;
  const int gw = lane / C::TR;
  const int c = warp * C::GPW + gw;
  const unsigned gmask =
      C::TR == 32 ? 0xffffffffu : (((1u << C::TR) - 1u) << (gw * C::TR));

  for (int e = threadIdx.x; e < C::W * C::W; e += C::NT) R[e] = 0.0;
  __syncthreads();

  double X[C::RPT][C::CPT];

  for (int64_t t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
    int s = 0;
    while (s + 1 < P.nseg && P.seg[s + 1].tile0 <= t) ++s;
    const TsqrSeg& sg = P.seg[s];
    const int64_t row0 = (t - sg.tile0) * C::B;
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
      const int64_t row = row0 + i * C::TR + r;
#pragma unroll
      for (int q = 0; q < C::CPT; ++q) {
        const int lc = col_of<C>(q, c) - sg.col_begin;
        X[i][q] = (row < sg.rows && lc >= 0 && lc < sg.cols)
                      ? __ldg(sg.data + row * sg.ld + lc)
                      : 0.0;
      }
    }

#pragma unroll
    for (int qb = 0; qb < C::CPT; ++qb) {
      for (int within = 0; within < C::TC; ++within) {
        const int k = qb * C::TC + within;
        const int ck = (qb & 1) ? C::TC - 1 - within : within;
        double* vb = vbuf + (k & 1) * C::B;
        if (c == ck) {
          double sig = 0.0;
#pragma unroll
          for (int i = 0; i < C::RPT; ++i) sig = fma(X[i][qb], X[i][qb], sig);
          sig = group_sum<C>(sig, gmask);
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
          double d = 0.0;
#pragma unroll
          for (int i = 0; i < C::RPT; ++i) d = fma(v[i], X[i][q], d);
          d = group_sum<C>(d, gmask);
          const double f = tau * (d + rkj);
#pragma unroll
          for (int i = 0; i < C::RPT; ++i) X[i][q] = fma(-f, v[i], X[i][q]);
          __syncwarp(gmask);
          if (r == 0) R[k * C::W + j] = rkj - f;
        }
      }
    }
    __syncthreads();
  }
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

using C4 = Cfg<4, 4, 32, 4>;
using C8 = Cfg<8, 4, 32, 4>;
using C16 = Cfg<16, 8, 16, 8>;
using C32 = Cfg<32, 16, 16, 4>;
using C64 = Cfg<64, 32, 8, 8>;
using C128 = Cfg<128, 32, 8, 8>;

int bucket(int w) {
  for (int b : {4, 8, 16, 32, 64, 128})
    if (w <= b) return b;
  return 0;
}

template <class C>
size_t smem_bytes() {
  return sizeof(double) * (C::W * C::W + 2 * C::B + 2);
}

template <class C>
int tile_rows() { return C::B; }

int tile_rows_for(int W) {
  switch (W) {
    case 4: return C4::B;
    case 8: return C8::B;
    case 16: return C16::B;
    case 32: return C32::B;
    case 64: return C64::B;
    default: return C128::B;
  }
}

template <class C>
int max_ctas(Context& ctx) {
  const size_t smem = smem_bytes<C>();
  FG_CUDA(cudaFuncSetAttribute(k_tsqr<C>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tsqr<C>,
                                                        C::NT, smem));
  return std::max(1, per_sm) * ctx.sm_count;
}

template <class C>
void launch(Context& ctx, const TsqrParams& p, int grid, double* out) {
  k_tsqr<C><<<grid, C::NT, smem_bytes<C>(), ctx.stream>>>(p, out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

int max_ctas_for(Context& ctx, int W) {
  switch (W) {
    case 4: return max_ctas<C4>(ctx);
    case 8: return max_ctas<C8>(ctx);
    case 16: return max_ctas<C16>(ctx);
    case 32: return max_ctas<C32>(ctx);
    case 64: return max_ctas<C64>(ctx);
    default: return max_ctas<C128>(ctx);
  }
}

void launch_for(Context& ctx, int W, const TsqrParams& p, int grid,
                double* out) {
  switch (W) {
    case 4: launch<C4>(ctx, p, grid, out); break;
    case 8: launch<C8>(ctx, p, grid, out); break;
    case 16: launch<C16>(ctx, p, grid, out); break;
    case 32: launch<C32>(ctx, p, grid, out); break;
    case 64: launch<C64>(ctx, p, grid, out); break;
    default: launch<C128>(ctx, p, grid, out); break;
  }
}

// A factor produced by one launch: `count` W x W matrices at `data`, whose
// meaningful width is `cols`, placed at `col_begin`.
struct Partial {
  const double* data;
  int count;
  int W;
  int cols;
  int col_begin;
};

// Factors a list of segments (all with the same bucket W); a CTA takes about
// `tiles_per_cta` tiles.  Returns the number of W x W partial factors.
int factor_segments(Context& ctx, int W, const std::vector<TsqrSeg>& segs,
                    int64_t tiles_per_cta, DevArray<double>& out) {
  const int B = tile_rows_for(W);
  const int cap = max_ctas_for(ctx, W);
  std::vector<TsqrParams> plans;
  std::vector<int> grids;
  int total = 0;
  for (size_t i = 0; i < segs.size();) {
    TsqrParams p{};
    int64_t tiles = 0;
    int n = 0;
    for (; i < segs.size() && n < kMaxSegs; ++i) {
      TsqrSeg s = segs[i];
      s.tile0 = tiles;
      tiles += ceil_div(s.rows, B);
      p.seg[n++] = s;
    }
    p.nseg = n;
    p.total_tiles = tiles;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>(cap, ceil_div(tiles, tiles_per_cta)));
    plans.push_back(p);
    grids.push_back(grid);
    total += grid;
  }
  out.alloc((size_t)total * W * W, ctx.stream);
  double* o = out.get();
  for (size_t l = 0; l < plans.size(); ++l) {
    launch_for(ctx, W, plans[l], grids[l], o);
    o += (int64_t)grids[l] * W * W;
  }
  return total;
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
    TsqrSeg seg{s.data, s.rows, s.ld, s.cols, 0, 0};
    const int cnt = factor_segments(ctx, W, {seg}, 4, out);
    parts.push_back({out.get(), cnt, W, s.cols, s.col_begin});
    keep.push_back(std::move(out));
  }

  // Merge levels in the n-wide space until a single factor remains.
  while (true) {
    int total = 0;
    for (const Partial& p : parts) total += p.count;
    if (total == 1 && parts[0].W == WN && parts[0].col_begin == 0) break;
    if (total == 0) break;
    std::vector<TsqrSeg> segs;
    for (const Partial& p : parts)
      for (int k = 0; k < p.count; ++k)
        segs.push_back({p.data + (int64_t)k * p.W * p.W, p.cols, p.W, p.cols,
                        p.col_begin, 0});
    // Roughly 8 partial factors per CTA.
    DevArray<double> out;
    const int cnt = factor_segments(ctx, WN, segs, 8, out);
    parts.clear();
    parts.push_back({out.get(), cnt, WN, n, 0});
    keep.push_back(std::move(out));
  }

  const int threads = 256;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(
                                                   ceil_div((int64_t)n * n, threads), 64));
  if (parts.empty()) {
    FG_CUDA(cudaMemsetAsync(R_out, 0, sizeof(double) * n * n, ctx.stream));
    return;
  }
  k_normalize<<<blocks, threads, 0, ctx.stream>>>(parts[0].data, WN, n, R_out);
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

}  // namespace fg
