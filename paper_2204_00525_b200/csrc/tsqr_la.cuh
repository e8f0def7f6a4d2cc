// Blocked TSQR for wide spans (W = 32 .. 128) with look-ahead: one
// accumulator R per CTA, panels of 8 columns factored by warp 0 in
// registers, the trailing update on the FP64 tensor cores (DMMA m8n8k4).
//
// Reference: triangularize_block / the THIN absorb (postprocess.hpp:35-169);
// the transformation is the structured Householder QR of [R; X] (LAPACK
// tpqrt: reflector k touches row k of R and the B tile rows), as in tsqr.cu.
//
// Schedule per B-row tile (X in shared memory):
//   stage the tile (cp.async; 16-byte copies when it lies inside one dense
//   segment; NBUF = 2 stages the next tile while this one is factored);
//   warp 0 factors panel 0;                                         barrier
//   for p = 0 .. NP-1:
//     warp 0     : block p+1 -= panel p (DMMA), then factors panel p+1
//     warps 1..  : blocks p+2 .. NP-1 -= panel p (DMMA)            barrier
// so the serial panel chain overlaps the tensor-core work of the previous
// panel instead of leaving the other warps at a barrier.  A panel whose tile
// columns are exactly zero (stacked triangular factors in merge levels) is
// the identity and is skipped together with the block updates it drives.
// The default configurations (tsqr.cu) are single-buffered with 64-row
// tiles; for large spans R is kept as upper-triangular 8 x 8 blocks (RTRI)
// so that 2-warp CTAs fit 4 per SM at W = 64.
//
// Panel (warp 0): lane (g, t) = (lane / 4, lane % 4) owns panel column g
// and tile rows 4i + t (the "quad" layout; the same registers are the A
// operand of the V^T X products).  A column step is one broadcast of the
// pivot column, one product pass and one two-level quad reduction: the pivot
// quad's product is the exact pivot norm, quads right of it get the update
// dots, quads left of it V^T v_k for the block reflector.  The next
// reflector comes from downdated norms (sigma' = sigma - 2 f p + f^2
// sigma_k) so its rsqrt latency overlaps the next product pass; a downdate
// that lost two bits, or a pivot outside the fast exponent range, is
// repaired after the next reduction (warp-uniform, rare).
// Reflectors are H_k = I - s_k^2 u u^T, u = [alpha - beta; x]; the block
// reflector uses u~ = s_k u so that H_0 ... H_7 = I - U~ T U~^T, unit-diagonal
// T (T[g][k] = -sum_j T[g][j] G~[j][k], G~ = U~^T U~), built inside the
// column loop from the same reductions.
//
// Trailing block J against panel P (one warp):
//   Y = U~^T [R_PJ; X_J]  (DMMA, K = tile rows),  W' = T^T Y,
//   R_PJ -= diag(u0~) W',  X_J -= V~ W'.
#pragma once

#include <cuda_pipeline.h>

#include "tsqr_blk.cuh"

namespace fg {

template <int W_, int B_, int WARPS_, int MINB_, int NBUF_ = 2, int RTRI_ = 0>
struct LCfg {
  static constexpr int W = W_;
  static constexpr int NP = W / 8;
  static constexpr int B = B_;
  static constexpr int RPL = B / 4;  // panel rows per lane
  static constexpr int WARPS = WARPS_;
  static constexpr int NT = 32 * WARPS;
  static constexpr int MINB = MINB_;
  static constexpr int NBUF = NBUF_;  // 2: the next tile is staged during this one
  // RTRI = 1: R kept as its NP (NP + 1) / 2 upper-triangular 8 x 8 blocks
  // (half the shared memory of the padded square; more CTAs per SM).
  static constexpr int RTRI = RTRI_;
  static constexpr int LDX = W + 4;
  static constexpr int LDR = W + 4;
  static_assert(W % 8 == 0 && B % 8 == 0 && WARPS >= 2, "shape");
  static_assert(NBUF == 1 || NBUF == 2, "buffers");
  static constexpr size_t r_doubles = RTRI ? (size_t)NP * (NP + 1) / 2 * 64 : (size_t)W * LDR;
  static constexpr size_t smem_doubles =
      r_doubles + NBUF * (size_t)B * LDX + 2 * 64 + 2 * 8 + 64 * WARPS;
  static constexpr size_t smem_bytes = smem_doubles * 8 + B * sizeof(int);
};

// Reflector in the scaled form: beta, u0 = alpha - beta and
// s = 1 / sqrt(nrm (nrm + |alpha|)) (H = I - s^2 u u^T; s = 0: H = I).
struct SRefl {
  double beta, u0, s;
};
__device__ __forceinline__ SRefl srefl_fast(double alpha, double sig) {
  SRefl h;
  const double q = fma(alpha, alpha, sig);
  const bool live = sig > 0.0;
  const double nrm = q * fast_rsqrt(q);
  const double s = fast_rsqrt(nrm * (nrm + fabs(alpha)));
  h.beta = live ? (alpha >= 0.0 ? -nrm : nrm) : alpha;
  h.u0 = alpha - h.beta;
  h.s = live ? s : 0.0;
  return h;
}
__device__ __forceinline__ bool srefl_ok(double alpha, double sig) {
  const double q = fma(alpha, alpha, sig);
  return !(sig > 0.0) || (q > 1e-250 && q < 1e250);
}
__device__ __noinline__ SRefl srefl_ieee(double alpha, double sig) {
  SRefl h;
  const double q = fma(alpha, alpha, sig);
  const bool live = sig > 0.0;
  const double nrm = sqrt(q);
  h.beta = live ? (alpha >= 0.0 ? -nrm : nrm) : alpha;
  h.u0 = alpha - h.beta;
  h.s = live ? sqrt(1.0 / nrm) * sqrt(1.0 / (nrm + fabs(alpha))) : 0.0;
  return h;
}

// Stages tile `tile` into X.  Fast path (CTA-uniform): the tile lies inside
// one dense, 16-byte aligned segment -- 16-byte cp.async with row/column
// arithmetic only; otherwise the general per-row segment path of stage_blk.
template <class C, class Seg>
__device__ __forceinline__ void la_stage(const Seg* __restrict__ segs, int nseg,
                                         int64_t total_rows, int64_t tile, double* X,
                                         int* rowseg) {
  const int64_t r0 = tile * C::B;
  int lo = 0, hi = nseg;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (segs[mid].row0 <= r0) lo = mid; else hi = mid;
  }
  const Seg& sg = segs[lo];
  const bool fast = r0 + C::B <= sg.row0 + sg.rows && sg.col_begin == 0 && sg.cols == C::W &&
                    (sg.ld & 1) == 0 && (reinterpret_cast<uintptr_t>(sg.data) & 15) == 0;
  if (!fast) {
    stage_blk<C>(segs, nseg, total_rows, tile, X, rowseg);
    return;
  }
  constexpr int HW = C::W / 2;
  const double* base = sg.data + (r0 - sg.row0) * sg.ld;
  for (int e = threadIdx.x; e < C::B * HW; e += C::NT) {
    const int row = e / HW, c2 = e - (e / HW) * HW;
    __pipeline_memcpy_async(X + row * C::LDX + 2 * c2, base + row * sg.ld + 2 * c2,
                            2 * sizeof(double));
  }
  __pipeline_commit();
}

// Pointer to R[8p][8j] (j >= p) and the row stride of that block.
template <class C>
__device__ __forceinline__ double* rblock(double* R, int p, int j) {
  if constexpr (C::RTRI) return R + (p * C::NP - p * (p - 1) / 2 + (j - p)) * 64;
  else return R + 8 * p * C::LDR + 8 * j;
}
template <class C>
constexpr int rld() { return C::RTRI ? 8 : C::LDR; }

__device__ __forceinline__ double qsum_l(double x) {
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  return x;
}

// Trailing block J0 of tile X against panel p0 (one warp, DMMA):
// Y = U~^T [R_PJ; X_J], W' = T^T Y, R_PJ -= diag(u0~) W', X_J -= V~ W'.
template <class C>
__device__ __forceinline__ void dm_trailing(double* __restrict__ X, double* __restrict__ R,
                                            int p0, int J0, const double* __restrict__ Ts,
                                            const double* __restrict__ ut,
                                            double* __restrict__ my, int lane) {
  const int g = lane >> 2, tg = lane & 3;
  double wa[4] = {0, 0, 0, 0}, wb[4] = {0, 0, 0, 0};
#pragma unroll
  for (int kk = 0; kk < C::B / 4; ++kk) {
    const double* row = X + (4 * kk + tg) * C::LDX;
    dmma(wa[kk & 3], wb[kk & 3], row[p0 + g], row[J0 + g]);
  }
  const double u = ut[g];
  double* rp = rblock<C>(R, p0 / 8, J0 / 8) + g * rld<C>() + 2 * tg;
  const double r0 = rp[0], r1 = rp[1];
  my[g * 8 + 2 * tg] = fma(u, r0, (wa[0] + wa[1]) + (wa[2] + wa[3]));
  my[g * 8 + 2 * tg + 1] = fma(u, r1, (wb[0] + wb[1]) + (wb[2] + wb[3]));
  __syncwarp();
  double v0 = 0.0, v1 = 0.0;
  dmma(v0, v1, Ts[tg * 8 + g], my[tg * 8 + g]);
  dmma(v0, v1, Ts[(4 + tg) * 8 + g], my[(4 + tg) * 8 + g]);
  __syncwarp();
  rp[0] = fma(-u, v0, r0);
  rp[1] = fma(-u, v1, r1);
  my[g * 8 + 2 * tg] = v0;
  my[g * 8 + 2 * tg + 1] = v1;
  __syncwarp();
  const double b0 = my[tg * 8 + g], b1 = my[(4 + tg) * 8 + g];
#pragma unroll 4
  for (int mt = 0; mt < C::B / 8; ++mt) {
    double* row = X + (8 * mt + g) * C::LDX;
    double2 c = *reinterpret_cast<double2*>(row + J0 + 2 * tg);
    dmma(c.x, c.y, -row[p0 + tg], b0);
    dmma(c.x, c.y, -row[p0 + 4 + tg], b1);
    *reinterpret_cast<double2*>(row + J0 + 2 * tg) = c;
  }
  __syncwarp();
}

// Panel p0 of tile X against R (warp 0).  Leaves V~ in X's panel columns,
// the finished diagonal block in R, u0~ in ut and T in Ts.
// Returns true (warp-uniform) when the panel's tile columns are all exactly
// zero: every reflector is the identity, so the panel and every block update
// it drives are skipped (triangular partial factors stacked in merge levels).
template <class C>
__device__ __forceinline__ bool la_panel(double* __restrict__ X, double* __restrict__ R,
                                         int p0, double* __restrict__ Ts,
                                         double* __restrict__ ut, int lane) {
  constexpr int RPL = C::RPL;
  const int g = lane >> 2, t = lane & 3;
  double Xp[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) Xp[i] = X[(4 * i + t) * C::LDX + p0 + g];
  double Rd[8];  // R[p0 + i][p0 + g], replicated over the quad
#pragma unroll
  for (int i = 0; i < 8; ++i) Rd[i] = rblock<C>(R, p0 / 8, p0 / 8)[i * rld<C>() + g];
  // exact tail norms of the panel columns
  double sig;
  {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i < RPL; i += 2) {
      a0 = fma(Xp[i], Xp[i], a0);
      if (i + 1 < RPL) a1 = fma(Xp[i + 1], Xp[i + 1], a1);
    }
    sig = qsum_l(a0 + a1);
  }
  if (__all_sync(0xffffffffu, sig == 0.0)) return true;
  double smax = sig;
  double sk = __shfl_sync(0xffffffffu, sig, 0);
  double al = __shfl_sync(0xffffffffu, Rd[0], 0);
  SRefl h = srefl_fast(al, sk);
  bool redo_norm = false, redo_refl = !srefl_ok(al, sk);
  // Row g of T, built column by column: T[g][k] = -sum_{j<k} T[g][j] G~[j][k]
  // with G~[j][k] = s_j s_k v_j . v_k (the X parts; u~'s R parts are on
  // different rows), gathered from the quads' reductions of step k.
  double Tr[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) Tr[k] = k == g ? 1.0 : 0.0;
  double my_s = 0.0, my_u = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double v[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) v[i] = __shfl_sync(0xffffffffu, Xp[i], 4 * k + t);
    double a[4];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      if (i < 4) a[i] = v[i] * Xp[i];
      else a[i & 3] = fma(v[i], Xp[i], a[i & 3]);
    }
    const double dot = qsum_l((a[0] + a[1]) + (a[2] + a[3]));
    if (redo_norm || redo_refl) {
      if (redo_norm) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; i += 2) {
          a0 = fma(Xp[i], Xp[i], a0);
          if (i + 1 < RPL) a1 = fma(Xp[i + 1], Xp[i + 1], a1);
        }
        sig = qsum_l(a0 + a1);
        smax = sig;
        sk = __shfl_sync(0xffffffffu, sig, 4 * k);
      }
      h = srefl_ok(al, sk) ? srefl_fast(al, sk) : srefl_ieee(al, sk);
    }
    const bool right = g > k;
    const double f = right ? (fma(h.u0, Rd[k], dot) * h.s) * h.s : 0.0;
#pragma unroll
    for (int i = 0; i < RPL; ++i) Xp[i] = fma(-f, v[i], Xp[i]);
    Rd[k] = right ? fma(-f, h.u0, Rd[k]) : (g == k ? h.beta : Rd[k]);
    if (right) {
      sig = fma(f, fma(f, sk, -2.0 * dot), sig);
      smax = fmax(smax, sig);
    }
    if (k > 0) {
      const double gt = dot * h.s * my_s;  // G~[g][k], valid for g < k
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < k; ++j) acc = fma(Tr[j], __shfl_sync(0xffffffffu, gt, 4 * j), acc);
      if (g < k) Tr[k] = -acc;
    }
    if (g == k) {
      my_s = h.s;
      my_u = h.u0 * h.s;
    }
    if (k + 1 < 8) {
      sk = __shfl_sync(0xffffffffu, sig, 4 * (k + 1));
      const double sm = __shfl_sync(0xffffffffu, smax, 4 * (k + 1));
      al = __shfl_sync(0xffffffffu, Rd[k + 1], 4 * (k + 1));
      redo_norm = !(sk >= 0.25 * sm);
      redo_refl = !srefl_ok(al, sk);
      h = srefl_fast(al, sk);
    }
  }
#pragma unroll
  for (int i = 0; i < RPL; ++i) X[(4 * i + t) * C::LDX + p0 + g] = Xp[i] * my_s;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if ((i & 3) == t) rblock<C>(R, p0 / 8, p0 / 8)[i * rld<C>() + g] = Rd[i];
  if (t == 0) ut[g] = my_u;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if ((k & 3) == t) Ts[g * 8 + k] = Tr[k];
  __syncwarp();
  return false;
}

template <class C, class Seg>
__global__ void __launch_bounds__(C::NT, C::MINB)
    k_tsqr_la(const Seg* __restrict__ segs, int nseg, int64_t total_rows,
              int64_t total_tiles, int64_t nunits, double* __restrict__ out) {
  constexpr int W = C::W, NP = C::NP;
  extern __shared__ __align__(16) double sm[];
  double* R = sm;                                // W x LDR
  double* Xb0 = R + C::r_doubles;                // B x LDX (x NBUF)
  double* Xb1 = Xb0 + (C::NBUF - 1) * C::B * C::LDX;
  double* Tsb = Xb1 + C::B * C::LDX;             // 2 x (8 x 8), by panel parity
  double* utb = Tsb + 128;                       // 2 x 8
  __shared__ int zpan[2];                        // panel of parity pb is the identity
  double* scr = utb + 16;                        // 64 per warp
  int* rowseg = reinterpret_cast<int*>(scr + 64 * C::WARPS);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my = scr + 64 * warp;

  for (int e = threadIdx.x; e < (int)C::r_doubles; e += C::NT) R[e] = 0.0;

  int64_t tt = blockIdx.x;
  if (C::NBUF == 2 && tt < total_tiles) la_stage<C>(segs, nseg, total_rows, tt, Xb0, rowseg);
  int buf = 0;
  for (; tt < total_tiles; tt += nunits, buf ^= (C::NBUF - 1)) {
    double* X = buf ? Xb1 : Xb0;
    if (C::NBUF == 1) la_stage<C>(segs, nseg, total_rows, tt, X, rowseg);
    __pipeline_wait_prior(0);
    __syncthreads();  // tile tt staged; the other buffer is free
    if (C::NBUF == 2 && tt + nunits < total_tiles)
      la_stage<C>(segs, nseg, total_rows, tt + nunits, buf ? Xb0 : Xb1, rowseg);
    if (warp == 0) {
      const bool z = la_panel<C>(X, R, 0, Tsb, utb, lane);
      if (lane == 0) zpan[0] = z;
    }
    __syncthreads();
    for (int p = 0; p < NP; ++p) {
      const int pb = p & 1;
      double* Tp = Tsb + 64 * pb;
      double* up = utb + 8 * pb;
      const bool zp = zpan[pb];
      if (warp == 0) {
        if (p + 1 < NP) {
          if (!zp) dm_trailing<C>(X, R, 8 * p, 8 * (p + 1), Tp, up, my, lane);
          const bool z = la_panel<C>(X, R, 8 * (p + 1), Tsb + 64 * (pb ^ 1), utb + 8 * (pb ^ 1),
                                     lane);
          if (lane == 0) zpan[pb ^ 1] = z;
        }
      } else if (!zp) {
        for (int j = p + 1 + warp; j < NP; j += C::WARPS - 1)
          dm_trailing<C>(X, R, 8 * p, 8 * j, Tp, up, my, lane);
      }
      __syncthreads();
    }
  }
  __syncthreads();
  double* o = out + (int64_t)blockIdx.x * W * W;
  for (int e = threadIdx.x; e < W * W; e += C::NT) {
    const int i = e / W, j = e - (e / W) * W;
    o[e] = (j >> 3) < (i >> 3) ? 0.0 : rblock<C>(R, i >> 3, j >> 3)[(i & 7) * rld<C>() + (j & 7)];
  }
}

}  // namespace fg
