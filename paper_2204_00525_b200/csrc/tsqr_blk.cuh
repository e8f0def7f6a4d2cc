// Blocked TSQR leaf for wide spans (W = 32, 64): Householder panels of 8
// columns factored by one warp in registers (tsqr_warp.cuh, shuffles only,
// no CTA barrier per column), and the GEMM-shaped trailing update applied as
// a compact-WY block reflector on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64).
//
// Per 128-row tile X (shared memory) and the CTA's accumulator R (shared):
//   for each panel P = [p0, p0+8):
//     warp 0: structured QR of [R_PP; X_P] (the LAPACK tpqrt shape of
//             tsqr.cu), recording every reflector H_k = I - t1 t2 v v^T with
//             v = [u0 e_k; y_k]; the vectors are rescaled to
//             v~ = sqrt(t1 t2) v so that H_k = I - v~ v~^T, then
//             G = Y~^T Y~ (DMMA) and the forward T (H_0..H_7 = I - V T V^T,
//             T[k][k] = 1, T[0:k,k] = -T[0:k,0:k] G[0:k,k]);
//     all warps, one 8-column block J each:
//             W  = Y~^T X_J + diag(u0~) R_PJ          (DMMA, K = 128)
//             W' = T^T W                              (DMMA)
//             R_PJ -= diag(u0~) W',  X_J -= Y~ W'      (DMMA)
// i.e. [R_J; X_J] <- (I - V T^T V^T) [R_J; X_J] = H_7 ... H_0 [R_J; X_J],
// the same transformation the column-by-column kernel applies.  7/8 of the
// flops of a 64-wide tile run on DMMA.
#pragma once

#include <cuda_pipeline.h>

#include "tsqr_warp.cuh"

namespace fg {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int W_, int B_ = 128>
struct BCfg {
  static constexpr int W = W_;
  static constexpr int NP = W / 8;   // panels
  static constexpr int B = B_;       // rows per tile
  static constexpr int MINB = B_ >= 128 ? 1 : 2;
  static constexpr int WARPS = 8;
  static constexpr int NT = 32 * WARPS;
  // Row strides = 4 (mod 8) doubles: the panel loads (8 rows x 4 adjacent
  // columns) and the DMMA fragment loads (4 rows x 8 columns) spread over
  // the banks.
  static constexpr int LDX = W + 4;
  static constexpr int LDR = W + 4;
  using P = WCfg<8, 2, B_ / 8, 1>;   // panel layout: TC = 4, TR = 8, B rows
  static_assert(P::B == B, "panel rows");
  static constexpr size_t smem_doubles =
      (size_t)W * LDR + (size_t)B * LDX + 24 + 8 + 64 + 64 + 64 * WARPS;
  static constexpr size_t smem_bytes = smem_doubles * 8 + B * sizeof(int);
};

// cp.async of tile t (rows t*B ..) into X (row stride LDX), zero outside a
// segment's column range; rowseg: scratch of B ints.
template <class C, class Seg>
__device__ __forceinline__ void stage_blk(const Seg* __restrict__ segs, int nseg,
                                          int64_t total_rows, int64_t t, double* X,
                                          int* rowseg) {
  const int64_t r0 = t * C::B;
  for (int row = threadIdx.x; row < C::B; row += C::NT) {
    const int64_t gr = r0 + row;
    int s = -1;
    if (gr < total_rows) {
      int lo = 0, hi = nseg;
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
    double* dst = X + row * C::LDX + col;
    const int s = rowseg[row];
    if (s >= 0) {
      const Seg& sg = segs[s];
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

template <class C, class Seg>
__global__ void __launch_bounds__(256, C::MINB)
    k_tsqr_blk(const Seg* __restrict__ segs, int nseg, int64_t total_rows,
               int64_t total_tiles, int64_t nunits, double* __restrict__ out) {
  constexpr int W = C::W;
  using P = typename C::P;
  extern __shared__ __align__(16) double sm[];
  double* R = sm;                        // W x LDR
  double* X = R + W * C::LDR;            // B x LDX
  double* rec = X + C::B * C::LDX;       // 8 x {u0, t1, t2}
  double* ut = rec + 24;                 // 8: scaled u0
  double* G = ut + 8;                    // 8 x 8
  double* T = G + 64;                    // 8 x 8
  double* scr = T + 64;                  // 64 per warp
  int* rowseg = reinterpret_cast<int*>(scr + 64 * C::WARPS);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my = scr + 64 * warp;
  const int g = lane >> 2, tg = lane & 3;  // DMMA fragment coordinates

  for (int e = threadIdx.x; e < W * C::LDR; e += C::NT) R[e] = 0.0;

  for (int64_t t = blockIdx.x; t < total_tiles; t += nunits) {
    __syncthreads();  // the previous tile is done with X
    stage_blk<C>(segs, nseg, total_rows, t, X, rowseg);
    __pipeline_wait_prior(0);
    __syncthreads();
    for (int p = 0; p < C::NP; ++p) {
      const int p0 = 8 * p;
      if (warp == 0) {
        // Panel: structured QR of [R_PP; X_P] in registers.
        const int r = lane % P::TR, c = lane / P::TR;
        int cols[P::CPT];
#pragma unroll
        for (int q = 0; q < P::CPT; ++q) cols[q] = wcol<P>(q, c);
        double Xp[P::RPT][P::CPT];
        double Racc[P::RR][P::CPT];
#pragma unroll
        for (int i = 0; i < P::RPT; ++i)
#pragma unroll
          for (int q = 0; q < P::CPT; ++q)
            Xp[i][q] = X[(i * P::TR + r) * C::LDX + p0 + cols[q]];
#pragma unroll
        for (int q = 0; q < P::CPT; ++q) Racc[0][q] = R[(p0 + r) * C::LDR + p0 + cols[q]];
        absorb_tile_rec<P>(Xp, Racc, r, c, cols, rec);
        __syncwarp();
        double sc[P::CPT];
#pragma unroll
        for (int q = 0; q < P::CPT; ++q)
          sc[q] = sqrt(rec[3 * cols[q] + 1]) * sqrt(rec[3 * cols[q] + 2]);
#pragma unroll
        for (int i = 0; i < P::RPT; ++i)
#pragma unroll
          for (int q = 0; q < P::CPT; ++q)
            X[(i * P::TR + r) * C::LDX + p0 + cols[q]] = Xp[i][q] * sc[q];
#pragma unroll
        for (int q = 0; q < P::CPT; ++q) R[(p0 + r) * C::LDR + p0 + cols[q]] = Racc[0][q];
        if (lane < 8)
          ut[lane] = rec[3 * lane] * (sqrt(rec[3 * lane + 1]) * sqrt(rec[3 * lane + 2]));
        __syncwarp();
        if (p + 1 < C::NP) {
          // G = Y~^T Y~ over the tile rows (four independent chains).
          double ga[4] = {0, 0, 0, 0}, gb[4] = {0, 0, 0, 0};
#pragma unroll
          for (int kk = 0; kk < C::B / 4; ++kk) {
            const double a = X[(4 * kk + tg) * C::LDX + p0 + g];
            dmma(ga[kk & 3], gb[kk & 3], a, a);
          }
          G[g * 8 + 2 * tg] = (ga[0] + ga[1]) + (ga[2] + ga[3]);
          G[g * 8 + 2 * tg + 1] = (gb[0] + gb[1]) + (gb[2] + gb[3]);
          __syncwarp();
          if (lane < 8) {
            // Row `lane` of T.
            double Tr[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) Tr[k] = k == lane ? 1.0 : 0.0;
#pragma unroll
            for (int k = 1; k < 8; ++k) {
              double s = 0.0;
#pragma unroll
              for (int j = 0; j < k; ++j)
                if (j >= lane) s = fma(Tr[j], G[j * 8 + k], s);
              if (lane < k) Tr[k] = -s;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) T[lane * 8 + k] = Tr[k];
          }
        }
      }
      __syncthreads();
      if (p + 1 < C::NP) {
        for (int j = p + 1 + warp; j < C::NP; j += C::WARPS) {
          const int J0 = 8 * j;
          double wa[4] = {0, 0, 0, 0}, wb[4] = {0, 0, 0, 0};
#pragma unroll
          for (int kk = 0; kk < C::B / 4; ++kk) {
            const double* row = X + (4 * kk + tg) * C::LDX;
            dmma(wa[kk & 3], wb[kk & 3], row[p0 + g], row[J0 + g]);
          }
          const double u = ut[g];
          double* rp = R + (p0 + g) * C::LDR + J0 + 2 * tg;
          const double r0 = rp[0], r1 = rp[1];
          my[g * 8 + 2 * tg] = fma(u, r0, (wa[0] + wa[1]) + (wa[2] + wa[3]));
          my[g * 8 + 2 * tg + 1] = fma(u, r1, (wb[0] + wb[1]) + (wb[2] + wb[3]));
          __syncwarp();
          double v0 = 0.0, v1 = 0.0;
          dmma(v0, v1, T[tg * 8 + g], my[tg * 8 + g]);
          dmma(v0, v1, T[(4 + tg) * 8 + g], my[(4 + tg) * 8 + g]);
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
            double c0 = row[J0 + 2 * tg], c1 = row[J0 + 2 * tg + 1];
            dmma(c0, c1, -row[p0 + tg], b0);
            dmma(c0, c1, -row[p0 + 4 + tg], b1);
            row[J0 + 2 * tg] = c0;
            row[J0 + 2 * tg + 1] = c1;
          }
          __syncwarp();
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  double* o = out + (int64_t)blockIdx.x * W * W;
  for (int e = threadIdx.x; e < W * W; e += C::NT) {
    const int i = e / W, j = e - (e / W) * W;
    o[e] = R[i * C::LDR + j];
  }
}

}  // namespace fg
