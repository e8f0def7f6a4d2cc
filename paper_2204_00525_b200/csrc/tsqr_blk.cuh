// Helpers of the blocked TSQR kernels (tsqr_la.cuh): the FP64 tensor-core
// MMA (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4) and the general tile staging
// (per-row segment lookup, zero fill outside a segment's column range).
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

}  // namespace fg
