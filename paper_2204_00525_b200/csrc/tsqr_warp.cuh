// Warp-level structured Householder core shared by the TSQR kernels
// (tsqr.cu) and the fused heads/tails -> TSQR kernel (headtail.cu).
#pragma once

#include "fg_internal.cuh"

namespace fg {

// 1/sqrt(q) and 1/q from the MUFU approximations plus two Newton steps
// (relative error ~1e-16; the IEEE sqrt+div sequence costs ~184 cycles of
// latency on B200, this ~60).
__device__ __forceinline__ double fast_rsqrt(double q) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  const double hq = 0.5 * q;
  r = r * fma(-hq * r, r, 1.5);
  r = r * fma(-hq * r, r, 1.5);
  return r;
}
__device__ __forceinline__ double fast_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = r * fma(-q, r, 2.0);
  r = r * fma(-q, r, 2.0);
  return r;
}

// Householder reflector of column k with pivot alpha and tail norm^2 sig in
// the unnormalised form H = I - tau * u u^T, u = [alpha - beta; x]:
//   beta = -sign(alpha) * nrm,  nrm = ||(alpha, x)||,
//   tau  = 1 / (nrm * (nrm + |alpha|)) = t1 * t2,
// kept as the two bounded factors t1 = 1/nrm and t2 = 1/(nrm + |alpha|)
// (tau itself overflows for numerically zero columns, nrm < 1e-154).
// Callers form g = (d * t1) * t2.  t1 = t2 = 0 when the tail is zero
// (H = I, beta = alpha).
struct Reflector {
  double beta, u0, t1, t2;
};
__device__ __forceinline__ Reflector make_reflector(double alpha, double sig) {
  Reflector h;
  const double q = fma(alpha, alpha, sig);
  const bool live = sig > 0.0;
  const double aa = fabs(alpha);
  double nrm, t1, t2;
  if (q > 1e-250 && q < 1e250) {
    // The .ftz approximations flush subnormals: only inside a safe range.
    t1 = fast_rsqrt(q);
    nrm = q * t1;
    t2 = fast_rcp(nrm + aa);
  } else {
    nrm = sqrt(q);
    t1 = 1.0 / nrm;
    t2 = 1.0 / (nrm + aa);
  }
  h.beta = live ? (alpha >= 0.0 ? -nrm : nrm) : alpha;
  h.u0 = alpha - h.beta;
  h.t1 = live ? t1 : 0.0;
  h.t2 = live ? t2 : 0.0;
  return h;
}

// The same for callers whose whole warp holds identical (alpha, sig) -- the
// register kernels broadcast both -- so the range test is a warp vote and
// the branch is uniform.
__device__ __forceinline__ Reflector make_reflector_warp(double alpha, double sig) {
  Reflector h;
  const double q = fma(alpha, alpha, sig);
  const bool live = sig > 0.0;
  const double aa = fabs(alpha);
  double nrm, t1, t2;
  if (__all_sync(0xffffffffu, q > 1e-250 && q < 1e250)) {
    t1 = fast_rsqrt(q);
    nrm = q * t1;
    t2 = fast_rcp(nrm + aa);
  } else {
    nrm = sqrt(q);
    t1 = 1.0 / nrm;
    t2 = 1.0 / (nrm + aa);
  }
  h.beta = live ? (alpha >= 0.0 ? -nrm : nrm) : alpha;
  h.u0 = alpha - h.beta;
  h.t1 = live ? t1 : 0.0;
  h.t2 = live ? t2 : 0.0;
  return h;
}

#ifndef FG_NCH
#define FG_NCH 4
#endif
#ifndef FG_ABSORB_OVL
#define FG_ABSORB_OVL 1
#endif
// ROLL_ = 1 keeps only the column-block loop unrolled in absorb_tile (the
// TC steps inside a block run as a loop): ~1/TC of the code, for kernels
// whose straight-line body overflows the instruction cache.
template <int W_, int CPT_, int RPT_, int MINB_ = 1, int ROLL_ = 0, int WARPS_ = 8>
struct WCfg {
  static constexpr int W = W_;
  static constexpr int CPT = CPT_;
  static constexpr int TC = W / CPT;
  static constexpr int TR = 32 / TC;
  static constexpr int RPT = RPT_;
  static constexpr int B = TR * RPT;
  static constexpr int RR = (W + TR - 1) / TR;  // accumulator rows per lane
  static constexpr int WARPS = WARPS_;
  static constexpr int NT = 32 * WARPS;
  static constexpr int MINB = MINB_;
  static constexpr int ROLL = ROLL_;
  static constexpr size_t smem_bytes = 0;
  static_assert(TC * TR == 32, "TC * TR must be a warp");
};

template <class C>
__device__ __forceinline__ int wcol(int q, int c) {
  return (q & 1) ? (q + 1) * C::TC - 1 - c : q * C::TC + c;
}

template <class C>
__device__ __forceinline__ double wgroup_sum(double x) {
#pragma unroll
  for (int o = C::TR / 2; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Sequential form of absorb_step: the dots are reduced after the reflector
// (u0 * R_kq folded in before the reduction) -- fewer live registers.
template <class C, int QB, bool REC = false>
__device__ __forceinline__ void absorb_step_seq(double (&X)[C::RPT][C::CPT],
                                            double (&Racc)[C::RR][C::CPT],
                                            int r, int c, const int (&cols)[C::CPT],
                                            int within, double* rec = nullptr) {
  const int k = QB * C::TC + within;
  const int ck = (QB & 1) ? C::TC - 1 - within : within;
  const int rk = k % C::TR;   // lane row holding accumulator row k
  const int mk = k / C::TR;
  constexpr int NCH = FG_NCH < C::RPT ? FG_NCH : C::RPT;
  double v[C::RPT];
  double sa[NCH];
#pragma unroll
  for (int i = 0; i < C::RPT; ++i) {
    v[i] = __shfl_sync(0xffffffffu, X[i][QB], r + ck * C::TR);
    if (i < NCH) sa[i] = v[i] * v[i];
    else sa[i % NCH] = fma(v[i], v[i], sa[i % NCH]);
  }
#pragma unroll
  for (int w = NCH / 2; w; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) sa[i] += sa[i + w];
  const double sig = wgroup_sum<C>(sa[0]);
  // Racc[mk][q] for a possibly run-time mk: a select chain over RR rows.
  auto racc = [&](int q) {
    double x = Racc[0][q];
#pragma unroll
    for (int m = 1; m < C::RR; ++m)
      if (mk == m) x = Racc[m][q];
    return x;
  };
  const double alpha = __shfl_sync(0xffffffffu, racc(QB), rk + ck * C::TR);
  const Reflector h = make_reflector_warp(alpha, sig);
  if constexpr (REC) {
    // Reflector k for the caller's block update: {u0, t1, t2}.
    if ((threadIdx.x & 31) == 0) {
      rec[3 * k] = h.u0;
      rec[3 * k + 1] = h.t1;
      rec[3 * k + 2] = h.t2;
    }
  }
#pragma unroll
  for (int q = QB; q < C::CPT; ++q) {
    // Slots past the pivot block hold only columns > k.
    const bool act = q > QB || cols[q] > k;
    double da[NCH];
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
      if (i < NCH) da[i] = v[i] * X[i][q];
      else da[i % NCH] = fma(v[i], X[i][q], da[i % NCH]);
    }
#pragma unroll
    for (int w = NCH / 2; w; w >>= 1)
#pragma unroll
      for (int i = 0; i < w; ++i) da[i] += da[i + w];
    double d = da[0];
    const double rq = racc(q);
    if (r == rk) d = fma(h.u0, rq, d);
    const double dsum = wgroup_sum<C>(d);  // all lanes shuffle
    const double f = act ? (dsum * h.t1) * h.t2 : 0.0;
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) X[i][q] = fma(-f, v[i], X[i][q]);
    if (r == rk) {
      const double nr = (q == QB && c == ck) ? h.beta : fma(-f, h.u0, rq);
#pragma unroll
      for (int m = 0; m < C::RR; ++m)
        if (mk == m) Racc[m][q] = nr;
    }
  }
}

// One column step k of absorb_tile; QB (the column block) is compile-time,
// the position inside the block may be a run-time value.
//
// Critical path per column: broadcast of column k (RPT shuffles), the
// squared norm and every trailing dot product x . X_q reduced TOGETHER in
// one xor tree (independent shuffles, so the latencies overlap), the
// reflector, and the update.  The pivot-row term u0 * R_kq of each dot
// (u0 = alpha - beta is known only after the reflector) is added after the
// reduction from a broadcast of accumulator row k that does not depend on
// this column's data.
template <class C, int QB, bool REC = false>
__device__ __forceinline__ void absorb_step(double (&X)[C::RPT][C::CPT],
                                            double (&Racc)[C::RR][C::CPT],
                                            int r, int c, const int (&cols)[C::CPT],
                                            int within, double* rec = nullptr) {
  // FG_ABSORB_OVL: 0 sequential everywhere, 1 overlapped everywhere,
  // 2 overlapped where registers allow (one CTA per SM, MINB == 1).
  if constexpr (FG_ABSORB_OVL == 0 || (FG_ABSORB_OVL == 2 && C::MINB != 1)) {
    absorb_step_seq<C, QB, REC>(X, Racc, r, c, cols, within, rec);
    return;
  }
  const int k = QB * C::TC + within;
  const int ck = (QB & 1) ? C::TC - 1 - within : within;
  const int rk = k % C::TR;   // lane row holding accumulator row k
  const int mk = k / C::TR;
  constexpr int NCH = FG_NCH < C::RPT ? FG_NCH : C::RPT;
  constexpr int NQ = C::CPT - QB;  // slots holding columns >= the pivot block
  // Racc[mk][q] for a possibly run-time mk: a select chain over RR rows.
  auto racc = [&](int q) {
    double x = Racc[0][q];
#pragma unroll
    for (int m = 1; m < C::RR; ++m)
      if (mk == m) x = Racc[m][q];
    return x;
  };
  // Accumulator row k, slot q, as seen by every lane of column group c.
  double rk_q[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) rk_q[j] = __shfl_sync(0xffffffffu, racc(QB + j), rk + c * C::TR);
  const double alpha = __shfl_sync(0xffffffffu, racc(QB), rk + ck * C::TR);
  double v[C::RPT];
  double sa[NCH];
#pragma unroll
  for (int i = 0; i < C::RPT; ++i) {
    v[i] = __shfl_sync(0xffffffffu, X[i][QB], r + ck * C::TR);
    if (i < NCH) sa[i] = v[i] * v[i];
    else sa[i % NCH] = fma(v[i], v[i], sa[i % NCH]);
  }
  double red[NQ + 1];
#pragma unroll
  for (int w = NCH / 2; w; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) sa[i] += sa[i + w];
  red[NQ] = sa[0];
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    double da[NCH];
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
      if (i < NCH) da[i] = v[i] * X[i][QB + j];
      else da[i % NCH] = fma(v[i], X[i][QB + j], da[i % NCH]);
    }
#pragma unroll
    for (int w = NCH / 2; w; w >>= 1)
#pragma unroll
      for (int i = 0; i < w; ++i) da[i] += da[i + w];
    red[j] = da[0];
  }
#pragma unroll
  for (int o = C::TR / 2; o; o >>= 1)
#pragma unroll
    for (int j = 0; j <= NQ; ++j) red[j] += __shfl_xor_sync(0xffffffffu, red[j], o);
  const Reflector h = make_reflector_warp(alpha, red[NQ]);
  if constexpr (REC) {
    // Reflector k for the caller's block update: {u0, t1, t2}.
    if ((threadIdx.x & 31) == 0) {
      rec[3 * k] = h.u0;
      rec[3 * k + 1] = h.t1;
      rec[3 * k + 2] = h.t2;
    }
  }
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int q = QB + j;
    // Slots past the pivot block hold only columns > k.
    const bool act = q > QB || cols[q] > k;
    const double dsum = fma(h.u0, rk_q[j], red[j]);
    const double f = act ? (dsum * h.t1) * h.t2 : 0.0;
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) X[i][q] = fma(-f, v[i], X[i][q]);
    if (r == rk) {
      const double nr = (q == QB && c == ck) ? h.beta : fma(-f, h.u0, rk_q[j]);
#pragma unroll
      for (int m = 0; m < C::RR; ++m)
        if (mk == m) Racc[m][q] = nr;
    }
  }
}

template <class C, int QB, bool REC = false>
__device__ __forceinline__ void absorb_blocks(double (&X)[C::RPT][C::CPT],
                                              double (&Racc)[C::RR][C::CPT],
                                              int r, int c, const int (&cols)[C::CPT],
                                              double* rec = nullptr) {
  if constexpr (QB < C::CPT) {
    if constexpr (C::ROLL) {
#pragma unroll 1
      for (int within = 0; within < C::TC; ++within)
        absorb_step<C, QB, REC>(X, Racc, r, c, cols, within, rec);
    } else {
#pragma unroll
      for (int within = 0; within < C::TC; ++within)
        absorb_step<C, QB, REC>(X, Racc, r, c, cols, within, rec);
    }
    absorb_blocks<C, QB + 1, REC>(X, Racc, r, c, cols, rec);
  }
}

// Absorbs one B x W tile (X, lane layout above) into the accumulator rows
// Racc: the W column steps of the structured Householder QR of [R; X]
// (postprocess.hpp:35-64 shape, LAPACK tpqrt), register code.
template <class C>
__device__ __forceinline__ void absorb_tile(double (&X)[C::RPT][C::CPT],
                                            double (&Racc)[C::RR][C::CPT],
                                            int r, int c, const int (&cols)[C::CPT]) {
  absorb_blocks<C, 0>(X, Racc, r, c, cols);
}

// Same, recording every reflector {u0, t1, t2} in rec[3k..3k+2] (lane 0).
template <class C>
__device__ __forceinline__ void absorb_tile_rec(double (&X)[C::RPT][C::CPT],
                                                double (&Racc)[C::RR][C::CPT],
                                                int r, int c, const int (&cols)[C::CPT],
                                                double* rec) {
  absorb_blocks<C, 0, true>(X, Racc, r, c, cols, rec);
}

}  // namespace fg
