// Dependent-chain latencies on the B200 (one warp, clock64 deltas):
// DFMA, DADD, SHFL (f64 xor), DMMA m8n8k4, LDS f64, bar.sync (8 warps),
// MUFU-based sqrt/div sequences.  Used to size the TSQR dependency chains.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void probe(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  double x = a + lane * 1e-9;
  long long t0, t1;
  if (threadIdx.x < 64) sm[threadIdx.x] = x;
  __syncthreads();
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, a, b);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x + b;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // SHFL xor + add chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // DMMA chain (accumulator dependency)
  double c0 = x, c1 = x;
  t0 = clock64();
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  x += c0 + c1;
  // LDS dependent chain (index from value)
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    double v = sm[idx & 63];
    idx = (int)v & 63;
    x += v * 1e-30;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // bar.sync with the whole CTA
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // sqrt + div chain
  t0 = clock64();
  for (int i = 0; i < N / 8; ++i) x = 1.0 / sqrt(x * x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) * 8;
  out[threadIdx.x] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 64);
  probe<<<1, 256>>>(out, cyc, 0.999, 1e-3);
  probe<<<1, 256>>>(out, cyc, 0.999, 1e-3);
  long long h[8];
  cudaMemcpy(h, cyc, sizeof(long long) * 7, cudaMemcpyDeviceToHost);
  printf("{\"dfma\": %.1f, \"dadd\": %.1f, \"shfl_add\": %.1f, \"dmma\": %.1f, "
         "\"lds\": %.1f, \"bar_sync_256\": %.1f, \"rsqrt_div_seq\": %.1f, \"err\": \"%s\"}\n",
         h[0] / (double)N, h[1] / (double)N, h[2] / (double)N, h[3] / (double)N,
         h[4] / (double)N, h[5] / (double)N, h[6] / (double)N,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
