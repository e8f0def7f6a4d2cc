// FP64 peak microbenchmark for the TSQR roofline denominator (B200 has no
// FP64 entry in MEASURED_PEAKS.json).  Measures dense DFMA (vector pipe) and
// DMMA m8n8k4 (mma.sync f64, the FP64 tensor path on sm_100a) throughput over
// all SMs with CUDA events.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 16;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
          "{%0,%1};\n"
          : "+d"(c[i][0]), "+d"(c[i][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256;
  const int blocks = sms * 8;
  const int iters = 4096;
  float best_dfma = 1e30f, best_dmma = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_dfma = ms < best_dfma ? ms : best_dfma;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters / 4, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_dmma = ms < best_dmma ? ms : best_dmma;
  }
  const double dfma_flops = 2.0 * kChains * (double)iters * blocks * threads;
  // m8n8k4: 8*8*4 FMA per warp instruction.
  const double dmma_flops =
      2.0 * 256.0 * kChains * (double)(iters / 4) * blocks * (threads / 32);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sms\": %d, "
         "\"clock_khz_attr\": %d, \"err\": \"%s\"}\n",
         dfma_flops / (best_dfma * 1e-3) / 1e12,
         dmma_flops / (best_dmma * 1e-3) / 1e12, sms, clk,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
