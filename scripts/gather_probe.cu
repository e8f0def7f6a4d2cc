// Probe: DRAM bytes read when gathering 64-byte rows through a random
// permutation (the heads/tails input pattern), for several load flavours.
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum ./gather_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#include <cuda_pipeline.h>

template <int MODE>
__device__ __forceinline__ double2 ld(const double2* p) {
  double2 v;
  if (MODE == 0) asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 1) asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 2) asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 3) asm volatile("ld.global.cv.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 4) asm volatile("ld.global.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 5) asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 6) asm volatile("ld.global.L2::128B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 7) asm volatile("ld.global.L1::evict_first.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  if (MODE == 8) asm volatile("ld.global.lu.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int MODE, int PK>  // PK packets (16 B) of each 64-byte row are read
__global__ void k_ld(const double2* __restrict__ d, const int* __restrict__ perm, long n, double* out) {
  double acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n * PK; i += (long)gridDim.x * blockDim.x) {
    const long r = perm[i / PK];
    const double2 v = ld<MODE>(&d[r * 4 + (i % PK)]);
    acc += v.x + v.y;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
  const long n = 50000000;
  std::vector<int> p(n);
  for (long i = 0; i < n; ++i) p[i] = (int)i;
  int *perm_rnd; double2* d; double* out;
  cudaMalloc(&perm_rnd, n * 4); cudaMalloc(&d, n * 64); cudaMalloc(&out, 8);
  cudaMemset(d, 0, n * 64);
  std::mt19937_64 g(1); std::shuffle(p.begin(), p.end(), g);
  cudaMemcpy(perm_rnd, p.data(), n * 4, cudaMemcpyHostToDevice);
  if (argc > 1) {
    size_t a = 0; cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
    cudaDeviceGetLimit(&a, cudaLimitMaxL2FetchGranularity); printf("L2 fetch granularity %zu\n", a);
  }
  const int grid = 148 * 8;
  k_ld<0, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<1, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<2, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<3, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<4, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<5, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<6, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<7, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<8, 4><<<grid, 256>>>(d, perm_rnd, n, out);
  k_ld<0, 2><<<grid, 256>>>(d, perm_rnd, n, out);  // 32 of every 64 bytes
  k_ld<0, 1><<<grid, 256>>>(d, perm_rnd, n, out);  // 16 of every 64 bytes
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
