// Microbenchmark: latency (cycles) of one warp-cooperative GF(2) jump
// (tm_device.cuh gf2_apply, nibble tables in shared memory), chained.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2009_04861_b200/csrc -o gf2_lat gf2_lat.cu
#include <cstdio>
#include "tm_device.cuh"
#ifndef CHAINS
#define CHAINS 1
#endif
using namespace tmg;
__global__ void lat(const uint32_t* tab_g, int iters, unsigned long long* out) {
  extern __shared__ __align__(16) uint32_t tab[];
  for (int k = threadIdx.x; k < kGf2TabWords; k += blockDim.x) tab[k] = tab_g[k];
  __syncthreads();
  const int lane = threadIdx.x;
  uint32_t s[CHAINS][8];
  for (int c = 0; c < CHAINS; ++c)
    for (int w = 0; w < 8; ++w) s[c][w] = w + 1 + 8 * c;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) gf2_apply(tab, s[c], lane);
  const long long t1 = clock64();
  uint32_t x = 0;
  for (int c = 0; c < CHAINS; ++c) x ^= s[c][0] ^ s[c][7];
  if (lane == 0) { out[0] = t1 - t0; out[1] = x; }
}
int main() {
  uint32_t* t; unsigned long long* d;
  cudaMalloc(&t, kGf2TabWords * 4); cudaMalloc(&d, 16);
  cudaMemset(t, 0x5a, kGf2TabWords * 4);
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, kGf2TabWords * 4);
  const int iters = 10000;
  lat<<<1, 32, kGf2TabWords * 4>>>(t, iters, d);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("{\"redux\": %d, \"chains\": %d, \"cycles_per_round\": %.1f}\n", TMG_GF2_REDUX, CHAINS, (double)h[0] / iters);
  return 0;
}
