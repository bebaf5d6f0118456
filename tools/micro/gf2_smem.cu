// Microbenchmark: the GF(2) jump with the XOR reduction through shared
// memory (partials [32][9], group sums [4][8]) instead of redux.sync,
// CHAINS independent jumps per round; checks the result against gf2_apply.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2009_04861_b200/csrc -DCHAINS=4 -o gf2_m4 gf2_smem.cu
#include <cstdio>
#include "tm_device.cuh"
using namespace tmg;
#ifndef CHAINS
#define CHAINS 1
#endif
__device__ __forceinline__ void gf2_apply_sm(const uint32_t* tab, uint32_t (&s)[8], int lane, uint32_t* scr) {
  const int ws = lane >> 2;
  uint32_t v = s[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) v = ws == k ? s[k] : v;
  const uint32_t byte = (v >> (8 * (lane & 3))) & 0xFFu;
  const uint4* e0 = reinterpret_cast<const uint4*>(tab + ((2 * lane) * 16 + (byte & 15u)) * 8);
  const uint4* e1 = reinterpret_cast<const uint4*>(tab + ((2 * lane + 1) * 16 + (byte >> 4)) * 8);
  const uint4 a0 = e0[0], a1 = e0[1], b0 = e1[0], b1 = e1[1];
  volatile uint32_t* P = scr;        // [32][9]
  volatile uint32_t* Q = scr + 288;  // [4][8]
  P[lane * 9 + 0] = a0.x ^ b0.x;
  P[lane * 9 + 1] = a0.y ^ b0.y;
  P[lane * 9 + 2] = a0.z ^ b0.z;
  P[lane * 9 + 3] = a0.w ^ b0.w;
  P[lane * 9 + 4] = a1.x ^ b1.x;
  P[lane * 9 + 5] = a1.y ^ b1.y;
  P[lane * 9 + 6] = a1.z ^ b1.z;
  P[lane * 9 + 7] = a1.w ^ b1.w;
  __syncwarp();
  const int w = lane & 7, g = lane >> 3;
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= P[(8 * g + k) * 9 + w];
  Q[g * 8 + w] = acc;
  __syncwarp();
  const uint4* q4 = reinterpret_cast<const uint4*>(scr + 288);
  uint4 r0 = q4[0], r1 = q4[1];
#pragma unroll
  for (int h = 1; h < 4; ++h) {
    const uint4 c0 = q4[2 * h], c1 = q4[2 * h + 1];
    r0.x ^= c0.x; r0.y ^= c0.y; r0.z ^= c0.z; r0.w ^= c0.w;
    r1.x ^= c1.x; r1.y ^= c1.y; r1.z ^= c1.z; r1.w ^= c1.w;
  }
  __syncwarp();
  s[0] = r0.x; s[1] = r0.y; s[2] = r0.z; s[3] = r0.w;
  s[4] = r1.x; s[5] = r1.y; s[6] = r1.z; s[7] = r1.w;
}

__global__ void lat(const uint32_t* tab_g, int iters, unsigned long long* out, uint32_t* chk) {
  extern __shared__ __align__(16) uint32_t tab[];
  __shared__ __align__(16) uint32_t scr[CHAINS][320];
  for (int k = threadIdx.x; k < kGf2TabWords; k += blockDim.x) tab[k] = tab_g[k];
  __syncthreads();
  const int lane = threadIdx.x;
  uint32_t s[CHAINS][8], t[8], u[8];
  for (int c = 0; c < CHAINS; ++c)
    for (int w = 0; w < 8; ++w) s[c][w] = w + 1 + 8 * c;
  for (int w = 0; w < 8; ++w) t[w] = u[w] = s[0][w];
  gf2_apply(tab, t, lane);  // the product's reduction
  gf2_apply_sm(tab, u, lane, scr[0]);
  uint32_t bad = 0;
  for (int w = 0; w < 8; ++w) bad |= t[w] ^ u[w];
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) gf2_apply_sm(tab, s[c], lane, scr[c]);
  const long long t1 = clock64();
  uint32_t x = 0;
  for (int c = 0; c < CHAINS; ++c) x ^= s[c][0] ^ s[c][7];
  if (lane == 0) {
    out[0] = t1 - t0;
    out[1] = x;
  }
  atomicOr(chk, bad);
}

int main() {
  uint32_t *t, *chk;
  unsigned long long* d;
  cudaMalloc(&t, kGf2TabWords * 4);
  cudaMalloc(&d, 16);
  cudaMalloc(&chk, 4);
  cudaMemset(chk, 0, 4);
  uint32_t* h = new uint32_t[kGf2TabWords];
  for (int k = 0; k < kGf2TabWords; ++k) h[k] = 2654435761u * (k + 1);
  cudaMemcpy(t, h, kGf2TabWords * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, kGf2TabWords * 4);
  const int iters = 10000;
  lat<<<1, 32, kGf2TabWords * 4>>>(t, iters, d, chk);
  unsigned long long r[2];
  uint32_t bad;
  cudaMemcpy(r, d, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(&bad, chk, 4, cudaMemcpyDeviceToHost);
  printf("{\"smem_reduce\": 1, \"chains\": %d, \"cycles_per_round\": %.1f, \"matches_redux\": %s}\n", CHAINS,
         (double)r[0] / iters, bad ? "false" : "true");
  return 0;
}
