// Microbenchmark: cycles per clause of the sequential replay's gate-scan loop
// shape (xoshiro256++ step, integer gate test, warp-uniform branch) run by one
// warp alone, vs the same with 63 other CTAs spinning on a global flag.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scan_loop scan_loop.cu
#include <cstdint>
#include <cstdio>
struct X {
  uint64_t s0, s1, s2, s3;
  __device__ __forceinline__ uint64_t next() {
    const uint64_t sum = s0 + s3, out = ((sum << 23) | (sum >> 41)) + s0, t = s1 << 17;
    s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = (s3 << 45) | (s3 >> 19);
    return out;
  }
};
__global__ void scan(uint64_t th, int n, unsigned long long* out, volatile int* flag) {
  if (blockIdx.x != 0) {  // spinners
    if (threadIdx.x == 0) while (*flag == 0) {}
    return;
  }
  if (threadIdx.x >= 32) return;
  X r{0x123456789abcdefULL, 0xfedcba9876543210ULL, 0x0f0f0f0f0f0f0f0fULL, 0x1234ULL};
  unsigned gw = 0, cnt = 0;
  const long long t0 = clock64();
  for (int j0 = 0; j0 < n; j0 += 32) {
    for (int b = 0; b < 32; ++b) {
      if (r.next() >= th) continue;
      gw |= 1u << b;
      if (!((0x55555555u >> b) & 1u)) continue;
      cnt += 1;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = gw + cnt; *flag = 1; }
}
int main() {
  unsigned long long* d; int* f;
  cudaMalloc(&d, 16); cudaMalloc(&f, 4);
  for (int grid : {1, 64}) for (double p : {0.0, 0.5, 1.0}) {
    cudaMemset(f, 0, 4);
    const uint64_t th = p >= 1.0 ? ~0ULL : (uint64_t)(p * 9007199254740992.0) << 11;
    const int n = 1 << 20;
    scan<<<grid, 1024>>>(th, n, d, f);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"grid\": %d, \"p\": %.1f, \"cycles_per_clause\": %.1f}\n", grid, p, (double)h[0] / n);
  }
  return 0;
}
