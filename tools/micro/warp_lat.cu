// Latency of the warp-collective steps the sequential replay chains (one warp,
// dependent chains of 256 ops, clock64 around them). nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned *out, long long *cyc, unsigned seed) {
  const int lane = threadIdx.x;
  unsigned v = seed + lane;
  long long t0, t1;
  __shared__ unsigned sm[64];
  sm[lane] = lane; sm[lane + 32] = lane;
  __syncwarp();
#define CHAIN(name, idx, body)                        \
  t0 = clock64();                                     \
  for (int i = 0; i < 256; i++) { body; }             \
  t1 = clock64();                                     \
  if (lane == 0) cyc[idx] = (t1 - t0);
  CHAIN("alu", 0, v = v * 3 + 1)
  CHAIN("redux_min", 1, v = __reduce_min_sync(0xffffffffu, v) + lane)
  CHAIN("redux_or", 2, v = __reduce_or_sync(0xffffffffu, v) + lane)
  CHAIN("ballot", 3, v = __ballot_sync(0xffffffffu, v & 1) + lane)
  CHAIN("shfl", 4, v = __shfl_sync(0xffffffffu, v, v & 31) + 1)
  CHAIN("lds", 5, v = sm[v & 63] + 1)
  CHAIN("syncwarp", 6, { __syncwarp(); v = v * 3 + 1; })
  CHAIN("sts_lds", 7, { sm[lane] = v; v = sm[(v + lane) & 31] + 1; })
  CHAIN("ballot_ffs_shfl", 8, { unsigned m = __ballot_sync(0xffffffffu, v & 1); v = __shfl_sync(0xffffffffu, v, __ffs(m | 1) - 1) + lane; })
  CHAIN("any", 9, v = __any_sync(0xffffffffu, v & 1) + v + lane)
  out[lane] = v;
}
int main() {
  unsigned *o; long long *c; cudaMalloc(&o, 128); cudaMalloc(&c, 16 * 8);
  k<<<1, 32>>>(o, c, 1); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 2); cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char *nm[] = {"alu(imad+iadd)", "redux_min", "redux_or", "ballot", "shfl", "lds", "syncwarp+alu", "sts+lds", "ballot+ffs+shfl", "any"};
  for (int i = 0; i < 10; i++) printf("%-18s %6.1f cycles/iter\n", nm[i], h[i] / 256.0);
}
