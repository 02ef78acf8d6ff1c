// Cycles per item of the gap-host resolve chain (one warp, lane p = priority p):
// vote(fit && last < ts) -> ffs -> lane select; fields broadcast one item ahead.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const int *ts_, const int *te_, const unsigned *f_, int n, int *out, long long *cyc, int variant) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x;
  int lastp = -1000000000;
  long long t0 = clock64();
  int acc = 0;
  for (int cb = 0; cb < n; cb += 32) {
    const int my_ts = ts_[cb + lane], my_te = te_[cb + lane];
    const unsigned fm = f_[cb + lane];
    int ts = __shfl_sync(FULL, my_ts, 0), te = __shfl_sync(FULL, my_te, 0);
    unsigned f = __shfl_sync(FULL, fm, 0);
    int my_code = 0;
    for (int k = 0; k < 32; k++) {
      const int k1 = (k + 1) & 31;
      const int nts = __shfl_sync(FULL, my_ts, k1), nte = __shfl_sync(FULL, my_te, k1);
      const unsigned nf = __shfl_sync(FULL, fm, k1);
      const unsigned m1 = __ballot_sync(FULL, ((f >> lane) & 1u) && lastp < ts);
      int code = 0;
      if (variant == 0) {
        const int host = __ffs(m1) - 1;
        lastp = lane == host ? te : lastp;
        code = host;
      } else {
        if (m1) {
          const int host = __ffs(m1) - 1;
          lastp = lane == host ? te : lastp;
          code = host;
        } else {
          code = 99;
        }
      }
      if (lane == k) my_code = code;
      ts = nts, te = nte, f = nf;
    }
    acc += my_code;
  }
  long long t1 = clock64();
  out[lane] = acc + lastp;
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  const int n = 1 << 20;
  int *ts, *te; unsigned *f; int *o; long long *c;
  cudaMallocManaged(&ts, n * 4); cudaMallocManaged(&te, n * 4); cudaMallocManaged(&f, n * 4);
  cudaMalloc(&o, 128); cudaMalloc(&c, 8);
  for (int i = 0; i < n; i++) { ts[i] = i; te[i] = i + 3 + (i % 7); f[i] = 0xffu; }
  for (int v = 0; v < 2; v++) {
    k<<<1, 32>>>(ts, te, f, n, o, c, v); cudaDeviceSynchronize();
    k<<<1, 32>>>(ts, te, f, n, o, c, v); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %.1f cycles/item\n", v, (double)h / n);
  }
}
