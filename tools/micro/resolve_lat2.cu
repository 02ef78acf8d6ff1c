// Cycles per item of the layer resolve step variants (one warp), c5-like data.
#include <climits>
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(const int *ts_, const int *te_, const unsigned *f_, int n, int *out, long long *cyc) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x;
  int lastp = INT_MIN, ne = INT_MIN, nnew = 0;
  int last8[8];
#pragma unroll
  for (int p = 0; p < 8; p++) last8[p] = INT_MIN;
  long long t0 = clock64();
  int acc = 0;
  int nx_ts = ts_[lane], nx_te = te_[lane];
  unsigned nx_fm = f_[lane];
  for (int cb = 0; cb < n; cb += 32) {
    const int my_ts = nx_ts, my_te = nx_te;
    const unsigned fm = nx_fm;
    if (cb + 32 < n) nx_ts = ts_[cb + 32 + lane], nx_te = te_[cb + 32 + lane], nx_fm = f_[cb + 32 + lane];
    int my_code = 0;
    auto step = [&](const int k) {
      const int ts = __shfl_sync(FULL, my_ts, k), te = __shfl_sync(FULL, my_te, k);
      const unsigned f = __shfl_sync(FULL, fm, k);
      int code;
      if (V <= 1) {
        const unsigned m1 = __ballot_sync(FULL, ((f >> lane) & 1u) && lastp < ts);
        if (m1) {
          lastp = ((m1 & (0u - m1)) >> lane) & 1u ? te : lastp;
          code = __ffs(m1) - 1;
        } else {
          const bool ca = lane < nnew && ne < ts;
          const int mx = __reduce_max_sync(FULL, ca ? ne : INT_MIN);
          const unsigned cma = __ballot_sync(FULL, ca && ne == mx);
          const int best = cma ? __ffs(cma) - 1 : nnew;
          if (lane == best) ne = te;
          nnew += cma ? 0 : 1;
          code = 32 + best;
        }
      } else {
        unsigned fr = 0;
#pragma unroll
        for (int p = 0; p < 8; p++) fr |= (last8[p] < ts ? 1u : 0u) << p;
        const unsigned m1 = f & fr;
        if (m1) {
          const unsigned low = m1 & (0u - m1);
#pragma unroll
          for (int p = 0; p < 8; p++) last8[p] = (low >> p) & 1u ? te : last8[p];
          code = __ffs(m1) - 1;
        } else {
          const bool ca = lane < nnew && ne < ts;
          const int mx = __reduce_max_sync(FULL, ca ? ne : INT_MIN);
          const unsigned cma = __ballot_sync(FULL, ca && ne == mx);
          const int best = cma ? __ffs(cma) - 1 : nnew;
          if (lane == best) ne = te;
          nnew += cma ? 0 : 1;
          code = 32 + best;
        }
      }
      my_code = lane == k ? code : my_code;
    };
    if (V == 4 || V == 5) {
      int k = 0;
      int ts = __shfl_sync(FULL, my_ts, 0), te = __shfl_sync(FULL, my_te, 0);
      unsigned f = __shfl_sync(FULL, fm, 0);
      while (true) {
#pragma unroll 2
        for (; k < 32; k++) {
          const int k1 = (k + 1) & 31;
          const int nts = __shfl_sync(FULL, my_ts, k1), nte = __shfl_sync(FULL, my_te, k1);
          const unsigned nf = __shfl_sync(FULL, fm, k1);
          const unsigned m1 = __ballot_sync(FULL, ((f >> lane) & 1u) && lastp < ts);
          if (!m1) break;
          lastp = ((m1 & (0u - m1)) >> lane) & 1u ? te : lastp;
          if (V == 4) my_code = lane == k ? __ffs(m1) - 1 : my_code;
          else my_code = lane == k ? (int)m1 : my_code;
          ts = nts, te = nte, f = nf;
        }
        if (k >= 32) break;
        {  // Alg. 1 for item k
          const bool ca = lane < nnew && ne < ts;
          const int mx = __reduce_max_sync(FULL, ca ? ne : INT_MIN);
          const unsigned cma = __ballot_sync(FULL, ca && ne == mx);
          const int best = cma ? __ffs(cma) - 1 : nnew;
          if (lane == best) ne = te;
          nnew += cma ? 0 : 1;
          my_code = lane == k ? 32 + best : my_code;
        }
        k++;
        if (k >= 32) break;
        ts = __shfl_sync(FULL, my_ts, k), te = __shfl_sync(FULL, my_te, k);
        f = __shfl_sync(FULL, fm, k);
      }
    } else if (V == 0 || V == 2) {
#pragma unroll
      for (int k = 0; k < 32; k++) step(k);
    } else {
#pragma unroll 4
      for (int k = 0; k < 32; k++) step(k);
    }
    acc += my_code;
  }
  long long t1 = clock64();
  out[lane] = acc + lastp + last8[0] + last8[7];
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  const int n = 1 << 20;
  int *ts, *te; unsigned *f; int *o; long long *c;
  cudaMallocManaged(&ts, n * 4); cudaMallocManaged(&te, n * 4); cudaMallocManaged(&f, n * 4);
  cudaMalloc(&o, 128); cudaMalloc(&c, 8);
  // 8 layers, items round-robin over them (c5-like: every item gap-inserted)
  for (int i = 0; i < n; i++) { ts[i] = 2 * i; te[i] = 2 * i + 9; f[i] = 0xffu; }
  const char *nm[] = {"vote, full unroll", "vote, unroll 4", "uniform8, full unroll", "uniform8, unroll 4", "vote, early exit", "vote, early exit, raw m1"};
  for (int v = 0; v < 6; v++) {
    for (int r = 0; r < 2; r++) {
      if (v == 0) k<0><<<1, 32>>>(ts, te, f, n, o, c);
      if (v == 1) k<1><<<1, 32>>>(ts, te, f, n, o, c);
      if (v == 2) k<2><<<1, 32>>>(ts, te, f, n, o, c);
      if (v == 3) k<3><<<1, 32>>>(ts, te, f, n, o, c);
      if (v == 4) k<4><<<1, 32>>>(ts, te, f, n, o, c);
      if (v == 5) k<5><<<1, 32>>>(ts, te, f, n, o, c);
      cudaDeviceSynchronize();
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %.1f cycles/item\n", nm[v], (double)h / n);
  }
}
