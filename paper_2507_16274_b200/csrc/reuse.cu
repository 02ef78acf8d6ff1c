// K8 -- dynamic reusable space (derive_reuse_map / compute_reusable_space,
// reuse.py:54-93).
//
// For key k with window [t_lo, t_hi]: occupied = union of [addr, addr+size)
// over static decisions with t_s < t_hi and t_lo < t_e; the result is
// [min addr, max end) minus occupied, coalesced (intervals.py:47-56, 157-162).
//
// Decisions are radix-sorted by address once (K2). One CTA per key then
// streams the address-sorted decisions, keeps a running maximum of occupied
// ends (block max-scan carried across chunks) and emits a gap wherever the next
// occupied interval starts above it. Two launches: count, then write at the
// scanned offsets.
#include <vector>

#include "planner.cuh"

namespace stw {

constexpr int kReuseThreads = 256;

#define GS2(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ long long warp_incl_max(long long v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long n = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v = n > v ? n : v;
  }
  return v;
}

// exclusive block max-scan (LLONG_MIN identity); *total = block max
__device__ long long block_excl_max(long long v, long long *sh, long long *total) {
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long inc = warp_incl_max(v);
  if (lane_id() == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    long long x = (int)lane_id() < nw ? sh[lane_id()] : LLONG_MIN;
    long long xi = warp_incl_max(x);
    long long ex = __shfl_up_sync(0xffffffffu, xi, 1);
    if (lane_id() == 0) ex = LLONG_MIN;
    if ((int)lane_id() < nw) sh[lane_id()] = ex;
    if ((int)lane_id() == nw - 1) sh[32] = xi;
  }
  __syncthreads();
  long long before_warp = sh[w];
  long long ex_in_warp = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane_id() == 0) ex_in_warp = LLONG_MIN;
  long long out = ex_in_warp > before_warp ? ex_in_warp : before_warp;
  *total = sh[32];
  __syncthreads();
  return out;
}

__global__ void k_addr_keys(const int64_t *__restrict__ addr, int64_t n, long long amin, uint64_t *__restrict__ key) {
  GS2(i, n) key[i] = (uint64_t)((long long)addr[i] - amin);
}

__global__ void k_bounds(const int64_t *__restrict__ addr, const int64_t *__restrict__ size, int64_t n,
                         long long *__restrict__ lohi) {
  GS2(i, n) {
    atomicMin(lohi, (long long)addr[i]);
    atomicMax(lohi + 1, (long long)(addr[i] + size[i]));
  }
}

__global__ void __launch_bounds__(kReuseThreads) k_reuse(const uint32_t *__restrict__ by_addr,
                                                         const int64_t *__restrict__ addr,
                                                         const int64_t *__restrict__ size,
                                                         const int32_t *__restrict__ ts, const int32_t *__restrict__ te,
                                                         int64_t n, const int64_t *__restrict__ t_lo,
                                                         const int64_t *__restrict__ t_hi,
                                                         const long long *__restrict__ lohi,
                                                         int64_t *__restrict__ count, const int64_t *__restrict__ off,
                                                         int64_t *__restrict__ out_lo, int64_t *__restrict__ out_hi) {
  const int64_t k = blockIdx.x;
  const long long ulo = lohi[0], uhi = lohi[1];
  const long long wlo = t_lo[k], whi = t_hi[k];
  __shared__ long long sh[33];
  __shared__ uint32_t shu[33];
  long long running = ulo;  // everything below `running` is occupied or outside the universe
  int64_t emitted = 0;
  const int64_t base = off ? off[k] : 0;
  for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
    int64_t j = c0 + threadIdx.x;
    bool live = false;
    long long lo = 0, hi = LLONG_MIN;
    if (j < n) {
      uint32_t i = by_addr[j];
      live = ts[i] < whi && wlo < te[i];
      if (live) {
        lo = addr[i];
        hi = addr[i] + size[i];
      }
    }
    long long tot;
    long long before = block_excl_max(live ? hi : LLONG_MIN, sh, &tot);
    long long prev = before > running ? before : running;
    bool gap = live && lo > prev;
    uint32_t ng;
    uint32_t pos = block_excl_sum<uint32_t>(gap ? 1u : 0u, shu, &ng);
    if (gap && off) {
      out_lo[base + emitted + pos] = prev;
      out_hi[base + emitted + pos] = lo;
    }
    emitted += ng;
    if (tot > running) running = tot;
  }
  if (threadIdx.x == 0) {
    bool tail = n > 0 && running < uhi;
    if (tail && off) {
      out_lo[base + emitted] = running;
      out_hi[base + emitted] = uhi;
    }
    if (!off) count[k] = emitted + (tail ? 1 : 0);
  }
}

int reuse_map(Ctx &ctx, int64_t n, const int64_t *addr, const int64_t *size, const int32_t *t_s, const int32_t *t_e,
              int64_t K, const int64_t *t_lo, const int64_t *t_hi, int64_t *out_off, int64_t *out_lo, int64_t *out_hi,
              int64_t cap, int64_t *total) {
  Arena ar(&ctx);
  *total = 0;
  if (K <= 0) {
    if (out_off) out_off[0] = 0;
    return ctx.rc;
  }
  int64_t by = 0;
  const int64_t *dad = stage(ctx, ar, addr, n, false, &by);
  const int64_t *dsz = stage(ctx, ar, size, n, false, &by);
  const int32_t *dts = stage(ctx, ar, t_s, n, false, &by);
  const int32_t *dte = stage(ctx, ar, t_e, n, false, &by);
  const int64_t *dlo = stage(ctx, ar, t_lo, K, false, &by);
  const int64_t *dhi = stage(ctx, ar, t_hi, K, false, &by);
  long long *lohi = ar.take<long long>(2);
  int64_t *cnt = ar.take<int64_t>(K + 1), *doff = ar.take<int64_t>(K + 1);
  uint32_t *perm = ar.take<uint32_t>(n + 1);
  uint64_t *key = ar.take<uint64_t>(n + 1);
  if (!ctx.ok()) return ctx.rc;
  long long init[2] = {LLONG_MAX, LLONG_MIN};
  STW_CUDA(ctx, cudaMemcpyAsync(lohi, init, sizeof(init), cudaMemcpyHostToDevice, ctx.stream));
  if (n > 0) {
    STW_KL(k_bounds, grid_for(n, 256), 256, ctx.stream, dad, dsz, n, lohi);
    long long h[2];
    STW_CUDA(ctx, cudaMemcpyAsync(h, lohi, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    if (!ctx.ok()) return ctx.rc;
    STW_KL(k_addr_keys, grid_for(n, 256), 256, ctx.stream, dad, n, h[0], key);
    sort_perm(ctx, ar, key, perm, n, bitlen_u64((uint64_t)(h[1] - h[0])));
  }
  STW_KL(k_reuse, (unsigned)K, kReuseThreads, ctx.stream, perm, dad, dsz, dts, dte, n, dlo, dhi, lohi, cnt,
         (const int64_t *)nullptr, (int64_t *)nullptr, (int64_t *)nullptr);
  STW_LAUNCHED(ctx);
  std::vector<int64_t> hc(K);
  STW_CUDA(ctx, cudaMemcpyAsync(hc.data(), cnt, K * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok()) return ctx.rc;
  std::vector<int64_t> ho(K + 1, 0);
  for (int64_t k = 0; k < K; k++) ho[k + 1] = ho[k] + hc[k];
  *total = ho[K];
  if (out_off) memcpy(out_off, ho.data(), (K + 1) * sizeof(int64_t));
  if (ho[K] > cap) {
    ctx.fail(STW_EARG, "reuse map needs %lld intervals (capacity %lld)", (long long)ho[K], (long long)cap);
    return ctx.rc;
  }
  if (ho[K] == 0) return ctx.rc;
  int64_t *olo = ar.take<int64_t>(ho[K]), *ohi = ar.take<int64_t>(ho[K]);
  if (!ctx.ok()) return ctx.rc;
  STW_CUDA(ctx, cudaMemcpyAsync(doff, ho.data(), (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx.stream));
  STW_KL(k_reuse, (unsigned)K, kReuseThreads, ctx.stream, perm, dad, dsz, dts, dte, n, dlo, dhi, lohi, cnt, doff, olo,
         ohi);
  STW_LAUNCHED(ctx);
  STW_CUDA(ctx, cudaMemcpyAsync(out_lo, olo, ho[K] * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaMemcpyAsync(out_hi, ohi, ho[K] * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  return ctx.rc;
}

}  // namespace stw
