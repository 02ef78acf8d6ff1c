// K1 -- peak live bytes (model.py:261-276) on a per-trace timeline.
//
// live(t) = sum(size : t_s <= t) - sum(size : t_e <= t) at every timestamp;
// frees precede allocs at equal t, so max_t live(t) is exactly the reference's
// running-sum maximum. Each event scatters +size at t_s and -size at t_e into
// its trace's timeline segment; every trace's deltas sum to zero, so one
// unsegmented inclusive scan over the concatenated timelines is already the
// per-trace scan, and a max-reduction per segment gives the peak.
#include "batch.cuh"

namespace stw {

__global__ void k_timeline_len(const int64_t *__restrict__ ev_off, int T, int64_t N,
                               const int32_t *__restrict__ t_s, const int32_t *__restrict__ t_e,
                               const int32_t *__restrict__ horizon, int *__restrict__ tmax) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    int t = trace_of(ev_off, T, i);
    int m = max(t_s[i], t_e[i]);
    if (m > horizon[t]) atomicMax(tmax + t, m);
  }
}

__global__ void k_init_len(const int32_t *__restrict__ horizon, int *__restrict__ tmax, int T) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) tmax[t] = horizon[t];
}

__global__ void k_timeline_scatter(const int64_t *__restrict__ ev_off, int T, int64_t N,
                                   const int64_t *__restrict__ size, const int32_t *__restrict__ t_s,
                                   const int32_t *__restrict__ t_e, const uint8_t *__restrict__ dyn,
                                   const int64_t *__restrict__ tl_off, unsigned long long *__restrict__ D,
                                   int static_only, const uint8_t *__restrict__ only) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (static_only && dyn[i]) continue;
    int t = trace_of(ev_off, T, i);
    if (!only[t]) continue;
    int64_t o = tl_off[t];
    unsigned long long s = (unsigned long long)size[i];
    atomicAdd(D + o + t_s[i], s);
    atomicAdd(D + o + t_e[i], (unsigned long long)(-(long long)s));
  }
}

__global__ void k_zero_selected(const uint8_t *__restrict__ only, int T, int64_t *__restrict__ peak) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
    if (only[t]) peak[t] = 0;
}

// per-segment max of the scanned timeline; each thread walks 8 consecutive
// entries and flushes one atomicMax per trace it touched
__global__ void k_segmax(const int64_t *__restrict__ P, int64_t H, const int64_t *__restrict__ tl_off, int T,
                         long long *__restrict__ peak) {  // peak[t] of the recomputed traces is pre-zeroed
  int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8;
  if (i0 >= H) return;
  int t = trace_of(tl_off, T, i0);
  long long best = 0;
  for (int64_t i = i0; i < i0 + 8 && i < H; i++) {
    while (i >= tl_off[t + 1]) {
      if (best > 0) atomicMax(peak + t, best);
      best = 0;
      t++;
    }
    long long v = P[i];
    if (v > best) best = v;
  }
  if (best > 0) atomicMax(peak + t, best);
}

// One CTA per trace whose timeline fits in shared memory (every c4 trace):
// deltas by shared-memory atomics, then each thread scans a contiguous chunk
// (local prefix + local max), one block scan of the chunk sums, and the peak
// is max(excl + local max) -- the timeline never touches HBM, so the kernel
// reads 17 B per event (t_s, t_e, size, dyn) and writes 8 B per trace. The
// timeline is sized by the batch's largest horizon (dynamic shared memory);
// a trace with a longer horizon or a timestamp outside [0, horizon] is
// flagged for the global-timeline path below.
constexpr int kPeakThreads = 128;
constexpr int kPeakSmemMax = 12288;  // timeline entries (96 KB)

__global__ void __launch_bounds__(kPeakThreads) k_peak_cta(const int64_t *__restrict__ ev_off,
                                                           const int64_t *__restrict__ size,
                                                           const int32_t *__restrict__ t_s,
                                                           const int32_t *__restrict__ t_e,
                                                           const uint8_t *__restrict__ dyn,
                                                           const int32_t *__restrict__ horizon, int hcap,
                                                           int static_only, long long *__restrict__ peak,
                                                           int *__restrict__ nbig, int32_t *__restrict__ big) {
  extern __shared__ unsigned long long D[];
  __shared__ long long sh[33];
  const int t = blockIdx.x, tid = threadIdx.x;
  const int64_t e0 = ev_off[t], e1 = ev_off[t + 1];
  const int H = horizon[t] + 1;  // timestamps are in [0, horizon] (model.py:240-241)
  if (H > hcap || H <= 0) {
    if (tid == 0) big[atomicAdd(nbig, 1)] = t;
    return;
  }
  for (int x = tid; x < H; x += kPeakThreads) D[x] = 0;
  __syncthreads();
  bool bad = false;
  for (int64_t i = e0 + tid; i < e1; i += kPeakThreads) {
    if (static_only && dyn[i]) continue;
    const int a = t_s[i], z = t_e[i];
    if ((unsigned)a >= (unsigned)H || (unsigned)z >= (unsigned)H) {
      bad = true;
      continue;
    }
    const unsigned long long sz = (unsigned long long)size[i];
    atomicAdd(D + a, sz);
    atomicAdd(D + z, 0ull - sz);
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) big[atomicAdd(nbig, 1)] = t;
    return;
  }
  const int per = (H + kPeakThreads - 1) / kPeakThreads;
  const int x0 = min(H, tid * per), x1 = min(H, x0 + per);
  long long run = 0, best = LLONG_MIN;
  for (int x = x0; x < x1; x++) {
    run += (long long)D[x];
    best = max(best, run);
  }
  long long tot;
  const long long ex = block_excl_sum<long long>(run, sh, &tot);
  long long cand = best == LLONG_MIN ? LLONG_MIN : ex + best;
  for (int o = 16; o; o >>= 1) cand = max(cand, __shfl_xor_sync(0xffffffffu, cand, o));
  if ((tid & 31) == 0) sh[tid >> 5] = cand;
  __syncthreads();
  if (tid == 0) {
    long long m = 0;  // the reference's running maximum starts at 0
    for (int w = 0; w < kPeakThreads / 32; w++) m = max(m, sh[w]);
    peak[t] = m;
  }
}

__global__ void k_big_offsets(const int32_t *__restrict__ big, const int *__restrict__ nbig, int T,
                              uint8_t *__restrict__ is_big) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < *nbig; x += gridDim.x * blockDim.x) is_big[big[x]] = 1;
}

static void peak_live_global(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak,
                             const uint8_t *only);

void peak_live(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak) {
  if (!ctx.ok() || b.T == 0) return;
  const int T = b.T;
  int *nbig = ar.take<int>(1);
  int32_t *big = ar.take<int32_t>(T);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemsetAsync(nbig, 0, sizeof(int), ctx.stream));
  int hmax = 0;
  for (int x : b.h_horizon) hmax = std::max(hmax, x);
  const int hcap = std::min(hmax + 1, kPeakSmemMax);
  const int smem = hcap * (int)sizeof(unsigned long long);
  STW_CUDA(ctx, cudaFuncSetAttribute(k_peak_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  STW_KLS(k_peak_cta, (unsigned)T, kPeakThreads, smem, ctx.stream, b.ev_off, b.size, b.t_s, b.t_e, b.dyn,
          b.horizon, hcap, static_only ? 1 : 0, (long long *)d_peak, nbig, big);
  STW_LAUNCHED(ctx);
  int h = 0;
  STW_CUDA(ctx, cudaMemcpyAsync(&h, nbig, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok() || h == 0) return;
  uint8_t *is_big = ar.take<uint8_t>(T);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemsetAsync(is_big, 0, T, ctx.stream));
  STW_KL(k_big_offsets, grid_for(h, 256), 256, ctx.stream, big, nbig, T, is_big);
  STW_LAUNCHED(ctx);
  peak_live_global(ctx, ar, b, static_only, d_peak, is_big);
}

// Traces with long timelines (e.g. c5, horizon 1,966,792): the timeline lives
// in HBM; `only` selects the traces to (re)compute.
static void peak_live_global(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak,
                             const uint8_t *only) {
  if (!ctx.ok()) return;
  const int T = b.T;
  int *tmax = ar.take<int>(T);
  int64_t *tl_len = ar.take<int64_t>(T + 1);
  if (!ctx.ok()) return;
  STW_KL(k_init_len, grid_for(T, 256), 256, ctx.stream, b.horizon, tmax, T);
  STW_KL(k_timeline_len, grid_for(b.N, 256), 256, ctx.stream, b.ev_off, T, b.N, b.t_s, b.t_e, b.horizon, tmax);
  STW_LAUNCHED(ctx);
  std::vector<int> h(T);
  STW_CUDA(ctx, cudaMemcpyAsync(h.data(), tmax, T * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok()) return;
  std::vector<int64_t> off(T + 1, 0);
  for (int t = 0; t < T; t++) off[t + 1] = off[t] + (int64_t)h[t] + 1;
  int64_t H = off[T];
  STW_CUDA(ctx, cudaMemcpyAsync(tl_len, off.data(), (T + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx.stream));
  int64_t *D = ar.take<int64_t>(H);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemsetAsync(D, 0, H * sizeof(int64_t), ctx.stream));
  STW_KL(k_zero_selected, grid_for(T, 256), 256, ctx.stream, only, T, d_peak);
  STW_KL(k_timeline_scatter, grid_for(b.N, 256), 256, ctx.stream, b.ev_off, T, b.N, b.size, b.t_s, b.t_e, b.dyn,
                                                                 tl_len, (unsigned long long *)D, static_only, only);
  STW_LAUNCHED(ctx);
  device_scan<int64_t>(ctx, ar, D, D, H, true);
  int64_t nthreads = (H + 7) / 8;
  STW_KL(k_segmax, (unsigned)((nthreads + 255) / 256), 256, ctx.stream, D, H, tl_len, T, (long long *)d_peak);
  STW_LAUNCHED(ctx);
}

}  // namespace stw
