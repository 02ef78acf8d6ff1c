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

// One warp per trace whose timeline fits in its shared-memory slice (every c4
// trace): deltas by shared-memory atomics, then each lane scans a contiguous
// chunk (local prefix + local max), one warp scan of the chunk sums, and the
// peak is max(excl + local max). The timeline never touches HBM, so the
// kernel reads 17 B per event (t_s, t_e, size, dyn) and writes 8 B per trace.
// Traces are packed host-side into CTAs by horizon (slices of 8 B x
// (horizon + 1), largest first), so there are no block-wide barriers and many
// traces per SM are in flight. A trace with a timestamp outside [0, horizon]
// (or too long a horizon) goes to the global-timeline path below.
constexpr int kPeakWarps = 8;
constexpr int kPeakSmem = 28 * 1024;  // bytes per CTA: eight CTAs per SM

// The timeline holds 32-bit deltas in units of 2^shift bytes (the alignment):
// half the shared memory of 64-bit deltas, so twice the traces in flight per
// SM, and native 32-bit shared atomics. A trace whose sizes are not multiples
// of 2^shift, or whose byte total in those units does not fit 31 bits (so a
// timeline entry could overflow), or with a timestamp outside [0, horizon],
// is flagged for the global-timeline path below.
__global__ void __launch_bounds__(kPeakWarps * 32) k_peak_warp(const int64_t *__restrict__ ev_off,
                                                               const int64_t *__restrict__ size,
                                                               const int32_t *__restrict__ t_s,
                                                               const int32_t *__restrict__ t_e,
                                                               const uint8_t *__restrict__ dyn,
                                                               const int32_t *__restrict__ horizon,
                                                               int static_only, int shift,
                                                               const int2 *__restrict__ wslot,
                                                               long long *__restrict__ peak, int *__restrict__ nbig,
                                                               int32_t *__restrict__ big) {
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ int pk_smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 slot = wslot[blockIdx.x * kPeakWarps + w];
  if (slot.x < 0) return;
  const int t = slot.x;
  int *D = pk_smem + slot.y;
  const int64_t e0 = ev_off[t], e1 = ev_off[t + 1];
  const int H = horizon[t] + 1;  // timestamps are in [0, horizon] (model.py:240-241)
  for (int x = lane; x < H; x += 32) D[x] = 0;
  __syncwarp();
  bool bad = false;
  long long units = 0;
  const long long low = (1ll << shift) - 1;
  constexpr int B = 4;  // events per lane loaded together (independent loads in flight)
  for (int64_t i0 = e0; i0 < e1; i0 += 32 * B) {
    int a[B], z[B];
    long long sz[B];
    bool use[B];
#pragma unroll
    for (int q = 0; q < B; q++) {
      const int64_t i = i0 + q * 32 + lane;
      use[q] = i < e1;
      a[q] = use[q] ? t_s[i] : 0;
      z[q] = use[q] ? t_e[i] : 0;
      sz[q] = use[q] ? (long long)size[i] : 0;
      if (static_only && use[q]) use[q] = dyn[i] == 0;
    }
#pragma unroll
    for (int q = 0; q < B; q++) {
      if (!use[q]) continue;
      if ((unsigned)a[q] >= (unsigned)H || (unsigned)z[q] >= (unsigned)H || sz[q] < 0 || (sz[q] & low)) {
        bad = true;
        continue;
      }
      const int u = (int)min(sz[q] >> shift, (long long)INT_MAX);
      units += sz[q] >> shift;
      atomicAdd(D + a[q], u);
      atomicAdd(D + z[q], -u);
    }
  }
  for (int o = 16; o; o >>= 1) units += __shfl_xor_sync(FULL, units, o);
  if (__any_sync(FULL, bad) || units > INT_MAX) {
    if (lane == 0) big[atomicAdd(nbig, 1)] = t;
    return;
  }
  __syncwarp();
  const int per = (H + 31) >> 5;
  const int x0 = min(H, lane * per), x1 = min(H, x0 + per);
  long long run = 0, best = LLONG_MIN;
  for (int x = x0; x < x1; x++) {
    run += D[x];
    best = max(best, run);
  }
  const long long inc = warp_incl_sum(run);
  long long cand = best == LLONG_MIN ? 0 : inc - run + best;  // the running maximum starts at 0
  for (int o = 16; o; o >>= 1) cand = max(cand, __shfl_xor_sync(FULL, cand, o));
  if (lane == 0) peak[t] = cand << shift;
}

__global__ void k_big_offsets(const int32_t *__restrict__ big, const int *__restrict__ nbig, int T,
                              uint8_t *__restrict__ is_big) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < *nbig; x += gridDim.x * blockDim.x) is_big[big[x]] = 1;
}

static void peak_live_global(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak,
                             const uint8_t *only);

void peak_live(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak) {
  PeakPending pp = peak_live_launch(ctx, ar, b, static_only, d_peak, 9);
  peak_live_finish(ctx, ar, b, static_only, d_peak, pp);
}

void peak_live_finish(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak,
                      const PeakPending &pp) {
  if (!ctx.ok() || !pp.nbig) return;
  int h = 0;
  STW_CUDA(ctx, cudaMemcpyAsync(&h, pp.nbig, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok() || h == 0) return;
  const int T = b.T;
  uint8_t *is_big = ar.take<uint8_t>(T);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemsetAsync(is_big, 0, T, ctx.stream));
  STW_KL(k_big_offsets, grid_for(h, 256), 256, ctx.stream, pp.big, pp.nbig, T, is_big);
  STW_LAUNCHED(ctx);
  peak_live_global(ctx, ar, b, static_only, d_peak, is_big);
}

PeakPending peak_live_launch(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak,
                             int shift, bool pinned) {
  PeakPending pp{};
  if (!ctx.ok() || b.T == 0) return pp;
  const int T = b.T;
  int *nbig = ar.take<int>(1);
  int32_t *big = ar.take<int32_t>(T);
  if (!ctx.ok()) return pp;
  pp.nbig = nbig;
  pp.big = big;
  STW_CUDA(ctx, cudaMemsetAsync(nbig, 0, sizeof(int), ctx.stream));
  // pack traces into CTAs by timeline size, largest first (counting sort by horizon)
  std::vector<int32_t> order, longh;
  order.reserve(T);
  int hmax = 0;
  for (int t = 0; t < T; t++) {
    const int64_t bytes = 4 * ((int64_t)b.h_horizon[t] + 1);
    if (b.h_horizon[t] < 0 || bytes > kPeakSmem)
      longh.push_back(t);
    else
      order.push_back(t), hmax = std::max(hmax, b.h_horizon[t]);
  }
  {
    std::vector<int32_t> pos(hmax + 2, 0), sorted(order.size());
    for (int32_t t : order) pos[hmax - b.h_horizon[t] + 1]++;
    for (int k = 0; k <= hmax; k++) pos[k + 1] += pos[k];
    for (int32_t t : order) sorted[pos[hmax - b.h_horizon[t]]++] = t;
    order.swap(sorted);
  }
  std::vector<int2> wslot;
  wslot.reserve(order.size() + kPeakWarps);
  const int cap = kPeakSmem / 4;
  for (size_t i = 0, j = order.size(); i < j;) {
    const size_t base = wslot.size();
    int used = 0, k = 0;
    auto put = [&](int32_t t) {
      wslot.push_back(make_int2(t, used));
      used += b.h_horizon[t] + 1;
      k++;
    };
    put(order[i++]);
    while (k < kPeakWarps && i < j && used + b.h_horizon[order[i]] + 1 <= cap) put(order[i++]);
    while (k < kPeakWarps && i < j && used + b.h_horizon[order[j - 1]] + 1 <= cap) put(order[--j]);
    while (wslot.size() < base + kPeakWarps) wslot.push_back(make_int2(-1, 0));
  }
  const int nctas = (int)(wslot.size() / kPeakWarps);
  int2 *d_wslot = nctas ? ar.take<int2>(wslot.size()) : nullptr;
  if (!ctx.ok()) return pp;
  if (!longh.empty()) {  // long horizons go straight to the global path
    const int nl = (int)longh.size();
    if (pinned) {
      h2d_async(ctx, big, longh.data(), longh.size() * sizeof(int32_t));
      h2d_async(ctx, nbig, &nl, sizeof(int));
    } else {
      STW_CUDA(ctx, cudaMemcpyAsync(big, longh.data(), longh.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                    ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(nbig, &nl, sizeof(int), cudaMemcpyHostToDevice, ctx.stream));
    }
  }
  if (nctas) {
    if (pinned)
      h2d_async(ctx, d_wslot, wslot.data(), wslot.size() * sizeof(int2));
    else
      STW_CUDA(ctx, cudaMemcpyAsync(d_wslot, wslot.data(), wslot.size() * sizeof(int2), cudaMemcpyHostToDevice,
                                    ctx.stream));
    STW_CUDA(ctx, cudaFuncSetAttribute(k_peak_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, kPeakSmem));
    STW_KLS(k_peak_warp, (unsigned)nctas, kPeakWarps * 32, kPeakSmem, ctx.stream, b.ev_off, b.size, b.t_s, b.t_e,
            b.dyn, b.horizon, static_only ? 1 : 0, shift, d_wslot, (long long *)d_peak, nbig, big);
  }
  STW_LAUNCHED(ctx);
  return pp;
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
