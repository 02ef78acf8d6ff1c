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
                                   int static_only) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (static_only && dyn[i]) continue;
    int t = trace_of(ev_off, T, i);
    int64_t o = tl_off[t];
    unsigned long long s = (unsigned long long)size[i];
    atomicAdd(D + o + t_s[i], s);
    atomicAdd(D + o + t_e[i], (unsigned long long)(-(long long)s));
  }
}

// per-segment max of the scanned timeline; each thread walks 8 consecutive
// entries and flushes one atomicMax per trace it touched
__global__ void k_segmax(const int64_t *__restrict__ P, int64_t H, const int64_t *__restrict__ tl_off, int T,
                         long long *__restrict__ peak) {
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

void peak_live(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak) {
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
  STW_CUDA(ctx, cudaMemsetAsync(d_peak, 0, T * sizeof(int64_t), ctx.stream));
  STW_KL(k_timeline_scatter, grid_for(b.N, 256), 256, ctx.stream, b.ev_off, T, b.N, b.size, b.t_s, b.t_e, b.dyn,
                                                                 tl_len, (unsigned long long *)D, static_only);
  STW_LAUNCHED(ctx);
  device_scan<int64_t>(ctx, ar, D, D, H, true);
  int64_t nthreads = (H + 7) / 8;
  STW_KL(k_segmax, (unsigned)((nthreads + 255) / 256), 256, ctx.stream, D, H, tl_len, T, (long long *)d_peak);
  STW_LAUNCHED(ctx);
}

}  // namespace stw
