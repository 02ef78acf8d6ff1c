// Device view of a stw_batch (include/stw.h): stages host inputs into HBM
// once per call and keeps host copies of the small per-trace arrays.
#pragma once
#include <vector>

#include "prims.cuh"

namespace stw {

struct DevBatch {
  int32_t T = 0;
  int64_t N = 0;
  const int64_t *ev_off = nullptr;
  const int64_t *id = nullptr, *size = nullptr;
  const int32_t *t_s = nullptr, *t_e = nullptr, *ps = nullptr, *pe = nullptr;
  const uint8_t *dyn = nullptr;
  const int32_t *horizon = nullptr, *n_sched = nullptr;
  std::vector<int64_t> h_ev_off;
  std::vector<int32_t> h_horizon, h_n_sched;
  int64_t max_trace_events = 0;
  int64_t h2d_bytes = 0;
};

template <class T>
static const T *stage(Ctx &ctx, Arena &ar, const T *src, int64_t n, bool on_device, int64_t *bytes) {
  if (on_device || n == 0 || !ctx.ok()) return src;
  T *d = ar.take<T>(n);
  if (!d) return nullptr;
  STW_CUDA(ctx, cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx.stream));
  *bytes += n * (int64_t)sizeof(T);
  return d;
}

template <class T>
static void fetch_small(Ctx &ctx, std::vector<T> &dst, const T *src, int64_t n, bool on_device) {
  dst.resize(n);
  if (n == 0 || !ctx.ok()) return;
  if (on_device) {
    d2h_async(ctx, dst.data(), src, n * sizeof(T));  // filled by stage_batch's host_sync
  } else {
    memcpy(dst.data(), src, n * sizeof(T));
  }
}

// a compact upload widened on the device: id = base + id32, size = size32 << shift (pipeline.cu)
__global__ void k_widen(const int32_t *__restrict__ id32, const uint32_t *__restrict__ s32, int64_t base, int shift,
                        int64_t n, int64_t *__restrict__ id, int64_t *__restrict__ size);

// `mirror` (optional): the same batch in host memory, read for the small
// per-trace arrays instead of a device round trip (stw_plan_batches stages its
// batches itself and keeps the host originals).
inline bool stage_batch(Ctx &ctx, Arena &ar, const stw_batch *b, DevBatch *d, const stw_batch *mirror = nullptr) {
  if (!b || b->n_traces < 0 || b->n_events < 0) {
    ctx.fail(STW_EARG, "bad batch descriptor");
    return false;
  }
  if (b->n_events > kSortMax) {  // every event-shaped sort goes through K2
    ctx.fail(STW_EARG, "batch too large: %lld events (limit 2^30-1)", (long long)b->n_events);
    return false;
  }
  bool dev = b->on_device != 0;
  d->T = b->n_traces;
  d->N = b->n_events;
  const stw_batch *hs = mirror ? mirror : b;
  const bool fetch_dev = mirror ? false : dev;
  fetch_small(ctx, d->h_ev_off, hs->ev_off, (int64_t)b->n_traces + 1, fetch_dev);
  fetch_small(ctx, d->h_horizon, hs->horizon, b->n_traces, fetch_dev);
  fetch_small(ctx, d->h_n_sched, hs->n_sched, b->n_traces, fetch_dev);
  if (fetch_dev) host_sync(ctx);  // one round trip for the three
  if (!ctx.ok()) return false;
  if (d->h_ev_off[0] != 0 || d->h_ev_off[d->T] != d->N) {
    ctx.fail(STW_EARG, "ev_off must span [0, n_events]");
    return false;
  }
  for (int t = 0; t < d->T; t++) {
    int64_t c = d->h_ev_off[t + 1] - d->h_ev_off[t];
    if (c < 0) {
      ctx.fail(STW_EARG, "ev_off not monotone");
      return false;
    }
    if (c > d->max_trace_events) d->max_trace_events = c;
  }
  int64_t *by = &d->h2d_bytes;
  d->ev_off = stage(ctx, ar, b->ev_off, (int64_t)d->T + 1, dev, by);
  if (!dev && b->id32 && b->size32) {  // compact host columns: 8 bytes less per event, widened on the device
    const int32_t *i32 = stage(ctx, ar, b->id32, d->N, dev, by);
    const uint32_t *s32 = stage(ctx, ar, b->size32, d->N, dev, by);
    int64_t *id = ar.take<int64_t>(d->N + 1), *size = ar.take<int64_t>(d->N + 1);
    if (ctx.ok() && d->N > 0) {
      STW_KL(k_widen, grid_for(d->N, 256), 256, ctx.stream, i32, s32, b->id_base, b->size_shift, d->N, id, size);
      STW_LAUNCHED(ctx);
    }
    d->id = id;
    d->size = size;
  } else {
    d->id = stage(ctx, ar, b->id, d->N, dev, by);
    d->size = stage(ctx, ar, b->size, d->N, dev, by);
  }
  d->t_s = stage(ctx, ar, b->t_s, d->N, dev, by);
  d->t_e = stage(ctx, ar, b->t_e, d->N, dev, by);
  d->ps = stage(ctx, ar, b->ps, d->N, dev, by);
  d->pe = stage(ctx, ar, b->pe, d->N, dev, by);
  d->dyn = stage(ctx, ar, b->dyn, d->N, dev, by);
  d->horizon = stage(ctx, ar, b->horizon, d->T, dev, by);
  d->n_sched = stage(ctx, ar, b->n_sched, d->T, dev, by);
  return ctx.ok();
}

// trace index of event i: binary search over ev_off (T+1 entries)
__device__ __forceinline__ int trace_of(const int64_t *__restrict__ ev_off, int T, int64_t i) {
  int lo = 0, hi = T;  // find last t with ev_off[t] <= i
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(ev_off + mid) <= i)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

void peak_live(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak);
// split form for callers that fold the check into a later host round trip:
// launch, then finish (runs the global-timeline path for flagged traces)
struct PeakPending {
  int *nbig;     // device: traces that need the global-timeline path
  int32_t *big;  // device list of those traces
};
// shift: timeline entries count bytes in units of 2^shift (traces whose sizes
// are not multiples fall back to the global-timeline path)
// pinned: upload the CTA packing through the pinned scratch (h2d_async; the
// caller ends with host_sync) instead of a copy-engine transfer
PeakPending peak_live_launch(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak, int shift,
                             bool pinned = false);
void peak_live_finish(Ctx &ctx, Arena &ar, const DevBatch &b, bool static_only, int64_t *d_peak,
                      const PeakPending &pp);

}  // namespace stw
