// Pipelined planner over a sequence of host batches (stw_plan_batches):
// double-buffered HBM staging on a copy stream so batch k+1's host->device copy
// and batch k-1's device->host results overlap batch k's planning on the
// compute stream. Per batch the work and the outputs are exactly those of
// stw_plan_batch on that batch.
#include <string.h>

#include <vector>

#include "planner.cuh"

namespace stw {

int plan_batch(Ctx &ctx, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out, const stw_batch *mirror,
               void (*after_uploads)(void *), void *hook_arg);

namespace {

template <class T>
void h2d(Ctx &ctx, T *dst, const T *src, int64_t n, cudaStream_t s) {
  if (n > 0) STW_CUDA(ctx, cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

template <class T>
void d2h(Ctx &ctx, T *dst, const T *src, int64_t n, cudaStream_t s) {
  if (dst && n > 0) STW_CUDA(ctx, cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

// a compact upload widened on the device: id = base + id32, size = size32 << shift
}  // namespace
__global__ void k_widen(const int32_t *__restrict__ id32, const uint32_t *__restrict__ s32, int64_t base, int shift,
                        int64_t n, int64_t *__restrict__ id, int64_t *__restrict__ size) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    id[i] = base + id32[i];
    size[i] = (int64_t)s32[i] << shift;
  }
}
namespace {

struct Slot {
  // device copies of one batch
  int32_t *id32 = nullptr;
  uint32_t *size32 = nullptr;
  int64_t *ev_off = nullptr, *id = nullptr, *size = nullptr;
  int32_t *t_s = nullptr, *t_e = nullptr, *ps = nullptr, *pe = nullptr, *horizon = nullptr, *n_sched = nullptr;
  uint8_t *dyn = nullptr;
  // device outputs of one batch (only the fields the caller asked for)
  stw_plan_out dout{};
  cudaEvent_t h2d, planned, d2h;
};

template <class T>
T *dalloc(Ctx &ctx, Arena &ar, bool want, int64_t n) {
  return want ? ar.take<T>(n > 0 ? n : 1) : nullptr;
}

}  // namespace

int plan_batches(Ctx &ctx, int n, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out) {
  if (n <= 0) return ctx.rc;
  for (int k = 0; k < n; k++)
    if (in[k].on_device || out[k].on_device) {
      ctx.fail(STW_EARG, "stw_plan_batches takes host batches and host outputs");
      return ctx.rc;
    }
  int64_t maxN = 0, maxT = 0;
  for (int k = 0; k < n; k++) {
    maxN = std::max<int64_t>(maxN, in[k].n_events);
    maxT = std::max<int64_t>(maxT, in[k].n_traces);
  }
  const int C = o->n_cand;
  const int64_t maxU = maxT * C;
  const stw_plan_out &want = out[0];
  // uploads on one copy stream, downloads on another: the two DMA directions
  // run at the same time
  cudaStream_t cs, ds;
  STW_CUDA(ctx, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  STW_CUDA(ctx, cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
  if (!ctx.ok()) return ctx.rc;
  Ctx cctx = ctx;  // copy-stream context (shares the error buffer)
  cctx.stream = cs;
  Ctx dctx = ctx;
  dctx.stream = ds;
  // upload batch k+1 when batch k starts (STW_PIPE_EARLY) or at its phase D
  // (default: measured faster -- the big upload then does not contend with
  // batch k's host round trips over the link)
  const bool early = getenv("STW_PIPE_EARLY") != nullptr;
  {
    Arena ar(&ctx);
    Slot sl[2];
    bool packed = false;
    for (int k = 0; k < n; k++) packed |= in[k].id32 && in[k].size32;
    for (Slot &s : sl) {
      if (packed) {
        s.id32 = ar.take<int32_t>(maxN + 1);
        s.size32 = ar.take<uint32_t>(maxN + 1);
      }
      s.ev_off = ar.take<int64_t>(maxT + 1);
      s.id = ar.take<int64_t>(maxN + 1);
      s.size = ar.take<int64_t>(maxN + 1);
      s.t_s = ar.take<int32_t>(maxN + 1);
      s.t_e = ar.take<int32_t>(maxN + 1);
      s.ps = ar.take<int32_t>(maxN + 1);
      s.pe = ar.take<int32_t>(maxN + 1);
      s.dyn = ar.take<uint8_t>(maxN + 1);
      s.horizon = ar.take<int32_t>(maxT + 1);
      s.n_sched = ar.take<int32_t>(maxT + 1);
      s.dout.on_device = 1;
      s.dout.rc = dalloc<int32_t>(ctx, ar, want.rc, maxU);
      s.dout.err_ids = dalloc<int64_t>(ctx, ar, want.err_ids, 2 * maxU);
      s.dout.stats = dalloc<int64_t>(ctx, ar, want.stats, maxU * STW_NSTATS);
      s.dout.addr = dalloc<int64_t>(ctx, ar, want.addr, C * maxN);
      s.dout.layer_of = dalloc<int32_t>(ctx, ar, want.layer_of, C * maxN);
      s.dout.layer_base = dalloc<int64_t>(ctx, ar, want.layer_base, C * maxN);
      s.dout.layer_size = dalloc<int64_t>(ctx, ar, want.layer_size, C * maxN);
      s.dout.fus_tmp = dalloc<double>(ctx, ar, want.fus_tmp, C * maxN);
      s.dout.fus_avg = dalloc<double>(ctx, ar, want.fus_avg, C * maxN);
      s.dout.order = dalloc<int32_t>(ctx, ar, want.order, maxN);
      s.dout.best_cand = dalloc<int32_t>(ctx, ar, want.best_cand, maxT);
      s.dout.addr_best = dalloc<int64_t>(ctx, ar, want.addr_best, maxN);
      s.dout.best_pool = dalloc<int64_t>(ctx, ar, want.best_pool, maxT);
      cudaEventCreateWithFlags(&s.h2d, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.planned, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.d2h, cudaEventDisableTiming);
    }
    // the slots' scratch was allocated on the compute stream: order the copy stream after it
    cudaEvent_t ready;
    cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    STW_CUDA(ctx, cudaEventRecord(ready, ctx.stream));
    STW_CUDA(ctx, cudaStreamWaitEvent(cs, ready, 0));
    STW_CUDA(ctx, cudaStreamWaitEvent(ds, ready, 0));
    auto stage = [&](int k) {
      Slot &s = sl[k & 1];
      const stw_batch &b = in[k];
      if (k >= 2) STW_CUDA(cctx, cudaStreamWaitEvent(cs, s.planned, 0));  // batch k-2 has read its inputs
      const int64_t N = b.n_events, T = b.n_traces;
      h2d(cctx, s.ev_off, b.ev_off, T + 1, cs);
      if (b.id32 && b.size32) {  // compact columns: 8 bytes less per event over the link
        h2d(cctx, s.id32, b.id32, N, cs);
        h2d(cctx, s.size32, b.size32, N, cs);
        if (N > 0) {
          const int slot = prof_pre(cs);
          k_widen<<<grid_for(N, 256), 256, 0, cs>>>(s.id32, s.size32, b.id_base, b.size_shift, N, s.id, s.size);
          prof_post(cs, "k_widen", slot);
          STW_LAUNCHED(cctx);
        }
      } else {
        h2d(cctx, s.id, b.id, N, cs);
        h2d(cctx, s.size, b.size, N, cs);
      }
      h2d(cctx, s.t_s, b.t_s, N, cs);
      h2d(cctx, s.t_e, b.t_e, N, cs);
      h2d(cctx, s.ps, b.ps, N, cs);
      h2d(cctx, s.pe, b.pe, N, cs);
      h2d(cctx, s.dyn, b.dyn, N, cs);
      h2d(cctx, s.horizon, b.horizon, T, cs);
      h2d(cctx, s.n_sched, b.n_sched, T, cs);
      STW_CUDA(cctx, cudaEventRecord(s.h2d, cs));
    };
    auto download = [&](int k) {  // batch k's results, once it is planned
      Slot &s = sl[k & 1];
      STW_CUDA(dctx, cudaStreamWaitEvent(ds, s.planned, 0));
      const int64_t N = in[k].n_events, T = in[k].n_traces, U = T * C;
      const stw_plan_out &h = out[k];
      d2h(dctx, h.rc, s.dout.rc, U, ds);
      d2h(dctx, h.err_ids, s.dout.err_ids, 2 * U, ds);
      d2h(dctx, h.stats, s.dout.stats, U * STW_NSTATS, ds);
      d2h(dctx, h.addr, s.dout.addr, C * N, ds);
      d2h(dctx, h.layer_of, s.dout.layer_of, C * N, ds);
      d2h(dctx, h.layer_base, s.dout.layer_base, C * N, ds);
      d2h(dctx, h.layer_size, s.dout.layer_size, C * N, ds);
      d2h(dctx, h.fus_tmp, s.dout.fus_tmp, C * N, ds);
      d2h(dctx, h.fus_avg, s.dout.fus_avg, C * N, ds);
      d2h(dctx, h.order, s.dout.order, N, ds);
      d2h(dctx, h.best_cand, s.dout.best_cand, T, ds);
      d2h(dctx, h.addr_best, s.dout.addr_best, N, ds);
      d2h(dctx, h.best_pool, s.dout.best_pool, T, ds);
      STW_CUDA(dctx, cudaEventRecord(s.d2h, ds));
    };
    // Batch k+1's upload and batch k-1's download are issued from inside batch
    // k's planning once its host round trips are done (at the phase D launch):
    // the planner's round trips then never wait behind them, and both overlap
    // the rest of batch k.
    struct Hook {
      int k, n;
      decltype(stage) *st;
      decltype(download) *dl;
      bool ran;
      static void run(void *p) {
        Hook *h = (Hook *)p;
        h->ran = true;
        if (h->k + 1 < h->n) (*h->st)(h->k + 1);
        if (h->k >= 1) (*h->dl)(h->k - 1);
      }
    };
    stage(0);
    int done = 0;  // batches whose download was issued
    for (int k = 0; k < n && ctx.ok() && cctx.ok(); k++) {
      Slot &s = sl[k & 1];
      STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, s.h2d, 0));
      if (k >= 2) STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, s.d2h, 0));  // the slot's results are out
      stw_batch db = in[k];
      db.on_device = 1;
      db.ev_off = s.ev_off;
      db.id = s.id;
      db.size = s.size;
      db.t_s = s.t_s;
      db.t_e = s.t_e;
      db.ps = s.ps;
      db.pe = s.pe;
      db.dyn = s.dyn;
      db.horizon = s.horizon;
      db.n_sched = s.n_sched;
      db.id32 = nullptr;
      db.size32 = nullptr;
      Hook hk{k, n, &stage, &download, false};
      if (early) {  // both transfers start with batch k's planning
        Hook::run(&hk);
        plan_batch(ctx, &db, o, &s.dout, &in[k], nullptr, nullptr);
      } else {
        plan_batch(ctx, &db, o, &s.dout, &in[k], &Hook::run, &hk);
      }
      if (!ctx.ok()) break;
      if (!hk.ran) Hook::run(&hk);  // a batch that returned before phase E (no traces)
      STW_CUDA(ctx, cudaEventRecord(s.planned, ctx.stream));
      done = k;  // downloads of batches < k were issued by the hook
    }
    if (ctx.ok() && cctx.ok())
      for (int k = done; k < n; k++) download(k);
    STW_CUDA(cctx, cudaStreamSynchronize(cs));
    STW_CUDA(dctx, cudaStreamSynchronize(ds));
    // the arena frees on the compute stream: order it after the copy streams' last use
    STW_CUDA(ctx, cudaEventRecord(ready, cs));
    STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, ready, 0));
    STW_CUDA(ctx, cudaEventRecord(ready, ds));
    STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, ready, 0));
    for (Slot &s : sl) {
      cudaEventDestroy(s.h2d);
      cudaEventDestroy(s.planned);
      cudaEventDestroy(s.d2h);
    }
    cudaEventDestroy(ready);
  }
  if (!cctx.ok() && ctx.ok()) ctx.rc = cctx.rc;
  if (!dctx.ok() && ctx.ok()) ctx.rc = dctx.rc;
  cudaStreamDestroy(cs);
  cudaStreamDestroy(ds);
  return ctx.rc;
}

}  // namespace stw
