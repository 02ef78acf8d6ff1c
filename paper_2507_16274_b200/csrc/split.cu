// One stw_plan_batch call (host batch) as two concurrent halves.
//
// A planner call has four host round trips (planner phases A-D decide launch
// shapes from device results) and host-side unit layout between them; the GPU
// idles through each (~20% of a c4 call). The traces of a batch are
// independent (every output is per trace, per unit or per event), so a large
// batch is cut at the trace nearest half of its events and the halves run as
// two ordinary calls at once: this thread drives the first on the caller's
// stream, a worker thread the second on its own stream. Each half's kernels
// fill the other's round-trip gaps. The outputs are the unsplit call's:
// contiguous fields are written in place at the half's offset, event indices
// in err_ids are rebased, and the [cand][n_events] fields go through a
// per-half staging buffer and one strided copy.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <iterator>
#include <mutex>
#include <thread>
#include <vector>

#include "planner.cuh"

namespace stw {

int plan_batch(Ctx &ctx, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out, const stw_batch *mirror,
               void (*after_uploads)(void *), void *hook_arg);

namespace {

constexpr int kMaxWorkers = 3;

// persistent worker threads (never joined: they outlive every call)
class Worker {
 public:
  static Worker &get(int i = 0) {  // workers 0 .. kMaxWorkers-1
    static Worker *w[kMaxWorkers] = {};
    static std::mutex mk;
    std::lock_guard<std::mutex> g(mk);
    if (!w[i]) w[i] = new Worker();
    return *w[i];
  }
  std::mutex busy;  // one split call at a time (others run unsplit)
  void run(std::function<void()> f) {
    std::lock_guard<std::mutex> lk(m_);
    job_ = std::move(f);
    has_ = true;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    cv_.wait(lk, [&] { return !has_; });
  }

 private:
  Worker() { std::thread([this] { loop(); }).detach(); }
  void loop() {
    std::unique_lock<std::mutex> lk(m_);
    for (;;) {
      cv_.wait(lk, [&] { return has_; });
      std::function<void()> f = std::move(job_);
      lk.unlock();
      f();
      lk.lock();
      has_ = false;
      cv_.notify_all();
    }
  }
  std::mutex m_;
  std::condition_variable cv_;
  std::function<void()> job_;
  bool has_ = false;
};

// the worker's stream on device `dev` (created once, non-blocking)
cudaStream_t worker_stream(int dev) {
  static thread_local cudaStream_t s[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!s[dev] && cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking) != cudaSuccess) s[dev] = nullptr;
  return s[dev];
}

__global__ void k_rebase_err(int64_t *e, int64_t n, int64_t base) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (e[i] >= 0) e[i] += base;
}

template <class T>
T *shift(T *p, int64_t k) {
  return p ? p + k : nullptr;
}

}  // namespace

// returns false when the call should run unsplit (nothing was done)
bool plan_batch_split(Ctx &ctx, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out) {
  const int64_t T = in->n_traces, N = in->n_events;
  // host batches only: a device batch would first need its per-trace arrays on
  // the host (one more round trip), and measured slower split (1.52 vs 1.42 ms
  // per c4 call with device outputs) than whole; a host batch gains 6% (its
  // uploads and downloads overlap the other half's planning too)
  if ((in->on_device && !getenv("STW_SPLIT_DEVICE")) || T < 1024 || N < (1 << 16) || getenv("STW_NO_SPLIT"))
    return false;
  Worker &wk = Worker::get();
  std::unique_lock<std::mutex> lk(wk.busy, std::try_to_lock);
  if (!lk.owns_lock()) return false;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaStream_t s1 = worker_stream(dev);
  if (!s1) return false;
  // the per-trace arrays on the host (one round trip for a device batch)
  std::vector<int64_t> off(T + 1);
  std::vector<int32_t> hz(T), ns(T);
  const bool dev_in = in->on_device != 0;
  if (dev_in) {
    STW_CUDA(ctx, cudaMemcpyAsync(off.data(), in->ev_off, (T + 1) * 8, cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaMemcpyAsync(hz.data(), in->horizon, T * 4, cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaMemcpyAsync(ns.data(), in->n_sched, T * 4, cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  } else {
    memcpy(off.data(), in->ev_off, (T + 1) * 8);
    memcpy(hz.data(), in->horizon, T * 4);
    memcpy(ns.data(), in->n_sched, T * 4);
  }
  if (!ctx.ok()) return true;
  if (off[0] != 0 || off[T] != N) return false;  // the unsplit call reports it
  int64_t tm = std::lower_bound(off.begin(), off.end(), N / 2) - off.begin();
  tm = std::min<int64_t>(std::max<int64_t>(tm, 1), T - 1);
  const int64_t t0[2] = {0, tm}, t1[2] = {tm, T};
  const int C = o->n_cand;
  Arena ar(&ctx);
  stw_batch sb[2], mir[2];
  stw_plan_out so[2];
  std::vector<int64_t> roff[2];
  int64_t *cn_tmp[2][6] = {};  // staged [cand][n_events] fields per half
  void *cn_dst[6] = {out->addr, out->layer_of, out->layer_base, out->layer_size, out->fus_tmp, out->fus_avg};
  const size_t cn_elt[6] = {8, 4, 8, 8, 8, 8};
  for (int k = 0; k < 2; k++) {
    const int64_t a = t0[k], b = t1[k], e0 = off[a], nk = off[b] - e0;
    roff[k].resize(b - a + 1);
    for (int64_t t = a; t <= b; t++) roff[k][t - a] = off[t] - e0;
    stw_batch s = *in;
    s.n_traces = (int32_t)(b - a);
    s.n_events = nk;
    s.id = shift(in->id, e0), s.size = shift(in->size, e0), s.t_s = shift(in->t_s, e0), s.t_e = shift(in->t_e, e0);
    s.ps = shift(in->ps, e0), s.pe = shift(in->pe, e0), s.dyn = shift(in->dyn, e0);
    s.horizon = shift(in->horizon, a), s.n_sched = shift(in->n_sched, a);
    s.id32 = shift(in->id32, e0), s.size32 = shift(in->size32, e0);
    if (dev_in) {
      int64_t *d = ar.take<int64_t>(b - a + 1);
      if (!ctx.ok()) return true;
      STW_CUDA(ctx, cudaMemcpyAsync(d, roff[k].data(), (b - a + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
      s.ev_off = d;
      mir[k] = s;
      mir[k].on_device = 0;
      mir[k].ev_off = roff[k].data();
      mir[k].horizon = hz.data() + a;
      mir[k].n_sched = ns.data() + a;
    } else {
      s.ev_off = roff[k].data();
    }
    sb[k] = s;
    const int64_t u0 = a * C;
    stw_plan_out q = *out;
    q.rc = shift(out->rc, u0);
    q.err_ids = shift(out->err_ids, 2 * u0);
    q.stats = shift(out->stats, u0 * STW_NSTATS);
    q.order = shift(out->order, e0);
    q.best_cand = shift(out->best_cand, a);
    q.addr_best = shift(out->addr_best, e0);
    q.best_pool = shift(out->best_pool, a);
    for (int f = 0; f < 6; f++) {
      if (!cn_dst[f]) continue;
      cn_tmp[k][f] = (int64_t *)ar.raw((size_t)C * nk * cn_elt[f] + 16);
      if (!ctx.ok()) return true;
    }
    if (out->addr || out->layer_of || out->layer_base || out->layer_size || out->fus_tmp || out->fus_avg) {
      // staged [cand][n_events] fields: the half writes them on the device
      q.on_device = 1;
      if (!out->on_device) {  // then every field of this half goes through the device
        q.rc = q.rc ? ar.take<int32_t>((b - a) * C) : nullptr;
        q.err_ids = q.err_ids ? ar.take<int64_t>(2 * (b - a) * C) : nullptr;
        q.stats = q.stats ? ar.take<int64_t>((b - a) * C * STW_NSTATS) : nullptr;
        q.order = q.order ? ar.take<int32_t>(nk) : nullptr;
        q.best_cand = q.best_cand ? ar.take<int32_t>(b - a) : nullptr;
        q.addr_best = q.addr_best ? ar.take<int64_t>(nk) : nullptr;
        q.best_pool = q.best_pool ? ar.take<int64_t>(b - a) : nullptr;
        if (!ctx.ok()) return true;
      }
    }
    q.addr = (int64_t *)cn_tmp[k][0];
    q.layer_of = (int32_t *)cn_tmp[k][1];
    q.layer_base = cn_tmp[k][2];
    q.layer_size = cn_tmp[k][3];
    q.fus_tmp = (double *)cn_tmp[k][4];
    q.fus_avg = (double *)cn_tmp[k][5];
    so[k] = q;
  }
  // fork: the second half waits for the uploads above
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  STW_CUDA(ctx, cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  STW_CUDA(ctx, cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  STW_CUDA(ctx, cudaEventRecord(ev_fork, ctx.stream));
  if (!ctx.ok()) return true;
  Ctx c1;
  c1.stream = s1;
  std::vector<char> err1(ctx.errlen ? ctx.errlen : 256, 0);
  c1.err = err1.data();
  c1.errlen = err1.size();
  stw_plan_opts o1 = *o;
  o1.stream = s1;
  wk.run([&] {
    cudaSetDevice(dev);
    STW_CUDA(c1, cudaStreamWaitEvent(s1, ev_fork, 0));
    if (c1.ok()) plan_batch(c1, &sb[1], &o1, &so[1], dev_in ? &mir[1] : nullptr, nullptr, nullptr);
    STW_CUDA(c1, cudaEventRecord(ev_join, s1));
  });
  plan_batch(ctx, &sb[0], o, &so[0], dev_in ? &mir[0] : nullptr, nullptr, nullptr);
  wk.wait();
  STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, ev_join, 0));
  if (!c1.ok() && ctx.ok()) ctx.fail(c1.rc, "%s", c1.err);
  if (ctx.ok() && !so[1].on_device && so[1].err_ids)  // host outputs: both halves' copies land first
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  // merge: event indices of the second half are rebased, staged fields placed
  const bool staged = out->addr || out->layer_of || out->layer_base || out->layer_size || out->fus_tmp ||
                      out->fus_avg;
  const cudaMemcpyKind kind = out->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (int k = 0; k < 2 && ctx.ok(); k++) {
    const int64_t a = t0[k], b = t1[k], e0 = off[a], nk = off[b] - e0, u0 = a * C, nu = (b - a) * C;
    const stw_plan_out &q = so[k];
    if (k == 1 && q.err_ids && nu > 0) {
      if (q.on_device) {
        k_rebase_err<<<(unsigned)std::min<int64_t>((2 * nu + 255) / 256, 1184), 256, 0, ctx.stream>>>(q.err_ids, 2 * nu,
                                                                                                     e0);
        STW_LAUNCHED(ctx);
      } else {
        for (int64_t i = 0; i < 2 * nu; i++)
          if (q.err_ids[i] >= 0) q.err_ids[i] += e0;
      }
    }
    if (staged && !out->on_device) {  // this half's contiguous fields were staged on the device too
      auto cp = [&](void *dst, const void *src, size_t bytes) {
        if (dst && src && bytes) STW_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, kind, ctx.stream));
      };
      cp(shift(out->rc, u0), q.rc, nu * 4);
      cp(shift(out->err_ids, 2 * u0), q.err_ids, 2 * nu * 8);
      cp(shift(out->stats, u0 * STW_NSTATS), q.stats, nu * STW_NSTATS * 8);
      cp(shift(out->order, e0), q.order, nk * 4);
      cp(shift(out->best_cand, a), q.best_cand, (b - a) * 4);
      cp(shift(out->addr_best, e0), q.addr_best, nk * 8);
      cp(shift(out->best_pool, a), q.best_pool, (b - a) * 8);
    }
    for (int f = 0; f < 6; f++) {
      if (!cn_dst[f] || nk == 0) continue;
      const size_t el = cn_elt[f];
      STW_CUDA(ctx, cudaMemcpy2DAsync((char *)cn_dst[f] + e0 * el, N * el, cn_tmp[k][f], nk * el, nk * el, C, kind,
                                      ctx.stream));
    }
  }
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));  // (the unsplit call returns with its outputs in place)
  cudaEventDestroy(ev_fork);
  cudaEventDestroy(ev_join);
  return true;
}

int plan_batches(Ctx &ctx, int n, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out);

// stw_plan_batches as L concurrent lanes (default 2, STW_LANES; measured on the
// c4 e2e run: 2 lanes 4.1e9 allocs/s, 3 lanes 0.7-2.6e9, 4 lanes 0.9-2.0e9 --
// beyond two the lanes' host threads, uploads and arena growth contend): batch k on
// lane k % L; lane 0 is the caller's thread and stream, lane j a persistent
// worker thread with its own stream. Each lane is the ordinary pipeline over
// its own subsequence (own staging slots and copy streams). The lanes' kernels
// fill each other's host round trips; every batch's outputs are what
// stw_plan_batch gives for it.
bool plan_batches_2lane(Ctx &ctx, int n, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out) {
  int L = 2;
  if (const char *e = getenv("STW_LANES")) L = atoi(e);
  L = std::min(std::min(L, n), kMaxWorkers + 1);
  if (L < 2 || getenv("STW_NO_SPLIT")) return false;
  {  // outputs shared by batches of different lanes keep the sequential semantics
     // (the last batch's results win): one lane. (Sharing inside a lane is sequential anyway.)
    std::vector<std::pair<const void *, int>> p;
    for (int k = 0; k < n; k++) {
      const stw_plan_out &q = out[k];
      for (const void *x : {(const void *)q.rc, (const void *)q.err_ids, (const void *)q.stats, (const void *)q.addr,
                            (const void *)q.layer_of, (const void *)q.layer_base, (const void *)q.layer_size,
                            (const void *)q.fus_tmp, (const void *)q.fus_avg, (const void *)q.order,
                            (const void *)q.best_cand, (const void *)q.addr_best, (const void *)q.best_pool})
        if (x) p.push_back({x, k % L});
    }
    std::sort(p.begin(), p.end());
    for (size_t i = 1; i < p.size(); i++)
      if (p[i].first == p[i - 1].first && p[i].second != p[i - 1].second) return false;
  }
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int j = 1; j < L; j++) {
    locks.emplace_back(Worker::get(j - 1).busy, std::try_to_lock);
    if (!locks.back().owns_lock()) return false;
  }
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::vector<std::vector<stw_batch>> bi(L);
  std::vector<std::vector<stw_plan_out>> oi(L);
  for (int k = 0; k < n; k++) {
    bi[k % L].push_back(in[k]);
    oi[k % L].push_back(out[k]);
  }
  // the other lanes start after whatever the caller queued before this call
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_join(L, nullptr);
  STW_CUDA(ctx, cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  for (int j = 1; j < L; j++) STW_CUDA(ctx, cudaEventCreateWithFlags(&ev_join[j], cudaEventDisableTiming));
  STW_CUDA(ctx, cudaEventRecord(ev_fork, ctx.stream));
  if (!ctx.ok()) return true;
  std::vector<Ctx> cj(L);
  std::vector<std::vector<char>> errs(L, std::vector<char>(ctx.errlen ? ctx.errlen : 256, 0));
  std::vector<stw_plan_opts> oj(L, *o);
  for (int j = 1; j < L; j++) {
    Ctx &c = cj[j];
    c.stream = nullptr;
    c.err = errs[j].data();
    c.errlen = errs[j].size();
    Worker::get(j - 1).run([&, j] {
      Ctx &c = cj[j];
      cudaSetDevice(dev);
      c.stream = worker_stream(dev);
      if (!c.stream) {
        c.fail(STW_ECUDA, "no worker stream");
        return;
      }
      oj[j].stream = c.stream;
      STW_CUDA(c, cudaStreamWaitEvent(c.stream, ev_fork, 0));
      if (c.ok()) plan_batches(c, (int)bi[j].size(), bi[j].data(), &oj[j], oi[j].data());
      STW_CUDA(c, cudaEventRecord(ev_join[j], c.stream));
      STW_CUDA(c, cudaStreamSynchronize(c.stream));
    });
  }
  plan_batches(ctx, (int)bi[0].size(), bi[0].data(), o, oi[0].data());
  for (int j = 1; j < L; j++) {
    Worker::get(j - 1).wait();
    if (ev_join[j]) STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, ev_join[j], 0));
    if (!cj[j].ok() && ctx.ok()) ctx.fail(cj[j].rc, "%s", cj[j].err);
  }
  cudaEventDestroy(ev_fork);
  for (int j = 1; j < L; j++) cudaEventDestroy(ev_join[j]);
  return true;
}

}  // namespace stw
