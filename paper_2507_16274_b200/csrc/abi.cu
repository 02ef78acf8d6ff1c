// C-ABI entry points of libstw (include/stw.h). Each wraps one hot-path
// stage in an error context + scratch arena and is synchronous on return.
#include "planner.cuh"

using namespace stw;

#define STW_ENTRY(stream_ptr, err, errlen) \
  Ctx ctx;                                  \
  ctx.stream = (cudaStream_t)(stream_ptr);  \
  ctx.err = (err);                          \
  ctx.errlen = (errlen);                    \
  if ((err) && (errlen)) (err)[0] = 0;      \
  bind_stream_device(ctx.stream);

static int finish(Ctx &ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx.stream);
  if (e != cudaSuccess) ctx.fail(STW_ECUDA, "stream sync: %s", cudaGetErrorString(e));
  return ctx.rc;
}

namespace stw {
int plan_batch(Ctx &ctx, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out, const stw_batch *mirror,
               void (*after_uploads)(void *), void *hook_arg);
bool plan_batch_split(Ctx &ctx, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out);
bool plan_batches_2lane(Ctx &ctx, int n, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out);
int plan_batches(Ctx &ctx, int n, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out);
int validate_plan_pairs(Ctx &ctx, int64_t n, const int64_t *id, const int64_t *addr, const int64_t *size,
                        const int32_t *t_s, const int32_t *t_e, int64_t *n_pairs, int32_t *pairs, int64_t cap);
int reuse_map(Ctx &ctx, int64_t n, const int64_t *addr, const int64_t *size, const int32_t *t_s, const int32_t *t_e,
              int64_t K, const int64_t *t_lo, const int64_t *t_hi, int64_t *out_off, int64_t *out_lo, int64_t *out_hi,
              int64_t cap, int64_t *total);
int replay(Ctx &ctx, const stw_batch *in, const stw_bundle *bun, stw_report *rep, stw_log *log, int64_t *err_id);
}  // namespace stw

extern "C" {

const char *stw_version(void) { return "stw 0.1.0 sm_100a"; }

int stw_peak_live(const stw_batch *b, int32_t static_only, int64_t *peak, void *stream, char *err,
                  size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  {
    Arena ar(&ctx);
    DevBatch d;
    if (stage_batch(ctx, ar, b, &d)) {
      int64_t *dp = ar.take<int64_t>(d.T > 0 ? d.T : 1);
      peak_live(ctx, ar, d, static_only != 0, dp);
      if (ctx.ok() && d.T > 0)
        STW_CUDA(ctx, cudaMemcpyAsync(peak, dp, d.T * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
    }
  }
  return finish(ctx);
}

int stw_radix_sort_pairs(uint64_t *keys, uint32_t *vals, int64_t n, int32_t begin_bit, int32_t end_bit,
                         void *stream, char *err, size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (begin_bit < 0 || end_bit > 64 || n < 0 || n > kSortMax) {
    ctx.fail(STW_EARG, "bad sort arguments");
    return ctx.rc;
  }
  {
    Arena ar(&ctx);
    radix_sort_pairs(ctx, ar, keys, vals, n, begin_bit, end_bit);
  }
  return finish(ctx);
}

int stw_scan_i64(const int64_t *in, int64_t *out, int64_t n, int32_t inclusive, void *stream, char *err,
                 size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (n < 0 || (n > 0 && (!in || !out))) {
    ctx.fail(STW_EARG, "bad scan arguments");
    return ctx.rc;
  }
  {
    Arena ar(&ctx);
    device_scan<int64_t>(ctx, ar, in, out, n, inclusive != 0);
  }
  return finish(ctx);
}

int stw_plan_batch(const stw_batch *b, const stw_plan_opts *opts, stw_plan_out *out, char *err, size_t errlen) {
  STW_ENTRY(opts ? opts->stream : nullptr, err, errlen);
  if (!b || !opts || !out) {
    ctx.fail(STW_EARG, "null argument");
    return ctx.rc;
  }
  if (!plan_batch_split(ctx, b, opts, out)) plan_batch(ctx, b, opts, out, nullptr, nullptr, nullptr);
  return finish(ctx);
}

int stw_plan_batches(int32_t n, const stw_batch *b, const stw_plan_opts *opts, stw_plan_out *out, char *err,
                     size_t errlen) {
  STW_ENTRY(opts ? opts->stream : nullptr, err, errlen);
  if (n < 0 || (n > 0 && (!b || !opts || !out))) {
    ctx.fail(STW_EARG, "null argument");
    return ctx.rc;
  }
  if (!plan_batches_2lane(ctx, n, b, opts, out)) plan_batches(ctx, n, b, opts, out);
  return finish(ctx);
}

int stw_validate(int64_t n, const int64_t *id, const int64_t *addr, const int64_t *size, const int32_t *t_s,
                 const int32_t *t_e, int64_t *n_pairs, int32_t *pairs, int64_t cap, void *stream, char *err,
                 size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (n < 0 || n > kSortMax || !n_pairs) {  // sorts n decisions (K2 limit)
    ctx.fail(STW_EARG, "bad validate arguments");
    return ctx.rc;
  }
  validate_plan_pairs(ctx, n, id, addr, size, t_s, t_e, n_pairs, pairs, cap);
  return finish(ctx);
}

int stw_validate_sets(const stw_rect_sets *r, int32_t shift, int64_t *count, void *stream, char *err,
                      size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (!r || !count || r->n_sets < 0 || r->n_cand <= 0 || r->n < 0 || shift < 0 || shift > 62) {
    ctx.fail(STW_EARG, "bad validate_sets arguments");
    return ctx.rc;
  }
  {
    Arena ar(&ctx);
    RectSets rs{r->n_sets, r->n, r->set_off, r->t_s, r->t_e, r->size, r->n_cand, r->addr};
    int *first = ar.take<int>((int64_t)r->n_sets * r->n_cand + 1);
    if (ctx.ok() && r->n_sets > 0) validate_sets(ctx, ar, rs, (long long *)count, first, shift);
  }
  return finish(ctx);
}

int stw_reuse_map(int64_t n, const int64_t *addr, const int64_t *size, const int32_t *t_s, const int32_t *t_e,
                  int64_t K, const int64_t *t_lo, const int64_t *t_hi, int64_t *out_off, int64_t *out_lo,
                  int64_t *out_hi, int64_t cap, int64_t *total, void *stream, char *err, size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (n < 0 || n > kSortMax || K < 0 || !total) {  // sorts n decisions (K2 limit)
    ctx.fail(STW_EARG, "bad reuse_map arguments");
    return ctx.rc;
  }
  reuse_map(ctx, n, addr, size, t_s, t_e, K, t_lo, t_hi, out_off, out_lo, out_hi, cap, total);
  return finish(ctx);
}

int stw_simulate(const stw_batch *trace, const stw_bundle *plan, stw_report *rep, stw_log *log, int64_t *err_id,
                 void *stream, char *err, size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (!trace || !plan || !rep || !err_id) {
    ctx.fail(STW_EARG, "null argument");
    return ctx.rc;
  }
  if (2 * trace->n_events > kSortMax) {  // the op order sorts 2n records
    ctx.fail(STW_EARG, "trace too large for replay: %lld events (limit 2^29-1)", (long long)trace->n_events);
    return ctx.rc;
  }
  replay(ctx, trace, plan, rep, log, err_id);
  return finish(ctx);
}

int stw_baseline(const stw_batch *trace, stw_report *rep, stw_log *log, int64_t *err_id, void *stream, char *err,
                 size_t errlen) {
  STW_ENTRY(stream, err, errlen);
  if (!trace || !rep || !err_id) {
    ctx.fail(STW_EARG, "null argument");
    return ctx.rc;
  }
  if (2 * trace->n_events > kSortMax) {  // the op order sorts 2n records
    ctx.fail(STW_EARG, "trace too large for replay: %lld events (limit 2^29-1)", (long long)trace->n_events);
    return ctx.rc;
  }
  replay(ctx, trace, nullptr, rep, log, err_id);
  return finish(ctx);
}

}  // extern "C"
