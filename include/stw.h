/*
 * libstw -- B200-native (sm_100a) spatio-temporal memory planner and trace
 * replay scorer. Plain C ABI: pointers, sizes and a cudaStream_t passed as
 * void*; no framework types. Every call is synchronous on return and keeps no
 * state between calls that changes its results; calls from different threads
 * may run concurrently. Kept across calls for speed (never for results): a
 * private device memory pool per device for scratch (its memory stays mapped
 * until stw_release_scratch), and per calling thread a mapped page-locked
 * staging buffer plus two side streams and events per device. There is no CPU
 * fallback: without a usable CUDA device every call returns STW_ECUDA.
 *
 * Each entry point replaces a function of the reference Python package
 * (/root/reference/pkg/src/memplan); the citation is next to it. The Python
 * mirror of the reference API (paper_2507_16274_b200/api.py) binds these via
 * ctypes; INTEGRATION.md shows the binding a memplan maintainer would add.
 */
#ifndef STW_H
#define STW_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes -> memplan exceptions (model.py:18-31) */
#define STW_OK 0
#define STW_ETRACE 1 /* TraceError */
#define STW_EPLAN 2  /* PlanError */
#define STW_ESIM 3   /* SimulationError */
#define STW_ECUDA 4  /* CUDA failure / no device */
#define STW_EARG 5   /* bad argument (ValueError) */

/* A batch of traces in structure-of-arrays form, concatenated. Trace t owns
 * events [ev_off[t], ev_off[t+1]). ps/pe are positions in the trace's phase
 * schedule; a value >= n_sched[t] marks a phase missing from the schedule.
 * horizon[t] = end of the last scheduled phase (model.py:197-199).
 * on_device: 1 if every pointer is a device pointer, 0 if all are host
 * pointers (the library then stages them to HBM itself). */
typedef struct {
  int32_t n_traces;
  int32_t on_device;
  int64_t n_events;
  const int64_t *ev_off;
  const int64_t *id;
  const int64_t *size;
  const int32_t *t_s;
  const int32_t *t_e;
  const int32_t *ps;
  const int32_t *pe;
  const uint8_t *dyn;
  const int32_t *horizon;
  const int32_t *n_sched;
  /* optional compact host columns, read by stw_plan_batch(es) when the batch is on the host (which then
   * uploads 8 bytes less per event): id[i] = id_base + id32[i], size[i] =
   * (int64_t)size32[i] << size_shift. NULL: upload id / size as they are. */
  const int32_t *id32;
  const uint32_t *size32;
  int64_t id_base;
  int32_t size_shift;
  int32_t reserved;
} stw_batch;

/* ---- K1: peak live bytes (model.py:261-281) ----------------------------
 * peak[t] = max over time of the bytes live in trace t (half-open lifespans,
 * frees before allocs at equal timestamps). static_only=1 restricts to
 * non-dynamic events (the planner's static_peak, planner.py:465),
 * static_only=0 is clique_lower_bound. peak is a host pointer [n_traces]. */
int stw_peak_live(const stw_batch *b, int32_t static_only, int64_t *peak, void *stream,
                  char *err, size_t errlen);

/* ---- K2: stable LSD radix sort of (u64 key, u32 value) pairs ------------
 * Device pointers, n < 2^30; sorts bits [begin_bit, end_bit) in place. Used by every
 * sort of the hot path (planner.py:82-83,392,419,455,483; sim.py:158,169). */
int stw_radix_sort_pairs(uint64_t *keys, uint32_t *vals, int64_t n, int32_t begin_bit,
                         int32_t end_bit, void *stream, char *err, size_t errlen);

/* ---- scan: device-wide prefix sum of int64 (device pointers; in == out
 * allowed). The running sums of every size / offset computation on the path
 * (pack_group's prefix sums planner.py:98-107, stacking :441-444, the live
 * bytes of peak_live_bytes model.py:261-276); single pass, decoupled
 * look-back. */
int stw_scan_i64(const int64_t *in, int64_t *out, int64_t n, int32_t inclusive, void *stream, char *err,
                 size_t errlen);

/* ---- planner: synthesize_static_plan (planner.py:357-473) ----------------
 * Plans every trace of the batch under each candidate (fusion, gap_insert)
 * setting. Unit u = trace * n_cand + cand. */
#define STW_CAND_FUSION 1
#define STW_CAND_GAP 2
#define STW_NSTATS 12 /* events, persistent, phase_groups, local_plans, residual_events,
                         fusion_attempts, fusion_accepted, gap_insertions, layers,
                         pool_size, static_peak, persistent_size (planner.py:261-294) */
typedef struct {
  int32_t n_cand;
  int32_t select_best; /* pick argmin (pool_size, cand) per trace */
  const uint8_t *cand; /* host [n_cand]: STW_CAND_* bits */
  int64_t alignment;   /* planner.py:362 */
  void *stream;
} stw_plan_opts;

/* Output pointers are host pointers unless on_device=1; any may be NULL.
 * Per-unit event-shaped arrays are laid out [cand][n_events] (the slice of
 * unit (t,c) is c*n_events + ev_off[t] .. ). Layer tables and accepted-fusion
 * audit pairs use the same per-unit slices (capacity = events of the trace). */
typedef struct {
  int32_t on_device;
  int32_t *rc;          /* [units] STW_OK / STW_ETRACE / STW_EPLAN */
  int64_t *err_ids;     /* [units*2] batch event indices named by the error (-1 = none) */
  int64_t *stats;       /* [units*STW_NSTATS] */
  int64_t *addr;        /* [n_cand*n_events] planned address, -1 for dynamic events */
  int32_t *layer_of;    /* [n_cand*n_events] layer index, -1 persistent/dynamic */
  int64_t *layer_base;  /* [n_cand*n_events] per-unit layer table (base) */
  int64_t *layer_size;  /* [n_cand*n_events] per-unit layer table (size) */
  double *fus_tmp;      /* [n_cand*n_events] PlanStats.accepted_fusions[k][0] */
  double *fus_avg;      /* [n_cand*n_events] PlanStats.accepted_fusions[k][1] */
  int32_t *order;       /* [n_events] trace-local index of the k-th event in (t_s,id) order */
  int32_t *best_cand;   /* [n_traces] (select_best) */
  int64_t *addr_best;   /* [n_events] addresses of the best candidate (select_best) */
  int64_t *best_pool;   /* [n_traces] */
} stw_plan_out;

int stw_plan_batch(const stw_batch *b, const stw_plan_opts *opts, stw_plan_out *out, char *err,
                   size_t errlen);

/* The same planner over a sequence of n host batches (host inputs, host
 * outputs out[k] for batch k; every out[k] requests the same fields). HBM
 * staging is double-buffered on a copy stream: batch k+1's host->device copy
 * and batch k-1's results overlap batch k's planning. Results are identical to
 * n stw_plan_batch calls. */
int stw_plan_batches(int32_t n, const stw_batch *b, const stw_plan_opts *opts, stw_plan_out *out, char *err,
                     size_t errlen);

/* ---- K7: validate_plan (planner.py:476-505) -----------------------------
 * Decisions (plan order) as SoA host pointers. Reproduces the reference
 * sweep's report exactly: pairs (i, j) index the decision arrays, in report
 * order. Returns the pair count in *n_pairs (may exceed cap; only cap pairs
 * are written). */
int stw_validate(int64_t n, const int64_t *id, const int64_t *addr, const int64_t *size,
                 const int32_t *t_s, const int32_t *t_e, int64_t *n_pairs, int32_t *pairs,
                 int64_t cap, void *stream, char *err, size_t errlen);

/* ---- K7 over many plans: validate_plan of every (set, candidate) ---------
 * The batched sweep's self-check as one call: decision set s owns
 * rectangles [set_off[s], set_off[s+1]) listed in its sweep order ((t_s, id)
 * order, planner.py:483); t_s/t_e/size are shared by the candidates and addr
 * is [n_cand][n]. All pointers are device pointers. count[s*n_cand + c] (device)
 * receives len(validate_plan(...)) of that plan -- 0 for a valid plan. Plans
 * whose addresses and sizes are multiples of 2^shift take the fast exact
 * overlap sweep; anything else (and any plan with a conflict) the exact
 * reporter. */
typedef struct {
  int32_t n_sets;
  int32_t n_cand;
  int64_t n;
  const int64_t *set_off;
  const int32_t *t_s, *t_e;
  const int64_t *size;
  const int64_t *addr;
} stw_rect_sets;

int stw_validate_sets(const stw_rect_sets *rs, int32_t shift, int64_t *count, void *stream, char *err,
                      size_t errlen);

/* ---- K8: derive_reuse_map (reuse.py:54-93) ------------------------------
 * Static decisions (host SoA) and K key windows [t_lo, t_hi]. Key k's free
 * intervals are out_lo/out_hi[out_off[k] .. out_off[k+1]). Returns STW_EARG
 * with *total set when cap is too small. */
int stw_reuse_map(int64_t n, const int64_t *addr, const int64_t *size, const int32_t *t_s,
                  const int32_t *t_e, int64_t K, const int64_t *t_lo, const int64_t *t_hi,
                  int64_t *out_off, int64_t *out_lo, int64_t *out_hi, int64_t cap, int64_t *total,
                  void *stream, char *err, size_t errlen);

/* ---- K9/K10: simulate (sim.py:143-238) and run_baseline (baseline.py:98-137) */
typedef struct {
  int64_t allocated_peak, reserved_peak, pool_size, fallback_count, fallback_bytes_peak,
      reuse_hits, mismatch_count;
  double efficiency, fragmentation;
} stw_report;

/* Columnar replay log; kind 0 init (size=pool), 1 reserve (size=bytes),
 * 2 alloc, 3 free; space 0 pool / 1 cache; route 0 planned, 1 reuse,
 * 2 fallback, 3 mismatch, 4 online, -1 n/a. Host pointers, capacity cap. */
typedef struct {
  int64_t cap;
  int64_t len;
  int8_t *kind;
  int64_t *t;
  int64_t *id;
  int64_t *size;
  int64_t *addr;
  int8_t *space;
  int8_t *route;
} stw_log;

/* The plan bundle (traceio.py:313-331): decisions in plan order, reuse
 * spaces per key (sp_off/sp_lo/sp_hi), and key[i] = reuse key of dynamic
 * event i of the trace (-1 when the bundle has no entry for it). */
typedef struct {
  int64_t pool_size;
  int64_t alignment;
  int64_t n_dec;
  const int64_t *d_id, *d_addr, *d_size;
  const int32_t *d_ts, *d_te;
  int64_t n_keys;
  const int64_t *sp_off, *sp_lo, *sp_hi;
  const int32_t *key;
  int32_t reuse;
} stw_bundle;

int stw_simulate(const stw_batch *trace, const stw_bundle *plan, stw_report *rep, stw_log *log,
                 int64_t *err_id, void *stream, char *err, size_t errlen);
int stw_baseline(const stw_batch *trace, stw_report *rep, stw_log *log, int64_t *err_id,
                 void *stream, char *err, size_t errlen);

/* ---- sub-operations (the reference's public helpers, one call each) -----
 * Host pointers in and out; the library stages them to HBM. */

/* group_by_phase (planner.py:74-85): rows sorted by (ps, pe, t_s, id) -- ps/pe
 * are order-preserving phase codes (PhaseId order: kind, microbatch, chunk) --
 * into perm[n]; group g = perm[grp_off[g] .. grp_off[g+1]), g < *n_groups
 * (grp_off needs n+1 entries). */
int stw_group_events(int64_t n, const int64_t *ps, const int64_t *pe, const int64_t *t_s, const int64_t *id,
                     int32_t *perm, int64_t *grp_off, int64_t *n_groups, void *stream, char *err, size_t errlen);

/* pack_group / _plan_from_decisions / compute_tmp (planner.py:88-115) over
 * n_plans plans, plan p = members [off[p], off[p+1]) in member order.
 * addr == NULL packs the members contiguously (prefix sums of sizes, written
 * to addr_out if non-NULL); otherwise the given addresses are used. height /
 * t_lo / t_hi = max end address, min t_s, max t_e unless the *_in overrides
 * are given (compute_tmp of an existing LocalPlan). tmp = sum(size * (t_e -
 * t_s)) / (height * (t_hi - t_lo)), correctly rounded (Python int / int);
 * rc[p] = STW_EPLAN for a degenerate lifespan (t_hi <= t_lo). */
typedef struct {
  int64_t n_plans, n;
  const int64_t *off, *size, *t_s, *t_e;
  const int64_t *addr;
  const int64_t *height_in, *t_lo_in, *t_hi_in;
  int64_t *addr_out, *height, *t_lo, *t_hi;
  double *tmp;
  int32_t *rc;
} stw_lplans;
int stw_local_plans(const stw_lplans *p, void *stream, char *err, size_t errlen);

/* weighted_tmp_average (planner.py:118-121): sum(tmp_i * height_i * dur_i) /
 * sum(height_i * dur_i) with CPython float semantics (float(int) round-half-
 * even, the builtin sum's compensated accumulation). */
int stw_weighted_tmp(int64_t n, const double *tmp, const int64_t *height, const int64_t *dur, double *out,
                     void *stream, char *err, size_t errlen);

/* fuse_plans / try_fuse (planner.py:124-182): places the smaller plan's
 * decisions (s_*) into the larger plan's (l_*) by the cursor walk. Outputs:
 * out_addr[i] = address of smaller decision i, out_order = smaller decision
 * indices in placement order; result_i = {fused height, t_s, t_e, rc};
 * result_d = {fused tmp, weighted_tmp_average([larger, smaller])} (given
 * each plan's tmp, height and duration). try_fuse accepts iff
 * result_d[0] > result_d[1]. */
typedef struct {
  int64_t n_large, n_small;
  const int64_t *l_addr, *l_size, *l_ts, *l_te;
  const int64_t *s_id, *s_size, *s_ts, *s_te;
  double l_tmp, s_tmp;
  int64_t l_height, l_dur, s_height, s_dur;
  int64_t *out_addr;
  int32_t *out_order;
  int64_t *result_i;
  double *result_d;
} stw_fusion;
int stw_fuse_plans(const stw_fusion *f, void *stream, char *err, size_t errlen);

/* build_layers_for_size, Alg. 1 (planner.py:236-254): items sorted by
 * (t_s, tie) (order[k] = item index), each joins the layer with the largest
 * end strictly below its start (ties: oldest), else opens a new one.
 * Timestamps are doubles (exact for integers < 2^53). */
int stw_build_layers(int64_t n, const double *t_s, const double *t_e, const int64_t *tie, int32_t *layer_of,
                     int32_t *order, int64_t *n_layers, void *stream, char *err, size_t errlen);

/* compute_metrics (sim.py:67-117) over a columnar log (stw_log encoding;
 * size = pool_size for init records, bytes for reserve records). */
int stw_metrics(int64_t n, const int8_t *kind, const int64_t *size, const int8_t *space, const int8_t *route,
                stw_report *rep, void *stream, char *err, size_t errlen);

/* Return the scratch pool's cached device memory to the driver (synchronizes
 * the device first). */
int stw_release_scratch(void);

/* library identification: returns "stw <version> sm_100a" */
const char *stw_version(void);

/* ---- tracing (diagnostics; off by default) ------------------------------
 * stw_launch_count: kernels launched by this library since load.
 * stw_prof_enable: bracket every launch with CUDA events on its stream.
 * stw_prof_collect: per-kernel launch counts and summed device ms (names in
 * 64-byte slots); returns the number of distinct kernels. */
long long stw_launch_count(void);
void stw_prof_enable(int on);
int stw_prof_collect(char *names, long long *counts, double *ms, int cap, int reset);

#ifdef __cplusplus
}
#endif
#endif
