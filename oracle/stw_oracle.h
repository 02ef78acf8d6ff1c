/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle.
 *
 * A plain, single-threaded C restatement of the reference `memplan` hot path
 * (/root/reference/pkg/src/memplan/{model,planner,reuse,sim,baseline}.py).
 * Each function cites the reference lines it follows. Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load it; the
 * product (libstw) never links or calls it.
 *
 * Pinned against the reference itself: tests/golden/ holds outputs of the
 * reference on the App. B configs and on fuzz traces (script:
 * tests/golden/make_golden.py), and tests/test_oracle_*.py compare them.
 */
#ifndef STW_ORACLE_H
#define STW_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One trace in SoA form (paper_2507_16274_b200/soa.py). ps/pe >= n_sched
 * means the phase is missing from the schedule. */
typedef struct {
  int64_t n;
  const int64_t *id, *size;
  const int32_t *t_s, *t_e, *ps, *pe;
  const uint8_t *dyn;
  int32_t horizon;
  int32_t n_sched;
} or_trace;

typedef struct {
  int64_t num_events, num_persistent, num_groups, num_plans, num_residuals;
  int64_t fusion_attempts, fusion_accepted, gap_insertions, num_layers;
  int64_t pool_size, static_peak, persistent_size, n_accepted;
} or_stats;

enum { OR_OK = 0, OR_TRACE_ERROR = 1, OR_PLAN_ERROR = 2, OR_SIM_ERROR = 3, OR_CAPACITY = 5 };

/* model.py:261-276 */
int64_t or_peak_live(int64_t n, const int64_t *size, const int32_t *t_s, const int32_t *t_e);

/* planner.py:357-473. addr[i] = planned address of event i (-1 for dynamic),
 * layer_of[i] = index into the layer table (-1 persistent/dynamic).
 * fus_tmp/fus_avg receive PlanStats.accepted_fusions. */
int or_plan(const or_trace *tr, int fusion, int gap_insert, int64_t alignment,
            int64_t *addr, int32_t *layer_of,
            int64_t *layer_base, int64_t *layer_size, int64_t layer_cap,
            double *fus_tmp, double *fus_avg, int64_t fus_cap,
            or_stats *st, char *err, size_t errlen);

/* planner.py:476-505 on decisions (id, addr, size, t_s, t_e) given in plan
 * order. Writes pair indices (into the decision arrays) in reference report
 * order; returns the total number of pairs (may exceed cap). */
int64_t or_validate(int64_t n, const int64_t *id, const int64_t *addr, const int64_t *size,
                    const int32_t *t_s, const int32_t *t_e, int32_t *pairs, int64_t cap);

/* reuse.py:54-80 for K keys: window [t_lo[k], t_hi[k]]. Output intervals of
 * key k are out_lo/out_hi[out_off[k] .. out_off[k+1]). Returns total count or
 * -1 when cap is too small. */
int64_t or_reuse(int64_t n, const int64_t *addr, const int64_t *size, const int32_t *t_s,
                 const int32_t *t_e, int64_t K, const int64_t *t_lo, const int64_t *t_hi,
                 int64_t *out_off, int64_t *out_lo, int64_t *out_hi, int64_t cap);

/* Columnar replay log (sim.py:157-232, baseline.py:98-137). */
typedef struct {
  int64_t cap, len;
  int8_t *kind;   /* 0 init, 1 reserve, 2 alloc, 3 free */
  int64_t *t, *id, *size, *addr;
  int8_t *space;  /* 0 pool, 1 cache */
  int8_t *route;  /* 0 planned, 1 reuse, 2 fallback, 3 mismatch, 4 online; -1 n/a */
  int32_t *key;   /* reuse key index of dynamic allocs, -1 otherwise */
} or_log;

typedef struct {
  int64_t allocated_peak, reserved_peak, pool_size, fallback_count, fallback_bytes_peak,
      reuse_hits, mismatch_count;
  double efficiency, fragmentation;
} or_report;

/* sim.py:143-238. Decisions (plan order) d_id/d_addr/d_size/d_ts/d_te; reuse
 * spaces per key k: sp_lo/sp_hi[sp_off[k]..sp_off[k+1]); key[i] = reuse key
 * index of dynamic event i (-1 = key absent from the plan's map). */
int or_simulate(const or_trace *tr, const int32_t *key, int64_t pool_size, int64_t alignment,
                int64_t nd, const int64_t *d_id, const int64_t *d_addr, const int64_t *d_size,
                const int32_t *d_ts, const int32_t *d_te, int64_t K, const int64_t *sp_off,
                const int64_t *sp_lo, const int64_t *sp_hi, int reuse, or_report *rep,
                or_log *log, int64_t *err_id, char *err, size_t errlen);

/* baseline.py:98-137 */
int or_baseline(const or_trace *tr, or_report *rep, or_log *log, int64_t *err_id, char *err,
                size_t errlen);

#ifdef __cplusplus
}
#endif
#endif
