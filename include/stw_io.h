/*
 * libstw_io -- trace and plan files natively (host C++).
 *
 * Replaces the reference's on-disk formats (memplan/traceio.py): JSONL trace
 * files in the raw (one op per line) and paired (one event per line) layouts,
 * and the single-document JSON plan file. Reading produces the structure-of-
 * arrays libstw consumes (no per-event objects); writing is byte-identical to
 * the reference's canonical output (sort_keys, compact lines / indent=2).
 *
 * Errors: rc STW_ETRACE (trace files) / STW_EPLAN (plan files) with
 * stw_io_error filled. kind STW_IOE_MSG carries the reference's complete
 * message; the other kinds name the line (1-based, header = line 1) whose JSON
 * did not decode or whose record did not convert, so the caller can report it
 * with the exact text of its language's own conversion error.
 */
#ifndef STW_IO_H
#define STW_IO_H
#include <stddef.h>
#include <stdint.h>

#include "stw.h"

#ifdef __cplusplus
extern "C" {
#endif

#define STW_IOE_MSG 1       /* text = the full message */
#define STW_IOE_JSON 2      /* line did not decode as JSON (plan: the document) */
#define STW_IOE_RECORD 3    /* record at `line` failed to convert (malformed record / bad size) */
#define STW_IOE_HEADER 4    /* paired header failed to convert */
#define STW_IOE_OS 5        /* file could not be opened / read / written (errno in `line`) */
#define STW_IOE_PLANDOC 6   /* plan document failed to convert */
#define STW_IOE_INDEX 7     /* raw writer: timestamp outside the slot table (text = index) */
#define STW_IOE_TYPE 8      /* a Python TypeError (text = its message), e.g. an unhashable layer name */

typedef struct {
  int32_t kind;
  int64_t line;
  char text[1024];
} stw_io_error;

/* A parsed, validated trace (parse_trace, traceio.py:48-215, then
 * Trace.validate, model.py:219-251). Phases are canonical tags: the first
 * n_sched form the schedule (with spans), any further ones are referenced by
 * events only. Layers: the first n_known_layers form the layer schedule. */
typedef struct stw_trace_file stw_trace_file;

int stw_trace_read(const char *path, stw_trace_file **out, stw_io_error *e);
void stw_trace_free(stw_trace_file *t);
/* sizes[5] = {events, phase tags, n_sched, layer names, n_known_layers} */
void stw_trace_sizes(const stw_trace_file *t, int64_t *sizes);
/* event columns in the trace's event order (raw: (t_s, id) order) */
void stw_trace_events(const stw_trace_file *t, int64_t *id, int64_t *size, int64_t *t_s, int64_t *t_e, int32_t *ps,
                      int32_t *pe, uint8_t *dyn, int32_t *ls, int32_t *le);
void stw_trace_schedules(const stw_trace_file *t, int64_t *ph_start, int64_t *ph_end, int64_t *ly_start,
                         int64_t *ly_end);
/* NUL-terminated canonical phase tag / layer name k */
const char *stw_trace_phase_tag(const stw_trace_file *t, int64_t k);
const char *stw_trace_layer_name(const stw_trace_file *t, int64_t k);

/* write_trace (traceio.py:222-291). Events as columns (ps/pe index
 * tags[], ls/le index names[] for dynamic events); the schedules as spans of
 * tags[0..n_sched) and names[0..n_layers). form 0 raw, 1 paired. */
typedef struct {
  int64_t n;
  const int64_t *id, *size, *t_s, *t_e;
  const int32_t *ps, *pe, *ls, *le;
  const uint8_t *dyn;
  int64_t n_tags;
  const char *const *tags;
  int64_t n_sched;
  const int64_t *ph_start, *ph_end;
  int64_t n_names;
  const char *const *names;
  int64_t n_layers;
  const int64_t *ly_start, *ly_end;
} stw_trace_cols;

int stw_trace_write(const stw_trace_cols *c, int32_t form, const char *path, stw_io_error *e);

/* Plan files (traceio.py:334-391). Reuse keys are string pairs (l_s, l_e);
 * key k's intervals are lo/hi[iv_off[k] .. iv_off[k+1]). write_plan sorts
 * the keys like the reference (by (l_s, l_e)). */
typedef struct {
  int64_t pool_size, alignment;
  int64_t n_dec;
  const int64_t *id, *addr, *size, *t_s, *t_e;
  int64_t n_keys;
  const char *const *l_s;
  const char *const *l_e;
  const int64_t *iv_off, *iv_lo, *iv_hi;
} stw_plan_cols;

int stw_plan_write(const stw_plan_cols *p, const char *path, stw_io_error *e);

typedef struct stw_plan_file stw_plan_file;
/* read_plan up to (not including) PlanBundle.validate: version check and
 * conversions; reuse intervals as given (the caller builds its interval sets). */
int stw_plan_read(const char *path, stw_plan_file **out, stw_io_error *e);
void stw_plan_free(stw_plan_file *p);
/* sizes[5] = {pool_size, alignment, decisions, keys, intervals} */
void stw_plan_sizes(const stw_plan_file *p, int64_t *sizes);
void stw_plan_decisions(const stw_plan_file *p, int64_t *id, int64_t *addr, int64_t *size, int64_t *t_s,
                        int64_t *t_e);
void stw_plan_reuse(const stw_plan_file *p, int64_t *iv_off, int64_t *iv_lo, int64_t *iv_hi);
const char *stw_plan_key(const stw_plan_file *p, int64_t k, int32_t which);

#ifdef __cplusplus
}
#endif
#endif
