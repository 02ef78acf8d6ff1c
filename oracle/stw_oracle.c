/*
 * TEST INFRASTRUCTURE ONLY -- parity oracle (see stw_oracle.h).
 *
 * Plain restatement of the reference algorithms, deliberately written as the
 * same greedy loops as the Python (no GPU-style decomposition), so that a
 * disagreement with libstw points at libstw. Data structures differ only
 * where the Python relies on O(n) list inserts that would make the full
 * configs take hours in any language (MemoryLayer uses a chunked sorted list
 * with identical bisect semantics).
 */
#define _GNU_SOURCE
#include "stw_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static void set_err(char *err, size_t errlen, const char *fmt, ...) {
  if (!err || !errlen) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

static void *xmalloc(size_t n) {
  void *p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "stw_oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------ */
/* Python numeric semantics                                            */

static int bitlen_u128(u128 x) {
  uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
  if (hi) return 128 - __builtin_clzll(hi);
  if (lo) return 64 - __builtin_clzll(lo);
  return 0;
}

/* Correctly rounded a / b (Python int.__truediv__), a, b > 0. */
static double py_truediv(u128 a, u128 b) {
  const u128 two53 = (u128)1 << 53;
  if (a == 0) return 0.0;
  if (a < two53 && b < two53) return (double)(uint64_t)a / (double)(uint64_t)b;
  u128 q = a / b, r = a % b;
  uint64_t mant;
  int exp, sticky, nq = bitlen_u128(q);
  if (nq >= 54) {
    int sh = nq - 54;
    mant = (uint64_t)(q >> sh);
    sticky = (sh && (q & (((u128)1 << sh) - 1)) != 0) || r != 0;
    exp = sh;
  } else {
    int have = nq;
    mant = (uint64_t)q;
    exp = 0;
    while (have < 54) {
      int carry = (int)(r >> 127);
      r <<= 1;
      int bit = 0;
      if (carry || r >= b) {
        r -= b;
        bit = 1;
      }
      mant = (mant << 1) | (uint64_t)bit;
      exp -= 1;
      if (have > 0 || bit) have++;
    }
    sticky = r != 0;
  }
  int round = (int)(mant & 1);
  mant >>= 1;
  exp += 1;
  if (round && (sticky || (mant & 1))) mant += 1;
  return ldexp((double)mant, exp);
}

/* float(int) -- round half even (PyLong_AsDouble). */
static double py_float(u128 x) { return (double)x; }

/* ------------------------------------------------------------------ */
/* peak_live_bytes: model.py:261-276                                   */

typedef struct {
  int64_t t;
  int is_alloc;
  int64_t size;
} delta_t;

static int cmp_delta(const void *a, const void *b) {
  const delta_t *x = a, *y = b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  if (x->is_alloc != y->is_alloc) return x->is_alloc < y->is_alloc ? -1 : 1;
  if (x->size != y->size) return x->size < y->size ? -1 : 1;
  return 0;
}

int64_t or_peak_live(int64_t n, const int64_t *size, const int32_t *t_s, const int32_t *t_e) {
  delta_t *d = xmalloc(sizeof(delta_t) * (size_t)(2 * n));
  for (int64_t i = 0; i < n; i++) {
    d[2 * i] = (delta_t){t_s[i], 1, size[i]};
    d[2 * i + 1] = (delta_t){t_e[i], 0, size[i]};
  }
  qsort(d, (size_t)(2 * n), sizeof(delta_t), cmp_delta);
  int64_t peak = 0, cur = 0;
  for (int64_t i = 0; i < 2 * n; i++) {
    if (d[i].is_alloc) {
      cur += d[i].size;
      if (cur > peak) peak = cur;
    } else {
      cur -= d[i].size;
    }
  }
  free(d);
  return peak;
}

/* ------------------------------------------------------------------ */
/* planner                                                             */

/* (t_s, id) order of event indices */
static int cmp_tsid(const void *a, const void *b, void *c) {
  const or_trace *tr = c;
  int32_t i = *(const int32_t *)a, j = *(const int32_t *)b;
  if (tr->t_s[i] != tr->t_s[j]) return tr->t_s[i] < tr->t_s[j] ? -1 : 1;
  if (tr->id[i] != tr->id[j]) return tr->id[i] < tr->id[j] ? -1 : 1;
  return 0;
}

/* group order: (phase_index(p_s), phase_index(p_e)) then members (t_s, id)
 * (planner.py:74-85, 390-392) */
static int cmp_group(const void *a, const void *b, void *c) {
  const or_trace *tr = c;
  int32_t i = *(const int32_t *)a, j = *(const int32_t *)b;
  if (tr->ps[i] != tr->ps[j]) return tr->ps[i] < tr->ps[j] ? -1 : 1;
  if (tr->pe[i] != tr->pe[j]) return tr->pe[i] < tr->pe[j] ? -1 : 1;
  return cmp_tsid(a, b, c);
}

typedef struct {
  int32_t ev;
  int64_t addr;
} dec_t;

typedef struct {
  int32_t k0, k1; /* phase indexes of the group key */
  dec_t *d;
  int64_t nd;
  int64_t height;
  int32_t t_s, t_e;
  double tmp;
} lplan_t;

/* _plan_from_decisions + compute_tmp (planner.py:88-115) */
static void plan_finish(const or_trace *tr, lplan_t *p) {
  int64_t h = 0;
  int32_t lo = INT32_MAX, hi = INT32_MIN;
  u128 used = 0;
  for (int64_t k = 0; k < p->nd; k++) {
    int32_t e = p->d[k].ev;
    int64_t end = p->d[k].addr + tr->size[e];
    if (end > h) h = end;
    if (tr->t_s[e] < lo) lo = tr->t_s[e];
    if (tr->t_e[e] > hi) hi = tr->t_e[e];
    used += (u128)tr->size[e] * (u128)(tr->t_e[e] - tr->t_s[e]);
  }
  p->height = h;
  p->t_s = lo;
  p->t_e = hi;
  /* hi > lo always: every event has t_e > t_s */
  p->tmp = py_truediv(used, (u128)h * (u128)(hi - lo));
}

static u128 space_time(const lplan_t *p) { return (u128)p->height * (u128)(p->t_e - p->t_s); }

/* weighted_tmp_average (planner.py:118-121), two plans */
static double weighted_avg2(const lplan_t *a, const lplan_t *b) {
  u128 wa = space_time(a), wb = space_time(b);
  double s = a->tmp * py_float(wa) + b->tmp * py_float(wb);
  return s / py_float(wa + wb);
}

static int conflicts(const or_trace *tr, const dec_t *fixed, int64_t nf, int32_t e, int64_t addr) {
  int64_t hi = addr + tr->size[e];
  for (int64_t k = 0; k < nf; k++) {
    int32_t f = fixed[k].ev;
    if (fixed[k].addr < hi && addr < fixed[k].addr + tr->size[f] && tr->t_s[f] < tr->t_e[e] &&
        tr->t_s[e] < tr->t_e[f])
      return 1;
  }
  return 0;
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return x < y ? -1 : x > y;
}

/* fuse_plans (planner.py:132-169); result owns fresh storage */
static lplan_t fuse_plans(const or_trace *tr, const lplan_t *L, const lplan_t *S) {
  int64_t na = 0;
  int64_t *anchors = xmalloc(sizeof(int64_t) * (size_t)L->nd);
  for (int64_t k = 0; k < L->nd; k++) anchors[k] = L->d[k].addr;
  qsort(anchors, (size_t)L->nd, sizeof(int64_t), cmp_i64);
  for (int64_t k = 0; k < L->nd; k++)
    if (na == 0 || anchors[na - 1] != anchors[k]) anchors[na++] = anchors[k];

  dec_t *fixed = xmalloc(sizeof(dec_t) * (size_t)(L->nd + S->nd));
  memcpy(fixed, L->d, sizeof(dec_t) * (size_t)L->nd);
  int64_t nf = L->nd;
  int32_t *rem = xmalloc(sizeof(int32_t) * (size_t)S->nd);
  for (int64_t k = 0; k < S->nd; k++) rem[k] = S->d[k].ev;
  qsort_r(rem, (size_t)S->nd, sizeof(int32_t), cmp_tsid, (void *)tr);
  char *gone = calloc((size_t)S->nd + 1, 1);
  int64_t left = S->nd, first = 0;
  int64_t addr = anchors[0];
  while (left) {
    int64_t pick = -1;
    for (int64_t k = first; k < S->nd; k++) {
      if (gone[k]) continue;
      if (!conflicts(tr, fixed, nf, rem[k], addr)) {
        pick = k;
        break;
      }
    }
    if (pick >= 0) {
      gone[pick] = 1;
      left--;
      while (first < S->nd && gone[first]) first++;
      fixed[nf++] = (dec_t){rem[pick], addr};
      addr += tr->size[rem[pick]];
    } else {
      int64_t nxt = INT64_MAX;
      for (int64_t k = 0; k < na; k++)
        if (anchors[k] > addr && anchors[k] < nxt) nxt = anchors[k];
      if (nxt == INT64_MAX) {
        nxt = INT64_MIN;
        for (int64_t k = 0; k < nf; k++) {
          int64_t end = fixed[k].addr + tr->size[fixed[k].ev];
          if (end > nxt) nxt = end;
        }
      }
      addr = nxt;
    }
  }
  lplan_t out;
  out.k0 = (L->t_s <= S->t_s ? L : S)->k0;
  out.k1 = (L->t_e >= S->t_e ? L : S)->k1;
  out.d = fixed; /* larger.decisions + placed */
  out.nd = nf;
  plan_finish(tr, &out);
  free(anchors);
  free(rem);
  free(gone);
  return out;
}

/* ---------------- memory layers (planner.py:189-212) --------------- */

#define CHUNK 256
typedef struct {
  int n;
  int32_t ts[CHUNK], te[CHUNK];
} chunk_t;

typedef struct {
  int64_t size;
  int64_t end; /* -1 initially */
  int64_t base;
  chunk_t **ch;
  int nch, capch;
} layer_t;

/* bisect_left over slot starts -> (chunk, offset); chunk == nch means end */
static void layer_pos(const layer_t *L, int32_t t, int *c, int *o) {
  int lo = 0, hi = L->nch; /* first chunk whose last start >= t */
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    const chunk_t *k = L->ch[mid];
    if (k->ts[k->n - 1] >= t)
      hi = mid;
    else
      lo = mid + 1;
  }
  *c = lo;
  if (lo == L->nch) {
    *o = 0;
    return;
  }
  const chunk_t *k = L->ch[lo];
  int a = 0, b = k->n;
  while (a < b) {
    int mid = (a + b) / 2;
    if (k->ts[mid] < t)
      a = mid + 1;
    else
      b = mid;
  }
  *o = a;
}

static int layer_fits_gap(const layer_t *L, int32_t t_s, int32_t t_e) {
  if (L->nch == 0) return 1;
  int c, o;
  layer_pos(L, t_s, &c, &o);
  /* predecessor */
  if (o > 0) {
    if (L->ch[c]->te[o - 1] >= t_s) return 0;
  } else if (c > 0) {
    const chunk_t *p = L->ch[c - 1];
    if (p->te[p->n - 1] >= t_s) return 0;
  }
  /* successor */
  if (c < L->nch && L->ch[c]->ts[o] <= t_e) return 0;
  return 1;
}

static void layer_insert(layer_t *L, int32_t t_s, int32_t t_e) {
  if (L->nch == 0) {
    L->capch = 4;
    L->ch = xmalloc(sizeof(chunk_t *) * 4);
    L->ch[0] = xmalloc(sizeof(chunk_t));
    L->ch[0]->n = 0;
    L->nch = 1;
  }
  int c, o;
  layer_pos(L, t_s, &c, &o);
  if (c == L->nch) {
    c = L->nch - 1;
    o = L->ch[c]->n;
  }
  chunk_t *k = L->ch[c];
  if (k->n == CHUNK) { /* split */
    if (L->nch == L->capch) {
      L->capch *= 2;
      L->ch = realloc(L->ch, sizeof(chunk_t *) * (size_t)L->capch);
    }
    chunk_t *nk = xmalloc(sizeof(chunk_t));
    int half = CHUNK / 2;
    nk->n = CHUNK - half;
    memcpy(nk->ts, k->ts + half, sizeof(int32_t) * (size_t)nk->n);
    memcpy(nk->te, k->te + half, sizeof(int32_t) * (size_t)nk->n);
    k->n = half;
    memmove(L->ch + c + 2, L->ch + c + 1, sizeof(chunk_t *) * (size_t)(L->nch - c - 1));
    L->ch[c + 1] = nk;
    L->nch++;
    if (o > half) {
      o -= half;
      k = nk;
    }
  }
  memmove(k->ts + o + 1, k->ts + o, sizeof(int32_t) * (size_t)(k->n - o));
  memmove(k->te + o + 1, k->te + o, sizeof(int32_t) * (size_t)(k->n - o));
  k->ts[o] = t_s;
  k->te[o] = t_e;
  k->n++;
  if (t_e > L->end) L->end = t_e;
}

static void layer_free(layer_t *L) {
  for (int i = 0; i < L->nch; i++) free(L->ch[i]);
  free(L->ch);
}

typedef struct {
  int64_t size;
  int32_t t_s, t_e;
  int64_t tie;
  int32_t plan; /* >= 0: plan index; -1: residual */
  int32_t ev;   /* residual event */
  int32_t layer;
} item_t;

static int cmp_item_class(const void *a, const void *b) {
  const item_t *x = *(item_t *const *)a, *y = *(item_t *const *)b;
  if (x->size != y->size) return x->size > y->size ? -1 : 1; /* classes descending */
  if (x->t_s != y->t_s) return x->t_s < y->t_s ? -1 : 1;
  if (x->tie != y->tie) return x->tie < y->tie ? -1 : 1;
  return 0;
}

/* validate core shared by or_plan and or_validate (planner.py:476-505) */
typedef struct {
  int64_t t;
  int is_alloc;
  int64_t id;
  int32_t k;
} vop_t;

static int cmp_vop(const void *a, const void *b) {
  const vop_t *x = a, *y = b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  if (x->is_alloc != y->is_alloc) return x->is_alloc < y->is_alloc ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

typedef struct {
  vop_t o;
  int64_t pos;
} sv_t;
static int cmp_sv(const void *a, const void *b) {
  const sv_t *x = a, *y = b;
  int c = cmp_vop(&x->o, &y->o);
  if (c) return c;
  return x->pos < y->pos ? -1 : x->pos > y->pos;
}

int64_t or_validate(int64_t n, const int64_t *id, const int64_t *addr, const int64_t *size,
                    const int32_t *t_s, const int32_t *t_e, int32_t *pairs, int64_t cap) {
  vop_t *ops = xmalloc(sizeof(vop_t) * (size_t)(2 * n));
  for (int64_t k = 0; k < n; k++) {
    ops[2 * k] = (vop_t){t_s[k], 1, id[k], (int32_t)k};
    ops[2 * k + 1] = (vop_t){t_e[k], 0, id[k], (int32_t)k};
  }
  /* Python's sort is stable: equal (t, is_alloc, id) keep list order */
  sv_t *sv = xmalloc(sizeof(sv_t) * (size_t)(2 * n));
  for (int64_t k = 0; k < 2 * n; k++) sv[k] = (sv_t){ops[k], k};
  qsort(sv, (size_t)(2 * n), sizeof(sv_t), cmp_sv);
  for (int64_t k = 0; k < 2 * n; k++) ops[k] = sv[k].o;
  free(sv);
  int64_t *alo = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  int32_t *act = xmalloc(sizeof(int32_t) * (size_t)(n + 1));
  int64_t na = 0, np = 0;
  for (int64_t q = 0; q < 2 * n; q++) {
    int32_t d = ops[q].k;
    int64_t a = addr[d], e = addr[d] + size[d];
    int64_t i = 0, hi = na; /* bisect_left(active_lo, a) */
    while (i < hi) {
      int64_t mid = (i + hi) / 2;
      if (alo[mid] < a)
        i = mid + 1;
      else
        hi = mid;
    }
    if (ops[q].is_alloc) {
      if (i > 0 && alo[i - 1] + size[act[i - 1]] > a) {
        if (np < cap) pairs[2 * np] = act[i - 1], pairs[2 * np + 1] = d;
        np++;
      }
      for (int64_t j = i; j < na && alo[j] < e; j++) {
        if (np < cap) pairs[2 * np] = act[j], pairs[2 * np + 1] = d;
        np++;
      }
      memmove(alo + i + 1, alo + i, sizeof(int64_t) * (size_t)(na - i));
      memmove(act + i + 1, act + i, sizeof(int32_t) * (size_t)(na - i));
      alo[i] = a;
      act[i] = d;
      na++;
    } else {
      while (i < na && act[i] != d) i++;
      if (i < na) {
        memmove(alo + i, alo + i + 1, sizeof(int64_t) * (size_t)(na - i - 1));
        memmove(act + i, act + i + 1, sizeof(int32_t) * (size_t)(na - i - 1));
        na--;
      }
    }
  }
  free(ops);
  free(alo);
  free(act);
  return np;
}

int or_plan(const or_trace *tr, int fusion, int gap_insert, int64_t alignment, int64_t *addr,
            int32_t *layer_of, int64_t *layer_base, int64_t *layer_size, int64_t layer_cap,
            double *fus_tmp, double *fus_avg, int64_t fus_cap, or_stats *st, char *err,
            size_t errlen) {
  const int64_t n = tr->n;
  memset(st, 0, sizeof(*st));
  for (int64_t i = 0; i < n; i++) {
    addr[i] = -1;
    layer_of[i] = -1;
  }
  int32_t *stat = xmalloc(sizeof(int32_t) * (size_t)(n + 1));
  int64_t ns = 0;
  for (int64_t i = 0; i < n; i++)
    if (!tr->dyn[i]) stat[ns++] = (int32_t)i;
  st->num_events = ns;
  for (int64_t k = 0; k < ns; k++) { /* planner.py:371-373 */
    int32_t e = stat[k];
    if (tr->size[e] % alignment) {
      set_err(err, errlen, "event %lld: size %lld not aligned", (long long)tr->id[e],
              (long long)tr->size[e]);
      free(stat);
      return OR_PLAN_ERROR;
    }
  }
  /* persistent block (planner.py:375-388) */
  int32_t *pers = xmalloc(sizeof(int32_t) * (size_t)(ns + 1));
  int32_t *scoped = xmalloc(sizeof(int32_t) * (size_t)(ns + 1));
  int64_t np_ = 0, nsc = 0;
  for (int64_t k = 0; k < ns; k++) {
    int32_t e = stat[k];
    if (tr->t_e[e] >= tr->horizon)
      pers[np_++] = e;
    else
      scoped[nsc++] = e;
  }
  st->num_persistent = np_;
  qsort_r(pers, (size_t)np_, sizeof(int32_t), cmp_tsid, (void *)tr);
  int64_t base = 0;
  for (int64_t k = 0; k < np_; k++) {
    addr[pers[k]] = base;
    base += tr->size[pers[k]];
  }
  int64_t persistent_size = base;

  /* groups (planner.py:390-393); unknown phases -> TraceError */
  for (int64_t k = 0; k < nsc; k++) {
    int32_t e = scoped[k];
    if (tr->ps[e] >= tr->n_sched || tr->pe[e] >= tr->n_sched) {
      set_err(err, errlen, "phase not in schedule");
      free(stat), free(pers), free(scoped);
      return OR_TRACE_ERROR;
    }
  }
  qsort_r(scoped, (size_t)nsc, sizeof(int32_t), cmp_group, (void *)tr);
  lplan_t *plans = xmalloc(sizeof(lplan_t) * (size_t)(nsc + 1));
  int64_t nplans = 0, ngroups = 0;
  int32_t *resid = xmalloc(sizeof(int32_t) * (size_t)(nsc + 1));
  int64_t nres = 0;
  for (int64_t a = 0; a < nsc;) {
    int64_t b = a;
    while (b < nsc && tr->ps[scoped[b]] == tr->ps[scoped[a]] &&
           tr->pe[scoped[b]] == tr->pe[scoped[a]])
      b++;
    ngroups++;
    if (tr->ps[scoped[a]] != tr->pe[scoped[a]]) { /* pack_group (planner.py:98-107) */
      lplan_t p;
      p.k0 = tr->ps[scoped[a]];
      p.k1 = tr->pe[scoped[a]];
      p.nd = b - a;
      p.d = xmalloc(sizeof(dec_t) * (size_t)p.nd);
      int64_t off = 0;
      for (int64_t k = a; k < b; k++) {
        p.d[k - a] = (dec_t){scoped[k], off};
        off += tr->size[scoped[k]];
      }
      plan_finish(tr, &p);
      plans[nplans++] = p;
    } else {
      for (int64_t k = a; k < b; k++) resid[nres++] = scoped[k];
    }
    a = b;
  }
  st->num_groups = ngroups;
  st->num_residuals = nres;

  /* fusion sweep (planner.py:329-354) */
  if (fusion && nplans > 1) {
    int changed = 1;
    while (changed) {
      changed = 0;
      for (int64_t i = 0; i < nplans && !changed; i++) {
        for (int64_t j = i + 1; j < nplans; j++) {
          lplan_t *a = &plans[i], *b = &plans[j];
          if (a->k1 != b->k0 && b->k1 != a->k0) continue;
          lplan_t *L = a->height >= b->height ? a : b;
          lplan_t *S = L == a ? b : a;
          st->fusion_attempts++;
          lplan_t f = fuse_plans(tr, L, S);
          double avg = weighted_avg2(L, S);
          if (!(f.tmp > avg)) {
            free(f.d);
            continue;
          }
          if (st->n_accepted < fus_cap) {
            fus_tmp[st->n_accepted] = f.tmp;
            fus_avg[st->n_accepted] = avg;
          }
          st->n_accepted++;
          st->fusion_accepted++;
          free(plans[i].d);
          free(plans[j].d);
          plans[i] = f;
          memmove(plans + j, plans + j + 1, sizeof(lplan_t) * (size_t)(nplans - j - 1));
          nplans--;
          changed = 1;
          break;
        }
      }
    }
  }
  st->num_plans = nplans;

  /* items (planner.py:408-412) */
  int64_t nit = nplans + nres;
  item_t *items = xmalloc(sizeof(item_t) * (size_t)(nit + 1));
  for (int64_t p = 0; p < nplans; p++) {
    int64_t mid = INT64_MAX;
    for (int64_t k = 0; k < plans[p].nd; k++)
      if (tr->id[plans[p].d[k].ev] < mid) mid = tr->id[plans[p].d[k].ev];
    items[p] = (item_t){plans[p].height, plans[p].t_s, plans[p].t_e, mid, (int32_t)p, -1, -1};
  }
  for (int64_t r = 0; r < nres; r++) {
    int32_t e = resid[r];
    items[nplans + r] = (item_t){tr->size[e], tr->t_s[e], tr->t_e[e], tr->id[e], -1, e, -1};
  }
  item_t **ord = xmalloc(sizeof(item_t *) * (size_t)(nit + 1));
  for (int64_t k = 0; k < nit; k++) ord[k] = &items[k];
  qsort(ord, (size_t)nit, sizeof(item_t *), cmp_item_class);

  /* layers per size class, descending (planner.py:414-438) */
  int64_t nl = 0, capl = 16;
  layer_t *layers = xmalloc(sizeof(layer_t) * (size_t)capl);
  item_t **leftover = xmalloc(sizeof(item_t *) * (size_t)(nit + 1));
  for (int64_t a = 0; a < nit;) {
    int64_t b = a;
    while (b < nit && ord[b]->size == ord[a]->size) b++;
    int64_t nleft = 0;
    for (int64_t k = a; k < b; k++) {
      item_t *it = ord[k];
      int64_t host = -1;
      if (gap_insert) {
        for (int64_t l = 0; l < nl; l++) {
          if (layers[l].size > it->size && (host < 0 || layers[l].size < layers[host].size) &&
              layer_fits_gap(&layers[l], it->t_s, it->t_e))
            host = l;
        }
      }
      if (host >= 0) {
        layer_insert(&layers[host], it->t_s, it->t_e);
        it->layer = (int32_t)host;
        st->gap_insertions++;
      } else {
        leftover[nleft++] = it;
      }
    }
    /* build_layers_for_size (planner.py:236-254); leftovers already (t_s, tie) */
    int64_t first_new = nl;
    for (int64_t k = 0; k < nleft; k++) {
      item_t *it = leftover[k];
      int64_t best = -1;
      for (int64_t l = first_new; l < nl; l++)
        if (layers[l].end < it->t_s && (best < 0 || layers[l].end > layers[best].end)) best = l;
      if (best < 0) {
        if (nl == capl) {
          capl *= 2;
          layers = realloc(layers, sizeof(layer_t) * (size_t)capl);
        }
        layers[nl] = (layer_t){it->size, -1, 0, NULL, 0, 0};
        best = nl++;
      }
      layer_insert(&layers[best], it->t_s, it->t_e);
      it->layer = (int32_t)best;
    }
    a = b;
  }
  st->num_layers = nl;

  /* stacking + emission (planner.py:441-455) */
  for (int64_t l = 0; l < nl; l++) {
    layers[l].base = base;
    if (l < layer_cap) {
      layer_base[l] = base;
      layer_size[l] = layers[l].size;
    }
    base += layers[l].size;
  }
  int64_t pool = base;
  for (int64_t k = 0; k < nit; k++) {
    item_t *it = &items[k];
    int64_t lb = layers[it->layer].base;
    if (it->plan >= 0) {
      lplan_t *p = &plans[it->plan];
      for (int64_t m = 0; m < p->nd; m++) {
        addr[p->d[m].ev] = p->d[m].addr + lb;
        layer_of[p->d[m].ev] = it->layer;
      }
    } else {
      addr[it->ev] = lb;
      layer_of[it->ev] = it->layer;
    }
  }
  st->pool_size = pool;
  st->persistent_size = persistent_size;

  /* self checks (planner.py:464-471) */
  int rc = OR_OK;
  {
    int64_t *ss = xmalloc(sizeof(int64_t) * (size_t)(ns + 1));
    int32_t *ts = xmalloc(sizeof(int32_t) * (size_t)(ns + 1));
    int32_t *te = xmalloc(sizeof(int32_t) * (size_t)(ns + 1));
    int64_t *ii = xmalloc(sizeof(int64_t) * (size_t)(ns + 1));
    int64_t *aa = xmalloc(sizeof(int64_t) * (size_t)(ns + 1));
    for (int64_t k = 0; k < ns; k++) {
      int32_t e = stat[k];
      ss[k] = tr->size[e];
      ts[k] = tr->t_s[e];
      te[k] = tr->t_e[e];
      ii[k] = tr->id[e];
      aa[k] = addr[e];
    }
    st->static_peak = or_peak_live(ns, ss, ts, te);
    if (pool < st->static_peak) {
      set_err(err, errlen, "pool below the static peak; planner invariant broken");
      rc = OR_PLAN_ERROR;
    } else {
      int32_t pr[2];
      int64_t nv = or_validate(ns, ii, aa, ss, ts, te, pr, 1);
      if (nv) {
        set_err(err, errlen, "planner emitted conflicting decisions %lld and %lld",
                (long long)ii[pr[0]], (long long)ii[pr[1]]);
        rc = OR_PLAN_ERROR;
      }
    }
    free(ss), free(ts), free(te), free(ii), free(aa);
  }

  for (int64_t l = 0; l < nl; l++) layer_free(&layers[l]);
  for (int64_t p = 0; p < nplans; p++) free(plans[p].d);
  free(layers), free(leftover), free(ord), free(items), free(plans);
  free(resid), free(stat), free(pers), free(scoped);
  return rc;
}

/* ------------------------------------------------------------------ */
/* reuse.py:54-80                                                      */

typedef struct {
  int64_t lo, hi;
} iv_t;

static int cmp_iv(const void *a, const void *b) {
  const iv_t *x = a, *y = b;
  if (x->lo != y->lo) return x->lo < y->lo ? -1 : 1;
  if (x->hi != y->hi) return x->hi < y->hi ? -1 : 1;
  return 0;
}

int64_t or_reuse(int64_t n, const int64_t *addr, const int64_t *size, const int32_t *t_s,
                 const int32_t *t_e, int64_t K, const int64_t *t_lo, const int64_t *t_hi,
                 int64_t *out_off, int64_t *out_lo, int64_t *out_hi, int64_t cap) {
  int64_t ulo = INT64_MAX, uhi = INT64_MIN;
  for (int64_t i = 0; i < n; i++) {
    if (addr[i] < ulo) ulo = addr[i];
    if (addr[i] + size[i] > uhi) uhi = addr[i] + size[i];
  }
  iv_t *occ = xmalloc(sizeof(iv_t) * (size_t)(n + 1));
  int64_t total = 0;
  for (int64_t k = 0; k < K; k++) {
    out_off[k] = total;
    if (n == 0) continue; /* empty universe */
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++)
      if (t_s[i] < t_hi[k] && t_lo[k] < t_e[i]) occ[m++] = (iv_t){addr[i], addr[i] + size[i]};
    qsort(occ, (size_t)m, sizeof(iv_t), cmp_iv);
    /* coalesce (intervals.py:47-56), then subtract from [ulo, uhi) */
    int64_t cur = ulo;
    int64_t j = 0;
    while (j < m) {
      int64_t lo = occ[j].lo, hi = occ[j].hi;
      j++;
      while (j < m && occ[j].lo <= hi) {
        if (occ[j].hi > hi) hi = occ[j].hi;
        j++;
      }
      if (lo > cur) {
        if (total >= cap) return -1;
        out_lo[total] = cur, out_hi[total] = lo, total++;
      }
      if (hi > cur) cur = hi;
    }
    if (cur < uhi) {
      if (total >= cap) return -1;
      out_lo[total] = cur, out_hi[total] = uhi, total++;
    }
  }
  out_off[K] = total;
  free(occ);
  return total;
}

/* ------------------------------------------------------------------ */
/* id-keyed hash map (Python dict stand-in)                            */

typedef struct {
  int64_t *key;
  int64_t *val;
  uint8_t *st; /* 0 empty, 1 full, 2 tomb */
  int64_t cap, used;
} hmap_t;

static void hm_init(hmap_t *h, int64_t n) {
  int64_t c = 16;
  while (c < 2 * n + 16) c <<= 1;
  h->cap = c;
  h->used = 0;
  h->key = xmalloc(sizeof(int64_t) * (size_t)c);
  h->val = xmalloc(sizeof(int64_t) * (size_t)c);
  h->st = calloc((size_t)c, 1);
}
static void hm_free(hmap_t *h) { free(h->key), free(h->val), free(h->st); }
static uint64_t hm_hash(int64_t k) {
  uint64_t x = (uint64_t)k * 0x9E3779B97F4A7C15ull;
  return x ^ (x >> 29);
}
static int64_t hm_find(const hmap_t *h, int64_t k) {
  uint64_t i = hm_hash(k) & (uint64_t)(h->cap - 1);
  for (;;) {
    if (h->st[i] == 0) return -1;
    if (h->st[i] == 1 && h->key[i] == k) return (int64_t)i;
    i = (i + 1) & (uint64_t)(h->cap - 1);
  }
}
static void hm_put(hmap_t *h, int64_t k, int64_t v) {
  int64_t f = hm_find(h, k);
  if (f >= 0) {
    h->val[f] = v;
    return;
  }
  uint64_t i = hm_hash(k) & (uint64_t)(h->cap - 1);
  while (h->st[i] == 1) i = (i + 1) & (uint64_t)(h->cap - 1);
  h->st[i] = 1;
  h->key[i] = k;
  h->val[i] = v;
}
static void hm_del(hmap_t *h, int64_t slot) { h->st[slot] = 2; }

/* ------------------------------------------------------------------ */
/* caching allocator (baseline.py:35-95)                               */

typedef struct {
  int64_t base, size;
  iv_t *fr;
  int64_t nfr, capfr;
} seg_t;

typedef struct {
  int64_t next_base, min_segment, reserved;
  seg_t *seg;
  int64_t nseg, capseg;
  hmap_t live;      /* id -> slot in lv arrays */
  int64_t *lv_seg, *lv_lo, *lv_hi;
  int64_t nlv, caplv;
} cache_t;

static void cache_init(cache_t *c, int64_t base, int64_t n) {
  memset(c, 0, sizeof(*c));
  c->next_base = base;
  c->min_segment = 2 * 1024 * 1024;
  c->capseg = 16;
  c->seg = xmalloc(sizeof(seg_t) * (size_t)c->capseg);
  hm_init(&c->live, n);
  c->caplv = 2 * n + 16;
  c->lv_seg = xmalloc(sizeof(int64_t) * (size_t)c->caplv);
  c->lv_lo = xmalloc(sizeof(int64_t) * (size_t)c->caplv);
  c->lv_hi = xmalloc(sizeof(int64_t) * (size_t)c->caplv);
}
static void cache_free_all(cache_t *c) {
  for (int64_t s = 0; s < c->nseg; s++) free(c->seg[s].fr);
  free(c->seg);
  hm_free(&c->live);
  free(c->lv_seg), free(c->lv_lo), free(c->lv_hi);
}
static void seg_insert(seg_t *s, int64_t i, iv_t v) {
  if (s->nfr == s->capfr) {
    s->capfr = s->capfr ? 2 * s->capfr : 8;
    s->fr = realloc(s->fr, sizeof(iv_t) * (size_t)s->capfr);
  }
  memmove(s->fr + i + 1, s->fr + i, sizeof(iv_t) * (size_t)(s->nfr - i));
  s->fr[i] = v;
  s->nfr++;
}
static void seg_erase(seg_t *s, int64_t i) {
  memmove(s->fr + i, s->fr + i + 1, sizeof(iv_t) * (size_t)(s->nfr - i - 1));
  s->nfr--;
}
static int64_t next_pow2(int64_t n) {
  int bl = 0;
  uint64_t x = (uint64_t)(n - 1);
  while (x) bl++, x >>= 1;
  return (int64_t)1 << bl;
}
/* returns 0 ok, -1 already live */
static int cache_malloc(cache_t *c, int64_t rid, int64_t size, int64_t *addr, int64_t *grown) {
  if (hm_find(&c->live, rid) >= 0) return -1;
  int64_t bs = -1, bi = -1, blen = 0;
  for (int64_t s = 0; s < c->nseg; s++)
    for (int64_t i = 0; i < c->seg[s].nfr; i++) {
      int64_t len = c->seg[s].fr[i].hi - c->seg[s].fr[i].lo;
      if (len >= size && (bs < 0 || len < blen)) bs = s, bi = i, blen = len;
    }
  *grown = 0;
  if (bs < 0) {
    int64_t ss = next_pow2(size);
    if (ss < c->min_segment) ss = c->min_segment;
    if (c->nseg == c->capseg) {
      c->capseg *= 2;
      c->seg = realloc(c->seg, sizeof(seg_t) * (size_t)c->capseg);
    }
    seg_t *s = &c->seg[c->nseg];
    memset(s, 0, sizeof(*s));
    s->base = c->next_base;
    s->size = ss;
    seg_insert(s, 0, (iv_t){s->base, s->base + ss});
    c->next_base = s->base + ss;
    c->reserved += ss;
    *grown = ss;
    bs = c->nseg++;
    bi = 0;
  }
  seg_t *s = &c->seg[bs];
  iv_t blk = s->fr[bi];
  seg_erase(s, bi);
  *addr = blk.lo;
  if (blk.lo + size < blk.hi) seg_insert(s, bi, (iv_t){blk.lo + size, blk.hi});
  if (c->nlv == c->caplv) {
    c->caplv *= 2;
    c->lv_seg = realloc(c->lv_seg, sizeof(int64_t) * (size_t)c->caplv);
    c->lv_lo = realloc(c->lv_lo, sizeof(int64_t) * (size_t)c->caplv);
    c->lv_hi = realloc(c->lv_hi, sizeof(int64_t) * (size_t)c->caplv);
  }
  c->lv_seg[c->nlv] = bs;
  c->lv_lo[c->nlv] = blk.lo;
  c->lv_hi[c->nlv] = blk.lo + size;
  hm_put(&c->live, rid, c->nlv++);
  return 0;
}
static int cache_owns(const cache_t *c, int64_t rid) { return hm_find(&c->live, rid) >= 0; }
static int cache_free(cache_t *c, int64_t rid, int64_t *addr, int64_t *size) {
  int64_t slot = hm_find(&c->live, rid);
  if (slot < 0) return -1;
  int64_t v = c->live.val[slot];
  hm_del(&c->live, slot);
  seg_t *s = &c->seg[c->lv_seg[v]];
  int64_t lo = c->lv_lo[v], hi = c->lv_hi[v];
  *addr = lo;
  *size = hi - lo;
  /* insort + index (tuple order) */
  int64_t i = 0;
  while (i < s->nfr && (s->fr[i].lo < lo || (s->fr[i].lo == lo && s->fr[i].hi <= hi))) i++;
  seg_insert(s, i, (iv_t){lo, hi});
  /* list.index finds the first equal tuple */
  for (int64_t k = 0; k < s->nfr; k++)
    if (s->fr[k].lo == lo && s->fr[k].hi == hi) {
      i = k;
      break;
    }
  if (i + 1 < s->nfr && s->fr[i + 1].lo == hi) {
    hi = s->fr[i + 1].hi;
    seg_erase(s, i + 1);
    s->fr[i].hi = hi;
  }
  if (i > 0 && s->fr[i - 1].hi == lo) {
    int64_t plo = s->fr[i - 1].lo;
    seg_erase(s, i - 1);
    s->fr[i - 1] = (iv_t){plo, hi};
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* replay                                                              */

static void log_push(or_log *g, int8_t kind, int64_t t, int64_t id, int64_t size, int8_t space,
                     int64_t addr, int8_t route, int32_t key) {
  if (!g) return;
  if (g->len < g->cap) {
    int64_t k = g->len;
    g->kind[k] = kind, g->t[k] = t, g->id[k] = id, g->size[k] = size;
    g->space[k] = space, g->addr[k] = addr, g->route[k] = route, g->key[k] = key;
  }
  g->len++;
}

typedef struct {
  int64_t alloc, cache_live, peak, cache_peak, reserved, fallback, reuse, mismatch;
} metr_t;

static void metr_alloc(metr_t *m, int64_t size, int cache, int route) {
  m->alloc += size;
  if (m->alloc > m->peak) m->peak = m->alloc;
  if (cache) {
    m->cache_live += size;
    if (m->cache_live > m->cache_peak) m->cache_peak = m->cache_live;
  }
  if (route == 2 || route == 3) m->fallback++;
  if (route == 3) m->mismatch++;
  if (route == 1) m->reuse++;
}
static void metr_free(metr_t *m, int64_t size, int cache) {
  m->alloc -= size;
  if (cache) m->cache_live -= size;
}
/* compute_metrics (sim.py:67-117) */
static void metr_report(const metr_t *m, int64_t pool, or_report *r) {
  r->allocated_peak = m->peak;
  r->reserved_peak = pool + m->reserved;
  r->efficiency = r->reserved_peak ? py_truediv((u128)m->peak, (u128)r->reserved_peak) : 1.0;
  r->fragmentation = 1.0 - r->efficiency;
  r->pool_size = pool;
  r->fallback_count = m->fallback;
  r->fallback_bytes_peak = m->cache_peak;
  r->reuse_hits = m->reuse;
  r->mismatch_count = m->mismatch;
}

typedef struct {
  int64_t t;
  int is_alloc;
  int64_t id;
  int64_t pos;
  int32_t ev;
} rop_t;
static int cmp_rop(const void *a, const void *b) {
  const rop_t *x = a, *y = b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  if (x->is_alloc != y->is_alloc) return x->is_alloc < y->is_alloc ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->pos < y->pos ? -1 : x->pos > y->pos;
}
static rop_t *build_ops(const or_trace *tr) {
  rop_t *ops = xmalloc(sizeof(rop_t) * (size_t)(2 * tr->n + 1));
  for (int64_t i = 0; i < tr->n; i++) {
    ops[2 * i] = (rop_t){tr->t_s[i], 1, tr->id[i], 2 * i, (int32_t)i};
    ops[2 * i + 1] = (rop_t){tr->t_e[i], 0, tr->id[i], 2 * i + 1, (int32_t)i};
  }
  qsort(ops, (size_t)(2 * tr->n), sizeof(rop_t), cmp_rop);
  return ops;
}

int or_baseline(const or_trace *tr, or_report *rep, or_log *log, int64_t *err_id, char *err,
                size_t errlen) {
  cache_t c;
  cache_init(&c, 0, tr->n);
  metr_t m = {0};
  if (log) log->len = 0;
  log_push(log, 0, 0, 0, 0, 0, 0, -1, -1);
  rop_t *ops = build_ops(tr);
  int rc = OR_OK;
  for (int64_t q = 0; q < 2 * tr->n; q++) {
    int32_t e = ops[q].ev;
    int64_t id = tr->id[e], t = ops[q].t;
    if (ops[q].is_alloc) {
      int64_t a, g;
      if (cache_malloc(&c, id, tr->size[e], &a, &g)) {
        set_err(err, errlen, "request %lld already live in cache", (long long)id);
        *err_id = id;
        rc = OR_SIM_ERROR;
        break;
      }
      if (g) {
        log_push(log, 1, t, 0, g, 0, 0, -1, -1);
        m.reserved += g;
      }
      log_push(log, 2, t, id, tr->size[e], 1, a, 4, -1);
      metr_alloc(&m, tr->size[e], 1, 4);
    } else {
      int64_t a, s;
      if (cache_free(&c, id, &a, &s)) {
        set_err(err, errlen, "free of unknown id %lld in cache", (long long)id);
        *err_id = id;
        rc = OR_SIM_ERROR;
        break;
      }
      log_push(log, 3, t, id, s, 1, a, -1, -1);
      metr_free(&m, s, 1);
    }
  }
  metr_report(&m, 0, rep);
  free(ops);
  cache_free_all(&c);
  return rc;
}

/* sorted coalesced interval set (intervals.py:37-176) */
typedef struct {
  iv_t *v;
  int64_t n, cap;
} ivs_t;
static void ivs_reserve(ivs_t *s, int64_t n) {
  if (n > s->cap) {
    s->cap = n * 2 + 8;
    s->v = realloc(s->v, sizeof(iv_t) * (size_t)s->cap);
  }
}
static int ivs_contains(const ivs_t *s, int64_t lo, int64_t hi) {
  int64_t a = 0, b = s->n; /* bisect_right on lo */
  while (a < b) {
    int64_t mid = (a + b) / 2;
    if (s->v[mid].lo <= lo)
      a = mid + 1;
    else
      b = mid;
  }
  int64_t i = a - 1;
  return i >= 0 && s->v[i].lo <= lo && hi <= s->v[i].hi;
}
static void ivs_remove(ivs_t *s, int64_t lo, int64_t hi) { /* intervals.py:113-129 */
  int64_t a = 0, b = s->n; /* bisect_right(ivs, lo, key=hi) */
  while (a < b) {
    int64_t mid = (a + b) / 2;
    if (s->v[mid].hi <= lo)
      a = mid + 1;
    else
      b = mid;
  }
  int64_t i = a, j = a;
  iv_t keep[2];
  int nk = 0;
  while (j < s->n && s->v[j].lo < hi) {
    if (s->v[j].lo < lo && nk < 2) keep[nk++] = (iv_t){s->v[j].lo, lo};
    if (s->v[j].hi > hi && nk < 2) keep[nk++] = (iv_t){hi, s->v[j].hi};
    j++;
  }
  int64_t newn = s->n - (j - i) + nk;
  ivs_reserve(s, newn + 1);
  memmove(s->v + i + nk, s->v + j, sizeof(iv_t) * (size_t)(s->n - j));
  for (int k = 0; k < nk; k++) s->v[i + k] = keep[k];
  s->n = newn;
}
static void ivs_add(ivs_t *s, int64_t lo, int64_t hi) { /* intervals.py:100-111 */
  int64_t a = 0, b = s->n; /* bisect_left key=hi, value lo */
  while (a < b) {
    int64_t mid = (a + b) / 2;
    if (s->v[mid].hi < lo)
      a = mid + 1;
    else
      b = mid;
  }
  int64_t li = a;
  a = li, b = s->n; /* bisect_right key=lo, value hi, lo=li */
  while (a < b) {
    int64_t mid = (a + b) / 2;
    if (s->v[mid].lo <= hi)
      a = mid + 1;
    else
      b = mid;
  }
  int64_t hiI = a;
  int64_t nlo = lo, nhi = hi;
  for (int64_t k = li; k < hiI; k++) {
    if (s->v[k].lo < nlo) nlo = s->v[k].lo;
    if (s->v[k].hi > nhi) nhi = s->v[k].hi;
  }
  int64_t newn = s->n - (hiI - li) + 1;
  ivs_reserve(s, newn + 1);
  memmove(s->v + li + 1, s->v + hiI, sizeof(iv_t) * (size_t)(s->n - hiI));
  s->v[li] = (iv_t){nlo, nhi};
  s->n = newn;
}

typedef struct {
  int64_t id, addr, size, t_s;
  int64_t pos;
} qd_t;
static int cmp_qd(const void *a, const void *b) {
  const qd_t *x = a, *y = b;
  if (x->t_s != y->t_s) return x->t_s < y->t_s ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->pos < y->pos ? -1 : x->pos > y->pos;
}

typedef struct {
  int32_t ph;
  int64_t size;
  int64_t ord;
  int64_t addr;
} qe_t;
static int cmp_qe(const void *a, const void *b) {
  const qe_t *x = a, *y = b;
  if (x->ph != y->ph) return x->ph < y->ph ? -1 : 1;
  if (x->size != y->size) return x->size < y->size ? -1 : 1;
  return x->ord < y->ord ? -1 : x->ord > y->ord;
}

int or_simulate(const or_trace *tr, const int32_t *key, int64_t pool_size, int64_t alignment,
                int64_t nd, const int64_t *d_id, const int64_t *d_addr, const int64_t *d_size,
                const int32_t *d_ts, const int32_t *d_te, int64_t K, const int64_t *sp_off,
                const int64_t *sp_lo, const int64_t *sp_hi, int reuse, or_report *rep,
                or_log *log, int64_t *err_id, char *err, size_t errlen) {
  (void)d_te;
  /* PlanBundle.validate (traceio.py:322-331) */
  for (int64_t k = 0; k < nd; k++) {
    if (d_addr[k] < 0 || d_addr[k] + d_size[k] > pool_size) {
      set_err(err, errlen, "decision %lld out of pool", (long long)d_id[k]);
      *err_id = d_id[k];
      return OR_PLAN_ERROR;
    }
    if (d_addr[k] % alignment) {
      set_err(err, errlen, "decision %lld misaligned address %lld", (long long)d_id[k],
              (long long)d_addr[k]);
      *err_id = d_id[k];
      return OR_PLAN_ERROR;
    }
  }
  for (int64_t k = 0; k < K; k++)
    for (int64_t j = sp_off[k]; j < sp_off[k + 1]; j++)
      if (sp_lo[j] < 0 || sp_hi[j] > pool_size) {
        set_err(err, errlen, "reuse entry outside pool");
        *err_id = k;
        return OR_PLAN_ERROR;
      }
  /* events_by_id: last event with a given id wins (dict comprehension) */
  hmap_t byid;
  hm_init(&byid, tr->n);
  for (int64_t i = 0; i < tr->n; i++) hm_put(&byid, tr->id[i], i);
  /* queues keyed by (ev.p_s, d.size), decisions in (t_s, id) order (sim.py:156-162) */
  qd_t *qd = xmalloc(sizeof(qd_t) * (size_t)(nd + 1));
  for (int64_t k = 0; k < nd; k++) qd[k] = (qd_t){d_id[k], d_addr[k], d_size[k], d_ts[k], k};
  qsort(qd, (size_t)nd, sizeof(qd_t), cmp_qd);
  /* queue key -> list; encode key as (phase index, size) and keep per-key FIFO via
   * sorting the eligible decisions by (key, plan order) */
  qe_t *qe = xmalloc(sizeof(qe_t) * (size_t)(nd + 1));
  int64_t nq = 0;
  for (int64_t k = 0; k < nd; k++) {
    int64_t s = hm_find(&byid, qd[k].id);
    if (s < 0) continue;
    int64_t e = byid.val[s];
    if (tr->dyn[e]) continue;
    qe[nq++] = (qe_t){tr->ps[e], qd[k].size, k, qd[k].addr};
  }
  qsort(qe, (size_t)nq, sizeof(qe_t), cmp_qe);
  int64_t *qcur = xmalloc(sizeof(int64_t) * (size_t)(nq + 1)); /* per-run cursor at run start */
  for (int64_t k = 0; k < nq; k++) qcur[k] = k;

  ivs_t fr = {0};
  if (pool_size) {
    ivs_reserve(&fr, 8);
    fr.v[0] = (iv_t){0, pool_size};
    fr.n = 1;
  }
  hmap_t live;
  hm_init(&live, tr->n);
  int64_t *lv_lo = xmalloc(sizeof(int64_t) * (size_t)(tr->n + 1));
  int64_t *lv_hi = xmalloc(sizeof(int64_t) * (size_t)(tr->n + 1));
  int64_t nlv = 0;
  cache_t c;
  cache_init(&c, pool_size, tr->n);
  metr_t m = {0};
  if (log) log->len = 0;
  log_push(log, 0, 0, 0, pool_size, 0, 0, -1, -1);
  rop_t *ops = build_ops(tr);
  ivs_t cand = {0};
  int rc = OR_OK;
  for (int64_t q = 0; q < 2 * tr->n && rc == OR_OK; q++) {
    int32_t e = ops[q].ev;
    int64_t id = tr->id[e], t = ops[q].t, size = tr->size[e];
    if (ops[q].is_alloc) {
      if (tr->dyn[e]) {
        int64_t addr = -1;
        int32_t k = key[e];
        if (reuse && k >= 0 && sp_off[k + 1] > sp_off[k]) { /* dynamic_allocate sim.py:120-140 */
          cand.n = 0;
          int64_t i = 0, j = sp_off[k];
          while (i < fr.n && j < sp_off[k + 1]) { /* intersect (intervals.py:138-154) */
            int64_t lo = fr.v[i].lo > sp_lo[j] ? fr.v[i].lo : sp_lo[j];
            int64_t hi = fr.v[i].hi < sp_hi[j] ? fr.v[i].hi : sp_hi[j];
            if (lo < hi) {
              ivs_reserve(&cand, cand.n + 1);
              cand.v[cand.n++] = (iv_t){lo, hi};
            }
            if (fr.v[i].hi < sp_hi[j])
              i++;
            else
              j++;
          }
          int64_t best = -1; /* best_fit (intervals.py:165-176) */
          for (int64_t z = 0; z < cand.n; z++) {
            int64_t len = cand.v[z].hi - cand.v[z].lo;
            if (len >= size && (best < 0 || len < cand.v[best].hi - cand.v[best].lo)) best = z;
          }
          if (best >= 0) {
            addr = cand.v[best].lo;
            ivs_remove(&fr, addr, addr + size);
          }
        }
        if (addr >= 0) {
          lv_lo[nlv] = addr, lv_hi[nlv] = addr + size;
          hm_put(&live, id, nlv++);
          log_push(log, 2, t, id, size, 0, addr, 1, k);
          metr_alloc(&m, size, 0, 1);
        } else {
          int64_t g;
          if (cache_malloc(&c, id, size, &addr, &g)) {
            set_err(err, errlen, "request %lld already live in cache", (long long)id);
            *err_id = id;
            rc = OR_SIM_ERROR;
            break;
          }
          if (g) {
            log_push(log, 1, t, 0, g, 0, 0, -1, -1);
            m.reserved += g;
          }
          log_push(log, 2, t, id, size, 1, addr, 2, k);
          metr_alloc(&m, size, 1, 2);
        }
      } else {
        /* find the queue for (ps, size): binary search over qe */
        int64_t a = 0, b = nq;
        while (a < b) {
          int64_t mid = (a + b) / 2;
          if (qe[mid].ph < tr->ps[e] || (qe[mid].ph == tr->ps[e] && qe[mid].size < size))
            a = mid + 1;
          else
            b = mid;
        }
        int64_t start = a;
        int have = start < nq && qe[start].ph == tr->ps[e] && qe[start].size == size;
        int64_t slot = -1;
        if (have) {
          slot = qcur[start];
          if (!(slot < nq && qe[slot].ph == tr->ps[e] && qe[slot].size == size)) slot = -1;
        }
        if (slot >= 0) {
          qcur[start] = slot + 1;
          int64_t lo = qe[slot].addr, hi = lo + size;
          if (!ivs_contains(&fr, lo, hi)) {
            set_err(err, errlen, "planned address %lld for event %lld is occupied", (long long)lo,
                    (long long)id);
            *err_id = id;
            rc = OR_SIM_ERROR;
            break;
          }
          ivs_remove(&fr, lo, hi);
          lv_lo[nlv] = lo, lv_hi[nlv] = hi;
          hm_put(&live, id, nlv++);
          log_push(log, 2, t, id, size, 0, lo, 0, -1);
          metr_alloc(&m, size, 0, 0);
        } else {
          int64_t addr, g;
          if (cache_malloc(&c, id, size, &addr, &g)) {
            set_err(err, errlen, "request %lld already live in cache", (long long)id);
            *err_id = id;
            rc = OR_SIM_ERROR;
            break;
          }
          if (g) {
            log_push(log, 1, t, 0, g, 0, 0, -1, -1);
            m.reserved += g;
          }
          log_push(log, 2, t, id, size, 1, addr, 3, -1);
          metr_alloc(&m, size, 1, 3);
        }
      }
    } else {
      int64_t s = hm_find(&live, id);
      if (s >= 0) {
        int64_t v = live.val[s];
        hm_del(&live, s);
        ivs_add(&fr, lv_lo[v], lv_hi[v]);
        log_push(log, 3, t, id, lv_hi[v] - lv_lo[v], 0, lv_lo[v], -1, -1);
        metr_free(&m, lv_hi[v] - lv_lo[v], 0);
      } else if (cache_owns(&c, id)) {
        int64_t a, sz;
        cache_free(&c, id, &a, &sz);
        log_push(log, 3, t, id, sz, 1, a, -1, -1);
        metr_free(&m, sz, 1);
      } else {
        set_err(err, errlen, "double free or free of unknown id %lld", (long long)id);
        *err_id = id;
        rc = OR_SIM_ERROR;
        break;
      }
    }
  }
  metr_report(&m, pool_size, rep);
  free(ops), free(cand.v), free(fr.v), free(lv_lo), free(lv_hi), free(qd), free(qe), free(qcur);
  hm_free(&live);
  hm_free(&byid);
  cache_free_all(&c);
  return rc;
}
