/*
 * memplan_oracle.c — sequential CPU restatement of the reference memplan
 * hot path.  TEST INFRASTRUCTURE ONLY (see memplan_oracle.h): used by
 * tests/ as the parity checker and by bench.py as the cpu_baseline port.
 *
 * Every function follows the reference Python line by line where the
 * arithmetic is observable (float folds, tie-breaks, max/min argument
 * order); data structures are C arrays instead of dicts/sets.  Compile with
 * -ffp-contract=off so no fused multiply-add changes a rounding.
 */
#include "memplan_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define INF (__builtin_inf())
#define EPS_US 1e-6 /* swapsim.py:31 */

static void set_err(mp_err *e, int32_t code, int64_t index, int64_t a0, int64_t a1) {
  if (!e) return;
  e->code = code;
  e->trace = 0;
  e->index = index;
  e->aux0 = a0;
  e->aux1 = a1;
  e->msg[0] = 0;
}

/* Python max(a, b): first maximal argument (b only if b > a) */
static inline double pmax(double a, double b) { return b > a ? b : a; }
static inline double pmin(double a, double b) { return b < a ? b : a; }

/* ---------------------------------------------------------------------- */
/* names: ids are lexicographic ranks; "base#ralloc" compared bytewise     */

static int name_cmp(orc_names nm, int32_t ab, int32_t ar, int32_t bb, int32_t br) {
  if (ar < 0 && br < 0) return (ab > bb) - (ab < bb);
  char sa[32], sb[32];
  int la = 0, lb = 0;
  if (ar >= 0) la = snprintf(sa, sizeof sa, "#%d", ar);
  if (br >= 0) lb = snprintf(sb, sizeof sb, "#%d", br);
  const uint8_t *pa = nm.blob + nm.off[ab], *pb = nm.blob + nm.off[bb];
  int64_t na = nm.off[ab + 1] - nm.off[ab], nb = nm.off[bb + 1] - nm.off[bb];
  int64_t ta = na + la, tb = nb + lb;
  for (int64_t i = 0; i < ta && i < tb; i++) {
    uint8_t ca = i < na ? pa[i] : (uint8_t)sa[i - na];
    uint8_t cb = i < nb ? pb[i] : (uint8_t)sb[i - nb];
    if (ca != cb) return ca < cb ? -1 : 1;
  }
  return (ta > tb) - (ta < tb);
}

/* ---------------------------------------------------------------------- */
/* validate_trace — trace.py:55-84                                          */

int orc_validate(const mp_trace_in *t, mp_err *err) {
  uint8_t *live = calloc((size_t)t->nvars + 1, 1);
  int64_t prev_t = 0;
  int rc = MP_OK;
  for (int64_t pos = 0; pos < t->n; pos++) {
    int64_t idx = t->index ? t->index[pos] : pos;
    if (idx != pos) { set_err(err, MP_E_INVARIANT, pos, MP_V_INDEX, idx); rc = MP_E_INVARIANT; break; }
    if (t->t_us[pos] < 0) { set_err(err, MP_E_INVARIANT, pos, MP_V_NEG_T, 0); rc = MP_E_INVARIANT; break; }
    if (pos > 0 && t->t_us[pos] < prev_t) { set_err(err, MP_E_INVARIANT, pos, MP_V_T_DEC, 0); rc = MP_E_INVARIANT; break; }
    prev_t = t->t_us[pos];
    int32_t v = t->var[pos];
    if (t->kind[pos] == MP_MALLOC) {
      if (t->size[pos] <= 0) { set_err(err, MP_E_INVARIANT, pos, MP_V_MALLOC_SIZE, v); rc = MP_E_INVARIANT; break; }
      if (live[v]) { set_err(err, MP_E_INVARIANT, pos, MP_V_MALLOC_LIVE, v); rc = MP_E_INVARIANT; break; }
      live[v] = 1;
    } else {
      if (t->size[pos] != 0) { set_err(err, MP_E_INVARIANT, pos, MP_V_SIZE_NONZERO, t->kind[pos]); rc = MP_E_INVARIANT; break; }
      if (!live[v]) {
        set_err(err, MP_E_INVARIANT, pos, t->kind[pos] == MP_FREE ? MP_V_FREE_DEAD : MP_V_USE_DEAD, v);
        rc = MP_E_INVARIANT;
        break;
      }
      if (t->kind[pos] == MP_FREE) live[v] = 0;
    }
  }
  free(live);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* detect_iteration — iteration.py:93-105                                   */

static inline int fp_eq(const mp_trace_in *t, int64_t i, int64_t j) {
  return t->kind[i] == t->kind[j] && t->size[i] == t->size[j];
}

/* the reference loop verbatim: O(p^2), small traces only */
int orc_detect_naive(const mp_trace_in *t, int64_t *period, mp_err *err) {
  int64_t n = t->n;
  for (int64_t p = 1; p <= n / 2; p++) {
    int ok = 1;
    for (int64_t i = 0; i < p && ok; i++) ok = fp_eq(t, n - p + i, n - 2 * p + i);
    if (ok) { *period = p; return MP_OK; }
  }
  set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0);
  return MP_E_PERIOD_NOT_FOUND;
}

/* Same answer in O(n): on the reversed fingerprint string R, the loop's
 * test fps[n-p:] == fps[n-2p:n-p] is R[0:p] == R[p:2p], i.e. Z_R[p] >= p. */
int orc_detect(const mp_trace_in *t, int64_t *period, mp_err *err) {
  int64_t n = t->n;
  if (n < 2) { set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0); return MP_E_PERIOD_NOT_FOUND; }
  int64_t *z = calloc((size_t)n, sizeof(int64_t));
#define R(i) (n - 1 - (i))
  int64_t l = 0, r = 0;
  for (int64_t i = 1; i < n; i++) {
    int64_t zi = 0;
    if (i < r) zi = (r - i < z[i - l]) ? r - i : z[i - l];
    while (i + zi < n && fp_eq(t, R(zi), R(i + zi))) zi++;
    z[i] = zi;
    if (i + zi > r) { l = i; r = i + zi; }
  }
#undef R
  int rc = MP_E_PERIOD_NOT_FOUND;
  for (int64_t p = 1; p <= n / 2; p++)
    if (z[p] >= p) { *period = p; rc = MP_OK; break; }
  free(z);
  if (rc) set_err(err, rc, n, 0, 0);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* extract_lifetimes + build_profile — iteration.py:124-301                 */

typedef struct acc_t { int32_t index; uint8_t kind, next; } acc_t;

typedef struct inst_t {
  int32_t base;
  int64_t size;
  int32_t alloc, free_;
  acc_t *acc;
  int64_t nacc, cap;
  int32_t nseg, seg[4];
  uint8_t persistent, wraps, removed, renamed;
  int32_t merged_into; /* old carry-in merged into a twin */
} inst_t;

struct orc_profile {
  mp_profile_dims d;
  int32_t *base, *alloc, *free_, *nseg, *seg, *acc_index, *op_owner;
  int64_t *size, *acc_off, *loads;
  uint8_t *flags, *acc_kind, *acc_next;
  double *op_times;
};

static void acc_push(inst_t *x, acc_t a) {
  if (x->nacc == x->cap) {
    x->cap = x->cap ? 2 * x->cap : 4;
    x->acc = realloc(x->acc, (size_t)x->cap * sizeof(acc_t));
  }
  x->acc[x->nacc++] = a;
}

static int cmp_acc(const void *a, const void *b) {
  const acc_t *x = a, *y = b;
  if (x->next != y->next) return x->next < y->next ? -1 : 1;
  return (x->index > y->index) - (x->index < y->index);
}

static int64_t g_ninst;
static inst_t *g_inst; /* qsort context for variable ordering */

static int cmp_var_order(const void *a, const void *b) {
  const inst_t *x = &g_inst[*(const int32_t *)a], *y = &g_inst[*(const int32_t *)b];
  /* (alloc or -1, name): alloc is unique for window instances; carry-ins
   * (alloc -1) keep their base name, which is unique among them */
  if (x->alloc != y->alloc) return x->alloc < y->alloc ? -1 : 1;
  return (x->base > y->base) - (x->base < y->base);
}

int orc_extract(const mp_trace_in *t, int64_t start, int64_t end, orc_profile **out, mp_err *err) {
  int64_t n = t->n;
  if (!(0 <= start && start < end && end <= n)) {
    set_err(err, MP_E_VALUE, start, end, n);
    return MP_E_VALUE;
  }
  int64_t p = end - start;
  /* op times and period duration: iteration.py:282-291 */
  double *op_times = malloc((size_t)p * sizeof(double));
  int64_t t0 = t->t_us[start];
  for (int64_t r = 0; r < p; r++) op_times[r] = (double)(t->t_us[start + r] - t0);
  double duration;
  if (start >= 1) {
    duration = (double)(t->t_us[end - 1] - t->t_us[start - 1]);
  } else {
    double tail = p > 1 ? op_times[p - 1] - op_times[p - 2] : 1.0;
    duration = op_times[p - 1] + pmax(tail, 1.0);
  }
  if (duration <= op_times[p - 1]) duration = op_times[p - 1] + 1.0;

  /* _live_at (iteration.py:124-132): last malloc/free before start */
  int32_t nv = t->nvars;
  int64_t *live_idx = malloc((size_t)(nv + 1) * sizeof(int64_t));
  for (int32_t v = 0; v < nv; v++) live_idx[v] = -1;
  for (int64_t i = 0; i < start; i++) {
    if (t->kind[i] == MP_MALLOC) live_idx[t->var[i]] = i;
    else if (t->kind[i] == MP_FREE) live_idx[t->var[i]] = -1;
  }

  int64_t cap = p + nv + 1;
  inst_t *inst = calloc((size_t)cap, sizeof(inst_t));
  int64_t ninst = 0;
  int32_t *open_i = malloc((size_t)(nv + 1) * sizeof(int32_t));
  int32_t *carry_i = malloc((size_t)(nv + 1) * sizeof(int32_t));
  int64_t *twin_rel = malloc((size_t)(nv + 1) * sizeof(int64_t));
  int32_t *resolved = malloc((size_t)p * sizeof(int32_t));
  int64_t *pre_b = malloc((size_t)(p + 1) * sizeof(int64_t));
  int64_t npre = 0;
  for (int32_t v = 0; v < nv; v++) { open_i[v] = -1; carry_i[v] = -1; }
  /* live_start: carry-ins (iteration.py:293-297, 154-157) */
  for (int32_t v = 0; v < nv; v++) {
    if (live_idx[v] < 0) continue;
    inst_t *x = &inst[ninst];
    x->base = v; x->size = t->size[live_idx[v]]; x->alloc = -1; x->free_ = -1;
    x->merged_into = -1;
    carry_i[v] = (int32_t)ninst++;
    twin_rel[v] = live_idx[v] >= start - p ? live_idx[v] - (start - p) : -1;
  }
  int rc = MP_OK;
  /* main pass, iteration.py:159-187 */
  for (int64_t r = 0; r < p && rc == MP_OK; r++) {
    int64_t i = start + r;
    int32_t b = t->var[i];
    uint8_t k = t->kind[i];
    if (k == MP_MALLOC) {
      if (open_i[b] >= 0) { set_err(err, MP_E_INVARIANT, r, MP_V_W_MALLOC_LIVE, b); rc = MP_E_INVARIANT; break; }
      inst_t *x = &inst[ninst];
      x->base = b; x->size = t->size[i]; x->alloc = (int32_t)r; x->free_ = -1; x->merged_into = -1;
      open_i[b] = (int32_t)ninst;
      resolved[r] = (int32_t)ninst++;
    } else if (k == MP_FREE) {
      if (open_i[b] >= 0) {
        inst_t *x = &inst[open_i[b]];
        x->free_ = (int32_t)r; x->nseg = 1; x->seg[0] = x->alloc; x->seg[1] = (int32_t)r;
        resolved[r] = open_i[b];
        open_i[b] = -1;
      } else if (carry_i[b] >= 0 && inst[carry_i[b]].free_ < 0) {
        inst[carry_i[b]].free_ = (int32_t)r;
        pre_b[npre++] = b;
        resolved[r] = carry_i[b];
      } else { set_err(err, MP_E_INVARIANT, r, MP_V_W_FREE_DEAD, b); rc = MP_E_INVARIANT; break; }
    } else {
      int32_t o;
      if (open_i[b] >= 0) o = open_i[b];
      else if (carry_i[b] >= 0 && inst[carry_i[b]].free_ < 0) o = carry_i[b];
      else { set_err(err, MP_E_INVARIANT, r, MP_V_W_USE_DEAD, b); rc = MP_E_INVARIANT; break; }
      acc_push(&inst[o], (acc_t){(int32_t)r, k, 0});
      resolved[r] = o;
    }
  }
  if (rc == MP_OK) {
    /* open_by_alloc: instances still open after the pass */
    int32_t *open_by_alloc = malloc((size_t)p * sizeof(int32_t));
    for (int64_t r = 0; r < p; r++) open_by_alloc[r] = -1;
    for (int64_t j = 0; j < ninst; j++)
      if (inst[j].alloc >= 0 && open_i[inst[j].base] == j) open_by_alloc[inst[j].alloc] = (int32_t)j;
    /* twin pairing, iteration.py:193-225 */
    for (int64_t q = 0; q < npre; q++) {
      int32_t b = (int32_t)pre_b[q];
      inst_t *old = &inst[carry_i[b]];
      int64_t r_f = old->free_;
      int32_t tw = twin_rel[b] >= 0 && twin_rel[b] < p ? open_by_alloc[twin_rel[b]] : -1;
      inst_t *twin = tw >= 0 ? &inst[tw] : NULL;
      if (twin && twin->size == old->size && twin->free_ < 0 && r_f <= twin->alloc) {
        twin->free_ = (int32_t)r_f; twin->wraps = 1; twin->nseg = 2;
        twin->seg[0] = twin->alloc; twin->seg[1] = (int32_t)p; twin->seg[2] = 0; twin->seg[3] = (int32_t)r_f;
        for (int64_t a = 0; a < old->nacc; a++) {
          acc_t e = old->acc[a];
          e.next = 1;
          acc_push(twin, e);
        }
        qsort(twin->acc, (size_t)twin->nacc, sizeof(acc_t), cmp_acc);
        open_i[twin->base] = -1;
        old->removed = 1;
        old->merged_into = tw;
      } else if (twin && twin->size == old->size && twin->free_ < 0) {
        old->nseg = 1; old->seg[0] = 0; old->seg[1] = (int32_t)r_f;
        twin->wraps = 1; twin->nseg = 1; twin->seg[0] = twin->alloc; twin->seg[1] = (int32_t)p;
        open_i[twin->base] = -1;
      } else {
        old->nseg = 1; old->seg[0] = 0; old->seg[1] = (int32_t)p; old->wraps = 1;
      }
      carry_i[b] = -1; /* popped from start_insts */
    }
    free(open_by_alloc);
    /* iteration.py:227-234 */
    for (int32_t v = 0; v < nv; v++) {
      if (carry_i[v] >= 0) {
        inst_t *x = &inst[carry_i[v]];
        x->persistent = 1; x->nseg = 1; x->seg[0] = 0; x->seg[1] = (int32_t)p;
      }
      if (open_i[v] >= 0) {
        inst_t *x = &inst[open_i[v]];
        x->persistent = 1; x->wraps = 1; x->nseg = 1; x->seg[0] = 0; x->seg[1] = (int32_t)p;
      }
    }
    /* renames, iteration.py:236-241 */
    int32_t *cnt = calloc((size_t)nv + 1, sizeof(int32_t));
    for (int64_t j = 0; j < ninst; j++) if (!inst[j].removed) cnt[inst[j].base]++;
    for (int64_t j = 0; j < ninst; j++)
      if (!inst[j].removed && cnt[inst[j].base] > 1 && inst[j].alloc >= 0) inst[j].renamed = 1;
    free(cnt);
    /* variable order (iteration.py:257-260) */
    int32_t *ord = malloc((size_t)(ninst + 1) * sizeof(int32_t));
    int64_t V = 0, ncarry = 0, nacc = 0;
    for (int64_t j = 0; j < ninst; j++) if (!inst[j].removed) ord[V++] = (int32_t)j;
    g_inst = inst;
    g_ninst = ninst;
    qsort(ord, (size_t)V, sizeof(int32_t), cmp_var_order);
    int32_t *pos_of = malloc((size_t)(ninst + 1) * sizeof(int32_t));
    for (int64_t q = 0; q < V; q++) {
      pos_of[ord[q]] = (int32_t)q;
      if (inst[ord[q]].alloc < 0) ncarry++;
      nacc += inst[ord[q]].nacc;
    }
    orc_profile *P = calloc(1, sizeof(orc_profile));
    P->d.period = p; P->d.nvars = V; P->d.ncarry = ncarry; P->d.naccess = nacc;
    P->d.duration_us = duration;
    P->base = malloc((size_t)(V + 1) * 4); P->alloc = malloc((size_t)(V + 1) * 4);
    P->free_ = malloc((size_t)(V + 1) * 4); P->nseg = malloc((size_t)(V + 1) * 4);
    P->seg = malloc((size_t)(V + 1) * 16); P->size = malloc((size_t)(V + 1) * 8);
    P->flags = malloc((size_t)(V + 1)); P->acc_off = malloc((size_t)(V + 1) * 8);
    P->acc_index = malloc((size_t)(nacc + 1) * 4); P->acc_kind = malloc((size_t)(nacc + 1));
    P->acc_next = malloc((size_t)(nacc + 1)); P->op_times = op_times;
    P->loads = malloc((size_t)p * 8); P->op_owner = malloc((size_t)p * 4);
    int64_t ao = 0;
    for (int64_t q = 0; q < V; q++) {
      inst_t *x = &inst[ord[q]];
      P->base[q] = x->base; P->alloc[q] = x->alloc; P->free_[q] = x->free_;
      P->nseg[q] = x->nseg; memcpy(&P->seg[4 * q], x->seg, 16); P->size[q] = x->size;
      P->flags[q] = (uint8_t)((x->persistent ? MP_F_PERSISTENT : 0) | (x->wraps ? MP_F_WRAPS : 0) |
                              (x->renamed ? MP_F_RENAMED : 0));
      P->acc_off[q] = ao;
      for (int64_t a = 0; a < x->nacc; a++, ao++) {
        P->acc_index[ao] = x->acc[a].index; P->acc_kind[ao] = x->acc[a].kind; P->acc_next[ao] = x->acc[a].next;
      }
    }
    P->acc_off[V] = ao;
    for (int64_t r = 0; r < p; r++) {
      int32_t o = resolved[r];
      if (inst[o].merged_into >= 0) o = inst[o].merged_into;
      P->op_owner[r] = pos_of[o];
    }
    /* compute_load_profile, iteration.py:304-320 */
    int64_t *diff = calloc((size_t)p + 1, 8);
    for (int64_t q = 0; q < V; q++)
      for (int s = 0; s < P->nseg[q]; s++) {
        diff[P->seg[4 * q + 2 * s]] += P->size[q];
        diff[P->seg[4 * q + 2 * s + 1]] -= P->size[q];
      }
    int64_t acc = 0, peak = 0, peak_i = 0;
    for (int64_t r = 0; r < p; r++) {
      acc += diff[r];
      P->loads[r] = acc;
      if (r == 0 || acc > peak) { peak = acc; peak_i = r; }
    }
    free(diff);
    P->d.peak_bytes = peak; P->d.peak_index = peak_i;
    free(ord); free(pos_of);
    *out = P;
    op_times = NULL;
  }
  for (int64_t j = 0; j < ninst; j++) free(inst[j].acc);
  free(inst); free(open_i); free(carry_i); free(twin_rel); free(resolved); free(pre_b);
  free(live_idx); free(op_times);
  return rc;
}

int orc_profile_dims(const orc_profile *p, mp_profile_dims *d) { *d = p->d; return MP_OK; }

int orc_profile_copy(const orc_profile *P, mp_profile_out *o) {
  int64_t V = P->d.nvars, A = P->d.naccess, p = P->d.period;
  memcpy(o->base, P->base, (size_t)V * 4); memcpy(o->size, P->size, (size_t)V * 8);
  memcpy(o->alloc, P->alloc, (size_t)V * 4); memcpy(o->free_, P->free_, (size_t)V * 4);
  memcpy(o->nseg, P->nseg, (size_t)V * 4); memcpy(o->seg, P->seg, (size_t)V * 16);
  memcpy(o->flags, P->flags, (size_t)V); memcpy(o->acc_off, P->acc_off, (size_t)(V + 1) * 8);
  memcpy(o->acc_index, P->acc_index, (size_t)A * 4); memcpy(o->acc_kind, P->acc_kind, (size_t)A);
  memcpy(o->acc_next, P->acc_next, (size_t)A); memcpy(o->op_times, P->op_times, (size_t)p * 8);
  memcpy(o->loads, P->loads, (size_t)p * 8); memcpy(o->op_owner, P->op_owner, (size_t)p * 4);
  return MP_OK;
}

void orc_profile_free(orc_profile *P) {
  if (!P) return;
  free(P->base); free(P->alloc); free(P->free_); free(P->nseg); free(P->seg); free(P->size);
  free(P->flags); free(P->acc_off); free(P->acc_index); free(P->acc_kind); free(P->acc_next);
  free(P->op_times); free(P->loads); free(P->op_owner); free(P);
}

/* ---------------------------------------------------------------------- */
/* conflict_graph_from_arcs — smartpool.py:51-79 (endpoint sweep)           */

struct orc_graph {
  int64_t V;
  int64_t *row_off;
  int32_t *col;
};

typedef struct ev_t { int64_t point; int32_t phase, var; } ev_t;

static int cmp_ev(const void *a, const void *b) {
  const ev_t *x = a, *y = b;
  if (x->point != y->point) return x->point < y->point ? -1 : 1;
  if (x->phase != y->phase) return x->phase - y->phase;
  return (x->var > y->var) - (x->var < y->var);
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

typedef struct vec32 { int32_t *a; int64_t n, cap; } vec32;
static void vpush(vec32 *v, int32_t x) {
  if (v->n == v->cap) { v->cap = v->cap ? 2 * v->cap : 8; v->a = realloc(v->a, (size_t)v->cap * 4); }
  v->a[v->n++] = x;
}

int orc_conflict(int32_t nvars, const int64_t *seg_off, const int32_t *lo, const int32_t *hi,
                 orc_graph **out) {
  int64_t ns = seg_off[nvars], ne = 0;
  ev_t *ev = malloc((size_t)(2 * ns + 1) * sizeof(ev_t));
  for (int32_t i = 0; i < nvars; i++)
    for (int64_t s = seg_off[i]; s < seg_off[i + 1]; s++) {
      if (hi[s] <= lo[s]) continue;
      ev[ne++] = (ev_t){lo[s], 1, i};
      ev[ne++] = (ev_t){hi[s], 0, i};
    }
  qsort(ev, (size_t)ne, sizeof(ev_t), cmp_ev);
  vec32 *adj = calloc((size_t)nvars + 1, sizeof(vec32));
  /* active set: dense list + position map */
  int32_t *act = malloc((size_t)nvars * 4 + 4), *where = malloc((size_t)nvars * 4 + 4);
  int64_t nact = 0;
  for (int32_t i = 0; i < nvars; i++) where[i] = -1;
  for (int64_t q = 0; q < ne; q++) {
    int32_t i = ev[q].var;
    if (ev[q].phase == 0) {
      if (where[i] >= 0) {
        int32_t w = where[i], last = act[--nact];
        act[w] = last; where[last] = w; where[i] = -1;
      }
    } else {
      for (int64_t a = 0; a < nact; a++) {
        int32_t j = act[a];
        if (j != i) { vpush(&adj[i], j); vpush(&adj[j], i); }
      }
      if (where[i] < 0) { where[i] = (int32_t)nact; act[nact++] = i; }
    }
  }
  orc_graph *g = malloc(sizeof(orc_graph));
  g->V = nvars;
  g->row_off = malloc((size_t)(nvars + 1) * 8);
  int64_t tot = 0;
  for (int32_t i = 0; i < nvars; i++) {
    qsort(adj[i].a, (size_t)adj[i].n, 4, cmp_i32);
    int64_t u = 0;
    for (int64_t k = 0; k < adj[i].n; k++)
      if (u == 0 || adj[i].a[k] != adj[i].a[u - 1]) adj[i].a[u++] = adj[i].a[k];
    adj[i].n = u;
    g->row_off[i] = tot;
    tot += u;
  }
  g->row_off[nvars] = tot;
  g->col = malloc((size_t)(tot + 1) * 4);
  for (int32_t i = 0; i < nvars; i++) {
    if (adj[i].n) memcpy(g->col + g->row_off[i], adj[i].a, (size_t)adj[i].n * 4);
    free(adj[i].a);
  }
  free(adj); free(ev); free(act); free(where);
  *out = g;
  return MP_OK;
}

int64_t orc_graph_nnz(const orc_graph *g) { return g->row_off[g->V]; }
void orc_graph_copy(const orc_graph *g, int64_t *row_off, int32_t *col) {
  memcpy(row_off, g->row_off, (size_t)(g->V + 1) * 8);
  memcpy(col, g->col, (size_t)g->row_off[g->V] * 4);
}
void orc_graph_free(orc_graph *g) {
  if (!g) return;
  free(g->row_off); free(g->col); free(g);
}

/* ---------------------------------------------------------------------- */
/* plan_pool — smartpool.py:91-144                                          */

typedef struct pctx { const int64_t *size, *alloc; const int32_t *nb, *nr; orc_names nm; } pctx;
static pctx g_p;

static int cmp_place(const void *a, const void *b) {
  int32_t i = *(const int32_t *)a, j = *(const int32_t *)b;
  /* key (-size, alloc, name) */
  if (g_p.size[i] != g_p.size[j]) return g_p.size[i] > g_p.size[j] ? -1 : 1;
  if (g_p.alloc[i] != g_p.alloc[j]) return g_p.alloc[i] < g_p.alloc[j] ? -1 : 1;
  return name_cmp(g_p.nm, g_p.nb[i], g_p.nr[i], g_p.nb[j], g_p.nr[j]);
}

typedef struct iv_t { int64_t s, e; } iv_t;
static int cmp_iv(const void *a, const void *b) {
  const iv_t *x = a, *y = b;
  if (x->s != y->s) return x->s < y->s ? -1 : 1;
  return (x->e > y->e) - (x->e < y->e);
}

/* _pick_offset, smartpool.py:101-119 */
static int64_t pick_offset(const iv_t *occ, int64_t m, int64_t need, int32_t policy) {
  int64_t top = 0, best_len = 0, best_off = 0;
  int have = 0;
  for (int64_t q = 0; q < m; q++) {
    int64_t s = occ[q].s, e = occ[q].e;
    if (s > top) {
      int64_t off = top, len = s - top;
      if (len >= need) {
        if (policy == 0) return off;
        if (!have || len < best_len || (len == best_len && off < best_off)) {
          best_len = len; best_off = off; have = 1;
        }
      }
    }
    if (e > top) top = e;
  }
  return have ? best_off : top;
}

int orc_plan(const orc_graph *g, const int64_t *size, const int64_t *alloc,
             const int32_t *name_base, const int32_t *name_ralloc, orc_names names,
             int32_t policy, int64_t *offsets, int64_t *footprint) {
  if (policy != 0 && policy != 1) return MP_E_VALUE;
  int64_t V = g->V;
  int32_t *ord = malloc((size_t)(V + 1) * 4);
  for (int64_t i = 0; i < V; i++) ord[i] = (int32_t)i;
  g_p = (pctx){size, alloc, name_base, name_ralloc, names};
  qsort(ord, (size_t)V, 4, cmp_place);
  uint8_t *placed = calloc((size_t)V + 1, 1);
  int64_t maxdeg = 0;
  for (int64_t i = 0; i < V; i++) {
    int64_t d = g->row_off[i + 1] - g->row_off[i];
    if (d > maxdeg) maxdeg = d;
  }
  iv_t *occ = malloc((size_t)(maxdeg + 1) * sizeof(iv_t));
  for (int64_t q = 0; q < V; q++) {
    int32_t i = ord[q];
    int64_t m = 0;
    for (int64_t k = g->row_off[i]; k < g->row_off[i + 1]; k++) {
      int32_t j = g->col[k];
      if (placed[j]) occ[m++] = (iv_t){offsets[j], offsets[j] + size[j]};
    }
    qsort(occ, (size_t)m, sizeof(iv_t), cmp_iv);
    offsets[i] = pick_offset(occ, m, size[i], policy);
    placed[i] = 1;
  }
  int64_t fp = 0;
  for (int64_t i = 0; i < V; i++) {
    int64_t e = offsets[i] + size[i];
    if (i == 0 || e > fp) fp = e;
  }
  *footprint = V ? fp : 0;
  free(ord); free(placed); free(occ);
  return MP_OK;
}

/* ---------------------------------------------------------------------- */
/* swap candidates — autoswap.py:26-116                                     */

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

int64_t orc_candidates(const mp_profile_dims *d, const mp_profile_out *P, int64_t threshold,
                       double bw, double lat, orc_cands *C) {
  int64_t p = d->period, k = 0, peak = d->peak_index;
  int64_t maxacc = 0;
  for (int64_t v = 0; v < d->nvars; v++) {
    int64_t m = P->acc_off[v + 1] - P->acc_off[v];
    if (m > maxacc) maxacc = m;
  }
  int64_t *co = malloc((size_t)(maxacc + 2) * 8);
  for (int64_t v = 0; v < d->nvars; v++) {
    if (P->size[v] < threshold) continue;
    /* _access_pairs, autoswap.py:53-66 */
    int64_t m = 0;
    for (int64_t a = P->acc_off[v]; a < P->acc_off[v + 1]; a++)
      co[m++] = P->acc_index[a] + (P->acc_next[a] ? p : 0);
    qsort(co, (size_t)m, 8, cmp_i64);
    int found = 0;
    int64_t c1 = 0, c2 = 0;
    int64_t npairs = m > 0 ? m - 1 : 0;
    int persistent = (P->flags[v] & MP_F_PERSISTENT) != 0;
    for (int64_t q = 0; q < npairs + ((persistent && m) ? 1 : 0) && !found; q++) {
      int64_t a, b;
      if (q < npairs) {
        a = co[q]; b = co[q + 1];
        if (!(a < b)) continue;
      } else {
        a = co[m - 1]; b = co[0] + p;
      }
      /* _peak_pair, autoswap.py:69-77 */
      if (a >= p) { a -= p; b -= p; }
      if ((a < peak && peak < b) || (a < peak + p && peak + p < b)) { c1 = a; c2 = b; found = 1; }
    }
    if (!found) continue;
    int spans = c2 >= p;
    double t1 = P->op_times[c1];
    double t2 = P->op_times[c2 % p] + (spans ? d->duration_us : 0.0);
    double delta = (double)P->size[v] / bw * 1e6 + lat;
    C->var[k] = (int32_t)v;
    C->size[k] = P->size[v];
    C->out_index[k] = (int32_t)c1;
    C->out_t[k] = t1;
    C->out_ready[k] = c1 + 1 < p ? P->op_times[c1 + 1] : d->duration_us;
    C->in_index[k] = (int32_t)(c2 % p);
    C->in_t[k] = t2;
    C->dout[k] = delta;
    C->din[k] = delta;
    C->spans[k] = (uint8_t)spans;
    C->name_base[k] = P->base[v];
    C->name_ralloc[k] = (P->flags[v] & MP_F_RENAMED) ? P->alloc[v] : -1;
    k++;
  }
  free(co);
  C->k = k;
  return k;
}

/* _step_area, autoswap.py:145-161 */
static double step_area(orc_load L, const double *cur, double a, double b) {
  if (b <= a) return 0.0;
  int64_t p = L.period;
  /* bisect_right(op_times, a) - 1, floored at 0 */
  int64_t lo = 0, hi = p;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (a < L.op_times[mid]) hi = mid; else lo = mid + 1;
  }
  int64_t r0 = lo - 1 < 0 ? 0 : lo - 1;
  double total = 0.0;
  for (int64_t r = r0; r < p; r++) {
    double s = L.op_times[r];
    double e = r + 1 < p ? L.op_times[r + 1] : L.duration;
    if (s >= b) break;
    double ov = pmin(b, e) - pmax(a, s);
    if (ov > 0) total += cur[r] * ov;
  }
  return total;
}

/* gap_area, autoswap.py:164-174 */
double orc_gap_area(orc_load L, const double *cur, double a, double b) {
  double d = L.duration;
  if (b <= d) return step_area(L, cur, a, b);
  return step_area(L, cur, a, d) + step_area(L, cur, 0.0, b - d);
}

/* apply_absence over absence_slots, autoswap.py:119-129 */
static void absence(int64_t p, const orc_cands *c, int64_t i, double *cur) {
  int64_t c2 = c->in_index[i] + (c->spans[i] ? p : 0);
  for (int64_t x = c->out_index[i] + 1; x < c2; x++) cur[x % p] -= (double)c->size[i];
}

static double vmax(const double *x, int64_t n) {
  double m = x[0];
  for (int64_t i = 1; i < n; i++) m = pmax(m, x[i]);
  return m;
}

/* exact Python float <= int comparison */
static int f_le_i(double f, int64_t i) {
  if (f != f) return 0;
  if (f >= 9223372036854775808.0) return 0;
  if (f < -9223372036854775808.0) return 1;
  double fl = floor(f);
  int64_t q = (int64_t)fl;
  if (q < i) return 1;
  if (q > i) return 0;
  return fl == f; /* q == i: f <= i iff f has no fractional part */
}

/* _swdoa_greedy, autoswap.py:181-207; peaks[j] = max(cur) after j picks */
static int64_t swdoa_greedy(orc_load L, const orc_cands *c, orc_names nm, int has_limit,
                            int64_t limit, int32_t *order, double *scores, double *cur) {
  int64_t k = c->k, p = L.period, npick = 0;
  for (int64_t r = 0; r < p; r++) cur[r] = (double)L.loads[r];
  uint8_t *taken = calloc((size_t)k + 1, 1);
  while (npick < k) {
    if (has_limit && f_le_i(vmax(cur, p), limit)) break;
    int64_t best = -1;
    double ba = 0;
    for (int64_t i = 0; i < k; i++) {
      if (taken[i]) continue;
      double area = orc_gap_area(L, cur, c->out_t[i], c->in_t[i]);
      int better = 0;
      if (best < 0) better = 1;
      else if (area > ba || (area == ba && c->size[i] > c->size[best])) better = 1;
      else if (area == ba && c->size[i] == c->size[best] &&
               name_cmp(nm, c->name_base[i], c->name_ralloc[i], c->name_base[best], c->name_ralloc[best]) < 0)
        better = 1;
      if (better) { best = i; ba = area; }
    }
    scores[best] = ba;
    absence(p, c, best, cur);
    taken[best] = 1;
    order[npick++] = (int32_t)best;
  }
  free(taken);
  return npick;
}

void orc_scores(orc_load L, const orc_cands *c, orc_names names, double *doa, double *aoa,
                double *wdoa, double *swdoa, int32_t *order) {
  int64_t k = c->k;
  double *cur = malloc((size_t)(L.period + 1) * 8);
  for (int64_t r = 0; r < L.period; r++) cur[r] = (double)L.loads[r];
  for (int64_t i = 0; i < k; i++) {
    /* score_doa / score_aoa, autoswap.py:132-142 */
    double gap = c->in_t[i] - c->out_t[i];
    doa[i] = gap - (c->dout[i] + c->din[i]);
    aoa[i] = doa[i] >= 0 ? (double)c->size[i] * doa[i] : doa[i] / (double)c->size[i];
    wdoa[i] = orc_gap_area(L, cur, c->out_t[i], c->in_t[i]);
  }
  swdoa_greedy(L, c, names, 0, 0, order, swdoa, cur);
  free(cur);
}

/* CPython 3.12 builtin sum() over floats: Neumaier compensated loop
 * (Python/bltinmodule.c, builtin_sum_impl); start value int 0 is absorbed
 * by the first float exactly. */
static double py_fsum(const double *x, int64_t n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0; /* int 0 + first float */
  for (int64_t i = 1; i < n; i++) {
    double t = f + x[i];
    if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
    else c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* the compiler must not fold pow(x, 2.0) into x*x: CPython calls libm pow,
 * which is not always correctly rounded */
static double (*volatile libm_pow)(double, double) = pow;

/* standardize, autoswap.py:228-238 (x ** 2 and var ** 0.5 are libm pow) */
void orc_standardize(const double *x, int64_t n, double *out) {
  if (n == 0) return;
  double mean = py_fsum(x, n) / (double)n;
  double *sq = malloc((size_t)n * 8);
  for (int64_t i = 0; i < n; i++) {
    /* float_pow (Objects/floatobject.c): 0**2 -> 0.0, negative base ->
     * pow(|x|, 2) (even exponent), 1**2 -> 1.0, else libm pow */
    double dv = x[i] - mean;
    if (dv == 0.0) sq[i] = 0.0;
    else if (isnan(dv)) sq[i] = dv;
    else {
      double a = fabs(dv);
      sq[i] = a == 1.0 ? 1.0 : libm_pow(a, 2.0);
    }
  }
  double var = py_fsum(sq, n) / (double)n;
  free(sq);
  if (var <= 0) { for (int64_t i = 0; i < n; i++) out[i] = 0.0; return; }
  double sd = var == 1.0 ? 1.0 : libm_pow(var, 0.5);
  for (int64_t i = 0; i < n; i++) out[i] = (x[i] - mean) / sd;
}

typedef struct sctx { const double *rank; const orc_cands *c; orc_names nm; } sctx;
static sctx g_s;
static int cmp_static(const void *a, const void *b) {
  int32_t i = *(const int32_t *)a, j = *(const int32_t *)b;
  double ri = -g_s.rank[i], rj = -g_s.rank[j];
  if (ri != rj) return ri < rj ? -1 : 1;
  int64_t si = -g_s.c->size[i], sj = -g_s.c->size[j];
  if (si != sj) return si < sj ? -1 : 1;
  int r = name_cmp(g_s.nm, g_s.c->name_base[i], g_s.c->name_ralloc[i], g_s.c->name_base[j],
                   g_s.c->name_ralloc[j]);
  if (r) return r;
  return (i > j) - (i < j); /* Python sort is stable */
}

/* select_by_score, autoswap.py:285-317 */
int orc_select(orc_load L, const orc_cands *c, orc_names names, int32_t score,
               const double *weights, int64_t limit, int32_t *sel, int64_t *nsel, mp_err *err) {
  int64_t k = c->k, p = L.period;
  if (score < 0 || score > 4) { set_err(err, MP_E_VALUE, 0, score, 0); return MP_E_VALUE; }
  double *cur = malloc((size_t)(p + 1) * 8);
  int64_t n = 0;
  int rc = MP_OK;
  if (score == 0) {
    double *sc = malloc((size_t)(k + 1) * 8);
    n = swdoa_greedy(L, c, names, 1, limit, sel, sc, cur);
    free(sc);
  } else {
    double *doa = malloc((size_t)(k + 1) * 8), *aoa = malloc((size_t)(k + 1) * 8);
    double *wdoa = malloc((size_t)(k + 1) * 8), *sw = malloc((size_t)(k + 1) * 8);
    double *rank = malloc((size_t)(k + 1) * 8);
    int32_t *ord = malloc((size_t)(k + 1) * 4);
    orc_scores(L, c, names, doa, aoa, wdoa, sw, ord);
    if (score == 1) memcpy(rank, doa, (size_t)k * 8);
    else if (score == 2) memcpy(rank, aoa, (size_t)k * 8);
    else if (score == 3) memcpy(rank, wdoa, (size_t)k * 8);
    else {
      /* combined_scores, autoswap.py:269-282: SCORE_NAMES order aoa, doa, wdoa, swdoa */
      const double *src[4] = {aoa, doa, wdoa, sw};
      double *z = malloc((size_t)(k + 1) * 8);
      for (int64_t i = 0; i < k; i++) rank[i] = 0.0;
      for (int s = 0; s < 4; s++) {
        orc_standardize(src[s], k, z);
        for (int64_t i = 0; i < k; i++) rank[i] += weights[s] * z[i];
      }
      free(z);
    }
    for (int64_t i = 0; i < k; i++) ord[i] = (int32_t)i;
    g_s = (sctx){rank, c, names};
    qsort(ord, (size_t)k, 4, cmp_static);
    for (int64_t r = 0; r < p; r++) cur[r] = (double)L.loads[r];
    for (int64_t q = 0; q < k; q++) {
      if (f_le_i(vmax(cur, p), limit)) break;
      absence(p, c, ord[q], cur);
      sel[n++] = ord[q];
    }
    free(doa); free(aoa); free(wdoa); free(sw); free(rank); free(ord);
  }
  double peak = p ? vmax(cur, p) : 0.0;
  if (!f_le_i(peak, limit)) {
    set_err(err, MP_E_LIMIT_UNREACHABLE, 0, limit, (int64_t)peak);
    rc = MP_E_LIMIT_UNREACHABLE;
  }
  free(cur);
  *nsel = n;
  return rc;
}

int64_t orc_load_min(orc_load L, const orc_cands *c) {
  int64_t p = L.period;
  if (!p) return 0;
  double *cur = malloc((size_t)p * 8);
  for (int64_t r = 0; r < p; r++) cur[r] = (double)L.loads[r];
  for (int64_t i = 0; i < c->k; i++) absence(p, c, i, cur);
  double m = vmax(cur, p);
  free(cur);
  return (int64_t)m;
}

/* ---------------------------------------------------------------------- */
/* _make_schedule — swapsim.py:62-108                                       */

typedef struct kctx { const double *key; const int32_t *who; const orc_cands *c; orc_names nm; } kctx;
static kctx g_k;
static int cmp_key_name(const void *a, const void *b) {
  int32_t i = *(const int32_t *)a, j = *(const int32_t *)b; /* positions in selection */
  double x = g_k.key[i], y = g_k.key[j];
  if (x != y) return x < y ? -1 : 1;
  int32_t ci = g_k.who[i], cj = g_k.who[j];
  int r = name_cmp(g_k.nm, g_k.c->name_base[ci], g_k.c->name_ralloc[ci], g_k.c->name_base[cj],
                   g_k.c->name_ralloc[cj]);
  if (r) return r;
  return (i > j) - (i < j);
}

static void make_schedule(const orc_cands *c, orc_names nm, const int32_t *sel, int64_t n,
                          const double *ready, const double *deadline, double *t_so, double *t_eo,
                          double *t_si, double *t_ei, int32_t *event_order) {
  int32_t *ord = malloc((size_t)(n + 1) * 4);
  for (int64_t q = 0; q < n; q++) ord[q] = (int32_t)q;
  g_k = (kctx){ready, sel, c, nm};
  qsort(ord, (size_t)n, 4, cmp_key_name);
  double busy = 0.0;
  for (int64_t q = 0; q < n; q++) {
    int32_t s = ord[q];
    double start = pmax(ready[s], busy);
    t_so[s] = start;
    busy = start + c->dout[sel[s]];
    t_eo[s] = busy;
  }
  for (int64_t q = 0; q < n; q++) ord[q] = (int32_t)q;
  g_k = (kctx){deadline, sel, c, nm};
  qsort(ord, (size_t)n, 4, cmp_key_name);
  double *desired = malloc((size_t)(n + 1) * 8);
  double cap = INF;
  for (int64_t q = n - 1; q >= 0; q--) {
    int32_t s = ord[q];
    double end = pmin(deadline[s], cap);
    desired[q] = end - c->din[sel[s]];
    cap = desired[q];
  }
  double prev_end = 0.0;
  for (int64_t q = 0; q < n; q++) {
    int32_t s = ord[q];
    double start = pmax(pmax(desired[q], t_eo[s]), prev_end);
    t_si[s] = start;
    prev_end = start + c->din[sel[s]];
    t_ei[s] = prev_end;
  }
  for (int64_t q = 0; q < n; q++) event_order[q] = (int32_t)q;
  g_k = (kctx){t_so, sel, c, nm};
  qsort(event_order, (size_t)n, 4, cmp_key_name);
  free(ord); free(desired);
}

void orc_schedule(const mp_profile_dims *d, const double *op_times, const orc_cands *c,
                  orc_names names, const int32_t *sel, int64_t nsel, double *t_so,
                  double *t_eo, double *t_si, double *t_ei, int32_t *event_order) {
  (void)d; (void)op_times;
  double *ready = malloc((size_t)(nsel + 1) * 8), *dl = malloc((size_t)(nsel + 1) * 8);
  for (int64_t q = 0; q < nsel; q++) { ready[q] = c->out_ready[sel[q]]; dl[q] = c->in_t[sel[q]]; }
  make_schedule(c, names, sel, nsel, ready, dl, t_so, t_eo, t_si, t_ei, event_order);
  free(ready); free(dl);
}

/* ---------------------------------------------------------------------- */
/* simulate — swapsim.py:147-395                                            */

typedef struct curve_t { double *t; int64_t *v; int64_t n; int64_t peak; double peak_t; int64_t load; } curve_t;

static void curve_point(curve_t *cv, double t) {
  if (cv->t[cv->n - 1] == t) cv->v[cv->n - 1] = cv->load;
  else { cv->t[cv->n] = t; cv->v[cv->n] = cv->load; cv->n++; }
  if (cv->load > cv->peak) { cv->peak = cv->load; cv->peak_t = t; }
}

/* _op_deltas, swapsim.py:147-163 */
static int64_t op_deltas(const mp_profile_dims *d, const mp_profile_out *P, int64_t *delta) {
  int64_t p = d->period, live0 = 0;
  for (int64_t r = 0; r < p; r++) delta[r] = 0;
  for (int64_t v = 0; v < d->nvars; v++)
    for (int s = 0; s < P->nseg[v]; s++) {
      int64_t lo = P->seg[4 * v + 2 * s], hi = P->seg[4 * v + 2 * s + 1];
      if (lo == 0) live0 += P->size[v];
      else delta[lo] += P->size[v];
      if (hi < p) delta[hi] -= P->size[v];
    }
  return live0;
}

typedef struct tde { double t; int64_t d; } tde;
static int cmp_tde(const void *a, const void *b) {
  const tde *x = a, *y = b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  return (x->d > y->d) - (x->d < y->d);
}

typedef struct replay_t {
  int64_t p, n, k_in, k_out, ncomp;
  int64_t *comp_sz; double *comp_t; int32_t *comp_who;
  double in_busy, head_floor, out_busy, delay;
  int64_t *in_order; double *plan_in, *in_done; uint8_t *in_has;
  int32_t *out_trigger, *in_wait; /* per op: selection position or -1 */
  curve_t cv;
  double *actual;
  int64_t *dl_idx; double *dl_us; int64_t ndl;
  int has_limit; int64_t limit;
} replay_t;

typedef struct ictx { const double *plan, *dl; const int32_t *sel; const orc_cands *c; orc_names nm; } ictx;
static ictx g_i;
static int cmp_inorder(const void *a, const void *b) {
  int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
  if (g_i.plan[i] != g_i.plan[j]) return g_i.plan[i] < g_i.plan[j] ? -1 : 1;
  if (g_i.dl[i] != g_i.dl[j]) return g_i.dl[i] < g_i.dl[j] ? -1 : 1;
  int32_t ci = g_i.sel[i], cj = g_i.sel[j];
  int r = name_cmp(g_i.nm, g_i.c->name_base[ci], g_i.c->name_ralloc[ci], g_i.c->name_base[cj],
                   g_i.c->name_ralloc[cj]);
  if (r) return r;
  return (i > j) - (i < j);
}

/* returns 1 = stepped, 0 = beyond horizon, -1 = IndexError (swapsim.py:266-267) */
static int rp_step(replay_t *R, const orc_cands *c, const int32_t *sel, double horizon) {
  double t_out = R->k_out < R->ncomp ? R->comp_t[R->k_out] : INF;
  double t_in = INF;
  int64_t hv = -1;
  if (R->k_in < R->n) {
    hv = R->in_order[R->k_in];
    double start = pmax(pmax(R->plan_in[hv], R->in_busy), R->head_floor);
    if (R->has_limit && R->cv.load + c->size[sel[hv]] > R->limit) start = INF;
    t_in = start;
  }
  double t = pmin(t_out, t_in);
  if (t > horizon) return 0;
  if (t_out <= t_in) {
    if (R->k_out >= R->ncomp) return -1;
    int64_t sz = R->comp_sz[R->k_out++];
    R->cv.load -= sz;
    R->head_floor = pmax(R->head_floor, t_out);
    curve_point(&R->cv, t_out);
  } else {
    R->cv.load += c->size[sel[hv]];
    curve_point(&R->cv, t_in);
    double end = t_in + c->din[sel[hv]];
    R->in_busy = end;
    R->in_done[hv] = end;
    R->in_has[hv] = 1;
    R->k_in++;
  }
  return 1;
}

/* one _Replay(...).run(); returns status */
static int replay_run(replay_t *R, const mp_profile_dims *d, const mp_profile_out *P, int64_t window0,
                      const int64_t *delta, int64_t live0, const orc_cands *c, orc_names nm,
                      const int32_t *sel, const double *t_si, const double *t_ei,
                      const int32_t *event_order, double d_actual, mp_err *err) {
  int64_t p = d->period, n = R->n;
  const double *tau = P->op_times;
  /* __init__, swapsim.py:208-246 */
  R->cv.load = live0;
  for (int64_t q = 0; q < n; q++) {
    int64_t s = event_order[q];
    int32_t ci = sel[s];
    if (c->spans[ci]) {
      R->cv.load -= c->size[ci];
      R->plan_in[s] = pmax(t_si[s] - d_actual, 0.0);
    } else {
      R->plan_in[s] = t_si[s];
    }
  }
  for (int64_t q = 0; q < n; q++) R->in_order[q] = event_order[q];
  g_i = (ictx){R->plan_in, t_ei, sel, c, nm};
  qsort(R->in_order, (size_t)n, 8, cmp_inorder);
  for (int64_t r = 0; r < p; r++) { R->out_trigger[r] = -1; R->in_wait[r] = -1; }
  for (int64_t s = 0; s < n; s++) { /* dict comprehension: later selection entries win */
    R->out_trigger[c->out_index[sel[s]]] = (int32_t)s;
    R->in_wait[c->in_index[sel[s]]] = (int32_t)s;
  }
  R->k_in = 0; R->in_busy = 0.0; R->head_floor = 0.0; R->ncomp = 0; R->k_out = 0;
  R->out_busy = 0.0; R->delay = 0.0; R->ndl = 0;
  for (int64_t s = 0; s < n; s++) R->in_has[s] = 0;
  R->cv.n = 1; R->cv.t[0] = 0.0; R->cv.v[0] = R->cv.load; R->cv.peak = R->cv.load; R->cv.peak_t = 0.0;
  /* run, swapsim.py:293-346 */
  for (int64_t r = 0; r < p; r++) {
    double t0 = tau[r] + R->delay, t = t0;
    int st;
    while ((st = rp_step(R, c, sel, t)) == 1) {}
    if (st < 0) return MP_E_SIM_INDEXERROR;
    int32_t w = R->in_wait[r];
    if (w >= 0) {
      while (!R->in_has[w]) {
        st = rp_step(R, c, sel, INF);
        if (st < 0) return MP_E_SIM_INDEXERROR;
        if (st == 0) {
          set_err(err, MP_E_SWAP_DEADLOCK, window0 + r, 1, sel[w]);
          return MP_E_SWAP_DEADLOCK;
        }
      }
      if (R->in_done[w] > t + EPS_US) {
        t = R->in_done[w];
        while ((st = rp_step(R, c, sel, t)) == 1) {}
        if (st < 0) return MP_E_SIM_INDEXERROR;
      }
    }
    int64_t dd = delta[r];
    if (dd > 0 && R->has_limit) {
      while (R->cv.load + dd > R->limit) {
        if (R->k_out >= R->ncomp) {
          set_err(err, MP_E_SWAP_DEADLOCK, window0 + r, 0, 0);
          return MP_E_SWAP_DEADLOCK;
        }
        double t_free = R->comp_t[R->k_out];
        int64_t sz = R->comp_sz[R->k_out++];
        R->cv.load -= sz;
        R->head_floor = pmax(R->head_floor, t_free);
        curve_point(&R->cv, t_free);
        t = pmax(t, t_free);
      }
    }
    if (t > t0 + EPS_US) {
      R->dl_idx[R->ndl] = window0 + r; R->dl_us[R->ndl] = t - t0; R->ndl++;
      R->delay += t - t0;
    } else {
      t = t0;
    }
    R->actual[r] = t;
    if (dd != 0) {
      R->cv.load += dd;
      curve_point(&R->cv, t);
      if (dd < 0) {
        R->head_floor = pmax(R->head_floor, t);
        while ((st = rp_step(R, c, sel, t)) == 1) {}
        if (st < 0) return MP_E_SIM_INDEXERROR;
      }
    }
    int32_t trig = R->out_trigger[r];
    if (trig >= 0) {
      double op_end = r + 1 < p ? tau[r + 1] : d->duration_us;
      double ready = t + (op_end - tau[r]);
      double start = pmax(ready, R->out_busy);
      R->out_busy = start + c->dout[sel[trig]];
      R->comp_t[R->ncomp] = R->out_busy; R->comp_sz[R->ncomp] = c->size[sel[trig]];
      R->comp_who[R->ncomp] = trig; R->ncomp++;
    }
  }
  return MP_OK;
}

int orc_simulate(const mp_profile_dims *d, const mp_profile_out *P, int64_t window0,
                 const orc_cands *c, orc_names names, const int32_t *sel, int64_t nsel,
                 int64_t limit, int32_t has_limit, int32_t max_rounds, orc_sim_out *o,
                 mp_err *err) {
  int64_t p = d->period, n = nsel;
  double dnat = d->duration_us;
  int64_t *delta = malloc((size_t)(p + 1) * 8);
  int64_t live0 = op_deltas(d, P, delta);
  /* initial schedule (build_schedule) — caller's o->t_* hold it on entry */
  double *si = malloc((size_t)(n + 1) * 8), *ei = malloc((size_t)(n + 1) * 8);
  double *so = malloc((size_t)(n + 1) * 8), *eo = malloc((size_t)(n + 1) * 8);
  int32_t *eord = malloc((size_t)(n + 1) * 4);
  memcpy(so, o->t_so, (size_t)n * 8); memcpy(eo, o->t_eo, (size_t)n * 8);
  memcpy(si, o->t_si, (size_t)n * 8); memcpy(ei, o->t_ei, (size_t)n * 8);
  memcpy(eord, o->event_order, (size_t)n * 4);
  /* LOAD' overlay, swapsim.py:184-202 */
  {
    tde *ev = malloc((size_t)(p + 2 * n + 1) * sizeof(tde));
    int64_t ne = 0, l0 = live0;
    for (int64_t r = 0; r < p; r++) if (delta[r] != 0) ev[ne++] = (tde){P->op_times[r], delta[r]};
    for (int64_t q = 0; q < n; q++) {
      int64_t s = eord[q];
      int32_t ci = sel[s];
      ev[ne++] = (tde){eo[s], -c->size[ci]};
      if (c->spans[ci]) { l0 -= c->size[ci]; ev[ne++] = (tde){pmax(si[s] - dnat, 0.0), c->size[ci]}; }
      else ev[ne++] = (tde){si[s], c->size[ci]};
    }
    /* _accumulate: stable sort on (t, delta) — equal keys are equal values */
    qsort(ev, (size_t)ne, sizeof(tde), cmp_tde);
    curve_t cv = {o->lp_t, o->lp_v, 1, l0, 0.0, l0};
    cv.t[0] = 0.0; cv.v[0] = l0;
    for (int64_t q = 0; q < ne; q++) { cv.load += ev[q].d; curve_point(&cv, ev[q].t); }
    o->n_lp = cv.n; o->lp_peak = cv.peak; o->lp_peak_t = cv.peak_t;
    free(ev);
  }
  replay_t R;
  memset(&R, 0, sizeof R);
  R.p = p; R.n = n; R.has_limit = has_limit; R.limit = limit;
  R.comp_sz = malloc((size_t)(n + 1) * 8); R.comp_t = malloc((size_t)(n + 1) * 8);
  R.comp_who = malloc((size_t)(n + 1) * 4);
  R.in_order = malloc((size_t)(n + 1) * 8); R.plan_in = malloc((size_t)(n + 1) * 8);
  R.in_done = malloc((size_t)(n + 1) * 8); R.in_has = malloc((size_t)(n + 1));
  R.out_trigger = malloc((size_t)(p + 1) * 4); R.in_wait = malloc((size_t)(p + 1) * 4);
  R.cv.t = o->ldp_t; R.cv.v = o->ldp_v;
  R.actual = malloc((size_t)(p + 1) * 8);
  R.dl_idx = o->delayed_index; R.dl_us = o->delayed_us;
  double prev_delay = 0.0;
  int have_prev = 0, rc = MP_OK;
  int64_t rounds = 0;
  double *ready = malloc((size_t)(n + 1) * 8), *dl = malloc((size_t)(n + 1) * 8);
  for (int32_t it = 0; it < max_rounds; it++) {
    rc = replay_run(&R, d, P, window0, delta, live0, c, names, sel, si, ei, eord,
                    dnat + (have_prev ? prev_delay : 0.0), err);
    if (rc) break;
    rounds++;
    if (n == 0 || R.delay == 0.0) break;
    if (have_prev && fabs(R.delay - prev_delay) < 1e-6) break;
    prev_delay = R.delay; have_prev = 1;
    double d_act = dnat + R.delay;
    for (int64_t s = 0; s < n; s++) {
      int32_t ci = sel[s];
      int64_t oi = c->out_index[ci];
      double op_end = oi + 1 < p ? P->op_times[oi + 1] : dnat;
      double dur = op_end - P->op_times[oi];
      ready[s] = R.actual[oi] + dur;
      dl[s] = R.actual[c->in_index[ci]] + (c->spans[ci] ? d_act : 0.0);
    }
    make_schedule(c, names, sel, n, ready, dl, so, eo, si, ei, eord);
  }
  if (rc == MP_E_SIM_INDEXERROR) set_err(err, rc, 0, 0, 0);
  if (rc == MP_OK) {
    memcpy(o->t_so, so, (size_t)n * 8); memcpy(o->t_eo, eo, (size_t)n * 8);
    memcpy(o->t_si, si, (size_t)n * 8); memcpy(o->t_ei, ei, (size_t)n * 8);
    memcpy(o->event_order, eord, (size_t)n * 4);
    o->n_ldp = R.cv.n; o->ldp_peak = R.cv.peak; o->ldp_peak_t = R.cv.peak_t;
    o->n_delayed = R.ndl; o->delay = R.delay; o->rounds = rounds;
  }
  free(ready); free(dl); free(delta); free(si); free(ei); free(so); free(eo); free(eord);
  free(R.comp_sz); free(R.comp_t); free(R.comp_who); free(R.in_order); free(R.plan_in);
  free(R.in_done); free(R.in_has); free(R.out_trigger); free(R.in_wait); free(R.actual);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* one sweep unit — what the estimators run for a trace (estimators.py:20-130):
 * validate_trace, detect_iteration, extract_lifetimes, build_conflict_graph +
 * plan_pool, filter_candidates, compute_load_min, then per budget
 * SwapPlanner(limit_bytes=int(peak * frac), score="swdoa").fit: the limit
 * checks (validation.py:32-34, estimators.py:98-100), select_by_score
 * (autoswap.py:285-301 -> select_by_swdoa, rerun per budget as the reference
 * does), build_schedule and simulate.  Records mirror mp_sweep_trace /
 * mp_sweep_budget; offsets and cand_order are sized to the trace's events. */

int orc_sweep_unit(const mp_trace_in *t, const mp_sweep_params *prm, mp_sweep_trace *rec,
                   mp_sweep_budget *brec, int64_t *offsets, int32_t *cand_order) {
  mp_err err;
  memset(rec, 0, sizeof *rec);
  for (int b = 0; b < prm->nbudget; b++) memset(&brec[b], 0, sizeof brec[b]);
  int rc = MP_OK;
  if (prm->validate) rc = orc_validate(t, &err);
  if (rc == MP_OK) {
    int64_t p;
    rc = orc_detect(t, &p, &err);
    if (rc == MP_OK) rec->period = p;
  }
  orc_profile *P = NULL;
  if (rc == MP_OK) rc = orc_extract(t, t->n - rec->period, t->n, &P, &err);
  if (rc != MP_OK) {
    rec->status = rc;
    rec->err_code = rc == MP_E_INVARIANT ? (int32_t)err.aux0 : 0;
    rec->err_index = err.index;
    for (int b = 0; b < prm->nbudget; b++) brec[b].status = rc;
    return rc;
  }
  mp_profile_dims d = P->d;
  int64_t V = d.nvars, p = d.period;
  rec->nvars = V; rec->ncarry = d.ncarry; rec->naccess = d.naccess;
  rec->peak_bytes = d.peak_bytes; rec->peak_index = d.peak_index; rec->duration_us = d.duration_us;
  mp_profile_out po = {P->base, P->size, P->alloc, P->free_, P->nseg, P->seg, P->flags, P->acc_off,
                       P->acc_index, P->acc_kind, P->acc_next, P->op_times, P->loads, P->op_owner};
  orc_names names = {t->name_blob, t->name_off};
  /* build_conflict_graph + plan_pool */
  int64_t *seg_off = malloc((size_t)(V + 1) * 8);
  int32_t *lo = malloc((size_t)(2 * V + 1) * 4), *hi = malloc((size_t)(2 * V + 1) * 4);
  int64_t *alloc64 = malloc((size_t)(V + 1) * 8);
  int32_t *ralloc = malloc((size_t)(V + 1) * 4);
  int64_t ns = 0;
  for (int64_t i = 0; i < V; i++) {
    seg_off[i] = ns;
    for (int s = 0; s < P->nseg[i]; s++) { lo[ns] = P->seg[4 * i + 2 * s]; hi[ns] = P->seg[4 * i + 2 * s + 1]; ns++; }
    alloc64[i] = P->alloc[i];
    ralloc[i] = (P->flags[i] & MP_F_RENAMED) ? P->alloc[i] : -1;
  }
  seg_off[V] = ns;
  orc_graph *g;
  orc_conflict((int32_t)V, seg_off, lo, hi, &g);
  rec->edges = orc_graph_nnz(g) / 2;
  orc_plan(g, P->size, alloc64, P->base, ralloc, names, prm->policy, offsets, &rec->footprint_bytes);
  orc_graph_free(g);
  /* filter_candidates + compute_load_min + the unbudgeted greedy order */
  orc_cands C;
  C.var = malloc((size_t)(V + 1) * 4); C.size = malloc((size_t)(V + 1) * 8);
  C.out_index = malloc((size_t)(V + 1) * 4); C.out_t = malloc((size_t)(V + 1) * 8);
  C.out_ready = malloc((size_t)(V + 1) * 8); C.in_index = malloc((size_t)(V + 1) * 4);
  C.in_t = malloc((size_t)(V + 1) * 8); C.dout = malloc((size_t)(V + 1) * 8);
  C.din = malloc((size_t)(V + 1) * 8); C.spans = malloc((size_t)(V + 1));
  C.name_base = malloc((size_t)(V + 1) * 4); C.name_ralloc = malloc((size_t)(V + 1) * 4);
  int64_t k = orc_candidates(&d, &po, prm->threshold, prm->bw, prm->lat, &C);
  rec->ncand = k;
  orc_load L = {p, P->loads, P->op_times, d.duration_us};
  int64_t load_min = orc_load_min(L, &C);
  rec->load_min = load_min;
  double *sc[4];
  for (int i = 0; i < 4; i++) sc[i] = malloc((size_t)(k + 1) * 8);
  int32_t *order = malloc((size_t)(k + 1) * 4);
  orc_scores(L, &C, names, sc[0], sc[1], sc[2], sc[3], order);
  /* the greedy prefix the budgets select from: up to the smallest limit that
   * passes SwapPlanner.fit's precheck (the device stops there too) */
  {
    int64_t stop = INT64_MAX;
    int need = 0;
    for (int b = 0; b < prm->nbudget; b++) {
      int64_t limit = (int64_t)((double)d.peak_bytes * prm->budget_frac[b]);
      if (limit <= 0 || (limit < d.peak_bytes && limit < load_min)) continue;
      need = 1;
      if (limit < stop) stop = limit;
    }
    int64_t norder = 0;
    if (need) {
      double *cur = malloc((size_t)(p + 1) * 8);
      for (int64_t r = 0; r < p; r++) cur[r] = (double)P->loads[r];
      while (norder < k && !f_le_i(vmax(cur, p), stop)) absence(p, &C, order[norder++], cur);
      free(cur);
    }
    rec->norder = norder;
    for (int64_t q = 0; q < norder; q++) cand_order[q] = C.var[order[q]];
  }
  /* per budget: SwapPlanner.fit */
  int32_t *sel = malloc((size_t)(k + 1) * 4);
  int64_t cap = 1 + p + 2 * k + 2;
  orc_sim_out so;
  double *tt[4];
  for (int i = 0; i < 4; i++) tt[i] = malloc((size_t)(k + 1) * 8);
  int32_t *eo = malloc((size_t)(k + 1) * 4);
  double *lp_t = malloc((size_t)cap * 8), *ldp_t = malloc((size_t)cap * 8), *du = malloc((size_t)(p + 1) * 8);
  int64_t *lp_v = malloc((size_t)cap * 8), *ldp_v = malloc((size_t)cap * 8), *di = malloc((size_t)(p + 1) * 8);
  for (int b = 0; b < prm->nbudget; b++) {
    mp_sweep_budget *rb = &brec[b];
    int64_t limit = (int64_t)((double)d.peak_bytes * prm->budget_frac[b]);
    rb->limit_bytes = limit;
    if (limit <= 0) { rb->status = MP_E_VALUE; continue; }
    if (limit < d.peak_bytes && limit < load_min) {
      rb->status = MP_E_LIMIT_UNREACHABLE; rb->err_aux = load_min; continue;
    }
    int64_t nsel = 0;
    int rs = orc_select(L, &C, names, 0, NULL, limit, sel, &nsel, &err);
    if (rs != MP_OK) { rb->status = rs; rb->err_aux = err.aux1; continue; }
    orc_schedule(&d, P->op_times, &C, names, sel, nsel, tt[0], tt[1], tt[2], tt[3], eo);
    so = (orc_sim_out){tt[0], tt[1], tt[2], tt[3], eo, lp_t, lp_v, 0, 0, 0.0, ldp_t, ldp_v, 0, 0, 0.0,
                       di, du, 0, 0.0, 0};
    int sr = orc_simulate(&d, &po, t->n - p, &C, names, sel, nsel, limit, 1, prm->max_rounds, &so, &err);
    int64_t bytes = 0;
    for (int64_t q = 0; q < nsel; q++) bytes += C.size[sel[q]];
    rb->status = sr;
    rb->nsel = nsel;
    rb->selected_bytes = bytes;
    if (sr == MP_OK) {
      rb->rounds = (int32_t)so.rounds;
      rb->overhead_us = so.delay;
      rb->achieved_peak_bytes = so.ldp_peak;
      rb->planned_peak_bytes = so.lp_peak;
    } else if (sr == MP_E_SWAP_DEADLOCK) {
      rb->err_index = err.index;
      rb->err_aux = err.aux1;
    }
  }
  free(seg_off); free(lo); free(hi); free(alloc64); free(ralloc);
  free(C.var); free(C.size); free(C.out_index); free(C.out_t); free(C.out_ready); free(C.in_index);
  free(C.in_t); free(C.dout); free(C.din); free(C.spans); free(C.name_base); free(C.name_ralloc);
  for (int i = 0; i < 4; i++) { free(sc[i]); free(tt[i]); }
  free(order); free(sel); free(eo); free(lp_t); free(ldp_t); free(du); free(lp_v); free(ldp_v); free(di);
  orc_profile_free(P);
  return MP_OK;
}
