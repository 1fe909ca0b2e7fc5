// ingest_dev.cuh — per-item bodies of validate_trace and extract_lifetimes.
//
// Shared by the grid-wide kernels of ingest.cu (one large trace, one thread
// per variable or op across the whole GPU) and by the one-CTA-per-trace
// batched sweep (sweep.cu), so both paths run the same state machines.
// Pointers are trace-relative: `perm` holds event positions inside the
// trace, `gstart[v]..gstart[v+1]` is variable v's run of `perm`.
#pragma once

#include "common.cuh"

// window-instance flags
#define WF_OPEN_END 1
#define WF_MERGED 2
#define WF_COEXIST 4
// carry-in cases
#define CC_PERSIST 0
#define CC_MERGED 1
#define CC_COEXIST 2
#define CC_CONSERVATIVE 3

#define NO_VIOLATION (~0ull)

struct ExScratch {
  // per window op r
  int32_t *owner;   // >= 0: window instance (malloc position); < 0: carry -(v+1)
  int32_t *w_free;  // free position of a window instance
  int32_t *w_nacc;
  uint8_t *w_flags;
  int32_t *w_mcarry;  // carry var merged into this twin
  int32_t *is_malloc; // scanned -> window instance ordinal
  // per variable
  uint8_t *c_live;
  int64_t *c_abs;
  int64_t *c_size;
  int32_t *c_free;
  int32_t *c_nacc;
  uint8_t *c_case;
  int32_t *c_twin;
  int32_t *c_surv;    // scanned -> carry ordinal
  int32_t *nmalloc;
};

struct ProfOut {
  int32_t *base, *alloc, *free_, *nseg, *seg, *acc_index, *op_owner;
  int64_t *size, *acc_off, *loads;
  uint8_t *flags, *acc_kind, *acc_next;
  double *op_times;
};

// ---------------------------------------------------------------------------
// validate_trace, trace.py:55-84

// element checks of position pos (trace.py:63-79); 0 = none
// checks: VC_STRUCT = index + kind/size, VC_TIMES = timestamps.  The codes
// are numbered in the reference's check order, so the minimum of
// (pos << 4 | code) over separate passes is the first violation of one pass.
enum { VC_STRUCT = 1, VC_TIMES = 2, VC_ALL = 3 };
__device__ __forceinline__ int validate_elem_code(const uint8_t *kind, const int64_t *size, const int64_t *t_us,
                                                  const int64_t *index, int64_t pos, int checks = VC_ALL) {
  if ((checks & VC_STRUCT) && index && index[pos] != pos) return MP_V_INDEX;
  if (checks & VC_TIMES) {
    if (t_us[pos] < 0) return MP_V_NEG_T;
    if (pos > 0 && t_us[pos] < t_us[pos - 1]) return MP_V_T_DEC;
  }
  if (!(checks & VC_STRUCT)) return 0;
  if (kind[pos] == MP_MALLOC) return size[pos] <= 0 ? MP_V_MALLOC_SIZE : 0;
  return size[pos] != 0 ? MP_V_SIZE_NONZERO : 0;
}

// live-set checks over one variable's run (trace.py:74-84): the first
// violation as (position << 4 | code), or NO_VIOLATION
__device__ __forceinline__ unsigned long long validate_var_first(const uint8_t *kind, const uint32_t *perm,
                                                                 int64_t q0, int64_t q1) {
  bool live = false;
  for (int64_t q = q0; q < q1; q++) {
    uint32_t e = perm[q];
    uint8_t k = kind[e];
    int code = 0;
    if (k == MP_MALLOC) {
      if (live) code = MP_V_MALLOC_LIVE;
      live = true;
    } else {
      if (!live) code = k == MP_FREE ? MP_V_FREE_DEAD : MP_V_USE_DEAD;
      if (k == MP_FREE) live = false;
    }
    if (code) return ((unsigned long long)e << 4) | (unsigned)code;
  }
  return NO_VIOLATION;
}

// ---------------------------------------------------------------------------
// extract_lifetimes / build_profile, iteration.py:124-301

// _live_at + the window walk of variable v (iteration.py:124-187): the
// first in-window violation as (r << 4 | code), or NO_VIOLATION
__device__ __forceinline__ unsigned long long ex_var_item(const uint8_t *kind, const int64_t *size,
                                                          const uint32_t *perm, const int64_t *gstart, int64_t v,
                                                          int64_t start, int64_t end, const ExScratch &s) {
  int64_t q = gstart[v], qe = gstart[v + 1];
  // _live_at: last malloc/free before the window
  int64_t live = -1;
  for (; q < qe; q++) {
    int64_t e = perm[q];
    if (e >= start) break;
    uint8_t k = kind[e];
    if (k == MP_MALLOC) live = e;
    else if (k == MP_FREE) live = -1;
  }
  s.c_live[v] = live >= 0;
  s.c_abs[v] = live;
  s.c_size[v] = live >= 0 ? size[live] : 0;
  s.c_free[v] = -1;
  s.c_case[v] = CC_PERSIST;
  s.c_twin[v] = -1;
  bool carry_alive = live >= 0;
  int32_t open = -1, nacc_c = 0, nm = 0;
  unsigned long long first = NO_VIOLATION;
  for (; q < qe; q++) {
    int64_t e = perm[q];
    if (e >= end) break;
    int32_t r = (int32_t)(e - start);
    uint8_t k = kind[e];
    int code = 0;
    if (k == MP_MALLOC) {
      if (open >= 0) code = MP_V_W_MALLOC_LIVE;
      else {
        open = r;
        nm++;
        s.w_free[r] = -1;
        s.w_nacc[r] = 0;
        s.w_flags[r] = 0;
        s.owner[r] = r;
      }
    } else if (k == MP_FREE) {
      if (open >= 0) { s.w_free[open] = r; s.owner[r] = open; open = -1; }
      else if (carry_alive) { s.c_free[v] = r; carry_alive = false; s.owner[r] = -(int32_t)(v + 1); }
      else code = MP_V_W_FREE_DEAD;
    } else {
      if (open >= 0) { s.w_nacc[open]++; s.owner[r] = open; }
      else if (carry_alive) { nacc_c++; s.owner[r] = -(int32_t)(v + 1); }
      else code = MP_V_W_USE_DEAD;
    }
    if (code) {
      first = ((unsigned long long)r << 4) | (unsigned)code;
      break;
    }
  }
  if (open >= 0) s.w_flags[open] |= WF_OPEN_END;
  s.c_nacc[v] = nacc_c;
  s.nmalloc[v] = nm;
  return first;
}

// twin pairing of carry-in v, iteration.py:193-225
__device__ __forceinline__ void ex_twin_item(const uint8_t *kind, const int64_t *size, int64_t v, int64_t start,
                                             int64_t p, const ExScratch &s) {
  int32_t surv = 0;
  if (s.c_live[v]) {
    surv = 1;
    int32_t r_f = s.c_free[v];
    if (r_f >= 0) {
      int64_t abs_idx = s.c_abs[v];
      int64_t tw = abs_idx >= start - p ? abs_idx - (start - p) : -1;
      bool ok = tw >= 0 && tw < p && kind[start + tw] == MP_MALLOC &&
                (s.w_flags[tw] & WF_OPEN_END) && size[start + tw] == s.c_size[v];
      if (ok && r_f <= tw) {
        s.c_case[v] = CC_MERGED;
        s.c_twin[v] = (int32_t)tw;
        s.w_flags[tw] |= WF_MERGED;
        s.w_mcarry[tw] = (int32_t)v;
        surv = 0;
      } else if (ok) {
        s.c_case[v] = CC_COEXIST;
        s.w_flags[tw] |= WF_COEXIST;
      } else {
        s.c_case[v] = CC_CONSERVATIVE;
      }
    }
  }
  s.c_surv[v] = surv;
}

// final record of a surviving carry-in (carry ordinal carry_ord[v])
__device__ __forceinline__ void ex_fill_carry_item(int64_t v, int64_t p, const ExScratch &s, const int32_t *carry_ord,
                                                   const ProfOut &o, int64_t *acc_cnt) {
  if (!s.c_live[v] || s.c_case[v] == CC_MERGED) return;
  int64_t i = carry_ord[v];
  o.base[i] = (int32_t)v;
  o.size[i] = s.c_size[v];
  o.alloc[i] = -1;
  o.free_[i] = s.c_free[v];
  o.nseg[i] = 1;
  uint8_t fl = 0;
  int32_t hi = (int32_t)p;
  switch (s.c_case[v]) {
    case CC_PERSIST: fl = MP_F_PERSISTENT; break;
    case CC_COEXIST: hi = s.c_free[v]; break;
    default: fl = MP_F_WRAPS; break;
  }
  o.seg[4 * i] = 0; o.seg[4 * i + 1] = hi; o.seg[4 * i + 2] = 0; o.seg[4 * i + 3] = 0;
  o.flags[i] = fl;
  acc_cnt[i] = s.c_nacc[v];
}

// final record of the window instance malloc'd at op r (alloc order)
__device__ __forceinline__ void ex_fill_window_item(const int32_t *var, const int64_t *size, int64_t start, int64_t r,
                                                    int64_t p, int64_t ncarry, const ExScratch &s,
                                                    const int32_t *win_ord, const int32_t *carry_survive,
                                                    const ProfOut &o, int64_t *acc_cnt) {
  if (!s.is_malloc[r]) return;
  int64_t i = ncarry + win_ord[r];
  int32_t b = var[start + r];
  o.base[i] = b;
  o.size[i] = size[start + r];
  o.alloc[i] = (int32_t)r;
  uint8_t wf = s.w_flags[r];
  uint8_t fl = 0;
  int32_t nseg = 1, l0 = (int32_t)r, h0 = s.w_free[r], l1 = 0, h1 = 0, fr = s.w_free[r];
  int64_t nacc = s.w_nacc[r];
  if (wf & WF_MERGED) {
    int32_t cv = s.w_mcarry[r];
    fr = s.c_free[cv];
    fl = MP_F_WRAPS;
    nseg = 2; h0 = (int32_t)p; l1 = 0; h1 = fr;
    nacc += s.c_nacc[cv];
  } else if (wf & WF_COEXIST) {
    fl = MP_F_WRAPS; fr = -1; h0 = (int32_t)p;
  } else if (wf & WF_OPEN_END) {
    fl = MP_F_PERSISTENT | MP_F_WRAPS; fr = -1; l0 = 0; h0 = (int32_t)p;
  }
  // renames, iteration.py:236-241: more than one instance of this base
  if (carry_survive[b] + s.nmalloc[b] > 1) fl |= MP_F_RENAMED;
  o.free_[i] = fr;
  o.nseg[i] = nseg;
  o.seg[4 * i] = l0; o.seg[4 * i + 1] = h0; o.seg[4 * i + 2] = l1; o.seg[4 * i + 3] = h1;
  o.flags[i] = fl;
  acc_cnt[i] = nacc;
}

// second walk of variable v: accesses into the final CSR, owners into
// op_owner (op_owner may be null)
__device__ __forceinline__ void ex_access_item(const uint8_t *kind, const uint32_t *perm, const int64_t *gstart,
                                               int64_t v, int64_t start, int64_t end, int64_t ncarry,
                                               const ExScratch &s, const int32_t *carry_ord, const int32_t *win_ord,
                                               const ProfOut &o) {
  int64_t q = gstart[v], qe = gstart[v + 1];
  while (q < qe && perm[q] < start) q++;
  // destination of carry-in accesses
  int64_t cdst = -1, cfinal = -1;
  uint8_t cnext = 0;
  if (s.c_live[v]) {
    if (s.c_case[v] == CC_MERGED) {
      int32_t tw = s.c_twin[v];
      cfinal = ncarry + win_ord[tw];
      cdst = o.acc_off[cfinal] + s.w_nacc[tw];
      cnext = 1;
    } else {
      cfinal = carry_ord[v];
      cdst = o.acc_off[cfinal];
    }
  }
  int64_t wdst = 0, wfinal = -1;
  for (; q < qe; q++) {
    int64_t e = perm[q];
    if (e >= end) break;
    int32_t r = (int32_t)(e - start);
    int32_t ow = s.owner[r];
    uint8_t k = kind[e];
    int64_t fin;
    if (ow >= 0) {
      if (k == MP_MALLOC) { wfinal = ncarry + win_ord[r]; wdst = o.acc_off[wfinal]; }
      fin = wfinal;
      if (k == MP_READ || k == MP_WRITE) {
        o.acc_index[wdst] = r;
        if (o.acc_kind) o.acc_kind[wdst] = k;
        o.acc_next[wdst] = 0;
        wdst++;
      }
    } else {
      fin = cfinal;
      if (k == MP_READ || k == MP_WRITE) {
        o.acc_index[cdst] = r;
        if (o.acc_kind) o.acc_kind[cdst] = k;
        o.acc_next[cdst] = cnext;
        cdst++;
      }
    }
    if (o.op_owner) o.op_owner[r] = (int32_t)fin;
  }
}

// period duration, iteration.py:283-291 (op_times[r] = t[start+r] - t[start])
__device__ __forceinline__ double ex_duration(const int64_t *t_us, int64_t start, int64_t end) {
  int64_t p = end - start;
  int64_t t0 = t_us[start];
  double last = (double)(t_us[end - 1] - t0);
  double d;
  if (start >= 1) {
    d = (double)(t_us[end - 1] - t_us[start - 1]);
  } else {
    double tail = p > 1 ? last - (double)(t_us[end - 2] - t0) : 1.0;
    d = last + pymax(tail, 1.0);
  }
  if (d <= last) d = last + 1.0;
  return d;
}
