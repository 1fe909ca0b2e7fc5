// swap_dev.cuh — device bodies of the AutoSwap path (autoswap.py,
// swapsim.py), shared by the per-trace kernels of swap.cu and the
// one-CTA-per-trace batched sweep (sweep.cu).
//
// Every float operation and comparison follows the reference's order and
// Python's max/min argument semantics (built with -fmad=false), so results
// are bit-identical to CPython's binary64 left folds.
#pragma once

#include <climits>

#include "common.cuh"

#define INF_D (__longlong_as_double(0x7ff0000000000000ll))
#define EPS_US 1e-6

struct CandView {
  int64_t k;
  const int64_t *size;
  const int32_t *out_index, *in_index, *name_rank;
  const double *out_t, *out_ready, *in_t, *dout, *din;
  const uint8_t *spans;
};

struct LoadView {
  int64_t p;
  const int64_t *loads;
  const double *op_times;
  double duration;
};

struct CandOut {
  int32_t *var, *out_index, *in_index;
  int64_t *size;
  double *out_t, *out_ready, *in_t, *dout, *din;
  uint8_t *spans;
};

struct ProfView {
  int64_t p, V, window0;
  double duration;
  const double *tau;
  const int32_t *nseg, *seg;
  const int64_t *size;
};

// ---------------------------------------------------------------------------
// filter_candidates, autoswap.py:53-116: variable v's candidate record in
// slot `slot` of o (returns false when v is not a candidate).  The access
// pairs walk the sorted multiset of coordinates (successor walk when the
// stored order is not already sorted).
__device__ __forceinline__ bool cand_item(int64_t v, int64_t slot, int64_t p, int64_t peak, const int64_t *size,
                                          const uint8_t *flags, const int64_t *acc_off, const int32_t *acc_index,
                                          const uint8_t *acc_next, const double *op_times, double duration,
                                          int64_t threshold, double bw, double lat, const CandOut &o) {
  if (size[v] < threshold) return false;
  int64_t a0 = acc_off[v], m = acc_off[v + 1] - a0;
  auto coord = [&](int64_t q) -> int64_t { return acc_index[a0 + q] + (acc_next[a0 + q] ? p : 0); };
  bool sorted = true;
  for (int64_t q = 1; q < m && sorted; q++) sorted = coord(q - 1) <= coord(q);
  // iterate consecutive pairs of the sorted multiset
  int64_t prev = 0, first = 0;
  bool found = false;
  int64_t c1 = 0, c2 = 0;
  int64_t last_v = -1, last_q = -1;  // successor-walk cursor
  for (int64_t q = 0; q < m && !found; q++) {
    int64_t cur;
    if (sorted) {
      cur = coord(q);
    } else {
      // smallest (value, index) strictly after (last_v, last_q)
      int64_t bv = LLONG_MAX, bq = -1;
      for (int64_t t = 0; t < m; t++) {
        int64_t cv = coord(t);
        bool after = cv > last_v || (cv == last_v && t > last_q);
        if (after && (cv < bv || (cv == bv && t < bq))) { bv = cv; bq = t; }
      }
      cur = bv;
      last_v = bv;
      last_q = bq;
    }
    if (q == 0) first = cur;
    if (q > 0 && prev < cur) {
      int64_t a = prev, b = cur;
      if (a >= p) { a -= p; b -= p; }
      if ((a < peak && peak < b) || (a < peak + p && peak + p < b)) { c1 = a; c2 = b; found = true; }
    }
    prev = cur;
  }
  if (!found && (flags[v] & MP_F_PERSISTENT) && m > 0) {
    int64_t a = prev, b = first + p;  // wrap pair (last, first + period)
    if (a >= p) { a -= p; b -= p; }
    if ((a < peak && peak < b) || (a < peak + p && peak + p < b)) { c1 = a; c2 = b; found = true; }
  }
  if (!found) return false;
  bool spans = c2 >= p;
  o.var[slot] = (int32_t)v;
  o.size[slot] = size[v];
  o.out_index[slot] = (int32_t)c1;
  o.out_t[slot] = op_times[c1];
  o.out_ready[slot] = c1 + 1 < p ? op_times[c1 + 1] : duration;
  o.in_index[slot] = (int32_t)(c2 % p);
  o.in_t[slot] = op_times[c2 % p] + (spans ? duration : 0.0);
  double delta = (double)size[v] / bw * 1e6 + lat;  // TransferModel.delta_us, autoswap.py:30-31
  o.dout[slot] = delta;
  o.din[slot] = delta;
  o.spans[slot] = spans;
  return true;
}

// ---------------------------------------------------------------------------
// gap areas

// _step_area, autoswap.py:145-161 (left fold in slot order)
__device__ __forceinline__ double step_area(const LoadView &L, const double *cur, const int64_t *iloads, double a,
                                            double b) {
  if (b <= a) return 0.0;
  int64_t p = L.p;
  int64_t lo = 0, hi = p;  // bisect_right(op_times, a)
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a < L.op_times[mid]) hi = mid; else lo = mid + 1;
  }
  int64_t r0 = lo - 1 < 0 ? 0 : lo - 1;
  // the reference stops at the first slot starting at or after b
  // (op_times is non-decreasing): bound the loop up front so the loads of
  // later slots are not held behind the exit test of earlier ones
  int64_t r1 = r0, hi2 = p;
  while (r1 < hi2) {
    int64_t mid = (r1 + hi2) >> 1;
    if (L.op_times[mid] < b) r1 = mid + 1; else hi2 = mid;
  }
  double total = 0.0;
  double s = r0 < r1 ? L.op_times[r0] : 0.0;
#pragma unroll 4
  for (int64_t r = r0; r < r1; r++) {
    const double e = r + 1 < p ? L.op_times[r + 1] : L.duration;
    const double ov = pymin(b, e) - pymax(a, s);
    const double x = cur ? cur[r] : (double)iloads[r];
    if (ov > 0) total += x * ov;
    s = e;
  }
  return total;
}

// gap_area, autoswap.py:164-174
__device__ __forceinline__ double gap_area(const LoadView &L, const double *cur, double a, double b) {
  double d = L.duration;
  if (b <= d) return step_area(L, cur, L.loads, a, b);
  return step_area(L, cur, L.loads, a, d) + step_area(L, cur, L.loads, 0.0, b - d);
}

// ---------------------------------------------------------------------------
// absence bookkeeping: slots strictly between the two accesses, modulo p
// (autoswap.py:119-129); a slot can be hit more than once only if the gap
// exceeds a period, and then the reference subtracts once per hit

__device__ __forceinline__ int absence_hits(int64_t r, int64_t lo, int64_t hi, int64_t p) {
  // number of x in (lo, hi) with x % p == r, for lo >= 0
  int h = 0;
  for (int64_t x = r; x < hi; x += p)
    if (x > lo) h++;
  return h;
}

// group-wide Python max (red: >= 33 doubles of shared memory)
template <class G>
__device__ __forceinline__ double block_max(const G &g, double v, double *red) {
  const int lane = g.idx() & 31, w = g.idx() >> 5, nw = (g.size() + 31) >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = pymax(v, __shfl_xor_sync(FULL_MASK, v, o));
  if (lane == 0) red[w] = v;
  g.sync();
  if (w == 0) {
    double x = lane < nw ? red[lane] : -INF_D;
#pragma unroll
    for (int o = 16; o; o >>= 1) x = pymax(x, __shfl_xor_sync(FULL_MASK, x, o));
    if (lane == 0) red[32] = x;
  }
  g.sync();
  double r = red[32];
  g.sync();
  return r;
}

template <class G>
__device__ __forceinline__ void apply_absence_block(const G &g, double *cur, int64_t p, const CandView &c, int32_t i) {
  int64_t lo = c.out_index[i];
  int64_t hi = c.in_index[i] + (c.spans[i] ? p : 0);
  double sz = (double)c.size[i];
  if (hi - lo - 1 <= p) {
    for (int64_t x = lo + 1 + g.idx(); x < hi; x += g.size()) cur[x % p] -= sz;
  } else {
    for (int64_t r = g.idx(); r < p; r += g.size()) {
      int h = absence_hits(r, lo, hi, p);
      for (int q = 0; q < h; q++) cur[r] -= sz;
    }
  }
  g.sync();
}

template <class G>
__device__ __forceinline__ double max_cur(const G &g, const double *cur, int64_t p, double *red) {
  double m = -INF_D;
  bool have = false;
  for (int64_t r = g.idx(); r < p; r += g.size()) {
    m = have ? pymax(m, cur[r]) : cur[r];
    have = true;
  }
  return block_max(g, m, red);
}

// key (area, size) then the smaller name: does candidate o beat b?
struct SwKey {
  int32_t i;   // -1: none
  int32_t rank;
  double area;
  int64_t size;
};
__device__ __forceinline__ bool swdoa_better(const SwKey &o, const SwKey &b) {
  return o.i >= 0 && (b.i < 0 || o.area > b.area ||
                      (o.area == b.area && (o.size > b.size || (o.size == b.size && o.rank < b.rank))));
}
__device__ __forceinline__ SwKey shfl_xor_key(const SwKey &k, int o) {
  return SwKey{__shfl_xor_sync(FULL_MASK, k.i, o), __shfl_xor_sync(FULL_MASK, k.rank, o),
               __shfl_xor_sync(FULL_MASK, k.area, o), __shfl_xor_sync(FULL_MASK, k.size, o)};
}

// ---------------------------------------------------------------------------
// exact gap areas
//
// Every operand of _step_area is an integer-valued double: op times and the
// period duration are differences of integer timestamps, loads and sizes
// are integers.  Its left fold only adds non-negative products cur[r] * ov,
// so while the exact integral stays below 2^53 every product and partial
// sum is an exactly representable integer and the fold returns the exact
// integral.  Then the integral can come from an int64 prefix sum
// W[j] = sum_{q<j} cur[q] * len_q in O(1) per candidate instead of an
// O(gap) fold; any candidate (or round) outside those bounds falls back to
// the reference fold.

#define EXACT_2_53 9007199254740992.0
#define EXACT_2_62 4611686018427387904.0

__device__ __forceinline__ bool int_valued(double x) { return x >= 0 && x < EXACT_2_53 && x == floor(x); }

// last slot r with op_times[r] <= x (bisect_right(op_times, x) - 1), >= 0
__device__ __forceinline__ int32_t slot_of(const LoadView &L, double x) {
  int64_t lo = 0, hi = L.p;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (x < L.op_times[mid]) hi = mid; else lo = mid + 1;
  }
  return (int32_t)(lo - 1 < 0 ? 0 : lo - 1);
}

// integral of the current load over [0, x] for x in slot j
__device__ __forceinline__ int64_t area_to(const LoadView &L, const double *cur, const int64_t *W, int32_t j,
                                           double x) {
  return W[j] + (int64_t)cur[j] * (int64_t)(x - L.op_times[j]);
}

// exact gap area of [a, b] (wrapping at the duration), or -1 when it may
// exceed 2^53 and the float fold has to run
__device__ __forceinline__ int64_t gap_area_exact(const LoadView &L, const double *cur, const int64_t *W, double a,
                                                  double b, int32_t ja, int32_t jb) {
  const double d = L.duration;
  int64_t ex;
  if (b <= d) {
    ex = b <= a ? 0 : area_to(L, cur, W, jb, b) - area_to(L, cur, W, ja, a);
  } else {
    int64_t x = d <= a ? 0 : W[L.p] - area_to(L, cur, W, ja, a);
    int64_t y = b - d <= 0 ? 0 : area_to(L, cur, W, jb, b - d);
    ex = x + y;
  }
  return ex < (int64_t)EXACT_2_53 ? ex : -1;
}

// the same integral without the 2^53 cut (int64; callers keep every
// integral below 2^62)
__device__ __forceinline__ int64_t gap_area_raw(const LoadView &L, const double *cur, const int64_t *W, double a,
                                                double b, int32_t ja, int32_t jb) {
  const double d = L.duration;
  if (b <= d) return b <= a ? 0 : area_to(L, cur, W, jb, b) - area_to(L, cur, W, ja, a);
  int64_t x = d <= a ? 0 : W[L.p] - area_to(L, cur, W, ja, a);
  int64_t y = b - d <= 0 ? 0 : area_to(L, cur, W, jb, b - d);
  return x + y;
}

// ---------------------------------------------------------------------------
// incremental gap areas.  Picking candidate c subtracts c.size from the
// load on c's absence slots, so every other candidate's exact integral
// drops by c.size times the wall time its gap shares with those slots:
// one O(1) update per candidate per round instead of a pass over the load.

// slot r spans [op_times[r], end(r)) in wall time
__device__ __forceinline__ double slot_end(const LoadView &L, int64_t r) {
  return r + 1 < L.p ? L.op_times[r + 1] : L.duration;
}

__device__ __forceinline__ double overlap(double x0, double x1, double y0, double y1) {
  const double lo = x0 > y0 ? x0 : y0, hi = x1 < y1 ? x1 : y1;
  return hi > lo ? hi - lo : 0.0;
}

// wall time of [y0, y1) inside candidate i's gap ([a, b], wrapping at the
// duration like gap_area)
__device__ __forceinline__ double gap_overlap(const LoadView &L, double a, double b, double y0, double y1) {
  const double d = L.duration;
  if (b <= d) return b <= a ? 0.0 : overlap(a, b, y0, y1);
  return (d <= a ? 0.0 : overlap(a, d, y0, y1)) + (b - d <= 0 ? 0.0 : overlap(0.0, b - d, y0, y1));
}

// The absence slots of candidate q (lo+1 .. hi-1 modulo p, each counted
// once per hit, as apply_absence subtracts once per hit: autoswap.py:119-129)
// as wall-time pieces: `full` whole periods plus up to two ranges.
struct AbsencePieces {
  double full;          // whole periods, each [op_times[0], duration)
  double y0[2], y1[2];  // partial ranges (empty when y1 <= y0)
};
__device__ __forceinline__ AbsencePieces absence_pieces(const LoadView &L, const CandView &c, int32_t q) {
  const int64_t p = L.p, lo = c.out_index[q], hi = c.in_index[q] + (c.spans[q] ? p : 0);
  AbsencePieces a{0.0, {0.0, 0.0}, {0.0, 0.0}};
  const int64_t n = hi - lo - 1;
  if (n <= 0) return a;
  const int64_t full = n / p, rem = n - full * p, st = (lo + 1) % p;
  a.full = (double)full;
  if (rem) {
    const int64_t last = st + rem - 1;
    a.y0[0] = L.op_times[st];
    if (last < p) {
      a.y1[0] = slot_end(L, last);
    } else {
      a.y1[0] = L.duration;
      a.y0[1] = L.op_times[0];
      a.y1[1] = slot_end(L, last - p);
    }
  }
  return a;
}

// wall time candidate i's gap [a, b] shares with those pieces
__device__ __forceinline__ double absence_overlap(const LoadView &L, const AbsencePieces &q, double a, double b) {
  double t = q.full != 0.0 ? q.full * gap_overlap(L, a, b, L.op_times[0], L.duration) : 0.0;
  if (q.y1[0] > q.y0[0]) t += gap_overlap(L, a, b, q.y0[0], q.y1[0]);
  if (q.y1[1] > q.y0[1]) t += gap_overlap(L, a, b, q.y0[1], q.y1[1]);
  return t;
}

// One pass over the current load: max(cur) (Python max: the first maximal
// value) and, when `exact` is requested and holds, W = the exclusive prefix
// of cur[q] * len_q (p + 1 entries).  `exact` comes back false when some cur
// is not an integer in [0, 2^53) or cur * duration may overflow.  Group-wide;
// sm: >= PM_SMEM long longs of shared memory.
constexpr int PM_SUM = 0, PM_TOT = 32, PM_MAX = 33, PM_MXR = 65, PM_OK = 66, PM_OKR = 98, PM_R0 = 100,
              PM_DONE = 101, PM_SMEM = 102;

template <class G>
__device__ double prefix_max_block(const G &g, const LoadView &L, const double *cur, int64_t *W, long long *sm,
                                   bool &exact) {
  const int tid = g.idx(), nt = g.size(), nw = (nt + 31) >> 5, lane = tid & 31;
  const int64_t p = L.p;
  int64_t per = (p + nt - 1) / nt;
  int64_t lo = tid * per, hi = lo + per < p ? lo + per : p;
  bool ok = exact;
  long long s = 0;
  double m = -INF_D;
  for (int64_t q = lo; q < hi; q++) {
    double c = cur[q];
    m = q == lo ? c : pymax(m, c);
    if (ok) {
      ok = int_valued(c) && c * L.duration < EXACT_2_62;
      double e = q + 1 < p ? L.op_times[q + 1] : L.duration;
      s += ok ? (long long)c * (long long)(e - L.op_times[q]) : 0;
    }
  }
  // threads are contiguous chunks in slot order, so combining in thread order
  // keeps Python's first-maximal semantics
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double u = __shfl_up_sync(FULL_MASK, m, o);
    if (lane >= o) m = pymax(u, m);
  }
  long long incl = warp_incl_scan_add(s);
  unsigned allok = __ballot_sync(FULL_MASK, ok);
  double *smd = reinterpret_cast<double *>(sm);
  if (lane == 31) {
    sm[PM_SUM + (tid >> 5)] = incl;
    smd[PM_MAX + (tid >> 5)] = m;
    sm[PM_OK + (tid >> 5)] = allok == FULL_MASK;
  }
  g.sync();
  if (tid == 0) {
    long long acc = 0, all = 1;
    double mx = smd[PM_MAX];
    for (int w = 0; w < nw; w++) {
      long long x = sm[PM_SUM + w];
      sm[PM_SUM + w] = acc;
      acc += x;
      if (w) mx = pymax(mx, smd[PM_MAX + w]);
      all &= sm[PM_OK + w];
    }
    smd[PM_MXR] = mx;
    sm[PM_TOT] = acc;
    sm[PM_OKR] = all;
  }
  g.sync();
  const bool all_exact = exact && sm[PM_OKR] != 0;
  const double mx = smd[PM_MXR];
  if (all_exact) {
    long long run = sm[PM_SUM + (tid >> 5)] + incl - s;
    for (int64_t q = lo; q < hi; q++) {
      W[q] = run;
      double e = q + 1 < p ? L.op_times[q + 1] : L.duration;
      run += (long long)cur[q] * (long long)(e - L.op_times[q]);
    }
    if (tid == 0) W[p] = sm[PM_TOT];
  }
  g.sync();
  exact = all_exact;
  return mx;
}

// scores + the SWDOA greedy (autoswap.py:132-215), group-wide.  peaks[j] =
// max(cur) after j picks, so a budgeted select_by_swdoa is the prefix
// order[0..m) with m the first j where peaks[j] <= limit.  With `stop` >= 0
// the greedy ends at the first planned peak <= stop (every budget at or
// above it is then decided); returns the number of picks made.  Any of
// doa/aoa/wdoa/swdoa may be null.  Scratch: W[p + 1], jx[2k]; shared
// memory keys >= 33 SwKey, sm >= PM_SMEM long longs.
// The rounds of the greedy on one warp, with incremental exact areas A[i]
// (see absence_overlap).  Runs while every round is exact in the sense of
// prefix_max_block (all loads integers in [0, 2^53), max * duration < 2^62);
// returns the first round it did not finish (== the pick count when it
// ended normally, with *done set).  Lane-strided; warp-collective.
static __device__ int64_t swdoa_rounds_warp(const LoadView &L, const CandView &c, double *cur, uint8_t *taken,
                                     double *swdoa, int32_t *order, double *peaks, int64_t *A, int64_t stop,
                                     bool &done) {
  const int lane = threadIdx.x & 31;
  const int64_t p = L.p, k = c.k;
  const double d = L.duration;
  done = false;
  for (int64_t round = 0;; round++) {
    double mx = -INF_D, mn = INF_D;
    for (int64_t r = lane; r < p; r += 32) {
      const double x = cur[r];
      mx = r == lane ? x : pymax(mx, x);
      mn = x < mn ? x : mn;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mx = pymax(mx, __shfl_xor_sync(FULL_MASK, mx, o));
      mn = fmin(mn, __shfl_xor_sync(FULL_MASK, mn, o));
    }
    if (lane == 0) peaks[round] = mx;
    if (round == k || (stop >= 0 && f_le_i(mx, stop))) {
      done = true;
      return round;
    }
    if (!(mn >= 0 && mx < EXACT_2_53 && mx * d < EXACT_2_62)) return round;
    SwKey best{-1, 0, 0.0, 0};
    for (int64_t i = lane; i < k; i += 32) {
      if (taken[i]) continue;
      const int64_t ex = A[i];
      SwKey o{(int32_t)i, c.name_rank[i], ex < (int64_t)EXACT_2_53 ? (double)ex : gap_area(L, cur, c.out_t[i], c.in_t[i]),
              c.size[i]};
      if (swdoa_better(o, best)) best = o;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      SwKey x = shfl_xor_key(best, o);
      if (swdoa_better(x, best)) best = x;
    }
    const int32_t pick = best.i;
    if (lane == 0) {
      order[round] = pick;
      if (swdoa) swdoa[pick] = best.area;
      taken[pick] = 1;
    }
    // the pick's absence, then every remaining candidate's area
    const int64_t lo = c.out_index[pick], hi = c.in_index[pick] + (c.spans[pick] ? p : 0);
    const double sz = (double)c.size[pick];
    if (hi - lo - 1 <= p) {
      // lo + 1 .. hi - 1, split at the period end (no modulo per slot)
      const int64_t e1 = hi < p ? hi : p;
      for (int64_t x = lo + 1 + lane; x < e1; x += 32) cur[x] -= sz;
      for (int64_t x = (lo + 1 > p ? lo + 1 - p : 0) + lane; x < hi - p; x += 32) cur[x] -= sz;
    } else {
      for (int64_t r = lane; r < p; r += 32) {
        const int h = absence_hits(r, lo, hi, p);
        for (int q = 0; q < h; q++) cur[r] -= sz;
      }
    }
    const AbsencePieces ap = absence_pieces(L, c, pick);
    const int64_t psz = c.size[pick];
    for (int64_t i = lane; i < k; i += 32) {
      if (i == pick || taken[i]) continue;
      A[i] -= psz * (int64_t)absence_overlap(L, ap, c.out_t[i], c.in_t[i]);
    }
    __syncwarp();
  }
}

template <class G>
__device__ int64_t swdoa_greedy_block(const G &g, const LoadView &L, const CandView &c, double *cur,
                                      uint8_t *taken, double *doa, double *aoa, double *wdoa, double *swdoa,
                                      int32_t *order, double *peaks, int64_t *W, int32_t *jx, SwKey *keys,
                                      long long *sm, int64_t stop = -1, int64_t *A = nullptr) {
  const int64_t p = L.p, k = c.k;
  const int tid = g.idx(), nt = g.size();
  bool times_ok = int_valued(L.duration);
  for (int64_t r = tid; r < p; r += nt) {
    cur[r] = (double)L.loads[r];
    times_ok &= int_valued(L.op_times[r]);
  }
  for (int64_t i = tid; i < k; i += nt) {
    double gap = c.in_t[i] - c.out_t[i];
    double d = gap - (c.dout[i] + c.din[i]);
    if (doa) doa[i] = d;
    if (aoa) aoa[i] = d >= 0 ? (double)c.size[i] * d : d / (double)c.size[i];
    if (wdoa) wdoa[i] = gap_area(L, nullptr, c.out_t[i], c.in_t[i]);
    taken[i] = 0;
    double a = c.out_t[i], b = c.in_t[i];
    times_ok &= int_valued(a) && int_valued(b);
    jx[2 * i] = slot_of(L, a);
    jx[2 * i + 1] = slot_of(L, b <= L.duration ? b : b - L.duration);
  }
  times_ok = g.sync_and(times_ok);
  const int lane = tid & 31, w = tid >> 5, nw = (nt + 31) >> 5;
  int64_t round0 = 0;
  if (A && times_ok) {
    // exact integrals of the initial load from its prefix, then the rounds
    // on warp 0 while they stay exact (the group waits at one barrier)
    bool exact = true;
    prefix_max_block(g, L, cur, W, sm, exact);
    if (exact) {
      for (int64_t i = tid; i < k; i += nt)
        A[i] = gap_area_raw(L, cur, W, c.out_t[i], c.in_t[i], jx[2 * i], jx[2 * i + 1]);
      g.sync();
      if (w == 0) {
        bool done;
        const int64_t r = swdoa_rounds_warp(L, c, cur, taken, swdoa, order, peaks, A, stop, done);
        if (lane == 0) {
          sm[PM_R0] = r;
          sm[PM_DONE] = done;
        }
      }
      g.sync();
      round0 = sm[PM_R0];
      const bool done = sm[PM_DONE] != 0;
      g.sync();
      if (done) return round0;
    }
  }
  for (int64_t round = round0;; round++) {
    bool exact = times_ok;
    const double pk = prefix_max_block(g, L, cur, W, sm, exact);
    if (tid == 0) peaks[round] = pk;
    if (round == k || (stop >= 0 && f_le_i(pk, stop))) return round;
    SwKey best{-1, 0, 0.0, 0};
    for (int64_t i = tid; i < k; i += nt) {
      if (taken[i]) continue;
      int64_t ex = exact ? gap_area_exact(L, cur, W, c.out_t[i], c.in_t[i], jx[2 * i], jx[2 * i + 1]) : -1;
      SwKey o{(int32_t)i, c.name_rank[i], ex >= 0 ? (double)ex : gap_area(L, cur, c.out_t[i], c.in_t[i]),
              c.size[i]};
      if (swdoa_better(o, best)) best = o;
    }
    // warp then group reduction of the argmax, keys carried in registers
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      SwKey x = shfl_xor_key(best, o);
      if (swdoa_better(x, best)) best = x;
    }
    if (lane == 0) keys[w] = best;
    g.sync();
    if (tid == 0) {
      SwKey b = keys[0];
      for (int q = 1; q < nw; q++)
        if (swdoa_better(keys[q], b)) b = keys[q];
      keys[32] = b;
      order[round] = b.i;
      if (swdoa) swdoa[b.i] = b.area;
      taken[b.i] = 1;
    }
    g.sync();
    const int32_t pick = keys[32].i;
    apply_absence_block(g, cur, p, c, pick);
  }
}

// ---------------------------------------------------------------------------
// _make_schedule + simulate: one warp per simulation.  The event loops are
// sequential (lane 0); the sorts are rank sorts across the warp's lanes.
// Every function below is warp-collective: all 32 lanes call it.

struct SimScratch {
  int32_t *ord;        // n
  double *desired;     // n
  int32_t *in_order;   // n
  double *plan_in, *in_done; uint8_t *in_has;  // n
  double *comp_t; int64_t *comp_sz;            // n
  int32_t *out_trigger, *in_wait;              // p
  uint32_t *busy_op;                           // (p + 31) / 32: ops a replay must visit
  int64_t *delta;                              // p
  double *actual;                              // p
  double *ready, *deadline;                    // n
  double *ev_t; int64_t *ev_d;                 // p (op events of the overlay)
  double *ev2_t; int64_t *ev2_d;               // 2n
  int32_t *ev2_ord;                            // 2n
};

// stable sort of positions 0..n-1 (ord[rank] = position) under a strict
// weak order: each lane ranks its positions by counting predecessors
template <class Less>
__device__ __forceinline__ void warp_rank_sort(int32_t *ord, int64_t n, Less less) {
  const int lane = threadIdx.x & 31;
  for (int64_t q = lane; q < n; q += 32) {
    int64_t r = 0;
    for (int64_t y = 0; y < n; y++) r += less(y, q) || (y < q && !less(q, y));
    ord[r] = (int32_t)q;
  }
  __syncwarp();
}

// positions of the selection ordered by (key, var name) (swapsim.py:76,82,98-102)
__device__ __forceinline__ void sort_by_key_name(int32_t *ord, int64_t n, const double *key, const int32_t *sel,
                                                 const CandView &c) {
  warp_rank_sort(ord, n, [&](int64_t y, int64_t x) {
    return key[y] < key[x] || (key[y] == key[x] && c.name_rank[sel[y]] < c.name_rank[sel[x]]);
  });
}

// _make_schedule, swapsim.py:62-108
static __device__ void make_schedule(const CandView &c, const int32_t *sel, int64_t n, const double *ready,
                              const double *deadline, double *t_so, double *t_eo, double *t_si, double *t_ei,
                              int32_t *eord, SimScratch &S) {
  const int lane = threadIdx.x & 31;
  sort_by_key_name(S.ord, n, ready, sel, c);
  if (lane == 0) {
    double busy = 0.0;
    for (int64_t q = 0; q < n; q++) {
      int32_t s = S.ord[q];
      double start = pymax(ready[s], busy);
      t_so[s] = start;
      busy = start + c.dout[sel[s]];
      t_eo[s] = busy;
    }
  }
  __syncwarp();
  sort_by_key_name(S.ord, n, deadline, sel, c);
  if (lane == 0) {
    double cap = INF_D;
    for (int64_t q = n - 1; q >= 0; q--) {
      int32_t s = S.ord[q];
      double end = pymin(deadline[s], cap);
      S.desired[q] = end - c.din[sel[s]];
      cap = S.desired[q];
    }
    double prev_end = 0.0;
    for (int64_t q = 0; q < n; q++) {
      int32_t s = S.ord[q];
      double start = pymax(pymax(S.desired[q], t_eo[s]), prev_end);
      t_si[s] = start;
      prev_end = start + c.din[sel[s]];
      t_ei[s] = prev_end;
    }
  }
  __syncwarp();
  sort_by_key_name(eord, n, t_so, sel, c);
}

// load curve with stored points (LoadCurve.points, swapsim.py:166-181/227-233)
struct Curve {
  double *t;
  int64_t *v;
  int64_t n, peak, load;
  double peak_t;
  __device__ void reset(int64_t l0) {
    n = 1; t[0] = 0.0; v[0] = l0; load = l0; peak = l0; peak_t = 0.0;
  }
  __device__ void point(double tt) {
    if (t[n - 1] == tt) v[n - 1] = load;
    else { t[n] = tt; v[n] = load; n++; }
    if (load > peak) { peak = load; peak_t = tt; }
  }
};

// the same curve when only its peak and point count are wanted (the sweep)
struct PeakCurve {
  double last_t;
  int64_t n, peak, load;
  double peak_t;
  __device__ void reset(int64_t l0) {
    n = 1; last_t = 0.0; load = l0; peak = l0; peak_t = 0.0;
  }
  __device__ void point(double tt) {
    if (last_t != tt) { last_t = tt; n++; }
    if (load > peak) { peak = load; peak_t = tt; }
  }
};

// replay state (lane 0 owns it).  The heads of both transfer queues — the
// next swap-out completion and the next planned swap-in with its size and
// duration — are cached in registers and refreshed only when a queue moves,
// so probing for the next transfer (every op, usually "nothing before this
// op") costs no shared-memory round trips.
template <class CurveT>
struct Replay {
  int64_t k_in, k_out, ncomp, n;
  double in_busy, head_floor, out_busy, delay;
  CurveT cv;
  int64_t ndl;
  bool has_limit;
  int64_t limit;
  double nx_t;      // comp_t[k_out], or INF when k_out >= ncomp
  int64_t nx_sz;    // comp_sz[k_out]
  int64_t hv;       // in_order[k_in], or -1 when k_in >= n
  double hv_plan, hv_din;
  int64_t hv_size;
};

template <class CurveT>
__device__ __forceinline__ void rp_out_head(Replay<CurveT> &R, const SimScratch &S) {
  if (R.k_out < R.ncomp) {
    R.nx_t = S.comp_t[R.k_out];
    R.nx_sz = S.comp_sz[R.k_out];
  } else {
    R.nx_t = INF_D;
  }
}

template <class CurveT>
__device__ __forceinline__ void rp_in_head(Replay<CurveT> &R, const SimScratch &S, const CandView &c,
                                           const int32_t *sel) {
  if (R.k_in < R.n) {
    R.hv = S.in_order[R.k_in];
    R.hv_plan = S.plan_in[R.hv];
    const int32_t ci = sel[R.hv];
    R.hv_size = c.size[ci];
    R.hv_din = c.din[ci];
  } else {
    R.hv = -1;
  }
}

// _Replay._step, swapsim.py:256-282: 1 stepped, 0 beyond horizon,
// -1 IndexError (the reference defect at swapsim.py:266-267)
template <class CurveT>
__device__ __forceinline__ int rp_step(Replay<CurveT> &R, SimScratch &S, const CandView &c, const int32_t *sel, double horizon) {
  const double t_out = R.nx_t;
  double t_in = INF_D;
  if (R.hv >= 0) {
    double start = pymax(pymax(R.hv_plan, R.in_busy), R.head_floor);
    if (R.has_limit && R.cv.load + R.hv_size > R.limit) start = INF_D;
    t_in = start;
  }
  double t = pymin(t_out, t_in);
  if (t > horizon) return 0;
  if (t_out <= t_in) {
    if (R.k_out >= R.ncomp) return -1;
    R.k_out++;
    R.cv.load -= R.nx_sz;
    R.head_floor = pymax(R.head_floor, t_out);
    R.cv.point(t_out);
    rp_out_head(R, S);
  } else {
    R.cv.load += R.hv_size;
    R.cv.point(t_in);
    double end = t_in + R.hv_din;
    R.in_busy = end;
    S.in_done[R.hv] = end;
    S.in_has[R.hv] = 1;
    R.k_in++;
    rp_in_head(R, S, c, sel);
  }
  return 1;
}

// one _Replay(...).run(), swapsim.py:205-346; returns the status (all lanes).
//
// Only ops with a load delta, an awaited swap-in or a triggered swap-out
// (and the last op) can change the replay state: at any other op the
// reference just processes pending transfers up to its start time, and
// doing that at the next visited op instead performs the same steps in the
// same order.  So lane 0 visits busy ops only; FILL_ACTUAL also writes the
// skipped ops' start times (tau[r] + delay: no delay accrues between busy
// ops), which only the delayed-op report needs.
template <bool FILL_ACTUAL, class CurveT>
__device__ int replay_run(Replay<CurveT> &R, SimScratch &S, const ProfView &P, const int64_t live0,
                          const CandView &c, const int32_t *sel, const double *t_si, const double *t_ei,
                          const int32_t *eord, double d_actual, int64_t *eidx, int64_t *eaux0, int64_t *eaux1) {
  const int lane = threadIdx.x & 31;
  const int64_t p = P.p, n = R.n;
  long long dl = 0;
  for (int64_t q = lane; q < n; q += 32) {
    int32_t s = eord[q];
    int32_t ci = sel[s];
    if (c.spans[ci]) {
      dl += c.size[ci];
      S.plan_in[s] = pymax(t_si[s] - d_actual, 0.0);
    } else {
      S.plan_in[s] = t_si[s];
    }
    S.in_has[s] = 0;
  }
  const int64_t l0 = live0 - warp_sum(dl);
  for (int64_t r = lane; r < p; r += 32) { S.out_trigger[r] = -1; S.in_wait[r] = -1; }
  __syncwarp();
  // in_order: (plan_in, deadline, name), swapsim.py:226-229
  warp_rank_sort(S.in_order, n, [&](int64_t y, int64_t x) {
    int32_t a = eord[y], b = eord[x];
    return S.plan_in[a] < S.plan_in[b] ||
           (S.plan_in[a] == S.plan_in[b] && (t_ei[a] < t_ei[b] ||
                                             (t_ei[a] == t_ei[b] && c.name_rank[sel[a]] < c.name_rank[sel[b]])));
  });
  for (int64_t q = lane; q < n; q += 32) S.in_order[q] = eord[S.in_order[q]];
  if (lane == 0)
    for (int64_t s = 0; s < n; s++) {  // dict comprehension: later entries win
      S.out_trigger[c.out_index[sel[s]]] = (int32_t)s;
      S.in_wait[c.in_index[sel[s]]] = (int32_t)s;
    }
  __syncwarp();
  const int64_t nwords = (p + 31) >> 5;
  for (int64_t w = lane; w < nwords; w += 32) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; b++) {
      int64_t r = w * 32 + b;
      if (r < p && (S.delta[r] != 0 || S.in_wait[r] >= 0 || S.out_trigger[r] >= 0 || r == p - 1))
        bits |= 1u << b;
    }
    S.busy_op[w] = bits;
  }
  __syncwarp();
  int status = MP_OK;
  if (lane == 0) {
    R.k_in = 0; R.in_busy = 0.0; R.head_floor = 0.0; R.ncomp = 0; R.k_out = 0;
    R.out_busy = 0.0; R.delay = 0.0; R.ndl = 0;
    R.cv.reset(l0);
    rp_out_head(R, S);
    rp_in_head(R, S, c, sel);
    int64_t filled = 0;
    for (int64_t w = 0; w < nwords && status == MP_OK; w++) {
      uint32_t bits = S.busy_op[w];
      while (bits) {
        const int64_t r = w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
        // this op's inputs, loaded together up front
        const double tau_r = P.tau[r];
        const int32_t wt = S.in_wait[r];
        const int64_t dd = S.delta[r];
        const int32_t trig = S.out_trigger[r];
        if (FILL_ACTUAL)
          for (; filled < r; filled++) S.actual[filled] = P.tau[filled] + R.delay;
        double t0 = tau_r + R.delay, t = t0;
        int st;
        while ((st = rp_step(R, S, c, sel, t)) == 1) {}
        if (st < 0) { status = MP_E_SIM_INDEXERROR; break; }
        if (wt >= 0) {
          int ws = 1;
          while (!S.in_has[wt]) {
            ws = rp_step(R, S, c, sel, INF_D);
            if (ws <= 0) break;
          }
          if (ws < 0) { status = MP_E_SIM_INDEXERROR; break; }
          if (ws == 0) {
            *eidx = P.window0 + r; *eaux0 = 1; *eaux1 = sel[wt];
            status = MP_E_SWAP_DEADLOCK;
            break;
          }
          if (S.in_done[wt] > t + EPS_US) {
            t = S.in_done[wt];
            while ((st = rp_step(R, S, c, sel, t)) == 1) {}
            if (st < 0) { status = MP_E_SIM_INDEXERROR; break; }
          }
        }
        if (dd > 0 && R.has_limit) {
          while (R.cv.load + dd > R.limit) {
            if (R.k_out >= R.ncomp) {
              *eidx = P.window0 + r; *eaux0 = 0; *eaux1 = 0;
              status = MP_E_SWAP_DEADLOCK;
              break;
            }
            const double t_free = R.nx_t;
            const int64_t sz = R.nx_sz;
            R.k_out++;
            rp_out_head(R, S);
            R.cv.load -= sz;
            R.head_floor = pymax(R.head_floor, t_free);
            R.cv.point(t_free);
            t = pymax(t, t_free);
          }
          if (status != MP_OK) break;
        }
        if (t > t0 + EPS_US) {
          R.ndl++;  // the list itself is rebuilt from actual starts (k_sim_delays)
          R.delay += t - t0;
        } else {
          t = t0;
        }
        S.actual[r] = t;
        filled = r + 1;
        if (dd != 0) {
          R.cv.load += dd;
          R.cv.point(t);
          if (dd < 0) {
            R.head_floor = pymax(R.head_floor, t);
            while ((st = rp_step(R, S, c, sel, t)) == 1) {}
            if (st < 0) { status = MP_E_SIM_INDEXERROR; break; }
          }
        }
        if (trig >= 0) {
          double op_end = r + 1 < p ? P.tau[r + 1] : P.duration;
          double ready = t + (op_end - tau_r);
          double start = pymax(ready, R.out_busy);
          R.out_busy = start + c.dout[sel[trig]];
          S.comp_t[R.ncomp] = R.out_busy;
          S.comp_sz[R.ncomp] = c.size[sel[trig]];
          R.ncomp++;
          if (R.k_out == R.ncomp - 1) { R.nx_t = R.out_busy; R.nx_sz = S.comp_sz[R.k_out]; }
        }
      }
    }
  }
  __syncwarp();
  return __shfl_sync(FULL_MASK, status, 0);
}

// (t, d) lexicographic
__device__ __forceinline__ bool td_less(double ta, int64_t da, double tb, int64_t db) {
  return ta < tb || (ta == tb && da < db);
}

// S.ev_t/ev_d <- the op events (t, delta) of _overlay_curve sorted by
// (t, delta) (swapsim.py:184-193); returns their count.  Independent of the
// selection, so a sweep builds it once per trace.  One thread.
__device__ __forceinline__ int64_t sim_op_events(const ProfView &P, const int64_t *delta, double *ev_t,
                                                 int64_t *ev_d) {
  int64_t na = 0;
  for (int64_t r = 0; r < P.p; r++)
    if (delta[r] != 0) { ev_t[na] = P.tau[r]; ev_d[na] = delta[r]; na++; }
  // op times are non-decreasing: sort equal-time runs by delta
  for (int64_t q = 1; q < na; q++) {
    double xt = ev_t[q];
    int64_t xd = ev_d[q];
    int64_t j = q - 1;
    while (j >= 0 && td_less(xt, xd, ev_t[j], ev_d[j])) { ev_t[j + 1] = ev_t[j]; ev_d[j + 1] = ev_d[j]; j--; }
    ev_t[j + 1] = xt;
    ev_d[j + 1] = xd;
  }
  return na;
}

// LOAD' overlay (swapsim.py:184-202) of the schedule (t_eo, t_si, eord)
// merged with na sorted op events; the curve is lane 0's
template <class CurveT>
__device__ void sim_overlay(const ProfView &P, const CandView &c, const int32_t *sel, int64_t n, int64_t live0,
                            const double *t_eo, const double *t_si, const int32_t *eord, const double *ev_t,
                            const int64_t *ev_d, int64_t na, SimScratch &S, CurveT &cv) {
  const int lane = threadIdx.x & 31;
  const double dnat = P.duration;
  long long dl = 0;
  for (int64_t q = lane; q < n; q += 32) {
    int32_t s = eord[q];
    int32_t ci = sel[s];
    S.ev2_t[2 * q] = t_eo[s];
    S.ev2_d[2 * q] = -c.size[ci];
    if (c.spans[ci]) { dl += c.size[ci]; S.ev2_t[2 * q + 1] = pymax(t_si[s] - dnat, 0.0); }
    else S.ev2_t[2 * q + 1] = t_si[s];
    S.ev2_d[2 * q + 1] = c.size[ci];
  }
  const int64_t l0 = live0 - warp_sum(dl);
  __syncwarp();
  const int64_t nb = 2 * n;
  warp_rank_sort(S.ev2_ord, nb, [&](int64_t y, int64_t x) {
    return td_less(S.ev2_t[y], S.ev2_d[y], S.ev2_t[x], S.ev2_d[x]);
  });
  if (lane == 0) {
    cv.reset(l0);
    int64_t ia = 0, ib = 0;
    while (ia < na || ib < nb) {
      int32_t jb = ib < nb ? S.ev2_ord[ib] : 0;
      bool take_a = ib >= nb || (ia < na && !td_less(S.ev2_t[jb], S.ev2_d[jb], ev_t[ia], ev_d[ia]));
      double t;
      int64_t d;
      if (take_a) { t = ev_t[ia]; d = ev_d[ia]; ia++; }
      else { t = S.ev2_t[jb]; d = S.ev2_d[jb]; ib++; }
      cv.load += d;
      cv.point(t);
    }
  }
  __syncwarp();
}

struct SimTimes {
  double *t_so, *t_eo, *t_si, *t_ei;
  int32_t *eord;
};

struct SimResult {
  int status;
  int64_t rounds, eidx, eaux0, eaux1;
  double delay;
};

// the LOAD'' replay with the fixed point on total delay (swapsim.py:349-395);
// T holds the initial schedule on entry and the last one on exit.  The
// result (and R) are lane 0's.
template <bool FILL_ACTUAL, class CurveT>
__device__ SimResult sim_fixed_point(const ProfView &P, const CandView &c, const int32_t *sel, int64_t n,
                                     int64_t limit, int has_limit, int max_rounds, int64_t live0, SimScratch &S,
                                     const SimTimes &T, Replay<CurveT> &R) {
  const int lane = threadIdx.x & 31;
  const int64_t p = P.p;
  const double dnat = P.duration;
  R.n = n;
  R.has_limit = has_limit;
  R.limit = limit;
  double prev_delay = 0.0;
  bool have_prev = false;
  SimResult out{MP_OK, 0, 0, 0, 0, 0.0};
  for (int it = 0; it < max_rounds; it++) {
    out.status = replay_run<FILL_ACTUAL>(R, S, P, live0, c, sel, T.t_si, T.t_ei, T.eord,
                                         dnat + (have_prev ? prev_delay : 0.0), &out.eidx, &out.eaux0, &out.eaux1);
    if (out.status) break;
    out.rounds++;
    const double delay = __shfl_sync(FULL_MASK, R.delay, 0);
    if (n == 0 || delay == 0.0) break;
    if (have_prev && fabs(delay - prev_delay) < 1e-6) break;
    prev_delay = delay;
    have_prev = true;
    double d_act = dnat + delay;
    for (int64_t s = lane; s < n; s += 32) {
      int32_t ci = sel[s];
      int64_t oi = c.out_index[ci];
      double op_end = oi + 1 < p ? P.tau[oi + 1] : dnat;
      double dur = op_end - P.tau[oi];
      S.ready[s] = S.actual[oi] + dur;
      S.deadline[s] = S.actual[c.in_index[ci]] + (c.spans[ci] ? d_act : 0.0);
    }
    __syncwarp();
    make_schedule(c, sel, n, S.ready, S.deadline, T.t_so, T.t_eo, T.t_si, T.t_ei, T.eord, S);
  }
  out.delay = R.delay;
  return out;
}
