// sweep.cu — batched planning sweep, one CTA per trace (BASELINE configs[4]).
//
// A sweep is thousands of small independent traces (models x batch sizes x
// swap budgets).  Each is far too small to fill a GPU with the grid-wide
// kernels of ingest.cu / conflict.cu / placement.cu / swap.cu, so here one
// CTA runs a trace's whole path — what the reference's estimators run for
// it (estimators.py:20-130):
//
//   validate_trace          trace.py:55-84        thread per position / variable
//   detect_iteration        iteration.py:93-105   warps race over candidate periods
//   extract_lifetimes       iteration.py:124-320  the same per-variable state
//                                                 machines as ingest.cu (ingest_dev.cuh)
//   build_conflict_graph +  smartpool.py:51-144   placement order by a CTA bitonic
//   plan_pool                                     sort; each step one warp gathers
//                                                 the placed neighbours (segment
//                                                 overlap tested on the fly) and
//                                                 replays _pick_offset (place_dev.cuh)
//   filter_candidates,      autoswap.py:80-225    swap_dev.cuh: thread per variable,
//   compute_load_min,       swapsim.py:398-405    slot-parallel, CTA-wide greedy
//   SWDOA greedy
//   per budget:             estimators.py:93-130  one warp (lane 0) per budget:
//   SwapPlanner.fit                               limit checks, the greedy prefix,
//                                                 _make_schedule, simulate
//
// Persistent CTAs pull traces from a work counter (largest first), and each
// CTA bump-allocates the trace's working arrays from its own slab of global
// scratch — small enough per trace to stay L2-resident.
#include <algorithm>

#include "handles.cuh"
#include "ingest_dev.cuh"
#include "place_dev.cuh"
#include "swap_dev.cuh"

#ifndef SW_THREADS_N
#define SW_THREADS_N 192  // 6 warps: 5 on the swap path, budgets of the largest traces start together (128: ~1 % slower)
#endif
constexpr int SW_THREADS = SW_THREADS_N;
constexpr int SW_WARPS = SW_THREADS / 32;
#ifndef SW_FAST_KB
#define SW_FAST_KB 88  // per-CTA shared arena: 2 CTAs/SM, the largest traces keep their budget scratch in smem (72 KB, 3 CTAs/SM: 3 % slower)
#endif
constexpr size_t SW_FAST_BYTES = SW_FAST_KB * 1024;
constexpr int SW_QUICK = 16;  // detect: fingerprint pairs of the quick filter
#ifndef PL_K_N
#define PL_K_N 4
#endif
constexpr int PL_K = PL_K_N;  // placement list entries per lane per pass

// ---------------------------------------------------------------------------
// scratch allocation.  Each CTA owns a slab of global scratch (bump
// allocated per trace, count-only when base is null: the host sizes slabs
// with the same calls the device makes) and a dynamic shared-memory arena
// that each phase refills from the bottom; Arena::take serves an array from
// shared memory when it fits and from the slab otherwise.

struct Bump {
  char *base;
  size_t top, cap;
  bool over;
  template <typename T>
  __host__ __device__ T *take(int64_t n) {
    size_t a = (top + 15) & ~(size_t)15;
    size_t b = a + (size_t)(n > 0 ? n : 1) * sizeof(T);
    top = b;
    if (b > cap) over = true;
    return (base && !over) ? reinterpret_cast<T *>(base + a) : nullptr;
  }
};

struct Arena {
  Bump fast, slow;
  template <typename T>
  __host__ __device__ T *take(int64_t n) {
    size_t a = (fast.top + 15) & ~(size_t)15;
    size_t b = a + (size_t)(n > 0 ? n : 1) * sizeof(T);
    if (fast.base && b <= fast.cap) {
      fast.top = b;
      return reinterpret_cast<T *>(fast.base + a);
    }
    return slow.take<T>(n);
  }
  __device__ void phase() { fast.top = 0; }
};

static __host__ __device__ int64_t pow2_at_least(int64_t x) {
  int64_t r = 1;
  while (r < x) r <<= 1;
  return r;
}

// the trace's kind/size columns staged on chip, and its events grouped by
// variable (perm, gstart) — read by validate, detect and extract
struct GroupArrays {
  uint8_t *kind;
  int64_t *size;
  int32_t *cnt;
  int64_t *gstart;
  uint32_t *perm;
  template <class A>
  __host__ __device__ void take(A &b, int64_t n, int64_t nv) {
    kind = b.template take<uint8_t>(n);
    size = b.template take<int64_t>(n);
    cnt = b.template take<int32_t>(nv + 1);
    gstart = b.template take<int64_t>(nv + 1);
    perm = b.template take<uint32_t>(n);
  }
};

struct ExtractArrays {
  ExScratch s;
  int32_t *carry_ord, *win_ord;
  template <class A>
  __host__ __device__ void take(A &b, int64_t p, int64_t nv) {
    s.owner = b.template take<int32_t>(p); s.w_free = b.template take<int32_t>(p);
    s.w_nacc = b.template take<int32_t>(p); s.w_flags = b.template take<uint8_t>(p);
    s.w_mcarry = b.template take<int32_t>(p); s.is_malloc = b.template take<int32_t>(p);
    win_ord = b.template take<int32_t>(p);
    s.c_live = b.template take<uint8_t>(nv); s.c_abs = b.template take<int64_t>(nv);
    s.c_size = b.template take<int64_t>(nv); s.c_free = b.template take<int32_t>(nv);
    s.c_nacc = b.template take<int32_t>(nv); s.c_case = b.template take<uint8_t>(nv);
    s.c_twin = b.template take<int32_t>(nv); s.c_surv = b.template take<int32_t>(nv);
    s.nmalloc = b.template take<int32_t>(nv);
    carry_ord = b.template take<int32_t>(nv);
  }
};

// per-op arrays every later stage reads
struct TimeArrays {
  double *op_times;
  int64_t *diff;  // p + 1: load diff, scanned in place (loads = diff + 1)
  template <class A>
  __host__ __device__ void take(A &b, int64_t p) {
    op_times = b.template take<double>(p);
    diff = b.template take<int64_t>(p + 1);
  }
};

struct ProfileArrays {
  int32_t *base, *alloc, *free_, *nseg, *seg, *acc_index;
  int64_t *size, *acc_off, *acc_cnt;
  uint8_t *flags, *acc_next;
  template <class A>
  __host__ __device__ void take(A &b, int64_t p, int64_t V) {
    base = b.template take<int32_t>(V); alloc = b.template take<int32_t>(V); free_ = b.template take<int32_t>(V);
    nseg = b.template take<int32_t>(V); seg = b.template take<int32_t>(4 * V); size = b.template take<int64_t>(V);
    flags = b.template take<uint8_t>(V); acc_off = b.template take<int64_t>(V + 1);
    acc_cnt = b.template take<int64_t>(V + 1);
    acc_index = b.template take<int32_t>(p); acc_next = b.template take<uint8_t>(p);
  }
};

// placement in rank space: position q of the placement order holds the
// q-th variable's segments, size and offset; row q of adj has bit j set
// for every earlier j < q it conflicts with
struct PlaceArrays {
  int32_t *order;
  int64_t *ksize;  // sort keys staged: size, alloc, base
  int32_t *kalloc, *kbase;
  int4 *rseg;
  int64_t *rsize;
  uint32_t *adj;
  // every placed range, sorted by start: start, end, rank
  int64_t *ls, *le;
  int32_t *lr;
  int64_t n2, words;
  template <class A>
  __host__ __device__ void take(A &b, int64_t V) {
    n2 = pow2_at_least(V > 1 ? V : 1);
    words = (V + 31) / 32;
    order = b.template take<int32_t>(n2);
    ksize = b.template take<int64_t>(V);
    kalloc = b.template take<int32_t>(V);
    kbase = b.template take<int32_t>(V);
    rseg = b.template take<int4>(V);
    rsize = b.template take<int64_t>(V);
    ls = b.template take<int64_t>(V);
    le = b.template take<int64_t>(V);
    lr = b.template take<int32_t>(V);
    adj = b.template take<uint32_t>(V * words);
  }
};

// swap-path arrays that live until the budgets are done (shared memory
// when they fit: the budget phase refills the arena above them)
struct SwapKeep {
  CandOut c;
  int32_t *name_rank, *order;
  double *peaks, *tau, *ev_t;
  int64_t *delta, *ev_d;
  template <class A>
  __host__ __device__ void take(A &b, int64_t p, int64_t V) {
    c.var = b.template take<int32_t>(V); c.out_index = b.template take<int32_t>(V);
    c.in_index = b.template take<int32_t>(V); c.size = b.template take<int64_t>(V);
    c.out_t = b.template take<double>(V); c.out_ready = b.template take<double>(V);
    c.in_t = b.template take<double>(V); c.dout = b.template take<double>(V);
    c.din = b.template take<double>(V); c.spans = b.template take<uint8_t>(V);
    name_rank = b.template take<int32_t>(V);
    order = b.template take<int32_t>(V);
    peaks = b.template take<double>(V + 1);
    tau = b.template take<double>(p);
    delta = b.template take<int64_t>(p);
  }
  // the overlay's op events are read once per budget: global scratch
  template <class A>
  __host__ __device__ void take_events(A &b, int64_t p) {
    ev_t = b.template take<double>(p);
    ev_d = b.template take<int64_t>(p);
  }
};

// candidates before compaction, and per-op scratch of the swap path
struct SwapScratch {
  int32_t *flag, *pos, *evpos, *cbase, *cralloc;
  CandOut tmp;
  int64_t *lmdiff;
  template <class A>
  __host__ __device__ void take(A &b, int64_t p, int64_t V) {
    flag = b.template take<int32_t>(V); pos = b.template take<int32_t>(V);
    cbase = b.template take<int32_t>(V); cralloc = b.template take<int32_t>(V);
    evpos = b.template take<int32_t>(p + 1);
    tmp.var = b.template take<int32_t>(V); tmp.out_index = b.template take<int32_t>(V);
    tmp.in_index = b.template take<int32_t>(V); tmp.size = b.template take<int64_t>(V);
    tmp.out_t = b.template take<double>(V); tmp.out_ready = b.template take<double>(V);
    tmp.in_t = b.template take<double>(V); tmp.dout = b.template take<double>(V);
    tmp.din = b.template take<double>(V); tmp.spans = b.template take<uint8_t>(V);
    lmdiff = b.template take<int64_t>(p + 1);
  }
};

// the greedy's working set
struct GreedyArrays {
  double *cur;
  int64_t *W;
  int64_t *area;  // incremental exact gap areas
  int32_t *jx;
  uint8_t *taken;
  template <class A>
  __host__ __device__ void take(A &b, int64_t p, int64_t k) {
    cur = b.template take<double>(p);
    W = b.template take<int64_t>(p + 1);
    area = b.template take<int64_t>(k);
    jx = b.template take<int32_t>(2 * k);
    taken = b.template take<uint8_t>(k);
  }
};

struct BudgetArrays {
  SimScratch S;
  SimTimes T;
  template <class A>
  __host__ __device__ void take(A &b, int64_t p, int64_t k) {
    S.ord = b.template take<int32_t>(k); S.desired = b.template take<double>(k);
    S.in_order = b.template take<int32_t>(k); S.plan_in = b.template take<double>(k);
    S.in_done = b.template take<double>(k); S.in_has = b.template take<uint8_t>(k);
    S.comp_t = b.template take<double>(k); S.comp_sz = b.template take<int64_t>(k);
    S.out_trigger = b.template take<int32_t>(p); S.in_wait = b.template take<int32_t>(p);
    S.busy_op = b.template take<uint32_t>((p + 31) / 32);
    S.delta = nullptr;  // shared per trace
    S.actual = b.template take<double>(p);
    S.ready = b.template take<double>(k); S.deadline = b.template take<double>(k);
    S.ev_t = nullptr; S.ev_d = nullptr;  // shared per trace
    S.ev2_t = b.template take<double>(2 * k); S.ev2_d = b.template take<int64_t>(2 * k);
    S.ev2_ord = b.template take<int32_t>(2 * k);
    T.t_so = b.template take<double>(k); T.t_eo = b.template take<double>(k);
    T.t_si = b.template take<double>(k); T.t_ei = b.template take<double>(k);
    T.eord = b.template take<int32_t>(k);
  }
};

// slab bytes a trace of n events and nv names can need (worst case: every
// array spills out of shared memory, the window is half the trace, every
// name carried in, every variable a candidate)
static size_t slab_bound(int64_t n, int64_t nv, int nb) {
  Bump b{nullptr, 0, SIZE_MAX, false};
  int64_t p = n / 2, V = nv + p;
  GroupArrays g; g.take(b, n, nv);
  ExtractArrays x; x.take(b, p, nv);
  TimeArrays ta; ta.take(b, p);
  ProfileArrays pa; pa.take(b, p, V);
  PlaceArrays pl; pl.take(b, V);
  SwapKeep kp; kp.take(b, p, V); kp.take_events(b, p);
  SwapScratch ss; ss.take(b, p, V);
  GreedyArrays gr; gr.take(b, p, V);
  for (int i = 0; i < nb; i++) { BudgetArrays ba; ba.take(b, p, V); }
  return (b.top + 255) & ~(size_t)255;
}

// ---------------------------------------------------------------------------
// group-wide helpers (CtaGroup or a WarpGroup of the CTA's warps)

// exclusive scan of n values (out may alias in); returns the total.
// sm: >= 33 long longs
template <class G, typename T, typename U>
__device__ U grp_excl_scan(const G &g, const T *in, U *out, int64_t n, long long *sm) {
  const int tid = g.idx(), nt = g.size(), nw = nt >> 5;
  int64_t per = (n + nt - 1) / nt;
  int64_t lo = tid * per, hi = lo + per < n ? lo + per : n;
  long long s = 0;
  for (int64_t i = lo; i < hi; i++) s += in[i];
  long long incl = warp_incl_scan_add(s);
  if ((tid & 31) == 31) sm[tid >> 5] = incl;
  g.sync();
  if (tid == 0) {
    long long acc = 0;
    for (int w = 0; w < nw; w++) { long long x = sm[w]; sm[w] = acc; acc += x; }
    sm[32] = acc;
  }
  g.sync();
  long long run = sm[tid >> 5] + incl - s;
  for (int64_t i = lo; i < hi; i++) { T x = in[i]; out[i] = (U)run; run += x; }
  U total = (U)sm[32];
  g.sync();
  return total;
}

template <class G>
__device__ __forceinline__ long long grp_sum(const G &g, long long v, long long *sm) {
  v = warp_sum(v);
  if ((g.idx() & 31) == 0) sm[g.idx() >> 5] = v;
  g.sync();
  long long t = 0;
  for (int w = 0; w < (g.size() >> 5); w++) t += sm[w];
  g.sync();
  return t;
}

template <class G>
__device__ __forceinline__ long long grp_max(const G &g, long long v, long long *sm) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    long long u = __shfl_xor_sync(FULL_MASK, v, o);
    v = u > v ? u : v;
  }
  if ((g.idx() & 31) == 0) sm[g.idx() >> 5] = v;
  g.sync();
  long long t = sm[0];
  for (int w = 1; w < (g.size() >> 5); w++) t = sm[w] > t ? sm[w] : t;
  g.sync();
  return t;
}

// placement order (smartpool.py:91-98): -size, alloc (carry-ins -1 first),
// name — carry-ins keep their base name, so the base id orders them
__device__ __forceinline__ bool place_less(const PlaceArrays &pl, int32_t x, int32_t y) {
  if (x < 0) return false;
  if (y < 0) return true;
  if (pl.ksize[x] != pl.ksize[y]) return pl.ksize[x] > pl.ksize[y];
  if (pl.kalloc[x] != pl.kalloc[y]) return pl.kalloc[x] < pl.kalloc[y];
  if (pl.kbase[x] != pl.kbase[y]) return pl.kbase[x] < pl.kbase[y];
  return x < y;
}

// ---------------------------------------------------------------------------

struct SweepArgs {
  int64_t T;
  const int64_t *ev_off, *var_off, *name_off;
  const uint8_t *kind, *blob;
  const int32_t *var;
  const int64_t *size, *t_us;
  const int32_t *work;
  int32_t *counter;
  mp_sweep_params prm;
  mp_sweep_trace *rec;
  mp_sweep_budget *brec;
  int64_t *offsets;
  int32_t *cand_order;
  char *slab;
  size_t slab_bytes;
  long long *prof;  // optional: clock64() at 8 phase marks per trace
};

#define SW_MARK(i) \
  do { if (a.prof && threadIdx.x == 0) a.prof[t * 16 + (i)] = clock64(); } while (0)

struct SweepShared {
  unsigned long long first;
  long long best_p;
  long long sm[33];          // CTA reductions
  long long gsm[PM_SMEM];    // swap-group reductions (concurrent with placement)
  double dur;
  long long edges;
  long long na;
  int bad, unsorted;
  double red[33];
  SwKey keys[33];
  int next_budget, swap_ready, nomem;
  BudgetArrays ba[MP_SWEEP_MAX_BUDGETS];
};

__device__ void sweep_fail(const SweepArgs &a, int64_t t, int status, int code, int64_t index,
                           const mp_sweep_trace &R) {
  if (threadIdx.x == 0) {
    mp_sweep_trace r = R;
    r.status = status;
    r.err_code = code;
    r.err_index = index;
    a.rec[t] = r;
  }
  for (int b = threadIdx.x; b < a.prm.nbudget; b += blockDim.x) {
    mp_sweep_budget rb{};
    rb.status = status;
    a.brec[t * a.prm.nbudget + b] = rb;
  }
  __syncthreads();
}

// SwapPlanner(limit, score="swdoa").fit (estimators.py:85-130) for budgets
// pulled from the shared counter, one warp each.
static __device__ __forceinline__ void sweep_budgets(SweepShared *shp, const SwapKeep kp, const ProfView P,
                                                  const int64_t peak, const double *fracs, const int nbudget,
                                                  const int max_rounds, mp_sweep_budget *brec, long long *prof) {
  SweepShared &sh = *shp;
  const int lane = threadIdx.x & 31;
  const int64_t k_ = sh.gsm[0], lmin = sh.gsm[1], l0 = sh.gsm[2], nord = sh.gsm[3], nevt = sh.gsm[4];
  const CandView cv{k_, kp.c.size, kp.c.out_index, kp.c.in_index, kp.name_rank, kp.c.out_t, kp.c.out_ready,
                    kp.c.in_t, kp.c.dout, kp.c.din, kp.c.spans};
  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(&sh.next_budget, 1);
    b = __shfl_sync(FULL_MASK, b, 0);
    if (b >= nbudget) break;
    mp_sweep_budget rb{};
    const int64_t limit = (int64_t)((double)peak * fracs[b]);
    rb.limit_bytes = limit;
    if (limit <= 0) {
      rb.status = MP_E_VALUE;  // check_positive, validation.py:32-34
    } else if (limit < peak && limit < lmin) {
      rb.status = MP_E_LIMIT_UNREACHABLE;  // estimators.py:98-100
      rb.err_aux = lmin;
    } else {
      // select_by_swdoa: the greedy stops at the first planned peak <= limit
      int64_t m = -1;
      for (int64_t j = 0; j <= nord; j++)
        if (f_le_i(kp.peaks[j], limit)) { m = j; break; }
      if (m < 0) {  // only when the greedy ran through every candidate
        rb.status = MP_E_LIMIT_UNREACHABLE;  // autoswap.py:222-224
        rb.err_aux = (int64_t)kp.peaks[nord];
      } else {
        SimScratch S = sh.ba[b].S;
        S.delta = kp.delta;
        const SimTimes T = sh.ba[b].T;
        const int32_t *sel = kp.order;
        long long bytes = 0;
        for (int64_t q = lane; q < m; q += 32) {
          S.ready[q] = cv.out_ready[sel[q]];   // build_schedule, swapsim.py:111-116
          S.deadline[q] = cv.in_t[sel[q]];
          bytes += cv.size[sel[q]];
        }
        bytes = warp_sum(bytes);
        __syncwarp();
        long long c0 = clock64();
        make_schedule(cv, sel, m, S.ready, S.deadline, T.t_so, T.t_eo, T.t_si, T.t_ei, T.eord, S);
        PeakCurve lp{};
        sim_overlay(P, cv, sel, m, l0, T.t_eo, T.t_si, T.eord, kp.ev_t, kp.ev_d, nevt, S, lp);
        long long c1 = clock64();
        Replay<PeakCurve> rep{};
        SimResult res = sim_fixed_point<false>(P, cv, sel, m, limit, 1, max_rounds, l0, S, T, rep);
        if (b == 0 && lane == 0 && prof) {
          prof[12] = c1 - c0;
          prof[13] = clock64() - c1;
          prof[14] = res.rounds;
          prof[15] = m;
        }
        rb.status = res.status;
        rb.nsel = m;
        rb.selected_bytes = bytes;
        if (res.status == MP_OK) {
          rb.rounds = (int32_t)res.rounds;
          rb.overhead_us = res.delay;
          rb.achieved_peak_bytes = rep.cv.peak;
          rb.planned_peak_bytes = lp.peak;
        } else if (res.status == MP_E_SWAP_DEADLOCK) {
          rb.err_index = res.eidx;
          rb.err_aux = res.eaux1;
        }
      }
    }
    if (lane == 0) brec[b] = rb;
    __syncwarp();
  }
}

__device__ void sweep_one(const SweepArgs &a, int64_t t, char *slab, char *fast, size_t fast_bytes,
                          SweepShared &sh) {
  const CtaGroup cta;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const mp_sweep_params &prm = a.prm;
  const int64_t e0 = a.ev_off[t], n = a.ev_off[t + 1] - e0;
  const int64_t nv = a.var_off[t + 1] - a.var_off[t];
  const int32_t *var = a.var + e0;
  const int64_t *t_us = a.t_us + e0;
  int64_t *offs = a.offsets + e0;
  int32_t *corder = a.cand_order + e0;
  mp_sweep_trace R{};
  Arena ar{Bump{fast, 0, fast_bytes, false}, Bump{slab, 0, a.slab_bytes, false}};
  Bump &bump = ar.slow;
  SW_MARK(0);

  // ---- stage kind/size, group events by variable (counts, scan, stable fill) ----
  GroupArrays g;
  g.take(ar, n, nv);
  TimeArrays ta;
  ta.take(bump, n / 2);
  if (bump.over) return sweep_fail(a, t, MP_E_NOMEM, 0, 0, R);
  const uint8_t *kind = g.kind;
  const int64_t *size = g.size;
  if (tid == 0) sh.bad = 0;
  for (int64_t i = tid; i < n; i += SW_THREADS) {
    g.kind[i] = a.kind[e0 + i];
    g.size[i] = a.size[e0 + i];
  }
  for (int64_t v = tid; v <= nv; v += SW_THREADS) g.cnt[v] = 0;
  __syncthreads();
  for (int64_t i = tid; i < n; i += SW_THREADS) {
    int32_t v = var[i];
    if (v < 0 || v >= nv) sh.bad = 1;
    else atomicAdd(&g.cnt[v], 1);
  }
  __syncthreads();
  if (sh.bad) return sweep_fail(a, t, MP_E_VALUE, 0, 0, R);
  grp_excl_scan(cta, g.cnt, g.gstart, nv, sh.sm);
  if (tid == 0) g.gstart[nv] = n;
  for (int64_t v = tid; v < nv; v += SW_THREADS) g.cnt[v] = 0;
  __syncthreads();
  if (warp == 0) {
    for (int64_t b0 = 0; b0 < n; b0 += 32) {
      int64_t i = b0 + lane;
      bool valid = i < n;
      int32_t v = valid ? var[i] : -1 - lane;
      unsigned peers = __match_any_sync(FULL_MASK, v);
      int rank = __popc(peers & lanemask_lt());
      int32_t cur = valid ? g.cnt[v] : 0;
      __syncwarp();
      if (valid) {
        if (rank == 0) g.cnt[v] = cur + __popc(peers);
        g.perm[g.gstart[v] + cur + rank] = (uint32_t)i;
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // ---- validate_trace ----
  if (prm.validate) {
    if (tid == 0) sh.first = NO_VIOLATION;
    __syncthreads();
    for (int64_t pos = tid; pos < n; pos += SW_THREADS) {
      int code = validate_elem_code(kind, size, t_us, nullptr, pos);
      if (code) atomicMin(&sh.first, ((unsigned long long)pos << 4) | (unsigned)code);
    }
    for (int64_t v = tid; v < nv; v += SW_THREADS) {
      unsigned long long f = validate_var_first(kind, g.perm, g.gstart[v], g.gstart[v + 1]);
      if (f != NO_VIOLATION) atomicMin(&sh.first, f);
    }
    __syncthreads();
    unsigned long long f = sh.first;
    if (f != NO_VIOLATION) return sweep_fail(a, t, MP_E_INVARIANT, (int)(f & 15), (int64_t)(f >> 4), R);
  }

  // ---- detect_iteration: smallest p with the last 2p fingerprints equal ----
  // Quick filter first: thread per candidate, a period must match its last
  // min(p, SW_QUICK) pairs; the smallest survivor is checked exactly by the
  // CTA.  Typical traces settle in one round; after a few rejected
  // survivors the warp-per-candidate search below takes over above them.
  int64_t lo_p = 1;
  long long found = LLONG_MAX;
  for (int it = 0; it < 4 && found == LLONG_MAX; it++) {
    if (tid == 0) sh.best_p = LLONG_MAX;
    __syncthreads();
    for (int64_t pp = lo_p + tid; pp <= n / 2; pp += SW_THREADS) {
      const int64_t qq = pp < SW_QUICK ? pp : SW_QUICK;
      bool ok = true;
      for (int64_t k = 1; k <= qq; k++)
        if (kind[n - k] != kind[n - pp - k] || size[n - k] != size[n - pp - k]) { ok = false; break; }
      if (ok) {
        atomicMin(&sh.best_p, (long long)pp);
        break;  // this thread's later candidates are larger
      }
    }
    __syncthreads();
    const long long c = sh.best_p;
    if (c == LLONG_MAX) { lo_p = n / 2 + 1; break; }  // every candidate left fails: no period
    bool good = true;
    for (int64_t i = tid; i < c; i += SW_THREADS)
      good &= kind[n - c + i] == kind[n - 2 * c + i] && size[n - c + i] == size[n - 2 * c + i];
    if (__syncthreads_and(good)) found = c;
    else lo_p = c + 1;
  }
  if (tid == 0) sh.best_p = found;
  __syncthreads();
  for (int64_t p = lo_p + warp; found == LLONG_MAX && p <= n / 2; p += SW_WARPS) {
    long long best = __shfl_sync(FULL_MASK, *(volatile long long *)&sh.best_p, 0);
    if (p >= best) break;
    bool ok = true;
    for (int64_t i0 = 0; i0 < p; i0 += 32) {
      int64_t i = i0 + lane;
      bool eq = i >= p || (kind[n - p + i] == kind[n - 2 * p + i] && size[n - p + i] == size[n - 2 * p + i]);
      if (!__all_sync(FULL_MASK, eq)) { ok = false; break; }
    }
    if (ok) {
      if (lane == 0) atomicMin(&sh.best_p, (long long)p);
      break;
    }
  }
  __syncthreads();
  const int64_t p = sh.best_p;
  if (p == LLONG_MAX) return sweep_fail(a, t, MP_E_PERIOD_NOT_FOUND, 0, n, R);
  R.period = p;
  const int64_t start = n - p, end = n;

  // ---- extract_lifetimes ----
  SW_MARK(1);
  ExtractArrays x;
  x.take(ar, p, nv);
  if (bump.over) return sweep_fail(a, t, MP_E_NOMEM, 0, 0, R);
  const ExScratch &s = x.s;
  if (tid == 0) sh.first = NO_VIOLATION;
  __syncthreads();
  for (int64_t v = tid; v < nv; v += SW_THREADS) {
    unsigned long long f = ex_var_item(kind, size, g.perm, g.gstart, v, start, end, s);
    if (f != NO_VIOLATION) atomicMin(&sh.first, f);
  }
  for (int64_t r = tid; r < p; r += SW_THREADS) s.is_malloc[r] = kind[start + r] == MP_MALLOC;
  __syncthreads();
  for (int64_t v = tid; v < nv; v += SW_THREADS) ex_twin_item(kind, size, v, start, p, s);
  __syncthreads();
  {
    unsigned long long f = sh.first;
    if (f != NO_VIOLATION) return sweep_fail(a, t, MP_E_INVARIANT, (int)(f & 15), (int64_t)(f >> 4), R);
  }
  const int64_t ncarry = grp_excl_scan(cta, s.c_surv, x.carry_ord, nv, sh.sm);
  const int64_t nwin = grp_excl_scan(cta, s.is_malloc, x.win_ord, p, sh.sm);
  const int64_t V = ncarry + nwin;
  R.nvars = V;
  R.ncarry = ncarry;
  ProfileArrays pa;
  pa.take(bump, p, V);
  if (bump.over) return sweep_fail(a, t, MP_E_NOMEM, 0, 0, R);
  int64_t *loads = ta.diff + 1;
  ProfOut o{pa.base, pa.alloc, pa.free_, pa.nseg, pa.seg, pa.acc_index, nullptr, pa.size, pa.acc_off, loads,
            pa.flags, nullptr, pa.acc_next, ta.op_times};
  for (int64_t v = tid; v < nv; v += SW_THREADS) ex_fill_carry_item(v, p, s, x.carry_ord, o, pa.acc_cnt);
  for (int64_t r = tid; r < p; r += SW_THREADS)
    ex_fill_window_item(var, a.size + e0, start, r, p, ncarry, s, x.win_ord, s.c_surv, o, pa.acc_cnt);
  __syncthreads();
  const int64_t naccess = grp_excl_scan(cta, pa.acc_cnt, pa.acc_off, V, sh.sm);
  if (tid == 0) pa.acc_off[V] = naccess;
  R.naccess = naccess;
  __syncthreads();
  for (int64_t v = tid; v < nv; v += SW_THREADS)
    ex_access_item(kind, g.perm, g.gstart, v, start, end, ncarry, s, x.carry_ord, x.win_ord, o);
  for (int64_t r = tid; r < p; r += SW_THREADS) {
    ta.op_times[r] = (double)(t_us[start + r] - t_us[start]);
    ta.diff[r] = 0;
  }
  if (tid == 0) {
    ta.diff[p] = 0;
    sh.dur = ex_duration(t_us, start, end);
  }
  __syncthreads();
  // compute_load_profile, iteration.py:304-320
  for (int64_t i = tid; i < V; i += SW_THREADS)
    for (int q = 0; q < pa.nseg[i]; q++) {
      atomicAdd((unsigned long long *)&ta.diff[pa.seg[4 * i + 2 * q]], (unsigned long long)pa.size[i]);
      atomicAdd((unsigned long long *)&ta.diff[pa.seg[4 * i + 2 * q + 1]], (unsigned long long)(-pa.size[i]));
    }
  __syncthreads();
  grp_excl_scan(cta, ta.diff, ta.diff, p + 1, sh.sm);
  const double dur = sh.dur;
  R.duration_us = dur;
  long long pk = LLONG_MIN;
  for (int64_t r = tid; r < p; r += SW_THREADS) pk = loads[r] > pk ? loads[r] : pk;
  const int64_t peak = grp_max(cta, pk, sh.sm);
  long long pi = LLONG_MAX;
  for (int64_t r = tid; r < p; r += SW_THREADS)
    if (loads[r] == peak && r < pi) pi = r;
  const int64_t peak_index = -grp_max(cta, -pi, sh.sm);
  R.peak_bytes = peak;
  R.peak_index = peak_index;

  // ---- placement order + conflict rows (whole CTA), swap arrays ----
  SW_MARK(2);
  ar.phase();
  SwapKeep kp;
  kp.take(ar, p, V);
  kp.take_events(bump, p);
  PlaceArrays pl;
  pl.take(ar, V);
  // the budgets refill the arena from here once the greedy's arrays are dead
  const size_t keep_top = ar.fast.top;
  const size_t keep_slow = ar.slow.top;
  GreedyArrays gr;
  gr.take(ar, p, V);
  SwapScratch ss;
  ss.take(ar, p, V);
  if (bump.over) return sweep_fail(a, t, MP_E_NOMEM, 0, 0, R);
  for (int64_t i = tid; i < V; i += SW_THREADS) {
    pl.ksize[i] = pa.size[i];
    pl.kalloc[i] = pa.alloc[i];
    pl.kbase[i] = pa.base[i];
  }
  for (int64_t i = tid; i < pl.n2; i += SW_THREADS) pl.order[i] = i < V ? (int32_t)i : -1;
  __syncthreads();
  for (int64_t k = 2; k <= pl.n2; k <<= 1)
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = tid; i < pl.n2; i += SW_THREADS) {
        int64_t ixj = i ^ j;
        if (ixj > i) {
          int32_t xa = pl.order[i], xb = pl.order[ixj];
          bool up = (i & k) == 0;
          if (up ? place_less(pl, xb, xa) : place_less(pl, xa, xb)) { pl.order[i] = xb; pl.order[ixj] = xa; }
        }
      }
      __syncthreads();
    }
  // rank space: segments (a one-segment variable's second is the empty
  // [0, 0), which overlaps nothing) and sizes in placement order
  for (int64_t q = tid; q < V; q += SW_THREADS) {
    int32_t u = pl.order[q];
    bool two = pa.nseg[u] > 1;
    pl.rseg[q] = make_int4(pa.seg[4 * u], pa.seg[4 * u + 1], two ? pa.seg[4 * u + 2] : 0, two ? pa.seg[4 * u + 3] : 0);
    pl.rsize[q] = pl.ksize[u];
  }
  __syncthreads();
  // conflict rows (conflict_graph_from_arcs, smartpool.py:51-79): an edge
  // iff some pair of half-open segments overlaps, max(lo) < min(hi)
  for (int64_t idx = tid; idx < V * pl.words; idx += SW_THREADS) {
    int64_t q = idx / pl.words, w0 = (idx % pl.words) * 32;
    uint32_t bits = 0;
    if (w0 < q) {
      const int4 u = pl.rseg[q];
      int64_t jn = q - w0 < 32 ? q - w0 : 32;
      for (int b = 0; b < jn; b++) {
        const int4 v = pl.rseg[w0 + b];
        bool hit = max(u.x, v.x) < min(u.y, v.y) || max(u.x, v.z) < min(u.y, v.w) ||
                   max(u.z, v.x) < min(u.w, v.y) || max(u.z, v.z) < min(u.w, v.w);
        bits |= (uint32_t)hit << b;
      }
    }
    pl.adj[idx] = bits;
  }
  if (tid == 0) {
    sh.next_budget = 0;
    sh.swap_ready = 0;
    sh.nomem = 0;
  }
  __syncthreads();

  const LoadView L{p, loads, kp.tau, dur};
  const ProfView P{p, V, start, dur, kp.tau, pa.nseg, pa.seg, pa.size};
  // SwapPlanner(limit, score="swdoa").fit for budgets pulled from a shared
  // counter, one warp each
  auto run_budgets = [&]() {
    sweep_budgets(&sh, kp, P, peak, a.prm.budget_frac, prm.nbudget, prm.max_rounds, a.brec + t * prm.nbudget,
                  a.prof ? a.prof + t * 16 : nullptr);
  };

  int64_t k = 0, load_min = 0, live0 = 0, na = 0, norder = 0;
  if (warp == 0) {
    // ---- plan_pool (smartpool.py:122-144), concurrently with the swap path ----
    // One warp walks the order.  All placed ranges are kept in one list
    // sorted by start; a step scans it with its conflict row as the validity
    // mask, so the placed neighbours arrive already sorted and _pick_offset
    // (smartpool.py:101-119) is one pass over it — then the new range
    // is inserted in order.
    int64_t edges = 0;
    int64_t *const ls = pl.ls, *const le = pl.le;
    int32_t *const lr = pl.lr;
    long long c_scan = 0, c_ins = 0, c_t0 = clock64();
    for (int64_t q = 0; q < V; q++) {
      const uint32_t *row = pl.adj + q * pl.words;
      long long c_a = clock64();
      const int64_t need = pl.rsize[q];
      for (int64_t w = lane; w * 32 < q; w += 32) edges += __popc(row[w]);
      // _pick_offset over the list, PL_K consecutive entries per lane: a hole
      // opens where a start exceeds the running max of earlier ends
      int64_t top = 0, ff_off = 0;
      bool ff_found = false;
      int64_t bl = INT64_MAX, bo = INT64_MAX;  // this lane's best fit (length, offset)
      for (int64_t c0 = 0; c0 < q && !ff_found; c0 += 32 * PL_K) {
        int64_t st[PL_K], en[PL_K];
        bool valid[PL_K];
        int64_t lmax = INT64_MIN;
#pragma unroll
        for (int jj = 0; jj < PL_K; jj++) {
          int64_t i = c0 + lane * PL_K + jj;
          valid[jj] = false;
          st[jj] = en[jj] = 0;
          if (i < q) {
            int32_t j = lr[i];
            valid[jj] = (row[j >> 5] >> (j & 31)) & 1u;
            st[jj] = ls[i];
            en[jj] = le[i];
            if (valid[jj] && en[jj] > lmax) lmax = en[jj];
          }
        }
        int64_t incl = warp_incl_scan_max(lmax);
        int64_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
        int64_t run = lane == 0 || excl < top ? top : excl;
        bool mine = false;
        int64_t my_off = 0;
#pragma unroll
        for (int jj = 0; jj < PL_K; jj++) {
          if (!valid[jj]) continue;
          if (st[jj] > run && st[jj] - run >= need) {
            int64_t len = st[jj] - run;
            if (!mine) { mine = true; my_off = run; }
            if (len < bl || (len == bl && run < bo)) { bl = len; bo = run; }
          }
          if (en[jj] > run) run = en[jj];
        }
        if (prm.policy == 0) {
          unsigned bal = __ballot_sync(FULL_MASK, mine);
          if (bal) {
            ff_off = __shfl_sync(FULL_MASK, my_off, __ffs(bal) - 1);
            ff_found = true;
          }
        }
        int64_t cmax = __shfl_sync(FULL_MASK, incl, 31);
        if (cmax > top) top = cmax;
      }
      int64_t off;
      if (prm.policy == 0) {
        off = ff_found ? ff_off : top;
      } else {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          int64_t ol = __shfl_xor_sync(FULL_MASK, bl, o), oo = __shfl_xor_sync(FULL_MASK, bo, o);
          if (ol < bl || (ol == bl && oo < bo)) { bl = ol; bo = oo; }
        }
        off = bl != INT64_MAX ? bo : top;
      }
      long long c_b = clock64();
      c_scan += c_b - c_a;
      // insert (off, off + need, q) before the first range starting at or after off
      int64_t pos = 0;
      for (int64_t c0 = 0; c0 < q; c0 += 32) {
        int64_t i = c0 + lane;
        pos += __popc(__ballot_sync(FULL_MASK, i < q && ls[i] < off));
      }
      // shift [pos, q) up by one in place, highest chunk first
      for (int64_t c1 = q; c1 > pos; c1 -= 32) {
        const int64_t i = c1 - 32 + lane;
        const bool mv = i >= pos;
        int64_t vs = 0, ve = 0;
        int32_t vr = 0;
        if (mv) { vs = ls[i]; ve = le[i]; vr = lr[i]; }
        __syncwarp();
        if (mv) { ls[i + 1] = vs; le[i + 1] = ve; lr[i + 1] = vr; }
        __syncwarp();
      }
      if (lane == 0) { ls[pos] = off; le[pos] = off + need; lr[pos] = (int32_t)q; }
      __syncwarp();
      c_ins += clock64() - c_b;
    }
    if (lane == 0 && a.prof) { a.prof[t * 16 + 8] = c_t0; a.prof[t * 16 + 9] = clock64(); a.prof[t * 16 + 10] = c_scan; a.prof[t * 16 + 11] = c_ins; }
    edges = warp_sum(edges);
    // scatter offsets back to profile order
    for (int64_t i = lane; i < V; i += 32) offs[pl.order[lr[i]]] = ls[i];
    if (lane == 0) sh.edges = edges;
    // then help with the budgets the swap path has not claimed yet
    if (lane == 0)
      while (!*(volatile int *)&sh.swap_ready) __nanosleep(64);
    __syncwarp();
    __threadfence_block();
    if (!*(volatile int *)&sh.nomem) run_budgets();
  } else {
    // ---- AutoSwap on warps 1..: candidates, load_min, SWDOA greedy ----
    const WarpGroup sg{1, SW_WARPS - 1, 1};
    const int gi = sg.idx(), gn = sg.size();
    for (int64_t v = gi; v < V; v += gn)
      ss.flag[v] = cand_item(v, v, p, peak_index, pa.size, pa.flags, pa.acc_off, pa.acc_index, pa.acc_next,
                             ta.op_times, dur, prm.threshold, prm.bw, prm.lat, ss.tmp);
    for (int64_t r = gi; r < p; r += gn) {
      kp.tau[r] = ta.op_times[r];
      kp.delta[r] = 0;
    }
    sg.sync();
    k = grp_excl_scan(sg, ss.flag, ss.pos, V, sh.gsm);
    CandOut &cc = kp.c;
    for (int64_t v = gi; v < V; v += gn) {
      if (!ss.flag[v]) continue;
      int64_t q = ss.pos[v];
      cc.var[q] = ss.tmp.var[v]; cc.out_index[q] = ss.tmp.out_index[v]; cc.in_index[q] = ss.tmp.in_index[v];
      cc.size[q] = ss.tmp.size[v]; cc.out_t[q] = ss.tmp.out_t[v]; cc.out_ready[q] = ss.tmp.out_ready[v];
      cc.in_t[q] = ss.tmp.in_t[v]; cc.dout[q] = ss.tmp.dout[v]; cc.din[q] = ss.tmp.din[v];
      cc.spans[q] = ss.tmp.spans[v];
      // the candidate's final name: base id, "#alloc" suffix when renamed
      ss.cbase[q] = pa.base[v];
      ss.cralloc[q] = (pa.flags[v] & MP_F_RENAMED) ? pa.alloc[v] : -1;
    }
    sg.sync();
    NameTable names{a.blob, a.name_off + a.var_off[t]};
    for (int64_t i = gi; i < k; i += gn) {
      const int32_t bi = ss.cbase[i], ri = ss.cralloc[i];
      int32_t rank = 0;
      for (int64_t j = 0; j < k; j++) rank += name_cmp(names, ss.cbase[j], ss.cralloc[j], bi, ri) < 0;
      kp.name_rank[i] = rank;
    }
    sg.sync();
    const CandView cv{k, cc.size, cc.out_index, cc.in_index, kp.name_rank, cc.out_t, cc.out_ready,
                      cc.in_t, cc.dout, cc.din, cc.spans};
    // compute_load_min (swapsim.py:398-405): every candidate absent.  While
    // every load and size sum is an integer below 2^53 the reference's float
    // subtractions are exact, so a difference array over the absence ranges
    // gives the same values; otherwise the slot-parallel fold runs.
    long long szsum = 0;
    bool short_gaps = true;
    for (int64_t q = gi; q < k; q += gn) {
      szsum += cv.size[q];
      short_gaps &= cv.in_index[q] + (cv.spans[q] ? p : 0) - cv.out_index[q] - 1 <= p;
    }
    for (int64_t r = gi; r <= p; r += gn) ss.lmdiff[r] = 0;
    szsum = grp_sum(sg, szsum, sh.gsm);
    const bool lm_fast = sg.sync_and(short_gaps) && (double)peak < EXACT_2_53 && (double)szsum < EXACT_2_53;
    double lm = -INF_D;
    if (lm_fast) {
      for (int64_t q = gi; q < k; q += gn) {
        int64_t lo = cv.out_index[q] + 1, hi = cv.in_index[q] + (cv.spans[q] ? p : 0);  // slots [lo, hi)
        unsigned long long neg = (unsigned long long)(-cv.size[q]), pos = (unsigned long long)cv.size[q];
        if (lo >= hi) continue;
        if (hi <= p) {
          atomicAdd((unsigned long long *)&ss.lmdiff[lo], neg);
          atomicAdd((unsigned long long *)&ss.lmdiff[hi], pos);
        } else {
          if (lo < p) {
            atomicAdd((unsigned long long *)&ss.lmdiff[lo], neg);
            atomicAdd((unsigned long long *)&ss.lmdiff[p], pos);
            lo = p;
          }
          atomicAdd((unsigned long long *)&ss.lmdiff[lo - p], neg);
          atomicAdd((unsigned long long *)&ss.lmdiff[hi - p], pos);
        }
      }
      sg.sync();
      grp_excl_scan(sg, ss.lmdiff, ss.lmdiff, p + 1, sh.gsm);
      // diff[r+1] after the exclusive scan = sum of diff[0..r]
      for (int64_t r = gi; r < p; r += gn) {
        double cur = (double)(loads[r] + ss.lmdiff[r + 1]);
        lm = r == gi ? cur : pymax(lm, cur);
      }
    } else {
      for (int64_t r = gi; r < p; r += gn) {
        double cur = (double)loads[r];
        for (int64_t q = 0; q < k; q++) {
          int64_t lo = cv.out_index[q], hi = cv.in_index[q] + (cv.spans[q] ? p : 0);
          int h = absence_hits(r, lo, hi, p);
          for (int z = 0; z < h; z++) cur -= (double)cv.size[q];
        }
        lm = r == gi ? cur : pymax(lm, cur);
      }
    }
    load_min = (int64_t)block_max(sg, lm, sh.red);
    // the smallest limit the greedy must reach: a budget below load_min (and
    // below the peak) is rejected by SwapPlanner.fit before selecting
    // (estimators.py:98-100), so every other budget is decided by the
    // greedy prefix up to it
    int64_t stop = INT64_MAX;
    bool need = false;
    for (int b = 0; b < prm.nbudget; b++) {
      const int64_t limit = (int64_t)((double)peak * prm.budget_frac[b]);
      if (limit <= 0 || (limit < peak && limit < load_min)) continue;
      need = true;
      stop = limit < stop ? limit : stop;
    }
    if (gi == 0 && a.prof) a.prof[t * 16 + 3] = clock64();
    norder = need ? swdoa_greedy_block(sg, L, cv, gr.cur, gr.taken, nullptr, nullptr, nullptr, nullptr, kp.order,
                                       kp.peaks, gr.W, gr.jx, sh.keys, sh.gsm, stop, gr.area)
                  : 0;
    if (gi == 0 && a.prof) a.prof[t * 16 + 4] = clock64();
    for (int64_t q = gi; q < norder; q += gn) corder[q] = cc.var[kp.order[q]];
    // ---- simulate prerequisites: _op_deltas and the sorted op events ----
    long long l0 = 0;
    for (int64_t i = gi; i < V; i += gn)
      for (int q = 0; q < pa.nseg[i]; q++) {
        int64_t lo = pa.seg[4 * i + 2 * q], hi = pa.seg[4 * i + 2 * q + 1];
        if (lo == 0) l0 += pa.size[i];
        else atomicAdd((unsigned long long *)&kp.delta[lo], (unsigned long long)pa.size[i]);
        if (hi < p) atomicAdd((unsigned long long *)&kp.delta[hi], (unsigned long long)(-pa.size[i]));
      }
    live0 = grp_sum(sg, l0, sh.gsm);
    // _overlay_curve's op events (t, delta != 0), swapsim.py:184-193: compacted
    // in op order, which is (t, delta) order unless equal times run backwards
    for (int64_t r = gi; r < p; r += gn) ss.evpos[r] = kp.delta[r] != 0;
    sg.sync();
    na = grp_excl_scan(sg, ss.evpos, ss.evpos, p, sh.gsm);
    for (int64_t r = gi; r < p; r += gn)
      if (kp.delta[r] != 0) {
        kp.ev_t[ss.evpos[r]] = kp.tau[r];
        kp.ev_d[ss.evpos[r]] = kp.delta[r];
      }
    sg.sync();
    bool sorted = true;
    for (int64_t q = gi; q + 1 < na; q += gn) sorted &= !td_less(kp.ev_t[q + 1], kp.ev_d[q + 1], kp.ev_t[q], kp.ev_d[q]);
    if (!sg.sync_and(sorted) && gi == 0) sim_op_events(P, kp.delta, kp.ev_t, kp.ev_d);
    // publish the scalars, lay out each budget's scratch (sized by its
    // selection) over the now-dead greedy arrays, then start the budgets
    if (gi == 0) {
      sh.gsm[0] = k;
      sh.gsm[1] = load_min;
      sh.gsm[2] = live0;
      sh.gsm[3] = norder;
      sh.gsm[4] = na;
      Arena bar = ar;
      bar.fast.top = keep_top;
      bar.slow.top = keep_slow;
      for (int b = 0; b < prm.nbudget; b++) {
        const int64_t limit = (int64_t)((double)peak * prm.budget_frac[b]);
        int64_t m = 0;
        if (limit > 0 && !(limit < peak && limit < load_min))
          while (m < norder && !f_le_i(kp.peaks[m], limit)) m++;
        sh.ba[b].take(bar, p, m);
      }
      sh.nomem = bar.slow.over;
      if (a.prof) a.prof[t * 16 + 5] = clock64();
    }
    sg.sync();
    if (gi == 0) {
      __threadfence_block();
      *(volatile int *)&sh.swap_ready = 1;
    }
    if (!sh.nomem) run_budgets();
  }
  __syncthreads();
  if (sh.nomem) return sweep_fail(a, t, MP_E_NOMEM, 0, 0, R);
  R.edges = sh.edges;
  R.ncand = sh.gsm[0];
  R.load_min = sh.gsm[1];
  R.norder = sh.gsm[3];
  long long fe = LLONG_MIN;
  for (int64_t i = tid; i < V; i += SW_THREADS) {
    long long e = offs[i] + pa.size[i];
    fe = e > fe ? e : fe;
  }
  const int64_t foot = grp_max(cta, fe, sh.sm);
  R.footprint_bytes = V ? foot : 0;
  SW_MARK(6);
  __syncwarp();
  __syncthreads();
  SW_MARK(7);
  if (tid == 0) {
    R.status = MP_OK;
    a.rec[t] = R;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SW_THREADS) k_sweep(SweepArgs a, size_t fast_bytes) {
  PDL_WAIT();
  __shared__ SweepShared sh;
  __shared__ int32_t s_item;
  extern __shared__ __align__(16) char s_fast[];
  char *slab = a.slab + (size_t)blockIdx.x * a.slab_bytes;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    int32_t item = s_item;
    __syncthreads();
    if (item >= a.T) break;
    sweep_one(a, a.work[item], slab, s_fast, fast_bytes, sh);
  }
}

// ---------------------------------------------------------------------------
// host side

struct mp_dsweep {
  mp_ctx *ctx = nullptr;
  int64_t T = 0, N = 0, NV = 0, nmax = 0, nvmax = 0;
  DBuf<int64_t> ev_off, var_off, name_off, size, t_us, offsets;
  DBuf<uint8_t> kind, blob;
  DBuf<int32_t> var, work, cand_order, counter;
  DBuf<mp_sweep_trace> rec;
  DBuf<mp_sweep_budget> brec;
  int32_t nbudget = 0;
  DBuf<char> slab;
  size_t slab_bytes = 0;
  int64_t nblocks = 0;
  DBuf<long long> prof;  // mp_sweep_set_profile
};

extern "C" int mp_sweep_upload(mp_ctx *ctx, const mp_sweep_in *in, mp_dsweep **out, mp_err *err) {
  CTX_GUARD(ctx);
  StageTimer tm(ctx, MP_ST_SWEEP);
  cudaStream_t st = ctx->stream;
  int64_t T = in->ntraces;
  if (T < 0 || (T && (!in->ev_off || !in->var_off))) {
    mp_set_err(err, MP_E_VALUE, 0, T, 0, "bad sweep batch");
    return MP_E_VALUE;
  }
  mp_dsweep *s = new mp_dsweep();
  s->ctx = ctx;
  s->T = T;
  s->N = T ? in->ev_off[T] : 0;
  s->NV = T ? in->var_off[T] : 0;
  std::vector<int32_t> work((size_t)T);
  for (int64_t t = 0; t < T; t++) {
    int64_t n = in->ev_off[t + 1] - in->ev_off[t], nv = in->var_off[t + 1] - in->var_off[t];
    if (n < 0 || nv < 0 || n > INT32_MAX) {
      delete s;
      mp_set_err(err, MP_E_VALUE, t, n, nv, "bad sweep batch");
      return MP_E_VALUE;
    }
    s->nmax = n > s->nmax ? n : s->nmax;
    s->nvmax = nv > s->nvmax ? nv : s->nvmax;
    work[(size_t)t] = (int32_t)t;
  }
  // largest traces first: the work counter then behaves like LPT
  std::stable_sort(work.begin(), work.end(), [&](int32_t x, int32_t y) {
    return in->ev_off[x + 1] - in->ev_off[x] > in->ev_off[y + 1] - in->ev_off[y];
  });
  int64_t N = s->N, NV = s->NV, nb = in->name_off ? in->name_off[NV] : 0;
  int rc = MP_OK;
  auto up = [&](auto &buf, const auto *src, int64_t cnt) -> cudaError_t {
    cudaError_t e = buf.alloc(cnt, st);
    if (e == cudaSuccess && cnt && src) e = cudaMemcpyAsync(buf.p, src, cnt * sizeof(*src), cudaMemcpyHostToDevice, st);
    return e;
  };
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = up(s->ev_off, in->ev_off, T + 1);
  if (e == cudaSuccess) e = up(s->var_off, in->var_off, T + 1);
  if (e == cudaSuccess) e = up(s->name_off, in->name_off, NV + 1);
  if (e == cudaSuccess) e = up(s->blob, in->name_blob, nb);
  if (e == cudaSuccess) e = up(s->kind, in->kind, N);
  if (e == cudaSuccess) e = up(s->var, in->var, N);
  if (e == cudaSuccess) e = up(s->size, in->size, N);
  if (e == cudaSuccess) e = up(s->t_us, in->t_us, N);
  if (e == cudaSuccess) e = up(s->work, work.data(), T);
  if (e == cudaSuccess) e = s->offsets.alloc(N, st);
  if (e == cudaSuccess) e = s->cand_order.alloc(N, st);
  // rows past a trace's variable / candidate count stay zero
  if (e == cudaSuccess && N) e = cudaMemsetAsync(s->offsets.p, 0, N * 8, st);
  if (e == cudaSuccess && N) e = cudaMemsetAsync(s->cand_order.p, 0, N * 4, st);
  if (e == cudaSuccess) e = s->rec.alloc(T, st);
  if (e == cudaSuccess) e = s->counter.alloc(1, st);
  // host staging (work) must outlive the async copy
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    delete s;
    mp_set_err(err, MP_E_CUDA, 0, (int64_t)e, __LINE__, cudaGetErrorString(e));
    return MP_E_CUDA;
  }
  (void)rc;
  *out = s;
  return MP_OK;
}

extern "C" int mp_sweep_free(mp_dsweep *s) {
  CTX_GUARD(s->ctx);
  delete s;
  return MP_OK;
}

extern "C" int mp_sweep_run(mp_ctx *ctx, mp_dsweep *s, const mp_sweep_params *prm, mp_err *err) {
  CTX_GUARD(ctx);
  StageTimer tm(ctx, MP_ST_SWEEP);
  cudaStream_t st = ctx->stream;
  if (prm->nbudget < 0 || prm->nbudget > MP_SWEEP_MAX_BUDGETS || (prm->policy != 0 && prm->policy != 1)) {
    mp_set_err(err, MP_E_VALUE, 0, prm->nbudget, prm->policy, "bad sweep parameters");
    return MP_E_VALUE;
  }
  if (s->T == 0) return MP_OK;
  if (s->nbudget != prm->nbudget || !s->brec.p) {
    CUDA_TRY(s->brec.alloc(s->T * (prm->nbudget > 0 ? prm->nbudget : 1), st));
    s->nbudget = prm->nbudget;
  }
  const size_t fast_bytes = SW_FAST_BYTES;
  CUDA_TRY(cudaFuncSetAttribute(k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_bytes));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep, SW_THREADS, fast_bytes));
  if (per_sm < 1) per_sm = 1;
  int64_t nblocks = (int64_t)ctx->num_sms * per_sm;
  if (nblocks > s->T) nblocks = s->T;
  size_t need = slab_bound(s->nmax, s->nvmax, prm->nbudget);
  if (need * (size_t)nblocks > (size_t)s->slab.n || nblocks > s->nblocks) {
    CUDA_TRY(s->slab.alloc((int64_t)(need * (size_t)nblocks), st));
    s->slab_bytes = need;
    s->nblocks = nblocks;
  } else {
    s->slab_bytes = (size_t)s->slab.n / (size_t)nblocks;
  }
  CUDA_TRY(cudaMemsetAsync(s->counter.p, 0, 4, st));
  SweepArgs a{s->T, s->ev_off.p, s->var_off.p, s->name_off.p, s->kind.p, s->blob.p, s->var.p, s->size.p,
              s->t_us.p, s->work.p, s->counter.p, *prm, s->rec.p, s->brec.p, s->offsets.p, s->cand_order.p,
              s->slab.p, s->slab_bytes, s->prof.p};
  LAUNCH(ctx, k_sweep, (unsigned)nblocks, SW_THREADS, fast_bytes, a, fast_bytes);
  return MP_OK;
}

extern "C" int mp_sweep_download(mp_ctx *ctx, mp_dsweep *s, mp_sweep_trace *traces, mp_sweep_budget *budgets,
                                 int64_t *offsets, int32_t *cand_order, mp_err *err) {
  CTX_GUARD(ctx);
  StageTimer tm(ctx, MP_ST_SWEEP);
  cudaStream_t st = ctx->stream;
  if (traces && s->T) CUDA_TRY(cudaMemcpyAsync(traces, s->rec.p, s->T * sizeof(mp_sweep_trace), cudaMemcpyDeviceToHost, st));
  if (budgets && s->T && s->nbudget)
    CUDA_TRY(cudaMemcpyAsync(budgets, s->brec.p, s->T * s->nbudget * sizeof(mp_sweep_budget), cudaMemcpyDeviceToHost, st));
  if (offsets && s->N) CUDA_TRY(cudaMemcpyAsync(offsets, s->offsets.p, s->N * 8, cudaMemcpyDeviceToHost, st));
  if (cand_order && s->N) CUDA_TRY(cudaMemcpyAsync(cand_order, s->cand_order.p, s->N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

extern "C" int mp_sweep_set_profile(mp_ctx *ctx, mp_dsweep *s, int on, mp_err *err) {
  CTX_GUARD(ctx);
  if (!on) { s->prof.release(); return MP_OK; }
  CUDA_TRY(s->prof.alloc(s->T * 16 > 0 ? s->T * 16 : 1, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(s->prof.p, 0, (s->T * 16 > 0 ? s->T * 16 : 1) * 8, ctx->stream));
  return MP_OK;
}

extern "C" int mp_sweep_profile_download(mp_ctx *ctx, mp_dsweep *s, long long *out, mp_err *err) {
  CTX_GUARD(ctx);
  if (!s->prof.p) { mp_set_err(err, MP_E_VALUE, 0, 0, 0, "profiling is off"); return MP_E_VALUE; }
  CUDA_TRY(cudaMemcpyAsync(out, s->prof.p, s->T * 16 * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MP_OK;
}
