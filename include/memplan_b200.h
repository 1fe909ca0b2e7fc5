/*
 * memplan_b200.h — C ABI of the B200-native memplan hot path.
 *
 * The drop-in boundary: the reference exposes this path as Python
 * functions of the `memplan` package (pkg/src/memplan/__init__.py:92-166).
 * Each entry point below replaces one of them; the Python package
 * `paper_1903_06631_b200` binds these symbols with ctypes and re-exposes
 * the reference's names, dataclasses and exceptions.
 *
 * Conventions
 *   - every call returns an int32 status: 0 = MP_OK, otherwise an MP_E_*
 *     code; details land in the caller's mp_err (may be NULL).
 *   - inputs are caller-owned, C-contiguous host arrays borrowed for the
 *     call; results go to caller-allocated host arrays sized from the
 *     *_dims queries, or stay device-resident behind an opaque handle.
 *   - variable ids are dense int32 ranks of the variable-name strings in
 *     lexicographic order; the UTF-8 names (blob + offsets) travel with the
 *     trace so renamed instances ("base#alloc", iteration.py:236-241) can be
 *     ordered exactly on the device.
 *   - all floating point is IEEE binary64 with no contraction (-fmad=false)
 *     and the reference's left-fold order, so results are bit-identical.
 *   - kind codes: 0 malloc, 1 free, 2 read, 3 write (trace.py:24-28).
 *   - threads: the reference's functions are reentrant.
 *     Every entry point that takes a context, or a handle (bound to the
 *     context that created it), holds that context's mutex for the call, so
 *     calls from several host threads on one context serialize and never
 *     share scratch; for parallel device work use one context per thread.
 *   - the plan-serving allocator and swap-copy hooks are declared in
 *     memplan_alloc.h (libmemplan_alloc.so).
 */
#ifndef MEMPLAN_B200_H
#define MEMPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_MALLOC 0
#define MP_FREE 1
#define MP_READ 2
#define MP_WRITE 3

/* status codes; mapping to the reference exceptions in errors.py */
enum {
  MP_OK = 0,
  MP_E_INVARIANT = 1,        /* InvariantViolation(index, reason)   errors.py:20 */
  MP_E_PERIOD_NOT_FOUND = 2, /* PeriodNotFound                      errors.py:36 */
  MP_E_LIMIT_UNREACHABLE = 3,/* LimitUnreachable(limit, achievable) errors.py:48 */
  MP_E_SWAP_DEADLOCK = 4,    /* SwapDeadlock(index, reason)         errors.py:62 */
  MP_E_SIM_INDEXERROR = 5,   /* reference defect swapsim.py:266-276 raises IndexError */
  MP_E_VALUE = 6,            /* ValueError (bad window / policy / score)          */
  MP_E_CUDA = 7,             /* CUDA runtime failure (no silent fallback)         */
  MP_E_NOMEM = 8,
  MP_E_UNSUPPORTED = 9
};

/* InvariantViolation reason codes (mp_err.aux0); reason text is formatted
 * by the host with the variable name in aux1 (a var id). */
enum {
  MP_V_INDEX = 1,        /* "index {index} not contiguous"   trace.py:64-65 (aux1 = bad index) */
  MP_V_NEG_T = 2,        /* "negative timestamp"              trace.py:66-67 */
  MP_V_T_DEC = 3,        /* "timestamp decreases"             trace.py:68-69 */
  MP_V_MALLOC_SIZE = 4,  /* "malloc size must be > 0"         trace.py:72-73 */
  MP_V_MALLOC_LIVE = 5,  /* "malloc of live id {var!r}"       trace.py:74-75 */
  MP_V_SIZE_NONZERO = 6, /* "{kind} size must be 0"           trace.py:78-79 (aux1 = kind) */
  MP_V_FREE_DEAD = 7,    /* "free of dead id {var!r}"         trace.py:80-82 */
  MP_V_USE_DEAD = 8,     /* "use of dead id {var!r}"          trace.py:80-82 */
  MP_V_W_MALLOC_LIVE = 9,/* "malloc of live id {base!r} in window" iteration.py:161-162 */
  MP_V_W_FREE_DEAD = 10, /* "free of dead id {base!r} in window"   iteration.py:177-178 */
  MP_V_W_USE_DEAD = 11   /* "use of dead id {base!r} in window"    iteration.py:184-185 */
};

typedef struct mp_err {
  int32_t code;
  int32_t trace; /* batch member the error belongs to */
  int64_t index;
  int64_t aux0;
  int64_t aux1;
  char msg[192];
} mp_err;

/* One trace in struct-of-arrays form (host memory). */
typedef struct mp_trace_in {
  int64_t n;
  const uint8_t *kind;
  const int32_t *var;
  const int64_t *size;
  const int64_t *t_us;
  const int64_t *index;     /* NULL when index == position */
  int32_t nvars;
  const uint8_t *name_blob; /* names of var ids, concatenated UTF-8 */
  const int64_t *name_off;  /* nvars + 1 offsets into name_blob */
} mp_trace_in;

/* Iteration profile (iteration.py:63-90) in flat form.  Variables are in
 * the reference order (alloc or -1, name) (iteration.py:257-260): the
 * `ncarry` carry-ins first, then window instances by alloc index. */
typedef struct mp_profile_dims {
  int64_t period, nvars, ncarry, naccess;
  int64_t peak_bytes, peak_index;
  double duration_us;
} mp_profile_dims;

#define MP_F_PERSISTENT 1
#define MP_F_WRAPS 2
#define MP_F_RENAMED 4 /* name is "base#alloc" */

typedef struct mp_profile_out {
  /* per variable [nvars] */
  int32_t *base;    /* var id of base_var */
  int64_t *size;
  int32_t *alloc;   /* -1 = None */
  int32_t *free_;   /* -1 = None */
  int32_t *nseg;    /* 1 or 2 */
  int32_t *seg;     /* [nvars][4] = lo0, hi0, lo1, hi1 */
  uint8_t *flags;   /* MP_F_* */
  int64_t *acc_off; /* [nvars + 1] */
  /* per access [naccess] */
  int32_t *acc_index;
  uint8_t *acc_kind;
  uint8_t *acc_next;
  /* per op [period] */
  double *op_times;
  int64_t *loads;
  int32_t *op_owner; /* variable index that op r resolved to */
} mp_profile_out;

/* ---------------------------------------------------------------------- */
/* device context                                                           */

typedef struct mp_ctx mp_ctx;
typedef struct mp_dtrace mp_dtrace;     /* device-resident trace  */
typedef struct mp_dprofile mp_dprofile; /* device-resident profile */
typedef struct mp_dgraph mp_dgraph;     /* device-resident CSR conflict graph */

int mp_version(void);
int mp_ctx_create(int device, mp_ctx **out, mp_err *err);
int mp_ctx_destroy(mp_ctx *ctx);
/* launches of this library's kernels since creation (bench evidence) */
int64_t mp_ctx_launches(mp_ctx *ctx);
int mp_ctx_sync(mp_ctx *ctx, mp_err *err);
/* stream the context launches on (cudaStream_t as void*) */
void *mp_ctx_stream(mp_ctx *ctx);

/* per-stage device time, measured with CUDA events recorded on the
 * context stream around each stage while timing is on */
enum {
  MP_ST_GROUP_SORT = 0, /* radix sort of events by variable */
  MP_ST_VALIDATE,       /* validate_trace kernels */
  MP_ST_DETECT,         /* period hashes + candidates + verify */
  MP_ST_EXTRACT,        /* per-variable state machines, twins, records */
  MP_ST_LOADS,          /* diff scatter + scan + peak */
  MP_ST_CONFLICT_PREP,  /* interval normalization, sorts, counts */
  MP_ST_CONFLICT_FILL,  /* CSR fill */
  MP_ST_PLACE_ORDER,    /* placement-order sort */
  MP_ST_PLACE_SPLIT,    /* row partition into preds / succs */
  MP_ST_PLACE,          /* wavefront placement kernel */
  MP_ST_FOOTPRINT,
  MP_ST_SWAP,           /* swap planning kernels */
  MP_ST_SWEEP,          /* batched sweep: upload, one-CTA-per-trace kernel, download */
  MP_NSTAGES = 16
};
int mp_ctx_set_timing(mp_ctx *ctx, int on);
/* accumulated ms and event-pair counts per stage since the last call */
int mp_ctx_timings(mp_ctx *ctx, double *ms, int64_t *count, mp_err *err);

/* validate_trace (trace.py:55-84) + upload.  Replaces
 * memplan.trace.validate_trace; the first violation is reported exactly as
 * the sequential reference would. */
int mp_trace_upload(mp_ctx *ctx, const mp_trace_in *in, mp_dtrace **out, mp_err *err);
/* the same upload without a host wait: the columns go up on a copy stream
 * (var, kind, size, index, t_us) and each stage waits only for the columns it
 * reads, so grouping and period detection overlap the rest of the transfer.
 * The input buffers stay borrowed until mp_trace_wait returns. */
int mp_trace_upload_async(mp_ctx *ctx, const mp_trace_in *in, mp_dtrace **out, mp_err *err);
/* the timestamp column of an asynchronous upload is sent only here (or when a
 * stage first needs it): call it before the placement, whose kernel a
 * concurrent host-to-device copy barely slows, unlike the readback-bound
 * stages before it.  Op times of profiles extracted meanwhile follow it. */
int mp_trace_flush(mp_dtrace *t, mp_err *err);
int mp_trace_wait(mp_dtrace *t, mp_err *err);
int mp_trace_free(mp_dtrace *t);
/* drop cached derived state (event grouping) so the next stage recomputes it */
int mp_trace_reset(mp_dtrace *t);
int mp_validate(mp_ctx *ctx, mp_dtrace *t, mp_err *err);
/* mp_validate in two passes, for a trace whose timestamps are still
 * uploading: mp_validate_structure checks everything but the timestamps
 * (on a violation it runs the full pass, so the error is the one
 * mp_validate reports), mp_validate_times only the timestamps.  Both passing
 * == mp_validate passing; the first failing pass names the first violation. */
int mp_validate_structure(mp_ctx *ctx, mp_dtrace *t, mp_err *err);
int mp_validate_times(mp_ctx *ctx, mp_dtrace *t, mp_err *err);

/* detect_iteration (iteration.py:93-105): smallest p with the last 2p
 * (kind, size) fingerprints equal pairwise; window = (n - p, n). */
int mp_detect(mp_ctx *ctx, mp_dtrace *t, int64_t *period, mp_err *err);
/* detect_iteration after validate_trace with one readback for both: a
 * violation is reported first (structure_only: everything but timestamps, a
 * violation then re-decided by the full pass, as mp_validate_structure);
 * without a period the full validation runs before PeriodNotFound. */
int mp_detect_validate(mp_ctx *ctx, mp_dtrace *t, int32_t structure_only, int64_t *period, mp_err *err);

/* extract_lifetimes (iteration.py:275-301) incl. build_profile and
 * compute_load_profile (iteration.py:135-272, 304-320). */
int mp_extract(mp_ctx *ctx, mp_dtrace *t, int64_t start, int64_t end,
               mp_dprofile **out, mp_err *err);
/* extract with caller-given op times / duration (build_profile as used by
 * combine_with_pool, swapsim.py:491) */
int mp_extract_times(mp_ctx *ctx, mp_dtrace *t, int64_t start, int64_t end, const double *op_times,
                     double duration, mp_dprofile **out, mp_err *err);
int mp_profile_get_dims(mp_dprofile *p, mp_profile_dims *dims);
int mp_profile_download(mp_ctx *ctx, mp_dprofile *p, mp_profile_out *out, mp_err *err);
int mp_profile_free(mp_dprofile *p);
/* upload a host-built profile (e.g. IterationProfile objects built in
 * Python); names must be interned so var ids are ranks, flags carry no
 * MP_F_RENAMED. */
int mp_profile_upload(mp_ctx *ctx, const mp_profile_dims *dims, const mp_profile_out *in,
                      const uint8_t *name_blob, const int64_t *name_off, int32_t nnames,
                      mp_dprofile **out, mp_err *err);

/* build_conflict_graph / conflict_graph_from_arcs (smartpool.py:51-88).
 * Edge iff two segments overlap as half-open intervals; the device CSR may
 * hold an edge more than once when a variable has two segments (sets on the
 * Python side deduplicate; planning is insensitive to repeats). */
int mp_conflict_from_profile(mp_ctx *ctx, mp_dprofile *p, mp_dgraph **out, mp_err *err);
int mp_conflict_from_arcs(mp_ctx *ctx, int32_t nvars, const int64_t *size,
                          const int64_t *tiekey, const int64_t *seg_off,
                          const int32_t *seg_lo, const int32_t *seg_hi,
                          mp_dgraph **out, mp_err *err);
int mp_graph_dims(mp_dgraph *g, int64_t *nvars, int64_t *nnz);
int mp_graph_download(mp_ctx *ctx, mp_dgraph *g, int64_t *row_off, int32_t *col, mp_err *err);
int mp_graph_free(mp_dgraph *g);
/* device pointer of the last plan's offsets (int64[nvars]) */
const int64_t *mp_graph_offsets_device(mp_dgraph *g);

/* plan_pool (smartpool.py:91-144).  policy 0 = first_fit, 1 = best_fit.
 * Placement order (-size, alloc, name) — the tie part comes from the
 * graph's tiekey (profile order for profiles).  offsets may be NULL: the
 * result then stays on the device (mp_graph_offsets_device). */
int mp_plan_pool(mp_ctx *ctx, mp_dgraph *g, int32_t policy, int64_t *offsets,
                 int64_t *footprint, int64_t *levels, mp_err *err);

/* upload a host CSR (e.g. a ConflictGraph built in Python); rows are
 * partitioned on the device by the placement order (-size, tiekey) */
int mp_graph_from_csr(mp_ctx *ctx, int32_t nvars, const int64_t *row_off, const int32_t *col,
                      const int64_t *size, const int64_t *tiekey, mp_dgraph **out, mp_err *err);
/* compute_load_profile (iteration.py:304-320) for an uploaded profile */
int mp_profile_compute_loads(mp_ctx *ctx, mp_dprofile *p, int64_t *loads, int64_t *peak, int64_t *peak_index,
                             mp_err *err);

/* ---------------------------------------------------------------------- */
/* AutoSwap planning (autoswap.py, swapsim.py)                              */

/* Swap candidates in columnar form (SwapCandidate, autoswap.py:34-50).
 * name_rank orders the candidates' var names (ties in every sort). */
typedef struct mp_cands_io {
  int64_t k;
  int32_t *var; /* profile variable index (output of mp_swap_candidates) */
  int64_t *size;
  int32_t *out_index;
  double *out_t;
  double *out_ready;
  int32_t *in_index;
  double *in_t;
  double *dout;
  double *din;
  uint8_t *spans;
  int32_t *name_rank;
} mp_cands_io;

/* filter_candidates (autoswap.py:80-116); arrays sized nvars */
int mp_swap_candidates(mp_ctx *ctx, mp_dprofile *p, int64_t threshold, double bw, double lat,
                       mp_cands_io *out, mp_err *err);
/* score_doa / score_aoa / score_wdoa and the unbudgeted SWDOA greedy
 * (autoswap.py:132-215): order[k], swdoa[k], and peaks[k+1] = max of the
 * planned load after j picks (a budgeted run is the prefix up to the first
 * peak <= limit). */
int mp_swap_scores(mp_ctx *ctx, mp_dprofile *p, const mp_cands_io *c, double *doa, double *aoa, double *wdoa,
                   double *swdoa, int32_t *order, double *peaks, mp_err *err);
/* gap_area (autoswap.py:164-174) of every candidate over `loads` (p
 * doubles; NULL = the profile's loads) */
int mp_swap_gap_area(mp_ctx *ctx, mp_dprofile *p, const mp_cands_io *c, const double *loads, double *area,
                     mp_err *err);
/* static-score selection (autoswap.py:305-317): order by (-ranked, -size,
 * name) and insert until the planned peak fits; MP_E_LIMIT_UNREACHABLE
 * with aux0 = limit, aux1 = int(peak) otherwise */
int mp_swap_select_static(mp_ctx *ctx, mp_dprofile *p, const mp_cands_io *c, const double *ranked,
                          int64_t limit, int32_t *sel, int64_t *nsel, mp_err *err);
/* max of the load with the given candidates absent (compute_load_min /
 * planned_peak, swapsim.py:398-405, autoswap.py:320-326); subset NULL = all */
int mp_swap_planned_peak(mp_ctx *ctx, mp_dprofile *p, const mp_cands_io *c, const int32_t *subset,
                         int64_t nsub, double *peak, mp_err *err);
/* _make_schedule (swapsim.py:62-108) for the selection `sel` */
int mp_swap_schedule(mp_ctx *ctx, const mp_cands_io *c, const int32_t *sel, int64_t n, const double *ready,
                     const double *deadline, double *t_so, double *t_eo, double *t_si, double *t_ei,
                     int32_t *event_order, mp_err *err);

typedef struct mp_sim_io {
  /* in: initial schedule (selection order); out: final schedule */
  double *t_so, *t_eo, *t_si, *t_ei;
  int32_t *event_order;
  /* out: LOAD' and LOAD'' curves (capacity 1 + period + 2n each) */
  double *lp_t; int64_t *lp_v; int64_t n_lp; int64_t lp_peak; double lp_peak_t;
  double *ldp_t; int64_t *ldp_v; int64_t n_ldp; int64_t ldp_peak; double ldp_peak_t;
  /* out: delayed ops (capacity period) */
  int64_t *delayed_index; double *delayed_us; int64_t n_delayed;
  double delay; int64_t rounds;
} mp_sim_io;

/* simulate (swapsim.py:349-395): LOAD' overlay + LOAD'' replay with the
 * fixed-point deadline refinement.  MP_E_SWAP_DEADLOCK (aux0 1: swap-in of
 * candidate aux1 cannot start) / MP_E_SIM_INDEXERROR mirror the reference. */
int mp_swap_simulate(mp_ctx *ctx, mp_dprofile *p, const mp_cands_io *c, const int32_t *sel, int64_t n,
                     int64_t limit, int32_t has_limit, int32_t max_rounds, mp_sim_io *io, mp_err *err);

/* Batched BO objective (SwapPlanner score="bo", estimators.py:114-120):
 * for each of m weight vectors (aoa, doa, wdoa, swdoa) the combined-score
 * selection (autoswap.py:269-317) + build_schedule + simulate at `limit`,
 * one warp per vector.  z = the candidates' standardized scores [4][k]
 * (mp_standardize, SCORE_NAMES order).  Per vector: status (MP_OK,
 * MP_E_LIMIT_UNREACHABLE with aux = int(peak), MP_E_SWAP_DEADLOCK with
 * aux = index, MP_E_SIM_INDEXERROR), overhead_us, nsel. */
int mp_swap_eval_weights(mp_ctx *ctx, mp_dprofile *p, const mp_cands_io *c, const double *z,
                         const double *weights, int64_t m, int64_t limit, int32_t max_rounds, int32_t *status,
                         double *overhead, int64_t *nsel, int64_t *aux, mp_err *err);

/* CPython-3.12 compatible standardize (autoswap.py:228-238): Neumaier
 * sum() and libm pow — host code, since device pow differs from glibc's */
int mp_standardize(const double *x, int64_t n, double *out);

/* ---------------------------------------------------------------------- */
/* Batched sweep (BASELINE configs[4]): many independent traces in one      */
/* launch, one CTA per trace.  Each trace runs what the reference's         */
/* estimators do for it (estimators.py:20-130): validate_trace ->            */
/* detect_iteration -> extract_lifetimes -> build_conflict_graph +          */
/* plan_pool -> filter_candidates -> compute_load_min -> the SWDOA greedy,  */
/* then per budget SwapPlanner(limit, score="swdoa").fit: the limit checks,  */
/* select_by_swdoa (the prefix of the greedy order), build_schedule and      */
/* simulate.  Budgets are fractions of each trace's own peak:               */
/* limit_bytes = int(peak_bytes * frac).                                    */

#define MP_SWEEP_MAX_BUDGETS 8

typedef struct mp_sweep_params {
  int32_t policy;      /* plan_pool policy: 0 first_fit, 1 best_fit */
  int32_t nbudget;     /* 0 .. MP_SWEEP_MAX_BUDGETS */
  int32_t max_rounds;  /* simulate(max_rounds=...) (swapsim.py:350) */
  int32_t validate;    /* 1: validate_trace first (IterationAnalyzer.fit) */
  int64_t threshold;   /* filter_candidates threshold_bytes */
  double bw, lat;      /* TransferModel(bandwidth_bytes_per_s, latency_us) */
  double budget_frac[MP_SWEEP_MAX_BUDGETS];
} mp_sweep_params;

/* traces concatenated column-wise; var ids are trace-local lexicographic
 * ranks of that trace's names */
typedef struct mp_sweep_in {
  int64_t ntraces;
  const int64_t *ev_off;   /* [ntraces + 1] */
  const uint8_t *kind;
  const int32_t *var;
  const int64_t *size;
  const int64_t *t_us;
  const int64_t *var_off;  /* [ntraces + 1]: trace t owns name ids var_off[t] .. var_off[t+1] */
  const uint8_t *name_blob;
  const int64_t *name_off; /* [var_off[ntraces] + 1] */
} mp_sweep_in;

/* per-trace result; status is MP_OK or the first failing stage's code
 * (MP_E_INVARIANT: err_index = event position / window op, err_code = MP_V_*;
 * MP_E_PERIOD_NOT_FOUND; MP_E_NOMEM when a trace outgrows the scratch) */
typedef struct mp_sweep_trace {
  int32_t status, err_code;
  int64_t err_index;
  int64_t period, nvars, ncarry, naccess;
  int64_t peak_bytes, peak_index;
  double duration_us;
  int64_t footprint_bytes;
  int64_t edges;     /* undirected conflict edges (ConflictGraph.adj) */
  int64_t ncand;     /* filter_candidates */
  int64_t load_min;  /* compute_load_min */
  int64_t norder;    /* SWDOA greedy picks computed (and stored in cand_order): up
                        to the smallest budget limit SwapPlanner.fit selects for */
} mp_sweep_trace;

/* per (trace, budget) result of SwapPlanner.fit; status MP_OK,
 * MP_E_VALUE (limit <= 0), MP_E_LIMIT_UNREACHABLE (err_aux = achievable),
 * MP_E_SWAP_DEADLOCK (err_index = absolute op index) or MP_E_SIM_INDEXERROR */
typedef struct mp_sweep_budget {
  int64_t limit_bytes;
  int32_t status, rounds;
  int64_t nsel;            /* selection = the first nsel greedy picks */
  int64_t selected_bytes;
  int64_t err_index, err_aux;
  double overhead_us;      /* SimulationResult.overhead_us */
  int64_t achieved_peak_bytes; /* LOAD'' peak */
  int64_t planned_peak_bytes;  /* LOAD' peak */
} mp_sweep_budget;

typedef struct mp_dsweep mp_dsweep; /* device-resident batch */

/* copy a batch to the device (stream-ordered on ctx) */
int mp_sweep_upload(mp_ctx *ctx, const mp_sweep_in *in, mp_dsweep **out, mp_err *err);
int mp_sweep_free(mp_dsweep *s);
/* run the sweep on the device; results stay in HBM until downloaded */
int mp_sweep_run(mp_ctx *ctx, mp_dsweep *s, const mp_sweep_params *prm, mp_err *err);
/* copy results out: traces[ntraces], budgets[ntraces * nbudget];
 * offsets / cand_order are laid out like the events (trace t's rows start
 * at ev_off[t]): plan_pool offsets in profile variable order, and the first
 * norder picks of the SWDOA greedy as profile variable indices (every
 * budget's selection is a prefix of them).  Any pointer may be NULL. */
int mp_sweep_download(mp_ctx *ctx, mp_dsweep *s, mp_sweep_trace *traces, mp_sweep_budget *budgets,
                      int64_t *offsets, int32_t *cand_order, mp_err *err);
/* diagnostics: per-trace clock64() at 8 phase marks of the sweep kernel
 * (start, extract, plan, candidates, greedy, simulate prep, budgets, end) */
int mp_sweep_set_profile(mp_ctx *ctx, mp_dsweep *s, int on, mp_err *err);
int mp_sweep_profile_download(mp_ctx *ctx, mp_dsweep *s, long long *out /* [ntraces * 16]: 8 marks + 8 counters */,
                              mp_err *err);

/* ---------------------------------------------------------------------- */
/* Native trace reader (host, threads): trace.py:87-151 for the canonical   */
/* record forms serialize_trace writes.  format 0 = JSONL, 1 = CSV.         */
/* Lines outside the canonical grammar are not decoded here: their 1-based  */
/* numbers come back as "slow lines" for the reference decoder, so every    */
/* MalformedRecord keeps its line and reason.  MP_E_UNSUPPORTED: the whole  */
/* buffer needs the reference reader (line separators other than \n/\r\n, */
/* CSV quoting, a missing or different CSV header).  Var ids are            */
/* lexicographic ranks of the names.  threads <= 0: all host cores.        */

typedef struct mp_reader mp_reader;

int mp_read_trace(const char *data, int64_t nbytes, int32_t format, int32_t threads, mp_reader **out,
                  mp_err *err);
int mp_reader_dims(mp_reader *r, int64_t *n, int64_t *nvars, int64_t *name_bytes, int64_t *nslow);
int mp_reader_copy(mp_reader *r, uint8_t *kind, int32_t *var, int64_t *size, int64_t *t_us, int64_t *index,
                   int64_t *line, uint8_t *name_blob, int64_t *name_off, int64_t *slow_lines);
int mp_reader_free(mp_reader *r);

/* ---- host-side small-instance oracle ------------------------------------ */

/* brute_force_optimal_footprint's search (smartpool.py:167-221), host code:
 * n variables in placement order with sizes size[k]; nb[nb_off[k]..nb_off[k+1])
 * the positions j < k of k's conflicting variables; cand[0..ncand) the
 * sorted subset sums of the sizes; *best in = the best-fit footprint, out =
 * the minimum found (search stops at the first layout <= lower). */
int mp_brute_force_footprint(int32_t n, const int64_t *size, const int64_t *nb_off, const int32_t *nb,
                             const int64_t *cand, int64_t ncand, int64_t lower, int64_t *best);

#ifdef __cplusplus
}
#endif

#endif /* MEMPLAN_B200_H */
