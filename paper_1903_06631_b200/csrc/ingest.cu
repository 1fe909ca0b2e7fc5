// ingest.cu — trace validation, period detection and lifetime extraction.
//
//   validate_trace      trace.py:55-84
//   detect_iteration    iteration.py:93-105
//   extract_lifetimes   iteration.py:124-301 (incl. build_profile)
//   compute_load_profile iteration.py:304-320
//
// Layout: one stable radix sort groups the trace's events by variable
// (perm, gstart).  Every per-variable state machine of the reference
// (live set, open instances, carry-ins) then runs as one thread per
// variable over its own run — the runs are independent, so the first
// violation in event order is the minimum over variables of each run's
// first violation.  Instances are addressed by their malloc position in the
// window (window instances) or by variable id (carry-ins); prefix sums turn
// them into the reference's variable order (carry-ins by name, then window
// instances by alloc index).
#include <climits>

#include "handles.cuh"
#include "ingest_dev.cuh"

// ---------------------------------------------------------------------------
// grouping

// gstart[v] = lower_bound(v) in the sorted keys: each position where the
// key changes writes the starts of the ids from the previous key + 1 up to
// its own (ids without events get an empty run); the last position closes
// the ids after the largest key.  n >= 1.
__global__ void k_group_bounds(const uint32_t *skeys, int64_t n, int32_t nvars, int64_t *gstart) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cur = skeys[i];
    const int64_t prev = i ? (int64_t)skeys[i - 1] : -1;
    for (int64_t v = prev + 1; v <= cur && v <= nvars; v++) gstart[v] = i;
    if (i == n - 1)
      for (int64_t v = cur + 1; v <= nvars; v++) gstart[v] = n;
  }
}

int build_groups(mp_ctx *ctx, mp_dtrace *t, mp_err *err) {
  if (t->grouped) return MP_OK;
  int rc0 = trace_need(ctx, t, TC_VAR, err);
  if (rc0) return rc0;
  StageTimer tm(ctx, MP_ST_GROUP_SORT);
  int64_t n = t->n;
  DBuf<uint32_t> keys;
  CUDA_TRY(keys.alloc(n, ctx->stream));
  CUDA_TRY(t->perm.alloc(n, ctx->stream));
  CUDA_TRY(t->gstart.alloc((int64_t)t->nvars + 1, ctx->stream));
  // the first pass reads the var column itself and carries the positions
  int rc = dev_radix_sort_u32_iota(ctx, (const uint32_t *)t->var.p, keys.p, t->perm.p, n,
                                   bits_for((uint64_t)(t->nvars > 0 ? t->nvars - 1 : 0)), err);
  if (rc) return rc;
  if (n) LAUNCH(ctx, k_group_bounds, grid_for(n, 256), 256, 0, keys.p, n, t->nvars, t->gstart.p);
  else CUDA_TRY(cudaMemsetAsync(t->gstart.p, 0, ((int64_t)t->nvars + 1) * 8, ctx->stream));
  t->grouped = true;
  return MP_OK;
}

// ---------------------------------------------------------------------------
// validate_trace

__global__ void k_validate_elem(const uint8_t *kind, const int64_t *size, const int64_t *t_us,
                                const int64_t *index, int64_t n, int checks, unsigned long long *first) {
  PDL_WAIT();
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < n; pos += (int64_t)gridDim.x * blockDim.x) {
    int code = validate_elem_code(kind, size, t_us, index, pos, checks);
    if (code) atomicMin(first, ((unsigned long long)pos << 4) | (unsigned)code);
  }
}

__global__ void k_validate_var(const uint8_t *kind, const uint32_t *perm, const int64_t *gstart,
                               int32_t nvars, unsigned long long *first) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvars; v += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long f = validate_var_first(kind, perm, gstart[v], gstart[v + 1]);
    if (f != NO_VIOLATION) atomicMin(first, f);
  }
}

// validate_trace (trace.py:55-84) restricted to `checks`: VC_STRUCT (index,
// kind/size, live-set walk: no timestamps), VC_TIMES (timestamps only) or
// VC_ALL.  Reports the first violation among the checks run.
static int validate_checks(mp_ctx *ctx, mp_dtrace *t, int checks, mp_err *err) {
  if (t->n == 0) return MP_OK;
  int rc = MP_OK;
  if (checks & VC_STRUCT) {
    rc = build_groups(ctx, t, err);
    if (rc) return rc;
  }
  rc = trace_need(ctx, t, checks == VC_ALL ? TC_ALL : checks == VC_TIMES ? TC_TUS : TC_ALL & ~TC_TUS, err);
  if (rc) return rc;
  StageTimer tm(ctx, MP_ST_VALIDATE);
  unsigned long long *d_first = (unsigned long long *)ctx->d_small;
  CUDA_TRY(cudaMemsetAsync(d_first, 0xff, 8, ctx->stream));
  LAUNCH(ctx, k_validate_elem, grid_for(t->n, 256, 4096), 256, 0, t->kind.p, t->size.p, t->t_us.p,
         t->index.p, t->n, checks, d_first);
  if (checks & VC_STRUCT)
    LAUNCH(ctx, k_validate_var, grid_for(t->nvars, 256), 256, 0, t->kind.p, t->perm.p, t->gstart.p,
           t->nvars, d_first);
  int64_t first;
  rc = dev_read_i64(ctx, (const int64_t *)d_first, &first, err);
  if (rc) return rc;
  if ((uint64_t)first == ~0ull) return MP_OK;
  int64_t pos = (int64_t)((uint64_t)first >> 4);
  int code = (int)(first & 15);
  int64_t aux1 = 0;
  if (code == MP_V_INDEX) {
    rc = dev_read_n(ctx, t->index.p + pos, &aux1, 8, err);
  } else if (code == MP_V_SIZE_NONZERO) {
    uint8_t k;
    rc = dev_read_n(ctx, t->kind.p + pos, &k, 1, err);
    aux1 = k;
  } else {
    int32_t v;
    rc = dev_read_n(ctx, t->var.p + pos, &v, 4, err);
    aux1 = v;
  }
  if (rc) return rc;
  mp_set_err(err, MP_E_INVARIANT, pos, code, aux1, "invariant violation");
  return MP_E_INVARIANT;
}

extern "C" int mp_validate(mp_ctx *ctx, mp_dtrace *t, mp_err *err) { CTX_GUARD(ctx); return validate_checks(ctx, t, VC_ALL, err); }

extern "C" int mp_validate_structure(mp_ctx *ctx, mp_dtrace *t, mp_err *err) {
  CTX_GUARD(ctx);
  int rc = validate_checks(ctx, t, VC_STRUCT, err);
  // a structural violation may still be preceded by a timestamp one: the
  // full pass decides which comes first
  if (rc == MP_E_INVARIANT) rc = validate_checks(ctx, t, VC_ALL, err);
  return rc;
}

extern "C" int mp_validate_times(mp_ctx *ctx, mp_dtrace *t, mp_err *err) {
  CTX_GUARD(ctx);
  return validate_checks(ctx, t, VC_TIMES, err);
}

// ---------------------------------------------------------------------------
// detect_iteration: polynomial hashes mod 2^61-1, all candidate periods
// tested in parallel, smallest hash-equal period verified exactly.

#define MODP 0x1fffffffffffffffull
#define HBASE 0x00b2d9c2e4f1a37bull

__device__ __forceinline__ uint64_t mulmod61(uint64_t a, uint64_t b) {
  uint64_t lo = a * b, hi = __umul64hi(a, b);
  uint64_t r = (lo & MODP) + (lo >> 61) + (hi << 3);
  r = (r & MODP) + (r >> 61);
  return r >= MODP ? r - MODP : r;
}
__device__ __forceinline__ uint64_t addmod61(uint64_t a, uint64_t b) {
  uint64_t r = a + b;
  return r >= MODP ? r - MODP : r;
}
__device__ __forceinline__ uint64_t submod61(uint64_t a, uint64_t b) { return a >= b ? a - b : a + MODP - b; }
__device__ uint64_t powmod61(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = mulmod61(r, b);
    b = mulmod61(b, b);
    e >>= 1;
  }
  return r;
}

__device__ __forceinline__ uint64_t fp_hash(uint8_t kind, int64_t size) {
  uint64_t x = (uint64_t)size * 4u + kind + 0x9e3779b97f4a7c15ull;
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return (x & MODP) % MODP;
}

struct HPair { uint64_t h, pw; };  // hash of a run and B^len
__device__ __forceinline__ HPair hcombine(HPair a, HPair b) { return {addmod61(mulmod61(a.h, b.pw), b.h), mulmod61(a.pw, b.pw)}; }

constexpr int DT_THREADS = 256;
constexpr int DT_ITEMS = 16;
constexpr int DT_TILE = DT_THREADS * DT_ITEMS;

__device__ HPair block_scan_hash(HPair v, HPair *total) {
  // exclusive scan of a non-commutative monoid, thread order
  __shared__ HPair s[DT_THREADS];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < DT_THREADS; o <<= 1) {
    HPair x = s[threadIdx.x];
    HPair y = threadIdx.x >= o ? s[threadIdx.x - o] : HPair{0, 1};
    __syncthreads();
    s[threadIdx.x] = hcombine(y, x);
    __syncthreads();
  }
  HPair incl = s[threadIdx.x];
  HPair excl = threadIdx.x ? s[threadIdx.x - 1] : HPair{0, 1};
  if (total) *total = s[DT_THREADS - 1];
  __syncthreads();
  (void)incl;
  return excl;
}

__global__ void __launch_bounds__(DT_THREADS) k_hash_tiles(const uint8_t *kind, const int64_t *size, int64_t n, HPair *tile_agg) {
  PDL_WAIT();
  int64_t base = (int64_t)blockIdx.x * DT_TILE + (int64_t)threadIdx.x * DT_ITEMS;
  HPair a{0, 1};
  for (int i = 0; i < DT_ITEMS; i++) {
    int64_t j = base + i;
    if (j < n) a = hcombine(a, HPair{fp_hash(kind[j], size[j]), HBASE});
  }
  __shared__ HPair tot;
  block_scan_hash(a, &tot);
  if (threadIdx.x == 0) tile_agg[blockIdx.x] = tot;
}

// exclusive prefix of the tile aggregates, one CTA in chunks of DT_THREADS
__global__ void __launch_bounds__(DT_THREADS) k_hash_tile_prefix(HPair *agg, int64_t ntiles) {
  PDL_WAIT();
  __shared__ HPair tot;
  HPair carry{0, 1};
  for (int64_t base = 0; base < ntiles; base += DT_THREADS) {
    int64_t t = base + threadIdx.x;
    HPair x = t < ntiles ? agg[t] : HPair{0, 1};
    HPair ex = block_scan_hash(x, &tot);
    __syncthreads();
    if (t < ntiles) agg[t] = hcombine(carry, ex);
    carry = hcombine(carry, tot);
    __syncthreads();
  }
}

// P[i] = hash of events [0, i) for i in [0, n]
__global__ void __launch_bounds__(DT_THREADS) k_hash_prefix(const uint8_t *kind, const int64_t *size, int64_t n,
                                                            const HPair *tile_pre, uint64_t *P) {
  PDL_WAIT();
  int64_t base = (int64_t)blockIdx.x * DT_TILE + (int64_t)threadIdx.x * DT_ITEMS;
  HPair a{0, 1};
  uint64_t f[DT_ITEMS];
  for (int i = 0; i < DT_ITEMS; i++) {
    int64_t j = base + i;
    f[i] = j < n ? fp_hash(kind[j], size[j]) : 0;
    if (j < n) a = hcombine(a, HPair{f[i], HBASE});
  }
  HPair ex = block_scan_hash(a, nullptr);
  HPair run = hcombine(tile_pre[blockIdx.x], ex);
  for (int i = 0; i < DT_ITEMS; i++) {
    int64_t j = base + i;
    if (j < n) {
      run = hcombine(run, HPair{f[i], HBASE});
      P[j + 1] = run.h;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P[0] = 0;
}

// each thread tests a run of PC_RUN consecutive periods, carrying B^p along
constexpr int PC_RUN = 32;
__global__ void k_period_candidates(const uint64_t *P, int64_t n, int64_t pmin, unsigned long long *best) {
  PDL_WAIT();
  int64_t nruns = (n / 2 - pmin + PC_RUN) / PC_RUN;
  for (int64_t run = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; run < nruns; run += (int64_t)gridDim.x * blockDim.x) {
    int64_t p0 = pmin + run * PC_RUN;
    uint64_t bp = powmod61(HBASE, (uint64_t)p0);
    uint64_t pn = P[n];
    for (int64_t p = p0; p < p0 + PC_RUN && p <= n / 2; p++) {
      uint64_t h1 = submod61(pn, mulmod61(P[n - p], bp));
      uint64_t h2 = submod61(P[n - p], mulmod61(P[n - 2 * p], bp));
      if (h1 == h2) {
        atomicMin(best, (unsigned long long)p);
        break;
      }
      bp = mulmod61(bp, HBASE);
    }
  }
}

__global__ void k_period_verify(const uint8_t *kind, const int64_t *size, int64_t n, const unsigned long long *pbest,
                                int *bad) {
  PDL_WAIT();
  unsigned long long pb = *pbest;
  if (pb == ~0ull) return;
  int64_t p = (int64_t)pb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = n - p + i, b = n - 2 * p + i;
    if (kind[a] != kind[b] || size[a] != size[b]) *bad = 1;
  }
}

// Quick filter: candidate p survives if its last min(p, DT_QUICK)
// fingerprint pairs match (a period must); the smallest survivor is then
// verified exactly.  Typical traces eliminate every non-period within a few
// pairs, so the prefix hashes are only needed when that survivor fails.
constexpr int DT_QUICK = 32;
__global__ void k_period_quick(const uint8_t *kind, const int64_t *size, int64_t n, unsigned long long *best) {
  PDL_WAIT();
  for (int64_t p = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= n / 2;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = p < DT_QUICK ? p : DT_QUICK;
    bool ok = true;
    for (int64_t k = 1; k <= q; k++)
      if (kind[n - k] != kind[n - p - k] || size[n - k] != size[n - p - k]) { ok = false; break; }
    if (ok) atomicMin(best, (unsigned long long)p);
  }
}

// the hash search above pmin (the quick filter's smallest survivor was not a
// period): fingerprint hash tiles, prefix hashes, every candidate, exact check
static int detect_hash(mp_ctx *ctx, mp_dtrace *t, int64_t pmin, int64_t *period, mp_err *err) {
  const int64_t n = t->n;
  unsigned long long *d_best = (unsigned long long *)ctx->d_small;
  int *d_bad = (int *)(ctx->d_small + 1);
  int64_t ntiles = (n + DT_TILE - 1) / DT_TILE;
  DBuf<HPair> agg;
  DBuf<uint64_t> P;
  CUDA_TRY(agg.alloc(ntiles, ctx->stream));
  CUDA_TRY(P.alloc(n + 1, ctx->stream));
  LAUNCH(ctx, k_hash_tiles, (unsigned)ntiles, DT_THREADS, 0, t->kind.p, t->size.p, n, agg.p);
  LAUNCH(ctx, k_hash_tile_prefix, 1, DT_THREADS, 0, agg.p, ntiles);
  LAUNCH(ctx, k_hash_prefix, (unsigned)ntiles, DT_THREADS, 0, t->kind.p, t->size.p, n, agg.p, P.p);
  for (;;) {
    if (pmin > n / 2) {
      mp_set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0, "no period");
      return MP_E_PERIOD_NOT_FOUND;
    }
    CUDA_TRY(cudaMemsetAsync(d_best, 0xff, 8, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, 4, ctx->stream));
    LAUNCH(ctx, k_period_candidates, grid_for((n / 2 - pmin + PC_RUN) / PC_RUN, 256, 8192), 256, 0, P.p, n, pmin,
           d_best);
    // exact check of the smallest hash match, read back together with it
    LAUNCH(ctx, k_period_verify, grid_for(n / 2, 256, 4096), 256, 0, t->kind.p, t->size.p, n,
           (const unsigned long long *)d_best, d_bad);
    int64_t h[2];
    int rc = dev_read_n(ctx, d_best, h, 16, err);
    if (rc) return rc;
    int64_t best = h[0];
    if ((uint64_t)best == ~0ull) {
      mp_set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0, "no period");
      return MP_E_PERIOD_NOT_FOUND;
    }
    if (!(int)h[1]) {
      *period = best;
      return MP_OK;
    }
    pmin = best + 1;  // hash collision: keep searching above it
  }
}

extern "C" int mp_detect(mp_ctx *ctx, mp_dtrace *t, int64_t *period, mp_err *err) {
  CTX_GUARD(ctx);
  int64_t n = t->n;
  if (n < 2) {
    mp_set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0, "no period");
    return MP_E_PERIOD_NOT_FOUND;
  }
  // group the events first: it needs only the var column, which an
  // asynchronous upload delivers before kind and size
  int rc0 = build_groups(ctx, t, err);
  if (rc0) return rc0;
  rc0 = trace_need(ctx, t, TC_KIND | TC_SIZE, err);
  if (rc0) return rc0;
  StageTimer tm(ctx, MP_ST_DETECT);
  unsigned long long *d_best = (unsigned long long *)ctx->d_small;
  int *d_bad = (int *)(ctx->d_small + 1);
  int64_t pmin = 1;
  {
    CUDA_TRY(cudaMemsetAsync(d_best, 0xff, 8, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, 4, ctx->stream));
    LAUNCH(ctx, k_period_quick, grid_for(n / 2, 256, 16384), 256, 0, t->kind.p, t->size.p, n, d_best);
    LAUNCH(ctx, k_period_verify, grid_for(n / 2, 256, 4096), 256, 0, t->kind.p, t->size.p, n,
           (const unsigned long long *)d_best, d_bad);
    int64_t h[2];
    int rc = dev_read_n(ctx, d_best, h, 16, err);
    if (rc) return rc;
    if ((uint64_t)h[0] == ~0ull) {  // no candidate survives: no period
      mp_set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0, "no period");
      return MP_E_PERIOD_NOT_FOUND;
    }
    if (!(int)h[1]) {
      *period = h[0];
      return MP_OK;
    }
    pmin = h[0] + 1;  // the smallest survivor is not a period: hash search above it
  }
  return detect_hash(ctx, t, pmin, period, err);
}

// detect_iteration and validate_trace in one round trip: the quick period
// filter + exact check and the validation kernels run back to back and one
// readback returns both.  A violation takes precedence (the reference
// validates first); a structural one is re-decided by the full pass, as
// mp_validate_structure does.  No period: the full validation decides between
// InvariantViolation and PeriodNotFound, as the pipeline's own fallback does.
extern "C" int mp_detect_validate(mp_ctx *ctx, mp_dtrace *t, int32_t structure_only, int64_t *period,
                                  mp_err *err) {
  CTX_GUARD(ctx);
  const int64_t n = t->n;
  const int checks = structure_only ? VC_STRUCT : VC_ALL;
  if (n < 2) {
    int rc = validate_checks(ctx, t, VC_ALL, err);
    if (rc) return rc;
    mp_set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0, "no period");
    return MP_E_PERIOD_NOT_FOUND;
  }
  int rc = build_groups(ctx, t, err);
  if (rc) return rc;
  rc = trace_need(ctx, t, checks == VC_ALL ? TC_ALL : TC_ALL & ~TC_TUS, err);
  if (rc) return rc;
  // d_small: [0] first violation, [2] best period, [3] its exact check
  unsigned long long *d_first = (unsigned long long *)ctx->d_small;
  unsigned long long *d_best = (unsigned long long *)(ctx->d_small + 2);
  int *d_bad = (int *)(ctx->d_small + 3);
  {
    StageTimer tm(ctx, MP_ST_DETECT);
    CUDA_TRY(cudaMemsetAsync(d_best, 0xff, 8, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, 4, ctx->stream));
    LAUNCH(ctx, k_period_quick, grid_for(n / 2, 256, 16384), 256, 0, t->kind.p, t->size.p, n, d_best);
    LAUNCH(ctx, k_period_verify, grid_for(n / 2, 256, 4096), 256, 0, t->kind.p, t->size.p, n,
           (const unsigned long long *)d_best, d_bad);
  }
  {
    StageTimer tm(ctx, MP_ST_VALIDATE);
    CUDA_TRY(cudaMemsetAsync(d_first, 0xff, 8, ctx->stream));
    LAUNCH(ctx, k_validate_elem, grid_for(n, 256, 4096), 256, 0, t->kind.p, t->size.p, t->t_us.p, t->index.p, n,
           checks, d_first);
    LAUNCH(ctx, k_validate_var, grid_for(t->nvars, 256), 256, 0, t->kind.p, t->perm.p, t->gstart.p, t->nvars,
           d_first);
  }
  int64_t h[4];
  rc = dev_read_n(ctx, ctx->d_small, h, 32, err);
  if (rc) return rc;
  if ((uint64_t)h[0] != ~0ull) return validate_checks(ctx, t, VC_ALL, err);  // names the first violation
  if ((uint64_t)h[2] == ~0ull) {
    rc = validate_checks(ctx, t, VC_ALL, err);
    if (rc) return rc;
    mp_set_err(err, MP_E_PERIOD_NOT_FOUND, n, 0, 0, "no period");
    return MP_E_PERIOD_NOT_FOUND;
  }
  if (!(int)h[3]) {
    *period = h[2];
    return MP_OK;
  }
  rc = detect_hash(ctx, t, h[2] + 1, period, err);
  if (rc == MP_E_PERIOD_NOT_FOUND) {
    mp_err e2{};
    const int vr = validate_checks(ctx, t, VC_ALL, &e2);
    if (vr) { *err = e2; return vr; }
  }
  return rc;
}


// ---------------------------------------------------------------------------
// extract_lifetimes

__global__ void k_ex_var(const uint8_t *kind, const int64_t *size, const uint32_t *perm,
                         const int64_t *gstart, int32_t nvars, int64_t start, int64_t end,
                         ExScratch s, unsigned long long *first) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvars; v += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long f = ex_var_item(kind, size, perm, gstart, v, start, end, s);
    if (f != NO_VIOLATION) atomicMin(first, f);
  }
}

// twin pairing, iteration.py:193-225, and the window's malloc marks (one
// launch: both only read k_ex_var's output or the trace)
__global__ void k_ex_twin(const uint8_t *kind, const int64_t *size, int32_t nvars, int64_t start,
                          int64_t p, ExScratch s, int32_t *is_malloc) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvars; v += (int64_t)gridDim.x * blockDim.x)
    ex_twin_item(kind, size, v, start, p, s);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p; r += (int64_t)gridDim.x * blockDim.x)
    is_malloc[r] = kind[start + r] == MP_MALLOC;
}

// final per-variable records (window instances, alloc order), and the
// carry-ins' (disjoint records and access counts: one launch)
__global__ void k_ex_fill_window(const int32_t *var, const int64_t *size, int64_t start, int64_t p,
                                 int64_t ncarry, ExScratch s, const int32_t *win_ord,
                                 const int32_t *carry_survive, ProfOut o, int64_t *acc_cnt, int32_t nvars,
                                 const int32_t *carry_ord) {
  PDL_WAIT();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p; r += (int64_t)gridDim.x * blockDim.x)
    ex_fill_window_item(var, size, start, r, p, ncarry, s, win_ord, carry_survive, o, acc_cnt);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvars; v += (int64_t)gridDim.x * blockDim.x)
    ex_fill_carry_item(v, p, s, carry_ord, o, acc_cnt);
}

// second walk: accesses into the final CSR, owners into op_owner
__global__ void k_ex_access(const uint8_t *kind, const uint32_t *perm, const int64_t *gstart,
                            int32_t nvars, int64_t start, int64_t end, int64_t ncarry, ExScratch s,
                            const int32_t *carry_ord, const int32_t *win_ord, ProfOut o) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvars; v += (int64_t)gridDim.x * blockDim.x)
    ex_access_item(kind, perm, gstart, v, start, end, ncarry, s, carry_ord, win_ord, o);
}

__global__ void k_ex_times(const int64_t *t_us, int64_t start, int64_t end, double *op_times, double *dur) {
  PDL_WAIT();
  int64_t p = end - start;
  int64_t t0 = t_us[start];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p; r += (int64_t)gridDim.x * blockDim.x)
    op_times[r] = (double)(t_us[start + r] - t0);
  if (blockIdx.x == 0 && threadIdx.x == 0) *dur = ex_duration(t_us, start, end);
}

// Enqueue the deferred timestamp upload on the copy stream (it starts at
// once), then the op times of the profiles extracted meanwhile, ordered
// after their allocations on the context stream.
int trace_flush_tus(mp_ctx *ctx, mp_dtrace *t, mp_err *err) {
  if (!t->tus_deferred) return MP_OK;
  t->tus_deferred = false;
  if (t->n && t->tus_host)
    CUDA_TRY(cudaMemcpyAsync(t->t_us.p, t->tus_host, t->n * 8, cudaMemcpyHostToDevice, ctx->copy));
  CUDA_TRY(cudaEventRecord(t->col_ev[4], ctx->copy));
  if (!t->tus_waiters.empty()) {
    cudaEvent_t ready;
    CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ready, ctx->stream));
    CUDA_TRY(cudaStreamWaitEvent(ctx->copy, ready, 0));
    CUDA_TRY(cudaEventDestroy(ready));
    for (mp_dprofile *P : t->tus_waiters) {
      const int64_t p = P->times_end - P->times_start;
      ctx->launches++;
      k_ex_times<<<grid_for(p, 256), 256, 0, ctx->copy>>>(t->t_us.p, P->times_start, P->times_end, P->op_times.p,
                                                         P->dur.p);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaEventRecord(P->times_ev, ctx->copy));
      P->times_src = nullptr;
    }
    t->tus_waiters.clear();
  }
  return MP_OK;
}

__global__ void k_load_diff(int64_t nv, const int32_t *nseg, const int32_t *seg, const int64_t *size,
                            unsigned long long *diff) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < nseg[i]; s++) {
      atomicAdd(&diff[seg[4 * i + 2 * s]], (unsigned long long)size[i]);
      atomicAdd(&diff[seg[4 * i + 2 * s + 1]], (unsigned long long)(-size[i]));
    }
  }
}

// peak and its earliest index in one pass: each block reduces its share to
// (max, first index of it); the last block to finish reduces the blocks'
// pairs (per-block cells, a finish counter it resets for the next call)
__global__ void k_load_peak_idx(const int64_t *loads, int64_t p, long long *bmax, long long *bidx,
                                unsigned int *finished, long long *peak, unsigned long long *idx) {
  PDL_WAIT();
  long long m = LLONG_MIN, mi = LLONG_MAX;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p; r += (int64_t)gridDim.x * blockDim.x) {
    const long long x = loads[r];
    if (x > m) { m = x; mi = r; }  // r increases along a thread's stride: the first wins ties
  }
  for (int o = 16; o; o >>= 1) {
    const long long um = __shfl_xor_sync(FULL_MASK, m, o), ui = __shfl_xor_sync(FULL_MASK, mi, o);
    if (um > m || (um == m && ui < mi)) { m = um; mi = ui; }
  }
  __shared__ long long sm[32], si[32];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) { sm[threadIdx.x >> 5] = m; si[threadIdx.x >> 5] = mi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (sm[w] > m || (sm[w] == m && si[w] < mi)) { m = sm[w]; mi = si[w]; }
    bmax[blockIdx.x] = m;
    bidx[blockIdx.x] = mi;
    __threadfence();
    last = atomicAdd(finished, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  m = LLONG_MIN;
  mi = LLONG_MAX;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const long long bm = *(volatile long long *)&bmax[b], bi = *(volatile long long *)&bidx[b];
    if (bm > m || (bm == m && bi < mi)) { m = bm; mi = bi; }
  }
  for (int o = 16; o; o >>= 1) {
    const long long um = __shfl_xor_sync(FULL_MASK, m, o), ui = __shfl_xor_sync(FULL_MASK, mi, o);
    if (um > m || (um == m && ui < mi)) { m = um; mi = ui; }
  }
  if ((threadIdx.x & 31) == 0) { sm[threadIdx.x >> 5] = m; si[threadIdx.x >> 5] = mi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (sm[w] > m || (sm[w] == m && si[w] < mi)) { m = sm[w]; mi = si[w]; }
    *peak = m;
    *idx = (unsigned long long)mi;
    *finished = 0;
  }
}


// loads + peak for any device profile (also used after uploads)
// loads + peak (left in ctx->d_small[0..1] = peak, earliest argmax)
int profile_loads_async(mp_ctx *ctx, mp_dprofile *P, mp_err *err) {
  StageTimer tm(ctx, MP_ST_LOADS);
  int64_t p = P->d.period, V = P->d.nvars;
  DBuf<int64_t> diff;
  CUDA_TRY(diff.alloc(p + 1, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(diff.p, 0, (p + 1) * 8, ctx->stream));
  LAUNCH(ctx, k_load_diff, grid_for(V, 256), 256, 0, V, P->nseg.p, P->seg.p, P->size.p,
         (unsigned long long *)diff.p);
  // loads[r] = sum diff[0..r]: inclusive scan straight into the profile
  int rc = dev_inclusive_scan<int64_t>(ctx, diff.p, P->loads.p, p, nullptr, err);
  if (rc) return rc;
  long long *d_peak = (long long *)ctx->d_small;
  unsigned long long *d_idx = (unsigned long long *)(ctx->d_small + 1);
  if (p == 0) {
    const long long lmin = LLONG_MIN;
    CUDA_TRY(cudaMemcpyAsync(d_peak, &lmin, 8, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(d_idx, 0xff, 8, ctx->stream));
    return MP_OK;
  }
  // per-block cells and the finish counter live in the context's small
  // scratch tail (the counter is left at zero by the last block)
  const unsigned nb = grid_for(p, 256, 1024);
  DBuf<long long> cells;
  CUDA_TRY(cells.alloc(2 * (int64_t)nb, ctx->stream));
  unsigned int *fin = (unsigned int *)(ctx->d_small + 63);
  LAUNCH(ctx, k_load_peak_idx, nb, 256, 0, P->loads.p, p, cells.p, cells.p + nb, fin, d_peak, d_idx);
  return MP_OK;
}

int profile_loads(mp_ctx *ctx, mp_dprofile *P, mp_err *err) {
  int rc = profile_loads_async(ctx, P, err);
  if (rc) return rc;
  int64_t p = P->d.period;
  int64_t h[2];
  rc = dev_read_n(ctx, ctx->d_small, h, 16, err);
  if (rc) return rc;
  P->d.peak_bytes = p ? h[0] : 0;
  P->d.peak_index = p ? h[1] : 0;
  return MP_OK;
}

int profile_alloc(mp_ctx *ctx, mp_dprofile *P, mp_err *err) {
  int64_t V = P->d.nvars, A = P->d.naccess, p = P->d.period;
  cudaStream_t s = ctx->stream;
  CUDA_TRY(P->base.alloc(V, s)); CUDA_TRY(P->alloc.alloc(V, s)); CUDA_TRY(P->free_.alloc(V, s));
  CUDA_TRY(P->nseg.alloc(V, s)); CUDA_TRY(P->seg.alloc(4 * V, s)); CUDA_TRY(P->size.alloc(V, s));
  CUDA_TRY(P->flags.alloc(V, s)); CUDA_TRY(P->acc_off.alloc(V + 1, s));
  CUDA_TRY(P->acc_index.alloc(A, s)); CUDA_TRY(P->acc_kind.alloc(A, s)); CUDA_TRY(P->acc_next.alloc(A, s));
  CUDA_TRY(P->op_times.alloc(p, s)); CUDA_TRY(P->loads.alloc(p, s)); CUDA_TRY(P->op_owner.alloc(p, s));
  return MP_OK;
}

static ProfOut prof_out(mp_dprofile *P) {
  return ProfOut{P->base.p, P->alloc.p, P->free_.p, P->nseg.p, P->seg.p, P->acc_index.p, P->op_owner.p,
                 P->size.p, P->acc_off.p, P->loads.p, P->flags.p, P->acc_kind.p, P->acc_next.p, P->op_times.p};
}

extern "C" int mp_extract(mp_ctx *ctx, mp_dtrace *t, int64_t start, int64_t end, mp_dprofile **out,
                          mp_err *err) {
  CTX_GUARD(ctx);
  int64_t n = t->n;
  if (!(0 <= start && start < end && end <= n)) {
    mp_set_err(err, MP_E_VALUE, start, end, n, "window out of range");
    return MP_E_VALUE;
  }
  int rc = build_groups(ctx, t, err);
  if (rc) return rc;
  // lifetimes need kind/var/size only; with the timestamps still uploading,
  // the op times are computed on the copy stream behind them (times_ev)
  const bool late_times = (t->pending & TC_TUS) && ctx->copy;
  rc = trace_need(ctx, t, late_times ? TC_ALL & ~TC_TUS : TC_ALL, err);
  if (rc) return rc;
  cudaStream_t st = ctx->stream;
  int64_t p = end - start;
  std::unique_ptr<StageTimer> tm(new StageTimer(ctx, MP_ST_EXTRACT));
  int32_t nv = t->nvars;
  DBuf<int32_t> owner, w_free, w_nacc, w_mcarry, is_malloc, win_ord, c_free, c_nacc, c_twin, c_surv,
      carry_ord, nmalloc;
  DBuf<uint8_t> w_flags, c_live, c_case;
  DBuf<int64_t> c_abs, c_size;
  CUDA_TRY(owner.alloc(p, st)); CUDA_TRY(w_free.alloc(p, st)); CUDA_TRY(w_nacc.alloc(p, st));
  CUDA_TRY(w_mcarry.alloc(p, st)); CUDA_TRY(is_malloc.alloc(p, st)); CUDA_TRY(win_ord.alloc(p, st));
  CUDA_TRY(w_flags.alloc(p, st));
  CUDA_TRY(c_free.alloc(nv, st)); CUDA_TRY(c_nacc.alloc(nv, st)); CUDA_TRY(c_twin.alloc(nv, st));
  CUDA_TRY(c_surv.alloc(nv, st)); CUDA_TRY(carry_ord.alloc(nv, st)); CUDA_TRY(nmalloc.alloc(nv, st));
  CUDA_TRY(c_live.alloc(nv, st)); CUDA_TRY(c_case.alloc(nv, st)); CUDA_TRY(c_abs.alloc(nv, st));
  CUDA_TRY(c_size.alloc(nv, st));
  ExScratch s{owner.p, w_free.p, w_nacc.p, w_flags.p, w_mcarry.p, is_malloc.p, c_live.p, c_abs.p,
              c_size.p, c_free.p, c_nacc.p, c_case.p, c_twin.p, c_surv.p, nmalloc.p};
  unsigned long long *d_first = (unsigned long long *)ctx->d_small;
  CUDA_TRY(cudaMemsetAsync(d_first, 0xff, 8, st));
  LAUNCH(ctx, k_ex_var, grid_for(nv, 128), 128, 0, t->kind.p, t->size.p, t->perm.p, t->gstart.p, nv,
         start, end, s, d_first);
  // twins and ordinals run before the violation check so one readback
  // returns both (on a violation their output is simply discarded)
  LAUNCH(ctx, k_ex_twin, grid_for(nv > p ? nv : p, 256), 256, 0, t->kind.p, t->size.p, nv, start, p, s,
         is_malloc.p);
  // carry ordinals (surviving carry-ins, by name = var id) and window ordinals
  int32_t *d_tot = (int32_t *)(ctx->d_small + 1);
  rc = dev_exclusive_scan<int32_t>(ctx, c_surv.p, carry_ord.p, nv, d_tot, err);
  if (rc) return rc;
  rc = dev_exclusive_scan<int32_t>(ctx, is_malloc.p, win_ord.p, p, d_tot + 1, err);
  if (rc) return rc;
  int64_t hs[2];
  rc = dev_read_n(ctx, ctx->d_small, hs, 16, err);
  if (rc) return rc;
  uint64_t first = (uint64_t)hs[0];
  if (first != ~0ull) {
    int64_t r = (int64_t)(first >> 4);
    int32_t v;
    rc = dev_read_n(ctx, t->var.p + start + r, &v, 4, err);
    if (rc) return rc;
    mp_set_err(err, MP_E_INVARIANT, r, (int64_t)(first & 15), v, "window invariant");
    return MP_E_INVARIANT;
  }
  int32_t tots[2];
  memcpy(tots, &hs[1], 8);
  int64_t ncarry = tots[0], nwin = tots[1];

  mp_dprofile *P = new mp_dprofile();
  P->ctx = ctx;
  P->window0 = start;
  P->d.period = p;
  P->d.nvars = ncarry + nwin;
  P->d.ncarry = ncarry;
  int64_t V = P->d.nvars;
  DBuf<int64_t> acc_cnt;
  CUDA_TRY(acc_cnt.alloc(V + 1, st));
  CUDA_TRY(P->acc_off.alloc(V + 1, st));
  // size everything but the access arrays first
  {
    cudaStream_t s2 = st;
    CUDA_TRY(P->base.alloc(V, s2)); CUDA_TRY(P->alloc.alloc(V, s2)); CUDA_TRY(P->free_.alloc(V, s2));
    CUDA_TRY(P->nseg.alloc(V, s2)); CUDA_TRY(P->seg.alloc(4 * V, s2)); CUDA_TRY(P->size.alloc(V, s2));
    CUDA_TRY(P->flags.alloc(V, s2));
    CUDA_TRY(P->op_times.alloc(p, s2)); CUDA_TRY(P->loads.alloc(p, s2)); CUDA_TRY(P->op_owner.alloc(p, s2));
  }
  ProfOut o = prof_out(P);
  // c_surv still holds the 0/1 flags (scan wrote carry_ord)
  LAUNCH(ctx, k_ex_fill_window, grid_for(nv > p ? nv : p, 256), 256, 0, t->var.p, t->size.p, start, p, ncarry, s,
         win_ord.p, c_surv.p, o, acc_cnt.p, nv, carry_ord.p);
  int64_t *d_atot = ctx->d_small + 2;
  rc = dev_exclusive_scan<int64_t>(ctx, acc_cnt.p, P->acc_off.p, V, d_atot, err);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(P->acc_off.p + V, d_atot, 8, cudaMemcpyDeviceToDevice, st));
  // accesses are window reads/writes: p bounds their count, no readback needed
  CUDA_TRY(P->acc_index.alloc(p, st)); CUDA_TRY(P->acc_kind.alloc(p, st)); CUDA_TRY(P->acc_next.alloc(p, st));
  o = prof_out(P);
  LAUNCH(ctx, k_ex_access, grid_for(nv, 128), 128, 0, t->kind.p, t->perm.p, t->gstart.p, nv, start, end,
         ncarry, s, carry_ord.p, win_ord.p, o);
  double *d_dur = (double *)(ctx->d_small + 3);
  if (late_times && t->tus_deferred) {
    // the timestamps are not on their way yet: trace_flush_tus computes the
    // op times right behind them
    CUDA_TRY(P->dur.alloc(1, st));
    CUDA_TRY(cudaEventCreateWithFlags(&P->times_ev, cudaEventDisableTiming));
    P->times_pending = true;
    P->times_src = t;
    P->times_start = start;
    P->times_end = end;
    t->tus_waiters.push_back(P);
  } else if (late_times) {
    CUDA_TRY(P->dur.alloc(1, st));
    cudaEvent_t ready;
    CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ready, st));  // op_times / dur allocated
    CUDA_TRY(cudaStreamWaitEvent(ctx->copy, ready, 0));
    CUDA_TRY(cudaEventDestroy(ready));
    ctx->launches++;
    k_ex_times<<<grid_for(p, 256), 256, 0, ctx->copy>>>(t->t_us.p, start, end, P->op_times.p, P->dur.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventCreateWithFlags(&P->times_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(P->times_ev, ctx->copy));
    P->times_pending = true;
  } else {
    LAUNCH(ctx, k_ex_times, grid_for(p, 256), 256, 0, t->t_us.p, start, end, P->op_times.p, d_dur);
  }
  tm.reset();
  rc = profile_loads_async(ctx, P, err);
  if (rc) { delete P; return rc; }
  // peak, peak index, access count, period duration: copied to pinned
  // memory without waiting (whoever reads them first calls profile_dims —
  // the conflict build's own readback has drained the stream by then)
  if (ctx->dims_owner) {
    rc = profile_dims(ctx, ctx->dims_owner, err);
    if (rc) { delete P; return rc; }
  }
  if (!ctx->dims_ev) CUDA_TRY(cudaEventCreateWithFlags(&ctx->dims_ev, cudaEventDisableTiming));
  CUDA_TRY(cudaMemcpyAsync(ctx->h_small + 40, ctx->d_small, 32, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaEventRecord(ctx->dims_ev, st));
  P->dims_pending = true;
  P->dims_late_times = late_times;
  ctx->dims_owner = P;
  P->nnames = t->nvars;
  *out = P;
  return MP_OK;
}

// build_profile with explicit op times (iteration.py:135-272 called from
// combine_with_pool, swapsim.py:491): the window's lifetimes come from the
// trace, its op times and period duration from the caller
extern "C" int mp_extract_times(mp_ctx *ctx, mp_dtrace *t, int64_t start, int64_t end, const double *op_times,
                                double duration, mp_dprofile **out, mp_err *err) {
  CTX_GUARD(ctx);
  int rc = mp_extract(ctx, t, start, end, out, err);
  if (rc) return rc;
  mp_dprofile *P = *out;
  rc = profile_times(ctx, P, err);  // the caller's times replace the computed ones
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(P->op_times.p, op_times, (end - start) * 8, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  P->d.duration_us = duration;
  return MP_OK;
}
