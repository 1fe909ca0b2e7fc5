// capi.cu — context and handle management of the C ABI (include/memplan_b200.h).
#include <math.h>

#include "handles.cuh"

int profile_loads(mp_ctx *ctx, mp_dprofile *P, mp_err *err);
int profile_alloc(mp_ctx *ctx, mp_dprofile *P, mp_err *err);

extern "C" int mp_version(void) { return 1; }

extern "C" int mp_ctx_create(int device, mp_ctx **out, mp_err *err) {
  mp_ctx *c = new mp_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    mp_set_err(err, MP_E_CUDA, 0, e, 0, cudaGetErrorString(e));
    delete c;
    return MP_E_CUDA;
  }
  CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaMallocHost((void **)&c->h_small, 64 * sizeof(int64_t)));
  CUDA_TRY(cudaMalloc((void **)&c->d_small, 64 * sizeof(int64_t)));
  CUDA_TRY(cudaMemset(c->d_small, 0, 64 * sizeof(int64_t)));  // [63]: k_load_peak_idx's finish counter
  // keep freed scratch in the pool instead of returning it to the driver
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return MP_OK;
}

extern "C" int mp_ctx_destroy(mp_ctx *c) {
  if (!c) return MP_OK;
  cudaStreamSynchronize(c->stream);
  cudaFreeHost(c->h_small);
  cudaFree(c->d_small);
  if (c->scan_vals) cudaFree(c->scan_vals);
  if (c->scan_ctr) cudaFree(c->scan_ctr);
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
  }
  cudaStreamDestroy(c->stream);
  delete c;
  return MP_OK;
}

extern "C" int64_t mp_ctx_launches(mp_ctx *c) { CTX_GUARD(c); return c->launches; }

extern "C" int mp_ctx_sync(mp_ctx *c, mp_err *err) {
  CTX_GUARD(c);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return MP_OK;
}

extern "C" void *mp_ctx_stream(mp_ctx *c) { return (void *)c->stream; }

extern "C" int mp_ctx_set_timing(mp_ctx *c, int on) {
  CTX_GUARD(c);
  c->timing = on != 0;
  return MP_OK;
}

extern "C" int mp_ctx_timings(mp_ctx *c, double *ms, int64_t *count, mp_err *err) {
  CTX_GUARD(c);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < MP_NSTAGES; i++) { ms[i] = 0.0; count[i] = 0; }
  for (auto &r : c->pending) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.id >= 0 && r.id < MP_NSTAGES) { ms[r.id] += t; count[r.id]++; }
    c->spare.push_back(r.a);
    c->spare.push_back(r.b);
  }
  c->pending.clear();
  return MP_OK;
}

extern "C" int mp_trace_reset(mp_dtrace *t) {
  CTX_GUARD(t->ctx);
  t->grouped = false;
  t->perm.release();
  t->gstart.release();
  return MP_OK;
}

static int trace_upload(mp_ctx *ctx, const mp_trace_in *in, mp_dtrace **out, bool async, mp_err *err) {
  cudaStream_t st = ctx->stream;
  mp_dtrace *t = new mp_dtrace();
  t->ctx = ctx;
  t->n = in->n;
  t->nvars = in->nvars;
  t->name_bytes = in->name_off ? in->name_off[in->nvars] : 0;
  int64_t n = in->n;
  CUDA_TRY(t->kind.alloc(n, st));
  CUDA_TRY(t->var.alloc(n, st));
  CUDA_TRY(t->size.alloc(n, st));
  CUDA_TRY(t->t_us.alloc(n, st));
  if (in->index) CUDA_TRY(t->index.alloc(n, st));
  // Names stay on the host: ids are lexicographic ranks, so every device
  // tie-break is an id compare (renamed instances only ever tie on alloc,
  // which is unique), and candidate name ranks arrive with the candidates.
  if (!async) {
    if (n) {
      CUDA_TRY(cudaMemcpyAsync(t->kind.p, in->kind, n, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(t->var.p, in->var, n * 4, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(t->size.p, in->size, n * 8, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(t->t_us.p, in->t_us, n * 8, cudaMemcpyHostToDevice, st));
      if (in->index) CUDA_TRY(cudaMemcpyAsync(t->index.p, in->index, n * 8, cudaMemcpyHostToDevice, st));
    }
    // inputs are borrowed for the duration of the call only
    CUDA_TRY(cudaStreamSynchronize(st));
    *out = t;
    return MP_OK;
  }
  // The columns go up on the copy stream in the order the stages need them
  // (var: grouping; kind, size: period detection; then the rest), each
  // followed by an event the consuming stage waits on (trace_need), so the
  // first stages run while the later columns are still in flight.
  if (!ctx->copy) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
  cudaEvent_t start;
  CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(start, st));  // after the allocations and earlier work
  CUDA_TRY(cudaStreamWaitEvent(ctx->copy, start, 0));
  CUDA_TRY(cudaEventDestroy(start));
  struct Col { int bit; void *dst; const void *src; size_t bytes; };
  const Col cols[5] = {{0, t->var.p, in->var, (size_t)n * 4}, {1, t->kind.p, in->kind, (size_t)n},
                       {2, t->size.p, in->size, (size_t)n * 8}, {3, t->index.p, in->index, (size_t)n * 8},
                       {4, t->t_us.p, in->t_us, (size_t)n * 8}};
  for (const Col &c : cols) {
    CUDA_TRY(cudaEventCreateWithFlags(&t->col_ev[c.bit], cudaEventDisableTiming));
    if (c.bit == 4) continue;  // timestamps: at trace_flush_tus
    if (n && c.src) CUDA_TRY(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, ctx->copy));
    CUDA_TRY(cudaEventRecord(t->col_ev[c.bit], ctx->copy));
  }
  t->tus_host = in->t_us;
  t->tus_deferred = true;
  t->pending = TC_ALL;
  *out = t;
  return MP_OK;
}

extern "C" int mp_trace_upload(mp_ctx *ctx, const mp_trace_in *in, mp_dtrace **out, mp_err *err) {
  CTX_GUARD(ctx);
  return trace_upload(ctx, in, out, false, err);
}

extern "C" int mp_trace_upload_async(mp_ctx *ctx, const mp_trace_in *in, mp_dtrace **out, mp_err *err) {
  CTX_GUARD(ctx);
  return trace_upload(ctx, in, out, true, err);
}

extern "C" int mp_trace_flush(mp_dtrace *t, mp_err *err) { CTX_GUARD(t->ctx); return trace_flush_tus(t->ctx, t, err); }

extern "C" int mp_trace_wait(mp_dtrace *t, mp_err *err) {
  CTX_GUARD(t->ctx);
  int rc = trace_flush_tus(t->ctx, t, err);
  if (rc) return rc;
  if (t->col_ev[4]) CUDA_TRY(cudaEventSynchronize(t->col_ev[4]));
  return MP_OK;
}

extern "C" int mp_trace_free(mp_dtrace *t) {
  CTX_GUARD(t->ctx);
  mp_err e{};
  trace_flush_tus(t->ctx, t, &e);  // profiles waiting for op times get them
  if (t->col_ev[4]) {
    // buffers are released stream-ordered on the context stream: after the copies
    cudaStreamWaitEvent(t->ctx->stream, t->col_ev[4], 0);
    for (cudaEvent_t &e : t->col_ev)
      if (e) cudaEventDestroy(e);
  }
  delete t;
  return MP_OK;
}

extern "C" int mp_profile_get_dims(mp_dprofile *p, mp_profile_dims *dims) {
  CTX_GUARD(p->ctx);
  mp_err e{};
  int rc = profile_times(p->ctx, p, &e);
  if (rc) return rc;
  *dims = p->d;
  return MP_OK;
}

extern "C" int mp_profile_download(mp_ctx *ctx, mp_dprofile *P, mp_profile_out *o, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc = profile_times(ctx, P, err);
    if (rc) return rc;
  }
  cudaStream_t st = ctx->stream;
  int64_t V = P->d.nvars, A = P->d.naccess, p = P->d.period;
#define DL(dst, src, bytes) \
  if ((bytes) > 0 && (dst)) CUDA_TRY(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, st))
  DL(o->base, P->base.p, V * 4);
  DL(o->size, P->size.p, V * 8);
  DL(o->alloc, P->alloc.p, V * 4);
  DL(o->free_, P->free_.p, V * 4);
  DL(o->nseg, P->nseg.p, V * 4);
  DL(o->seg, P->seg.p, V * 16);
  DL(o->flags, P->flags.p, V);
  DL(o->acc_off, P->acc_off.p, (V + 1) * 8);
  DL(o->acc_index, P->acc_index.p, A * 4);
  DL(o->acc_kind, P->acc_kind.p, A);
  DL(o->acc_next, P->acc_next.p, A);
  DL(o->op_times, P->op_times.p, p * 8);
  DL(o->loads, P->loads.p, p * 8);
  DL(o->op_owner, P->op_owner.p, p * 4);
#undef DL
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

extern "C" int mp_profile_free(mp_dprofile *p) {
  CTX_GUARD(p->ctx);
  if (p->ctx->dims_owner == p) p->ctx->dims_owner = nullptr;
  if (p->times_src) {  // still registered with a deferred timestamp upload
    auto &w = p->times_src->tus_waiters;
    for (size_t i = 0; i < w.size(); i++)
      if (w[i] == p) { w.erase(w.begin() + i); break; }
    p->times_src = nullptr;
  }
  if (p->times_ev) {
    // buffers are released stream-ordered on the context stream: after the op times
    cudaStreamWaitEvent(p->ctx->stream, p->times_ev, 0);
    cudaEventDestroy(p->times_ev);
  }
  delete p;
  return MP_OK;
}

extern "C" int mp_profile_upload(mp_ctx *ctx, const mp_profile_dims *dims, const mp_profile_out *in,
                                 const uint8_t *name_blob, const int64_t *name_off, int32_t nnames,
                                 mp_dprofile **out, mp_err *err) {
  CTX_GUARD(ctx);
  cudaStream_t st = ctx->stream;
  mp_dprofile *P = new mp_dprofile();
  P->ctx = ctx;
  P->d = *dims;
  int rc = profile_alloc(ctx, P, err);
  if (rc) { delete P; return rc; }
  int64_t V = P->d.nvars, A = P->d.naccess, p = P->d.period;
#define UL(dst, src, bytes) \
  if ((bytes) > 0 && (src)) CUDA_TRY(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, st))
  UL(P->base.p, in->base, V * 4);
  UL(P->size.p, in->size, V * 8);
  UL(P->alloc.p, in->alloc, V * 4);
  UL(P->free_.p, in->free_, V * 4);
  UL(P->nseg.p, in->nseg, V * 4);
  UL(P->seg.p, in->seg, V * 16);
  UL(P->flags.p, in->flags, V);
  UL(P->acc_off.p, in->acc_off, (V + 1) * 8);
  UL(P->acc_index.p, in->acc_index, A * 4);
  UL(P->acc_kind.p, in->acc_kind, A);
  UL(P->acc_next.p, in->acc_next, A);
  UL(P->op_times.p, in->op_times, p * 8);
  UL(P->loads.p, in->loads, p * 8);
  UL(P->op_owner.p, in->op_owner, p * 4);
  (void)name_blob;
  (void)name_off;
  P->nnames = nnames;
#undef UL
  CUDA_TRY(cudaStreamSynchronize(st));
  *out = P;
  return MP_OK;
}

// ---------------------------------------------------------------------------
// host-side helpers

// CPython's float pow goes to libm; the compiler must not turn pow(x, 2.0)
// into x*x (glibc pow is not always correctly rounded)
static double (*volatile libm_pow)(double, double) = pow;

// builtin sum() over floats in CPython 3.12: Neumaier compensation
static double py_fsum(const double *x, int64_t n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0;
  for (int64_t i = 1; i < n; i++) {
    double t = f + x[i];
    if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
    else c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

// standardize, autoswap.py:228-238 (float_pow special cases as CPython)
extern "C" int mp_standardize(const double *x, int64_t n, double *out) {
  if (n == 0) return MP_OK;
  double mean = py_fsum(x, n) / (double)n;
  std::vector<double> sq((size_t)n);
  for (int64_t i = 0; i < n; i++) {
    double dv = x[i] - mean;
    if (dv == 0.0) sq[i] = 0.0;
    else if (dv != dv) sq[i] = dv;
    else {
      double a = fabs(dv);
      sq[i] = a == 1.0 ? 1.0 : libm_pow(a, 2.0);
    }
  }
  double var = py_fsum(sq.data(), n) / (double)n;
  if (var <= 0) {
    for (int64_t i = 0; i < n; i++) out[i] = 0.0;
    return MP_OK;
  }
  double sd = var == 1.0 ? 1.0 : libm_pow(var, 0.5);
  for (int64_t i = 0; i < n; i++) out[i] = (x[i] - mean) / sd;
  return MP_OK;
}

extern "C" int mp_profile_compute_loads(mp_ctx *ctx, mp_dprofile *P, int64_t *loads, int64_t *peak,
                                        int64_t *peak_index, mp_err *err) {
  CTX_GUARD(ctx);
  int rc = profile_dims(ctx, P, err);  // settle the extraction's values before recomputing
  if (rc) return rc;
  rc = profile_loads(ctx, P, err);
  if (rc) return rc;
  if (P->d.period) CUDA_TRY(cudaMemcpyAsync(loads, P->loads.p, P->d.period * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *peak = P->d.peak_bytes;
  *peak_index = P->d.peak_index;
  return MP_OK;
}
