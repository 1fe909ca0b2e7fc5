// swap.cu — AutoSwap planning on the device (autoswap.py, swapsim.py).
//
//   filter_candidates       autoswap.py:53-116   thread per variable + compaction
//   doa / aoa / wdoa         autoswap.py:132-178  thread per candidate
//   SWDOA greedy             autoswap.py:181-215  one CTA: per round every
//                            remaining candidate folds its gap area (binary64
//                            left fold, -fmad=false), a block argmax picks
//                            (area, size, name), the absence is subtracted
//                            slot-parallel, the planned peak is reduced
//   static selection         autoswap.py:285-317  one CTA
//   compute_load_min /       swapsim.py:398-405,  slot-parallel; each slot
//   planned_peak             autoswap.py:320-326  subtracts in candidate order
//   _make_schedule           swapsim.py:62-108    one thread (k is small)
//   simulate / _Replay       swapsim.py:147-395   one thread: the replay is a
//                            sequential event loop (one simulation per
//                            thread is how the batched sweep scales)
//
// Every float operation and comparison follows the reference's order and
// Python's max/min argument semantics, so results are bit-identical.
#include "handles.cuh"
#include "swap_dev.cuh"

struct CandDev {
  int64_t k = 0;
  DBuf<int32_t> var, out_index, in_index, name_rank;
  DBuf<int64_t> size;
  DBuf<double> out_t, out_ready, in_t, dout, din;
  DBuf<uint8_t> spans;
};

static int upload_cands(mp_ctx *ctx, const mp_cands_io *c, CandDev &d, CandView &v, mp_err *err) {
  cudaStream_t st = ctx->stream;
  int64_t k = c->k;
  d.k = k;
  CUDA_TRY(d.size.alloc(k, st)); CUDA_TRY(d.out_index.alloc(k, st)); CUDA_TRY(d.in_index.alloc(k, st));
  CUDA_TRY(d.name_rank.alloc(k, st)); CUDA_TRY(d.out_t.alloc(k, st)); CUDA_TRY(d.out_ready.alloc(k, st));
  CUDA_TRY(d.in_t.alloc(k, st)); CUDA_TRY(d.dout.alloc(k, st)); CUDA_TRY(d.din.alloc(k, st));
  CUDA_TRY(d.spans.alloc(k, st));
  if (k) {
    CUDA_TRY(cudaMemcpyAsync(d.size.p, c->size, k * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.out_index.p, c->out_index, k * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.in_index.p, c->in_index, k * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.name_rank.p, c->name_rank, k * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.out_t.p, c->out_t, k * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.out_ready.p, c->out_ready, k * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.in_t.p, c->in_t, k * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.dout.p, c->dout, k * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.din.p, c->din, k * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.spans.p, c->spans, k, cudaMemcpyHostToDevice, st));
  }
  v = CandView{k, d.size.p, d.out_index.p, d.in_index.p, d.name_rank.p, d.out_t.p, d.out_ready.p, d.in_t.p,
               d.dout.p, d.din.p, d.spans.p};
  return MP_OK;
}

// ---------------------------------------------------------------------------
// filter_candidates

__global__ void k_swap_candidates(int64_t V, int64_t p, int64_t peak, const int64_t *size, const uint8_t *flags,
                                  const int64_t *acc_off, const int32_t *acc_index, const uint8_t *acc_next,
                                  const double *op_times, double duration, int64_t threshold, double bw, double lat,
                                  int32_t *flag, CandOut o) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    flag[v] = cand_item(v, v, p, peak, size, flags, acc_off, acc_index, acc_next, op_times, duration, threshold, bw,
                        lat, o);
}

template <typename T>
__global__ void k_compact(int64_t V, const int32_t *flag, const int32_t *pos, const T *src, T *dst) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    if (flag[v]) dst[pos[v]] = src[v];
}

extern "C" int mp_swap_candidates(mp_ctx *ctx, mp_dprofile *P, int64_t threshold, double bw, double lat,
                                  mp_cands_io *out, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc_t = profile_times(ctx, P, err);
    if (rc_t) return rc_t;
  }
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  int64_t V = P->d.nvars;
  out->k = 0;
  if (V == 0) return MP_OK;
  DBuf<int32_t> flag, pos, var, oi, ii, var2, oi2, ii2;
  DBuf<int64_t> size, size2;
  DBuf<double> ot, orr, it, dout, din, ot2, orr2, it2, dout2, din2;
  DBuf<uint8_t> spans, spans2;
  CUDA_TRY(flag.alloc(V, st)); CUDA_TRY(pos.alloc(V, st)); CUDA_TRY(var.alloc(V, st)); CUDA_TRY(oi.alloc(V, st));
  CUDA_TRY(ii.alloc(V, st)); CUDA_TRY(size.alloc(V, st)); CUDA_TRY(ot.alloc(V, st)); CUDA_TRY(orr.alloc(V, st));
  CUDA_TRY(it.alloc(V, st)); CUDA_TRY(dout.alloc(V, st)); CUDA_TRY(din.alloc(V, st)); CUDA_TRY(spans.alloc(V, st));
  CandOut o{var.p, oi.p, ii.p, size.p, ot.p, orr.p, it.p, dout.p, din.p, spans.p};
  LAUNCH(ctx, k_swap_candidates, grid_for(V, 128), 128, 0, V, P->d.period, P->d.peak_index, P->size.p,
         P->flags.p, P->acc_off.p, P->acc_index.p, P->acc_next.p, P->op_times.p, P->d.duration_us, threshold, bw,
         lat, flag.p, o);
  int32_t *d_k = (int32_t *)ctx->d_small;
  int rc = dev_exclusive_scan<int32_t>(ctx, flag.p, pos.p, V, d_k, err);
  if (rc) return rc;
  int32_t k;
  rc = dev_read_n(ctx, d_k, &k, 4, err);
  if (rc) return rc;
  out->k = k;
  if (!k) return MP_OK;
  CUDA_TRY(var2.alloc(k, st)); CUDA_TRY(oi2.alloc(k, st)); CUDA_TRY(ii2.alloc(k, st)); CUDA_TRY(size2.alloc(k, st));
  CUDA_TRY(ot2.alloc(k, st)); CUDA_TRY(orr2.alloc(k, st)); CUDA_TRY(it2.alloc(k, st)); CUDA_TRY(dout2.alloc(k, st));
  CUDA_TRY(din2.alloc(k, st)); CUDA_TRY(spans2.alloc(k, st));
  unsigned g = grid_for(V, 256);
  LAUNCH(ctx, k_compact<int32_t>, g, 256, 0, V, flag.p, pos.p, var.p, var2.p);
  LAUNCH(ctx, k_compact<int32_t>, g, 256, 0, V, flag.p, pos.p, oi.p, oi2.p);
  LAUNCH(ctx, k_compact<int32_t>, g, 256, 0, V, flag.p, pos.p, ii.p, ii2.p);
  LAUNCH(ctx, k_compact<int64_t>, g, 256, 0, V, flag.p, pos.p, size.p, size2.p);
  LAUNCH(ctx, k_compact<double>, g, 256, 0, V, flag.p, pos.p, ot.p, ot2.p);
  LAUNCH(ctx, k_compact<double>, g, 256, 0, V, flag.p, pos.p, orr.p, orr2.p);
  LAUNCH(ctx, k_compact<double>, g, 256, 0, V, flag.p, pos.p, it.p, it2.p);
  LAUNCH(ctx, k_compact<double>, g, 256, 0, V, flag.p, pos.p, dout.p, dout2.p);
  LAUNCH(ctx, k_compact<double>, g, 256, 0, V, flag.p, pos.p, din.p, din2.p);
  LAUNCH(ctx, k_compact<uint8_t>, g, 256, 0, V, flag.p, pos.p, spans.p, spans2.p);
  CUDA_TRY(cudaMemcpyAsync(out->var, var2.p, k * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->out_index, oi2.p, k * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->in_index, ii2.p, k * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->size, size2.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->out_t, ot2.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->out_ready, orr2.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->in_t, it2.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->dout, dout2.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->din, din2.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->spans, spans2.p, k, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

// ---------------------------------------------------------------------------
// gap areas

__global__ void k_gap_areas(LoadView L, CandView c, const double *cur, double *area) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.k; i += (int64_t)gridDim.x * blockDim.x)
    area[i] = gap_area(L, cur, c.out_t[i], c.in_t[i]);
}

// scores + the unbudgeted SWDOA greedy, one CTA
__global__ void __launch_bounds__(512) k_swap_greedy(LoadView L, CandView c, double *cur, uint8_t *taken,
                                                     double *doa, double *aoa, double *wdoa, double *swdoa,
                                                     int32_t *order, double *peaks, int64_t *W, int32_t *jx,
                                                     int64_t *area) {
  PDL_WAIT();
  __shared__ SwKey keys[33];
  __shared__ long long sm[PM_SMEM];
  swdoa_greedy_block(CtaGroup{}, L, c, cur, taken, doa, aoa, wdoa, swdoa, order, peaks, W, jx, keys, sm, -1, area);
}

// the greedy's rounds run on one warp with incremental areas up to this
// many load slots (a round is then O(p / 32 + k / 32) on the warp instead
// of a CTA pass with six barriers); longer windows keep the CTA rounds
constexpr int64_t SWAP_WARP_ROUNDS_MAX_P = 8192;

static LoadView load_view(mp_dprofile *P) { return LoadView{P->d.period, P->loads.p, P->op_times.p, P->d.duration_us}; }

extern "C" int mp_swap_scores(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, double *doa, double *aoa,
                              double *wdoa, double *swdoa, int32_t *order, double *peaks, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc_t = profile_times(ctx, P, err);
    if (rc_t) return rc_t;
  }
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  int64_t k = c->k, p = P->d.period;
  DBuf<double> cur, o_doa, o_aoa, o_wdoa, o_sw, o_peaks;
  DBuf<int32_t> o_order;
  DBuf<uint8_t> taken;
  CUDA_TRY(cur.alloc(p, st)); CUDA_TRY(o_doa.alloc(k, st)); CUDA_TRY(o_aoa.alloc(k, st));
  CUDA_TRY(o_wdoa.alloc(k, st)); CUDA_TRY(o_sw.alloc(k, st)); CUDA_TRY(o_peaks.alloc(k + 1, st));
  CUDA_TRY(o_order.alloc(k, st)); CUDA_TRY(taken.alloc(k, st));
  DBuf<int64_t> W, area;
  DBuf<int32_t> jx;
  CUDA_TRY(W.alloc(p + 1, st)); CUDA_TRY(jx.alloc(2 * k, st)); CUDA_TRY(area.alloc(k, st));
  LAUNCH(ctx, k_swap_greedy, 1, 512, 0, load_view(P), cv, cur.p, taken.p, o_doa.p, o_aoa.p, o_wdoa.p, o_sw.p,
         o_order.p, o_peaks.p, W.p, jx.p, p <= SWAP_WARP_ROUNDS_MAX_P ? area.p : nullptr);
  if (k) {
    CUDA_TRY(cudaMemcpyAsync(doa, o_doa.p, k * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(aoa, o_aoa.p, k * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(wdoa, o_wdoa.p, k * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(swdoa, o_sw.p, k * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(order, o_order.p, k * 4, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaMemcpyAsync(peaks, o_peaks.p, (k + 1) * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

extern "C" int mp_swap_gap_area(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, const double *loads,
                                double *area, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc_t = profile_times(ctx, P, err);
    if (rc_t) return rc_t;
  }
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  int64_t k = c->k, p = P->d.period;
  if (!k) return MP_OK;
  DBuf<double> cur, out;
  CUDA_TRY(out.alloc(k, st));
  if (loads) {
    CUDA_TRY(cur.alloc(p, st));
    CUDA_TRY(cudaMemcpyAsync(cur.p, loads, p * 8, cudaMemcpyHostToDevice, st));
  }
  LAUNCH(ctx, k_gap_areas, grid_for(k, 128), 128, 0, load_view(P), cv, cur.p, out.p);
  CUDA_TRY(cudaMemcpyAsync(area, out.p, k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

// ---------------------------------------------------------------------------
// static-score selection, one CTA

__global__ void __launch_bounds__(512) k_swap_static(LoadView L, CandView c, const double *ranked, int64_t limit,
                                                     double *cur, int32_t *ord, int32_t *sel, int64_t *nsel,
                                                     double *peak_out) {
  PDL_WAIT();
  __shared__ double red[33];
  const int64_t p = L.p, k = c.k;
  // order by (-ranked, -size, name): rank_i = #keys smaller than key_i
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
    double ri = -ranked[i];
    int64_t si = -c.size[i];
    int64_t pos = 0;
    for (int64_t j = 0; j < k; j++) {
      double rj = -ranked[j];
      int64_t sj = -c.size[j];
      bool less = rj < ri || (rj == ri && (sj < si || (sj == si && (c.name_rank[j] < c.name_rank[i] ||
                                                                    (c.name_rank[j] == c.name_rank[i] && j < i)))));
      pos += less;
    }
    ord[pos] = (int32_t)i;
  }
  for (int64_t r = threadIdx.x; r < p; r += blockDim.x) cur[r] = (double)L.loads[r];
  __syncthreads();
  int64_t n = 0;
  double pk = max_cur(CtaGroup{}, cur, p, red);
  for (int64_t q = 0; q < k; q++) {
    if (f_le_i(pk, limit)) break;
    int32_t i = ord[q];
    apply_absence_block(CtaGroup{}, cur, p, c, i);
    if (threadIdx.x == 0) sel[n] = i;
    n++;
    pk = max_cur(CtaGroup{}, cur, p, red);
  }
  if (threadIdx.x == 0) {
    *nsel = n;
    *peak_out = pk;
  }
}

extern "C" int mp_swap_select_static(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, const double *ranked,
                                     int64_t limit, int32_t *sel, int64_t *nsel, mp_err *err) {
  CTX_GUARD(ctx);
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  int64_t k = c->k, p = P->d.period;
  DBuf<double> rk, cur;
  DBuf<int32_t> ord, osel;
  CUDA_TRY(rk.alloc(k, st)); CUDA_TRY(cur.alloc(p, st)); CUDA_TRY(ord.alloc(k, st)); CUDA_TRY(osel.alloc(k, st));
  if (k) CUDA_TRY(cudaMemcpyAsync(rk.p, ranked, k * 8, cudaMemcpyHostToDevice, st));
  int64_t *d_n = ctx->d_small;
  double *d_pk = (double *)(ctx->d_small + 1);
  LAUNCH(ctx, k_swap_static, 1, 512, 0, load_view(P), cv, rk.p, limit, cur.p, ord.p, osel.p, d_n, d_pk);
  int64_t h[2];
  rc = dev_read_n(ctx, ctx->d_small, h, 16, err);
  if (rc) return rc;
  *nsel = h[0];
  if (h[0]) CUDA_TRY(cudaMemcpyAsync(sel, osel.p, h[0] * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  double pk;
  memcpy(&pk, &h[1], 8);
  if (p && !f_le_i(pk, limit)) {
    mp_set_err(err, MP_E_LIMIT_UNREACHABLE, 0, limit, (int64_t)pk, "limit unreachable");
    return MP_E_LIMIT_UNREACHABLE;
  }
  return MP_OK;
}

// ---------------------------------------------------------------------------
// planned peak / load_min: slot-parallel, candidate order per slot

__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_planned_peak(LoadView L, CandView c, const int32_t *subset, int64_t nsub,
                               unsigned long long *best) {
  PDL_WAIT();
  const int64_t p = L.p;
  unsigned long long m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p; r += (int64_t)gridDim.x * blockDim.x) {
    double cur = (double)L.loads[r];
    for (int64_t q = 0; q < nsub; q++) {
      int32_t i = subset ? subset[q] : (int32_t)q;
      int64_t lo = c.out_index[i], hi = c.in_index[i] + (c.spans[i] ? p : 0);
      int h = absence_hits(r, lo, hi, p);
      for (int t = 0; t < h; t++) cur -= (double)c.size[i];
    }
    unsigned long long kx = dkey(cur);
    m = kx > m ? kx : m;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(FULL_MASK, m, o);
    m = u > m ? u : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(best, m);
}

extern "C" int mp_swap_planned_peak(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, const int32_t *subset,
                                    int64_t nsub, double *peak, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc_t = profile_times(ctx, P, err);
    if (rc_t) return rc_t;
  }
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  DBuf<int32_t> sub;
  if (subset) {
    CUDA_TRY(sub.alloc(nsub, st));
    if (nsub) CUDA_TRY(cudaMemcpyAsync(sub.p, subset, nsub * 4, cudaMemcpyHostToDevice, st));
  } else {
    nsub = c->k;
  }
  unsigned long long *d_best = (unsigned long long *)ctx->d_small;
  CUDA_TRY(cudaMemsetAsync(d_best, 0, 8, st));
  LAUNCH(ctx, k_planned_peak, grid_for(P->d.period, 256, 4096), 256, 0, load_view(P), cv, subset ? sub.p : nullptr,
         nsub, d_best);
  unsigned long long b;
  rc = dev_read_n(ctx, d_best, &b, 8, err);
  if (rc) return rc;
  // decode on the host (same transform)
  unsigned long long bits = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
  memcpy(peak, &bits, 8);
  return MP_OK;
}

// ---------------------------------------------------------------------------
// _make_schedule + simulate: one thread

__global__ void k_swap_schedule(CandView c, const int32_t *sel, int64_t n, const double *ready, const double *deadline,
                                double *t_so, double *t_eo, double *t_si, double *t_ei, int32_t *eord, SimScratch S) {
  PDL_WAIT();
  if (blockIdx.x || threadIdx.x >= 32) return;
  make_schedule(c, sel, n, ready, deadline, t_so, t_eo, t_si, t_ei, eord, S);
}

extern "C" int mp_swap_schedule(mp_ctx *ctx, const mp_cands_io *c, const int32_t *sel, int64_t n,
                                const double *ready, const double *deadline, double *t_so, double *t_eo,
                                double *t_si, double *t_ei, int32_t *event_order, mp_err *err) {
  CTX_GUARD(ctx);
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  if (n == 0) return MP_OK;
  DBuf<int32_t> dsel, eord, ord;
  DBuf<double> rd, dl, so, eo, si, ei, des;
  CUDA_TRY(dsel.alloc(n, st)); CUDA_TRY(eord.alloc(n, st)); CUDA_TRY(ord.alloc(n, st));
  CUDA_TRY(rd.alloc(n, st)); CUDA_TRY(dl.alloc(n, st)); CUDA_TRY(so.alloc(n, st)); CUDA_TRY(eo.alloc(n, st));
  CUDA_TRY(si.alloc(n, st)); CUDA_TRY(ei.alloc(n, st)); CUDA_TRY(des.alloc(n, st));
  CUDA_TRY(cudaMemcpyAsync(dsel.p, sel, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(rd.p, ready, n * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dl.p, deadline, n * 8, cudaMemcpyHostToDevice, st));
  SimScratch S{};
  S.ord = ord.p;
  S.desired = des.p;
  LAUNCH(ctx, k_swap_schedule, 1, 32, 0, cv, dsel.p, n, rd.p, dl.p, so.p, eo.p, si.p, ei.p, eord.p, S);
  CUDA_TRY(cudaMemcpyAsync(t_so, so.p, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(t_eo, eo.p, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(t_si, si.p, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(t_ei, ei.p, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(event_order, eord.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

struct SimOutDev {
  double *t_so, *t_eo, *t_si, *t_ei;
  int32_t *eord;
  double *lp_t; int64_t *lp_v;
  double *ldp_t; int64_t *ldp_v;
  int64_t *dl_idx; double *dl_us;
  int64_t *scalars;  // n_lp, lp_peak, lp_peak_t, n_ldp, ldp_peak, ldp_peak_t, n_delayed, delay, rounds, status, idx, aux0, aux1
};

__global__ void k_op_deltas(ProfView P, int64_t *delta, unsigned long long *live0) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < P.V; v += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < P.nseg[v]; s++) {
      int64_t lo = P.seg[4 * v + 2 * s], hi = P.seg[4 * v + 2 * s + 1];
      if (lo == 0) atomicAdd(live0, (unsigned long long)P.size[v]);
      else atomicAdd((unsigned long long *)&delta[lo], (unsigned long long)P.size[v]);
      if (hi < P.p) atomicAdd((unsigned long long *)&delta[hi], (unsigned long long)(-P.size[v]));
    }
  }
}

__global__ void k_swap_simulate(ProfView P, CandView c, const int32_t *sel, int64_t n, int64_t limit, int has_limit,
                                int max_rounds, const unsigned long long *live0p, SimScratch S, SimOutDev O) {
  PDL_WAIT();
  if (blockIdx.x || threadIdx.x >= 32) return;  // one warp
  const int lane = threadIdx.x;
  int64_t live0 = (int64_t)*live0p;
  int64_t *sc = O.scalars;
  // ---- LOAD' overlay (swapsim.py:184-202) on the initial schedule ----
  {
    int64_t na = 0;
    if (lane == 0) na = sim_op_events(P, S.delta, S.ev_t, S.ev_d);
    na = __shfl_sync(FULL_MASK, na, 0);
    __syncwarp();
    Curve cv{O.lp_t, O.lp_v, 1, 0, 0, 0.0};
    sim_overlay(P, c, sel, n, live0, O.t_eo, O.t_si, O.eord, S.ev_t, S.ev_d, na, S, cv);
    if (lane == 0) {
      sc[0] = cv.n; sc[1] = cv.peak;
      memcpy(&sc[2], &cv.peak_t, 8);
    }
  }
  // ---- LOAD'' replay with the fixed point (swapsim.py:349-395) ----
  Replay<Curve> R{};
  R.cv.t = O.ldp_t;
  R.cv.v = O.ldp_v;
  SimTimes T{O.t_so, O.t_eo, O.t_si, O.t_ei, O.eord};
  SimResult res = sim_fixed_point<true>(P, c, sel, n, limit, has_limit, max_rounds, live0, S, T, R);
  if (lane == 0) {
    sc[9] = res.status;
    sc[10] = res.eidx; sc[11] = res.eaux0; sc[12] = res.eaux1;
    if (res.status == MP_OK) {
      sc[3] = R.cv.n; sc[4] = R.cv.peak;
      memcpy(&sc[5], &R.cv.peak_t, 8);
      sc[6] = R.ndl;
      memcpy(&sc[7], &res.delay, 8);
      sc[8] = res.rounds;
    }
  }
}

// the delayed-op list of the last replay, recomputed from actual starts
__global__ void k_sim_delays(ProfView P, const double *actual, double delay_total, int64_t *dl_idx, double *dl_us,
                             int64_t *ndl) {
  PDL_WAIT();
  (void)delay_total;
  if (threadIdx.x || blockIdx.x) return;
  // a delayed op r adds (t - t0) where t0 = tau[r] + accumulated delay
  double acc = 0.0;
  int64_t n = 0;
  for (int64_t r = 0; r < P.p; r++) {
    double t0 = P.tau[r] + acc;
    double t = actual[r];
    if (t > t0 + EPS_US) {
      dl_idx[n] = P.window0 + r;
      dl_us[n] = t - t0;
      n++;
      acc += t - t0;
    }
  }
  *ndl = n;
}

extern "C" int mp_swap_simulate(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, const int32_t *sel, int64_t n,
                                int64_t limit, int32_t has_limit, int32_t max_rounds, mp_sim_io *io, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc_t = profile_times(ctx, P, err);
    if (rc_t) return rc_t;
  }
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  int64_t p = P->d.period, cap = 1 + p + 2 * n;
  DBuf<int32_t> dsel, ord, eord, out_trigger, in_wait, in_order, ev2_ord;
  DBuf<uint32_t> busy_op;
  DBuf<double> desired, plan_in, in_done, comp_t, actual, ready, deadline, ev_t, ev2_t, so, eo, si, ei, lp_t, ldp_t, dl_us;
  DBuf<int64_t> comp_sz, delta, ev_d, ev2_d, lp_v, ldp_v, dl_idx, scal;
  DBuf<uint8_t> in_has;
  int64_t nn = n > 0 ? n : 1;
  CUDA_TRY(dsel.alloc(nn, st)); CUDA_TRY(ord.alloc(nn, st)); CUDA_TRY(eord.alloc(nn, st));
  CUDA_TRY(out_trigger.alloc(p, st)); CUDA_TRY(in_wait.alloc(p, st)); CUDA_TRY(desired.alloc(nn, st));
  CUDA_TRY(plan_in.alloc(nn, st)); CUDA_TRY(in_done.alloc(nn, st)); CUDA_TRY(comp_t.alloc(nn, st));
  CUDA_TRY(actual.alloc(p, st)); CUDA_TRY(ready.alloc(nn, st)); CUDA_TRY(deadline.alloc(nn, st));
  CUDA_TRY(ev_t.alloc(p, st)); CUDA_TRY(ev_d.alloc(p, st)); CUDA_TRY(ev2_t.alloc(2 * nn, st)); CUDA_TRY(ev2_d.alloc(2 * nn, st));
  CUDA_TRY(so.alloc(nn, st)); CUDA_TRY(eo.alloc(nn, st)); CUDA_TRY(si.alloc(nn, st)); CUDA_TRY(ei.alloc(nn, st));
  CUDA_TRY(lp_t.alloc(cap, st)); CUDA_TRY(lp_v.alloc(cap, st)); CUDA_TRY(ldp_t.alloc(cap, st)); CUDA_TRY(ldp_v.alloc(cap, st));
  CUDA_TRY(dl_idx.alloc(p, st)); CUDA_TRY(dl_us.alloc(p, st)); CUDA_TRY(scal.alloc(16, st));
  CUDA_TRY(in_order.alloc(nn, st)); CUDA_TRY(comp_sz.alloc(nn, st)); CUDA_TRY(delta.alloc(p, st));
  CUDA_TRY(in_has.alloc(nn, st)); CUDA_TRY(ev2_ord.alloc(2 * nn, st)); CUDA_TRY(busy_op.alloc((p + 31) / 32, st));
  if (n) {
    CUDA_TRY(cudaMemcpyAsync(dsel.p, sel, n * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(so.p, io->t_so, n * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(eo.p, io->t_eo, n * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(si.p, io->t_si, n * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ei.p, io->t_ei, n * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(eord.p, io->event_order, n * 4, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaMemsetAsync(delta.p, 0, p * 8, st));
  unsigned long long *d_live0 = (unsigned long long *)ctx->d_small;
  CUDA_TRY(cudaMemsetAsync(d_live0, 0, 8, st));
  ProfView pv{p, P->d.nvars, P->window0, P->d.duration_us, P->op_times.p, P->nseg.p, P->seg.p, P->size.p};
  LAUNCH(ctx, k_op_deltas, grid_for(P->d.nvars, 256), 256, 0, pv, delta.p, d_live0);
  SimScratch S{ord.p, desired.p, in_order.p, plan_in.p, in_done.p, in_has.p, comp_t.p, comp_sz.p,
               out_trigger.p, in_wait.p, busy_op.p, delta.p, actual.p, ready.p, deadline.p, ev_t.p, ev_d.p,
               ev2_t.p, ev2_d.p, ev2_ord.p};
  SimOutDev O{so.p, eo.p, si.p, ei.p, eord.p, lp_t.p, lp_v.p, ldp_t.p, ldp_v.p, dl_idx.p, dl_us.p, scal.p};
  LAUNCH(ctx, k_swap_simulate, 1, 32, 0, pv, cv, dsel.p, n, limit, has_limit, max_rounds, d_live0, S, O);
  int64_t h[16];
  rc = dev_read_n(ctx, scal.p, h, 13 * 8, err);
  if (rc) return rc;
  int status = (int)h[9];
  if (status == MP_E_SWAP_DEADLOCK) {
    mp_set_err(err, status, h[10], h[11], h[12], "swap deadlock");
    return status;
  }
  if (status == MP_E_SIM_INDEXERROR) {
    mp_set_err(err, status, 0, 0, 0, "IndexError in replay");
    return status;
  }
  double delay;
  memcpy(&delay, &h[7], 8);
  LAUNCH(ctx, k_sim_delays, 1, 32, 0, pv, actual.p, delay, dl_idx.p, dl_us.p, scal.p + 14);
  int64_t ndl;
  rc = dev_read_n(ctx, scal.p + 14, &ndl, 8, err);
  if (rc) return rc;
  io->n_lp = h[0]; io->lp_peak = h[1]; memcpy(&io->lp_peak_t, &h[2], 8);
  io->n_ldp = h[3]; io->ldp_peak = h[4]; memcpy(&io->ldp_peak_t, &h[5], 8);
  io->n_delayed = ndl;
  io->delay = delay;
  io->rounds = h[8];
  if (n) {
    CUDA_TRY(cudaMemcpyAsync(io->t_so, so.p, n * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(io->t_eo, eo.p, n * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(io->t_si, si.p, n * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(io->t_ei, ei.p, n * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(io->event_order, eord.p, n * 4, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaMemcpyAsync(io->lp_t, lp_t.p, io->n_lp * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(io->lp_v, lp_v.p, io->n_lp * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(io->ldp_t, ldp_t.p, io->n_ldp * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(io->ldp_v, ldp_v.p, io->n_ldp * 8, cudaMemcpyDeviceToHost, st));
  if (ndl) {
    CUDA_TRY(cudaMemcpyAsync(io->delayed_index, dl_idx.p, ndl * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(io->delayed_us, dl_us.p, ndl * 8, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}

// ---------------------------------------------------------------------------
// batched BO evaluator: the SwapPlanner(score="bo") objective for m weight
// vectors at once (estimators.py:114-120 -> _select_and_simulate with
// score="combined"), one warp per vector:
//   combined_scores  autoswap.py:269-282  sum over SCORE_NAMES of w * z (the
//                                         z-scores are weight-free: host C)
//   select_by_score  autoswap.py:303-317  static order (-score, -size, name),
//                                         insert until max(cur) <= limit
//   build_schedule + simulate             the warp-collective replay above
// Only the overhead (and failures) come back: the winning weights are
// re-run through the regular path by the caller.

struct EvalArgs {
  LoadView L;
  ProfView P;
  CandView c;
  const double *z;   // [4][k]: standardized aoa, doa, wdoa, swdoa
  const double *w;   // [m][4]
  int64_t m, limit;
  int max_rounds;
  const unsigned long long *live0;
  const int64_t *delta;
  const double *ev_t;
  const int64_t *ev_d;
  const int64_t *na;
  char *scratch;
  size_t per_warp;
  int32_t *status, *rounds;
  double *overhead;
  int64_t *nsel, *aux;
};

struct EvalScratch {
  double *comb, *cur;
  int32_t *ord, *sel;
  SimScratch S;
  SimTimes T;
};

template <class A>
__host__ __device__ void eval_take(A &b, EvalScratch &x, int64_t p, int64_t k) {
  x.comb = b.template take<double>(k); x.cur = b.template take<double>(p);
  x.ord = b.template take<int32_t>(k); x.sel = b.template take<int32_t>(k);
  SimScratch &S = x.S;
  S.ord = b.template take<int32_t>(k); S.desired = b.template take<double>(k);
  S.in_order = b.template take<int32_t>(k); S.plan_in = b.template take<double>(k);
  S.in_done = b.template take<double>(k); S.in_has = b.template take<uint8_t>(k);
  S.comp_t = b.template take<double>(k); S.comp_sz = b.template take<int64_t>(k);
  S.out_trigger = b.template take<int32_t>(p); S.in_wait = b.template take<int32_t>(p);
  S.busy_op = b.template take<uint32_t>((p + 31) / 32);
  S.actual = b.template take<double>(p);
  S.ready = b.template take<double>(k); S.deadline = b.template take<double>(k);
  S.ev2_t = b.template take<double>(2 * k); S.ev2_d = b.template take<int64_t>(2 * k);
  S.ev2_ord = b.template take<int32_t>(2 * k);
  x.T.t_so = b.template take<double>(k); x.T.t_eo = b.template take<double>(k);
  x.T.t_si = b.template take<double>(k); x.T.t_ei = b.template take<double>(k);
  x.T.eord = b.template take<int32_t>(k);
}

struct LinearAlloc {  // bump allocation over one warp's scratch (count-only when base is null)
  char *base;
  size_t top;
  template <typename T>
  __host__ __device__ T *take(int64_t n) {
    size_t a = (top + 15) & ~(size_t)15;
    top = a + (size_t)(n > 0 ? n : 1) * sizeof(T);
    return base ? reinterpret_cast<T *>(base + a) : nullptr;
  }
};

__device__ __forceinline__ double warp_pymax_cur(const double *cur, int64_t p) {
  const int lane = threadIdx.x & 31;
  double m = -INF_D;
  for (int64_t r = lane; r < p; r += 32) m = r == lane ? cur[r] : pymax(m, cur[r]);
  // lanes hold interleaved slots: the maximum value is the same whichever
  // copy is kept (a tie is the same double)
#pragma unroll
  for (int o = 16; o; o >>= 1) m = pymax(m, __shfl_xor_sync(FULL_MASK, m, o));
  return m;
}

__global__ void k_op_events(ProfView P, const int64_t *delta, double *ev_t, int64_t *ev_d, int64_t *na) {
  PDL_WAIT();
  if (blockIdx.x || threadIdx.x) return;
  *na = sim_op_events(P, delta, ev_t, ev_d);
}

__global__ void __launch_bounds__(128) k_swap_eval_weights(EvalArgs a) {
  PDL_WAIT();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t p = a.L.p, k = a.c.k;
  const CandView &c = a.c;
  LinearAlloc al{a.scratch + (size_t)gw * a.per_warp, 0};
  EvalScratch x;
  eval_take(al, x, p, k);
  x.S.delta = const_cast<int64_t *>(a.delta);
  const int64_t live0 = (int64_t)*a.live0, na = *a.na;
  for (int64_t e = gw; e < a.m; e += nw) {
    const double *w = a.w + 4 * e;
    for (int64_t i = lane; i < k; i += 32) {
      double s = 0.0;
      for (int q = 0; q < 4; q++) s = s + w[q] * a.z[q * k + i];
      x.comb[i] = s;
    }
    __syncwarp();
    warp_rank_sort(x.ord, k, [&](int64_t y, int64_t q) {
      double ry = -x.comb[y], rq = -x.comb[q];
      if (ry != rq) return ry < rq;
      if (c.size[y] != c.size[q]) return -c.size[y] < -c.size[q];
      return c.name_rank[y] < c.name_rank[q];
    });
    for (int64_t r = lane; r < p; r += 32) x.cur[r] = (double)a.L.loads[r];
    __syncwarp();
    int64_t n = 0;
    double mx = warp_pymax_cur(x.cur, p);
    for (int64_t q = 0; q < k; q++) {
      if (f_le_i(mx, a.limit)) break;
      const int32_t i = x.ord[q];
      const int64_t lo = c.out_index[i], hi = c.in_index[i] + (c.spans[i] ? p : 0);
      const double sz = (double)c.size[i];
      if (hi - lo - 1 <= p) {
        for (int64_t s = lo + 1 + lane; s < hi; s += 32) x.cur[s % p] -= sz;
      } else {
        for (int64_t r = lane; r < p; r += 32) {
          int h = absence_hits(r, lo, hi, p);
          for (int z = 0; z < h; z++) x.cur[r] -= sz;
        }
      }
      if (lane == 0) x.sel[n] = i;
      n++;
      __syncwarp();
      mx = warp_pymax_cur(x.cur, p);
    }
    int status = MP_OK, rounds = 0;
    double overhead = 0.0;
    int64_t aux = 0;
    if (!f_le_i(mx, a.limit)) {
      status = MP_E_LIMIT_UNREACHABLE;  // autoswap.py:315-316
      aux = (int64_t)mx;
    } else {
      for (int64_t q = lane; q < n; q += 32) {
        x.S.ready[q] = c.out_ready[x.sel[q]];
        x.S.deadline[q] = c.in_t[x.sel[q]];
      }
      __syncwarp();
      make_schedule(c, x.sel, n, x.S.ready, x.S.deadline, x.T.t_so, x.T.t_eo, x.T.t_si, x.T.t_ei, x.T.eord, x.S);
      // the overlay curve is not part of the objective; only the replay is
      Replay<PeakCurve> rep{};
      SimResult res = sim_fixed_point<false>(a.P, c, x.sel, n, a.limit, 1, a.max_rounds, live0, x.S, x.T, rep);
      status = res.status;
      rounds = (int)res.rounds;
      overhead = res.delay;
      aux = res.status == MP_E_SWAP_DEADLOCK ? res.eidx : 0;
      (void)na;
    }
    if (lane == 0) {
      a.status[e] = status;
      a.rounds[e] = rounds;
      a.overhead[e] = overhead;
      a.nsel[e] = n;
      a.aux[e] = aux;
    }
    __syncwarp();
  }
}

extern "C" int mp_swap_eval_weights(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, const double *z,
                                    const double *weights, int64_t m, int64_t limit, int32_t max_rounds,
                                    int32_t *status, double *overhead, int64_t *nsel, int64_t *aux, mp_err *err) {
  CTX_GUARD(ctx);
  {
    int rc_t = profile_times(ctx, P, err);
    if (rc_t) return rc_t;
  }
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  if (m <= 0) return MP_OK;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  const int64_t p = P->d.period, k = c->k;
  DBuf<double> dz, dw, ev_t, ov;
  DBuf<int64_t> delta, ev_d, dn, dnsel, daux;
  DBuf<int32_t> dst, drounds;
  DBuf<char> scratch;
  CUDA_TRY(dz.alloc(4 * k, st)); CUDA_TRY(dw.alloc(4 * m, st)); CUDA_TRY(ev_t.alloc(p, st));
  CUDA_TRY(ov.alloc(m, st)); CUDA_TRY(delta.alloc(p, st)); CUDA_TRY(ev_d.alloc(p, st)); CUDA_TRY(dn.alloc(2, st));
  CUDA_TRY(dnsel.alloc(m, st)); CUDA_TRY(daux.alloc(m, st)); CUDA_TRY(dst.alloc(m, st)); CUDA_TRY(drounds.alloc(m, st));
  if (k) CUDA_TRY(cudaMemcpyAsync(dz.p, z, 4 * k * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dw.p, weights, 4 * m * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(delta.p, 0, p * 8, st));
  CUDA_TRY(cudaMemsetAsync(dn.p, 0, 16, st));
  ProfView pv{p, P->d.nvars, P->window0, P->d.duration_us, P->op_times.p, P->nseg.p, P->seg.p, P->size.p};
  unsigned long long *d_live0 = (unsigned long long *)(dn.p + 1);
  LAUNCH(ctx, k_op_deltas, grid_for(P->d.nvars, 256), 256, 0, pv, delta.p, d_live0);
  LAUNCH(ctx, k_op_events, 1, 32, 0, pv, delta.p, ev_t.p, ev_d.p, dn.p);
  LinearAlloc cnt{nullptr, 0};
  EvalScratch xs;
  eval_take(cnt, xs, p, k);
  const size_t per = (cnt.top + 255) & ~(size_t)255;
  int64_t warps = m < (int64_t)ctx->num_sms * 16 ? m : (int64_t)ctx->num_sms * 16;
  CUDA_TRY(scratch.alloc((int64_t)(per * (size_t)warps), st));
  EvalArgs a{load_view(P), pv, cv, dz.p, dw.p, m, limit, max_rounds, d_live0, delta.p, ev_t.p, ev_d.p, dn.p,
             scratch.p, per, dst.p, drounds.p, ov.p, dnsel.p, daux.p};
  LAUNCH(ctx, k_swap_eval_weights, (unsigned)((warps + 3) / 4), 128, 0, a);
  CUDA_TRY(cudaMemcpyAsync(status, dst.p, m * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(overhead, ov.p, m * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(nsel, dnsel.p, m * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(aux, daux.p, m * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MP_OK;
}
