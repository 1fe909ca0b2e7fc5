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
#include <climits>

#include "handles.cuh"

#define INF_D (__longlong_as_double(0x7ff0000000000000ll))
#define EPS_US 1e-6

struct CandDev {
  int64_t k = 0;
  DBuf<int32_t> var, out_index, in_index, name_rank;
  DBuf<int64_t> size;
  DBuf<double> out_t, out_ready, in_t, dout, din;
  DBuf<uint8_t> spans;
};

struct CandView {
  int64_t k;
  const int64_t *size;
  const int32_t *out_index, *in_index, *name_rank;
  const double *out_t, *out_ready, *in_t, *dout, *din;
  const uint8_t *spans;
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

struct LoadView {
  int64_t p;
  const int64_t *loads;
  const double *op_times;
  double duration;
};

// ---------------------------------------------------------------------------
// filter_candidates

struct CandOut {
  int32_t *var, *out_index, *in_index;
  int64_t *size;
  double *out_t, *out_ready, *in_t, *dout, *din;
  uint8_t *spans;
};

// coordinate q-th in sorted order of the access multiset (successor walk
// when the stored order is not already sorted)
__global__ void k_swap_candidates(int64_t V, int64_t p, int64_t peak, const int64_t *size, const uint8_t *flags,
                                  const int64_t *acc_off, const int32_t *acc_index, const uint8_t *acc_next,
                                  const double *op_times, double duration, int64_t threshold, double bw, double lat,
                                  int32_t *flag, CandOut o) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    flag[v] = 0;
    if (size[v] < threshold) continue;
    int64_t a0 = acc_off[v], m = acc_off[v + 1] - a0;
    auto coord = [&](int64_t q) -> int64_t { return acc_index[a0 + q] + (acc_next[a0 + q] ? p : 0); };
    bool sorted = true;
    for (int64_t q = 1; q < m && sorted; q++) sorted = coord(q - 1) <= coord(q);
    // iterate consecutive pairs of the sorted multiset
    int64_t prev = 0, prev_q = -1, first = 0;
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
      prev_q = q;
    }
    (void)prev_q;
    if (!found && (flags[v] & MP_F_PERSISTENT) && m > 0) {
      int64_t a = prev, b = first + p;  // wrap pair (last, first + period)
      if (a >= p) { a -= p; b -= p; }
      if ((a < peak && peak < b) || (a < peak + p && peak + p < b)) { c1 = a; c2 = b; found = true; }
    }
    if (!found) continue;
    bool spans = c2 >= p;
    flag[v] = 1;
    o.var[v] = (int32_t)v;
    o.size[v] = size[v];
    o.out_index[v] = (int32_t)c1;
    o.out_t[v] = op_times[c1];
    o.out_ready[v] = c1 + 1 < p ? op_times[c1 + 1] : duration;
    o.in_index[v] = (int32_t)(c2 % p);
    o.in_t[v] = op_times[c2 % p] + (spans ? duration : 0.0);
    double delta = (double)size[v] / bw * 1e6 + lat;
    o.dout[v] = delta;
    o.din[v] = delta;
    o.spans[v] = spans;
  }
}

template <typename T>
__global__ void k_compact(int64_t V, const int32_t *flag, const int32_t *pos, const T *src, T *dst) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    if (flag[v]) dst[pos[v]] = src[v];
}

extern "C" int mp_swap_candidates(mp_ctx *ctx, mp_dprofile *P, int64_t threshold, double bw, double lat,
                                  mp_cands_io *out, mp_err *err) {
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

// _step_area, autoswap.py:145-161 (left fold in slot order)
__device__ double step_area(const LoadView &L, const double *cur, const int64_t *iloads, double a, double b) {
  if (b <= a) return 0.0;
  int64_t p = L.p;
  int64_t lo = 0, hi = p;  // bisect_right(op_times, a)
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a < L.op_times[mid]) hi = mid; else lo = mid + 1;
  }
  int64_t r0 = lo - 1 < 0 ? 0 : lo - 1;
  double total = 0.0;
  for (int64_t r = r0; r < p; r++) {
    double s = L.op_times[r];
    double e = r + 1 < p ? L.op_times[r + 1] : L.duration;
    if (s >= b) break;
    double ov = pymin(b, e) - pymax(a, s);
    if (ov > 0) total += (cur ? cur[r] : (double)iloads[r]) * ov;
  }
  return total;
}

// gap_area, autoswap.py:164-174
__device__ double gap_area(const LoadView &L, const double *cur, double a, double b) {
  double d = L.duration;
  if (b <= d) return step_area(L, cur, L.loads, a, b);
  return step_area(L, cur, L.loads, a, d) + step_area(L, cur, L.loads, 0.0, b - d);
}

__global__ void k_gap_areas(LoadView L, CandView c, const double *cur, double *area) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.k; i += (int64_t)gridDim.x * blockDim.x)
    area[i] = gap_area(L, cur, c.out_t[i], c.in_t[i]);
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

__device__ __forceinline__ double block_max(double v, double *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = pymax(v, __shfl_xor_sync(FULL_MASK, v, o));
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double x = lane < nw ? red[lane] : -INF_D;
#pragma unroll
    for (int o = 16; o; o >>= 1) x = pymax(x, __shfl_xor_sync(FULL_MASK, x, o));
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

__device__ void apply_absence_block(double *cur, int64_t p, const CandView &c, int32_t i) {
  int64_t lo = c.out_index[i];
  int64_t hi = c.in_index[i] + (c.spans[i] ? p : 0);
  double sz = (double)c.size[i];
  if (hi - lo - 1 <= p) {
    for (int64_t x = lo + 1 + threadIdx.x; x < hi; x += blockDim.x) cur[x % p] -= sz;
  } else {
    for (int64_t r = threadIdx.x; r < p; r += blockDim.x) {
      int h = absence_hits(r, lo, hi, p);
      for (int q = 0; q < h; q++) cur[r] -= sz;
    }
  }
  __syncthreads();
}

__device__ double max_cur(const double *cur, int64_t p, double *red) {
  double m = -INF_D;
  bool have = false;
  for (int64_t r = threadIdx.x; r < p; r += blockDim.x) {
    m = have ? pymax(m, cur[r]) : cur[r];
    have = true;
  }
  return block_max(m, red);
}

// scores + the unbudgeted SWDOA greedy, one CTA
__global__ void __launch_bounds__(512) k_swap_greedy(LoadView L, CandView c, double *cur, uint8_t *taken,
                                                     double *doa, double *aoa, double *wdoa, double *swdoa,
                                                     int32_t *order, double *peaks) {
  __shared__ double red[33];
  __shared__ double s_area[32];
  __shared__ int32_t s_idx[32];
  __shared__ int32_t s_best;
  __shared__ double s_best_area;
  const int64_t p = L.p, k = c.k;
  for (int64_t r = threadIdx.x; r < p; r += blockDim.x) cur[r] = (double)L.loads[r];
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
    double gap = c.in_t[i] - c.out_t[i];
    double d = gap - (c.dout[i] + c.din[i]);
    doa[i] = d;
    aoa[i] = d >= 0 ? (double)c.size[i] * d : d / (double)c.size[i];
    wdoa[i] = gap_area(L, nullptr, c.out_t[i], c.in_t[i]);
    taken[i] = 0;
  }
  __syncthreads();
  peaks[0] = max_cur(cur, p, red);  // all threads agree
  for (int64_t round = 0; round < k; round++) {
    // best key: max (area, size), ties to the smaller name
    int32_t bi = -1;
    double ba = 0;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
      if (taken[i]) continue;
      double area = gap_area(L, cur, c.out_t[i], c.in_t[i]);
      bool better = bi < 0 || area > ba || (area == ba && (c.size[i] > c.size[bi] ||
                                                          (c.size[i] == c.size[bi] && c.name_rank[i] < c.name_rank[bi])));
      if (better) { bi = (int32_t)i; ba = area; }
    }
    // warp then block reduction of the argmax
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      int32_t oi = __shfl_xor_sync(FULL_MASK, bi, o);
      double oa = __shfl_xor_sync(FULL_MASK, ba, o);
      bool take = oi >= 0 && (bi < 0 || oa > ba || (oa == ba && (c.size[oi] > c.size[bi] ||
                                                                  (c.size[oi] == c.size[bi] && c.name_rank[oi] < c.name_rank[bi]))));
      if (take) { bi = oi; ba = oa; }
    }
    if (lane == 0) { s_idx[w] = bi; s_area[w] = ba; }
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t b = -1;
      double a = 0;
      for (int q = 0; q < nw; q++) {
        int32_t oi = s_idx[q];
        double oa = s_area[q];
        bool take = oi >= 0 && (b < 0 || oa > a || (oa == a && (c.size[oi] > c.size[b] ||
                                                                (c.size[oi] == c.size[b] && c.name_rank[oi] < c.name_rank[b]))));
        if (take) { b = oi; a = oa; }
      }
      s_best = b;
      s_best_area = a;
      order[round] = b;
      swdoa[b] = a;
      taken[b] = 1;
    }
    __syncthreads();
    apply_absence_block(cur, p, c, s_best);
    double pk = max_cur(cur, p, red);
    if (threadIdx.x == 0) peaks[round + 1] = pk;
  }
  (void)s_best_area;
}

static LoadView load_view(mp_dprofile *P) { return LoadView{P->d.period, P->loads.p, P->op_times.p, P->d.duration_us}; }

extern "C" int mp_swap_scores(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, double *doa, double *aoa,
                              double *wdoa, double *swdoa, int32_t *order, double *peaks, mp_err *err) {
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
  LAUNCH(ctx, k_swap_greedy, 1, 512, 0, load_view(P), cv, cur.p, taken.p, o_doa.p, o_aoa.p, o_wdoa.p, o_sw.p,
         o_order.p, o_peaks.p);
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
  double pk = max_cur(cur, p, red);
  for (int64_t q = 0; q < k; q++) {
    if (f_le_i(pk, limit)) break;
    int32_t i = ord[q];
    apply_absence_block(cur, p, c, i);
    if (threadIdx.x == 0) sel[n] = i;
    n++;
    pk = max_cur(cur, p, red);
  }
  if (threadIdx.x == 0) {
    *nsel = n;
    *peak_out = pk;
  }
}

extern "C" int mp_swap_select_static(mp_ctx *ctx, mp_dprofile *P, const mp_cands_io *c, const double *ranked,
                                     int64_t limit, int32_t *sel, int64_t *nsel, mp_err *err) {
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

struct SimScratch {
  int32_t *ord;        // n
  double *desired;     // n
  int64_t *in_order;   // n
  double *plan_in, *in_done; uint8_t *in_has;  // n
  double *comp_t; int64_t *comp_sz;            // n
  int32_t *out_trigger, *in_wait;              // p
  int64_t *delta;                              // p
  double *actual;                              // p
  double *ready, *deadline;                    // n
  double *ev_t; int64_t *ev_d;                 // p + 2n (overlay events)
  double *ev2_t; int64_t *ev2_d;               // 2n
};

// insertion sort of positions by (key, name rank, position)
__device__ void sort_by_key_name(int32_t *ord, int64_t n, const double *key, const int32_t *sel, const CandView &c) {
  for (int64_t q = 0; q < n; q++) ord[q] = (int32_t)q;
  for (int64_t q = 1; q < n; q++) {
    int32_t x = ord[q];
    int64_t j = q - 1;
    while (j >= 0) {
      int32_t y = ord[j];
      bool gt = key[y] > key[x] || (key[y] == key[x] && (c.name_rank[sel[y]] > c.name_rank[sel[x]] ||
                                                       (c.name_rank[sel[y]] == c.name_rank[sel[x]] && y > x)));
      if (!gt) break;
      ord[j + 1] = y;
      j--;
    }
    ord[j + 1] = x;
  }
}

// _make_schedule, swapsim.py:62-108
__device__ void make_schedule(const CandView &c, const int32_t *sel, int64_t n, const double *ready,
                              const double *deadline, double *t_so, double *t_eo, double *t_si, double *t_ei,
                              int32_t *eord, SimScratch &S) {
  sort_by_key_name(S.ord, n, ready, sel, c);
  double busy = 0.0;
  for (int64_t q = 0; q < n; q++) {
    int32_t s = S.ord[q];
    double start = pymax(ready[s], busy);
    t_so[s] = start;
    busy = start + c.dout[sel[s]];
    t_eo[s] = busy;
  }
  sort_by_key_name(S.ord, n, deadline, sel, c);
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
  sort_by_key_name(eord, n, t_so, sel, c);
}

__global__ void k_swap_schedule(CandView c, const int32_t *sel, int64_t n, const double *ready, const double *deadline,
                                double *t_so, double *t_eo, double *t_si, double *t_ei, int32_t *eord, SimScratch S) {
  if (threadIdx.x || blockIdx.x) return;
  make_schedule(c, sel, n, ready, deadline, t_so, t_eo, t_si, t_ei, eord, S);
}

extern "C" int mp_swap_schedule(mp_ctx *ctx, const mp_cands_io *c, const int32_t *sel, int64_t n,
                                const double *ready, const double *deadline, double *t_so, double *t_eo,
                                double *t_si, double *t_ei, int32_t *event_order, mp_err *err) {
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

struct Curve {
  double *t;
  int64_t *v;
  int64_t n, peak, load;
  double peak_t;
  __device__ void point(double tt) {
    if (t[n - 1] == tt) v[n - 1] = load;
    else { t[n] = tt; v[n] = load; n++; }
    if (load > peak) { peak = load; peak_t = tt; }
  }
};

struct SimOutDev {
  double *t_so, *t_eo, *t_si, *t_ei;
  int32_t *eord;
  double *lp_t; int64_t *lp_v;
  double *ldp_t; int64_t *ldp_v;
  int64_t *dl_idx; double *dl_us;
  int64_t *scalars;  // n_lp, lp_peak, lp_peak_t, n_ldp, ldp_peak, ldp_peak_t, n_delayed, delay, rounds, status, idx, aux0, aux1
};

struct Replay {
  int64_t k_in, k_out, ncomp, n;
  double in_busy, head_floor, out_busy, delay;
  Curve cv;
  int64_t ndl;
  bool has_limit;
  int64_t limit;
};

// 1 stepped, 0 beyond horizon, -1 IndexError (swapsim.py:266-267)
__device__ int rp_step(Replay &R, SimScratch &S, const CandView &c, const int32_t *sel, double horizon) {
  double t_out = R.k_out < R.ncomp ? S.comp_t[R.k_out] : INF_D;
  double t_in = INF_D;
  int64_t hv = -1;
  if (R.k_in < R.n) {
    hv = S.in_order[R.k_in];
    double start = pymax(pymax(S.plan_in[hv], R.in_busy), R.head_floor);
    if (R.has_limit && R.cv.load + c.size[sel[hv]] > R.limit) start = INF_D;
    t_in = start;
  }
  double t = pymin(t_out, t_in);
  if (t > horizon) return 0;
  if (t_out <= t_in) {
    if (R.k_out >= R.ncomp) return -1;
    int64_t sz = S.comp_sz[R.k_out++];
    R.cv.load -= sz;
    R.head_floor = pymax(R.head_floor, t_out);
    R.cv.point(t_out);
  } else {
    R.cv.load += c.size[sel[hv]];
    R.cv.point(t_in);
    double end = t_in + c.din[sel[hv]];
    R.in_busy = end;
    S.in_done[hv] = end;
    S.in_has[hv] = 1;
    R.k_in++;
  }
  return 1;
}

struct ProfView {
  int64_t p, V, window0;
  double duration;
  const double *tau;
  const int32_t *nseg, *seg;
  const int64_t *size;
};

// one _Replay(...).run(), swapsim.py:205-346; returns status
__device__ int replay_run(Replay &R, SimScratch &S, const ProfView &P, const int64_t live0, const CandView &c,
                          const int32_t *sel, const double *t_si, const double *t_ei, const int32_t *eord,
                          double d_actual, int64_t *eidx, int64_t *eaux0, int64_t *eaux1) {
  const int64_t p = P.p, n = R.n;
  R.cv.load = live0;
  for (int64_t q = 0; q < n; q++) {
    int32_t s = eord[q];
    int32_t ci = sel[s];
    if (c.spans[ci]) {
      R.cv.load -= c.size[ci];
      S.plan_in[s] = pymax(t_si[s] - d_actual, 0.0);
    } else {
      S.plan_in[s] = t_si[s];
    }
  }
  // in_order: (plan_in, deadline, name)
  for (int64_t q = 0; q < n; q++) S.in_order[q] = eord[q];
  for (int64_t q = 1; q < n; q++) {
    int64_t x = S.in_order[q];
    int64_t j = q - 1;
    while (j >= 0) {
      int64_t y = S.in_order[j];
      bool gt = S.plan_in[y] > S.plan_in[x] ||
                (S.plan_in[y] == S.plan_in[x] && (t_ei[y] > t_ei[x] ||
                                                  (t_ei[y] == t_ei[x] && c.name_rank[sel[y]] > c.name_rank[sel[x]])));
      if (!gt) break;
      S.in_order[j + 1] = y;
      j--;
    }
    S.in_order[j + 1] = x;
  }
  for (int64_t r = 0; r < p; r++) { S.out_trigger[r] = -1; S.in_wait[r] = -1; }
  for (int64_t s = 0; s < n; s++) {  // dict comprehension: later entries win
    S.out_trigger[c.out_index[sel[s]]] = (int32_t)s;
    S.in_wait[c.in_index[sel[s]]] = (int32_t)s;
  }
  R.k_in = 0; R.in_busy = 0.0; R.head_floor = 0.0; R.ncomp = 0; R.k_out = 0;
  R.out_busy = 0.0; R.delay = 0.0; R.ndl = 0;
  for (int64_t s = 0; s < n; s++) S.in_has[s] = 0;
  R.cv.n = 1; R.cv.t[0] = 0.0; R.cv.v[0] = R.cv.load; R.cv.peak = R.cv.load; R.cv.peak_t = 0.0;
  for (int64_t r = 0; r < p; r++) {
    double t0 = P.tau[r] + R.delay, t = t0;
    int st;
    while ((st = rp_step(R, S, c, sel, t)) == 1) {}
    if (st < 0) return MP_E_SIM_INDEXERROR;
    int32_t w = S.in_wait[r];
    if (w >= 0) {
      while (!S.in_has[w]) {
        st = rp_step(R, S, c, sel, INF_D);
        if (st < 0) return MP_E_SIM_INDEXERROR;
        if (st == 0) { *eidx = P.window0 + r; *eaux0 = 1; *eaux1 = sel[w]; return MP_E_SWAP_DEADLOCK; }
      }
      if (S.in_done[w] > t + EPS_US) {
        t = S.in_done[w];
        while ((st = rp_step(R, S, c, sel, t)) == 1) {}
        if (st < 0) return MP_E_SIM_INDEXERROR;
      }
    }
    int64_t dd = S.delta[r];
    if (dd > 0 && R.has_limit) {
      while (R.cv.load + dd > R.limit) {
        if (R.k_out >= R.ncomp) { *eidx = P.window0 + r; *eaux0 = 0; *eaux1 = 0; return MP_E_SWAP_DEADLOCK; }
        double t_free = S.comp_t[R.k_out];
        int64_t sz = S.comp_sz[R.k_out++];
        R.cv.load -= sz;
        R.head_floor = pymax(R.head_floor, t_free);
        R.cv.point(t_free);
        t = pymax(t, t_free);
      }
    }
    if (t > t0 + EPS_US) {
      R.ndl++;  // the list itself is rebuilt from actual starts (k_sim_delays)
      R.delay += t - t0;
    } else {
      t = t0;
    }
    S.actual[r] = t;
    if (dd != 0) {
      R.cv.load += dd;
      R.cv.point(t);
      if (dd < 0) {
        R.head_floor = pymax(R.head_floor, t);
        while ((st = rp_step(R, S, c, sel, t)) == 1) {}
        if (st < 0) return MP_E_SIM_INDEXERROR;
      }
    }
    int32_t trig = S.out_trigger[r];
    if (trig >= 0) {
      double op_end = r + 1 < p ? P.tau[r + 1] : P.duration;
      double ready = t + (op_end - P.tau[r]);
      double start = pymax(ready, R.out_busy);
      R.out_busy = start + c.dout[sel[trig]];
      S.comp_t[R.ncomp] = R.out_busy;
      S.comp_sz[R.ncomp] = c.size[sel[trig]];
      R.ncomp++;
    }
  }
  return MP_OK;
}

__global__ void k_op_deltas(ProfView P, int64_t *delta, unsigned long long *live0) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < P.V; v += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < P.nseg[v]; s++) {
      int64_t lo = P.seg[4 * v + 2 * s], hi = P.seg[4 * v + 2 * s + 1];
      if (lo == 0) atomicAdd(live0, (unsigned long long)P.size[v]);
      else atomicAdd((unsigned long long *)&delta[lo], (unsigned long long)P.size[v]);
      if (hi < P.p) atomicAdd((unsigned long long *)&delta[hi], (unsigned long long)(-P.size[v]));
    }
  }
}

// (t, d) lexicographic
__device__ __forceinline__ bool td_less(double ta, int64_t da, double tb, int64_t db) {
  return ta < tb || (ta == tb && da < db);
}

__global__ void k_swap_simulate(ProfView P, CandView c, const int32_t *sel, int64_t n, int64_t limit, int has_limit,
                                int max_rounds, const unsigned long long *live0p, SimScratch S, SimOutDev O) {
  if (threadIdx.x || blockIdx.x) return;
  const int64_t p = P.p;
  const double dnat = P.duration;
  int64_t live0 = (int64_t)*live0p;
  int64_t *sc = O.scalars;
  // ---- LOAD' overlay (swapsim.py:184-202) on the initial schedule ----
  {
    // op events are already in time order; sort equal-time runs by delta
    int64_t na = 0;
    for (int64_t r = 0; r < p; r++)
      if (S.delta[r] != 0) { S.ev_t[na] = P.tau[r]; S.ev_d[na] = S.delta[r]; na++; }
    for (int64_t q = 1; q < na; q++) {
      double xt = S.ev_t[q];
      int64_t xd = S.ev_d[q];
      int64_t j = q - 1;
      while (j >= 0 && td_less(xt, xd, S.ev_t[j], S.ev_d[j])) { S.ev_t[j + 1] = S.ev_t[j]; S.ev_d[j + 1] = S.ev_d[j]; j--; }
      S.ev_t[j + 1] = xt;
      S.ev_d[j + 1] = xd;
    }
    int64_t nb = 0, l0 = live0;
    for (int64_t q = 0; q < n; q++) {
      int32_t s = O.eord[q];
      int32_t ci = sel[s];
      S.ev2_t[nb] = O.t_eo[s]; S.ev2_d[nb] = -c.size[ci]; nb++;
      if (c.spans[ci]) { l0 -= c.size[ci]; S.ev2_t[nb] = pymax(O.t_si[s] - dnat, 0.0); }
      else S.ev2_t[nb] = O.t_si[s];
      S.ev2_d[nb] = c.size[ci];
      nb++;
    }
    for (int64_t q = 1; q < nb; q++) {
      double xt = S.ev2_t[q];
      int64_t xd = S.ev2_d[q];
      int64_t j = q - 1;
      while (j >= 0 && td_less(xt, xd, S.ev2_t[j], S.ev2_d[j])) { S.ev2_t[j + 1] = S.ev2_t[j]; S.ev2_d[j + 1] = S.ev2_d[j]; j--; }
      S.ev2_t[j + 1] = xt;
      S.ev2_d[j + 1] = xd;
    }
    Curve cv{O.lp_t, O.lp_v, 1, l0, l0, 0.0};
    cv.t[0] = 0.0;
    cv.v[0] = l0;
    int64_t ia = 0, ib = 0;
    while (ia < na || ib < nb) {
      bool take_a = ib >= nb || (ia < na && !td_less(S.ev2_t[ib], S.ev2_d[ib], S.ev_t[ia], S.ev_d[ia]));
      double t;
      int64_t d;
      if (take_a) { t = S.ev_t[ia]; d = S.ev_d[ia]; ia++; }
      else { t = S.ev2_t[ib]; d = S.ev2_d[ib]; ib++; }
      cv.load += d;
      cv.point(t);
    }
    sc[0] = cv.n; sc[1] = cv.peak;
    memcpy(&sc[2], &cv.peak_t, 8);
  }
  // ---- LOAD'' replay with the fixed point (swapsim.py:349-395) ----
  Replay R{};
  R.n = n;
  R.has_limit = has_limit;
  R.limit = limit;
  R.cv.t = O.ldp_t;
  R.cv.v = O.ldp_v;
  double prev_delay = 0.0;
  bool have_prev = false;
  int rc = MP_OK;
  int64_t rounds = 0, eidx = 0, ea0 = 0, ea1 = 0;
  for (int it = 0; it < max_rounds; it++) {
    rc = replay_run(R, S, P, live0, c, sel, O.t_si, O.t_ei, O.eord, dnat + (have_prev ? prev_delay : 0.0),
                    &eidx, &ea0, &ea1);
    if (rc) break;
    rounds++;
    if (n == 0 || R.delay == 0.0) break;
    if (have_prev && fabs(R.delay - prev_delay) < 1e-6) break;
    prev_delay = R.delay;
    have_prev = true;
    double d_act = dnat + R.delay;
    for (int64_t s = 0; s < n; s++) {
      int32_t ci = sel[s];
      int64_t oi = c.out_index[ci];
      double op_end = oi + 1 < p ? P.tau[oi + 1] : dnat;
      double dur = op_end - P.tau[oi];
      S.ready[s] = S.actual[oi] + dur;
      S.deadline[s] = S.actual[c.in_index[ci]] + (c.spans[ci] ? d_act : 0.0);
    }
    make_schedule(c, sel, n, S.ready, S.deadline, O.t_so, O.t_eo, O.t_si, O.t_ei, O.eord, S);
  }
  sc[9] = rc;
  sc[10] = eidx; sc[11] = ea0; sc[12] = ea1;
  if (rc == MP_OK) {
    sc[3] = R.cv.n; sc[4] = R.cv.peak;
    memcpy(&sc[5], &R.cv.peak_t, 8);
    sc[6] = R.ndl;
    memcpy(&sc[7], &R.delay, 8);
    sc[8] = rounds;
  }
}

// the delayed-op list of the last replay, recomputed from actual starts
__global__ void k_sim_delays(ProfView P, const double *actual, double delay_total, int64_t *dl_idx, double *dl_us,
                             int64_t *ndl) {
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
  StageTimer tm(ctx, MP_ST_SWAP);
  cudaStream_t st = ctx->stream;
  CandDev d;
  CandView cv;
  int rc = upload_cands(ctx, c, d, cv, err);
  if (rc) return rc;
  int64_t p = P->d.period, cap = 1 + p + 2 * n;
  DBuf<int32_t> dsel, ord, eord, out_trigger, in_wait;
  DBuf<double> desired, plan_in, in_done, comp_t, actual, ready, deadline, ev_t, ev2_t, so, eo, si, ei, lp_t, ldp_t, dl_us;
  DBuf<int64_t> in_order, comp_sz, delta, ev_d, ev2_d, lp_v, ldp_v, dl_idx, scal;
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
  CUDA_TRY(in_has.alloc(nn, st));
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
               out_trigger.p, in_wait.p, delta.p, actual.p, ready.p, deadline.p, ev_t.p, ev_d.p, ev2_t.p, ev2_d.p};
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
