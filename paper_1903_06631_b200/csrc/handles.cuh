// handles.cuh — device-resident objects behind the opaque C-ABI handles.
#pragma once
#include <vector>

#include "common.cuh"

struct mp_dprofile;

struct mp_dtrace {
  mp_ctx *ctx = nullptr;
  int64_t n = 0;
  int32_t nvars = 0;
  int64_t name_bytes = 0;
  DBuf<uint8_t> kind;
  DBuf<int32_t> var;
  DBuf<int64_t> size;
  DBuf<int64_t> t_us;
  DBuf<int64_t> index;  // empty when index == position
  DBuf<uint8_t> blob;
  DBuf<int64_t> name_off;
  // events grouped by variable: perm = event indices sorted by (var, index),
  // gstart[v] .. gstart[v+1] = var v's run (built once, reused by validate,
  // live-at and extraction)
  bool grouped = false;
  DBuf<uint32_t> perm;
  DBuf<int64_t> gstart;
  // asynchronous upload (mp_trace_upload_async): one event per column on
  // the copy stream; `pending` = columns the context stream has not yet
  // waited for
  cudaEvent_t col_ev[5] = {};
  unsigned pending = 0;
  // the timestamp column of an asynchronous upload goes up only at
  // trace_flush_tus (before the placement, which a concurrent H2D copy barely
  // slows, unlike the readback-bound stages before it); profiles extracted
  // meanwhile get their op times then
  const int64_t *tus_host = nullptr;
  bool tus_deferred = false;
  std::vector<mp_dprofile *> tus_waiters;
};

int trace_flush_tus(mp_ctx *ctx, mp_dtrace *t, mp_err *err);

enum { TC_VAR = 1, TC_KIND = 2, TC_SIZE = 4, TC_INDEX = 8, TC_TUS = 16, TC_ALL = 31 };

// order the context stream after the upload of the columns in `mask`
inline int trace_need(mp_ctx *ctx, mp_dtrace *t, unsigned mask, mp_err *err) {
  if ((mask & TC_TUS) && t->tus_deferred) {
    int rc = trace_flush_tus(ctx, t, err);
    if (rc) return rc;
  }
  unsigned m = mask & t->pending;
  for (int b = 0; b < 5; b++)
    if (m & (1u << b)) CUDA_TRY(cudaStreamWaitEvent(ctx->stream, t->col_ev[b], 0));
  t->pending &= ~m;
  return MP_OK;
}

struct mp_dprofile {
  mp_ctx *ctx = nullptr;
  mp_profile_dims d{};
  int64_t window0 = 0;
  DBuf<int32_t> base, alloc, free_, nseg, seg, acc_index, op_owner;
  DBuf<int64_t> size, acc_off, loads;
  DBuf<uint8_t> flags, acc_kind, acc_next;
  DBuf<double> op_times;
  DBuf<uint8_t> blob;
  DBuf<int64_t> name_off;
  int32_t nnames = 0;
  // op times computed behind an asynchronous trace upload (mp_extract on a
  // trace whose t_us column is still in flight): ready at times_ev
  cudaEvent_t times_ev = nullptr;
  bool times_pending = false;
  // peak / peak index / access count (and the duration unless times are
  // late) still on their way to ctx->h_small[40..43] (profile_dims)
  bool dims_pending = false, dims_late_times = false;
  DBuf<double> dur;
  mp_dtrace *times_src = nullptr;  // registered with a deferred timestamp upload
  int64_t times_start = 0, times_end = 0;
};

// the extraction's final scalars, read back without a stream sync of its own
inline int profile_dims(mp_ctx *ctx, mp_dprofile *P, mp_err *err) {
  if (!P->dims_pending) return MP_OK;
  CUDA_TRY(cudaEventSynchronize(ctx->dims_ev));
  const int64_t *h = ctx->h_small + 40;
  const int64_t p = P->d.period;
  P->d.peak_bytes = p ? h[0] : 0;
  P->d.peak_index = p ? h[1] : 0;
  P->d.naccess = h[2];
  if (!P->dims_late_times) memcpy(&P->d.duration_us, &h[3], 8);
  P->dims_pending = false;
  if (ctx->dims_owner == P) ctx->dims_owner = nullptr;
  return MP_OK;
}

// wait for deferred op times (device order on the context stream, and the
// period duration on the host); resolves the deferred dims first
inline int profile_times(mp_ctx *ctx, mp_dprofile *P, mp_err *err) {
  {
    int rc = profile_dims(ctx, P, err);
    if (rc) return rc;
  }
  if (!P->times_pending) return MP_OK;
  if (P->times_src) {
    int rc = trace_flush_tus(ctx, P->times_src, err);
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamWaitEvent(ctx->stream, P->times_ev, 0));
  CUDA_TRY(cudaEventSynchronize(P->times_ev));
  CUDA_TRY(cudaMemcpy(&P->d.duration_us, P->dur.p, 8, cudaMemcpyDeviceToHost));
  P->times_pending = false;
  return MP_OK;
}

struct mp_dgraph {
  mp_ctx *ctx = nullptr;
  int64_t nvars = 0;
  int64_t nnz = 0;
  DBuf<int64_t> row_off;
  DBuf<int32_t> col;
  DBuf<int64_t> size;     // vertex weights
  DBuf<int64_t> tiekey;   // placement tie-break after -size (empty: vertex order)
  DBuf<int64_t> offsets;  // last plan
  DBuf<int32_t> rank;     // position in the placement order (-size, tie)
  DBuf<int32_t> pcnt;     // row prefix holding the placement predecessors
  int64_t arena_need = 0; // scratch ranges for rows longer than 128
  int64_t size_lo = INT64_MIN, size_hi = INT64_MAX;  // vertex weight range (when the build knows it)
  int64_t peak_hint = -1;  // peak load of the profile the graph came from (a footprint lower bound), -1 unknown
};

// descending size as an ascending unsigned key (placement order, smartpool.py:91-98)
__device__ __forceinline__ uint64_t desc_size_key(int64_t s) { return ~((uint64_t)s ^ 0x8000000000000000ull); }

int build_groups(mp_ctx *ctx, mp_dtrace *t, mp_err *err);
int placement_rank(mp_ctx *ctx, int64_t V, const int64_t *size, const int64_t *tiekey, int32_t *rank,
                   mp_err *err);
int placement_rank_keys(mp_ctx *ctx, int64_t V, const int64_t *size, unsigned long long *mm, mp_err *err);
int placement_rank_sort(mp_ctx *ctx, int64_t V, const int64_t *size, const int64_t *tiekey, int32_t *rank,
                        uint64_t kmin, uint64_t kmax, mp_err *err);
