// conflict.cu — weighted interval-conflict graph as CSR (smartpool.py:51-88).
//
// The reference sweeps sorted endpoints and unions an active set into
// adjacency sets.  Here the same relation is built sort-and-sweep style:
//   1. per variable, segments are normalized into the disjoint "effective"
//      intervals the reference's add/discard toggling produces (identity
//      for profile lifetimes; matters only for self-overlapping arcs);
//   2. intervals are radix-sorted by start (and, separately, by end);
//   3. interval k overlaps exactly the sorted run (k, ub(end_k)) after it
//      ("forward") plus the earlier intervals still open at start_k
//      ("backward", counted with one binary search over sorted ends);
//   4. row k's forward run is copied contiguously, and each forward pair is
//      mirrored into the partner's backward slots with an atomic cursor.
// The CSR may repeat an edge when a variable owns two intervals; plan_pool
// only looks at the union of neighbour ranges, and the Python adjacency
// sets deduplicate.
#include <algorithm>
#include <utility>

#include "handles.cuh"

constexpr int MAXSEG = 64;

// effective intervals of each variable: [lo_k, min{hi_m > lo_k}) merged
// GENERAL = false: every variable has at most two segments (profiles); the
// kernel then carries no per-thread segment arrays
template <bool GENERAL>
__global__ void k_norm_count(int64_t nv, const int64_t *seg_off, const int32_t *lo, const int32_t *hi,
                             int64_t *ecnt, int32_t *ea, int32_t *eb, int *overflow, int write,
                             const int64_t *eoff, int32_t *ivar) {
  PDL_WAIT();
  // counting pass (write == 0): eb doubles as the (min start, max end) cell
  int32_t lmin = INT32_MAX, lmax = INT32_MIN;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = seg_off[v], s1 = seg_off[v + 1];
    if (!GENERAL || s1 - s0 <= 2) {
      // profile variables (at most two segments): the same rule in registers
      int32_t l0 = 0, h0 = 0, l1 = 0, h1 = 0;
      int mm = 0;
      for (int64_t s = s0; s < s1; s++) {
        int32_t a = lo[s], b = hi[s];
        if (b <= a) continue;
        if (mm == 0) { l0 = a; h0 = b; }
        else if (a < l0) { l1 = l0; h1 = h0; l0 = a; h0 = b; }
        else { l1 = a; h1 = b; }
        mm++;
      }
      int64_t out = write ? eoff[v] : 0, c = 0;
      int32_t cur_end = INT32_MIN;
      for (int k = 0; k < mm; k++) {
        const int32_t lk = k ? l1 : l0;
        if (lk < cur_end) continue;
        int32_t ne = INT32_MAX;
        if (h0 > lk && h0 < ne) ne = h0;
        if (mm > 1 && h1 > lk && h1 < ne) ne = h1;
        if (write) {
          ea[out + c] = lk;
          eb[out + c] = ne;
          ivar[out + c] = (int32_t)v;
        } else {
          lmin = min(lmin, lk);
          lmax = max(lmax, ne);
        }
        c++;
        cur_end = ne;
      }
      if (!write) ecnt[v] = c;
      continue;
    }
    if constexpr (GENERAL) {
    if (s1 - s0 > MAXSEG) {
      // many segments: walk the chain a_0 = min lo, e_i = min{hi > a_i},
      // a_{i+1} = min{lo >= e_i} straight from global memory (the same
      // intervals as the sorted pass below, O(m) reads per interval)
      int64_t out = write ? eoff[v] : 0, c = 0;
      int64_t want = INT64_MIN;  // next start must be >= want
      for (;;) {
        int64_t a = INT64_MAX;
        for (int64_t s = s0; s < s1; s++)
          if (hi[s] > lo[s] && lo[s] >= want && lo[s] < a) a = lo[s];
        if (a == INT64_MAX) break;
        int32_t ne = INT32_MAX;
        for (int64_t s = s0; s < s1; s++)
          if (hi[s] > lo[s] && hi[s] > a && hi[s] < ne) ne = hi[s];
        if (write) {
          ea[out + c] = (int32_t)a;
          eb[out + c] = ne;
          ivar[out + c] = (int32_t)v;
        } else {
          lmin = min(lmin, (int32_t)a);
          lmax = max(lmax, ne);
        }
        c++;
        want = ne;
      }
      if (!write) ecnt[v] = c;
      continue;
    }
    int32_t L[MAXSEG], H[MAXSEG];
    int m = 0;
    for (int64_t s = s0; s < s1; s++) {
      if (hi[s] <= lo[s]) continue;  // empty segments never enter the sweep
      // insertion sort by lo
      int j = m++;
      while (j > 0 && L[j - 1] > lo[s]) { L[j] = L[j - 1]; H[j] = H[j - 1]; j--; }
      L[j] = lo[s];
      H[j] = hi[s];
    }
    int64_t out = write ? eoff[v] : 0, c = 0;
    int32_t cur_end = INT32_MIN;
    for (int k = 0; k < m; k++) {
      if (L[k] < cur_end) continue;  // inside the current effective interval
      int32_t ne = INT32_MAX;
      for (int q = 0; q < m; q++)
        if (H[q] > L[k] && H[q] < ne) ne = H[q];
      if (write) {
        ea[out + c] = L[k];
        eb[out + c] = ne;
        ivar[out + c] = (int32_t)v;
      } else {
        lmin = min(lmin, L[k]);
        lmax = max(lmax, ne);
      }
      c++;
      cur_end = ne;
    }
    if (!write) ecnt[v] = c;
    }
  }
  if (!write) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      lmin = min(lmin, __shfl_xor_sync(FULL_MASK, lmin, o));
      lmax = max(lmax, __shfl_xor_sync(FULL_MASK, lmax, o));
    }
    if ((threadIdx.x & 31) == 0 && lmin <= lmax) {
      atomicMin(&eb[0], lmin);
      atomicMax(&eb[1], lmax);
    }
  }
}

__global__ void k_iv_keys(int64_t n, const int32_t *a, uint32_t *keys, uint32_t *vals) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint32_t)a[i] ^ 0x80000000u;  // order-preserving for signed bounds
    vals[i] = (uint32_t)i;
  }
}

// fwd/bwd counts per interval (indexed by interval id), plus per sorted
// position the interval's variable, that variable's placement rank and the
// forward count (the fill reads these contiguously instead of chasing
// perm -> ivar -> rank)
__global__ void k_iv_counts(int64_t n, const uint32_t *sstart, const uint32_t *perm, const uint32_t *send,
                            const int32_t *eb, int64_t *cnt, const int32_t *ivar, const int32_t *rank,
                            int32_t *sv) {
  PDL_WAIT();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t iid = perm[k];
    uint32_t a = sstart[k], b = (uint32_t)eb[iid] ^ 0x80000000u;
    int64_t lo = k + 1, hi = n;  // first sorted start >= b
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sstart[mid] < b) lo = mid + 1; else hi = mid;
    }
    int64_t f = lo - k - 1;
    lo = 0; hi = n;  // number of ends <= a
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (send[mid] <= a) lo = mid + 1; else hi = mid;
    }
    int64_t bw = k - lo;
    cnt[iid] = f + bw;
    int32_t v = ivar[iid];
    sv[3 * k] = v;
    sv[3 * k + 1] = rank[v];
    sv[3 * k + 2] = (int32_t)f;
  }
}

__global__ void k_arena_need(int64_t V, const int64_t *row_off, unsigned long long *need) {
  PDL_WAIT();
  unsigned long long s = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = row_off[v + 1] - row_off[v];
    if (d > 128) {
      unsigned long long n2 = 64;
      while (n2 < (unsigned long long)d) n2 <<= 1;
      s += n2;
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(need, s);
}

__global__ void k_iv_minmax(int64_t n, const int32_t *ea, const int32_t *eb, int *mm) {
  PDL_WAIT();
  int lo = INT32_MAX, hi = INT32_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    lo = min(lo, ea[i]);
    hi = max(hi, eb[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(FULL_MASK, lo, o));
    hi = max(hi, __shfl_xor_sync(FULL_MASK, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

__global__ void k_iv_hist(int64_t n, const int32_t *ea, const int32_t *eb, int32_t base, int32_t *hs, int32_t *he) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&hs[ea[i] - base], 1);
    atomicAdd(&he[eb[i] - base], 1);  // exclusive scan: cum_e[x - base + 1] = #ends <= x
  }
}

__global__ void k_iv_scatter(int64_t n, const int32_t *ea, int32_t base, const int32_t *offs, int32_t *cur,
                             uint32_t *perm) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = ea[i] - base;
    perm[offs[x] + atomicAdd(&cur[x], 1)] = (uint32_t)i;
  }
}

// forward run = sorted positions (k, #starts < end); backward = k - #ends <= start
__global__ void k_iv_counts_dense(int64_t n, const uint32_t *perm, const int32_t *ea, const int32_t *eb, int32_t base,
                                  const int32_t *offs, const int32_t *cum_e, int64_t *cnt, const int32_t *ivar,
                                  const int32_t *rank, int32_t *sv) {
  PDL_WAIT();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t iid = perm[k];
    int64_t f = (int64_t)offs[eb[iid] - base] - k - 1;
    int64_t bw = k - cum_e[ea[iid] - base + 1];
    cnt[iid] = f + bw;
    int32_t v = ivar[iid];
    sv[3 * k] = v;
    sv[3 * k + 1] = rank[v];
    sv[3 * k + 2] = (int32_t)f;
  }
}

__global__ void k_row_off(int64_t nv, const int64_t *eoff, const int64_t *sub_off, int64_t *row_off) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= nv; v += (int64_t)gridDim.x * blockDim.x)
    row_off[v] = sub_off[eoff[v]];
}

// warp per sorted interval: the forward run and its mirror, written straight
// into placement-partitioned rows (predecessors grow from the row start,
// successors from the row end) so plan_pool needs no separate split pass
#ifndef IV_FILL_MINB
#define IV_FILL_MINB 8  // 32 registers, 64 warps per SM: more cursor atomics in flight (6: 1.5 % slower)
#endif
__global__ void __launch_bounds__(256, IV_FILL_MINB) k_iv_fill(int64_t n, const int32_t *sv, const int64_t *row_off,
                                                              int32_t *pc, int32_t *sc, int32_t *col) {
  PDL_WAIT();
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = lanemask_lt();
  for (int64_t k = warp; k < n; k += nwarps) {
    // the first 32 partners are read with the interval itself (their
    // addresses do not depend on its forward count)
    const int64_t k0 = k + 1 + lane;
    const int32_t j0 = k0 < n ? sv[3 * k0] : 0, rj0 = k0 < n ? sv[3 * k0 + 1] : 0;
    const int32_t u = sv[3 * k], ru = sv[3 * k + 1], f = sv[3 * k + 2];
    int64_t rbu = row_off[u], reu = row_off[u + 1];
    for (int32_t base = 0; base < f; base += 32) {
      int32_t jx = base + lane;
      bool valid = jx < f;
      int32_t j = j0, rj = rj0;
      if (base && valid) {
        j = sv[3 * (k + 1 + jx)];
        rj = sv[3 * (k + 1 + jx) + 1];
      }
      bool isp = valid && rj < ru;  // j precedes u in placement order
      unsigned bp = __ballot_sync(FULL_MASK, isp);
      unsigned bs = __ballot_sync(FULL_MASK, valid && !isp);
      // the mirrored slot in j's row and u's own cursors are independent
      // round trips: issue both before waiting on either
      int32_t qj = 0;
      int64_t mj = 0;
      if (isp) {
        qj = atomicAdd(&sc[j], 1);  // u succeeds j
        mj = row_off[j + 1] - 1;
      } else if (valid) {
        qj = atomicAdd(&pc[j], 1);  // u precedes j
        mj = row_off[j];
      }
      int32_t p0 = 0, s0 = 0;
      if (lane == 0) {
        if (bp) p0 = atomicAdd(&pc[u], __popc(bp));
        if (bs) s0 = atomicAdd(&sc[u], __popc(bs));
      }
      p0 = __shfl_sync(FULL_MASK, p0, 0);
      s0 = __shfl_sync(FULL_MASK, s0, 0);
      if (isp) {
        col[rbu + p0 + __popc(bp & lt)] = j;
        col[mj - qj] = u;
      } else if (valid) {
        col[reu - 1 - (s0 + __popc(bs & lt))] = j;
        col[mj + qj] = u;
      }
    }
  }
}

static int build_csr(mp_ctx *ctx, int64_t nv, const int64_t *seg_off_d, const int32_t *lo_d,
                     const int32_t *hi_d, bool general, mp_dgraph *g, mp_err *err) {
  auto norm = general ? k_norm_count<true> : k_norm_count<false>;
  cudaStream_t st = ctx->stream;
  // placement order first: the fill writes rows already split by it
  CUDA_TRY(g->rank.alloc(nv, st));
  CUDA_TRY(g->pcnt.alloc(nv, st));
  std::unique_ptr<StageTimer> tm(new StageTimer(ctx, MP_ST_CONFLICT_PREP));
  DBuf<int64_t> ecnt, eoff;
  CUDA_TRY(ecnt.alloc(nv + 1, st));
  CUDA_TRY(eoff.alloc(nv + 1, st));
  // d_small: [0] overflow flag, [1] interval count, [4] (min start, max end),
  // [6..7] size-key range for the placement order — one readback for all
  int *d_over = (int *)ctx->d_small;
  int *d_mm = (int *)(ctx->d_small + 4);
  unsigned long long *d_kmm = (unsigned long long *)(ctx->d_small + 6);
  CUDA_TRY(cudaMemsetAsync(d_over, 0, 4, st));
  int mm_init[2] = {INT32_MAX, INT32_MIN};
  CUDA_TRY(cudaMemcpyAsync(d_mm, mm_init, 8, cudaMemcpyHostToDevice, st));
  int rc = placement_rank_keys(ctx, nv, g->size.p, d_kmm, err);
  if (rc) return rc;
  LAUNCH(ctx, norm, grid_for(nv, 128), 128, 0, nv, seg_off_d, lo_d, hi_d, ecnt.p, (int32_t *)nullptr,
         d_mm, d_over, 0, (const int64_t *)nullptr, (int32_t *)nullptr);
  int64_t *d_tot = ctx->d_small + 1;
  rc = dev_exclusive_scan<int64_t>(ctx, ecnt.p, eoff.p, nv, d_tot, err);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(eoff.p + nv, d_tot, 8, cudaMemcpyDeviceToDevice, st));
  int64_t h[8];
  rc = dev_read_n(ctx, ctx->d_small, h, 64, err);
  if (rc) return rc;
  if ((int)h[0]) {
    mp_set_err(err, MP_E_UNSUPPORTED, 0, MAXSEG, 0, "more than 64 segments on one variable");
    return MP_E_UNSUPPORTED;
  }
  int64_t ni = h[1];
  int mm[2];
  memcpy(mm, &h[4], 8);
  if (nv) {
    // size keys are descending-order encodings: kmin holds the largest size
    g->size_hi = (int64_t)(~(uint64_t)h[6] ^ 0x8000000000000000ull);
    g->size_lo = (int64_t)(~(uint64_t)h[7] ^ 0x8000000000000000ull);
    rc = placement_rank_sort(ctx, nv, g->size.p, g->tiekey.p, g->rank.p, (uint64_t)h[6], (uint64_t)h[7], err);
    if (rc) return rc;
  }
  DBuf<int32_t> ea, eb, ivar, sv, scur;
  CUDA_TRY(ea.alloc(ni, st)); CUDA_TRY(eb.alloc(ni, st)); CUDA_TRY(ivar.alloc(ni, st));
  CUDA_TRY(sv.alloc(3 * ni, st)); CUDA_TRY(scur.alloc(nv, st));
  LAUNCH(ctx, norm, grid_for(nv, 128), 128, 0, nv, seg_off_d, lo_d, hi_d, ecnt.p, ea.p, eb.p,
         d_over, 1, eoff.p, ivar.p);
  // order intervals by start.  Interval bounds are op positions, so when
  // their range is small a counting sort does it (order among equal starts
  // is irrelevant: each overlapping pair is still emitted exactly once); the
  // backward counts then need only a histogram of ends, no sorted copy.
  DBuf<uint32_t> skey, perm;
  CUDA_TRY(skey.alloc(ni, st)); CUDA_TRY(perm.alloc(ni, st));
  DBuf<int64_t> cnt, sub_off;
  CUDA_TRY(cnt.alloc(ni + 1, st));
  CUDA_TRY(sub_off.alloc(ni + 1, st));
  int64_t range = ni ? (int64_t)mm[1] - mm[0] + 1 : 1;
  if (range <= 8 * ni + 4096) {
    DBuf<int32_t> hs, he, offs_s, cum_e, curs;
    CUDA_TRY(hs.alloc(range + 1, st)); CUDA_TRY(he.alloc(range + 2, st)); CUDA_TRY(offs_s.alloc(range + 1, st));
    CUDA_TRY(cum_e.alloc(range + 2, st)); CUDA_TRY(curs.alloc(range + 1, st));
    CUDA_TRY(cudaMemsetAsync(hs.p, 0, (range + 1) * 4, st));
    CUDA_TRY(cudaMemsetAsync(he.p, 0, (range + 2) * 4, st));
    CUDA_TRY(cudaMemsetAsync(curs.p, 0, (range + 1) * 4, st));
    LAUNCH(ctx, k_iv_hist, grid_for(ni, 256), 256, 0, ni, ea.p, eb.p, mm[0], hs.p, he.p);
    rc = dev_exclusive_scan<int32_t>(ctx, hs.p, offs_s.p, range + 1, nullptr, err);
    if (rc) return rc;
    rc = dev_exclusive_scan<int32_t>(ctx, he.p, cum_e.p, range + 2, nullptr, err);
    if (rc) return rc;
    LAUNCH(ctx, k_iv_scatter, grid_for(ni, 256), 256, 0, ni, ea.p, mm[0], offs_s.p, curs.p, perm.p);
    LAUNCH(ctx, k_iv_counts_dense, grid_for(ni, 256), 256, 0, ni, perm.p, ea.p, eb.p, mm[0], offs_s.p, cum_e.p,
           cnt.p, ivar.p, g->rank.p, sv.p);
  } else {
    DBuf<uint32_t> ekey, edummy;
    CUDA_TRY(ekey.alloc(ni, st)); CUDA_TRY(edummy.alloc(ni, st));
    LAUNCH(ctx, k_iv_keys, grid_for(ni, 256), 256, 0, ni, ea.p, skey.p, perm.p);
    LAUNCH(ctx, k_iv_keys, grid_for(ni, 256), 256, 0, ni, eb.p, ekey.p, edummy.p);
    rc = dev_radix_sort_u32(ctx, skey.p, perm.p, ni, 32, err);
    if (rc) return rc;
    rc = dev_radix_sort_u32(ctx, ekey.p, edummy.p, ni, 32, err);
    if (rc) return rc;
    LAUNCH(ctx, k_iv_counts, grid_for(ni, 256), 256, 0, ni, skey.p, perm.p, ekey.p, eb.p, cnt.p, ivar.p, g->rank.p,
           sv.p);
  }
  rc = dev_exclusive_scan<int64_t>(ctx, cnt.p, sub_off.p, ni, d_tot, err);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(sub_off.p + ni, d_tot, 8, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(g->row_off.alloc(nv + 1, st));
  LAUNCH(ctx, k_row_off, grid_for(nv + 1, 256), 256, 0, nv, eoff.p, sub_off.p, g->row_off.p);
  // placement scratch for rows longer than the register sorts (degree bounds
  // the predecessor count), read back with nnz
  unsigned long long *d_arena = (unsigned long long *)(ctx->d_small + 2);
  CUDA_TRY(cudaMemsetAsync(d_arena, 0, 8, st));
  LAUNCH(ctx, k_arena_need, grid_for(nv, 256, 2048), 256, 0, nv, g->row_off.p, d_arena);
  int64_t h2[2];
  rc = dev_read_n(ctx, d_tot, h2, 16, err);
  if (rc) return rc;
  int64_t nnz = h2[0];
  g->nvars = nv;
  g->nnz = nnz;
  g->arena_need = h2[1];
  CUDA_TRY(g->col.alloc(nnz, st));
  CUDA_TRY(cudaMemsetAsync(scur.p, 0, nv * 4, st));
  CUDA_TRY(cudaMemsetAsync(g->pcnt.p, 0, nv * 4, st));
  tm.reset();
  StageTimer fill(ctx, MP_ST_CONFLICT_FILL);
  LAUNCH(ctx, k_iv_fill, grid_for(ni * 32, 256, 148 * 64), 256, 0, ni, sv.p, g->row_off.p, g->pcnt.p, scur.p,
         g->col.p);
  return MP_OK;
}

__global__ void k_prof_segs(int64_t nv, const int32_t *nseg, const int32_t *seg, int64_t *seg_off,
                            int32_t *lo, int32_t *hi) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    seg_off[v] = 2 * v;
    int ns = nseg[v];
    lo[2 * v] = seg[4 * v]; hi[2 * v] = seg[4 * v + 1];
    lo[2 * v + 1] = ns > 1 ? seg[4 * v + 2] : 0;
    hi[2 * v + 1] = ns > 1 ? seg[4 * v + 3] : 0;  // empty when absent
    if (v == nv - 1) seg_off[nv] = 2 * nv;
  }
}

// ---------------------------------------------------------------------------
// Profile fast path.  A profile variable has one or two segments with bounds
// in [0, period], so its effective intervals (at most two) get fixed slots
// 2v, 2v+1 and need no counting pass or offset scan; one kernel computes
// them, histograms their starts and ends for the counting sort (bounds are
// op positions: base 0, range period + 1) and reduces the size-key range
// the placement order needs, so the build reads back once before the
// placement-order sort instead of twice.

// effective intervals of one <= 2-segment variable (k_norm_count's rule):
// returns their count, intervals in (a0, b0), (a1, b1)
__device__ __forceinline__ int prof_effective(int ns, int4 sg, int32_t &a0, int32_t &b0, int32_t &a1, int32_t &b1) {
  int32_t l0 = 0, h0 = 0, l1 = 0, h1 = 0;
  int mm = 0;
  for (int q = 0; q < ns; q++) {
    const int32_t a = q ? sg.z : sg.x, b = q ? sg.w : sg.y;
    if (b <= a) continue;
    if (mm == 0) { l0 = a; h0 = b; }
    else if (a < l0) { l1 = l0; h1 = h0; l0 = a; h0 = b; }
    else { l1 = a; h1 = b; }
    mm++;
  }
  int c = 0;
  int32_t cur_end = INT32_MIN;
  for (int k = 0; k < mm; k++) {
    const int32_t lk = k ? l1 : l0;
    if (lk < cur_end) continue;
    int32_t ne = INT32_MAX;
    if (h0 > lk && h0 < ne) ne = h0;
    if (mm > 1 && h1 > lk && h1 < ne) ne = h1;
    if (c == 0) { a0 = lk; b0 = ne; } else { a1 = lk; b1 = ne; }
    c++;
    cur_end = ne;
  }
  return c;
}

// hse[x]: starts at x in the low 32 bits, ends at x in the high 32 bits, so
// ONE 64-bit scan gives both prefix counts (the low sum never carries: fewer
// than 2^31 intervals)
__global__ void k_prof_intervals(int64_t nv, const int32_t *nseg, const int32_t *seg, const int64_t *size,
                                 int32_t *ea, int32_t *eb, int64_t *cnt, unsigned long long *hse,
                                 unsigned long long *kmm, int32_t *curs, int64_t ncurs,
                                 unsigned long long *arena, unsigned long long *cells, unsigned int *finished) {
  PDL_WAIT();
  // scratch the later kernels of the build count into (no memsets)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncurs; i += (int64_t)gridDim.x * blockDim.x)
    curs[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *arena = 0;
  unsigned long long lmn = ~0ull, lmx = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int4 sg = reinterpret_cast<const int4 *>(seg)[v];
    int32_t a0 = -1, b0 = -1, a1 = -1, b1 = -1;
    const int c = prof_effective(nseg[v], sg, a0, b0, a1, b1);
    reinterpret_cast<int2 *>(ea)[v] = make_int2(c > 0 ? a0 : -1, c > 1 ? a1 : -1);
    reinterpret_cast<int2 *>(eb)[v] = make_int2(b0, b1);
    if (c > 0) { atomicAdd(&hse[a0], 1ull); atomicAdd(&hse[b0], 1ull << 32); }
    if (c > 1) { atomicAdd(&hse[a1], 1ull); atomicAdd(&hse[b1], 1ull << 32); }
    cnt[2 * v] = 0;
    cnt[2 * v + 1] = 0;
    const uint64_t k = desc_size_key(size[v]);
    lmn = k < lmn ? k : lmn;
    lmx = k > lmx ? k : lmx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(FULL_MASK, lmn, o), y = __shfl_xor_sync(FULL_MASK, lmx, o);
    lmn = x < lmn ? x : lmn;
    lmx = y > lmx ? y : lmx;
  }
  // per-block pairs, reduced by the last block to finish (the range needs
  // no initialised cell, so no memset ahead of the kernel)
  __shared__ unsigned long long smn[32], smx[32];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) { smn[w] = lmn; smx[w] = lmx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; i++) {
      lmn = smn[i] < lmn ? smn[i] : lmn;
      lmx = smx[i] > lmx ? smx[i] : lmx;
    }
    cells[blockIdx.x] = lmn;
    cells[gridDim.x + blockIdx.x] = lmx;
    __threadfence();
    last = atomicAdd(finished, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  lmn = ~0ull;
  lmx = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const unsigned long long x = *(volatile unsigned long long *)&cells[b];
    const unsigned long long y = *(volatile unsigned long long *)&cells[gridDim.x + b];
    lmn = x < lmn ? x : lmn;
    lmx = y > lmx ? y : lmx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(FULL_MASK, lmn, o), y = __shfl_xor_sync(FULL_MASK, lmx, o);
    lmn = x < lmn ? x : lmn;
    lmx = y > lmx ? y : lmx;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) { smn[w] = lmn; smx[w] = lmx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; i++) {
      lmn = smn[i] < lmn ? smn[i] : lmn;
      lmx = smx[i] > lmx ? smx[i] : lmx;
    }
    kmm[0] = lmn;
    kmm[1] = lmx;
    *finished = 0;  // ready for the next build
  }
}

// slots in start order (counting sort; order among equal starts is free)
__global__ void k_prof_scatter(int64_t nslots, const int32_t *ea, const int64_t *pref, int32_t *cur, uint32_t *perm) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = ea[i];
    if (x >= 0) perm[(int32_t)(uint32_t)pref[x] + atomicAdd(&cur[x], 1)] = (uint32_t)i;
  }
}

// k_iv_counts_dense with the slot's variable implicit (slot >> 1)
// (the interval count is read on the device: the low half of the packed
// start/end total; the rank column of sv is written by k_prof_sv_rank once
// the size order exists)
__global__ void k_prof_counts(const int64_t *d_ni, const uint32_t *perm, const int32_t *ea, const int32_t *eb,
                              const int64_t *pref, int64_t *cnt, int32_t *sv) {
  PDL_WAIT();
  const int64_t n = (int64_t)(uint32_t)*d_ni;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t iid = perm[k];
    const int64_t f = (int64_t)(uint32_t)pref[eb[iid]] - k - 1;       // starts before the end
    const int64_t bw = k - (int64_t)(pref[ea[iid] + 1] >> 32);         // ends at or before the start
    cnt[iid] = f + bw;
    const int32_t v = (int32_t)(iid >> 1);
    sv[3 * k] = v;
    sv[3 * k + 2] = (int32_t)f;
  }
}

__global__ void k_prof_sv_rank(int64_t n, const int32_t *rank, int32_t *sv) {
  PDL_WAIT();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    sv[3 * k + 1] = rank[sv[3 * k]];
}

// row bounds from the slot scan, and the long-row scratch bound
// (sub_off has 2 nv entries; its total, the slot scan's, is read from *tot)
__global__ void k_prof_rows(int64_t nv, const int64_t *sub_off, const int64_t *tot, int64_t *row_off,
                            unsigned long long *need, int32_t *scur, int32_t *pcnt) {
  PDL_WAIT();
  unsigned long long s = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = v < nv ? sub_off[2 * v] : *tot;
    row_off[v] = r0;
    if (v < nv) {
      scur[v] = 0;  // the fill's row cursors
      pcnt[v] = 0;
      const int64_t d = (v + 1 < nv ? sub_off[2 * v + 2] : *tot) - r0;
      if (d > 128) {
        unsigned long long n2 = 64;
        while (n2 < (unsigned long long)d) n2 <<= 1;
        s += n2;
      }
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(need, s);
}

static int build_csr_profile(mp_ctx *ctx, mp_dprofile *P, mp_dgraph *g, mp_err *err) {
  cudaStream_t st = ctx->stream;
  const int64_t nv = P->d.nvars, p = P->d.period, ns = 2 * nv;
  CUDA_TRY(g->rank.alloc(nv, st));
  CUDA_TRY(g->pcnt.alloc(nv, st));
  std::unique_ptr<StageTimer> tm(new StageTimer(ctx, MP_ST_CONFLICT_PREP));
  DBuf<int32_t> ea, eb, curs, sv, scur;
  DBuf<int64_t> cnt, sub_off, hse, pref;
  CUDA_TRY(ea.alloc(ns, st)); CUDA_TRY(eb.alloc(ns, st));
  CUDA_TRY(hse.alloc(p + 2, st)); CUDA_TRY(pref.alloc(p + 2, st)); CUDA_TRY(curs.alloc(p + 1, st));
  CUDA_TRY(cnt.alloc(ns + 1, st)); CUDA_TRY(sub_off.alloc(ns + 1, st));
  CUDA_TRY(cudaMemsetAsync(hse.p, 0, (p + 2) * 8, st));
  // d_small: [0..1] size-key range, [2] interval count, [3] arena need, [4] nnz
  unsigned long long *d_kmm = (unsigned long long *)ctx->d_small;
  int64_t *d_ni = ctx->d_small + 2;
  unsigned long long *d_arena = (unsigned long long *)(ctx->d_small + 3);
  const unsigned ib = grid_for(nv, 256, (int64_t)ctx->num_sms * 8);
  DBuf<unsigned long long> kcells;
  CUDA_TRY(kcells.alloc(2 * (int64_t)ib, st));
  LAUNCH(ctx, k_prof_intervals, ib, 256, 0, nv, P->nseg.p, P->seg.p, P->size.p, ea.p, eb.p, cnt.p,
         (unsigned long long *)hse.p, d_kmm, curs.p, p + 1, d_arena, kcells.p, (unsigned int *)(ctx->d_small + 62));
  int rc = dev_exclusive_scan<int64_t>(ctx, hse.p, pref.p, p + 2, d_ni, err);
  if (rc) return rc;
  // everything up to the row bounds runs without the host: buffers indexed
  // by sorted interval are sized for every slot that can hold one (ni <= ns)
  DBuf<uint32_t> perm;
  CUDA_TRY(perm.alloc(ns, st)); CUDA_TRY(sv.alloc(3 * ns, st)); CUDA_TRY(scur.alloc(nv, st));
  LAUNCH(ctx, k_prof_scatter, grid_for(ns, 256), 256, 0, ns, ea.p, pref.p, curs.p, perm.p);
  LAUNCH(ctx, k_prof_counts, grid_for(ns, 256), 256, 0, d_ni, perm.p, ea.p, eb.p, pref.p, cnt.p, sv.p);
  int64_t *d_tot = ctx->d_small + 4;
  rc = dev_exclusive_scan<int64_t>(ctx, cnt.p, sub_off.p, ns, d_tot, err);
  if (rc) return rc;
  CUDA_TRY(g->row_off.alloc(nv + 1, st));
  LAUNCH(ctx, k_prof_rows, grid_for(nv + 1, 256, 2048), 256, 0, nv, sub_off.p, d_tot, g->row_off.p, d_arena,
         scur.p, g->pcnt.p);
  // one readback: size-key range, interval count, long-row scratch, nnz
  int64_t h[5];
  rc = dev_read_n(ctx, ctx->d_small, h, 40, err);
  if (rc) return rc;
  const int64_t ni = (int64_t)(uint32_t)h[2];  // low half of the packed total: the interval count
  g->size_hi = (int64_t)(~(uint64_t)h[0] ^ 0x8000000000000000ull);
  g->size_lo = (int64_t)(~(uint64_t)h[1] ^ 0x8000000000000000ull);
  g->nvars = nv;
  g->nnz = h[4];
  g->arena_need = h[3];
  CUDA_TRY(g->col.alloc(g->nnz, st));
  rc = placement_rank_sort(ctx, nv, g->size.p, nullptr, g->rank.p, (uint64_t)h[0], (uint64_t)h[1], err);
  if (rc) return rc;
  LAUNCH(ctx, k_prof_sv_rank, grid_for(ni, 256), 256, 0, ni, g->rank.p, sv.p);

  tm.reset();
  StageTimer fill(ctx, MP_ST_CONFLICT_FILL);
  LAUNCH(ctx, k_iv_fill, grid_for(ni * 32, 256, 148 * 64), 256, 0, ni, sv.p, g->row_off.p, g->pcnt.p, scur.p,
         g->col.p);
  return MP_OK;
}

#ifndef CONFLICT_PROFILE_FAST
#define CONFLICT_PROFILE_FAST 1
#endif

extern "C" int mp_conflict_from_profile(mp_ctx *ctx, mp_dprofile *P, mp_dgraph **out, mp_err *err) {
  CTX_GUARD(ctx);
  cudaStream_t st = ctx->stream;
  int64_t nv = P->d.nvars;
  if (CONFLICT_PROFILE_FAST && nv > 0 && P->d.period + 1 <= 16 * nv + 4096 && 2 * nv < INT32_MAX) {
    mp_dgraph *g = new mp_dgraph();
    g->ctx = ctx;
    CUDA_TRY(g->size.alloc(nv, st));
    CUDA_TRY(cudaMemcpyAsync(g->size.p, P->size.p, nv * 8, cudaMemcpyDeviceToDevice, st));
    int rc = build_csr_profile(ctx, P, g, err);
    if (rc) { delete g; return rc; }
    rc = profile_dims(ctx, P, err);  // drained by the build's readbacks: no wait
    if (rc) { delete g; return rc; }
    g->peak_hint = P->d.peak_bytes;
    *out = g;
    return MP_OK;
  }
  DBuf<int64_t> so;
  DBuf<int32_t> lo, hi;
  CUDA_TRY(so.alloc(nv + 1, st)); CUDA_TRY(lo.alloc(2 * nv, st)); CUDA_TRY(hi.alloc(2 * nv, st));
  if (nv == 0) CUDA_TRY(cudaMemsetAsync(so.p, 0, 8, st));
  else LAUNCH(ctx, k_prof_segs, grid_for(nv, 256), 256, 0, nv, P->nseg.p, P->seg.p, so.p, lo.p, hi.p);
  mp_dgraph *g = new mp_dgraph();
  g->ctx = ctx;
  CUDA_TRY(g->size.alloc(nv, st));
  if (nv) CUDA_TRY(cudaMemcpyAsync(g->size.p, P->size.p, nv * 8, cudaMemcpyDeviceToDevice, st));
  // profile variables are already in (alloc or -1, name) order: the
  // placement tie-break is the vertex index
  int rc = build_csr(ctx, nv, so.p, lo.p, hi.p, false, g, err);
  if (rc) { delete g; return rc; }
  rc = profile_dims(ctx, P, err);
  if (rc) { delete g; return rc; }
  g->peak_hint = P->d.peak_bytes;
  *out = g;
  return MP_OK;
}

extern "C" int mp_conflict_from_arcs(mp_ctx *ctx, int32_t nvars, const int64_t *size, const int64_t *tiekey,
                                     const int64_t *seg_off, const int32_t *seg_lo, const int32_t *seg_hi,
                                     mp_dgraph **out, mp_err *err) {
  CTX_GUARD(ctx);
  cudaStream_t st = ctx->stream;
  int64_t nv = nvars, ns = seg_off[nvars];
  DBuf<int64_t> so;
  DBuf<int32_t> lo, hi;
  CUDA_TRY(so.alloc(nv + 1, st)); CUDA_TRY(lo.alloc(ns, st)); CUDA_TRY(hi.alloc(ns, st));
  CUDA_TRY(cudaMemcpyAsync(so.p, seg_off, (nv + 1) * 8, cudaMemcpyHostToDevice, st));
  if (ns) {
    CUDA_TRY(cudaMemcpyAsync(lo.p, seg_lo, ns * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(hi.p, seg_hi, ns * 4, cudaMemcpyHostToDevice, st));
  }
  mp_dgraph *g = new mp_dgraph();
  g->ctx = ctx;
  CUDA_TRY(g->size.alloc(nv, st));
  CUDA_TRY(g->tiekey.alloc(nv, st));
  if (nv) {
    CUDA_TRY(cudaMemcpyAsync(g->size.p, size, nv * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(g->tiekey.p, tiekey, nv * 8, cudaMemcpyHostToDevice, st));
  }
  int rc = build_csr(ctx, nv, so.p, lo.p, hi.p, true, g, err);
  if (rc) { delete g; return rc; }
  CUDA_TRY(cudaStreamSynchronize(st));  // host arrays are only borrowed for the call
  *out = g;
  return MP_OK;
}

extern "C" int mp_graph_dims(mp_dgraph *g, int64_t *nvars, int64_t *nnz) {
  CTX_GUARD(g->ctx);
  *nvars = g->nvars;
  *nnz = g->nnz;
  return MP_OK;
}

extern "C" int mp_graph_download(mp_ctx *ctx, mp_dgraph *g, int64_t *row_off, int32_t *col, mp_err *err) {
  CTX_GUARD(ctx);
  CUDA_TRY(cudaMemcpyAsync(row_off, g->row_off.p, (g->nvars + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (g->nnz) CUDA_TRY(cudaMemcpyAsync(col, g->col.p, g->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MP_OK;
}

extern "C" int mp_graph_free(mp_dgraph *g) {
  CTX_GUARD(g->ctx);
  delete g;
  return MP_OK;
}

// rows of a host CSR split by placement order (warp per row)
__global__ void k_partition_rows(int64_t V, const int64_t *row_off, const int32_t *col_in, const int32_t *rank,
                                 int32_t *col, int32_t *pcnt) {
  PDL_WAIT();
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = lanemask_lt();
  for (int64_t v = warp; v < V; v += nwarps) {
    int64_t rb = row_off[v], deg = row_off[v + 1] - rb;
    int32_t rv = rank[v];
    int32_t pc = 0, sc = 0;
    for (int64_t base = 0; base < deg; base += 32) {
      int64_t idx = base + lane;
      bool valid = idx < deg;
      int32_t j = valid ? col_in[rb + idx] : 0;
      bool isp = valid && rank[j] < rv;
      unsigned bp = __ballot_sync(FULL_MASK, isp);
      unsigned bs = __ballot_sync(FULL_MASK, valid && !isp);
      if (isp) col[rb + pc + __popc(bp & lt)] = j;
      else if (valid) col[rb + deg - 1 - (sc + __popc(bs & lt))] = j;
      pc += __popc(bp);
      sc += __popc(bs);
    }
    if (lane == 0) pcnt[v] = pc;
  }
}

// The device placement counts, per vertex, the neighbours placed before it
// and is released by each of them, so it needs each row to hold exactly the
// vertex's earlier-placed neighbours plus the later-placed vertices that
// list it.  A caller's graph need not be symmetric: the reference reads only
// adj[i] when placing i (smartpool.py:131-135), so u constrains v iff
// u in adj[v] and u precedes v.  Rebuild that relation, mirrored, on the
// host (self loops and duplicates dropped, ids checked).
static int normalize_host_csr(int64_t nv, const int64_t *row_off, const int32_t *col, const int64_t *size,
                              const int64_t *tiekey, std::vector<int64_t> &row_out, std::vector<int32_t> &col_out,
                              mp_err *err) {
  std::vector<int64_t> pos(nv);
  {
    std::vector<int32_t> order(nv);
    for (int64_t i = 0; i < nv; i++) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      if (size[a] != size[b]) return size[a] > size[b];
      int64_t ta = tiekey ? tiekey[a] : a, tb = tiekey ? tiekey[b] : b;
      return ta < tb;
    });
    for (int64_t k = 0; k < nv; k++) pos[order[k]] = k;
  }
  std::vector<std::pair<int32_t, int32_t>> pairs;
  pairs.reserve((size_t)row_off[nv] * 2);
  for (int64_t v = 0; v < nv; v++) {
    if (row_off[v + 1] < row_off[v]) {
      mp_set_err(err, MP_E_VALUE, v, row_off[v], row_off[v + 1], "row offsets must be non-decreasing");
      return MP_E_VALUE;
    }
    for (int64_t e = row_off[v]; e < row_off[v + 1]; e++) {
      int32_t u = col[e];
      if (u < 0 || u >= nv) {
        mp_set_err(err, MP_E_VALUE, v, u, e, "list index out of range");
        return MP_E_VALUE;
      }
      if (pos[u] < pos[v]) {
        pairs.push_back({(int32_t)v, u});
        pairs.push_back({u, (int32_t)v});
      }
    }
  }
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  row_out.assign(nv + 1, 0);
  col_out.resize(pairs.size());
  for (size_t k = 0; k < pairs.size(); k++) {
    row_out[pairs[k].first + 1]++;
    col_out[k] = pairs[k].second;
  }
  for (int64_t v = 0; v < nv; v++) row_out[v + 1] += row_out[v];
  return MP_OK;
}

extern "C" int mp_graph_from_csr(mp_ctx *ctx, int32_t nvars, const int64_t *row_off_in, const int32_t *col_in,
                                 const int64_t *size, const int64_t *tiekey, mp_dgraph **out, mp_err *err) {
  CTX_GUARD(ctx);
  cudaStream_t st = ctx->stream;
  int64_t nv = nvars;
  std::vector<int64_t> row_v;
  std::vector<int32_t> col_v;
  int nrc = normalize_host_csr(nv, row_off_in, col_in, size, tiekey, row_v, col_v, err);
  if (nrc) return nrc;
  const int64_t *row_off = row_v.data();
  const int32_t *col = col_v.data();
  int64_t nnz = row_off[nv];
  mp_dgraph *g = new mp_dgraph();
  g->ctx = ctx;
  g->nvars = nv;
  g->nnz = nnz;
  CUDA_TRY(g->size.alloc(nv, st)); CUDA_TRY(g->row_off.alloc(nv + 1, st)); CUDA_TRY(g->col.alloc(nnz, st));
  CUDA_TRY(g->rank.alloc(nv, st)); CUDA_TRY(g->pcnt.alloc(nv, st));
  DBuf<int32_t> cin;
  CUDA_TRY(cin.alloc(nnz, st));
  CUDA_TRY(cudaMemcpyAsync(g->row_off.p, row_off, (nv + 1) * 8, cudaMemcpyHostToDevice, st));
  if (nnz) CUDA_TRY(cudaMemcpyAsync(cin.p, col, nnz * 4, cudaMemcpyHostToDevice, st));
  if (nv) {
    CUDA_TRY(cudaMemcpyAsync(g->size.p, size, nv * 8, cudaMemcpyHostToDevice, st));
    if (tiekey) {
      CUDA_TRY(g->tiekey.alloc(nv, st));
      CUDA_TRY(cudaMemcpyAsync(g->tiekey.p, tiekey, nv * 8, cudaMemcpyHostToDevice, st));
    }
    int rc = placement_rank(ctx, nv, g->size.p, g->tiekey.p, g->rank.p, err);
    if (rc) { delete g; return rc; }
    LAUNCH(ctx, k_partition_rows, grid_for(nv * 32, 256, 148 * 64), 256, 0, nv, g->row_off.p, cin.p, g->rank.p,
           g->col.p, g->pcnt.p);
    unsigned long long *d_arena = (unsigned long long *)(ctx->d_small + 2);
    CUDA_TRY(cudaMemsetAsync(d_arena, 0, 8, st));
    LAUNCH(ctx, k_arena_need, grid_for(nv, 256, 2048), 256, 0, nv, g->row_off.p, d_arena);
    int64_t need;
    rc = dev_read_i64(ctx, (const int64_t *)d_arena, &need, err);
    if (rc) { delete g; return rc; }
    g->arena_need = need;
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  *out = g;
  return MP_OK;
}
