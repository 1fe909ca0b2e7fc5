// placement.cu — SmartPool greedy offset assignment (smartpool.py:91-144).
//
// The reference places variables one at a time in (-size, alloc, name)
// order; each offset depends only on the already-placed neighbours.  A
// variable can therefore be placed as soon as every neighbour that precedes
// it in that order is placed: the placement order defines a DAG, and
// processing it level by level (Kahn wavefronts) reproduces the sequential
// result bit for bit while exposing every independent variable at once.
//
// Per variable, one warp gathers the placed neighbours' [off, off+size)
// ranges, sorts them by (start, end) with a bitonic network (registers for
// <= 32, shared memory up to the per-warp capacity, global scratch beyond),
// and replays _pick_offset (smartpool.py:101-119) as an exclusive max-scan
// of range ends: a hole opens where a start exceeds the running top.
// first_fit takes the lowest qualifying hole (ballot + ffs), best_fit the
// (length, offset) minimum (warp reduction), otherwise the running top.
//
// One persistent cooperative kernel runs all levels with a grid barrier
// between them; tiny graphs use a single CTA and __syncthreads.
#include <cooperative_groups.h>

#include "handles.cuh"

namespace cg = cooperative_groups;

struct IV {
  int64_t s, e;
};

struct PlaceArgs {
  int64_t V;
  const int64_t *row_off;
  const int32_t *col2;  // row partitioned: preds first, then succs
  const int32_t *pcnt;
  const int64_t *size;
  int64_t *off;
  int32_t *remaining;
  int32_t *F0, *F1;
  int32_t *counts;  // 3 rotating frontier counters
  int policy;       // 0 first_fit, 1 best_fit
  int cap;          // shared-memory ranges per warp
  IV *gscratch;
  int64_t gcap;
  int32_t *levels;
};

__device__ __forceinline__ bool iv_less(int64_t as, int64_t ae, int64_t bs, int64_t be) {
  return as < bs || (as == bs && ae < be);
}

__device__ __forceinline__ void warp_bitonic32(int64_t &s, int64_t &e) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      int64_t os = __shfl_xor_sync(FULL_MASK, s, j);
      int64_t oe = __shfl_xor_sync(FULL_MASK, e, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      bool other_less = iv_less(os, oe, s, e);
      bool take_other = (lower == up) ? other_less : iv_less(s, e, os, oe);
      if (take_other) { s = os; e = oe; }
    }
  }
}

__device__ void warp_bitonic_mem(IV *buf, int n2) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < n2; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = (i & k) == 0;
          IV a = buf[i], b = buf[ixj];
          bool sw = up ? iv_less(b.s, b.e, a.s, a.e) : iv_less(a.s, a.e, b.s, b.e);
          if (sw) { buf[i] = b; buf[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
}

struct HoleState {
  int64_t top;       // running max end (starts at 0)
  int64_t best_len;  // best_fit candidate
  int64_t best_off;
  bool found;
};

// one chunk of 32 sorted ranges; returns true when first_fit is decided
__device__ __forceinline__ bool hole_chunk(HoleState &h, int64_t s, int64_t e, bool valid, int64_t need,
                                           int policy) {
  const int lane = threadIdx.x & 31;
  int64_t incl = warp_incl_scan_max(valid ? e : INT64_MIN);
  int64_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
  if (lane == 0) excl = INT64_MIN;
  int64_t tb = excl > h.top ? excl : h.top;
  bool hole = valid && s > tb;
  int64_t len = s - tb;
  bool ok = hole && len >= need;
  unsigned bal = __ballot_sync(FULL_MASK, ok);
  if (policy == 0) {
    if (bal) {
      int first = __ffs(bal) - 1;
      h.best_off = __shfl_sync(FULL_MASK, tb, first);
      h.found = true;
      return true;
    }
  } else if (bal) {
    int64_t bl = ok ? len : INT64_MAX, bo = ok ? tb : INT64_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      int64_t ol = __shfl_xor_sync(FULL_MASK, bl, o), oo = __shfl_xor_sync(FULL_MASK, bo, o);
      if (ol < bl || (ol == bl && oo < bo)) { bl = ol; bo = oo; }
    }
    if (!h.found || bl < h.best_len || (bl == h.best_len && bo < h.best_off)) {
      h.best_len = bl;
      h.best_off = bo;
      h.found = true;
    }
  }
  int64_t cmax = __shfl_sync(FULL_MASK, incl, 31);
  if (cmax > h.top) h.top = cmax;
  return false;
}

__device__ int64_t place_one(const PlaceArgs &a, int64_t v, IV *wbuf, IV *gbuf) {
  const int lane = threadIdx.x & 31;
  int64_t rb = a.row_off[v];
  int m = a.pcnt[v];
  int64_t need = a.size[v];
  if (m == 0) return 0;
  HoleState h{0, 0, 0, false};
  if (m <= 32) {
    int64_t s = INT64_MAX, e = INT64_MAX;
    if (lane < m) {
      int32_t j = a.col2[rb + lane];
      s = __ldcg(&a.off[j]);
      e = s + a.size[j];
    }
    warp_bitonic32(s, e);
    hole_chunk(h, s, e, lane < m, need, a.policy);
  } else {
    IV *buf = m <= a.cap ? wbuf : gbuf;
    int n2 = 64;
    while (n2 < m) n2 <<= 1;
    for (int i = lane; i < n2; i += 32) {
      IV x{INT64_MAX, INT64_MAX};
      if (i < m) {
        int32_t j = a.col2[rb + i];
        x.s = __ldcg(&a.off[j]);
        x.e = x.s + a.size[j];
      }
      buf[i] = x;
    }
    __syncwarp();
    warp_bitonic_mem(buf, n2);
    for (int base = 0; base < m; base += 32) {
      int i = base + lane;
      IV x = i < m ? buf[i] : IV{0, 0};
      if (hole_chunk(h, x.s, x.e, i < m, need, a.policy)) break;
    }
    __syncwarp();
  }
  return h.found ? h.best_off : h.top;
}

template <bool GRID>
__global__ void __launch_bounds__(256) k_place(PlaceArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  IV *sbuf = (IV *)smem_raw;
  const int lane = threadIdx.x & 31;
  IV *wbuf = sbuf + (threadIdx.x >> 5) * a.cap;
  int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  IV *gbuf = a.gscratch ? a.gscratch + gwarp * a.gcap : nullptr;
  bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  int r = 0;
  for (;;) {
    int n = __ldcg(&a.counts[r % 3]);
    if (n == 0) break;
    const int32_t *cur = (r & 1) ? a.F1 : a.F0;
    int32_t *nxt = (r & 1) ? a.F0 : a.F1;
    if (leader) a.counts[(r + 2) % 3] = 0;
    for (int64_t q = gwarp; q < n; q += nwarps) {
      int32_t v = __ldcg(&cur[q]);
      int64_t o = place_one(a, v, wbuf, gbuf);
      if (lane == 0) a.off[v] = o;
      __threadfence();
      int64_t rb = a.row_off[v], deg = a.row_off[v + 1] - rb;
      for (int64_t i = a.pcnt[v] + lane; i < deg; i += 32) {
        int32_t j = a.col2[rb + i];
        if (atomicSub(&a.remaining[j], 1) == 1) {
          int slot = atomicAdd(&a.counts[(r + 1) % 3], 1);
          nxt[slot] = j;
        }
      }
    }
    if (GRID) {
      __threadfence();
      cg::this_grid().sync();
    } else {
      __threadfence_block();
      __syncthreads();
    }
    r++;
  }
  if (leader) *a.levels = r;
}

// ---------------------------------------------------------------------------
// placement order and row partition

__global__ void k_tie_keys(int64_t V, const int64_t *tiekey, uint64_t *keys, uint32_t *vals) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    keys[v] = (uint64_t)tiekey[v] ^ 0x8000000000000000ull;
    vals[v] = (uint32_t)v;
  }
}

// descending size as an ascending unsigned key
__device__ __forceinline__ uint64_t desc_size_key(int64_t s) { return ~((uint64_t)s ^ 0x8000000000000000ull); }

__global__ void k_size_keys(int64_t V, const int64_t *size, const uint32_t *vals, uint64_t *keys,
                            unsigned long long *mn, unsigned long long *mx) {
  unsigned long long lmn = ~0ull, lmx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = desc_size_key(size[vals[i]]);
    keys[i] = k;
    lmn = k < lmn ? k : lmn;
    lmx = k > lmx ? k : lmx;
  }
  atomicMin(mn, lmn);
  atomicMax(mx, lmx);
}

__global__ void k_sub_keys(int64_t V, uint64_t *keys, const unsigned long long *mn) {
  uint64_t m = *mn;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] -= m;
}

__global__ void k_iota(int64_t V, uint32_t *vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    vals[i] = (uint32_t)i;
}

__global__ void k_rank(int64_t V, const uint32_t *order, int32_t *rank) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < V; q += (int64_t)gridDim.x * blockDim.x)
    rank[order[q]] = (int32_t)q;
}

__global__ void k_partition(int64_t V, const int64_t *row_off, const int32_t *col, const int32_t *rank,
                            int32_t *col2, int32_t *pcnt, int32_t *remaining, int32_t *F0, int32_t *count0,
                            int32_t *maxpred) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < V; v += nwarps) {
    int64_t rb = row_off[v], deg = row_off[v + 1] - rb;
    int32_t rv = rank[v];
    int32_t pc = 0, sc = 0;
    for (int64_t base = 0; base < deg; base += 32) {
      int64_t idx = base + lane;
      bool valid = idx < deg;
      int32_t j = valid ? col[rb + idx] : 0;
      bool isp = valid && rank[j] < rv;
      unsigned bp = __ballot_sync(FULL_MASK, isp);
      unsigned bs = __ballot_sync(FULL_MASK, valid && !isp);
      if (isp) col2[rb + pc + __popc(bp & lanemask_lt())] = j;
      else if (valid) col2[rb + deg - 1 - (sc + __popc(bs & lanemask_lt()))] = j;
      pc += __popc(bp);
      sc += __popc(bs);
    }
    if (lane == 0) {
      pcnt[v] = pc;
      remaining[v] = pc;
      atomicMax(maxpred, pc);
      if (pc == 0) F0[atomicAdd(count0, 1)] = (int32_t)v;
    }
  }
}

__global__ void k_footprint(int64_t V, const int64_t *off, const int64_t *size, long long *fp) {
  long long m = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    long long e = off[i] + size[i];
    if (e > m) m = e;
  }
  for (int o = 16; o; o >>= 1) {
    long long u = __shfl_xor_sync(FULL_MASK, m, o);
    if (u > m) m = u;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(fp, m);
}

extern "C" int mp_plan_pool(mp_ctx *ctx, mp_dgraph *g, int32_t policy, int64_t *offsets, int64_t *footprint,
                            int64_t *levels, mp_err *err) {
  if (policy != 0 && policy != 1) {
    mp_set_err(err, MP_E_VALUE, 0, policy, 0, "unknown policy");
    return MP_E_VALUE;
  }
  cudaStream_t st = ctx->stream;
  int64_t V = g->nvars;
  if (V == 0) {
    *footprint = 0;
    if (levels) *levels = 0;
    return MP_OK;
  }
  // placement order: sort by tie key (when given), then stable by -size
  DBuf<uint64_t> keys;
  DBuf<uint32_t> order;
  CUDA_TRY(keys.alloc(V, st));
  CUDA_TRY(order.alloc(V, st));
  int rc;
  if (g->tiekey.p) {
    LAUNCH(ctx, k_tie_keys, grid_for(V, 256), 256, 0, V, g->tiekey.p, keys.p, order.p);
    rc = dev_radix_sort_u64(ctx, keys.p, order.p, V, 64, err);
    if (rc) return rc;
  } else {
    LAUNCH(ctx, k_iota, grid_for(V, 256), 256, 0, V, order.p);
  }
  unsigned long long *d_mn = (unsigned long long *)ctx->d_small, *d_mx = d_mn + 1;
  CUDA_TRY(cudaMemsetAsync(d_mn, 0xff, 8, st));
  CUDA_TRY(cudaMemsetAsync(d_mx, 0, 8, st));
  LAUNCH(ctx, k_size_keys, grid_for(V, 256, 1024), 256, 0, V, g->size.p, order.p, keys.p, d_mn, d_mx);
  uint64_t mm[2];
  rc = dev_read_n(ctx, d_mn, mm, 16, err);
  if (rc) return rc;
  LAUNCH(ctx, k_sub_keys, grid_for(V, 256), 256, 0, V, keys.p, d_mn);
  rc = dev_radix_sort_u64(ctx, keys.p, order.p, V, bits_for(mm[1] - mm[0]), err);
  if (rc) return rc;
  DBuf<int32_t> rank, col2, pcnt, remaining, F0, F1, counts;
  CUDA_TRY(rank.alloc(V, st)); CUDA_TRY(col2.alloc(g->nnz, st)); CUDA_TRY(pcnt.alloc(V, st));
  CUDA_TRY(remaining.alloc(V, st)); CUDA_TRY(F0.alloc(V, st)); CUDA_TRY(F1.alloc(V, st));
  CUDA_TRY(counts.alloc(8, st));
  CUDA_TRY(cudaMemsetAsync(counts.p, 0, 32, st));
  LAUNCH(ctx, k_rank, grid_for(V, 256), 256, 0, V, order.p, rank.p);
  int32_t *d_maxpred = counts.p + 4;
  LAUNCH(ctx, k_partition, grid_for(V * 32, 256, 148 * 64), 256, 0, V, g->row_off.p, g->col.p, rank.p, col2.p,
         pcnt.p, remaining.p, F0.p, counts.p, d_maxpred);
  int32_t maxpred;
  rc = dev_read_n(ctx, d_maxpred, &maxpred, 4, err);
  if (rc) return rc;
  DBuf<int64_t> off;
  CUDA_TRY(off.alloc(V, st));
  const int cap = 256;
  const int threads = 256;
  size_t smem = (size_t)(threads / 32) * cap * sizeof(IV);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_place<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_place<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  bool grid_mode = V > 4096;
  int nblocks = 1;
  if (grid_mode) {
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_place<true>, threads, smem));
    if (per_sm < 1) per_sm = 1;
    nblocks = per_sm * ctx->num_sms;
  }
  DBuf<IV> gscratch;
  int64_t gcap = 0;
  if (maxpred > cap) {
    gcap = 64;
    while (gcap < maxpred) gcap <<= 1;
    CUDA_TRY(gscratch.alloc(gcap * (int64_t)nblocks * (threads / 32), st));
  }
  PlaceArgs a{V, g->row_off.p, col2.p, pcnt.p, g->size.p, off.p, remaining.p, F0.p, F1.p, counts.p, policy,
              cap, gscratch.p, gcap, counts.p + 5};
  ctx->launches++;
  if (grid_mode) {
    void *args[] = {&a};
    CUDA_TRY(cudaLaunchCooperativeKernel((void *)k_place<true>, dim3(nblocks), dim3(threads), args, smem, st));
  } else {
    k_place<false><<<1, threads, smem, st>>>(a);
    CUDA_TRY(cudaGetLastError());
  }
  long long *d_fp = (long long *)ctx->d_small;
  const long long lmin = LLONG_MIN;
  CUDA_TRY(cudaMemcpyAsync(d_fp, &lmin, 8, cudaMemcpyHostToDevice, st));
  LAUNCH(ctx, k_footprint, grid_for(V, 256, 1024), 256, 0, V, off.p, g->size.p, d_fp);
  CUDA_TRY(cudaMemcpyAsync(offsets, off.p, V * 8, cudaMemcpyDeviceToHost, st));
  int64_t fp;
  rc = dev_read_i64(ctx, (const int64_t *)d_fp, &fp, err);
  if (rc) return rc;
  *footprint = fp;
  if (levels) {
    int32_t lv;
    rc = dev_read_n(ctx, counts.p + 5, &lv, 4, err);
    if (rc) return rc;
    *levels = lv;
  }
  return MP_OK;
}
