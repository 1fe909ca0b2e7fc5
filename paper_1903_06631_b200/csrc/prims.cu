// prims.cu — device-wide scan and stable LSD radix sort (sm_100a).
//
// The radix sort is the "vectorised radix sort" the ingest and conflict
// stages stand on, two variants of 8-bit digit passes:
//  * reduce-then-scan (large inputs): per pass a tile histogram kernel, one
//    exclusive scan of the digit-major (digit, tile) count matrix, and a
//    scatter kernel that ranks keys stably inside the tile (ballot
//    multisplit), stages the tile in shared memory in digit order and writes
//    each digit run out contiguously;
//  * one-sweep (inputs of about one wave of tiles): the global digit
//    histograms of every pass up front, then one kernel per pass whose tiles
//    resolve their digit offsets by decoupled look-back.
#include "common.cuh"

void mp_set_err(mp_err *e, int32_t code, int64_t index, int64_t a0, int64_t a1, const char *msg) {
  if (!e) return;
  e->code = code;
  e->trace = 0;
  e->index = index;
  e->aux0 = a0;
  e->aux1 = a1;
  if (msg) {
    strncpy(e->msg, msg, sizeof(e->msg) - 1);
    e->msg[sizeof(e->msg) - 1] = 0;
  } else {
    e->msg[0] = 0;
  }
}

int dev_read_n(mp_ctx *ctx, const void *d, void *h, size_t bytes, mp_err *err) {
  CUDA_TRY(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MP_OK;
}

int dev_read_i64(mp_ctx *ctx, const int64_t *d, int64_t *h, mp_err *err) {
  CUDA_TRY(cudaMemcpyAsync(ctx->h_small, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *h = ctx->h_small[0];
  return MP_OK;
}

// ----------------------------------------------------------------------------
// exclusive scan: block partials -> scan of partials -> block scan + offset

#ifndef SCAN_VEC
#define SCAN_VEC 1  // 16-byte loads/stores of full tiles
#endif
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ T block_excl_scan(T v, T *total) {
  __shared__ T warp_tot[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan_add(v);
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < SCAN_THREADS / 32 ? warp_tot[lane] : T(0);
    T xi = warp_incl_scan_add(x);
    if (lane < SCAN_THREADS / 32) warp_tot[lane] = xi - x;
    if (lane == SCAN_THREADS / 32 - 1) *total = xi;
  }
  __syncthreads();
  T r = warp_tot[w] + inc - v;
  __syncthreads();
  return r;
}

// Single-pass scan with decoupled look-back: tiles take ids in launch order
// from a counter, publish their aggregate, then resolve their exclusive
// prefix from predecessors (aggregate or inclusive prefix, whichever is
// posted first) and post their own inclusive prefix.
//
// Posting carries no fence: every posted value travels in 64-bit words that
// hold the scan's epoch in the high half and 32 bits of the value in the low
// half (an int64 value takes two words), so a reader that sees the epoch in
// a word has that word's half of the value — the word is its own flag.  A
// word from an earlier scan carries another epoch and reads as "not
// posted", so the words never need clearing.  words = [agg lo | agg hi |
// pfx lo | pfx hi] x cap.
template <typename T>
__device__ __forceinline__ void scan_post(uint64_t *w, int64_t cap, int64_t tile, uint64_t tag, T v) {
  if (sizeof(T) == 8) *(volatile uint64_t *)&w[cap + tile] = tag | (uint32_t)((uint64_t)(int64_t)v >> 32);
  *(volatile uint64_t *)&w[tile] = tag | (uint32_t)(uint64_t)(int64_t)v;
}

// 0: nothing posted yet, 1: aggregate, 2: inclusive prefix (value in *v)
template <typename T>
__device__ __forceinline__ int scan_peek(const uint64_t *w, int64_t cap, int64_t q, uint64_t tag, T *v) {
#pragma unroll
  for (int st = 2; st >= 1; st--) {
    const uint64_t *b = w + (int64_t)(st == 2 ? 2 : 0) * cap;
    const uint64_t lo = *(volatile const uint64_t *)&b[q];
    if ((lo & 0xffffffff00000000ull) != tag) continue;
    if (sizeof(T) == 8) {
      uint64_t hi;
      do hi = *(volatile const uint64_t *)&b[cap + q];
      while ((hi & 0xffffffff00000000ull) != tag);  // posted right after the low word
      *v = (T)(int64_t)((hi << 32) | (uint32_t)lo);
    } else {
      *v = (T)(int32_t)(uint32_t)lo;
    }
    return st;
  }
  return 0;
}

template <typename T, bool INCL>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_onepass(const T *in, T *out, int64_t n, uint64_t *words,
                                                               int64_t cap, int32_t *tile_ctr, T *total,
                                                               uint32_t epoch, uint32_t tile_base) {
  PDL_WAIT();
  __shared__ int32_t s_tile;
  __shared__ T s_excl, s_tot;
  const uint64_t tag = (uint64_t)epoch << 32;
  uint64_t *const wagg = words, *const wpfx = words + 2 * cap;
  if (threadIdx.x == 0) s_tile = (int32_t)((uint32_t)atomicAdd(tile_ctr, 1) - tile_base);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SCAN_TILE;
  union {
    T v[SCAN_ITEMS];
    uint4 q[SCAN_ITEMS * sizeof(T) / 16];
  } u;
  T *const v = u.v;
  T s = 0;
  // full tiles of 16-byte aligned arrays: each thread's run is read as
  // 16-byte vectors (its SCAN_ITEMS values are contiguous)
  const bool vec = SCAN_VEC && base + SCAN_TILE <= n && ((((uintptr_t)in) | ((uintptr_t)out)) & 15) == 0;
  if (vec) {
    const uint4 *src = (const uint4 *)(in + base + (int64_t)threadIdx.x * SCAN_ITEMS);
#pragma unroll
    for (int i = 0; i < (int)(SCAN_ITEMS * sizeof(T) / 16); i++) u.q[i] = src[i];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) s += v[i];
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
      int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
      v[i] = j < n ? in[j] : T(0);
      s += v[i];
    }
  }
  T pre = block_excl_scan(s, &s_tot);
  if (threadIdx.x < 32) {
    // warp 0 posts the tile, then looks back 32 predecessors at a time: sum
    // aggregates up to the nearest posted inclusive prefix
    const int lane = threadIdx.x;
    const T sum = s_tot;
    T excl = 0;
    if (tile == 0) {
      if (lane == 0) scan_post<T>(wpfx, cap, 0, tag, sum);
    } else {
      if (lane == 0) scan_post<T>(wagg, cap, tile, tag, sum);
      for (int64_t p = tile - 1;; p -= 32) {
        const int64_t q = p - lane;
        T val = 0;
        int st = q >= 0 ? scan_peek<T>(words, cap, q, tag, &val) : 2;
        while (__any_sync(FULL_MASK, st == 0))
          if (st == 0) st = scan_peek<T>(words, cap, q, tag, &val);
        const unsigned pfx = __ballot_sync(FULL_MASK, st == 2);
        const int stop = pfx ? __ffs(pfx) - 1 : 31;
        excl += warp_sum(lane <= stop ? val : T(0));
        if (pfx) break;
      }
      if (lane == 0) scan_post<T>(wpfx, cap, tile, tag, excl + sum);
    }
    if (lane == 0) {
      s_excl = excl;
      if (total && base + SCAN_TILE >= n) *total = excl + sum;
    }
  }
  __syncthreads();
  T run = s_excl + pre;
  if (vec) {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
      T x = v[i];
      if (INCL) {
        run += x;
        v[i] = run;
      } else {
        v[i] = run;
        run += x;
      }
    }
    uint4 *dst = (uint4 *)(out + base + (int64_t)threadIdx.x * SCAN_ITEMS);
#pragma unroll
    for (int i = 0; i < (int)(SCAN_ITEMS * sizeof(T) / 16); i++) dst[i] = u.q[i];
    return;
  }
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    if (INCL) run += v[i];
    if (j < n) out[j] = run;
    if (!INCL) run += v[i];
  }
}

template <typename T, bool INCL>
static int dev_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err) {
  if (n <= 0) {
    if (total) CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(T), ctx->stream));
    return MP_OK;
  }
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  // persistent per-context flags / values / tile counter (see mp_ctx)
  if (nb > ctx->scan_cap || ctx->scan_epoch >= 0xfffffff0u) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (ctx->scan_vals) cudaFree(ctx->scan_vals);
    if (!ctx->scan_ctr) CUDA_TRY(cudaMalloc((void **)&ctx->scan_ctr, 16));
    int64_t cap = nb < 4096 ? 4096 : nb;
    CUDA_TRY(cudaMalloc((void **)&ctx->scan_vals, 4 * cap * 8));
    CUDA_TRY(cudaMemsetAsync(ctx->scan_vals, 0, 4 * cap * 8, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->scan_ctr, 0, 16, ctx->stream));
    ctx->scan_cap = cap;
    ctx->scan_epoch = 0;
    ctx->scan_base = 0;
  }
  const uint32_t epoch = ++ctx->scan_epoch;
  const uint32_t base = ctx->scan_base;
  ctx->scan_base += (uint32_t)nb;
  LAUNCH(ctx, (k_scan_onepass<T, INCL>), (unsigned)nb, SCAN_THREADS, 0, in, out, n, (uint64_t *)ctx->scan_vals,
         ctx->scan_cap, ctx->scan_ctr, total, epoch, base);
  return MP_OK;
}

template <typename T>
int dev_exclusive_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err) {
  return dev_scan<T, false>(ctx, in, out, n, total, err);
}
template <typename T>
int dev_inclusive_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err) {
  return dev_scan<T, true>(ctx, in, out, n, total, err);
}

template int dev_exclusive_scan<int32_t>(mp_ctx *, const int32_t *, int32_t *, int64_t, int32_t *, mp_err *);
template int dev_exclusive_scan<int64_t>(mp_ctx *, const int64_t *, int64_t *, int64_t, int64_t *, mp_err *);
template int dev_inclusive_scan<int64_t>(mp_ctx *, const int64_t *, int64_t *, int64_t, int64_t *, mp_err *);

// ----------------------------------------------------------------------------
// radix sort

#ifndef RS_LOOKBACK_BATCH
#define RS_LOOKBACK_BATCH 8  // predecessor digit counts read per look-back round trip (1: 5 % slower passes)
#endif
#ifndef RS_ITEMS32
#define RS_ITEMS32 16  // keys per thread of a 32-bit one-sweep pass tile
#endif
#ifndef RS_RTS_ITEMS32
#define RS_RTS_ITEMS32 12  // keys per thread of a 32-bit reduce-then-scan tile (16: 119 registers, 8: 4 % slower)
#endif
#ifndef RS_RTS_MIN_N32
#define RS_RTS_MIN_N32 500000  // 32-bit keys: 1 M-key placement order 0.100 -> 0.090 ms by reduce-then-scan
#endif
#ifndef RS_RTS_MIN_N
#define RS_RTS_MIN_N 2000000  // below this many keys a one-sweep pass's look-back is short: keep it
#endif
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_BINS = 256;

// One-sweep LSD radix sort (8-bit digits): one kernel computes every pass's
// global digit histogram up front, then each pass is a single kernel whose
// tiles (ids in launch order) rank their keys per warp (match_any), post
// their digit counts, resolve each digit's exclusive prefix by decoupled
// look-back over earlier tiles (32-bit flag|count words), and scatter
// through shared memory so global writes stay coalesced per digit run.

// lanes of the warp holding the same digit (d < 1 << RB), among `valid` lanes
template <int RB>
__device__ __forceinline__ unsigned multisplit_peers(unsigned d, unsigned valid) {
  unsigned peers = valid;
#pragma unroll
  for (int b = 0; b < RB; b++) {
    const bool bit = (d >> b) & 1u;
    const unsigned bb = __ballot_sync(FULL_MASK, bit);
    peers &= bit ? bb : ~bb;
  }
  return peers;
}

#ifndef OS_MATCH
#define OS_MATCH 0  // 1: rank with match.any
#endif

constexpr uint32_t OS_AGG = 1u << 30, OS_PFX = 2u << 30, OS_MASK = (1u << 30) - 1;
constexpr int OS_MAX_PASSES = 8;

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_os_hist(const K *keys, int64_t n, int passes, int32_t *ghist) {
  PDL_WAIT();
  __shared__ int32_t h[OS_MAX_PASSES][RS_BINS];
  for (int i = threadIdx.x; i < passes * RS_BINS; i += RS_THREADS) h[i / RS_BINS][i % RS_BINS] = 0;
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)RS_THREADS + threadIdx.x; j < n; j += (int64_t)gridDim.x * RS_THREADS) {
    K k = keys[j];
    for (int p = 0; p < passes; p++) atomicAdd(&h[p][(unsigned)((k >> (8 * p)) & 0xff)], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RS_BINS; i += RS_THREADS) {
    int32_t c = h[i / RS_BINS][i % RS_BINS];
    if (c) atomicAdd(&ghist[i], c);
  }
}

// per pass: exclusive prefix of the 256 digit counts (one warp per pass)
__global__ void k_os_prefix(int32_t *ghist, int passes) {
  PDL_WAIT();
  const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
  if (p >= passes) return;
  int32_t c = 0;
  for (int chunk = 0; chunk < RS_BINS; chunk += 32) {
    int32_t x = ghist[p * RS_BINS + chunk + lane];
    int32_t xi = warp_incl_scan_add(x);
    ghist[p * RS_BINS + chunk + lane] = c + xi - x;
    c += __shfl_sync(FULL_MASK, xi, 31);
  }
}

template <typename K, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS) k_os_pass(const K *keys, const uint32_t *vals, K *okeys,
                                                         uint32_t *ovals, int64_t n, int shift,
                                                         const int32_t *gstart, uint32_t *look,
                                                         int32_t *tile_ctr) {
  PDL_WAIT();
  constexpr int TILE = RS_THREADS * ITEMS;
  constexpr int PER_WARP = 32 * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K *sk = (K *)smem_raw;
  uint32_t *sv = (uint32_t *)(sk + TILE);
  __shared__ int32_t whist[RS_WARPS][RS_BINS];
  __shared__ int32_t dprefix[RS_BINS];
  __shared__ int32_t gbase[RS_BINS];
  __shared__ int32_t s_tile;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1);
  for (int d = lane; d < RS_BINS; d += 32) whist[w][d] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * (int64_t)TILE;

  K k[ITEMS];
  uint32_t v[ITEMS];
  int dig[ITEMS];
  int loc[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    int64_t j = base + (int64_t)w * PER_WARP + i * 32 + lane;
    bool ok = j < n;
    k[i] = ok ? keys[j] : K(0);
    v[i] = ok ? vals[j] : 0u;
    dig[i] = ok ? (int)((k[i] >> shift) & 0xff) : RS_BINS;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
#if OS_MATCH
    unsigned peers = __match_any_sync(FULL_MASK, dig[i]);
#else
    // eight ballots instead of match.any (whose result latency dominated
    // the pass's stalls)
    unsigned peers = multisplit_peers<8>((unsigned)dig[i] & 0xffu, __ballot_sync(FULL_MASK, dig[i] < RS_BINS));
#endif
    int rank = __popc(peers & lanemask_lt());
    int cnt = __popc(peers);
    int leader = __ffs(peers) - 1;
    int b = 0;
    if (dig[i] < RS_BINS) b = whist[w][dig[i]];
    loc[i] = b + rank;
    __syncwarp();
    if (lane == leader && dig[i] < RS_BINS) whist[w][dig[i]] = b + cnt;
    __syncwarp();
  }
  __syncthreads();
  {
    // per digit: exclusive prefix over warps, the tile's count, its posting
    // and the look-back for its global position
    const int d = threadIdx.x;  // RS_THREADS == RS_BINS
    int32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++) {
      int32_t t = whist[ww][d];
      whist[ww][d] = run;
      run += t;
    }
    dprefix[d] = run;
    uint32_t *mine = look + tile * RS_BINS + d;
    if (tile == 0) {
      atomicExch(mine, OS_PFX | (uint32_t)run);
      gbase[d] = gstart[d];
    } else {
      atomicExch(mine, OS_AGG | (uint32_t)run);
      uint32_t excl = 0;
#if RS_LOOKBACK_BATCH > 1
      // RS_LOOKBACK_BATCH predecessors per round trip, consumed in order
      for (int64_t p = tile - 1;; p -= RS_LOOKBACK_BATCH) {
        uint32_t x[RS_LOOKBACK_BATCH];
#pragma unroll
        for (int i = 0; i < RS_LOOKBACK_BATCH; i++)
          x[i] = p - i >= 0 ? *(volatile uint32_t *)(look + (p - i) * RS_BINS + d) : 0u;
        bool done = false;
#pragma unroll
        for (int i = 0; i < RS_LOOKBACK_BATCH; i++) {
          uint32_t v = x[i];
          while (!(v & ~OS_MASK)) v = *(volatile uint32_t *)(look + (p - i) * RS_BINS + d);
          excl += v & OS_MASK;
          if (v & OS_PFX) { done = true; break; }
        }
        if (done) break;
      }
#else
      for (int64_t p = tile - 1;;) {
        uint32_t x = *(volatile uint32_t *)(look + p * RS_BINS + d);
        if (!(x & ~OS_MASK)) continue;
        excl += x & OS_MASK;
        if (x & OS_PFX) break;
        p--;
      }
#endif
      atomicExch(mine, OS_PFX | (excl + (uint32_t)run));
      gbase[d] = gstart[d] + (int32_t)excl;
    }
  }
  __syncthreads();
  // exclusive scan of the tile digit counts (256 values, one warp)
  if (w == 0) {
    int32_t c = 0;
    for (int chunk = 0; chunk < RS_BINS; chunk += 32) {
      int32_t x = dprefix[chunk + lane];
      int32_t xi = warp_incl_scan_add(x);
      dprefix[chunk + lane] = c + xi - x;
      c += __shfl_sync(FULL_MASK, xi, 31);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    if (dig[i] < RS_BINS) {
      int pos = dprefix[dig[i]] + whist[w][dig[i]] + loc[i];
      sk[pos] = k[i];
      sv[pos] = v[i];
    }
  }
  __syncthreads();
  int64_t cnt = n - base;
  if (cnt > TILE) cnt = TILE;
  for (int i = threadIdx.x; i < cnt; i += RS_THREADS) {
    K key = sk[i];
    int d = (int)((key >> shift) & 0xff);
    int64_t pos = (int64_t)gbase[d] + (i - dprefix[d]);
    okeys[pos] = key;
    ovals[pos] = sv[i];
  }
}

// ----------------------------------------------------------------------------
// Reduce-then-scan LSD radix sort (the default; RS_ONESWEEP=1 restores the
// one-sweep kernels above).  Per pass: (1) k_rs_hist counts each tile's
// digits into a digit-major matrix mat[d * ntiles + tile]; (2) one exclusive
// scan of the matrix gives every (digit, tile) run its global start — the
// digit base and the tile prefix at once, so no tile waits on a look-back
// (the one-sweep passes spent a quarter of their time there: a tile posted
// late in a wave walks back over every tile of the wave still in flight);
// (3) k_rs_scatter ranks each tile's keys stably and writes each digit run
// contiguously through shared memory.  Ranking uses a ballot multisplit (one
// vote per digit bit) instead of match.any, whose latency serialised the
// per-warp ranking loop.
#ifndef RS_ONESWEEP
#define RS_ONESWEEP 0
#endif

template <typename K, int RB, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K *keys, int64_t n, int shift, int32_t ntiles,
                                                        int32_t *mat) {
  PDL_WAIT();
  constexpr int BINS = 1 << RB;
  constexpr int TILE = RS_THREADS * ITEMS;
  constexpr int VK = 16 / sizeof(K);  // keys per 16-byte vector
  __shared__ int32_t h[2][BINS];  // two copies halve same-address contention on skewed digits
  for (int i = threadIdx.x; i < 2 * BINS; i += RS_THREADS) h[i / BINS][i % BINS] = 0;
  const int64_t base = (int64_t)blockIdx.x * TILE;
  int32_t *hh = h[(threadIdx.x >> 5) & 1];
  // every load issued before the first atomic
  union {
    uint4 q[ITEMS / VK];
    K k[ITEMS];
  } u;
  const bool full = base + TILE <= n && (((uintptr_t)keys) & 15) == 0;
  if (full) {
    const uint4 *src = (const uint4 *)(keys + base);
#pragma unroll
    for (int i = 0; i < ITEMS / VK; i++) u.q[i] = src[i * RS_THREADS + threadIdx.x];
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
      const int64_t j = base + (int64_t)i * RS_THREADS + threadIdx.x;
      u.k[i] = j < n ? keys[j] : K(0);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const int64_t j = full ? 0 : base + (int64_t)i * RS_THREADS + threadIdx.x;
    if (j < n) atomicAdd(&hh[(unsigned)(u.k[i] >> shift) & (BINS - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) mat[(int64_t)d * ntiles + blockIdx.x] = h[0][d] + h[1][d];
}

// vals == nullptr: the values are the input positions (iota)
#ifndef RS_MINB
#define RS_MINB 3  // resident scatter CTAs per SM the register budget must allow
#endif
#ifndef RS_MATCH
#define RS_MATCH 0  // rank with match.any instead of the ballot multisplit
#endif
template <typename K, int RB, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS, RS_MINB) k_rs_scatter(const K *keys, const uint32_t *vals, K *okeys,
                                                           uint32_t *ovals, int64_t n, int shift, int32_t ntiles,
                                                           const int32_t *offs, int32_t *rank_out) {
  PDL_WAIT();
  constexpr int BINS = 1 << RB;
  constexpr int TILE = RS_THREADS * ITEMS;
  constexpr int PER_WARP = 32 * ITEMS;
  // dynamic: the staged tile, then the per-warp digit counts and the tile's
  // digit starts / global positions
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K *sk = (K *)smem_raw;
  uint32_t *sv = (uint32_t *)(sk + TILE);
  int32_t(*whist)[BINS] = (int32_t(*)[BINS])(sv + TILE);
  int32_t *dstart = &whist[RS_WARPS][0];
  int32_t *gpos = dstart + BINS;
  __shared__ int32_t wtot[RS_WARPS];

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * (int64_t)TILE;
  for (int d = lane; d < BINS; d += 32) whist[w][d] = 0;
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) gpos[d] = offs[(int64_t)d * ntiles + tile];
  K k[ITEMS];
  uint32_t v[ITEMS];
  int loc[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const int64_t j = base + (int64_t)w * PER_WARP + i * 32 + lane;
    const bool ok = j < n;
    k[i] = ok ? keys[j] : K(0);
    v[i] = ok ? (vals ? vals[j] : (uint32_t)j) : 0u;
  }
  __syncwarp();
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const int64_t j = base + (int64_t)w * PER_WARP + i * 32 + lane;
    const unsigned valid = __ballot_sync(FULL_MASK, j < n);
    const unsigned d = (unsigned)(k[i] >> shift) & (BINS - 1);
#if RS_MATCH
    const unsigned peers = __match_any_sync(FULL_MASK, j < n ? d : (1u << RB) + lane) & valid;
#else
    const unsigned peers = multisplit_peers<RB>(d, valid);
#endif
    int b = 0;
    if (j < n) b = whist[w][d];
    loc[i] = b + __popc(peers & lt);
    __syncwarp();
    if (j < n && (peers & lt) == 0) whist[w][d] = b + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps; the tile's count of the digit
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) {
    int32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++) {
      const int32_t t = whist[ww][d];
      whist[ww][d] = run;
      run += t;
    }
    dstart[d] = run;
  }
  __syncthreads();
  // exclusive scan of the tile's digit counts: SW warps scan BINS / SW each
  {
    constexpr int SW = BINS >= 32 * RS_WARPS ? RS_WARPS : BINS / 32;  // scanning warps
    constexpr int PER = BINS / SW;  // contiguous digits per scanning warp (>= 32)
    int32_t c = 0;
    if (w < SW)
      for (int ch = 0; ch < PER; ch += 32) {
        const int d = w * PER + ch + lane;
        const int32_t x = dstart[d];
        const int32_t xi = warp_incl_scan_add(x);
        dstart[d] = c + xi - x;
        c += __shfl_sync(FULL_MASK, xi, 31);
      }
    if (lane == 0) wtot[w] = c;
    __syncthreads();
    int32_t add = 0;
    for (int ww = 0; ww < w; ww++) add += wtot[ww];
    if (w < SW)
      for (int ch = 0; ch < PER; ch += 32) dstart[w * PER + ch + lane] += add;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const int64_t j = base + (int64_t)w * PER_WARP + i * 32 + lane;
    if (j < n) {
      const unsigned d = (unsigned)(k[i] >> shift) & (BINS - 1);
      const int pos = dstart[d] + whist[w][d] + loc[i];
      sk[pos] = k[i];
      sv[pos] = v[i];
    }
  }
  __syncthreads();
  int64_t cnt = n - base;
  if (cnt > TILE) cnt = TILE;
  for (int i = threadIdx.x; i < cnt; i += RS_THREADS) {
    const K key = sk[i];
    const unsigned d = (unsigned)(key >> shift) & (BINS - 1);
    const int64_t pos = (int64_t)gpos[d] + (i - dstart[d]);
    if (rank_out) {
      rank_out[sv[i]] = (int32_t)pos;  // last pass of a ranking: each value's sorted position
    } else {
      okeys[pos] = key;
      ovals[pos] = sv[i];
    }
  }
}

__global__ void k_rs_iota(uint32_t *v, int64_t n) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

// stable sort of (kin, vin) on key bits [0, bits) into (kout, vout); vin ==
// nullptr sorts the positions 0..n-1.  kin/vin may alias kout/vout.
#ifndef RS_RTS_EXACT_RB
#define RS_RTS_EXACT_RB 1  // a 7- or 9-bit pass uses 128 / 512 bins (smaller digit matrix and tile scans)
#endif
#ifndef RS_RTS_MAXRB
#define RS_RTS_MAXRB 10  // widest digit of a reduce-then-scan pass (config 4's 21-bit ids: 3 passes of 7 bits; 11: 2 passes, 35 % slower)
#endif

// one reduce-then-scan pass with RB-bit digits (the digit is masked to w bits)
template <typename K, int RB, int ITEMS>
static int rts_pass(mp_ctx *ctx, const K *sk, const uint32_t *sv, K *dk, uint32_t *dv, int64_t n, int shift,
                    int32_t ntiles, int32_t *mat, int32_t *rank_out, mp_err *err) {
  constexpr int BINS = 1 << RB;
  constexpr int TILE = RS_THREADS * ITEMS;
  const size_t smem = (size_t)TILE * (sizeof(K) + sizeof(uint32_t)) + (size_t)(RS_WARPS + 2) * BINS * sizeof(int32_t);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_rs_scatter<K, RB, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  LAUNCH(ctx, (k_rs_hist<K, RB, ITEMS>), (unsigned)ntiles, RS_THREADS, 0, sk, n, shift, ntiles, mat);
  int rc = dev_exclusive_scan<int32_t>(ctx, mat, mat, (int64_t)BINS * ntiles, nullptr, err);
  if (rc) return rc;
  LAUNCH(ctx, (k_rs_scatter<K, RB, ITEMS>), (unsigned)ntiles, RS_THREADS, smem, sk, sv, dk, dv, n, shift, ntiles,
         (const int32_t *)mat, rank_out);
  return MP_OK;
}

template <typename K, int ITEMS>
static int radix_sort_rts(mp_ctx *ctx, const K *kin, const uint32_t *vin, K *kout, uint32_t *vout, int64_t n,
                          int bits, mp_err *err, int32_t *rank_out = nullptr) {
  constexpr int TILE = RS_THREADS * ITEMS;
  cudaStream_t st = ctx->stream;
  if (n <= 0) return MP_OK;
  if (n > (int64_t)INT32_MAX) {
    mp_set_err(err, MP_E_UNSUPPORTED, 0, n, 0, "radix sort of more than 2^31 keys");
    return MP_E_UNSUPPORTED;
  }
  // as few passes as RS_RTS_MAXRB-bit digits allow, the bits split evenly
  const int passes = bits <= 0 ? 0 : (bits + RS_RTS_MAXRB - 1) / RS_RTS_MAXRB;
  if (passes == 0) {
    if (kout != kin) CUDA_TRY(cudaMemcpyAsync(kout, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    if (!vin) LAUNCH(ctx, k_rs_iota, grid_for(n, 256), 256, 0, vout, n);
    else if (vout != vin) CUDA_TRY(cudaMemcpyAsync(vout, vin, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    return MP_OK;
  }
  const int32_t ntiles = (int32_t)((n + TILE - 1) / TILE);
  DBuf<K> ka, kb;
  DBuf<uint32_t> va, vb;
  const int wbase = bits / passes, wextra = bits % passes;  // the first wextra passes take one bit more
  const int wmax = wbase + (wextra ? 1 : 0);
  // digits as wide as the pass (RS_RTS_EXACT_RB), else rounded up to 8 / 10 / 11
  auto rb_for = [](int w) { return RS_RTS_EXACT_RB ? (w <= 7 ? 7 : w) : (w <= 8 ? 8 : w <= 10 ? 10 : 11); };
  const int rbmax = rb_for(wmax);
  DBuf<int32_t> mat;
  CUDA_TRY(mat.alloc((int64_t)ntiles << rbmax, st));
  const bool alias = kout == kin || (vin && vout == vin);
  // pass p reads src and writes dst; the last pass writes the caller's
  // output unless it aliases the input of a single pass
  const int need = passes > 1 ? 2 : (alias ? 1 : 0);
  if (need >= 1) { CUDA_TRY(ka.alloc(n, st)); CUDA_TRY(va.alloc(n, st)); }
  if (need >= 2 && passes > 2) { CUDA_TRY(kb.alloc(n, st)); CUDA_TRY(vb.alloc(n, st)); }
  const K *sk = kin;
  int shift = 0;
  const uint32_t *sv = vin;
  for (int p = 0; p < passes; p++) {
    K *dk;
    uint32_t *dv;
    const bool last = p == passes - 1;
    if (last && !(passes == 1 && alias)) { dk = kout; dv = vout; }
    else if ((p & 1) == 0) { dk = ka.p; dv = va.p; }
    else { dk = kb.p; dv = vb.p; }
    // a pass of w bits reads digits (k >> shift) & (2^RB - 1): bits above
    // shift + w are zero in the key range (or sorted by a later pass)
    const int w = wbase + (p < wextra ? 1 : 0);
    int32_t *ro = last ? rank_out : (int32_t *)nullptr;
    int rc;
    switch (rb_for(w)) {
      case 7: rc = rts_pass<K, 7, ITEMS>(ctx, sk, sv, dk, dv, n, shift, ntiles, mat.p, ro, err); break;
      case 8: rc = rts_pass<K, 8, ITEMS>(ctx, sk, sv, dk, dv, n, shift, ntiles, mat.p, ro, err); break;
      case 9: rc = rts_pass<K, 9, ITEMS>(ctx, sk, sv, dk, dv, n, shift, ntiles, mat.p, ro, err); break;
      case 10: rc = rts_pass<K, 10, ITEMS>(ctx, sk, sv, dk, dv, n, shift, ntiles, mat.p, ro, err); break;
      default: rc = rts_pass<K, 11, ITEMS>(ctx, sk, sv, dk, dv, n, shift, ntiles, mat.p, ro, err); break;
    }
    if (rc) return rc;
    shift += w;
    sk = dk;
    sv = dv;
  }
  if (!rank_out && sk != kout) {
    CUDA_TRY(cudaMemcpyAsync(kout, sk, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(vout, sv, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  return MP_OK;
}

// rank[i] = position of key i in the stable order of kin (bits [0, bits)),
// the last pass scattering positions instead of keys and values; returns 1
// (nothing done) below dev_radix_rank_min_n() keys
int64_t dev_radix_rank_min_n() { return RS_RTS_MIN_N32; }
int dev_radix_rank_u32(mp_ctx *ctx, const uint32_t *kin, int64_t n, int bits, int32_t *rank, mp_err *err) {
  if (n < RS_RTS_MIN_N32 || bits <= 0) return 1;
  return radix_sort_rts<uint32_t, RS_RTS_ITEMS32>(ctx, kin, nullptr, nullptr, nullptr, n, bits, err, rank);
}

int dev_radix_sort_u32_iota(mp_ctx *ctx, const uint32_t *kin, uint32_t *kout, uint32_t *vout, int64_t n, int bits,
                            mp_err *err) {
  return radix_sort_rts<uint32_t, RS_RTS_ITEMS32>(ctx, kin, nullptr, kout, vout, n, bits, err);
}

template <typename K, int ITEMS, int RTS_ITEMS>
static int radix_sort_impl(mp_ctx *ctx, K *keys, uint32_t *vals, int64_t n, int bits, mp_err *err) {
  if (n <= 1 || bits <= 0) return MP_OK;
  if (!RS_ONESWEEP && n >= (sizeof(K) == 4 ? RS_RTS_MIN_N32 : RS_RTS_MIN_N)) return radix_sort_rts<K, RTS_ITEMS>(ctx, keys, vals, keys, vals, n, bits, err);
  if (n > (int64_t)OS_MASK) {
    mp_set_err(err, MP_E_UNSUPPORTED, 0, n, 0, "radix sort of more than 2^30 keys");
    return MP_E_UNSUPPORTED;
  }
  constexpr int TILE = RS_THREADS * ITEMS;
  const int64_t ntiles = (n + TILE - 1) / TILE;
  const int passes = (bits + 7) / 8;
  cudaStream_t st = ctx->stream;
  DBuf<K> k2;
  DBuf<uint32_t> v2;
  DBuf<int32_t> meta;  // [passes][256] digit starts, then per pass a tile counter
  DBuf<uint32_t> look;
  CUDA_TRY(k2.alloc(n, st));
  CUDA_TRY(v2.alloc(n, st));
  CUDA_TRY(meta.alloc(passes * RS_BINS + passes, st));
  CUDA_TRY(look.alloc(ntiles * RS_BINS * passes, st));
  CUDA_TRY(cudaMemsetAsync(meta.p, 0, (passes * RS_BINS + passes) * sizeof(int32_t), st));
  CUDA_TRY(cudaMemsetAsync(look.p, 0, ntiles * RS_BINS * passes * sizeof(uint32_t), st));
  size_t smem = (size_t)TILE * (sizeof(K) + sizeof(uint32_t));
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_os_pass<K, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  unsigned hgrid = grid_for(n, RS_THREADS, (int64_t)ctx->num_sms * 8);
  LAUNCH(ctx, k_os_hist<K>, hgrid, RS_THREADS, 0, keys, n, passes, meta.p);
  LAUNCH(ctx, k_os_prefix, 1, 32 * passes, 0, meta.p, passes);
  // buffers: the caller's (0) and scratch (1, 2); the last pass always writes
  // the caller's, odd pass counts route through the third buffer
  DBuf<K> k3;
  DBuf<uint32_t> v3;
  if ((passes & 1) && passes > 1) {
    CUDA_TRY(k3.alloc(n, st));
    CUDA_TRY(v3.alloc(n, st));
  }
  K *bk[3] = {keys, k2.p, k3.p};
  uint32_t *bv[3] = {vals, v2.p, v3.p};
  int src = 0;
  for (int p = 0; p < passes; p++) {
    int dst;
    if (p == passes - 1) dst = passes == 1 ? 1 : 0;
    else if (passes & 1) dst = src == 1 ? 2 : 1;
    else dst = src ^ 1;
    LAUNCH(ctx, (k_os_pass<K, ITEMS>), (unsigned)ntiles, RS_THREADS, smem, bk[src], bv[src], bk[dst], bv[dst], n,
           8 * p, meta.p + p * RS_BINS, look.p + (int64_t)p * ntiles * RS_BINS, meta.p + passes * RS_BINS + p);
    src = dst;
  }
  if (src != 0) {  // a single pass
    CUDA_TRY(cudaMemcpyAsync(keys, bk[src], n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(vals, bv[src], n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  return MP_OK;
}

int dev_radix_sort_u32(mp_ctx *ctx, uint32_t *keys, uint32_t *vals, int64_t n, int bits, mp_err *err) {
  return radix_sort_impl<uint32_t, RS_ITEMS32, RS_RTS_ITEMS32>(ctx, keys, vals, n, bits, err);
}

int dev_radix_sort_u64(mp_ctx *ctx, uint64_t *keys, uint32_t *vals, int64_t n, int bits, mp_err *err) {
  return radix_sort_impl<uint64_t, 8, 8>(ctx, keys, vals, n, bits, err);
}
