// prims.cu — device-wide scan and stable LSD radix sort (sm_100a).
//
// The radix sort is the "vectorised radix sort" the ingest and conflict
// stages stand on: per 8-bit digit pass, (1) a tile histogram kernel,
// (2) an exclusive scan of the digit-major count matrix, (3) a scatter
// kernel that ranks keys inside the tile with warp match_any (stable: warp w
// owns a contiguous run, processed round by round in lane order), stages
// the tile in shared memory in digit order and writes each digit run out
// contiguously so global stores coalesce.
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

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partials(const T *in, int64_t n, T *part) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    int64_t j = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
    if (j < n) s += in[j];
  }
  __shared__ T tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_single(T *a, int64_t n, T *total) {
  // one block scans n partials in place (n up to ~ millions, looped)
  __shared__ T carry_s, tot;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += SCAN_TILE) {
    T v[SCAN_ITEMS];
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
      int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
      v[i] = j < n ? a[j] : T(0);
      s += v[i];
    }
    T pre = block_excl_scan(s, &tot);
    T c = carry_s;
    T run = c + pre;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
      int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
      if (j < n) a[j] = run;
      run += v[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry_s = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry_s;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(const T *in, T *out, int64_t n, const T *part) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  T v[SCAN_ITEMS];
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    v[i] = j < n ? in[j] : T(0);
    s += v[i];
  }
  __shared__ T tot;
  T run = part[blockIdx.x] + block_excl_scan(s, &tot);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    if (j < n) out[j] = run;
    run += v[i];
  }
}

template <typename T>
int dev_exclusive_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err) {
  if (n <= 0) {
    if (total) CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(T), ctx->stream));
    return MP_OK;
  }
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 1) {
    if (out != in) CUDA_TRY(cudaMemcpyAsync(out, in, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
    LAUNCH(ctx, k_scan_single<T>, 1, SCAN_THREADS, 0, out, n, total);
    return MP_OK;
  }
  DBuf<T> part;
  CUDA_TRY(part.alloc(nb, ctx->stream));
  LAUNCH(ctx, k_scan_partials<T>, (unsigned)nb, SCAN_THREADS, 0, in, n, part.p);
  LAUNCH(ctx, k_scan_single<T>, 1, SCAN_THREADS, 0, part.p, nb, total);
  LAUNCH(ctx, k_scan_apply<T>, (unsigned)nb, SCAN_THREADS, 0, in, out, n, part.p);
  return MP_OK;
}

template int dev_exclusive_scan<int32_t>(mp_ctx *, const int32_t *, int32_t *, int64_t, int32_t *, mp_err *);
template int dev_exclusive_scan<int64_t>(mp_ctx *, const int64_t *, int64_t *, int64_t, int64_t *, mp_err *);

// ----------------------------------------------------------------------------
// radix sort

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_BINS = 256;

template <typename K, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K *keys, int64_t n, int shift,
                                                         int64_t ntiles, int32_t *counts) {
  __shared__ int32_t h[RS_BINS];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * (int64_t)(RS_THREADS * ITEMS);
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    int64_t j = base + (int64_t)i * RS_THREADS + threadIdx.x;
    if (j < n) atomicAdd(&h[(unsigned)((keys[j] >> shift) & 0xff)], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + tile] = h[threadIdx.x];
}

template <typename K, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const K *keys, const uint32_t *vals,
                                                            K *okeys, uint32_t *ovals, int64_t n,
                                                            int shift, int64_t ntiles,
                                                            const int32_t *offsets) {
  constexpr int TILE = RS_THREADS * ITEMS;
  constexpr int PER_WARP = 32 * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K *sk = (K *)smem_raw;
  uint32_t *sv = (uint32_t *)(sk + TILE);
  __shared__ int32_t whist[RS_WARPS][RS_BINS];
  __shared__ int32_t dprefix[RS_BINS];
  __shared__ int32_t gbase[RS_BINS];

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * (int64_t)TILE;
  for (int d = lane; d < RS_BINS; d += 32) whist[w][d] = 0;
  if (threadIdx.x < RS_BINS) gbase[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + tile];
  __syncwarp();

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
    unsigned peers = __match_any_sync(FULL_MASK, dig[i]);
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
  // per digit: exclusive prefix over warps; tile totals
  {
    int d = threadIdx.x;  // RS_THREADS == RS_BINS
    int32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++) {
      int32_t t = whist[ww][d];
      whist[ww][d] = run;
      run += t;
    }
    dprefix[d] = run;
  }
  __syncthreads();
  // exclusive scan of tile digit totals (256 values, one warp)
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

template <typename K, int ITEMS>
static int radix_sort_impl(mp_ctx *ctx, K *keys, uint32_t *vals, int64_t n, int bits, mp_err *err) {
  if (n <= 1 || bits <= 0) return MP_OK;
  constexpr int TILE = RS_THREADS * ITEMS;
  int64_t ntiles = (n + TILE - 1) / TILE;
  DBuf<K> k2;
  DBuf<uint32_t> v2;
  DBuf<int32_t> counts;
  CUDA_TRY(k2.alloc(n, ctx->stream));
  CUDA_TRY(v2.alloc(n, ctx->stream));
  CUDA_TRY(counts.alloc(ntiles * RS_BINS, ctx->stream));
  size_t smem = (size_t)TILE * (sizeof(K) + sizeof(uint32_t));
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_rs_scatter<K, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  K *src_k = keys, *dst_k = k2.p;
  uint32_t *src_v = vals, *dst_v = v2.p;
  int passes = 0;
  for (int shift = 0; shift < bits; shift += 8, passes++) {
    LAUNCH(ctx, (k_rs_hist<K, ITEMS>), (unsigned)ntiles, RS_THREADS, 0, src_k, n, shift, ntiles, counts.p);
    int rc = dev_exclusive_scan<int32_t>(ctx, counts.p, counts.p, ntiles * RS_BINS, nullptr, err);
    if (rc) return rc;
    LAUNCH(ctx, (k_rs_scatter<K, ITEMS>), (unsigned)ntiles, RS_THREADS, smem, src_k, src_v, dst_k, dst_v,
           n, shift, ntiles, counts.p);
    K *tk = src_k; src_k = dst_k; dst_k = tk;
    uint32_t *tv = src_v; src_v = dst_v; dst_v = tv;
  }
  if (passes & 1) {
    CUDA_TRY(cudaMemcpyAsync(keys, src_k, n * sizeof(K), cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(vals, src_v, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return MP_OK;
}

int dev_radix_sort_u32(mp_ctx *ctx, uint32_t *keys, uint32_t *vals, int64_t n, int bits, mp_err *err) {
  return radix_sort_impl<uint32_t, 16>(ctx, keys, vals, n, bits, err);
}

int dev_radix_sort_u64(mp_ctx *ctx, uint64_t *keys, uint32_t *vals, int64_t n, int bits, mp_err *err) {
  return radix_sort_impl<uint64_t, 8>(ctx, keys, vals, n, bits, err);
}
