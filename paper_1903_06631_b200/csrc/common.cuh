// common.cuh — shared device/host plumbing for libmemplan_b200 (sm_100a).
//
// Context, stream-ordered scratch, launch accounting, Python-exact float
// helpers and the device-wide primitives (scan, reductions) every stage
// uses.  All kernels are built with -fmad=false: the swap path reproduces
// CPython's binary64 left folds bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <memory>
#include <vector>

#include "../../include/memplan_b200.h"

#define MP_WARP 32
#define FULL_MASK 0xffffffffu

struct mp_stage_rec {
  int id;
  cudaEvent_t a, b;
};

struct mp_ctx {
  // every C-ABI entry point that uses the context (its stream, scratch
  // cells, timing records) or a handle bound to it holds this for the call:
  // calls from several host threads on one context serialize
  std::recursive_mutex mu;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // asynchronous trace uploads (created on first use)
  long long launches = 0;
  // pinned host staging for small scalar readbacks
  int64_t *h_small = nullptr;
  int64_t *d_small = nullptr;
  // single-pass scan state kept across calls (dev_exclusive_scan): per-tile
  // aggregates / inclusive prefixes as value words tagged with a per-scan
  // epoch, so no scan has to clear them first, and the tile-id counter
  // (each scan consumes exactly its tile count from it)
  int64_t *scan_vals = nullptr;   // [4 * scan_cap] 64-bit words (prims.cu k_scan_onepass)
  int32_t *scan_ctr = nullptr;
  int64_t scan_cap = 0;
  uint32_t scan_epoch = 0;
  uint32_t scan_base = 0;
  // the last extraction's final scalars (peak, peak index, access count,
  // duration) travel to h_small[40..43] asynchronously; dims_owner is the
  // profile they belong to until read (handles.cuh profile_dims)
  struct mp_dprofile *dims_owner = nullptr;
  cudaEvent_t dims_ev = nullptr;
  // stage timing (CUDA events on `stream`)
  bool timing = false;
  struct StageTimer *open_timer = nullptr;  // innermost running stage
  std::vector<mp_stage_rec> pending;
  std::vector<cudaEvent_t> spare;
  cudaEvent_t event() {
    cudaEvent_t e;
    if (!spare.empty()) { e = spare.back(); spare.pop_back(); }
    else cudaEventCreate(&e);
    return e;
  }
};

#define CTX_GUARD(c) std::lock_guard<std::recursive_mutex> _ctx_guard((c)->mu)

// RAII: brackets a stage with events on the context stream when timing is on.
// Stages nest exclusively: while an inner stage runs (the size-order sort
// inside the conflict build) the outer one is paused, so per-stage times add
// up to the step instead of counting the inner work twice.
struct StageTimer {
  mp_ctx *c;
  int id;
  cudaEvent_t a = nullptr;
  StageTimer *outer = nullptr;
  StageTimer(mp_ctx *c_, int id_) : c(c_), id(id_) {
    if (c->timing) {
      outer = c->open_timer;
      if (outer) outer->stop();
      c->open_timer = this;
      start();
    }
  }
  void start() {
    a = c->event();
    cudaEventRecord(a, c->stream);
  }
  void stop() {
    if (!a) return;
    cudaEvent_t b = c->event();
    cudaEventRecord(b, c->stream);
    c->pending.push_back({id, a, b});
    a = nullptr;
  }
  ~StageTimer() {
    if (c->open_timer != this) return;
    stop();
    c->open_timer = outer;
    if (outer) outer->start();
  }
};

// ----------------------------------------------------------------------------
// error plumbing

struct MpStatus {
  int code = MP_OK;
};

void mp_set_err(mp_err *e, int32_t code, int64_t index, int64_t a0, int64_t a1, const char *msg);

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      mp_set_err(err, MP_E_CUDA, 0, (int64_t)_e, __LINE__, cudaGetErrorString(_e));     \
      return MP_E_CUDA;                                                                 \
    }                                                                                   \
  } while (0)

// Programmatic dependent launch: a kernel may be scheduled while the one
// before it on the stream drains, and waits (griddepcontrol.wait, the first
// statement of every kernel here) until that one has completed and its
// writes are visible — the launch latency and block ramp-up of each kernel
// overlap its predecessor's tail.  Every __global__ function in csrc/ starts
// with PDL_WAIT() (tests/test_cpu_host.py checks it): a kernel that returned
// before waiting could complete ahead of its predecessor and let the next
// kernel read unfinished data.
#ifndef MP_PDL
#define MP_PDL 1
#endif
#define PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

// launch wrapper: counts launches on the context and checks the config
#define LAUNCH(ctx, kernel, grid, block, smem, ...)                                      \
  do {                                                                                  \
    (ctx)->launches++;                                                                  \
    cudaLaunchConfig_t _cfg = {};                                                       \
    _cfg.gridDim = dim3(grid);                                                          \
    _cfg.blockDim = dim3(block);                                                        \
    _cfg.dynamicSmemBytes = (smem);                                                     \
    _cfg.stream = (ctx)->stream;                                                        \
    cudaLaunchAttribute _at[1];                                                         \
    _at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                     \
    _at[0].val.programmaticStreamSerializationAllowed = MP_PDL;                         \
    _cfg.attrs = _at;                                                                   \
    _cfg.numAttrs = 1;                                                                  \
    cudaError_t _le = cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__);                   \
    if (_le == cudaSuccess) _le = cudaGetLastError();                                   \
    if (_le != cudaSuccess) {                                                           \
      mp_set_err(err, MP_E_CUDA, 0, (int64_t)_le, __LINE__, cudaGetErrorString(_le));   \
      return MP_E_CUDA;                                                                 \
    }                                                                                   \
  } while (0)

static inline unsigned grid_for(int64_t n, int block, int64_t cap = 1 << 20) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// stream-ordered device buffer (cudaMallocAsync on the context stream)
template <typename T>
struct DBuf {
  T *p = nullptr;
  int64_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  cudaError_t alloc(int64_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T);
    return cudaMallocAsync((void **)&p, bytes, st);
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
};

// ----------------------------------------------------------------------------
// Python-exact float helpers (builtin max/min keep the first maximal arg)

__host__ __device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }
__host__ __device__ __forceinline__ double pymin(double a, double b) { return b < a ? b : a; }

// exact Python `float <= int` (no int->double rounding)
__host__ __device__ __forceinline__ bool f_le_i(double f, int64_t i) {
  if (f != f) return false;
  if (f >= 9223372036854775808.0) return false;
  if (f < -9223372036854775808.0) return true;
  double fl = floor(f);
  int64_t q = (int64_t)fl;
  if (q < i) return true;
  if (q > i) return false;
  return fl == f;
}

// ----------------------------------------------------------------------------
// names: var ids are lexicographic ranks; renamed instances "base#alloc"
// fall back to a byte comparison of the virtual strings.

struct NameTable {
  const uint8_t *blob;
  const int64_t *off;
};

__host__ __device__ inline int dec_digits(int32_t v, char *buf) {
  // writes '#' + decimal(v) (v >= 0), returns length
  char tmp[12];
  int n = 0;
  do { tmp[n++] = (char)('0' + v % 10); v /= 10; } while (v);
  buf[0] = '#';
  for (int i = 0; i < n; i++) buf[1 + i] = tmp[n - 1 - i];
  return n + 1;
}

__host__ __device__ inline int name_cmp(NameTable nm, int32_t ab, int32_t ar, int32_t bb, int32_t br) {
  if (ar < 0 && br < 0) return (ab > bb) - (ab < bb);
  char sa[16], sb[16];
  int la = ar >= 0 ? dec_digits(ar, sa) : 0;
  int lb = br >= 0 ? dec_digits(br, sb) : 0;
  const uint8_t *pa = nm.blob + nm.off[ab];
  const uint8_t *pb = nm.blob + nm.off[bb];
  int64_t na = nm.off[ab + 1] - nm.off[ab], nb = nm.off[bb + 1] - nm.off[bb];
  int64_t ta = na + la, tb = nb + lb;
  for (int64_t i = 0; i < ta && i < tb; i++) {
    uint8_t ca = i < na ? pa[i] : (uint8_t)sa[i - na];
    uint8_t cb = i < nb ? pb[i] : (uint8_t)sb[i - nb];
    if (ca != cb) return ca < cb ? -1 : 1;
  }
  return (ta > tb) - (ta < tb);
}

// ----------------------------------------------------------------------------
// device-wide primitives (prims.cu)

// exclusive scan of n values; out may alias in; total (if non-null) is a
// device pointer receiving the sum.  T in {int32_t, int64_t}.
template <typename T>
int dev_exclusive_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err);
// out[i] = in[0] + ... + in[i] (T = int64_t)
template <typename T>
int dev_inclusive_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err);

// stable LSD radix sort of (key, value) pairs on bits [0, bits)
int dev_radix_sort_u32(mp_ctx *ctx, uint32_t *keys, uint32_t *vals, int64_t n, int bits,
                       mp_err *err);
int dev_radix_sort_u64(mp_ctx *ctx, uint64_t *keys, uint32_t *vals, int64_t n, int bits,
                       mp_err *err);
// stable sort of kin's bits [0, bits) into kout, the positions 0..n-1 carried
// into vout (kin may alias kout)
int64_t dev_radix_rank_min_n();
int dev_radix_rank_u32(mp_ctx *ctx, const uint32_t *kin, int64_t n, int bits, int32_t *rank, mp_err *err);
int dev_radix_sort_u32_iota(mp_ctx *ctx, const uint32_t *kin, uint32_t *kout, uint32_t *vout, int64_t n, int bits,
                            mp_err *err);

// read back one int64 from device memory (synchronizes the stream)
int dev_read_i64(mp_ctx *ctx, const int64_t *d, int64_t *h, mp_err *err);
int dev_read_n(mp_ctx *ctx, const void *d, void *h, size_t bytes, mp_err *err);

static inline int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b)) b++;
  return b;
}

// ----------------------------------------------------------------------------
// warp helpers

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan_add(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(FULL_MASK, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

__device__ __forceinline__ int64_t warp_incl_scan_max(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t u = __shfl_up_sync(FULL_MASK, v, o);
    if (lane >= o && u > v) v = u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// ----------------------------------------------------------------------------
// thread groups for CTA-level helpers: the whole CTA, or a run of warps
// synchronizing on a named barrier (so different warps of one CTA can run
// different stages of a trace concurrently)

struct CtaGroup {
  __device__ __forceinline__ int idx() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ bool sync_and(bool v) const { return __syncthreads_and(v); }
};

struct WarpGroup {
  int first_warp, nwarps, bar;  // bar: named barrier 1..15
  __device__ __forceinline__ int idx() const { return (int)threadIdx.x - 32 * first_warp; }
  __device__ __forceinline__ int size() const { return 32 * nwarps; }
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * nwarps) : "memory");
  }
  __device__ __forceinline__ bool sync_and(bool v) const {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.and.pred q, %2, %3, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"((unsigned)v), "r"(bar), "r"(32 * nwarps)
        : "memory");
    return r != 0;
  }
};
