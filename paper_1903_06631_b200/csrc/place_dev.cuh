// place_dev.cuh — warp-level pieces of the SmartPool placement step
// (_pick_offset, smartpool.py:101-119): bitonic sorts of neighbour ranges
// and the hole scan.  Shared by the grid-wide dataflow placement
// (placement.cu) and the one-CTA-per-trace sweep (sweep.cu).
#pragma once

#include <climits>

#include "common.cuh"

struct IV {
  int64_t s, e;
};

__device__ __forceinline__ bool iv_less(int64_t as, int64_t ae, int64_t bs, int64_t be) {
  return as < bs || (as == bs && ae < be);
}

// bitonic sort of 32*K (start, end) pairs held as element i = r*32 + lane
template <int K>
__device__ __forceinline__ void warp_bitonic_reg(int64_t (&s)[K], int64_t (&e)[K]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < K; r++) {
          if ((r & jr) == 0) {
            const int r2 = r | jr;
            const bool up = ((r * 32) & k) == 0;
            bool gt = iv_less(s[r2], e[r2], s[r], e[r]);
            if (up == gt) {
              int64_t ts = s[r], te = e[r];
              s[r] = s[r2]; e[r] = e[r2]; s[r2] = ts; e[r2] = te;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < K; r++) {
          int64_t os = __shfl_xor_sync(FULL_MASK, s[r], j);
          int64_t oe = __shfl_xor_sync(FULL_MASK, e[r], j);
          const bool up = ((r * 32 + lane) & k) == 0;
          const bool lower = (lane & j) == 0;
          bool take = (lower == up) ? iv_less(os, oe, s[r], e[r]) : iv_less(s[r], e[r], os, oe);
          if (take) { s[r] = os; e[r] = oe; }
        }
      }
    }
  }
}

// bitonic sort of n2 pairs in memory (shared or global), one warp
template <typename P>
__device__ void warp_bitonic_mem(P buf, int n2) {
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
  bool ok = valid && s > tb && s - tb >= need;
  int64_t len = s - tb;
  unsigned bal = __ballot_sync(FULL_MASK, ok);
  if (policy == 0) {
    if (bal) {
      h.best_off = __shfl_sync(FULL_MASK, tb, __ffs(bal) - 1);
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

__device__ __forceinline__ int warp_max_i32(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}

// One compare-exchange step of a bitonic network on a 64-bit key: one
// 64-bit compare and one select (the keys are unique up to equal padding,
// so "take the partner" is a single predicate: the lane keeps the minimum
// iff it sits low in an ascending block, and the partner is the minimum
// iff it compares below).
__device__ __forceinline__ uint64_t cx_key(uint64_t x, uint64_t o, bool keep_min) {
  return ((o < x) == keep_min) ? o : x;
}

// bitonic sort of 32*K unsigned keys held as element i = r*32 + lane
template <int K>
__device__ __forceinline__ void warp_bitonic_keys(uint64_t (&x)[K]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < K; r++) {
          if ((r & jr) == 0) {
            const int r2 = r | jr;
            const bool up = ((r * 32) & k) == 0;
            bool sw = (x[r2] < x[r]) == up;
            uint64_t a = sw ? x[r2] : x[r], b = sw ? x[r] : x[r2];
            x[r] = a;
            x[r2] = b;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < K; r++) {
          uint64_t o = __shfl_xor_sync(FULL_MASK, x[r], j);
          const bool up = ((r * 32 + lane) & k) == 0;
          const bool lower = (lane & j) == 0;
          x[r] = cx_key(x[r], o, lower == up);
        }
      }
    }
  }
}

// The same network with the stage loops rolled (runtime k, j): a fraction
// of the code of the unrolled form, for the rarer long rows, so the hot
// loop stays inside the instruction cache.
template <int K>
__device__ __forceinline__ void warp_bitonic_keys_rolled(uint64_t (&x)[K]) {
  static_assert(K == 2 || K == 4, "rolled network is for 64 or 128 keys");
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        if (K == 4 && j == 64) {
#pragma unroll
          for (int r = 0; r < 2; r++) {
            const bool up = ((r * 32) & k) == 0;
            bool sw = (x[r + 2] < x[r]) == up;
            uint64_t a = sw ? x[r + 2] : x[r], b = sw ? x[r] : x[r + 2];
            x[r] = a;
            x[r + 2] = b;
          }
        } else {
#pragma unroll
          for (int r = 0; r < K; r += 2) {
            const bool up = ((r * 32) & k) == 0;
            bool sw = (x[r + 1] < x[r]) == up;
            uint64_t a = sw ? x[r + 1] : x[r], b = sw ? x[r] : x[r + 1];
            x[r] = a;
            x[r + 1] = b;
          }
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < K; r++) {
          uint64_t o = __shfl_xor_sync(FULL_MASK, x[r], j);
          const bool up = ((r * 32 + lane) & k) == 0;
          x[r] = cx_key(x[r], o, lower == up);
        }
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Lane-major forms for 64-128 ranges: sorted position p = lane * K + r.  The
// bitonic network is the same, with the low log2(K) index bits inside a
// lane's registers: every stage with j < K is a register compare-exchange
// (13 of the 28 stages for K = 4, against 3 in the register-major form),
// and _pick_offset becomes ONE pass: a lane's K consecutive ranges in
// order, one warp max-scan of the lanes' end maxima, one reduction.

template <int K>
__device__ __forceinline__ void lm_cx_regs(uint64_t (&x)[K], int j, int k, int lane) {
#pragma unroll
  for (int r = 0; r < K; r++) {
    if ((r & j) == 0) {
      const int r2 = r | j;
      const bool up = ((lane * K + r) & k) == 0;
      const bool sw = (x[r2] < x[r]) == up;
      const uint64_t a = sw ? x[r2] : x[r], b = sw ? x[r] : x[r2];
      x[r] = a;
      x[r2] = b;
    }
  }
}

// unrolled
template <int K>
__device__ __forceinline__ void warp_bitonic_keys_lm_unrolled(uint64_t (&x)[K]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < K) {
        lm_cx_regs<K>(x, j, k, lane);
      } else {
        const int jl = j / K;
        const bool lower = (lane & jl) == 0;
#pragma unroll
        for (int r = 0; r < K; r++) {
          const uint64_t o = __shfl_xor_sync(FULL_MASK, x[r], jl);
          const bool up = ((lane * K + r) & k) == 0;
          x[r] = cx_key(x[r], o, lower == up);
        }
      }
    }
  }
}

// rolled stage loops (runtime k, j); j < K branches to the register form
template <int K>
__device__ __forceinline__ void warp_bitonic_keys_lm(uint64_t (&x)[K]) {
  static_assert(K == 2 || K == 4, "lane-major network is for 64 or 128 keys");
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < K) {
        if (K == 4 && j == 2) lm_cx_regs<K>(x, 2, k, lane);
        else lm_cx_regs<K>(x, 1, k, lane);
      } else {
        const int jl = j / K;
        const bool lower = (lane & jl) == 0;
#pragma unroll
        for (int r = 0; r < K; r++) {
          const uint64_t o = __shfl_xor_sync(FULL_MASK, x[r], jl);
          const bool up = ((lane * K + r) & k) == 0;
          x[r] = cx_key(x[r], o, lower == up);
        }
      }
    }
  }
}

// _pick_offset over 32 * K sorted ranges held lane-major (s[r], e[r] of
// position lane * K + r, valid below m); returns the offset
template <int K>
__device__ __forceinline__ int64_t hole_lm(const int64_t (&s)[K], const int64_t (&e)[K], int m, int64_t need,
                                           int policy) {
  const int lane = threadIdx.x & 31;
  int64_t lmax = INT64_MIN;
#pragma unroll
  for (int r = 0; r < K; r++)
    if (lane * K + r < m && e[r] > lmax) lmax = e[r];
  const int64_t incl = warp_incl_scan_max(lmax);
  int64_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
  if (lane == 0) excl = INT64_MIN;
  int64_t run = excl > 0 ? excl : 0;
  bool mine = false;
  int64_t my_off = 0, bl = INT64_MAX, bo = INT64_MAX;
#pragma unroll
  for (int r = 0; r < K; r++) {
    if (lane * K + r >= m) continue;
    if (s[r] > run && s[r] - run >= need) {
      const int64_t len = s[r] - run;
      if (!mine) { mine = true; my_off = run; }
      if (len < bl || (len == bl && run < bo)) { bl = len; bo = run; }
    }
    if (e[r] > run) run = e[r];
  }
  const int64_t cmax = __shfl_sync(FULL_MASK, incl, 31);
  const int64_t top = cmax > 0 ? cmax : 0;
  if (policy == 0) {
    const unsigned bal = __ballot_sync(FULL_MASK, mine);
    return bal ? __shfl_sync(FULL_MASK, my_off, __ffs(bal) - 1) : top;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t ol = __shfl_xor_sync(FULL_MASK, bl, o), oo = __shfl_xor_sync(FULL_MASK, bo, o);
    if (ol < bl || (ol == bl && oo < bo)) { bl = ol; bo = oo; }
  }
  return bl != INT64_MAX ? bo : top;
}

// bitonic sort of the first N (<= 32) lanes' keys, one per lane: lanes >= N
// hold the all-ones padding already, so the 32-key result is sorted too
template <int N>
__device__ __forceinline__ void warp_bitonic_keys_first(uint64_t &x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(FULL_MASK, x, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = cx_key(x, o, lower == up);
    }
  }
}

// hole_lm on 32-bit values (every end below 2^31): one shuffle per scan
// level and redux reductions
// L = the lanes that can hold ranges (m <= L * K): a row of at most 8 / 16
// ranges needs 3 / 4 scan levels, and the top is lane L - 1's prefix
template <int K, int L = 32>
__device__ __forceinline__ int64_t hole_lm32(const int32_t (&s)[K], const int32_t (&e)[K], int m, int32_t need,
                                             int policy) {
  const int lane = threadIdx.x & 31;
  int32_t lmax = INT32_MIN;
#pragma unroll
  for (int r = 0; r < K; r++)
    if (lane * K + r < m && e[r] > lmax) lmax = e[r];
  int32_t incl = lmax;
#pragma unroll
  for (int o = 1; o < L; o <<= 1) {
    const int32_t u = __shfl_up_sync(FULL_MASK, incl, o);
    if (lane >= o && u > incl) incl = u;
  }
  int32_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
  if (lane == 0) excl = INT32_MIN;
  int32_t run = excl > 0 ? excl : 0;
  bool mine = false;
  int32_t my_off = 0, bl = INT32_MAX, bo = INT32_MAX;
#pragma unroll
  for (int r = 0; r < K; r++) {
    if (lane * K + r >= m) continue;
    if (s[r] > run && s[r] - run >= need) {
      const int32_t len = s[r] - run;
      if (!mine) { mine = true; my_off = run; }
      if (len < bl || (len == bl && run < bo)) { bl = len; bo = run; }
    }
    if (e[r] > run) run = e[r];
  }
  const int32_t cmax = __shfl_sync(FULL_MASK, incl, L - 1);
  const int32_t top = cmax > 0 ? cmax : 0;
  if (policy == 0) {
    const unsigned bal = __ballot_sync(FULL_MASK, mine);
    return bal ? __shfl_sync(FULL_MASK, my_off, __ffs(bal) - 1) : top;
  }
  // (length, offset) minimum: non-negative, so the unsigned redux order is right
  const unsigned ml = __reduce_min_sync(FULL_MASK, (unsigned)bl);
  const unsigned mo = __reduce_min_sync(FULL_MASK, (unsigned)bl == ml ? (unsigned)bo : 0xffffffffu);
  return ml != (unsigned)INT32_MAX ? (int64_t)mo : (int64_t)top;
}
