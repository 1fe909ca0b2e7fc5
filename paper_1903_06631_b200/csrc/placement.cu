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
// Scheduling is asynchronous dataflow: a ready queue (claimed in order,
// published by the last predecessor to finish) feeds persistent warps, so
// a variable starts as soon as its own predecessors are placed instead of
// waiting for a whole wavefront.  The CSR rows arrive partitioned into
// predecessors and successors by the conflict build (conflict.cu).
//
// Memory protocol: offsets and levels are written once,
// from the sentinels -1 / 0, with relaxed stores; successor counters,
// queue slots and polls are relaxed too.  A variable whose counter reached
// zero reads its predecessors' offsets until none is a sentinel (a
// non-sentinel value is final), so no release fence has to wait for the
// offset store before the counters go down (3.5 % faster than acq_rel
// counters + fences).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "handles.cuh"
#include "place_dev.cuh"

// PLACE_TRACE=1 builds (tools/place_trace.py) record per-variable
// %globaltimer stamps: placed, claimed, made ready, gathered, sorted.
#ifndef PLACE_REC
#define PLACE_REC 1
#endif
#ifndef PLACE_TRACE
#define PLACE_TRACE 0
#endif
// experiment switches (tools/ab_place.sh)
#ifndef PLACE_SUCC_PIPE
#define PLACE_SUCC_PIPE 2  // successor decrements batched 128 per round trip: 1 always, 2 rows with > 32 successors, 0 never
#endif
#ifndef PLACE_BACKOFF
#define PLACE_BACKOFF 1    // exponential idle backoff
#endif
#ifndef PLACE_LANE_MAJOR
#define PLACE_LANE_MAJOR 1  // 64-128 predecessors: lane-major network + one-pass hole scan
#endif
#ifndef PLACE_LM_KMIN
#define PLACE_LM_KMIN 2  // 4: only the 65-128 rows (1.28 ms), 2: also 33-64 (1.21 ms vs 1.34 register-major)
#endif
#ifndef PLACE_HOLE32
#define PLACE_HOLE32 1  // 32-bit hole scan when every end is below 2^31
#endif
#ifndef PLACE_SE_KEYS
#define PLACE_SE_KEYS 1  // narrow variables sort (start << 32 | end) keys
#endif
#ifndef PLACE_SHORT_SCANS
#define PLACE_SHORT_SCANS 1  // rows of <= 8 / 16 ranges: 3 / 4-level hole scans
#endif
#ifndef PLACE_SHORT_NETS
#define PLACE_SHORT_NETS 1  // rows of <= 8 / 16 predecessors sort with an 8 / 16-wide network
#endif
#ifndef PLACE_LM_K4_UNROLLED
#define PLACE_LM_K4_UNROLLED 0
#endif
#ifndef PLACE_K4_ROLLED
#define PLACE_K4_ROLLED 1  // rolled stage loops for 65..128 predecessors
#endif
#define PT_STAMP(slot, v)                                                 \
  do {                                                                    \
    if (PLACE_TRACE && a.tdone) {                                         \
      unsigned long long t_;                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory");    \
      a.tdone[(slot) * a.V + (v)] = t_;                                   \
    }                                                                     \
  } while (0)

struct PlaceArgs {
  int64_t V;
  const int64_t *row_off;
  const int32_t *col;   // rows partitioned: preds (earlier in placement order) first
  const int32_t *pcnt;
  const int64_t *size;
  int64_t *off;
  int32_t *level;       // DAG depth of each placed variable
  int32_t *remaining;   // unplaced preds
  int32_t *queue;       // ready variables, v + 1 (0 = slot not yet published)
  int32_t *head, *tail;
  int32_t *done;        // variables placed (flushed per queue claim)
  int policy;           // 0 first_fit, 1 best_fit
  IV *wscratch;         // 128 ranges per warp (packed-key fallback)
  IV *arena;            // long rows (> 128 preds) bump-allocate here
  unsigned long long *arena_top;
  long long *footprint;
  int32_t *depth;
  int32_t dbg_v;
  unsigned long long *tdone;  // debug (MP_PLACE_TRACE): %globaltimer when each variable was placed
  longlong2 *rec;       // placed-variable records (k_place_async<true>, see pred_range)
};

__device__ __forceinline__ int64_t ld_relaxed_s64(const int64_t *p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_relaxed_s32(const int32_t *p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Range [s, e) and level of placed predecessor j.  Offsets and levels are
// written once (from -1 / 0 sentinels) with relaxed stores and the counters
// carry no release/acquire, so a predecessor counted as placed may not be
// visible yet — read until it is (a non-sentinel value is final).  REC: one
// 16-byte record {offset, size | level << 32} per variable, written by one
// store from all-ones (a half not yet visible reads offset -1 or level -1),
// so the gather is one load per predecessor instead of three; 1.35 vs 1.38
// ms on config 4.  Used when every size fits 32 bits.
template <bool REC>
__device__ __forceinline__ void pred_range(const PlaceArgs &a, int32_t j, int64_t &s, int64_t &e, int &l) {
  if constexpr (REC) {
    for (;;) {
      long long w0, w1;
      asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(a.rec + j) : "memory");
      l = (int)(w1 >> 32);
      if (w0 >= 0 && l > 0) {
        s = w0;
        e = w0 + (int64_t)(uint32_t)w1;
        return;
      }
      __nanosleep(32);
    }
  } else {
    for (;;) {
      s = ld_relaxed_s64(&a.off[j]);
      l = ld_relaxed_s32(&a.level[j]);
      if (s >= 0 && l > 0) break;
      __nanosleep(32);
    }
    e = s + a.size[j];
  }
}

// Gather the predecessors' ranges, sort them by start and replay
// _pick_offset.  Ranges are sorted as one 64-bit key (start << IB | slot):
// equal starts may come in any order (the hole scan only sees the running
// max of ends), so the slot just makes keys unique and carries the end.
template <bool REC, int K, bool NARROW>
__device__ __forceinline__ int64_t place_reg(const PlaceArgs &a, int64_t rb, int m, int64_t need, int &lvl,
                                             bool &ok) {
  const int lane = threadIdx.x & 31;
  constexpr int IB = K == 1 ? 5 : K == 2 ? 6 : K == 4 ? 7 : 8;
  uint64_t x[K];
  int64_t e[K];
  int lv = 0;
  bool big = false;
#pragma unroll
  for (int r = 0; r < K; r++) {
    int i = r * 32 + lane;
    x[r] = ~0ull;
    e[r] = INT64_MIN;
    if (i < m) {
      int32_t j = a.col[rb + i];
      int64_t s;
      int l;
      pred_range<REC>(a, j, s, e[r], l);
      lv = max(lv, l);
      big |= (uint64_t)s >> (63 - IB) != 0;
      x[r] = ((uint64_t)s << IB) | (uint64_t)i;
    }
  }
  ok = !__any_sync(FULL_MASK, big);
  if (!ok) return 0;
  // NARROW kernel (pools under 2^31 bytes): every end and the request below
  // 2^31 lets the hole scan run in 32 bits; any wider value takes the 64-bit
  // scan for this variable
  bool narrow = false;
  if constexpr (NARROW) {
    bool wide = need >= (int64_t)INT32_MAX;
#pragma unroll
    for (int r = 0; r < K; r++) wide |= e[r] >= (int64_t)INT32_MAX;
    narrow = !__any_sync(FULL_MASK, wide);
  }
  lvl = (int)__reduce_max_sync(FULL_MASK, (unsigned)lv) + 1;
  if (lane == 0) PT_STAMP(3, a.dbg_v);
  if constexpr ((PLACE_LANE_MAJOR && K >= PLACE_LM_KMIN) || (K == 1 && NARROW)) {
    // lane-major network and one-pass hole scan (place_dev.cuh)
    if (PLACE_SE_KEYS && NARROW && narrow) {
      // starts and ends both fit 31 bits: the key is (start << 32 | end),
      // so the sorted keys carry the ends and no lookup by slot follows
#pragma unroll
      for (int r = 0; r < K; r++)
        if (x[r] != ~0ull) x[r] = ((x[r] >> IB) << 32) | (uint64_t)(uint32_t)e[r];
    }
    if constexpr (K == 1) {
      if (m <= 8) warp_bitonic_keys_first<8>(x[0]);
      else if (m <= 16) warp_bitonic_keys_first<16>(x[0]);
      else warp_bitonic_keys_first<32>(x[0]);
    } else if constexpr (K == 2 || PLACE_LM_K4_UNROLLED) {
      warp_bitonic_keys_lm_unrolled<K>(x);
    } else {
      warp_bitonic_keys_lm<K>(x);
    }
    if (lane == 0) PT_STAMP(4, a.dbg_v);
    if (PLACE_SE_KEYS && NARROW && narrow) {
      int32_t s32[K], e32[K];
#pragma unroll
      for (int r = 0; r < K; r++) { s32[r] = (int32_t)(x[r] >> 32); e32[r] = (int32_t)(uint32_t)x[r]; }
      if constexpr (K == 1 && PLACE_SHORT_SCANS) {
        if (m <= 8) return hole_lm32<1, 8>(s32, e32, m, (int32_t)need, a.policy);
        if (m <= 16) return hole_lm32<1, 16>(s32, e32, m, (int32_t)need, a.policy);
      }
      return hole_lm32<K>(s32, e32, m, (int32_t)need, a.policy);
    }
    int64_t ss[K], es[K];
#pragma unroll
    for (int r = 0; r < K; r++) {
      const int src = (int)(x[r] & ((1u << IB) - 1));
      es[r] = INT64_MIN;
#pragma unroll
      for (int q = 0; q < K; q++) {
        const int64_t t = __shfl_sync(FULL_MASK, e[q], src & 31);
        if ((src >> 5) == q) es[r] = t;
      }
      ss[r] = (int64_t)(x[r] >> IB);
    }
    if (NARROW && narrow) {
      int32_t s32[K], e32[K];
#pragma unroll
      for (int r = 0; r < K; r++) { s32[r] = (int32_t)ss[r]; e32[r] = (int32_t)es[r]; }
      return hole_lm32<K>(s32, e32, m, (int32_t)need, a.policy);
    }
    return hole_lm<K>(ss, es, m, need, a.policy);
  }
  if constexpr (K == 1 && PLACE_SHORT_NETS) {
    // a network only as wide as the row (m <= 8 / 16: 6 / 10 stages, not 15)
    if (m <= 8) warp_bitonic_keys_first<8>(x[0]);
    else if (m <= 16) warp_bitonic_keys_first<16>(x[0]);
    else warp_bitonic_keys_first<32>(x[0]);
  } else if constexpr (K <= 2 || !PLACE_K4_ROLLED) {
    warp_bitonic_keys<K>(x);
  } else {
    warp_bitonic_keys_rolled<K>(x);
  }
  if (lane == 0) PT_STAMP(4, a.dbg_v);
  HoleState h{0, 0, 0, false};
#pragma unroll
  for (int r = 0; r < K; r++) {
    if (r * 32 >= m) break;
    // end of the range now at sorted position r*32 + lane
    int src = (int)(x[r] & ((1u << IB) - 1));
    int64_t es = INT64_MIN;
#pragma unroll
    for (int q = 0; q < K; q++) {
      int64_t t = __shfl_sync(FULL_MASK, e[q], src & 31);
      if ((src >> 5) == q) es = t;
    }
    bool valid = r * 32 + lane < m;
    int64_t ss = (int64_t)(x[r] >> IB);
    if (hole_chunk(h, ss, es, valid, need, a.policy)) break;
  }
  return h.found ? h.best_off : h.top;
}

template <bool REC, typename P>
__device__ int64_t place_mem(const PlaceArgs &a, P buf, int64_t rb, int m, int64_t need, int &lvl) {
  const int lane = threadIdx.x & 31;
  int n2 = 64;
  while (n2 < m) n2 <<= 1;
  int lv = 0;
  for (int i = lane; i < n2; i += 32) {
    IV x{INT64_MAX, INT64_MAX};
    if (i < m) {
      int32_t j = a.col[rb + i];
      int l;
      pred_range<REC>(a, j, x.s, x.e, l);
      lv = max(lv, l);
    }
    buf[i] = x;
  }
  lvl = (int)__reduce_max_sync(FULL_MASK, (unsigned)lv) + 1;
  __syncwarp();
  warp_bitonic_mem(buf, n2);
  HoleState h{0, 0, 0, false};
  for (int base = 0; base < m; base += 32) {
    int i = base + lane;
    IV x = i < m ? buf[i] : IV{0, 0};
    if (hole_chunk(h, x.s, x.e, i < m, need, a.policy)) break;
  }
  __syncwarp();
  return h.found ? h.best_off : h.top;
}

__device__ __forceinline__ int atom_dec_relaxed(int32_t *p) {
  int old;
  asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}


#ifndef PLACE_SUCC_BATCH
#define PLACE_SUCC_BATCH 2  // round 2 re-tune: 2 rows of 32 per round trip (4: +1.5 %, 1: +2 %)
#endif
constexpr int SUCC_BATCH = PLACE_SUCC_BATCH;  // successor rows of 32 decremented per round trip
#ifndef PLACE_SLEEP0_NS
#define PLACE_SLEEP0_NS 64
#endif
#ifndef PLACE_DONE_MASK
#define PLACE_DONE_MASK 7
#endif
#ifndef PLACE_MAX_SLEEP_NS
#define PLACE_MAX_SLEEP_NS 1024  // 256: 3.5 % slower, 4096: 3 % slower
#endif
constexpr unsigned PLACE_MAX_SLEEP = PLACE_MAX_SLEEP_NS;  // ns, idle-warp poll backoff cap

constexpr int PLACE_THREADS = 256;
#ifndef PLACE_MIN_BLOCKS
#define PLACE_MIN_BLOCKS 5  // <= 48 registers: 40 resident warps per SM
#endif



// offset of one variable whose predecessors are all placed (warp-wide)
template <bool REC, bool NARROW>
__device__ __forceinline__ int64_t place_var(const PlaceArgs &a, int32_t v, int64_t gwarp, int64_t rb, int m,
                                             int64_t need, int &lvl) {
  const int lane = threadIdx.x & 31;
  int64_t o = 0;
  bool ok = true;
  lvl = 1;
  if (m == 0) o = 0;
  else if (m <= 32) o = place_reg<REC, 1, NARROW>(a, rb, m, need, lvl, ok);
  else if (m <= 64) o = place_reg<REC, 2, NARROW>(a, rb, m, need, lvl, ok);
  else if (m <= 128) o = place_reg<REC, 4, NARROW>(a, rb, m, need, lvl, ok);
  else ok = false;
  // long rows, or offsets too large to pack: sort (start, end) pairs in
  // global scratch
  if (!ok) {
    IV *buf = a.wscratch + gwarp * 128;
    if (m > 128) {
      unsigned long long n2 = 64;
      while (n2 < (unsigned long long)m) n2 <<= 1;
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(a.arena_top, n2);
      buf = a.arena + __shfl_sync(FULL_MASK, at, 0);
    }
    o = place_mem<REC>(a, buf, rb, m, need, lvl);
  }
  return o;
}

// Asynchronous dataflow placement: warps claim ready variables from a
// queue in order; placing a variable decrements its successors' counters
// and the last predecessor to finish publishes the successor.  No grid-wide
// barrier: a variable starts the moment its last predecessor is placed.
template <bool REC, bool NARROW>
__global__ void __launch_bounds__(PLACE_THREADS, PLACE_MIN_BLOCKS) k_place_async(PlaceArgs a) {
  PDL_WAIT();
  const int lane = threadIdx.x & 31;
  int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  long long fp = LLONG_MIN;
  int dmax = 0;
  // up to two successors this warp made ready and kept for itself, taken
  // in the order they became ready (a deeper private stack, or LIFO order,
  // starves the other warps: 1.9-4.7 ms instead of 1.45)
  int32_t next = -1, next2 = -1;
  int local_done = 0;    // placements not yet added to the global count
  for (;;) {
    int32_t v;
    if (next >= 0) {
      v = next;
      next = next2;
      next2 = -1;
    } else {
      int i = 0;
      if (lane == 0) {
        if (local_done) atomicAdd(a.done, local_done);
        i = atomicAdd(a.head, 1);
      }
      local_done = 0;
      int v1 = 0;
      if (lane == 0) {
        // continuation means not every variable passes through the queue,
        // so an empty slot ends the warp once all are placed; idle warps back
        // off exponentially and look at the done count only now and then
        // (thousands of pollers on one line slow the L2 slice the counters
        // live in)
        const int32_t *q = a.queue + (i < a.V ? i : 0);
        unsigned ns = PLACE_SLEEP0_NS;
        for (int spin = 0; !v1; spin++) {
          if (i < a.V) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v1) : "l"(q) : "memory");
          if (v1) break;
          if ((!PLACE_BACKOFF || (spin & PLACE_DONE_MASK) == PLACE_DONE_MASK) && *(volatile int *)a.done >= a.V) { v1 = -1; break; }
          __nanosleep(PLACE_BACKOFF ? ns : 20);
          if (ns < PLACE_MAX_SLEEP) ns <<= 1;
        }
      }
      v1 = __shfl_sync(FULL_MASK, v1, 0);
      if (v1 < 0) break;
      v = v1 - 1;
    }
    if (lane == 0) PT_STAMP(1, v);
    int64_t rb = a.row_off[v], re = a.row_off[v + 1];
    int m = a.pcnt[v];
    int64_t need = a.size[v];
    int lvl;
#if PLACE_TRACE
    PlaceArgs ad = a;
    ad.dbg_v = v;
    int64_t o = place_var<REC, NARROW>(ad, v, gwarp, rb, m, need, lvl);
#else
    int64_t o = place_var<REC, NARROW>(a, v, gwarp, rb, m, need, lvl);
#endif
    if (lane == 0) {
      if constexpr (REC) {
        long long w1 = (long long)(((uint64_t)(uint32_t)lvl << 32) | (uint64_t)(uint32_t)need);
        asm volatile("st.relaxed.gpu.global.v2.s64 [%0], {%1, %2};" ::"l"(a.rec + v), "l"(o), "l"(w1) : "memory");
        a.off[v] = o;
        if (PLACE_TRACE) a.level[v] = lvl;
      } else {
        asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(a.level + v), "r"(lvl) : "memory");
        asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(a.off + v), "l"(o) : "memory");
      }
      if (o + need > fp) fp = o + need;
      if (lvl > dmax) dmax = lvl;
      PT_STAMP(0, v);
    }
    local_done++;
    __syncwarp();
    if (PLACE_SUCC_PIPE && re - (rb + m) > (PLACE_SUCC_PIPE == 2 ? 32 : 0)) {
      // decrement every successor's counter, SUCC_BATCH rows of 32 in
      // flight at once instead of one round trip per 32
      for (int64_t base = rb + m; base < re; base += 32 * SUCC_BATCH) {
        int32_t jj[SUCC_BATCH];
        int rem[SUCC_BATCH];
#pragma unroll
        for (int c = 0; c < SUCC_BATCH; c++) {
          int64_t k = base + c * 32 + lane;
          jj[c] = k < re ? a.col[k] : -1;
        }
#pragma unroll
        for (int c = 0; c < SUCC_BATCH; c++) rem[c] = jj[c] >= 0 ? atom_dec_relaxed(&a.remaining[jj[c]]) : 0;
        bool any = false;
#pragma unroll
        for (int c = 0; c < SUCC_BATCH; c++) any |= rem[c] == 1;
        if (!__any_sync(FULL_MASK, any)) continue;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < SUCC_BATCH; c++) {
          bool ready = rem[c] == 1;
          int32_t j = jj[c];
          if (ready) PT_STAMP(2, j);
          unsigned bal = __ballot_sync(FULL_MASK, ready);
          // keep newly ready successors while the stack has room; publish the rest
          while (bal && next2 < 0) {
            int keep = __ffs(bal) - 1;
            int32_t jk = __shfl_sync(FULL_MASK, j, keep);
            if (next < 0) next = jk;
            else next2 = jk;
            if (lane == keep) ready = false;
            bal &= bal - 1;
          }
          if (bal) {
            int qb = 0;
            if (lane == __ffs(bal) - 1) qb = atomicAdd(a.tail, __popc(bal));
            qb = __shfl_sync(FULL_MASK, qb, __ffs(bal) - 1);
            if (ready) {
              int32_t *q = a.queue + qb + __popc(bal & lanemask_lt());
              asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(q), "r"(j + 1) : "memory");
            }
          }
        }
      }
    }
    if (!PLACE_SUCC_PIPE || (PLACE_SUCC_PIPE == 2 && re - (rb + m) <= 32)) {
    for (int64_t k = rb + m + lane; k - lane < re; k += 32) {
      bool ready = false;
      int32_t j = 0;
      if (k < re) {
        j = a.col[k];
        ready = atom_dec_relaxed(&a.remaining[j]) == 1;
      }
      if (ready) PT_STAMP(2, j);
      unsigned bal = __ballot_sync(FULL_MASK, ready);
      while (bal && next2 < 0) {
        int keep = __ffs(bal) - 1;
        int32_t jk = __shfl_sync(FULL_MASK, j, keep);
        if (next < 0) next = jk;
        else next2 = jk;
        if (lane == keep) ready = false;
        bal &= bal - 1;
      }
      if (bal) {
        int qb = 0;
        if (lane == __ffs(bal) - 1) qb = atomicAdd(a.tail, __popc(bal));
        qb = __shfl_sync(FULL_MASK, qb, __ffs(bal) - 1);
        if (ready) {
          int32_t *q = a.queue + qb + __popc(bal & lanemask_lt());
          asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(q), "r"(j + 1) : "memory");
        }
      }
    }
    }
  }
  if (lane == 0) {
    atomicMax(a.footprint, fp);
    atomicMax(a.depth, dmax);
  }
}

// ---------------------------------------------------------------------------
// placement order and row partition

__global__ void k_tie_keys(int64_t V, const int64_t *tiekey, uint64_t *keys, uint32_t *vals) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    keys[v] = (uint64_t)tiekey[v] ^ 0x8000000000000000ull;
    vals[v] = (uint32_t)v;
  }
}


__global__ void k_size_keys(int64_t V, const int64_t *size, const uint32_t *vals, uint64_t *keys,
                            unsigned long long *mn, unsigned long long *mx) {
  PDL_WAIT();
  unsigned long long lmn = ~0ull, lmx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = desc_size_key(size[vals[i]]);
    keys[i] = k;
    lmn = k < lmn ? k : lmn;
    lmx = k > lmx ? k : lmx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(FULL_MASK, lmn, o), b = __shfl_xor_sync(FULL_MASK, lmx, o);
    lmn = a < lmn ? a : lmn;
    lmx = b > lmx ? b : lmx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mn, lmn);
    atomicMax(mx, lmx);
  }
}

__global__ void k_sub_keys(int64_t V, uint64_t *keys, const unsigned long long *mn) {
  PDL_WAIT();
  uint64_t m = *mn;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] -= m;
}

__global__ void k_iota(int64_t V, uint32_t *vals) {
  PDL_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    vals[i] = (uint32_t)i;
}

__global__ void k_rank(int64_t V, const uint32_t *order, int32_t *rank) {
  PDL_WAIT();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < V; q += (int64_t)gridDim.x * blockDim.x)
    rank[order[q]] = (int32_t)q;
}

// counters, the initial ready queue, the placement sentinels (record
// all-ones, or offset -1 / level 0) and the footprint's starting value
__global__ void k_ready_init(int64_t V, const int32_t *pcnt, int32_t *remaining, int32_t *queue, int32_t *tail,
                             unsigned long long *arena_need, longlong2 *rec, int64_t *off, int32_t *level,
                             long long *footprint) {
  PDL_WAIT();
  if (blockIdx.x == 0 && threadIdx.x == 0) *footprint = LLONG_MIN;
  unsigned long long need = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    int c = pcnt[v];
    remaining[v] = c;
    if (rec) {
      rec[v] = make_longlong2(-1, -1);
    } else {
      off[v] = -1;
      level[v] = 0;
    }
    if (c > 128) {
      unsigned long long n2 = 64;
      while (n2 < (unsigned long long)c) n2 <<= 1;
      need += n2;
    }
    // one tail atomic per warp (thousands of single increments on one
    // address serialise in L2)
    const unsigned am = __activemask();
    const unsigned z = __ballot_sync(am, c == 0);
    if (z) {
      const int lead = __ffs(z) - 1;
      int qb = 0;
      if ((int)(threadIdx.x & 31) == lead) qb = atomicAdd(tail, __popc(z));
      qb = __shfl_sync(am, qb, lead);
      if (c == 0) queue[qb + __popc(z & lanemask_lt())] = (int32_t)(v + 1);
    }
  }
  need = warp_sum(need);
  if ((threadIdx.x & 31) == 0 && need) atomicAdd(arena_need, need);
}

// placement rank of every vertex: (-size, tiekey or vertex index)
__global__ void k_size_range(int64_t V, const int64_t *size, unsigned long long *mm) {
  PDL_WAIT();
  unsigned long long lmn = ~0ull, lmx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = desc_size_key(size[i]);
    lmn = k < lmn ? k : lmn;
    lmx = k > lmx ? k : lmx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(FULL_MASK, lmn, o), b = __shfl_xor_sync(FULL_MASK, lmx, o);
    lmn = a < lmn ? a : lmn;
    lmx = b > lmx ? b : lmx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lmn);
    atomicMax(&mm[1], lmx);
  }
}

// the size-key range (so the order sort only passes over the bits that
// vary); left in mm[0..1] on the device for the caller's next readback
int placement_rank_keys(mp_ctx *ctx, int64_t V, const int64_t *size, unsigned long long *mm, mp_err *err) {
  CUDA_TRY(cudaMemsetAsync(mm, 0xff, 8, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(mm + 1, 0, 8, ctx->stream));
  if (V) LAUNCH(ctx, k_size_range, grid_for(V, 256, 1024), 256, 0, V, size, mm);
  return MP_OK;
}

// rank[v] = position in (-size, tiekey or vertex) order, size keys in [kmin, kmax]
__global__ void k_size_keys32(int64_t V, const int64_t *size, uint64_t kmin, uint32_t *keys, uint32_t *vals) {
  PDL_WAIT();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    keys[v] = (uint32_t)(desc_size_key(size[v]) - kmin);
    if (vals) vals[v] = (uint32_t)v;
  }
}

int placement_rank_sort(mp_ctx *ctx, int64_t V, const int64_t *size, const int64_t *tiekey, int32_t *rank,
                        uint64_t kmin, uint64_t kmax, mp_err *err) {
  StageTimer tm(ctx, MP_ST_PLACE_ORDER);
  cudaStream_t st = ctx->stream;
  if (!tiekey && kmax - kmin <= 0xffffffffull) {
    // vertex-order ties and a size range that fits 32 bits: one stable sort
    // of 32-bit keys (a third less traffic per pass than the 64-bit path)
    DBuf<uint32_t> k32, order;
    CUDA_TRY(k32.alloc(V, st));
    if (V >= dev_radix_rank_min_n() && bits_for(kmax - kmin) > 0) {
      // the sort's last pass writes the ranks itself
      LAUNCH(ctx, k_size_keys32, grid_for(V, 256), 256, 0, V, size, kmin, k32.p, (uint32_t *)nullptr);
      return dev_radix_rank_u32(ctx, k32.p, V, bits_for(kmax - kmin), rank, err);
    }
    CUDA_TRY(order.alloc(V, st));
    LAUNCH(ctx, k_size_keys32, grid_for(V, 256), 256, 0, V, size, kmin, k32.p, order.p);
    int rc = dev_radix_sort_u32(ctx, k32.p, order.p, V, bits_for(kmax - kmin), err);
    if (rc) return rc;
    LAUNCH(ctx, k_rank, grid_for(V, 256), 256, 0, V, order.p, rank);
    return MP_OK;
  }
  DBuf<uint64_t> keys;
  DBuf<uint32_t> order;
  CUDA_TRY(keys.alloc(V, st));
  CUDA_TRY(order.alloc(V, st));
  int rc;
  if (tiekey) {
    LAUNCH(ctx, k_tie_keys, grid_for(V, 256), 256, 0, V, tiekey, keys.p, order.p);
    rc = dev_radix_sort_u64(ctx, keys.p, order.p, V, 64, err);
    if (rc) return rc;
  } else {
    LAUNCH(ctx, k_iota, grid_for(V, 256), 256, 0, V, order.p);
  }
  unsigned long long *d_mn = (unsigned long long *)ctx->d_small + 12;
  CUDA_TRY(cudaMemcpyAsync(d_mn, &kmin, 8, cudaMemcpyHostToDevice, st));
  LAUNCH(ctx, k_size_keys, grid_for(V, 256, 1024), 256, 0, V, size, order.p, keys.p, d_mn + 1, d_mn + 2);
  LAUNCH(ctx, k_sub_keys, grid_for(V, 256), 256, 0, V, keys.p, d_mn);
  rc = dev_radix_sort_u64(ctx, keys.p, order.p, V, bits_for(kmax - kmin), err);
  if (rc) return rc;
  LAUNCH(ctx, k_rank, grid_for(V, 256), 256, 0, V, order.p, rank);
  return MP_OK;
}

int placement_rank(mp_ctx *ctx, int64_t V, const int64_t *size, const int64_t *tiekey, int32_t *rank, mp_err *err) {
  unsigned long long *mm = (unsigned long long *)ctx->d_small + 10;
  int rc = placement_rank_keys(ctx, V, size, mm, err);
  if (rc) return rc;
  uint64_t h[2];
  rc = dev_read_n(ctx, mm, h, 16, err);
  if (rc) return rc;
  return placement_rank_sort(ctx, V, size, tiekey, rank, h[0], h[1], err);
}

int placement_rank_legacy(mp_ctx *ctx, int64_t V, const int64_t *size, const int64_t *tiekey, int32_t *rank,
                          mp_err *err) {
  StageTimer tm(ctx, MP_ST_PLACE_ORDER);
  cudaStream_t st = ctx->stream;
  DBuf<uint64_t> keys;
  DBuf<uint32_t> order;
  CUDA_TRY(keys.alloc(V, st));
  CUDA_TRY(order.alloc(V, st));
  int rc;
  if (tiekey) {
    LAUNCH(ctx, k_tie_keys, grid_for(V, 256), 256, 0, V, tiekey, keys.p, order.p);
    rc = dev_radix_sort_u64(ctx, keys.p, order.p, V, 64, err);
    if (rc) return rc;
  } else {
    LAUNCH(ctx, k_iota, grid_for(V, 256), 256, 0, V, order.p);
  }
  unsigned long long *d_mn = (unsigned long long *)ctx->d_small, *d_mx = d_mn + 1;
  CUDA_TRY(cudaMemsetAsync(d_mn, 0xff, 8, st));
  CUDA_TRY(cudaMemsetAsync(d_mx, 0, 8, st));
  LAUNCH(ctx, k_size_keys, grid_for(V, 256, 1024), 256, 0, V, size, order.p, keys.p, d_mn, d_mx);
  uint64_t mm[2];
  rc = dev_read_n(ctx, d_mn, mm, 16, err);
  if (rc) return rc;
  LAUNCH(ctx, k_sub_keys, grid_for(V, 256), 256, 0, V, keys.p, d_mn);
  rc = dev_radix_sort_u64(ctx, keys.p, order.p, V, bits_for(mm[1] - mm[0]), err);
  if (rc) return rc;
  LAUNCH(ctx, k_rank, grid_for(V, 256), 256, 0, V, order.p, rank);
  return MP_OK;
}

extern "C" int mp_plan_pool(mp_ctx *ctx, mp_dgraph *g, int32_t policy, int64_t *offsets, int64_t *footprint,
                            int64_t *levels, mp_err *err) {
  CTX_GUARD(ctx);
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
  DBuf<int32_t> remaining, queue, level, ctr;
  CUDA_TRY(remaining.alloc(V, st)); CUDA_TRY(queue.alloc(V, st)); CUDA_TRY(level.alloc(V, st));
  CUDA_TRY(ctr.alloc(16, st));
  // ctr: [0] head [1] tail [2] done [3] depth [4..5] footprint [6..7] arena need [8..9] arena top
  long long *d_fp = (long long *)(ctr.p + 4);
  unsigned long long *d_need = (unsigned long long *)(ctr.p + 6);
  // the conflict build bounded the long-row scratch by degree (no readback)
  uint64_t arena_need = (uint64_t)g->arena_need;
  static int per_sm_cached[4] = {0, 0, 0, 0};
  DBuf<int64_t> &off = g->offsets;
  CUDA_TRY(off.alloc(V, st));
  // sentinels: -1 offsets, level 0 or -1 (see pred_range)
  DBuf<longlong2> rec;
  const bool use_rec = PLACE_REC && g->size_lo >= 0 && g->size_hi <= (int64_t)0xffffffffll;
  if (use_rec) CUDA_TRY(rec.alloc(V, st));  // sentinels written by k_ready_init
  size_t smem = 0;
  // the 32-bit hole scan pays off only when the pool fits 2^31 bytes: the
  // narrow kernel when the traced peak (a lower bound of the footprint) does
  const bool narrow = PLACE_HOLE32 && g->peak_hint >= 0 && g->peak_hint < (int64_t)INT32_MAX;
  void (*kern)(PlaceArgs) = use_rec ? (narrow ? k_place_async<true, true> : k_place_async<true, false>)
                                    : (narrow ? k_place_async<false, true> : k_place_async<false, false>);
  int &cached = per_sm_cached[2 * use_rec + narrow];
  if (!cached) CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached, kern, PLACE_THREADS, smem));
  int per_sm = cached < 1 ? 1 : cached;
  if (const char *e = getenv("MP_PLACE_BLOCKS_PER_SM")) per_sm = atoi(e) < per_sm ? atoi(e) : per_sm;  // experiments
  // all warps resident: spinning consumers must never starve producers
  int64_t warps_needed = V;
  int64_t nblocks = (int64_t)per_sm * ctx->num_sms;
  int64_t need_blocks = (warps_needed * 32 + PLACE_THREADS - 1) / PLACE_THREADS;
  if (need_blocks < nblocks) nblocks = need_blocks;
  // scratch for rows the register sorts do not take: 128 ranges per warp,
  // plus a bump arena sized for every row longer than 128
  DBuf<IV> wscratch, arena;
  CUDA_TRY(wscratch.alloc(128 * nblocks * (PLACE_THREADS / 32), st));
  CUDA_TRY(arena.alloc((int64_t)arena_need, st));
  PlaceArgs a{V, g->row_off.p, g->col.p, g->pcnt.p, g->size.p, off.p, level.p, remaining.p, queue.p,
              ctr.p, ctr.p + 1, ctr.p + 2, policy, wscratch.p, arena.p, (unsigned long long *)(ctr.p + 8), d_fp, ctr.p + 3,
              0, nullptr, use_rec ? rec.p : nullptr};
  const char *trace_path = PLACE_TRACE ? getenv("MP_PLACE_TRACE") : nullptr;
  DBuf<unsigned long long> tdone;
  if (trace_path) {
    CUDA_TRY(tdone.alloc(5 * V, st));
    CUDA_TRY(cudaMemsetAsync(tdone.p, 0, 5 * V * 8, st));
    a.tdone = tdone.p;
  }
  {
    {
      StageTimer tm(ctx, MP_ST_PLACE_SPLIT);
      CUDA_TRY(cudaMemsetAsync(queue.p, 0, V * 4, st));
      CUDA_TRY(cudaMemsetAsync(ctr.p, 0, 64, st));
      LAUNCH(ctx, k_ready_init, grid_for(V, 256, 2048), 256, 0, V, g->pcnt.p, remaining.p, queue.p, ctr.p + 1,
             d_need, use_rec ? rec.p : (longlong2 *)nullptr, off.p, level.p, d_fp);
    }
    StageTimer ptm(ctx, MP_ST_PLACE);
    LAUNCH(ctx, kern, (unsigned)nblocks, PLACE_THREADS, smem, a);
  }
  if (offsets) CUDA_TRY(cudaMemcpyAsync(offsets, off.p, V * 8, cudaMemcpyDeviceToHost, st));
  if (trace_path) {
    // debug dump: V, level[V] (int32), predecessor count[V] (int32), time
    // placed[V], time claimed[V], time made ready[V] (ns, 0 = no predecessors)
    std::vector<int32_t> hl(2 * V);
    std::vector<unsigned long long> ht(5 * V);
    CUDA_TRY(cudaMemcpyAsync(hl.data(), level.p, V * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(hl.data() + V, g->pcnt.p, V * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(ht.data(), tdone.p, 5 * V * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (FILE *f = fopen(trace_path, "wb")) {
      fwrite(&V, 8, 1, f);
      fwrite(hl.data(), 4, 2 * V, f);
      fwrite(ht.data(), 8, 5 * V, f);
      fclose(f);
    }
  }
  int32_t tail4[6];
  int rc = dev_read_n(ctx, ctr.p, tail4, 24, err);
  if (rc) return rc;
  *footprint = *(int64_t *)(tail4 + 4);
  if (levels) *levels = tail4[3];
  return MP_OK;
}

extern "C" const int64_t *mp_graph_offsets_device(mp_dgraph *g) { return g->offsets.p; }
