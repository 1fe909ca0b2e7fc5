// alloc.cpp — PyTorch CUDAPluggableAllocator hooks serving a SmartPool plan.
//
// The paper's Device::Malloc/Free backed by the static
// pool: in RECORD mode every allocation is stream-ordered cudaMallocAsync
// and logged (op ordinal, kind, pointer, size rounded to 512 B) so one
// training iteration becomes a memplan trace; in SERVE mode the k-th
// allocation of an iteration gets pool_base + offset[k] from the plan's
// lookup table (smartpool.py:224-254) and frees are no-ops — a size mismatch
// falls back to cudaMallocAsync and is counted as a miss.
//
// Signatures follow torch.cuda.memory.CUDAPluggableAllocator:
//   void* alloc(ssize_t size, int device, cudaStream_t stream)
//   void  free(void* ptr, ssize_t size, int device, cudaStream_t stream)
#include <cuda_runtime.h>
#include <stdint.h>
#include <sys/types.h>

#include <time.h>

#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/memplan_alloc.h"

namespace {

constexpr int64_t ALIGN = 512;

struct LogRec {
  int64_t seq;
  int32_t kind;  // 0 malloc, 1 free
  int64_t ptr;
  int64_t size;
};

struct State {
  std::mutex mu;
  int mode = 0;  // 0 record/passthrough, 1 serve
  bool logging = false;
  int64_t seq = 0;  // op ordinal set by the tracer
  std::vector<LogRec> log;
  std::unordered_map<int64_t, int64_t> live;  // ptr -> size (passthrough allocations)
  // serve
  char *pool = nullptr;
  int64_t pool_bytes = 0;
  std::vector<int64_t> slot_off, slot_size;
  int64_t ordinal = 0, misses = 0, hits = 0, conflicts = 0;
  std::unordered_map<int64_t, int64_t> pool_live;  // offset -> size of served blocks
  std::unordered_map<int64_t, int64_t> pool_who;   // offset -> iteration * 2^20 + ordinal
  int64_t iteration = 0;
  std::vector<int64_t> clash_log;                  // (iteration, ordinal, other) triples
  int64_t cur_bytes = 0, peak_bytes = 0;  // passthrough bytes live
  // pools replaced by a later plan while blocks served from them were still
  // referenced (e.g. gradients freed by the next iteration's zero_grad):
  // each stays mapped until its last block is freed, so no later
  // allocation can reuse the address range under a live tensor
  struct Retired {
    int64_t base, bytes;
    std::unordered_map<int64_t, int64_t> live;  // offset -> size
  };
  std::vector<Retired> retired;
  // offsets of swapped-out blocks: PyTorch still holds their pointers, so
  // no other block may be served at the same address while they are out
  std::unordered_map<int64_t, int64_t> swapped_out;
  int64_t aliases = 0;
  // host-side cost of the hooks (entry to return, lock wait included)
  int64_t alloc_calls = 0, alloc_ns = 0, free_calls = 0, free_ns = 0;
};

State &S() {
  static State s;
  return s;
}

inline int64_t round_up(int64_t n) { return (n + ALIGN - 1) / ALIGN * ALIGN; }

inline int64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000 + ts.tv_nsec;
}

// adds the time since `start` (taken before the lock) to (calls, ns) when
// the enclosing hook returns
struct HookTimer {
  int64_t t0, &calls, &ns;
  HookTimer(int64_t &c, int64_t &n, int64_t start) : t0(start), calls(c), ns(n) {}
  ~HookTimer() {
    calls++;
    ns += now_ns() - t0;
  }
};

}  // namespace

extern "C" {

void *mp_torch_alloc(ssize_t size, int device, cudaStream_t stream) {
  State &s = S();
  const int64_t t0 = now_ns();
  std::lock_guard<std::mutex> g(s.mu);
  HookTimer tm(s.alloc_calls, s.alloc_ns, t0);
  int64_t rs = round_up(size > 0 ? size : 1);
  void *p = nullptr;
  if (s.mode == 1) {
    int64_t k = s.ordinal++;
    if (k < (int64_t)s.slot_off.size() && s.slot_size[k] == rs) {
      int64_t lo = s.slot_off[k], hi = lo + rs;
      // guard: the slot must not overlap a pool block that is still live
      // (a program whose lifetimes drift from the recorded ones)
      bool clash = s.swapped_out.count(lo) != 0;
      int64_t other = -1;
      if (clash) s.aliases++;
      if (!clash)
        for (auto &kv : s.pool_live)
        if (kv.first < hi && lo < kv.first + kv.second) { clash = true; other = s.pool_who[kv.first]; break; }
      if (clash) {
        s.conflicts++;
        if (s.clash_log.size() < 3 * 64) {
          s.clash_log.push_back(s.iteration);
          s.clash_log.push_back(k);
          s.clash_log.push_back(other);
        }
      } else {
        p = s.pool + lo;
        s.pool_live[lo] = rs;
        s.pool_who[lo] = (s.iteration << 20) | k;
        s.hits++;
      }
    } else {
      s.misses++;
    }
  }
  if (!p) {
    (void)device;
    if (cudaMallocAsync(&p, rs, stream) != cudaSuccess) return nullptr;
    s.live[(int64_t)p] = rs;
    s.cur_bytes += rs;
    if (s.cur_bytes > s.peak_bytes) s.peak_bytes = s.cur_bytes;
  }
  if (s.logging) s.log.push_back({s.seq, 0, (int64_t)p, rs});
  return p;
}

void mp_torch_free(void *ptr, ssize_t size, int device, cudaStream_t stream) {
  State &s = S();
  const int64_t t0 = now_ns();
  std::lock_guard<std::mutex> g(s.mu);
  HookTimer tm(s.free_calls, s.free_ns, t0);
  (void)size;
  (void)device;
  if (s.logging) s.log.push_back({s.seq, 1, (int64_t)ptr, 0});
  char *c = (char *)ptr;
  const int64_t a = (int64_t)c;
  // retired pools first: their ranges are still mapped, so no current
  // block can lie inside one
  for (size_t r = 0; r < s.retired.size(); r++) {
    auto &rp = s.retired[r];
    if (a >= rp.base && a < rp.base + rp.bytes) {
      rp.live.erase(a - rp.base);
      if (rp.live.empty()) {
        cudaFree((void *)rp.base);  // synchronizes: pending work on the block is done
        s.retired.erase(s.retired.begin() + r);
      }
      return;
    }
  }
  if (s.pool && c >= s.pool && c < s.pool + s.pool_bytes) {  // pool slots are static
    s.pool_live.erase(a - (int64_t)s.pool);
    s.swapped_out.erase(a - (int64_t)s.pool);
    return;
  }
  auto it = s.live.find(a);
  if (it != s.live.end()) {
    s.cur_bytes -= it->second;
    s.live.erase(it);
  }
  cudaFreeAsync(ptr, stream);
}

// ---- control (ctypes) ----
void mp_alloc_set_seq(int64_t seq) { S().seq = seq; }
void mp_alloc_logging(int on) {
  std::lock_guard<std::mutex> g(S().mu);
  S().logging = on != 0;
}
int64_t mp_alloc_log_size() { return (int64_t)S().log.size(); }
void mp_alloc_log_drain(int64_t *seq, int32_t *kind, int64_t *ptr, int64_t *size) {
  State &s = S();
  std::lock_guard<std::mutex> g(s.mu);
  for (size_t i = 0; i < s.log.size(); i++) {
    seq[i] = s.log[i].seq;
    kind[i] = s.log[i].kind;
    ptr[i] = s.log[i].ptr;
    size[i] = s.log[i].size;
  }
  s.log.clear();
}
// install a plan: n slots (offset, rounded size) in allocation order
int mp_alloc_set_plan(int64_t pool_bytes, int64_t n, const int64_t *off, const int64_t *size) {
  State &s = S();
  std::lock_guard<std::mutex> g(s.mu);
  if (s.pool) {
    // blocks PyTorch still holds (served or swapped out) keep the old pool
    // mapped; an unreferenced pool goes back to the driver now
    State::Retired rp{(int64_t)s.pool, s.pool_bytes, std::move(s.pool_live)};
    for (auto &kv : s.swapped_out) rp.live[kv.first] = kv.second;
    if (rp.live.empty()) cudaFree(s.pool);
    else s.retired.push_back(std::move(rp));
  }
  s.pool = nullptr;
  s.pool_bytes = pool_bytes;
  if (pool_bytes > 0 && cudaMalloc((void **)&s.pool, pool_bytes) != cudaSuccess) return 1;
  s.slot_off.assign(off, off + n);
  s.slot_size.assign(size, size + n);
  s.ordinal = 0;
  s.pool_live.clear();
  s.swapped_out.clear();
  return 0;
}
void mp_alloc_mode(int mode) {
  std::lock_guard<std::mutex> g(S().mu);
  S().mode = mode;
}
void mp_alloc_begin_iteration() {
  std::lock_guard<std::mutex> g(S().mu);
  S().ordinal = 0;
  S().iteration++;
}
int64_t mp_alloc_clash_log(int64_t *out, int64_t cap) {
  State &s = S();
  std::lock_guard<std::mutex> g(s.mu);
  int64_t n = (int64_t)s.clash_log.size();
  for (int64_t i = 0; i < n && i < cap; i++) out[i] = s.clash_log[i];
  return n;
}
void mp_alloc_stats(int64_t *out) {
  State &s = S();
  std::lock_guard<std::mutex> g(s.mu);
  out[6] = s.conflicts;
  out[0] = s.hits;
  out[1] = s.misses;
  out[2] = s.pool_bytes;
  out[3] = s.cur_bytes;
  out[4] = s.peak_bytes;
  out[5] = s.ordinal;
  out[7] = (int64_t)s.pool_live.size();
  out[8] = s.aliases;
  out[9] = (int64_t)s.retired.size();
}
// swap executor: a swapped-out block's bytes are free for the planned
// co-tenants until it is swapped back in
void mp_alloc_pool_release(int64_t off) {
  std::lock_guard<std::mutex> g(S().mu);
  auto it = S().pool_live.find(off);
  if (it != S().pool_live.end()) {
    S().swapped_out[off] = it->second;
    S().pool_live.erase(it);
  }
}
// returns 0, or 1 if a live block still overlaps [off, off+size)
int mp_alloc_pool_reclaim(int64_t off, int64_t size) {
  State &s = S();
  std::lock_guard<std::mutex> g(s.mu);
  for (auto &kv : s.pool_live)
    if (kv.first < off + size && off < kv.first + kv.second) {
      s.conflicts++;
      return 1;
    }
  s.swapped_out.erase(off);
  s.pool_live[off] = size;
  return 0;
}
void mp_alloc_call_stats(int64_t *out) {
  State &s = S();
  std::lock_guard<std::mutex> g(s.mu);
  out[0] = s.alloc_calls;
  out[1] = s.alloc_ns;
  out[2] = s.free_calls;
  out[3] = s.free_ns;
}
void mp_alloc_reset_peak() {
  std::lock_guard<std::mutex> g(S().mu);
  S().alloc_calls = S().alloc_ns = S().free_calls = S().free_ns = 0;
  S().peak_bytes = S().cur_bytes;
  S().hits = S().misses = S().conflicts = S().aliases = 0;
}
int64_t mp_alloc_pool_base() { return (int64_t)S().pool; }
int mp_alloc_peek_error() { return (int)cudaPeekAtLastError(); }
// swap executor copies: d2h=1 copies dev -> host, else host -> dev
int mp_alloc_copy_async(void *dev, void *host, int64_t n, int d2h, cudaStream_t stream) {
  cudaError_t e = d2h ? cudaMemcpyAsync(host, dev, n, cudaMemcpyDeviceToHost, stream)
                      : cudaMemcpyAsync(dev, host, n, cudaMemcpyHostToDevice, stream);
  return (int)e;
}

}  // extern "C"
