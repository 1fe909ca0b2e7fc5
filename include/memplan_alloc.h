/*
 * memplan_alloc.h — C ABI of the plan-serving allocator and the swap
 * executor's copy hooks (libmemplan_alloc.so, csrc/alloc.cpp).
 *
 * The reference package stops at the plan (LookupTable, smartpool.py:224-254;
 * SwapSchedule, swapsim.py:34-116); the paper's runtime serves it from its
 * Device::Malloc/Free.  Here that runtime is a PyTorch
 * CUDAPluggableAllocator: mp_torch_alloc / mp_torch_free have exactly the
 * signatures torch.cuda.memory.CUDAPluggableAllocator binds, and the control
 * calls below are what torchmem.py / swapexec.py drive through ctypes.
 *
 * State is process-wide (one allocator per process, as PyTorch installs it)
 * and every call takes one mutex, so the hooks may be called from any host
 * thread; mp_torch_alloc never synchronizes the device.
 */
#ifndef MEMPLAN_ALLOC_H
#define MEMPLAN_ALLOC_H

#include <stdint.h>
#include <sys/types.h>

#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- the PyTorch allocator hooks ------------------------------------- */

/* RECORD mode (0): stream-ordered cudaMallocAsync, logged when logging is
 * on.  SERVE mode (1): the k-th allocation of an iteration returns
 * pool_base + offset[k] when its 512-byte-rounded size equals the planned
 * slot and the slot overlaps no live pool block; anything else is a miss
 * (or a conflict) served by cudaMallocAsync. */
void *mp_torch_alloc(ssize_t size, int device, cudaStream_t stream);
/* pool blocks are static: a free only marks the slot dead.  Blocks of a
 * pool replaced by mp_alloc_set_plan keep it mapped until the last one is
 * freed. */
void mp_torch_free(void *ptr, ssize_t size, int device, cudaStream_t stream);

/* ---- control ----------------------------------------------------------- */

/* install a plan: n slots (offset, rounded size) in malloc order — the
 * window's LookupTable (smartpool.py:246-254) flattened by ordinal.  The
 * previous pool is released now if no block of it is referenced, else
 * retired.  Returns 0, or 1 if the pool allocation failed. */
int mp_alloc_set_plan(int64_t pool_bytes, int64_t n, const int64_t *off, const int64_t *size);
void mp_alloc_mode(int mode);             /* 0 record/passthrough, 1 serve */
void mp_alloc_begin_iteration(void);      /* malloc ordinal back to 0 */
int64_t mp_alloc_pool_base(void);
/* out[10]: hits, misses, pool_bytes, passthrough live bytes, passthrough
 * peak bytes, ordinal, conflicts, live pool blocks, swap alias fallbacks,
 * retired pools still mapped */
void mp_alloc_stats(int64_t *out);
/* out[4]: mp_torch_alloc calls, their total host ns, mp_torch_free calls,
 * their total host ns (entry to return, lock wait included); zeroed by
 * mp_alloc_reset_peak */
void mp_alloc_call_stats(int64_t *out);
void mp_alloc_reset_peak(void);
/* (iteration, ordinal, clashing block) triples of refused slots */
int64_t mp_alloc_clash_log(int64_t *out, int64_t cap);

/* ---- trace recording (torchmem.Tracer) --------------------------------- */

void mp_alloc_set_seq(int64_t seq);       /* op ordinal stamped on log records */
void mp_alloc_logging(int on);
int64_t mp_alloc_log_size(void);
/* move the log out: per record (op ordinal, kind 0 malloc / 1 free,
 * pointer, rounded size) */
void mp_alloc_log_drain(int64_t *seq, int32_t *kind, int64_t *ptr, int64_t *size);

/* ---- swap executor (swapexec.py) --------------------------------------- */

/* a swapped-out block's bytes become free for its planned co-tenants ... */
void mp_alloc_pool_release(int64_t off);
/* ... until it is swapped back in: 0, or 1 if a live block still overlaps */
int mp_alloc_pool_reclaim(int64_t off, int64_t size);
/* cudaMemcpyAsync on the executor's copy stream: d2h != 0 copies device ->
 * pinned host, else host -> device; returns the cudaError_t */
int mp_alloc_copy_async(void *dev, void *host, int64_t n, int d2h, cudaStream_t stream);
int mp_alloc_peek_error(void);

#ifdef __cplusplus
}
#endif

#endif /* MEMPLAN_ALLOC_H */
