/*
 * libstw_alloc -- runtime allocator that serves a plan.
 *
 * Loadable by torch.cuda.memory.CUDAPluggableAllocator(path, "stw_malloc",
 * "stw_free"); the two entry points match torch's
 * std::function<void*(size_t, int, cudaStream_t)> and
 * std::function<void(void*, size_t, int, cudaStream_t)>.
 *
 * Semantics are the reference replay's routing (sim.py:143-232): one reserved
 * pool of pool_size bytes; a static request is matched to the next planned
 * decision of key (current phase, size) and lands at its planned offset; a
 * dynamic request (stw_set_layer(key, 1)) gets the best fit inside its key's
 * reusable space intersected with the pool's free space; everything else goes
 * to a fallback region with the CachingAllocator policy (baseline.py:35-95:
 * best fit over all cached blocks, power-of-two segments >= 2 MiB, split /
 * merge), whose virtual addresses start at pool_size like the replay's.
 * Thread-safe (one mutex); the stream argument does not affect placement.
 */
#ifndef STW_ALLOC_H
#define STW_ALLOC_H
#include <stddef.h>
#include <stdint.h>

#include "stw.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Reserve ONE virtual range on `device`: the pool [0, pool_size) backed at
 * once, then fallback_va bytes (0 = 256 GiB) where the fallback segments are
 * mapped on first use. Device pointer = range base + the replay's address
 * (pool offset, or cache address >= pool_size). STW_EARG if already
 * initialised. */
int stw_alloc_init(int device, int64_t pool_size, int64_t alignment);
int stw_alloc_init_ex(int device, int64_t pool_size, int64_t alignment, int64_t fallback_va);

/* Load (or reload) the plan: decisions (any order) with the phase index of
 * their event, size, planned offset, t_s and id (queue order = (t_s, id),
 * sim.py:156-162), and the reuse spaces per dynamic key (key k:
 * sp_lo/sp_hi[sp_off[k]..sp_off[k+1])). Live allocations are kept; STW_EPLAN
 * if a decision or space leaves the reserved pool. */
int stw_alloc_load_plan(int64_t n_dec, const int32_t *phase, const int64_t *size, const int64_t *addr,
                        const int32_t *t_s, const int64_t *id, int64_t n_keys, const int64_t *sp_off,
                        const int64_t *sp_lo, const int64_t *sp_hi);

/* Request-matcher hooks: the phase the next requests belong to, and whether
 * they are dynamic (with their reuse key index; -1 = no reuse entry). */
void stw_set_phase(int32_t phase);
void stw_set_layer(int32_t key, int32_t dynamic);

/* CUDAPluggableAllocator entry points. stw_malloc commits nothing (queue
 * position, counters) unless the memory is there: on failure it returns NULL
 * with the state unchanged. Unknown or double frees are counted (the replay
 * raises SimulationError for them, sim.py:231-232) and make stw_alloc_report
 * return STW_ESIM. */
void *stw_malloc(size_t size, int device, void *stream);
void stw_free(void *ptr, size_t size, int device, void *stream);

/* Replay address of a live block (pool offset, or cache address >=
 * pool_size), -1 if unknown; route of its allocation (0 planned, 1 reuse,
 * 2 fallback, 3 mismatch). */
int64_t stw_alloc_vaddr(const void *ptr, int32_t *route);

/* Replay metrics of everything served so far (sim.py:67-117); STW_ESIM if a
 * planned address was found occupied or an unknown pointer was freed. */
int stw_alloc_report(stw_report *rep);

/* out[7] = {initialised, pool_size, live blocks, occupied-planned count,
 * bad frees, mapped bytes of the range, range base}. */
int stw_alloc_status(int64_t *out);

/* Unmap and release the range and forget the plan; STW_EARG (nothing done)
 * while any block is live. */
int stw_alloc_shutdown(void);

/* ---- Allocation Profiler (paper §4) + request matcher ---
 * Modes: 0 passthrough (plain cudaMalloc / cudaFree; the default before a
 * plan is loaded), 1 profiling (passthrough, and every malloc / free issued
 * while profiling is recorded with the current phase / module / dynamic tags,
 * in call order -- the raw trace of traceio.py:6-11; frees of blocks allocated
 * before profiling began are not recorded), 2 serving the plan (the mode
 * stw_alloc_init enters). Blocks allocated in passthrough keep being freed
 * through cudaFree in any mode. */
int stw_alloc_set_mode(int32_t mode);
/* tags of the next requests while profiling: phase / module are the caller's
 * interned indices */
void stw_prof_set(int32_t phase, int32_t module, int32_t dynamic);
/* the recording so far (op 0 alloc / 1 free, dynamic, phase, module, id,
 * bytes); returns the record count (only cap are written) */
int64_t stw_prof_records(int8_t *op, int8_t *dyn, int32_t *phase, int32_t *module, int64_t *id, int64_t *size,
                         int64_t cap);
/* (route, replay address) of every request served since stw_alloc_init, in
 * call order; returns the count (only cap are written) */
int64_t stw_alloc_served(int8_t *route, int64_t *vaddr, int64_t cap);
/* dynamic requests matched by layer instance: instance l's dynamic
 * allocations take reuse keys keys[off[l] .. off[l+1]) in order (-1 = none);
 * stw_set_layer_instance names the instance the next requests come from */
int stw_alloc_load_dyn_keys(int32_t n_layers, const int64_t *off, const int32_t *keys);
void stw_set_layer_instance(int32_t layer, int32_t dynamic);

/* ---- the same policies as standalone host objects ----------------------
 * CachingAllocator (baseline.py:35-95) over virtual addresses starting at
 * `base`: malloc returns STW_ESIM if rid is live, free STW_ESIM if unknown. */
void *stw_cache_new(int64_t base, int64_t min_segment);
void stw_cache_delete(void *cache);
int stw_cache_malloc(void *cache, int64_t rid, int64_t size, int64_t *addr, int64_t *grown);
int stw_cache_free(void *cache, int64_t rid, int64_t *addr, int64_t *size);
int stw_cache_owns(void *cache, int64_t rid);
/* out[5] = {reserved, live_bytes, segments, free blocks, next base} */
void stw_cache_stats(void *cache, int64_t *out);
/* segment g: base/size, free blocks blk_lo/blk_hi[blk_off[g] .. blk_off[g+1]) */
void stw_cache_segments(void *cache, int64_t *seg_base, int64_t *seg_size, int64_t *blk_off, int64_t *blk_lo,
                        int64_t *blk_hi);

/* dynamic_allocate's placement (sim.py:120-140): best fit of `size` in
 * free ∩ space (both sorted, coalesced); lowest address of the chosen piece,
 * -1 when nothing fits. */
int64_t stw_reuse_best_fit(int64_t n_free, const int64_t *free_lo, const int64_t *free_hi, int64_t n_space,
                           const int64_t *sp_lo, const int64_t *sp_hi, int64_t size);

#ifdef __cplusplus
}
#endif
#endif
