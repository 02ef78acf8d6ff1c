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

/* Reserve the pool on `device` (cudaMalloc of pool_size bytes). */
int stw_alloc_init(int device, int64_t pool_size, int64_t alignment);

/* Load the plan: decisions (any order) with the phase index of their event,
 * size, planned offset, t_s and id (queue order = (t_s, id), sim.py:156-162),
 * and the reuse spaces per dynamic key (key k: sp_lo/sp_hi[sp_off[k]..sp_off[k+1])). */
int stw_alloc_load_plan(int64_t n_dec, const int32_t *phase, const int64_t *size, const int64_t *addr,
                        const int32_t *t_s, const int64_t *id, int64_t n_keys, const int64_t *sp_off,
                        const int64_t *sp_lo, const int64_t *sp_hi);

/* Request-matcher hooks: the phase the next requests belong to, and whether
 * they are dynamic (with their reuse key index; -1 = no reuse entry). */
void stw_set_phase(int32_t phase);
void stw_set_layer(int32_t key, int32_t dynamic);

/* CUDAPluggableAllocator entry points */
void *stw_malloc(size_t size, int device, void *stream);
void stw_free(void *ptr, size_t size, int device, void *stream);

/* Virtual address of a live block (pool offset, or cache virtual address >=
 * pool_size), -1 if unknown; route of its allocation (0 planned, 1 reuse,
 * 2 fallback, 3 mismatch). */
int64_t stw_alloc_vaddr(const void *ptr, int32_t *route);

/* Replay metrics of everything served so far (sim.py:67-117). */
int stw_alloc_report(stw_report *rep);

/* Release every device allocation and forget the plan. */
void stw_alloc_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif
