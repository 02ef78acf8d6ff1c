// Device-wide primitives: exclusive/inclusive scan and stable LSD radix sort.
#pragma once
#include "common.cuh"

namespace stw {

// ---------------------------------------------------------------------------
// scan: single pass with decoupled look-back, 2048 elements per block (256 threads x 8)

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

struct Arena;
template <class T>
void device_scan(Ctx &ctx, Arena &ar, const T *in, T *out, int64_t n, bool inclusive);

// ---------------------------------------------------------------------------
// radix sort

// K2's records per sort: the decoupled look-back packs each digit's running
// count into 30 bits (flag bits above), so every sort checks n <= kSortMax.
constexpr int64_t kSortMax = ((int64_t)1 << 30) - 1;


void radix_sort_pairs(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *vals, int64_t n, int begin_bit,
                      int end_bit);

// Convenience: sort (key, value) where value starts as the identity
// permutation; returns the permutation in `perm` and sorted keys in `keys`.
void sort_perm(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *perm, int64_t n, int bits);

__global__ void k_iota(uint32_t *p, int64_t n);

}  // namespace stw
