// Device-wide primitives: exclusive/inclusive scan and stable LSD radix sort.
#pragma once
#include "common.cuh"

namespace stw {

// ---------------------------------------------------------------------------
// scan: reduce-then-scan, 2048 elements per block (256 threads x 8)

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__global__ void k_tile_reduce(const T *__restrict__ in, T *__restrict__ sums, int64_t n) {
  __shared__ T sh[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++)
    if (base + k < n) acc += in[base + k];
  T total;
  block_excl_sum<T>(acc, sh, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <class T>
__global__ void k_tile_scan(const T *__restrict__ in, T *__restrict__ out, const T *__restrict__ carry,
                            int64_t n, int inclusive) {
  __shared__ T sh[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    v[k] = base + k < n ? in[base + k] : T(0);
    acc += v[k];
  }
  T pre = block_excl_sum<T>(acc, sh, nullptr) + (carry ? carry[blockIdx.x] : T(0));
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    if (base + k < n) out[base + k] = inclusive ? pre + v[k] : pre;
    pre += v[k];
  }
}

struct Arena;
template <class T>
void device_scan(Ctx &ctx, Arena &ar, const T *in, T *out, int64_t n, bool inclusive);

// ---------------------------------------------------------------------------
// radix sort


void radix_sort_pairs(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *vals, int64_t n, int begin_bit,
                      int end_bit);

// Convenience: sort (key, value) where value starts as the identity
// permutation; returns the permutation in `perm` and sorted keys in `keys`.
void sort_perm(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *perm, int64_t n, int bits);

__global__ void k_iota(uint32_t *p, int64_t n);

}  // namespace stw
