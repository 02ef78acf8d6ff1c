// Shared device/host helpers for libstw (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/stw.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libstw is written for sm_100a only"
#endif

namespace stw {

typedef unsigned __int128 u128;

constexpr int kWarp = 32;
constexpr int kSMs = 148;  // B200; kernels size grids as multiples of this

// ---------------------------------------------------------------------------
// error plumbing: every entry point runs inside a Ctx that records the first
// failure; CUDA errors map to STW_ECUDA.

struct Ctx {
  cudaStream_t stream;
  char *err;
  size_t errlen;
  int rc = STW_OK;
  void fail(int code, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
  bool ok() const { return rc == STW_OK; }
};

#define STW_CUDA(ctx, call)                                                        \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      (ctx).fail(STW_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                 cudaGetErrorString(_e));                                          \
    }                                                                              \
  } while (0)

#define STW_LAUNCHED(ctx) STW_CUDA(ctx, cudaGetLastError())

// libstw links its own (static) CUDA runtime: an entry point given a stream
// binds that runtime to the stream's device, so a caller on device k (one
// process per GPU, torch.cuda.set_device(k)) is served on device k. Without a
// stream the runtime uses the thread's current context, as any CUDA library.
inline void bind_stream_device(cudaStream_t s) {
  if (!s || s == cudaStreamLegacy || s == cudaStreamPerThread) return;
  int dev = -1, cur = -1;
  if (cudaStreamGetDevice(s, &dev) != cudaSuccess) {
    cudaGetLastError();  // (not a stream of this process: the launch reports it)
    return;
  }
  if (cudaGetDevice(&cur) == cudaSuccess && cur != dev) cudaSetDevice(dev);
}

// Every kernel launch goes through STW_KL: it counts launches and, when the
// opt-in profiler is on (stw_prof_enable), brackets the launch with CUDA
// events recorded on the launching stream.
int prof_pre(cudaStream_t s);
void prof_post(cudaStream_t s, const char *name, int slot);
#define STW_KL(kern, grid, block, stream, ...)               \
  do {                                                       \
    int _stw_slot = ::stw::prof_pre(stream);                 \
    kern<<<(grid), (block), 0, (stream)>>>(__VA_ARGS__);     \
    ::stw::prof_post(stream, #kern, _stw_slot);              \
  } while (0)

#define STW_KLS(kern, grid, block, smem, stream, ...)         \
  do {                                                       \
    int _stw_slot = ::stw::prof_pre(stream);                 \
    kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__); \
    ::stw::prof_post(stream, #kern, _stw_slot);              \
  } while (0)

// Stream-ordered scratch: every take() is a cudaMallocAsync on the call's
// stream (served from the device's default pool, whose release threshold is
// raised once so repeated calls do not remap); everything is returned with
// cudaFreeAsync when the Arena goes out of scope.
struct Arena {
  Ctx *ctx;
  void *ptrs[512];
  int n = 0;
  char *cur = nullptr;  // bump pointer inside the newest chunk
  size_t left = 0;
  explicit Arena(Ctx *c) : ctx(c) {}
  void *raw(size_t bytes);
  template <class T>
  T *take(size_t n_elems) {
    return reinterpret_cast<T *>(raw(n_elems * sizeof(T)));
  }
  void release();
  ~Arena() { release(); }
};

// Small host<->device transfers of the planner's round trips, kept off the
// copy engines: a copy engine works through its queue in order, so a few-byte
// pageable copy issued while stw_plan_batches streams the next batch in (or
// the previous results out) would wait behind megabytes. These go through a
// mapped page-locked scratch instead and are moved by copy kernels on the
// caller's stream (pending uploads: one launch right before the stream's next
// kernel; downloads: one launch at host_sync, where they land in `dst`).
// The scratch is reused after each host_sync (every kernel that read it ran).
void h2d_async(Ctx &ctx, void *ddst, const void *hsrc, size_t bytes);
void h2d_flush(Ctx &ctx);  // before another stream (or an event) must see the uploads
void d2h_async(Ctx &ctx, void *dst, const void *dsrc, size_t bytes);
void host_sync(Ctx &ctx);
// drop anything a failed earlier call left pending (start of a planner call)
void pinned_reset();

// NVTX ranges (header-only NVTX3; no-ops unless a profiler is attached): the
// call, then one range per phase, for nsys / ncu --nvtx filtering
struct NvtxPhases {
  bool open = false;
  explicit NvtxPhases(const char *call) { nvtxRangePushA(call); }
  void next(const char *phase) {
    if (open) nvtxRangePop();
    nvtxRangePushA(phase);
    open = true;
  }
  ~NvtxPhases() {
    if (open) nvtxRangePop();
    nvtxRangePop();
  }
};

// host-side size helpers

inline int bitlen_u64(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

inline unsigned grid_for(int64_t n, int block, int64_t cap = 148 * 64) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ int bitlen_dev(u128 x) {
  uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
  if (hi) return 128 - __clzll((long long)hi);
  if (lo) return 64 - __clzll((long long)lo);
  return 0;
}

// int -> double, round half even (Python float(int)), exact for < 2^53
__device__ __forceinline__ double u128_to_double_rne(u128 x) {
  int n = bitlen_dev(x);
  if (n <= 53) return (double)(uint64_t)x;
  int sh = n - 54;  // keep 54 bits: 53 + round bit
  uint64_t m = (uint64_t)(x >> sh);
  bool sticky = (x & (((u128)1 << sh) - 1)) != 0;
  bool rnd = m & 1;
  m >>= 1;
  if (rnd && (sticky || (m & 1))) m += 1;
  return scalbn((double)m, sh + 1);
}

// Correctly rounded a / b for positive integers (Python int true division).
static __device__ __noinline__ double exact_div(u128 a, u128 b) {
  const u128 two53 = (u128)1 << 53;
  if (a == 0) return 0.0;
  if (a < two53 && b < two53) return __ddiv_rn((double)(uint64_t)a, (double)(uint64_t)b);
  u128 q = a / b, r = a % b;
  uint64_t mant;
  int ex, nq = bitlen_dev(q);
  bool sticky;
  if (nq >= 54) {
    int sh = nq - 54;
    mant = (uint64_t)(q >> sh);
    sticky = (sh > 0 && (q & (((u128)1 << sh) - 1)) != 0) || r != 0;
    ex = sh;
  } else {
    int have = nq;
    mant = (uint64_t)q;
    ex = 0;
    while (have < 54) {
      bool carry = (r >> 127) != 0;
      r <<= 1;
      uint64_t bit = 0;
      if (carry || r >= b) {
        r -= b;
        bit = 1;
      }
      mant = (mant << 1) | bit;
      ex -= 1;
      if (have > 0 || bit) have++;
    }
    sticky = r != 0;
  }
  bool rnd = mant & 1;
  mant >>= 1;
  ex += 1;
  if (rnd && (sticky || (mant & 1))) mant += 1;
  return scalbn((double)mant, ex);
}

// 128-bit unsigned atomic add built from two 64-bit atomics (carry owned by
// the adder that overflowed the low word).
__device__ __forceinline__ void atomic_add_u128(unsigned long long *lohi, u128 v) {
  unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  unsigned long long old = atomicAdd(lohi, lo);
  if (old + lo < old) hi += 1;
  if (hi) atomicAdd(lohi + 1, hi);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
__device__ __forceinline__ T warp_incl_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

// Block exclusive sum; returns total via *total. `sh` needs >= 33 elements.
template <class T>
__device__ __forceinline__ T block_excl_sum(T v, T *sh, T *total) {
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T inc = warp_incl_sum(v);
  if (lane_id() == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = (int)lane_id() < nw ? sh[lane_id()] : T(0);
    T xi = warp_incl_sum(x);
    if ((int)lane_id() < nw) sh[lane_id()] = xi - x;
    if ((int)lane_id() == nw - 1) sh[32] = xi;
  }
  __syncthreads();
  T out = inc - v + sh[w];
  if (total) *total = sh[32];
  __syncthreads();
  return out;
}

}  // namespace stw
