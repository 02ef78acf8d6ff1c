// Host runtime pieces shared by every entry point: error context, scratch
// arena, device-wide scan and the stable LSD radix sort (K2).
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "prims.cuh"

namespace stw {

// ---------------------------------------------------------------------------
// launch counter + opt-in per-kernel event profiler

static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_prof_on{false};
static std::mutex g_prof_mu;
struct Pending {
  const char *name;
  cudaEvent_t a, b;
};
static std::vector<Pending> g_pending;
static std::vector<cudaEvent_t> g_free_events;
struct Agg {
  long long count = 0;
  double ms = 0;
};
static std::map<std::string, Agg> g_agg;

static cudaEvent_t get_event() {
  if (!g_free_events.empty()) {
    cudaEvent_t e = g_free_events.back();
    g_free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

int prof_pre(cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on.load(std::memory_order_relaxed)) return -1;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  Pending p{nullptr, get_event(), get_event()};
  cudaEventRecord(p.a, s);
  g_pending.push_back(p);
  return (int)g_pending.size() - 1;
}

void prof_post(cudaStream_t s, const char *name, int slot) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_pending[slot].name = name;
  cudaEventRecord(g_pending[slot].b, s);
}

// Correctly rounded a / b (Python int true division) on the host.
double exact_div_host(unsigned long long a, unsigned long long b) {
  if (a == 0 || b == 0) return 0.0;
  if (a < (1ull << 53) && b < (1ull << 53)) return (double)a / (double)b;
  unsigned long long q = a / b, r = a % b;
  int nq = q ? 64 - __builtin_clzll(q) : 0;
  unsigned long long mant;
  int ex;
  bool sticky;
  if (nq >= 54) {
    int sh = nq - 54;
    mant = q >> sh;
    sticky = (sh > 0 && (q & ((1ull << sh) - 1))) || r;
    ex = sh;
  } else {
    int have = nq;
    mant = q;
    ex = 0;
    while (have < 54) {
      bool carry = (r >> 63) != 0;
      r <<= 1;
      unsigned long long bit = 0;
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
  return ldexp((double)mant, ex);
}

void Ctx::fail(int code, const char *fmt, ...) {
  if (rc != STW_OK) return;  // keep the first failure
  rc = code;
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
}

static void raise_pool_threshold() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

// Scratch is bump-allocated (256 B aligned) from stream-ordered chunks of at
// least 32 MiB, so a planner call costs a handful of cudaMallocAsync calls
// instead of one per buffer.
void *Arena::raw(size_t bytes) {
  if (!ctx->ok()) return nullptr;
  const size_t need = ((bytes ? bytes : 16) + 255) & ~(size_t)255;
  if (need > left) {
    if (n == (int)(sizeof(ptrs) / sizeof(ptrs[0]))) {
      ctx->fail(STW_ECUDA, "scratch arena: too many chunks");
      return nullptr;
    }
    raise_pool_threshold();
    const size_t chunk = need > (32u << 20) ? need : (32u << 20);
    void *p = nullptr;
    STW_CUDA(*ctx, cudaMallocAsync(&p, chunk, ctx->stream));
    if (!ctx->ok()) return nullptr;
    ptrs[n++] = p;
    cur = (char *)p;
    left = chunk;
  }
  void *out = cur;
  cur += need;
  left -= need;
  return out;
}

void Arena::release() {
  for (int i = 0; i < n; i++) cudaFreeAsync(ptrs[i], ctx->stream);
  n = 0;
  cur = nullptr;
  left = 0;
}

template <class T>
void device_scan(Ctx &ctx, Arena &ar, const T *in, T *out, int64_t n, bool inclusive) {
  if (n <= 0 || !ctx.ok()) return;
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb == 1) {
    STW_KL(k_tile_scan<T>, 1, kScanThreads, ctx.stream, in, out, nullptr, n, inclusive);
    STW_LAUNCHED(ctx);
    return;
  }
  T *sums = ar.take<T>(nb);
  if (!sums) return;
  STW_KL(k_tile_reduce<T>, (unsigned)nb, kScanThreads, ctx.stream, in, sums, n);
  STW_LAUNCHED(ctx);
  device_scan<T>(ctx, ar, sums, sums, nb, false);
  STW_KL(k_tile_scan<T>, (unsigned)nb, kScanThreads, ctx.stream, in, out, sums, n, inclusive);
  STW_LAUNCHED(ctx);
}
template void device_scan<uint32_t>(Ctx &, Arena &, const uint32_t *, uint32_t *, int64_t, bool);
template void device_scan<int64_t>(Ctx &, Arena &, const int64_t *, int64_t *, int64_t, bool);
template void device_scan<uint64_t>(Ctx &, Arena &, const uint64_t *, uint64_t *, int64_t, bool);
template void device_scan<int32_t>(Ctx &, Arena &, const int32_t *, int32_t *, int64_t, bool);

// ---------------------------------------------------------------------------
// K2: LSD radix sort, 8-bit digits.
// Pass = upsweep (per-tile digit histogram, digit-major) -> exclusive scan ->
// downsweep (stable rank inside the tile via warp match_any, scatter).

__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint64_t *__restrict__ keys,
                                                             uint32_t *__restrict__ counts, int64_t n,
                                                             int shift, uint32_t mask, int ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int j = 0; j < kSortItems; j++) {
    int64_t i = base + j * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(uint32_t)(keys[i] >> shift) & mask], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, const uint32_t *__restrict__ offs, int64_t n, int shift, uint32_t mask,
    int ntiles) {
  constexpr int W = kSortThreads / 32;
  __shared__ uint32_t base[256];
  __shared__ uint32_t wc[W][256];
  const int tid = threadIdx.x, warp = tid >> 5;
  base[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
  int64_t tile0 = (int64_t)blockIdx.x * kSortTile;
  for (int j = 0; j < kSortItems; j++) {
#pragma unroll
    for (int w = 0; w < W; w++) wc[w][tid] = 0;
    __syncthreads();
    int64_t i = tile0 + j * kSortThreads + tid;
    bool valid = i < n;
    uint64_t k = valid ? kin[i] : 0;
    uint32_t v = valid ? vin[i] : 0;
    uint32_t d = (uint32_t)(k >> shift) & mask;
    unsigned vm = __ballot_sync(0xffffffffu, valid);
    unsigned peers = 0, rank = 0;
    if (valid) {
      peers = __match_any_sync(vm, d);
      rank = __popc(peers & lanemask_lt());
      if (rank == 0) wc[warp][d] = __popc(peers);
    }
    __syncthreads();
    {  // exclusive prefix over warps for digit tid
      uint32_t s = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        uint32_t c = wc[w][tid];
        wc[w][tid] = s;
        s += c;
      }
      __syncthreads();
      if (valid) {
        uint32_t pos = base[d] + wc[warp][d] + rank;
        kout[pos] = k;
        vout[pos] = v;
      }
      __syncthreads();
      base[tid] += s;
    }
    __syncthreads();
  }
}

void radix_sort_pairs(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *vals, int64_t n, int begin_bit,
                      int end_bit) {
  if (n <= 1 || end_bit <= begin_bit || !ctx.ok()) return;
  int ntiles = (int)((n + kSortTile - 1) / kSortTile);
  uint64_t *k2 = ar.take<uint64_t>(n);
  uint32_t *v2 = ar.take<uint32_t>(n);
  uint32_t *counts = ar.take<uint32_t>((size_t)256 * ntiles);
  if (!ctx.ok()) return;
  uint64_t *ka = keys, *kb = k2;
  uint32_t *va = vals, *vb = v2;
  int passes = 0;
  for (int b = begin_bit; b < end_bit; b += 8) {
    int w = end_bit - b < 8 ? end_bit - b : 8;
    uint32_t mask = (1u << w) - 1;
    STW_KL(k_radix_hist, ntiles, kSortThreads, ctx.stream, ka, counts, n, b, mask, ntiles);
    STW_LAUNCHED(ctx);
    device_scan<uint32_t>(ctx, ar, counts, counts, (int64_t)256 * ntiles, false);
    STW_KL(k_radix_scatter, ntiles, kSortThreads, ctx.stream, ka, va, kb, vb, counts, n, b, mask, ntiles);
    STW_LAUNCHED(ctx);
    uint64_t *tk = ka;
    ka = kb;
    kb = tk;
    uint32_t *tv = va;
    va = vb;
    vb = tv;
    passes++;
  }
  if (passes & 1) {
    STW_CUDA(ctx, cudaMemcpyAsync(keys, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx.stream));
    STW_CUDA(ctx, cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx.stream));
  }
}

__global__ void k_iota(uint32_t *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

void sort_perm(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *perm, int64_t n, int bits) {
  if (!ctx.ok()) return;
  STW_KL(k_iota, grid_for(n, 256), 256, ctx.stream, perm, n);
  STW_LAUNCHED(ctx);
  radix_sort_pairs(ctx, ar, keys, perm, n, 0, bits);
}

}  // namespace stw

extern "C" {

long long stw_launch_count(void) { return stw::g_launches.load(); }

void stw_prof_enable(int on) { stw::g_prof_on.store(on != 0); }

// Drain recorded launches into per-kernel aggregates; then copy up to cap
// entries (name NUL-padded into 64-byte slots, launch count, summed ms).
int stw_prof_collect(char *names, long long *counts, double *ms, int cap, int reset) {
  using namespace stw;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto &p : g_pending) {
    cudaEventSynchronize(p.b);
    float t = 0;
    cudaEventElapsedTime(&t, p.a, p.b);
    Agg &a = g_agg[p.name ? p.name : "?"];
    a.count++;
    a.ms += t;
    g_free_events.push_back(p.a);
    g_free_events.push_back(p.b);
  }
  g_pending.clear();
  int n = 0;
  for (auto &kv : g_agg) {
    if (n < cap) {
      strncpy(names + 64 * n, kv.first.c_str(), 63);
      names[64 * n + 63] = 0;
      counts[n] = kv.second.count;
      ms[n] = kv.second.ms;
    }
    n++;
  }
  if (reset) g_agg.clear();
  return n;
}

}  // extern "C"
