// Host runtime pieces shared by every entry point: error context, scratch
// arena, device-wide scan and the stable LSD radix sort (K2).
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
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

void h2d_flush_stream(cudaStream_t s);

int prof_pre(cudaStream_t s) {
  h2d_flush_stream(s);  // uploads queued by h2d_async land before the kernel
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

// The arena draws from a private memory pool per device (not the device's
// default pool, which torch's cudaMallocAsync backend shares): its release
// threshold is raised so chunks stay mapped between calls, and
// stw_release_scratch() trims it back to the driver.
static std::mutex g_pool_mu;
static std::map<int, cudaMemPool_t> g_pools;

static cudaMemPool_t scratch_pool(Ctx &ctx) {
  int dev = 0;
  STW_CUDA(ctx, cudaGetDevice(&dev));
  if (!ctx.ok()) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_pools.find(dev);
  if (it != g_pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  STW_CUDA(ctx, cudaMemPoolCreate(&pool, &props));
  if (!ctx.ok()) return nullptr;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  g_pools[dev] = pool;
  return pool;
}

// Scratch is bump-allocated (256 B aligned) from stream-ordered chunks of at
// least 256 MiB, so a planner call costs a handful of cudaMallocAsync calls
// instead of one per buffer.
constexpr size_t kArenaChunk = (size_t)256 << 20;

void *Arena::raw(size_t bytes) {
  if (!ctx->ok()) return nullptr;
  const size_t need = ((bytes ? bytes : 16) + 255) & ~(size_t)255;
  if (need > left) {
    if (n == (int)(sizeof(ptrs) / sizeof(ptrs[0]))) {
      ctx->fail(STW_ECUDA, "scratch arena: too many chunks");
      return nullptr;
    }
    cudaMemPool_t pool = scratch_pool(*ctx);
    if (!pool) return nullptr;
    // large chunks: one planner call takes a few (each cudaMallocAsync is host
    // time the GPU may wait on); the pool keeps them cached between calls
    const size_t chunk = need > kArenaChunk ? need : kArenaChunk;
    void *p = nullptr;
    STW_CUDA(*ctx, cudaMallocFromPoolAsync(&p, chunk, pool, ctx->stream));
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

// Single-pass scan with decoupled look-back: tiles of kScanTile claimed in
// order by an atomic counter; each tile publishes its aggregate, then a warp
// looks back over up to 128 predecessors at a time for the nearest inclusive
// prefix; one launch and one read + one write of the data. The first
// kScanDirect tiles instead sum all their predecessors' aggregates at once.
//
// Look-back records are 16 bytes {token, value}, written and read as single
// 16-byte accesses (naturally aligned vector accesses are single-copy atomic
// on this hardware), so neither side needs a fence between flag and value.
// A record is valid iff its token equals the launch's token (unique per
// launch), so the record arrays need no clearing. Each tile has an aggregate
// record and an inclusive-prefix record (the direct path needs aggregates).
constexpr int64_t kScanDirect = 1024;
constexpr int kScanWin = 4;  // look-back entries per lane (window = 128 tiles)

struct __align__(16) ScanRec {
  unsigned long long tok, val;
};
__device__ __forceinline__ void scan_rec_put(ScanRec *p, unsigned long long tok, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(tok), "l"(v) : "memory");
}
__device__ __forceinline__ ScanRec scan_rec_get(const ScanRec *p) {
  ScanRec r;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.tok), "=l"(r.val) : "l"(p) : "memory");
  return r;
}
template <class T>
__device__ __forceinline__ unsigned long long scan_bits(T v) {
  return (unsigned long long)(long long)v;  // 32-bit types widen; only the low bits are read back
}

// Tile I/O is coalesced: 16-byte vector loads / stores over the tile (thread
// t moves vectors t, t + 256, ...), staged through shared memory (padded one
// element per 16 against bank conflicts), where each thread then scans its
// kScanItems consecutive elements in place (nothing held in registers across
// the look-back).
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_lb(const T *__restrict__ in, T *__restrict__ out, int64_t n,
                                                          int inclusive, ScanRec *__restrict__ agg,
                                                          ScanRec *__restrict__ pre, uint32_t *__restrict__ ctr,
                                                          unsigned long long tok) {
  constexpr int kVec = 16 / sizeof(T);          // elements per 16-byte vector
  constexpr int kVecs = kScanTile / kVec;       // vectors per tile
  constexpr int kPad = kScanTile + kScanTile / 16;
  __shared__ __align__(16) T st[kPad];
  __shared__ T sh[33];
  __shared__ uint32_t s_tile;
  __shared__ T s_excl;
  auto at = [](int i) { return i + (i >> 4); };  // padded position of tile element i
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t t0 = (int64_t)tile * kScanTile;
  const int cnt = (int)(n - t0 < kScanTile ? n - t0 : kScanTile);
  const bool vec_ok = cnt == kScanTile && (reinterpret_cast<uintptr_t>(in + t0) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(out + t0) & 15) == 0;
  if (vec_ok) {
    const uint4 *src = reinterpret_cast<const uint4 *>(in + t0);
    uint4 w[kVecs / kScanThreads];
#pragma unroll
    for (int j = 0; j < kVecs / kScanThreads; j++) w[j] = __ldcs(src + j * kScanThreads + tid);  // streamed once
#pragma unroll
    for (int j = 0; j < kVecs / kScanThreads; j++) {
      const int q = j * kScanThreads + tid;
      const T *e = reinterpret_cast<const T *>(&w[j]);
#pragma unroll
      for (int x = 0; x < kVec; x++) st[at(q * kVec + x)] = e[x];
    }
  } else {
    for (int i = tid; i < kScanTile; i += kScanThreads) st[at(i)] = i < cnt ? in[t0 + i] : T(0);
  }
  __syncthreads();
  T acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) acc += st[at(tid * kScanItems + k)];
  T total;
  const T ex = block_excl_sum<T>(acc, sh, &total);
  if (tid == 0) {
    scan_rec_put(agg + tile, tok, scan_bits(total));
    if (tile == 0) scan_rec_put(pre, tok, scan_bits(total));
  }
  if (tile > 0 && tile <= kScanDirect) {
    // few tiles: sum every predecessor's aggregate directly -- they are all
    // published at about the same time, so there is no prefix chain to wait on
    T part = 0;
    for (int64_t t = tid; t < (int64_t)tile; t += kScanThreads) {
      ScanRec r;
      do r = scan_rec_get(agg + t);
      while (r.tok != tok);
      part += (T)r.val;
    }
    T excl;
    block_excl_sum<T>(part, sh, &excl);
    if (tid == 0) {
      scan_rec_put(pre + tile, tok, scan_bits(excl + total));  // for the look-back of later tiles
      s_excl = excl;
    }
  } else if (tid < 32) {
    T excl = 0;
    if (tile > 0) {
      // window of 128 predecessors, entry d = j * 32 + lane at tile tw - d:
      // the nearest published inclusive prefix ends the walk, aggregates
      // between it and this tile are added; every entry must be published
      for (int64_t tw = (int64_t)tile - 1;; tw -= 32 * kScanWin) {
        T val[kScanWin];
        bool isp[kScanWin];
#pragma unroll
        for (int j = 0; j < kScanWin; j++) {
          const int64_t t = tw - j * 32 - lane;
          val[j] = 0;
          isp[j] = t < 0;  // before tile 0: acts as a zero prefix
          if (t >= 0) {
            const ScanRec p = scan_rec_get(pre + t);
            if (p.tok == tok) {
              isp[j] = true;
              val[j] = (T)p.val;
            } else {
              ScanRec a;
              do {
                a = scan_rec_get(agg + t);
              } while (a.tok != tok);
              // an inclusive prefix may have landed meanwhile; either is exact
              val[j] = (T)a.val;
            }
          }
        }
        int stop = 32 * kScanWin;  // first entry (by distance) holding a prefix
#pragma unroll
        for (int j = kScanWin - 1; j >= 0; j--) {
          const unsigned pm = __ballot_sync(0xffffffffu, isp[j]);
          if (pm) stop = j * 32 + __ffs(pm) - 1;
        }
        T part = 0;
#pragma unroll
        for (int j = 0; j < kScanWin; j++) part += j * 32 + lane <= stop ? val[j] : T(0);
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (stop < 32 * kScanWin) break;
      }
      if (lane == 0) scan_rec_put(pre + tile, tok, scan_bits(excl + total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  T run = ex + s_excl;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    T &x = st[at(tid * kScanItems + k)];
    const T v = x;
    x = inclusive ? run + v : run;
    run += v;
  }
  __syncthreads();
  if (vec_ok) {
    uint4 *dst = reinterpret_cast<uint4 *>(out + t0);
#pragma unroll
    for (int j = 0; j < kVecs / kScanThreads; j++) {
      const int q = j * kScanThreads + tid;
      uint4 w;
      T *e = reinterpret_cast<T *>(&w);
#pragma unroll
      for (int x = 0; x < kVec; x++) e[x] = st[at(q * kVec + x)];
      __stcs(dst + q, w);
    }
  } else {
    for (int i = tid; i < cnt; i += kScanThreads) out[t0 + i] = st[at(i)];
  }
}

static std::atomic<unsigned long long> g_scan_tok{0x5ca1ab1e00000000ull};

template <class T>
void device_scan(Ctx &ctx, Arena &ar, const T *in, T *out, int64_t n, bool inclusive) {
  if (n <= 0 || !ctx.ok()) return;
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  ScanRec *agg = ar.take<ScanRec>(nb), *pre = ar.take<ScanRec>(nb);
  uint32_t *ctr = ar.take<uint32_t>(1);
  if (!ctx.ok()) return;
  // a token no earlier launch used: stale records in recycled scratch never match it
  const unsigned long long tok = g_scan_tok.fetch_add(1, std::memory_order_relaxed) + 1;
  STW_CUDA(ctx, cudaMemsetAsync(ctr, 0, sizeof(uint32_t), ctx.stream));
  STW_KL(k_scan_lb<T>, (unsigned)nb, kScanThreads, ctx.stream, in, out, n, inclusive ? 1 : 0, agg, pre, ctr, tok);
  STW_LAUNCHED(ctx);
}
template void device_scan<uint32_t>(Ctx &, Arena &, const uint32_t *, uint32_t *, int64_t, bool);
template void device_scan<int64_t>(Ctx &, Arena &, const int64_t *, int64_t *, int64_t, bool);
template void device_scan<uint64_t>(Ctx &, Arena &, const uint64_t *, uint64_t *, int64_t, bool);
template void device_scan<int32_t>(Ctx &, Arena &, const int32_t *, int32_t *, int64_t, bool);

// ---------------------------------------------------------------------------
// K2: stable LSD radix sort, 8-bit digits, one kernel per pass ("onesweep":
// decoupled look-back instead of a separate upsweep/scan/downsweep).
//
//  k_os_hist  one read of the keys -> the digit histograms of every pass
//  k_os_bins  exclusive scan of each pass's 256 bins
//  k_os_pass  per 3840-key tile (tile ids handed out in launch order by an
//             atomic counter): warp-level stable ranking (8 ballots) into
//             per-warp digit counters, publish the tile's digit counts (the
//             sum of the warps' counters), look
//             back over earlier tiles' published counts/prefixes (one thread
//             per digit), stage the tile in shared memory in digit order and
//             write it out in digit runs (coalesced).
// Traffic per pass: 12 B read + 12 B written per (key, value) pair.

constexpr int kOsThreads = 256;  // one thread per digit in the look-back
constexpr int kOsItems = 15;
constexpr int kOsTile = kOsThreads * kOsItems;
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsAhead = 148 * 2;  // tiles ahead (measured: 2 per SM beats 3 and 6)
constexpr uint32_t kOsAgg = 1u << 30, kOsPrefix = 2u << 30, kOsVal = kOsAgg - 1;
constexpr size_t kOsSmem = (size_t)kOsTile * 12 + (size_t)kOsWarps * 256 * 4 + 256 * 4 + 256 * 8 + 256 * 4 + 16;

// One read of the keys -> the digit histograms of every pass (one shared
// histogram per CTA; 16-byte loads, four in flight per thread).
__global__ void __launch_bounds__(256) k_os_hist(const uint64_t *__restrict__ keys, int64_t n, int begin_bit,
                                                 int end_bit, int passes, uint32_t *__restrict__ hist) {
  __shared__ uint32_t h[8][256];
  for (int x = threadIdx.x; x < 8 * 256; x += blockDim.x) (&h[0][0])[x] = 0;
  __syncthreads();
  const int64_t n2 = n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
  const ulonglong2 *k2 = reinterpret_cast<const ulonglong2 *>(keys);
  const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
  auto count = [&](uint64_t k) {
    for (int p = 0; p < passes; p++) {
      const int b = begin_bit + 8 * p, w = min(8, end_bit - b);
      atomicAdd(&h[p][(uint32_t)(k >> b) & ((1u << w) - 1)], 1u);
    }
  };
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (vec) {
    for (; i + 3 * stride < n2; i += 4 * stride) {
      const ulonglong2 a = k2[i], b = k2[i + stride], c = k2[i + 2 * stride], d = k2[i + 3 * stride];
      count(a.x), count(a.y), count(b.x), count(b.y), count(c.x), count(c.y), count(d.x), count(d.y);
    }
    for (; i < n2; i += stride) {
      const ulonglong2 a = k2[i];
      count(a.x), count(a.y);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) count(keys[n - 1]);
  } else {
    for (; i < n; i += stride) count(keys[i]);
  }
  __syncthreads();
  for (int x = threadIdx.x; x < passes * 256; x += blockDim.x) {
    const uint32_t c = (&h[0][0])[x];
    if (c) atomicAdd(hist + x, c);
  }
}

__global__ void __launch_bounds__(256) k_os_bins(uint32_t *__restrict__ hist) {
  __shared__ uint32_t sh[33];
  uint32_t *hp = hist + blockIdx.x * 256;
  const uint32_t v = hp[threadIdx.x];
  hp[threadIdx.x] = block_excl_sum<uint32_t>(v, sh, nullptr);
}

template <int W>  // digit bits of this pass (8, or fewer for a key's last bits)
__global__ void __launch_bounds__(kOsThreads, 3) k_os_pass(const uint64_t *__restrict__ kin,
                                                        const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
                                                        uint32_t *__restrict__ vout, int64_t n, int shift,
                                                        uint32_t mask, const uint32_t *__restrict__ bins,
                                                        uint32_t *__restrict__ status, uint32_t *__restrict__ ctr,
                                                        uint32_t *__restrict__ status_next) {
  extern __shared__ __align__(16) unsigned char os_smem[];
  uint64_t *sk = (uint64_t *)os_smem;
  uint32_t *sv = (uint32_t *)(sk + kOsTile);
  uint32_t *wh = sv + kOsTile;             // [warp][digit] counts, then warp offsets
  uint32_t *texcl = wh + kOsWarps * 256;   // tile-local exclusive offsets per digit
  int64_t *gbase = (int64_t *)(texcl + 256);  // global base per digit (minus texcl)
  uint32_t *stile = (uint32_t *)(gbase + 256) + 256;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (tid == 0) *stile = atomicAdd(ctr, 1u);
  for (int x = tid; x < kOsWarps * 256; x += kOsThreads) wh[x] = 0;
  __syncthreads();
  const uint32_t tile = *stile;
  // the next pass's look-back flags start cleared: each tile clears its own
  // (this pass's predecessor left them set; the next pass starts after this one)
  if (status_next) status_next[(int64_t)tile * 256 + tid] = 0;
  const int64_t base = (int64_t)tile * kOsTile + (int64_t)w * (kOsItems * 32);
  uint64_t k[kOsItems];
#pragma unroll
  for (int j = 0; j < kOsItems; j++) {
    const int64_t i = base + j * 32 + lane;
    k[j] = i < n ? kin[i] : 0;
  }
  {  // warm L2 for the tile a CTA will claim about one residency wave from now
    const int64_t ahead = (int64_t)kOsAhead * kOsTile;
#pragma unroll
    for (int j = 0; j < kOsItems; j += 2) {  // one 128-byte line per 16 lanes and key row pair
      const int64_t i = base + ahead + j * 32 + lane * 2;
      if (i < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(kin + i));
    }
    const int64_t iv = base + ahead + lane * 32;  // 32 values = one line
    if (lane < 15 && iv < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(vin + iv));
  }
  // stable rank inside the warp: peers with the same digit from 8 ballots (one
  // per digit bit, independent, so they pipeline); the highest peer bumps the
  // warp's counter with one shared atomic and broadcasts the old value. The
  // warp's atomics on a counter execute in program order, so rows j keep order.
  uint16_t rk[kOsItems];
  uint32_t *myh = wh + w * 256;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kOsItems; j++) {
    const bool valid = base + j * 32 + lane < n;
    const uint32_t d = (uint32_t)(k[j] >> shift) & mask;
    unsigned peers = __ballot_sync(0xffffffffu, valid);  // (8 ballots beat __match_any_sync here: 6.6 vs 8.7 ms)
#pragma unroll
    for (int b = 0; b < W; b++) {
      const bool bit = (d >> b) & 1u;
      const unsigned bb = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bb : ~bb;
    }
    const int leader = 31 - __clz(peers | 1u);
    uint32_t old = 0;
    if (valid && lane == leader) old = atomicAdd(myh + d, (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader);
    rk[j] = (uint16_t)(old + __popc(peers & lt));
  }
  __syncthreads();
  // digit tid: offsets of each warp inside the tile's run of that digit; the
  // warps' counts sum to the tile's count, published at once
  uint32_t cnt;
  {
    uint32_t run = 0;
#pragma unroll
    for (int x = 0; x < kOsWarps; x++) {
      const uint32_t c = wh[x * 256 + tid];
      wh[x * 256 + tid] = run;
      run += c;
    }
    cnt = run;
  }
  if (tile == 0) {
    atomicExch(status + tid, kOsPrefix | cnt);
  } else {
    atomicExch(status + (int64_t)tile * 256 + tid, kOsAgg | cnt);
  }
  // the tile's digit runs (block scan) and each (warp, digit) block's start:
  // the staging needs nothing from earlier tiles, so it runs before the
  // look-back (which then finds more predecessors published)
  __shared__ uint32_t shs[33];
  const uint32_t tx = block_excl_sum<uint32_t>(cnt, shs, nullptr);
#pragma unroll
  for (int x = 0; x < kOsWarps; x++) wh[x * 256 + tid] += tx;
  __syncthreads();
  // stage the tile in digit order
#pragma unroll
  for (int j = 0; j < kOsItems; j++) {
    const int64_t i = base + j * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)(k[j] >> shift) & mask;
      const uint32_t pos = wh[w * 256 + d] + rk[j];
      sk[pos] = k[j];
      sv[pos] = vin[i];
    }
  }
  // look back over the earlier tiles for this digit
  volatile uint32_t *st = status;
  uint32_t excl = 0;
  if (tile > 0) {
    // windows of 4 predecessors (measured: 4 beats 2, 8 and 16) loaded together (independent L2 loads), consumed
    // newest-first until an inclusive prefix is found; an unpublished entry
    // restarts the window there
    constexpr int W = 4;
    for (int64_t t = (int64_t)tile - 1;;) {
      uint32_t sw[W];
#pragma unroll
      for (int i = 0; i < W; i++) sw[i] = t - i >= 0 ? (uint32_t)st[(t - i) * 256 + tid] : (uint32_t)kOsPrefix;
      int i = 0;
      bool done = false;
#pragma unroll
      for (int q = 0; q < W; q++) {
        if (done || sw[q] == 0 || i != q) continue;
        excl += sw[q] & kOsVal;
        done = (sw[q] & kOsPrefix) != 0;
        i = q + 1;
      }
      if (done) break;
      t -= i;
    }
    atomicExch(status + (int64_t)tile * 256 + tid, kOsPrefix | (excl + cnt));
  }
  gbase[tid] = (int64_t)bins[tid] + excl - tx;
  __syncthreads();
  const int64_t t0 = (int64_t)tile * kOsTile;
  const int cnt_tile = (int)(n - t0 < kOsTile ? n - t0 : kOsTile);
  for (int i = tid; i < cnt_tile; i += kOsThreads) {
    const uint64_t key = sk[i];
    const uint32_t d = (uint32_t)(key >> shift) & mask;
    const int64_t g = gbase[d] + i;
    kout[g] = key;
    vout[g] = sv[i];
  }
}

void radix_sort_pairs(Ctx &ctx, Arena &ar, uint64_t *keys, uint32_t *vals, int64_t n, int begin_bit,
                      int end_bit) {
  if (n <= 1 || end_bit <= begin_bit || !ctx.ok()) return;
  if (n > kSortMax) {  // the look-back status words hold 30-bit counts
    ctx.fail(STW_EARG, "radix sort of %lld records exceeds the limit of 2^30-1", (long long)n);
    return;
  }
  const int passes = (end_bit - begin_bit + 7) / 8;
  const int64_t ntiles = (n + kOsTile - 1) / kOsTile;
  uint64_t *k2 = ar.take<uint64_t>(n);
  uint32_t *v2 = ar.take<uint32_t>(n);
  uint32_t *hist = ar.take<uint32_t>((size_t)passes * 256);
  uint32_t *status = ar.take<uint32_t>((size_t)ntiles * 256 * 2);  // two buffers, alternating by pass
  uint32_t *ctr = ar.take<uint32_t>(passes);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemsetAsync(hist, 0, (size_t)passes * 256 * sizeof(uint32_t), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(ctr, 0, passes * sizeof(uint32_t), ctx.stream));
  STW_KL(k_os_hist, grid_for(n, 256, 148 * 8), 256, ctx.stream, keys, n, begin_bit, end_bit, passes, hist);
  STW_KL(k_os_bins, passes, 256, ctx.stream, hist);
  STW_LAUNCHED(ctx);
  auto pass_kernel = [](int w) {
    switch (w) {
      case 1: return k_os_pass<1>;
      case 2: return k_os_pass<2>;
      case 3: return k_os_pass<3>;
      case 4: return k_os_pass<4>;
      case 5: return k_os_pass<5>;
      case 6: return k_os_pass<6>;
      case 7: return k_os_pass<7>;
      default: return k_os_pass<8>;
    }
  };
  uint64_t *ka = keys, *kb = k2;
  uint32_t *va = vals, *vb = v2;
  for (int p = 0; p < passes && ctx.ok(); p++) {
    const int b = begin_bit + 8 * p, w = end_bit - b < 8 ? end_bit - b : 8;
    uint32_t *cur = status + (size_t)(p & 1) * ntiles * 256, *nxt = status + (size_t)((p + 1) & 1) * ntiles * 256;
    if (p == 0) STW_CUDA(ctx, cudaMemsetAsync(cur, 0, (size_t)ntiles * 256 * sizeof(uint32_t), ctx.stream));
    auto kern = pass_kernel(w);
    STW_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOsSmem));
    {
      const int slot = prof_pre(ctx.stream);
      kern<<<(unsigned)ntiles, kOsThreads, kOsSmem, ctx.stream>>>(ka, va, kb, vb, n, b, (1u << w) - 1, hist + p * 256,
                                                                  cur, ctr + p, p + 1 < passes ? nxt : nullptr);
      prof_post(ctx.stream, "k_os_pass", slot);
    }
    STW_LAUNCHED(ctx);
    std::swap(ka, kb);
    std::swap(va, vb);
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


// ---------------------------------------------------------------------------
// mapped page-locked scratch for small transfers (see common.cuh). Pending
// uploads are moved by ONE multi-copy kernel launched just before the next
// kernel on their stream (prof_pre) or at an explicit h2d_flush; pending
// downloads by one launch at host_sync.

namespace {
struct CopyDesc {
  const unsigned char *src;
  unsigned char *dst;
  int64_t bytes;
};
constexpr int kMaxCopies = 48;
struct CopyBatch {
  CopyDesc d[kMaxCopies];
};

__global__ void k_copy_multi(CopyBatch cb) {
  const CopyDesc c = cb.d[blockIdx.y];
  const bool vec = ((reinterpret_cast<uintptr_t>(c.src) | reinterpret_cast<uintptr_t>(c.dst)) & 15) == 0;
  const int64_t n16 = vec ? c.bytes >> 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = t; i < n16; i += stride)
    reinterpret_cast<uint4 *>(c.dst)[i] = reinterpret_cast<const uint4 *>(c.src)[i];
  for (int64_t i = (n16 << 4) + t; i < c.bytes; i += stride) c.dst[i] = c.src[i];
}

struct PinnedScratch {
  std::vector<std::pair<char *, size_t>> blocks;
  size_t blk = 0, off = 0;
  std::vector<CopyDesc> up, down;  // pending uploads / downloads
  cudaStream_t up_stream = nullptr;
  struct HostCopy {
    void *dst;
    const void *src;
    size_t bytes;
  };
  std::vector<HostCopy> out;  // pinned -> caller memory at host_sync
  char *take(Ctx &ctx, size_t bytes) {
    bytes = (bytes + 15) & ~(size_t)15;
    while (blk < blocks.size() && off + bytes > blocks[blk].second) blk++, off = 0;
    if (blk == blocks.size()) {
      const size_t cap = std::max<size_t>(bytes, 4 << 20);
      void *p = nullptr;
      STW_CUDA(ctx, cudaHostAlloc(&p, cap, cudaHostAllocMapped | cudaHostAllocPortable));
      if (!p) return nullptr;
      blocks.push_back({(char *)p, cap});
      off = 0;
    }
    char *p = blocks[blk].first + off;
    off += bytes;
    return p;
  }
};
thread_local PinnedScratch g_pin;

void launch_copies(std::vector<CopyDesc> &v, cudaStream_t s) {
  for (size_t i = 0; i < v.size(); i += kMaxCopies) {
    CopyBatch cb;
    const int n = (int)std::min<size_t>(kMaxCopies, v.size() - i);
    int64_t mx = 0;
    for (int k = 0; k < n; k++) cb.d[k] = v[i + k], mx = std::max(mx, v[i + k].bytes);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_copy_multi<<<dim3(grid_for((mx + 15) / 16, 256, 64), n), 256, 0, s>>>(cb);
  }
  v.clear();
}
}  // namespace

void pinned_reset() {
  g_pin.up.clear();
  g_pin.down.clear();
  g_pin.out.clear();
  g_pin.blk = 0;
  g_pin.off = 0;
}

void h2d_flush_stream(cudaStream_t s) {
  if (!g_pin.up.empty() && s == g_pin.up_stream) launch_copies(g_pin.up, s);
}

void h2d_flush(Ctx &ctx) {
  if (g_pin.up.empty()) return;
  launch_copies(g_pin.up, g_pin.up_stream);
  STW_LAUNCHED(ctx);
}

void h2d_async(Ctx &ctx, void *ddst, const void *hsrc, size_t bytes) {
  if (!bytes || !ctx.ok()) return;
  if (!g_pin.up.empty() && g_pin.up_stream != ctx.stream) h2d_flush(ctx);
  char *p = g_pin.take(ctx, bytes);
  if (!p) return;
  memcpy(p, hsrc, bytes);
  g_pin.up.push_back({(const unsigned char *)p, (unsigned char *)ddst, (int64_t)bytes});
  g_pin.up_stream = ctx.stream;
}

void d2h_async(Ctx &ctx, void *dst, const void *dsrc, size_t bytes) {
  if (!bytes || !ctx.ok()) return;
  char *p = g_pin.take(ctx, bytes);
  if (!p) return;
  g_pin.down.push_back({(const unsigned char *)dsrc, (unsigned char *)p, (int64_t)bytes});
  g_pin.out.push_back({dst, p, bytes});
}

void host_sync(Ctx &ctx) {
  h2d_flush(ctx);
  if (!g_pin.down.empty()) {
    launch_copies(g_pin.down, ctx.stream);
    STW_LAUNCHED(ctx);
  }
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (ctx.ok())
    for (auto &q : g_pin.out) memcpy(q.dst, q.src, q.bytes);
  g_pin.out.clear();
  g_pin.up.clear();
  g_pin.down.clear();
  g_pin.blk = 0;
  g_pin.off = 0;
}

}  // namespace stw

extern "C" {

long long stw_launch_count(void) { return stw::g_launches.load(); }

int stw_release_scratch(void) {
  using namespace stw;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (cudaDeviceSynchronize() != cudaSuccess) return STW_ECUDA;
  for (auto &kv : g_pools)
    if (cudaMemPoolTrimTo(kv.second, 0) != cudaSuccess) return STW_ECUDA;
  return STW_OK;
}

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
