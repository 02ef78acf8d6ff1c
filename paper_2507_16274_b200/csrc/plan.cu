// Batched static planner (synthesize_static_plan, planner.py:357-473) for a
// batch of traces x candidate (fusion, gap_insert) settings.
//
// Pipeline (every stage runs on the device; the host only sizes buffers):
//   A  canonical ranks    q = id rank, r = (t_s, id) rank per trace      (K2 sorts)
//   B  phase groups       one stable sort by (trace, class, p_s, p_e, r);
//                         persistent block, HomoPhase groups, packing by a
//                         global exclusive scan of sizes, per-plan height /
//                         span / used / TMP                              (K3)
//   C  fusion sweep       one CTA per trace, block-parallel cursor search  (K4)
//   D  layer items        plans + residuals, sorted by (size desc, t_s, tie)
//   E  HomoSize layers    one CTA per unit; per size class: parallel
//                         fixed-slot fit masks -> warp-serial resolve of gap
//                         insertion + Alg. 1 -> merge of the slot CSR      (K5)
//   F  stacking/emission  layer bases by scan, addresses per event        (K6)
//   G  self-check         static peak (K1) and the rectangle sweep (K7)
//
// Decomposition used by E (exactly equivalent to MemoryLayer.fits_gap,
// planner.py:199-212, because every layer's slots are pairwise disjoint as
// closed intervals): an item of class S fits layer L iff it does not overlap
// the slots L held before class S started, and every class-S item already
// gap-inserted into L ended before the item starts.
#include <algorithm>
#include <vector>

#include <cooperative_groups.h>

#include "planner.cuh"

namespace stw {

constexpr int kPlanThreads = 256;
constexpr int kFitWords = 4;      // fit masks kept for the first 128 layers of a class
constexpr int kSmemLayers = 1024;  // per-class resolve state kept in shared memory up to this

// ---------------------------------------------------------------------------
// generic helpers

template <class T>
__device__ T block_reduce_min(T v, T *sh) {
  for (int o = 16; o; o >>= 1) {
    T n = __shfl_down_sync(0xffffffffu, v, o);
    v = n < v ? n : v;
  }
  int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane_id() == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T m = sh[0];
    for (int k = 1; k < nw; k++) m = sh[k] < m ? sh[k] : m;
    sh[32] = m;
  }
  __syncthreads();
  T out = sh[32];
  __syncthreads();
  return out;
}

template <class T>
__device__ T block_reduce_max(T v, T *sh) {
  for (int o = 16; o; o >>= 1) {
    T n = __shfl_down_sync(0xffffffffu, v, o);
    v = n > v ? n : v;
  }
  int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane_id() == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T m = sh[0];
    for (int k = 1; k < nw; k++) m = sh[k] > m ? sh[k] : m;
    sh[32] = m;
  }
  __syncthreads();
  T out = sh[32];
  __syncthreads();
  return out;
}

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_fill_i32(int32_t *__restrict__ p, int64_t n, int32_t v) { GRID_STRIDE(i, n) p[i] = v; }

// trace index of every event: one warp per trace writes its run (coalesced)
// Phase A in one pass, one CTA per trace: the trace index of every event
// (coalesced runs); flags[0] = 1 unless every trace's ids increase strictly
// and its t_s never decrease (then its id order and its (t_s, id) order are
// both the listing order); id range (mm[0], mm[1]) and max t_s (flags[1]) for
// the sort key widths; the input checks -- bad_align[t] / bad_phase[t] = the
// first static event (trace-local index) whose size is not aligned
// (planner.py:371-373) / whose timestamps leave [0, horizon] (model.py:240-241)
// or whose scoped phases are missing from the schedule (model.py:201-205),
// INT_MAX if none -- and flags[2] = the largest phase
// index of a scoped static event.
__global__ void __launch_bounds__(128) k_trace_scan(
    const int64_t *__restrict__ ev_off, int T, const int64_t *__restrict__ id, const int32_t *__restrict__ ts,
    const int32_t *__restrict__ te, const int64_t *__restrict__ size, const int32_t *__restrict__ ps,
    const int32_t *__restrict__ pe, const uint8_t *__restrict__ dyn, const int32_t *__restrict__ horizon,
    const int32_t *__restrict__ n_sched, long long align, int32_t *__restrict__ tr, int *__restrict__ bad_align,
    int *__restrict__ bad_phase, int *__restrict__ flags, long long *__restrict__ mm, int64_t chunk) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ int s_ba, s_bp;
  // blockIdx.y: the part of a long trace (gridDim.y > 1 only when some trace
  // has more than `chunk` events; then bad_* were filled with INT_MAX first)
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_ba = s_bp = INT_MAX;
  __syncthreads();
  const int64_t e0 = ev_off[t], te1 = ev_off[t + 1];
  const int64_t p0 = e0 + (int64_t)blockIdx.y * chunk;
  if (gridDim.y > 1 && p0 >= te1 && blockIdx.y > 0) return;
  const int64_t e1 = gridDim.y > 1 ? min(te1, p0 + chunk) : te1;
  const int hz = horizon[t], ns = n_sched[t];
  bool bad = false;
  long long idmin = LLONG_MAX, idmax = LLONG_MIN;
  int tsmax = 0, pmax = 0, ba = INT_MAX, bp = INT_MAX;
  const bool pow2 = (align & (align - 1)) == 0;
  // every column loaded up front and branch-free (more loads in flight per warp)
#pragma unroll 2
  for (int64_t i = (gridDim.y > 1 ? p0 : e0) + tid; i < e1; i += blockDim.x) {
    const int64_t my_id = id[i], sz = size[i];
    const int my_ts = ts[i], my_te = te[i], a = ps[i], z = pe[i];
    const bool dy = dyn[i] != 0;
    const int64_t prev_id = i > e0 ? id[i - 1] : LLONG_MIN;
    const int prev_ts = i > e0 ? ts[i - 1] : INT_MIN;
    tr[i] = t;
    idmin = min(idmin, (long long)my_id);
    idmax = max(idmax, (long long)my_id);
    tsmax = max(tsmax, my_ts);
    bad |= !(prev_id < my_id && prev_ts <= my_ts);
    const int loc = (int)(i - e0);
    if (my_ts < 0 || my_ts >= hz || my_te > hz) bp = min(bp, loc);  // model.py:240-241
    const bool misal = pow2 ? (sz & (align - 1)) != 0 : (sz % align) != 0;
    if (!dy && misal) ba = min(ba, loc);
    if (!dy && my_te < hz) {
      if (a >= ns || z >= ns) bp = min(bp, loc);
      pmax = max(pmax, max(a, z));
    }
  }
  ba = __reduce_min_sync(FULL, ba);
  bp = __reduce_min_sync(FULL, bp);
  for (int o = 16; o; o >>= 1) {
    idmin = min(idmin, __shfl_xor_sync(FULL, idmin, o));
    idmax = max(idmax, __shfl_xor_sync(FULL, idmax, o));
  }
  tsmax = __reduce_max_sync(FULL, tsmax);
  pmax = __reduce_max_sync(FULL, pmax);
  const bool anybad = __any_sync(FULL, bad);
  __shared__ int s_bad, s_ts, s_pm;
  __shared__ long long s_lo, s_hi;
  if (tid == 0) {
    s_bad = 0, s_ts = 0, s_pm = 0;
    s_lo = LLONG_MAX, s_hi = LLONG_MIN;
  }
  __syncthreads();
  if (lane == 0) {
    if (ba != INT_MAX) atomicMin(&s_ba, ba);
    if (bp != INT_MAX) atomicMin(&s_bp, bp);
    if (anybad) s_bad = 1;
    atomicMax(&s_ts, tsmax);
    atomicMax(&s_pm, pmax);
    atomicMin(&s_lo, idmin);
    atomicMax(&s_hi, idmax);
  }
  __syncthreads();
  if (tid == 0) {
    if (gridDim.y == 1) {
      bad_align[t] = s_ba;
      bad_phase[t] = s_bp;
    } else {
      if (s_ba != INT_MAX) atomicMin(bad_align + t, s_ba);
      if (s_bp != INT_MAX) atomicMin(bad_phase + t, s_bp);
    }
    // batch-wide values: one CTA-level update each, and only when it changes the
    // current value (thousands of CTAs would otherwise serialise on five words)
    volatile int *vf = flags;
    volatile long long *vm = mm;
    if (s_bad) atomicOr(flags, 1);
    if (s_ts > vf[1]) atomicMax(flags + 1, s_ts);
    if (s_pm > vf[2]) atomicMax(flags + 2, s_pm);
    if (s_lo != LLONG_MAX) {
      if (s_lo < vm[0]) atomicMin(mm, s_lo);
      if (s_hi > vm[1]) atomicMax(mm + 1, s_hi);
    }
  }
}

// off[0..n] = exclusive prefix sums of cnt[0..n) (uint32), one CTA
__global__ void __launch_bounds__(1024) k_offsets_u32(const uint32_t *__restrict__ cnt, int n,
                                                      uint32_t *__restrict__ off) {
  __shared__ uint32_t sh[33];
  uint32_t carry = 0;
  for (int b = 0; b < n; b += blockDim.x) {
    const int i = b + threadIdx.x;
    const uint32_t v = i < n ? cnt[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_sum<uint32_t>(v, sh, &tot);
    if (i < n) off[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = carry;
}

// off[0..n] = exclusive prefix sums of cnt[0..n) (int64), one CTA
__global__ void __launch_bounds__(1024) k_offsets_i32(const int *__restrict__ cnt, int n, int64_t *__restrict__ off) {
  __shared__ long long sh[33];
  long long carry = 0;
  for (int b = 0; b < n; b += blockDim.x) {
    const int i = b + threadIdx.x;
    const long long v = i < n ? cnt[i] : 0;
    long long tot;
    const long long ex = block_excl_sum<long long>(v, sh, &tot);
    if (i < n) off[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = carry;
}

__global__ void k_minmax_i64(const int64_t *__restrict__ v, int64_t n, long long *mn, long long *mx) {
  __shared__ long long sh[33];
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  GRID_STRIDE(i, n) {
    lo = min(lo, (long long)v[i]);
    hi = max(hi, (long long)v[i]);
  }
  lo = block_reduce_min(lo, sh);
  hi = block_reduce_max(hi, sh);
  if (threadIdx.x == 0) {
    atomicMin(mn, lo);
    atomicMax(mx, hi);
  }
}

__global__ void k_max_i32(const int32_t *__restrict__ v, int64_t n, int *mx) {
  __shared__ int sh[33];
  int hi = 0;
  GRID_STRIDE(i, n) hi = max(hi, v[i]);
  hi = block_reduce_max(hi, sh);
  if (threadIdx.x == 0) atomicMax(mx, hi);
}

__global__ void k_concat_key(uint64_t *__restrict__ hi, const uint64_t *__restrict__ lo, int lobits, int64_t n) {
  GRID_STRIDE(i, n) hi[i] = (lobits >= 64 ? 0 : (hi[i] << lobits)) | lo[i];
}

__global__ void k_gather_u64(const uint64_t *__restrict__ src, const uint32_t *__restrict__ perm,
                             uint64_t *__restrict__ dst, int64_t n) {
  GRID_STRIDE(i, n) dst[i] = src[perm[i]];
}

void sort_perm2(Ctx &ctx, Arena &ar, uint64_t *hi, int hibits, uint64_t *lo, int lobits, uint32_t *perm,
                int64_t n) {
  if (!ctx.ok() || n == 0) return;
  if (hibits + lobits <= 64) {
    STW_KL(k_concat_key, grid_for(n, 256), 256, ctx.stream, hi, lo, lobits, n);
    STW_LAUNCHED(ctx);
    sort_perm(ctx, ar, hi, perm, n, hibits + lobits);
    return;
  }
  sort_perm(ctx, ar, lo, perm, n, lobits);
  STW_KL(k_gather_u64, grid_for(n, 256), 256, ctx.stream, hi, perm, lo, n);  // lo := hi[perm]
  STW_LAUNCHED(ctx);
  radix_sort_pairs(ctx, ar, lo, perm, n, 0, hibits);
}


// ---------------------------------------------------------------------------
// CTA-local segmented sort: one CTA per segment (trace or (variant, trace)),
// an LSD radix sort of (key, index) pairs in shared memory -- a stable sort of
// the segment in one global read + write. Used whenever every segment fits
// kSegSortMax elements; otherwise the global LSD radix sort (K2) runs.

constexpr int kSegSortMax = 4096;

__global__ void k_local_key(uint64_t *__restrict__ hi, const uint64_t *__restrict__ lo, uint64_t mask, int lobits,
                            int64_t n) {
  GRID_STRIDE(i, n) hi[i] = (lobits >= 64 ? 0 : ((hi[i] & mask) << lobits)) | lo[i];
}

// Segmented LSD radix sort in shared memory: one CTA per segment, 8-bit
// digits, only the key bits [bit0, bits) (a caller whose elements are already
// ordered by the lower bits starts above them). Per pass each warp ranks its
// contiguous block of the segment row by row -- peers from one ballot per
// digit bit, the highest peer bumps the warp's digit counter with one shared
// atomic -- then one thread per digit turns the (digit, warp) counts into
// offsets and the elements are scattered to the other shared buffer. Stable;
// ~40 instructions per element per pass instead of the bitonic network's
// ~log2(P)^2/2 compare-exchanges.
// The passes of the CTA-local sort: (key, value) pairs kA/vA[0, n) in shared
// memory, stable by key bits [bit0, bits); wh = 8 x 256 counters; sh = 33.
template <int IPT>
__device__ __forceinline__ void cta_radix(uint64_t *kA, uint32_t *vA, uint32_t *wh, uint32_t *sh, int n, int bit0,
                                          int bits) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const unsigned lt = lanemask_lt();
  const int R = (n + 255) >> 8;  // rows of 32 per warp actually used (<= IPT)
  const int run = 32 * R;        // each warp owns a contiguous block of the segment
  for (int b = bit0, width; b < bits; b += width) {
    // the fewest 8-bit-or-narrower passes, widths balanced (fewer ballots per pass)
    const int left = bits - b;
    width = (left + (left + 7) / 8 - 1) / ((left + 7) / 8);
    const uint32_t mask = (1u << width) - 1;
    for (int x = tid; x < 8 * 256; x += 256) wh[x] = 0;
    __syncthreads();
    uint64_t k[IPT];
    uint32_t v[IPT];
    uint16_t rk[IPT];
    uint32_t *myh = wh + w * 256;
#pragma unroll
    for (int j = 0; j < IPT; j++) {
      if (j >= R) break;
      const int e = w * run + j * 32 + lane;
      const bool valid = e < n;
      k[j] = valid ? kA[e] : 0;
      v[j] = valid ? vA[e] : 0;
      const uint32_t d = (uint32_t)(k[j] >> b) & mask;
      unsigned peers = __ballot_sync(0xffffffffu, valid);
      for (int q = 0; q < width; q++) {
        const bool bit = (d >> q) & 1u;
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
    {  // digit tid: offsets of (digit, warp) blocks in digit-major order
      uint32_t run = 0;
#pragma unroll
      for (int x = 0; x < 8; x++) {
        const uint32_t c = wh[x * 256 + tid];
        wh[x * 256 + tid] = run;
        run += c;
      }
      const uint32_t base = block_excl_sum<uint32_t>(run, sh, nullptr);
#pragma unroll
      for (int x = 0; x < 8; x++) wh[x * 256 + tid] += base;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; j++) {
      if (j >= R) break;
      const int e = w * run + j * 32 + lane;
      if (e < n) {
        const uint32_t d = (uint32_t)(k[j] >> b) & mask;
        const uint32_t pos = myh[d] + rk[j];
        kA[pos] = k[j];
        vA[pos] = v[j];
      }
    }
    __syncthreads();
  }
}

template <int IPT>
__global__ void __launch_bounds__(256) k_seg_radix(uint64_t *__restrict__ keys, uint32_t *__restrict__ perm,
                                                   const int64_t *__restrict__ seg_off, int bit0, int bits) {
  constexpr int P = 256 * IPT;
  extern __shared__ __align__(16) unsigned char srx[];
  uint64_t *kA = (uint64_t *)srx;  // one buffer: a pass holds its elements in registers
  uint32_t *vA = (uint32_t *)(kA + P);
  uint32_t *wh = vA + P;  // [8 warps][256 digits]
  __shared__ uint32_t sh[33];
  const int64_t s0 = seg_off[blockIdx.x];
  const int n = (int)(seg_off[blockIdx.x + 1] - s0);
  const int tid = threadIdx.x;
  {
    bool all = true;  // no bits to sort, or already in order: the stable result is the identity
    if (bit0 < bits)
      for (int i = tid; i + 1 < n; i += 256) all &= keys[s0 + i] <= keys[s0 + i + 1];
    if (__syncthreads_and(all)) {
      for (int i = tid; i < n; i += 256) perm[s0 + i] = (uint32_t)(s0 + i);
      return;
    }
  }
  for (int i = tid; i < n; i += 256) {
    kA[i] = keys[s0 + i];
    vA[i] = (uint32_t)(s0 + i);
  }
  __syncthreads();
  cta_radix<IPT>(kA, vA, wh, sh, n, bit0, bits);
  for (int i = tid; i < n; i += 256) {
    keys[s0 + i] = kA[i];
    perm[s0 + i] = vA[i];
  }
}

// Stable sort of n elements by (segment, hi & ~segment bits, lo), segments
// given by seg_off[nseg+1] (device) and contiguous. hi/lo are consumed.
static void seg_sort(Ctx &ctx, Arena &ar, uint64_t *hi, int hibits, int segbits, uint64_t *lo, int lobits,
                     uint32_t *perm, int64_t n, const int64_t *seg_off, int64_t nseg, int64_t max_seg,
                     bool lo_in_order = false) {
  if (!ctx.ok() || n == 0) return;
  const int local_hi = hibits - segbits;
  if (max_seg <= kSegSortMax && local_hi + lobits <= 64) {
    uint64_t mask = local_hi >= 64 ? ~0ull : ((1ull << local_hi) - 1);
    STW_KL(k_local_key, grid_for(n, 256), 256, ctx.stream, hi, lo, mask, lobits, n);
    // lo_in_order: every segment already lists its elements by the low key bits,
    // so a stable sort on the high bits alone is the full sort
    const int bit0 = lo_in_order ? lobits : 0, bits = local_hi + lobits;
    if (max_seg <= 2048) {
      constexpr int smem = 2048 * 12 + 8 * 256 * 4;
      STW_KLS(k_seg_radix<8>, (unsigned)nseg, 256, smem, ctx.stream, hi, perm, seg_off, bit0, bits);
    } else {
      constexpr int smem = 4096 * 12 + 8 * 256 * 4;
      STW_CUDA(ctx, cudaFuncSetAttribute(k_seg_radix<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      STW_KLS(k_seg_radix<16>, (unsigned)nseg, 256, smem, ctx.stream, hi, perm, seg_off, bit0, bits);
    }
    STW_LAUNCHED(ctx);
    return;
  }
  sort_perm2(ctx, ar, hi, hibits, lo, lobits, perm, n);
}

// traces in recorded order: both canonical ranks are the position in the trace
__global__ void k_identity_ranks(const int32_t *__restrict__ tr, const int64_t *__restrict__ ev_off, int64_t n,
                                 int32_t *__restrict__ q, int32_t *__restrict__ r, uint32_t *__restrict__ rperm,
                                 int32_t *__restrict__ local_order) {
  GRID_STRIDE(i, n) {
    const int32_t k = (int32_t)(i - ev_off[tr[i]]);
    q[i] = k;
    r[i] = k;
    rperm[i] = (uint32_t)i;
    local_order[i] = k;
  }
}

// rank[perm[k]] = k - ev_off[trace]; optional per-trace local permutation
__global__ void k_rank_from_perm(const uint32_t *__restrict__ perm, const int32_t *__restrict__ tr,
                                 const int64_t *__restrict__ ev_off, int64_t n, int32_t *__restrict__ rank,
                                 int32_t *__restrict__ local_order) {
  GRID_STRIDE(k, n) {
    uint32_t i = perm[k];
    int64_t b = ev_off[tr[i]];
    rank[i] = (int32_t)(k - b);
    if (local_order) local_order[k] = (int32_t)(i - b);
  }
}

__device__ __forceinline__ int ev_class(uint8_t dyn, int32_t te, int32_t horizon) {
  return dyn ? 2 : (te >= horizon ? 0 : 1);  // 0 persistent, 1 scoped static, 2 dynamic
}

// ---------------------------------------------------------------------------
// A: keys

__global__ void k_key_q(const int32_t *__restrict__ tr, const int64_t *__restrict__ id, int64_t n, long long idmin,
                        uint64_t *__restrict__ hi, uint64_t *__restrict__ lo) {
  GRID_STRIDE(i, n) {
    hi[i] = (uint64_t)tr[i];
    lo[i] = (uint64_t)((long long)id[i] - idmin);
  }
}

__global__ void k_key_r(const int32_t *__restrict__ tr, const int32_t *__restrict__ ts, const int32_t *__restrict__ q,
                        int64_t n, int qb, uint64_t *__restrict__ hi, uint64_t *__restrict__ lo) {
  GRID_STRIDE(i, n) {
    hi[i] = (uint64_t)tr[i];
    lo[i] = ((uint64_t)(uint32_t)ts[i] << qb) | (uint32_t)q[i];
  }
}

__global__ void k_key_group(const int32_t *__restrict__ tr, const int32_t *__restrict__ te,
                            const int32_t *__restrict__ ps, const int32_t *__restrict__ pe,
                            const uint8_t *__restrict__ dyn, const int32_t *__restrict__ horizon,
                            const int32_t *__restrict__ r, int64_t n, int pb, uint64_t *__restrict__ hi,
                            uint64_t *__restrict__ lo) {
  GRID_STRIDE(i, n) {
    int t = tr[i];
    int c = ev_class(dyn[i], te[i], horizon[t]);
    uint64_t a = c == 1 ? (uint32_t)ps[i] : 0, b = c == 1 ? (uint32_t)pe[i] : 0;
    hi[i] = ((uint64_t)t << (2 + 2 * pb)) | ((uint64_t)c << (2 * pb)) | (a << pb) | b;
    lo[i] = (uint32_t)r[i];
  }
}

// ---------------------------------------------------------------------------
// B: groups

struct Ev {
  const int32_t *tr, *ts, *te, *ps, *pe, *q;
  const int64_t *size;
  const uint8_t *dyn;
  const int32_t *horizon;
};

__device__ __forceinline__ void group_key(const Ev &e, uint32_t i, int *c, int *a, int *b) {
  *c = ev_class(e.dyn[i], e.te[i], e.horizon[e.tr[i]]);
  *a = *c == 1 ? e.ps[i] : 0;
  *b = *c == 1 ? e.pe[i] : 0;
}

__global__ void k_group_heads(Ev e, const uint32_t *__restrict__ gperm, const int64_t *__restrict__ ev_off, int64_t n,
                              uint32_t *__restrict__ head, int64_t *__restrict__ szs) {
  GRID_STRIDE(k, n) {
    uint32_t i = gperm[k];
    szs[k] = e.size[i];
    int t = e.tr[i];
    uint32_t h = 1;
    if (k != ev_off[t]) {
      int c1, a1, b1, c0, a0, b0;
      group_key(e, i, &c1, &a1, &b1);
      group_key(e, gperm[k - 1], &c0, &a0, &b0);
      h = (c1 != c0 || a1 != a0 || b1 != b0);
    }
    head[k] = h;
  }
}

struct Groups {
  int64_t *start;  // first sorted position
  int32_t *tr, *cls, *ps, *pe;
  int64_t *height;
};

struct TraceCounts {
  int *n_static, *n_pers, *n_groups, *n_plans, *n_res;
  int64_t *pers_size;
};

// Phase B fused (traces of <= 4096 events): one CTA per trace sorts the
// trace's events by (class, p_s, p_e, r) in shared memory (k_key_group + the
// segmented sort) and builds the whole group table from the sorted order --
// the work of k_group_heads, the two global scans, k_group_table, k_group_rel
// and k_trace_counts -- without a round trip through HBM. Group ids are sparse:
// trace t's groups take [ev_off[t], ev_off[t] + groups of t) (a trace has no
// more groups than events), so no cross-trace offset is needed; the gaps read
// as non-plan groups (is_plan is zeroed). pidx gets each plan group's rank
// among the trace's plan groups (the global plan index is pl_off[t] + that).
template <int IPT>
__global__ void __launch_bounds__(256, IPT == 8 ? 4 : 1) k_groups_fused(Ev e, const int64_t *__restrict__ ev_off,
                                                      const int32_t *__restrict__ r, int pb, int qb, int bit0,
                                                      uint32_t *__restrict__ gperm, Groups g,
                                                      int64_t *__restrict__ rel, int32_t *__restrict__ gof,
                                                      TraceCounts tc, uint32_t *__restrict__ is_plan,
                                                      uint32_t *__restrict__ pidx) {
  constexpr int CAP = 256 * IPT;
  extern __shared__ __align__(16) unsigned char sgs[];
  uint64_t *kA = (uint64_t *)sgs;
  uint32_t *vA = (uint32_t *)(kA + CAP);
  uint32_t *wh = vA + CAP;
  long long *gS = (long long *)(wh + 8 * 256);  // [CAP + 1] group start offsets (prefix of sizes)
  uint8_t *gc = (uint8_t *)(gS + CAP + 1);      // [CAP] class | plan << 2
  __shared__ uint32_t sh[33];
  __shared__ long long shl[33];
  __shared__ int cnt[4];  // static events, persistent events, residual events, class-1 groups
  const int t = blockIdx.x, tid = threadIdx.x;
  const int64_t g0 = ev_off[t];
  const int n = (int)(ev_off[t + 1] - g0);
  const int hz = e.horizon[t];
  if (tid < 4) cnt[tid] = 0;
  for (int j = tid; j < n; j += blockDim.x) {
    const int64_t i = g0 + j;
    const int c = ev_class(e.dyn[i], e.te[i], hz);
    const uint64_t a = c == 1 ? (uint32_t)e.ps[i] : 0, b = c == 1 ? (uint32_t)e.pe[i] : 0;
    kA[j] = ((((uint64_t)c << (2 * pb)) | (a << pb) | b) << qb) | (uint32_t)r[i];
    vA[j] = (uint32_t)j;
  }
  __syncthreads();
  cta_radix<IPT>(kA, vA, wh, sh, n, bit0, qb + 2 + 2 * pb);
  const uint64_t pmask = (1ull << pb) - 1;
  // chunked scans: thread tid owns sorted positions [c0, c1)
  const int per = (n + 255) >> 8, c0 = min(n, tid * per), c1 = min(n, c0 + per);
  uint32_t hm = 0, nh = 0, np = 0;  // head bits of the chunk (per <= 16), heads, plan heads
  long long ssum = 0;
  for (int k = c0; k < c1; k++) {
    const uint64_t key = kA[k] >> qb;
    const bool h = k == 0 || key != (kA[k - 1] >> qb);
    hm |= (h ? 1u : 0u) << (k - c0);
    nh += h;
    np += h && (key >> (2 * pb)) == 1 && ((key >> pb) & pmask) != (key & pmask);
    const int64_t i = g0 + vA[k];
    gperm[g0 + k] = (uint32_t)i;
    ssum += e.size[i];
  }
  uint32_t htot;
  const uint32_t hex = block_excl_sum<uint32_t>(nh, sh, &htot);
  uint32_t ptot;
  const uint32_t pex = block_excl_sum<uint32_t>(np, sh, &ptot);
  long long stot;
  const long long sex = block_excl_sum<long long>(ssum, shl, &stot);
  // heads: the group table; every position: its offset (kept in kA)
  uint32_t gcount = hex, pcount = pex;
  long long run = sex;
  for (int k = c0; k < c1; k++) {
    const uint64_t key = kA[k] >> qb;
    const long long sz = e.size[g0 + vA[k]];
    if ((hm >> (k - c0)) & 1u) {
      const int lg = (int)gcount++;
      const int c = (int)(key >> (2 * pb));
      const int a = (int)((key >> pb) & pmask), b = (int)(key & pmask);
      const bool plan = c == 1 && a != b;
      const int64_t gi = g0 + lg;
      g.start[gi] = g0 + k;
      g.tr[gi] = t;
      g.cls[gi] = c;
      g.ps[gi] = a;
      g.pe[gi] = b;
      is_plan[gi] = plan;
      if (plan) pidx[gi] = pcount++;
      gS[lg] = run;
      gc[lg] = (uint8_t)(c | (plan ? 4 : 0));
    }
    kA[k] = (uint64_t)run;
    run += sz;
  }
  if (tid == 0) gS[htot] = stot;
  __syncthreads();
  // every event: its offset inside its group, its group; the event counts
  gcount = hex;
  int nst = 0, npe = 0, nre = 0;
  for (int k = c0; k < c1; k++) {
    gcount += (hm >> (k - c0)) & 1u;
    const int lg = (int)gcount - 1;
    const int64_t i = g0 + vA[k];
    rel[i] = (long long)kA[k] - gS[lg];
    gof[i] = (int32_t)(g0 + lg);
    const int m = gc[lg];
    nst += (m & 3) <= 1;
    npe += (m & 3) == 0;
    nre += m == 1;
  }
  // every group: its height; the group counts
  int ngr = 0;
  for (int lg = tid; lg < (int)htot; lg += blockDim.x) {
    const long long h = gS[lg + 1] - gS[lg];
    g.height[g0 + lg] = h;
    const int m = gc[lg];
    if ((m & 3) == 0) tc.pers_size[t] = h;
    ngr += (m & 3) == 1;
  }
  if (nst) atomicAdd(&cnt[0], nst);
  if (npe) atomicAdd(&cnt[1], npe);
  if (nre) atomicAdd(&cnt[2], nre);
  if (ngr) atomicAdd(&cnt[3], ngr);
  __syncthreads();
  if (tid == 0) {
    tc.n_static[t] = cnt[0];
    tc.n_pers[t] = cnt[1];
    tc.n_res[t] = cnt[2];
    tc.n_groups[t] = cnt[3];
    tc.n_plans[t] = (int)ptot;
  }
}

// goff (optional): per-trace group offsets when gid holds trace-local ids
// (k_groups_fused); gid is rewritten to the global inclusive id
__global__ void k_group_table(Ev e, const uint32_t *__restrict__ gperm, const uint32_t *__restrict__ head,
                              uint32_t *__restrict__ gid_incl, const uint32_t *__restrict__ goff, int64_t n,
                              Groups g) {
  GRID_STRIDE(k, n) {
    uint32_t i = gperm[k];
    if (goff) gid_incl[k] += goff[e.tr[i]];
    if (!head[k]) continue;
    int gi = (int)gid_incl[k] - 1;
    int c, a, b;
    group_key(e, i, &c, &a, &b);
    g.start[gi] = k;
    g.tr[gi] = e.tr[i];
    g.cls[gi] = c;
    g.ps[gi] = a;
    g.pe[gi] = b;
  }
}

__global__ void k_group_rel(const uint32_t *__restrict__ gperm, const uint32_t *__restrict__ gid_incl,
                            const int64_t *__restrict__ S, const int64_t *__restrict__ szs, Groups g,
                            int64_t n, const uint32_t *__restrict__ Gp, int64_t *__restrict__ rel,
                            int32_t *__restrict__ gof) {
  const int G = (int)*Gp;  // number of groups
  GRID_STRIDE(k, n) {
    int gi = (int)gid_incl[k] - 1;
    uint32_t i = gperm[k];
    rel[i] = S[k] - S[g.start[gi]];
    gof[i] = gi;
    int64_t end = gi + 1 < G ? g.start[gi + 1] : n;
    if (k == end - 1) g.height[gi] = S[k] + szs[k] - S[g.start[gi]];
  }
}

__global__ void k_trace_counts(Groups g, const uint32_t *__restrict__ Gp, int64_t n, TraceCounts tc,
                               uint32_t *__restrict__ is_plan) {
  const int G = (int)*Gp;  // launched over an upper bound (n); groups past G idle
  GRID_STRIDE(gi, (int64_t)G) {
    int t = g.tr[gi];
    int64_t cnt = (gi + 1 < G ? g.start[gi + 1] : n) - g.start[gi];
    int c = g.cls[gi];
    uint32_t plan = 0;
    if (c == 0) {
      tc.n_pers[t] = (int)cnt;
      tc.pers_size[t] = g.height[gi];
      atomicAdd(tc.n_static + t, (int)cnt);
    } else if (c == 1) {
      atomicAdd(tc.n_groups + t, 1);
      atomicAdd(tc.n_static + t, (int)cnt);
      if (g.ps[gi] != g.pe[gi]) {
        plan = 1;
        atomicAdd(tc.n_plans + t, 1);
      } else {
        atomicAdd(tc.n_res + t, (int)cnt);
      }
    }
    is_plan[gi] = plan;
  }
}

// plan table (one entry per cross-phase group, planner.py:88-115)
struct Plans {
  int32_t *grp, *tr;
  int64_t *h;
  int32_t *ts, *te, *k0, *k1, *minq;
  unsigned long long *used;  // 2 words per plan
  double *tmp;
  uint8_t *alive;
};

// pl_off: pidx holds trace-local plan ranks (k_groups_fused), else global ones;
// Gp: the group count (nullptr: sparse ids below gcap)
__global__ void k_plan_init(Groups g, const uint32_t *__restrict__ Gp, int64_t gcap, const uint32_t *__restrict__ is_plan,
                            const uint32_t *__restrict__ pidx, const int64_t *__restrict__ pl_off,
                            const uint32_t *__restrict__ gperm, Ev e, Plans p) {
  const int64_t G = Gp ? (int64_t)*Gp : gcap;
  GRID_STRIDE(gi, G) {
    if (!is_plan[gi]) continue;
    const int64_t k = pidx[gi] + (pl_off ? pl_off[g.tr[gi]] : 0);
    p.grp[k] = (int)gi;
    p.tr[k] = g.tr[gi];
    p.h[k] = g.height[gi];
    p.ts[k] = e.ts[gperm[g.start[gi]]];  // members are (t_s, id) ordered
    p.te[k] = INT_MIN;
    p.minq[k] = INT_MAX;
    p.k0[k] = g.ps[gi];
    p.k1[k] = g.pe[gi];
    p.used[2 * k] = 0;
    p.used[2 * k + 1] = 0;
    p.alive[k] = 1;
  }
}

__global__ void k_plan_members(const uint32_t *__restrict__ gperm, const int32_t *__restrict__ gof,
                               const uint32_t *__restrict__ is_plan, const uint32_t *__restrict__ pidx,
                               const int64_t *__restrict__ pl_off, Ev e, int64_t n, Plans p,
                               int32_t *__restrict__ pid) {
  GRID_STRIDE(k, n) {
    uint32_t i = gperm[k];
    int gi = gof[i];
    if (!is_plan[gi]) {
      pid[i] = -1;
      continue;
    }
    const int64_t pk = pidx[gi] + (pl_off ? pl_off[e.tr[i]] : 0);
    pid[i] = (int)pk;
    atomicMax(p.te + pk, e.te[i]);
    atomicMin(p.minq + pk, e.q[i]);
    atomic_add_u128(p.used + 2 * pk, (u128)(uint64_t)e.size[i] * (u128)(uint32_t)(e.te[i] - e.ts[i]));
  }
}

__global__ void k_plan_tmp(Plans p, int64_t P) {
  GRID_STRIDE(k, P) {
    u128 used = ((u128)p.used[2 * k + 1] << 64) | p.used[2 * k];
    p.tmp[k] = exact_div(used, (u128)(uint64_t)p.h[k] * (u128)(uint32_t)(p.te[k] - p.ts[k]));
  }
}

// ---------------------------------------------------------------------------
// C: fusion sweep (planner.py:124-182, 329-354), one CTA per trace

struct FusionArgs {
  const int64_t *ev_off;
  const uint32_t *rperm;  // events in (trace, t_s, id) order
  Ev e;
  const int64_t *pl_off;  // [T+1]
  Plans p;                // variant-1 plan state (mutated)
  int32_t *lst;           // plan list order, per trace segment
  int32_t *pid;           // per event plan (mutated)
  int64_t *frel;          // per event address inside its plan (mutated)
  // per-trace scratch, segment [ev_off[t], ev_off[t+1])
  int64_t *fx_addr, *fx_end;
  int32_t *fx_ts, *fx_te;
  int32_t *rm_ev;
  int64_t *rm_new;
  uint8_t *rm_gone;
  uint32_t *memo;
  const int64_t *memo_off;  // bit offsets per trace (memo disabled when off[t]==off[t+1])
  int64_t *attempts, *accepted;
  double *acc_tmp, *acc_avg;  // indexed by pl_off[t] + k
};

__device__ __forceinline__ u128 plan_used(const Plans &p, int k) {
  return ((u128)p.used[2 * k + 1] << 64) | p.used[2 * k];
}
__device__ __forceinline__ u128 space_time(const Plans &p, int k) {
  return (u128)(uint64_t)p.h[k] * (u128)(uint32_t)(p.te[k] - p.ts[k]);
}

// weighted_tmp_average([a, b]) with CPython float semantics (planner.py:118-121)
__device__ double weighted_avg2(const Plans &p, int a, int b) {
  u128 wa = space_time(p, a), wb = space_time(p, b);
  double s = __dadd_rn(__dmul_rn(p.tmp[a], u128_to_double_rne(wa)), __dmul_rn(p.tmp[b], u128_to_double_rne(wb)));
  return __ddiv_rn(s, u128_to_double_rne(wa + wb));
}

// block-wide compaction of one trace's plan members (in (t_s,id) order)
__device__ void gather_members(const FusionArgs &A, int64_t base, int64_t nt, int L, int S, int *nf, int *nr,
                               uint32_t *shu) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    *nf = 0;
    *nr = 0;
  }
  __syncthreads();
  for (int64_t c = 0; c < nt; c += blockDim.x) {
    int64_t j = c + tid;
    uint32_t i = j < nt ? A.rperm[base + j] : 0;
    int who = j < nt ? A.pid[i] : -1;
    uint32_t isL = who == L, isS = who == S;
    uint32_t tl, ts_;
    uint32_t pl = block_excl_sum<uint32_t>(isL, shu, &tl);
    uint32_t ps = block_excl_sum<uint32_t>(isS, shu, &ts_);
    int fbase = *nf, rbase = *nr;
    if (isL) {
      int64_t o = base + fbase + pl;
      A.fx_addr[o] = A.frel[i];
      A.fx_end[o] = A.frel[i] + A.e.size[i];
      A.fx_ts[o] = A.e.ts[i];
      A.fx_te[o] = A.e.te[i];
    }
    if (isS) {
      int64_t o = base + rbase + ps;
      A.rm_ev[o] = (int32_t)i;
      A.rm_gone[o] = 0;
    }
    __syncthreads();
    if (tid == 0) {
      *nf += (int)tl;
      *nr += (int)ts_;
    }
    __syncthreads();
  }
}

__global__ void k_fusion_prep(Plans p0, Plans p1, int64_t np, const int32_t *__restrict__ pid0,
                              int32_t *__restrict__ pid1, const int64_t *__restrict__ rel, int64_t *__restrict__ frel1,
                              int64_t ne, int32_t *__restrict__ lst, uint32_t *__restrict__ memo, int64_t nmemo) {
  GRID_STRIDE(i, max(max(np, ne), nmemo)) {
    if (i < np) {
      p1.grp[i] = p0.grp[i];
      p1.tr[i] = p0.tr[i];
      p1.h[i] = p0.h[i];
      p1.ts[i] = p0.ts[i];
      p1.te[i] = p0.te[i];
      p1.k0[i] = p0.k0[i];
      p1.k1[i] = p0.k1[i];
      p1.minq[i] = p0.minq[i];
      p1.used[2 * i] = p0.used[2 * i];
      p1.used[2 * i + 1] = p0.used[2 * i + 1];
      p1.tmp[i] = p0.tmp[i];
      p1.alive[i] = p0.alive[i];
      lst[i] = (int32_t)i;
    }
    if (i < ne) {
      pid1[i] = pid0[i];
      frel1[i] = rel[i];
    }
    if (i < nmemo) memo[i] = 0;
  }
}

constexpr int kFuseCap = 384;  // rectangles of one try staged in shared memory

__global__ void __launch_bounds__(kPlanThreads, 8) k_fusion(FusionArgs A, int T) {
  const int t = blockIdx.x;
  const int64_t p0 = A.pl_off[t];
  int P = (int)(A.pl_off[t + 1] - p0);
  if (A.attempts && threadIdx.x == 0) {
    A.attempts[t] = 0;
    A.accepted[t] = 0;
  }
  if (P <= 1) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  const int NW = blockDim.x >> 5;
  const int64_t base = A.ev_off[t], nt = A.ev_off[t + 1] - base;
  const int64_t P0 = P;
  const bool use_memo = A.memo_off[t + 1] > A.memo_off[t];
  __shared__ uint32_t shu[33];
  __shared__ long long shl[33];
  __shared__ int sh_nf, sh_nr, sh_pick, sh_first, sh_left, sh_okw[32];
  __shared__ long long sh_addr, sh_maxend;
  __shared__ long long s_fa[kFuseCap], s_fe[kFuseCap], s_csz[kFuseCap], s_new[kFuseCap];
  __shared__ int s_fts[kFuseCap], s_fte[kFuseCap], s_cts[kFuseCap], s_cte[kFuseCap];
  __shared__ uint8_t s_gone[kFuseCap];
  __shared__ long long sh_att, sh_acc;
  int32_t *lst = A.lst + p0;
  if (tid == 0) {
    sh_att = 0;
    sh_acc = 0;
  }
  __syncthreads();

  // Scan order of the reference's `for i: for j>i:` restart loop
  // (planner.py fusion): (ci, cj) is where the scan resumes -- after a
  // rejected try at (i, j+1), after an accepted one at (0, 1).
  __shared__ int sh_si, sh_sj;
  int ci = 0, cj = 1;
  while (true) {
    int i, jstar;
    if (P <= 32) {
      // one warp finds the next adjacent, not memo-rejected pair with ballots:
      // one barrier per try instead of two block reductions per row
      if (warp == 0) {
        int fi = -1, fj = -1;
        uint32_t natt = 0;
        for (int r = ci; r < P - 1; r++) {
          const int a = lst[r];
          const int j0 = r == ci ? cj : r + 1;
          const int jj = j0 + lane;
          bool adj = false, fresh = false;
          if (jj < P) {
            const int b = lst[jj];
            adj = A.p.k1[a] == A.p.k0[b] || A.p.k1[b] == A.p.k0[a];
            if (adj) {
              fresh = true;
              if (use_memo) {
                int x = min(a, b) - (int)p0, y = max(a, b) - (int)p0;
                int64_t bit = A.memo_off[t] + (int64_t)x * P0 + y;
                fresh = !((A.memo[bit >> 5] >> (bit & 31)) & 1u);
              }
            }
          }
          const uint32_t ma = __ballot_sync(0xffffffffu, adj);
          const uint32_t mf = __ballot_sync(0xffffffffu, adj && fresh);
          if (mf) {
            const int k = __ffs(mf) - 1;
            natt += __popc(ma & (0xffffffffu >> (31 - k)));  // attempts up to and incl. the pick
            fi = r;
            fj = j0 + k;
            break;
          }
          natt += __popc(ma);
        }
        if (lane == 0) {
          sh_si = fi;
          sh_sj = fj;
          sh_att += natt;
        }
      }
      __syncthreads();
      i = sh_si;
      jstar = sh_sj;
    } else {
      i = -1;
      jstar = -1;
      for (int r = ci; r < P - 1 && i < 0; r++) {
        const int a = lst[r];
        for (int j = r == ci ? cj : r + 1; j < P; j += blockDim.x) {
          // next adjacent (and not memo-rejected) partner in list order
          int jj = j + tid;
          bool adj = false, fresh = false;
          if (jj < P) {
            int b = lst[jj];
            adj = A.p.k1[a] == A.p.k0[b] || A.p.k1[b] == A.p.k0[a];
            if (adj) {
              fresh = true;
              if (use_memo) {
                int x = min(a, b) - (int)p0, y = max(a, b) - (int)p0;
                int64_t bit = A.memo_off[t] + (int64_t)x * P0 + y;
                fresh = !((A.memo[bit >> 5] >> (bit & 31)) & 1u);
              }
            }
          }
          int cand = (adj && fresh) ? jj : INT_MAX;
          int js = block_reduce_min(cand, (int *)shu);
          // attempts counted for every adjacent pair up to and including js
          uint32_t cnt_adj = (adj && jj <= js) ? 1u : 0u;
          uint32_t tot;
          block_excl_sum<uint32_t>(cnt_adj, shu, &tot);
          if (tid == 0) sh_att += tot;
          if (js != INT_MAX) {
            i = r;
            jstar = js;
            break;
          }
        }
      }
    }
    if (i < 0) break;
    {
      {
        const int a = lst[i];
        // ---- try_fuse(larger, smaller) --------------------------------------
        const int b = lst[jstar];
        const int L = A.p.h[a] >= A.p.h[b] ? a : b;
        const int S = L == a ? b : a;
        gather_members(A, base, nt, L, S, &sh_nf, &sh_nr, shu);
        const int nf0 = sh_nf, nr = sh_nr;
        long long amin = LLONG_MAX, emax = LLONG_MIN;
        for (int k = tid; k < nf0; k += blockDim.x) {
          amin = min(amin, (long long)A.fx_addr[base + k]);
          emax = max(emax, (long long)A.fx_end[base + k]);
        }
        amin = block_reduce_min(amin, shl);
        emax = block_reduce_max(emax, shl);
        if (tid == 0) {
          sh_addr = amin;
          sh_maxend = emax;
          sh_left = nr;
          sh_first = 0;
          sh_nf = nf0;
        }
        __syncthreads();
        if (nf0 + nr <= kFuseCap) {
          // Shared-memory cursor walk (every c4 try): the fixed rectangles and the
          // candidates' sizes / lifespans are staged once, so each placement step
          // is shared-memory loads and barriers instead of L2 round trips.
          for (int k = tid; k < nf0; k += blockDim.x) {
            s_fa[k] = A.fx_addr[base + k];
            s_fe[k] = A.fx_end[base + k];
            s_fts[k] = A.fx_ts[base + k];
            s_fte[k] = A.fx_te[base + k];
          }
          for (int k = tid; k < nr; k += blockDim.x) {
            const int ev = A.rm_ev[base + k];
            s_csz[k] = A.e.size[ev];
            s_cts[k] = A.e.ts[ev];
            s_cte[k] = A.e.te[ev];
            s_gone[k] = 0;
          }
          __syncthreads();
          while (sh_left > 0) {
            const long long addr = sh_addr;
            const int nf = sh_nf;
            if (tid == 0) sh_pick = -1;
            __syncthreads();
            for (int cb = sh_first; cb < nr; cb += NW) {
              const int k = cb + warp;
              bool ok = false;
              if (k < nr && !s_gone[k]) {
                const long long hi = addr + s_csz[k];
                const int ets = s_cts[k], ete = s_cte[k];
                bool conflict = false;
                for (int f = lane; f < nf && !conflict; f += 32)
                  conflict = s_fa[f] < hi && addr < s_fe[f] && s_fts[f] < ete && ets < s_fte[f];
                ok = !__any_sync(0xffffffffu, conflict);
              }
              if (lane == 0) sh_okw[warp] = ok ? k : INT_MAX;
              __syncthreads();
              if (tid == 0) {
                int mk = INT_MAX;
                for (int w = 0; w < NW; w++) mk = min(mk, sh_okw[w]);
                if (mk != INT_MAX) sh_pick = mk;
              }
              __syncthreads();
              if (sh_pick >= 0) break;
            }
            if (sh_pick >= 0) {
              if (tid == 0) {
                const int k = sh_pick;
                const long long sz = s_csz[k];
                s_gone[k] = 1;
                s_new[k] = addr;
                s_fa[nf] = addr;
                s_fe[nf] = addr + sz;
                s_fts[nf] = s_cts[k];
                s_fte[nf] = s_cte[k];
                sh_nf = nf + 1;
                if (addr + sz > sh_maxend) sh_maxend = addr + sz;
                sh_addr = addr + sz;
                sh_left--;
                int f = sh_first;
                while (f < nr && s_gone[f]) f++;
                sh_first = f;
              }
            } else {
              // next anchor strictly above the cursor, else the top of everything fixed
              long long nx = LLONG_MAX;
              for (int k = tid; k < nf0; k += blockDim.x) {
                const long long v = s_fa[k];
                if (v > addr && v < nx) nx = v;
              }
              nx = block_reduce_min(nx, shl);
              if (tid == 0) sh_addr = nx != LLONG_MAX ? nx : sh_maxend;
            }
            __syncthreads();
          }
          for (int k = tid; k < nr; k += blockDim.x) A.rm_new[base + k] = s_new[k];
          __syncthreads();
        }
        while (sh_left > 0) {  // large tries: the same walk over global scratch
          const long long addr = sh_addr;
          const int nf = sh_nf;
          if (tid == 0) sh_pick = -1;
          __syncthreads();
          for (int cb = sh_first; cb < nr; cb += NW) {
            int k = cb + warp;
            bool ok = false;
            if (k < nr && !A.rm_gone[base + k]) {
              int ev = A.rm_ev[base + k];
              long long hi = addr + A.e.size[ev];
              int ets = A.e.ts[ev], ete = A.e.te[ev];
              bool conflict = false;
              for (int f = lane; f < nf && !conflict; f += 32) {
                int64_t o = base + f;
                conflict = A.fx_addr[o] < hi && addr < A.fx_end[o] && A.fx_ts[o] < ete && ets < A.fx_te[o];
              }
              ok = !__any_sync(0xffffffffu, conflict);
            }
            if (lane == 0) sh_okw[warp] = ok ? k : INT_MAX;
            __syncthreads();
            if (tid == 0) {
              int m = INT_MAX;
              for (int w = 0; w < NW; w++) m = min(m, sh_okw[w]);
              if (m != INT_MAX) sh_pick = m;
            }
            __syncthreads();
            if (sh_pick >= 0) break;
          }
          if (sh_pick >= 0) {
            if (tid == 0) {
              int k = sh_pick;
              int ev = A.rm_ev[base + k];
              long long sz = A.e.size[ev];
              A.rm_gone[base + k] = 1;
              A.rm_new[base + k] = addr;
              int64_t o = base + sh_nf;
              A.fx_addr[o] = addr;
              A.fx_end[o] = addr + sz;
              A.fx_ts[o] = A.e.ts[ev];
              A.fx_te[o] = A.e.te[ev];
              sh_nf++;
              if (addr + sz > sh_maxend) sh_maxend = addr + sz;
              sh_addr = addr + sz;
              sh_left--;
              int f = sh_first;
              while (f < nr && A.rm_gone[base + f]) f++;
              sh_first = f;
            }
          } else {
            // next anchor strictly above the cursor, else the top of everything fixed
            long long nx = LLONG_MAX;
            for (int k = tid; k < nf0; k += blockDim.x) {
              long long v = A.fx_addr[base + k];
              if (v > addr && v < nx) nx = v;
            }
            nx = block_reduce_min(nx, shl);
            if (tid == 0) sh_addr = nx != LLONG_MAX ? nx : sh_maxend;
          }
          __syncthreads();
        }
        // fused plan statistics (_plan_from_decisions) and acceptance (try_fuse)
        const long long fh = sh_maxend;
        const int fts = min(A.p.ts[L], A.p.ts[S]), fte = max(A.p.te[L], A.p.te[S]);
        const u128 fused = plan_used(A.p, L) + plan_used(A.p, S);
        const double ftmp = exact_div(fused, (u128)(uint64_t)fh * (u128)(uint32_t)(fte - fts));
        const double avg = weighted_avg2(A.p, L, S);
        const bool accept = ftmp > avg;
        if (!accept) {
          if (tid == 0 && use_memo) {
            int x = min(a, b) - (int)p0, y = max(a, b) - (int)p0;
            int64_t bit = A.memo_off[t] + (int64_t)x * P0 + y;
            A.memo[bit >> 5] |= 1u << (bit & 31);
          }
          __syncthreads();
          ci = i;
          cj = jstar + 1;
          continue;
        }
        // commit: plans[i] = fused; del plans[j]
        const int si = a, sj = b;
        for (int k = tid; k < nr; k += blockDim.x) A.frel[A.rm_ev[base + k]] = A.rm_new[base + k];
        for (int64_t k = tid; k < nt; k += blockDim.x) {
          uint32_t ev = A.rperm[base + k];
          int w = A.pid[ev];
          if (w == si || w == sj) A.pid[ev] = si;
        }
        if (tid == 0) {
          int nk0 = (A.p.ts[L] <= A.p.ts[S] ? A.p.k0[L] : A.p.k0[S]);
          int nk1 = (A.p.te[L] >= A.p.te[S] ? A.p.k1[L] : A.p.k1[S]);
          int nminq = min(A.p.minq[L], A.p.minq[S]);
          A.acc_tmp[p0 + sh_acc] = ftmp;
          A.acc_avg[p0 + sh_acc] = avg;
          sh_acc++;
          A.p.h[si] = fh;
          A.p.ts[si] = fts;
          A.p.te[si] = fte;
          A.p.used[2 * si] = (unsigned long long)fused;
          A.p.used[2 * si + 1] = (unsigned long long)(fused >> 64);
          A.p.tmp[si] = ftmp;
          A.p.k0[si] = nk0;
          A.p.k1[si] = nk1;
          A.p.minq[si] = nminq;
          A.p.alive[sj] = 0;
        }
        // memo: forget every verdict involving the rewritten slot
        if (use_memo) {
          int x0 = si - (int)p0;
          for (int k = tid; k < P0; k += blockDim.x) {
            int x = min(x0, k), y = max(x0, k);
            int64_t bit = A.memo_off[t] + (int64_t)x * P0 + y;
            atomicAnd(A.memo + (bit >> 5), ~(1u << (bit & 31)));
          }
        }
        // delete list position jstar
        int moved[8];
        int nm = 0;
        for (int k = jstar + 1 + tid; k < P && nm < 8; k += blockDim.x) moved[nm++] = lst[k];
        __syncthreads();
        nm = 0;
        for (int k = jstar + 1 + tid; k < P && nm < 8; k += blockDim.x) lst[k - 1] = moved[nm++];
        __syncthreads();
        if (P - jstar - 1 > 8 * (int)blockDim.x) {  // long lists: serial tail shift
          if (tid == 0)
            for (int k = jstar + 1 + 8 * blockDim.x; k < P; k++) lst[k - 1] = lst[k];
          __syncthreads();
        }
        P -= 1;
        ci = 0;
        cj = 1;
      }
    }
  }
  if (tid == 0) {
    A.attempts[t] = sh_att;
    A.accepted[t] = sh_acc;
  }
}

// ---------------------------------------------------------------------------
// D: items per (variant, trace): final plans + residual events

struct Items {
  int64_t *size;
  int32_t *ts, *te, *tie, *ref;  // ref >= 0 plan id, < 0 ~event
};


// Phase D for segments too large for one CTA (e.g. a single 10^6-event trace).
// A segment's items are the variant's surviving plans in plan order
// (planner.py:408-411), then the trace's residual events -- scoped statics of
// single-phase groups -- in event order (planner.py:397-401, 412-417). All
// segments form one virtual sequence -- per variant v, per trace t: its plans,
// then its events -- whose selected entries are compacted by one global scan;
// the scan value at an entry is its item index (segments are in item order).
__device__ __forceinline__ bool item_virtual(int64_t x, int T, int64_t P, int64_t N, const int64_t *pl_off,
                                             const int64_t *ev_off, int *v, int *t, int64_t *src, bool *is_plan) {
  *v = (int)(x / (P + N));
  const int64_t y = x - (int64_t)*v * (P + N);  // position inside the variant: pl_off[t] + ev_off[t] + ...
  int lo = 0, hi = T;  // last t with pl_off[t] + ev_off[t] <= y
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pl_off[mid] + ev_off[mid] <= y)
      lo = mid;
    else
      hi = mid;
  }
  *t = lo;
  const int64_t r = y - pl_off[lo] - ev_off[lo], np = pl_off[lo + 1] - pl_off[lo];
  *is_plan = r < np;
  *src = *is_plan ? pl_off[lo] + r : ev_off[lo] + (r - np);
  return true;
}

__global__ void k_item_flags(Plans p0, Plans p1, int want0, int want1, const int64_t *__restrict__ pl_off, Ev e,
                             const int64_t *__restrict__ ev_off, const int32_t *__restrict__ gof, Groups g,
                             const int32_t *__restrict__ pid0, int T, int64_t P, int64_t N, uint32_t *__restrict__ f) {
  GRID_STRIDE(x, 2 * (P + N)) {
    int v, t;
    int64_t src;
    bool pl;
    item_virtual(x, T, P, N, pl_off, ev_off, &v, &t, &src, &pl);
    bool sel = false;
    if (v ? want1 : want0) {
      if (pl)
        sel = (v ? p1 : p0).alive[src];
      else
        sel = !e.dyn[src] && pid0[src] < 0 && g.cls[gof[src]] == 1;
    }
    f[x] = sel ? 1u : 0u;
  }
}

__global__ void k_item_scatter(Plans p0, Plans p1, const int64_t *__restrict__ pl_off, Ev e,
                               const int64_t *__restrict__ ev_off, int T, int64_t P, int64_t N,
                               const uint32_t *__restrict__ f, const uint32_t *__restrict__ pos, Items it) {
  GRID_STRIDE(x, 2 * (P + N)) {
    if (!f[x]) continue;
    int v, t;
    int64_t src;
    bool pl;
    item_virtual(x, T, P, N, pl_off, ev_off, &v, &t, &src, &pl);
    const int64_t o = pos[x];
    if (pl) {
      const Plans &pv = v ? p1 : p0;
      it.size[o] = pv.h[src];
      it.ts[o] = pv.ts[src];
      it.te[o] = pv.te[src];
      it.tie[o] = pv.minq[src];
      it.ref[o] = (int32_t)src;
    } else {
      it.size[o] = e.size[src];
      it.ts[o] = e.ts[src];
      it.te[o] = e.te[src];
      it.tie[o] = e.q[src];
      it.ref[o] = ~(int32_t)src;
    }
  }
}

// class ends for large segments: items are sorted by size descending inside
// their segment, so j's class ends at the first later item of smaller size
// (binary search; the segment from io by binary search)
__global__ void k_class_ends_bs(Items it, const int64_t *__restrict__ io, int VT, int64_t n,
                                int64_t *__restrict__ cend) {
  GRID_STRIDE(j, n) {
    int lo = 0, hi = VT;  // segment: last s with io[s] <= j
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (io[mid] <= j)
        lo = mid;
      else
        hi = mid;
    }
    while (io[lo + 1] <= j) lo++;  // skip empty segments
    const int64_t b = io[lo + 1];
    const int64_t sz = it.size[j];
    int64_t a = j + 1, z = b;  // first k in [j+1, b) with size < sz
    while (a < z) {
      const int64_t m = (a + z) >> 1;
      if (it.size[m] < sz)
        z = m;
      else
        a = m + 1;
    }
    cend[j] = a;
  }
}

// Phase D fused (segments of <= 4096 items, keys of <= 64 bits): one CTA per
// (variant, trace) gathers the segment's items (alive plans in plan order,
// then residual events in event order), sorts
// (size desc, t_s, tie) keys with their source refs in shared memory
// (cta_radix, stable) and writes the items in sorted order together with the
// plan/event -> item maps: the gather + k_item_keys + the segmented sort +
// k_item_permute in one pass over the data.
template <int IPT>
__global__ void __launch_bounds__(256, IPT == 8 ? 5 : 1) k_items_sorted(Plans p0, Plans p1, int want0, int want1,
                                                      const int64_t *__restrict__ pl_off, Ev e,
                                                      const int64_t *__restrict__ ev_off,
                                                      const int32_t *__restrict__ gof, Groups g,
                                                      const int32_t *__restrict__ pid0, const int64_t *__restrict__ io,
                                                      int T, int64_t P, int64_t N, Items it,
                                                      int32_t *__restrict__ item_of_plan,
                                                      int32_t *__restrict__ item_of_res, long long maxsu, int ashift,
                                                      long long align, int qb, int lobits, int in_order,
                                                      int64_t *__restrict__ cend) {
  constexpr int CAP = 256 * IPT;
  extern __shared__ __align__(16) unsigned char sis[];
  uint64_t *kA = (uint64_t *)sis;
  uint32_t *vA = (uint32_t *)(kA + CAP);
  uint32_t *wh = vA + CAP;
  __shared__ uint32_t sh[33];
  const int sgi = blockIdx.x, tid = threadIdx.x;
  const int v = sgi >= T, t = sgi - v * T;
  if (!(v ? want1 : want0)) return;
  const Plans &pv = v ? p1 : p0;
  auto key = [&](int64_t size, int ts, int tie) -> uint64_t {
    const long long su = ashift >= 0 ? (size >> ashift) : size / align;
    const uint64_t lo = in_order ? (uint64_t)(uint32_t)tie : ((uint64_t)(uint32_t)ts << qb) | (uint32_t)tie;
    return ((uint64_t)(maxsu - su) << lobits) | lo;
  };
  int pos = 0;
  for (int64_t k0 = pl_off[t]; k0 < pl_off[t + 1]; k0 += blockDim.x) {
    const int64_t k = k0 + tid;
    const bool alive = k < pl_off[t + 1] && pv.alive[k];
    uint32_t tot;
    const uint32_t ex = block_excl_sum<uint32_t>(alive ? 1u : 0u, sh, &tot);
    if (alive) {
      kA[pos + ex] = key(pv.h[k], pv.ts[k], pv.minq[k]);
      vA[pos + ex] = (uint32_t)k;
    }
    pos += tot;
  }
  // residual events: scoped static events of a single-phase group (class 1,
  // p_s == p_e: no cross-phase plan, so pid0 < 0) -- from the event's own
  // columns (coalesced) rather than the pid0 -> gof -> group-class gathers
  const int ehz = e.horizon[t];
  for (int64_t i0 = ev_off[t]; i0 < ev_off[t + 1]; i0 += blockDim.x) {
    const int64_t i = i0 + tid;
    const bool res = i < ev_off[t + 1] && ev_class(e.dyn[i], e.te[i], ehz) == 1 && e.ps[i] == e.pe[i];
    uint32_t tot;
    const uint32_t ex = block_excl_sum<uint32_t>(res ? 1u : 0u, sh, &tot);
    if (res) {
      kA[pos + ex] = key(e.size[i], e.ts[i], e.q[i]);
      vA[pos + ex] = (uint32_t)~(int32_t)i;
    }
    pos += tot;
  }
  __syncthreads();
  const int n = pos;
  cta_radix<IPT>(kA, vA, wh, sh, n, 0, lobits + bitlen_dev((u128)maxsu));
  const int64_t o0 = io[sgi];
  for (int j = tid; j < n; j += blockDim.x) {
    const int32_t r = (int32_t)vA[j];
    const int64_t o = o0 + j;
    if (r >= 0) {
      it.size[o] = pv.h[r];
      it.ts[o] = pv.ts[r];
      it.te[o] = pv.te[r];
      it.tie[o] = pv.minq[r];
      item_of_plan[(int64_t)v * P + r] = (int32_t)o;
    } else {
      const int64_t i = ~r;
      it.size[o] = e.size[i];
      it.ts[o] = e.ts[i];
      it.te[o] = e.te[i];
      it.tie[o] = e.q[i];
      item_of_res[(int64_t)v * N + i] = (int32_t)o;
    }
    it.ref[o] = r;
  }
  // class ends: cend[j] = the first class edge after j, an edge
  // being the segment's last item or a change of the key's size bits. Edges go
  // to vA (read above), then a suffix minimum: per-thread chunks + warp shuffles.
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x)
    vA[j] = (j + 1 == n || lobits >= 64 || (kA[j + 1] >> lobits) != (kA[j] >> lobits)) ? (uint32_t)(j + 1)
                                                                                       : 0xffffffffu;
  __syncthreads();
  const int per = (n + 255) >> 8, c0 = min(n, tid * per), c1 = min(n, c0 + per);
  uint32_t agg = 0xffffffffu;
  for (int j = c0; j < c1; j++) agg = min(agg, vA[j]);
  const int w = tid >> 5, lane = tid & 31;
  uint32_t x = agg;  // inclusive suffix minimum over the warp's lanes
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, x, d);
    if (lane + d < 32) x = min(x, y);
  }
  uint32_t later = __shfl_down_sync(0xffffffffu, x, 1);
  if (lane == 31) later = 0xffffffffu;
  __shared__ uint32_t wmin[8];
  if (lane == 0) wmin[w] = x;
  __syncthreads();
  for (int w2 = w + 1; w2 < 8; w2++) later = min(later, wmin[w2]);
  for (int j = c1 - 1; j >= c0; j--) {
    later = min(later, vA[j]);
    cend[o0 + j] = o0 + later;
  }
}

// in_order: every trace is listed in recorded order, so q (the id rank) is the
// position and t_s never decreases along it. An item's (t_s, tie) is then the
// (t_s, q) of one event -- its own, or a plan's earliest member (whose t_s is
// the plan's min t_s and whose q is its min q, fused plans included) -- and
// (t_s, tie) order is tie order: the low key is tie alone.
__global__ void k_item_keys(Items it, int64_t n, const int64_t *__restrict__ io, int VT, int qb, long long align,
                            long long maxsu, int sb, int in_order, uint64_t *__restrict__ hi,
                            uint64_t *__restrict__ lo) {
  GRID_STRIDE(j, n) {
    int vt = 0;
    {  // segment of j in io[0..VT]
      int a = 0, b = VT;
      while (b - a > 1) {
        int m = (a + b) >> 1;
        if (io[m] <= j)
          a = m;
        else
          b = m;
      }
      vt = a;
    }
    long long su = it.size[j] / align;
    hi[j] = ((uint64_t)vt << sb) | (uint64_t)(maxsu - su);
    lo[j] = in_order ? (uint64_t)(uint32_t)it.tie[j] : ((uint64_t)(uint32_t)it.ts[j] << qb) | (uint32_t)it.tie[j];
  }
}

// gather items into sorted order; item_of_* map plans/residuals of variant v
// (items of variant 0 precede those of variant 1) to sorted positions
__global__ void k_item_permute(Items src, Items dst, const uint32_t *__restrict__ perm, int64_t n,
                               const int64_t *__restrict__ io, int T, int64_t P, int64_t N,
                               int32_t *__restrict__ item_of_plan, int32_t *__restrict__ item_of_res) {
  GRID_STRIDE(j, n) {
    uint32_t s = perm[j];
    dst.size[j] = src.size[s];
    dst.ts[j] = src.ts[s];
    dst.te[j] = src.te[s];
    dst.tie[j] = src.tie[s];
    int r = src.ref[s];
    dst.ref[j] = r;
    int v = j >= io[T] ? 1 : 0;
    if (r >= 0)
      item_of_plan[(int64_t)v * P + r] = (int32_t)j;
    else
      item_of_res[(int64_t)v * N + ~r] = (int32_t)j;
  }
}


// ---------------------------------------------------------------------------
// E: HomoSize layers, one CTA per unit (planner.py:189-254, 414-439)

struct LayerArgs {
  int C, T;
  const uint8_t *cand;
  const int32_t *var_of;
  const int64_t *io;  // [V*T+1]
  const int64_t *uo;  // [U+1] unit scratch offsets
  Items it;
  const int64_t *cend;
  const int64_t *pers_size;
  const int32_t *horizon;                  // [T]
  int32_t *sA_ts, *sA_te, *sB_ts, *sB_te;  // [total]
  int32_t *loffA, *loffB;                  // [total + U]
  int32_t *prioA, *prioB, *lastEnd, *nend, *newcnt, *runoff, *run_ts, *run_te;
  uint32_t *fitw;  // [total * kFitWords]
  int32_t *ilayer, *irank;
  int64_t *lsize, *lbase;
  int32_t *nlayers;
  int64_t *gapins, *pool;
};

// fits_gap of item [ts, te] against layer slots [lo, hi) of buffer (sts, ste)
__device__ __forceinline__ bool slot_fit(const int32_t *__restrict__ sts, const int32_t *__restrict__ ste, int lo,
                                         int hi, int ts, int te) {
  int a = lo, b = hi;  // first slot with start > te
  while (a < b) {
    int m = (a + b) >> 1;
    if (sts[m] <= te)
      a = m + 1;
    else
      b = m;
  }
  return a == lo || ste[a - 1] < ts;
}

__device__ __forceinline__ int lower_bound_i32(const int32_t *__restrict__ v, int lo, int hi, int x) {
  while (lo < hi) {
    int m = (lo + hi) >> 1;
    if (v[m] < x)
      lo = m + 1;
    else
      hi = m;
  }
  return lo;
}

// block exclusive scan of f(l) for l in [0, n) into out[0..n], out[n] = total
template <class F>
__device__ void block_scan_into(int n, F f, int32_t *out, int *shi) {
  int carry = 0;
  for (int c = 0; c < n; c += blockDim.x) {
    int l = c + threadIdx.x;
    int v = l < n ? f(l) : 0;
    int tot;
    int ex = block_excl_sum<int>(v, shi, &tot);
    if (l < n) out[l] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
  __syncthreads();
}

__device__ void layers_unit(const LayerArgs &A, const int u);
#ifdef STW_LAYERS_CLOCK
__device__ unsigned long long g_layers_clk[8];
__device__ unsigned long long g_class_clk[64][3];  // per class of the big unit: cycles, items, nl
#define LCLK(i) if (threadIdx.x == 0) { long long _n = clock64(); atomicAdd(&g_layers_clk[i], (unsigned long long)(_n - _lc)); _lc = _n; }
#else
#define LCLK(i)
#endif

// ulist[0 .. *ucount) (or [0, gridDim.x) without a count), grid-stride
__global__ void __launch_bounds__(kPlanThreads) k_layers(LayerArgs A, const int32_t *__restrict__ ulist,
                                                         const int *__restrict__ ucount) {
  const int n = ucount ? *ucount : (int)gridDim.x;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    layers_unit(A, ulist[i]);
    __syncthreads();
  }
}

// Step 2 of a class (planner.py:414-439): the warp-serial resolve -- gap
// insertion (the lowest fitting priority whose same-class last end is before
// t_s), else Alg. 1 among this class's new layers. Run by a whole CTA (warp 0
// works). Writes ilayer / irank / newcnt, *out_nnew and adds to *out_gap
// (shared variables of the calling CTA).
__device__ void resolve_class(const LayerArgs &A, const bool gap, const int nl, const int64_t j0, const int64_t j1,
                              const int64_t a0, const int64_t off, const uint32_t *__restrict__ fitw,
                              const int32_t *__restrict__ prioA, const int32_t *__restrict__ sAts,
                              const int32_t *__restrict__ sAte, const int32_t *__restrict__ loffA, int32_t *last,
                              int32_t *newcnt, int32_t *ilayer, int32_t *irank, int32_t *sm_nend, int *out_nnew,
                              long long *out_gap, const int hz) {
  const int warp = threadIdx.x >> 5, lane = lane_id();
  // ---- 2. warp-serial resolve: gap insertion, else Alg. 1 among this class's new layers.
  // Narrow case (<= 32 layers): the register-resident chain of k_layers_w32;
  // if the class would open a 33rd layer it is redone by the general loop.
  __shared__ int sh_cnt[32], sh_fast;
  if (warp == 0) {
    constexpr unsigned FULL = 0xffffffffu;
    bool fast = nl <= 32;
    int nnew = 0, gapc = 0;
    if (fast) {
      int lastp = INT_MIN, ne = INT_MIN;
      sh_cnt[lane] = 0;
      __syncwarp();
      const int my_prio = lane < nl ? prioA[lane] : 0;  // lane p: the layer at priority p
      // Alg. 1 keys pack (end << 5 | 31 - lane) when every end is in [0, 2^26)
      const bool packed = hz < (1 << 26);  // ends are <= horizon
      // each chunk's item fields are loaded one chunk ahead (the chain never waits on global memory)
      int nx_ts = 0, nx_te = 0;
      unsigned nx_fm = 0;
      if (j0 + lane < j1) {
        nx_ts = A.it.ts[j0 + lane];
        nx_te = A.it.te[j0 + lane];
        if (gap && nl > 0) nx_fm = fitw[(j0 + lane - a0) * kFitWords];
      }
      for (int64_t cb = j0; cb < j1 && fast; cb += 32) {
        const int64_t mine = cb + lane;
        const int cnt = (int)min((int64_t)32, j1 - cb);
        const int my_ts = nx_ts, my_te = nx_te;
        const unsigned fm = nx_fm;
        if (mine + 32 < j1) {
          nx_ts = A.it.ts[mine + 32];
          nx_te = A.it.te[mine + 32];
          if (gap && nl > 0) nx_fm = fitw[(mine + 32 - a0) * kFitWords];
        }
        int my_code = 0;
#ifdef STW_LAYERS_CLOCK
        long long _c0 = clock64();
#endif
        // Hot loop: consecutive gap-hosted items, one vote each (lane p:
        // priority p). The host lane tests (m1 & lanemask_le) == lanemask_eq;
        // the raw vote is kept by lane k and decoded (ffs) after the chunk, so
        // nothing variable-latency sits on the per-item chain. The next item's
        // fields are broadcast one item ahead. An item no layer hosts leaves
        // the loop for Alg. 1 (a max-reduction over the class's new layers).
        const unsigned lm_eq = 1u << lane, lm_le = lm_eq | (lm_eq - 1u);
        unsigned my_m1 = 0;  // lane k: item k's vote (0: Alg. 1, code in my_code)
        int k = 0;
        int ts = __shfl_sync(FULL, my_ts, 0), te = __shfl_sync(FULL, my_te, 0);
        unsigned f = __shfl_sync(FULL, fm, 0);
        while (k < cnt) {
          if (gap && nl > 0) {
            for (; k < cnt; k++) {
              const int k1 = (k + 1) & 31;
              const int nts = __shfl_sync(FULL, my_ts, k1), nte = __shfl_sync(FULL, my_te, k1);
              const unsigned nf = __shfl_sync(FULL, fm, k1);
              const unsigned m1 = __ballot_sync(FULL, (f & lm_eq) && lastp < ts);
              if (!m1) break;
              lastp = (m1 & lm_le) == lm_eq ? te : lastp;
              my_m1 = lane == k ? m1 : my_m1;
              ts = nts, te = nte, f = nf;
            }
            if (k >= cnt) break;
          }
          // Alg. 1 for item k (planner.py:236-254): the largest end < t_s among
          // the class's new layers, ties to the oldest -- one max-reduction over
          // (end << 5 | 31 - lane) keys when ends fit 26 bits; none: a new layer
          int best;
          bool found;
          if (packed) {
            const int key = __reduce_max_sync(
                FULL, lane < nnew && ne < ts ? (int)(((unsigned)ne << 5) | (unsigned)(31 - lane)) : -1);
            found = key >= 0;
            best = found ? 31 - (key & 31) : nnew;
          } else {
            const bool ca = lane < nnew && ne < ts;
            const int mx = __reduce_max_sync(FULL, ca ? ne : INT_MIN);
            const unsigned cma = __ballot_sync(FULL, ca && ne == mx);
            found = cma != 0;
            best = found ? __ffs(cma) - 1 : nnew;
          }
          if (!found && nl + nnew == 32) {
            fast = false;
            break;
          }
          if (lane == best) ne = te;
          nnew += found ? 0 : 1;
          if (lane == k) my_m1 = 0, my_code = 32 + best;
          k++;
          const int kk = k & 31;
          ts = __shfl_sync(FULL, my_ts, kk), te = __shfl_sync(FULL, my_te, kk);
          f = __shfl_sync(FULL, fm, kk);
        }
        if (my_m1) my_code = __ffs(my_m1) - 1;
#ifdef STW_LAYERS_CLOCK
        if (lane == 0) atomicAdd(&g_layers_clk[3], (unsigned long long)(clock64() - _c0)), atomicAdd(&g_layers_clk[5], (unsigned long long)cnt);
#endif
        if (!fast) break;
        const bool act = lane < cnt;
        const int hp = __shfl_sync(FULL, my_prio, my_code & 31);  // layer of priority my_code (gap host)
        const int layer = my_code < 32 ? hp : nl + (my_code - 32);
        gapc += __popc(__ballot_sync(FULL, act && my_code < 32));
        const unsigned peers = __match_any_sync(FULL, act ? layer : -1 - lane);
        const int r = __popc(peers & lanemask_lt());
        const int base = act ? sh_cnt[layer] : 0;
        __syncwarp();
        if (act) {
          ilayer[mine - a0] = layer;
          irank[mine - a0] = base + r;
          if (r == __popc(peers) - 1) sh_cnt[layer] = base + __popc(peers);
        }
        __syncwarp();
      }
      if (fast) {
        for (int l = lane; l < nl + nnew; l += 32) newcnt[l] = sh_cnt[l];
        if (lane == 0) {
          *out_nnew = nnew;
          *out_gap += gapc;
        }
      } else {  // restart the class on the general path
        nnew = 0;
        for (int p = lane; p < nl; p += 32) last[p] = INT_MIN;
        for (int l = lane; l < nl; l += 32) newcnt[l] = 0;
        __syncwarp();
      }
    }
    if (lane == 0) sh_fast = fast;
  }
  __syncthreads();
  if (!sh_fast && warp == 0) {
    int nnew = 0;
    long long gapc = 0;
    int32_t *nend = A.nend + off;  // spill path when a class opens > kSmemLayers layers
    for (int64_t cb = j0; cb < j1; cb += 32) {
      int64_t mine = cb + lane;
      int my_ts = 0, my_te = 0;
      uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
      if (mine < j1) {
        my_ts = A.it.ts[mine];
        my_te = A.it.te[mine];
        if (gap && nl > 0) {
          const uint32_t *f = fitw + (mine - a0) * kFitWords;
          w0 = f[0];
          w1 = f[1];
          w2 = f[2];
          w3 = f[3];
        }
      }
      const int cnt = (int)min((int64_t)32, j1 - cb);
      for (int k = 0; k < cnt; k++) {
        const int ts = __shfl_sync(0xffffffffu, my_ts, k), te = __shfl_sync(0xffffffffu, my_te, k);
        const uint32_t f0 = __shfl_sync(0xffffffffu, w0, k), f1 = __shfl_sync(0xffffffffu, w1, k),
                       f2 = __shfl_sync(0xffffffffu, w2, k), f3 = __shfl_sync(0xffffffffu, w3, k);
        const int64_t jj = cb + k;
        int host_p = -1;
        if (gap) {
          for (int pb = 0; pb < nl && host_p < 0; pb += 32) {
            int p = pb + lane;
            bool ok = false;
            if (p < nl) {
              bool fit;
              if (p < 32 * kFitWords) {
                uint32_t w = pb == 0 ? f0 : pb == 32 ? f1 : pb == 64 ? f2 : f3;
                fit = (w >> lane) & 1u;
              } else {
                int l = prioA[p];
                fit = slot_fit(sAts, sAte, loffA[l], loffA[l + 1], ts, te);
              }
              ok = fit && last[p] < ts;
            }
            unsigned msk = __ballot_sync(0xffffffffu, ok);
            if (msk) host_p = pb + __ffs(msk) - 1;
          }
        }
        int layer;
        if (host_p >= 0) {
          layer = prioA[host_p];
          if (lane == 0) last[host_p] = te;
          gapc++;
        } else {
          int32_t *ne = nnew <= kSmemLayers ? sm_nend : nend;
          int best_k = -1, best_e = INT_MIN;
          for (int kb = 0; kb < nnew; kb += 32) {
            int kk = kb + lane;
            int e = kk < nnew ? ne[kk] : INT_MIN;
            bool cand = kk < nnew && e < ts;
            int mx = __reduce_max_sync(0xffffffffu, cand ? e : INT_MIN);
            unsigned cm = __ballot_sync(0xffffffffu, cand && e == mx);
            if (cm && (best_k < 0 || mx > best_e)) {
              best_e = mx;
              best_k = kb + __ffs(cm) - 1;
            }
          }
          if (best_k < 0) {
            best_k = nnew++;
            if (nnew == kSmemLayers + 1) {  // spill the new-layer ends to global memory
              for (int x = lane; x < kSmemLayers; x += 32) nend[x] = sm_nend[x];
              __syncwarp();
            }
            if (lane == 0) newcnt[nl + best_k] = 0;
          }
          int32_t *ne2 = nnew <= kSmemLayers ? sm_nend : nend;
          if (lane == 0) ne2[best_k] = te;
          layer = nl + best_k;
        }
        if (lane == 0) {
          ilayer[jj - a0] = layer;
          irank[jj - a0] = newcnt[layer]++;
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      *out_nnew = nnew;
      *out_gap += gapc;
    }
  }
  __syncthreads();

}

__device__ void layers_unit(const LayerArgs &A, const int u) {
  const int c = u % A.C, t = u / A.C;
  const int v = A.var_of[c];
  const bool gap = (A.cand[c] & STW_CAND_GAP) != 0;
  const int64_t a0 = A.io[(int64_t)v * A.T + t], a1 = A.io[(int64_t)v * A.T + t + 1];
  const int64_t off = A.uo[u];
  const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  __shared__ int shi[33];
  __shared__ int sm_last[kSmemLayers], sm_nend[kSmemLayers];
  __shared__ int sh_nl, sh_nnew;
  __shared__ long long sh_gap;

  int32_t *sAts = A.sA_ts + off, *sAte = A.sA_te + off, *sBts = A.sB_ts + off, *sBte = A.sB_te + off;
  int32_t *loffA = A.loffA + off + u, *loffB = A.loffB + off + u;
  int32_t *prioA = A.prioA + off, *prioB = A.prioB + off;
  int32_t *newcnt = A.newcnt + off, *runoff = A.runoff + off + u;
  int32_t *run_ts = A.run_ts + off, *run_te = A.run_te + off;
  int32_t *ilayer = A.ilayer + off, *irank = A.irank + off;
  uint32_t *fitw = A.fitw + off * kFitWords;
  int64_t *lsize = A.lsize + off;
  if (tid == 0) {
    sh_nl = 0;
    sh_gap = 0;
    loffA[0] = 0;
  }
  __syncthreads();

#ifdef STW_LAYERS_CLOCK
  long long _lc = clock64();
  if (threadIdx.x == 0) atomicAdd(&g_layers_clk[7], 1ull);
#endif
  for (int64_t j0 = a0; j0 < a1;) {
    const int64_t j1 = A.cend[j0];
    const int m = (int)(j1 - j0);
    const int64_t S = A.it.size[j0];
#ifdef STW_LAYERS_CLOCK
    if (threadIdx.x == 0) atomicAdd(&g_layers_clk[6], 1ull);
#endif
    const int nl = sh_nl;
    const int nfit = min(nl, 32 * kFitWords);
    int32_t *last = nl <= kSmemLayers ? sm_last : A.lastEnd + off;
    // ---- 1. fit masks against the slots of earlier classes
    if (gap && nl > 0) {
      for (int x = tid; x < m * kFitWords; x += blockDim.x) fitw[(j0 - a0) * kFitWords + x] = 0;
      for (int p = tid; p < nl; p += blockDim.x) last[p] = INT_MIN;
      __syncthreads();
      for (int64_t x = tid; x < (int64_t)m * nfit; x += blockDim.x) {
        int jj = (int)(x / nfit), p = (int)(x % nfit);
        int64_t it = j0 + jj;
        int l = prioA[p];
        if (slot_fit(sAts, sAte, loffA[l], loffA[l + 1], A.it.ts[it], A.it.te[it]))
          atomicOr(fitw + (it - a0) * kFitWords + (p >> 5), 1u << (p & 31));
      }
    }
    for (int l = tid; l < nl; l += blockDim.x) newcnt[l] = 0;
    __syncthreads();
    LCLK(0)
    // ---- 2. warp-serial resolve (resolve_class)
    resolve_class(A, gap, nl, j0, j1, a0, off, fitw, prioA, sAts, sAte, loffA, last, newcnt, ilayer, irank, sm_nend,
                  &sh_nnew, &sh_gap, A.horizon[t]);
    LCLK(1)
    // ---- 3. merge this class's slots into the per-layer sorted slot CSR
    const int nnew = sh_nnew, nl2 = nl + nnew;
    for (int x = tid; x < nnew; x += blockDim.x) lsize[nl + x] = S;
    block_scan_into(nl2, [&](int l) { return (l < nl ? loffA[l + 1] - loffA[l] : 0) + newcnt[l]; }, loffB, shi);
    block_scan_into(nl2, [&](int l) { return newcnt[l]; }, runoff, shi);
    for (int x = tid; x < m; x += blockDim.x) {
      int l = ilayer[j0 - a0 + x];
      int pos = runoff[l] + irank[j0 - a0 + x];
      run_ts[pos] = A.it.ts[j0 + x];
      run_te[pos] = A.it.te[j0 + x];
    }
    __syncthreads();
    const int nold = nl > 0 ? loffA[nl] : 0;
    for (int s = tid; s < nold; s += blockDim.x) {
      int a = 0, b = nl;  // layer of slot s
      while (b - a > 1) {
        int mid = (a + b) >> 1;
        if (loffA[mid] <= s)
          a = mid;
        else
          b = mid;
      }
      int l = a;
      while (loffA[l + 1] <= s) l++;  // skip empty layers
      int ts = sAts[s];
      int k = newcnt[l] ? lower_bound_i32(run_ts, runoff[l], runoff[l] + newcnt[l], ts) - runoff[l] : 0;
      int dst = loffB[l] + (s - loffA[l]) + k;
      sBts[dst] = ts;
      sBte[dst] = sAte[s];
    }
    for (int x = tid; x < m; x += blockDim.x) {
      int l = ilayer[j0 - a0 + x];
      int ts = A.it.ts[j0 + x];
      int k = l < nl ? lower_bound_i32(sAts, loffA[l], loffA[l + 1], ts) - loffA[l] : 0;
      int dst = loffB[l] + irank[j0 - a0 + x] + k;
      sBts[dst] = ts;
      sBte[dst] = A.it.te[j0 + x];
    }
    // priority order for later classes: newest (smallest) layers first, creation order within
    for (int x = tid; x < nl2; x += blockDim.x) prioB[x] = x < nnew ? nl + x : prioA[x - nnew];
    __syncthreads();
    {
      int32_t *tp;
      tp = sAts, sAts = sBts, sBts = tp;
      tp = sAte, sAte = sBte, sBte = tp;
      tp = loffA, loffA = loffB, loffB = tp;
      tp = prioA, prioA = prioB, prioB = tp;
    }
    if (tid == 0) sh_nl = nl2;
    __syncthreads();
    LCLK(2)
    j0 = j1;
  }
  // ---- F: stacking (planner.py:441-444)
  const int nl = sh_nl;
  int64_t *lbase = A.lbase + off;
  long long carry = A.pers_size[t];
  for (int c0 = 0; c0 < nl; c0 += blockDim.x) {
    int l = c0 + tid;
    long long v0 = l < nl ? lsize[l] : 0;
    __shared__ long long shl[33];
    long long tot;
    long long ex = block_excl_sum<long long>(v0, shl, &tot);
    if (l < nl) lbase[l] = carry + ex;
    carry += tot;
  }
  if (tid == 0) {
    A.nlayers[u] = nl;
    A.gapins[u] = sh_gap;
    A.pool[u] = carry;
  }
}


// ---------------------------------------------------------------------------
// E for the largest units (e.g. c5's single 10^6-item trace): one unit spread
// over the whole GPU. A cooperative launch walks the unit's classes; per class
// the fit masks (a binary search of each item in every earlier layer's sorted
// slots) and the slot merge run on every SM, the serial resolve on one warp,
// with grid-wide barriers between the steps (the single-CTA k_layers spent
// 40% of c5's time in those two data-parallel steps on one SM).
// Gap insertion of one class, per layer, on the whole GPU. For the layer at
// priority p the greedy (planner.py:420-431: each item takes the first fitting
// layer in priority order whose same-class slots all end before its start) is
// a chain over the class's items in (t_s, tie) order: the candidates are the
// items that fit layer p and no higher-priority layer took; the layer takes
// the first candidate, then the first candidate starting after that item's
// end, and so on -- so layer p's members are the chain head -> nx -> nx ...
// with nx(i) = the first candidate at or after the first position whose t_s
// exceeds t_e(i) (t_s is sorted, so a binary search). Layers are processed in
// priority order (layer p's candidates exclude what layers < p took).
// Per layer: (A) per 4096-item block a suffix-min of candidate positions,
// (B) nx of every candidate, (C) per block each candidate's exit from the
// block by pointer jumping in shared memory, (D) one thread walks the chain
// over block entries (exits), (E) per block one thread walks the members
// from the block's entry, recording their rank. Items no layer takes go
// through Alg. 1 afterwards (few: c5 has 54 of 983,279).
constexpr int kChainB = 4096;
constexpr int kChainMaxL = 32;

struct ChainScratch {
  int32_t *ipri;    // [n] priority that took the item, -1: none yet
  int32_t *nxl;     // [n] first candidate at or after x inside x's block (m: none)
  int32_t *nx;      // [n] chain successor of a candidate (m: none)
  int32_t *ex;      // [n] first chain node after x outside x's block (m: none)
  int32_t *lrank;   // [n] rank of a member among its layer's members in its block
  int32_t *bfirst;  // [nb] first candidate of the block (m: none)
  int32_t *bsfx;    // [nb + 1] first candidate at or after the block
  int32_t *bent;    // [nb] the chain's first node in the block (-1: none)
  int32_t *bcnt;    // [nb * kChainMaxL] members of priority p in block b, then their exclusive prefix
};

struct BigState {
  int nl, nnew;
  long long gap;
  int use_chain, over;
  ChainScratch cs;
};

// thread t of a 256-thread CTA: minimum of v over threads > t (`none` if none); *total = minimum over all
__device__ __forceinline__ int block_suffix_min_excl(int v, int none, int *sh, int *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;  // suffix (inclusive) inside the warp
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_down_sync(0xffffffffu, inc, o);
    if (lane + o < 32) inc = min(inc, y);
  }
  if (lane == 0) sh[w] = inc;
  __syncthreads();
  int after = none;  // warps after w
  for (int x = w + 1; x < (int)(blockDim.x >> 5); x++) after = min(after, sh[x]);
  int ex = __shfl_down_sync(0xffffffffu, inc, 1);
  if (lane == 31) ex = none;
  ex = min(ex, after);
  if (total) {
    int t = none;
    for (int x = 0; x < (int)(blockDim.x >> 5); x++) t = min(t, sh[x]);
    *total = t;
  }
  __syncthreads();
  return ex;
}

__device__ __forceinline__ int chain_nxc(const ChainScratch &cs, int y, int m) {
  if (y >= m) return m;
  const int v = cs.nxl[y];
  return v < m ? v : cs.bsfx[y / kChainB + 1];
}

// returns false when the class must be redone by resolve_class (Alg. 1 would
// need more than 32 layers in all); on success ilayer / irank / newcnt are
// written for every item of the class, *nnew_out = new layers, *gap_out += gapped
__device__ bool chain_class(const LayerArgs &A, const ChainScratch &cs, const int nl, const int64_t j0,
                            const int64_t j1, const int64_t a0, const uint32_t *__restrict__ fitw,
                            const int32_t *__restrict__ prioA, int32_t *newcnt, int32_t *ilayer, int32_t *irank,
                            int *sh_flag, int *sh_nnew, long long *sh_gap, const bool lead, const int hz,
                            cooperative_groups::grid_group &grid) {
  constexpr unsigned FULL = 0xffffffffu;
  const int m = (int)(j1 - j0);
  const int nb = (m + kChainB - 1) / kChainB;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + tid, gs = (int64_t)gridDim.x * blockDim.x;
  const int32_t *ts = A.it.ts + j0, *te = A.it.te + j0;
  const uint32_t *fw = fitw + (j0 - a0) * kFitWords;
  __shared__ int s_J[kChainB];
  __shared__ int s_sh[33];
  for (int64_t x = gt; x < m; x += gs) cs.ipri[x] = -1;
  grid.sync();
  for (int p = 0; p < nl; p++) {
    // (A) per block: suffix-min of candidate positions; the block's first candidate
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
      const int base = b * kChainB, cnt = min(kChainB, m - base);
      constexpr int IPT = kChainB / kPlanThreads;
      int v[IPT];
      int tmin = m;
#pragma unroll
      for (int k = IPT - 1; k >= 0; k--) {
        const int x = base + tid * IPT + k;
        const bool c = tid * IPT + k < cnt && ((fw[(int64_t)x * kFitWords + (p >> 5)] >> (p & 31)) & 1u) &&
                       cs.ipri[x] < 0;
        tmin = c ? x : tmin;
        v[k] = tmin;
      }
      int tot;
      const int after = block_suffix_min_excl(tmin, m, s_sh, &tot);
#pragma unroll
      for (int k = 0; k < IPT; k++) {
        const int x = base + tid * IPT + k;
        if (tid * IPT + k < cnt) cs.nxl[x] = min(v[k], after);
      }
      if (tid == 0) {
        cs.bfirst[b] = tot;
        cs.bent[b] = -1;
      }
    }
    grid.sync();
    if (lead && tid == 0) {  // suffix over the blocks
      int r = m;
      cs.bsfx[nb] = m;
      for (int b = nb - 1; b >= 0; b--) r = min(r, cs.bfirst[b]), cs.bsfx[b] = r;
    }
    grid.sync();
    // (B) chain successors of the candidates
    for (int64_t x = gt; x < m; x += gs) {
      if (cs.nxl[x] != (int)x) continue;  // not a candidate
      const int e = te[x];
      int lo = (int)x + 1, hi = m;  // first position with t_s > t_e(x) (> x: t_s(x) <= t_e(x))
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ts[mid] <= e)
          lo = mid + 1;
        else
          hi = mid;
      }
      cs.nx[x] = chain_nxc(cs, lo, m);
    }
    grid.sync();
    // (C) per block: each candidate's first chain node outside the block (pointer jumping)
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
      const int base = b * kChainB, cnt = min(kChainB, m - base);
      for (int i = tid; i < cnt; i += blockDim.x) s_J[i] = cs.nxl[base + i] == base + i ? cs.nx[base + i] : m;
      __syncthreads();
      for (int round = 0; round < 14; round++) {  // every round reads, then (after a barrier) writes
        constexpr int IPT = kChainB / kPlanThreads;
        int nv[IPT];
        bool moved = false;
#pragma unroll
        for (int k = 0; k < IPT; k++) {
          const int i = tid + k * kPlanThreads;
          nv[k] = m;
          if (i < cnt) {
            const int j = s_J[i];
            nv[k] = j < base + cnt ? s_J[j - base] : j;  // inside the block: jump
            moved |= j < base + cnt;
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < IPT; k++) {
          const int i = tid + k * kPlanThreads;
          if (i < cnt) s_J[i] = nv[k];
        }
        if (!__syncthreads_or(moved)) break;
      }
      for (int i = tid; i < cnt; i += blockDim.x)
        if (cs.nxl[base + i] == base + i) cs.ex[base + i] = s_J[i];
      __syncthreads();
    }
    grid.sync();
    // (D) the chain's entry into every block it visits
    if (lead && tid == 0) {
      for (int e = chain_nxc(cs, 0, m); e < m; e = cs.ex[e]) cs.bent[e / kChainB] = e;
    }
    grid.sync();
    // (E) per block: the members from the entry, their ranks, the block's count
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
      const int base = b * kChainB, cnt = min(kChainB, m - base);
      const int ent = cs.bent[b];
      if (ent >= 0) {
        for (int i = tid; i < cnt; i += blockDim.x) s_J[i] = cs.nx[base + i];  // only members are read
        __syncthreads();
        if (tid == 0) {
          int r = 0;
          for (int x = ent; x < base + cnt; x = s_J[x - base]) {
            cs.ipri[x] = p;
            cs.lrank[x] = r++;
          }
          cs.bcnt[b * kChainMaxL + p] = r;
        }
        __syncthreads();
      } else if (tid == 0) {
        cs.bcnt[b * kChainMaxL + p] = 0;
      }
    }
    grid.sync();
  }
  // member ranks: prefix of each priority's block counts; the layers' counts
  __shared__ unsigned long long s_gapped;
  if (lead) {
    if (tid == 0) s_gapped = 0;
    __syncthreads();
    for (int p = tid; p < nl; p += blockDim.x) {
      int r = 0;
      for (int b = 0; b < nb; b++) {
        const int c = cs.bcnt[b * kChainMaxL + p];
        cs.bcnt[b * kChainMaxL + p] = r;
        r += c;
      }
      newcnt[prioA[p]] = r;
      atomicAdd(&s_gapped, (unsigned long long)r);
    }
  }
  grid.sync();
  for (int64_t x = gt; x < m; x += gs) {
    const int p = cs.ipri[x];
    if (p >= 0) {
      ilayer[j0 - a0 + x] = prioA[p];
      irank[j0 - a0 + x] = cs.bcnt[(x / kChainB) * kChainMaxL + p] + cs.lrank[x];
    }
  }
  // leftovers: Alg. 1 among the class's new layers (planner.py:236-254), in item order
  bool ok = true;
  if (lead) {
    if (tid < 32) {
      const bool packed = hz < (1 << 26);
      int ne = INT_MIN, nnew = 0, my_cnt = 0;
      for (int cb = 0; cb < m && ok; cb += 32) {
        const int x = cb + lane;
        const bool left = x < m && cs.ipri[x] < 0;
        unsigned lm = __ballot_sync(FULL, left);
        const int my_ts = left ? ts[x] : 0, my_te = left ? te[x] : 0;
        while (lm) {
          const int k = __ffs(lm) - 1;
          lm &= lm - 1;
          const int t0 = __shfl_sync(FULL, my_ts, k), t1 = __shfl_sync(FULL, my_te, k);
          int best;
          bool found;
          if (packed) {
            const int key = __reduce_max_sync(
                FULL, lane < nnew && ne < t0 ? (int)(((unsigned)ne << 5) | (unsigned)(31 - lane)) : -1);
            found = key >= 0;
            best = found ? 31 - (key & 31) : nnew;
          } else {
            const bool ca = lane < nnew && ne < t0;
            const int mx = __reduce_max_sync(FULL, ca ? ne : INT_MIN);
            const unsigned cma = __ballot_sync(FULL, ca && ne == mx);
            found = cma != 0;
            best = found ? __ffs(cma) - 1 : nnew;
          }
          if (!found && nl + nnew == kChainMaxL) {
            ok = false;
            break;
          }
          const int rk = __shfl_sync(FULL, my_cnt, best);
          if (lane == best) ne = t1, my_cnt++;
          nnew += found ? 0 : 1;
          if (lane == k) ilayer[j0 - a0 + x] = nl + best, irank[j0 - a0 + x] = rk;
        }
      }
      if (ok && lane < nnew) newcnt[nl + lane] = my_cnt;
      if (lane == 0) {
        *sh_nnew = nnew, *sh_flag = ok ? 1 : 0;
        if (ok) *sh_gap += (long long)s_gapped;
      }
    }
    __syncthreads();
    ok = *sh_flag != 0;
    if (!ok)  // resolve_class redoes the class: the gap layers' counts start from zero again
      for (int l = tid; l < nl; l += blockDim.x) newcnt[l] = 0;
    __syncthreads();
  }
  return ok;
}

__device__ void layers_unit_big(const LayerArgs &A, const int u, BigState *st, cooperative_groups::grid_group &grid) {
  const int c = u % A.C, t = u / A.C;
  const int v = A.var_of[c];
  const bool gap = (A.cand[c] & STW_CAND_GAP) != 0;
  const int64_t a0 = A.io[(int64_t)v * A.T + t], a1 = A.io[(int64_t)v * A.T + t + 1];
  const int64_t off = A.uo[u];
  const int tid = threadIdx.x;
  const bool lead = blockIdx.x == 0;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + tid, gs = (int64_t)gridDim.x * blockDim.x;
  __shared__ int shi[33];
  __shared__ int sm_nend[kSmemLayers];
  __shared__ int sh_nnew;
  __shared__ long long sh_gap;
  volatile BigState *vst = st;

  int32_t *sAts = A.sA_ts + off, *sAte = A.sA_te + off, *sBts = A.sB_ts + off, *sBte = A.sB_te + off;
  int32_t *loffA = A.loffA + off + u, *loffB = A.loffB + off + u;
  int32_t *prioA = A.prioA + off, *prioB = A.prioB + off;
  int32_t *newcnt = A.newcnt + off, *runoff = A.runoff + off + u;
  int32_t *run_ts = A.run_ts + off, *run_te = A.run_te + off;
  int32_t *ilayer = A.ilayer + off, *irank = A.irank + off;
  int32_t *last = A.lastEnd + off;
  uint32_t *fitw = A.fitw + off * kFitWords;
  int64_t *lsize = A.lsize + off;
  if (lead && tid == 0) {
    vst->nl = 0;
    vst->gap = 0;
    loffA[0] = 0;
  }
  if (lead && tid == 0) sh_gap = 0;
  grid.sync();
#ifdef STW_LAYERS_CLOCK
  long long _lc = clock64();
#define BCLK(i) if (lead && tid == 0) { long long _n = clock64(); atomicAdd(&g_layers_clk[i], (unsigned long long)(_n - _lc)); _lc = _n; }
#else
#define BCLK(i)
#endif
  for (int64_t j0 = a0; j0 < a1;) {
    const int64_t j1 = A.cend[j0];
    const int m = (int)(j1 - j0);
    const int64_t S = A.it.size[j0];
    const int nl = vst->nl;
    const int nfit = min(nl, 32 * kFitWords);
    // ---- 1. fit masks against the slots of earlier classes (every SM)
    for (int64_t x = gt; x < (int64_t)m * kFitWords; x += gs) fitw[(j0 - a0) * kFitWords + x] = 0;
    for (int64_t l = gt; l < nl; l += gs) last[l] = INT_MIN, newcnt[l] = 0;
    grid.sync();
    if (gap && nl > 0) {
      for (int64_t x = gt; x < (int64_t)m * nfit; x += gs) {
        const int jj = (int)(x / nfit), p = (int)(x % nfit);
        const int64_t it = j0 + jj;
        const int l = prioA[p];
        if (slot_fit(sAts, sAte, loffA[l], loffA[l + 1], A.it.ts[it], A.it.te[it]))
          atomicOr(fitw + (it - a0) * kFitWords + (p >> 5), 1u << (p & 31));
      }
    }
    grid.sync();
    BCLK(0)
    // ---- 2. the serial resolve (one CTA, warp 0)
#ifdef STW_LAYERS_CLOCK
    const long long _r0 = clock64();
#endif
    bool done = false;
    if (st->use_chain && gap && nl > 0 && nl <= kChainMaxL) {  // the chain resolve (grid-wide; uniform condition)
      __shared__ int sh_flag;
      done = chain_class(A, st->cs, nl, j0, j1, a0, fitw, prioA, newcnt, ilayer, irank, &sh_flag, &sh_nnew, &sh_gap,
                         lead, A.horizon[t], grid);
    }
    if (lead) {
      if (!done)
        resolve_class(A, gap, nl, j0, j1, a0, off, fitw, prioA, sAts, sAte, loffA, last, newcnt, ilayer, irank,
                      sm_nend, &sh_nnew, &sh_gap, A.horizon[t]);
      __syncthreads();
      if (tid == 0) vst->nnew = sh_nnew;
#ifdef STW_LAYERS_CLOCK
      if (tid == 0) {
        static __device__ int cls_i = 0;
        const int ci = atomicAdd(&cls_i, 1) & 63;
        g_class_clk[ci][0] = clock64() - _r0, g_class_clk[ci][1] = m, g_class_clk[ci][2] = nl;
      }
#endif
    }
    grid.sync();
    BCLK(1)
    // ---- 3. merge this class's slots into the per-layer sorted slot CSR (every SM)
    const int nnew = vst->nnew, nl2 = nl + nnew;
    if (lead) {
      for (int x = tid; x < nnew; x += blockDim.x) lsize[nl + x] = S;
      block_scan_into(nl2, [&](int l) { return (l < nl ? loffA[l + 1] - loffA[l] : 0) + newcnt[l]; }, loffB, shi);
      block_scan_into(nl2, [&](int l) { return newcnt[l]; }, runoff, shi);
    }
    grid.sync();
    for (int64_t x = gt; x < m; x += gs) {
      const int l = ilayer[j0 - a0 + x];
      const int pos = runoff[l] + irank[j0 - a0 + x];
      run_ts[pos] = A.it.ts[j0 + x];
      run_te[pos] = A.it.te[j0 + x];
    }
    grid.sync();
    const int nold = nl > 0 ? loffA[nl] : 0;
    for (int64_t s = gt; s < nold; s += gs) {
      int a = 0, b = nl;  // layer of slot s
      while (b - a > 1) {
        const int mid = (a + b) >> 1;
        if (loffA[mid] <= s)
          a = mid;
        else
          b = mid;
      }
      int l = a;
      while (loffA[l + 1] <= s) l++;  // skip empty layers
      const int ts = sAts[s];
      const int k = newcnt[l] ? lower_bound_i32(run_ts, runoff[l], runoff[l] + newcnt[l], ts) - runoff[l] : 0;
      const int dst = loffB[l] + ((int)s - loffA[l]) + k;
      sBts[dst] = ts;
      sBte[dst] = sAte[s];
    }
    for (int64_t x = gt; x < m; x += gs) {
      const int l = ilayer[j0 - a0 + x];
      const int ts = A.it.ts[j0 + x];
      const int k = l < nl ? lower_bound_i32(sAts, loffA[l], loffA[l + 1], ts) - loffA[l] : 0;
      const int dst = loffB[l] + irank[j0 - a0 + x] + k;
      sBts[dst] = ts;
      sBte[dst] = A.it.te[j0 + x];
    }
    // priority order for later classes: newest (smallest) layers first, creation order within
    for (int64_t x = gt; x < nl2; x += gs) prioB[x] = x < nnew ? nl + (int)x : prioA[x - nnew];
    grid.sync();
    {
      int32_t *tp;
      tp = sAts, sAts = sBts, sBts = tp;
      tp = sAte, sAte = sBte, sBte = tp;
      tp = loffA, loffA = loffB, loffB = tp;
      tp = prioA, prioA = prioB, prioB = tp;
    }
    if (lead && tid == 0) vst->nl = nl2;
    grid.sync();
    BCLK(2)
    j0 = j1;
  }
  // ---- F: stacking (planner.py:441-444)
  if (lead) {
    const int nl = vst->nl;
    int64_t *lbase = A.lbase + off;
    long long carry = A.pers_size[t];
    for (int c0 = 0; c0 < nl; c0 += blockDim.x) {
      const int l = c0 + tid;
      const long long v0 = l < nl ? lsize[l] : 0;
      __shared__ long long shl[33];
      long long tot;
      const long long ex = block_excl_sum<long long>(v0, shl, &tot);
      if (l < nl) lbase[l] = carry + ex;
      carry += tot;
    }
    if (tid == 0) {
      A.nlayers[u] = nl;
      A.gapins[u] = sh_gap;
      A.pool[u] = carry;
    }
  }
}

__global__ void __launch_bounds__(kPlanThreads) k_layers_big(LayerArgs A, const int32_t *__restrict__ ulist, int nu,
                                                             BigState *st) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  for (int i = 0; i < nu; i++) {
    layers_unit_big(A, ulist[i], st + i, grid);
    grid.sync();
  }
}

__device__ __forceinline__ int warp_excl_scan(int v, int *total) {
  int inc = warp_incl_sum(v);
  *total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

// ---------------------------------------------------------------------------
// E (narrow units, <= 32 layers -- every c4 unit): one warp per unit; the
// per-item greedy is a short dependency chain. Lane p holds the same-class last
// end of the layer at priority p and lane q the end of the class's new layer q;
// each item is one ballot (gap host: the lowest fitting priority) raced against
// one max-reduction + ballot (Alg. 1), both speculative, then a select. Layer
// ids, insertion ranks (match_any) and the gap count are resolved lane-parallel
// after each 32-item chunk; ilayer/irank and the merge's output buffer live in
// global scratch (L2), so the shared footprint is the slot CSR and the class
// runs (4 ints per item). Units are packed host-side into CTAs of a fixed
// shared-memory budget, largest first; `wslot` gives each warp its unit and
// shared-memory offset (unit -1: idle warp). A unit that would open a 33rd
// layer is handed to the CTA kernel.

constexpr int kWN = 32;
constexpr int kWarpsPerCta = 8;
constexpr int kLayerSmemInts = 14336;  // 56 KB per CTA: four CTAs per SM

// gap units: per layer an occupancy bitmap over the trace's timeline and its
// per-word prefix popcounts (see below), kWN layers, plus the priority list
__host__ __device__ constexpr int gap_words(int horizon) { return (horizon >> 5) + 2; }
// bitmap words (32 bits) + their prefix counts (16 bits: at most 32 * Wn < 2^16
// set bits before a word, as a CTA's budget caps Wn) + the priority list
__host__ __device__ constexpr int gap_pfx_ints(int horizon) { return (kWN * gap_words(horizon) + 1) / 2; }
__host__ __device__ constexpr int warpn_smem_ints(int horizon) {
  return kWN * gap_words(horizon) + gap_pfx_ints(horizon) + kWN + 1;
}

// GAP = the unit's candidate inserts into gaps of earlier classes' layers.
// Without gap insertion a class only ever fills its own new layers (Alg. 1),
// so the slot CSR, the fit masks, the insertion ranks and the per-class merge
// are not needed at all: such a unit uses no shared memory and its per-item
// step is the Alg. 1 max-reduce + ballot alone.
// Gap units keep, per layer, a bitmap of the timestamps its slots occupy
// (closed slot intervals, pairwise disjoint) and the prefix popcount of every
// bitmap word. fits_gap of [t_s, t_e] against the slots of earlier classes
// (planner.py:196-205) is then "no set bit in [t_s, t_e]": two rank lookups.
// A class's slots are added after the class (its own items only meet each
// other through the `last < t_s` rule), then the touched layers' prefix
// counts are rebuilt.
template <bool GAP>
__device__ __forceinline__ void layers_w32_unit(const LayerArgs &A, int32_t *__restrict__ smem, const int2 slot,
                                                int32_t *__restrict__ over, int *__restrict__ nover) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = lane_id();
  const int u = slot.x;
  const int c = u % A.C, t = u / A.C;
  const int v = A.var_of[c];
  const int64_t a0 = A.io[(int64_t)v * A.T + t], a1 = A.io[(int64_t)v * A.T + t + 1];
  const int n = (int)(a1 - a0);
  const int64_t off = A.uo[u];
  const int hz = A.horizon[t];
  const int Wn = GAP ? gap_words(hz) : 0;
  uint32_t *bits = (uint32_t *)smem;                  // [kWN][Wn]
  uint16_t *pfx = (uint16_t *)(bits + kWN * Wn);       // [kWN][Wn]
  int32_t *prio = (int32_t *)(bits + kWN * Wn) + (GAP ? gap_pfx_ints(hz) : 0);
  const int32_t *gts = A.it.ts + a0, *gte = A.it.te + a0;
  const int64_t *gcend = A.cend + a0;
  int32_t *ilayer = A.ilayer + off;
  int64_t *lsize = A.lsize + off;
  if (GAP) {
    for (int x = lane; x < kWN * Wn + gap_pfx_ints(hz); x += 32) bits[x] = 0;
  }
  int nl = 0, gapc = 0;
  __syncwarp();
  // set bits below x in layer l
  auto rank = [&](int l, int x) -> int {
    const int w = x >> 5;
    return (int)pfx[l * Wn + w] + __popc(bits[l * Wn + w] & ((1u << (x & 31)) - 1u));
  };
  for (int j0 = 0; j0 < n;) {
    const int j1 = (int)(gcend[j0] - a0);
    const int m = j1 - j0;
    const int64_t S = A.it.size[a0 + j0];
    // lane q: end of the class's new layer q (INT_MAX while unopened)
    int last = INT_MIN, ne = INT_MAX, nnew = 0;
    for (int cb = j0; cb < j1; cb += 32) {
      const int mine = cb + lane;
      const int cnt = min(32, j1 - cb);
      int my_ts = 0, my_te = 0;
      unsigned fm = 0;
      if (mine < j1) {
        my_ts = gts[mine];
        my_te = gte[mine];
        if (GAP) {
          // only a trace the input check rejects has times outside [0, horizon];
          // clamp so its bitmap lookups stay in bounds
          my_ts = min(max(my_ts, 0), hz);
          my_te = min(max(my_te, 0), hz);
          for (int p = 0; p < nl; p++) {
            const int l = prio[p];
            if (rank(l, my_te + 1) == rank(l, my_ts)) fm |= 1u << p;
          }
        }
      }
      int my_code = 0;
      if (GAP) {
        // gap host (planner.py:420-431): first fitting layer in priority order
        // whose same-class slots all end before ts. Hot loop: consecutive
        // gap-hosted items, one vote each; the host lane tests (m1 & le) == eq,
        // the raw vote is decoded (ffs) after the chunk; the next item's fields
        // are broadcast one item ahead. An item no layer hosts leaves the loop
        // for Alg. 1.
        const unsigned lm_eq = 1u << lane, lm_le = lm_eq | (lm_eq - 1u);
        unsigned my_m1 = 0;
        int k = 0;
        int ts = __shfl_sync(FULL, my_ts, 0), te = __shfl_sync(FULL, my_te, 0);
        unsigned f = __shfl_sync(FULL, fm, 0);
        while (true) {
          for (; k < cnt; k++) {
            const int k1 = (k + 1) & 31;
            const int nts = __shfl_sync(FULL, my_ts, k1), nte = __shfl_sync(FULL, my_te, k1);
            const unsigned nf = __shfl_sync(FULL, fm, k1);
            const unsigned m1 = __ballot_sync(FULL, (f & lm_eq) && last < ts);
            if (!m1) break;
            last = (m1 & lm_le) == lm_eq ? te : last;
            my_m1 = lane == k ? m1 : my_m1;
            ts = nts, te = nte, f = nf;
          }
          if (k >= cnt) break;
          // Alg. 1 (planner.py:244-252) for item k: the new layer with the largest
          // end < ts, ties to the oldest -- one max-reduction over (end, 31 - lane)
          // keys (ends < 2^26: the host routes longer timelines to the CTA kernel)
          const int key = __reduce_max_sync(FULL, ne < ts ? (int)(((unsigned)ne << 5) | (unsigned)(31 - lane)) : -1);
          const int tgt = key >= 0 ? 31 - (key & 31) : nnew;  // nnew: open a layer
          if (lane == tgt) ne = te;
          nnew += key < 0 ? 1 : 0;
          if (lane == k) my_m1 = 0, my_code = kWN + tgt;
          if (++k >= cnt) break;
          ts = __shfl_sync(FULL, my_ts, k), te = __shfl_sync(FULL, my_te, k);
          f = __shfl_sync(FULL, fm, k);
        }
        if (my_m1) my_code = __ffs(my_m1) - 1;
      } else {
        for (int kg = 0; kg < cnt; kg += 8) {
#pragma unroll
          for (int kk = 0; kk < 8; kk++) {
            const int k = kg + kk;
            const bool valid = k < cnt;  // warp-uniform
            const int ts = __shfl_sync(FULL, my_ts, k & 31), te = __shfl_sync(FULL, my_te, k & 31);
            // Alg. 1 (planner.py:244-252): the new layer with the largest end < ts,
            // ties to the oldest -- one max-reduction over (end, 31 - lane) keys
            const int key = __reduce_max_sync(FULL, ne < ts ? (int)(((unsigned)ne << 5) | (unsigned)(31 - lane)) : -1);
            const int tgt = key >= 0 ? 31 - (key & 31) : nnew;  // nnew: open a layer
            if (valid && lane == tgt) ne = te;
            nnew += (valid && key < 0) ? 1 : 0;
            if (lane == k) my_code = kWN + tgt;
          }
        }
      }
      if (nl + nnew > kWN) {  // a 33rd layer: the CTA kernel redoes the unit
        if (lane == 0) over[atomicAdd(nover, 1)] = u;
        return;
      }
      // lane-parallel: layer ids and the gap count
      const bool act = lane < cnt;
      if (!GAP) {  // no shared memory here: every code is a new layer of the class
        if (act) ilayer[mine] = nl + (my_code - kWN);
        continue;
      }
      const int layer = my_code < kWN ? prio[my_code] : nl + (my_code - kWN);
      gapc += __popc(__ballot_sync(FULL, act && my_code < kWN));
      if (act) ilayer[mine] = layer;
    }
    const int nl2 = nl + nnew;
    if (lane < nnew) lsize[nl + lane] = S;
    if (!GAP || j1 >= n) {  // nothing reads the bitmaps after the last class
      nl = nl2;
      j0 = j1;
      continue;
    }
    __syncwarp();
    // ---- add the class's slots to its layers' bitmaps, then rebuild the touched
    // layers' prefix counts
    unsigned touched = 0;
    for (int x = lane; x < m; x += 32) {
      const int l = ilayer[j0 + x];
      const int ts = min(max(gts[j0 + x], 0), hz), te = min(max(gte[j0 + x], 0), hz);
      touched |= 1u << l;
      uint32_t *row = bits + l * Wn;
      for (int w = ts >> 5; w <= (te >> 5); w++) {
        const int lo = max(ts, w << 5) & 31, hi = min(te, (w << 5) + 31) & 31;
        const uint32_t msk = (hi == 31 ? 0xffffffffu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u);
        atomicOr(row + w, msk);
      }
    }
    for (int o = 16; o; o >>= 1) touched |= __shfl_xor_sync(FULL, touched, o);
    __syncwarp();
    while (touched) {
      const int l = __ffs(touched) - 1;
      touched &= touched - 1;
      uint32_t carry = 0;
      for (int w0 = 0; w0 < Wn; w0 += 32) {
        const int w = w0 + lane;
        const uint32_t c1 = w < Wn ? (uint32_t)__popc(bits[l * Wn + w]) : 0u;
        uint32_t inc = c1;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += y;
        }
        if (w < Wn) pfx[l * Wn + w] = (uint16_t)(carry + inc - c1);
        carry += __shfl_sync(FULL, inc, 31);
      }
    }
    // priority order for later classes: the class's new layers (creation order), then the old list
    {
      const int po = lane < nl ? prio[lane] : 0;
      const int sv = __shfl_sync(FULL, po, (lane - nnew) & 31);
      __syncwarp();
      if (lane < nl2) prio[lane] = lane < nnew ? nl + lane : sv;
    }
    __syncwarp();
    nl = nl2;
    j0 = j1;
  }
  // stacking (planner.py:441-444)
  const long long sz = lane < nl ? lsize[lane] : 0;
  const long long inc = warp_incl_sum(sz);
  const long long base = A.pers_size[t], total = __shfl_sync(FULL, inc, 31);
  if (lane < nl) A.lbase[off + lane] = base + inc - sz;
  if (lane == 0) {
    A.nlayers[u] = nl;
    A.gapins[u] = gapc;
    A.pool[u] = base + total;
  }
}

__global__ void __launch_bounds__(kWarpsPerCta * 32, 5) k_layers_w32(LayerArgs A, const int2 *__restrict__ wslot,
                                                                  int32_t *__restrict__ over, int *__restrict__ nover) {
  extern __shared__ int32_t smem[];
  const int2 slot = wslot[blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5)];
  if (slot.x < 0) return;
  const int c = slot.x % A.C;
  if (A.cand[c] & STW_CAND_GAP)
    layers_w32_unit<true>(A, smem + slot.y, slot, over, nover);
  else
    layers_w32_unit<false>(A, smem, slot, over, nover);
}

// ---------------------------------------------------------------------------
// F: emission (planner.py:446-455)

struct EmitArgs {
  int C, T;
  int64_t N, P;
  const int32_t *var_of;
  Ev e;
  const int64_t *rel, *frel1;
  const int32_t *pid0, *pid1;
  const int32_t *item_of_plan, *item_of_res;  // [V * P], [V * N]
  const int64_t *io, *uo;
  const int32_t *ilayer;
  const int64_t *lbase;
  const uint32_t *rperm;  // events in sweep order (trace, t_s, id)
  const uint32_t *sflag, *spos;  // per sweep position: static event, its rectangle slot
  int64_t NS;
  int64_t *addr;    // [C * N] event order, or nullptr (not requested)
  int32_t *layer;   // [C * N] event order, or nullptr
  int32_t *rts, *rte;  // [NS] sweep-order rectangles of the static events (validate_plan)
  int64_t *rsz, *raddr;  // [NS], [C * NS]
};

// emission (planner.py:446-455) straight into the self-check's sweep order:
// thread per sweep position, every candidate in turn (the event's columns are
// read once and the candidates' dependent lookups item -> layer -> base
// overlap). The static events' rectangles are written in sweep order, the
// event-order address / layer tables only when the caller asked for them.
__global__ void k_emit(EmitArgs A) {
  GRID_STRIDE(k, A.N) {
    const uint32_t i = A.rperm[k];
    const int t = A.e.tr[i];
    const int cl = ev_class(A.e.dyn[i], A.e.te[i], A.e.horizon[t]);
    const int64_t rel = cl == 2 ? 0 : A.rel[i];
    const int p0 = cl == 1 ? A.pid0[i] : -1;
    const int p1 = cl == 1 && A.pid1 ? A.pid1[i] : -1;
    // (sflag == nullptr: every event static and listed in sweep order -- the
    // rectangles are the batch's own columns and the event-order addresses)
    const bool st = A.sflag ? A.sflag[k] != 0 : true;
    const int64_t o = !st ? 0 : A.spos ? (int64_t)A.spos[k] : k;
    if (st && A.rts) {
      A.rts[o] = A.e.ts[i];
      A.rte[o] = A.e.te[i];
      A.rsz[o] = A.e.size[i];
    }
    for (int c = 0; c < A.C; c++) {
      const int64_t u = (int64_t)t * A.C + c;
      const int v = A.var_of[c];
      long long ad = -1;
      int ly = -1;
      if (cl == 0) {
        ad = rel;
      } else if (cl == 1) {
        const int p = v ? p1 : p0;
        int64_t j;
        long long fr = 0;
        if (p >= 0) {
          j = A.item_of_plan[(int64_t)v * A.P + p];
          fr = v ? A.frel1[i] : rel;
        } else {
          j = A.item_of_res[(int64_t)v * A.N + i];
        }
        const int64_t local = j - A.io[(int64_t)v * A.T + t];
        ly = A.ilayer[A.uo[u] + local];
        ad = A.lbase[A.uo[u] + ly] + fr;
      }
      if (st && A.raddr != A.addr) A.raddr[(int64_t)c * A.NS + o] = ad;
      if (A.addr) A.addr[(int64_t)c * A.N + i] = ad;
      if (A.layer) A.layer[(int64_t)c * A.N + i] = ly;
    }
  }
}

// sweep-order rectangle sets for the self-check: static events in (t_s, id) order
__global__ void k_static_flag(const uint32_t *__restrict__ rperm, const uint8_t *__restrict__ dyn, int64_t n,
                              uint32_t *__restrict__ f) {
  GRID_STRIDE(k, n) f[k] = dyn[rperm[k]] ? 0u : 1u;
}

// the event behind each rectangle (only the conflict report needs it)
__global__ void k_rect_events(const uint32_t *__restrict__ rperm, const uint32_t *__restrict__ f,
                              const uint32_t *__restrict__ pos, int64_t n, int32_t *__restrict__ rs_ev) {
  GRID_STRIDE(k, n) {
    if (!f || f[k]) rs_ev[pos ? pos[k] : k] = (int32_t)rperm[k];
  }
}

// ---------------------------------------------------------------------------
// finalisation: verdicts (planner.py:371-373, 392, 464-471), stats, best pick

struct FinalArgs {
  int T, C;
  const int32_t *var_of;
  TraceCounts tc;
  const int64_t *att, *acc;  // per trace (nullptr when no fusion variant ran)
  const int64_t *gapins;
  const int32_t *nlayers;
  const int64_t *pool, *peak;
  const int *bad_align, *bad_phase;
  const long long *vcount;
  const int64_t *ev_off;
  int32_t *rc;
  int64_t *err, *stats;
  int *nconf;
};

__global__ void k_unit_finalize(FinalArgs A) {
  GRID_STRIDE(u, (int64_t)A.T * A.C) {
    int t = (int)(u / A.C), c = (int)(u % A.C);
    bool fus_ran = A.var_of[c] == 1 && A.tc.n_plans[t] > 1 && A.att;
    int64_t *st = A.stats + u * STW_NSTATS;
    int64_t acc = fus_ran ? A.acc[t] : 0;
    st[0] = A.tc.n_static[t];
    st[1] = A.tc.n_pers[t];
    st[2] = A.tc.n_groups[t];
    st[3] = A.tc.n_plans[t] - acc;
    st[4] = A.tc.n_res[t];
    st[5] = fus_ran ? A.att[t] : 0;
    st[6] = acc;
    st[7] = A.gapins[u];
    st[8] = A.nlayers[u];
    st[9] = A.pool[u];
    st[10] = A.peak[t];
    st[11] = A.tc.pers_size[t];
    int rc = STW_OK;
    int64_t e0 = -1;
    if (A.bad_align[t] != INT_MAX) {
      rc = STW_EPLAN;
      e0 = A.ev_off[t] + A.bad_align[t];
    } else if (A.bad_phase[t] != INT_MAX) {
      rc = STW_ETRACE;
      e0 = A.ev_off[t] + A.bad_phase[t];
    } else if (A.pool[u] < A.peak[t]) {
      rc = STW_EPLAN;
    } else if (A.vcount[u] > 0) {
      rc = STW_EPLAN;
      atomicAdd(A.nconf, 1);
    }
    A.rc[u] = rc;
    A.err[2 * u] = e0;
    A.err[2 * u + 1] = -1;
  }
}

// best candidate per trace: argmin (pool_size, candidate index) over clean units
__global__ void k_select_best(const int32_t *__restrict__ rc, const int64_t *__restrict__ pool, int T, int C,
                              int32_t *__restrict__ best, int64_t *__restrict__ bpool) {
  GRID_STRIDE(t, (int64_t)T) {
    int b = -1;
    long long bp = -1;
    for (int c = 0; c < C; c++) {
      int64_t u = t * C + c;
      if (rc[u] != STW_OK) continue;
      if (b < 0 || pool[u] < bp) b = c, bp = pool[u];
    }
    best[t] = b;
    bpool[t] = bp;
  }
}

// the best candidate's addresses, event order, from the sweep-order rectangles
// (dynamic events: -1, as emitted)
__global__ void k_gather_best(const int32_t *__restrict__ tr, const int32_t *__restrict__ best,
                              const uint32_t *__restrict__ rperm, const uint32_t *__restrict__ f,
                              const uint32_t *__restrict__ pos, const int64_t *__restrict__ raddr, int64_t NS,
                              int64_t N, int64_t *__restrict__ out) {
  GRID_STRIDE(k, N) {
    const uint32_t i = rperm[k];
    const int b = best[tr[i]];
    out[i] = b >= 0 && (!f || f[k]) ? raddr[(int64_t)b * NS + (pos ? (int64_t)pos[k] : k)] : -1;
  }
}

__global__ void k_scatter_layers(const int64_t *__restrict__ uo, int64_t U, int C, const int64_t *__restrict__ ev_off,
                                 int64_t N, const int32_t *__restrict__ nl, const int64_t *__restrict__ lbase,
                                 const int64_t *__restrict__ lsize, int64_t *__restrict__ ob, int64_t *__restrict__ os,
                                 int64_t TU) {
  GRID_STRIDE(x, TU) {
    int64_t a = 0, z = U;  // unit owning scratch slot x
    while (z - a > 1) {
      int64_t m = (a + z) >> 1;
      if (uo[m] <= x)
        a = m;
      else
        z = m;
    }
    while (uo[a + 1] <= x) a++;
    int64_t l = x - uo[a];
    if (l >= nl[a]) continue;
    int t = (int)(a / C), c = (int)(a % C);
    int64_t dst = (int64_t)c * N + ev_off[t] + l;
    ob[dst] = lbase[x];
    os[dst] = lsize[x];
  }
}

__global__ void k_scatter_fusions(const int32_t *__restrict__ ptr, const int64_t *__restrict__ pl_off,
                                  const int64_t *__restrict__ acc, const int32_t *__restrict__ var_of, int C,
                                  const int64_t *__restrict__ ev_off, int64_t N, const double *__restrict__ ft,
                                  const double *__restrict__ fa, double *__restrict__ ot, double *__restrict__ oa,
                                  int64_t P) {
  GRID_STRIDE(p, P) {
    int t = ptr[p];
    int64_t k = p - pl_off[t];
    if (k >= acc[t]) continue;
    for (int c = 0; c < C; c++) {
      if (var_of[c] != 1) continue;
      int64_t dst = (int64_t)c * N + ev_off[t] + k;
      ot[dst] = ft[p];
      oa[dst] = fa[p];
    }
  }
}

// ---------------------------------------------------------------------------
// host orchestration

// Per-thread cache of forked streams/events for concurrent launches inside one
// call (created once per host thread, reused; the call stays synchronous).
// per-thread side stream and fork/join events (a call's work is joined back
// into its own stream before the call returns)
// per thread and per device (streams and events belong to the device that was
// current when they were created)
constexpr int kMaxDevices = 64;
static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < kMaxDevices ? d : 0;
}
static cudaStream_t side_stream() {
  thread_local cudaStream_t s[kMaxDevices] = {};
  cudaStream_t &x = s[cur_device()];
  if (!x) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  return x;
}
static cudaEvent_t side_event(int i) {
  thread_local cudaEvent_t e[kMaxDevices][2] = {};
  cudaEvent_t &x = e[cur_device()][i];
  if (!x) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  return x;
}

template <class T>
static void d2h(Ctx &ctx, std::vector<T> &h, const T *d, int64_t n) {
  h.resize(n);
  if (n > 0) d2h_async(ctx, h.data(), d, n * sizeof(T));  // filled at the next sync
}
template <class T>
static T *h2d(Ctx &ctx, Arena &ar, const std::vector<T> &h) {
  T *d = ar.take<T>(h.size() ? h.size() : 1);
  if (d && h.size()) h2d_async(ctx, d, h.data(), h.size() * sizeof(T));
  return d;
}
static void sync(Ctx &ctx) { host_sync(ctx); }

template <class T>
static void out_copy(Ctx &ctx, T *dst, const T *src, int64_t n, bool dst_dev) {
  if (!dst || dst == src || n <= 0 || !ctx.ok()) return;
  STW_CUDA(ctx, cudaMemcpyAsync(dst, src, n * sizeof(T), dst_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                ctx.stream));
}

#define LAUNCH(kern, n, ...)                                                     \
  do {                                                                           \
    if (ctx.ok() && (n) > 0) {                                                   \
      STW_KL(kern, grid_for((n), 256), 256, ctx.stream, __VA_ARGS__);          \
      STW_LAUNCHED(ctx);                                                         \
    }                                                                            \
  } while (0)

// grid-stride reductions: a few CTAs per SM, many elements per thread
#define LAUNCH_RED(kern, n, ...)                                                 \
  do {                                                                           \
    if (ctx.ok() && (n) > 0) {                                                   \
      STW_KL(kern, grid_for((n), 256, 148 * 4), 256, ctx.stream, __VA_ARGS__);   \
      STW_LAUNCHED(ctx);                                                         \
    }                                                                            \
  } while (0)

// STW_DEBUG_TIMING=1: synchronise at phase boundaries and print host wall time per phase.
// STW_DEBUG_TIMING=2: no extra syncs; print, per phase, the host time at which
// the phase's last work was enqueued and the GPU time (events) at which it ended.
struct PhaseTimer {
  Ctx &ctx;
  int mode;
  double t0, tstart;
  std::vector<std::pair<const char *, double>> host;
  std::vector<cudaEvent_t> ev;
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  explicit PhaseTimer(Ctx &c) : ctx(c), mode(0), t0(now()), tstart(t0) {
    if (const char *e = getenv("STW_DEBUG_TIMING")) mode = atoi(e) == 2 ? 2 : 1;
    if (mode == 2) mark0();
  }
  void mark0() {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, ctx.stream);
    ev.push_back(e);
  }
  void mark(const char *name) {
    if (!mode) return;
    if (mode == 2) {
      mark0();
      host.push_back({name, now() - tstart});
      return;
    }
    cudaStreamSynchronize(ctx.stream);
    double t = now();
    fprintf(stderr, "[stw plan] %-24s %8.3f ms\n", name, t - t0);
    t0 = t;
  }
  ~PhaseTimer() {
    if (mode != 2) return;
    cudaStreamSynchronize(ctx.stream);
    for (size_t i = 0; i < host.size(); i++) {
      float g = 0, d = 0;
      cudaEventElapsedTime(&g, ev[0], ev[i + 1]);
      cudaEventElapsedTime(&d, ev[i], ev[i + 1]);
      fprintf(stderr, "[stw plan] %-24s host enq %8.3f ms   gpu end %8.3f ms  (phase %7.3f)\n", host[i].first,
              host[i].second, g, d);
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
};

int plan_batch(Ctx &ctx, const stw_batch *in, const stw_plan_opts *o, stw_plan_out *out, const stw_batch *mirror,
               void (*after_uploads)(void *), void *hook_arg) {
  pinned_reset();  // a call that failed midway may have left transfers pending
  NvtxPhases nv("stw_plan_batch");
  PhaseTimer pt(ctx);
  Arena ar(&ctx);
  DevBatch b;
  if (!o || o->n_cand <= 0 || !o->cand || o->alignment <= 0) {
    ctx.fail(STW_EARG, "bad plan options");
    return ctx.rc;
  }
  if (!stage_batch(ctx, ar, in, &b, mirror)) return ctx.rc;
  const int T = b.T, C = o->n_cand;
  const int64_t N = b.N, U = (int64_t)T * C;
  std::vector<uint8_t> hcand(o->cand, o->cand + C);
  std::vector<int32_t> var_of(C);
  bool want[2] = {false, false};
  for (int c = 0; c < C; c++) {
    var_of[c] = (hcand[c] & STW_CAND_FUSION) ? 1 : 0;
    want[var_of[c]] = true;
  }
  const int V = 2;
  if (T == 0) return ctx.rc;

  pt.mark("stage");
  nv.next("A ranks");
  // ---- A: canonical ranks
  int32_t *tr = ar.take<int32_t>(N + 1);
  int32_t *q = ar.take<int32_t>(N + 1), *r = ar.take<int32_t>(N + 1);
  uint64_t *khi = ar.take<uint64_t>(N + 1), *klo = ar.take<uint64_t>(N + 1);
  uint32_t *perm = ar.take<uint32_t>(N + 1), *rperm = ar.take<uint32_t>(N + 1), *gperm = ar.take<uint32_t>(N + 1);
  int32_t *order_local = ar.take<int32_t>(N + 1);
  long long *mm = ar.take<long long>(2);
  int *im = ar.take<int>(4);
  if (!ctx.ok()) return ctx.rc;
  long long mm_init[2] = {LLONG_MAX, LLONG_MIN};
  h2d_async(ctx, mm, mm_init, sizeof(mm_init));
  STW_CUDA(ctx, cudaMemsetAsync(im, 0, 4 * sizeof(int), ctx.stream));
  // one warp-per-trace pass: tr, presortedness, key widths and the input checks
  int *bad_align = ar.take<int>(T), *bad_phase = ar.take<int>(T);
  if (!ctx.ok()) return ctx.rc;
  if (T > 0) {
    // long traces (c5: 10^6 events in one trace) are split into parts of
    // kScanChunk events, one CTA each, combined by atomics
    constexpr int64_t kScanChunk = 16384;
    const int64_t parts = std::max<int64_t>(1, (b.max_trace_events + kScanChunk - 1) / kScanChunk);
    if (parts > 1) {
      LAUNCH(k_fill_i32, T, bad_align, (int64_t)T, INT_MAX);
      LAUNCH(k_fill_i32, T, bad_phase, (int64_t)T, INT_MAX);
    }
    STW_KL(k_trace_scan, dim3((unsigned)T, (unsigned)parts), 128, ctx.stream, b.ev_off, T, b.id, b.t_s, b.t_e,
           b.size, b.ps, b.pe, b.dyn, b.horizon, b.n_sched, (long long)o->alignment, tr, bad_align, bad_phase, im, mm,
           kScanChunk);
    STW_LAUNCHED(ctx);
  }
  long long hmm[2] = {0, 0};
  int him[4] = {0, 0, 0, 0};
  d2h_async(ctx, hmm, mm, sizeof(hmm));
  d2h_async(ctx, him, im, sizeof(him));
  sync(ctx);
  if (!ctx.ok()) return ctx.rc;
  const int tb = bitlen_u64((uint64_t)(T - 1));
  const int idb = N ? bitlen_u64((uint64_t)(hmm[1] - hmm[0])) : 0;
  const int qb = bitlen_u64((uint64_t)(b.max_trace_events > 0 ? b.max_trace_events - 1 : 0));
  const int tsb = bitlen_u64((uint64_t)him[1]);
  if (him[0] == 0) {  // recorded order: both ranks are the position in the trace
    LAUNCH(k_identity_ranks, N, tr, b.ev_off, N, q, r, rperm, order_local);
  } else {
    // q: id rank within trace
    LAUNCH(k_key_q, N, tr, b.id, N, hmm[0], khi, klo);
    seg_sort(ctx, ar, khi, tb, tb, klo, idb, perm, N, b.ev_off, T, b.max_trace_events);
    LAUNCH(k_rank_from_perm, N, perm, tr, b.ev_off, N, q, (int32_t *)nullptr);
    // r: (t_s, id) rank within trace
    LAUNCH(k_key_r, N, tr, b.t_s, q, N, qb, khi, klo);
    seg_sort(ctx, ar, khi, tb, tb, klo, tsb + qb, rperm, N, b.ev_off, T, b.max_trace_events);
    LAUNCH(k_rank_from_perm, N, rperm, tr, b.ev_off, N, r, order_local);
  }

  pt.mark("A ranks");
  const int pb = bitlen_u64((uint64_t)him[2]);

  pt.mark("A checks");
  nv.next("B groups");
  // ---- B: phase groups
  Ev e{tr, b.t_s, b.t_e, b.ps, b.pe, q, b.size, b.dyn, b.horizon};
  int64_t *rel = ar.take<int64_t>(N + 1);
  int32_t *gof = ar.take<int32_t>(N + 1);
  const int G = (int)N;  // capacity (a trace has no more groups than events)
  Groups g{ar.take<int64_t>(G + 1), ar.take<int32_t>(G + 1), ar.take<int32_t>(G + 1), ar.take<int32_t>(G + 1),
           ar.take<int32_t>(G + 1), ar.take<int64_t>(G + 1)};
  // per-trace counters and the plan flags in one zeroed block
  const size_t tc_bytes = (size_t)T * (5 * sizeof(int) + sizeof(int64_t)) + (size_t)(G + 1) * sizeof(uint32_t);
  char *tcb = ar.take<char>(tc_bytes + 64);
  uint32_t *pidx = ar.take<uint32_t>(G + 1);
  if (!ctx.ok()) return ctx.rc;
  int64_t *tc_pers = (int64_t *)tcb;  // 8-byte aligned first
  int *tc_ints = (int *)(tc_pers + T);
  TraceCounts tc{tc_ints, tc_ints + T, tc_ints + 2 * T, tc_ints + 3 * T, tc_ints + 4 * T, tc_pers};
  uint32_t *is_plan = (uint32_t *)(tc_ints + 5 * T);
  STW_CUDA(ctx, cudaMemsetAsync(tcb, 0, tc_bytes, ctx.stream));
  // the group count stays on the device (G <= N): tables are sized by N and
  // the group kernels read G themselves (fused: sparse ids, no count)
  const uint32_t *d_G = nullptr;
  const bool fused_groups = T > 0 && b.max_trace_events <= kSegSortMax && qb + 2 + 2 * pb <= 64;
  if (fused_groups) {
    const int gbit0 = him[0] == 0 ? qb : 0;  // recorded order: r is the position, already in order
    if (b.max_trace_events <= 2048) {
      constexpr int smem = 2048 * 12 + 8 * 256 * 4 + 2049 * 8 + 2048;
      STW_CUDA(ctx, cudaFuncSetAttribute(k_groups_fused<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      STW_KLS(k_groups_fused<8>, (unsigned)T, 256, smem, ctx.stream, e, b.ev_off, r, pb, qb, gbit0, gperm, g, rel,
              gof, tc, is_plan, pidx);
    } else {
      constexpr int smem = 4096 * 12 + 8 * 256 * 4 + 4097 * 8 + 4096;
      STW_CUDA(ctx, cudaFuncSetAttribute(k_groups_fused<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      STW_KLS(k_groups_fused<16>, (unsigned)T, 256, smem, ctx.stream, e, b.ev_off, r, pb, qb, gbit0, gperm, g, rel,
              gof, tc, is_plan, pidx);
    }
    STW_LAUNCHED(ctx);
  } else {
    uint32_t *head = ar.take<uint32_t>(N + 1), *gid = ar.take<uint32_t>(N + 1);
    int64_t *szs = ar.take<int64_t>(N + 1), *S = ar.take<int64_t>(N + 1);
    if (!ctx.ok()) return ctx.rc;
    LAUNCH(k_key_group, N, tr, b.t_e, b.ps, b.pe, b.dyn, b.horizon, r, N, pb, khi, klo);
    seg_sort(ctx, ar, khi, tb + 2 + 2 * pb, tb, klo, qb, gperm, N, b.ev_off, T, b.max_trace_events,
             /*lo_in_order=*/him[0] == 0);
    LAUNCH(k_group_heads, N, e, gperm, b.ev_off, N, head, szs);
    device_scan<uint32_t>(ctx, ar, head, gid, N, true);
    device_scan<int64_t>(ctx, ar, szs, S, N, false);
    d_G = gid + (N > 0 ? N - 1 : 0);
    LAUNCH(k_group_table, N, e, gperm, head, gid, (const uint32_t *)nullptr, N, g);
    LAUNCH(k_group_rel, N, gperm, gid, S, szs, g, N, d_G, rel, gof);
    LAUNCH(k_trace_counts, G, g, d_G, N, tc, is_plan);
    device_scan<uint32_t>(ctx, ar, is_plan, pidx, G, false);
  }
  std::vector<int> h_nplans, h_nstatic, h_nres;
  d2h(ctx, h_nplans, tc.n_plans, T);
  d2h(ctx, h_nstatic, tc.n_static, T);
  d2h(ctx, h_nres, tc.n_res, T);
  sync(ctx);
  if (!ctx.ok()) return ctx.rc;
  std::vector<int64_t> pl_off(T + 1, 0);
  for (int t = 0; t < T; t++) pl_off[t + 1] = pl_off[t] + h_nplans[t];
  const int64_t P = pl_off[T];
  int64_t *d_pl_off = h2d(ctx, ar, pl_off);
  auto mk_plans = [&]() {
    return Plans{ar.take<int32_t>(P + 1), ar.take<int32_t>(P + 1), ar.take<int64_t>(P + 1),
                 ar.take<int32_t>(P + 1), ar.take<int32_t>(P + 1), ar.take<int32_t>(P + 1),
                 ar.take<int32_t>(P + 1), ar.take<int32_t>(P + 1), ar.take<unsigned long long>(2 * P + 2),
                 ar.take<double>(P + 1), ar.take<uint8_t>(P + 1)};
  };
  Plans p0 = mk_plans();
  int32_t *pid0 = ar.take<int32_t>(N + 1);
  if (!ctx.ok()) return ctx.rc;
  const int64_t *pl_local = fused_groups ? d_pl_off : nullptr;  // fused: trace-local plan ranks
  LAUNCH(k_plan_init, G, g, d_G, (int64_t)G, is_plan, pidx, pl_local, gperm, e, p0);
  LAUNCH(k_plan_members, N, gperm, gof, is_plan, pidx, pl_local, e, N, p0, pid0);
  LAUNCH(k_plan_tmp, P, p0, P);

  pt.mark("B groups");
  nv.next("C fusion");
  // ---- C: fusion variant
  Plans p1 = p0;
  int32_t *pid1 = pid0;
  int64_t *frel1 = rel;
  std::vector<int64_t> h_att(T, 0), h_acc(T, 0);
  double *acc_tmp = nullptr, *acc_avg = nullptr;
  int64_t *att_dev = nullptr, *acc_dev = nullptr;
  if (want[1]) {
    p1 = mk_plans();
    pid1 = ar.take<int32_t>(N + 1);
    frel1 = ar.take<int64_t>(N + 1);
    int32_t *lst = ar.take<int32_t>(P + 1);
    acc_tmp = ar.take<double>(P + 1);
    acc_avg = ar.take<double>(P + 1);
    int64_t *att = ar.take<int64_t>(T), *acc = ar.take<int64_t>(T);
    att_dev = att;
    acc_dev = acc;
    std::vector<int64_t> moff(T + 1, 0);
    const int64_t kMemoMax = 4096;
    for (int t = 0; t < T; t++) {
      int64_t pp = h_nplans[t];
      moff[t + 1] = moff[t] + ((pp > 1 && pp <= kMemoMax) ? pp * pp : 0);
      moff[t + 1] = (moff[t + 1] + 31) & ~(int64_t)31;
    }
    int64_t *d_moff = h2d(ctx, ar, moff);
    uint32_t *memo = ar.take<uint32_t>(moff[T] / 32 + 1);
    FusionArgs F{b.ev_off, rperm, e, d_pl_off, p1, lst, pid1, frel1,
                 ar.take<int64_t>(N + 1), ar.take<int64_t>(N + 1), ar.take<int32_t>(N + 1), ar.take<int32_t>(N + 1),
                 ar.take<int32_t>(N + 1), ar.take<int64_t>(N + 1), ar.take<uint8_t>(N + 1), memo, d_moff, att, acc,
                 acc_tmp, acc_avg};
    if (!ctx.ok()) return ctx.rc;
    // variant-1 state starts as a copy of variant 0; the plan list is the identity;
    // the rejection memo is clear -- one pass
    const int64_t nmemo = moff[T] / 32 + 1, nprep = std::max<int64_t>(std::max<int64_t>(P + 1, N + 1), nmemo);
    STW_KL(k_fusion_prep, grid_for(nprep, 256), 256, ctx.stream, p0, p1, P + 1, pid0, pid1, rel, frel1, N + 1, lst,
           memo, nmemo);
    STW_LAUNCHED(ctx);
    if (ctx.ok()) {
      STW_KL(k_fusion, T, kPlanThreads, ctx.stream, F, T);
      STW_LAUNCHED(ctx);
    }
    d2h(ctx, h_att, att, T);
    d2h(ctx, h_acc, acc, T);
  }

  // largest item size (plan heights of both variants, event sizes): sizes the
  // item sort key, read with the fusion counts
  long long *d_imax = ar.take<long long>(2);
  long long h_imax[2] = {LLONG_MAX, 0};
  if (!ctx.ok()) return ctx.rc;
  h2d_async(ctx, d_imax, h_imax, sizeof(h_imax));
  LAUNCH_RED(k_minmax_i64, P, p0.h, P, d_imax, d_imax + 1);
  if (want[1]) LAUNCH_RED(k_minmax_i64, P, p1.h, P, d_imax, d_imax + 1);
  LAUNCH_RED(k_minmax_i64, N, b.size, N, d_imax, d_imax + 1);
  d2h_async(ctx, h_imax, d_imax, sizeof(h_imax));

  pt.mark("C fusion");
  nv.next("D items");
  // ---- D: items per (variant, trace)
  std::vector<int64_t> io(V * T + 1, 0);
  sync(ctx);
  if (!ctx.ok()) return ctx.rc;
  for (int v = 0; v < V; v++)
    for (int t = 0; t < T; t++) {
      int64_t na = want[v] ? (v ? h_nplans[t] - h_acc[t] : h_nplans[t]) : 0;
      int64_t cnt = want[v] ? na + h_nres[t] : 0;
      io[v * T + t + 1] = io[v * T + t] + cnt;
    }
  const int64_t NI = io[V * T];
  int64_t *d_io = h2d(ctx, ar, io);
  Items it{ar.take<int64_t>(NI + 1), ar.take<int32_t>(NI + 1), ar.take<int32_t>(NI + 1), ar.take<int32_t>(NI + 1),
           ar.take<int32_t>(NI + 1)};
  int32_t *item_of_plan = ar.take<int32_t>(V * (P + 1)), *item_of_res = ar.take<int32_t>(V * (N + 1));
  if (!ctx.ok()) return ctx.rc;
  // sort items by (variant-trace, size desc, t_s, tie)
  const long long maxsu = NI ? std::max(0ll, h_imax[1]) / o->alignment : 0;
  const int vtb = bitlen_u64((uint64_t)(V * T - 1)), sb = bitlen_u64((uint64_t)maxsu);
  if (vtb + sb > 64) {
    ctx.fail(STW_EARG, "item sort key exceeds 64 bits");
    return ctx.rc;
  }
  const bool in_order = him[0] == 0;
  const int ilobits = in_order ? qb : tsb + qb;
  int64_t max_items = 0;
  for (int64_t x = 0; x < V * T; x++) max_items = std::max(max_items, io[x + 1] - io[x]);
  const long long al = o->alignment;
  const int ashift = (al & (al - 1)) == 0 ? __builtin_ctzll((unsigned long long)al) : -1;
  int64_t *cend = ar.take<int64_t>(NI + 1);
  if (!ctx.ok()) return ctx.rc;
  const bool fused_items = T > 0 && max_items <= kSegSortMax && sb + ilobits <= 64;
  if (fused_items) {
    // fused gather + sort + write (every c4 segment)
    if (max_items <= 2048) {
      constexpr int smem = 2048 * 12 + 8 * 256 * 4;
      STW_KLS(k_items_sorted<8>, (unsigned)(V * T), 256, smem, ctx.stream, p0, p1, want[0] ? 1 : 0,
              want[1] ? 1 : 0, d_pl_off, e, b.ev_off, gof, g, pid0, d_io, T, P, N, it, item_of_plan, item_of_res,
              maxsu, ashift, al, qb, ilobits, in_order ? 1 : 0, cend);
    } else {
      constexpr int smem = 4096 * 12 + 8 * 256 * 4;
      STW_CUDA(ctx, cudaFuncSetAttribute(k_items_sorted<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      STW_KLS(k_items_sorted<16>, (unsigned)(V * T), 256, smem, ctx.stream, p0, p1, want[0] ? 1 : 0,
              want[1] ? 1 : 0, d_pl_off, e, b.ev_off, gof, g, pid0, d_io, T, P, N, it, item_of_plan, item_of_res,
              maxsu, ashift, al, qb, ilobits, in_order ? 1 : 0, cend);
    }
    STW_LAUNCHED(ctx);
    pt.mark("D items");
    // a pipelining caller starts streaming its next batch in (and the previous
    // results out) here: the round trips are behind us, and the remaining small
    // uploads of phase E go through the pinned scratch (kernel copies), so the
    // transfer overlaps phases D-G (measured best among the hook points)
    if (after_uploads) after_uploads(hook_arg), after_uploads = nullptr;
  } else {
    Items it0{ar.take<int64_t>(NI + 1), ar.take<int32_t>(NI + 1), ar.take<int32_t>(NI + 1),
              ar.take<int32_t>(NI + 1), ar.take<int32_t>(NI + 1)};
    uint64_t *ihi = ar.take<uint64_t>(NI + 1), *ilo = ar.take<uint64_t>(NI + 1);
    uint32_t *iperm = ar.take<uint32_t>(NI + 1);
    if (!ctx.ok()) return ctx.rc;
    if (T > 0) {  // one global compaction (segments this large would serialise a CTA each)
      const int64_t NV = 2 * (P + N);
      uint32_t *iflag = ar.take<uint32_t>(NV + 1), *ipos = ar.take<uint32_t>(NV + 1);
      if (!ctx.ok()) return ctx.rc;
      LAUNCH(k_item_flags, NV, p0, p1, want[0] ? 1 : 0, want[1] ? 1 : 0, d_pl_off, e, b.ev_off, gof, g, pid0, T,
             P, N, iflag);
      device_scan<uint32_t>(ctx, ar, iflag, ipos, NV, false);
      LAUNCH(k_item_scatter, NV, p0, p1, d_pl_off, e, b.ev_off, T, P, N, iflag, ipos, it0);
    }
    pt.mark("D items");
    LAUNCH(k_item_keys, NI, it0, NI, d_io, V * T, qb, al, maxsu, sb, in_order ? 1 : 0, ihi, ilo);
    seg_sort(ctx, ar, ihi, vtb + sb, vtb, ilo, ilobits, iperm, NI, d_io, (int64_t)V * T, max_items);
    LAUNCH(k_item_permute, NI, it0, it, iperm, NI, d_io, T, P, N, item_of_plan, item_of_res);
  }
  // host-side preparation of phase E, overlapped with the D kernels: unit
  // scratch offsets and the warp-per-unit CTA packing (flat per-unit arrays:
  // this runs while the GPU sorts the items and must finish before it does)
  std::vector<int64_t> uo(U + 1, 0);
  std::vector<int32_t> ucnt(U), uneed(U);
  {
    std::vector<uint8_t> gapc(C);
    for (int c = 0; c < C; c++) gapc[c] = (hcand[c] & STW_CAND_GAP) ? 1 : 0;
    int64_t acc = 0;
    for (int t = 0, u = 0; t < T; t++) {
      const int wn = warpn_smem_ints(std::max(0, b.h_horizon[t]));
      for (int c = 0; c < C; c++, u++) {
        const int v = var_of[c];
        const int64_t n_u = io[(int64_t)v * T + t + 1] - io[(int64_t)v * T + t];
        ucnt[u] = (int32_t)std::min<int64_t>(n_u, INT_MAX);
        uneed[u] = gapc[c] ? wn : 0;
        acc += n_u;
        uo[u + 1] = acc;
      }
    }
  }
  pt.mark("D host uo");
  // narrow units: one warp each, packed into fixed-budget CTAs (largest unit
  // first, then the smallest ones that still fit); units too large for a
  // CTA's budget, and any unit that needs > 32 layers, go to the CTA kernel
  std::vector<int32_t> order, bigs;
  order.reserve(U);
  for (int t = 0, u = 0; t < T; t++) {
    const bool longh = b.h_horizon[t] >= (1 << 26);
    for (int c = 0; c < C; c++, u++) {
      if (uneed[u] <= kLayerSmemInts && ucnt[u] < INT_MAX / 8 && !longh)
        order.push_back(u);
      else
        bigs.push_back(u);
    }
  }
  pt.mark("D host order");
  if (order.size() < 1024) {  // few units (one huge trace): a comparison sort
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return ucnt[x] > ucnt[y]; });
  } else {  // stable counting sort by item count, descending
    int32_t mx = 0;
    for (int32_t u : order) mx = std::max(mx, ucnt[u]);
    std::vector<int32_t> pos(mx + 2, 0);
    for (int32_t u : order) pos[mx - ucnt[u] + 1]++;
    for (int32_t k = 0; k <= mx; k++) pos[k + 1] += pos[k];
    std::vector<int32_t> sorted(order.size());
    for (int32_t u : order) sorted[pos[mx - ucnt[u]]++] = u;
    order.swap(sorted);
  }
  pt.mark("D host csort");
  // gap units: CTAs packed to the shared-memory budget; non-gap units need no
  // shared memory and go eight to a CTA in a second launch (dynamic smem 0),
  // which runs concurrently on a side stream
  std::vector<int2> wslot, wslot_ng;
  int cta_smem_ints = 0;  // the largest packed CTA's footprint: the launch asks for no more
  {
    std::vector<int32_t> og;
    og.reserve(order.size());
    wslot_ng.reserve(order.size() + kWarpsPerCta);
    for (int32_t u : order) {
      if (uneed[u] > 0)
        og.push_back(u);
      else
        wslot_ng.push_back(make_int2(u, 0));
    }
    while (wslot_ng.size() % kWarpsPerCta) wslot_ng.push_back(make_int2(-1, 0));
    wslot.resize(og.size() * kWarpsPerCta + kWarpsPerCta);  // upper bound: one unit per CTA
    size_t ws = 0;
    cta_smem_ints = 0;
    for (size_t i = 0, j = og.size(); i < j;) {
      const size_t base = ws;
      int used = 0, k = 0;
      auto put = [&](int32_t u) {
        wslot[ws++] = make_int2(u, used);
        used += uneed[u];
        k++;
      };
      put(og[i++]);
      while (k < kWarpsPerCta && i < j && used + uneed[og[i]] <= kLayerSmemInts) put(og[i++]);
      while (k < kWarpsPerCta && i < j && used + uneed[og[j - 1]] <= kLayerSmemInts) put(og[--j]);
      while (ws < base + kWarpsPerCta) wslot[ws++] = make_int2(-1, 0);
      cta_smem_ints = std::max(cta_smem_ints, used);
    }
    wslot.resize(ws);
  }
  pt.mark("D sort");
  // classes (written by k_items_sorted on the fused path)
  if (V * T > 0 && !fused_items) LAUNCH(k_class_ends_bs, NI, it, d_io, V * T, NI, cend);

  pt.mark("D classes");
  nv.next("E layers");
  // ---- E: layers per unit (host-side unit layout and CTA packing were prepared during D)
  const int64_t TU = uo[U];
  int64_t *d_uo = h2d(ctx, ar, uo);
  uint8_t *d_cand = h2d(ctx, ar, hcand);
  int32_t *d_var = h2d(ctx, ar, var_of);
  LayerArgs LA{C, T, d_cand, d_var, d_io, d_uo, it, cend, tc.pers_size, b.horizon,
               ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1),
               ar.take<int32_t>(TU + U + 1), ar.take<int32_t>(TU + U + 1),
               ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1),
               ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + U + 1), ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1),
               ar.take<uint32_t>((TU + 1) * kFitWords),
               ar.take<int32_t>(TU + 1), ar.take<int32_t>(TU + 1), ar.take<int64_t>(TU + 1), ar.take<int64_t>(TU + 1),
               ar.take<int32_t>(U), ar.take<int64_t>(U), ar.take<int64_t>(U)};
  if (!ctx.ok()) return ctx.rc;
  {
    const int nctas = (int)(wslot.size() / kWarpsPerCta), nctas_ng = (int)(wslot_ng.size() / kWarpsPerCta);
    // overflow lists (units that need > 32 layers), one per launch: each launch's
    // overflow units are redone by the CTA kernel on that launch's stream
    int32_t *d_over = ar.take<int32_t>(U + 1), *d_over_ng = ar.take<int32_t>(U + 1);
    int *d_nover = ar.take<int>(2), *d_nover_ng = d_nover + 1;
    int2 *d_wslot = nctas ? h2d(ctx, ar, wslot) : nullptr;
    int2 *d_wslot_ng = nctas_ng ? h2d(ctx, ar, wslot_ng) : nullptr;
    int32_t *d_bigs = bigs.empty() ? nullptr : h2d(ctx, ar, bigs);
    if (!ctx.ok()) return ctx.rc;
    STW_CUDA(ctx, cudaMemsetAsync(d_nover, 0, 2 * sizeof(int), ctx.stream));
    cudaStream_t side = nullptr;
    if (nctas_ng) {  // fork: non-gap units (and their overflow) on the side stream
      side = side_stream();
      h2d_flush(ctx);  // the side stream reads the unit tables uploaded above
      STW_CUDA(ctx, cudaEventRecord(side_event(0), ctx.stream));
      STW_CUDA(ctx, cudaStreamWaitEvent(side, side_event(0), 0));
      STW_KLS(k_layers_w32, (unsigned)nctas_ng, kWarpsPerCta * 32, 0, side, LA, d_wslot_ng, d_over_ng, d_nover_ng);
      STW_LAUNCHED(ctx);
      STW_KL(k_layers, 296, kPlanThreads, side, LA, d_over_ng, d_nover_ng);
      STW_LAUNCHED(ctx);
      STW_CUDA(ctx, cudaEventRecord(side_event(1), side));
    }
    if (nctas) {
      const int smem = cta_smem_ints * (int)sizeof(int32_t);
      STW_CUDA(ctx, cudaFuncSetAttribute(k_layers_w32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kLayerSmemInts * (int)sizeof(int32_t)));
      STW_KLS(k_layers_w32, (unsigned)nctas, kWarpsPerCta * 32, smem, ctx.stream, LA, d_wslot, d_over, d_nover);
      STW_LAUNCHED(ctx);
    }
    if (!bigs.empty()) {  // units too large for a warp's shared memory (runs beside the side stream)
      if (bigs.size() <= 4 && !getenv("STW_NO_BIG_COOP")) {
        // a few huge units (one long trace): each spread over the whole GPU
        int occ = 0;
        STW_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_layers_big, kPlanThreads, 0));
        int dev = 0, nsm = kSMs;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        // one CTA per SM: a co-resident CTA spinning in grid.sync would compete with the resolve warp for issue slots
        unsigned grid = (unsigned)nsm;
        if (getenv("STW_BIG_GRID")) grid = (unsigned)atoi(getenv("STW_BIG_GRID"));  // diagnostics
        (void)occ;
        // the chain resolve's scratch, shared by the big units (they run one after another)
        int64_t maxn = 1;
        for (int32_t u : bigs) maxn = std::max<int64_t>(maxn, uo[u + 1] - uo[u]);
        const int64_t nbk = (maxn + kChainB - 1) / kChainB + 1;
        ChainScratch cs{ar.take<int32_t>(maxn), ar.take<int32_t>(maxn), ar.take<int32_t>(maxn),
                        ar.take<int32_t>(maxn), ar.take<int32_t>(maxn), ar.take<int32_t>(nbk),
                        ar.take<int32_t>(nbk + 1), ar.take<int32_t>(nbk), ar.take<int32_t>(nbk * kChainMaxL)};
        std::vector<BigState> hst(bigs.size());
        for (auto &h : hst) h = BigState{0, 0, 0, getenv("STW_NO_CHAIN") ? 0 : 1, 0, cs};
        BigState *d_st = h2d(ctx, ar, hst);
        int nb = (int)bigs.size();
        if (!ctx.ok()) return ctx.rc;
        void *args[] = {(void *)&LA, (void *)&d_bigs, (void *)&nb, (void *)&d_st};
        const int slot = prof_pre(ctx.stream);
        STW_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)k_layers_big, dim3(grid), dim3(kPlanThreads), args, 0,
                                                  ctx.stream));
        prof_post(ctx.stream, "k_layers_big", slot);
      } else {
        STW_KL(k_layers, (unsigned)bigs.size(), kPlanThreads, ctx.stream, LA, d_bigs, (const int *)nullptr);
      }
      STW_LAUNCHED(ctx);
    }
    if (nctas) {  // gap units that overflowed 32 layers (count read on the device)
      STW_KL(k_layers, 296, kPlanThreads, ctx.stream, LA, d_over, d_nover);
      STW_LAUNCHED(ctx);
    }
    if (side) STW_CUDA(ctx, cudaStreamWaitEvent(ctx.stream, side_event(1), 0));  // join
  }

  if (getenv("STW_DEBUG_DUMP")) {  // developer aid: dump unit 0's sorted items and layer choices
    int64_t n0 = uo[1] - uo[0];
    int v0 = var_of[0];
    int64_t j0 = io[(int64_t)v0 * T];
    std::vector<int64_t> hs, hce;
    std::vector<int32_t> hts, hte, htie, href, hil, hir;
    d2h(ctx, hs, it.size + j0, n0);
    d2h(ctx, hts, it.ts + j0, n0);
    d2h(ctx, hte, it.te + j0, n0);
    d2h(ctx, htie, it.tie + j0, n0);
    d2h(ctx, href, it.ref + j0, n0);
    d2h(ctx, hce, cend + j0, n0);
    d2h(ctx, hil, LA.ilayer, n0);
    d2h(ctx, hir, LA.irank, n0);
    sync(ctx);
    fprintf(stderr, "unit0: v=%d items=%lld (j0=%lld)\n", v0, (long long)n0, (long long)j0);
    for (int64_t k = 0; k < n0; k++)
      fprintf(stderr, "  it %lld size=%lld ts=%d te=%d tie=%d ref=%d cend=%lld -> layer %d rank %d\n", (long long)k,
              (long long)hs[k], hts[k], hte[k], htie[k], href[k], (long long)(hce[k] - j0), hil[k], hir[k]);
  }

#ifdef STW_LAYERS_CLOCK
  {
    unsigned long long hc[8];
    cudaStreamSynchronize(ctx.stream);
    cudaMemcpyFromSymbol(hc, g_layers_clk, sizeof(hc));
    fprintf(stderr, "k_layers phases (Mcycles, thread 0 of each CTA): fit %.1f resolve %.1f merge %.1f; item loops %.1f (%llu items); units %llu classes %llu\n",
            hc[0] / 1e6, hc[1] / 1e6, hc[2] / 1e6, hc[3] / 1e6, hc[5], hc[7], hc[6]);
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_layers_clk, z, sizeof(z));
    unsigned long long cc[64][3];
    cudaMemcpyFromSymbol(cc, g_class_clk, sizeof(cc));
    for (int i = 0; i < 64 && cc[i][1]; i++)
      fprintf(stderr, "  class %d: %llu items, %llu earlier layers, %.1f Mcycles (%.0f / item)\n", i, cc[i][1],
              cc[i][2], cc[i][0] / 1e6, (double)cc[i][0] / cc[i][1]);
  }
#endif
  pt.mark("E layers");
  if (after_uploads) after_uploads(hook_arg);  // the unfused path: after phase E
  nv.next("F emission");
  // ---- F + G: emission in sweep order, the self-check's rectangles with it;
  // static peak (K1) and the sweep validator (K7)
  int64_t *peak = ar.take<int64_t>(T);
  if (!ctx.ok()) return ctx.rc;
  // finished at the finalize round trip
  const PeakPending ppk =
      peak_live_launch(ctx, ar, b, true, peak, __builtin_ctzll((unsigned long long)o->alignment), /*pinned=*/true);
  std::vector<int64_t> so(T + 1, 0);
  for (int t = 0; t < T; t++) so[t + 1] = so[t] + h_nstatic[t];
  const int64_t NS = so[T];
  // every event static and every trace in recorded order: the sweep order is the
  // event order, so the self-check's rectangles are the batch's own columns and
  // the event-order addresses (no flags, positions, or copies)
  const bool ident = NS == N && him[0] == 0;
  uint32_t *sflag = nullptr, *spos = nullptr;
  const int64_t *d_so = b.ev_off;
  int32_t *rts = nullptr, *rte = nullptr;
  int64_t *rsz = nullptr;
  if (!ident) {
    sflag = ar.take<uint32_t>(N + 1), spos = ar.take<uint32_t>(N + 1);
    int64_t *so_dev = ar.take<int64_t>(T + 1);  // the same offsets, made on the device (no upload)
    rts = ar.take<int32_t>(NS + 1), rte = ar.take<int32_t>(NS + 1), rsz = ar.take<int64_t>(NS + 1);
    if (!ctx.ok()) return ctx.rc;
    LAUNCH(k_static_flag, N, rperm, b.dyn, N, sflag);
    device_scan<uint32_t>(ctx, ar, sflag, spos, N, false);
    STW_KL(k_offsets_i32, 1, 1024, ctx.stream, tc.n_static, T, so_dev);
    STW_LAUNCHED(ctx);
    d_so = so_dev;
  }
  // device outputs are emitted in place; host outputs are staged
  int64_t *addr = !out->addr ? nullptr : out->on_device ? out->addr : ar.take<int64_t>((int64_t)C * N + 1);
  int32_t *layer = !out->layer_of ? nullptr : out->on_device ? out->layer_of : ar.take<int32_t>((int64_t)C * N + 1);
  int64_t *raddr = ident && addr ? addr : ar.take<int64_t>((int64_t)C * NS + 1);
  long long *vcount = ar.take<long long>(U);
  int *vfirst = ar.take<int>(U);
  if (!ctx.ok()) return ctx.rc;
  EmitArgs EA{C, T, N, P, d_var, e, rel, frel1, pid0, pid1, item_of_plan, item_of_res, d_io, d_uo,
              LA.ilayer, LA.lbase, rperm, sflag, spos, NS, addr, layer, rts, rte, rsz, raddr};
  LAUNCH(k_emit, N, EA);
  pt.mark("F emit");
  nv.next("G self-check");
  RectSets rs{T, NS, d_so, ident ? b.t_s : rts, ident ? b.t_e : rte, ident ? b.size : rsz, C, raddr};
  // fast validity test now; its verdict is read at the finalize round trip
  STW_CUDA(ctx, cudaMemsetAsync(vcount, 0, U * sizeof(long long), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(vfirst, 0x7f, U * sizeof(int), ctx.stream));
  const int32_t *d_vorder = nullptr;  // traces by static event count, largest first
  if (T > 1 && !getenv("STW_K7_NATURAL")) {
    std::vector<int32_t> ord(T);
    for (int t = 0; t < T; t++) ord[t] = t;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int c) { return h_nstatic[a] > h_nstatic[c]; });
    d_vorder = h2d(ctx, ar, ord);
  }
  int *d_nflag = overlap_launch(ctx, ar, rs, __builtin_ctzll((unsigned long long)o->alignment), d_vorder);
  if (!ctx.ok()) return ctx.rc;

  pt.mark("G check");
  // ---- per-unit verdicts, stats and best-candidate selection on the device
  int32_t *d_rc = ar.take<int32_t>(U);
  int64_t *d_err = ar.take<int64_t>(2 * U), *d_stats = ar.take<int64_t>(U * STW_NSTATS);
  int32_t *d_best = ar.take<int32_t>(T);
  int64_t *d_bpool = ar.take<int64_t>(T), *d_abest = ar.take<int64_t>(N + 1);
  int *d_nconf = ar.take<int>(1);
  int64_t *d_att = att_dev, *d_acc = acc_dev;
  if (!ctx.ok()) return ctx.rc;
  FinalArgs FA{T, C, d_var, tc, d_att, d_acc, LA.gapins, LA.nlayers, LA.pool, peak, bad_align, bad_phase, vcount,
               b.ev_off, d_rc, d_err, d_stats, d_nconf};
  auto finalize = [&]() {
    STW_CUDA(ctx, cudaMemsetAsync(d_nconf, 0, sizeof(int), ctx.stream));
    LAUNCH(k_unit_finalize, U, FA);
    LAUNCH(k_select_best, T, d_rc, LA.pool, T, C, d_best, d_bpool);
    LAUNCH(k_gather_best, N, tr, d_best, rperm, sflag, spos, raddr, NS, N, d_abest);
  };
  finalize();
  // one host round trip for the deferred checks: conflicts, units the fast
  // validity test could not decide, traces whose peak needs the global timeline
  int hq[3] = {0, 0, 0};
  d2h_async(ctx, hq, d_nconf, sizeof(int));
  if (d_nflag) d2h_async(ctx, hq + 1, d_nflag, sizeof(int));
  if (ppk.nbig) d2h_async(ctx, hq + 2, ppk.nbig, sizeof(int));
  sync(ctx);
  if (!ctx.ok()) return ctx.rc;
  if (hq[1] > 0 || hq[2] > 0) {  // rare: redo the verdicts with the exact validator / global peaks
    if (hq[2] > 0) peak_live_finish(ctx, ar, b, true, peak, ppk);
    if (hq[1] > 0) validate_exact(ctx, ar, rs, vcount, vfirst);
    finalize();
    d2h_async(ctx, hq, d_nconf, sizeof(int));
    sync(ctx);
    if (!ctx.ok()) return ctx.rc;
  }
  const int h_nconf = hq[0];
  if (h_nconf > 0) {  // error path: name the first reported pair of every conflicting unit
    std::vector<long long> h_vc;
    std::vector<int> h_vf;
    std::vector<int32_t> h_rc2;
    std::vector<int64_t> h_err2;
    d2h(ctx, h_vc, vcount, U);
    d2h(ctx, h_vf, vfirst, U);
    d2h(ctx, h_rc2, d_rc, U);
    d2h(ctx, h_err2, d_err, 2 * U);
    int32_t *rs_ev = ar.take<int32_t>(NS + 1);
    if (ctx.ok()) LAUNCH(k_rect_events, N, rperm, sflag, spos, N, rs_ev);
    sync(ctx);
    for (int64_t u = 0; u < U && ctx.ok(); u++) {
      if (h_vc[u] <= 0 || h_err2[2 * u] >= 0) continue;
      int t = (int)(u / C), c = (int)(u % C);
      int pa = -1, pbb = -1;
      first_pair(ctx, rs, t, c, h_vf[u], &pa, &pbb);
      if (pa >= 0) {
        int32_t ev2[2] = {-1, -1};
        STW_CUDA(ctx, cudaMemcpy(&ev2[0], rs_ev + so[t] + pa, sizeof(int32_t), cudaMemcpyDeviceToHost));
        STW_CUDA(ctx, cudaMemcpy(&ev2[1], rs_ev + so[t] + pbb, sizeof(int32_t), cudaMemcpyDeviceToHost));
        h_err2[2 * u] = ev2[0];
        h_err2[2 * u + 1] = ev2[1];
      }
    }
    h2d_async(ctx, d_err, h_err2.data(), 2 * U * sizeof(int64_t));
    sync(ctx);
  }
  pt.mark("finalize");

  // ---- outputs
  const bool od = out->on_device != 0;
  out_copy(ctx, out->rc, d_rc, U, od);
  out_copy(ctx, out->err_ids, d_err, 2 * U, od);
  out_copy(ctx, out->stats, d_stats, U * STW_NSTATS, od);
  out_copy(ctx, out->addr, addr, (int64_t)C * N, od);
  out_copy(ctx, out->layer_of, layer, (int64_t)C * N, od);
  out_copy(ctx, out->order, order_local, N, od);
  if (out->layer_base || out->layer_size || out->fus_tmp || out->fus_avg) {
    int64_t *lb_out = ar.take<int64_t>((int64_t)C * N + 1), *ls_out = ar.take<int64_t>((int64_t)C * N + 1);
    double *ft_out = ar.take<double>((int64_t)C * N + 1), *fa_out = ar.take<double>((int64_t)C * N + 1);
    if (!ctx.ok()) return ctx.rc;
    for (void *p : {(void *)lb_out, (void *)ls_out, (void *)ft_out, (void *)fa_out})  // unused slots read as 0
      STW_CUDA(ctx, cudaMemsetAsync(p, 0, ((int64_t)C * N + 1) * 8, ctx.stream));
    LAUNCH(k_scatter_layers, TU, d_uo, (int64_t)U, C, b.ev_off, N, LA.nlayers, LA.lbase, LA.lsize, lb_out, ls_out, TU);
    if (want[1]) LAUNCH(k_scatter_fusions, P, p0.tr, d_pl_off, d_acc, d_var, C, b.ev_off, N, acc_tmp, acc_avg, ft_out, fa_out, P);
    out_copy(ctx, out->layer_base, lb_out, (int64_t)C * N, od);
    out_copy(ctx, out->layer_size, ls_out, (int64_t)C * N, od);
    out_copy(ctx, out->fus_tmp, ft_out, (int64_t)C * N, od);
    out_copy(ctx, out->fus_avg, fa_out, (int64_t)C * N, od);
  }
  if (o->select_best) {
    out_copy(ctx, out->best_cand, d_best, T, od);
    out_copy(ctx, out->best_pool, d_bpool, T, od);
    out_copy(ctx, out->addr_best, d_abest, N, od);
  }
  sync(ctx);
  pt.mark("outputs");
  return ctx.rc;
}

}  // namespace stw
