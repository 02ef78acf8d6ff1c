// K9/K10 sequential residue, register-resident variant.
//
// The replay's state is small on real traces -- the caching allocator's free
// blocks number at most one or two per segment (c1: 29, c3: 68, c5: 129), the
// pool's free set a handful of intervals -- but the general warp (replay.cu,
// k_replay) pays a chain of dependent shared/global loads per op. Here the
// whole state lives in the registers of one warp (R rows per lane: cache
// blocks {lo, hi, segment base}, pool free intervals {lo, hi}, all in units
// of the largest power of two dividing every size / address of the call, so
// 32-bit), and every query is a few lane-parallel compares plus one or two
// warp reductions (REDUX) or ballots:
//
//   best fit (baseline.py:54-61, intervals.py:165-176) = min length, ties to
//     the lowest address (segments are appended at increasing bases, so the
//     cache's (segment, free-list) order is address order): REDUX.MIN over
//     the lengths, then over the addresses of the rows that tie;
//   free + merge (baseline.py:79-95, intervals.py:100-111): two ballots find
//     the neighbours that end at lo / start at hi (same segment), the owning
//     lanes update their own rows;
//   planned placement (sim.py:196-203): one ballot finds the free interval
//     that contains the request, its lane splits it.
//
// Ops stream through in windows of 32 (one per lane) with a three-stage
// prefetch: op records two windows ahead, the allocation a free releases one
// window ahead (it was written at the end of an earlier window; allocations
// of the current or previous window are forwarded through shared memory), so
// no global latency sits on the per-op chain. Per-op results {addr, segment,
// flags} are written once per window; the replay log is built from them by a
// parallel kernel afterwards, and the metrics (sim.py:67-117) are folded
// inside the loop. Preconditions (checked, otherwise the call falls back to
// k_replay): unique ids (so the id-level errors cannot occur), every value a
// multiple of the unit below 2^31 units, and the state within 32 R rows.
#include <algorithm>

#include "planner.cuh"

namespace stw {

#define GS4(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

enum { RR_PLANNED = 0, RR_REUSE = 1, RR_FALLBACK = 2, RR_MISMATCH = 3, RR_ONLINE = 4, RR_DYN = 5 };
constexpr unsigned kRFull = 0xffffffffu;
constexpr long long kRMinSegment = 2ll * 1024 * 1024;

struct RegArgs {
  int64_t n;  // events; ops = 2n
  const uint32_t *operm;
  const int32_t *apos;
  const int64_t *id, *size;
  const int32_t *ts, *te;
  const uint8_t *dyn;
  const int8_t *route0;
  const int64_t *paddr;
  const int32_t *key;
  const int64_t *sp_off, *sp_lo, *sp_hi;
  int64_t nsp;
  int reuse, baseline;
  long long pool;
  unsigned long long *unit;  // [0] OR of every value, [1] max value
  int4 *ops;                 // per op: {size_u, flags, z, w}
  int4 *res;                 // per op: {addr_u, segment base_u, flags, 0}
  long long *out;            // see k_replay_reg
  // resume after the cache outgrew its rows: resume[0] = op to continue at
  // (0: start), [1] next segment base, [2] cache rows dumped; dump[r * 32 + lane]
  long long *resume;
  int4 *dump;
  int sp_staged;  // the reuse spaces (in units) are staged in dynamic shared memory
  // off-chain mode (simulate): the planned static allocations and their frees
  // are not replayed; ridx maps a full op index to its replayed index
  const uint32_t *ridx;
  int64_t nops;  // ops replayed (2n, or the kept ops)
};

// a static event whose allocation got a planned address (sim.py:189-203)
__device__ __forceinline__ bool reg_planned(const RegArgs &A, int e) {
  return !A.baseline && !A.dyn[e] && A.route0[e] == RR_PLANNED;
}
constexpr int64_t kSpSmemMax = 16384;  // intervals staged in shared memory (128 KB)

// the unit: OR of every size / planned address / space bound / the pool and the 2 MiB segment minimum
__global__ void k_reg_unit(RegArgs A) {
  unsigned long long o = 0, mx = 0;
  GS4(e, A.n) {
    const unsigned long long s = (unsigned long long)A.size[e];
    o |= s;
    mx = max(mx, s);
    if (!A.baseline && !A.dyn[e] && A.route0[e] == RR_PLANNED) {
      const unsigned long long a = (unsigned long long)A.paddr[e];
      o |= a;
      mx = max(mx, a + s);
    }
  }
  if (!A.baseline) GS4(j, A.nsp) {
      o |= (unsigned long long)A.sp_lo[j] | (unsigned long long)A.sp_hi[j];
      mx = max(mx, (unsigned long long)A.sp_hi[j]);
    }
  for (int d = 16; d; d >>= 1) {
    o |= __shfl_xor_sync(kRFull, o, d);
    mx = max(mx, __shfl_xor_sync(kRFull, mx, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(A.unit, o);
    atomicMax(A.unit + 1, mx);
  }
}

__device__ __forceinline__ int reg_shift(const RegArgs &A) {
  const unsigned long long o = A.unit[0] | (unsigned long long)kRMinSegment | (unsigned long long)A.pool;
  return __ffsll((long long)o) - 1;
}

// op records in op order: x = size in units, y = is_alloc | route << 1,
// z = planned address (PLANNED) / first space interval (DYN) / the op index
// of the allocation a free releases, w = end of the space intervals (DYN)
__global__ void k_reg_ops(RegArgs A) {
  const int sh = reg_shift(A);
  GS4(k, 2 * A.n) {
    const uint32_t o = A.operm[k];
    const int e = (int)(o >> 1);
    if (A.ridx && reg_planned(A, e)) continue;  // off the chain
    const int64_t j = A.ridx ? (int64_t)A.ridx[k] : k;
    const bool alloc = !(o & 1);
    int4 r;
    r.x = (int)((unsigned long long)A.size[e] >> sh);
    r.z = r.w = 0;
    if (alloc) {
      int route = RR_ONLINE;
      if (!A.baseline) {
        if (A.dyn[e]) {
          route = RR_DYN;
          const int kk = A.key[e];
          if (A.reuse && kk >= 0) {
            r.z = (int)A.sp_off[kk];
            r.w = (int)A.sp_off[kk + 1];
          }
        } else {
          route = A.route0[e];
          if (route == RR_PLANNED) r.z = (int)((unsigned long long)A.paddr[e] >> sh);
        }
      }
      r.y = 1 | (route << 1);
    } else {
      r.y = 0;
      r.z = A.ridx ? (int)A.ridx[A.apos[e]] : A.apos[e];
    }
    A.ops[j] = r;
  }
}

// Row helpers. Empty rows hold sentinels that no query matches: a cache row
// {0, 0, kNoSeg} (length 0, no segment), a pool row {kRFull, kRFull}.
constexpr uint32_t kNoSeg = kRFull;

// this lane (eq = 1 << lane, computed once per kernel: no S2R on the chain) is
// the lowest set bit of m (lanemask compare: no variable-latency ffs either)
__device__ __forceinline__ bool lowest_lane(unsigned m, unsigned eq) { return (m & (eq | (eq - 1u))) == eq; }

// first empty row of the first lane that has one; false if the state is full
template <int R, bool CACHE>
__device__ __forceinline__ bool reg_insert(uint32_t (&lo)[R], uint32_t (&hi)[R], uint32_t (&sg)[R], uint32_t a,
                                           uint32_t b, uint32_t s, unsigned eq) {
  bool has = false;
#pragma unroll
  for (int r = 0; r < R; r++) has |= CACHE ? sg[r] == kNoSeg : hi[r] == kRFull;
  const unsigned m = __ballot_sync(kRFull, has);
  if (!m) return false;
  if (lowest_lane(m, eq)) {
    bool done = false;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const bool e = !done && (CACHE ? sg[r] == kNoSeg : hi[r] == kRFull);
      if (e) {
        lo[r] = a, hi[r] = b;
        if (CACHE) sg[r] = s;
      }
      done |= e;
    }
  }
  return true;
}

// the first empty row of lane ffs(me) - 1 takes [a, b) (segment s)
template <int R, bool CACHE>
__device__ __forceinline__ void reg_put(uint32_t (&lo)[R], uint32_t (&hi)[R], uint32_t (&sg)[R], unsigned me,
                                        uint32_t a, uint32_t b, uint32_t s, unsigned eq) {
  if (lowest_lane(me, eq)) {
    bool done = false;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const bool e = !done && (CACHE ? sg[r] == kNoSeg : hi[r] == kRFull);
      if (e) {
        lo[r] = a, hi[r] = b;
        if (CACHE) sg[r] = s;
      }
      done |= e;
    }
  }
}

// release [a, b) (segment s for the cache): merge with the free neighbours that
// end at a / start at b (baseline.py:79-95, intervals.py:100-111). The four
// collectives (left, right, empty-row votes, the right neighbour's end) are
// independent and issued together; the updates are predicated.
template <int R, bool CACHE>
__device__ __forceinline__ bool reg_release(uint32_t (&lo)[R], uint32_t (&hi)[R], uint32_t (&sg)[R], uint32_t a,
                                            uint32_t b, uint32_t s, unsigned eq) {
  unsigned lm = 0, rm = 0;
  uint32_t rhi = 0;
  bool has_e = false;
#pragma unroll
  for (int r = 0; r < R; r++) {
    const bool same = !CACHE || sg[r] == s;  // empty cache rows: kNoSeg; empty pool rows: kRFull bounds
    const bool L = same && hi[r] == a, Rr = same && lo[r] == b;
    lm |= (unsigned)L << r;
    rm |= (unsigned)Rr << r;
    if (Rr) rhi = hi[r];
    has_e |= CACHE ? sg[r] == kNoSeg : hi[r] == kRFull;
  }
  const unsigned ml = __ballot_sync(kRFull, lm != 0), mr = __ballot_sync(kRFull, rm != 0);
  const unsigned me = __ballot_sync(kRFull, has_e);
  const uint32_t nh = __reduce_max_sync(kRFull, rhi);  // the right neighbour's end
#pragma unroll
  for (int r = 0; r < R; r++) {
    if ((lm >> r) & 1) hi[r] = mr ? nh : b;
    if ((rm >> r) & 1) {
      if (ml) {  // swallowed by the left neighbour
        lo[r] = CACHE ? 0u : kRFull;
        hi[r] = CACHE ? 0u : kRFull;
        if (CACHE) sg[r] = kNoSeg;
      } else {
        lo[r] = a;
      }
    }
  }
  if (ml | mr) return true;
  if (!me) return false;
  reg_put<R, CACHE>(lo, hi, sg, me, a, b, s, eq);
  return true;
}

// take [a, a + n) out of the pool free interval holding it (sim.py:196-203);
// 0 ok, 1 not free (SimulationError), 2 no row for the split's upper part.
// The votes (owner, split, empty row) and the owner's end are issued together.
template <int R>
__device__ __forceinline__ int reg_pool_take(uint32_t (&fl)[R], uint32_t (&fh)[R], uint32_t (&dummy)[R], uint32_t a,
                                             uint32_t n, unsigned eq) {
  const uint32_t e = a + n;
  bool own = false, split = false, has_e = false;
  uint32_t oh = 0;
#pragma unroll
  for (int r = 0; r < R; r++) {
    has_e |= fh[r] == kRFull;
    if (fl[r] <= a && e <= fh[r]) {  // empty rows: fl = kRFull > a
      own = true;
      oh = fh[r];
      split = fl[r] < a && e < oh;
      if (fl[r] < a) fh[r] = a;
      else if (e < oh) fl[r] = e;
      else fl[r] = fh[r] = kRFull;
    }
  }
  const unsigned mo = __ballot_sync(kRFull, own), ms = __ballot_sync(kRFull, split);
  const unsigned me = __ballot_sync(kRFull, has_e);
  const uint32_t nh = __reduce_max_sync(kRFull, split ? oh : 0u);
  if (!mo) return 1;
  if (ms) {
    if (!me) return 2;
    reg_put<R, false>(fl, fh, dummy, me, e, nh, 0, eq);
  }
  return 0;
}

// shared-memory accesses by 32-bit shared-window address: the bases are
// computed once (plain __shared__ indexing re-derives the window address from
// SR_CgaCtaId on every access inside the op loop)
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  uint32_t r;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// pairwise (tree) minimum over a lane's rows: log2(R) dependent steps, not R
template <int R>
__device__ __forceinline__ uint32_t rows_min(uint32_t (&v)[R]) {
#pragma unroll
  for (int w = 1; w < R; w *= 2)
#pragma unroll
    for (int r = 0; r + w < R; r += 2 * w) v[r] = min(v[r], v[r + w]);
  return v[0];
}

#ifdef STW_REPLAY_PROF
__device__ unsigned long long g_rr_prof[4][2];
#endif

// out: [0] status (0 done, 1 outside the preconditions: more rows / k_replay,
// 2 replay error), [2] error id, [3] error address
template <int R, int RP, bool SIM>
__global__ void __launch_bounds__(32) k_replay_reg(RegArgs A) {
  // per window: op records, the allocations its frees release, the first space
  // intervals of its dynamic ops, and its results ({addr, segment base, flags,
  // grown}, uniform: every lane writes the same record and reads its own write)
  __shared__ int4 s_op[32], s_info[32], s_res[32];
  __shared__ uint4 s_sp[32];
  const int lane = threadIdx.x;
  const unsigned leq = 1u << lane;
  const int sh = reg_shift(A);
  const int64_t n2 = A.nops;
  long long *out = A.out;
  if (A.unit[1] >> sh >= (1ull << 31) || ((unsigned long long)A.pool >> sh) >= (1ull << 31)) {
    if (lane == 0) out[0] = 1;  // values must fit 31 bits in units
    return;
  }
  const uint32_t a_op = smem_addr(s_op), a_info = smem_addr(s_info), a_res = smem_addr(s_res),
                 a_sp = smem_addr(s_sp);
  extern __shared__ uint2 s_spc[];  // the whole reuse-space table, when A.sp_staged
  if (SIM && A.sp_staged) {
    for (int64_t j = lane; j < A.nsp; j += 32)
      s_spc[j] = make_uint2((uint32_t)((unsigned long long)A.sp_lo[j] >> sh), (uint32_t)((unsigned long long)A.sp_hi[j] >> sh));
    __syncwarp();
  }
  // cache blocks {cl, ch, cs} (R rows per lane) and pool free intervals {fl, fh} (RP rows)
  uint32_t cl[R], ch[R], cs[R], fl[RP], fh[RP], fs[RP];
#pragma unroll
  for (int r = 0; r < R; r++) cl[r] = ch[r] = 0, cs[r] = kNoSeg;
#pragma unroll
  for (int r = 0; r < RP; r++) fl[r] = fh[r] = kRFull, fs[r] = 0;
  int over = 0;  // which structure outgrew its rows: 1 cache, 2 pool
  const uint32_t pool_u = (uint32_t)((unsigned long long)A.pool >> sh);
  if (SIM && pool_u > 0 && lane == 0) fl[0] = 0, fh[0] = pool_u;
  uint32_t next_base = SIM ? pool_u : 0u;
  // resuming (baseline only: the cache is the whole state): the previous
  // launch's rows, the next segment base, and the first op not yet replayed
  const int64_t start = SIM ? 0 : A.resume[0];
  if (start > 0) {
    next_base = (uint32_t)A.resume[1];
    const int rd = (int)A.resume[2];
#pragma unroll
    for (int r = 0; r < R; r++)
      if (r < rd) {
        const int4 q = A.dump[r * 32 + lane];
        cl[r] = (uint32_t)q.x, ch[r] = (uint32_t)q.y, cs[r] = (uint32_t)q.z;
      }
  }
  const uint32_t minseg = (uint32_t)(kRMinSegment >> sh);
  int status = 0;
  long long err_op = 0, err_addr = 0, done_ops = 0;
  bool too_big = false;

  // caching-allocator malloc (baseline.py:49-77): best fit = min length, ties
  // to the lowest address; none fits: a fresh segment at the next base. The
  // block's segment base comes back uniform (one max-reduction, read late).
  auto cache_malloc = [&](uint32_t n, uint32_t *addr, uint32_t *sbase, uint32_t *grown) -> bool {
    uint32_t key[R], t[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint32_t len = ch[r] - cl[r];  // empty rows: 0, never >= n
      key[r] = len >= n ? len : kRFull;
      t[r] = key[r];
    }
    const uint32_t m = __reduce_min_sync(kRFull, rows_min<R>(t));
    if (m != kRFull) {
#pragma unroll
      for (int r = 0; r < R; r++) t[r] = key[r] == m ? cl[r] : kRFull;
      const uint32_t a = __reduce_min_sync(kRFull, rows_min<R>(t));
      uint32_t bs = 0;
#pragma unroll
      for (int r = 0; r < R; r++) {
        if (key[r] == m && cl[r] == a) {  // the one winning row of the warp
          bs = cs[r];
          cl[r] += n;
          if (cl[r] == ch[r]) cl[r] = ch[r] = 0, cs[r] = kNoSeg;
        }
      }
      *sbase = __reduce_max_sync(kRFull, bs);  // (only the winner is non-zero)
      *addr = a;
      *grown = 0;
      return true;
    }
    uint32_t ss = 1;
    while (ss < n) ss <<= 1;
    if (ss < minseg) ss = minseg;
    if ((unsigned long long)next_base + ss >= (1ull << 31)) {
      too_big = true;  // values past 31 bits: the general warp
      return false;
    }
    const uint32_t base = next_base;
    if (ss > n && !reg_insert<R, true>(cl, ch, cs, base + n, base + ss, base, leq)) return false;  // state untouched
    next_base += ss;
    *grown = ss, *addr = base, *sbase = base;
    return true;
  };

  // three-stage prefetch: O1/O2 = op records of the next two windows, F1 = the
  // allocation results the next window's frees release (written before this
  // window), SP1 = the next window's first two space intervals per dynamic op
  const int4 z4 = make_int4(0, 0, 0, 0);
  int4 O1 = start + lane < n2 ? A.ops[start + lane] : z4;
  int4 O2 = start + 32 + lane < n2 ? A.ops[start + 32 + lane] : z4;
  int4 F1 = z4;  // a resumed run's first window: every earlier allocation is in A.res
  if (start > 0 && start + lane < n2 && !(O1.y & 1) && O1.z < start) F1 = A.res[O1.z];
  long long SP1[4] = {0, 0, 0, 0};
  auto load_sp = [&](const int4 &o, long long *sp) {
    sp[0] = sp[1] = sp[2] = sp[3] = 0;
    if (SIM && !A.sp_staged && (o.y & 1) && (o.y >> 1) == RR_DYN) {
      if (o.w > o.z) sp[0] = A.sp_lo[o.z], sp[1] = A.sp_hi[o.z];
      if (o.w > o.z + 1) sp[2] = A.sp_lo[o.z + 1], sp[3] = A.sp_hi[o.z + 1];
    }
  };
  load_sp(O1, SP1);
  for (int64_t w0 = start; w0 < n2; w0 += 32) {
    const int4 O0 = O1;
    const int4 F0 = F1;
    const uint4 SP0 = make_uint4((uint32_t)((unsigned long long)SP1[0] >> sh), (uint32_t)((unsigned long long)SP1[1] >> sh),
                                 (uint32_t)((unsigned long long)SP1[2] >> sh), (uint32_t)((unsigned long long)SP1[3] >> sh));
    O1 = O2;
    O2 = w0 + 64 + lane < n2 ? A.ops[w0 + 64 + lane] : z4;
    F1 = z4;
    if (w0 + 32 + lane < n2 && !(O1.y & 1) && O1.z < w0) F1 = A.res[O1.z];
    load_sp(O1, SP1);
    // this window's frees: allocation of an earlier window (F0) or of the previous one (s_res)
    int4 info = F0;
    if (w0 > start && !(O0.y & 1) && O0.z >= w0 - 32 && O0.z < w0) info = lds128(a_res + 16 * (int)(O0.z - (w0 - 32)));
    __syncwarp();
    sts128(a_op + 16 * lane, O0);
    sts128(a_info + 16 * lane, info);
    if (SIM) sts128(a_sp + 16 * lane, make_int4((int)SP0.x, (int)SP0.y, (int)SP0.z, (int)SP0.w));
    __syncwarp();
    const int cnt = (int)min((int64_t)32, n2 - w0);
    int4 op = lds128(a_op), fi = lds128(a_info);
    for (int k = 0; k < cnt; k++) {
#ifdef STW_REPLAY_PROF
      const long long c0 = clock64();
#endif
      const uint32_t nk = 16 * ((k + 1) & 31);
      const int4 nop = lds128(a_op + nk), nfi = lds128(a_info + nk);  // next op, off the chain
      const uint32_t n = (uint32_t)op.x;
      int4 rec;
      if (op.y & 1) {
        int route = op.y >> 1;
        bool to_cache = true;
        uint32_t a = 0;
        if (SIM && route == RR_PLANNED) {
          a = (uint32_t)op.z;
          const int st = reg_pool_take<RP>(fl, fh, fs, a, n, leq);
          if (st) {
            status = st == 1 ? 2 : 1;
            over = 2;
            err_op = w0 + k;
            err_addr = (long long)a << sh;
            break;
          }
          to_cache = false;
        } else if (SIM && route == RR_DYN) {
          // best fit in free ∩ space (sim.py:120-140, intervals.py:138-176)
          route = RR_FALLBACK;
          if (op.w > op.z) {
            const int4 sp4 = lds128(a_sp + 16 * k);
            const uint4 sp = make_uint4((uint32_t)sp4.x, (uint32_t)sp4.y, (uint32_t)sp4.z, (uint32_t)sp4.w);
            // per lane: its best piece as (length << 32 | address), min over the
            // spaces and rows without branches (ties to the lowest address)
            unsigned long long best = ~0ull;
            for (int j = op.z; j < op.w; j++) {
              uint32_t slo, shi;
              if (A.sp_staged) {
                const uint2 q = s_spc[j];
                slo = q.x, shi = q.y;
              } else if (j == op.z) {
                slo = sp.x, shi = sp.y;
              } else if (j == op.z + 1) {
                slo = sp.z, shi = sp.w;
              } else {
                slo = (uint32_t)((unsigned long long)A.sp_lo[j] >> sh), shi = (uint32_t)((unsigned long long)A.sp_hi[j] >> sh);
              }
#pragma unroll
              for (int r = 0; r < RP; r++) {
                const uint32_t lo = max(fl[r], slo), hi = min(fh[r], shi);
                const unsigned long long k = ((unsigned long long)(hi - lo) << 32) | lo;
                best = hi > lo && hi - lo >= n && k < best ? k : best;
              }
            }
            const uint32_t bl = (uint32_t)(best >> 32), bo = (uint32_t)best;
            const uint32_t m = __reduce_min_sync(kRFull, bl);
            if (m != kRFull) {
              a = __reduce_min_sync(kRFull, bl == m ? bo : kRFull);
              if (reg_pool_take<RP>(fl, fh, fs, a, n, leq)) {  // inside a free interval: only a full state fails
                status = 1;
                over = 2;
                break;
              }
              route = RR_REUSE;
              to_cache = false;
            }
          }
        }
        if (to_cache) {
          uint32_t grown, sb;
          if (!cache_malloc(n, &a, &sb, &grown)) {
            status = 1;
            err_op = w0 + k;  // (resumable unless too_big: the state is untouched)
            over = 1;
            break;
          }
          rec = make_int4((int)a, (int)sb, 1 | (route << 1) | (grown ? 16 : 0), (int)grown);
        } else {
          rec = make_int4((int)a, 0, route << 1, 0);
        }
      } else {
        int4 ai = fi;
        if (op.z >= w0) ai = lds128(a_res + 16 * (op.z - w0));  // allocation of this window: forwarded
        const bool cache = !SIM || (ai.z & 1);
        bool ok;
        if (cache)
          ok = reg_release<R, true>(cl, ch, cs, (uint32_t)ai.x, (uint32_t)ai.x + n, (uint32_t)ai.y, leq);
        else
          ok = reg_release<RP, false>(fl, fh, fs, (uint32_t)ai.x, (uint32_t)ai.x + n, 0, leq);
        if (!ok) {
          status = 1;
          err_op = w0 + k;
          over = cache ? 1 : 2;
          break;
        }
        rec = make_int4(ai.x, 0, ai.z & 1, 0);
      }
      sts128(a_res + 16 * k, rec);  // every lane writes the same record (each later reads its own write)
      __syncwarp();  // later reads of the record by other lanes are ordered after every lane's write (racecheck-clean; no measurable cost)
#ifdef STW_REPLAY_PROF
      {  // cycles per op kind: [0] alloc pool, [1] alloc cache, [2] free pool, [3] free cache
        const int kind = (op.y & 1) ? ((rec.z & 1) ? 1 : 0) : ((rec.z & 1) ? 3 : 2);
        __syncwarp();
        if (lane == 0) {
          atomicAdd(&g_rr_prof[kind][0], (unsigned long long)(clock64() - c0));
          atomicAdd(&g_rr_prof[kind][1], 1ull);
        }
      }
#endif
      op = nop, fi = nfi;
    }
    if (status) {
      done_ops = w0;
      if (!SIM && status == 1 && !too_big) {  // resumable: flush this window's finished ops, dump the rows
        const int kk = (int)(err_op - w0);
        __syncwarp();
        if (lane < kk) A.res[w0 + lane] = lds128(a_res + 16 * lane);
#pragma unroll
        for (int r = 0; r < R; r++) A.dump[r * 32 + lane] = make_int4((int)cl[r], (int)ch[r], (int)cs[r], 0);
        if (lane == 0) A.resume[0] = err_op, A.resume[1] = next_base, A.resume[2] = R;
        done_ops = err_op;
      }
      break;
    }
    __syncwarp();
    if (lane < cnt) A.res[w0 + lane] = lds128(a_res + 16 * lane);
  }
  if (lane == 0) {
    out[0] = status;
    out[1] = over;
    out[3] = err_addr;
    if (status == 2) out[2] = A.ridx ? -1 : A.id[A.operm[err_op] >> 1];  // (off-chain: no planned op replayed)
    out[4] = status == 1 ? done_ops : n2;  // ops replayed before an overflow (diagnostics)
  }
}

// the report (sim.py:67-117) from the per-op results: signed live deltas of
// every op and of the cache ops (peaks: prefix sums + max), and the counts
__global__ void k_reg_metrics(RegArgs A, int64_t *__restrict__ dl, int64_t *__restrict__ dc,
                              unsigned long long *__restrict__ cnt) {
  const int sh = reg_shift(A);
  unsigned long long grown = 0, ng = 0, fb = 0, mm = 0, ru = 0;
  GS4(k, 2 * A.n) {
    const uint32_t o = A.operm[k];
    const long long z = A.size[o >> 1];
    const int4 r = A.res[k];
    const bool alloc = !(o & 1);
    dl[k] = alloc ? z : -z;
    dc[k] = (r.z & 1) ? (alloc ? z : -z) : 0;
    if (alloc) {
      const int route = (r.z >> 1) & 7;
      if (r.z & 16) grown += (unsigned long long)(uint32_t)r.w << sh, ng++;
      fb += route == RR_FALLBACK || route == RR_MISMATCH;
      mm += route == RR_MISMATCH;
      ru += route == RR_REUSE;
    }
  }
  for (int d = 16; d; d >>= 1) {
    grown += __shfl_xor_sync(kRFull, grown, d);
    ng += __shfl_xor_sync(kRFull, ng, d);
    fb += __shfl_xor_sync(kRFull, fb, d);
    mm += __shfl_xor_sync(kRFull, mm, d);
    ru += __shfl_xor_sync(kRFull, ru, d);
  }
  if ((threadIdx.x & 31) == 0) {
    if (grown) atomicAdd(cnt + 0, grown);
    if (ng) atomicAdd(cnt + 1, ng);
    if (fb) atomicAdd(cnt + 2, fb);
    if (mm) atomicAdd(cnt + 3, mm);
    if (ru) atomicAdd(cnt + 4, ru);
  }
}

__global__ void k_max_scan(const int64_t *__restrict__ v, int64_t n, long long *__restrict__ mx);

__global__ void k_reg_grown(const int4 *__restrict__ res, int64_t n2, uint32_t *__restrict__ g) {
  GS4(k, n2) g[k] = (res[k].z & 16) ? 1u : 0u;
}

// the replay log (sim.py:171-229 record order) from the per-op results:
// op k's record lands at 1 + k + (reserve records before it), a reserve
// record right before its allocation
__global__ void k_reg_log(RegArgs A, const uint32_t *__restrict__ gex, int8_t *lkind, int8_t *lspace,
                          int8_t *lroute, int64_t *lt, int64_t *lid, int64_t *lsize, int64_t *laddr) {
  const int sh = reg_shift(A);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    lkind[0] = 0, lt[0] = 0, lid[0] = 0, lsize[0] = A.baseline ? 0 : A.pool, lspace[0] = 0, laddr[0] = 0,
    lroute[0] = -1;
  }
  GS4(k, 2 * A.n) {
    const uint32_t o = A.operm[k];
    const int e = (int)(o >> 1);
    const bool alloc = !(o & 1);
    const int4 r = A.res[k];
    int64_t p = 1 + k + gex[k];
    const long long t = alloc ? A.ts[e] : A.te[e];
    if (alloc && (r.z & 16)) {
      lkind[p] = 1, lt[p] = t, lid[p] = 0, lsize[p] = (long long)(uint32_t)r.w << sh, lspace[p] = 0, laddr[p] = 0,
      lroute[p] = -1;
      p++;
    }
    lkind[p] = alloc ? 2 : 3;
    lt[p] = t;
    lid[p] = A.id[e];
    lsize[p] = A.size[e];
    lspace[p] = (int8_t)(r.z & 1);
    laddr[p] = (long long)(uint32_t)r.x << sh;
    lroute[p] = alloc ? (int8_t)((r.z >> 1) & 7) : (int8_t)-1;
  }
}

// off-chain mode: every op's result in full op order -- a planned allocation
// and its free land at the planned address in the pool (route PLANNED)
__global__ void k_reg_expand(RegArgs A, const int4 *__restrict__ rres, int4 *__restrict__ res) {
  const int sh = reg_shift(A);
  GS4(k, 2 * A.n) {
    const int e = (int)(A.operm[k] >> 1);
    res[k] = reg_planned(A, e) ? make_int4((int)((unsigned long long)A.paddr[e] >> sh), 0, 0, 0) : rres[A.ridx[k]];
  }
}

// ---------------------------------------------------------------------------
// Planned static allocations off the sequential chain (simulate).
//
// A planned allocation's outcome is fixed (its planned address, or the
// "occupied" SimulationError); it feeds the chain only through the pool's
// free set, i.e. through (a) the error test of later planned allocations and
// (b) the free-set pieces a dynamic request sees inside its reuse space
// (sim.py:120-140). Both vanish when
//   1. the planned rectangles (event lifespan x planned interval) are pairwise
//      disjoint -- no planned allocation fails against another (the K7 test);
//   2. no planned rectangle meets (space x [t_s, t_e)) for any reuse space of
//      any dynamic request that may take the reuse route -- so no planned
//      interval is live inside a space while a dynamic request of that space
//      is placed or alive (then a dynamic placement never collides with a
//      planned one either, and free ∩ space is the same with or without the
//      planned intervals).
// derive_reuse_map builds spaces that hold this (reuse.py:54-80: the spaces
// avoid every decision live in the key's window). When both hold, the chain
// replays only the dynamic and mismatched requests with the pool's free set
// taken as [0, pool) minus the live dynamic placements, which gives every op
// the result the full replay gives; otherwise the full chain runs (and
// reports the reference's exact error, if any).

struct OffArgs {
  int64_t n;
  const uint32_t *operm;
  const uint8_t *dyn;
  const int8_t *route0;
  const int32_t *ts, *te, *key;
  const int64_t *size, *paddr, *sp_off, *sp_lo, *sp_hi;
  int reuse;
  uint32_t *af, *rank, *keep;
  int32_t *rts, *rte;
  int64_t *rsz, *raddr, *roff;
  int *bad;
};

__device__ __forceinline__ bool off_planned(const OffArgs &A, int e) { return !A.dyn[e] && A.route0[e] == RR_PLANNED; }

__global__ void k_off_flags(OffArgs A) {
  GS4(k, 2 * A.n) {
    const uint32_t o = A.operm[k];
    const bool p = off_planned(A, (int)(o >> 1));
    A.af[k] = p && !(o & 1) ? 1u : 0u;  // planned allocations, in op order
    A.keep[k] = p ? 0u : 1u;            // ops that stay on the chain
  }
}

// the planned rectangles in op order of their allocations ((t_s, id) order)
__global__ void k_off_rects(OffArgs A) {
  GS4(k, 2 * A.n) {
    if (k == 2 * A.n - 1) A.roff[1] = (int64_t)A.rank[k] + A.af[k];
    if (!A.af[k]) continue;
    const int e = (int)(A.operm[k] >> 1);
    const uint32_t r = A.rank[k];
    A.rts[r] = A.ts[e];
    A.rte[r] = A.te[e];
    A.rsz[r] = A.size[e];
    A.raddr[r] = A.paddr[e];
  }
}

// per reuse key: the hull [min t_s, max t_e) of its dynamic requests
__global__ void k_off_hull(OffArgs A, int32_t *__restrict__ hlo, int32_t *__restrict__ hhi) {
  GS4(e, A.n) {
    if (!A.dyn[e] || !A.reuse) continue;
    const int kk = A.key[e];
    if (kk < 0 || A.sp_off[kk + 1] <= A.sp_off[kk]) continue;
    atomicMin(hlo + kk, A.ts[e]);
    atomicMax(hhi + kk, A.te[e]);
  }
}

// condition 2 on the key's hull (it covers every request of the key, so it
// is sufficient), one CTA per key
__global__ void __launch_bounds__(256) k_off_spaces(OffArgs A, const int32_t *__restrict__ hlo,
                                                    const int32_t *__restrict__ hhi) {
  const int kk = blockIdx.x;
  const int32_t ets = hlo[kk], ete = hhi[kk];
  if (ets >= ete) return;  // no request of this key can take the reuse route
  const int64_t s0 = A.sp_off[kk], s1 = A.sp_off[kk + 1];
  const int ns = s1 - s0 < 4 ? (int)(s1 - s0) : 4;
  long long sl[4], sh[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    sl[q] = q < ns ? A.sp_lo[s0 + q] : 0;
    sh[q] = q < ns ? A.sp_hi[s0 + q] : 0;
  }
  const int64_t np = A.roff[1];
  // rectangles are in t_s order: only those starting before the hull's end can meet it
  int64_t lo = 0, hi = np;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (A.rts[m] < ete)
      lo = m + 1;
    else
      hi = m;
  }
  bool hit = false;
  for (int64_t j = threadIdx.x; j < lo; j += blockDim.x) {
    if (A.rte[j] <= ets) continue;
    const long long a = A.raddr[j], b = a + A.rsz[j];
#pragma unroll
    for (int q = 0; q < 4; q++) hit |= q < ns && a < sh[q] && sl[q] < b;
    for (int64_t s = s0 + 4; s < s1; s++) hit |= a < A.sp_hi[s] && A.sp_lo[s] < b;  // (keys of > 4 spaces)
  }
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(A.bad, 1);
}

bool offchain_check(Ctx &ctx, Arena &ar, RegIn &in, int64_t nkeys) {
  in.ridx = nullptr;
  in.nkept = 2 * in.n;
  const int64_t n = in.n, n2 = 2 * n;
  if (!ctx.ok() || in.baseline || n <= 0 || n > (1 << 20)) return false;
  OffArgs A{n, in.operm, in.dyn, in.route0, in.ts, in.te, in.key, in.size, in.paddr, in.sp_off, in.sp_lo, in.sp_hi,
            in.reuse};
  A.af = ar.take<uint32_t>(n2);
  A.rank = ar.take<uint32_t>(n2);
  A.keep = ar.take<uint32_t>(n2);
  A.rts = ar.take<int32_t>(n + 1);
  A.rte = ar.take<int32_t>(n + 1);
  A.rsz = ar.take<int64_t>(n + 1);
  A.raddr = ar.take<int64_t>(n + 1);
  A.roff = ar.take<int64_t>(2);
  A.bad = ar.take<int>(1);
  uint32_t *ridx = ar.take<uint32_t>(n2);
  if (!ctx.ok()) return false;
  STW_CUDA(ctx, cudaMemsetAsync(A.roff, 0, 2 * sizeof(int64_t), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(A.bad, 0, sizeof(int), ctx.stream));
  STW_KL(k_off_flags, grid_for(n2, 256), 256, ctx.stream, A);
  device_scan<uint32_t>(ctx, ar, A.af, A.rank, n2, false);
  device_scan<uint32_t>(ctx, ar, A.keep, ridx, n2, false);
  STW_KL(k_off_rects, grid_for(n2, 256), 256, ctx.stream, A);
  STW_LAUNCHED(ctx);
  if (in.reuse && nkeys > 0) {
    int32_t *hlo = ar.take<int32_t>(nkeys), *hhi = ar.take<int32_t>(nkeys);
    if (!ctx.ok()) return false;
    STW_CUDA(ctx, cudaMemsetAsync(hlo, 0x7f, nkeys * sizeof(int32_t), ctx.stream));
    STW_CUDA(ctx, cudaMemsetAsync(hhi, 0, nkeys * sizeof(int32_t), ctx.stream));
    STW_KL(k_off_hull, grid_for(n, 256), 256, ctx.stream, A, hlo, hhi);
    STW_KL(k_off_spaces, (unsigned)nkeys, 256, ctx.stream, A, hlo, hhi);
    STW_LAUNCHED(ctx);
  }
  // condition 1: the exact tiled reporter (the whole GPU on one trace) over the
  // np planned rectangles
  long long np = 0;
  STW_CUDA(ctx, cudaMemcpyAsync(&np, A.roff + 1, sizeof(long long), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok() || np == 0) return false;
  RectSets rs{1, np, A.roff, A.rts, A.rte, A.rsz, 1, A.raddr};
  long long *cnt = ar.take<long long>(1);
  int *first = ar.take<int>(1);
  if (!ctx.ok()) return false;
  validate_exact(ctx, ar, rs, cnt, first);
  if (!ctx.ok()) return false;
  long long hf = 1;
  int hb = 1;
  STW_CUDA(ctx, cudaMemcpyAsync(&hf, cnt, sizeof(long long), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaMemcpyAsync(&hb, A.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok() || hf != 0 || hb != 0) return false;
  in.ridx = ridx;
  in.nkept = n2 - 2 * np;
  return true;
}

// Runs the register-resident replay; returns 0 when it produced the result
// (hout[4..10] = metrics, log written when asked), 1 when the call must fall
// back to k_replay (state or values outside the preconditions), 2 on a replay
// error (hout[2] id, hout[3] address).
int replay_reg(Ctx &ctx, Arena &ar, RegIn &in, long long *hout, stw_log *log) {
  if (!ctx.ok()) return 1;
  const int64_t n = in.n, n2 = 2 * n;
  RegArgs A{};
  A.n = n;
  A.operm = in.operm;
  A.apos = in.apos;
  A.id = in.id;
  A.size = in.size;
  A.ts = in.ts;
  A.te = in.te;
  A.dyn = in.dyn;
  A.route0 = in.route0;
  A.paddr = in.paddr;
  A.key = in.key;
  A.sp_off = in.sp_off;
  A.sp_lo = in.sp_lo;
  A.sp_hi = in.sp_hi;
  A.nsp = in.nsp;
  A.reuse = in.reuse;
  A.baseline = in.baseline;
  A.pool = in.pool;
  A.ridx = in.ridx;
  A.nops = in.ridx ? in.nkept : n2;
  A.unit = ar.take<unsigned long long>(2);
  A.ops = ar.take<int4>(A.nops + 1);
  A.res = ar.take<int4>(A.nops + 1);
  A.out = ar.take<long long>(16);
  A.resume = ar.take<long long>(4);
  A.dump = ar.take<int4>(16 * 32);
  if (!ctx.ok()) return 1;
  STW_CUDA(ctx, cudaMemsetAsync(A.resume, 0, 4 * sizeof(long long), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(A.unit, 0, 2 * sizeof(unsigned long long), ctx.stream));
  STW_KL(k_reg_unit, grid_for(std::max<int64_t>(n, in.nsp), 256, 148 * 8), 256, ctx.stream, A);
  STW_KL(k_reg_ops, grid_for(n2, 256), 256, ctx.stream, A);
  // rows per lane (32 blocks / intervals per row): a run that outgrows them
  // restarts with more rows for the structure that overflowed (the state
  // grows early in a trace, so failed runs are short). Simulate: the pool's
  // free set has one row (c3: at most 3 intervals) or as many as the cache.
  const bool sim = !in.baseline;
  A.sp_staged = sim && in.nsp > 0 && in.nsp <= kSpSmemMax;
  const int sp_smem = A.sp_staged ? (int)(in.nsp * sizeof(uint2)) : 0;
  int rc = 1, rp = 1;
  hout[0] = 1;
  while (hout[0] == 1 && rc <= 16) {  // (rc beyond 16: the general warp)
    bool launched = false;
#define STW_RR(RC)                                                                                       \
  if (rc == RC) {                                                                                        \
    if (!sim) {                                                                                          \
      STW_KL((k_replay_reg<RC, 1, false>), 1, 32, ctx.stream, A);                                        \
    } else if (rp == 1) {                                                                                \
      cudaFuncSetAttribute(k_replay_reg<RC, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp_smem); \
      STW_KLS((k_replay_reg<RC, 1, true>), 1, 32, sp_smem, ctx.stream, A);                               \
    } else {                                                                                             \
      cudaFuncSetAttribute(k_replay_reg<RC, RC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp_smem); \
      STW_KLS((k_replay_reg<RC, RC, true>), 1, 32, sp_smem, ctx.stream, A);                              \
    }                                                                                                    \
    launched = true;                                                                                     \
  }
    STW_RR(1) STW_RR(2) STW_RR(3) STW_RR(5) STW_RR(8) STW_RR(16)
#undef STW_RR
    if (!launched) break;
    STW_LAUNCHED(ctx);
    STW_CUDA(ctx, cudaMemcpyAsync(hout, A.out, 16 * sizeof(long long), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    if (!ctx.ok()) return 1;
#ifdef STW_REPLAY_CLOCK
    fprintf(stderr, "replay_reg rows=%d/%d ops=%lld: status %lld over %lld after %lld ops\n", rc, rp, (long long)n2,
            hout[0], hout[1], hout[4]);
#endif
#ifdef STW_REPLAY_PROF
    {
      unsigned long long hp[4][2];
      cudaMemcpyFromSymbol(hp, g_rr_prof, sizeof(hp));
      const char *nm[4] = {"alloc pool", "alloc cache", "free pool", "free cache"};
      for (int q = 0; q < 4; q++)
        if (hp[q][1]) fprintf(stderr, "  %s: %llu ops, %.0f cycles/op\n", nm[q], hp[q][1], (double)hp[q][0] / hp[q][1]);
      unsigned long long z[4][2] = {};
      cudaMemcpyToSymbol(g_rr_prof, z, sizeof(z));
    }
#endif
    if (hout[0] != 1) break;
    // the baseline resumes where the cache outgrew its rows (A.resume / A.dump
    // were written); a simulate run restarts from the first op
    if (hout[1] == 2 && sim && rp < rc) {  // pool outgrew its single row
      rp = rc;
    } else {  // 1 -> 2 -> 3 -> 5 -> 8 -> 16 rows (32 blocks each): c1 29, c3 68, c5 129 blocks
      rc = rc == 1 ? 2 : rc == 2 ? 3 : rc == 3 ? 5 : rc == 5 ? 8 : 16 * (rc / 8 + 1);
      rp = rp == 1 ? 1 : rc;
    }
    if (sim || hout[1] != 1) STW_CUDA(ctx, cudaMemsetAsync(A.resume, 0, 4 * sizeof(long long), ctx.stream));
  }
  if (hout[0] != 0) return (int)hout[0];
  if (A.ridx) {  // every op's result in full op order
    int4 *full = ar.take<int4>(n2 + 1);
    if (!ctx.ok()) return 1;
    STW_KL(k_reg_expand, grid_for(n2, 256), 256, ctx.stream, A, A.res, full);
    STW_LAUNCHED(ctx);
    A.res = full;
    A.ridx = nullptr;
    A.nops = n2;
  }
  // metrics
  int64_t *dl = ar.take<int64_t>(n2), *dc = ar.take<int64_t>(n2);
  unsigned long long *cnt = ar.take<unsigned long long>(8);
  long long *pk = ar.take<long long>(2);
  if (!ctx.ok()) return 1;
  STW_CUDA(ctx, cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(pk, 0, 2 * sizeof(long long), ctx.stream));
  STW_KL(k_reg_metrics, grid_for(n2, 256, 148 * 8), 256, ctx.stream, A, dl, dc, cnt);
  device_scan<int64_t>(ctx, ar, dl, dl, n2, true);
  device_scan<int64_t>(ctx, ar, dc, dc, n2, true);
  STW_KL(k_max_scan, grid_for(n2, 256, 148 * 4), 256, ctx.stream, dl, n2, pk);
  STW_KL(k_max_scan, grid_for(n2, 256, 148 * 4), 256, ctx.stream, dc, n2, pk + 1);
  unsigned long long hc[8];
  long long hpk[2];
  STW_CUDA(ctx, cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaMemcpyAsync(hpk, pk, sizeof(hpk), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok()) return 1;
  hout[4] = hpk[0];
  hout[5] = (long long)hc[0];
  hout[6] = hpk[1];
  hout[7] = (long long)hc[2];
  hout[8] = (long long)hc[4];
  hout[9] = (long long)hc[3];
  hout[10] = (long long)hc[1];
  if (log) {
    const int64_t nlog = 1 + n2 + hout[10];
    uint32_t *g = ar.take<uint32_t>(n2 + 1);
    int8_t *lkind = ar.take<int8_t>(nlog), *lspace = ar.take<int8_t>(nlog), *lroute = ar.take<int8_t>(nlog);
    int64_t *lt = ar.take<int64_t>(nlog), *lid = ar.take<int64_t>(nlog), *lsize = ar.take<int64_t>(nlog),
            *laddr = ar.take<int64_t>(nlog);
    if (!ctx.ok()) return 1;
    if (n2) {
      STW_KL(k_reg_grown, grid_for(n2, 256), 256, ctx.stream, A.res, n2, g);
      device_scan<uint32_t>(ctx, ar, g, g, n2, false);
    }
    STW_KL(k_reg_log, grid_for(n2 + 1, 256), 256, ctx.stream, A, g, lkind, lspace, lroute, lt, lid, lsize, laddr);
    STW_LAUNCHED(ctx);
    log->len = nlog;
    const int64_t m = std::min<int64_t>(nlog, log->cap);
    if (m > 0) {
      STW_CUDA(ctx, cudaMemcpyAsync(log->kind, lkind, m, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->space, lspace, m, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->route, lroute, m, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->t, lt, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->id, lid, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->size, lsize, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->addr, laddr, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
    }
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    if (!ctx.ok()) return 1;
  }
  return 0;
}

}  // namespace stw
