// K7 -- tiled pairwise (time x address) rectangle validator reproducing the
// reference sweep (validate_plan, planner.py:476-505) exactly.
//
// The sweep visits allocations in (t_s, id) order ("sweep position" r). When
// decision d is allocated, the active set is {c : r(c) < r(d), t_e(c) > t_s(d)}
// (frees precede allocs at equal t). The reference reports
//   * (pred, d) where pred is the active decision at the insertion point
//     minus one of the address-sorted active list -- the largest address below
//     d.addr, ties to the earliest inserted -- if pred.end > d.addr, and
//   * (c, d) for every active c with d.addr <= c.addr < d.end, in list order
//     (address ascending, ties most recently inserted first).
// It under-reports on invalid plans; reproducing it keeps
// validate_plan's output identical.
//
// Tiling: each set's sweep-ordered rectangles are cut into tiles of kTile.
// The decisions still live when tile b starts (r < first(b), t_e > T0(b)) are
// listed per tile once (a stabbing list built with a difference array + two
// scans); one CTA then checks every decision of the tile against that list
// and the tile's own earlier decisions from shared memory.
#include <algorithm>
#include <vector>

#include "planner.cuh"

namespace stw {

constexpr int kTile = 128;
constexpr int kLiveSmem = 1024;

#define GS(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

struct Tiles {
  int64_t NB;
  const int64_t *bo;  // [S+1] first tile of each set
  int32_t *bset;      // [NB]
  int32_t *T0;        // [NB] t_s of the tile's first decision
  int64_t *loff;      // [NB+1] live list offsets
  int32_t *live;      // set-local positions
};

__global__ void k_tile_meta(const int64_t *__restrict__ off, const int64_t *__restrict__ bo, int S,
                            const int32_t *__restrict__ ts, int32_t *__restrict__ bset, int32_t *__restrict__ T0,
                            int64_t NB) {
  GS(b, NB) {
    int a = 0, z = S;  // set of tile b
    while (z - a > 1) {
      int m = (a + z) >> 1;
      if (bo[m] <= b)
        a = m;
      else
        z = m;
    }
    while (bo[a + 1] <= b) a++;
    bset[b] = a;
    T0[b] = ts[off[a] + (b - bo[a]) * kTile];
  }
}

// last tile of set s (tiles [b0, b1)) whose start time is < te
__device__ __forceinline__ int64_t last_tile_before(const int32_t *__restrict__ T0, int64_t b0, int64_t b1, int te) {
  int64_t lo = b0, hi = b1;  // first tile with T0 >= te
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (T0[m] < te)
      lo = m + 1;
    else
      hi = m;
  }
  return lo - 1;
}

__global__ void k_live_count(const int64_t *__restrict__ off, int S, int64_t n, const int32_t *__restrict__ ts,
                             const int32_t *__restrict__ te, const int64_t *__restrict__ bo,
                             const int32_t *__restrict__ T0, int *__restrict__ diff) {
  GS(k, n) {
    int a = 0, z = S;
    while (z - a > 1) {
      int m = (a + z) >> 1;
      if (off[m] <= k)
        a = m;
      else
        z = m;
    }
    while (off[a + 1] <= k) a++;
    int64_t b = bo[a] + (k - off[a]) / kTile;
    int64_t last = last_tile_before(T0, b + 1, bo[a + 1], te[k]);
    if (last > b) {
      atomicAdd(diff + b + 1, 1);
      atomicAdd(diff + last + 1, -1);
    }
  }
}

// a decision live into more than kLongSpan later tiles (c5's persistent
// allocations span thousands) is handed to k_live_fill_long, where a CTA
// spreads its tiles over the threads, instead of one thread walking them
constexpr int64_t kLongSpan = 32;

__global__ void k_live_fill(const int64_t *__restrict__ off, int S, int64_t n, const int32_t *__restrict__ te,
                            const int64_t *__restrict__ bo, const int32_t *__restrict__ T0,
                            const int64_t *__restrict__ loff, int *__restrict__ cursor, int32_t *__restrict__ live,
                            int *__restrict__ nlong, int4 *__restrict__ longs) {
  GS(k, n) {
    int a = 0, z = S;
    while (z - a > 1) {
      int m = (a + z) >> 1;
      if (off[m] <= k)
        a = m;
      else
        z = m;
    }
    while (off[a + 1] <= k) a++;
    int64_t b = bo[a] + (k - off[a]) / kTile;
    int64_t last = last_tile_before(T0, b + 1, bo[a + 1], te[k]);
    if (last - b > kLongSpan) {  // (tile indices < 2^31: the batch guard caps n)
      longs[atomicAdd(nlong, 1)] = make_int4((int)(b + 1), (int)last, (int)(k - off[a]), 0);
      continue;
    }
    for (int64_t x = b + 1; x <= last; x++) {
      int slot = atomicAdd(cursor + x, 1);
      live[loff[x] + slot] = (int32_t)(k - off[a]);
    }
  }
}

__global__ void k_live_fill_long(const int *__restrict__ nlong, const int4 *__restrict__ longs,
                                 const int64_t *__restrict__ loff, int *__restrict__ cursor,
                                 int32_t *__restrict__ live) {
  for (int i = blockIdx.x; i < *nlong; i += gridDim.x) {
    const int4 q = longs[i];
    for (int x = q.x + threadIdx.x; x <= q.y; x += blockDim.x) {
      const int slot = atomicAdd(cursor + x, 1);
      live[loff[x] + slot] = q.z;
    }
  }
}

struct Cand {
  long long addr, end;
  int ts, te, r;
};

// per-decision evaluation of the reference report; returns the count and
// (optionally) the predecessor
__device__ __forceinline__ void eval_one(const Cand &d, const Cand &c, long long &pa, int &pr, long long &pend,
                                         int &fwd) {
  if (c.te <= d.ts) return;  // freed before d is allocated
  if (c.addr < d.addr) {
    if (c.addr > pa || (c.addr == pa && c.r < pr)) {
      pa = c.addr;
      pr = c.r;
      pend = c.end;
    }
  } else if (c.addr < d.end) {
    fwd++;
  }
}

// One CTA per (tile, candidate). Writes per-decision report counts (optional)
// and per-unit totals / first reporting position.
__global__ void __launch_bounds__(kTile) k_validate_tiles(RectSets rs, Tiles tl, long long *__restrict__ count,
                                                          int *__restrict__ first, int32_t *__restrict__ per_d) {
  const int64_t b = blockIdx.x;
  const int c = blockIdx.y;
  const int s = tl.bset[b];
  const int64_t s0 = rs.off[s], s1 = rs.off[s + 1];
  const int64_t k0 = s0 + (b - tl.bo[s]) * kTile;
  const int nb = (int)min((int64_t)kTile, s1 - k0);
  const int64_t *addr = rs.addr + (int64_t)c * rs.n;
  __shared__ Cand tile[kTile];
  __shared__ Cand lv[kLiveSmem];
  __shared__ long long sh_cnt;
  __shared__ int sh_first;
  const int tid = threadIdx.x;
  if (tid == 0) {
    sh_cnt = 0;
    sh_first = INT_MAX;
  }
  if (tid < nb) {
    int64_t k = k0 + tid;
    tile[tid] = Cand{addr[k], addr[k] + rs.size[k], rs.ts[k], rs.te[k], (int)(k - s0)};
  }
  const int64_t l0 = tl.loff[b], nl = tl.loff[b + 1] - l0;
  Cand d{};
  long long pa = LLONG_MIN, pend = 0;
  int pr = INT_MAX, fwd = 0;
  __syncthreads();
  if (tid < nb) d = tile[tid];
  for (int64_t cb = 0; cb < nl; cb += kLiveSmem) {
    int m = (int)min((int64_t)kLiveSmem, nl - cb);
    __syncthreads();
    for (int x = tid; x < m; x += blockDim.x) {
      int64_t k = s0 + tl.live[l0 + cb + x];
      lv[x] = Cand{addr[k], addr[k] + rs.size[k], rs.ts[k], rs.te[k], (int)(k - s0)};
    }
    __syncthreads();
    if (tid < nb)
      for (int x = 0; x < m; x++) eval_one(d, lv[x], pa, pr, pend, fwd);
  }
  int cnt = 0;
  if (tid < nb) {
    for (int x = 0; x < tid; x++) eval_one(d, tile[x], pa, pr, pend, fwd);
    cnt = fwd + ((pa != LLONG_MIN && pend > d.addr) ? 1 : 0);
    if (per_d) per_d[k0 + tid] = cnt;
    if (cnt) {
      atomicAdd((unsigned long long *)&sh_cnt, (unsigned long long)cnt);
      atomicMin(&sh_first, d.r);
    }
  }
  __syncthreads();
  if (tid == 0 && sh_cnt) {
    int64_t u = (int64_t)s * rs.n_cand + c;
    atomicAdd((unsigned long long *)(count + u), (unsigned long long)sh_cnt);
    atomicMin(first + u, sh_first);
  }
}

static void build_tiles(Ctx &ctx, Arena &ar, const RectSets &rs, Tiles *tl) {
  std::vector<int64_t> off(rs.S + 1), bo(rs.S + 1, 0);
  if (rs.S > 0)
    STW_CUDA(ctx, cudaMemcpyAsync(off.data(), rs.off, (rs.S + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  for (int s = 0; s < rs.S; s++) bo[s + 1] = bo[s] + (off[s + 1] - off[s] + kTile - 1) / kTile;
  tl->NB = bo[rs.S];
  int64_t *dbo = ar.take<int64_t>(rs.S + 1);
  tl->bo = dbo;
  tl->bset = ar.take<int32_t>(tl->NB + 1);
  tl->T0 = ar.take<int32_t>(tl->NB + 1);
  tl->loff = ar.take<int64_t>(tl->NB + 2);
  int *diff = ar.take<int>(tl->NB + 2);
  int *cnt = ar.take<int>(tl->NB + 2);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemcpyAsync(dbo, bo.data(), (rs.S + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(diff, 0, (tl->NB + 2) * sizeof(int), ctx.stream));
  if (tl->NB == 0) return;
  STW_KL(k_tile_meta, grid_for(tl->NB, 256), 256, ctx.stream, rs.off, dbo, rs.S, rs.ts, tl->bset, tl->T0, tl->NB);
  STW_KL(k_live_count, grid_for(rs.n, 256), 256, ctx.stream, rs.off, rs.S, rs.n, rs.ts, rs.te, dbo, tl->T0, diff);
  STW_LAUNCHED(ctx);
  device_scan<int>(ctx, ar, diff, cnt, tl->NB + 1, true);  // cnt[b] = live entries of tile b
  if (!ctx.ok()) return;
  {
    std::vector<int> h(tl->NB + 1);
    STW_CUDA(ctx, cudaMemcpyAsync(h.data(), cnt, (tl->NB + 1) * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    std::vector<int64_t> lo(tl->NB + 2, 0);
    for (int64_t b = 0; b < tl->NB; b++) lo[b + 1] = lo[b] + h[b];
    STW_CUDA(ctx, cudaMemcpyAsync(tl->loff, lo.data(), (tl->NB + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                  ctx.stream));
    tl->live = ar.take<int32_t>(lo[tl->NB] + 1);
  }
  int *cursor = ar.take<int>(tl->NB + 2);  // [NB + 1]: the long-span count
  int4 *longs = ar.take<int4>(rs.n + 1);
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemsetAsync(cursor, 0, (tl->NB + 2) * sizeof(int), ctx.stream));
  STW_KL(k_live_fill, grid_for(rs.n, 256), 256, ctx.stream, rs.off, rs.S, rs.n, rs.te, dbo, tl->T0, tl->loff, cursor,
         tl->live, cursor + tl->NB + 1, longs);
  STW_KL(k_live_fill_long, 148 * 2, 256, ctx.stream, cursor + tl->NB + 1, longs, tl->loff, cursor, tl->live);
  STW_LAUNCHED(ctx);
}


// ---------------------------------------------------------------------------
// Fast path: exact "does the reference report anything" test, one warp per
// (set, candidate). The reference reports at least one pair iff some decision
// overlaps (address x half-open lifespan) a decision allocated before it in
// sweep order (the first such decision reports its predecessor or a forward
// neighbour: any other active rectangle it could hit would itself have been a
// conflict earlier), so a valid plan needs only the overlap test. The warp
// sweeps 32 decisions at a time, scaled to int4 (address and end in units of
// 2^shift, t_s, t_e). The active list -- decisions still live at the tile
// start -- is kept sorted by address; while no conflict has been seen its
// entries are pairwise disjoint, so each lane finds the entries meeting its
// address range by binary search (O(log active) instead of a scan of the
// list). The tile's earlier decisions are tested pairwise from shared memory.
// Between tiles the entries that end before the next tile starts are
// compacted away and the tile's surviving decisions merged in. The rectangles
// stream through once (24 B each, next tile prefetched). A unit that
// conflicts, does not scale to 32 bits, overflows the active list, or is too
// long for a serial sweep is flagged and the exact tiled reporter above runs
// instead.
#ifdef STW_K7_STATS
__device__ unsigned long long g_k7_stats[4];  // max active, sum active, tiles, sum survivors
#endif
constexpr int kOvWarps = 8;
constexpr int kOvCap = 320;
constexpr int64_t kOvMaxSerial = 1 << 16;

__global__ void __launch_bounds__(kOvWarps * 32, 5) k_overlap_sweep(RectSets rs, int shift, int *__restrict__ nflag,
                                                                    const int32_t *__restrict__ order) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ int4 act[kOvWarps][kOvCap];
  __shared__ int4 tile[kOvWarps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * kOvWarps + w;
  if (u >= (int64_t)rs.S * rs.n_cand) return;
  const int s = order ? order[u / rs.n_cand] : (int)(u / rs.n_cand), c = (int)(u % rs.n_cand);
  const int64_t s0 = rs.off[s], n = rs.off[s + 1] - s0;
  if (n > kOvMaxSerial) {
    if (lane == 0) atomicAdd(nflag, 1);
    return;
  }
  const int64_t *addr = rs.addr + (int64_t)c * rs.n + s0, *size = rs.size + s0;
  const int32_t *ts = rs.ts + s0, *te = rs.te + s0;
  int4 *A = act[w], *Tt = tile[w];
  const long long low = (1ll << shift) - 1;
  const unsigned lt = lanemask_lt();
  int na = 0;
  long long pa = 0, psz = 0;
  int pts = 0, pte = 0;
  if (lane < n) {
    pa = addr[lane];
    psz = size[lane];
    pts = ts[lane];
    pte = te[lane];
  }
  for (int64_t k0 = 0; k0 < n; k0 += 32) {
    const bool valid = k0 + lane < n;
    const long long a = pa, sz = psz;
    const int dts = pts, dte = pte;
    const int64_t kn = k0 + 32 + lane;
    pa = psz = 0;  // past the end: an empty rectangle
    pts = pte = 0;
    if (kn < n) {
      pa = addr[kn];
      psz = size[kn];
      pts = ts[kn];
      pte = te[kn];
    }
    const long long end = a + sz;
    const bool ok = !valid || (a >= 0 && sz > 0 && dts >= 0 && dte > dts && ((a | sz) & low) == 0 && (end >> shift) <= INT_MAX);
    if (__any_sync(FULL, !ok)) {
      if (lane == 0) atomicAdd(nflag, 1);
      return;
    }
    const int da = (int)(a >> shift), de = (int)(end >> shift);
    const int4 mine = make_int4(da, de, dts, dte);  // all zero past the end: meets nothing
    Tt[lane] = mine;
    __syncwarp();
    bool hit = false;
    if (valid) {
      // The active list is address-sorted and pairwise disjoint (its entries are all
      // live at the tile start and were checked against each other), so the entries
      // meeting [da, de) are a contiguous run from the first one ending above da;
      // any of them still live at dts is a conflict.
      int lo = 0, hi = na;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid].y > da)
          hi = mid;
        else
          lo = mid + 1;
      }
      for (int q = lo; q < na; q++) {
        const int4 e = A[q];
        if (e.x >= de) break;
        if (e.w > dts) {
          hit = true;
          break;
        }
      }
    }
    // the tile's decisions among themselves, each unordered pair once: lane i meets
    // lane i - o (mod 32), o = 1..16. Overlap <=> (c.addr - d.end), (d.addr - c.end),
    // (d.ts - c.te) and (c.ts - d.te) all negative: the sign bit of their AND
    // (operands in [0, 2^31)); for a pair in sweep order the last one always is.
    int acc = 0;
#pragma unroll
    for (int o = 1; o <= 16; o++) {
      const int4 q = Tt[(lane - o) & 31];
      acc |= (q.x - de) & (da - q.y) & (dts - q.w) & (q.z - dte);
    }
    hit |= acc < 0;
    if (__any_sync(FULL, hit)) {
      if (lane == 0) atomicAdd(nflag, 1);
      return;
    }
    if (k0 + 32 >= n) break;  // nothing reads the list after the last tile
    // 1. drop the entries that end by the tile's last start (order kept). What
    // stays is live at that instant, hence pairwise checked and disjoint.
    const int t0n = __shfl_sync(FULL, dts, 31);
    int nn = 0;
    for (int cb = 0; cb < na; cb += 32) {
      const int j = cb + lane;
      const int4 q = j < na ? A[j] : make_int4(0, 0, 0, 0);
      const bool keep = j < na && q.w > t0n;
      const unsigned m = __ballot_sync(FULL, keep);
      __syncwarp();
      if (keep) A[nn + __popc(m & lt)] = q;
      nn += __popc(m);
      __syncwarp();
    }
    // 2. the tile's decisions still live then, merged in address order
    const bool keep = valid && dte > t0n;
    const unsigned m = __ballot_sync(FULL, keep);
    const int ns = __popc(m);
    if (nn + ns > kOvCap) {
      if (lane == 0) atomicAdd(nflag, 1);
      return;
    }
    if (ns) {
      int rk = 0;  // rank among the survivors (addresses distinct: pairwise disjoint)
      for (unsigned mm = m; mm; mm &= mm - 1) rk += __shfl_sync(FULL, da, __ffs(mm) - 1) < da ? 1 : 0;
      int pos = 0;  // survivors' slot: old entries below it + survivors below it
      if (keep) {
        int lo = 0, hi = nn;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (A[mid].x < da)
            lo = mid + 1;
          else
            hi = mid;
        }
        pos = lo + rk;
      }
      __syncwarp();
      if (keep) Tt[rk] = mine;  // survivors sorted by address
      __syncwarp();
      // old entry i moves up by the survivors below it; back to front, a chunk is
      // read before the next one down overwrites it, and destinations increase
      for (int cb = (nn - 1) & ~31; cb >= 0; cb -= 32) {
        const int j = cb + lane;
        int4 q = make_int4(0, 0, 0, 0);
        int dst = j;
        if (j < nn) {
          q = A[j];
          int lo = 0, hi = ns;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (Tt[mid].x < q.x)
              lo = mid + 1;
            else
              hi = mid;
          }
          dst = j + lo;
        }
        __syncwarp();
        if (j < nn && dst != j) A[dst] = q;
        __syncwarp();
      }
      if (keep) A[pos] = mine;
    }
    na = nn + ns;
#ifdef STW_K7_STATS
    if (lane == 0) {
      atomicMax(&g_k7_stats[0], (unsigned long long)na);
      atomicAdd(&g_k7_stats[1], (unsigned long long)na);
      atomicAdd(&g_k7_stats[2], 1ull);
      atomicAdd(&g_k7_stats[3], (unsigned long long)ns);
    }
#endif
    __syncwarp();
  }
}

// launches the fast test; returns the device counter of units that need the
// exact reporter (valid after the stream reaches it)
int *overlap_launch(Ctx &ctx, Arena &ar, const RectSets &rs, int shift, const int32_t *order) {
  if (!ctx.ok()) return nullptr;
  const int64_t U = (int64_t)rs.S * rs.n_cand;
  int *nflag = ar.take<int>(1);
  if (!ctx.ok()) return nullptr;
  STW_CUDA(ctx, cudaMemsetAsync(nflag, 0, sizeof(int), ctx.stream));
  if (U > 0) {
    STW_KL(k_overlap_sweep, (unsigned)((U + kOvWarps - 1) / kOvWarps), kOvWarps * 32, ctx.stream, rs, shift, nflag,
           order);
    STW_LAUNCHED(ctx);
  }
  return nflag;
}

int overlap_flags(Ctx &ctx, Arena &ar, const RectSets &rs, int shift) {
  int *nflag = overlap_launch(ctx, ar, rs, shift);
  if (!nflag) return -1;
#ifdef STW_K7_STATS
  {
    unsigned long long h[4];
    cudaStreamSynchronize(ctx.stream);
    cudaMemcpyFromSymbol(h, g_k7_stats, sizeof(h));
    fprintf(stderr, "K7: max active %llu, mean active %.1f, mean survivors %.1f over %llu tiles\n", h[0],
            (double)h[1] / h[2], (double)h[3] / h[2], h[2]);
    unsigned long long z[4] = {};
    cudaMemcpyToSymbol(g_k7_stats, z, sizeof(z));
  }
#endif
  int h = 0;
  STW_CUDA(ctx, cudaMemcpyAsync(&h, nflag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  return ctx.ok() ? h : -1;
}

void validate_sets(Ctx &ctx, Arena &ar, const RectSets &rs, long long *d_count, int *d_first, int shift) {
  if (!ctx.ok()) return;
  int64_t U = (int64_t)rs.S * rs.n_cand;
  STW_CUDA(ctx, cudaMemsetAsync(d_count, 0, U * sizeof(long long), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(d_first, 0x7f, U * sizeof(int), ctx.stream));  // 0x7f7f7f7f: no report
  // one warp per unit: with few units the serial sweep leaves the GPU idle, and
  // the tiled reporter (CTA per 128-decision tile) is faster outright
  if (U >= 148 && overlap_flags(ctx, ar, rs, shift) == 0) return;  // every unit valid: nothing reported
  validate_exact(ctx, ar, rs, d_count, d_first);
}

// the exact tiled reporter over every unit (counts and first reporting position)
void validate_exact(Ctx &ctx, Arena &ar, const RectSets &rs, long long *d_count, int *d_first) {
  if (!ctx.ok()) return;
  int64_t U = (int64_t)rs.S * rs.n_cand;
  STW_CUDA(ctx, cudaMemsetAsync(d_count, 0, U * sizeof(long long), ctx.stream));
  std::vector<int> big(U, INT_MAX);
  STW_CUDA(ctx, cudaMemcpyAsync(d_first, big.data(), U * sizeof(int), cudaMemcpyHostToDevice, ctx.stream));
  Tiles tl;
  build_tiles(ctx, ar, rs, &tl);
  if (!ctx.ok() || tl.NB == 0) {
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    return;
  }
  dim3 grid((unsigned)tl.NB, (unsigned)rs.n_cand);
  STW_KL(k_validate_tiles, grid, kTile, ctx.stream, rs, tl, d_count, d_first, nullptr);
  STW_LAUNCHED(ctx);
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
}

// Error path only: rebuild the first reported pair of one unit on the host.
void first_pair(Ctx &ctx, const RectSets &rs, int set, int cand, int first, int *pa, int *pb) {
  *pa = *pb = -1;
  std::vector<int64_t> off(rs.S + 1);
  STW_CUDA(ctx, cudaMemcpy(off.data(), rs.off, (rs.S + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  int64_t s0 = off[set], n = off[set + 1] - s0;
  if (first < 0 || first >= n) return;
  std::vector<int64_t> ad(n), sz(n);
  std::vector<int32_t> ts(n), te(n);
  STW_CUDA(ctx, cudaMemcpy(ad.data(), rs.addr + (int64_t)cand * rs.n + s0, n * 8, cudaMemcpyDeviceToHost));
  STW_CUDA(ctx, cudaMemcpy(sz.data(), rs.size + s0, n * 8, cudaMemcpyDeviceToHost));
  STW_CUDA(ctx, cudaMemcpy(ts.data(), rs.ts + s0, n * 4, cudaMemcpyDeviceToHost));
  STW_CUDA(ctx, cudaMemcpy(te.data(), rs.te + s0, n * 4, cudaMemcpyDeviceToHost));
  if (!ctx.ok()) return;
  const int d = first;
  long long best = LLONG_MIN;
  int pr = INT_MAX;
  long long fa = LLONG_MAX;
  int fr = -1;
  for (int c = 0; c < d; c++) {
    if (te[c] <= ts[d]) continue;
    if (ad[c] < ad[d]) {
      if (ad[c] > best || (ad[c] == best && c < pr)) best = ad[c], pr = c;
    } else if (ad[c] < ad[d] + sz[d]) {
      if (ad[c] < fa || (ad[c] == fa && c > fr)) fa = ad[c], fr = c;
    }
  }
  if (pr != INT_MAX && ad[pr] + sz[pr] > ad[d])
    *pa = pr;
  else
    *pa = fr;
  *pb = d;
}

// ---------------------------------------------------------------------------
// standalone validate_plan with the full ordered pair list

__global__ void k_pairs(RectSets rs, Tiles tl, const int64_t *__restrict__ pos, int32_t *__restrict__ pairs,
                        int64_t cap, const uint32_t *__restrict__ sweep2orig) {
  // one thread per decision; candidate scan straight from global memory (error path sizes)
  GS(k, rs.n) {
    int64_t start = pos[k], stop = pos[k + 1];
    if (start == stop) continue;
    const int64_t b = k / kTile;
    Cand d{rs.addr[k], rs.addr[k] + rs.size[k], rs.ts[k], rs.te[k], (int)k};
    long long pa = LLONG_MIN, pend = 0;
    int pr = INT_MAX, fwd = 0;
    auto visit = [&](int64_t x) {
      Cand c{rs.addr[x], rs.addr[x] + rs.size[x], rs.ts[x], rs.te[x], (int)x};
      eval_one(d, c, pa, pr, pend, fwd);
    };
    for (int64_t x = tl.loff[b]; x < tl.loff[b + 1]; x++) visit(tl.live[x]);
    for (int64_t x = b * kTile; x < k; x++) visit(x);
    int64_t w = start;
    if (pa != LLONG_MIN && pend > d.addr) {
      if (w < cap) pairs[2 * w] = (int32_t)sweep2orig[pr], pairs[2 * w + 1] = (int32_t)sweep2orig[k];
      w++;
    }
    // forward candidates in (addr asc, sweep position desc) order: selection by repeated scans
    long long last_a = LLONG_MIN;
    int last_r = INT_MAX;
    for (int rep = 0; rep < fwd; rep++) {
      long long ba = LLONG_MAX;
      int br = -1;
      auto pick = [&](int64_t x) {
        if (rs.te[x] <= d.ts) return;
        long long a = rs.addr[x];
        if (a < d.addr || a >= d.end) return;
        bool after = a > last_a || (a == last_a && (int)x < last_r);
        if (!after) return;
        if (a < ba || (a == ba && (int)x > br)) ba = a, br = (int)x;
      };
      for (int64_t x = tl.loff[b]; x < tl.loff[b + 1]; x++) pick(tl.live[x]);
      for (int64_t x = b * kTile; x < k; x++) pick(x);
      if (w < cap) pairs[2 * w] = (int32_t)sweep2orig[br], pairs[2 * w + 1] = (int32_t)sweep2orig[k];
      w++;
      last_a = ba;
      last_r = br;
    }
  }
}

__global__ void k_gather_rect(const uint32_t *__restrict__ perm, const int64_t *__restrict__ addr,
                              const int64_t *__restrict__ size, const int32_t *__restrict__ ts,
                              const int32_t *__restrict__ te, int64_t n, int64_t *__restrict__ a2,
                              int64_t *__restrict__ s2, int32_t *__restrict__ ts2, int32_t *__restrict__ te2) {
  GS(k, n) {
    uint32_t i = perm[k];
    a2[k] = addr[i];
    s2[k] = size[i];
    ts2[k] = ts[i];
    te2[k] = te[i];
  }
}

__global__ void k_sweep_keys(const int64_t *__restrict__ id, const int32_t *__restrict__ ts, int64_t n, long long idmin,
                             uint64_t *__restrict__ hi, uint64_t *__restrict__ lo) {
  GS(k, n) {
    hi[k] = (uint32_t)ts[k];
    lo[k] = (uint64_t)((long long)id[k] - idmin);
  }
}

__global__ void k_minmax_id(const int64_t *__restrict__ v, int64_t n, long long *mn, long long *mx) {
  GS(i, n) {
    atomicMin(mn, (long long)v[i]);
    atomicMax(mx, (long long)v[i]);
  }
}

__global__ void k_or_bits(const int64_t *__restrict__ a, const int64_t *__restrict__ b, int64_t n,
                          unsigned long long *out) {
  unsigned long long v = 0;
  GS(i, n) v |= (unsigned long long)a[i] | (unsigned long long)b[i];
  for (int o = 16; o; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicOr(out, v);
}

__global__ void k_max_ts(const int32_t *__restrict__ v, int64_t n, int *mx) {
  GS(i, n) atomicMax(mx, v[i]);
}

int validate_plan_pairs(Ctx &ctx, int64_t n, const int64_t *id, const int64_t *addr, const int64_t *size,
                        const int32_t *t_s, const int32_t *t_e, int64_t *n_pairs, int32_t *pairs, int64_t cap) {
  Arena ar(&ctx);
  *n_pairs = 0;
  if (n <= 0) return ctx.rc;
  int64_t by = 0;
  const int64_t *did = stage(ctx, ar, id, n, false, &by);
  const int64_t *dad = stage(ctx, ar, addr, n, false, &by);
  const int64_t *dsz = stage(ctx, ar, size, n, false, &by);
  const int32_t *dts = stage(ctx, ar, t_s, n, false, &by);
  const int32_t *dte = stage(ctx, ar, t_e, n, false, &by);
  long long *mm = ar.take<long long>(2);
  int *mts = ar.take<int>(1);
  uint64_t *hi = ar.take<uint64_t>(n), *lo = ar.take<uint64_t>(n);
  uint32_t *perm = ar.take<uint32_t>(n);
  if (!ctx.ok()) return ctx.rc;
  long long init[2] = {LLONG_MAX, LLONG_MIN};
  STW_CUDA(ctx, cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(mts, 0, sizeof(int), ctx.stream));
  STW_KL(k_minmax_id, grid_for(n, 256), 256, ctx.stream, did, n, mm, mm + 1);
  STW_KL(k_max_ts, grid_for(n, 256), 256, ctx.stream, dts, n, mts);
  long long h[2];
  int hts = 0;
  STW_CUDA(ctx, cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaMemcpyAsync(&hts, mts, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok()) return ctx.rc;
  STW_KL(k_sweep_keys, grid_for(n, 256), 256, ctx.stream, did, dts, n, h[0], hi, lo);
  sort_perm2(ctx, ar, hi, bitlen_u64((uint64_t)hts), lo, bitlen_u64((uint64_t)(h[1] - h[0])), perm, n);
  int64_t *a2 = ar.take<int64_t>(n), *s2 = ar.take<int64_t>(n);
  int32_t *ts2 = ar.take<int32_t>(n), *te2 = ar.take<int32_t>(n);
  int64_t *off = ar.take<int64_t>(2);
  long long *cnt = ar.take<long long>(1);
  int *first = ar.take<int>(1);
  int32_t *per_d = ar.take<int32_t>(n + 1);
  int64_t *pos = ar.take<int64_t>(n + 1);
  if (!ctx.ok()) return ctx.rc;
  STW_KL(k_gather_rect, grid_for(n, 256), 256, ctx.stream, perm, dad, dsz, dts, dte, n, a2, s2, ts2, te2);
  int64_t hoff[2] = {0, n};
  STW_CUDA(ctx, cudaMemcpyAsync(off, hoff, sizeof(hoff), cudaMemcpyHostToDevice, ctx.stream));
  RectSets rs{1, n, off, ts2, te2, s2, 1, a2};
  {  // fast path: a valid plan reports nothing
    unsigned long long *orv = ar.take<unsigned long long>(1);
    if (!ctx.ok()) return ctx.rc;
    STW_CUDA(ctx, cudaMemsetAsync(orv, 0, sizeof(unsigned long long), ctx.stream));
    STW_KL(k_or_bits, grid_for(n, 256), 256, ctx.stream, a2, s2, n, orv);
    unsigned long long hor = 0;
    STW_CUDA(ctx, cudaMemcpyAsync(&hor, orv, sizeof(hor), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    const int shift = hor ? std::min(__builtin_ctzll(hor), 62) : 0;
    if (overlap_flags(ctx, ar, rs, shift) == 0) return ctx.rc;
    if (!ctx.ok()) return ctx.rc;
  }
  Tiles tl;
  build_tiles(ctx, ar, rs, &tl);
  STW_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(long long), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(first, 0x7f, sizeof(int), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(per_d, 0, (n + 1) * sizeof(int32_t), ctx.stream));
  if (!ctx.ok()) return ctx.rc;
  STW_KL(k_validate_tiles, dim3((unsigned)tl.NB, 1), kTile, ctx.stream, rs, tl, cnt, first, per_d);
  STW_LAUNCHED(ctx);
  // pair slots per decision: exclusive scan of per-decision counts (as int64)
  {
    std::vector<int32_t> hp(n + 1);
    STW_CUDA(ctx, cudaMemcpyAsync(hp.data(), per_d, (n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    std::vector<int64_t> hpos(n + 1, 0);
    for (int64_t k = 0; k < n; k++) hpos[k + 1] = hpos[k] + hp[k];
    *n_pairs = hpos[n];
    if (hpos[n] == 0 || !ctx.ok()) return ctx.rc;
    STW_CUDA(ctx, cudaMemcpyAsync(pos, hpos.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx.stream));
  }
  int64_t wcap = std::min<int64_t>(cap, *n_pairs);
  int32_t *dpairs = ar.take<int32_t>(2 * wcap + 2);
  if (!ctx.ok()) return ctx.rc;
  STW_KL(k_pairs, grid_for(n, 128), 128, ctx.stream, rs, tl, pos, dpairs, wcap, perm);
  STW_LAUNCHED(ctx);
  if (wcap > 0)
    STW_CUDA(ctx, cudaMemcpyAsync(pairs, dpairs, 2 * wcap * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  return ctx.rc;
}

}  // namespace stw
