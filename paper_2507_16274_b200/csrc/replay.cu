// K9/K10 -- trace replay against a plan (simulate, sim.py:143-238) and the
// online caching-allocator baseline (run_baseline, baseline.py:98-137).
//
// Parallel preprocessing on the device:
//   * plan bundle validation (traceio.py:322-331)
//   * dense id classes (the reference keys its live maps and events_by_id by id)
//   * static matching: the k-th static alloc (in op order) of key
//     (p_s, size) receives the k-th decision of that key in (t_s, id) order
//     (sim.py:156-162, 189-191) -- a joint radix sort of decisions and static
//     events by (p_s, size, side, order), then ranks inside each key
//   * op order (t, is_alloc, id), frees first (sim.py:165-169)
// Sequential residue on one warp: the pool free-interval set, dynamic best-fit
// inside the reuse space (sim.py:120-140), the caching allocator
// (baseline.py:49-95), the replay log and the metrics (sim.py:67-117). The
// warp prefetches 32 ops at a time; interval lists live in shared memory.
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "planner.cuh"

namespace stw {

#define GS3(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// kernels shared with plan.cu
__global__ void k_minmax_i64(const int64_t *__restrict__ v, int64_t n, long long *mn, long long *mx);
__global__ void k_max_i32(const int32_t *__restrict__ v, int64_t n, int *mx);
__global__ void k_gather_u64(const uint64_t *__restrict__ src, const uint32_t *__restrict__ perm,
                             uint64_t *__restrict__ dst, int64_t n);
double exact_div_host(unsigned long long a, unsigned long long b);

constexpr int kFreeSmem = 4096;   // pool free intervals kept in shared memory
constexpr int kBlockSmem = 4096;  // cache free blocks kept in shared memory
constexpr int kSpaceSmem = 2048;  // reuse-space intervals of one key staged in shared memory
constexpr size_t kReplaySmem = (size_t)kFreeSmem * 16 + (size_t)kBlockSmem * 20 + (size_t)kSpaceSmem * 16;
constexpr long long kMinSegment = 2ll * 1024 * 1024;

enum { R_PLANNED = 0, R_REUSE = 1, R_FALLBACK = 2, R_MISMATCH = 3, R_ONLINE = 4 };

// ---------------------------------------------------------------------------
// preprocessing kernels

__global__ void k_bundle_check(const int64_t *__restrict__ d_addr, const int64_t *__restrict__ d_size, int64_t nd,
                               long long pool, long long align, int *__restrict__ first_bad,
                               const int64_t *__restrict__ sp_off, const int64_t *__restrict__ sp_lo,
                               const int64_t *__restrict__ sp_hi, int64_t K, int *__restrict__ first_bad_key) {
  GS3(k, nd) {
    if (d_addr[k] < 0 || d_addr[k] + d_size[k] > pool || d_addr[k] % align) atomicMin(first_bad, (int)k);
  }
  GS3(k, K) {
    for (int64_t j = sp_off[k]; j < sp_off[k + 1]; j++)
      if (sp_lo[j] < 0 || sp_hi[j] > pool) {
        atomicMin(first_bad_key, (int)k);
        break;
      }
  }
}

__global__ void k_id_keys(const int64_t *__restrict__ id, int64_t n, long long idmin, uint64_t *__restrict__ key) {
  GS3(i, n) key[i] = (uint64_t)((long long)id[i] - idmin);
}

// did (dense id class) per event, last event index per class, sorted unique ids
__global__ void k_id_classes(const uint32_t *__restrict__ perm, const uint64_t *__restrict__ skey, int64_t n,
                             const uint32_t *__restrict__ cls_incl, int32_t *__restrict__ did, int32_t *__restrict__ last_of,
                             uint64_t *__restrict__ ukey) {
  GS3(k, n) {
    uint32_t i = perm[k];
    int c = (int)cls_incl[k] - 1;
    did[i] = c;
    if (k + 1 == n || skey[k + 1] != skey[k]) {
      last_of[c] = (int32_t)i;  // stable sort: the largest index of the class comes last
      ukey[c] = skey[k];
    }
  }
}

// ids strictly increasing in listing order (the usual trace): *bad stays 0
__global__ void k_ids_increasing(const int64_t *__restrict__ id, int64_t n, int *__restrict__ bad) {
  int b = 0;
  GS3(i, n - 1) b |= id[i] >= id[i + 1] ? 1 : 0;
  b = __reduce_or_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(bad, 1);
}

// the id classes of increasing ids: the identity (what the sort + scan give)
__global__ void k_id_identity(const int64_t *__restrict__ id, int64_t n, long long idmin, int32_t *__restrict__ did,
                              int32_t *__restrict__ last_of, uint64_t *__restrict__ ukey) {
  GS3(i, n) {
    did[i] = (int32_t)i;
    last_of[i] = (int32_t)i;
    ukey[i] = (uint64_t)((long long)id[i] - idmin);
  }
}

__global__ void k_heads_u64(const uint64_t *__restrict__ skey, int64_t n, uint32_t *__restrict__ head) {
  GS3(k, n) head[k] = (k == 0 || skey[k] != skey[k - 1]) ? 1u : 0u;
}

// op keys, stage 1 (id) and stage 2 (t, is_alloc); ops are (alloc e, free e) = (2e, 2e+1)
__global__ void k_op_keys_id(const int64_t *__restrict__ id, int64_t n, long long idmin, uint64_t *__restrict__ key) {
  GS3(o, 2 * n) key[o] = (uint64_t)((long long)id[o >> 1] - idmin);
}
__global__ void k_op_keys_t(const uint32_t *__restrict__ perm, const int32_t *__restrict__ ts,
                            const int32_t *__restrict__ te, int64_t n, uint64_t *__restrict__ key) {
  GS3(k, 2 * n) {
    uint32_t o = perm[k];
    uint32_t e = o >> 1;
    bool alloc = !(o & 1);
    key[k] = ((uint64_t)(uint32_t)(alloc ? ts[e] : te[e]) << 1) | (alloc ? 1u : 0u);
  }
}
__global__ void k_op_rank(const uint32_t *__restrict__ operm, int64_t n2, int32_t *__restrict__ apos) {
  GS3(k, n2) {
    uint32_t o = operm[k];
    if (!(o & 1)) apos[o >> 1] = (int32_t)k;
  }
}

// decisions: find the event carrying the id (events_by_id keeps the last one)
__global__ void k_dec_lookup(const int64_t *__restrict__ d_id, int64_t nd, const uint64_t *__restrict__ ukey, int64_t nu,
                             long long idmin, const int32_t *__restrict__ last_of, const uint8_t *__restrict__ dyn,
                             int32_t *__restrict__ d_ev) {
  GS3(k, nd) {
    long long x = (long long)d_id[k] - idmin;
    int e = -1;
    if (x >= 0) {
      uint64_t ux = (uint64_t)x;
      int64_t lo = 0, hi = nu;
      while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (ukey[m] < ux)
          lo = m + 1;
        else
          hi = m;
      }
      if (lo < nu && ukey[lo] == ux) e = last_of[lo];
    }
    d_ev[k] = (e >= 0 && !dyn[e]) ? e : -1;
  }
}

// decision queue order: (t_s, id, plan position)
__global__ void k_dec_keys(const int32_t *__restrict__ d_ts, const int64_t *__restrict__ d_id, int64_t nd,
                           long long idmin, uint64_t *__restrict__ hi, uint64_t *__restrict__ lo) {
  GS3(k, nd) {
    hi[k] = (uint32_t)d_ts[k];
    lo[k] = (uint64_t)((long long)d_id[k] - idmin);
  }
}
__global__ void k_scatter_rank(const uint32_t *__restrict__ perm, int64_t n, int32_t *__restrict__ rank) {
  GS3(k, n) rank[perm[k]] = (int32_t)k;
}

// joint records for queue matching. record r < nd: decision; else static event
struct MatchRec {
  int64_t nd, n;
  const int32_t *d_ev, *d_rank;
  const int64_t *d_size;
  const int32_t *ps;
  const int64_t *size;
  const uint8_t *dyn;
  const int32_t *apos;
};
__global__ void k_match_keys(MatchRec M, uint64_t *__restrict__ k_ord, uint64_t *__restrict__ k_size,
                             uint64_t *__restrict__ k_ps) {
  GS3(r, M.nd + M.n) {
    uint64_t side, ord, sz, ph;
    if (r < M.nd) {
      int e = M.d_ev[r];
      side = 0;
      ord = (uint32_t)M.d_rank[r];
      sz = (uint64_t)M.d_size[r];
      ph = e >= 0 ? (uint32_t)M.ps[e] : 0xFFFFFFFFu;  // ineligible decisions sort last, never matched
    } else {
      int64_t e = r - M.nd;
      side = 1;
      ord = (uint32_t)M.apos[e];
      sz = (uint64_t)M.size[e];
      ph = M.dyn[e] ? 0xFFFFFFFFu : (uint32_t)M.ps[e];
    }
    k_ord[r] = (side << 32) | ord;
    k_size[r] = sz;
    k_ps[r] = ph;
  }
}

__global__ void k_match_heads(const uint32_t *__restrict__ perm, MatchRec M, uint32_t *__restrict__ head) {
  GS3(k, M.nd + M.n) {
    auto key = [&](uint32_t r, uint64_t *ph, uint64_t *sz) {
      if (r < M.nd) {
        int e = M.d_ev[r];
        *ph = e >= 0 ? (uint32_t)M.ps[e] : 0xFFFFFFFFu;
        *sz = (uint64_t)M.d_size[r];
      } else {
        int64_t e = r - M.nd;
        *ph = M.dyn[e] ? 0xFFFFFFFFu : (uint32_t)M.ps[e];
        *sz = (uint64_t)M.size[e];
      }
    };
    uint32_t h = 1;
    if (k > 0) {
      uint64_t a, b, c, d;
      key(perm[k], &a, &b);
      key(perm[k - 1], &c, &d);
      h = (a != c || b != d);
    }
    head[k] = h;
  }
}

__global__ void k_match_groups(const uint32_t *__restrict__ perm, const uint32_t *__restrict__ gid_incl, int64_t nr,
                               int64_t nd, int64_t *__restrict__ gstart, int32_t *__restrict__ gndec) {
  GS3(k, nr) {
    int g = (int)gid_incl[k] - 1;
    if (k == 0 || gid_incl[k - 1] != gid_incl[k]) gstart[g] = k;
    if (perm[k] < nd) atomicAdd(gndec + g, 1);
  }
}

__global__ void k_match_assign(const uint32_t *__restrict__ perm, const uint32_t *__restrict__ gid_incl, int64_t nr,
                               MatchRec M, const int64_t *__restrict__ gstart, const int32_t *__restrict__ gndec,
                               const int64_t *__restrict__ d_addr, int8_t *__restrict__ route,
                               int64_t *__restrict__ paddr) {
  GS3(k, nr) {
    uint32_t r = perm[k];
    if (r < M.nd) continue;
    int64_t e = r - M.nd;
    if (M.dyn[e]) continue;
    int g = (int)gid_incl[k] - 1;
    int64_t rank = k - gstart[g] - gndec[g];
    if (rank < gndec[g]) {
      route[e] = R_PLANNED;
      paddr[e] = d_addr[perm[gstart[g] + rank]];
    } else {
      route[e] = R_MISMATCH;
      paddr[e] = -1;
    }
  }
}

// ---------------------------------------------------------------------------
// sequential replay warp

struct ReplayArgs {
  int64_t n;
  const uint32_t *operm;
  const int64_t *id, *size;
  const int32_t *ts, *te;
  const uint8_t *dyn;
  const int32_t *did;
  const int8_t *route0;  // R_PLANNED / R_MISMATCH for static events; baseline: all R_ONLINE
  const int64_t *paddr;
  const int32_t *key;
  const int64_t *sp_off, *sp_lo, *sp_hi;
  int reuse, baseline;
  long long pool;
  // state (global, per dense id class)
  int64_t *plo, *phi;
  int8_t *pflag;
  int64_t *clo, *chi;
  int32_t *cseg;
  int8_t *cflag;
  int64_t *gflo, *gfhi;              // spill storage for the free list (cap n + 2)
  int64_t *gblo, *gbhi;              // spill storage for cache blocks (cap 2n + 2)
  int32_t *gbseg;
  int64_t *sbase;                    // segment bases (cap n + 1)
  // log (cap 1 + 3n)
  int8_t *lkind, *lspace, *lroute;
  int64_t *lt, *lid, *lsize, *laddr;
  // results
  long long *res;  // [0] nlog, [1] err code, [2] err id, [3] err addr, metrics [4..]
};

// warp helpers ---------------------------------------------------------------
constexpr unsigned kFull = 0xffffffffu;

// min of (k1, k2, k3) lexicographic over the warp, result in every lane
__device__ __forceinline__ void warp_min3(long long &k1, long long &k2, int &k3) {
  for (int o = 16; o; o >>= 1) {
    const long long a = __shfl_xor_sync(kFull, k1, o), b = __shfl_xor_sync(kFull, k2, o);
    const int c = __shfl_xor_sync(kFull, k3, o);
    if (a < k1 || (a == k1 && b < k2)) k1 = a, k2 = b, k3 = c;
  }
}

__device__ __forceinline__ void warp_min_pair(long long &k1, long long &k2) {
  for (int o = 16; o; o >>= 1) {
    long long a = __shfl_xor_sync(kFull, k1, o), b = __shfl_xor_sync(kFull, k2, o);
    if (a < k1 || (a == k1 && b < k2)) k1 = a, k2 = b;
  }
}

// The sequential residue of the replay on one warp. Interval lists are kept
// UNSORTED in shared memory (spilling to global beyond the smem capacity):
// every query is a lane-parallel scan + ballot, every update O(1) by lane 0
// (in place, append, or swap-remove), so no op pays for a binary search or a
// shifted array. Order-dependent tie-breaks are order-free here: best fit =
// min (length, address) -- the cache's (segment, address) order is address
// order, since segments are appended at increasing bases (baseline.py:54-66).
// Per op window (32 ops, one per lane) every lane prefetches its op's fields
// AND the per-id state it will read (pool / cache liveness, interval,
// segment, the reuse key's space range), so the chain of dependent global
// loads is paid once per 32 ops; state an earlier op of the same window
// changes is forwarded lane to lane.
__global__ void __launch_bounds__(32) k_replay(ReplayArgs A) {
  extern __shared__ int64_t dsm[];
  int64_t *s_flo = dsm, *s_fhi = dsm + kFreeSmem;
  int64_t *s_blo = dsm + 2 * kFreeSmem, *s_bhi = s_blo + kBlockSmem;
  int32_t *s_bseg = (int32_t *)(s_bhi + kBlockSmem);
  int64_t *s_sp = (int64_t *)(s_bseg + kBlockSmem);  // staged reuse space of the current key: lo, hi pairs
  const int lane = (int)lane_id();
  // lists start in shared memory and move to their global spill arrays the
  // first time they would outgrow it
  int64_t *flo = s_flo, *fhi = s_fhi;
  int64_t *blo = s_blo, *bhi = s_bhi;
  int32_t *bseg = s_bseg;
  int nf = 0, nb = 0, ns = 0;
  auto grow_free = [&]() {  // before a free-list append
    if (flo != s_flo || nf + 1 < kFreeSmem) return;
    for (int i = lane; i < nf; i += 32) A.gflo[i] = s_flo[i], A.gfhi[i] = s_fhi[i];
    __syncwarp();
    flo = A.gflo;
    fhi = A.gfhi;
  };
  auto grow_blocks = [&]() {  // before a cache-block append
    if (blo != s_blo || nb + 1 < kBlockSmem) return;
    for (int i = lane; i < nb; i += 32) A.gblo[i] = s_blo[i], A.gbhi[i] = s_bhi[i], A.gbseg[i] = s_bseg[i];
    __syncwarp();
    blo = A.gblo;
    bhi = A.gbhi;
    bseg = A.gbseg;
  };
  long long next_base = A.baseline ? 0 : A.pool;
  if (!A.baseline && A.pool > 0) {
    if (lane == 0) {
      flo[0] = 0;
      fhi[0] = A.pool;
    }
    nf = 1;
    __syncwarp();  // the other lanes read it (racecheck)
  }
  long long nlog = 0, live = 0, peak = 0, clive = 0, cpeak = 0, reserved = 0;
  long long n_fb = 0, n_reuse = 0, n_mm = 0;
  long long err = 0, err_id = 0, err_addr = 0;
  long long max_nb = 0, max_nf = 0, sum_nb = 0, sum_nf = 0;  // list sizes (diagnostics, res[10..13])
  auto logrec = [&](int kind, long long t, long long id, long long size, int space, long long addr, int route) {
    if (lane == 0) {
      A.lkind[nlog] = (int8_t)kind;
      A.lt[nlog] = t;
      A.lid[nlog] = id;
      A.lsize[nlog] = size;
      A.lspace[nlog] = (int8_t)space;
      A.laddr[nlog] = addr;
      A.lroute[nlog] = (int8_t)route;
    }
    nlog++;
  };
  logrec(0, 0, 0, A.baseline ? 0 : A.pool, 0, 0, -1);

  // pool free set -----------------------------------------------------------
  // index of the free interval holding [lo, hi) entirely, -1 if none (contains_interval, intervals.py:95-98)
  auto free_holding = [&](long long lo, long long hi) -> int {
    for (int base = 0; base < nf; base += 32) {
      const int i = base + lane;
      const unsigned m = __ballot_sync(kFull, i < nf && flo[i] <= lo && hi <= fhi[i]);
      if (m) return base + __ffs(m) - 1;
    }
    return -1;
  };
  // remove [lo, hi) lying inside free interval i (IntervalSet.remove, intervals.py:113-129)
  auto free_remove = [&](int i, long long lo, long long hi) {
    grow_free();
    const long long a = flo[i], b = fhi[i];
    __syncwarp();
    if (lane == 0) {
      if (a < lo && b > hi) {
        fhi[i] = lo;
        flo[nf] = hi;
        fhi[nf] = b;
      } else if (a < lo) {
        fhi[i] = lo;
      } else if (b > hi) {
        flo[i] = hi;
      } else {
        flo[i] = flo[nf - 1];
        fhi[i] = fhi[nf - 1];
      }
    }
    nf += (a < lo && b > hi) ? 1 : (a < lo || b > hi) ? 0 : -1;
    __syncwarp();
  };
  // IntervalSet.add (intervals.py:100-111) of an interval disjoint from the free
  // set (it was live): merge with the neighbours it touches
  auto free_add = [&](long long lo, long long hi) {
    grow_free();
    int l = -1, r = -1;
    for (int base = 0; base < nf; base += 32) {
      const int i = base + lane;
      const bool in = i < nf;
      const long long a = in ? flo[i] : 0, b = in ? fhi[i] : 0;
      const unsigned ml = __ballot_sync(kFull, in && b == lo), mr = __ballot_sync(kFull, in && a == hi);
      if (ml) l = base + __ffs(ml) - 1;
      if (mr) r = base + __ffs(mr) - 1;
    }
    __syncwarp();
    if (lane == 0) {
      if (l >= 0 && r >= 0) {
        fhi[l] = fhi[r];
        flo[r] = flo[nf - 1];
        fhi[r] = fhi[nf - 1];
      } else if (l >= 0) {
        fhi[l] = hi;
      } else if (r >= 0) {
        flo[r] = lo;
      } else {
        flo[nf] = lo;
        fhi[nf] = hi;
      }
    }
    nf += (l >= 0 && r >= 0) ? -1 : (l < 0 && r < 0) ? 1 : 0;
    __syncwarp();
  };

  // caching allocator (baseline.py:49-95) ------------------------------------
  // malloc: returns the address, sets *grown and *sg (segment)
  auto cache_malloc = [&](long long size, long long *grown, int *sg) -> long long {
    long long bl = LLONG_MAX, ba = LLONG_MAX;
    int bi = -1;
    for (int i = lane; i < nb; i += 32) {
      const long long a = blo[i], len = bhi[i] - a;
      if (len >= size && (len < bl || (len == bl && a < ba))) bl = len, ba = a, bi = i;
    }
    warp_min3(bl, ba, bi);
    *grown = 0;
    if (bi < 0) {  // a fresh segment at the next base
      grow_blocks();
      long long ss = 1;
      while (ss < size) ss <<= 1;
      if (ss < kMinSegment) ss = kMinSegment;
      if (lane == 0) {
        A.sbase[ns] = next_base;
        blo[nb] = next_base;
        bhi[nb] = next_base + ss;
        bseg[nb] = ns;
      }
      __syncwarp();
      bi = nb++;
      ns++;
      ba = next_base;
      next_base += ss;
      *grown = ss;
    }
    const long long hi = bhi[bi];
    *sg = bseg[bi];
    __syncwarp();
    if (lane == 0) {
      if (ba + size < hi) {  // split: the remainder stays
        blo[bi] = ba + size;
      } else {  // exact fit: swap-remove
        blo[bi] = blo[nb - 1];
        bhi[bi] = bhi[nb - 1];
        bseg[bi] = bseg[nb - 1];
      }
    }
    if (ba + size >= hi) nb--;
    __syncwarp();
    return ba;
  };
  // free: merge with the same segment's free neighbours (baseline.py:79-95)
  auto cache_free = [&](long long lo, long long hi, int sg) {
    grow_blocks();
    int l = -1, r = -1;
    for (int base = 0; base < nb; base += 32) {
      const int i = base + lane;
      const bool in = i < nb;
      const bool same = in && bseg[i] == sg;
      const unsigned ml = __ballot_sync(kFull, same && bhi[i] == lo), mr = __ballot_sync(kFull, same && blo[i] == hi);
      if (ml) l = base + __ffs(ml) - 1;
      if (mr) r = base + __ffs(mr) - 1;
    }
    __syncwarp();
    if (lane == 0) {
      if (l >= 0 && r >= 0) {
        bhi[l] = bhi[r];
        blo[r] = blo[nb - 1];
        bhi[r] = bhi[nb - 1];
        bseg[r] = bseg[nb - 1];
        if (l == nb - 1) bhi[r] = bhi[l];  // l itself moved into r's slot
      } else if (l >= 0) {
        bhi[l] = hi;
      } else if (r >= 0) {
        blo[r] = lo;
      } else {
        blo[nb] = lo;
        bhi[nb] = hi;
        bseg[nb] = sg;
      }
    }
    nb += (l >= 0 && r >= 0) ? -1 : (l < 0 && r < 0) ? 1 : 0;
    __syncwarp();
  };

  const int64_t n2 = 2 * A.n;
  for (int64_t cb = 0; cb < n2 && !err; cb += 32) {
    // prefetch one op per lane, with the state it reads
    const int64_t mine = cb + lane;
    const uint32_t o = mine < n2 ? A.operm[mine] : 0;
    const int e = (int)(o >> 1);
    const bool is_alloc = !(o & 1);
    long long my_t = 0, my_id = 0, my_size = 0, my_paddr = -1;
    int my_did = -1, my_key = -1, my_route = R_ONLINE;
    long long my_s0 = 0, my_s1 = 0;
    // per-id state: pool (flag, lo, hi), cache (flag, lo, hi, segment)
    int my_pf = 0, my_cf = 0, my_cs = 0;
    long long my_plo = 0, my_phi = 0, my_clo = 0, my_chi = 0;
    if (mine < n2) {
      my_t = is_alloc ? A.ts[e] : A.te[e];
      my_id = A.id[e];
      my_size = A.size[e];
      my_did = A.did[e];
      const bool dyn = A.dyn[e] != 0;
      if (!A.baseline) {
        my_route = dyn ? -1 : A.route0[e];
        my_paddr = dyn ? -1 : A.paddr[e];
        my_key = dyn ? A.key[e] : -1;
        if (my_key >= 0 && A.reuse) {
          my_s0 = A.sp_off[my_key];
          my_s1 = A.sp_off[my_key + 1];
        }
      }
      my_pf = A.pflag[my_did];
      my_cf = A.cflag[my_did];
      if (!is_alloc) {
        my_plo = A.plo[my_did];
        my_phi = A.phi[my_did];
        my_clo = A.clo[my_did];
        my_chi = A.chi[my_did];
        my_cs = A.cseg[my_did];
      }
    }
    const int cnt = (int)min((int64_t)32, n2 - cb);
    for (int k = 0; k < cnt && !err; k++) {
#ifdef STW_REPLAY_STATS
      max_nb = max(max_nb, (long long)nb), max_nf = max(max_nf, (long long)nf), sum_nb += nb, sum_nf += nf;
#endif
      const bool alloc = __shfl_sync(kFull, (int)is_alloc, k);
      const long long t = __shfl_sync(kFull, my_t, k), id = __shfl_sync(kFull, my_id, k);
      const long long size = __shfl_sync(kFull, my_size, k);
      const int c = __shfl_sync(kFull, my_did, k);
      const bool same = my_did == c;  // lanes whose op touches the same id (state forwarding)
      if (alloc) {
        const int route = __shfl_sync(kFull, my_route, k);
        bool to_pool = false, to_cache = false;
        long long a = -1;
        int rt = route;
        if (route == R_PLANNED) {
          a = __shfl_sync(kFull, my_paddr, k);
          const int i = free_holding(a, a + size);
          if (i < 0) {
            err = STW_ESIM;
            err_id = id;
            err_addr = a;
            break;
          }
          free_remove(i, a, a + size);
          to_pool = true;
        } else if (route == R_MISMATCH || route == R_ONLINE) {
          to_cache = true;
        } else {  // dynamic: best fit in free ∩ space[key] (sim.py:120-140), else the fallback
          const long long s0 = __shfl_sync(kFull, my_s0, k), s1 = __shfl_sync(kFull, my_s1, k);
          const int ns_ = (int)(s1 - s0);
          rt = R_FALLBACK;
          if (ns_ > 0) {
            // the key's space, staged in shared memory when it fits
            const bool staged = ns_ <= kSpaceSmem;
            if (staged) {
              for (int j = lane; j < ns_; j += 32) {
                s_sp[2 * j] = A.sp_lo[s0 + j];
                s_sp[2 * j + 1] = A.sp_hi[s0 + j];
              }
              __syncwarp();
            }
            auto sp_lo = [&](int64_t j) { return staged ? s_sp[2 * j] : (long long)A.sp_lo[s0 + j]; };
            auto sp_hi = [&](int64_t j) { return staged ? s_sp[2 * j + 1] : (long long)A.sp_hi[s0 + j]; };
            long long best_len = LLONG_MAX, best_lo = LLONG_MAX;
            for (int i = lane; i < nf; i += 32) {
              const long long fa = flo[i], fb = fhi[i];
              int64_t x = 0, y = ns_;  // first space interval with hi > fa
              while (x < y) {
                const int64_t m = (x + y) >> 1;
                if (sp_hi(m) <= fa)
                  x = m + 1;
                else
                  y = m;
              }
              for (int64_t j = x; j < ns_ && sp_lo(j) < fb; j++) {
                const long long lo = max(fa, sp_lo(j)), hi = min(fb, sp_hi(j));
                const long long len = hi - lo;
                if (len >= size && (len < best_len || (len == best_len && lo < best_lo))) best_len = len, best_lo = lo;
              }
            }
            warp_min_pair(best_len, best_lo);
            __syncwarp();
            if (best_len != LLONG_MAX) {
              a = best_lo;
              free_remove(free_holding(a, a + size), a, a + size);
              to_pool = true;
              rt = R_REUSE;
            }
          }
          if (!to_pool) to_cache = true;
        }
        if (to_pool) {
          if (lane == 0) {
            A.plo[c] = a;
            A.phi[c] = a + size;
            A.pflag[c] = 1;
          }
          if (same) my_pf = 1, my_plo = a, my_phi = a + size;
          logrec(2, t, id, size, 0, a, rt);
          live += size;
          peak = max(peak, live);
          if (rt == R_REUSE) n_reuse++;
        } else if (to_cache) {
          if (__shfl_sync(kFull, my_cf, k)) {  // request already live in cache
            err = STW_ESIM + 100;
            err_id = id;
            break;
          }
          long long grown;
          int sg;
          a = cache_malloc(size, &grown, &sg);
          if (lane == 0) {
            A.clo[c] = a;
            A.chi[c] = a + size;
            A.cseg[c] = sg;
            A.cflag[c] = 1;
          }
          if (same) my_cf = 1, my_clo = a, my_chi = a + size, my_cs = sg;
          if (grown) {
            logrec(1, t, 0, grown, 0, 0, -1);
            reserved += grown;
          }
          logrec(2, t, id, size, 1, a, rt);
          live += size;
          peak = max(peak, live);
          clive += size;
          cpeak = max(cpeak, clive);
          if (rt == R_MISMATCH || rt == R_FALLBACK) n_fb++;
          if (rt == R_MISMATCH) n_mm++;
        }
      } else {
        if (__shfl_sync(kFull, my_pf, k)) {
          const long long lo = __shfl_sync(kFull, my_plo, k), hi = __shfl_sync(kFull, my_phi, k);
          if (lane == 0) A.pflag[c] = 0;
          if (same) my_pf = 0;
          free_add(lo, hi);
          logrec(3, t, id, hi - lo, 0, lo, -1);
          live -= hi - lo;
        } else if (__shfl_sync(kFull, my_cf, k)) {
          const long long lo = __shfl_sync(kFull, my_clo, k), hi = __shfl_sync(kFull, my_chi, k);
          const int sg = __shfl_sync(kFull, my_cs, k);
          if (lane == 0) A.cflag[c] = 0;
          if (same) my_cf = 0;
          cache_free(lo, hi, sg);
          logrec(3, t, id, hi - lo, 1, lo, -1);
          live -= hi - lo;
          clive -= hi - lo;
        } else {
          err = STW_ESIM + 200;  // double free / unknown id
          err_id = id;
          break;
        }
      }
    }
    __syncwarp();  // this window's state stores are visible to the next window's prefetch
  }
  if (lane == 0) {
    A.res[0] = nlog;
    A.res[1] = err;
    A.res[2] = err_id;
    A.res[3] = err_addr;
    A.res[4] = peak;
    A.res[5] = reserved;
    A.res[6] = cpeak;
    A.res[7] = n_fb;
    A.res[8] = n_reuse;
    A.res[9] = n_mm;
    A.res[10] = max_nb;
    A.res[11] = max_nf;
    A.res[12] = sum_nb;
    A.res[13] = sum_nf;
  }
}

__global__ void k_fill_i8(int8_t *p, int64_t n, int8_t v) { GS3(i, n) p[i] = v; }

// ---------------------------------------------------------------------------
// Parallel replay of a fully planned static trace. When every event is static
// with a unique id and the queue matching gave every allocation a planned
// address, the replay's only state is the pool's free set, and a planned
// allocation lands iff its interval is free -- i.e. iff no earlier live planned
// rectangle overlaps it (the K7 test on the (lifespan x planned interval)
// rectangles in op order). Then the log is a function of the op order and the
// metrics are a prefix sum: allocated_peak = max over op order of live bytes,
// reserved = pool, no fallbacks/reuse. Any conflict falls back to the
// sequential warp, which reports the reference's exact error.

__global__ void k_fast_flags(const int8_t *__restrict__ route, const uint8_t *__restrict__ dyn, int64_t n,
                             int *__restrict__ bad) {
  int b = 0;
  GS3(e, n) b |= (dyn[e] != 0 || route[e] != R_PLANNED) ? 1 : 0;
  b = __reduce_or_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(bad, 1);
}

// rectangles in op order of the allocations (= (t_s, id) order), and the
// signed size delta of every op
__global__ void k_fast_rects(const uint32_t *__restrict__ operm, int64_t n,
                             const int32_t *__restrict__ ts, const int32_t *__restrict__ te,
                             const int64_t *__restrict__ size, const int64_t *__restrict__ paddr,
                             const int32_t *__restrict__ arank, int32_t *__restrict__ rts, int32_t *__restrict__ rte,
                             int64_t *__restrict__ rsz, int64_t *__restrict__ raddr, int64_t *__restrict__ delta) {
  GS3(k, 2 * n) {
    const uint32_t o = operm[k];
    const uint32_t e = o >> 1;
    const bool alloc = !(o & 1);
    delta[k] = alloc ? size[e] : -size[e];
    if (alloc) {
      const int32_t r = arank[k];
      rts[r] = ts[e];
      rte[r] = te[e];
      rsz[r] = size[e];
      raddr[r] = paddr[e];
    }
  }
}

__global__ void k_alloc_flag(const uint32_t *__restrict__ operm, int64_t n2, uint32_t *__restrict__ f) {
  GS3(k, n2) f[k] = (operm[k] & 1) ? 0u : 1u;
}

__global__ void k_fast_log(const uint32_t *__restrict__ operm, int64_t n, const int32_t *__restrict__ ts,
                           const int32_t *__restrict__ te, const int64_t *__restrict__ id,
                           const int64_t *__restrict__ size, const int64_t *__restrict__ paddr, long long pool,
                           int8_t *__restrict__ lkind, int8_t *__restrict__ lspace, int8_t *__restrict__ lroute,
                           int64_t *__restrict__ lt, int64_t *__restrict__ lid, int64_t *__restrict__ lsize,
                           int64_t *__restrict__ laddr) {
  GS3(k, 2 * n + 1) {
    if (k == 0) {  // init record (sim.py:153)
      lkind[0] = 0, lspace[0] = 0, lroute[0] = -1, lt[0] = 0, lid[0] = 0, lsize[0] = pool, laddr[0] = 0;
      continue;
    }
    const uint32_t o = operm[k - 1];
    const uint32_t e = o >> 1;
    const bool alloc = !(o & 1);
    lkind[k] = alloc ? 2 : 3;
    lspace[k] = 0;
    lroute[k] = alloc ? R_PLANNED : -1;
    lt[k] = alloc ? ts[e] : te[e];
    lid[k] = id[e];
    lsize[k] = size[e];
    laddr[k] = paddr[e];
  }
}

__global__ void k_max_scan(const int64_t *__restrict__ v, int64_t n, long long *__restrict__ mx) {
  long long m = 0;
  GS3(i, n) m = max(m, (long long)v[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(mx, m);
}

// ---------------------------------------------------------------------------
// host


int replay(Ctx &ctx, const stw_batch *in, const stw_bundle *bun, stw_report *rep, stw_log *log, int64_t *err_id) {
  NvtxPhases nv(bun ? "stw_simulate" : "stw_baseline");
  nv.next("prepare");
  Arena ar(&ctx);
  DevBatch b;
  if (!stage_batch(ctx, ar, in, &b)) return ctx.rc;
  if (b.T != 1) {
    ctx.fail(STW_EARG, "replay takes exactly one trace");
    return ctx.rc;
  }
  const bool baseline = bun == nullptr;
  const int64_t n = b.N;
  const long long pool = baseline ? 0 : bun->pool_size;
  const int64_t nd = baseline ? 0 : bun->n_dec;
  const int64_t K = baseline ? 0 : bun->n_keys;
  *err_id = 0;
  int64_t by = 0;
  const int64_t *d_id = nullptr, *d_addr = nullptr, *d_size = nullptr, *sp_off = nullptr, *sp_lo = nullptr,
                *sp_hi = nullptr;
  const int32_t *d_ts = nullptr, *key = nullptr;
  if (!baseline) {
    d_id = stage(ctx, ar, bun->d_id, nd, false, &by);
    d_addr = stage(ctx, ar, bun->d_addr, nd, false, &by);
    d_size = stage(ctx, ar, bun->d_size, nd, false, &by);
    d_ts = stage(ctx, ar, bun->d_ts, nd, false, &by);
    std::vector<int64_t> off1(1, 0);
    sp_off = stage(ctx, ar, K ? bun->sp_off : off1.data(), K + 1, false, &by);
    int64_t nsp = K ? bun->sp_off[K] : 0;
    sp_lo = stage(ctx, ar, bun->sp_lo, nsp, false, &by);
    sp_hi = stage(ctx, ar, bun->sp_hi, nsp, false, &by);
    key = stage(ctx, ar, bun->key, n, false, &by);
    // PlanBundle.validate
    int *bad = ar.take<int>(2);
    if (!ctx.ok()) return ctx.rc;
    int init[2] = {INT_MAX, INT_MAX};
    STW_CUDA(ctx, cudaMemcpyAsync(bad, init, sizeof(init), cudaMemcpyHostToDevice, ctx.stream));
    int64_t g = std::max<int64_t>(nd, K);
    if (g > 0)
      STW_KL(k_bundle_check, grid_for(g, 256), 256, ctx.stream, d_addr, d_size, nd, pool, (long long)bun->alignment,
             bad, sp_off, sp_lo, sp_hi, K, bad + 1);
    int hb[2];
    STW_CUDA(ctx, cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    if (!ctx.ok()) return ctx.rc;
    if (hb[0] != INT_MAX) {
      int64_t k = hb[0];
      *err_id = bun->d_id[k];
      if (bun->d_addr[k] < 0 || bun->d_addr[k] + bun->d_size[k] > pool)
        ctx.fail(STW_EPLAN, "decision %lld out of pool", (long long)bun->d_id[k]);
      else
        ctx.fail(STW_EPLAN, "decision %lld misaligned address %lld", (long long)bun->d_id[k],
                 (long long)bun->d_addr[k]);
      return ctx.rc;
    }
    if (hb[1] != INT_MAX) {
      *err_id = hb[1];
      ctx.fail(STW_EPLAN, "reuse entry %d outside pool", hb[1]);
      return ctx.rc;
    }
  }
  // id classes
  long long *mm = ar.take<long long>(2);
  int *mt = ar.take<int>(1);
  uint64_t *k1 = ar.take<uint64_t>(2 * n + nd + 1), *k2 = ar.take<uint64_t>(2 * n + nd + 1);
  uint64_t *k3 = ar.take<uint64_t>(2 * n + nd + 1);
  uint32_t *perm = ar.take<uint32_t>(2 * n + nd + 1), *head = ar.take<uint32_t>(2 * n + nd + 1);
  uint32_t *cls = ar.take<uint32_t>(2 * n + nd + 1);
  int32_t *did = ar.take<int32_t>(n + 1), *last_of = ar.take<int32_t>(n + 1);
  uint64_t *ukey = ar.take<uint64_t>(n + 1);
  uint32_t *operm = ar.take<uint32_t>(2 * n + 1);
  int32_t *apos = ar.take<int32_t>(n + 1);
  if (!ctx.ok()) return ctx.rc;
  int *notinc = ar.take<int>(1);
  if (!ctx.ok()) return ctx.rc;
  long long init[2] = {LLONG_MAX, LLONG_MIN};
  STW_CUDA(ctx, cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(mt, 0, sizeof(int), ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(notinc, 0, sizeof(int), ctx.stream));
  if (n > 1) STW_KL(k_ids_increasing, grid_for(n, 256, 148 * 4), 256, ctx.stream, b.id, n, notinc);
  if (n) STW_KL(k_minmax_i64, grid_for(n, 256), 256, ctx.stream, b.id, n, mm, mm + 1);
  if (nd) STW_KL(k_minmax_i64, grid_for(nd, 256), 256, ctx.stream, d_id, nd, mm, mm + 1);
  if (n) STW_KL(k_max_i32, grid_for(n, 256), 256, ctx.stream, b.t_e, n, mt);
  if (nd) STW_KL(k_max_i32, grid_for(nd, 256), 256, ctx.stream, d_ts, nd, mt);
  long long hm[2] = {0, 0};
  int hmt = 0, hni = 1;
  STW_CUDA(ctx, cudaMemcpyAsync(hm, mm, sizeof(hm), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaMemcpyAsync(&hmt, mt, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaMemcpyAsync(&hni, notinc, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok()) return ctx.rc;
  const long long idmin = n || nd ? hm[0] : 0;
  const int idb = n || nd ? bitlen_u64((uint64_t)(hm[1] - hm[0])) : 0;
  const int tb = bitlen_u64((uint64_t)hmt);
  int64_t nu = 0;
  const bool inc = hni == 0;  // ids strictly increasing: every sort by id is the identity
  if (n && inc) {
    STW_KL(k_id_identity, grid_for(n, 256), 256, ctx.stream, b.id, n, idmin, did, last_of, ukey);
    nu = n;
    // op order: by id (the listing order: ops 2e, 2e + 1), then by (t, is_alloc)
    STW_KL(k_iota, grid_for(2 * n, 256), 256, ctx.stream, operm, 2 * n);
  } else if (n) {
    STW_KL(k_id_keys, grid_for(n, 256), 256, ctx.stream, b.id, n, idmin, k1);
    sort_perm(ctx, ar, k1, perm, n, idb);
    STW_KL(k_heads_u64, grid_for(n, 256), 256, ctx.stream, k1, n, head);
    device_scan<uint32_t>(ctx, ar, head, cls, n, true);
    STW_KL(k_id_classes, grid_for(n, 256), 256, ctx.stream, perm, k1, n, cls, did, last_of, ukey);
    uint32_t hn = 0;
    STW_CUDA(ctx, cudaMemcpyAsync(&hn, cls + n - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    nu = hn;
    // op order: stable by id, then by (t, is_alloc)
    STW_KL(k_op_keys_id, grid_for(2 * n, 256), 256, ctx.stream, b.id, n, idmin, k1);
    sort_perm(ctx, ar, k1, operm, 2 * n, idb);
  }
  if (n) {
    STW_KL(k_op_keys_t, grid_for(2 * n, 256), 256, ctx.stream, operm, b.t_s, b.t_e, n, k1);
    radix_sort_pairs(ctx, ar, k1, operm, 2 * n, 0, tb + 1);
    STW_KL(k_op_rank, grid_for(2 * n, 256), 256, ctx.stream, operm, 2 * n, apos);
  }
  int8_t *route = ar.take<int8_t>(n + 1);
  int64_t *paddr = ar.take<int64_t>(n + 1);
  if (!ctx.ok()) return ctx.rc;
  STW_KL(k_fill_i8, grid_for(n + 1, 256), 256, ctx.stream, route, n + 1, (int8_t)(baseline ? R_ONLINE : R_MISMATCH));
  if (!baseline && n && nd) {
    int32_t *d_ev = ar.take<int32_t>(nd), *d_rank = ar.take<int32_t>(nd);
    if (!ctx.ok()) return ctx.rc;
    STW_KL(k_dec_lookup, grid_for(nd, 256), 256, ctx.stream, d_id, nd, ukey, nu, idmin, last_of, b.dyn, d_ev);
    // queue order of decisions: (t_s, id, plan position)
    STW_KL(k_dec_keys, grid_for(nd, 256), 256, ctx.stream, d_ts, d_id, nd, idmin, k2, k3);
    sort_perm2(ctx, ar, k2, tb, k3, idb, perm, nd);
    STW_KL(k_scatter_rank, grid_for(nd, 256), 256, ctx.stream, perm, nd, d_rank);
    MatchRec M{nd, n, d_ev, d_rank, d_size, b.ps, b.size, b.dyn, apos};
    const int64_t nr = nd + n;
    STW_KL(k_match_keys, grid_for(nr, 256), 256, ctx.stream, M, k1, k2, k3);
    // LSD: (side, order) then size then phase
    sort_perm(ctx, ar, k1, perm, nr, 33);
    STW_KL(k_gather_u64, grid_for(nr, 256), 256, ctx.stream, k2, perm, k1, nr);
    radix_sort_pairs(ctx, ar, k1, perm, nr, 0, 64);
    STW_KL(k_gather_u64, grid_for(nr, 256), 256, ctx.stream, k3, perm, k1, nr);
    radix_sort_pairs(ctx, ar, k1, perm, nr, 0, 32);
    STW_KL(k_match_heads, grid_for(nr, 256), 256, ctx.stream, perm, M, head);
    device_scan<uint32_t>(ctx, ar, head, cls, nr, true);
    uint32_t ng = 0;
    STW_CUDA(ctx, cudaMemcpyAsync(&ng, cls + nr - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    int64_t *gstart = ar.take<int64_t>(ng + 1);
    int32_t *gndec = ar.take<int32_t>(ng + 1);
    if (!ctx.ok()) return ctx.rc;
    STW_CUDA(ctx, cudaMemsetAsync(gndec, 0, (ng + 1) * sizeof(int32_t), ctx.stream));
    STW_KL(k_match_groups, grid_for(nr, 256), 256, ctx.stream, perm, cls, nr, nd, gstart, gndec);
    STW_KL(k_match_assign, grid_for(nr, 256), 256, ctx.stream, perm, cls, nr, M, gstart, gndec, d_addr, route, paddr);
  }
  const int64_t cap_log = 1 + 3 * n;
  // parallel fast path (static-only, every allocation planned, unique ids)
  nv.next("parallel replay");
  if (!baseline && n > 0 && nu == n && nd > 0) {
    int *bad = ar.take<int>(1);
    if (!ctx.ok()) return ctx.rc;
    STW_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), ctx.stream));
    STW_KL(k_fast_flags, grid_for(n, 256, 148 * 4), 256, ctx.stream, route, b.dyn, n, bad);
    int hbad = 1;
    STW_CUDA(ctx, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    if (!ctx.ok()) return ctx.rc;
    if (!hbad) {
      int32_t *rts = ar.take<int32_t>(n), *rte = ar.take<int32_t>(n), *arank = ar.take<int32_t>(2 * n);
      int64_t *rsz = ar.take<int64_t>(n), *raddr = ar.take<int64_t>(n), *delta = ar.take<int64_t>(2 * n);
      uint32_t *af = ar.take<uint32_t>(2 * n);
      int64_t *roff = ar.take<int64_t>(2);
      long long *cnt = ar.take<long long>(1), *pk = ar.take<long long>(1);
      int *first = ar.take<int>(1);
      if (!ctx.ok()) return ctx.rc;
      STW_KL(k_alloc_flag, grid_for(2 * n, 256), 256, ctx.stream, operm, 2 * n, af);
      device_scan<uint32_t>(ctx, ar, af, (uint32_t *)arank, 2 * n, false);
      STW_KL(k_fast_rects, grid_for(2 * n, 256), 256, ctx.stream, operm, n, b.t_s, b.t_e, b.size, paddr,
             arank, rts, rte, rsz, raddr, delta);
      int64_t hoff[2] = {0, n};
      STW_CUDA(ctx, cudaMemcpyAsync(roff, hoff, sizeof(hoff), cudaMemcpyHostToDevice, ctx.stream));
      RectSets rs{1, n, roff, rts, rte, rsz, 1, raddr};
      const long long al = bun->alignment > 0 ? bun->alignment : 1;
      validate_sets(ctx, ar, rs, cnt, first, __builtin_ctzll((unsigned long long)al));
      long long hcnt = -1;
      STW_CUDA(ctx, cudaMemcpyAsync(&hcnt, cnt, sizeof(hcnt), cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
      if (!ctx.ok()) return ctx.rc;
      if (hcnt == 0) {
        device_scan<int64_t>(ctx, ar, delta, delta, 2 * n, true);
        STW_CUDA(ctx, cudaMemsetAsync(pk, 0, sizeof(long long), ctx.stream));
        STW_KL(k_max_scan, grid_for(2 * n, 256, 148 * 4), 256, ctx.stream, delta, 2 * n, pk);
        const int64_t nlog = 1 + 2 * n;
        int8_t *lkind = ar.take<int8_t>(nlog), *lspace = ar.take<int8_t>(nlog), *lroute = ar.take<int8_t>(nlog);
        int64_t *lt = ar.take<int64_t>(nlog), *lid = ar.take<int64_t>(nlog), *lsize = ar.take<int64_t>(nlog),
                *laddr = ar.take<int64_t>(nlog);
        if (!ctx.ok()) return ctx.rc;
        if (log)
          STW_KL(k_fast_log, grid_for(nlog, 256), 256, ctx.stream, operm, n, b.t_s, b.t_e, b.id, b.size, paddr, pool,
                 lkind, lspace, lroute, lt, lid, lsize, laddr);
        long long hpk = 0;
        STW_CUDA(ctx, cudaMemcpyAsync(&hpk, pk, sizeof(hpk), cudaMemcpyDeviceToHost, ctx.stream));
        if (log) {
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
        }
        STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
        if (!ctx.ok()) return ctx.rc;
        rep->allocated_peak = hpk;
        rep->reserved_peak = pool;
        rep->pool_size = pool;
        rep->fallback_count = 0;
        rep->fallback_bytes_peak = 0;
        rep->reuse_hits = 0;
        rep->mismatch_count = 0;
        rep->efficiency = rep->reserved_peak ? exact_div_host(rep->allocated_peak, rep->reserved_peak) : 1.0;
        rep->fragmentation = 1.0 - rep->efficiency;
        return ctx.rc;
      }
    }
  }
  // sequential replay: the register-resident warp when ids are unique and the
  // state fits (replay_reg.cu), else the general warp below
  if (n > 0 && nu == n && !getenv("STW_REPLAY_GENERAL")) {
    nv.next("sequential replay (registers)");
    RegIn ri{n, operm, apos, b.id, b.size, b.t_s, b.t_e, b.dyn, route, paddr, key, sp_off, sp_lo, sp_hi,
             baseline ? 0 : (K ? bun->sp_off[K] : 0), baseline ? 0 : bun->reuse, baseline ? 1 : 0, pool,
             nullptr, 2 * n};
    // simulate: the planned static allocations leave the chain when that is exact
    const bool off = !baseline && !getenv("STW_REPLAY_FULL_CHAIN") && offchain_check(ctx, ar, ri, K);
    if (!ctx.ok()) return ctx.rc;
    if (getenv("STW_REPLAY_STATS"))
      fprintf(stderr, "replay: %s chain, %lld of %lld ops\n", off ? "off-planned" : "full", (long long)ri.nkept,
              (long long)(2 * n));
    long long ho[16] = {0};
    int st = replay_reg(ctx, ar, ri, ho, log);
    if (!ctx.ok()) return ctx.rc;
    if (off && st == 2) {  // (cannot happen when the conditions hold) the full chain decides
      ri.ridx = nullptr;
      ri.nkept = 2 * n;
      st = replay_reg(ctx, ar, ri, ho, log);
      if (!ctx.ok()) return ctx.rc;
    }
    if (st == 2) {
      *err_id = ho[2];
      ctx.fail(STW_ESIM, "planned address %lld for event %lld is occupied", ho[3], ho[2]);
      return ctx.rc;
    }
    if (st == 0) {
      rep->allocated_peak = ho[4];
      rep->reserved_peak = pool + ho[5];
      rep->pool_size = pool;
      rep->fallback_count = ho[7];
      rep->fallback_bytes_peak = ho[6];
      rep->reuse_hits = ho[8];
      rep->mismatch_count = ho[9];
      rep->efficiency = rep->reserved_peak ? exact_div_host(rep->allocated_peak, rep->reserved_peak) : 1.0;
      rep->fragmentation = 1.0 - rep->efficiency;
      return ctx.rc;
    }
  }
  nv.next("sequential replay");
  ReplayArgs R{};
  R.n = n;
  R.operm = operm;
  R.id = b.id;
  R.size = b.size;
  R.ts = b.t_s;
  R.te = b.t_e;
  R.dyn = b.dyn;
  R.did = did;
  R.route0 = route;
  R.paddr = paddr;
  R.key = key;
  R.sp_off = sp_off;
  R.sp_lo = sp_lo;
  R.sp_hi = sp_hi;
  R.reuse = baseline ? 0 : bun->reuse;
  R.baseline = baseline;
  R.pool = pool;
  R.plo = ar.take<int64_t>(n + 1);
  R.phi = ar.take<int64_t>(n + 1);
  R.pflag = ar.take<int8_t>(n + 1);
  R.clo = ar.take<int64_t>(n + 1);
  R.chi = ar.take<int64_t>(n + 1);
  R.cseg = ar.take<int32_t>(n + 1);
  R.cflag = ar.take<int8_t>(n + 1);
  R.gflo = ar.take<int64_t>(n + 3);
  R.gfhi = ar.take<int64_t>(n + 3);
  R.gblo = ar.take<int64_t>(2 * n + 3);
  R.gbhi = ar.take<int64_t>(2 * n + 3);
  R.gbseg = ar.take<int32_t>(2 * n + 3);
  R.sbase = ar.take<int64_t>(n + 2);
  R.lkind = ar.take<int8_t>(cap_log);
  R.lspace = ar.take<int8_t>(cap_log);
  R.lroute = ar.take<int8_t>(cap_log);
  R.lt = ar.take<int64_t>(cap_log);
  R.lid = ar.take<int64_t>(cap_log);
  R.lsize = ar.take<int64_t>(cap_log);
  R.laddr = ar.take<int64_t>(cap_log);
  R.res = ar.take<long long>(16);
  if (!ctx.ok()) return ctx.rc;
  STW_CUDA(ctx, cudaMemsetAsync(R.pflag, 0, n + 1, ctx.stream));
  STW_CUDA(ctx, cudaMemsetAsync(R.cflag, 0, n + 1, ctx.stream));
  STW_CUDA(ctx, cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kReplaySmem));
  {
    int slot = prof_pre(ctx.stream);
    k_replay<<<1, 32, kReplaySmem, ctx.stream>>>(R);
    prof_post(ctx.stream, "k_replay", slot);
  }
  STW_LAUNCHED(ctx);
  long long res[16];
  STW_CUDA(ctx, cudaMemcpyAsync(res, R.res, sizeof(res), cudaMemcpyDeviceToHost, ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  if (!ctx.ok()) return ctx.rc;
  const long long nlog = res[0], err = res[1];
  if (getenv("STW_REPLAY_STATS"))  // list sizes, when built with -DSTW_REPLAY_STATS
    fprintf(stderr, "replay: n=%lld max_nb=%lld max_nf=%lld avg_nb=%.1f avg_nf=%.1f\n", (long long)n, res[10], res[11],
            (double)res[12] / (2.0 * n), (double)res[13] / (2.0 * n));
  if (err) {
    *err_id = res[2];
    if (err == STW_ESIM)
      ctx.fail(STW_ESIM, "planned address %lld for event %lld is occupied", res[3], res[2]);
    else if (err == STW_ESIM + 100)
      ctx.fail(STW_ESIM, "request %lld already live in cache", res[2]);
    else
      ctx.fail(STW_ESIM, baseline ? "free of unknown id %lld in cache" : "double free or free of unknown id %lld",
               res[2]);
    return ctx.rc;
  }
  // compute_metrics (sim.py:67-117)
  rep->allocated_peak = res[4];
  rep->reserved_peak = pool + res[5];
  rep->pool_size = pool;
  rep->fallback_count = res[7];
  rep->fallback_bytes_peak = res[6];
  rep->reuse_hits = res[8];
  rep->mismatch_count = res[9];
  rep->efficiency = rep->reserved_peak ? exact_div_host(rep->allocated_peak, rep->reserved_peak) : 1.0;
  rep->fragmentation = 1.0 - rep->efficiency;
  if (log) {
    log->len = nlog;
    int64_t m = std::min<int64_t>(nlog, log->cap);
    if (m > 0) {
      STW_CUDA(ctx, cudaMemcpyAsync(log->kind, R.lkind, m, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->space, R.lspace, m, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->route, R.lroute, m, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->t, R.lt, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->id, R.lid, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->size, R.lsize, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
      STW_CUDA(ctx, cudaMemcpyAsync(log->addr, R.laddr, m * 8, cudaMemcpyDeviceToHost, ctx.stream));
    }
  }
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  return ctx.rc;
}

}  // namespace stw
