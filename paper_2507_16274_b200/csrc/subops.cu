// The reference planner's and replay's public sub-operations, one call each
// (include/stw.h "sub-operations"): the same arithmetic the batched planner
// runs per trace, exposed for callers that drive the pieces themselves.
//
//   stw_group_events   group_by_phase            planner.py:74-85
//   stw_local_plans    pack_group / _plan_from_decisions / compute_tmp   planner.py:88-115
//   stw_weighted_tmp   weighted_tmp_average      planner.py:118-121
//   stw_fuse_plans     fuse_plans / try_fuse     planner.py:124-182
//   stw_build_layers   build_layers_for_size     planner.py:236-254
//   stw_metrics        compute_metrics           sim.py:67-117
//
// Inputs are host pointers (staged to HBM here), outputs host pointers.
#include <string.h>

#include <vector>

#include "planner.cuh"

namespace stw {

#define GSX(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

namespace {

template <class T>
T *upload(Ctx &ctx, Arena &ar, const T *h, int64_t n) {
  if (!ctx.ok()) return nullptr;
  T *d = ar.take<T>(n > 0 ? n : 1);
  if (d && n > 0) STW_CUDA(ctx, cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, ctx.stream));
  return d;
}

template <class T>
void download(Ctx &ctx, T *h, const T *d, int64_t n) {
  if (ctx.ok() && h && n > 0) STW_CUDA(ctx, cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, ctx.stream));
}

// order-preserving maps onto u64: signed integers flip the sign bit; IEEE
// doubles flip every bit of negatives and the sign bit of the rest
__device__ __forceinline__ uint64_t okey_i64(int64_t v) { return (uint64_t)v ^ (1ull << 63); }
__device__ __forceinline__ uint64_t okey_f64(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v == 0.0 ? 0.0 : v);  // -0.0 == 0.0
  return (b >> 63) ? ~b : b | (1ull << 63);
}

__global__ void k_okeys_i64(const int64_t *__restrict__ v, int64_t n, uint64_t *__restrict__ k) {
  GSX(i, n) k[i] = okey_i64(v[i]);
}
__global__ void k_okeys_f64(const double *__restrict__ v, int64_t n, uint64_t *__restrict__ k) {
  GSX(i, n) k[i] = okey_f64(v[i]);
}

__global__ void k_umin_umax(const uint64_t *__restrict__ v, int64_t n, unsigned long long *mm) {
  unsigned long long lo = ~0ull, hi = 0;
  GSX(i, n) {
    lo = min(lo, (unsigned long long)v[i]);
    hi = max(hi, (unsigned long long)v[i]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void k_gather_rebased(const uint64_t *__restrict__ col, const uint32_t *__restrict__ perm,
                                 unsigned long long lo, int64_t n, uint64_t *__restrict__ key) {
  GSX(i, n) key[i] = col[perm[i]] - lo;
}

// Stable lexicographic sort of n rows by k order-preserving u64 columns
// (cols[0] primary): LSD over the columns, each a K2 radix sort of the column
// (rebased to its minimum, only its significant bits) gathered through the
// permutation so far. perm receives the row order.
void lexsort(Ctx &ctx, Arena &ar, uint64_t *const *cols, int k, int64_t n, uint32_t *perm) {
  if (!ctx.ok() || n <= 0) return;
  unsigned long long *dmm = ar.take<unsigned long long>(2 * k);
  std::vector<unsigned long long> mm(2 * k);
  for (int c = 0; c < k; c++) {
    mm[2 * c] = ~0ull;
    mm[2 * c + 1] = 0;
  }
  if (!ctx.ok()) return;
  STW_CUDA(ctx, cudaMemcpyAsync(dmm, mm.data(), 2 * k * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                                ctx.stream));
  for (int c = 0; c < k; c++) STW_KL(k_umin_umax, grid_for(n, 256, 148 * 4), 256, ctx.stream, cols[c], n, dmm + 2 * c);
  STW_LAUNCHED(ctx);
  STW_CUDA(ctx, cudaMemcpyAsync(mm.data(), dmm, 2 * k * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                ctx.stream));
  STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  uint64_t *key = ar.take<uint64_t>(n);
  if (!ctx.ok()) return;
  STW_KL(k_iota, grid_for(n, 256), 256, ctx.stream, perm, n);
  for (int c = k - 1; c >= 0 && ctx.ok(); c--) {
    const int bits = bitlen_u64(mm[2 * c + 1] - mm[2 * c]);
    if (bits == 0) continue;  // constant column
    STW_KL(k_gather_rebased, grid_for(n, 256), 256, ctx.stream, cols[c], perm, mm[2 * c], n, key);
    STW_LAUNCHED(ctx);
    radix_sort_pairs(ctx, ar, key, perm, n, 0, bits);
  }
}

// ---------------------------------------------------------------------------
// group_by_phase: rows sorted by (p_s, p_e, t_s, id); a group starts where
// (p_s, p_e) changes.

__global__ void k_group_heads(const uint32_t *__restrict__ perm, const uint64_t *__restrict__ ps,
                              const uint64_t *__restrict__ pe, int64_t n, int64_t *__restrict__ head) {
  GSX(i, n) {
    const uint32_t a = perm[i];
    int64_t h = 1;
    if (i > 0) {
      const uint32_t b = perm[i - 1];
      h = (ps[a] != ps[b] || pe[a] != pe[b]) ? 1 : 0;
    }
    head[i] = h;
  }
}

__global__ void k_group_offsets(const int64_t *__restrict__ head, const int64_t *__restrict__ gid, int64_t n,
                                int64_t *__restrict__ off) {
  GSX(i, n) {
    if (head[i]) off[gid[i]] = i;
    if (i == n - 1) off[gid[i] + head[i]] = n;  // one past the last group
  }
}

__global__ void k_perm_i32(const uint32_t *__restrict__ p, int64_t n, int32_t *__restrict__ o) {
  GSX(i, n) o[i] = (int32_t)p[i];
}

// ---------------------------------------------------------------------------
// local plans: one CTA per plan over its members (in the given order)

constexpr int kLpThreads = 256;

struct LocalPlanArgs {
  int64_t P;
  const int64_t *off, *size, *t_s, *t_e, *addr_in;
  const int64_t *h_in, *ts_in, *te_in;
  int64_t *addr_out, *height, *t_lo, *t_hi;
  double *tmp;
  int32_t *rc;
};

__device__ __forceinline__ u128 shfl_down_u128(u128 v, int o) {
  const uint64_t lo = __shfl_down_sync(0xffffffffu, (unsigned long long)(uint64_t)v, o);
  const uint64_t hi = __shfl_down_sync(0xffffffffu, (unsigned long long)(uint64_t)(v >> 64), o);
  return ((u128)hi << 64) | lo;
}

// block-wide (max, min, max, sum) of one value each; results valid in every thread
struct Red4 {
  long long hmax, tmin, tmax;
  u128 used;
};

__device__ Red4 block_red4(Red4 r, Red4 *sh) {
  for (int o = 16; o; o >>= 1) {
    r.hmax = max(r.hmax, __shfl_down_sync(0xffffffffu, r.hmax, o));
    r.tmin = min(r.tmin, __shfl_down_sync(0xffffffffu, r.tmin, o));
    r.tmax = max(r.tmax, __shfl_down_sync(0xffffffffu, r.tmax, o));
    r.used += shfl_down_u128(r.used, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    Red4 a = sh[0];
    for (int k = 1; k < nw; k++) {
      a.hmax = max(a.hmax, sh[k].hmax);
      a.tmin = min(a.tmin, sh[k].tmin);
      a.tmax = max(a.tmax, sh[k].tmax);
      a.used += sh[k].used;
    }
    sh[32] = a;
  }
  __syncthreads();
  Red4 out = sh[32];
  __syncthreads();
  return out;
}

// tmp = used / (height * (t_e - t_s)), Python int/int (planner.py:110-115)
__device__ double tmp_of(u128 used, long long height, long long t_lo, long long t_hi, int32_t *rc) {
  if (t_hi <= t_lo) {
    *rc = STW_EPLAN;  // "degenerate lifespan"
    return 0.0;
  }
  if (height <= 0) {
    *rc = STW_EARG;  // division by zero
    return 0.0;
  }
  *rc = STW_OK;
  return exact_div(used, (u128)(uint64_t)height * (u128)(uint64_t)(t_hi - t_lo));
}

__global__ void __launch_bounds__(kLpThreads) k_local_plans(LocalPlanArgs A) {
  __shared__ Red4 sh[33];
  __shared__ long long shs[33];
  for (int64_t p = blockIdx.x; p < A.P; p += gridDim.x) {
    const int64_t s0 = A.off[p], s1 = A.off[p + 1];
    Red4 r{LLONG_MIN, LLONG_MAX, LLONG_MIN, 0};
    long long carry = 0;  // packing: running prefix of sizes in member order
    for (int64_t b = s0; b < s1; b += kLpThreads) {
      const int64_t i = b + threadIdx.x;
      const bool in = i < s1;
      const long long sz = in ? A.size[i] : 0;
      long long a;
      if (A.addr_in) {
        a = in ? A.addr_in[i] : 0;
      } else {
        long long tot;
        a = carry + block_excl_sum<long long>(sz, shs, &tot);
        carry += tot;
      }
      if (in) {
        if (A.addr_out) A.addr_out[i] = a;
        const long long ts = A.t_s[i], te = A.t_e[i];
        r.hmax = max(r.hmax, a + sz);
        r.tmin = min(r.tmin, ts);
        r.tmax = max(r.tmax, te);
        r.used += (u128)(uint64_t)sz * (u128)(uint64_t)(te - ts);
      }
    }
    r = block_red4(r, sh);
    if (threadIdx.x == 0) {
      const long long h = A.h_in ? A.h_in[p] : r.hmax;
      const long long lo = A.ts_in ? A.ts_in[p] : r.tmin;
      const long long hi = A.te_in ? A.te_in[p] : r.tmax;
      int32_t rc;
      const double t = s1 > s0 || A.h_in ? tmp_of(r.used, h, lo, hi, &rc) : (rc = STW_EPLAN, 0.0);
      A.height[p] = h;
      A.t_lo[p] = lo;
      A.t_hi[p] = hi;
      A.tmp[p] = t;
      A.rc[p] = rc;
    }
  }
}

// ---------------------------------------------------------------------------
// weighted_tmp_average (planner.py:118-121) with CPython 3.12 float semantics:
// each term float(tmp) * float(int weight) (int -> double round-half-even), the
// builtin sum's Neumaier-compensated accumulation, then / float(sum of weights).

__device__ double weighted_avg(int n, const double *tmp, const u128 *w) {
  double f = 0.0, c = 0.0;
  u128 tw = 0;
  for (int i = 0; i < n; i++) {
    const double x = __dmul_rn(tmp[i], u128_to_double_rne(w[i]));
    tw += w[i];
    if (i == 0) {
      f = __dadd_rn(0.0, x);  // int 0 + float
      continue;
    }
    const double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x))
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
    else
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
  return __ddiv_rn(f, u128_to_double_rne(tw));
}

__global__ void k_weighted_tmp(int64_t n, const double *__restrict__ tmp, const int64_t *__restrict__ h,
                               const int64_t *__restrict__ dur, u128 *__restrict__ w, double *out) {
  for (int64_t i = 0; i < n; i++) w[i] = (u128)(uint64_t)h[i] * (u128)(uint64_t)dur[i];
  *out = weighted_avg((int)n, tmp, w);
}

// ---------------------------------------------------------------------------
// fuse_plans: the cursor walk of planner.py:132-169 in one CTA. Each step the
// CTA tests the unplaced smaller-plan decisions (in (t_s, id) order) against
// every fixed rectangle, a chunk of blockDim at a time, and takes the first
// conflict-free one; with none, the cursor jumps to the next anchor above it
// or to the top of everything fixed.

constexpr int kFuseThreads = 512;

struct FuseArgs {
  int64_t nL, nS;
  const int64_t *L_addr, *L_size, *L_ts, *L_te;
  const int64_t *S_size, *S_ts, *S_te;
  const uint32_t *S_order;  // smaller's decisions in (t_s, id) order
  const uint64_t *anchors;  // larger's addresses, sorted (okey)
  int64_t *F_addr, *F_size, *F_ts, *F_te;  // fixed rectangles (nL + nS)
  uint8_t *placed;
  int64_t *out_addr;   // [nS] per smaller decision (input order)
  int32_t *out_order;  // [nS] placement order (input indices)
  // fused plan (planner.py:165-169 via _plan_from_decisions) and acceptance
  double L_tmp, S_tmp;
  int64_t L_h, L_dur, S_h, S_dur;
  int64_t *res_i;  // height, t_lo, t_hi, rc
  double *res_d;   // fused tmp, weighted average of (larger, smaller)
};

__global__ void __launch_bounds__(kFuseThreads) k_fuse(FuseArgs A) {
  __shared__ long long s_addr, s_top;
  __shared__ int64_t s_nF, s_k;
  __shared__ int s_found;
  __shared__ Red4 sh[33];
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < A.nL; i += blockDim.x) {
    A.F_addr[i] = A.L_addr[i];
    A.F_size[i] = A.L_size[i];
    A.F_ts[i] = A.L_ts[i];
    A.F_te[i] = A.L_te[i];
  }
  for (int64_t i = tid; i < A.nS; i += blockDim.x) A.placed[i] = 0;
  {
    Red4 r{LLONG_MIN, 0, 0, 0};
    for (int64_t i = tid; i < A.nL; i += blockDim.x) r.hmax = max(r.hmax, (long long)(A.L_addr[i] + A.L_size[i]));
    r = block_red4(r, sh);
    if (tid == 0) {
      s_top = r.hmax;
      s_addr = (long long)(A.anchors[0] ^ (1ull << 63));
      s_nF = A.nL;
      s_k = 0;
    }
  }
  __syncthreads();
  while (s_k < A.nS) {
    const long long addr = s_addr;
    const int64_t nF = s_nF;
    if (tid == 0) s_found = INT_MAX;
    __syncthreads();
    for (int64_t b = 0; b < A.nS; b += blockDim.x) {
      const int64_t j = b + tid;
      bool ok = j < A.nS && !A.placed[j];
      if (ok) {
        const uint32_t s = A.S_order[j];
        const long long hi = addr + A.S_size[s], ts = A.S_ts[s], te = A.S_te[s];
        for (int64_t f = 0; f < nF; f++) {
          const long long fa = A.F_addr[f];
          if (fa < hi && addr < fa + A.F_size[f] && A.F_ts[f] < te && ts < A.F_te[f]) {
            ok = false;
            break;
          }
        }
      }
      if (ok) atomicMin(&s_found, (int)j);
      __syncthreads();
      const int found = s_found;
      __syncthreads();
      if (found != INT_MAX) break;
    }
    if (tid == 0) {
      const int j = s_found;
      if (j != INT_MAX) {
        const uint32_t s = A.S_order[j];
        const int64_t f = s_nF;
        A.F_addr[f] = addr;
        A.F_size[f] = A.S_size[s];
        A.F_ts[f] = A.S_ts[s];
        A.F_te[f] = A.S_te[s];
        A.placed[j] = 1;
        A.out_addr[s] = addr;
        A.out_order[s_k] = (int32_t)s;
        s_top = max(s_top, addr + (long long)A.S_size[s]);
        s_addr = addr + A.S_size[s];
        s_nF = f + 1;
        s_k = s_k + 1;
      } else {
        // next anchor strictly above the cursor (planner.py:163-164)
        int64_t lo = 0, hi = A.nL;
        const uint64_t key = (uint64_t)addr ^ (1ull << 63);
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (A.anchors[mid] <= key)
            lo = mid + 1;
          else
            hi = mid;
        }
        s_addr = lo < A.nL ? (long long)(A.anchors[lo] ^ (1ull << 63)) : s_top;
      }
    }
    __syncthreads();
  }
  // the fused plan's height / span / tmp over larger + placed
  Red4 r{LLONG_MIN, LLONG_MAX, LLONG_MIN, 0};
  const int64_t nF = A.nL + A.nS;
  for (int64_t i = tid; i < nF; i += blockDim.x) {
    const long long a = A.F_addr[i], sz = A.F_size[i], ts = A.F_ts[i], te = A.F_te[i];
    r.hmax = max(r.hmax, a + sz);
    r.tmin = min(r.tmin, ts);
    r.tmax = max(r.tmax, te);
    r.used += (u128)(uint64_t)sz * (u128)(uint64_t)(te - ts);
  }
  r = block_red4(r, sh);
  if (tid == 0) {
    int32_t rc;
    const double t = tmp_of(r.used, r.hmax, r.tmin, r.tmax, &rc);
    double tm[2] = {A.L_tmp, A.S_tmp};
    u128 w[2] = {(u128)(uint64_t)A.L_h * (u128)(uint64_t)A.L_dur, (u128)(uint64_t)A.S_h * (u128)(uint64_t)A.S_dur};
    A.res_i[0] = r.hmax;
    A.res_i[1] = r.tmin;
    A.res_i[2] = r.tmax;
    A.res_i[3] = rc;
    A.res_d[0] = t;
    A.res_d[1] = (w[0] + w[1]) != 0 ? weighted_avg(2, tm, w) : 0.0;
  }
}

// ---------------------------------------------------------------------------
// build_layers_for_size (Alg. 1): items in (t_s, tie) order; each joins the
// layer with the largest end strictly below its start (ties: oldest layer),
// else opens a new one. One warp; lanes stride over the layers.

__global__ void __launch_bounds__(32) k_alg1(const uint32_t *__restrict__ order, const double *__restrict__ ts,
                                             const double *__restrict__ te, int64_t n, double *__restrict__ lend,
                                             int32_t *__restrict__ layer_of, int64_t *n_layers) {
  const int lane = threadIdx.x;
  int64_t L = 0;
  for (int64_t k = 0; k < n; k++) {
    const uint32_t it = order[k];
    const double s = ts[it];
    double best = 0.0;
    int64_t bl = -1;
    for (int64_t l = lane; l < L; l += 32) {
      const double e = lend[l];
      if (e < s && (bl < 0 || e > best)) best = e, bl = l;  // l increasing: first max kept
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, o);
      const long long ol = __shfl_down_sync(0xffffffffu, (long long)bl, o);
      if (ol >= 0 && (bl < 0 || ob > best || (ob == best && ol < bl))) best = ob, bl = ol;
    }
    bl = __shfl_sync(0xffffffffu, (long long)bl, 0);
    if (lane == 0) {
      const double e = te[it];
      if (bl < 0) {
        lend[L] = e;
        layer_of[it] = (int32_t)L;
      } else {
        if (e > lend[bl]) lend[bl] = e;  // MemoryLayer.insert keeps the max end
        layer_of[it] = (int32_t)bl;
      }
    }
    if (bl < 0) L++;
    __syncwarp();
  }
  if (lane == 0) *n_layers = L;
}

// ---------------------------------------------------------------------------
// compute_metrics: one CTA folds the log tile by tile (block scans of the live
// byte deltas for the running peaks, block sums for the counts).

constexpr int kMtThreads = 1024;

__global__ void __launch_bounds__(kMtThreads) k_metrics(int64_t n, const int8_t *__restrict__ kind,
                                                        const int64_t *__restrict__ size,
                                                        const int8_t *__restrict__ space,
                                                        const int8_t *__restrict__ route, stw_report *rep) {
  __shared__ long long sh[33];
  long long live = 0, cache = 0, peak = 0, cpeak = 0;
  long long reserved = 0, fb = 0, mm = 0, ru = 0, init_at = -1;
  for (int64_t b = 0; b < n; b += kMtThreads) {
    const int64_t i = b + threadIdx.x;
    long long d = 0, dc = 0, res = 0, f = 0, m = 0, r = 0, ia = -1;
    if (i < n) {
      const int k = kind[i];
      const long long sz = size[i];
      if (k == 0) ia = i;
      if (k == 1) res = sz;
      if (k == 2) {
        d = sz;
        if (space[i] == 1) dc = sz;
        const int rt = route[i];
        f = (rt == 2 || rt == 3);
        m = rt == 3;
        r = rt == 1;
      }
      if (k == 3) {
        d = -sz;
        if (space[i] == 1) dc = -sz;
      }
    }
    long long tot;
    const long long pre = block_excl_sum<long long>(d, sh, &tot) + d + live;  // inclusive running live
    live += tot;
    const long long prec = block_excl_sum<long long>(dc, sh, &tot) + dc + cache;
    cache += tot;
    long long pk = i < n && kind[i] == 2 ? pre : LLONG_MIN, cpk = i < n && kind[i] == 2 && space[i] == 1 ? prec : LLONG_MIN;
    for (int o = 16; o; o >>= 1) {
      pk = max(pk, __shfl_down_sync(0xffffffffu, pk, o));
      cpk = max(cpk, __shfl_down_sync(0xffffffffu, cpk, o));
      res += __shfl_down_sync(0xffffffffu, res, o);
      f += __shfl_down_sync(0xffffffffu, f, o);
      m += __shfl_down_sync(0xffffffffu, m, o);
      r += __shfl_down_sync(0xffffffffu, r, o);
      ia = max(ia, __shfl_down_sync(0xffffffffu, ia, o));
    }
    __shared__ long long wv[7][32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      wv[0][w] = pk, wv[1][w] = cpk, wv[2][w] = res, wv[3][w] = f, wv[4][w] = m, wv[5][w] = r, wv[6][w] = ia;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int x = 0; x < kMtThreads / 32; x++) {
        peak = max(peak, wv[0][x]);
        cpeak = max(cpeak, wv[1][x]);
        reserved += wv[2][x];
        fb += wv[3][x];
        mm += wv[4][x];
        ru += wv[5][x];
        init_at = max(init_at, wv[6][x]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const long long pool = init_at >= 0 ? size[init_at] : 0;
    rep->allocated_peak = peak;
    rep->reserved_peak = pool + reserved;
    rep->pool_size = pool;
    rep->fallback_count = fb;
    rep->fallback_bytes_peak = cpeak;
    rep->reuse_hits = ru;
    rep->mismatch_count = mm;
    const long long rp = pool + reserved;
    rep->efficiency = rp ? exact_div((u128)(uint64_t)peak, (u128)(uint64_t)rp) : 1.0;
    rep->fragmentation = __dsub_rn(1.0, rep->efficiency);
  }
}

}  // namespace

}  // namespace stw

using namespace stw;

#define STW_SUB_ENTRY(stream_ptr, err, errlen) \
  Ctx ctx;                                      \
  ctx.stream = (cudaStream_t)(stream_ptr);      \
  ctx.err = (err);                              \
  ctx.errlen = (errlen);                        \
  if ((err) && (errlen)) (err)[0] = 0;          \
  bind_stream_device(ctx.stream);

static int sub_finish(Ctx &ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx.stream);
  if (e != cudaSuccess) ctx.fail(STW_ECUDA, "stream sync: %s", cudaGetErrorString(e));
  return ctx.rc;
}

static constexpr int64_t kSubMax = kSortMax;  // every sub-operation sorts its rows with K2

extern "C" {

int stw_group_events(int64_t n, const int64_t *ps, const int64_t *pe, const int64_t *t_s, const int64_t *id,
                     int32_t *perm, int64_t *grp_off, int64_t *n_groups, void *stream, char *err, size_t errlen) {
  STW_SUB_ENTRY(stream, err, errlen);
  if (n < 0 || n > kSubMax || !n_groups || (n > 0 && (!ps || !pe || !t_s || !id || !perm || !grp_off))) {
    ctx.fail(STW_EARG, "bad group_events arguments");
    return ctx.rc;
  }
  *n_groups = 0;
  if (n == 0) return STW_OK;
  {
    Arena ar(&ctx);
    const int64_t *src[4] = {ps, pe, t_s, id};
    uint64_t *cols[4];
    for (int c = 0; c < 4; c++) {
      int64_t *d = upload(ctx, ar, src[c], n);
      cols[c] = ar.take<uint64_t>(n);
      if (!ctx.ok()) break;
      STW_KL(k_okeys_i64, grid_for(n, 256), 256, ctx.stream, d, n, cols[c]);
    }
    uint32_t *p = ar.take<uint32_t>(n);
    lexsort(ctx, ar, cols, 4, n, p);
    int64_t *head = ar.take<int64_t>(n), *gid = ar.take<int64_t>(n), *off = ar.take<int64_t>(n + 1);
    int32_t *p32 = ar.take<int32_t>(n);
    if (ctx.ok()) {
      STW_KL(k_group_heads, grid_for(n, 256), 256, ctx.stream, p, cols[0], cols[1], n, head);
      device_scan<int64_t>(ctx, ar, head, gid, n, false);
      STW_KL(k_group_offsets, grid_for(n, 256), 256, ctx.stream, head, gid, n, off);
      STW_KL(k_perm_i32, grid_for(n, 256), 256, ctx.stream, p, n, p32);
      STW_LAUNCHED(ctx);
    }
    int64_t last[2] = {0, 0};
    download(ctx, last, gid + n - 1, 1);
    download(ctx, last + 1, head + n - 1, 1);
    download(ctx, perm, p32, n);
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
    if (ctx.ok()) {
      *n_groups = last[0] + last[1];
      download(ctx, grp_off, off, *n_groups + 1);
    }
  }
  return sub_finish(ctx);
}

int stw_local_plans(const stw_lplans *lp, void *stream, char *err, size_t errlen) {
  STW_SUB_ENTRY(stream, err, errlen);
  if (!lp || lp->n_plans < 0 || lp->n < 0 || lp->n > kSubMax || !lp->off || !lp->height || !lp->t_lo ||
      !lp->t_hi || !lp->tmp || !lp->rc || (lp->n > 0 && (!lp->size || !lp->t_s || !lp->t_e))) {
    ctx.fail(STW_EARG, "bad local_plans arguments");
    return ctx.rc;
  }
  const int64_t P = lp->n_plans, n = lp->n;
  if (P == 0) return STW_OK;
  {
    Arena ar(&ctx);
    LocalPlanArgs A{};
    A.P = P;
    A.off = upload(ctx, ar, lp->off, P + 1);
    A.size = upload(ctx, ar, lp->size, n);
    A.t_s = upload(ctx, ar, lp->t_s, n);
    A.t_e = upload(ctx, ar, lp->t_e, n);
    A.addr_in = lp->addr ? upload(ctx, ar, lp->addr, n) : nullptr;
    A.h_in = lp->height_in ? upload(ctx, ar, lp->height_in, P) : nullptr;
    A.ts_in = lp->t_lo_in ? upload(ctx, ar, lp->t_lo_in, P) : nullptr;
    A.te_in = lp->t_hi_in ? upload(ctx, ar, lp->t_hi_in, P) : nullptr;
    A.addr_out = lp->addr_out ? ar.take<int64_t>(n > 0 ? n : 1) : nullptr;
    A.height = ar.take<int64_t>(P);
    A.t_lo = ar.take<int64_t>(P);
    A.t_hi = ar.take<int64_t>(P);
    A.tmp = ar.take<double>(P);
    A.rc = ar.take<int32_t>(P);
    if (ctx.ok()) {
      STW_KL(k_local_plans, (unsigned)std::min<int64_t>(P, 148 * 16), kLpThreads, ctx.stream, A);
      STW_LAUNCHED(ctx);
    }
    if (lp->addr_out) download(ctx, lp->addr_out, A.addr_out, n);
    download(ctx, lp->height, A.height, P);
    download(ctx, lp->t_lo, A.t_lo, P);
    download(ctx, lp->t_hi, A.t_hi, P);
    download(ctx, lp->tmp, A.tmp, P);
    download(ctx, lp->rc, A.rc, P);
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  }
  return sub_finish(ctx);
}

int stw_weighted_tmp(int64_t n, const double *tmp, const int64_t *height, const int64_t *dur, double *out,
                     void *stream, char *err, size_t errlen) {
  STW_SUB_ENTRY(stream, err, errlen);
  if (n <= 0 || n > (1 << 24) || !tmp || !height || !dur || !out) {
    ctx.fail(STW_EARG, "bad weighted_tmp arguments");
    return ctx.rc;
  }
  {
    Arena ar(&ctx);
    const double *t = upload(ctx, ar, tmp, n);
    const int64_t *h = upload(ctx, ar, height, n), *d = upload(ctx, ar, dur, n);
    u128 *w = ar.take<u128>(n);
    double *o = ar.take<double>(1);
    if (ctx.ok()) {
      STW_KL(k_weighted_tmp, 1, 1, ctx.stream, n, t, h, d, w, o);
      STW_LAUNCHED(ctx);
    }
    download(ctx, out, o, 1);
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  }
  return sub_finish(ctx);
}

int stw_fuse_plans(const stw_fusion *fz, void *stream, char *err, size_t errlen) {
  STW_SUB_ENTRY(stream, err, errlen);
  if (!fz || fz->n_large <= 0 || fz->n_small <= 0 || fz->n_large + fz->n_small > kSubMax || !fz->out_addr ||
      !fz->out_order || !fz->result_i || !fz->result_d) {
    ctx.fail(STW_EARG, "bad fuse arguments");
    return ctx.rc;
  }
  const int64_t nL = fz->n_large, nS = fz->n_small;
  {
    Arena ar(&ctx);
    FuseArgs A{};
    A.nL = nL;
    A.nS = nS;
    int64_t *la = upload(ctx, ar, fz->l_addr, nL);
    A.L_addr = la;
    A.L_size = upload(ctx, ar, fz->l_size, nL);
    A.L_ts = upload(ctx, ar, fz->l_ts, nL);
    A.L_te = upload(ctx, ar, fz->l_te, nL);
    int64_t *sts = upload(ctx, ar, fz->s_ts, nS), *sid = upload(ctx, ar, fz->s_id, nS);
    A.S_size = upload(ctx, ar, fz->s_size, nS);
    A.S_ts = sts;
    A.S_te = upload(ctx, ar, fz->s_te, nS);
    // smaller's decisions in (t_s, id) order (planner.py:147); larger's addresses sorted (planner.py:145)
    uint64_t *ck[2] = {ar.take<uint64_t>(nS), ar.take<uint64_t>(nS)};
    uint64_t *anc = ar.take<uint64_t>(nL);
    uint32_t *sorder = ar.take<uint32_t>(nS), *aperm = ar.take<uint32_t>(nL);
    if (ctx.ok()) {
      STW_KL(k_okeys_i64, grid_for(nS, 256), 256, ctx.stream, sts, nS, ck[0]);
      STW_KL(k_okeys_i64, grid_for(nS, 256), 256, ctx.stream, sid, nS, ck[1]);
      STW_KL(k_okeys_i64, grid_for(nL, 256), 256, ctx.stream, la, nL, anc);
      STW_KL(k_iota, grid_for(nL, 256), 256, ctx.stream, aperm, nL);
      STW_LAUNCHED(ctx);
    }
    lexsort(ctx, ar, ck, 2, nS, sorder);
    radix_sort_pairs(ctx, ar, anc, aperm, nL, 0, 64);
    A.S_order = sorder;
    A.anchors = anc;
    A.F_addr = ar.take<int64_t>(nL + nS);
    A.F_size = ar.take<int64_t>(nL + nS);
    A.F_ts = ar.take<int64_t>(nL + nS);
    A.F_te = ar.take<int64_t>(nL + nS);
    A.placed = ar.take<uint8_t>(nS);
    A.out_addr = ar.take<int64_t>(nS);
    A.out_order = ar.take<int32_t>(nS);
    A.L_tmp = fz->l_tmp;
    A.S_tmp = fz->s_tmp;
    A.L_h = fz->l_height;
    A.L_dur = fz->l_dur;
    A.S_h = fz->s_height;
    A.S_dur = fz->s_dur;
    A.res_i = ar.take<int64_t>(4);
    A.res_d = ar.take<double>(2);
    if (ctx.ok()) {
      STW_KL(k_fuse, 1, kFuseThreads, ctx.stream, A);
      STW_LAUNCHED(ctx);
    }
    download(ctx, fz->out_addr, A.out_addr, nS);
    download(ctx, fz->out_order, A.out_order, nS);
    download(ctx, fz->result_i, A.res_i, 4);
    download(ctx, fz->result_d, A.res_d, 2);
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  }
  return sub_finish(ctx);
}

int stw_build_layers(int64_t n, const double *t_s, const double *t_e, const int64_t *tie, int32_t *layer_of,
                     int32_t *order, int64_t *n_layers, void *stream, char *err, size_t errlen) {
  STW_SUB_ENTRY(stream, err, errlen);
  if (n < 0 || n > kSubMax || !n_layers || (n > 0 && (!t_s || !t_e || !tie || !layer_of || !order))) {
    ctx.fail(STW_EARG, "bad build_layers arguments");
    return ctx.rc;
  }
  *n_layers = 0;
  if (n == 0) return STW_OK;
  {
    Arena ar(&ctx);
    double *ts = upload(ctx, ar, t_s, n), *te = upload(ctx, ar, t_e, n);
    int64_t *tk = upload(ctx, ar, tie, n);
    uint64_t *ck[2] = {ar.take<uint64_t>(n), ar.take<uint64_t>(n)};
    uint32_t *p = ar.take<uint32_t>(n);
    double *lend = ar.take<double>(n);
    int32_t *lof = ar.take<int32_t>(n), *p32 = ar.take<int32_t>(n);
    int64_t *nl = ar.take<int64_t>(1);
    if (ctx.ok()) {
      STW_KL(k_okeys_f64, grid_for(n, 256), 256, ctx.stream, ts, n, ck[0]);
      STW_KL(k_okeys_i64, grid_for(n, 256), 256, ctx.stream, tk, n, ck[1]);
      STW_LAUNCHED(ctx);
    }
    lexsort(ctx, ar, ck, 2, n, p);
    if (ctx.ok()) {
      STW_KL(k_alg1, 1, 32, ctx.stream, p, ts, te, n, lend, lof, nl);
      STW_KL(k_perm_i32, grid_for(n, 256), 256, ctx.stream, p, n, p32);
      STW_LAUNCHED(ctx);
    }
    download(ctx, layer_of, lof, n);
    download(ctx, order, p32, n);
    download(ctx, n_layers, nl, 1);
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  }
  return sub_finish(ctx);
}

int stw_metrics(int64_t n, const int8_t *kind, const int64_t *size, const int8_t *space, const int8_t *route,
                stw_report *rep, void *stream, char *err, size_t errlen) {
  STW_SUB_ENTRY(stream, err, errlen);
  if (n < 0 || !rep || (n > 0 && (!kind || !size || !space || !route))) {
    ctx.fail(STW_EARG, "bad metrics arguments");
    return ctx.rc;
  }
  {
    Arena ar(&ctx);
    const int8_t *k = upload(ctx, ar, kind, n), *sp = upload(ctx, ar, space, n), *rt = upload(ctx, ar, route, n);
    const int64_t *sz = upload(ctx, ar, size, n);
    stw_report *d = ar.take<stw_report>(1);
    if (ctx.ok()) {
      STW_KL(k_metrics, 1, kMtThreads, ctx.stream, n, k, sz, sp, rt, d);
      STW_LAUNCHED(ctx);
    }
    download(ctx, rep, d, 1);
    STW_CUDA(ctx, cudaStreamSynchronize(ctx.stream));
  }
  return sub_finish(ctx);
}

}  // extern "C"
