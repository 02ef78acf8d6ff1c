// libstw_alloc -- CUDAPluggableAllocator serving a plan at runtime (include/stw_alloc.h).
//
// Host-side state machine with the reference replay's routing (sim.py:143-232,
// baseline.py:35-95); the memory itself is one cudaMalloc'd pool plus
// power-of-two fallback segments in HBM.
#include "../../include/stw_alloc.h"

#include <cuda_runtime.h>

#include <math.h>

#include <algorithm>
#include <deque>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace {

constexpr int64_t kMinSegment = 2ll * 1024 * 1024;

struct Segment {
  int64_t vbase, size;
  char *dev;
  std::vector<std::pair<int64_t, int64_t>> free;  // sorted (lo, hi) virtual
};

struct Live {
  int space;  // 0 pool, 1 cache
  int route;
  int64_t vaddr, size;
  int seg;
};

struct State {
  std::mutex mu;
  int device = 0;
  int64_t pool_size = 0, alignment = 512;
  char *pool = nullptr;
  std::map<int64_t, int64_t> free;  // coalesced free intervals of the pool (lo -> hi)
  std::map<std::pair<int32_t, int64_t>, std::deque<int64_t>> queues;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> spaces;
  std::vector<Segment> segs;
  int64_t next_vbase = 0;
  std::unordered_map<const void *, Live> live;
  int32_t phase = 0, key = -1, dynamic = 0;
  // metrics (sim.py:67-117)
  int64_t cur = 0, peak = 0, cache_cur = 0, cache_peak = 0, reserved = 0;
  int64_t fallback = 0, reuse = 0, mismatch = 0, occupied = 0;
};

State &S() {
  static State s;
  return s;
}

bool pool_contains(State &s, int64_t lo, int64_t hi) {
  auto it = s.free.upper_bound(lo);
  if (it == s.free.begin()) return false;
  --it;
  return it->first <= lo && hi <= it->second;
}

void pool_remove(State &s, int64_t lo, int64_t hi) {  // [lo, hi) lies inside one free interval
  auto it = s.free.upper_bound(lo);
  --it;
  int64_t a = it->first, b = it->second;
  s.free.erase(it);
  if (a < lo) s.free[a] = lo;
  if (hi < b) s.free[hi] = b;
}

void pool_add(State &s, int64_t lo, int64_t hi) {  // IntervalSet.add (intervals.py:100-111)
  auto it = s.free.lower_bound(lo);
  if (it != s.free.begin()) {
    auto p = std::prev(it);
    if (p->second >= lo) it = p;
  }
  while (it != s.free.end() && it->first <= hi) {
    lo = std::min(lo, it->first);
    hi = std::max(hi, it->second);
    it = s.free.erase(it);
  }
  s.free[lo] = hi;
}

// best fit inside free ∩ space (sim.py:120-140, intervals.py:138-176)
int64_t reuse_fit(State &s, int key, int64_t size) {
  if (key < 0 || key >= (int)s.spaces.size() || s.spaces[key].empty()) return -1;
  int64_t best_len = INT64_MAX, best_lo = -1;
  for (auto &sp : s.spaces[key]) {
    auto it = s.free.upper_bound(sp.first);
    if (it != s.free.begin()) --it;
    for (; it != s.free.end() && it->first < sp.second; ++it) {
      int64_t lo = std::max(it->first, sp.first), hi = std::min(it->second, sp.second);
      if (hi - lo >= size && hi - lo < best_len) best_len = hi - lo, best_lo = lo;
    }
  }
  return best_lo;
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// CachingAllocator.malloc (baseline.py:49-77); returns virtual address or -1
int64_t cache_malloc(State &s, int64_t size, int *seg_out) {
  int bs = -1, bi = -1;
  int64_t blen = 0;
  for (int g = 0; g < (int)s.segs.size(); g++)
    for (int i = 0; i < (int)s.segs[g].free.size(); i++) {
      int64_t len = s.segs[g].free[i].second - s.segs[g].free[i].first;
      if (len >= size && (bs < 0 || len < blen)) bs = g, bi = i, blen = len;
    }
  if (bs < 0) {
    int64_t ss = std::max(kMinSegment, next_pow2(size));
    Segment seg{s.next_vbase, ss, nullptr, {}};
    if (cudaMalloc(&seg.dev, (size_t)ss) != cudaSuccess) return -1;
    seg.free.push_back({seg.vbase, seg.vbase + ss});
    s.next_vbase += ss;
    s.reserved += ss;
    s.segs.push_back(std::move(seg));
    bs = (int)s.segs.size() - 1;
    bi = 0;
  }
  Segment &seg = s.segs[bs];
  auto blk = seg.free[bi];
  seg.free.erase(seg.free.begin() + bi);
  if (blk.first + size < blk.second) seg.free.insert(seg.free.begin() + bi, {blk.first + size, blk.second});
  *seg_out = bs;
  return blk.first;
}

void cache_free(State &s, int g, int64_t lo, int64_t size) {  // CachingAllocator.free (baseline.py:79-95)
  auto &fr = s.segs[g].free;
  int64_t hi = lo + size;
  auto pos = std::lower_bound(fr.begin(), fr.end(), std::make_pair(lo, hi));
  size_t i = pos - fr.begin();
  fr.insert(pos, {lo, hi});
  if (i + 1 < fr.size() && fr[i + 1].first == hi) {
    fr[i].second = fr[i + 1].second;
    fr.erase(fr.begin() + i + 1);
  }
  if (i > 0 && fr[i - 1].second == lo) {
    fr[i - 1].second = fr[i].second;
    fr.erase(fr.begin() + i);
  }
}

// correctly rounded a / b, like Python's int true division (sim.py:103-106)
double exact_div(uint64_t a, uint64_t b) {
  if (a == 0) return 0.0;
  if (a < (1ull << 53) && b < (1ull << 53)) return (double)a / (double)b;
  uint64_t q = a / b, r = a % b, mant;
  int nq = q ? 64 - __builtin_clzll(q) : 0, ex;
  bool sticky;
  if (nq >= 54) {
    int sh = nq - 54;
    mant = q >> sh;
    sticky = (sh && (q & ((1ull << sh) - 1))) || r;
    ex = sh;
  } else {
    int have = nq;
    mant = q;
    ex = 0;
    while (have < 54) {
      bool carry = r >> 63;
      r <<= 1;
      uint64_t bit = 0;
      if (carry || r >= b) r -= b, bit = 1;
      mant = (mant << 1) | bit;
      ex--;
      if (have > 0 || bit) have++;
    }
    sticky = r != 0;
  }
  bool rnd = mant & 1;
  mant >>= 1;
  ex++;
  if (rnd && (sticky || (mant & 1))) mant++;
  return ldexp((double)mant, ex);
}

void account_alloc(State &s, int64_t size, bool cache, int route) {
  s.cur += size;
  s.peak = std::max(s.peak, s.cur);
  if (cache) {
    s.cache_cur += size;
    s.cache_peak = std::max(s.cache_peak, s.cache_cur);
  }
  if (route == 2 || route == 3) s.fallback++;
  if (route == 3) s.mismatch++;
  if (route == 1) s.reuse++;
}

}  // namespace

extern "C" {

int stw_alloc_init(int device, int64_t pool_size, int64_t alignment) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (s.pool) return STW_EARG;
  if (cudaSetDevice(device) != cudaSuccess) return STW_ECUDA;
  s.device = device;
  s.pool_size = pool_size;
  s.alignment = alignment > 0 ? alignment : 512;
  if (pool_size > 0 && cudaMalloc(&s.pool, (size_t)pool_size) != cudaSuccess) {
    s.pool = nullptr;
    return STW_ECUDA;
  }
  s.free.clear();
  if (pool_size > 0) s.free[0] = pool_size;
  s.next_vbase = pool_size;
  return STW_OK;
}

int stw_alloc_load_plan(int64_t n_dec, const int32_t *phase, const int64_t *size, const int64_t *addr,
                        const int32_t *t_s, const int64_t *id, int64_t n_keys, const int64_t *sp_off,
                        const int64_t *sp_lo, const int64_t *sp_hi) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  std::vector<int64_t> order(n_dec);
  for (int64_t k = 0; k < n_dec; k++) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return t_s[a] != t_s[b] ? t_s[a] < t_s[b] : id[a] < id[b];
  });
  s.queues.clear();
  for (int64_t k : order) {
    if (addr[k] < 0 || addr[k] + size[k] > s.pool_size) return STW_EPLAN;
    s.queues[{phase[k], size[k]}].push_back(addr[k]);
  }
  s.spaces.assign(n_keys, {});
  for (int64_t k = 0; k < n_keys; k++)
    for (int64_t j = sp_off[k]; j < sp_off[k + 1]; j++) s.spaces[k].push_back({sp_lo[j], sp_hi[j]});
  return STW_OK;
}

void stw_set_phase(int32_t phase) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  s.phase = phase;
}

void stw_set_layer(int32_t key, int32_t dynamic) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  s.key = key;
  s.dynamic = dynamic;
}

void *stw_malloc(size_t nbytes, int device, void *stream) {
  (void)device;
  (void)stream;
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (nbytes == 0) nbytes = 1;
  int64_t size = (int64_t)((nbytes + s.alignment - 1) / s.alignment * s.alignment);
  int route;
  int64_t vaddr = -1;
  if (s.dynamic) {
    vaddr = reuse_fit(s, s.key, size);
    if (vaddr >= 0) {
      pool_remove(s, vaddr, vaddr + size);
      route = 1;
    } else {
      route = 2;
    }
  } else {
    route = 3;
    auto q = s.queues.find({s.phase, size});
    if (q != s.queues.end() && !q->second.empty()) {
      int64_t a = q->second.front();
      q->second.pop_front();
      if (pool_contains(s, a, a + size)) {
        pool_remove(s, a, a + size);
        vaddr = a;
        route = 0;
      } else {
        s.occupied++;  // the replay would raise SimulationError; a live run falls back instead
      }
    }
  }
  Live lv{0, route, vaddr, size, -1};
  char *ptr;
  if (route == 0 || route == 1) {
    ptr = s.pool + vaddr;
  } else {
    int g;
    int64_t before = s.reserved;
    vaddr = cache_malloc(s, size, &g);
    if (vaddr < 0) return nullptr;
    (void)before;
    ptr = s.segs[g].dev + (vaddr - s.segs[g].vbase);
    lv = Live{1, route, vaddr, size, g};
  }
  account_alloc(s, size, lv.space == 1, route);
  s.live[ptr] = lv;
  return ptr;
}

void stw_free(void *ptr, size_t nbytes, int device, void *stream) {
  (void)nbytes;
  (void)device;
  (void)stream;
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  auto it = s.live.find(ptr);
  if (it == s.live.end()) return;
  Live lv = it->second;
  s.live.erase(it);
  s.cur -= lv.size;
  if (lv.space == 0) {
    pool_add(s, lv.vaddr, lv.vaddr + lv.size);
  } else {
    s.cache_cur -= lv.size;
    cache_free(s, lv.seg, lv.vaddr, lv.size);
  }
}

int64_t stw_alloc_vaddr(const void *ptr, int32_t *route) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  auto it = s.live.find(ptr);
  if (it == s.live.end()) return -1;
  if (route) *route = it->second.route;
  return it->second.vaddr;
}

int stw_alloc_report(stw_report *rep) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  rep->allocated_peak = s.peak;
  rep->reserved_peak = s.pool_size + s.reserved;
  rep->pool_size = s.pool_size;
  rep->fallback_count = s.fallback;
  rep->fallback_bytes_peak = s.cache_peak;
  rep->reuse_hits = s.reuse;
  rep->mismatch_count = s.mismatch;
  rep->efficiency = rep->reserved_peak ? exact_div((uint64_t)rep->allocated_peak, (uint64_t)rep->reserved_peak) : 1.0;
  rep->fragmentation = 1.0 - rep->efficiency;
  return s.occupied ? STW_ESIM : STW_OK;
}

void stw_alloc_shutdown(void) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (s.pool) cudaFree(s.pool);
  for (auto &g : s.segs) cudaFree(g.dev);
  s.pool = nullptr;
  s.segs.clear();
  s.free.clear();
  s.queues.clear();
  s.spaces.clear();
  s.live.clear();
  s.cur = s.peak = s.cache_cur = s.cache_peak = s.reserved = 0;
  s.fallback = s.reuse = s.mismatch = s.occupied = 0;
  s.phase = 0;
  s.key = -1;
  s.dynamic = 0;
}

}  // extern "C"
