// libstw_alloc -- the runtime side of a plan (include/stw_alloc.h).
//
// 1. A CUDAPluggableAllocator serving a plan with the reference replay's
//    routing (sim.py:143-232): planned offsets for static requests, best fit
//    inside the reuse space for dynamic ones, the CachingAllocator policy
//    (baseline.py:35-95) for everything else. All of it lives in ONE reserved
//    virtual range: [base, base + pool_size) is the pool, the fallback
//    segments follow at base + pool_size + ... exactly where the replay puts
//    them (sim.py:154), each backed by physical memory mapped on first use
//    (cuMemCreate / cuMemMap; segments are never returned, like the
//    reference's). So device pointer = base + replay address for every route.
// 2. The same CachingAllocator and reuse best fit as standalone host objects
//    (stw_cache_*, stw_reuse_best_fit) -- what the Python mirror's
//    CachingAllocator / dynamic_allocate call.
//
// Driver entry points come through cudaGetDriverEntryPoint, so the library
// loads (and the standalone allocator objects work) without a GPU.
#include "../../include/stw_alloc.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <deque>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace {

constexpr int64_t kMinSegment = 2ll * 1024 * 1024;  // baseline.py:17
constexpr int64_t kDefaultFallbackVa = 256ll << 30;

typedef std::pair<int64_t, int64_t> Iv;  // [lo, hi)

int64_t next_pow2(int64_t n) {  // baseline.py:20-21
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// ---------------------------------------------------------------------------
// CachingAllocator policy over virtual addresses (baseline.py:35-95)

struct Seg {
  int64_t base, size;
  std::vector<Iv> free;  // sorted, disjoint
};

struct CacheCore {
  int64_t next_base = 0, min_segment = kMinSegment, reserved = 0, live_bytes = 0;
  std::vector<Seg> segs;

  // best fit over every free block in (segment, address) order; the first
  // minimal block wins (baseline.py:54-59)
  bool find(int64_t size, int *g, int *i) const {
    int bg = -1, bi = -1;
    int64_t blen = 0;
    for (int s = 0; s < (int)segs.size(); s++)
      for (int k = 0; k < (int)segs[s].free.size(); k++) {
        const int64_t len = segs[s].free[k].second - segs[s].free[k].first;
        if (len >= size && (bg < 0 || len < blen)) bg = s, bi = k, blen = len;
      }
    *g = bg;
    *i = bi;
    return bg >= 0;
  }
  int64_t segment_size(int64_t size) const { return std::max(min_segment, next_pow2(size)); }
  int add_segment(int64_t ss) {  // a miss: a fresh segment at the next base (baseline.py:61-69)
    segs.push_back(Seg{next_base, ss, {Iv(next_base, next_base + ss)}});
    next_base += ss;
    reserved += ss;
    return (int)segs.size() - 1;
  }
  int64_t carve(int g, int i, int64_t size) {  // split the block (baseline.py:71-76)
    auto &fr = segs[g].free;
    const Iv b = fr[i];
    fr.erase(fr.begin() + i);
    if (b.first + size < b.second) fr.insert(fr.begin() + i, Iv(b.first + size, b.second));
    live_bytes += size;
    return b.first;
  }
  void give_back(int g, int64_t lo, int64_t size) {  // insort + merge (baseline.py:79-95)
    auto &fr = segs[g].free;
    const int64_t hi = lo + size;
    auto pos = std::lower_bound(fr.begin(), fr.end(), Iv(lo, hi));
    size_t i = pos - fr.begin();
    fr.insert(pos, Iv(lo, hi));
    if (i + 1 < fr.size() && fr[i + 1].first == hi) {
      fr[i].second = fr[i + 1].second;
      fr.erase(fr.begin() + i + 1);
    }
    if (i > 0 && fr[i - 1].second == lo) {
      fr[i - 1].second = fr[i].second;
      fr.erase(fr.begin() + i);
    }
    live_bytes -= size;
  }
};

// ---------------------------------------------------------------------------
// best fit inside free ∩ space (sim.py:120-140 over intervals.py:138-176): the
// smallest intersection piece holding `size`, ties to the lowest address.
// Free and space are coalesced, so the pieces come out disjoint and ascending.

template <class It>
int64_t best_fit_pieces(It f, It fend, const Iv *sp, int64_t nsp, int64_t size) {
  int64_t best_len = INT64_MAX, best_lo = -1;
  for (int64_t s = 0; s < nsp; s++) {
    while (f != fend && f->second <= sp[s].first) ++f;
    for (It g = f; g != fend && g->first < sp[s].second; ++g) {
      const int64_t lo = std::max(g->first, sp[s].first), hi = std::min(g->second, sp[s].second);
      if (hi - lo >= size && hi - lo < best_len) best_len = hi - lo, best_lo = lo;
    }
  }
  return best_lo;
}

// ---------------------------------------------------------------------------
// driver entry points (virtual memory management)

struct Drv {
  bool ok = false;
  decltype(&cuMemAddressReserve) addressReserve;
  decltype(&cuMemAddressFree) addressFree;
  decltype(&cuMemCreate) create;
  decltype(&cuMemRelease) release;
  decltype(&cuMemMap) map;
  decltype(&cuMemUnmap) unmap;
  decltype(&cuMemSetAccess) setAccess;
  decltype(&cuMemGetAllocationGranularity) granularity;
};

template <class F>
bool entry(const char *name, F *f) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
  *f = reinterpret_cast<F>(p);
  return true;
}

Drv &drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuMemAddressReserve", &d.addressReserve) && entry("cuMemAddressFree", &d.addressFree) &&
           entry("cuMemCreate", &d.create) && entry("cuMemRelease", &d.release) && entry("cuMemMap", &d.map) &&
           entry("cuMemUnmap", &d.unmap) && entry("cuMemSetAccess", &d.setAccess) &&
           entry("cuMemGetAllocationGranularity", &d.granularity);
  });
  return d;
}

// ---------------------------------------------------------------------------
// the pluggable allocator's state

struct Live {
  int space;  // 0 pool, 1 cache
  int route;
  int64_t vaddr, size;
  int seg;
};

struct Mapping {
  int64_t off, size;
  CUmemGenericAllocationHandle h;
};

struct State {
  std::mutex mu;
  bool inited = false;
  int device = 0;
  int64_t pool_size = 0, alignment = 512;
  CUdeviceptr base = 0;
  int64_t va_size = 0, gran = 0, mapped_hi = 0;  // [0, mapped_hi) of the range is backed
  std::vector<Mapping> maps;
  std::map<int64_t, int64_t> free;  // coalesced free intervals of the pool (lo -> hi)
  std::map<std::pair<int32_t, int64_t>, std::deque<int64_t>> queues;
  std::vector<std::vector<Iv>> spaces;
  CacheCore cache;
  std::unordered_map<const void *, Live> live;
  int32_t phase = 0, key = -1, dynamic = 0;
  // metrics (sim.py:67-117)
  int64_t cur = 0, peak = 0, cache_cur = 0, cache_peak = 0;
  int64_t fallback = 0, reuse = 0, mismatch = 0, occupied = 0, bad_frees = 0;
  // request matcher for dynamic requests: per layer instance, the reuse keys of
  // its dynamic allocations in recorded order (-1 = no entry); layer = current instance
  std::vector<std::deque<int32_t>> dyn_keys;
  int32_t layer = -1;
  bool dyn_by_layer = false;
  // modes: 0 passthrough (cudaMalloc / cudaFree), 1 profiling (passthrough +
  // recording), 2 serving the plan (stw_alloc_init switches to it)
  int mode = 0;
  std::unordered_map<const void *, int64_t> passthrough;  // ptr -> size
  // the Allocation Profiler's records: one per op, raw-trace order
  struct Rec {
    int8_t op;  // 0 alloc, 1 free
    int8_t dyn;
    int32_t phase, module;
    int64_t id, size;
  };
  std::vector<Rec> recs;
  std::unordered_map<const void *, int64_t> rec_id;  // live recorded block -> its id
  int64_t next_id = 0;
  int32_t p_phase = 0, p_module = 0, p_dyn = 0;
  std::vector<std::pair<int8_t, int64_t>> served;  // (route, replay address) of every served request
};

State &S() {
  static State s;
  return s;
}

// back [mapped_hi, roundup(end)) of the reserved range with fresh physical memory
bool map_upto(State &s, int64_t end) {
  if (end <= s.mapped_hi) return true;
  if (end > s.va_size) return false;
  Drv &d = drv();
  const int64_t hi = (end + s.gran - 1) / s.gran * s.gran, sz = hi - s.mapped_hi;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = s.device;
  CUmemGenericAllocationHandle h;
  if (d.create(&h, (size_t)sz, &prop, 0) != CUDA_SUCCESS) return false;
  if (d.map(s.base + s.mapped_hi, (size_t)sz, 0, h, 0) != CUDA_SUCCESS) {
    d.release(h);
    return false;
  }
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = s.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (d.setAccess(s.base + s.mapped_hi, (size_t)sz, &acc, 1) != CUDA_SUCCESS) {
    d.unmap(s.base + s.mapped_hi, (size_t)sz);
    d.release(h);
    return false;
  }
  s.maps.push_back(Mapping{s.mapped_hi, sz, h});
  s.mapped_hi = hi;
  return true;
}

void unmap_all(State &s) {
  Drv &d = drv();
  for (auto &m : s.maps) {
    d.unmap(s.base + m.off, (size_t)m.size);
    d.release(m.h);
  }
  s.maps.clear();
  if (s.base) d.addressFree(s.base, (size_t)s.va_size);
  s.base = 0;
  s.va_size = s.mapped_hi = 0;
}

void reset(State &s) {
  s.inited = false;
  s.served.clear();
  s.dyn_keys.clear();
  s.dyn_by_layer = false;
  s.layer = -1;
  s.free.clear();
  s.queues.clear();
  s.spaces.clear();
  s.cache = CacheCore();
  s.live.clear();
  s.cur = s.peak = s.cache_cur = s.cache_peak = 0;
  s.fallback = s.reuse = s.mismatch = s.occupied = s.bad_frees = 0;
  s.phase = 0;
  s.key = -1;
  s.dynamic = 0;
}

bool pool_contains(State &s, int64_t lo, int64_t hi) {  // IntervalSet.contains_interval (intervals.py:95-98)
  auto it = s.free.upper_bound(lo);
  if (it == s.free.begin()) return false;
  --it;
  return it->first <= lo && hi <= it->second;
}

void pool_remove(State &s, int64_t lo, int64_t hi) {  // [lo, hi) lies inside one free interval
  auto it = s.free.upper_bound(lo);
  --it;
  const int64_t a = it->first, b = it->second;
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

int64_t reuse_fit(State &s, int key, int64_t size) {
  if (key < 0 || key >= (int)s.spaces.size() || s.spaces[key].empty()) return -1;
  const auto &sp = s.spaces[key];
  auto f = s.free.upper_bound(sp[0].first);
  if (f != s.free.begin()) --f;
  return best_fit_pieces(f, s.free.end(), sp.data(), (int64_t)sp.size(), size);
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

// standalone CachingAllocator object of the handle API
struct CacheObj {
  CacheCore core;
  struct Blk {
    int seg;
    int64_t lo, size;
  };
  std::unordered_map<int64_t, Blk> live;
};

}  // namespace

extern "C" {

int stw_alloc_init_ex(int device, int64_t pool_size, int64_t alignment, int64_t fallback_va) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (s.inited || pool_size < 0) return STW_EARG;
  Drv &d = drv();
  if (!d.ok || cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return STW_ECUDA;
  reset(s);
  s.device = device;
  s.pool_size = pool_size;
  s.alignment = alignment > 0 ? alignment : 512;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  size_t g = 0;
  if (d.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0) return STW_ECUDA;
  s.gran = (int64_t)g;
  const int64_t fb = fallback_va > 0 ? fallback_va : kDefaultFallbackVa;
  s.va_size = ((pool_size + fb) + s.gran - 1) / s.gran * s.gran;
  if (d.addressReserve(&s.base, (size_t)s.va_size, 0, 0, 0) != CUDA_SUCCESS) {
    s.base = 0;
    return STW_ECUDA;
  }
  s.mapped_hi = 0;
  if (pool_size > 0 && !map_upto(s, pool_size)) {  // the pool is backed up front
    unmap_all(s);
    return STW_ECUDA;
  }
  if (pool_size > 0) s.free[0] = pool_size;
  s.cache.next_base = pool_size;  // the replay's cache starts at pool_size (sim.py:154)
  s.inited = true;
  s.mode = 2;
  return STW_OK;
}

int stw_alloc_init(int device, int64_t pool_size, int64_t alignment) {
  return stw_alloc_init_ex(device, pool_size, alignment, 0);
}

int stw_alloc_load_plan(int64_t n_dec, const int32_t *phase, const int64_t *size, const int64_t *addr,
                        const int32_t *t_s, const int64_t *id, int64_t n_keys, const int64_t *sp_off,
                        const int64_t *sp_lo, const int64_t *sp_hi) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (!s.inited) return STW_EARG;
  std::vector<int64_t> order(n_dec);
  for (int64_t k = 0; k < n_dec; k++) {
    order[k] = k;
    if (addr[k] < 0 || addr[k] + size[k] > s.pool_size) return STW_EPLAN;
  }
  for (int64_t k = 0; k < n_keys; k++)
    for (int64_t j = sp_off[k]; j < sp_off[k + 1]; j++)
      if (sp_lo[j] < 0 || sp_hi[j] > s.pool_size) return STW_EPLAN;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return t_s[a] != t_s[b] ? t_s[a] < t_s[b] : id[a] < id[b];
  });
  s.queues.clear();
  for (int64_t k : order) s.queues[{phase[k], size[k]}].push_back(addr[k]);
  s.spaces.assign(n_keys, {});
  for (int64_t k = 0; k < n_keys; k++)
    for (int64_t j = sp_off[k]; j < sp_off[k + 1]; j++) s.spaces[k].push_back(Iv(sp_lo[j], sp_hi[j]));
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
  if (s.mode != 2) {  // passthrough, recorded when profiling
    void *p = nullptr;
    if (cudaMalloc(&p, nbytes) != cudaSuccess) return nullptr;
    s.passthrough[p] = (int64_t)nbytes;
    if (s.mode == 1) {
      const int64_t id = s.next_id++;
      s.rec_id[p] = id;
      s.recs.push_back(State::Rec{0, (int8_t)s.p_dyn, s.p_phase, s.p_module, id, (int64_t)nbytes});
    }
    return p;
  }
  if (!s.inited) return nullptr;
  const int64_t size = (int64_t)((nbytes + s.alignment - 1) / s.alignment * s.alignment);
  // decide the route first; nothing is committed until the memory is there
  int route;
  int64_t vaddr = -1;
  std::deque<int64_t> *q = nullptr;
  if (s.dynamic) {
    int32_t key = s.key;
    if (s.dyn_by_layer) {  // the layer instance's next recorded key (popped once served)
      key = -1;
      if (s.layer >= 0 && s.layer < (int32_t)s.dyn_keys.size() && !s.dyn_keys[s.layer].empty())
        key = s.dyn_keys[s.layer].front();
    }
    vaddr = reuse_fit(s, key, size);
    route = vaddr >= 0 ? 1 : 2;
  } else {
    route = 3;
    auto it = s.queues.find({s.phase, size});
    if (it != s.queues.end() && !it->second.empty()) {
      q = &it->second;
      if (pool_contains(s, q->front(), q->front() + size)) {
        vaddr = q->front();
        route = 0;
      }
    }
  }
  Live lv{0, route, vaddr, size, -1};
  if (route == 2 || route == 3) {
    int g, i;
    if (!s.cache.find(size, &g, &i)) {
      const int64_t ss = s.cache.segment_size(size);
      if (!map_upto(s, s.cache.next_base + ss)) return nullptr;  // out of memory: state untouched
      g = s.cache.add_segment(ss);
      i = 0;
    }
    lv = Live{1, route, s.cache.carve(g, i, size), size, g};
    // the replay raises SimulationError on an occupied planned address; a live
    // run serves the request from the cache and reports it (stw_alloc_report)
    if (q && route == 3) s.occupied++;
  } else if (route == 0 || route == 1) {
    pool_remove(s, vaddr, vaddr + size);
  }
  if (q) q->pop_front();
  if (s.dynamic && s.dyn_by_layer && s.layer >= 0 && s.layer < (int32_t)s.dyn_keys.size() &&
      !s.dyn_keys[s.layer].empty())
    s.dyn_keys[s.layer].pop_front();
  account_alloc(s, size, lv.space == 1, route);
  s.served.push_back({(int8_t)route, lv.vaddr});
  void *ptr = reinterpret_cast<void *>(s.base + lv.vaddr);
  s.live[ptr] = lv;
  return ptr;
}

void stw_free(void *ptr, size_t nbytes, int device, void *stream) {
  (void)nbytes;
  (void)device;
  (void)stream;
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  auto pt = s.passthrough.find(ptr);
  if (pt != s.passthrough.end()) {
    if (s.mode == 1) {
      auto r = s.rec_id.find(ptr);
      if (r != s.rec_id.end()) {  // frees of blocks allocated before profiling began are not part of the trace
        s.recs.push_back(State::Rec{1, 0, s.p_phase, s.p_module, r->second, pt->second});
        s.rec_id.erase(r);
      }
    }
    cudaFree(ptr);
    s.passthrough.erase(pt);
    return;
  }
  auto it = s.live.find(ptr);
  if (it == s.live.end()) {  // unknown or double free (sim.py:231-232): counted, reported by stw_alloc_report
    s.bad_frees++;
    return;
  }
  const Live lv = it->second;
  s.live.erase(it);
  s.cur -= lv.size;
  if (lv.space == 0) {
    pool_add(s, lv.vaddr, lv.vaddr + lv.size);
  } else {
    s.cache_cur -= lv.size;
    s.cache.give_back(lv.seg, lv.vaddr, lv.size);
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
  rep->reserved_peak = s.pool_size + s.cache.reserved;
  rep->pool_size = s.pool_size;
  rep->fallback_count = s.fallback;
  rep->fallback_bytes_peak = s.cache_peak;
  rep->reuse_hits = s.reuse;
  rep->mismatch_count = s.mismatch;
  rep->efficiency = rep->reserved_peak ? exact_div((uint64_t)rep->allocated_peak, (uint64_t)rep->reserved_peak) : 1.0;
  rep->fragmentation = 1.0 - rep->efficiency;
  return s.occupied || s.bad_frees ? STW_ESIM : STW_OK;
}

int stw_alloc_status(int64_t *out) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  out[0] = s.inited;
  out[1] = s.pool_size;
  out[2] = (int64_t)s.live.size();
  out[3] = s.occupied;
  out[4] = s.bad_frees;
  out[5] = s.mapped_hi;
  out[6] = (int64_t)s.base;
  return STW_OK;
}

int stw_alloc_shutdown(void) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (!s.live.empty()) return STW_EARG;  // live tensors still point into the range
  if (s.inited) unmap_all(s);
  reset(s);
  s.mode = 0;
  return STW_OK;
}

// ---- Allocation Profiler + request matcher ----------------------------------

int stw_alloc_set_mode(int32_t mode) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  if (mode < 0 || mode > 2 || (mode == 2 && !s.inited)) return STW_EARG;
  if (mode == 1 && s.mode != 1) {  // a fresh recording
    s.recs.clear();
    s.rec_id.clear();
    s.next_id = 0;
  }
  s.mode = mode;
  return STW_OK;
}

void stw_prof_set(int32_t phase, int32_t module, int32_t dynamic) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  s.p_phase = phase;
  s.p_module = module;
  s.p_dyn = dynamic;
}

int64_t stw_prof_records(int8_t *op, int8_t *dyn, int32_t *phase, int32_t *module, int64_t *id, int64_t *size,
                         int64_t cap) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  const int64_t n = (int64_t)s.recs.size();
  for (int64_t k = 0; k < n && k < cap; k++) {
    const State::Rec &r = s.recs[k];
    op[k] = r.op, dyn[k] = r.dyn, phase[k] = r.phase, module[k] = r.module, id[k] = r.id, size[k] = r.size;
  }
  return n;
}

int stw_alloc_load_dyn_keys(int32_t n_layers, const int64_t *off, const int32_t *keys) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  s.dyn_keys.assign(n_layers, {});
  for (int32_t l = 0; l < n_layers; l++)
    for (int64_t j = off[l]; j < off[l + 1]; j++) s.dyn_keys[l].push_back(keys[j]);
  s.dyn_by_layer = true;
  return STW_OK;
}

int64_t stw_alloc_served(int8_t *route, int64_t *vaddr, int64_t cap) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  const int64_t n = (int64_t)s.served.size();
  for (int64_t k = 0; k < n && k < cap; k++) route[k] = s.served[k].first, vaddr[k] = s.served[k].second;
  return n;
}

void stw_set_layer_instance(int32_t layer, int32_t dynamic) {
  State &s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  s.layer = layer;
  s.dynamic = dynamic;
}

// ---- standalone allocator objects ---------------------------------------

void *stw_cache_new(int64_t base, int64_t min_segment) {
  CacheObj *c = new CacheObj();
  c->core.next_base = base;
  c->core.min_segment = min_segment;
  return c;
}

void stw_cache_delete(void *h) { delete static_cast<CacheObj *>(h); }

int stw_cache_malloc(void *h, int64_t rid, int64_t size, int64_t *addr, int64_t *grown) {
  CacheObj *c = static_cast<CacheObj *>(h);
  if (c->live.count(rid)) return STW_ESIM;  // "request {rid} already live in cache"
  int g, i;
  *grown = 0;
  if (!c->core.find(size, &g, &i)) {
    const int64_t ss = c->core.segment_size(size);
    g = c->core.add_segment(ss);
    i = 0;
    *grown = ss;
  }
  *addr = c->core.carve(g, i, size);
  c->live[rid] = CacheObj::Blk{g, *addr, size};
  return STW_OK;
}

int stw_cache_free(void *h, int64_t rid, int64_t *addr, int64_t *size) {
  CacheObj *c = static_cast<CacheObj *>(h);
  auto it = c->live.find(rid);
  if (it == c->live.end()) return STW_ESIM;  // "free of unknown id {rid} in cache"
  const CacheObj::Blk b = it->second;
  c->live.erase(it);
  c->core.give_back(b.seg, b.lo, b.size);
  *addr = b.lo;
  *size = b.size;
  return STW_OK;
}

int stw_cache_owns(void *h, int64_t rid) { return static_cast<CacheObj *>(h)->live.count(rid) ? 1 : 0; }

void stw_cache_stats(void *h, int64_t *out) {
  CacheObj *c = static_cast<CacheObj *>(h);
  int64_t blocks = 0;
  for (auto &g : c->core.segs) blocks += (int64_t)g.free.size();
  out[0] = c->core.reserved;
  out[1] = c->core.live_bytes;
  out[2] = (int64_t)c->core.segs.size();
  out[3] = blocks;
  out[4] = c->core.next_base;
}

void stw_cache_segments(void *h, int64_t *seg_base, int64_t *seg_size, int64_t *blk_off, int64_t *blk_lo,
                        int64_t *blk_hi) {
  CacheObj *c = static_cast<CacheObj *>(h);
  int64_t k = 0;
  for (size_t g = 0; g < c->core.segs.size(); g++) {
    const Seg &s = c->core.segs[g];
    seg_base[g] = s.base;
    seg_size[g] = s.size;
    blk_off[g] = k;
    for (auto &b : s.free) blk_lo[k] = b.first, blk_hi[k] = b.second, k++;
  }
  blk_off[c->core.segs.size()] = k;
}

int64_t stw_reuse_best_fit(int64_t n_free, const int64_t *free_lo, const int64_t *free_hi, int64_t n_space,
                           const int64_t *sp_lo, const int64_t *sp_hi, int64_t size) {
  std::vector<Iv> fr(n_free), sp(n_space);
  for (int64_t k = 0; k < n_free; k++) fr[k] = Iv(free_lo[k], free_hi[k]);
  for (int64_t k = 0; k < n_space; k++) sp[k] = Iv(sp_lo[k], sp_hi[k]);
  if (sp.empty()) return -1;
  auto f = std::upper_bound(fr.begin(), fr.end(), Iv(sp[0].first, INT64_MAX));
  if (f != fr.begin()) --f;
  return best_fit_pieces(f, fr.end(), sp.data(), n_space, size);
}

}  // extern "C"
