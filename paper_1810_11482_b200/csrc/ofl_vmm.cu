// Large device buffers through the CUDA virtual-memory API.
//
// The stream-ordered pool (ofl_runtime.cu) makes frees cheap, but growing it
// is slow: ~70 ms per GiB on B200 against 2.3 ms for cudaMalloc (profiles/
// r02_alloc_probe.txt), so the first 2 x 8 GiB of config 4 cost a second.
// cudaMalloc, in turn, pays a device-wide synchronisation on every
// cudaFree (profiles/r02_vmm_probe.txt: a 1 MiB cudaFree waits 54 ms for
// a kernel on another stream).  Buffers of kVmmMin bytes and up therefore
// get their own physical allocation (cuMemCreate + cuMemAddressReserve +
// cuMemMap + cuMemSetAccess: ~2 ms per GiB), and their free is deferred:
// ofl_free records a fence event on every live stream and hands the mapping
// to a reaper thread, which waits for those events and then caches it for
// reuse by an allocation of the same size (unmapped — cuMemUnmap does not
// synchronise with other streams, same probe — only when an allocation runs
// out of memory), so no stream ever stalls on a dropped buffer and
// steady-state allocations make no driver call.
//
// Driver entry points come from cudaGetDriverEntryPoint (libofl.so does not
// link libcuda; the runtime resolves the driver it already loaded).
#include <cuda.h>

#include <condition_variable>
#include <deque>
#include <iterator>
#include <map>
#include <set>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ofl_internal.h"

namespace {

using CreateFn = CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                              unsigned long long);
using ReleaseFn = CUresult (*)(CUmemGenericAllocationHandle);
using ReserveFn = CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
using AddrFreeFn = CUresult (*)(CUdeviceptr, size_t);
using MapFn = CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                           unsigned long long);
using UnmapFn = CUresult (*)(CUdeviceptr, size_t);
using AccessFn = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
using GranFn = CUresult (*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);

struct Driver {
  CreateFn create = nullptr;
  ReleaseFn release = nullptr;
  ReserveFn reserve = nullptr;
  AddrFreeFn addr_free = nullptr;
  MapFn map = nullptr;
  UnmapFn unmap = nullptr;
  AccessFn access = nullptr;
  GranFn gran = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    (void)cudaGetLastError();
    return false;
  }
  *out = reinterpret_cast<F>(fn);
  return true;
}

const Driver& driver() {
  static Driver d = [] {
    Driver x;
    x.ok = entry("cuMemCreate", &x.create) && entry("cuMemRelease", &x.release) &&
           entry("cuMemAddressReserve", &x.reserve) && entry("cuMemAddressFree", &x.addr_free) &&
           entry("cuMemMap", &x.map) && entry("cuMemUnmap", &x.unmap) &&
           entry("cuMemSetAccess", &x.access) &&
           entry("cuMemGetAllocationGranularity", &x.gran);
    return x;
  }();
  return d;
}

struct Mapping {
  int dev;
  CUdeviceptr va;
  size_t size;
};

std::mutex g_mu;                              // mappings, cache, peer grants
std::unordered_map<uintptr_t, Mapping> g_live;
// released mappings whose fences have passed, by size: reused as they are
// (a fresh physical allocation can wait behind queued work, a cached one
// never does); unmapped only when an allocation runs out of memory
std::multimap<size_t, Mapping> g_cache[ofl::kMaxDev];
std::set<int> g_peers[ofl::kMaxDev];          // devices granted access to dev's buffers

// deferred frees: a mapping and the fence events it must outlive
struct Pending {
  Mapping m;
  std::vector<cudaEvent_t> fences;
};
// The reaper thread is detached and may be waiting when the process exits:
// its queue and condition variables live on the heap and are never
// destroyed (destroying a condition variable that has a waiter blocks).
struct Queue {
  std::mutex mu;
  std::condition_variable cv, idle_cv;
  std::deque<Pending> q;
  int busy = 0;
};
Queue& queue() {
  static Queue* q = new Queue();
  return *q;
}

void unmap(const Mapping& m) {
  const Driver& d = driver();
  d.unmap(m.va, m.size);
  d.addr_free(m.va, m.size);
}

void reaper() {
  Queue& Q = queue();
  for (;;) {
    Pending p;
    {
      std::unique_lock<std::mutex> lk(Q.mu);
      Q.cv.wait(lk, [&] { return !Q.q.empty(); });
      p = std::move(Q.q.front());
      Q.q.pop_front();
      ++Q.busy;
    }
    for (cudaEvent_t e : p.fences) {
      cudaEventSynchronize(e);  // blocks this thread only
      cudaEventDestroy(e);
    }
    (void)cudaGetLastError();
    {
      std::lock_guard<std::mutex> g(g_mu);
      g_cache[p.m.dev].emplace(p.m.size, p.m);
    }
    {
      std::lock_guard<std::mutex> lk(Q.mu);
      --Q.busy;
      if (Q.q.empty() && Q.busy == 0) Q.idle_cv.notify_all();
    }
  }
}

void start_reaper() {
  static std::once_flag once;
  std::call_once(once, [] { std::thread(reaper).detach(); });
}

CUmemAllocationProp prop_for(int dev) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  return p;
}

}  // namespace

namespace ofl {

bool vmm_available() { return driver().ok; }

// a mapped allocation of at least `bytes` on `dev`,
// readable and writable by dev and every device granted peer access to it
int vmm_alloc(int dev, size_t bytes, void** out) {
  const Driver& d = driver();
  if (!d.ok) return set_error(OFL_ERR_INTERNAL, "virtual-memory API unavailable");
  CUmemAllocationProp prop = prop_for(dev);
  size_t gran = 0;
  if (d.gran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !gran)
    gran = 2u << 20;
  const size_t size = (bytes + gran - 1) / gran * gran;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_cache[dev].find(size);
    if (it != g_cache[dev].end()) {  // a released mapping of this size
      const Mapping m = it->second;
      g_cache[dev].erase(it);
      g_live[(uintptr_t)m.va] = m;
      *out = reinterpret_cast<void*>(m.va);
      return OFL_OK;
    }
  }
  CUmemGenericAllocationHandle h;
  CUresult r = d.create(&h, size, &prop, 0);
  if (r == CUDA_ERROR_OUT_OF_MEMORY)  // the caller reclaims freed memory and retries
    return set_error(OFL_ERR_OOM, "cuda" + std::to_string(dev) + ": " + std::to_string(bytes) +
                                      " bytes requested, allocation failed");
  if (r != CUDA_SUCCESS) return set_error(OFL_ERR_CUDA, "cuMemCreate failed: " + std::to_string(r));
  CUdeviceptr va = 0;
  r = d.reserve(&va, size, gran, 0, 0);
  if (r == CUDA_SUCCESS) r = d.map(va, size, 0, h, 0);
  d.release(h);  // the mapping keeps the physical memory until it is unmapped
  if (r != CUDA_SUCCESS) {
    if (va) d.addr_free(va, size);
    return set_error(OFL_ERR_CUDA, "cuMemAddressReserve/cuMemMap failed: " + std::to_string(r));
  }
  std::lock_guard<std::mutex> g(g_mu);
  std::vector<CUmemAccessDesc> acc;
  CUmemAccessDesc a{};
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  a.location.id = dev;
  acc.push_back(a);
  for (int p : g_peers[dev]) {
    a.location.id = p;
    acc.push_back(a);
  }
  r = d.access(va, size, acc.data(), acc.size());
  if (r != CUDA_SUCCESS) {
    d.unmap(va, size);
    d.addr_free(va, size);
    return set_error(OFL_ERR_CUDA, "cuMemSetAccess failed: " + std::to_string(r));
  }
  g_live[(uintptr_t)va] = Mapping{dev, va, size};
  *out = reinterpret_cast<void*>(va);
  return OFL_OK;
}

// true (and the mapping is queued for release after `fences`) when p is a
// live VMM allocation; the events are destroyed by the reaper
bool vmm_free_after(void* p, std::vector<cudaEvent_t>& fences) {
  Mapping m;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_live.find((uintptr_t)p);
    if (it == g_live.end()) return false;
    m = it->second;
    g_live.erase(it);
  }
  start_reaper();
  Queue& Q = queue();
  {
    std::lock_guard<std::mutex> lk(Q.mu);
    Q.q.push_back(Pending{m, std::move(fences)});
  }
  Q.cv.notify_one();
  return true;
}

bool vmm_owns(void* p) {
  std::lock_guard<std::mutex> g(g_mu);
  return g_live.count((uintptr_t)p) != 0;
}

// every deferred free released (used before retrying a failed allocation)
void vmm_drain() {
  Queue& Q = queue();
  std::unique_lock<std::mutex> lk(Q.mu);
  Q.idle_cv.wait(lk, [&] { return Q.q.empty() && Q.busy == 0; });
}

// unmap cached mappings of `dev`, largest first, until `need` bytes are
// released (0: all of them) -- before retrying a failed allocation; the
// small ones stay cached for the allocations that reuse them
void vmm_trim(int dev, size_t need) {
  std::vector<Mapping> drop;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto& c = g_cache[dev];
    size_t got = 0;
    while (!c.empty() && (need == 0 || got < need)) {
      auto it = std::prev(c.end());
      got += it->second.size;
      drop.push_back(it->second);
      c.erase(it);
    }
  }
  for (auto& m : drop) unmap(m);
}

// `from` may now read and write `to`'s VMM buffers, current and future
void vmm_grant_peer(int from, int to) {
  const Driver& d = driver();
  if (!d.ok || from < 0 || to < 0 || from >= kMaxDev || to >= kMaxDev) return;
  std::lock_guard<std::mutex> g(g_mu);
  if (!g_peers[to].insert(from).second) return;
  CUmemAccessDesc a{};
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.location.id = from;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (auto& kv : g_live)
    if (kv.second.dev == to) d.access(kv.second.va, kv.second.size, &a, 1);
  for (auto& kv : g_cache[to]) d.access(kv.second.va, kv.second.size, &a, 1);
}

}  // namespace ofl
