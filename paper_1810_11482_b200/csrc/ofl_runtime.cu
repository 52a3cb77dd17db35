// libofl.so runtime core: discovery, streams with ticket logs, lazily placed
// completion markers, host-function completions into an eventfd-signalled
// queue, device/pinned memory and stream-ordered copies.
//
// Replaces, below the dispatch seam of the reference (runtime.py:30-120):
//   DeviceObject + _StreamWorker   device.py:129-157,188-328
//   BufferObject storage/copies    buffer.py:26-55
//   Promise fulfilment on workers  futures.py:76-89,133-174
#include <sys/eventfd.h>
#include <unistd.h>

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include <set>
#include <unordered_set>

#include "ofl_internal.h"

namespace ofl {

// ---------------------------------------------------------------- errors ---
static thread_local std::string t_last_error;

int set_error(int code, const std::string& msg) {
  t_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* what) {
  int code = (e == cudaErrorMemoryAllocation) ? OFL_ERR_OOM : OFL_ERR_CUDA;
  return set_error(code, std::string(what) + ": " + cudaGetErrorName(e) + ": " +
                             cudaGetErrorString(e));
}

cudaError_t use_device(int dev) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return e;
  if (cur == dev) return cudaSuccess;
  return cudaSetDevice(dev);
}

static int g_sms[kMaxDev];

int num_sms(int dev) {
  if (dev < 0 || dev >= kMaxDev) return 148;
  if (g_sms[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    g_sms[dev] = v;
  }
  return g_sms[dev];
}

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ------------------------------------------------------------ event pool ---
// Markers are DisableTiming events, recycled per device.
struct EventPool {
  std::mutex mu;
  std::vector<cudaEvent_t> free_list;
};
static EventPool g_pools[kMaxDev];

static cudaError_t pool_get(int dev, cudaEvent_t* ev) {
  {
    std::lock_guard<std::mutex> g(g_pools[dev].mu);
    if (!g_pools[dev].free_list.empty()) {
      *ev = g_pools[dev].free_list.back();
      g_pools[dev].free_list.pop_back();
      return cudaSuccess;
    }
  }
  return cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
}

static void pool_put(int dev, cudaEvent_t ev) {
  std::lock_guard<std::mutex> g(g_pools[dev].mu);
  g_pools[dev].free_list.push_back(ev);
}

EvBox::~EvBox() { pool_put(dev, ev); }

static inline void raise_done(ofl_stream* s, uint64_t t) {
  uint64_t cur = s->done.load(std::memory_order_acquire);
  while (cur < t && !s->done.compare_exchange_weak(cur, t, std::memory_order_acq_rel)) {
  }
}

// Pop markers that have completed (caller holds s->mu).  Returns an error
// status if the stream hit a sticky device fault.
static int reap(ofl_stream* s) {
  while (!s->markers.empty()) {
    auto& m = s->markers.front();
    cudaError_t e = cudaEventQuery(m->ev);
    if (e == cudaErrorNotReady) {
      (void)cudaGetLastError();
      break;
    }
    if (e != cudaSuccess) return cuda_error(e, "device fault");
    raise_done(s, m->ticket);
    s->markers.pop_front();
  }
  return OFL_OK;
}

// Marker covering `ticket` (the first placed at or after it); places one at
// the tail if none exists.  Caller holds s->mu.
static int covering(ofl_stream* s, uint64_t ticket, std::shared_ptr<EvBox>* out) {
  for (auto& m : s->markers)
    if (m->ticket >= ticket) {
      *out = m;
      return OFL_OK;
    }
  cudaError_t e = use_device(s->dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  cudaEvent_t ev;
  e = pool_get(s->dev, &ev);
  if (e != cudaSuccess) return cuda_error(e, "cudaEventCreate");
  e = cudaEventRecord(ev, s->cs);
  if (e != cudaSuccess) {
    pool_put(s->dev, ev);
    return cuda_error(e, "cudaEventRecord");
  }
  auto box = std::shared_ptr<EvBox>(new EvBox{s->dev, ev, s->tail});
  s->markers.push_back(box);
  *out = box;
  return OFL_OK;
}

// --------------------------------------------------------- completions ---
struct CompletionQueue {
  std::mutex mu;
  std::deque<uint64_t> ids;
  int efd = -1;
};
static CompletionQueue g_cq;
static std::once_flag g_cq_once;

static void cq_init() {
  std::call_once(g_cq_once, [] { g_cq.efd = eventfd(0, EFD_CLOEXEC); });
}

static void cq_post(uint64_t id) {
  cq_init();
  {
    std::lock_guard<std::mutex> g(g_cq.mu);
    g_cq.ids.push_back(id);
  }
  uint64_t one = 1;
  ssize_t r;
  do {
    r = write(g_cq.efd, &one, sizeof(one));
  } while (r < 0 && errno == EINTR);
}

struct NotifyPayload {
  ofl_stream* s;
  uint64_t ticket;
  uint64_t id;
};

// Runs on the CUDA driver's callback thread after every prior operation on
// the stream finished.  Must not call CUDA.
static void CUDART_CB host_complete(void* p) {
  auto* pl = static_cast<NotifyPayload*>(p);
  raise_done(pl->s, pl->ticket);
  cq_post(pl->id);
  delete pl;
}

// ------------------------------------------------------------- memory ---
// Buffers of kVmmMin bytes and up are VMM mappings (ofl_vmm.cu); smaller
// ones come from each device's stream-ordered memory pool (cudaMallocAsync
// on a per-device internal stream; the pool keeps freed memory for reuse
// instead of returning it to the driver).  A free is ordered on the device
// after the work enqueued so far on every stream of the process — the
// internal stream waits on a fence event recorded on each, then
// cudaFreeAsync — instead of cudaFree's implicit device-wide
// synchronisation, which stalled every stream (including other devices'
// fused exchanges) whenever a buffer was dropped.  Buffers shared with other
// processes through CUDA IPC are plain cudaMalloc allocations (IPC handles
// do not cover stream-ordered allocations): ofl_malloc_shareable.
static std::mutex g_zero_mu[kMaxDev];
static cudaStream_t g_zero_stream[kMaxDev];  // allocation + zero fill
static std::mutex g_free_mu[kMaxDev];
static cudaStream_t g_free_stream[kMaxDev];  // frees, each after fence waits
static bool g_pool_ready[kMaxDev];
static std::mutex g_streams_mu;                 // live streams (free fences)
static std::set<ofl_stream*> g_streams;
static std::mutex g_legacy_mu;                  // cudaMalloc'd (shareable) buffers
static std::unordered_set<void*> g_legacy;

// the internal stream of `dev` (created on first use; caller holds
// g_zero_mu[dev]), at the device's highest priority: a zero fill is a short
// kernel that must not queue behind the pending CTAs of a long kernel chain
// on another stream (it gets the SMs at the chain's next kernel boundary)
static cudaError_t internal_stream(int dev) {
  if (g_zero_stream[dev]) return cudaSuccess;
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e != cudaSuccess) return e;
  return cudaStreamCreateWithPriority(&g_zero_stream[dev], cudaStreamNonBlocking, greatest);
}

static cudaError_t pool_setup(int dev) {
  if (g_pool_ready[dev]) return cudaSuccess;
  cudaMemPool_t pool;
  cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return e;
  uint64_t keep = UINT64_MAX;  // never trim at synchronisation points
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e != cudaSuccess) return e;
  // an allocation may reuse memory whose free has already completed, but
  // the pool must not make the allocation stream wait on a pending free
  // (that would turn every allocation after a free into a wait for the
  // work the free is ordered after)
  int no = 0;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  if (e != cudaSuccess) return e;
  g_pool_ready[dev] = true;
  return cudaSuccess;
}

// Direct peer access for copies and kernel peer stores (once per pair).
static std::mutex g_peer_mu;
static bool g_peer_done[kMaxDev][kMaxDev];

void enable_peer(int from, int to) {
  if (from == to || from < 0 || to < 0 || from >= kMaxDev || to >= kMaxDev) return;
  std::lock_guard<std::mutex> g(g_peer_mu);
  if (g_peer_done[from][to]) return;
  g_peer_done[from][to] = true;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, from, to) == cudaSuccess && can) {
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(from);
    cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
    // stream-ordered and VMM allocations need an explicit grant per
    // accessing device
    vmm_grant_peer(from, to);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, to) == cudaSuccess) {
      cudaMemAccessDesc d{};
      d.location.type = cudaMemLocationTypeDevice;
      d.location.id = from;
      d.flags = cudaMemAccessFlagsProtReadWrite;
      (void)cudaMemPoolSetAccess(pool, &d, 1);
    }
    if (cur >= 0) cudaSetDevice(cur);
  }
  (void)cudaGetLastError();
}

}  // namespace ofl

using namespace ofl;

extern "C" {

int ofl_abi_version(void) { return OFL_ABI_VERSION; }
const char* ofl_last_error(void) { return t_last_error.c_str(); }
uint64_t ofl_kernel_launches(void) { return g_launches.load(); }

// -------------------------------------------------------------- devices ---
int ofl_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    *count = 0;
    return cuda_error(e, "cudaGetDeviceCount");
  }
  *count = n;
  return OFL_OK;
}

int ofl_device_props(int dev, char* name, int name_cap, int* cc_major, int* cc_minor,
                     uint64_t* mem_bytes, int* sms, uint64_t* l2_bytes) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaGetDeviceProperties");
  if (name && name_cap > 0) {
    std::snprintf(name, (size_t)name_cap, "%s", p.name);
  }
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  if (mem_bytes) *mem_bytes = p.totalGlobalMem;
  if (sms) *sms = p.multiProcessorCount;
  if (l2_bytes) *l2_bytes = (uint64_t)p.l2CacheSize;
  return OFL_OK;
}

int ofl_device_pci_bus_id(int dev, char* out, int cap) {
  if (!out || cap < 13) return set_error(OFL_ERR_BAD_ARGS, "pci bus id: buffer of >= 13 bytes");
  cudaError_t e = cudaDeviceGetPCIBusId(out, cap, dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaDeviceGetPCIBusId");
  for (char* c = out; *c; ++c) *c = (char)std::tolower((unsigned char)*c);
  return OFL_OK;
}

// -------------------------------------------------------------- streams ---
int ofl_stream_create(int dev, ofl_stream** out) {
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  auto* s = new ofl_stream();
  s->dev = dev;
  // non-blocking: never implicitly ordered with the legacy default stream
  e = cudaStreamCreateWithFlags(&s->cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->fence, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    if (s->cs) cudaStreamDestroy(s->cs);
    delete s;
    return cuda_error(e, "cudaStreamCreate");
  }
  {
    std::lock_guard<std::mutex> l(g_streams_mu);
    g_streams.insert(s);
  }
  *out = s;
  return OFL_OK;
}

int ofl_stream_destroy(ofl_stream* s) {
  OFL_CHECK_STREAM(s);
  {
    std::lock_guard<std::mutex> l(g_streams_mu);
    g_streams.erase(s);
  }
  use_device(s->dev);
  cudaStreamSynchronize(s->cs);
  {
    std::lock_guard<std::mutex> g(s->mu);
    s->markers.clear();
    if (s->scratch) cudaFree(s->scratch);
  }
  if (s->fence) cudaEventDestroy(s->fence);
  cudaStreamDestroy(s->cs);
  delete s;
  return OFL_OK;
}

uint64_t ofl_stream_tail(ofl_stream* s) {
  std::lock_guard<std::mutex> g(s->mu);
  return s->tail;
}

uint64_t ofl_stream_done(ofl_stream* s) { return s->done.load(std::memory_order_acquire); }
void* ofl_stream_handle(ofl_stream* s) { return (void*)s->cs; }

// --------------------------------------------------------------- memory ---
// ------------------------------------------------------------- CUDA IPC ---
// Device allocations shared between the processes of one node (one process
// per GPU under torchrun): the owner exports a handle, the others map it and
// reach the memory over NVLink (peer access enabled lazily by the driver).
int ofl_ipc_handle(void* dptr, char* out64) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dptr);
  if (e != cudaSuccess) return cuda_error(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  memcpy(out64, &h, sizeof(h));
  return OFL_OK;
}

int ofl_ipc_open(int dev, const char* handle64, void** dptr) {
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_error(e, "cudaIpcOpenMemHandle");
  return OFL_OK;
}

int ofl_ipc_close(int dev, void* dptr) {
  cudaError_t e = use_device(dev);
  if (e == cudaSuccess) e = cudaIpcCloseMemHandle(dptr);
  if (e != cudaSuccess) return cuda_error(e, "cudaIpcCloseMemHandle");
  return OFL_OK;
}

static int oom(int dev, uint64_t bytes) {
  return set_error(OFL_ERR_OOM, "cuda" + std::to_string(dev) + ": " + std::to_string(bytes) +
                                    " bytes requested, allocation failed");
}

// Hand memory that freed buffers hold back to the device (before retrying an
// allocation that ran out).  First without waiting for anything: the pool's
// kept blocks and the released VMM mappings cached for reuse.  Only with
// `wait` also the frees still queued behind other streams' work (their fence
// events), which can take as long as those streams' kernel chains -- so an
// allocation that the caches can satisfy never stalls behind them.
static void reclaim(int dev, bool wait, size_t need) {
  if (wait) {
    std::lock_guard<std::mutex> f(g_free_mu[dev]);
    if (g_free_stream[dev]) cudaStreamSynchronize(g_free_stream[dev]);
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  if (wait) vmm_drain();
  // the first pass unmaps only what the request needs (largest cached
  // mappings first); waiting frees everything
  vmm_trim(dev, wait ? 0 : need);
  (void)cudaGetLastError();
}

int ofl_trim_memory(int dev) {
  if (dev < 0 || dev >= kMaxDev) return set_error(OFL_ERR_BAD_ARGS, "bad device ordinal");
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  std::lock_guard<std::mutex> g(g_zero_mu[dev]);
  reclaim(dev, true, 0);
  return OFL_OK;
}

int ofl_malloc(int dev, uint64_t bytes, void** dptr) {
  if (bytes == 0) return set_error(OFL_ERR_BAD_ARGS, "buffer size must be positive");
  if (dev < 0 || dev >= kMaxDev) return set_error(OFL_ERR_BAD_ARGS, "bad device ordinal");
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  std::lock_guard<std::mutex> g(g_zero_mu[dev]);
  e = internal_stream(dev);
  if (e == cudaSuccess) e = pool_setup(dev);
  if (e != cudaSuccess) return cuda_error(e, "memory pool setup");
  // a request beyond the device's capacity fails at once
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && bytes > total_b) return oom(dev, bytes);
  void* p = nullptr;
  if (bytes >= kVmmMin && vmm_available()) {
    // large buffers: their own mapping (fast to create, freed without any
    // device-wide synchronisation; ofl_vmm.cu)
    int st = vmm_alloc(dev, bytes, &p);
    for (int wait = 0; st == OFL_ERR_OOM && wait < 2; ++wait) {
      reclaim(dev, wait != 0, bytes);
      st = vmm_alloc(dev, bytes, &p);
    }
    if (st) return st;
    e = cudaMemsetAsync(p, 0, bytes, g_zero_stream[dev]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g_zero_stream[dev]);
    if (e != cudaSuccess) {
      std::vector<cudaEvent_t> none;
      vmm_free_after(p, none);
      return cuda_error(e, "zero fill");
    }
    *dptr = p;
    return OFL_OK;
  }
  e = cudaMallocAsync(&p, bytes, g_zero_stream[dev]);
  for (int wait = 0; e == cudaErrorMemoryAllocation && wait < 2; ++wait) {
    (void)cudaGetLastError();
    reclaim(dev, wait != 0, bytes);
    e = cudaMallocAsync(&p, bytes, g_zero_stream[dev]);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) return oom(dev, bytes);
    return cuda_error(e, "cudaMallocAsync");
  }
  // zero-initialised like the reference's np.zeros storage (buffer.py:32);
  // complete before any stream can see the pointer.
  e = cudaMemsetAsync(p, 0, bytes, g_zero_stream[dev]);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g_zero_stream[dev]);
  if (e != cudaSuccess) {
    cudaFreeAsync(p, g_zero_stream[dev]);
    return cuda_error(e, "zero fill");
  }
  *dptr = p;
  return OFL_OK;
}

int ofl_malloc_shareable(int dev, uint64_t bytes, void** dptr) {
  if (bytes == 0) return set_error(OFL_ERR_BAD_ARGS, "buffer size must be positive");
  if (dev < 0 || dev >= kMaxDev) return set_error(OFL_ERR_BAD_ARGS, "bad device ordinal");
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  void* p = nullptr;
  e = cudaMalloc(&p, bytes);
  for (int wait = 0; e == cudaErrorMemoryAllocation && wait < 2; ++wait) {
    (void)cudaGetLastError();
    reclaim(dev, wait != 0, bytes);
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) return oom(dev, bytes);
    return cuda_error(e, "cudaMalloc");
  }
  std::lock_guard<std::mutex> g(g_zero_mu[dev]);
  e = internal_stream(dev);
  if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, bytes, g_zero_stream[dev]);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g_zero_stream[dev]);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_error(e, "zero fill");
  }
  {
    std::lock_guard<std::mutex> l(g_legacy_mu);
    g_legacy.insert(p);
  }
  *dptr = p;
  return OFL_OK;
}

int ofl_free(int dev, void* dptr) {
  if (!dptr) return OFL_OK;
  if (dev < 0 || dev >= kMaxDev) return set_error(OFL_ERR_BAD_ARGS, "bad device ordinal");
  bool legacy;
  {
    std::lock_guard<std::mutex> l(g_legacy_mu);
    legacy = g_legacy.erase(dptr) > 0;
  }
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  if (legacy) {
    // shareable buffers: cudaFree synchronises with in-flight work, so they
    // drain before they are released (registry.py:104-109 semantics)
    e = cudaFree(dptr);
    if (e != cudaSuccess) return cuda_error(e, "cudaFree");
    return OFL_OK;
  }
  if (vmm_owns(dptr)) {
    // released by the reaper once a fence recorded now on every live stream
    // (of any device: peer copies, peer stores) has passed
    std::vector<cudaEvent_t> fences;
    {
      std::lock_guard<std::mutex> l(g_streams_mu);
      for (ofl_stream* s : g_streams) {
        if (use_device(s->dev) != cudaSuccess) continue;
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) continue;
        if (cudaEventRecord(ev, s->cs) == cudaSuccess)
          fences.push_back(ev);
        else
          cudaEventDestroy(ev);
      }
    }
    (void)cudaGetLastError();
    use_device(dev);
    vmm_free_after(dptr, fences);
    return OFL_OK;
  }
  // ordered after the work enqueued so far on every live stream (any device
  // may reach the buffer: peer copies, peer stores), without blocking them
  std::lock_guard<std::mutex> g(g_free_mu[dev]);
  if (!g_free_stream[dev]) {
    e = cudaStreamCreateWithFlags(&g_free_stream[dev], cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_error(e, "cudaStreamCreate");
  }
  {
    std::lock_guard<std::mutex> l(g_streams_mu);
    for (ofl_stream* s : g_streams) {
      if (use_device(s->dev) != cudaSuccess) continue;
      if (cudaEventRecord(s->fence, s->cs) == cudaSuccess)
        (void)cudaStreamWaitEvent(g_free_stream[dev], s->fence, 0);
    }
  }
  e = use_device(dev);
  if (e == cudaSuccess) e = cudaFreeAsync(dptr, g_free_stream[dev]);
  if (e != cudaSuccess) return cuda_error(e, "cudaFreeAsync");
  return OFL_OK;
}

int ofl_host_alloc(uint64_t bytes, void** hptr) {
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return cuda_error(e, "cudaHostAlloc");
  }
  *hptr = p;
  return OFL_OK;
}

int ofl_host_free(void* hptr) {
  if (!hptr) return OFL_OK;
  cudaError_t e = cudaFreeHost(hptr);
  if (e != cudaSuccess) return cuda_error(e, "cudaFreeHost");
  return OFL_OK;
}

// --------------------------------------------------------------- copies ---
static int copy_op(ofl_stream* s, void* dst, const void* src, uint64_t bytes, cudaMemcpyKind k,
                   uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  Enqueue q(s, "ofl:copy");
  if (!q.ok()) return q.status;
  if (bytes) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, k, s->cs);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync");
  }
  return q.finish(ticket);
}

int ofl_h2d(ofl_stream* s, void* dst, const void* src, uint64_t bytes, uint64_t* ticket) {
  return copy_op(s, dst, src, bytes, cudaMemcpyHostToDevice, ticket);
}
int ofl_d2h(ofl_stream* s, void* dst, const void* src, uint64_t bytes, uint64_t* ticket) {
  return copy_op(s, dst, src, bytes, cudaMemcpyDeviceToHost, ticket);
}
int ofl_d2h_rows(ofl_stream* s, void* dst, uint64_t dst_pitch, const void* src,
                 uint64_t row_bytes, uint64_t rows, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (dst_pitch < row_bytes) return set_error(OFL_ERR_BAD_ARGS, "destination pitch < row bytes");
  Enqueue q(s, "ofl:d2h_rows");
  if (!q.ok()) return q.status;
  if (row_bytes && rows) {
    // contiguous rows: one linear DMA (a 2-D copy pays per row)
    cudaError_t e = dst_pitch == row_bytes
                        ? cudaMemcpyAsync(dst, src, row_bytes * rows, cudaMemcpyDeviceToHost, s->cs)
                        : cudaMemcpy2DAsync(dst, dst_pitch, src, row_bytes, row_bytes, rows,
                                            cudaMemcpyDeviceToHost, s->cs);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpy2DAsync");
  }
  return q.finish(ticket);
}
int ofl_d2d(ofl_stream* s, void* dst, const void* src, uint64_t bytes, uint64_t* ticket) {
  return copy_op(s, dst, src, bytes, cudaMemcpyDeviceToDevice, ticket);
}

int ofl_p2p(ofl_stream* s, void* dst, int dst_dev, const void* src, int src_dev, uint64_t bytes,
            uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (dst_dev == src_dev) return copy_op(s, dst, src, bytes, cudaMemcpyDeviceToDevice, ticket);
  enable_peer(dst_dev, src_dev);
  enable_peer(src_dev, dst_dev);
  Enqueue q(s, "ofl:p2p");
  if (!q.ok()) return q.status;
  if (bytes) {
    cudaError_t e = cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes, s->cs);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyPeerAsync");
  }
  return q.finish(ticket);
}

int ofl_stream_wait(ofl_stream* waiter, ofl_stream* on, uint64_t ticket) {
  OFL_CHECK_STREAM(waiter);
  OFL_CHECK_STREAM(on);
  if (ticket == 0 || on->done.load(std::memory_order_acquire) >= ticket) return OFL_OK;
  std::shared_ptr<EvBox> box;
  {
    std::lock_guard<std::mutex> g(on->mu);
    if (ticket > on->tail) return set_error(OFL_ERR_BAD_ARGS, "ticket not yet enqueued");
    int st = covering(on, ticket, &box);
    if (st) return st;
  }
  if (waiter == on) return OFL_OK;  // same stream: already ordered
  std::lock_guard<std::mutex> g(waiter->mu);
  cudaError_t e = use_device(waiter->dev);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(waiter->cs, box->ev, 0);
  if (e != cudaSuccess) return cuda_error(e, "cudaStreamWaitEvent");
  return OFL_OK;
}

// ----------------------------------------------------------- completion ---
int ofl_query(ofl_stream* s, uint64_t ticket, int* ready) {
  OFL_CHECK_STREAM(s);
  *ready = 0;
  if (ticket == 0 || s->done.load(std::memory_order_acquire) >= ticket) {
    *ready = 1;
    return OFL_OK;
  }
  std::lock_guard<std::mutex> g(s->mu);
  if (ticket > s->tail) return set_error(OFL_ERR_BAD_ARGS, "ticket not yet enqueued");
  int st = reap(s);
  if (st) return st;
  if (s->done.load() >= ticket) {
    *ready = 1;
    return OFL_OK;
  }
  std::shared_ptr<EvBox> box;
  st = covering(s, ticket, &box);
  if (st) return st;
  cudaError_t e = cudaEventQuery(box->ev);
  if (e == cudaErrorNotReady) {
    (void)cudaGetLastError();
    return OFL_OK;
  }
  if (e != cudaSuccess) return cuda_error(e, "device fault");
  raise_done(s, box->ticket);
  *ready = 1;
  return reap(s);
}

int ofl_wait(ofl_stream* s, uint64_t ticket) {
  OFL_CHECK_STREAM(s);
  if (ticket == 0 || s->done.load(std::memory_order_acquire) >= ticket) return OFL_OK;
  std::shared_ptr<EvBox> box;
  uint64_t tail_sync = 0;
  {
    std::lock_guard<std::mutex> g(s->mu);
    if (ticket > s->tail) return set_error(OFL_ERR_BAD_ARGS, "ticket not yet enqueued");
    int st = reap(s);
    if (st) return st;
    if (s->done.load() >= ticket) return OFL_OK;
    if (ticket == s->tail && (s->markers.empty() || s->markers.back()->ticket < ticket)) {
      tail_sync = s->tail;  // waiting on the newest op: no marker needed
    } else {
      st = covering(s, ticket, &box);
      if (st) return st;
    }
  }
  if (tail_sync) {
    cudaError_t e = use_device(s->dev);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->cs);
    if (e != cudaSuccess) return cuda_error(e, "device fault");
    raise_done(s, tail_sync);
    std::lock_guard<std::mutex> g(s->mu);
    return reap(s);
  }
  cudaError_t e = cudaEventSynchronize(box->ev);
  if (e != cudaSuccess) return cuda_error(e, "device fault");
  raise_done(s, box->ticket);
  std::lock_guard<std::mutex> g(s->mu);
  return reap(s);
}

int ofl_notify(ofl_stream* s, uint64_t ticket, uint64_t token_id) {
  OFL_CHECK_STREAM(s);
  if (ticket == 0 || s->done.load(std::memory_order_acquire) >= ticket) {
    cq_post(token_id);
    return OFL_OK;
  }
  cq_init();
  std::lock_guard<std::mutex> g(s->mu);
  if (ticket > s->tail) return set_error(OFL_ERR_BAD_ARGS, "ticket not yet enqueued");
  cudaError_t e = use_device(s->dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  // The host function lands at the current tail, which covers `ticket`.
  auto* pl = new NotifyPayload{s, s->tail, token_id};
  e = cudaLaunchHostFunc(s->cs, host_complete, pl);
  if (e != cudaSuccess) {
    delete pl;
    return cuda_error(e, "cudaLaunchHostFunc");
  }
  return OFL_OK;
}

int ofl_completion_fd(void) {
  cq_init();
  return g_cq.efd;
}

int ofl_completion_post(uint64_t token_id) {
  cq_post(token_id);
  return OFL_OK;
}

int ofl_drain(uint64_t* ids, int cap, int* count) {
  std::lock_guard<std::mutex> g(g_cq.mu);
  int n = 0;
  while (n < cap && !g_cq.ids.empty()) {
    ids[n++] = g_cq.ids.front();
    g_cq.ids.pop_front();
  }
  *count = n;
  return OFL_OK;
}

// --------------------------------------------------------------- events ---
int ofl_event_create(int dev, ofl_event** out) {
  cudaError_t e = use_device(dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  auto* ev = new ofl_event();
  ev->dev = dev;
  e = cudaEventCreate(&ev->ev);
  if (e != cudaSuccess) {
    delete ev;
    return cuda_error(e, "cudaEventCreate");
  }
  *out = ev;
  return OFL_OK;
}

int ofl_event_record(ofl_event* ev, ofl_stream* s) {
  OFL_CHECK_STREAM(s);
  std::lock_guard<std::mutex> g(s->mu);
  cudaError_t e = use_device(s->dev);
  if (e == cudaSuccess) e = cudaEventRecord(ev->ev, s->cs);
  if (e != cudaSuccess) return cuda_error(e, "cudaEventRecord");
  return OFL_OK;
}

int ofl_event_elapsed_ms(ofl_event* a, ofl_event* b, float* ms) {
  cudaError_t e = cudaEventSynchronize(b->ev);
  if (e == cudaSuccess) e = cudaEventElapsedTime(ms, a->ev, b->ev);
  if (e != cudaSuccess) return cuda_error(e, "cudaEventElapsedTime");
  return OFL_OK;
}

int ofl_event_destroy(ofl_event* ev) {
  if (!ev) return OFL_OK;
  cudaEventDestroy(ev->ev);
  delete ev;
  return OFL_OK;
}

}  // extern "C"

namespace ofl {

int stream_scratch(ofl_stream* s, size_t bytes, void** out) {
  if (s->scratch_bytes < bytes) {
    if (s->scratch) {
      cudaStreamSynchronize(s->cs);
      cudaFree(s->scratch);
      s->scratch = nullptr;
      s->scratch_bytes = 0;
    }
    size_t want = bytes < 65536 ? 65536 : bytes;
    cudaError_t e = cudaMalloc(&s->scratch, want);
    if (e != cudaSuccess) return cuda_error(e, "scratch cudaMalloc");
    e = cudaMemsetAsync(s->scratch, 0, want, s->cs);  // ordered before first use
    if (e != cudaSuccess) return cuda_error(e, "scratch memset");
    s->scratch_bytes = want;
  }
  *out = s->scratch;
  return OFL_OK;
}

}  // namespace ofl
