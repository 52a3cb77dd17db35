// Host side of large transfers between pageable memory and HBM.
//
// Writes (BufferObject.enqueue_write with a plain `bytes`/numpy payload; the
// reference makes three host copies, buffer.py:40-47): the payload is cut
// into chunks that the copy threads stage into a ring of pinned slots; each
// chunk is DMA'd as soon as its copy is done, while the copies of the next
// chunks proceed, so host copies and the PCIe transfer overlap.  The caller
// returns once the last chunk is staged: the payload may then be reused, as
// in the reference (which owns a copy once the call returns).  The stream
// lock is held for the whole write, so it stays one atomic stream operation
// with one ticket.
//
// Reads (BufferObject.enqueue_read -> `bytes`, buffer.py:49-55): the D2H
// goes to a pinned staging block in chunks, each followed by an event
// (ofl_d2h_chunked); collecting (ofl_collect, run by the token's finish
// step) waits for each chunk's event and hands it to the copy threads, so
// the copy into the pageable destination of chunk k overlaps the DMA of the
// chunks after it.
#include <immintrin.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <thread>
#include <vector>

#include "ofl_internal.h"

namespace {

constexpr size_t kSlotBytes = 8u << 20;  // 8 MiB per staging slot
constexpr int kSlots = 8;                // 64 MiB of pinned write staging per process
constexpr size_t kPart = 1u << 20;       // copy task granularity
constexpr size_t kHugePage = 2u << 20;   // reads into fresh memory: one task per huge page
constexpr int kLag = 3;                  // chunks being copied ahead of the DMA issue

// A fixed pool of copy threads taking independent memcpy tasks; a Group
// counts the outstanding tasks of one chunk (or of one whole copy).
struct Group {
  std::atomic<int> left{0};
  std::mutex mu;
  std::condition_variable cv;
  void done_one() {
    if (left.fetch_sub(1, std::memory_order_acq_rel) == 1) {
      std::lock_guard<std::mutex> g(mu);
      cv.notify_all();
    }
  }
  void wait() {
    if (left.load(std::memory_order_acquire) == 0) return;
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return left.load(std::memory_order_acquire) == 0; });
  }
};

struct Task {
  char* dst;
  const char* src;
  size_t n;
  Group* g;
};

// Copy with non-temporal (streaming) stores: the destination lines go to
// DRAM without being read first (no read-for-ownership) and without
// evicting the cache.  On the GPU box's host, 15 threads copy 256 MiB into
// resident memory at 80 GB/s this way against 54 GB/s with memcpy
// (profiles/r02_nt_copy.txt, scripts/probes/nt_copy_probe.c).
__attribute__((target("avx2"))) void copy_stream(char* d, const char* s, size_t n) {
  size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(d, s, head);
  d += head, s += head, n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
  }
  std::memcpy(d + i, s + i, n - i);
  _mm_sfence();  // the streamed lines are globally visible before the task counts as done
}

const bool g_avx2 = __builtin_cpu_supports("avx2");
const uintptr_t g_page = (uintptr_t)sysconf(_SC_PAGESIZE);

// One copy task.  Into resident memory (pinned staging slots, a caller's
// array) streaming stores win; into fresh memory — a new bytes object,
// first-touched by this very copy — the page fault dominates and plain
// memcpy is slightly faster (44.7 vs 42.0 GB/s), so the task asks the kernel
// whether its first destination page is resident (mincore: one syscall per
// task of up to 2 MiB).
void run_task(const Task& t) {
  if (g_avx2 && t.n >= 4096) {
    unsigned char resident = 0;
    void* page = (void*)((uintptr_t)t.dst & ~(g_page - 1));
    if (mincore(page, 1, &resident) == 0 && (resident & 1)) {
      copy_stream(t.dst, t.src, t.n);
      return;
    }
  }
  std::memcpy(t.dst, t.src, t.n);
}

class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int n = (int)std::max(2u, std::min(15u, hw ? hw - 1 : 4u));
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  // split [src, src+n) -> dst into tasks of `part` bytes counted by g; the
  // cuts fall on multiples of `part` in the DESTINATION's address space, so
  // no two threads first-touch the same (2 MiB huge) page of a fresh buffer
  void submit(void* dst, const void* src, size_t n, Group* g, size_t part = kPart) {
    std::vector<Task> tasks;
    size_t off = 0;
    while (off < n) {
      const uintptr_t d = (uintptr_t)dst + off;
      const size_t to_cut = part - (size_t)(d % part);
      const size_t len = std::min(to_cut, n - off);
      tasks.push_back(Task{(char*)dst + off, (const char*)src + off, len, g});
      off += len;
    }
    g->left.fetch_add((int)tasks.size(), std::memory_order_acq_rel);
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (auto& t : tasks) q_.push_back(t);
    }
    cv_.notify_all();
  }
  // copy now, using the pool and the calling thread
  void copy(void* dst, const void* src, size_t n) {
    Group g;
    submit(dst, src, n, &g);
    help(&g);
    g.wait();
  }
  // run queued tasks on the calling thread until g is done or the queue is empty
  void help(Group* g) {
    while (g->left.load(std::memory_order_acquire) > 0) {
      Task t;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (q_.empty()) return;
        t = q_.front();
        q_.pop_front();
      }
      run_task(t);
      t.g->done_one();
    }
  }

 private:
  void loop() {
    for (;;) {
      Task t;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return !q_.empty(); });
        t = q_.front();
        q_.pop_front();
      }
      run_task(t);
      t.g->done_one();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Task> q_;
  std::vector<std::thread> workers_;
};

CopyPool& pool() {
  static CopyPool* p = new CopyPool();  // never destroyed (process lifetime)
  return *p;
}

struct Slot {
  void* host = nullptr;
  cudaEvent_t done = nullptr;  // recorded after the slot's DMA
  int dev = -1;
  bool used = false;
  Group copied;                // the slot's host copy
};

struct Ring {
  std::mutex mu;  // one staged write at a time
  Slot slots[kSlots];
};
Ring g_ring;

int prepare_slot(Slot& slot, int dev) {
  cudaError_t e;
  if (!slot.host) {
    e = cudaHostAlloc(&slot.host, kSlotBytes, cudaHostAllocPortable);
    if (e != cudaSuccess) return ofl::cuda_error(e, "staging cudaHostAlloc");
  }
  if (slot.used) {
    e = cudaEventSynchronize(slot.done);  // the slot's previous DMA finished
    if (e != cudaSuccess) return ofl::cuda_error(e, "staging slot wait");
    slot.used = false;
  }
  if (slot.dev != dev) {  // events belong to a device
    if (slot.done) cudaEventDestroy(slot.done);
    e = cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming);
    if (e != cudaSuccess) return ofl::cuda_error(e, "staging event");
    slot.dev = dev;
  }
  return OFL_OK;
}

}  // namespace

// pending chunked device->host read (ofl_d2h_chunked / ofl_collect)
struct ofl_read {
  int dev;
  const char* staging;
  uint64_t bytes, chunk;
  std::vector<cudaEvent_t> events;  // one per chunk, recorded after its DMA
};

// Host memcpy on the copy threads (large staging <-> pageable copies).
extern "C" int ofl_host_memcpy(void* dst, const void* src, uint64_t bytes) {
  if (bytes >= (4u << 20))
    pool().copy(dst, src, (size_t)bytes);
  else if (bytes)
    std::memcpy(dst, src, (size_t)bytes);
  return OFL_OK;
}

extern "C" int ofl_h2d_pageable(ofl_stream* s, void* dst, const void* src, uint64_t bytes,
                                uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  std::lock_guard<std::mutex> ring_lock(g_ring.mu);
  ofl::Enqueue q(s, "ofl:h2d_pageable");
  if (!q.ok()) return q.status;
  const uint64_t nchunks = (bytes + kSlotBytes - 1) / kSlotBytes;
  auto len_of = [&](uint64_t k) {
    return (size_t)std::min<uint64_t>(kSlotBytes, bytes - k * kSlotBytes);
  };
  // chunk k uses slot k % kSlots; its copy is submitted kLag chunks before
  // its DMA is issued, so up to kLag chunks are being staged while the
  // caller waits for the oldest one and hands it to the copy engine
  auto stage = [&](uint64_t k) -> int {
    Slot& slot = g_ring.slots[k % kSlots];
    const int st = prepare_slot(slot, s->dev);
    if (st) return st;
    pool().submit(slot.host, (const char*)src + k * kSlotBytes, len_of(k), &slot.copied);
    return OFL_OK;
  };
  int status = OFL_OK;
  uint64_t staged = 0;
  for (uint64_t k = 0; k < nchunks && status == OFL_OK; ++k) {
    while (staged < nchunks && staged <= k + kLag && status == OFL_OK) status = stage(staged++);
    if (status) break;
    Slot& slot = g_ring.slots[k % kSlots];
    pool().help(&slot.copied);
    slot.copied.wait();
    cudaError_t e = cudaMemcpyAsync((char*)dst + k * kSlotBytes, slot.host, len_of(k),
                                    cudaMemcpyHostToDevice, s->cs);
    if (e == cudaSuccess) e = cudaEventRecord(slot.done, s->cs);
    if (e != cudaSuccess) status = ofl::cuda_error(e, "staged H2D");
    slot.used = true;
  }
  // never leave copy tasks running into slots after an error
  for (auto& slot : g_ring.slots) slot.copied.wait();
  if (status) return status;
  return q.finish(ticket);
}

extern "C" int ofl_d2h_chunked(ofl_stream* s, void* staging, const void* src, uint64_t bytes,
                               uint64_t chunk, ofl_read** out, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (!out || !staging || !chunk) return ofl::set_error(OFL_ERR_BAD_ARGS, "d2h_chunked arguments");
  *out = nullptr;
  auto* r = new ofl_read{s->dev, (const char*)staging, bytes, chunk, {}};
  ofl::Enqueue q(s, "ofl:d2h_chunked");
  if (!q.ok()) {
    delete r;
    return q.status;
  }
  for (uint64_t off = 0; off < bytes; off += chunk) {
    const uint64_t len = std::min(chunk, bytes - off);
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((char*)staging + off, (const char*)src + off, len,
                          cudaMemcpyDeviceToHost, s->cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev, s->cs);
    if (e != cudaSuccess) {
      for (auto x : r->events) cudaEventDestroy(x);
      delete r;
      return ofl::cuda_error(e, "chunked D2H");
    }
    r->events.push_back(ev);
  }
  const int st = q.finish(ticket);
  if (st) {
    for (auto x : r->events) cudaEventDestroy(x);
    delete r;
    return st;
  }
  *out = r;
  return OFL_OK;
}

extern "C" int ofl_collect(ofl_read* r, void* dst) {
  if (!r) return ofl::set_error(OFL_ERR_BAD_ARGS, "null read handle");
  cudaError_t e = ofl::use_device(r->dev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "cudaSetDevice");
  Group g;
  int status = OFL_OK;
  for (size_t i = 0; i < r->events.size(); ++i) {
    e = cudaEventSynchronize(r->events[i]);
    if (e != cudaSuccess) {
      status = ofl::cuda_error(e, "device fault");
      break;
    }
    const uint64_t off = i * r->chunk;
    pool().submit((char*)dst + off, r->staging + off, (size_t)std::min(r->chunk, r->bytes - off),
                  &g, kHugePage);
  }
  pool().help(&g);
  g.wait();
  return status;
}

extern "C" int ofl_read_release(ofl_read* r) {
  if (!r) return OFL_OK;
  if (ofl::use_device(r->dev) == cudaSuccess)
    for (auto x : r->events) cudaEventDestroy(x);
  delete r;
  return OFL_OK;
}
