// Pageable host -> device writes (BufferObject.enqueue_write with a plain
// `bytes`/numpy payload; reference buffer.py:40-47 makes three host copies).
//
// The payload is cut into chunks that are copied into a ring of pinned
// staging slots by a small pool of host threads and DMA'd from there, so the
// host copy of chunk k+1 overlaps the PCIe transfer of chunk k.  The caller
// returns once the last chunk is staged: the payload may then be reused, as
// in the reference (which owns a copy once the call returns).  The stream
// lock is held for the whole write, so the write stays one atomic stream
// operation with one ticket.
#include <condition_variable>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "ofl_internal.h"

namespace {

constexpr size_t kSlotBytes = 8u << 20;  // 8 MiB per slot
constexpr int kSlots = 8;                // 64 MiB of pinned staging per process
constexpr int kCopyThreads = 4;

struct Slot {
  void* host = nullptr;
  cudaEvent_t done = nullptr;  // recorded after the slot's DMA
  int dev = -1;
  bool used = false;
};

struct Ring {
  std::mutex mu;  // one staged write at a time
  Slot slots[kSlots];
  int next = 0;
};
Ring g_ring;

// minimal fork-join pool for the host copies
class CopyPool {
 public:
  CopyPool() {
    for (int i = 0; i < kCopyThreads; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // copy [src, src+n) to dst using all workers plus the caller
  void copy(void* dst, const void* src, size_t n) {
    const size_t parts = kCopyThreads + 1;
    const size_t per = (n + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> g(mu_);
      pending_ = 0;
      for (size_t p = 1; p < parts; ++p) {
        const size_t lo = p * per;
        if (lo >= n) break;
        const size_t len = (lo + per <= n) ? per : n - lo;
        jobs_.push_back([=] { std::memcpy((char*)dst + lo, (const char*)src + lo, len); });
        ++pending_;
      }
    }
    cv_.notify_all();
    std::memcpy(dst, src, per < n ? per : n);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return stop_ || !jobs_.empty(); });
        if (stop_) return;
        job = std::move(jobs_.back());
        jobs_.pop_back();
      }
      job();
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::function<void()>> jobs_;
  std::vector<std::thread> workers_;
  int pending_ = 0;
  bool stop_ = false;
};

CopyPool& pool() {
  static CopyPool* p = new CopyPool();  // never destroyed (process lifetime)
  return *p;
}

}  // namespace

// Host memcpy on the copy pool (large staging <-> pageable copies).
extern "C" int ofl_host_memcpy(void* dst, const void* src, uint64_t bytes) {
  if (bytes >= (4u << 20)) {
    static std::mutex mu;  // the pool runs one fork-join copy at a time
    std::lock_guard<std::mutex> g(mu);
    std::lock_guard<std::mutex> r(g_ring.mu);
    pool().copy(dst, src, (size_t)bytes);
  } else if (bytes) {
    std::memcpy(dst, src, (size_t)bytes);
  }
  return OFL_OK;
}

extern "C" int ofl_h2d_pageable(ofl_stream* s, void* dst, const void* src, uint64_t bytes,
                                uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  std::lock_guard<std::mutex> ring_lock(g_ring.mu);
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  uint64_t off = 0;
  while (off < bytes) {
    Slot& slot = g_ring.slots[g_ring.next];
    g_ring.next = (g_ring.next + 1) % kSlots;
    cudaError_t e;
    if (!slot.host) {
      e = cudaHostAlloc(&slot.host, kSlotBytes, cudaHostAllocPortable);
      if (e != cudaSuccess) return ofl::cuda_error(e, "staging cudaHostAlloc");
    }
    if (slot.used) {
      e = cudaEventSynchronize(slot.done);  // the slot's previous DMA finished
      if (e != cudaSuccess) return ofl::cuda_error(e, "staging slot wait");
    }
    if (slot.dev != s->dev) {  // events belong to a device
      if (slot.done) cudaEventDestroy(slot.done);
      e = cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming);
      if (e != cudaSuccess) return ofl::cuda_error(e, "staging event");
      slot.dev = s->dev;
    }
    const size_t len = bytes - off < kSlotBytes ? (size_t)(bytes - off) : kSlotBytes;
    if (len >= (1u << 20))
      pool().copy(slot.host, (const char*)src + off, len);
    else
      std::memcpy(slot.host, (const char*)src + off, len);
    e = cudaMemcpyAsync((char*)dst + off, slot.host, len, cudaMemcpyHostToDevice, s->cs);
    if (e == cudaSuccess) e = cudaEventRecord(slot.done, s->cs);
    if (e != cudaSuccess) return ofl::cuda_error(e, "staged H2D");
    slot.used = true;
    off += len;
  }
  return q.finish(ticket);
}
