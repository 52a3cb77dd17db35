// Internal declarations shared by the libofl.so translation units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ofl.h"

namespace ofl {

// A completion marker: a CUDA event recorded right after ticket `ticket`.
// Shared between the stream's marker list and any thread blocked on it; the
// event returns to the per-device pool when the last holder lets go.
struct EvBox {
  int dev;
  cudaEvent_t ev;
  uint64_t ticket;
  ~EvBox();
};

}  // namespace ofl

struct ofl_stream {
  int dev;
  cudaStream_t cs;
  std::mutex mu;                   // serialises enqueue + ticket assignment
  uint64_t tail = 0;               // last ticket enqueued
  std::atomic<uint64_t> done{0};   // highest ticket known complete
  std::deque<std::shared_ptr<ofl::EvBox>> markers;  // ascending, placed lazily
  // per-stream device scratch for multi-block reductions / work queues
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // recorded by ofl_free to order a stream-ordered free after this stream's
  // work enqueued so far (the free's stream waits on it)
  cudaEvent_t fence = nullptr;
};

struct ofl_event {
  int dev;
  cudaEvent_t ev;
};

namespace ofl {

constexpr int kMaxDev = 64;
// device buffers of this size and up are VMM mappings (ofl_vmm.cu)
constexpr size_t kVmmMin = 2u << 20;

int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);
cudaError_t use_device(int dev);
int num_sms(int dev);
void count_launch(uint64_t n = 1);
// the STREAM launcher behind ofl_stream_op (k_stream.cu), shared with the
// raw-CUDA chain of the overhead benchmark so both launch identical kernels
cudaError_t stream_launch(cudaStream_t st, int sms, int op, double* a, const double* b,
                          const double* c, double scalar, uint64_t n);
// cudaDeviceEnablePeerAccess(from -> to) once per pair, if the pair supports it
void enable_peer(int from, int to);
// VMM allocations (ofl_vmm.cu)
bool vmm_available();
int vmm_alloc(int dev, size_t bytes, void** out);
bool vmm_owns(void* p);
bool vmm_free_after(void* p, std::vector<cudaEvent_t>& fences);
void vmm_drain();
void vmm_trim(int dev, size_t need = 0);
void vmm_grant_peer(int from, int to);
// Scratch of at least `bytes` on the stream's device (caller holds s->mu).
int stream_scratch(ofl_stream* s, size_t bytes, void** out);

// RAII: locks the stream, makes its device current; finish() assigns the
// ticket after the CUDA call(s) succeeded.
// Every stream operation enqueues under its stream's lock and takes the next
// ticket.  It is also an NVTX range named after the entry point ("ofl:heat",
// "ofl:stream_op", ...), so nsys timelines and `ncu --nvtx --nvtx-include`
// filters see the runtime's operations; NVTX3 is header-only and a no-op
// unless a profiler injects itself.
struct Enqueue {
  ofl_stream* s;
  std::unique_lock<std::mutex> lk;
  int status = OFL_OK;
  const char* what;
  explicit Enqueue(ofl_stream* st, const char* name = nullptr) : s(st), lk(st->mu), what(name) {
    if (what) nvtxRangePushA(what);
    cudaError_t e = use_device(st->dev);
    if (e != cudaSuccess) status = cuda_error(e, "cudaSetDevice");
  }
  ~Enqueue() {
    if (what) nvtxRangePop();
  }
  Enqueue(const Enqueue&) = delete;
  Enqueue& operator=(const Enqueue&) = delete;
  bool ok() const { return status == OFL_OK; }
  int finish(uint64_t* ticket) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "enqueue");
    s->tail += 1;
    if (ticket) *ticket = s->tail;
    return OFL_OK;
  }
};

}  // namespace ofl

#define OFL_CHECK_STREAM(s) \
  do { if (!(s)) return ofl::set_error(OFL_ERR_BAD_ARGS, "null stream"); } while (0)
