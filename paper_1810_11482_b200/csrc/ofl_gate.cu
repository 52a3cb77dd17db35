// Device-side ordering between processes (one process per GPU): a pass on
// one GPU must start only after its neighbours' previous pass finished, and
// with one process per GPU there is no shared stream or event to express
// that.  Instead each rank owns a 64-bit completion counter in device memory
// that the other ranks map through CUDA IPC:
//   ofl_gate_signal — after this rank's work: fence, counter = value
//   ofl_gate_wait   — before the next work: one thread polls the given
//                     counters (peer memory over NVLink) until each reaches
//                     its target, then lets the stream continue.
// Both are one-thread kernels, so the ordering stays on the device (no host
// round trip per exchange).  The wait is bounded: after ~20 s it gives up
// and records a timeout in *status (the caller's counter block).
#include "ofl_internal.h"

namespace {

__global__ void k_gate_signal(unsigned long long* counter, unsigned long long value) {
  __threadfence_system();  // this stream's earlier writes (incl. peer stores) first
  *reinterpret_cast<volatile unsigned long long*>(counter) = value;
  __threadfence_system();
}

__global__ void k_gate_wait(const unsigned long long* const* counters, int count,
                            unsigned long long target, unsigned long long* status) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < count; ++i) {
    const volatile unsigned long long* c = counters[i];
    while (*c < target) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20ull * 1000 * 1000 * 1000) {
        *status = 1;
        return;
      }
      __nanosleep(500);
    }
  }
  __threadfence_system();
}

}  // namespace

extern "C" int ofl_gate_signal(ofl_stream* s, unsigned long long* counter, uint64_t value,
                               uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  ofl::Enqueue q(s, "ofl:gate_signal");
  if (!q.ok()) return q.status;
  k_gate_signal<<<1, 1, 0, s->cs>>>(counter, value);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ofl::cuda_error(e, "gate signal");
  ofl::count_launch();
  return q.finish(ticket);
}

extern "C" int ofl_gate_wait(ofl_stream* s, const unsigned long long* const* counters_dev,
                             int count, uint64_t target, unsigned long long* status,
                             uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (count < 0 || count > 64) return ofl::set_error(OFL_ERR_BAD_ARGS, "gate: 0..64 counters");
  ofl::Enqueue q(s, "ofl:gate_wait");
  if (!q.ok()) return q.status;
  if (count) {
    k_gate_wait<<<1, 1, 0, s->cs>>>(counters_dev, count, target, status);
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "gate wait");
    ofl::count_launch();
  }
  return q.finish(ticket);
}
