// Raw-CUDA reference loops for the futurization-overhead benchmark
// (BASELINE config 5): the same H2D copy + kernel launch chain
// the futurized API issues, written directly against the CUDA runtime with
// no tokens, no tickets and no Python.  (t_futurized - t_raw) / K is the
// per-step overhead of the futures layer.
#include <chrono>

#include "ofl_internal.h"

// FP64 issue-rate probe for the Mandelbrot roofline: independent DMUL and
// DADD chains (no FMA — the bit-exact kernel may not contract either).
__global__ void k_fp64_peak(double* out, double a, double b, int iters) {
  double x[8], y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    x[k] = threadIdx.x + k;
    y[k] = blockIdx.x + k;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[k] = __dmul_rn(x[k], a);
      y[k] = __dadd_rn(y[k], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k] + y[k];
  if (s == 1234.5) out[0] = s;  // keep the chains alive
}

extern "C" int ofl_bench_fp64_peak(ofl_stream* s, double* ops_per_s) {
  OFL_CHECK_STREAM(s);
  std::lock_guard<std::mutex> g(s->mu);
  cudaError_t e = ofl::use_device(s->dev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "cudaSetDevice");
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int blocks = ofl::num_sms(s->dev) * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_fp64_peak<<<blocks, threads, 0, s->cs>>>(out, 0.999999, 1e-9, 64);  // warm-up
  cudaEventRecord(a, s->cs);
  k_fp64_peak<<<blocks, threads, 0, s->cs>>>(out, 0.999999, 1e-9, iters);
  cudaEventRecord(b, s->cs);
  e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return ofl::cuda_error(e, "fp64 probe");
  *ops_per_s = (double)blocks * threads * iters * 16 / (ms * 1e-3);
  ofl::count_launch(2);
  return OFL_OK;
}

// mode 0: stream order only, one sync at the end
// mode 1: additionally record an event after each step and make the next step
//         wait on it (cudaStreamWaitEvent) — explicit dependency chaining
// mode 2: cudaStreamSynchronize after every step (round-trip latency)
extern "C" int ofl_bench_raw_chain(ofl_stream* s, void* dst, const void* src, uint64_t bytes,
                                   double* a, const double* b, const double* c, uint64_t n,
                                   uint64_t steps, int mode, double* seconds) {
  OFL_CHECK_STREAM(s);
  std::lock_guard<std::mutex> g(s->mu);
  cudaError_t e = ofl::use_device(s->dev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "cudaSetDevice");
  cudaEvent_t ev = nullptr;
  if (mode == 1) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  const int sms = ofl::num_sms(s->dev);
  cudaStreamSynchronize(s->cs);
  auto t0 = std::chrono::steady_clock::now();
  for (uint64_t k = 0; k < steps; ++k) {
    if (mode == 1 && k) cudaStreamWaitEvent(s->cs, ev, 0);
    cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s->cs);
    // the same kernel and launch (attributes included) ofl_stream_op issues,
    // so the difference to the futurized chain is the runtime alone
    ofl::stream_launch(s->cs, sms, OFL_STREAM_TRIAD, a, b, c, 3.0, n);
    if (mode == 1) cudaEventRecord(ev, s->cs);
    if (mode == 2) cudaStreamSynchronize(s->cs);
  }
  e = cudaStreamSynchronize(s->cs);
  auto t1 = std::chrono::steady_clock::now();
  if (ev) cudaEventDestroy(ev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "raw chain");
  *seconds = std::chrono::duration<double>(t1 - t0).count();
  ofl::count_launch(steps);
  return OFL_OK;
}
