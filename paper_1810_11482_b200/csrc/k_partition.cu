// Pythagorean identity over global element indices (partition.k,
// /root/reference/pkg/src/offloadrt/bench/kernels/partition.k:3-8), the
// kernel of the paper's Alg. 1 partition benchmark (harness.py:236-335):
//   out[i] = sqrt(sin(v)*sin(v) + cos(v)*cos(v)),  v = f64((offset + i) mod 2^32)
// Products and sum are separate round-to-nearest ops; sin/cos are CUDA's
// double-precision functions (<= 2 ulp), so parity with the libm CPU path is
// by tolerance (1e-12 absolute on outputs of ~1.0, test_acceptance.py:77-84).
#include "ofl_internal.h"

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) k_partition(double* __restrict__ out, uint32_t offset,
                                                        uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < count; i += stride) {
    const double v = (double)(uint32_t)(offset + (uint32_t)i);
    double sv, cv;
    sincos(v, &sv, &cv);
    __stcs(out + i, __dsqrt_rn(__dadd_rn(__dmul_rn(sv, sv), __dmul_rn(cv, cv))));
  }
}

}  // namespace

extern "C" int ofl_partition(ofl_stream* s, double* out, uint32_t offset, uint64_t count,
                             uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  ofl::Enqueue q(s, "ofl:partition");
  if (!q.ok()) return q.status;
  if (count) {
    uint64_t blocks = (count + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)ofl::num_sms(s->dev) * 8;
    if (blocks > cap) blocks = cap;
    k_partition<<<(unsigned)blocks, kThreads, 0, s->cs>>>(out, offset, count);
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "partition launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}
