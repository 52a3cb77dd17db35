// STREAM copy / scale / add / triad over fp64 vectors (BASELINE config 1).
//
// The reference has no STREAM kernel; these are the sm_100a kernels bound to
// the .k programs in paper_1810_11482_b200/kernels/stream.k, whose semantics
// are the reference executor's (kernel/codegen.py:107-128): item gtid < n
// stores a[gtid] = f(b[gtid], c[gtid]).  Elements are independent, so the
// grid-stride order is free; the arithmetic is IEEE round-to-nearest with no
// FMA contraction (__dmul_rn/__dadd_rn), bit-identical to the CPU path.
//
// HBM-bound: 16 B/elem (copy, scale), 24 B/elem (add, triad).  Each thread
// keeps kUnroll independent 128-bit loads per input in flight; loads bypass
// L1 (.nc + L1::no_allocate), stores are evict-first (.cs) so the streamed
// output does not displace anything useful from L2.
#include "ofl_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

template <int OP>
__device__ __forceinline__ double apply(double b, double c, double s) {
  if constexpr (OP == OFL_STREAM_COPY) return b;
  else if constexpr (OP == OFL_STREAM_SCALE) return __dmul_rn(s, b);
  else if constexpr (OP == OFL_STREAM_ADD) return __dadd_rn(b, c);
  else return __dadd_rn(b, __dmul_rn(s, c));
}

template <int OP>
__device__ __forceinline__ double2 apply2(double2 b, double2 c, double s) {
  return make_double2(apply<OP>(b.x, c.x, s), apply<OP>(b.y, c.y, s));
}

template <int OP>
__global__ void __launch_bounds__(kThreads) k_stream_vec(double* __restrict__ a,
                                                         const double* __restrict__ b,
                                                         const double* __restrict__ c, double s,
                                                         uint64_t n) {
  constexpr bool kC = (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD);
  const uint64_t n2 = n >> 1;
  double2* __restrict__ a2 = reinterpret_cast<double2*>(a);
  const double2* __restrict__ b2 = reinterpret_cast<const double2*>(b);
  const double2* __restrict__ c2 = reinterpret_cast<const double2*>(c);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x;

  for (; i + (kUnroll - 1) * stride < n2; i += kUnroll * stride) {
    double2 vb[kUnroll], vc[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      vb[u] = ld_stream(b2 + i + u * stride);
      if constexpr (kC) vc[u] = ld_stream(c2 + i + u * stride);
      else vc[u] = vb[u];
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_stream(a2 + i + u * stride, apply2<OP>(vb[u], vc[u], s));
  }
  for (; i < n2; i += stride) {
    double2 vb = ld_stream(b2 + i);
    double2 vc = kC ? ld_stream(c2 + i) : vb;
    st_stream(a2 + i, apply2<OP>(vb, vc, s));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t j = n - 1;
    a[j] = apply<OP>(b[j], kC ? c[j] : 0.0, s);
  }
}

// Fallback for operands that are not 16-byte aligned.
template <int OP>
__global__ void __launch_bounds__(kThreads) k_stream_scalar(double* a, const double* b,
                                                            const double* c, double s,
                                                            uint64_t n) {
  constexpr bool kC = (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    a[i] = apply<OP>(b[i], kC ? c[i] : 0.0, s);
}

template <int OP>
cudaError_t launch(cudaStream_t st, int sms, double* a, const double* b, const double* c,
                   double s, uint64_t n) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                         reinterpret_cast<uintptr_t>(c)) & 15) == 0;
  // 8 resident 256-thread CTAs per SM (2048 threads); grid-stride beyond.
  const uint64_t per_wave = (uint64_t)sms * 8;
  const uint64_t units = aligned ? (n >> 1) : n;
  uint64_t blocks = (units + kThreads * kUnroll - 1) / (kThreads * kUnroll);
  if (blocks > per_wave) blocks = per_wave;
  if (blocks == 0) blocks = 1;
  if (aligned)
    k_stream_vec<OP><<<(unsigned)blocks, kThreads, 0, st>>>(a, b, c, s, n);
  else
    k_stream_scalar<OP><<<(unsigned)blocks, kThreads, 0, st>>>(a, b, c, s, n);
  return cudaPeekAtLastError();
}

}  // namespace

extern "C" int ofl_stream_op(ofl_stream* s, int op, double* a, const double* b, const double* c,
                             double scalar, uint64_t n, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (op < OFL_STREAM_COPY || op > OFL_STREAM_TRIAD)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "unknown STREAM op");
  if (!c) c = b;
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  if (n) {
    const int sms = ofl::num_sms(s->dev);
    cudaError_t e;
    switch (op) {
      case OFL_STREAM_COPY: e = launch<OFL_STREAM_COPY>(s->cs, sms, a, b, c, scalar, n); break;
      case OFL_STREAM_SCALE: e = launch<OFL_STREAM_SCALE>(s->cs, sms, a, b, c, scalar, n); break;
      case OFL_STREAM_ADD: e = launch<OFL_STREAM_ADD>(s->cs, sms, a, b, c, scalar, n); break;
      default: e = launch<OFL_STREAM_TRIAD>(s->cs, sms, a, b, c, scalar, n); break;
    }
    if (e != cudaSuccess) return ofl::cuda_error(e, "STREAM launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}
