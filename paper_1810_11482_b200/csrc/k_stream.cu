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
// keeps its 128-bit loads per input in flight; loads bypass L1 (.nc +
// L1::no_allocate), stores are evict-first (.cs) so the streamed output does
// not displace anything useful from L2.
#include "ofl_internal.h"

namespace {

constexpr int kThreads = 256;

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

// Tile form: one CTA per contiguous tile of T*U double2, no loop; the
// hardware block scheduler load-balances the (many) tiles.
template <int OP, int T, int U, bool kPDL>
__global__ void __launch_bounds__(T) k_stream_tile(double* __restrict__ a,
                                                  const double* __restrict__ b,
                                                  const double* __restrict__ c, double s,
                                                  uint64_t n) {
  constexpr bool kC = (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD);
  if constexpr (kPDL) {
    // programmatic dependent launch: let the next grid on the stream start
    // launching its CTAs while this one drains, and wait here until the
    // previous grid has completed and its memory is visible
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const uint64_t n2 = n >> 1;
  double2* __restrict__ a2 = reinterpret_cast<double2*>(a);
  const double2* __restrict__ b2 = reinterpret_cast<const double2*>(b);
  const double2* __restrict__ c2 = reinterpret_cast<const double2*>(c);
  const uint64_t base = (uint64_t)blockIdx.x * (T * U) + threadIdx.x;
  if (base + (U - 1) * T < n2) {
    double2 vb[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vb[u] = ld_stream(b2 + base + u * T);
      if constexpr (kC) vc[u] = ld_stream(c2 + base + u * T);
      else vc[u] = vb[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st_stream(a2 + base + u * T, apply2<OP>(vb[u], vc[u], s));
  } else {
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + u * T;
      if (i < n2) {
        double2 vb = ld_stream(b2 + i);
        double2 vc = kC ? ld_stream(c2 + i) : vb;
        st_stream(a2 + i, apply2<OP>(vb, vc, s));
      }
    }
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

template <int OP, int T, int U>
void launch_tile_pdl(cudaStream_t st, double* a, const double* b, const double* c, double s,
                     uint64_t n) {
  uint64_t blocks = ((n >> 1) + (uint64_t)T * U - 1) / ((uint64_t)T * U);
  if (blocks == 0) blocks = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_stream_tile<OP, T, U, true>, a, b, c, s, n);
}

template <int OP>
cudaError_t launch(cudaStream_t st, int sms, double* a, const double* b, const double* c,
                   double s, uint64_t n) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                         reinterpret_cast<uintptr_t>(c)) & 15) == 0;
  if (!aligned) {
    uint64_t blocks = (n + kThreads - 1) / kThreads;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    k_stream_scalar<OP><<<(unsigned)(blocks ? blocks : 1), kThreads, 0, st>>>(a, b, c, s, n);
    return cudaPeekAtLastError();
  }
  // measured best on B200 (profiles/r01_stream_sweep.txt: 19 launch shapes,
  // grid-stride and TMA forms; the alternatives were removed): one-shot
  // tiles, 512 threads; 1 double2 per input per thread for the 2-input ops,
  // 2 for the 1-input ops; launched with programmatic dependent launch so
  // back-to-back launches overlap CTA scheduling with the previous drain
  if constexpr (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD)
    launch_tile_pdl<OP, 512, 1>(st, a, b, c, s, n);
  else
    launch_tile_pdl<OP, 512, 2>(st, a, b, c, s, n);
  return cudaPeekAtLastError();
}

}  // namespace

namespace ofl {
cudaError_t stream_launch(cudaStream_t st, int sms, int op, double* a, const double* b,
                          const double* c, double scalar, uint64_t n) {
  switch (op) {
    case OFL_STREAM_COPY: return launch<OFL_STREAM_COPY>(st, sms, a, b, c, scalar, n);
    case OFL_STREAM_SCALE: return launch<OFL_STREAM_SCALE>(st, sms, a, b, c, scalar, n);
    case OFL_STREAM_ADD: return launch<OFL_STREAM_ADD>(st, sms, a, b, c, scalar, n);
    default: return launch<OFL_STREAM_TRIAD>(st, sms, a, b, c, scalar, n);
  }
}
}  // namespace ofl

extern "C" int ofl_stream_op(ofl_stream* s, int op, double* a, const double* b, const double* c,
                             double scalar, uint64_t n, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (op < OFL_STREAM_COPY || op > OFL_STREAM_TRIAD)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "unknown STREAM op");
  if (!c) c = b;
  ofl::Enqueue q(s, "ofl:stream_op");
  if (!q.ok()) return q.status;
  if (n) {
    const cudaError_t e = ofl::stream_launch(s->cs, ofl::num_sms(s->dev), op, a, b, c, scalar, n);
    if (e != cudaSuccess) return ofl::cuda_error(e, "STREAM launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}
