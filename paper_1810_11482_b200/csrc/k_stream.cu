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
#include <cstdlib>

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

// Grid-stride form: a fixed grid of T-thread CTAs (MINB resident per SM)
// sweeps the vector; each thread keeps U 128-bit loads per input in flight.
template <int OP, int T, int U, int MINB>
__global__ void __launch_bounds__(T, MINB) k_stream_vec(double* __restrict__ a,
                                                       const double* __restrict__ b,
                                                       const double* __restrict__ c, double s,
                                                       uint64_t n) {
  constexpr bool kC = (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD);
  const uint64_t n2 = n >> 1;
  double2* __restrict__ a2 = reinterpret_cast<double2*>(a);
  const double2* __restrict__ b2 = reinterpret_cast<const double2*>(b);
  const double2* __restrict__ c2 = reinterpret_cast<const double2*>(c);
  const uint64_t stride = (uint64_t)gridDim.x * T;
  uint64_t i = (uint64_t)blockIdx.x * T + threadIdx.x;

  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 vb[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vb[u] = ld_stream(b2 + i + u * stride);
      if constexpr (kC) vc[u] = ld_stream(c2 + i + u * stride);
      else vc[u] = vb[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st_stream(a2 + i + u * stride, apply2<OP>(vb[u], vc[u], s));
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

// Tile form: one CTA per contiguous tile of T*U double2, no loop; the
// hardware block scheduler load-balances the (many) tiles.
template <int OP, int T, int U, bool kPDL = false>
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

// TMA (bulk-copy engine) form: one elected thread moves each input tile
// global->shared with cp.async.bulk completing on an mbarrier, the CTA
// computes in shared memory (in place over b), and the tile goes back with
// one shared->global bulk store.  Tiles of kTmaTile doubles per input.
constexpr int kTmaThreads = 256;
constexpr int kTmaTile = 2048;  // 16 KiB per input tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int OP, int TILE = kTmaTile>
__global__ void __launch_bounds__(kTmaThreads) k_stream_tma(double* __restrict__ a,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ c,
                                                          double s, uint64_t n) {
  constexpr bool kC = (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD);
  __shared__ alignas(128) double sb[TILE];
  __shared__ alignas(128) double sc[kC ? TILE : 1];
  __shared__ alignas(8) uint64_t bar;
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
  const uint64_t count = n - base < (uint64_t)TILE ? n - base : (uint64_t)TILE;
  const uint32_t bytes = (uint32_t)(count * 8) & ~15u;  // bulk sizes are 16-byte multiples
  const uint32_t bar_a = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                 "r"(kC ? 2 * bytes : bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(sb)), "l"(b + base), "r"(bytes), "r"(bar_a)
        : "memory");
    if constexpr (kC)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(sc)), "l"(c + base), "r"(bytes), "r"(bar_a)
          : "memory");
  }
  if (bytes) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar_a)
          : "memory");
  }
  const uint32_t m = bytes / 8;  // elements covered by the bulk copies
  for (uint32_t i = threadIdx.x; i < m; i += kTmaThreads)
    sb[i] = apply<OP>(sb[i], kC ? sc[i] : 0.0, s);
  for (uint64_t i = base + m + threadIdx.x; i < base + count; i += kTmaThreads)
    a[i] = apply<OP>(b[i], kC ? c[i] : 0.0, s);  // < 2 leftover elements
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a + base),
                 "r"(smem_u32(sb)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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

template <int OP, int T, int U, int MINB>
void launch_vec(cudaStream_t st, int sms, int per_sm, double* a, const double* b,
                const double* c, double s, uint64_t n) {
  uint64_t blocks = ((n >> 1) + (uint64_t)T * U - 1) / ((uint64_t)T * U);
  const uint64_t cap = (uint64_t)sms * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  k_stream_vec<OP, T, U, MINB><<<(unsigned)blocks, T, 0, st>>>(a, b, c, s, n);
}

template <int OP, int T, int U>
void launch_tile(cudaStream_t st, double* a, const double* b, const double* c, double s,
                 uint64_t n) {
  uint64_t blocks = ((n >> 1) + (uint64_t)T * U - 1) / ((uint64_t)T * U);
  if (blocks == 0) blocks = 1;
  k_stream_tile<OP, T, U><<<(unsigned)blocks, T, 0, st>>>(a, b, c, s, n);
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

// Launch-shape variants (OFL_STREAM_VARIANT, for tuning sweeps); the default
// is the one measured fastest on B200 (profiles/).
int stream_variant() {
  static int v = [] {
    const char* e = getenv("OFL_STREAM_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
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
  switch (stream_variant()) {
    case 1: launch_vec<OP, 256, 4, 4>(st, sms, 4, a, b, c, s, n); break;
    case 2: launch_vec<OP, 256, 2, 8>(st, sms, 8, a, b, c, s, n); break;
    case 3: launch_vec<OP, 512, 4, 2>(st, sms, 2, a, b, c, s, n); break;
    case 4: launch_vec<OP, 128, 8, 8>(st, sms, 8, a, b, c, s, n); break;
    case 5: launch_tile<OP, 256, 4>(st, a, b, c, s, n); break;
    case 6: launch_tile<OP, 256, 2>(st, a, b, c, s, n); break;
    case 7: launch_tile<OP, 128, 8>(st, a, b, c, s, n); break;
    case 8: launch_vec<OP, 256, 8, 2>(st, sms, 4, a, b, c, s, n); break;
    case 9: launch_vec<OP, kThreads, kUnroll, 1>(st, sms, 8, a, b, c, s, n); break;
    case 10: launch_tile<OP, 256, 1>(st, a, b, c, s, n); break;
    case 11: launch_tile<OP, 512, 1>(st, a, b, c, s, n); break;
    case 12: launch_tile<OP, 512, 2>(st, a, b, c, s, n); break;
    case 13: launch_tile<OP, 1024, 1>(st, a, b, c, s, n); break;
    case 14: launch_tile<OP, 128, 4>(st, a, b, c, s, n); break;
    case 15: launch_tile<OP, 128, 2>(st, a, b, c, s, n); break;
    case 16: {
      const uint64_t blocks = (n + 2047) / 2048;
      k_stream_tma<OP, 2048><<<(unsigned)(blocks ? blocks : 1), kTmaThreads, 0, st>>>(a, b, c, s, n);
      break;
    }
    case 18:
      if constexpr (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD)
        launch_tile_pdl<OP, 512, 1>(st, a, b, c, s, n);
      else
        launch_tile_pdl<OP, 512, 2>(st, a, b, c, s, n);
      break;
    case 17: {
      const uint64_t blocks = (n + 1023) / 1024;
      k_stream_tma<OP, 1024><<<(unsigned)(blocks ? blocks : 1), kTmaThreads, 0, st>>>(a, b, c, s, n);
      break;
    }
    case 19:  // the default shape without programmatic dependent launch
      if constexpr (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD)
        launch_tile<OP, 512, 1>(st, a, b, c, s, n);
      else
        launch_tile<OP, 512, 2>(st, a, b, c, s, n);
      break;
    default:
      // measured best on B200 (profiles/r01_stream_sweep.txt): one-shot tiles,
      // 512 threads; 1 double2 per input per thread for the 2-input ops,
      // 2 for the 1-input ops; launched with programmatic dependent launch so
      // back-to-back launches overlap CTA scheduling with the previous drain
      if constexpr (OP == OFL_STREAM_ADD || OP == OFL_STREAM_TRIAD)
        launch_tile_pdl<OP, 512, 1>(st, a, b, c, s, n);
      else
        launch_tile_pdl<OP, 512, 2>(st, a, b, c, s, n);
      break;
  }
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
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  if (n) {
    const cudaError_t e = ofl::stream_launch(s->cs, ofl::num_sms(s->dev), op, a, b, c, scalar, n);
    if (e != cudaSuccess) return ofl::cuda_error(e, "STREAM launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}
