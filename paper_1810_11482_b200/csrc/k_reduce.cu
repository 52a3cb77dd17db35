// Reductions: u32 wrap-around sum (sum.k, /root/reference/pkg/src/offloadrt/
// bench/kernels/sum.k:3-11; oracle harness.py:129-130) and the fp32 dot
// product with fp64 accumulation (BASELINE config 4; no reference kernel —
// the language has no f32, kernel/lang.py:29).
//
// One kernel per reduction: vectorised 128-bit loads, per-thread partials,
// warp shuffle tree, block tree in shared memory, one partial per CTA to a
// per-stream scratch array, and the last CTA to finish (threadfence +
// atomic ticket) folds the partials in CTA order and writes res[0].
//   - u32 addition mod 2^32 is associative and commutative, so the parallel
//     order gives exactly the sequential result (bit-exact).
//   - fp64 partials are folded in a fixed order for a given grid, so the dot
//     result is run-to-run deterministic; each fp32*fp32 product is exact in
//     fp64, only the accumulation rounds.
#include <cstdlib>

#include "ofl_internal.h"

namespace {

constexpr int kThreads = 512;
constexpr int kMaxBlocks = 148 * 4;
constexpr int kSumCtasPerSm = 3;
constexpr int kDotCtasPerSm = 2;

// Lives at kScratchOffset of the per-stream scratch (the Mandelbrot work
// queue uses offset 32768); `partial` has one slot per CTA of the launch.
constexpr size_t kScratchOffset = 65536;
struct Scratch {
  unsigned int counter;
  unsigned int pad[63];
  uint64_t partial[1];  // u32 sums or fp64 bit patterns, gridDim.x of them
};

size_t scratch_bytes(uint64_t blocks) { return kScratchOffset + 256 + 8 * blocks; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v) {
  __shared__ T red[kThreads / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = 0;
  if (w == 0) {
    r = (l < kThreads / 32) ? red[l] : T(0);
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// Last-CTA fold; returns true in thread 0 of the final CTA with the total.
template <typename T>
__device__ __forceinline__ bool fold(Scratch* sc, T mine, T* total) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    sc->partial[blockIdx.x] = *reinterpret_cast<uint64_t*>(&mine);
    __threadfence();
    const unsigned int done = atomicAdd(&sc->counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // fixed-order fold: each thread strides the partials, then a block tree
  T acc = 0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += kThreads) {
    uint64_t bits = *reinterpret_cast<volatile uint64_t*>(&sc->partial[b]);
    acc += *reinterpret_cast<T*>(&bits);
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    *total = acc;
    sc->counter = 0;  // ready for the next launch on this stream
  }
  return threadIdx.x == 0;
}

__global__ void __launch_bounds__(kThreads) k_sum_u32(const uint32_t* __restrict__ in,
                                                      uint32_t* __restrict__ res, uint64_t n,
                                                      Scratch* sc) {
  const uint64_t n4 = n >> 2;
  const uint4* in4 = reinterpret_cast<const uint4*>(in);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const uint4 v0 = __ldcs(in4 + i), v1 = __ldcs(in4 + i + stride);
    const uint4 v2 = __ldcs(in4 + i + 2 * stride), v3 = __ldcs(in4 + i + 3 * stride);
    a0 += v0.x + v0.y + v0.z + v0.w;
    a1 += v1.x + v1.y + v1.z + v1.w;
    a2 += v2.x + v2.y + v2.z + v2.w;
    a3 += v3.x + v3.y + v3.z + v3.w;
  }
  for (; i < n4; i += stride) {
    const uint4 v = __ldcs(in4 + i);
    a0 += v.x + v.y + v.z + v.w;
  }
  uint32_t acc = a0 + a1 + a2 + a3;
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) acc += in[(n & ~3ull) + threadIdx.x];
  acc = block_sum(acc);
  uint32_t total;
  if (fold<uint32_t>(sc, acc, &total)) res[0] = total;
}

// Exchange block of one rank for the fused dot + allreduce (ofl_dot_f32_allreduce),
// in that rank's device memory and written by every rank over NVLink.
struct Xchg {
  unsigned long long arrivals;  // monotonically counts partials received
  unsigned long long status;    // non-zero: a rank gave up waiting (timeout)
  double slot[2][OFL_MAX_PEER_RANKS];  // [round parity][rank]
};

struct PeerReduce {
  Xchg* peers[OFL_MAX_PEER_RANKS];  // every rank's block (peer pointers)
  int rank, nranks;
  unsigned long long round;  // 0, 1, 2, ... per call on this group
};

// Last CTA of rank `rank`: publish the partial to every rank, then wait for
// all partials of this round and sum them in rank order (identical bits on
// every rank).  Bounded wait: after ~20 s the rank records a timeout.
__device__ void peer_allreduce(const PeerReduce& pr, double partial, double* res) {
  const int par = (int)(pr.round & 1);
  for (int r = 0; r < pr.nranks; ++r)
    *reinterpret_cast<volatile double*>(&pr.peers[r]->slot[par][pr.rank]) = partial;
  __threadfence_system();
  for (int r = 0; r < pr.nranks; ++r) atomicAdd_system(&pr.peers[r]->arrivals, 1ull);
  Xchg* mine = pr.peers[pr.rank];
  const unsigned long long target = (pr.round + 1) * (unsigned long long)pr.nranks;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*reinterpret_cast<volatile unsigned long long*>(&mine->arrivals) < target) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20ull * 1000 * 1000 * 1000) {
      mine->status = 1;
      res[0] = __longlong_as_double(0x7ff8000000000000ll);
      return;
    }
    __nanosleep(200);
  }
  __threadfence_system();
  double total = 0.0;
  for (int r = 0; r < pr.nranks; ++r)
    total += *reinterpret_cast<volatile double*>(&mine->slot[par][r]);
  res[0] = total;
}

template <bool kPeer = false>
__global__ void __launch_bounds__(kThreads) k_dot_f32(const float* __restrict__ a,
                                                      const float* __restrict__ b,
                                                      double* __restrict__ res, uint64_t n,
                                                      Scratch* sc, PeerReduce pr = PeerReduce{}) {
  const uint64_t n4 = n >> 2;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  double s0 = 0.0, s1 = 0.0;
  for (; i + stride < n4; i += 2 * stride) {
    const float4 x0 = __ldcs(a4 + i), y0 = __ldcs(b4 + i);
    const float4 x1 = __ldcs(a4 + i + stride), y1 = __ldcs(b4 + i + stride);
    // fp32*fp32 is exact in fp64, so fma == add(product)
    s0 = fma((double)x0.x, (double)y0.x, s0);
    s0 = fma((double)x0.y, (double)y0.y, s0);
    s0 = fma((double)x0.z, (double)y0.z, s0);
    s0 = fma((double)x0.w, (double)y0.w, s0);
    s1 = fma((double)x1.x, (double)y1.x, s1);
    s1 = fma((double)x1.y, (double)y1.y, s1);
    s1 = fma((double)x1.z, (double)y1.z, s1);
    s1 = fma((double)x1.w, (double)y1.w, s1);
  }
  for (; i < n4; i += stride) {
    const float4 x = __ldcs(a4 + i), y = __ldcs(b4 + i);
    s0 = fma((double)x.x, (double)y.x, s0);
    s0 = fma((double)x.y, (double)y.y, s0);
    s0 = fma((double)x.z, (double)y.z, s0);
    s0 = fma((double)x.w, (double)y.w, s0);
  }
  double acc = s0 + s1;
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const uint64_t j = (n & ~3ull) + threadIdx.x;
    acc = fma((double)a[j], (double)b[j], acc);
  }
  acc = block_sum(acc);
  double total;
  if (fold<double>(sc, acc, &total)) {
    if (kPeer) peer_allreduce(pr, total, res);
    else res[0] = total;
  }
}

// Grid: persistent, `cps` CTAs of 512 threads per SM with a grid-stride
// loop.  A one-shot grid (one unrolled round per thread) measured slower on
// B200 — 0.198 vs 0.167 ms for sum 2^28, 3.46 vs 2.60 ms for dot 2^31
// (profiles/r01_reduce_grid.txt): the per-CTA atomic ticket and the last
// CTA's fold over ~10^5 partials cost more than the tail it balances.  CTAs
// per SM per kernel from the read-bandwidth sweep (scripts/probes/
// read_bw_probe.cu, scripts/reduce_sweep.sh).
int grid_for(ofl_stream* s, uint64_t vec_units, int unroll, int cps) {
  uint64_t blocks = (vec_units + (uint64_t)kThreads * unroll - 1) / ((uint64_t)kThreads * unroll);
  uint64_t cap = (uint64_t)ofl::num_sms(s->dev) * cps;
  if (cap > kMaxBlocks) cap = kMaxBlocks;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return (int)blocks;
}

Scratch* reduce_scratch(void* base) {
  return reinterpret_cast<Scratch*>(static_cast<char*>(base) + kScratchOffset);
}

}  // namespace

extern "C" int ofl_sum_u32(ofl_stream* s, const uint32_t* in, uint32_t* res, uint64_t n,
                           uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (reinterpret_cast<uintptr_t>(in) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "sum input must be 16-byte aligned");
  ofl::Enqueue q(s, "ofl:sum_u32");
  if (!q.ok()) return q.status;
  const int blocks = grid_for(s, n >> 2, 4, kSumCtasPerSm);
  void* scratch = nullptr;
  int st = ofl::stream_scratch(s, scratch_bytes(blocks), &scratch);
  if (st) return st;
  k_sum_u32<<<blocks, kThreads, 0, s->cs>>>(in, res, n, reduce_scratch(scratch));
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ofl::cuda_error(e, "sum launch");
  ofl::count_launch();
  return q.finish(ticket);
}

extern "C" int ofl_dot_f32(ofl_stream* s, const float* a, const float* b, double* res,
                           uint64_t n, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "dot operands must be 16-byte aligned");
  ofl::Enqueue q(s, "ofl:dot_f32");
  if (!q.ok()) return q.status;
  const int blocks = grid_for(s, n >> 2, 2, kDotCtasPerSm);
  void* scratch = nullptr;
  int st = ofl::stream_scratch(s, scratch_bytes(blocks), &scratch);
  if (st) return st;
  k_dot_f32<<<blocks, kThreads, 0, s->cs>>>(a, b, res, n, reduce_scratch(scratch));
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ofl::cuda_error(e, "dot launch");
  ofl::count_launch();
  return q.finish(ticket);
}

extern "C" int ofl_xchg_bytes(void) { return (int)sizeof(Xchg); }

extern "C" int ofl_dot_f32_allreduce(ofl_stream* s, const float* a, const float* b, double* res,
                                     uint64_t n, int rank, int nranks, void* const* xchg,
                                     const int* devs, uint64_t round, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "dot operands must be 16-byte aligned");
  if (nranks < 1 || nranks > OFL_MAX_PEER_RANKS || rank < 0 || rank >= nranks)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "dot allreduce: bad rank / group size");
  PeerReduce pr{};
  for (int r = 0; r < nranks; ++r) {
    if (!xchg[r]) return ofl::set_error(OFL_ERR_BAD_ARGS, "dot allreduce: missing exchange block");
    pr.peers[r] = static_cast<Xchg*>(xchg[r]);
    if (devs[r] != s->dev) ofl::enable_peer(s->dev, devs[r]);
  }
  pr.rank = rank;
  pr.nranks = nranks;
  pr.round = round;
  ofl::Enqueue q(s, "ofl:dot_f32_allreduce");
  if (!q.ok()) return q.status;
  const int blocks = grid_for(s, n >> 2, 2, kDotCtasPerSm);
  void* scratch = nullptr;
  int st = ofl::stream_scratch(s, scratch_bytes(blocks), &scratch);
  if (st) return st;
  k_dot_f32<true><<<blocks, kThreads, 0, s->cs>>>(a, b, res, n, reduce_scratch(scratch), pr);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ofl::cuda_error(e, "dot allreduce launch");
  ofl::count_launch();
  return q.finish(ticket);
}
