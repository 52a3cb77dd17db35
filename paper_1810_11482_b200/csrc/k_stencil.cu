// 1-D 3-point stencil (stencil.k, /root/reference/pkg/src/offloadrt/bench/
// kernels/stencil.k:2-10) and its iteration as a heat equation (BASELINE
// config 2).
//
//   y[i] = x[i]                                   i == 0 or i == n-1
//   y[i] = (0.5*x[i-1] + x[i]) + 0.5*x[i+1]       otherwise
//
// evaluated left to right with round-to-nearest and no contraction, exactly
// the reference executor's order (kernel/codegen.py:241-289: every binary
// operation is a separate IEEE operation).  Items are independent, so the
// parallel order is free.
//
// Single step (k_stencil_smem): each thread owns aligned pairs of cells
// loaded as 128-bit vectors and staged in shared memory with the two cells
// just outside the CTA's range, so every cell is read from HBM once: 16 B/cell.
//
// Temporal blocking (k_heat_pipe, below): a warp holds a tile of cells plus
// a halo of `tb` cells each side in registers, advances it `tb` steps (the
// valid region shrinks by one cell per side per step), and writes the
// centre back: 16 B/cell per `tb` steps instead of per step.  Global
// endpoints are fixed points of the update, exactly as stencil.k.


#include "ofl_internal.h"

namespace {


// read-only, L1-bypassing 128-bit load (as the STREAM kernels)
__device__ __forceinline__ double2 ld_nc(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

__device__ __forceinline__ double point(double l, double c, double r) {
  return __dadd_rn(__dadd_rn(__dmul_rn(0.5, l), c), __dmul_rn(0.5, r));
}

// m  = number of items that execute (min(n, grid*block of the .k launch))
// hi = highest readable x index = min(m, n-1)
// Shared-memory form: the CTA's U*T pairs are staged once in shared memory
// with the two cells just outside the CTA's range (loaded by threads 0 and
// T-1), so each cell's outer neighbours come from shared memory instead of a
// warp-edge load per warp: 2 extra loads per 2*U*T cells instead of 2 per
// 64 — the per-warp edge loads cost the shuffle form ~13% against a copy.
template <int T, int U, bool kPDL>
__global__ void __launch_bounds__(T) k_stencil_smem(const double* __restrict__ x,
                                                    double* __restrict__ y, uint64_t n,
                                                    uint64_t m) {
  if constexpr (kPDL) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  constexpr int kCells = 2 * T * U;
  __shared__ double tile[kCells + 2];  // tile[1 + i] = x[c0 + i]
  const uint64_t hi = (m < n - 1) ? m : n - 1;  // highest readable index
  const uint64_t c0 = (uint64_t)blockIdx.x * kCells;
  double2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t j = c0 / 2 + (uint64_t)u * T + threadIdx.x;
    const uint64_t lo = 2 * j;
    v[u] = make_double2(0.0, 0.0);
    if (lo + 1 <= hi) v[u] = ld_nc(reinterpret_cast<const double2*>(x) + j);
    else if (lo <= hi) v[u].x = x[lo];
  }
  if (threadIdx.x == 0) tile[0] = (c0 >= 1 && c0 - 1 <= hi) ? x[c0 - 1] : 0.0;
  if (threadIdx.x == T - 1) tile[kCells + 1] = (c0 + kCells <= hi) ? x[c0 + kCells] : 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = 2 * (u * T + threadIdx.x);
    tile[1 + i] = v[u].x;
    tile[2 + i] = v[u].y;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = 2 * (u * T + threadIdx.x);
    const uint64_t lo = c0 + i;
    if (lo < m) {
      const double left = tile[i], right = tile[i + 3];
      const double r0 = (lo == 0 || lo == n - 1) ? v[u].x : point(left, v[u].x, v[u].y);
      if (lo + 1 < m) {
        const double r1 = (lo + 1 == n - 1) ? v[u].y : point(v[u].x, v[u].y, right);
        __stcs(reinterpret_cast<double2*>(y + lo), make_double2(r0, r1));
      } else {
        y[lo] = r0;
      }
    }
  }
}

template <int T, int U>
void launch_stencil_smem(cudaStream_t cs, const double* x, double* y, uint64_t n, uint64_t m) {
  const uint64_t cells = 2ull * T * U;
  const unsigned blocks = (unsigned)((m + cells - 1) / cells);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(T);
  cfg.stream = cs;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_stencil_smem<T, U, true>, x, y, n, m);
}

// One stencil step, the shape measured fastest on B200 (2^28 cells back to
// back: 621 us/step, 6.91 TB/s = copy speed; the warp-shuffle form with
// per-warp edge loads and other launch shapes measured 630-786 us and were
// removed, profiles/r01_stencil_ncu.txt).
void launch_stencil(cudaStream_t cs, const double* x, double* y, uint64_t n, uint64_t m) {
  launch_stencil_smem<256, 4>(cs, x, y, n, m);
}

// ---------------------------------------------------------------- heat ---
// T steps of stencil.k (BASELINE config 2) in passes of up to tb steps; a
// pass keeps each tile in registers for all its steps, so HBM sees 16 B per
// cell per pass instead of per step and the FP64 pipe is the bound.  Earlier
// forms (shared-memory tiles, CTA register tiles with a barrier per step,
// two-level warp ghosts, one tile per warp; profiles/r01_heat_sweep.txt,
// r02_heat_sweep.txt) were removed once this one beat them.
// Warp tiles: every warp owns its own tile of 32*R consecutive cells (R per
// lane, in registers) including a halo of tb cells each side that is
// computed redundantly, so a step needs two shuffles and no barrier at all;
// per-thread ILP (R independent cells) hides the FP64 latency.
constexpr int kWarpThreads = 128;

// Fused form of point(): when 0.5*l and 0.5*r are exact (no result below
// 2^-1022), round(0.5*l + c) is exactly __dadd_rn(__dmul_rn(0.5, l), c), so
//   (0.5*l + c) + 0.5*r  ==  fma(0.5, r, fma(0.5, l, c))      bit for bit
// — two DFMA instead of DMUL + 2 DADD (3 after CSE).  Only valid under the
// tile guard (warp_tile_steps).
__device__ __forceinline__ double point_fma(double l, double c, double r) {
  return __fma_rn(0.5, r, __fma_rn(0.5, l, c));
}

// One step of a warp tile.  kEdge: some lane holds global cell 0 or n-1
// (held fixed), decided warp-uniformly so the common case has no per-step
// test.  kClamp: lanes 0 / 31 use their own edge cell as the outer
// neighbour; without it they read an arbitrary finite-or-not value, which
// is harmless: garbage enters at the tile ends and moves one cell per step,
// so after tb steps it has reached only the tb-cell halo that is never
// written back (the valid cells' dependency cones lie inside the tile).
template <int R, bool kFma, bool kEdge, bool kClamp = false>
__device__ __forceinline__ void warp_step(const double (&in)[R], double (&out)[R], int lane,
                                          int64_t g0, int64_t nn) {
  double left = __shfl_up_sync(0xffffffffu, in[R - 1], 1);
  double right = __shfl_down_sync(0xffffffffu, in[0], 1);
  if (kClamp) {
    if (lane == 0) left = in[0];
    if (lane == 31) right = in[R - 1];
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const double l = i > 0 ? in[i - 1] : left;
    const double r = i + 1 < R ? in[i + 1] : right;
    out[i] = kFma ? point_fma(l, in[i], r) : point(l, in[i], r);
  }
  if (kEdge) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t g = g0 + i;
      if (g <= 0 || g >= nn - 1) out[i] = in[i];
    }
  }
}

template <int R, bool kFma, bool kEdge>
__device__ __forceinline__ bool warp_steps(double (&a)[R], double (&b)[R], int lane, int64_t g0,
                                           int64_t nn, int tb) {
  int s = 0;
  for (; s + 1 < tb; s += 2) {
    warp_step<R, kFma, kEdge>(a, b, lane, g0, nn);
    warp_step<R, kFma, kEdge>(b, a, lane, g0, nn);
  }
  if (s < tb) warp_step<R, kFma, kEdge>(a, b, lane, g0, nn);
  return s < tb;
}

// tb steps of a warp tile held in registers (a -> a or b; returns true when
// the result is in b).  Tile guard for the fused update: every cell is +0 or
// a positive number >= 2^(tb-1020) (inf/nan included).  With non-negative
// inputs a cell never decreases and a new non-zero is at least half a
// non-zero neighbour, so over tb steps every operand stays >= 2^-1020 or
// zero and 0.5*x is exact.  Otherwise (signs, -0, tiny values) the warp takes
// the unfused path.  The guard is warp-uniform (__all_sync).
template <int R>
__device__ __forceinline__ bool warp_tile_steps(double (&a)[R], double (&b)[R], int lane,
                                                bool edge, int64_t g0, int64_t nn, int tb,
                                                bool fma_ok) {
  bool safe = fma_ok;
  if (safe) {
    const uint64_t lo_bits = (uint64_t)(tb + 3) << 52;  // 2^(tb-1020)
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t u = (uint64_t)__double_as_longlong(a[i]);
      safe &= (u == 0) || (u >= lo_bits && u < 0x8000000000000000ull);
    }
  }
  safe = __all_sync(0xffffffffu, safe);
  if (__any_sync(0xffffffffu, edge))
    return safe ? warp_steps<R, true, true>(a, b, lane, g0, nn, tb)
                : warp_steps<R, false, true>(a, b, lane, g0, nn, tb);
  return safe ? warp_steps<R, true, false>(a, b, lane, g0, nn, tb)
              : warp_steps<R, false, false>(a, b, lane, g0, nn, tb);
}

// Where a slab pass (ofl_heat_slab) puts its results: only the owned cells
// [own_lo, own_hi) of y, plus the first / last h owned cells straight into
// the neighbouring slabs' ghost cells (left / right, usually on peer GPUs:
// the stores travel over NVLink from this kernel, no separate copy).
struct SlabOut {
  int64_t own_lo, own_hi, h;
  double* left;   // receives y[own_lo, own_lo + h), or null
  double* right;  // receives y[own_hi - h, own_hi), or null
};

// Cells per lane of the windows the general path advances (below): 32*kSlowR
// cells fit two register arrays without spilling, and exceed 2*tb (tb <= 128).
constexpr int kSlowR = 32;

// tb steps of one window of 32*RS consecutive cells starting at w0 >= 0, in
// registers (lane l holds cells w0 + l*RS ...); cells [vlo, vhi) are stored.
// A window flush with the field's start (w0 == 0) holds global cell 0 at
// lane 0 / index 0, one flush with its end holds cell n-1 at lane 31 /
// index RS-1: those cells are put back after every step (one predicated move,
// no per-cell edge test), and since a fixed cell never reads its outer
// neighbour, nothing beyond it matters.  Only a field shorter than the window
// takes the per-cell edge test (cells past n-1 are zeros nobody reads).
template <int RS, bool kSlab>
__device__ __noinline__ void heat_window(const double* __restrict__ x, double* __restrict__ y,
                                         int64_t nn, int tb, bool fma_ok, int64_t w0, int64_t vlo,
                                         int64_t vhi, int lane, int64_t own_lo, int64_t own_hi,
                                         int64_t h, double* left, double* right) {
  constexpr int64_t kW = 32 * RS;
  const int64_t g0 = w0 + (int64_t)lane * RS;
  double a[RS], b[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) a[i] = g0 + i < nn ? __ldg(x + g0 + i) : 0.0;
  bool fused = fma_ok;
  if (fused) {
    const uint64_t lo_bits = (uint64_t)(tb + 3) << 52;  // 2^(tb-1020), see warp_tile_steps
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const uint64_t u = (uint64_t)__double_as_longlong(a[i]);
      fused &= (u == 0) || (u >= lo_bits && u < 0x8000000000000000ull);
    }
  }
  fused = __all_sync(0xffffffffu, fused);
  bool odd;
  if (w0 + kW > nn) {  // the whole field inside one window
    odd = fused ? warp_steps<RS, true, true>(a, b, lane, g0, nn, tb)
                : warp_steps<RS, false, true>(a, b, lane, g0, nn, tb);
  } else {
    const bool fix_lo = w0 == 0 && lane == 0;
    const bool fix_hi = w0 + kW == nn && lane == 31;
    int st = 0;
    for (; st + 1 < tb; st += 2) {
      if (fused) {
        warp_step<RS, true, false>(a, b, lane, g0, nn);
      } else {
        warp_step<RS, false, false>(a, b, lane, g0, nn);
      }
      if (fix_lo) b[0] = a[0];
      if (fix_hi) b[RS - 1] = a[RS - 1];
      if (fused) {
        warp_step<RS, true, false>(b, a, lane, g0, nn);
      } else {
        warp_step<RS, false, false>(b, a, lane, g0, nn);
      }
      if (fix_lo) a[0] = b[0];
      if (fix_hi) a[RS - 1] = b[RS - 1];
    }
    odd = st < tb;
    if (odd) {
      if (fused) {
        warp_step<RS, true, false>(a, b, lane, g0, nn);
      } else {
        warp_step<RS, false, false>(a, b, lane, g0, nn);
      }
      if (fix_lo) b[0] = a[0];
      if (fix_hi) b[RS - 1] = a[RS - 1];
    }
  }
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    const int64_t g = g0 + i;
    if (g >= vlo && g < vhi) {
      const double v = odd ? b[i] : a[i];
      if (!kSlab) {
        y[g] = v;
      } else if (g >= own_lo && g < own_hi) {
        y[g] = v;
        if (left && g < own_lo + h) left[g - own_lo] = v;
        if (right && g >= own_hi - h) right[g - (own_hi - h)] = v;
      }
    }
  }
}

// The general path for a whole tile (cells [c_lo, c_hi) after tb steps):
// tiles at the field's ends, overhanging it, or (slab passes) reaching the
// strips sent to the neighbours.  The range is covered by windows of
// 32*kSlowR cells — flush with cell 0 / n-1 where the tile touches them,
// else with tb halo cells each side — so the general path never holds a
// 32*R-cell tile in registers (which spilled and made these few tiles the
// critical path of a short pass: a ~0.3 ms floor per pass).
template <int R, bool kSlab>
__device__ __forceinline__ void heat_tile_slow(const double* __restrict__ x, double* __restrict__ y,
                                               int64_t nn, int tb, bool fma_ok, int64_t c_lo,
                                               int64_t c_hi, int lane, int64_t own_lo,
                                               int64_t own_hi, int64_t h, double* left,
                                               double* right) {
  constexpr int64_t kW = 32 * kSlowR;
  int64_t pos = c_lo;
  while (pos < c_hi) {
    int64_t w0, end;
    if (nn <= kW || pos <= tb) {  // flush with cell 0 (or the field is one window)
      w0 = 0;
      end = nn <= kW ? nn : kW - tb;
    } else if (pos - tb + kW >= nn) {  // flush with cell n-1
      w0 = nn - kW;
      end = nn;
    } else {
      w0 = pos - tb;
      end = pos + kW - 2 * tb;
    }
    const int64_t hi = end < c_hi ? end : c_hi;
    heat_window<kSlowR, kSlab>(x, y, nn, tb, fma_ok, w0, pos, hi, lane, own_lo, own_hi, h, left,
                               right);
    pos = hi;
  }
}

// Persistent warps with the tiles moved by the bulk-copy engine (TMA).
// Every warp owns one shared-memory tile buffer (32R+2 doubles) and an
// mbarrier, and walks its tiles t = warp, warp + W, ...:
//   * the NEXT tile's cells are prefetched into the buffer by one
//     cp.async.bulk while the current tile is advanced in registers, so the
//     HBM load overlaps the FP64 work instead of every warp of an SM loading
//     at the same moment (one-tile-per-warp grids run in lock step: all
//     warps load, then all compute, and the FP64 pipe idles ~16% of a pass);
//   * at the end of a tile each lane swaps its R results with its R cells of
//     the prefetched tile (registers <-> shared memory), and the valid centre
//     goes back to HBM with one cp.async.bulk store, read out of the buffer
//     before the following prefetch overwrites it;
//   * global loads and stores are whole contiguous tiles (the register
//     layout, R consecutive cells per lane, would make them 32-way strided).
// Tiles touching global cell 0 or n-1, or reaching past n, and tiles that
// fail the fused-update guard run heat_tile_slow (global loads/stores).
// Alignment: a tile's load starts at the even index lo & ~1 and spans 32R+2
// cells; the valid centre starts at the even index t*valid (valid = 32R-2tb)
// and sits at the even buffer offset tb + (tb & 1): both 16-byte aligned.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const double* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

template <int R>
__host__ __device__ constexpr int heat_pipe_buf() {  // doubles per warp buffer (16-byte multiple)
  return 32 * R + 2;
}

// cells per lane of the production heat pass (odd: conflict-free 8-byte
// shared-memory accesses at a lane stride of R doubles)
constexpr int kHeatPipeR = 99;

template <int R>
constexpr int heat_pipe_min_blocks() {
  return R <= 63 ? 3 : 2;
}

// Tiles are handed out by an atomic counter (grabbed one tile ahead, so
// the prefetch can start): the few tiles the pipeline cannot take — those
// holding global cell 0 or n-1 or reaching past n-1 — come first and run
// the general path before the pipelined loop, so no call sits inside the
// loop (its live values would be spilled) and the warps that took them
// simply grab fewer tiles later.  The counter is reset once per heat call;
// pass p of a call reads it relative to `base` (every pass hands out
// exactly ntiles + warps values: each warp stops at its first index past
// the end).
template <int R, bool kSlab = false>
__global__ void __launch_bounds__(kWarpThreads, heat_pipe_min_blocks<R>())
    k_heat_pipe(const double* __restrict__ x, double* __restrict__ y, uint64_t n, int tb,
                bool fma_ok, unsigned long long* ctr, unsigned long long base,
                SlabOut so = SlabOut{}) {
  constexpr int kCells = 32 * R;
  constexpr int kBuf = heat_pipe_buf<R>();
  constexpr int kWarps = kWarpThreads / 32;
  extern __shared__ __align__(128) double heat_smem[];
  __shared__ __align__(8) uint64_t bars[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* buf = heat_smem + warp * kBuf;
  const uint32_t buf_a = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&bars[warp]));
  const int64_t nn = (int64_t)n;
  const int64_t valid = kCells - 2 * tb;
  const int64_t ntiles = (nn + valid - 1) / valid;
  // eligible tiles are [t_lo, t_hi]: lo = t*valid - tb >= 1, the aligned
  // load range [lo & ~1, (lo & ~1) + kBuf) ends at or before n-1, and (slab
  // passes) the stored centre lies inside the owned cells minus the strips
  // that go to the neighbours' ghost cells
  const int64_t own_lo = kSlab ? so.own_lo + (so.left ? so.h : 0) : 0;
  const int64_t own_hi = kSlab ? so.own_hi - (so.right ? so.h : 0) : nn;
  int64_t t_lo = (tb + 1 + valid - 1) / valid;
  if (kSlab && t_lo * valid < own_lo) t_lo = (own_lo + valid - 1) / valid;
  int64_t t_hi = (nn - 1 - kBuf + tb + 1) / valid;  // (lo & ~1) <= lo <= lo+1
  if (t_hi > ntiles - 1) t_hi = ntiles - 1;
  while (t_hi >= 0 && (((t_hi * valid - tb) & ~(int64_t)1) + kBuf > nn - 1 ||
                       (kSlab && t_hi * valid + valid > own_hi)))
    --t_hi;
  const int64_t n_elig = t_hi >= t_lo ? t_hi - t_lo + 1 : 0;
  const int64_t n_edge = ntiles - n_elig;  // handed out first
  // hand-out order: tiles [0, t_lo), then (t_hi, ntiles), then [t_lo, t_hi]
  auto tile_of = [&](int64_t k) -> int64_t {
    if (n_elig == 0) return k;
    if (k < n_edge) return k < t_lo ? k : t_hi + 1 + (k - t_lo);
    return t_lo + (k - n_edge);
  };
  auto grab = [&]() -> int64_t {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1ull) - base;
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  // valid is even, so every tile's first cell t*valid - tb has the parity
  // of tb: one buffer offset d for all tiles
  const int d = tb & 1;
  auto prefetch = [&](int64_t tile) {  // lane 0 only
    const int64_t lo_al = (tile * valid - tb) & ~(int64_t)1;
    bulk_load(buf_a, x + lo_al, kBuf * 8u, bar);
  };
  int64_t k = grab();
  while (k < n_edge) {  // edge / overhanging tiles: general path, global memory
    const int64_t te = tile_of(k);
    heat_tile_slow<R, kSlab>(x, y, nn, tb, fma_ok, te * valid,
                             te * valid + valid < nn ? te * valid + valid : nn, lane,
                             so.own_lo, so.own_hi, so.h, so.left, so.right);
    k = grab();
  }
  if (k >= ntiles) return;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  double a[R], b[R];
  int64_t t = tile_of(k);
  if (lane == 0) prefetch(t);
  mbar_wait(bar, phase);
  phase ^= 1;
#pragma unroll
  for (int i = 0; i < R; ++i) a[i] = buf[lane * R + d + i];
  bool store_pending = false;  // lane 0's bulk store may still be reading the buffer
  while (true) {
    const int64_t kn = grab();
    const bool next = kn < ntiles;
    const int64_t tn = next ? tile_of(kn) : 0;
    // the buffer is free once every lane has read the current tile out of
    // it and the previous bulk store has read its results
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0 && store_pending) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    if (next && lane == 0) prefetch(tn);
    bool fused = fma_ok;
    if (fused) {
      const uint64_t lo_bits = (uint64_t)(tb + 3) << 52;  // 2^(tb-1020), see warp_tile_steps
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint64_t u = (uint64_t)__double_as_longlong(a[i]);
        fused &= (u == 0) || (u >= lo_bits && u < 0x8000000000000000ull);
      }
    }
    fused = __all_sync(0xffffffffu, fused);
    const int64_t g0 = t * valid - tb + (int64_t)lane * R;
    if (fused) {
      int s = 0;
      for (; s + 1 < tb; s += 2) {
        warp_step<R, true, false>(a, b, lane, g0, nn);
        warp_step<R, true, false>(b, a, lane, g0, nn);
      }
      if (s < tb) {
        warp_step<R, true, false>(a, b, lane, g0, nn);
#pragma unroll
        for (int i = 0; i < R; ++i) a[i] = b[i];
      }
    } else {  // rare (signs, -0, tiny values): the unfused update, same tile
      int s = 0;
      for (; s + 1 < tb; s += 2) {
        warp_step<R, false, false>(a, b, lane, g0, nn);
        warp_step<R, false, false>(b, a, lane, g0, nn);
      }
      if (s < tb) {
        warp_step<R, false, false>(a, b, lane, g0, nn);
#pragma unroll
        for (int i = 0; i < R; ++i) a[i] = b[i];
      }
    }
    if (next) {
      mbar_wait(bar, phase);  // the next tile has landed
      phase ^= 1;
      // results of t into the buffer, cells of tn into registers
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double v = buf[lane * R + d + i];
        buf[lane * R + d + i] = a[i];
        a[i] = v;
      }
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) buf[lane * R + d + i] = a[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(y + t * valid),
                   "r"(buf_a + (uint32_t)(tb + d) * 8u), "r"((uint32_t)valid * 8u)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    store_pending = true;
    if (!next) break;
    t = tn;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace

extern "C" int ofl_stencil(ofl_stream* s, const double* x, double* y, uint64_t n, uint64_t items,
                           uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  const uint64_t m = items < n ? items : n;
  if (m && (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "stencil operands must be 16-byte aligned");
  ofl::Enqueue q(s, "ofl:stencil");
  if (!q.ok()) return q.status;
  if (m) {
    launch_stencil(s->cs, x, y, n, m);
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "stencil launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}

// Fused two-DFMA update under the tile guard (always on; the unfused update
// runs for tiles the guard rejects).
static bool heat_fused() { return true; }

extern "C" int ofl_heat(ofl_stream* s, double* x, double* y, uint64_t n, uint64_t steps, int tb,
                        uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (n < 1) return ofl::set_error(OFL_ERR_BAD_ARGS, "heat needs n >= 1");
  if (tb < 1 || tb > 128) return ofl::set_error(OFL_ERR_BAD_ARGS, "temporal block must be 1..128");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "heat operands must be 16-byte aligned");
  ofl::Enqueue q(s, "ofl:heat");
  if (!q.ok()) return q.status;
  const int sms = ofl::num_sms(s->dev);
  double* src = x;
  double* dst = y;
  // Pass schedule: the fewest passes of at most tb steps whose count has the
  // parity of `steps` (each pass swaps the buffers, so the state must end
  // where the single-step ping-pong would leave it: x if steps is even, else
  // y), with the steps spread evenly over them — no short remainder pass and
  // no extra single-step pass to fix the parity.
  uint64_t passes = (steps + (uint64_t)tb - 1) / (uint64_t)tb;
  if ((passes & 1) != (steps & 1)) ++passes;
  const uint64_t base_k = passes ? steps / passes : 0, longer = passes ? steps % passes : 0;
  constexpr int R = kHeatPipeR;
  const int smem = (int)(sizeof(double) * (kWarpThreads / 32) * heat_pipe_buf<R>());
  const uint64_t cap = (uint64_t)sms * heat_pipe_min_blocks<R>();
  unsigned long long* ctr = nullptr;  // k_heat_pipe's tile counter, reset once per call
  unsigned long long base = 0;        // values the earlier passes of this call handed out
  uint64_t launches = 0;
  for (uint64_t i = 0; i < passes; ++i) {
    const int k = (int)(base_k + (i < longer ? 1 : 0));
    if (k == 1) {
      launch_stencil(s->cs, src, dst, n, n);
    } else {
      if (!ctr) {
        void* scratch = nullptr;
        const int st = ofl::stream_scratch(s, 65536, &scratch);
        if (st) return st;
        ctr = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + 40960);
        cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s->cs);
        if (e != cudaSuccess) return ofl::cuda_error(e, "heat counter reset");
        cudaFuncSetAttribute(k_heat_pipe<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      }
      const uint64_t valid = 32ull * R - 2 * (uint64_t)k;
      const uint64_t tiles = (n + valid - 1) / valid;
      const uint64_t want = (tiles + kWarpThreads / 32 - 1) / (kWarpThreads / 32);
      const unsigned blocks = (unsigned)(want < cap ? want : cap);
      k_heat_pipe<R><<<blocks, kWarpThreads, smem, s->cs>>>(src, dst, n, k, heat_fused(), ctr, base);
      base += tiles + (uint64_t)blocks * (kWarpThreads / 32);
    }
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "heat launch");
    ++launches;
    double* t = src;
    src = dst;
    dst = t;
  }
  ofl::count_launch(launches);
  return q.finish(ticket);
}

extern "C" int ofl_heat_slab(ofl_stream* s, const double* x, double* y, uint64_t n, int k,
                             uint64_t own_lo, uint64_t own_hi, double* left_ghost, int left_dev,
                             double* right_ghost, int right_dev, uint64_t h, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (n < 1 || k < 1 || k > 128)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "heat slab needs n >= 1 and 1 <= k <= 128");
  if (own_lo > own_hi || own_hi > n || h > own_hi - own_lo)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "heat slab: bad owned range / halo");
  if (x == y) return ofl::set_error(OFL_ERR_BAD_ARGS, "heat slab: x and y must differ");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "heat slab operands must be 16-byte aligned");
  if (left_ghost && left_dev != s->dev) ofl::enable_peer(s->dev, left_dev);
  if (right_ghost && right_dev != s->dev) ofl::enable_peer(s->dev, right_dev);
  ofl::Enqueue q(s, "ofl:heat_slab");
  if (!q.ok()) return q.status;
  SlabOut so{(int64_t)own_lo, (int64_t)own_hi, (int64_t)h, h ? left_ghost : nullptr,
             h ? right_ghost : nullptr};
  // the single-device pass kernel (k_heat_pipe) with the slab epilogue: tiles
  // whose centre reaches the strips sent to the neighbours run the general
  // path, which also stores those strips into the peers' ghost cells
  constexpr int R = kHeatPipeR;
  const int sms = ofl::num_sms(s->dev);
  const uint64_t valid = 32ull * R - 2 * (uint64_t)k;
  const uint64_t tiles = (n + valid - 1) / valid;
  const uint64_t want = (tiles + kWarpThreads / 32 - 1) / (kWarpThreads / 32);
  const uint64_t cap = (uint64_t)sms * heat_pipe_min_blocks<R>();
  const unsigned blocks = (unsigned)(want < cap ? want : cap);
  void* scratch = nullptr;
  const int st = ofl::stream_scratch(s, 65536, &scratch);
  if (st) return st;
  auto* ctr = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + 40960);
  cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s->cs);
  if (e != cudaSuccess) return ofl::cuda_error(e, "heat slab counter reset");
  const int smem = (int)(sizeof(double) * (kWarpThreads / 32) * heat_pipe_buf<R>());
  cudaFuncSetAttribute(k_heat_pipe<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_heat_pipe<R, true><<<blocks, kWarpThreads, smem, s->cs>>>(x, y, n, k, heat_fused(), ctr, 0ull,
                                                               so);
  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ofl::cuda_error(e, "heat slab launch");
  ofl::count_launch();
  return q.finish(ticket);
}
