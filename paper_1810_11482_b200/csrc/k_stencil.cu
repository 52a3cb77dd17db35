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
// Single step (k_stencil): each thread owns an aligned pair of cells loaded
// as one 128-bit vector; the outer neighbours come from the adjacent lanes by
// warp shuffle, so every cell is read from HBM once: 16 B/cell.
//
// Temporal blocking (k_heat_tb): a CTA stages a tile of kTile cells plus a
// halo of `tb` cells each side in shared memory, advances it `tb` steps in
// place (the valid region shrinks by one cell per side per step), and writes
// the centre back: 16 B/cell per `tb` steps instead of per step.  Global
// endpoints are fixed points of the update, exactly as stencil.k.
#include <cstdlib>

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
// One-shot tiles (as the STREAM kernels: the block scheduler balances many
// CTAs better than a persistent grid): a CTA of T threads covers U*T cell
// pairs; thread t owns pairs base + t + u*T (cells 2j, 2j+1), so every load
// instruction of a warp is one contiguous 512-byte run.  kPDL: programmatic
// dependent launch (see k_stream.cu) for back-to-back steps.
template <int T, int U, bool kPDL>
__global__ void __launch_bounds__(T) k_stencil(const double* __restrict__ x,
                                               double* __restrict__ y, uint64_t n, uint64_t m) {
  if constexpr (kPDL) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const int lane = threadIdx.x & 31;
  const uint64_t hi = (m < n - 1) ? m : n - 1;
  double edge[U];
  double2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t j = (uint64_t)blockIdx.x * (T * U) + (uint64_t)u * T + threadIdx.x;
    const uint64_t lo = 2 * j;
    // the warp-edge neighbours are loaded together with the main vectors, so
    // a warp waits for one memory latency, not two
    edge[u] = 0.0;
    if (lane == 0 && lo >= 1 && lo - 1 <= hi) edge[u] = x[lo - 1];
    if (lane == 31 && lo + 2 <= hi) edge[u] = x[lo + 2];
    v[u] = make_double2(0.0, 0.0);
    if (lo + 1 <= hi) {
      v[u] = ld_nc(reinterpret_cast<const double2*>(x) + j);
    } else if (lo <= hi) {
      v[u].x = x[lo];
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t j = (uint64_t)blockIdx.x * (T * U) + (uint64_t)u * T + threadIdx.x;
    const uint64_t lo = 2 * j;
    double left = __shfl_up_sync(0xffffffffu, v[u].y, 1);
    double right = __shfl_down_sync(0xffffffffu, v[u].x, 1);
    if (lane == 0) left = edge[u];
    if (lane == 31) right = edge[u];
    if (lo < m) {
      const double r0 = (lo == 0 || lo == n - 1) ? v[u].x : point(left, v[u].x, v[u].y);
      if (lo + 1 < m) {
        const double r1 = (lo + 1 == n - 1) ? v[u].y : point(v[u].x, v[u].y, right);
        __stcs(reinterpret_cast<double2*>(y) + j, make_double2(r0, r1));
      } else {
        y[lo] = r0;
      }
    }
  }
}

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

// single-step launch shape (OFL_STENCIL_VARIANT, sweeps; 2^28 cells, back
// to back): 0 = shared-memory staging, 256 threads x 4 pairs, PDL (default:
// 621 us/step, 6.91 TB/s — copy speed); shuffle form 1 = 256 x 1 (the first
// version, 713 us), 2 = 512 x 1 + PDL (742), 3 = 256 x 4 + PDL (770),
// 7 = 512 x 2 + PDL (706); smem form 4 = 512 x 2 (630), 5 = 512 x 1 (786)
int stencil_variant() {
  static int v = [] {
    const char* e = getenv("OFL_STENCIL_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int T, int U, bool kPDL>
void launch_stencil_t(cudaStream_t cs, const double* x, double* y, uint64_t n, uint64_t m) {
  const uint64_t npairs = (m + 1) >> 1;
  const unsigned blocks = (unsigned)((npairs + (uint64_t)T * U - 1) / ((uint64_t)T * U));
  if (!kPDL) {
    k_stencil<T, U, false><<<blocks, T, 0, cs>>>(x, y, n, m);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(T);
  cfg.stream = cs;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_stencil<T, U, true>, x, y, n, m);
}

void launch_stencil(cudaStream_t cs, const double* x, double* y, uint64_t n, uint64_t m) {
  switch (stencil_variant()) {
    case 1: launch_stencil_t<256, 1, false>(cs, x, y, n, m); break;
    case 2: launch_stencil_t<512, 1, true>(cs, x, y, n, m); break;
    case 3: launch_stencil_t<256, 4, true>(cs, x, y, n, m); break;
    case 4: launch_stencil_smem<512, 2>(cs, x, y, n, m); break;
    case 5: launch_stencil_smem<512, 1>(cs, x, y, n, m); break;
    case 7: launch_stencil_t<512, 2, true>(cs, x, y, n, m); break;
    default: launch_stencil_smem<256, 4>(cs, x, y, n, m); break;
  }
}

// ---------------------------------------------------------------- heat ---
constexpr int kTbThreads = 512;
constexpr int kTile = 8192;  // cells written per CTA pass

// One pass = `tb` steps over the whole vector (x -> y).  Tile t covers
// cells [t*kTile, (t+1)*kTile); smem holds [t*kTile - tb, (t+1)*kTile + tb).
__global__ void __launch_bounds__(kTbThreads) k_heat_tb(const double* __restrict__ x,
                                                        double* __restrict__ y, uint64_t n,
                                                        int tb) {
  extern __shared__ double sm[];  // two buffers of kTile + 2*tb
  const int w = kTile + 2 * tb;
  double* a = sm;
  double* b = sm + w;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t g0 = (int64_t)(t * kTile) - tb;  // global index of smem[0]
    for (int k = threadIdx.x; k < w; k += kTbThreads) {
      const int64_t g = g0 + k;
      a[k] = (g >= 0 && g < (int64_t)n) ? __ldcs(x + g) : 0.0;
    }
    __syncthreads();
    for (int s = 1; s <= tb; ++s) {
      // valid after s steps: smem [s, w - s)
      for (int k = s + threadIdx.x; k < w - s; k += kTbThreads) {
        const int64_t g = g0 + k;
        double v;
        if (g <= 0 || g >= (int64_t)n - 1) v = a[k];
        else v = point(a[k - 1], a[k], a[k + 1]);
        b[k] = v;
      }
      __syncthreads();
      double* tmp = a;
      a = b;
      b = tmp;
    }
    for (int k = tb + threadIdx.x; k < tb + kTile; k += kTbThreads) {
      const int64_t g = g0 + k;
      if (g < (int64_t)n) __stcs(y + g, a[k]);
    }
    __syncthreads();
  }
}

// Register-blocked temporal blocking.  A CTA of kRegThreads threads holds a
// tile of kRegThreads*R consecutive cells in registers (thread t owns cells
// [t*R, t*R+R) of the tile), advances it `tb` steps without touching memory
// — in-warp neighbours by shuffle, warp-edge cells through a double-
// buffered shared array, one __syncthreads per step — and writes the centre
// kRegThreads*R - 2*tb cells.  Errors from the clamped tile ends travel one
// cell per step, so they stay inside the tb-cell halo.  Shared-memory
// traffic per cell-step drops from ~32 B (k_heat_tb) to ~2 warp-edge words,
// which leaves the FP64 pipe (4 DP ops per cell-step) as the limiter.
constexpr int kRegThreads = 256;

// One step of the register tile: in[] -> out[] (distinct register arrays,
// so an unrolled pair of steps needs no register moves).  Step parity p
// selects the half of the warp-edge exchange buffer.
template <int R>
__device__ __forceinline__ void reg_step(const double (&in)[R], double (&out)[R],
                                         double (*edge_l)[kRegThreads / 32],
                                         double (*edge_r)[kRegThreads / 32], int p, int lane,
                                         int warp, bool edge, int64_t g0, int64_t nn) {
  constexpr int kWarps = kRegThreads / 32;
  if (lane == 0) edge_l[p][warp] = in[0];
  if (lane == 31) edge_r[p][warp] = in[R - 1];
  double left = __shfl_up_sync(0xffffffffu, in[R - 1], 1);
  double right = __shfl_down_sync(0xffffffffu, in[0], 1);
  __syncthreads();
  if (lane == 0) left = warp > 0 ? edge_r[p][warp - 1] : in[0];
  if (lane == 31) right = warp < kWarps - 1 ? edge_l[p][warp + 1] : in[R - 1];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const double l = i > 0 ? in[i - 1] : left;
    const double r = i + 1 < R ? in[i + 1] : right;
    out[i] = point(l, in[i], r);
  }
  if (edge) {  // rare: my cells include global cell 0 or n-1 (held fixed)
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t g = g0 + i;
      if (g <= 0 || g >= nn - 1) out[i] = in[i];
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kRegThreads) k_heat_reg(const double* __restrict__ x,
                                                          double* __restrict__ y, uint64_t n,
                                                          int tb) {
  constexpr int kWarps = kRegThreads / 32;
  constexpr int kCells = kRegThreads * R;
  __shared__ double edge_l[2][kWarps];  // first cell of each warp
  __shared__ double edge_r[2][kWarps];  // last cell of each warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t valid = kCells - 2 * tb;
  const int64_t t0 = (int64_t)blockIdx.x * valid - tb;  // global index of tile cell 0
  const int64_t g0 = t0 + (int64_t)threadIdx.x * R;      // global index of my c[0]
  const int64_t nn = (int64_t)n;

  double a[R], b[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t g = g0 + i;
    a[i] = (g >= 0 && g < nn) ? x[g] : 0.0;
  }
  // does my range contain a global endpoint (0 or n-1)?  rare
  const bool edge = (g0 <= 0 && g0 + R > 0) || (g0 <= nn - 1 && g0 + R > nn - 1);

  int s = 0;
  for (; s + 1 < tb; s += 2) {
    reg_step<R>(a, b, edge_l, edge_r, 0, lane, warp, edge, g0, nn);
    reg_step<R>(b, a, edge_l, edge_r, 1, lane, warp, edge, g0, nn);
  }
  const bool odd = s < tb;
  if (odd) reg_step<R>(a, b, edge_l, edge_r, 0, lane, warp, edge, g0, nn);
  // write the valid centre [tb, kCells - tb) of the tile
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int local = threadIdx.x * R + i;
    const int64_t g = g0 + i;
    if (local >= tb && local < kCells - tb && g >= 0 && g < nn) y[g] = odd ? b[i] : a[i];
  }
}

// Warp-independent variant: every warp owns its own tile of 32*R cells
// (halo tb each side, computed redundantly), so a step needs two shuffles
// and no barrier at all; per-thread ILP (R independent cells) hides latency
// instead of occupancy.
constexpr int kWarpThreads = 128;

// Fused form of point(): when 0.5*l and 0.5*r are exact (no result below
// 2^-1022), round(0.5*l + c) is exactly __dadd_rn(__dmul_rn(0.5, l), c), so
//   (0.5*l + c) + 0.5*r  ==  fma(0.5, r, fma(0.5, l, c))      bit for bit
// — two DFMA instead of DMUL + 2 DADD (3 after CSE).  Only valid under the
// tile guard in k_heat_warp (heat_fma_safe).
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

// Residency by tile size (profiles/r01_heat_sweep.txt): four 128-thread
// CTAs per SM for R <= 24 (128 registers), three for R <= 30 (168), two
// above.  Default R=30 at 3 CTAs/SM: 41.2 ms for config 2 (R=24 at 4 CTAs:
// 43.9; 13% instead of 17% redundant halo cells outweighs the lower
// residency); R=32 at 3 CTAs spills inside the step loop (50.0 ms).
// The slab form (extra peer stores) would spill at 128, so it gets three.
template <int R, bool kSlab>
constexpr int heat_warp_min_blocks() {
  return kSlab ? 3 : (R <= 24 ? 4 : (R <= 30 ? 3 : 2));
}

template <int R, bool kSlab = false>
__global__ void __launch_bounds__(kWarpThreads, heat_warp_min_blocks<R, kSlab>()) k_heat_warp(const double* __restrict__ x,
                                                            double* __restrict__ y, uint64_t n,
                                                            int tb, bool fma_ok,
                                                            SlabOut so = SlabOut{}) {
  constexpr int kCells = 32 * R;
  const int lane = threadIdx.x & 31;
  const int64_t wtile = (int64_t)blockIdx.x * (kWarpThreads / 32) + (threadIdx.x >> 5);
  const int64_t valid = kCells - 2 * tb;
  const int64_t nn = (int64_t)n;
  const int64_t g0 = wtile * valid - tb + (int64_t)lane * R;
  if (wtile * valid >= nn) return;  // whole warp past the end (warp-uniform)
  double a[R], b[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t g = g0 + i;
    a[i] = (g >= 0 && g < nn) ? x[g] : 0.0;
  }
  const bool edge = (g0 <= 0 && g0 + R > 0) || (g0 <= nn - 1 && g0 + R > nn - 1);
  const bool odd = warp_tile_steps<R>(a, b, lane, edge, g0, nn, tb, fma_ok);
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int local = lane * R + i;
    const int64_t g = g0 + i;
    if (local >= tb && local < kCells - tb && g >= 0 && g < nn) {
      const double v = odd ? b[i] : a[i];
      if (!kSlab) {
        y[g] = v;
      } else if (g >= so.own_lo && g < so.own_hi) {
        y[g] = v;
        if (so.left && g < so.own_lo + so.h) so.left[g - so.own_lo] = v;
        if (so.right && g >= so.own_hi - so.h) so.right[g - (so.own_hi - so.h)] = v;
      }
    }
  }
}

// Two-level temporal blocking.  Each warp runs warp-independent steps (two
// shuffles, no barrier) on a warp tile of 32*R cells whose outer K cells on
// each side are ghosts (K <= R/2, so they live in lanes 0 and 31); every K
// steps the warps refresh their ghosts from their neighbours' boundary cells
// through double-buffered shared memory (one barrier per K steps).  The
// CTA's outer tb cells are the tile halo.  Redundant work drops from 2*tb per
// warp (k_heat_warp) to 2*K per warp + 2*tb per CTA, barriers from one per
// step (k_heat_reg) to one per K steps.
constexpr int kHierWarps = 4;

// lanes 0 / 31 publish their first / last K owned cells, barrier, then pull
// the neighbours' into their ghosts (static register indices only)
template <int R, int K>
__device__ __forceinline__ void ghost_exchange(double (&c)[R], double (*sl)[K], double (*sr)[K],
                                               int lane, int warp) {
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) sl[warp][i] = c[K + i];
  }
  if (lane == 31) {
#pragma unroll
    for (int i = 0; i < K; ++i) sr[warp][i] = c[R - 2 * K + i];
  }
  __syncthreads();
  if (lane == 0 && warp > 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = sr[warp - 1][i];
  }
  if (lane == 31 && warp < kHierWarps - 1) {
#pragma unroll
    for (int i = 0; i < K; ++i) c[R - K + i] = sl[warp + 1][i];
  }
}

// tb steps of the two-level scheme: K barrier-free warp steps, then a ghost
// refresh from the neighbouring warps; returns whether the state is in a.
template <int R, int K, bool kFma, bool kEdge>
__device__ __forceinline__ bool hier_steps(double (&a)[R], double (&b)[R], int lane, int warp,
                                           int64_t g0, int64_t nn, int tb,
                                           double (*sh_l)[kHierWarps][K],
                                           double (*sh_r)[kHierWarps][K]) {
  int s = 0, ex = 0;
  bool in_a = true;
  while (s < tb) {
    int k = 0;
    for (; k + 1 < K && s + k + 1 < tb; k += 2) {
      if (in_a) {
        warp_step<R, kFma, kEdge>(a, b, lane, g0, nn);
        warp_step<R, kFma, kEdge>(b, a, lane, g0, nn);
      } else {
        warp_step<R, kFma, kEdge>(b, a, lane, g0, nn);
        warp_step<R, kFma, kEdge>(a, b, lane, g0, nn);
      }
    }
    if (k < K && s + k < tb) {
      if (in_a) warp_step<R, kFma, kEdge>(a, b, lane, g0, nn);
      else warp_step<R, kFma, kEdge>(b, a, lane, g0, nn);
      in_a = !in_a;
      ++k;
    }
    s += k;
    if (s >= tb) break;
    const int p = ex & 1;
    ++ex;
    if (in_a)
      ghost_exchange<R, K>(a, sh_l[p], sh_r[p], lane, warp);
    else
      ghost_exchange<R, K>(b, sh_l[p], sh_r[p], lane, warp);
  }
  return in_a;
}

template <int R, int K>
__global__ void __launch_bounds__(kHierWarps * 32) k_heat_hier(const double* __restrict__ x,
                                                               double* __restrict__ y,
                                                               uint64_t n, int tb, bool fma_ok) {
  static_assert(2 * K <= R, "ghosts must fit in the edge lanes");
  constexpr int kOwn = 32 * R - 2 * K;        // owned cells per warp
  constexpr int kSpan = kHierWarps * kOwn;    // owned cells per CTA (incl. CTA halo)
  __shared__ double sh_l[2][kHierWarps][K];   // each warp's first K owned cells
  __shared__ double sh_r[2][kHierWarps][K];   // each warp's last K owned cells
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = (int64_t)n;
  const int64_t cta0 = (int64_t)blockIdx.x * (kSpan - 2 * tb) - tb;  // global of CTA owned[0]
  const int64_t g0 = cta0 + (int64_t)warp * kOwn - K + (int64_t)lane * R;  // my c[0]
  double a[R], b[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t g = g0 + i;
    a[i] = (g >= 0 && g < nn) ? x[g] : 0.0;
  }
  // CTA-uniform update form: ghosts carry neighbouring warps' values into a
  // warp's tile, so the fused update's guard (warp_tile_steps) must hold for
  // the whole CTA tile; the endpoint fix-up is likewise decided per CTA
  bool safe = fma_ok;
  if (safe) {
    const uint64_t lo_bits = (uint64_t)(tb + 3) << 52;  // 2^(tb-1020)
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t u = (uint64_t)__double_as_longlong(a[i]);
      safe &= (u == 0) || (u >= lo_bits && u < 0x8000000000000000ull);
    }
  }
  safe = __syncthreads_and(safe);
  const bool edge = __syncthreads_or((g0 <= 0 && g0 + R > 0) || (g0 <= nn - 1 && g0 + R > nn - 1));
  bool in_a;
  if (safe)
    in_a = edge ? hier_steps<R, K, true, true>(a, b, lane, warp, g0, nn, tb, sh_l, sh_r)
                : hier_steps<R, K, true, false>(a, b, lane, warp, g0, nn, tb, sh_l, sh_r);
  else
    in_a = edge ? hier_steps<R, K, false, true>(a, b, lane, warp, g0, nn, tb, sh_l, sh_r)
                : hier_steps<R, K, false, false>(a, b, lane, warp, g0, nn, tb, sh_l, sh_r);
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int own = warp * kOwn - K + lane * R + i;  // CTA owned coordinate
    const int64_t g = g0 + i;
    const bool mine = (lane * R + i >= K) && (lane * R + i < 32 * R - K);
    if (mine && own >= tb && own < kSpan - tb && g >= 0 && g < nn) y[g] = in_a ? a[i] : b[i];
  }
}

}  // namespace

extern "C" int ofl_stencil(ofl_stream* s, const double* x, double* y, uint64_t n, uint64_t items,
                           uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  const uint64_t m = items < n ? items : n;
  if (m && (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "stencil operands must be 16-byte aligned");
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  if (m) {
    launch_stencil(s->cs, x, y, n, m);
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "stencil launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}

// heat pass kernel (OFL_HEAT_KERNEL): 2 = warp-independent register tiles
// (default, fastest measured), 0 = CTA register tiles with a barrier per
// step, 1 = shared-memory tiles, 3 = two-level (warp ghosts + CTA halo)
static int heat_kernel() {
  static int v = [] {
    const char* e = getenv("OFL_HEAT_KERNEL");
    return e ? atoi(e) : 2;
  }();
  return v;
}

// cells per thread of the register kernels (OFL_HEAT_R: 8, 16, 20, 24, 26, 28, 30, 32);
// default per kernel from profiles/r01_heat_sweep.txt
static int heat_cells_per_thread() {
  static int v = [] {
    const char* e = getenv("OFL_HEAT_R");
    const int dflt = heat_kernel() == 2 ? 30 : 8;
    const int r = e ? atoi(e) : dflt;
    return (r == 8 || r == 16 || r == 20 || r == 24 || r == 26 || r == 28 || r == 30 || r == 32) ? r : dflt;
  }();
  return v;
}

// fused two-DFMA update under the tile guard (OFL_HEAT_FMA=0 disables; the
// unfused kernel is kept for the sweep and for tiles the guard rejects)
static bool heat_fused() {
  static bool v = [] {
    const char* e = getenv("OFL_HEAT_FMA");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

extern "C" int ofl_heat(ofl_stream* s, double* x, double* y, uint64_t n, uint64_t steps, int tb,
                        uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (n < 1) return ofl::set_error(OFL_ERR_BAD_ARGS, "heat needs n >= 1");
  if (tb < 1 || tb > 128) return ofl::set_error(OFL_ERR_BAD_ARGS, "temporal block must be 1..128");
  if (heat_kernel() != 2 && tb > 64) tb = 64;  // the sweep kernels size their tiles for <= 64
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "heat operands must be 16-byte aligned");
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  const int sms = ofl::num_sms(s->dev);
  double* src = x;
  double* dst = y;
  const size_t smem = sizeof(double) * 2 * (kTile + 2 * 64);
  // per-device attribute; cheap to (re)apply
  cudaFuncSetAttribute(k_heat_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // Pass schedule: the fewest passes of at most tb steps whose count has the
  // parity of `steps` (each pass swaps the buffers, so the state must end
  // where the single-step ping-pong would leave it: x if steps is even, else
  // y), with the steps spread evenly over them — no short remainder pass and
  // no extra single-step pass to fix the parity.
  uint64_t passes = (steps + (uint64_t)tb - 1) / (uint64_t)tb;
  if ((passes & 1) != (steps & 1)) ++passes;
  const uint64_t base_k = passes ? steps / passes : 0, longer = passes ? steps % passes : 0;
  uint64_t launches = 0;
  auto run_pass = [&](int k) -> cudaError_t {
    if (k == 1) {
      launch_stencil(s->cs, src, dst, n, n);
    } else if (heat_kernel() == 1) {
      const uint64_t ntiles = (n + kTile - 1) / kTile;
      uint64_t blocks = ntiles < (uint64_t)sms * 2 ? ntiles : (uint64_t)sms * 2;
      const size_t sm_k = sizeof(double) * 2 * (kTile + 2 * k);
      k_heat_tb<<<(unsigned)blocks, kTbThreads, sm_k, s->cs>>>(src, dst, n, k);
    } else if (heat_kernel() == 3) {
      const int r = heat_cells_per_thread();
      constexpr int K = 8;
      const uint64_t span = (uint64_t)kHierWarps * (32 * (uint64_t)r - 2 * K);
      const uint64_t valid = span - 2 * (uint64_t)k;
      const unsigned blocks = (unsigned)((n + valid - 1) / valid);
      if (r == 24)
        k_heat_hier<24, K><<<blocks, kHierWarps * 32, 0, s->cs>>>(src, dst, n, k, heat_fused());
      else
        k_heat_hier<16, K><<<blocks, kHierWarps * 32, 0, s->cs>>>(src, dst, n, k, heat_fused());
    } else if (heat_kernel() == 2) {
      const int r = heat_cells_per_thread();
      const bool fma = heat_fused();
      const uint64_t valid = 32ull * r - 2 * (uint64_t)k;
      const uint64_t warps = (n + valid - 1) / valid;
      const unsigned blocks = (unsigned)((warps + kWarpThreads / 32 - 1) / (kWarpThreads / 32));
      if (r == 32)
        k_heat_warp<32><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
      else if (r == 24)
        k_heat_warp<24><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
      else if (r == 20)
        k_heat_warp<20><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
      else if (r == 28)
        k_heat_warp<28><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
      else if (r == 26)
        k_heat_warp<26><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
      else if (r == 30)
        k_heat_warp<30><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
      else
        k_heat_warp<16><<<blocks, kWarpThreads, 0, s->cs>>>(src, dst, n, k, fma);
    } else {
      const int r = heat_cells_per_thread();
      const uint64_t valid = (uint64_t)kRegThreads * r - 2 * (uint64_t)k;
      const unsigned blocks = (unsigned)((n + valid - 1) / valid);
      if (r == 8)
        k_heat_reg<8><<<blocks, kRegThreads, 0, s->cs>>>(src, dst, n, k);
      else if (r == 32)
        k_heat_reg<32><<<blocks, kRegThreads, 0, s->cs>>>(src, dst, n, k);
      else
        k_heat_reg<16><<<blocks, kRegThreads, 0, s->cs>>>(src, dst, n, k);
    }
    ++launches;
    double* t = src;
    src = dst;
    dst = t;
    return cudaPeekAtLastError();
  };
  for (uint64_t i = 0; i < passes; ++i) {
    const int k = (int)(base_k + (i < longer ? 1 : 0));
    cudaError_t e = run_pass(k);
    if (e != cudaSuccess) return ofl::cuda_error(e, "heat launch");
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
  if (left_ghost && left_dev != s->dev) ofl::enable_peer(s->dev, left_dev);
  if (right_ghost && right_dev != s->dev) ofl::enable_peer(s->dev, right_dev);
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  SlabOut so{(int64_t)own_lo, (int64_t)own_hi, (int64_t)h, h ? left_ghost : nullptr,
             h ? right_ghost : nullptr};
  const uint64_t valid = 32ull * 24 - 2 * (uint64_t)k;
  const uint64_t warps = (n + valid - 1) / valid;
  const unsigned blocks = (unsigned)((warps + kWarpThreads / 32 - 1) / (kWarpThreads / 32));
  k_heat_warp<24, true><<<blocks, kWarpThreads, 0, s->cs>>>(x, y, n, k, heat_fused(), so);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ofl::cuda_error(e, "heat slab launch");
  ofl::count_launch();
  return q.finish(ticket);
}
