// 2-D 5-point Jacobi step (paper_1810_11482_b200/kernels/stencil2d.k; the
// reference has only the 1-D stencil.k — this is the same language run by
// the same executor rules, kernel/codegen.py:107-128):
//
//   cells = (w*h) mod 2^32; for gtid < min(items, cells), row = gtid / w,
//   col = gtid - row*w (u32):
//     boundary ring (row 0 / h-1, col 0 / w-1):  y[g] = x[g]
//     interior: y[g] = 0.25 * (((x[g-w] + x[g-1]) + x[g+1]) + x[g+w])
//
// evaluated left to right, round-to-nearest, no contraction: bit-exact.
//
// HBM-bound (16 B per cell: one read, one write).  k_stencil2d_march: a warp
// owns a 64-column x R-row strip; each lane holds two adjacent columns as one
// double2 and marches down the rows keeping (up, cur, down) in registers, so
// every cell is loaded from HBM once (+2/R for the strip's halo rows); the
// west/east neighbours come from the adjacent lanes by shuffle, the two
// outside the strip from a scalar load by lanes 0 / 31 (L2 hits: the
// neighbouring strips load them too).  Stores are 128-bit, streaming.
// k_stencil2d_cells: one thread per cell with u32 index arithmetic exactly
// as the .k text — odd widths (unaligned rows), grids whose w*h wraps 2^32,
// unaligned buffers.
#include <cstdlib>

#include "ofl_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kRows = 32;  // rows per warp strip

__device__ __forceinline__ double interior(double n, double w, double e, double s) {
  return __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(n, w), e), s));
}

// Multi-GPU row slabs (ofl_stencil2d_slab): only the owned local rows
// [own_lo, own_hi) are written; the first / last owned row also goes
// straight into the neighbouring slabs' ghost rows (peer stores over NVLink).
struct SlabRows {
  int64_t own_lo, own_hi;
  double* up;    // receives row own_lo (w cells), or null
  double* down;  // receives row own_hi - 1, or null
};

__device__ __forceinline__ double2 ld2(const double* x, uint64_t idx, uint64_t lx) {
  // idx is even (16-byte aligned pair); either half may lie past the buffer
  if (idx + 1 < lx) return __ldcs(reinterpret_cast<const double2*>(x + idx));
  double2 v = make_double2(0.0, 0.0);
  if (idx < lx) v.x = x[idx];
  return v;
}

__device__ __forceinline__ double ld1(const double* x, uint64_t idx, uint64_t lx) {
  return idx < lx ? x[idx] : 0.0;
}

// w even, w*h < 2^32, x and y 16-byte aligned.  m = cells that execute.
__global__ void __launch_bounds__(kThreads) k_stencil2d_march(const double* __restrict__ x,
                                                              double* __restrict__ y, uint32_t w,
                                                              uint32_t h, uint64_t m, uint64_t lx,
                                                              uint32_t col_chunks) {
  const int lane = threadIdx.x & 31;
  const uint64_t wid = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const uint64_t cx = wid % col_chunks, ry = wid / col_chunks;
  const uint32_t c0 = (uint32_t)cx * 64u;
  const uint32_t r0 = (uint32_t)ry * kRows;
  if (r0 >= h) return;  // warp-uniform
  const uint32_t r1 = (r0 + kRows < h) ? r0 + kRows : h;
  const uint32_t j = c0 + 2u * (uint32_t)lane;  // my columns j, j+1 (j even)
  const bool mine = j < w;                      // w even: j < w => j+1 < w
  // (up, cur) of the first row; rows outside the grid read as 0 (never used)
  double2 up = make_double2(0.0, 0.0), cur = make_double2(0.0, 0.0);
  if (mine && r0 > 0) up = ld2(x, (uint64_t)(r0 - 1) * w + j, lx);
  if (mine) cur = ld2(x, (uint64_t)r0 * w + j, lx);
  double eL = 0.0, eR = 0.0;  // the strip's outside neighbours (lanes 0 / 31)
  if (lane == 0 && c0 > 0) eL = ld1(x, (uint64_t)r0 * w + c0 - 1, lx);
  if (lane == 31 && c0 + 64 < w) eR = ld1(x, (uint64_t)r0 * w + c0 + 64, lx);
#pragma unroll 4
  for (uint32_t i = r0; i < r1; ++i) {
    const uint64_t g = (uint64_t)i * w + j;
    double2 down = make_double2(0.0, 0.0);
    if (mine && i + 1 < h) down = ld2(x, g + w, lx);
    // next row's strip-edge cells, issued early
    double nL = 0.0, nR = 0.0;
    if (i + 1 < r1) {
      if (lane == 0 && c0 > 0) nL = ld1(x, g + w - 1, lx);
      if (lane == 31 && c0 + 64 < w) nR = ld1(x, g + w + 2, lx);  // j + 2 = c0 + 64
    }
    double west = __shfl_up_sync(0xffffffffu, cur.y, 1);
    double east = __shfl_down_sync(0xffffffffu, cur.x, 1);
    if (lane == 0) west = eL;
    if (lane == 31) east = eR;
    if (mine && g < m) {
      const bool edge_row = (i == 0) || (i == h - 1);
      const double o0 = (edge_row || j == 0) ? cur.x : interior(up.x, west, cur.y, down.x);
      const double o1 = (edge_row || j + 1 == w - 1) ? cur.y : interior(up.y, cur.x, east, down.y);
      if (g + 1 < m) {
        __stcs(reinterpret_cast<double2*>(y + g), make_double2(o0, o1));
      } else {
        y[g] = o0;
      }
    }
    up = cur;
    cur = down;
    eL = nL;
    eR = nR;
  }
}

// Batched form: a warp owns 64 columns x RB rows, issues all RB + 2 row
// loads (and the strip-edge loads) up front — RB + 2 independent 512-byte
// requests per warp in flight — then computes and stores the RB rows.  The
// two halo rows per strip mostly hit L2 (the neighbouring strips load them).
template <int RB, bool kSlab = false, bool kPDL = false>
__global__ void __launch_bounds__(kThreads) k_stencil2d_batch(const double* __restrict__ x,
                                                              double* __restrict__ y, uint32_t w,
                                                              uint32_t h, uint64_t m, uint64_t lx,
                                                              uint32_t col_chunks,
                                                              SlabRows sr = SlabRows{}) {
  if constexpr (kPDL) {  // programmatic dependent launch (see k_stream.cu)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const int lane = threadIdx.x & 31;
  const uint64_t wid = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const uint64_t cx = wid % col_chunks, ry = wid / col_chunks;
  const uint32_t c0 = (uint32_t)cx * 64u;
  const int64_t r0 = (int64_t)ry * RB;
  if (r0 >= h) return;  // warp-uniform
  const uint32_t j = c0 + 2u * (uint32_t)lane;
  const bool mine = j < w;
  static_assert(RB <= 32, "one strip-edge value per lane");
  double2 v[RB + 2];  // rows r0-1 .. r0+RB
#pragma unroll
  for (int k = 0; k < RB + 2; ++k) {
    const int64_t r = r0 - 1 + k;
    v[k] = (mine && r >= 0 && r < h) ? ld2(x, (uint64_t)r * w + j, lx) : make_double2(0.0, 0.0);
  }
  // strip-edge cells: lane k holds x[r0+k][c0-1] and x[r0+k][c0+64]
  const int64_t re = r0 + lane;
  const bool erow = lane < RB && re < h;
  const double eLv = (erow && c0 > 0) ? ld1(x, (uint64_t)re * w + c0 - 1, lx) : 0.0;
  const double eRv = (erow && c0 + 64 < w) ? ld1(x, (uint64_t)re * w + c0 + 64, lx) : 0.0;
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    const int64_t i = r0 + k;
    const double2 up = v[k], cur = v[k + 1], down = v[k + 2];
    double west = __shfl_up_sync(0xffffffffu, cur.y, 1);
    double east = __shfl_down_sync(0xffffffffu, cur.x, 1);
    const double wl = __shfl_sync(0xffffffffu, eLv, k);
    const double er = __shfl_sync(0xffffffffu, eRv, k);
    if (lane == 0) west = wl;
    if (lane == 31) east = er;
    const uint64_t g = (uint64_t)i * w + j;
    if (i < h && mine && g < m) {
      const bool edge_row = (i == 0) || (i == (int64_t)h - 1);
      const double o0 = (edge_row || j == 0) ? cur.x : interior(up.x, west, cur.y, down.x);
      const double o1 = (edge_row || j + 1 == w - 1) ? cur.y : interior(up.y, cur.x, east, down.y);
      if (kSlab) {
        if (i >= sr.own_lo && i < sr.own_hi) {
          const double2 o = make_double2(o0, o1);
          __stcs(reinterpret_cast<double2*>(y + g), o);
          if (sr.up && i == sr.own_lo) *reinterpret_cast<double2*>(sr.up + j) = o;
          if (sr.down && i == sr.own_hi - 1) *reinterpret_cast<double2*>(sr.down + j) = o;
        }
      } else if (g + 1 < m) {
        __stcs(reinterpret_cast<double2*>(y + g), make_double2(o0, o1));
      } else {
        y[g] = o0;
      }
    }
  }
}

// CTA form of the batch kernel: the CTA's 8 warps sit side by side (512
// columns x RB rows), so a warp's west / east strip-edge cells are its
// neighbour warps' first / last columns, exchanged through shared memory;
// only the CTA's two outer strips load edge cells from global memory (2 per
// 8 warps instead of 2 per warp — per-warp edge loads cost the 1-D stencil
// 13% against a copy, profiles/r01_stencil2d_sweep.txt).
template <int RB>
__global__ void __launch_bounds__(kThreads) k_stencil2d_cta(const double* __restrict__ x,
                                                            double* __restrict__ y, uint32_t w,
                                                            uint32_t h, uint64_t m, uint64_t lx,
                                                            uint32_t cta_cols) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int kWarps = kThreads / 32;
  __shared__ double s_first[kWarps][RB], s_last[kWarps][RB];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const uint32_t bx = blockIdx.x % cta_cols, by = blockIdx.x / cta_cols;
  const uint32_t c0 = bx * (64u * kWarps) + 64u * (uint32_t)wq;
  const int64_t r0 = (int64_t)by * RB;
  const uint32_t j = c0 + 2u * (uint32_t)lane;
  const bool mine = j < w;
  double2 v[RB + 2];  // rows r0-1 .. r0+RB
#pragma unroll
  for (int k = 0; k < RB + 2; ++k) {
    const int64_t r = r0 - 1 + k;
    v[k] = (mine && r >= 0 && r < h) ? ld2(x, (uint64_t)r * w + j, lx) : make_double2(0.0, 0.0);
  }
  // outer strips only: lane k holds the edge cell of row r0+k
  const int64_t re = r0 + lane;
  const bool erow = lane < RB && re < h;
  const double eLv = (wq == 0 && erow && c0 > 0) ? ld1(x, (uint64_t)re * w + c0 - 1, lx) : 0.0;
  const double eRv = (wq == kWarps - 1 && erow && c0 + 64 < w)
                         ? ld1(x, (uint64_t)re * w + c0 + 64, lx) : 0.0;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < RB; ++k) s_first[wq][k] = v[k + 1].x;
  }
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < RB; ++k) s_last[wq][k] = v[k + 1].y;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    const int64_t i = r0 + k;
    const double2 up = v[k], cur = v[k + 1], down = v[k + 2];
    double west = __shfl_up_sync(0xffffffffu, cur.y, 1);
    double east = __shfl_down_sync(0xffffffffu, cur.x, 1);
    const double wl = __shfl_sync(0xffffffffu, eLv, k);
    const double er = __shfl_sync(0xffffffffu, eRv, k);
    if (lane == 0) west = wq > 0 ? s_last[wq - 1][k] : wl;
    if (lane == 31) east = wq < kWarps - 1 ? s_first[wq + 1][k] : er;
    const uint64_t g = (uint64_t)i * w + j;
    if (i < h && mine && g < m) {
      const bool edge_row = (i == 0) || (i == (int64_t)h - 1);
      const double o0 = (edge_row || j == 0) ? cur.x : interior(up.x, west, cur.y, down.x);
      const double o1 = (edge_row || j + 1 == w - 1) ? cur.y : interior(up.y, cur.x, east, down.y);
      if (g + 1 < m) {
        __stcs(reinterpret_cast<double2*>(y + g), make_double2(o0, o1));
      } else {
        y[g] = o0;
      }
    }
  }
}

// TMA-staged form (full grids, w even, w*h < 2^32): persistent CTAs walk
// 64-column x 32-row output tiles; one elected thread stages each tile's 34
// input rows (cols c0-2 .. c0+65, clipped to the grid; 16-byte aligned) into
// shared memory with cp.async.bulk on an mbarrier, S stages deep so the
// next tiles' copies overlap this tile's compute.  Measured 0.92 of the
// register-batch kernel (profiles/r01_stencil2d_sweep.txt): kept for the
// sweep, not the default.  Each warp computes 4 rows
// from shared memory (128-bit reads of the centre / north / south pairs,
// 64-bit reads of the west / east neighbours) and stores 128-bit streaming.
constexpr int kTmaCols = 64, kTmaRows = 32;
constexpr int kTmaPitch = kTmaCols + 4;  // doubles per staged row (cols c0-2 .. c0+65)
constexpr int kTmaStage = (kTmaRows + 2) * kTmaPitch;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tma_stage_tile(const double* x, double* stage, uint32_t bar,
                                               uint32_t w, uint32_t h, uint32_t c0, int64_t r0) {
  const int64_t lo = (int64_t)c0 - 2 < 0 ? 0 : (int64_t)c0 - 2;
  const int64_t hi = (int64_t)c0 + kTmaCols + 2 > (int64_t)w ? (int64_t)w : (int64_t)c0 + kTmaCols + 2;
  const uint32_t row_bytes = (uint32_t)(hi - lo) * 8u;
  const uint32_t soff = (uint32_t)(lo - ((int64_t)c0 - 2)) * 8u;
  const int64_t ra = r0 - 1 < 0 ? 0 : r0 - 1;
  const int64_t rb = r0 + kTmaRows + 1 > (int64_t)h ? (int64_t)h : r0 + kTmaRows + 1;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"((uint32_t)(rb - ra) * row_bytes)
               : "memory");
  for (int64_t r = ra; r < rb; ++r) {
    const uint32_t dst = smem_u32(stage + (r - (r0 - 1)) * kTmaPitch) + soff;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst), "l"(x + (uint64_t)r * w + lo), "r"(row_bytes), "r"(bar)
        : "memory");
  }
}

template <int S>
__global__ void __launch_bounds__(kThreads) k_stencil2d_tma(const double* __restrict__ x,
                                                            double* __restrict__ y, uint32_t w,
                                                            uint32_t h, uint32_t col_tiles,
                                                            uint64_t ntiles) {
  extern __shared__ __align__(128) double tma_smem[];  // S stages
  __shared__ __align__(8) uint64_t bars[S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t t0 = blockIdx.x;
  if (t0 >= ntiles) return;
  // prologue: the first S-1 tiles of this CTA in flight
  if (threadIdx.x == 0)
    for (int k = 0; k < S - 1; ++k) {
      const uint64_t tk = t0 + (uint64_t)k * gridDim.x;
      if (tk < ntiles)
        tma_stage_tile(x, tma_smem + k * kTmaStage, smem_u32(&bars[k]), w, h,
                       (uint32_t)(tk % col_tiles) * kTmaCols, (int64_t)(tk / col_tiles) * kTmaRows);
    }
  uint32_t it = 0;
  for (uint64_t t = t0; t < ntiles; t += gridDim.x, ++it) {
    const uint32_t st = it % S;
    const uint64_t tn = t + (uint64_t)(S - 1) * gridDim.x;
    if (threadIdx.x == 0 && tn < ntiles) {
      // stage (it+S-1)%S was last read in iteration it-1 (barrier below)
      const uint32_t sn = (it + S - 1) % S;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma_stage_tile(x, tma_smem + sn * kTmaStage, smem_u32(&bars[sn]), w, h,
                     (uint32_t)(tn % col_tiles) * kTmaCols, (int64_t)(tn / col_tiles) * kTmaRows);
    }
    const uint32_t bar = smem_u32(&bars[st]);
    const uint32_t parity = (it / S) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar), "r"(parity)
          : "memory");
    const double* tile = tma_smem + st * kTmaStage;
    const uint32_t c0 = (uint32_t)(t % col_tiles) * kTmaCols;
    const int64_t r0 = (int64_t)(t / col_tiles) * kTmaRows;
    const uint32_t j = c0 + 2u * (uint32_t)lane;
    const int cc = 2 * lane + 2;  // staged column of j
    const int rr0 = 1 + warp * 4; // staged row of this warp's first output row
    if (j < w) {
      double2 up = *reinterpret_cast<const double2*>(tile + (rr0 - 1) * kTmaPitch + cc);
      double2 cur = *reinterpret_cast<const double2*>(tile + rr0 * kTmaPitch + cc);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t i = r0 + warp * 4 + k;
        const int rr = rr0 + k;
        if (i >= (int64_t)h) break;
        const double2 down = *reinterpret_cast<const double2*>(tile + (rr + 1) * kTmaPitch + cc);
        const double west = tile[rr * kTmaPitch + cc - 1];
        const double east = tile[rr * kTmaPitch + cc + 2];
        const bool edge_row = (i == 0) || (i == (int64_t)h - 1);
        const double o0 = (edge_row || j == 0) ? cur.x : interior(up.x, west, cur.y, down.x);
        const double o1 = (edge_row || j + 1 == w - 1) ? cur.y : interior(up.y, cur.x, east, down.y);
        __stcs(reinterpret_cast<double2*>(y + (uint64_t)i * w + j), make_double2(o0, o1));
        up = cur;
        cur = down;
      }
    }
    __syncthreads();  // this stage may be refilled from iteration it+1 on
  }
}

template <int S>
void launch_stencil2d_tma(cudaStream_t cs, int sms, const double* x, double* y, uint32_t w,
                          uint32_t h) {
  const uint32_t col_tiles = (w + kTmaCols - 1) / kTmaCols;
  const uint64_t ntiles = (uint64_t)col_tiles * ((h + kTmaRows - 1) / kTmaRows);
  const size_t smem = (size_t)S * kTmaStage * sizeof(double);
  cudaFuncSetAttribute(k_stencil2d_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stencil2d_tma<S>, kThreads, smem);
  const uint64_t cap = (uint64_t)sms * (occ > 0 ? occ : 1);
  const unsigned g = (unsigned)(ntiles < cap ? ntiles : cap);
  k_stencil2d_tma<S><<<g, kThreads, smem, cs>>>(x, y, w, h, col_tiles, ntiles);
}

// One thread per cell, u32 arithmetic exactly as stencil2d.k.
template <bool kSlab = false>
__global__ void __launch_bounds__(kThreads) k_stencil2d_cells(const double* __restrict__ x,
                                                              double* __restrict__ y, uint32_t w,
                                                              uint32_t h, uint64_t m,
                                                              SlabRows sr = SlabRows{}) {
  const uint64_t t = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (t >= m) return;
  const uint32_t g = (uint32_t)t;
  const uint32_t row = g / w;
  const uint32_t col = g - row * w;
  if (kSlab && (row < sr.own_lo || row >= sr.own_hi)) return;
  double v;
  if (row == 0 || row == h - 1u || col == 0 || col == w - 1u) {
    v = x[g];
  } else {
    v = interior(x[(uint32_t)(g - w)], x[g - 1u], x[g + 1u], x[(uint32_t)(g + w)]);
  }
  y[g] = v;
  if (kSlab) {
    if (sr.up && row == sr.own_lo) sr.up[col] = v;
    if (sr.down && row == sr.own_hi - 1) sr.down[col] = v;
  }
}

// Launch with programmatic stream serialization: the kernel's CTAs may be
// scheduled while the previous kernel on the stream drains; they wait in
// griddepcontrol.wait before touching memory.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), unsigned blocks, cudaStream_t cs, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = cs;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// OFL_STENCIL2D_VARIANT (sweeps, profiles/r01_stencil2d_sweep.txt): 0 = CTA
// form, 8 warps side by side x 8 rows (default), 6 = per-warp batch of 8
// rows, 1 = row marching (32 rows), 2/3/4 = batch of 16/4/12 rows, 5 =
// TMA-staged tiles (4 stages; full grids)
int stencil2d_variant() {
  static int v = [] {
    const char* e = getenv("OFL_STENCIL2D_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

}  // namespace

extern "C" int ofl_stencil2d(ofl_stream* s, const double* x, double* y, uint32_t w, uint32_t h,
                             uint64_t items, uint64_t x_elems, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (x == y && items) return ofl::set_error(OFL_ERR_BAD_ARGS, "stencil2d: x and y must differ");
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  const uint64_t cells = (uint64_t)(uint32_t)(w * h);  // u32 wrap as stencil2d.k
  const uint64_t m = items < cells ? items : cells;
  if (m) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    const bool fits = (uint64_t)w * h < (1ull << 32);
    if (aligned && fits && (w & 1u) == 0) {
      const uint32_t col_chunks = (w + 63u) / 64u;
      const uint64_t rows_needed = (m + w - 1) / w;  // rows holding executed cells
      const int v = stencil2d_variant();
      const uint64_t rows_per_warp = v == 1 ? kRows : v == 2 ? 16 : v == 3 ? 4 : v == 4 ? 12 : 8;
      const uint64_t row_chunks = (rows_needed + rows_per_warp - 1) / rows_per_warp;
      const uint64_t warps = (uint64_t)col_chunks * row_chunks;
      const unsigned blocks = (unsigned)((warps + kThreads / 32 - 1) / (kThreads / 32));
      cudaStream_t cs = s->cs;
      if (v == 5 && m == cells) {
        launch_stencil2d_tma<4>(cs, ofl::num_sms(s->dev), x, y, w, h);
      } else if (v == 0) {
        constexpr int RB = 8;
        const uint32_t cta_cols = (w + 64u * (kThreads / 32) - 1) / (64u * (kThreads / 32));
        const uint64_t row_blocks = (rows_needed + RB - 1) / RB;
        launch_pdl(k_stencil2d_cta<RB>, (unsigned)(cta_cols * row_blocks), cs, x, y, w, h, m,
                   x_elems, cta_cols);
      } else if (v == 1)
        k_stencil2d_march<<<blocks, kThreads, 0, cs>>>(x, y, w, h, m, x_elems, col_chunks);
      else if (v == 2)
        k_stencil2d_batch<16><<<blocks, kThreads, 0, cs>>>(x, y, w, h, m, x_elems, col_chunks);
      else if (v == 3)
        k_stencil2d_batch<4><<<blocks, kThreads, 0, cs>>>(x, y, w, h, m, x_elems, col_chunks);
      else if (v == 4)
        k_stencil2d_batch<12><<<blocks, kThreads, 0, cs>>>(x, y, w, h, m, x_elems, col_chunks);
      else  // v == 6
        launch_pdl(k_stencil2d_batch<8, false, true>, blocks, cs, x, y, w, h, m, x_elems,
                   col_chunks, SlabRows{});
    } else {
      const uint64_t blocks = (m + kThreads - 1) / kThreads;
      k_stencil2d_cells<<<(unsigned)blocks, kThreads, 0, s->cs>>>(x, y, w, h, m);
    }
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "stencil2d launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}

extern "C" int ofl_stencil2d_slab(ofl_stream* s, const double* x, double* y, uint32_t w,
                                  uint32_t h, uint32_t own_lo, uint32_t own_hi, double* up_ghost,
                                  int up_dev, double* down_ghost, int down_dev,
                                  uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (x == y) return ofl::set_error(OFL_ERR_BAD_ARGS, "stencil2d slab: x and y must differ");
  if ((uint64_t)w * h >= (1ull << 32) || own_lo > own_hi || own_hi > h)
    return ofl::set_error(OFL_ERR_BAD_ARGS, "stencil2d slab: bad shape or owned rows");
  if (up_ghost && up_dev != s->dev) ofl::enable_peer(s->dev, up_dev);
  if (down_ghost && down_dev != s->dev) ofl::enable_peer(s->dev, down_dev);
  ofl::Enqueue q(s);
  if (!q.ok()) return q.status;
  const uint64_t m = (uint64_t)w * h;
  if (m && own_lo < own_hi) {
    SlabRows sr{(int64_t)own_lo, (int64_t)own_hi, up_ghost, down_ghost};
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                           reinterpret_cast<uintptr_t>(up_ghost) |
                           reinterpret_cast<uintptr_t>(down_ghost)) & 15) == 0;
    if (aligned && (w & 1u) == 0) {
      constexpr int RB = 8;
      const uint32_t col_chunks = (w + 63u) / 64u;
      const uint64_t warps = (uint64_t)col_chunks * ((h + RB - 1) / RB);
      const unsigned blocks = (unsigned)((warps + kThreads / 32 - 1) / (kThreads / 32));
      k_stencil2d_batch<RB, true><<<blocks, kThreads, 0, s->cs>>>(x, y, w, h, m, m, col_chunks, sr);
    } else {
      const unsigned blocks = (unsigned)((m + kThreads - 1) / kThreads);
      k_stencil2d_cells<true><<<blocks, kThreads, 0, s->cs>>>(x, y, w, h, m, sr);
    }
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return ofl::cuda_error(e, "stencil2d slab launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}
