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
// HBM-bound (16 B per cell: one read, one write).  Each lane holds two
// adjacent columns as one double2 and keeps the rows it needs in registers,
// so every cell is loaded from HBM once (+ the tile's halo rows, L2 hits);
// the west/east neighbours come from the adjacent lanes by shuffle.  Stores
// are 128-bit, streaming.
// k_stencil2d_cells: one thread per cell with u32 index arithmetic exactly
// as the .k text — odd widths (unaligned rows), grids whose w*h wraps 2^32,
// unaligned buffers.
#include "ofl_internal.h"

namespace {

constexpr int kThreads = 256;

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

}  // namespace

extern "C" int ofl_stencil2d(ofl_stream* s, const double* x, double* y, uint32_t w, uint32_t h,
                             uint64_t items, uint64_t x_elems, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (x == y && items) return ofl::set_error(OFL_ERR_BAD_ARGS, "stencil2d: x and y must differ");
  ofl::Enqueue q(s, "ofl:stencil2d");
  if (!q.ok()) return q.status;
  const uint64_t cells = (uint64_t)(uint32_t)(w * h);  // u32 wrap as stencil2d.k
  const uint64_t m = items < cells ? items : cells;
  if (m) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    const bool fits = (uint64_t)w * h < (1ull << 32);
    if (aligned && fits && (w & 1u) == 0) {
      // CTA form: 8 warps side by side x 8 rows (fastest of the row-march,
      // per-warp batch and TMA-staged forms, profiles/r01_stencil2d_sweep.txt)
      constexpr int RB = 8;
      const uint64_t rows_needed = (m + w - 1) / w;  // rows holding executed cells
      const uint32_t cta_cols = (w + 64u * (kThreads / 32) - 1) / (64u * (kThreads / 32));
      const uint64_t row_blocks = (rows_needed + RB - 1) / RB;
      launch_pdl(k_stencil2d_cta<RB>, (unsigned)(cta_cols * row_blocks), s->cs, x, y, w, h, m,
                 x_elems, cta_cols);
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
  ofl::Enqueue q(s, "ofl:stencil2d_slab");
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
