// Escape-time Mandelbrot (mandelbrot.k, /root/reference/pkg/src/offloadrt/
// bench/kernels/mandelbrot.k:6-29; validator harness.py:133-158).
//
// Per pixel gtid < total = (width*height) mod 2^32:
//   px = gtid mod width, py = gtid / width
//   cre = re0 + ((f64(px) + 0.5) * (re1 - re0)) / f64(width)
//   cim = im0 + ((f64(py) + 0.5) * (im1 - im0)) / f64(height)
//   repeat max_iter times: break if zr*zr + zi*zi > esc (checked BEFORE the
//   increment); t = (zr*zr - zi*zi) + cre; zi = (2*zr)*zi + cim; zr = t; ++count
// Every operation is a separate round-to-nearest IEEE op (no FMA), so the
// counts are bit-identical to the reference's CPU executor.
//
// FP64-issue bound.  Divergence: a warp works on a compact 8x4 pixel tile
// (neighbouring pixels escape at similar counts), and warps pull units of
// kTilesPerUnit tiles from an atomic queue so the slow (bounded) regions do
// not leave SMs idle.  Multi-GPU: rows py = row_first + k*row_step only
// (cyclic row split); tiles index those rows densely.
#include <cmath>
#include <cstdlib>

#include "ofl_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kTileW = 8, kTileH = 4;  // one warp
constexpr int kTilesPerUnit = 4;       // 32x4 pixels per queue pop
#ifndef OFL_PERIOD_CHECK
#define OFL_PERIOD_CHECK 16
#endif
constexpr uint32_t kPeriodCheck = OFL_PERIOD_CHECK;  // cycle test every k iterations (power of 2)

struct MandelArgs {
  uint32_t* out;
  uint32_t width, height;
  double re0, re1, im0, im1, esc;
  uint32_t max_iter;
  uint64_t limit;  // pixels gtid < limit are computed
  uint32_t row_first, row_step, rows;  // rows owned by this launch
  uint32_t tiles_x;
  uint64_t units;
  int compact;  // 1: row r of this launch lands at out[r*width + px]
  int fused;    // allow the FUSED iteration (escape_countP) under its guard
  int period;   // exact cycle detection (escape_countP PERIOD)
};

// INTCMP: the escape test `mag > esc` done on the bit patterns (int64
// compare on the ALU pipe instead of DSETP on the FP64 pipe).  Exact when
// mag >= +0 and esc > 0 are finite, which the host guarantees by enabling it
// only for esc in (0, 1e10] and a viewport inside [-1e10, 1e10]: then every
// executed iteration starts from |z|^2 <= 1e10 and nothing overflows.
// P pixels per thread in lock step (ILP P for the FP64 pipe, branch-free
// body): an escaped pixel keeps iterating harmlessly but its count is
// frozen; the loop ends when all have escaped or max_iter is hit.
//
// FUSED: zi' = (2*zr)*zi + cim is evaluated as fma(2, zr*zi, cim) — 7 DP ops
// per iteration instead of 8.  Bit-identical to the reference whenever
// zr*zi is zero or normal (then round((2zr)*zi) = 2*round(zr*zi), and 2p is
// exact, so fma(2, p, cim) = round(2p + cim)).  The caller enables it only
// with INTCMP's bounds (|z|^2 <= 1e10 before every update: no overflow) and
// when every pixel of the warp has |cre|, |cim| >= 2^-400: a sum of two
// doubles one of which is >= 2^-400 is 0 or >= 2^-454 in magnitude, so zr
// and zi stay in {0} U [2^-454, 1e5] and zr*zi in {0} U [2^-908, 1e10].
//
// PERIOD: exact cycle detection (Brent).  The iteration is a deterministic
// map on the double pair (zr, zi); if the state after iteration i is bit-
// for-bit the state saved after iteration s < i, the orbit repeats forever,
// every value on the cycle already passed the escape test, so the pixel
// never escapes: its count is max_iter — exactly what iterating to max_iter
// gives.  States are saved at iterations 16, 32, 64, ... and compared every
// 16th iteration (64-bit integer compares on the ALU pipe; every 4/8/16/32:
// 2.98/2.71/2.68/2.97 ms for config 3, profiles/r01_mandel_sweep.txt).
//
// PERIOD also skips pixels that provably never escape: c inside the main
// cardioid with the fixed point's multiplier |1 - sqrt(1 - 4c)| <= 0.99, or
// inside the period-2 bulb with |4(c + 1)| <= 0.99.  There the critical
// orbit is attracted to a cycle and stays in the filled Julia set, which
// lies in |z| <= (1 + sqrt(1 + 4|c|)) / 2 < 1.52 — |z|^2 < 2.31, far below
// any bailout >= 4 (the host enables the test only then) — so the reference
// counts max_iter for them; the 1% margin keeps the classification away
// from the boundary, where the basin thins out.  Checked bit for bit on the
// full config-3 image and on cardioid / bulb viewports at up to 5000
// iterations (tests/test_gpu_parity.py).
__device__ __forceinline__ bool never_escapes(double cr, double ci) {
  const double b = (cr + 1.0) * (cr + 1.0) + ci * ci;  // period-2 bulb
  if (b <= 0.06125625) return true;                      // (0.99 / 4)^2
  const double wr = 1.0 - 4.0 * cr, wi = -4.0 * ci;      // 1 - 4c
  const double m = sqrt(wr * wr + wi * wi);
  const double sr = sqrt(0.5 * (m + wr));
  const double si = copysign(sqrt(fmax(0.5 * (m - wr), 0.0)), wi);
  const double lr = 1.0 - sr;                            // multiplier 1 - sqrt(1 - 4c)
  return lr * lr + si * si <= 0.9801;                    // 0.99^2
}

template <bool INTCMP, int P, bool FUSED = false, bool PERIOD = false>
__device__ __forceinline__ void escape_countP(const double (&cr)[P], const double (&ci)[P],
                                              double esc, uint32_t max_iter, uint32_t (&n)[P],
                                              bool interior_ok = false) {
  // zr^2 and zi^2 are carried from one iteration to the next (computed
  // right after the update) so each is evaluated once per iteration.
  double zr[P], zi[P], r2[P], i2[P];
  long long sr[P], si[P];  // saved state (bit patterns) for PERIOD
  bool live[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    zr[p] = zi[p] = r2[p] = i2[p] = 0.0;
    sr[p] = si[p] = 0x7ff8000000000001ll;  // matches no iterate
    n[p] = 0;
    live[p] = true;
    if (PERIOD && interior_ok && never_escapes(cr[p], ci[p])) {
      n[p] = max_iter;
      live[p] = false;
    }
  }
  const long long esc_bits = __double_as_longlong(esc);
  uint32_t save_at = kPeriodCheck;
  // one iteration for every pixel; false once no pixel of the thread is live
  auto iterate = [&]() -> bool {
    bool any = false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const double m = __dadd_rn(r2[p], i2[p]);
      const bool out = INTCMP ? (__double_as_longlong(m) > esc_bits) : (m > esc);
      live[p] = live[p] && !out;
      any = any || live[p];
    }
    if (!any) return false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      // predicated increment (one instruction; the plain `n += live` form
      // compiles to add + select + move around the loop back edge)
      asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q add.u32 %0, %0, 1;\n\t}"
          : "+r"(n[p])
          : "r"((uint32_t)live[p]));
      const double t = __dadd_rn(__dsub_rn(r2[p], i2[p]), cr[p]);
      zi[p] = FUSED ? __fma_rn(2.0, __dmul_rn(zr[p], zi[p]), ci[p])
                    : __dadd_rn(__dmul_rn(__dmul_rn(2.0, zr[p]), zi[p]), ci[p]);
      zr[p] = t;
      r2[p] = __dmul_rn(zr[p], zr[p]);
      i2[p] = __dmul_rn(zi[p], zi[p]);
    }
    return true;
  };
  if constexpr (!PERIOD) {
    for (uint32_t i = 0; i < max_iter; ++i)
      if (!iterate()) return;
  } else {
    // blocks of kPeriodCheck iterations, the cycle test after each full block
    for (uint32_t base = 0; base < max_iter; base += kPeriodCheck) {
      const uint32_t len = max_iter - base < kPeriodCheck ? max_iter - base : kPeriodCheck;
      for (uint32_t j = 0; j < len; ++j)
        if (!iterate()) return;
      if (len < kPeriodCheck) return;
      // state after iteration base + kPeriodCheck
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const long long zb = __double_as_longlong(zr[p]), wb = __double_as_longlong(zi[p]);
        if (live[p] && zb == sr[p] && wb == si[p]) {
          n[p] = max_iter;  // periodic: never escapes
          live[p] = false;
        }
      }
      if (base + kPeriodCheck == save_at) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          sr[p] = __double_as_longlong(zr[p]);
          si[p] = __double_as_longlong(zi[p]);
        }
        save_at <<= 1;
      }
    }
  }
}

// warp-uniform FUSED guard (see escape_countP)
template <int P>
__device__ __forceinline__ bool fused_ok(const double (&cr)[P], const double (&ci)[P]) {
  bool ok = true;
#pragma unroll
  for (int p = 0; p < P; ++p) ok &= fabs(cr[p]) >= 0x1p-400 && fabs(ci[p]) >= 0x1p-400;
  return __all_sync(0xffffffffu, ok);
}

// ILP-P variant: lane l handles the same position of the P tiles of a unit.
// PERIOD keeps two more saved doubles per pixel; its launch bound asks for 4
// CTAs/SM (at P = 2 the registers fit without spilling)
template <bool INTCMP, int P, bool PERIOD = false>
__global__ void __launch_bounds__(kThreads, PERIOD ? 4 : 1) k_mandelbrotP(MandelArgs a,
                                                                       unsigned int* queue) {
  static_assert(kTilesPerUnit % P == 0, "P must divide the unit");
  const int lane = threadIdx.x & 31;
  const double dre = __dsub_rn(a.re1, a.re0);
  const double dim = __dsub_rn(a.im1, a.im0);
  const double fw = (double)a.width, fh = (double)a.height;
  while (true) {
    unsigned int u = 0;
    if (lane == 0) u = atomicAdd(queue, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if ((uint64_t)u >= a.units) break;
#pragma unroll 1
    for (int k = 0; k < kTilesPerUnit; k += P) {
      uint64_t at[P];
      double cr[P], ci[P];
      bool ok[P];
      uint32_t cnt[P];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const uint64_t tile = (uint64_t)u * kTilesPerUnit + k + j;
        const uint32_t ty = (uint32_t)(tile / a.tiles_x);
        const uint32_t tx = (uint32_t)(tile % a.tiles_x);
        const uint32_t px = tx * kTileW + (lane & (kTileW - 1));
        const uint32_t r = ty * kTileH + (lane / kTileW);
        const uint32_t py = a.row_first + r * a.row_step;
        const uint64_t gtid = (uint64_t)py * a.width + px;
        ok[j] = r < a.rows && px < a.width && gtid < a.limit;
        at[j] = a.compact ? (uint64_t)r * a.width + px : gtid;
        const double c_re =
            __dadd_rn(a.re0, __ddiv_rn(__dmul_rn(__dadd_rn((double)px, 0.5), dre), fw));
        const double c_im =
            __dadd_rn(a.im0, __ddiv_rn(__dmul_rn(__dadd_rn((double)py, 0.5), dim), fh));
        cr[j] = ok[j] ? c_re : 1e3;  // off-image lanes escape at once, never stored
        ci[j] = ok[j] ? c_im : 1.0;
      }
      const bool interior_ok = a.esc >= 4.0;  // see never_escapes
      if (INTCMP && a.fused && fused_ok<P>(cr, ci))
        escape_countP<INTCMP, P, true, PERIOD>(cr, ci, a.esc, a.max_iter, cnt, interior_ok);
      else
        escape_countP<INTCMP, P, false, PERIOD>(cr, ci, a.esc, a.max_iter, cnt, interior_ok);
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (ok[j]) a.out[at[j]] = cnt[j];
    }
  }
}

}  // namespace

extern "C" int ofl_mandelbrot(ofl_stream* s, uint32_t* out, uint32_t width, uint32_t height,
                              double re0, double re1, double im0, double im1, double esc,
                              uint32_t max_iter, uint64_t items, uint32_t row_first,
                              uint32_t row_step, int compact, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (row_step == 0) return ofl::set_error(OFL_ERR_BAD_ARGS, "row_step must be >= 1");
  const uint64_t total = (uint64_t)((uint32_t)(width * height));  // u32 wrap as mandelbrot.k
  const uint64_t limit = items < total ? items : total;
  ofl::Enqueue q(s, "ofl:mandelbrot");
  if (!q.ok()) return q.status;
  if (limit && width && row_first < height) {
    MandelArgs a;
    a.out = out;
    a.width = width;
    a.height = height;
    a.re0 = re0;
    a.re1 = re1;
    a.im0 = im0;
    a.im1 = im1;
    a.esc = esc;
    a.max_iter = max_iter;
    a.limit = limit;
    a.row_first = row_first;
    a.row_step = row_step;
    a.compact = compact;
    a.fused = 1;  // fused zi update wherever its guard proves it bit-identical
    // exact cycle detection on by default; OFL_MANDEL_PERIOD=0 runs the plain
    // escape loop — the FP64-roofline measurement of config 3 (bench.py
    // refuses the switch for headline runs)
    static const int period = [] {
      const char* e = getenv("OFL_MANDEL_PERIOD");
      return e ? atoi(e) != 0 : 1;
    }();
    a.period = period;
    // rows of this launch that can hold a pixel with gtid < limit
    const uint64_t last_row = (limit - 1) / width;  // highest py needed
    const uint64_t max_py = last_row < (uint64_t)height - 1 ? last_row : (uint64_t)height - 1;
    a.rows = max_py < row_first ? 0 : (uint32_t)((max_py - row_first) / row_step + 1);
    a.tiles_x = (width + kTileW - 1) / kTileW;
    const uint64_t tiles = (uint64_t)a.tiles_x * ((a.rows + kTileH - 1) / kTileH);
    a.units = (tiles + kTilesPerUnit - 1) / kTilesPerUnit;
    if (a.units) {
      void* scratch = nullptr;
      // queue word lives past the reductions' scratch (k_reduce.cu)
      int st = ofl::stream_scratch(s, 65536, &scratch);
      if (st) return st;
      unsigned int* queue = reinterpret_cast<unsigned int*>(static_cast<char*>(scratch) + 32768);
      cudaError_t e = cudaMemsetAsync(queue, 0, sizeof(unsigned int), s->cs);
      if (e != cudaSuccess) return ofl::cuda_error(e, "queue reset");
      uint64_t warps = a.units;
      uint64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
      const uint64_t cap = (uint64_t)ofl::num_sms(s->dev) * 8;
      if (blocks > cap) blocks = cap;
      const double lim = 1e10;
      const bool intcmp = esc > 0.0 && esc <= lim && fabs(re0) <= lim && fabs(re1) <= lim &&
                          fabs(im0) <= lim && fabs(im1) <= lim;
      // pixels per thread in lock step: the plain kernel 4 (fastest of 1-4,
      // profiles/r01_mandel_sweep.txt); with cycle detection 2 (a warp then
      // waits on the slowest of 64 pixels, not 128: 1.20 vs 1.32 ms for
      // config 3, profiles/r02_mandel_p_sweep.txt)
      if (intcmp)
        if (a.period)
          k_mandelbrotP<true, 2, true><<<(unsigned)blocks, kThreads, 0, s->cs>>>(a, queue);
        else
          k_mandelbrotP<true, 4><<<(unsigned)blocks, kThreads, 0, s->cs>>>(a, queue);
      else if (a.period)
        k_mandelbrotP<false, 2, true><<<(unsigned)blocks, kThreads, 0, s->cs>>>(a, queue);
      else
        k_mandelbrotP<false, 4><<<(unsigned)blocks, kThreads, 0, s->cs>>>(a, queue);
      e = cudaPeekAtLastError();
      if (e != cudaSuccess) return ofl::cuda_error(e, "mandelbrot launch");
      ofl::count_launch();
    }
  }
  return q.finish(ticket);
}
