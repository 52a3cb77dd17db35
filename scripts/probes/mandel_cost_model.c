// Per-pixel cost model of config 3 under the kernel scheme (interior shortcut,
// cycle test every 16 iterations, saves at powers of two): warp-iterations of
// the one-phase kernel vs a two-phase (defer-and-resume) variant.
//   gcc -O2 -fopenmp -ffp-contract=off scripts/probes/mandel_cost_model.c -lm && ./a.out
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static int never_escapes(double cr, double ci) {
  double b = (cr + 1.0) * (cr + 1.0) + ci * ci;
  if (b <= 0.06125625) return 1;
  double wr = 1.0 - 4.0 * cr, wi = -4.0 * ci;
  double m = sqrt(wr * wr + wi * wi);
  double sr = sqrt(0.5 * (m + wr));
  double si = copysign(sqrt(fmax(0.5 * (m - wr), 0.0)), wi);
  double lr = 1.0 - sr;
  return lr * lr + si * si <= 0.9801;
}
int main() {
  const uint32_t W = 7680, H = 4320, IT = 2000;
  uint32_t* c = malloc(sizeof(uint32_t) * W * H);
  #pragma omp parallel for schedule(dynamic, 4)
  for (uint32_t py = 0; py < H; ++py)
    for (uint32_t px = 0; px < W; ++px) {
      double cr = -2 + ((px + 0.5) * 3.0) / W, ci = -1.5 + ((py + 0.5) * 3.0) / H;
      if (never_escapes(cr, ci)) { c[(size_t)py * W + px] = 0; continue; }
      double zr = 0, zi = 0, r2 = 0, i2 = 0; int64_t sr = 0x7ff8000000000001ll, si = sr; uint32_t save_at = 16; uint32_t cost = IT, n = 0;
      for (uint32_t base = 0; base < IT; base += 16) {
        int d = 0;
        for (int j = 0; j < 16; ++j) { if (r2 + i2 > 4.0) { d = 1; break; } n++; double t = (r2 - i2) + cr; zi = (2.0 * zr) * zi + ci; zr = t; r2 = zr * zr; i2 = zi * zi; }
        if (d) { cost = n + 1; break; }
        int64_t zb, wb; memcpy(&zb, &zr, 8); memcpy(&wb, &zi, 8);
        if (zb == sr && wb == si) { cost = base + 16; break; }
        if (base + 16 == save_at) { sr = zb; si = wb; save_at <<= 1; }
      }
      c[(size_t)py * W + px] = cost;
    }
  for (uint32_t T1 = 32; T1 <= 1024; T1 *= 2) {
    double p1 = 0, p2 = 0; long unf = 0;
    for (uint32_t ty = 0; ty < H / 4; ++ty)
      for (uint32_t ux = 0; ux < W / 32; ++ux) {
        uint32_t mx = 0;
        for (int r = 0; r < 4; ++r) for (int x = 0; x < 32; ++x) {
          uint32_t v = c[(size_t)(ty * 4 + r) * W + ux * 32 + x]; if (v > mx) mx = v;
          if (v > T1) { p2 += v - T1; unf++; } }
        p1 += mx < T1 ? mx : T1;
      }
    printf("T1 %4u: phase1 warp-iters %.3e  phase2 (packed, /128) %.3e  total %.3e  queued %ld\n", T1, p1, p2 / 128, p1 + p2 / 128, unf);
  }
}
