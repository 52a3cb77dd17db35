#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int V>
__device__ __forceinline__ double2 ld(const double2* p) {
  double2 r;
  if (V == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
template <int V>
__device__ __forceinline__ void st(double2* p, double2 v) {
  if (V == 3) asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
  else asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
template <int V, int T, int U>
__global__ void __launch_bounds__(T) triad(double* a, const double* b, const double* c, double s, uint64_t n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t n2 = n >> 1;
  double2* a2 = (double2*)a; const double2* b2 = (const double2*)b; const double2* c2 = (const double2*)c;
  const uint64_t base = (uint64_t)blockIdx.x * (T * U) + threadIdx.x;
  double2 vb[U], vc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { uint64_t i = base + u * T; if (i < n2) { vb[u] = ld<V>(b2 + i); vc[u] = ld<V>(c2 + i); } }
#pragma unroll
  for (int u = 0; u < U; ++u) { uint64_t i = base + u * T; if (i < n2) st<V>(a2 + i, make_double2(__dadd_rn(vb[u].x, __dmul_rn(s, vc[u].x)), __dadd_rn(vb[u].y, __dmul_rn(s, vc[u].y)))); }
}
// 256-bit loads: each thread handles 4 doubles
template <int T>
__global__ void __launch_bounds__(T) triad4(double* a, const double* b, const double* c, double s, uint64_t n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t i = ((uint64_t)blockIdx.x * T + threadIdx.x) * 4;
  if (i + 3 < n) {
    double b0, b1, b2_, b3, c0, c1, c2_, c3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(b0), "=d"(b1), "=d"(b2_), "=d"(b3) : "l"(b + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(c0), "=d"(c1), "=d"(c2_), "=d"(c3) : "l"(c + i));
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(a + i), "d"(__dadd_rn(b0, __dmul_rn(s, c0))), "d"(__dadd_rn(b1, __dmul_rn(s, c1))), "d"(__dadd_rn(b2_, __dmul_rn(s, c2_))), "d"(__dadd_rn(b3, __dmul_rn(s, c3))) : "memory");
  }
}
template <typename K>
float timeit(K kern, unsigned blocks, unsigned threads, double* a, double* b, double* c, uint64_t n, int reps) {
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(threads);
  cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, kern, a, (const double*)b, (const double*)c, 3.0, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, kern, a, (const double*)b, (const double*)c, 3.0, n);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return 24.0 * n * reps / (ms * 1e-3) / 1e9;
}
int main() {
  for (int lg = 25; lg <= 28; lg += 3) {
  uint64_t n = 1ull << lg;
  double *a, *b, *c; cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8);
  cudaMemset(b, 0, n * 8); cudaMemset(c, 0, n * 8);
  int reps = lg == 25 ? 1000 : 125;
  for (int rep = 0; rep < 2; ++rep) {
  printf("n=2^%d v0 512x1: %.1f\n", lg, timeit(triad<0, 512, 1>, (unsigned)((n / 2 + 511) / 512), 512, a, b, c, n, reps));
  printf("n=2^%d v1 L2::256B: %.1f\n", lg, timeit(triad<1, 512, 1>, (unsigned)((n / 2 + 511) / 512), 512, a, b, c, n, reps));
  printf("n=2^%d v3 st default: %.1f\n", lg, timeit(triad<3, 512, 1>, (unsigned)((n / 2 + 511) / 512), 512, a, b, c, n, reps));
  printf("n=2^%d v0 256x2: %.1f\n", lg, timeit(triad<0, 256, 2>, (unsigned)((n / 2 + 511) / 512), 256, a, b, c, n, reps));
  printf("n=2^%d v1 256x2: %.1f\n", lg, timeit(triad<1, 256, 2>, (unsigned)((n / 2 + 511) / 512), 256, a, b, c, n, reps));
  printf("n=2^%d v4x256 512: %.1f\n", lg, timeit(triad4<512>, (unsigned)((n / 4 + 511) / 512), 512, a, b, c, n, reps));
  printf("n=2^%d v4x256 256: %.1f\n", lg, timeit(triad4<256>, (unsigned)((n / 4 + 255) / 256), 256, a, b, c, n, reps));
  }
  cudaFree(a); cudaFree(b); cudaFree(c);
  }
  return 0;
}
