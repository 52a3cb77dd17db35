// Read-bandwidth probe for the reduction kernels (dot f32, 2 x 8 GiB): load
// flavour x unroll x grid.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o /tmp/rbw scripts/probes/read_bw_probe.cu && /tmp/rbw
#include <cstdio>
#include <cstdint>

template <int FLAVOR>
__device__ __forceinline__ float4 ld(const float4* p) {
  float4 v;
  if (FLAVOR == 0) {
    v = __ldcs(p);
  } else if (FLAVOR == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else if (FLAVOR == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else {
    v = __ldg(p);
  }
  return v;
}

template <int FLAVOR, int U>
__global__ void __launch_bounds__(512) kdot(const float4* a, const float4* b, double* out, uint64_t n4) {
  const uint64_t stride = (uint64_t)gridDim.x * 512;
  uint64_t i = (uint64_t)blockIdx.x * 512 + threadIdx.x;
  double s[U];
#pragma unroll
  for (int u = 0; u < U; ++u) s[u] = 0;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { x[u] = ld<FLAVOR>(a + i + u * stride); y[u] = ld<FLAVOR>(b + i + u * stride); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s[u] = fma((double)x[u].x, (double)y[u].x, s[u]);
      s[u] = fma((double)x[u].y, (double)y[u].y, s[u]);
      s[u] = fma((double)x[u].z, (double)y[u].z, s[u]);
      s[u] = fma((double)x[u].w, (double)y[u].w, s[u]);
    }
  }
  double t = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) t += s[u];
  if (t == 12345.0) out[0] = t;
}

__global__ void fill(float* p, uint64_t n, uint32_t seed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    p[i] = (h >> 8) * (1.0f / 16777216.0f);
  }
}

template <int FLAVOR, int U>
void run(const float4* a, const float4* b, double* out, uint64_t n4, int cps, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int blocks = sms * cps;
  kdot<FLAVOR, U><<<blocks, 512>>>(a, b, out, n4);
  cudaEventRecord(e0);
  const int K = 10;
  for (int k = 0; k < K; ++k) kdot<FLAVOR, U><<<blocks, 512>>>(a, b, out, n4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("flavor %d unroll %d CTAs/SM %d: %.3f ms  %.1f GB/s\n", FLAVOR, U, cps, ms / K,
         2.0 * n4 * 16 / (ms / K * 1e-3) / 1e9);
}

int main() {
  uint64_t n = 1ull << 31, n4 = n / 4;
  float4 *a, *b;
  double* out;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMalloc(&out, 8);
  fill<<<4096, 256>>>((float*)a, n, 1u);
  fill<<<4096, 256>>>((float*)b, n, 7u);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cps : {1, 2, 3}) {
    run<0, 1>(a, b, out, n4, cps, sms);
    run<0, 2>(a, b, out, n4, cps, sms);
    run<0, 4>(a, b, out, n4, cps, sms);
    run<0, 8>(a, b, out, n4, cps, sms);
  }
  return 0;
}
