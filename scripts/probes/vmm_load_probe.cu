// Does a fresh physical allocation (cuMemCreate + map, cudaMalloc,
// cudaMallocAsync growth) wait for kernels that are already running?
// nvcc -gencode arch=compute_100a,code=sm_100a vmm_load_probe.cu
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
__global__ void busy(double* x, long long cycles) {  // every SM busy
  long long t0 = clock64();
  double v = threadIdx.x;
  while (clock64() - t0 < cycles) v = v * 1.0000001 + 1e-9;
  if (v == 12345.0) x[0] = v;
}
typedef CUresult (*CreateFn)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
int main() {
  cudaFree(0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuMemCreate", &fn, cudaEnableDefault, &q);
  CreateFn create = (CreateFn)fn;
  cudaStream_t w, s;
  cudaStreamCreateWithFlags(&w, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* x;
  cudaMalloc(&x, 8);
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = 0;
  for (int load = 0; load < 2; ++load) {
    for (int i = 0; i < 3; ++i) {
      if (load) busy<<<148 * 8, 256, 0, w>>>(x, 100000000);  // ~50 ms, full GPU
      auto t = std::chrono::steady_clock::now();
      CUmemGenericAllocationHandle h;
      create(&h, 32u << 20, &p, 0);
      double a = ms_since(t);
      t = std::chrono::steady_clock::now();
      void* m;
      cudaMalloc(&m, 32u << 20);
      double b = ms_since(t);
      t = std::chrono::steady_clock::now();
      void* n;
      cudaMallocAsync(&n, (64u << 20) * (i + 1 + 4 * load), s);
      cudaStreamSynchronize(s);
      double c = ms_since(t);
      printf("load=%d: cuMemCreate 32 MiB %.2f ms, cudaMalloc 32 MiB %.2f ms, pool growth %.2f ms, kernel still running=%d\n",
             load, a, b, c, cudaStreamQuery(w) == cudaErrorNotReady);
      cudaStreamSynchronize(w);
    }
  }
  return 0;
}
