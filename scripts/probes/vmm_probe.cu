// Where does stream-ordered pool growth spend its time, and do VMM frees
// (cuMemUnmap/cuMemRelease) wait for a kernel running on another stream?
// nvcc -gencode arch=compute_100a,code=sm_100a vmm_probe.cu -lcuda
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
int main() {
  cudaFree(0);
  cudaStream_t s, w;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&w, cudaStreamNonBlocking);
  // custom pool
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = 0;
  cudaMemPool_t pool;
  cudaMemPoolCreate(&pool, &props);
  unsigned long long keep = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  for (int i = 0; i < 3; ++i) {
    void* p;
    auto t = std::chrono::steady_clock::now();
    cudaMallocFromPoolAsync(&p, 1ull << 30, pool, s);
    cudaStreamSynchronize(s);
    printf("custom pool growth 1 GiB: %.2f ms\n", ms_since(t));
  }
  // VMM: one 1 GiB physical allocation
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  size_t gran = 0;
  cuMemGetAllocationGranularity(&gran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  printf("granularity %zu\n", gran);
  for (int i = 0; i < 3; ++i) {
    size_t sz = 1ull << 30;
    auto t = std::chrono::steady_clock::now();
    CUmemGenericAllocationHandle h;
    CUresult r1 = cuMemCreate(&h, sz, &ap, 0);
    double c = ms_since(t);
    CUdeviceptr va;
    cuMemAddressReserve(&va, sz, 0, 0, 0);
    cuMemMap(va, sz, 0, h, 0);
    CUmemAccessDesc d = {};
    d.location = ap.location;
    d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cuMemSetAccess(va, sz, &d, 1);
    double m = ms_since(t);
    spin<<<1, 1, 0, w>>>(100000000);  // ~50 ms on another stream
    auto t2 = std::chrono::steady_clock::now();
    cuMemUnmap(va, sz);
    cuMemRelease(h);
    cuMemAddressFree(va, sz);
    double u = ms_since(t2);
    int busy = cudaStreamQuery(w) == cudaErrorNotReady;
    printf("VMM 1 GiB: create %.2f ms, create+map+access %.2f ms (rc %d); unmap+release %.2f ms, kernel still running=%d\n", c, m, (int)r1, u, busy);
    cudaStreamSynchronize(w);
  }
  // legacy cudaFree while a kernel runs elsewhere
  for (int i = 0; i < 2; ++i) {
    void* p;
    cudaMalloc(&p, 1 << 20);
    spin<<<1, 1, 0, w>>>(100000000);
    auto t = std::chrono::steady_clock::now();
    cudaFree(p);
    printf("cudaFree(1 MiB) with a kernel on another stream: %.2f ms, kernel still running=%d\n", ms_since(t), cudaStreamQuery(w) == cudaErrorNotReady);
    cudaStreamSynchronize(w);
  }
  return 0;
}
