// Stream-ordered pool behaviour: does cudaMallocAsync (+ memset + sync of its
// own stream) ever wait for a long kernel on another stream, with frees
// queued behind that kernel?  nvcc -gencode arch=compute_100a,code=sm_100a
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
int main() {
  cudaStream_t work, zero, fre;
  cudaStreamCreateWithFlags(&work, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&zero, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&fre, cudaStreamNonBlocking);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long keep = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  int no = 0;
  cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  cudaEvent_t fence;
  cudaEventCreateWithFlags(&fence, cudaEventDisableTiming);
  for (int trial = 0; trial < 6; ++trial) {
    void *big1, *big2;
    cudaMallocAsync(&big1, 1ull << 30, zero);
    cudaMallocAsync(&big2, 1ull << 30, zero);
    cudaStreamSynchronize(zero);
    spin<<<1, 1, 0, work>>>(100000000);  // ~50 ms
    void* tmp;
    auto t0 = std::chrono::steady_clock::now();
    cudaMallocAsync(&tmp, 1 << 20, zero);
    double a = ms_since(t0);
    cudaMemsetAsync(tmp, 0, 1 << 20, zero);
    cudaStreamSynchronize(zero);
    double b = ms_since(t0);
    cudaEventRecord(fence, work);
    cudaStreamWaitEvent(fre, fence, 0);
    cudaFreeAsync(tmp, fre);
    void* fresh;
    auto t1 = std::chrono::steady_clock::now();
    cudaMallocAsync(&fresh, 32 << 20, zero);
    double c = ms_since(t1);
    cudaMemsetAsync(fresh, 0, 32 << 20, zero);
    cudaStreamSynchronize(zero);
    double d = ms_since(t1);
    printf("trial %d: malloc 1MiB %.2f ms (+memset+sync %.2f); after free: malloc 32MiB %.2f ms (+memset+sync %.2f); work done=%d\n",
           trial, a, b, c, d, cudaStreamQuery(work) == cudaSuccess);
    cudaStreamSynchronize(work);
    cudaFreeAsync(big1, fre);
    cudaFreeAsync(big2, fre);
    cudaFreeAsync(fresh, fre);
    cudaStreamSynchronize(fre);
  }
  return 0;
}
