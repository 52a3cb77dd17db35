// Allocation cost: cudaMalloc vs cudaMallocAsync pool growth vs pool reuse,
// per GiB.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
int main() {
  cudaFree(0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long keep = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  const size_t sizes[] = {1u << 20, 64u << 20, 1ull << 30, 8ull << 30};
  for (size_t sz : sizes) {
    void* p[4];
    auto t = std::chrono::steady_clock::now();
    for (auto& q : p) cudaMalloc(&q, sz);
    double a = ms_since(t) / 4;
    t = std::chrono::steady_clock::now();
    for (auto& q : p) cudaFree(q);
    double f = ms_since(t) / 4;
    t = std::chrono::steady_clock::now();
    for (auto& q : p) cudaMallocAsync(&q, sz, s);
    cudaStreamSynchronize(s);
    double g = ms_since(t) / 4;
    for (auto& q : p) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
    t = std::chrono::steady_clock::now();
    for (auto& q : p) cudaMallocAsync(&q, sz, s);
    cudaStreamSynchronize(s);
    double r = ms_since(t) / 4;
    t = std::chrono::steady_clock::now();
    for (auto& q : p) cudaMemsetAsync(q, 0, sz, s);
    cudaStreamSynchronize(s);
    double z = ms_since(t) / 4;
    for (auto& q : p) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
    printf("%8zu MiB: cudaMalloc %.3f ms, cudaFree %.3f ms, pool growth %.3f ms, pool reuse %.3f ms, memset %.3f ms\n",
           sz >> 20, a, f, g, r, z);
  }
  return 0;
}
