// FP64 instruction-throughput probe (B200): DADD / DMUL / DFMA chains, 8
// independent chains per thread, 148*k CTAs of 256 threads.  Prints warp-
// level ops/s per instruction kind.  Build+run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64 scripts/probes/fp64_probe.cu && /tmp/fp64
#include <cstdio>

template <int MODE>
__global__ void k(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) x[j] = __dadd_rn(x[j], b);
      if (MODE == 1) x[j] = __dmul_rn(x[j], a);
      if (MODE == 2) x[j] = __fma_rn(x[j], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5) out[0] = s;
}

template <int MODE>
double run(double* out, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192;
  k<MODE><<<blocks, 256>>>(out, 0.999999, 1e-9, 64);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(out, 0.999999, 1e-9, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return (double)blocks * 256 * iters * 8 / (ms * 1e-3);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {4, 8}) {
    printf("CTAs/SM=%d  DADD %.2f T/s  DMUL %.2f T/s  DFMA %.2f T/s (instr per s, thread level)\n", occ,
           run<0>(out, sms * occ) / 1e12, run<1>(out, sms * occ) / 1e12, run<2>(out, sms * occ) / 1e12);
  }
  return 0;
}
