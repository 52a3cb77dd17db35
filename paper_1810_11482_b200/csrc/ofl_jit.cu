// Run-time compilation of kernel-language programs that have no hand-written
// binding: the Python code generator (kernel/cuda_codegen.py) lowers the
// validated IR to CUDA C, NVRTC compiles it for sm_100a (the paper compiles
// with NVRTC too), and the cubin is loaded through the
// runtime's library API (cudaLibraryLoadData / cudaLibraryGetKernel), so no
// driver-API linkage is needed.  This replaces the reference's numba
// whole-grid compilation (kernel/codegen.py:319-337) for such kernels.
//
// libnvrtc is dlopen'ed on first use (path hint from the caller, then the
// CUDA toolkit), so libofl.so itself has no NVRTC dependency.
#include <dlfcn.h>
#include <nvrtc.h>

#include <string>
#include <vector>

#include "ofl_internal.h"

struct ofl_jit {
  int dev;
  cudaLibrary_t lib;
  cudaKernel_t kern;
};

namespace {

struct NvrtcApi {
  void* h = nullptr;
  nvrtcResult (*Create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*Compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*LogSize)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*Log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*CubinSize)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*Cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*Destroy)(nvrtcProgram*) = nullptr;
  const char* (*Err)(nvrtcResult) = nullptr;
};

NvrtcApi g_nv;
std::mutex g_nv_mu;

int nvrtc_load(const char* hint) {
  std::lock_guard<std::mutex> g(g_nv_mu);
  if (g_nv.h) return OFL_OK;
  // the toolkit's NVRTC matches the cudart this library links statically
  const char* cands[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", hint, "libnvrtc.so.12",
                         "libnvrtc.so"};
  void* h = nullptr;
  for (const char* c : cands)
    if (c && *c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return ofl::set_error(OFL_ERR_COMPILE, std::string("dlopen libnvrtc: ") + dlerror());
#define OFL_NV(f, n)                                                          \
  g_nv.f = reinterpret_cast<decltype(g_nv.f)>(dlsym(h, n));                   \
  if (!g_nv.f) return ofl::set_error(OFL_ERR_COMPILE, std::string("missing ") + n);
  OFL_NV(Create, "nvrtcCreateProgram")
  OFL_NV(Compile, "nvrtcCompileProgram")
  OFL_NV(LogSize, "nvrtcGetProgramLogSize")
  OFL_NV(Log, "nvrtcGetProgramLog")
  OFL_NV(CubinSize, "nvrtcGetCUBINSize")
  OFL_NV(Cubin, "nvrtcGetCUBIN")
  OFL_NV(Destroy, "nvrtcDestroyProgram")
  OFL_NV(Err, "nvrtcGetErrorString")
#undef OFL_NV
  g_nv.h = h;
  return OFL_OK;
}

}  // namespace

extern "C" {

int ofl_jit_available(const char* nvrtc_path) { return nvrtc_load(nvrtc_path); }

int ofl_jit_compile(int dev, const char* src, const char* entry, ofl_jit** out, char* log,
                    int logcap) {
  int st = nvrtc_load(nullptr);
  if (st) return st;
  cudaError_t e = ofl::use_device(dev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "cudaSetDevice");
  cudaDeviceProp p;
  e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "cudaGetDeviceProperties");
  std::string arch = "--gpu-architecture=sm_" + std::to_string(p.major) +
                     std::to_string(p.minor) + (p.major >= 9 ? "a" : "");
  const char* opts[] = {arch.c_str(), "--fmad=false", "--std=c++17", "-default-device",
                        "--extra-device-vectorization"};
  nvrtcProgram prog;
  nvrtcResult r = g_nv.Create(&prog, src, "ofl_kernel.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return ofl::set_error(OFL_ERR_COMPILE, g_nv.Err(r));
  r = g_nv.Compile(prog, 5, opts);
  size_t ls = 0;
  g_nv.LogSize(prog, &ls);
  std::string text(ls, '\0');
  if (ls) g_nv.Log(prog, &text[0]);
  if (log && logcap > 0) std::snprintf(log, (size_t)logcap, "%s", text.c_str());
  if (r != NVRTC_SUCCESS) {
    g_nv.Destroy(&prog);
    return ofl::set_error(OFL_ERR_COMPILE, std::string("nvrtc: ") + g_nv.Err(r) + "\n" + text);
  }
  size_t cs = 0;
  g_nv.CubinSize(prog, &cs);
  std::vector<char> cubin(cs);
  g_nv.Cubin(prog, cubin.data());
  g_nv.Destroy(&prog);
  auto* k = new ofl_jit();
  k->dev = dev;
  e = cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&k->kern, k->lib, entry);
  if (e != cudaSuccess) {
    delete k;
    return ofl::cuda_error(e, "load jit module");
  }
  *out = k;
  return OFL_OK;
}

// params: kernel parameter pointers (cudaLaunchKernel convention)
int ofl_jit_launch(ofl_stream* s, ofl_jit* k, void** params, uint64_t blocks, int threads,
                   uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  if (!k) return ofl::set_error(OFL_ERR_BAD_ARGS, "null jit kernel");
  ofl::Enqueue q(s, "ofl:jit_launch");
  if (!q.ok()) return q.status;
  if (blocks) {
    cudaError_t e = cudaLaunchKernel((const void*)k->kern, dim3((unsigned)blocks), dim3(threads),
                                     params, 0, s->cs);
    if (e != cudaSuccess) return ofl::cuda_error(e, "jit launch");
    ofl::count_launch();
  }
  return q.finish(ticket);
}

int ofl_jit_destroy(ofl_jit* k) {
  if (!k) return OFL_OK;
  ofl::use_device(k->dev);
  cudaLibraryUnload(k->lib);
  delete k;
  return OFL_OK;
}

// 0xFF-fill `bytes` of device memory on the stream (error-record reset)
int ofl_fill_ones(ofl_stream* s, void* dptr, uint64_t bytes, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  ofl::Enqueue q(s, "ofl:fill_ones");
  if (!q.ok()) return q.status;
  cudaError_t e = cudaMemsetAsync(dptr, 0xFF, bytes, s->cs);
  if (e != cudaSuccess) return ofl::cuda_error(e, "memset");
  return q.finish(ticket);
}

}  // extern "C"
