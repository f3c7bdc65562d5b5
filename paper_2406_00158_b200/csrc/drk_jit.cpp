// drk_jit.cpp — run-time compilation of traced view expressions (NVRTC -> sm_100a cubin).
//
// The reference evaluates arbitrary Python lambdas over numpy arrays
// (views.py:164-181 `_apply_elementwise`, algorithms.py:101-111 vectorised for_each).  The
// B200 runtime traces such a lambda once into an expression, generates a functor in CUDA
// C++ that plugs into the map/reduce/scan templates of drk_device.cuh, and compiles it
// here.  NVRTC is loaded lazily with dlopen so the library (and every AOT kernel) works on
// hosts without it; modules are loaded with cudaLibraryLoadData, which makes the kernels
// available on every device of the process.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/drk.h"

typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;

namespace {

struct Nvrtc {
  bool tried = false;
  bool ok = false;
  std::string why;
  const char* (*GetErrorString)(nvrtcResult_t);
  nvrtcResult_t (*CreateProgram)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                                 const char* const*);
  nvrtcResult_t (*DestroyProgram)(nvrtcProgram_t*);
  nvrtcResult_t (*CompileProgram)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*GetProgramLogSize)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*GetProgramLog)(nvrtcProgram_t, char*);
  nvrtcResult_t (*GetCUBINSize)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*GetCUBIN)(nvrtcProgram_t, char*);
};

std::mutex g_jit_mu;
Nvrtc g_nv;

bool load_nvrtc(std::string& why) {
  if (g_nv.tried) {
    why = g_nv.why;
    return g_nv.ok;
  }
  g_nv.tried = true;
  const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void* h = nullptr;
  for (const char* n : names) {
    h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    if (h) break;
  }
  if (!h) {
    g_nv.why = "NVRTC (libnvrtc.so.12) not found";
    why = g_nv.why;
    return false;
  }
#define DRK_SYM(field, sym)                                     \
  *(void**)(&g_nv.field) = dlsym(h, sym);                        \
  if (!g_nv.field) {                                             \
    g_nv.why = std::string("NVRTC symbol missing: ") + sym;      \
    why = g_nv.why;                                              \
    return false;                                                \
  }
  DRK_SYM(GetErrorString, "nvrtcGetErrorString");
  DRK_SYM(CreateProgram, "nvrtcCreateProgram");
  DRK_SYM(DestroyProgram, "nvrtcDestroyProgram");
  DRK_SYM(CompileProgram, "nvrtcCompileProgram");
  DRK_SYM(GetProgramLogSize, "nvrtcGetProgramLogSize");
  DRK_SYM(GetProgramLog, "nvrtcGetProgramLog");
  DRK_SYM(GetCUBINSize, "nvrtcGetCUBINSize");
  DRK_SYM(GetCUBIN, "nvrtcGetCUBIN");
#undef DRK_SYM
  g_nv.ok = true;
  return true;
}

thread_local std::string g_jit_error;

int jit_error(int code, const std::string& msg) {
  g_jit_error = msg;
  return code;
}

void copy_log(const std::string& s, char* log, size_t log_bytes) {
  if (!log || !log_bytes) return;
  size_t n = s.size() < log_bytes - 1 ? s.size() : log_bytes - 1;
  memcpy(log, s.data(), n);
  log[n] = 0;
}

int compile_cubin(const char* source, const char* name, const char* include_dir, std::vector<char>& cubin,
                  std::string& log) {
  std::string why;
  std::lock_guard<std::mutex> lk(g_jit_mu);
  if (!load_nvrtc(why)) {
    log = why;
    return DRK_E_JIT;
  }
  nvrtcProgram_t prog = nullptr;
  nvrtcResult_t r = g_nv.CreateProgram(&prog, source, name ? name : "drk_jit.cu", 0, nullptr, nullptr);
  if (r != 0) {
    log = std::string("nvrtcCreateProgram: ") + g_nv.GetErrorString(r);
    return DRK_E_JIT;
  }
  std::string inc = std::string("-I") + (include_dir ? include_dir : ".");
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-fmad=false", "-lineinfo",
                        inc.c_str()};
  r = g_nv.CompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t ls = 0;
  g_nv.GetProgramLogSize(prog, &ls);
  if (ls > 1) {
    std::string l(ls, '\0');
    g_nv.GetProgramLog(prog, &l[0]);
    log = l;
  }
  if (r != 0) {
    log = std::string("nvrtcCompileProgram: ") + g_nv.GetErrorString(r) + "\n" + log;
    g_nv.DestroyProgram(&prog);
    return DRK_E_JIT;
  }
  size_t cs = 0;
  g_nv.GetCUBINSize(prog, &cs);
  cubin.resize(cs);
  g_nv.GetCUBIN(prog, cubin.data());
  g_nv.DestroyProgram(&prog);
  return 0;
}

}  // namespace

extern "C" int drk_jit_cubin(const char* source, const char* name, const char* include_dir, void* cubin_out,
                             size_t* cubin_bytes, char* log, size_t log_bytes) {
  if (!source || !cubin_bytes) return jit_error(DRK_E_ARG, "drk_jit_cubin: null argument");
  std::vector<char> cubin;
  std::string l;
  int rc = compile_cubin(source, name, include_dir, cubin, l);
  copy_log(l, log, log_bytes);
  if (rc) return rc;
  if (cubin_out) {
    if (*cubin_bytes < cubin.size()) {
      *cubin_bytes = cubin.size();
      return DRK_E_ARG;
    }
    memcpy(cubin_out, cubin.data(), cubin.size());
  }
  *cubin_bytes = cubin.size();
  return 0;
}

extern "C" int drk_jit_load(const void* cubin, void** handle) {
  if (!cubin || !handle) return jit_error(DRK_E_ARG, "drk_jit_load: null argument");
  cudaLibrary_t lib = nullptr;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) return jit_error((int)e, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
  *handle = (void*)lib;
  return 0;
}

extern "C" int drk_jit_compile(const char* source, const char* name, const char* include_dir, void** handle,
                               char* log, size_t log_bytes) {
  if (!source || !handle) return jit_error(DRK_E_ARG, "drk_jit_compile: null argument");
  std::vector<char> cubin;
  std::string l;
  int rc = compile_cubin(source, name, include_dir, cubin, l);
  copy_log(l, log, log_bytes);
  if (rc) return rc;
  return drk_jit_load(cubin.data(), handle);
}

static int get_kernel(void* handle, const char* kernel, cudaKernel_t* k) {
  if (!handle || !kernel) return jit_error(DRK_E_ARG, "drk_jit: null handle/kernel");
  cudaError_t e = cudaLibraryGetKernel(k, (cudaLibrary_t)handle, kernel);
  if (e != cudaSuccess)
    return jit_error((int)e, std::string("cudaLibraryGetKernel(") + kernel + "): " + cudaGetErrorString(e));
  return 0;
}

extern "C" int64_t drk_note_launch(void);

// the kernel `kernel` of module `handle` as a function pointer for cudaLaunchKernelExC
// (libdrk's own launchers of NVRTC scans, drk_jit_scan_view)
extern "C" int drk_get_jit_kernel(void* handle, const char* kernel, const void** fn) {
  cudaKernel_t k;
  if (int rc = get_kernel(handle, kernel, &k)) return rc;
  *fn = (const void*)k;
  return 0;
}

extern "C" int drk_jit_launch(void* handle, const char* kernel, unsigned grid, unsigned block, unsigned smem,
                              const void* params, size_t params_bytes, int device, void* stream) {
  (void)params_bytes;
  cudaKernel_t k;
  if (int rc = get_kernel(handle, kernel, &k)) return rc;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return jit_error((int)e, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  void* args[] = {const_cast<void*>(params)};
  cudaError_t e = cudaLaunchKernel((const void*)k, dim3(grid), dim3(block), args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return jit_error((int)e, std::string("cudaLaunchKernel: ") + cudaGetErrorString(e));
  drk_note_launch();
  return 0;
}

extern "C" int drk_jit_occupancy(void* handle, const char* kernel, unsigned block, unsigned smem, int device,
                                 int* blocks_per_sm, int* sm_count) {
  cudaKernel_t k;
  if (int rc = get_kernel(handle, kernel, &k)) return rc;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) cudaSetDevice(device);
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, (const void*)k, (int)block, (size_t)smem);
  if (e != cudaSuccess) return jit_error((int)e, std::string("occupancy: ") + cudaGetErrorString(e));
  if (blocks_per_sm) *blocks_per_sm = n;
  if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device);
  return 0;
}

extern "C" const char* drk_jit_last_error(void) { return g_jit_error.c_str(); }
