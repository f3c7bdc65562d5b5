// drk_kernels.cu — ahead-of-time sm_100a kernels and the C ABI declared in include/drk.h.
//
// Hot-path kernels of the distributed-ranges shp runtime (reference: segrange, pure
// Python/numpy; see the per-entry citations in include/drk.h).  All kernels are
// HBM-bandwidth bound streaming kernels; nothing here is a contraction, so there are no
// tensor-core paths.  Template machinery lives in drk_device.cuh (shared with NVRTC).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "drk_host.h"

using namespace drk;

// ---------------------------------------------------------------------------------------
// error plumbing

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

namespace drk_host {
int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  return set_error((int)e, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace drk_host
using namespace drk_host;

extern "C" const char* drk_last_error(void) { return g_last_error.c_str(); }
int drk_error(int code, const char* msg) { return set_error(code, msg); }
int drk_cuda_error(cudaError_t e, const char* what) { return cuda_status(e, what); }
extern "C" int drk_version(void) { return 1; }
extern "C" int64_t drk_launch_count(void) { return g_launches.load(); }
extern "C" int64_t drk_note_launch(void) { return g_launches.fetch_add(1) + 1; }

int g_memcpy_chunk = 256;  // MiB per cudaMemcpyAsync of drk_memcpy_async (0: one copy); e2e 131.9 -> 141.1 GB/s

extern "C" int drk_memcpy_async(void* dst, const void* src, size_t bytes, int device, void* stream) {
  if (bytes == 0) return 0;
  if (!dst || !src) return set_error(DRK_E_ARG, "drk_memcpy_async: null pointer");
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) DRK_CHECK(cudaSetDevice(device));
  // large host<->device copies go as a train of chunks: with both PCIe directions busy
  // (bench e2e) the copy engines interleave chunk trains better than two multi-GB copies
  const size_t chunk = g_memcpy_chunk > 0 ? ((size_t)g_memcpy_chunk << 20) : bytes;
  for (size_t off = 0; off < bytes; off += chunk) {
    const size_t b = bytes - off < chunk ? bytes - off : chunk;
    DRK_CHECK(cudaMemcpyAsync((char*)dst + off, (const char*)src + off, b, cudaMemcpyDefault, (cudaStream_t)stream));
  }
  return 0;
}

// Result readback through the SMs: a few 8-byte words stored straight into mapped pinned
// host memory.  A cudaMemcpyAsync D2H of 8 bytes would queue on the copy engine behind any
// multi-GB download in flight on another stream (bench.py e2e), stalling the compute stream.
__global__ void readback_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                                int words) {
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}

extern "C" int drk_readback(void* host_dst, const void* dev_src, size_t bytes, int device, void* stream) {
  if (bytes == 0) return 0;
  if (!host_dst || !dev_src) return set_error(DRK_E_ARG, "drk_readback: null pointer");
  if (bytes % 8) return set_error(DRK_E_ARG, "drk_readback: bytes must be a multiple of 8");
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) DRK_CHECK(cudaSetDevice(device));
  void* dptr = nullptr;
  DRK_CHECK(cudaHostGetDevicePointer(&dptr, host_dst, 0));  // fails unless host_dst is mapped pinned memory
  const int words = (int)(bytes / 8);
  readback_kernel<<<1, words < 256 ? ((words + 31) / 32) * 32 : 256, 0, (cudaStream_t)stream>>>(
      (unsigned long long*)dptr, (const unsigned long long*)dev_src, words);
  g_launches.fetch_add(1);
  DRK_CHECK(cudaGetLastError());
  return 0;
}

extern "C" int drk_mapped_ptr(const void* host, void** dev) {
  if (!host || !dev) return set_error(DRK_E_ARG, "drk_mapped_ptr: null pointer");
  DRK_CHECK(cudaHostGetDevicePointer(dev, const_cast<void*>(host), 0));
  return 0;
}

extern "C" int drk_memset_async(void* dst, int value, size_t bytes, int device, void* stream) {
  if (bytes == 0) return 0;
  if (!dst) return set_error(DRK_E_ARG, "drk_memset_async: null pointer");
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) DRK_CHECK(cudaSetDevice(device));
  DRK_CHECK(cudaMemsetAsync(dst, value, bytes, (cudaStream_t)stream));
  return 0;
}

extern "C" int drk_stream_synchronize(int device, void* stream) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) DRK_CHECK(cudaSetDevice(device));
  DRK_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

extern "C" int drk_enable_peer_access(int device, int peer) {
  int can = 0;
  DRK_CHECK(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return set_error(DRK_E_ARG, "drk_enable_peer_access: devices cannot access each other");
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) DRK_CHECK(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  return cuda_status(e, "cudaDeviceEnablePeerAccess");
}

extern "C" int drk_device_count(int* count) {
  if (!count) return set_error(DRK_E_ARG, "drk_device_count: null count");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    *count = 0;
    return 0;
  }
  return cuda_status(e, "cudaGetDeviceCount");
}

// ---------------------------------------------------------------------------------------
// launch geometry and knobs (declared in drk_host.h)

namespace drk_host {
std::mutex g_mu;
int g_map_waves = 0;
int g_reduce_waves = 1;
int g_reduce_grid = 0;  // experiments: cap on the reduce grid (0: SMs x occupancy x waves)
int g_scan_sub = 0;  // 0: by segment size (drk_scan.cu)
int g_scan_l2dyn = 1;
int g_scan_l2_min = 1 << 22;
int g_scan_l2_subs = 0;
int g_scan_l2_pre = 2;
int g_scan_l2_ring = 3;
int g_scan_debug = 0;
int g_scan_stagger = -1;
int g_scan_smem_pad = 0;
int g_scan_rescan_pol = 0;
int g_scan_keep_tail = 1;
int g_scan_lb_snap = 0;
int g_scan_2p_lo_kb = 0, g_scan_2p_hi_kb = 0;
thread_local int g_chain_launch = 0;
void* g_scan_trace = nullptr;

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
      v = 148;
    cache[device] = v;
  }
  return cache[device];
}

int epilogue(const char* what) {
  g_launches.fetch_add(1);
  return cuda_status(cudaGetLastError(), what);
}

// Per-scratch launch epochs (tile descriptors of older launches then read as stale).
static std::unordered_map<uintptr_t, uint64_t> g_scan_epochs;
uint64_t next_epoch(void* scratch) {
  std::lock_guard<std::mutex> lk(g_mu);
  return ++g_scan_epochs[(uintptr_t)scratch];
}
}  // namespace drk_host

extern "C" int drk_scan_set_trace(void* buf) {
  g_scan_trace = buf;
  return 0;
}

extern "C" int drk_tune(const char* name, int value) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!name) return -1;
  int old = -1;
  if (!strcmp(name, "map_waves")) {
    old = g_map_waves;
    g_map_waves = value;
  } else if (!strcmp(name, "reduce_grid")) {
    old = g_reduce_grid;
    g_reduce_grid = value;
  } else if (!strcmp(name, "reduce_waves")) {
    old = g_reduce_waves;
    g_reduce_waves = value;
  } else if (!strcmp(name, "scan_l2dyn")) {
    old = g_scan_l2dyn;
    g_scan_l2dyn = value;
  } else if (!strcmp(name, "scan_l2_subs")) {
    old = g_scan_l2_subs;
    g_scan_l2_subs = value;
  } else if (!strcmp(name, "scan_l2_ring")) {
    old = g_scan_l2_ring;
    g_scan_l2_ring = value;
  } else if (!strcmp(name, "scan_l2_pre")) {
    old = g_scan_l2_pre;
    g_scan_l2_pre = value;
  } else if (!strcmp(name, "scan_stagger")) {
    old = g_scan_stagger;
    g_scan_stagger = value;
  } else if (!strcmp(name, "scan_debug")) {
    old = g_scan_debug;
    g_scan_debug = value;
  } else if (!strcmp(name, "scan_l2_min")) {
    old = g_scan_l2_min;
    g_scan_l2_min = value;
  } else if (!strcmp(name, "scan_smem_pad")) {
    old = g_scan_smem_pad;
    g_scan_smem_pad = value;
  } else if (!strcmp(name, "memcpy_chunk_mb")) {
    old = g_memcpy_chunk;
    g_memcpy_chunk = value;
  } else if (!strcmp(name, "scan_2p_lo_kb")) {
    old = g_scan_2p_lo_kb;
    g_scan_2p_lo_kb = value;
  } else if (!strcmp(name, "scan_2p_hi_kb")) {
    old = g_scan_2p_hi_kb;
    g_scan_2p_hi_kb = value;
  } else if (!strcmp(name, "scan_lb_snap")) {
    old = g_scan_lb_snap;
    g_scan_lb_snap = value;
  } else if (!strcmp(name, "scan_keep_tail")) {
    old = g_scan_keep_tail;
    g_scan_keep_tail = value;
  } else if (!strcmp(name, "scan_rescan_pol")) {
    old = g_scan_rescan_pol;
    g_scan_rescan_pol = value;
  } else if (!strcmp(name, "l2_persist_mb")) {
    // persisting-L2 set-aside of the current device (evict_last lines): experiments
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    old = (int)(cur >> 20);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)value << 20);
  } else if (!strcmp(name, "scan_sub")) {
    old = g_scan_sub;
    if (value >= 0 && value <= 4) g_scan_sub = value;
  }
  return old;
}

// ---------------------------------------------------------------------------------------
// map functors

template <class T> struct CopyF {
  struct Params {
    T* out;
    const T* in;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {
    T a[E];
  };
  static __device__ __forceinline__ void load(const Params& p, i64 i, Regs& r) { ldv<T, E>(p.in + i, r.a); }
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs& r) { stv<T, E>(p.out + i, r.a); }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) { p.out[i] = p.in[i]; }
};

template <class T> struct FillF {
  struct Params {
    T* out;
    T value;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {};
  static __device__ __forceinline__ void load(const Params&, i64, Regs&) {}
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs&) {
    T a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = p.value;
    stv<T, E>(p.out + i, a);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) { p.out[i] = p.value; }
};

template <class T> struct IotaF {
  struct Params {
    T* out;
    i64 start;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {};
  static __device__ __forceinline__ void load(const Params&, i64, Regs&) {}
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs&) {
    T a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = (T)(p.start + i + e);
    stv<T, E>(p.out + i, a);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) { p.out[i] = (T)(p.start + i); }
};

template <class T> struct ScaleF {
  struct Params {
    T* out;
    const T* in;
    T alpha;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {
    T a[E];
  };
  static __device__ __forceinline__ void load(const Params& p, i64 i, Regs& r) { ldv<T, E>(p.in + i, r.a); }
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs& r) {
    T o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = Arith<T>::mul(p.alpha, r.a[e]);
    stv<T, E>(p.out + i, o);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) {
    p.out[i] = Arith<T>::mul(p.alpha, p.in[i]);
  }
};

template <class T> struct AddF {
  struct Params {
    T* out;
    const T* a;
    const T* b;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {
    T a[E], b[E];
  };
  static __device__ __forceinline__ void load(const Params& p, i64 i, Regs& r) {
    ldv<T, E>(p.a + i, r.a);
    ldv<T, E>(p.b + i, r.b);
  }
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs& r) {
    T o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = Arith<T>::add(r.a[e], r.b[e]);
    stv<T, E>(p.out + i, o);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) {
    p.out[i] = Arith<T>::add(p.a[i], p.b[i]);
  }
};

#ifndef BS_E
#define BS_E 2  // 16-byte vectors per operand per thread (ILP of the transcendental chain)
#endif

// a = b + alpha * c with numpy's two roundings (weak-scalar alpha already in T).
template <class T> struct TriadF {
  struct Params {
    T* out;
    const T* b;
    const T* c;
    T alpha;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {
    T b[E], c[E];
  };
  static __device__ __forceinline__ void load(const Params& p, i64 i, Regs& r) {
    ldv<T, E>(p.b + i, r.b);
    ldv<T, E>(p.c + i, r.c);
  }
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs& r) {
    T o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = Arith<T>::add(r.b[e], Arith<T>::mul(p.alpha, r.c[e]));
    stv<T, E>(p.out + i, o);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) {
    p.out[i] = Arith<T>::add(p.b[i], Arith<T>::mul(p.alpha, p.c[i]));
  }
};

template <class T, class M = BSMath<T>> struct BlackScholesF {
  struct Params {
    T* out;
    const T *S, *K, *r, *v, *t;
  };
  // the fp32 SFU tier needs ILP (BS_E vectors per thread); the fp64 reference chain is
  // register-bound, so it runs one vector per thread and more warps
#ifndef BS_REF_E
#define BS_REF_E 1
#endif
  static constexpr int E = (is_same<M, BSMath<T>>::value ? BS_E : BS_REF_E) * 16 / sizeof(T);
#ifndef BS_REF_MINB
#define BS_REF_MINB 4
#endif
  static constexpr int MINB = is_same<M, BSMath<T>>::value ? 0 : BS_REF_MINB;
  static constexpr int U = 1;  // transcendental-heavy: fewer registers, more warps
  struct Regs {
    T S[E], K[E], r[E], v[E], t[E];
  };
  static __device__ __forceinline__ void load(const Params& p, i64 i, Regs& g) {
    ldv<T, E>(p.S + i, g.S);
    ldv<T, E>(p.K + i, g.K);
    ldv<T, E>(p.r + i, g.r);
    ldv<T, E>(p.v + i, g.v);
    ldv<T, E>(p.t + i, g.t);
  }
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs& g) {
    T o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = M::price(g.S[e], g.K[e], g.r[e], g.v[e], g.t[e]);
    stv<T, E>(p.out + i, o);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) {
    p.out[i] = M::price(p.S[i], p.K[i], p.r[i], p.v[i], p.t[i]);
  }
};

// splitmix64 (repro.py:21-30): draw i of stream `seed` mixes seed + (i+1)*golden.
__device__ __forceinline__ u64 splitmix64_at(u64 seed, u64 i) {
  u64 z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <class T> struct GenF {
  struct Params {
    T* out;
    u64 seed, start;
    int kind;
    double a, b;
  };
  static constexpr int E = 16 / sizeof(T);
  struct Regs {};
  static __device__ __forceinline__ T gen(const Params& p, i64 i) {
    const u64 bits = splitmix64_at(p.seed, p.start + (u64)i);
    if (p.kind == DRK_GEN_UNIFORM) {
      // unit_doubles: (bits >> 11) * 2^-53, exact; uniform: lo + (hi - lo) * u (two roundings)
      double u = (double)(bits >> 11) * 1.1102230246251565e-16;
      if (!(p.a == 0.0 && p.b == 1.0)) u = __dadd_rn(p.a, __dmul_rn(__dsub_rn(p.b, p.a), u));
      return (T)u;
    }
    const i64 m = (i64)(bits % (u64)p.a);
    return (T)(m + (i64)p.b);
  }
  static __device__ __forceinline__ void load(const Params&, i64, Regs&) {}
  static __device__ __forceinline__ void store(const Params& p, i64 i, const Regs&) {
    T a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = gen(p, i + e);
    stv<T, E>(p.out + i, a);
  }
  static __device__ __forceinline__ void scalar(const Params& p, i64 i) { p.out[i] = gen(p, i); }
};

template <class F, class = void> struct UnrollOf { static constexpr int value = MAP_U; };
template <class F> struct UnrollOf<F, decltype((void)F::U, void())> { static constexpr int value = F::U; };

template <class F>
static int launch_map(const typename F::Params& p, int64_t n, bool vec_ok, int device, void* stream,
                      const char* what) {
  if (n < 0) return set_error(DRK_E_ARG, std::string(what) + ": negative length");
  if (n == 0) return 0;
  if (int rc = prologue(device, what)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int sms = sm_count(device);
  if (vec_ok) {
    constexpr int U = UnrollOf<F>::value;
    auto k = map_vec_fn<F, BLOCK, U>();
    const int64_t nchunk = n / F::E;
    int64_t grid = (nchunk + (int64_t)BLOCK * U - 1) / ((int64_t)BLOCK * U);
    if (g_map_waves > 0) {
      const int64_t cap = (int64_t)sms * occupancy(k, BLOCK, 0) * g_map_waves;
      if (grid > cap) grid = cap;
    }
    // the scalar tail (n % E elements) is handled by the first threads of the grid
    if (grid < 1) grid = 1;
    if (grid > 0x7fffffff) grid = 0x7fffffff;
    k<<<(unsigned)grid, BLOCK, 0, s>>>(p, n);
  } else {
    auto k = map_striped_fn<F, BLOCK, MAP_U>();
    int64_t grid = (n + (int64_t)BLOCK * MAP_U - 1) / ((int64_t)BLOCK * MAP_U);
    const int64_t cap = (int64_t)sms * occupancy(k, BLOCK, 0) * 8;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    k<<<(unsigned)grid, BLOCK, 0, s>>>(p, n);
  }
  return epilogue(what);
}

static int need(const void* p, const char* what, const char* arg) {
  if (!p) return set_error(DRK_E_ARG, std::string(what) + ": null " + arg);
  return 0;
}

extern "C" int drk_copy(int dtype, void* out, const void* in, int64_t n, int device, void* stream) {
  if (n > 0 && (need(out, "drk_copy", "out") || need(in, "drk_copy", "in"))) return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_copy", T, {
    typename CopyF<T>::Params p{(T*)out, (const T*)in};
    return launch_map<CopyF<T>>(p, n, aligned16(out) && aligned16(in), device, stream, "drk_copy");
  });
}

extern "C" int drk_fill(int dtype, void* out, int64_t n, const void* value, int device, void* stream) {
  if (need(value, "drk_fill", "value")) return DRK_E_ARG;
  if (n > 0 && need(out, "drk_fill", "out")) return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_fill", T, {
    typename FillF<T>::Params p{(T*)out, *(const T*)value};
    return launch_map<FillF<T>>(p, n, aligned16(out), device, stream, "drk_fill");
  });
}

extern "C" int drk_iota(int dtype, void* out, int64_t n, int64_t start, int device, void* stream) {
  if (n > 0 && need(out, "drk_iota", "out")) return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_iota", T, {
    typename IotaF<T>::Params p{(T*)out, start};
    return launch_map<IotaF<T>>(p, n, aligned16(out), device, stream, "drk_iota");
  });
}

extern "C" int drk_scale(int dtype, void* out, const void* in, int64_t n, const void* alpha, int device,
                         void* stream) {
  if (need(alpha, "drk_scale", "alpha")) return DRK_E_ARG;
  if (n > 0 && (need(out, "drk_scale", "out") || need(in, "drk_scale", "in"))) return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_scale", T, {
    typename ScaleF<T>::Params p{(T*)out, (const T*)in, *(const T*)alpha};
    return launch_map<ScaleF<T>>(p, n, aligned16(out) && aligned16(in), device, stream, "drk_scale");
  });
}

extern "C" int drk_add(int dtype, void* out, const void* a, const void* b, int64_t n, int device,
                       void* stream) {
  if (n > 0 && (need(out, "drk_add", "out") || need(a, "drk_add", "a") || need(b, "drk_add", "b")))
    return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_add", T, {
    typename AddF<T>::Params p{(T*)out, (const T*)a, (const T*)b};
    return launch_map<AddF<T>>(p, n, aligned16(out) && aligned16(a) && aligned16(b), device, stream,
                               "drk_add");
  });
}

extern "C" int drk_triad(int dtype, void* out, const void* b, const void* c, int64_t n, const void* alpha,
                         int device, void* stream) {
  if (need(alpha, "drk_triad", "alpha")) return DRK_E_ARG;
  if (n > 0 && (need(out, "drk_triad", "out") || need(b, "drk_triad", "b") || need(c, "drk_triad", "c")))
    return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_triad", T, {
    typename TriadF<T>::Params p{(T*)out, (const T*)b, (const T*)c, *(const T*)alpha};
    return launch_map<TriadF<T>>(p, n, aligned16(out) && aligned16(b) && aligned16(c), device, stream,
                                 "drk_triad");
  });
}

extern "C" int drk_black_scholes_ex(int dtype, int flags, void* out, const void* S, const void* K, const void* r,
                                    const void* v, const void* t, int64_t n, int device, void* stream) {
  if (n > 0 && (need(out, "drk_black_scholes", "out") || need(S, "drk_black_scholes", "spot") ||
                need(K, "drk_black_scholes", "strike") || need(r, "drk_black_scholes", "rate") ||
                need(v, "drk_black_scholes", "volatility") || need(t, "drk_black_scholes", "expiry")))
    return DRK_E_ARG;
  if (flags & ~DRK_BS_FAST) return set_error(DRK_E_ARG, "drk_black_scholes: unknown flags");
  DRK_DISPATCH_FLOAT(dtype, "drk_black_scholes", T, {
    const bool al = aligned16(out) && aligned16(S) && aligned16(K) && aligned16(r) && aligned16(v) &&
                    aligned16(t);
    if (flags & DRK_BS_FAST) {
      typename BlackScholesF<T>::Params p{(T*)out, (const T*)S, (const T*)K, (const T*)r, (const T*)v,
                                          (const T*)t};
      return launch_map<BlackScholesF<T>>(p, n, al, device, stream, "drk_black_scholes");
    }
    typename BlackScholesF<T, BSRef<T>>::Params p{(T*)out, (const T*)S, (const T*)K, (const T*)r, (const T*)v,
                                                   (const T*)t};
    return launch_map<BlackScholesF<T, BSRef<T>>>(p, n, al, device, stream, "drk_black_scholes");
  });
}

extern "C" int drk_black_scholes(int dtype, void* out, const void* S, const void* K, const void* r,
                                 const void* v, const void* t, int64_t n, int device, void* stream) {
  return drk_black_scholes_ex(dtype, 0, out, S, K, r, v, t, n, device, stream);
}

extern "C" int drk_generate(int dtype, void* out, int64_t n, uint64_t seed, uint64_t start, int kind,
                            double a, double b, int device, void* stream) {
  if (n > 0 && need(out, "drk_generate", "out")) return DRK_E_ARG;
  if (kind != DRK_GEN_UNIFORM && kind != DRK_GEN_MOD)
    return set_error(DRK_E_ARG, "drk_generate: unknown kind");
  if (kind == DRK_GEN_MOD && !(a >= 1.0)) return set_error(DRK_E_ARG, "drk_generate: modulus must be >= 1");
  DRK_DISPATCH(dtype, "drk_generate", T, {
    typename GenF<T>::Params p{(T*)out, seed, start, kind, a, b};
    return launch_map<GenF<T>>(p, n, aligned16(out), device, stream, "drk_generate");
  });
}

// ---------------------------------------------------------------------------------------
// reductions

template <class T> struct IdentLoad {
  typedef T V;
  struct Params {
    const T* x;
  };
  static constexpr int E = 16 / sizeof(T);
  static __device__ __forceinline__ void load(const Params& p, i64 i, T (&v)[E]) { ldv<T, E>(p.x + i, v); }
  static __device__ __forceinline__ T one(const Params& p, i64 i) { return p.x[i]; }
};

// x[i] * y[i] rounded in T, as numpy's `t[0] * t[1]` temporary (bench.py:89).
template <class T> struct ProdLoad {
  typedef T V;
  struct Params {
    const T* x;
    const T* y;
  };
  static constexpr int E = 16 / sizeof(T);
  static __device__ __forceinline__ void load(const Params& p, i64 i, T (&v)[E]) {
    T a[E], b[E];
    ldv<T, E>(p.x + i, a);
    ldv<T, E>(p.y + i, b);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = Arith<T>::mul(a[e], b[e]);
  }
  static __device__ __forceinline__ T one(const Params& p, i64 i) { return Arith<T>::mul(p.x[i], p.y[i]); }
};

extern "C" size_t drk_reduce_scratch_bytes(void) {
  return 128 + (size_t)MAX_RED_GRID * (8 + 4);
}

static int acc_code(int dtype, int op) {
  const bool widen = (op == DRK_ADD || op == DRK_MUL);
  switch (dtype) {
    case DRK_F32: return widen ? DRK_F64 : DRK_F32;
    case DRK_F64: return DRK_F64;
    case DRK_I32: return widen ? DRK_I64 : DRK_I32;
    case DRK_I64: return DRK_I64;
  }
  return -1;
}
extern "C" int drk_acc_dtype(int dtype, int op) { return acc_code(dtype, op); }

static ReduceScratch carve_reduce(void* scratch) {
  ReduceScratch s;
  char* b = (char*)scratch;
  s.counter = (u32*)b;
  s.partials = (void*)(b + 128);
  s.has = (int*)(b + 128 + (size_t)MAX_RED_GRID * 8);
  return s;
}

template <class LD, class Op>
static int launch_reduce(const typename LD::Params& p, int64_t n, bool vec_ok, void* result, void* scratch,
                         int device, void* stream, const char* what) {
  typedef typename WideAcc<typename LD::V, Op>::type A;
  if (n < 1) return set_error(DRK_E_ARG, std::string(what) + ": n must be >= 1");
  if (!result || !scratch) return set_error(DRK_E_ARG, std::string(what) + ": null result/scratch");
  if (int rc = prologue(device, what)) return rc;
  auto k = reduce_kernel<LD, Op, BLOCK, RED_U>;
  const int64_t work = vec_ok ? (n / LD::E) * 1 + 1 : n;
  int64_t grid = (work + (int64_t)BLOCK * RED_U - 1) / ((int64_t)BLOCK * RED_U);
  const int64_t cap = (int64_t)sm_count(device) * occupancy(k, BLOCK, 0) * (g_reduce_waves > 0 ? g_reduce_waves : 1);
  if (grid > cap) grid = cap;
  if (grid > MAX_RED_GRID) grid = MAX_RED_GRID;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, BLOCK, 0, (cudaStream_t)stream>>>(p, n, vec_ok ? 1 : 0, carve_reduce(scratch), (A*)result,
                                                       nullptr);
  return epilogue(what);
}

template <class T>
static int reduce_op(int op, const T* x, int64_t n, void* result, void* scratch, int device, void* stream) {
  typename IdentLoad<T>::Params p{x};
  const bool v = aligned16(x);
  switch (op) {
    case DRK_ADD: return launch_reduce<IdentLoad<T>, OpAdd>(p, n, v, result, scratch, device, stream, "drk_reduce");
    case DRK_MUL: return launch_reduce<IdentLoad<T>, OpMul>(p, n, v, result, scratch, device, stream, "drk_reduce");
    case DRK_MIN: return launch_reduce<IdentLoad<T>, OpMin>(p, n, v, result, scratch, device, stream, "drk_reduce");
    case DRK_MAX: return launch_reduce<IdentLoad<T>, OpMax>(p, n, v, result, scratch, device, stream, "drk_reduce");
  }
  return set_error(DRK_E_ARG, "drk_reduce: unknown op");
}

extern "C" int drk_reduce(int dtype, int op, const void* x, int64_t n, void* result_dev, void* scratch,
                          int device, void* stream) {
  if (need(x, "drk_reduce", "x")) return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_reduce", T, { return reduce_op<T>(op, (const T*)x, n, result_dev, scratch, device, stream); });
}

// Batched reductions: the segments of a vector that share a GPU reduced by one launch; the
// one wave of CTAs is split between the segments in proportion to their lengths, and each
// segment folds its own CTA partials (same determinism as drk_reduce).  `results` gets one
// 8-byte slot per segment, `scratch` nseg x drk_reduce_scratch_bytes().
// the fused cross-GPU combine of one call (FusedCombine in drk_device.cuh), host side
struct FusedSpec {
  void* slots;
  u32* counter;
  u32 total;
  u64 init_bits;
  void* result;
  u64* flag;
  u64 epoch;
  const int* gslot;  // global slot of each of this launch's segments
};

template <class LD, class Op>
static int launch_reduce_batch(int nseg, const typename LD::Params* ps, const int64_t* ns, const bool* vec_ok,
                               void* results, void* flags, uint64_t epoch, void* scratch, int device, void* stream,
                               const char* what, const FusedSpec* fs = nullptr) {
  typedef typename WideAcc<typename LD::V, Op>::type A;
  if (nseg < 1 || nseg > DRK_RED_SEGS) return set_error(DRK_E_ARG, std::string(what) + ": nseg out of range");
  if (!results || !scratch) return set_error(DRK_E_ARG, std::string(what) + ": null results/scratch");
  int64_t total = 0;
  for (int k = 0; k < nseg; ++k) {
    if (ns[k] < 1) return set_error(DRK_E_ARG, std::string(what) + ": empty segment");
    total += ns[k];
  }
  if (int rc = prologue(device, what)) return rc;
  auto kern = reduce_batch_kernel<LD, Op, BLOCK, RED_U>;
  int64_t cap = (int64_t)sm_count(device) * occupancy(kern, BLOCK, 0) * (g_reduce_waves > 0 ? g_reduce_waves : 1);
  if (g_reduce_grid > 0 && cap > g_reduce_grid) cap = g_reduce_grid;
  ReduceBatch<LD, A> b;
  memset(&b, 0, sizeof(b));
  b.nseg = nseg;
  u32 first = 0;
  const size_t sbytes = 128 + (size_t)MAX_RED_GRID * (8 + 4);
  for (int k = 0; k < nseg; ++k) {
    const int64_t work = vec_ok[k] ? (ns[k] / LD::E) + 1 : ns[k];
    int64_t g = (work + (int64_t)BLOCK * RED_U - 1) / ((int64_t)BLOCK * RED_U);
    const int64_t share = (cap * ns[k] + total - 1) / total;
    if (g > share) g = share;
    if (g > MAX_RED_GRID) g = MAX_RED_GRID;
    if (g < 1) g = 1;
    b.cta_first[k] = first;
    first += (u32)g;
    b.p[k] = ps[k];
    b.n[k] = ns[k];
    b.vec_ok[k] = vec_ok[k] ? 1 : 0;
    b.s[k] = carve_reduce((char*)scratch + (size_t)k * sbytes);
    b.result[k] = (A*)((char*)results + 8 * (size_t)k);
    b.flag[k] = flags ? (u64*)flags + k : nullptr;
    if (fs) b.gslot[k] = (u32)fs->gslot[k];
  }
  b.epoch = epoch;
  if (fs) {
    b.fused = 1;
    b.fc.slots = (A*)fs->slots;
    b.fc.counter = fs->counter;
    b.fc.total = fs->total;
    b.fc.init_bits = fs->init_bits;
    b.fc.result = fs->result;
    b.fc.flag = fs->flag;
    b.fc.epoch = fs->epoch;
  }
  b.cta_first[nseg] = first;
  kern<<<first, BLOCK, 0, (cudaStream_t)stream>>>(b);
  return epilogue(what);
}

template <class T>
static int reduce_batch_op(int op, int nseg, const void* const* xs, const int64_t* ns, void* results, void* flags,
                           uint64_t epoch, void* scratch, int device, void* stream, const FusedSpec* fs = nullptr) {
  typename IdentLoad<T>::Params ps[DRK_RED_SEGS];
  bool v[DRK_RED_SEGS];
  if (nseg < 1 || nseg > DRK_RED_SEGS) return set_error(DRK_E_ARG, "drk_reduce_batch: nseg out of range");
  for (int k = 0; k < nseg; ++k) {
    if (!xs[k]) return set_error(DRK_E_ARG, "drk_reduce_batch: null segment");
    ps[k].x = (const T*)xs[k];
    v[k] = aligned16(xs[k]);
  }
  const char* w = "drk_reduce_batch";
  switch (op) {
    case DRK_ADD: return launch_reduce_batch<IdentLoad<T>, OpAdd>(nseg, ps, ns, v, results, flags, epoch, scratch, device, stream, w, fs);
    case DRK_MUL: return launch_reduce_batch<IdentLoad<T>, OpMul>(nseg, ps, ns, v, results, flags, epoch, scratch, device, stream, w, fs);
    case DRK_MIN: return launch_reduce_batch<IdentLoad<T>, OpMin>(nseg, ps, ns, v, results, flags, epoch, scratch, device, stream, w, fs);
    case DRK_MAX: return launch_reduce_batch<IdentLoad<T>, OpMax>(nseg, ps, ns, v, results, flags, epoch, scratch, device, stream, w, fs);
  }
  return set_error(DRK_E_ARG, "drk_reduce_batch: unknown op");
}

extern "C" int drk_reduce_batch_ex(int dtype, int op, int nseg, const void* const* xs, const int64_t* ns,
                                   void* results, void* flags, uint64_t epoch, void* scratch, int device,
                                   void* stream) {
  if (!xs || !ns) return set_error(DRK_E_ARG, "drk_reduce_batch: null segment arrays");
  DRK_DISPATCH(dtype, "drk_reduce_batch", T,
               { return reduce_batch_op<T>(op, nseg, xs, ns, results, flags, epoch, scratch, device, stream); });
}

extern "C" int drk_reduce_batch(int dtype, int op, int nseg, const void* const* xs, const int64_t* ns, void* results,
                                void* scratch, int device, void* stream) {
  return drk_reduce_batch_ex(dtype, op, nseg, xs, ns, results, nullptr, 0, scratch, device, stream);
}

static int dot_batch_any(int dtype, int nseg, const void* const* xs, const void* const* ys, const int64_t* ns,
                         void* results, void* flags, uint64_t epoch, void* scratch, int device, void* stream,
                         const FusedSpec* fs) {
  if (!xs || !ys || !ns) return set_error(DRK_E_ARG, "drk_dot_batch: null segment arrays");
  if (nseg < 1 || nseg > DRK_RED_SEGS) return set_error(DRK_E_ARG, "drk_dot_batch: nseg out of range");
  DRK_DISPATCH(dtype, "drk_dot_batch", T, {
    typename ProdLoad<T>::Params ps[DRK_RED_SEGS];
    bool v[DRK_RED_SEGS];
    for (int k = 0; k < nseg; ++k) {
      if (!xs[k] || !ys[k]) return set_error(DRK_E_ARG, "drk_dot_batch: null segment");
      ps[k] = typename ProdLoad<T>::Params{(const T*)xs[k], (const T*)ys[k]};
      v[k] = aligned16(xs[k]) && aligned16(ys[k]);
    }
    return launch_reduce_batch<ProdLoad<T>, OpAdd>(nseg, ps, ns, v, results, flags, epoch, scratch, device, stream,
                                                  "drk_dot_batch", fs);
  });
}

extern "C" int drk_dot_batch_ex(int dtype, int nseg, const void* const* xs, const void* const* ys, const int64_t* ns,
                                void* results, void* flags, uint64_t epoch, void* scratch, int device, void* stream) {
  return dot_batch_any(dtype, nseg, xs, ys, ns, results, flags, epoch, scratch, device, stream, nullptr);
}

extern "C" int drk_dot_batch(int dtype, int nseg, const void* const* xs, const void* const* ys, const int64_t* ns,
                             void* results, void* scratch, int device, void* stream) {
  return drk_dot_batch_ex(dtype, nseg, xs, ys, ns, results, nullptr, 0, scratch, device, stream);
}

// Every GPU's batched reduction of one algorithm call in one entry (the multi-device form of
// drk_reduce_batch_ex / drk_dot_batch_ex): segments are listed device by device, counts[d] of
// them for devices[d], and each device gets its own results / flags / scratch.  Arguments of
// every device are validated before anything is enqueued.
extern "C" int drk_reduce_multi(int kind, int dtype, int op, int ndev, const int* devices, void* const* streams,
                                const int* counts, const void* const* xs, const void* const* ys, const int64_t* ns,
                                void* const* results, void* const* flags, uint64_t epoch, void* const* scratch) {
  const char* what = "drk_reduce_multi";
  if (kind != 0 && kind != 1) return set_error(DRK_E_ARG, "drk_reduce_multi: kind must be 0 (reduce) or 1 (dot)");
  if (ndev < 1 || !devices || !streams || !counts || !xs || !ns || !results || !scratch || (kind == 1 && !ys))
    return set_error(DRK_E_ARG, "drk_reduce_multi: null argument");
  int off = 0;
  for (int d = 0; d < ndev; ++d) {
    if (counts[d] < 1 || counts[d] > DRK_RED_SEGS) return set_error(DRK_E_ARG, "drk_reduce_multi: count out of range");
    if (!results[d] || !scratch[d]) return set_error(DRK_E_ARG, "drk_reduce_multi: null result / scratch");
    for (int k = off; k < off + counts[d]; ++k)
      if (!xs[k] || (kind == 1 && !ys[k]) || ns[k] < 1) return set_error(DRK_E_ARG, "drk_reduce_multi: bad segment");
    off += counts[d];
  }
  (void)what;
  off = 0;
  for (int d = 0; d < ndev; ++d) {
    void* f = flags ? flags[d] : nullptr;
    const int rc = kind == 0 ? drk_reduce_batch_ex(dtype, op, counts[d], xs + off, ns + off, results[d], f, epoch,
                                                   scratch[d], devices[d], streams[d])
                             : drk_dot_batch_ex(dtype, counts[d], xs + off, ys + off, ns + off, results[d], f, epoch,
                                                scratch[d], devices[d], streams[d]);
    if (rc) return rc;
    off += counts[d];
  }
  return 0;
}

// CUDA graphs for launch-bound plans: a cached plan that issues several kernels on one stream
// (a vector spread over several locales of one GPU) is captured once and replayed with one
// cudaGraphLaunch.  The capture is thread-local, so other threads' streams are unaffected.
namespace {
struct GraphExec {
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;  // kernels in the graph (drk_launch_count accounting per replay)
  int64_t noted_at_begin = 0;
};
thread_local int64_t g_capture_mark = 0;
}  // namespace

extern "C" int drk_graph_begin(int device, void* stream) {
  if (int rc = prologue(device, "drk_graph_begin")) return rc;
  g_capture_mark = drk_launch_count();
  DRK_CHECK(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return 0;
}

extern "C" int drk_graph_end(int device, void* stream, void** exec) {
  if (!exec) return set_error(DRK_E_ARG, "drk_graph_end: null exec");
  *exec = nullptr;
  if (int rc = prologue(device, "drk_graph_end")) return rc;
  cudaGraph_t graph = nullptr;
  DRK_CHECK(cudaStreamEndCapture((cudaStream_t)stream, &graph));
  cudaGraphExec_t ge = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&ge, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate");
  GraphExec* g = new GraphExec();
  g->exec = ge;
  g->launches = drk_launch_count() - g_capture_mark;
  // the captured launches did not run: take them back out of the launch count
  g_launches.fetch_sub(g->launches);
  *exec = g;
  return 0;
}

extern "C" int drk_graph_launch(void* exec, int device, void* stream) {
  if (!exec) return set_error(DRK_E_ARG, "drk_graph_launch: null exec");
  if (int rc = prologue(device, "drk_graph_launch")) return rc;
  GraphExec* g = (GraphExec*)exec;
  DRK_CHECK(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
  g_launches.fetch_add(g->launches);
  return 0;
}

extern "C" int drk_graph_destroy(void* exec) {
  if (!exec) return 0;
  GraphExec* g = (GraphExec*)exec;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
  return 0;
}

// drk_reduce_multi with the cross-GPU combine fused into the kernels (FusedCombine): segment k
// of the listing stores its partial into home_slots[slot_of[k]] (8-byte slots on devices[0],
// peer memory for the others), and the last CTA of the call folds them in slot order from
// init (partial dtype) into result_host_mapped and sets flag_host_mapped to epoch.  One wait
// on one word, no fold on the host.  home_counter (4 bytes on devices[0]) must be zero.
extern "C" int drk_reduce_fused(int kind, int dtype, int op, int ndev, const int* devices, void* const* streams,
                                const int* counts, const void* const* xs, const void* const* ys, const int64_t* ns,
                                const int* slot_of, void* home_slots, void* home_counter, const void* init,
                                void* result_host_mapped, void* flag_host_mapped, uint64_t epoch,
                                void* const* scratch) {
  if (kind != 0 && kind != 1) return set_error(DRK_E_ARG, "drk_reduce_fused: kind must be 0 (reduce) or 1 (dot)");
  if (ndev < 1 || !devices || !streams || !counts || !xs || !ns || !slot_of || !home_slots || !home_counter ||
      !init || !result_host_mapped || !flag_host_mapped || !scratch || (kind == 1 && !ys))
    return set_error(DRK_E_ARG, "drk_reduce_fused: null argument");
  int total = 0;
  for (int d = 0; d < ndev; ++d) {
    if (counts[d] < 1 || counts[d] > DRK_RED_SEGS) return set_error(DRK_E_ARG, "drk_reduce_fused: count out of range");
    if (!scratch[d]) return set_error(DRK_E_ARG, "drk_reduce_fused: null scratch");
    total += counts[d];
  }
  if (total > DRK_FOLD_MAX) return set_error(DRK_E_ARG, "drk_reduce_fused: more than DRK_FOLD_MAX segments");
  for (int k = 0; k < total; ++k) {
    if (slot_of[k] < 0 || slot_of[k] >= total) return set_error(DRK_E_ARG, "drk_reduce_fused: slot out of range");
    if (!xs[k] || (kind == 1 && !ys[k]) || ns[k] < 1) return set_error(DRK_E_ARG, "drk_reduce_fused: bad segment");
  }
  const int pd = drk_partial_dtype(dtype, op);
  if (pd < 0) return set_error(DRK_E_DTYPE, "drk_reduce_fused: unknown dtype");
  FusedSpec fs;
  fs.slots = home_slots;
  fs.counter = (u32*)home_counter;
  fs.total = (u32)total;
  fs.init_bits = 0;
  memcpy(&fs.init_bits, init, (pd == DRK_F32 || pd == DRK_I32) ? 4 : 8);
  fs.result = result_host_mapped;
  fs.flag = (u64*)flag_host_mapped;
  fs.epoch = epoch;
  int off = 0;
  for (int d = 0; d < ndev; ++d) {
    fs.gslot = slot_of + off;
    int rc;
    if (kind == 0) {
      DRK_DISPATCH(dtype, "drk_reduce_fused", T, {
        rc = reduce_batch_op<T>(op, counts[d], xs + off, ns + off, home_slots, nullptr, 0, scratch[d], devices[d],
                                streams[d], &fs);
        break;
      });
    } else {
      rc = dot_batch_any(dtype, counts[d], xs + off, ys + off, ns + off, home_slots, nullptr, 0, scratch[d],
                         devices[d], streams[d], &fs);
    }
    if (rc) return rc;
    off += counts[d];
  }
  return 0;
}

// Host-side wait for completion words written by a kernel into mapped pinned memory: spin
// (a pause per poll) until every one of `count` words equals `epoch`; the stream is queried
// every few thousand polls so a failed launch surfaces as its error instead of a hang.
extern "C" int drk_wait_flags(const void* host_flags, int count, uint64_t epoch, int device, void* stream) {
  if (count <= 0) return 0;
  if (!host_flags) return set_error(DRK_E_ARG, "drk_wait_flags: null flags");
  const volatile uint64_t* f = (const volatile uint64_t*)host_flags;
  for (uint64_t spins = 1;; ++spins) {
    int k = 0;
    while (k < count && f[k] == epoch) ++k;
    if (k == count) return 0;
    __builtin_ia32_pause();
    if ((spins & 4095) == 0) {
      const cudaError_t e = cudaStreamQuery((cudaStream_t)stream);
      if (e == cudaSuccess) {
        k = 0;
        while (k < count && f[k] == epoch) ++k;
        if (k == count) return 0;
        return set_error(DRK_E_ARG, "drk_wait_flags: the stream is idle but the completion words were not written");
      }
      if (e != cudaErrorNotReady) return cuda_status(e, "drk_wait_flags");
    }
  }
}

extern "C" int drk_dot(int dtype, const void* x, const void* y, int64_t n, void* result_dev, void* scratch,
                       int device, void* stream) {
  if (need(x, "drk_dot", "x") || need(y, "drk_dot", "y")) return DRK_E_ARG;
  DRK_DISPATCH(dtype, "drk_dot", T, {
    typename ProdLoad<T>::Params p{(const T*)x, (const T*)y};
    return launch_reduce<ProdLoad<T>, OpAdd>(p, n, aligned16(x) && aligned16(y), result_dev, scratch, device,
                                             stream, "drk_dot");
  });
}

// ---------------------------------------------------------------------------------------
// cross-segment carry on the device (reference algorithms.py:256-262, the driver's fold of
// segment totals).  A segment's GPU folds the totals of the segments before it straight from
// where they were reduced (peer memory over NVLink, or an all-gathered buffer), so the scan
// of a vector spread over several GPUs needs no host round trip between its two passes.

// identity of the fold, used only when nothing precedes a segment: -0.0 for float sums
// (x + -0.0 == x bit-for-bit, including x = -0.0), 1 for products, +-inf / int limits for
// minimum / maximum
template <class Op, class A> struct FoldIdent;
template <class A> struct FoldIdent<OpAdd, A> {
  static __device__ A v() { return is_float<A>::value ? (A)(-0.0) : (A)0; }
};
template <class A> struct FoldIdent<OpMul, A> {
  static __device__ A v() { return (A)1; }
};
template <class A> struct FoldIdent<OpMin, A> {
  static __device__ A v() {
    if (is_float<A>::value) return (A)__longlong_as_double(0x7ff0000000000000ll);
    return sizeof(A) == 4 ? (A)0x7fffffff : (A)0x7fffffffffffffffll;
  }
};
template <class A> struct FoldIdent<OpMax, A> {
  static __device__ A v() {
    if (is_float<A>::value) return (A)__longlong_as_double((long long)0xfff0000000000000ull);
    return sizeof(A) == 4 ? (A)(-0x7fffffff - 1) : (A)(-0x7fffffffffffffffll - 1);
  }
};

struct CarryArgs {
  const void* val[DRK_CARRY_MAX];
  const long long* has[DRK_CARRY_MAX];
};

template <class T, class Op>
__global__ void carry_fold_kernel(const CarryArgs a, int count, int has_in, typename WideAcc<T, Op>::type carry_in,
                                  const typename WideAcc<T, Op>::type* carry_in_dev,
                                  typename WideAcc<T, Op>::type* out) {
  typedef typename LocalAcc<T, Op>::type L;
  typedef typename WideAcc<T, Op>::type A;
  Opt<A> acc;
  acc.has = has_in;
  acc.v = carry_in;
  if (carry_in_dev) {  // an earlier fold: already in the accumulator type
    Opt<A> c;
    c.has = 1;
    c.v = *carry_in_dev;
    acc = opt_combine<Op>(acc, c);
  }
  for (int j = 0; j < count; ++j) {
    if (a.has[j] && *a.has[j] == 0) continue;
    Opt<A> v;
    v.has = 1;
    v.v = (A)(L) * (const A*)a.val[j];  // the reference folds the segment totals in numpy's dtype
    acc = opt_combine<Op>(acc, v);
  }
  *out = acc.has ? acc.v : FoldIdent<Op, A>::v();
}

template <class T, class Op>
static int carry_fold_t(const CarryArgs& a, int count, const void* carry_in_host, const void* carry_in_dev, void* out,
                        int device, void* stream) {
  typedef typename WideAcc<T, Op>::type A;
  if (int rc = prologue(device, "drk_carry_fold")) return rc;
  A cin = A();
  if (carry_in_host) memcpy(&cin, carry_in_host, sizeof(A));
  carry_fold_kernel<T, Op><<<1, 1, 0, (cudaStream_t)stream>>>(a, count, carry_in_host != nullptr, cin,
                                                               (const A*)carry_in_dev, (A*)out);
  return epilogue("drk_carry_fold");
}

extern "C" int drk_carry_fold(int dtype, int op, const void* const* totals, const void* const* has, int count,
                              const void* carry_in_host, const void* carry_in_dev, void* carry_out_dev, int device,
                              void* stream) {
  if (count < 0 || count > DRK_CARRY_MAX) return set_error(DRK_E_ARG, "drk_carry_fold: count out of range");
  if (!carry_out_dev || (count > 0 && !totals)) return set_error(DRK_E_ARG, "drk_carry_fold: null pointer");
  CarryArgs a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < count; ++j) {
    if (!totals[j]) return set_error(DRK_E_ARG, "drk_carry_fold: null total pointer");
    a.val[j] = totals[j];
    a.has[j] = has ? (const long long*)has[j] : nullptr;
  }
  DRK_DISPATCH(dtype, "drk_carry_fold", T, {
    switch (op) {
      case DRK_ADD: return carry_fold_t<T, OpAdd>(a, count, carry_in_host, carry_in_dev, carry_out_dev, device, stream);
      case DRK_MUL: return carry_fold_t<T, OpMul>(a, count, carry_in_host, carry_in_dev, carry_out_dev, device, stream);
      case DRK_MIN: return carry_fold_t<T, OpMin>(a, count, carry_in_host, carry_in_dev, carry_out_dev, device, stream);
      case DRK_MAX: return carry_fold_t<T, OpMax>(a, count, carry_in_host, carry_in_dev, carry_out_dev, device, stream);
    }
    return set_error(DRK_E_ARG, "drk_carry_fold: unknown op");
  });
}

// ---------------------------------------------------------------------------------------
// scans of NVRTC-compiled kernels (custom associative operators)

extern "C" int drk_jit_launch(void* handle, const char* kernel, unsigned grid, unsigned block, unsigned smem,
                              const void* params, size_t params_bytes, int device, void* stream);

template <class A>
static int jit_scan_impl(void* handle, const char* kernel, int tile, int smem_bytes, int exclusive, const void* in,
                         void* out, int64_t n, const void* init_host, const void* carry_host, const void* carry_dev,
                         void* seg_total, void* carry_out, void* scratch, size_t scratch_bytes, int device,
                         void* stream) {
  if (n < 1 || tile < 1) return set_error(DRK_E_ARG, "drk_jit_scan: n and tile must be >= 1");
  if (!in || !out) return set_error(DRK_E_ARG, "drk_jit_scan: null in/out");
  if (exclusive && !init_host) return set_error(DRK_E_ARG, "drk_jit_scan: exclusive scan needs init");
  if (carry_host && carry_dev) return set_error(DRK_E_ARG, "drk_jit_scan: give at most one carry");
  const int64_t nt = (n + tile - 1) / tile;
  if (!scratch || scratch_bytes < 128 + (size_t)nt * 16)
    return set_error(DRK_E_SCRATCH, "drk_jit_scan: scratch too small");
  ScanParams<A, const void*> p;
  memset(&p, 0, sizeof(p));
  p.in = in;
  p.out = out;
  p.n = n;
  p.ntiles = (u32)nt;
  p.exclusive = exclusive;
  p.has_init = init_host != nullptr;
  if (init_host) memcpy(&p.init, init_host, sizeof(A));
  p.carry_kind = carry_host ? 1 : (carry_dev ? 2 : 0);
  if (carry_host) memcpy(&p.carry_val, carry_host, sizeof(A));
  p.carry_ptr = (const A*)carry_dev;
  p.seg_total = (A*)seg_total;
  p.carry_out = (A*)carry_out;
  p.counter = (u32*)scratch;
  p.desc = (u64*)((char*)scratch + 128);
  p.epoch = next_epoch(scratch);
  p.bulk_ok = 0;
  p.trace = nullptr;
  return drk_jit_launch(handle, kernel, (unsigned)nt, BLOCK, (unsigned)smem_bytes, &p, sizeof(p), device, stream);
}

extern "C" size_t drk_jit_scan_scratch_bytes(int64_t n, int tile) {
  if (n < 1) n = 1;
  if (tile < 1) tile = 1;
  return 128 + (size_t)((n + tile - 1) / tile) * 16;
}

extern "C" int drk_jit_scan(void* handle, const char* kernel, int acc_bytes, int tile, int smem_bytes, int exclusive,
                            const void* in, void* out, int64_t n, const void* init_host, const void* carry_host,
                            const void* carry_dev, void* seg_total_dev, void* carry_out_dev, void* scratch,
                            size_t scratch_bytes, int device, void* stream) {
  if (acc_bytes == 8)
    return jit_scan_impl<double>(handle, kernel, tile, smem_bytes, exclusive, in, out, n, init_host, carry_host,
                                 carry_dev, seg_total_dev, carry_out_dev, scratch, scratch_bytes, device, stream);
  if (acc_bytes == 4)
    return jit_scan_impl<float>(handle, kernel, tile, smem_bytes, exclusive, in, out, n, init_host, carry_host,
                                carry_dev, seg_total_dev, carry_out_dev, scratch, scratch_bytes, device, stream);
  return set_error(DRK_E_ARG, "drk_jit_scan: acc_bytes must be 4 or 8");
}

