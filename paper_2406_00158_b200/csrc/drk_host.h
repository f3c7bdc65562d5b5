// drk_host.h — host-side plumbing shared by the translation units of libdrk.so
// (drk_kernels.cu: plumbing, maps, reductions, carry fold, NVRTC scans; drk_scan.cu: the
// scan kernels' launchers).  Launch knobs are defined once in drk_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/drk.h"
#include "drk_device.cuh"

namespace drk_host {
using namespace drk;

int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);
#define DRK_CHECK(call)                                  \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_status(_e, #call); \
  } while (0)

static constexpr int BLOCK = 256;
static constexpr int MAP_U = 4;
static constexpr int RED_U = 4;
static constexpr int MAX_RED_GRID = 4096;

extern std::mutex g_mu;
extern int g_map_waves;     // 0: size grid to cover the work once (non-persistent)
extern int g_reduce_waves;  // reduce grid = SMs * occupancy * waves
extern int g_scan_sub;      // scan sub-tiles per CTA tile (1..4; 0: by size)
extern int g_scan_l2dyn;    // L2-resident two-touch scan for large aligned segments
extern int g_scan_l2_min;
extern int g_scan_l2_subs;  // sub-tiles per L2 tile (0: 8 = 160 KB for 4-byte types)
extern int g_scan_l2_pre;   // sub-tiles scanned prefix-free during the look-back
extern int g_scan_l2_ring;  // TMA ring slots of the L2 re-scan (2 or 3)
extern int g_scan_debug;    // ScanParams::debug (experiments only)
extern int g_scan_stagger;     // ns between first-wave tile starts of the L2 scan (-1: automatic)
extern int g_scan_smem_pad;    // extra dynamic smem of the L2 scan (caps CTAs per SM): experiments
extern int g_scan_rescan_pol;  // ScanParams::rescan_pol (experiments)
extern int g_scan_keep_tail;   // ScanParams::keep_tail
extern int g_scan_lb_snap;     // ScanParams::lb_snap
extern int g_scan_2p_lo_kb, g_scan_2p_hi_kb;  // two-launch L2 scan for inputs of [lo, hi] KB (0 0: never)
extern thread_local int g_chain_launch;  // drk_scan_ex flag DRK_SCAN_CHAINED for this call
extern void* g_scan_trace;  // debug: per-tile timestamps of the next scans

int sm_count(int device);

template <class K> static int occupancy(K kernel, int block, size_t smem) {
  static std::unordered_map<uint64_t, int> cache;
  std::lock_guard<std::mutex> lk(g_mu);
  const uint64_t key = ((uint64_t)(uintptr_t)kernel << 20) ^ (uint64_t)smem ^ ((uint64_t)block << 40);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, smem) != cudaSuccess || n < 1)
    n = 1;
  cache[key] = n;
  return n;
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static inline int prologue(int device, const char* what) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, what);
  }
  return 0;
}

int epilogue(const char* what);

#define DRK_DISPATCH(dtype, what, T, ...)                                         \
  switch (dtype) {                                                               \
    case DRK_F32: { typedef float T; __VA_ARGS__; }                              \
    case DRK_F64: { typedef double T; __VA_ARGS__; }                             \
    case DRK_I32: { typedef int T; __VA_ARGS__; }                                \
    case DRK_I64: { typedef long long T; __VA_ARGS__; }                          \
    default: return set_error(DRK_E_DTYPE, std::string(what) + ": unknown dtype"); \
  }

#define DRK_DISPATCH_FLOAT(dtype, what, T, ...)                                       \
  switch (dtype) {                                                                   \
    case DRK_F32: { typedef float T; __VA_ARGS__; }                                  \
    case DRK_F64: { typedef double T; __VA_ARGS__; }                                 \
    default: return set_error(DRK_E_DTYPE, std::string(what) + ": needs float32/float64"); \
  }


template <class T, class Op> struct ScanItems {
  // ITEMS * sizeof(T) / 16 odd => conflict-free 16-byte LDS of per-thread runs.
  // (int32 sums keep 64-bit running partials; 20 still fits without spills: 64 registers)
  static constexpr int value = sizeof(T) == 4 ? 20 : 10;
};

template <class T, class Op> static size_t scan_scratch(int64_t n) {
  // sized for the smallest tile (SUB = 1) so any g_scan_sub fits
  constexpr int TILE = BLOCK * ScanItems<T, Op>::value;
  const size_t nt = (size_t)((n + TILE - 1) / TILE);
  return 128 + nt * 16;
}

// Per-scratch launch epochs (tile descriptors of older launches then read as stale).
uint64_t next_epoch(void* scratch);


}  // namespace drk_host
