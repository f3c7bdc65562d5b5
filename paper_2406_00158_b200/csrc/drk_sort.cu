// drk_sort.cu — sort entry points of include/drk.h: this library's own LSD radix sort (below),
// the gather of a permutation and the sample sort's splitter search.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/drk.h"
#include "drk_device.cuh"

using namespace drk;

extern "C" int64_t drk_note_launch(void);
extern "C" size_t drk_scan_scratch_bytes(int dtype, int op, int64_t n);
extern "C" int drk_scan(int dtype, int op, int exclusive, const void* in, void* out, int64_t n, const void* init_host,
                        const void* carry_host, const void* carry_dev, void* seg_total_dev, void* carry_out_dev,
                        void* scratch, size_t scratch_bytes, int device, void* stream);
int drk_error(int code, const char* msg);  // drk_kernels.cu
int drk_cuda_error(cudaError_t e, const char* what);

#define DRK_CHECK(call)                                       \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return drk_cuda_error(_e, #call);  \
  } while (0)

static int set_device(int device) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) DRK_CHECK(cudaSetDevice(device));
  return 0;
}

#define DRK_DISPATCH(dtype, what, T, ...)                          \
  switch (dtype) {                                                \
    case DRK_F32: { typedef float T; __VA_ARGS__; }               \
    case DRK_F64: { typedef double T; __VA_ARGS__; }              \
    case DRK_I32: { typedef int T; __VA_ARGS__; }                 \
    case DRK_I64: { typedef long long T; __VA_ARGS__; }           \
    case DRK_U32: { typedef unsigned int T; __VA_ARGS__; }        \
    case DRK_U64: { typedef unsigned long long T; __VA_ARGS__; }  \
    default: return drk_error(DRK_E_DTYPE, what ": unknown dtype"); \
  }

// ---------------------------------------------------------------------------------------
// sort (reference algorithms.py:315-432): the local and chunk sorts of the sample sort are
// an LSD radix sort of one contiguous buffer, 8-bit digits, three kernels per digit pass:
//   upsweep    one 4096-key tile per CTA: the tile's digit histogram -> counts[d][tile]
//   scan       exclusive scan of counts in (digit, tile) order (drk_scan, this library's
//              decoupled look-back scan) -> the global offset of every (digit, tile) run
//   downsweep  the tile re-read, keys ranked stably by digit inside the tile (warp
//              __match_any_sync + per-warp digit counters), exchanged through shared memory
//              into digit order, then written as contiguous digit runs (coalesced)
// Passes alternate between the buffer and its alternate; an even number of passes (4 for
// 4-byte, 8 for 8-byte keys) leaves the result in place.  Order: numpy's (np.sort /
// argsort kind="stable", reference :336-340): keys map to unsigned radix keys with the usual
// sign twiddles, every NaN after +inf.  Keys-only sorts keep -0.0 before +0.0 (equal under
// numpy's comparison, whose quicksort leaves their order unspecified) and return NaNs with
// the sign bit cleared; pair sorts (the stable argsort of a key function) rank -0.0 and +0.0
// as equal, so ties keep their input order exactly as argsort(kind="stable") does.
namespace {

constexpr int RX_BLOCK = 256;
constexpr int RX_WARPS = RX_BLOCK / 32;
#ifndef DRK_RX_IPT
#define DRK_RX_IPT 16
#endif
constexpr int RX_IPT = DRK_RX_IPT;               // keys per thread
constexpr int RX_TILE = RX_BLOCK * RX_IPT;       // 4096 keys per tile
constexpr int RX_DIGITS = 256;

// Keys travel as their raw bit patterns (U): every step below is integer arithmetic on the
// bits, so no floating-point operation can touch a key (signed zeros, denormals and NaN
// payloads are moved exactly).  RadixOf<K>::to maps bits to an unsigned radix key in numpy's
// order; canon gives the bits written back (NaNs with the sign cleared in keys-only sorts).
template <class K> struct RadixOf;
template <> struct RadixOf<unsigned int> {
  typedef unsigned int U;
  static __device__ __forceinline__ U to(U k, bool) { return k; }
  static __device__ __forceinline__ U canon(U k) { return k; }
};
template <> struct RadixOf<unsigned long long> {
  typedef unsigned long long U;
  static __device__ __forceinline__ U to(U k, bool) { return k; }
  static __device__ __forceinline__ U canon(U k) { return k; }
};
template <> struct RadixOf<int> {
  typedef unsigned int U;
  static __device__ __forceinline__ U to(U k, bool) { return k ^ 0x80000000u; }
  static __device__ __forceinline__ U canon(U k) { return k; }
};
template <> struct RadixOf<long long> {
  typedef unsigned long long U;
  static __device__ __forceinline__ U to(U k, bool) { return k ^ 0x8000000000000000ull; }
  static __device__ __forceinline__ U canon(U k) { return k; }
};
template <> struct RadixOf<float> {
  typedef unsigned int U;
  static __device__ __forceinline__ U to(U u, bool pairs) {
    const U mag = u & 0x7fffffffu;
    if (mag > 0x7f800000u) u = mag;                    // every NaN after +inf
    else if (pairs && u == 0x80000000u) u = 0u;        // -0.0 ranks with +0.0
    return u ^ ((u >> 31) ? 0xffffffffu : 0x80000000u);
  }
  static __device__ __forceinline__ U canon(U u) {
    const U mag = u & 0x7fffffffu;
    return mag > 0x7f800000u ? mag : u;
  }
};
template <> struct RadixOf<double> {
  typedef unsigned long long U;
  static __device__ __forceinline__ U to(U u, bool pairs) {
    const U mag = u & 0x7fffffffffffffffull;
    if (mag > 0x7ff0000000000000ull) u = mag;
    else if (pairs && u == 0x8000000000000000ull) u = 0ull;
    return u ^ ((u >> 63) ? 0xffffffffffffffffull : 0x8000000000000000ull);
  }
  static __device__ __forceinline__ U canon(U u) {
    const U mag = u & 0x7fffffffffffffffull;
    return mag > 0x7ff0000000000000ull ? mag : u;
  }
};

template <class K> __device__ __forceinline__ int digit_of(typename RadixOf<K>::U k, int shift, bool pairs) {
  return (int)((RadixOf<K>::to(k, pairs) >> shift) & 0xffu);
}

// key index of item j of lane l in warp w (warp-striped: a warp's 512 keys are contiguous,
// item-major, so (warp, item, lane) is the keys' order)
__device__ __forceinline__ int rx_index(int w, int j, int l) { return w * 32 * RX_IPT + j * 32 + l; }

template <class K>
__global__ void __launch_bounds__(RX_BLOCK) radix_upsweep(const typename RadixOf<K>::U* __restrict__ keys, i64 n,
                                                           int shift, int pairs, u32* __restrict__ counts,
                                                           u32 ntiles) {
  typedef typename RadixOf<K>::U U;
  // per-warp histograms (shared-memory atomics, no warp matching: the count is all that is
  // needed here), summed per digit at the end
  __shared__ u32 hist[RX_WARPS][RX_DIGITS];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int k = 0; k < RX_WARPS; ++k) hist[k][tid] = 0;
  __syncthreads();
  const i64 base = (i64)blockIdx.x * RX_TILE;
  U key[RX_IPT];
#pragma unroll
  for (int j = 0; j < RX_IPT; ++j) {
    const i64 i = base + rx_index(w, j, lane);
    key[j] = i < n ? keys[i] : U(0);
  }
#pragma unroll
  for (int j = 0; j < RX_IPT; ++j) {
    const i64 i = base + rx_index(w, j, lane);
    const int d = i < n ? digit_of<K>(key[j], shift, pairs != 0) : RX_DIGITS;
    const int d0 = __shfl_sync(0xffffffffu, d, 0);
    if (__all_sync(0xffffffffu, d == d0)) {
      // one digit for the whole warp (narrow key ranges, upper digits): one update, not 32
      // serialised ones on the same counter
      if (lane == 0 && d0 < RX_DIGITS) hist[w][d0] += 32u;
    } else if (d < RX_DIGITS) {
      atomicAdd(&hist[w][d], 1u);
    }
  }
  __syncthreads();
  u32 c = 0;
#pragma unroll
  for (int k = 0; k < RX_WARPS; ++k) c += hist[k][tid];
  counts[(size_t)tid * ntiles + blockIdx.x] = c;
}

// lanes of the warp holding the same 8-bit digit (d < 256; d = 256 marks an empty slot):
// eight ballots on the digit's bits (cheaper than MATCH.ANY on this pipe)
__device__ __forceinline__ u32 digit_peers(int d) {
  u32 peers = __ballot_sync(0xffffffffu, d >> 8);
  peers = (d >> 8) ? peers : ~peers;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const u32 m = __ballot_sync(0xffffffffu, (d >> b) & 1);
    peers &= ((d >> b) & 1) ? m : ~m;
  }
  return peers;
}

template <class K, bool HAS_V>
__global__ void __launch_bounds__(RX_BLOCK, 4) radix_downsweep(
    const typename RadixOf<K>::U* __restrict__ keys_in, typename RadixOf<K>::U* __restrict__ keys_out,
                                                             const i64* __restrict__ vals_in, i64* __restrict__ vals_out,
                                                             i64 n, int shift, int pairs, const u32* __restrict__ offsets,
                                                             u32 ntiles) {
  __shared__ u32 whist[RX_WARPS][RX_DIGITS];  // per-warp digit counts -> exclusive prefix over warps
  __shared__ u32 tstart[RX_DIGITS];           // exclusive prefix of the tile's digit counts
  __shared__ u32 gstart[RX_DIGITS];           // global position of the tile's run of digit d
  __shared__ u32 wsum[RX_WARPS];
  typedef typename RadixOf<K>::U U;
  extern __shared__ __align__(16) unsigned char rx_smem[];
  U* skeys = (U*)rx_smem;
  i64* svals = (i64*)(rx_smem + RX_TILE * sizeof(K));
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 tile = blockIdx.x;
  const i64 base = (i64)tile * RX_TILE;
  const int valid = (int)((n - base) < RX_TILE ? (n - base) : RX_TILE);
#pragma unroll
  for (int k = 0; k < RX_WARPS; ++k) whist[k][tid] = 0;
  gstart[tid] = offsets[(size_t)tid * ntiles + tile];
  __syncthreads();
  const u32 lt = (1u << lane) - 1u;
  U key[RX_IPT];
  i64 val[RX_IPT];
  int dig[RX_IPT];
  u32 rank[RX_IPT];
#pragma unroll
  for (int j = 0; j < RX_IPT; ++j) {
    const int li = rx_index(w, j, lane);
    const bool ok = li < valid;
    key[j] = ok ? keys_in[base + li] : U(0);
    if constexpr (HAS_V) val[j] = ok ? vals_in[base + li] : 0;
    dig[j] = ok ? digit_of<K>(key[j], shift, pairs != 0) : RX_DIGITS;
  }
  // the warp's digit counters are read by every lane and bumped by each digit group's leader,
  // item after item: volatile accesses keep the compiler from hoisting the next item's reads
  // above this item's (other lanes') updates, and __syncwarp orders them between lanes
  volatile u32* wh = whist[w];
#pragma unroll
  for (int j = 0; j < RX_IPT; ++j) {
    const int d = dig[j];
    const u32 peers = digit_peers(d);
    const u32 before = d < RX_DIGITS ? wh[d] : 0u;
    rank[j] = before + (u32)__popc(peers & lt);
    __syncwarp();
    if (d < RX_DIGITS && lane == __ffs(peers) - 1) wh[d] = before + (u32)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // digit tid: exclusive prefix over warps, and the tile's count
  u32 run = 0;
#pragma unroll
  for (int k = 0; k < RX_WARPS; ++k) {
    const u32 c = whist[k][tid];
    whist[k][tid] = run;
    run += c;
  }
  // exclusive prefix of the tile's digit counts (block scan over 256 values)
  u32 incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  u32 woff = 0;
#pragma unroll
  for (int k = 0; k < RX_WARPS; ++k)
    if (k < w) woff += wsum[k];
  tstart[tid] = woff + incl - run;
  __syncthreads();
  // exchange into digit order
#pragma unroll
  for (int j = 0; j < RX_IPT; ++j) {
    const int d = dig[j];
    if (d < RX_DIGITS) {
      const u32 pos = tstart[d] + whist[w][d] + rank[j];
      skeys[pos] = pairs ? key[j] : RadixOf<K>::canon(key[j]);
      if constexpr (HAS_V) svals[pos] = val[j];
    }
  }
  __syncthreads();
  // contiguous digit runs to their global positions
  for (int i = tid; i < valid; i += RX_BLOCK) {
    const U k = skeys[i];
    const int d = digit_of<K>(k, shift, pairs != 0);
    const u32 g = gstart[d] + (u32)i - tstart[d];
    keys_out[g] = k;
    if constexpr (HAS_V) vals_out[g] = svals[i];
  }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// scratch: counts and offsets (256 x ntiles u32 each) and the scan's scratch
size_t radix_scratch(int64_t n) {
  const size_t ntiles = (size_t)((n + RX_TILE - 1) / RX_TILE);
  const size_t m = (size_t)RX_DIGITS * ntiles;
  return 2 * align256(m * 4) + align256(drk_scan_scratch_bytes(DRK_I32, DRK_ADD, (int64_t)m)) + 256;
}

template <class K, bool HAS_V>
int radix_sort(K* keys, K* alt, i64* vals, i64* vals_alt, int64_t n, bool pairs, void* scratch, int device,
               cudaStream_t s) {
  const u32 ntiles = (u32)((n + RX_TILE - 1) / RX_TILE);
  const size_t m = (size_t)RX_DIGITS * ntiles;
  char* b = (char*)(((uintptr_t)scratch + 255) & ~(uintptr_t)255);
  u32* counts = (u32*)b;
  u32* offsets = (u32*)(b + align256(m * 4));
  void* sscr = b + 2 * align256(m * 4);
  const size_t sbytes = align256(drk_scan_scratch_bytes(DRK_I32, DRK_ADD, (int64_t)m));
  const size_t smem = (size_t)RX_TILE * sizeof(K) + (HAS_V ? (size_t)RX_TILE * 8 : 0);
  auto down = radix_downsweep<K, HAS_V>;
  DRK_CHECK(cudaFuncSetAttribute(down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // the scan's scratch (ticket counter, epoch-tagged tile descriptors) starts zeroed; its
  // epochs then separate the passes
  DRK_CHECK(cudaMemsetAsync(sscr, 0, sbytes, s));
  const long long zero = 0;  // the int32 scan's accumulator is int64
  K* src = keys;
  K* dst = alt;
  i64* vsrc = vals;
  i64* vdst = vals_alt;
  for (int shift = 0; shift < (int)(8 * sizeof(K)); shift += 8) {
    typedef typename RadixOf<K>::U U;
    radix_upsweep<K><<<ntiles, RX_BLOCK, 0, s>>>((const U*)src, n, shift, pairs ? 1 : 0, counts, ntiles);
    drk_note_launch();
    if (int rc = drk_scan(DRK_I32, DRK_ADD, 1, counts, offsets, (int64_t)m, &zero, nullptr, nullptr, nullptr,
                          nullptr, sscr, sbytes, device, s))
      return rc;
    down<<<ntiles, RX_BLOCK, smem, s>>>((const U*)src, (U*)dst, vsrc, vdst, n, shift, pairs ? 1 : 0, offsets, ntiles);
    drk_note_launch();
    DRK_CHECK(cudaGetLastError());
    K* t = src; src = dst; dst = t;
    i64* tv = vsrc; vsrc = vdst; vdst = tv;
  }
  return 0;  // an even number of passes: the result is back in keys / vals
}

}  // namespace

template <class K> static int sort_keys_t(void* keys, void* alt, int64_t n, void* scratch, size_t* bytes,
                                          int device, void* stream) {
  const size_t need = radix_scratch(n);
  if (!scratch) {
    *bytes = need;
    return 0;
  }
  if (*bytes < need) return drk_error(DRK_E_SCRATCH, "drk_sort_keys: scratch too small");
  if (int rc = set_device(device)) return rc;
  return radix_sort<K, false>((K*)keys, (K*)alt, nullptr, nullptr, n, false, scratch, device, (cudaStream_t)stream);
}

/* Sort `keys` (n elements of dtype) ascending in place; `alt` is an n-element buffer of
 * the same dtype.  With scratch == NULL, *scratch_bytes receives the needed size. */
extern "C" int drk_sort_keys(int dtype, void* keys, void* alt, int64_t n, void* scratch, size_t* scratch_bytes,
                             int device, void* stream) {
  if (!scratch_bytes) return drk_error(DRK_E_ARG, "drk_sort_keys: null scratch_bytes");
  if (n < 2) {
    if (!scratch) *scratch_bytes = 0;
    return 0;
  }
  if (n > 0x7fffffffLL) return drk_error(DRK_E_ARG, "drk_sort_keys: n must be < 2^31");
  if (!keys || !alt) return drk_error(DRK_E_ARG, "drk_sort_keys: null buffer");
  DRK_DISPATCH(dtype, "drk_sort_keys", T, return sort_keys_t<T>(keys, alt, n, scratch, scratch_bytes, device, stream));
}

template <class K> static int sort_pairs_t(void* keys, void* keys_alt, int64_t* idx, int64_t* idx_alt, int64_t n,
                                           void* scratch, size_t* bytes, int device, void* stream) {
  const size_t need = radix_scratch(n);
  if (!scratch) {
    *bytes = need;
    return 0;
  }
  if (*bytes < need) return drk_error(DRK_E_SCRATCH, "drk_sort_pairs: scratch too small");
  if (int rc = set_device(device)) return rc;
  return radix_sort<K, true>((K*)keys, (K*)keys_alt, (i64*)idx, (i64*)idx_alt, n, true, scratch, device,
                             (cudaStream_t)stream);
}

/* Stable sort of (key, index) pairs by key: afterwards keys[] is sorted and idx[] holds
 * the permutation that sorted it (idx[] comes in as the values to carry, e.g. an iota). */
extern "C" int drk_sort_pairs(int key_dtype, void* keys, void* keys_alt, void* idx, void* idx_alt, int64_t n,
                              void* scratch, size_t* scratch_bytes, int device, void* stream) {
  if (!scratch_bytes) return drk_error(DRK_E_ARG, "drk_sort_pairs: null scratch_bytes");
  if (n < 2) {
    if (!scratch) *scratch_bytes = 0;
    return 0;
  }
  if (n > 0x7fffffffLL) return drk_error(DRK_E_ARG, "drk_sort_pairs: n must be < 2^31");
  if (!keys || !keys_alt || !idx || !idx_alt) return drk_error(DRK_E_ARG, "drk_sort_pairs: null buffer");
  DRK_DISPATCH(key_dtype, "drk_sort_pairs", K,
               return sort_pairs_t<K>(keys, keys_alt, (int64_t*)idx, (int64_t*)idx_alt, n, scratch, scratch_bytes,
                                      device, stream));
}

template <class T>
__global__ void __launch_bounds__(256) gather_kernel(T* out, const T* in, const long long* idx, i64 n) {
  const i64 G = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += G) out[i] = in[idx[i]];
}

/* out[i] = in[idx[i]] */
extern "C" int drk_gather(int dtype, void* out, const void* in, const void* idx, int64_t n, int device,
                          void* stream) {
  if (n <= 0) return 0;
  if (!out || !in || !idx) return drk_error(DRK_E_ARG, "drk_gather: null buffer");
  if (int rc = set_device(device)) return rc;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int64_t grid = (n + 255) / 256;
  if (grid > (int64_t)sms * 16) grid = (int64_t)sms * 16;
  DRK_DISPATCH(dtype, "drk_gather", T, {
    gather_kernel<T><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>((T*)out, (const T*)in, (const long long*)idx, n);
    drk_note_launch();
    DRK_CHECK(cudaGetLastError());
    return 0;
  });
}

// numpy's sort order: NaN after everything else (npy_sort's LT macro for floats)
template <class T> __device__ __forceinline__ bool np_lt(T a, T b) { return a < b; }
template <> __device__ __forceinline__ bool np_lt<float>(float a, float b) { return a < b || (b != b && a == a); }
template <> __device__ __forceinline__ bool np_lt<double>(double a, double b) {
  return a < b || (b != b && a == a);
}

// bounds[j] = number of elements of the sorted run that are not greater than split[j]
// (np.searchsorted(sorted, split[j], side="right")), one binary search per thread.
template <class T>
__global__ void __launch_bounds__(128) sort_bounds_kernel(const T* sorted, i64 n, const T* split, int nsplit,
                                                          long long* bounds) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsplit) return;
  const T s = split[j];
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = lo + ((hi - lo) >> 1);
    if (np_lt(s, sorted[mid])) hi = mid; else lo = mid + 1;
  }
  bounds[j] = lo;
}

/* Splitter positions in a sorted run for the sample sort's redistribution
 * (reference algorithms.py:371-378 `_count_task`: element x goes to chunk
 * searchsorted(split, x, side="left"); on a sorted run the end of chunk j is
 * searchsorted(run, split[j], side="right")).  split and bounds are device arrays of
 * nsplit entries (bounds: int64). */
extern "C" int drk_sort_bounds(int dtype, const void* sorted, int64_t n, const void* split, int nsplit,
                               void* bounds, int device, void* stream) {
  if (nsplit <= 0) return 0;
  if (n < 0) return drk_error(DRK_E_ARG, "drk_sort_bounds: negative length");
  if (!split || !bounds || (n > 0 && !sorted)) return drk_error(DRK_E_ARG, "drk_sort_bounds: null buffer");
  if (int rc = set_device(device)) return rc;
  DRK_DISPATCH(dtype, "drk_sort_bounds", T, {
    sort_bounds_kernel<T><<<(nsplit + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        (const T*)sorted, n, (const T*)split, nsplit, (long long*)bounds);
    drk_note_launch();
    DRK_CHECK(cudaGetLastError());
    return 0;
  });
}
