// drk_sort.cu — sort entry points of include/drk.h (CUB device radix sort + gather).
// Separate translation unit: CUB's radix-sort instantiations dominate compile time.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/drk.h"
#include "drk_device.cuh"

using namespace drk;

extern "C" int64_t drk_note_launch(void);
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
// sort (reference algorithms.py:315-432): device radix sort of one contiguous buffer.
// CUB's DeviceRadixSort is library code; the distributed part (gathering segments,
// writing them back in order) is the caller's.

template <class K> static int sort_keys_t(void* keys, void* alt, int64_t n, void* scratch, size_t* bytes,
                                          int device, void* stream) {
  cub::DoubleBuffer<K> db((K*)keys, (K*)alt);
  size_t need = 0;
  DRK_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, need, db, n, 0, (int)(sizeof(K) * 8), (cudaStream_t)stream));
  if (!scratch) {
    *bytes = need;
    return 0;
  }
  if (*bytes < need) return drk_error(DRK_E_SCRATCH, "drk_sort_keys: scratch too small");
  if (int rc = set_device(device)) return rc;
  DRK_CHECK(cub::DeviceRadixSort::SortKeys(scratch, need, db, n, 0, (int)(sizeof(K) * 8), (cudaStream_t)stream));
  drk_note_launch();
  if (db.Current() != (K*)keys)
    DRK_CHECK(cudaMemcpyAsync(keys, db.Current(), n * sizeof(K), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return 0;
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
  if (!keys || !alt) return drk_error(DRK_E_ARG, "drk_sort_keys: null buffer");
  DRK_DISPATCH(dtype, "drk_sort_keys", T, return sort_keys_t<T>(keys, alt, n, scratch, scratch_bytes, device, stream));
}

template <class K> static int sort_pairs_t(void* keys, void* keys_alt, int64_t* idx, int64_t* idx_alt, int64_t n,
                                           void* scratch, size_t* bytes, int device, void* stream) {
  cub::DoubleBuffer<K> dk((K*)keys, (K*)keys_alt);
  cub::DoubleBuffer<int64_t> dv(idx, idx_alt);
  size_t need = 0;
  DRK_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, need, dk, dv, n, 0, (int)(sizeof(K) * 8), (cudaStream_t)stream));
  if (!scratch) {
    *bytes = need;
    return 0;
  }
  if (*bytes < need) return drk_error(DRK_E_SCRATCH, "drk_sort_pairs: scratch too small");
  if (int rc = set_device(device)) return rc;
  DRK_CHECK(cub::DeviceRadixSort::SortPairs(scratch, need, dk, dv, n, 0, (int)(sizeof(K) * 8), (cudaStream_t)stream));
  drk_note_launch();
  if (dv.Current() != idx)
    DRK_CHECK(cudaMemcpyAsync(idx, dv.Current(), n * sizeof(int64_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  if (dk.Current() != (K*)keys)
    DRK_CHECK(cudaMemcpyAsync(keys, dk.Current(), n * sizeof(K), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return 0;
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
