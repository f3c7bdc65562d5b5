/* c_host.c — the drop-in boundary used from plain C: no Python, no torch.
 *
 * A host program that owns its device memory and stream and calls libdrk.so through
 * include/drk.h only, the way a segrange maintainer's FFI (or any C/C++/cgo/JNI host) would:
 * a distributed vector of 2 segments on GPU 0, filled by the device twin of the reference's
 * generator (repro.py:21-40), then dot (bench.py:87-90), STREAM triad (bench.py:93-99) and an
 * inclusive scan with the carry passed from segment 0 to segment 1 on the device
 * (algorithms.py:234-308).  Results are checked on the host against plain C loops.
 *
 *   make -C examples && examples/c_host [log2n]      (prints one line, exit 0 = all checks pass)
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include "../include/drk.h"

#define CK(x)                                                                     \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_) {                                                                    \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, drk_last_error());         \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CU(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                    \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(int argc, char** argv) {
  const int log2n = argc > 1 ? atoi(argv[1]) : 22;
  const int64_t n = (int64_t)1 << log2n, half = n / 2;
  const int dev = 0;
  int count = 0;
  CK(drk_device_count(&count));
  if (count < 1) {
    fprintf(stderr, "no CUDA device\n");
    return 1;
  }
  CU(cudaSetDevice(dev));
  cudaStream_t s;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

  float *b, *c, *a;
  int32_t *xi, *yi;
  CU(cudaMalloc((void**)&b, n * sizeof(float)));
  CU(cudaMalloc((void**)&c, n * sizeof(float)));
  CU(cudaMalloc((void**)&a, n * sizeof(float)));
  CU(cudaMalloc((void**)&xi, n * sizeof(int32_t)));
  CU(cudaMalloc((void**)&yi, n * sizeof(int32_t)));
  void* red = NULL;
  CU(cudaMalloc(&red, drk_reduce_scratch_bytes()));
  CU(cudaMemsetAsync(red, 0, drk_reduce_scratch_bytes(), s));
  const size_t sb = drk_scan_scratch_bytes(DRK_I32, DRK_ADD, half);
  void* scan_scratch = NULL;
  CU(cudaMalloc(&scan_scratch, sb));
  CU(cudaMemsetAsync(scan_scratch, 0, sb, s));
  double* res = NULL;  /* result slots: [dot seg0, dot seg1, carry] */
  CU(cudaMalloc((void**)&res, 4 * sizeof(double)));

  /* inputs: b = unit_doubles(1, 0, n), c = unit_doubles(1, n, n), x = splitmix % 2001 - 1000 */
  CK(drk_generate(DRK_F32, b, n, 1, 0, DRK_GEN_UNIFORM, 0.0, 1.0, dev, s));
  CK(drk_generate(DRK_F32, c, n, 1, (uint64_t)n, DRK_GEN_UNIFORM, 0.0, 1.0, dev, s));
  CK(drk_generate(DRK_I32, xi, n, 1, 0, DRK_GEN_MOD, 2001.0, -1000.0, dev, s));

  /* dot: one fused kernel per segment; the driver folds the two partials in order */
  CK(drk_dot(DRK_F32, b, c, half, &res[0], red, dev, s));
  CK(drk_dot(DRK_F32, b + half, c + half, n - half, &res[1], red, dev, s));
  /* triad: a = b + 3 c */
  const float alpha = 3.0f;
  CK(drk_triad(DRK_F32, a, b, c, n, &alpha, dev, s));
  /* scan: segment 1's carry is segment 0's carry_out, read on the device */
  CK(drk_scan(DRK_I32, DRK_ADD, 0, xi, yi, half, NULL, NULL, NULL, NULL, &res[2], scan_scratch, sb, dev, s));
  CK(drk_scan(DRK_I32, DRK_ADD, 0, xi + half, yi + half, n - half, NULL, NULL, &res[2], NULL, NULL, scan_scratch,
              sb, dev, s));
  /* the driver's fold of the two dot partials on the device (drk_reduce_fold: numpy's
   * reduce dtype, float32 for float32 data), starting from init 0.0f */
  const float zero = 0.0f;
  const void* parts[2] = {&res[0], &res[1]};
  CK(drk_reduce_fold(DRK_F32, DRK_ADD, parts, 2, &zero, &res[3], NULL, dev, s));
  /* sort a copy of x with the library's radix sort */
  int32_t *sx, *salt;
  CU(cudaMalloc((void**)&sx, n * sizeof(int32_t)));
  CU(cudaMalloc((void**)&salt, n * sizeof(int32_t)));
  CU(cudaMemcpyAsync(sx, xi, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  size_t sort_bytes = 0;
  CK(drk_sort_keys(DRK_I32, sx, salt, n, NULL, &sort_bytes, dev, s));
  void* sort_scratch = NULL;
  CU(cudaMalloc(&sort_scratch, sort_bytes));
  CK(drk_sort_keys(DRK_I32, sx, salt, n, sort_scratch, &sort_bytes, dev, s));
  CK(drk_stream_synchronize(dev, s));

  /* host checks */
  float* hb = (float*)malloc(n * sizeof(float));
  float* hc = (float*)malloc(n * sizeof(float));
  float* ha = (float*)malloc(n * sizeof(float));
  int32_t* hx = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* hy = (int32_t*)malloc(n * sizeof(int32_t));
  double hres[4];
  CU(cudaMemcpy(hb, b, n * sizeof(float), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hc, c, n * sizeof(float), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(ha, a, n * sizeof(float), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hx, xi, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hy, yi, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hres, res, 4 * sizeof(double), cudaMemcpyDeviceToHost));
  int32_t* hs = (int32_t*)malloc(n * sizeof(int32_t));
  CU(cudaMemcpy(hs, sx, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  double dot = 0.0, want = 0.0;
  dot = (double)(float)hres[0] + (double)(float)hres[1];
  float folded;
  memcpy(&folded, &hres[3], sizeof(float));
  const int fold_ok = folded == (float)(zero + (float)hres[0]) + (float)hres[1];
  int bad_triad = 0, bad_scan = 0;
  int64_t run = 0;
  for (int64_t i = 0; i < n; ++i) {
    want += (double)hb[i] * (double)hc[i];
    volatile float t = 3.0f * hc[i]; /* numpy: b + fp32(3 c), two roundings */
    if (ha[i] != hb[i] + t) ++bad_triad;
    run += hx[i];
    if (hy[i] != (int32_t)run) ++bad_scan;
  }
  /* sorted, and the same multiset (the sum and the count of each residue mod 7) */
  int bad_sort = 0;
  int64_t sum_x = 0, sum_s = 0;
  int64_t res_x[7] = {0}, res_s[7] = {0};
  for (int64_t i = 0; i < n; ++i) {
    if (i && hs[i - 1] > hs[i]) ++bad_sort;
    sum_x += hx[i];
    sum_s += hs[i];
    ++res_x[((hx[i] % 7) + 7) % 7];
    ++res_s[((hs[i] % 7) + 7) % 7];
  }
  if (sum_x != sum_s || memcmp(res_x, res_s, sizeof(res_x))) ++bad_sort;
  const double rel = fabs(dot - want) / fabs(want);
  const int ok = rel <= 1e-5 && bad_triad == 0 && bad_scan == 0 && bad_sort == 0 && fold_ok;
  printf("{\"n\": %lld, \"dot\": %.9g, \"dot_rel_err\": %.3g, \"triad_mismatches\": %d, \"scan_mismatches\": %d, "
         "\"sort_errors\": %d, \"device_fold_ok\": %s, \"launches\": %lld, \"ok\": %s}\n",
         (long long)n, dot, rel, bad_triad, bad_scan, bad_sort, fold_ok ? "true" : "false",
         (long long)drk_launch_count(), ok ? "true" : "false");
  return ok ? 0 : 1;
}
