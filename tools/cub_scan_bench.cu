// Calibration only (not part of the product): CUB 2.8 DeviceScan / DeviceReduce on the
// same sizes as tools/kbench.py, to know what a library scan reaches on this B200.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <algorithm>

template <class T> void run(const char* name, size_t n) {
  T *in, *out;
  cudaMalloc(&in, n * sizeof(T));
  cudaMalloc(&out, n * sizeof(T));
  cudaMemset(in, 0, n * sizeof(T));
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, (int64_t)n);
  void* d_tmp;
  cudaMalloc(&d_tmp, tmp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> ts;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a);
    cub::DeviceScan::InclusiveSum(d_tmp, tmp, in, out, (int64_t)n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  double med = ts[ts.size() / 2];
  printf("cub_scan_%s n=%zu ms=%.4f GB/s=%.1f err=%s\n", name, n, med, 2.0 * n * sizeof(T) / (med * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(in);
  cudaFree(out);
  cudaFree(d_tmp);
}

int main() {
  run<float>("f32", size_t(1) << 30);
  run<int>("i32", size_t(1) << 30);
  run<double>("f64", size_t(1) << 29);
  return 0;
}
