// Launch cost of a kernel by the size of its by-value parameter block (the batched reduce
// passes a ~1.3 KB ReduceBatch): R back-to-back launches between one event pair, queue kept
// full.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/param_probe tools/param_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct P { unsigned char b[B]; };
template <int B> __global__ void k(const P<B> p, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = p.b[B - 1];
}
__global__ void spin(long long ns) { long long t0 = clock64(); while (clock64() - t0 < ns) {} }
template <int B> void run(float* out) {
  P<B> p = {};
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  for (int i = 0; i < 10; ++i) k<B><<<256, 256>>>(p, out);
  cudaDeviceSynchronize();
  spin<<<1, 1>>>(20000000);
  cudaEventRecord(s);
  const int R = 500;
  for (int i = 0; i < R; ++i) k<B><<<256, 256>>>(p, out);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  printf("{\"param_bytes\": %d, \"us_per_launch\": %.3f}\n", B, ms * 1e3 / R);
}
int main() {
  float* out; cudaMalloc(&out, 64);
  run<16>(out); run<256>(out); run<1024>(out); run<1400>(out); run<2048>(out); run<4000>(out);
  return 0;
}
