// Microbenchmark: throughput of F2F.F64.F32 conversion, DADD/DFMA and fp32 TwoSum on sm_100a.
// Used once to size the PID-mean kernel's arithmetic.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_f2f(float seed, double* out) {
  double acc[8] = {0};
  float x = seed + threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc[j] += (double)x; x = x * 1.0000001f; }
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_dadd(double seed, double* out) {
  double acc[8] = {0}; double x = seed + threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc[j] = fma(acc[j], 1.0000001, x); }
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_twosum(float seed, float* out) {
  float s[8] = {0}, c[8] = {0}; float x = seed + threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float t = s[j] + x; float bp = t - s[j]; float e = (s[j] - (t - bp)) + (x - bp);
      s[j] = t; c[j] += e; x = x * 1.0000001f;
    }
  }
  float r = 0; for (int j = 0; j < 8; ++j) r += s[j] + c[j];
  if (r == 12345.0f) out[0] = r;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  dim3 grid(sms * 8), block(256);
  double elems = (double)grid.x * block.x * ITERS * 8;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); k_f2f<<<grid, block>>>(1.0f, d); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("f2f+dadd: %.3e elem/s  (%.2f per SM per ns)\n", elems / (ms * 1e-3), elems / (ms * 1e-3) / sms / 1e9);
    cudaEventRecord(a); k_dadd<<<grid, block>>>(1.0, d); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("dfma: %.3e op/s  (%.2f per SM per ns)\n", elems / (ms * 1e-3), elems / (ms * 1e-3) / sms / 1e9);
    cudaEventRecord(a); k_twosum<<<grid, block>>>(1.0f, (float*)d); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("twosum: %.3e elem/s  (%.2f per SM per ns)\n", elems / (ms * 1e-3), elems / (ms * 1e-3) / sms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
