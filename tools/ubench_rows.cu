// Row-segment width vs HBM read throughput for the K5 tile shape, with a
// per-tile hold that mimics the sweeps keeping a stage busy before refill:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_rows tools/ubench_rows.cu -lcuda
// N = 200 member rows per box, W floats per row segment, `stages` ring
// buffers per CTA, 148 CTAs; hold = spin of `hold` ns per 256 B of row width
// after a tile lands and before its buffer is refilled.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>

#include "../paper_2512_15187_b200/csrc/common.cuh"

using namespace pidb;

__global__ void __launch_bounds__(128) rows(const __grid_constant__ CUtensorMap tm, int N, int W,
                                            int stages, long long tiles, long long hold_cycles,
                                            unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  const uint32_t tile_bytes = (uint32_t)N * W * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)stages * tile_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const long long G = gridDim.x;
  const long long mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / G + 1 : 0;
  const uint64_t pol = policy_evict_first();
  auto issue = [&](long long j) {
    const int s = (int)(j % stages);
    mbar_arrive_expect_tx(&full[s], tile_bytes);
    tma_load_2d(ring + (size_t)s * tile_bytes, &tm, (int)((blockIdx.x + j * G) * W), 0, &full[s], pol);
  };
  if (threadIdx.x == 0)
    for (long long j = 0; j < mine && j < stages; ++j) issue(j);
  unsigned long long acc = 0;
  for (long long j = 0; j < mine; ++j) {
    const int s = (int)(j % stages);
    mbar_wait(&full[s], (uint32_t)((j / stages) & 1));
    acc += ring[(size_t)s * tile_bytes + threadIdx.x * 4];
    if (hold_cycles) {
      const long long t0 = clock64();
      while (clock64() - t0 < hold_cycles) {}
    }
    __syncthreads();
    if (threadIdx.x == 0 && j + stages < mine) issue(j + stages);
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  const size_t bytes = (size_t)24 << 30;
  float* d = nullptr;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 200;
  for (int hold_ns : {0, 400, 800, 1600}) {
    for (int W : {64, 80, 96, 128}) {
      for (int stages = 2; stages <= 4; ++stages) {
        const size_t tile_bytes = (size_t)N * W * 4;
        const size_t smem = 1024 + stages * tile_bytes + 256;
        if (smem > 227 * 1024) continue;
        const long long M = (long long)(bytes / 4 / N) / 1024 * 1024;
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N};
        cuuint64_t strides[1] = {(cuuint64_t)M * 4};
        cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)N};
        cuuint32_t es[2] = {1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          printf("encode W=%d failed\n", W);
          continue;
        }
        const long long tiles = M / W;
        const long long hold = (long long)hold_ns * W / 64 * 19 / 10;  // ~1.9 GHz
        cudaFuncSetAttribute(rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float ms = 1e30f;  // best of 8 (the first is a warm-up)
        for (int rep = 0; rep < 8; ++rep) {
          float t = 0;
          cudaEventRecord(a);
          rows<<<148, 128, smem>>>(tm, N, W, stages, tiles, hold, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&t, a, b);
          if (rep > 0 && t < ms) ms = t;
        }
        printf("hold=%4d ns/256B row=%4d B stages=%d stage=%6zu B: %7.1f GB/s (%s)\n", hold_ns,
               W * 4, stages, tile_bytes, (double)tiles * W * N * 4 / 1e9 / (ms * 1e-3),
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
