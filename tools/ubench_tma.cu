// Microbenchmark: HBM streaming bandwidth of 2D TMA tiles (no compute).
// A tile = `boxes` boxes of (32 fp32 x R rows) from an (N x M) row-major
// matrix; each CTA streams tiles round-robin through a ring of `stages`
// buffers.  Reports GB/s for several (N, R, column-boxes, stages) shapes to
// size the K5/K9 tiles.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2512_15187_b200/csrc/common.cuh"

namespace pidb {
void set_error(const char*, ...) {}
int check_cuda(cudaError_t e, const char*) { return e == cudaSuccess ? 0 : -2; }
int sm_count() { return 148; }
}  // namespace pidb

using namespace pidb;

__global__ void __launch_bounds__(128) stream_tiles(const __grid_constant__ CUtensorMap tm, int N, int R,
                                                       int ncb, int stages, long long tiles, int V,
                                                       unsigned long long* sink, int hint) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  const int nrb = (N + R - 1) / R;
  const uint32_t tile_bytes = (uint32_t)ncb * nrb * R * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)stages * tile_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const long long G = gridDim.x;
  const long long mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / G + 1 : 0;
  const uint64_t pol = hint == 1 ? policy_evict_first() : (hint == 2 ? policy_evict_last() : 0ull);
  auto issue = [&](long long j) {
    const int s = (int)(j % stages);
    const long long tile = blockIdx.x + j * G;
    unsigned char* dst = ring + (size_t)s * tile_bytes;
    mbar_arrive_expect_tx(&full[s], tile_bytes);
    for (int cb = 0; cb < ncb; ++cb)
      for (int rb = 0; rb < nrb; ++rb)
        if (hint)
          tma_load_2d(dst + (size_t)(cb * nrb + rb) * R * 128, &tm, (int)(tile * V + cb * 32), rb * R,
                      &full[s], pol);
        else
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst + (size_t)(cb * nrb + rb) * R * 128)),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&full[s])), "r"((int)(tile * V + cb * 32)),
              "r"(rb * R)
              : "memory");
  };
  if (threadIdx.x == 0)
    for (long long j = 0; j < mine && j < stages; ++j) issue(j);
  unsigned long long acc = 0;
  for (long long j = 0; j < mine; ++j) {
    const int s = (int)(j % stages);
    mbar_wait(&full[s], (uint32_t)((j / stages) & 1));
    acc += ring[(size_t)s * tile_bytes + threadIdx.x * 4];
    __syncthreads();
    if (threadIdx.x == 0 && j + stages < mine) issue(j + stages);
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

__global__ void __launch_bounds__(128) stream_wide(const __grid_constant__ CUtensorMap tm, int N, int W,
                                                    int stages, long long tiles, unsigned long long* sink) {
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
    const long long tile = blockIdx.x + j * G;
    mbar_arrive_expect_tx(&full[s], tile_bytes);
    tma_load_2d(ring + (size_t)s * tile_bytes, &tm, (int)(tile * W), 0, &full[s], pol);
  };
  if (threadIdx.x == 0)
    for (long long j = 0; j < mine && j < stages; ++j) issue(j);
  unsigned long long acc = 0;
  for (long long j = 0; j < mine; ++j) {
    const int s = (int)(j % stages);
    mbar_wait(&full[s], (uint32_t)((j / stages) & 1));
    acc += ring[(size_t)s * tile_bytes + threadIdx.x * 4];
    __syncthreads();
    if (threadIdx.x == 0 && j + stages < mine) issue(j + stages);
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

// 1D bulk copies: one cp.async.bulk per member row segment of `seg` bytes.
__global__ void __launch_bounds__(128) stream_bulk(const float* base, long long M, int N, int seg,
                                                    int stages, long long tiles,
                                                    unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  const uint32_t tile_bytes = (uint32_t)N * seg;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)stages * tile_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const long long G = gridDim.x;
  const long long mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / G + 1 : 0;
  const int V = seg / 4;
  auto issue = [&](long long j) {  // issued by warp 0 lanes
    const int s = (int)(j % stages);
    const long long tile = blockIdx.x + j * G;
    unsigned char* dst = ring + (size_t)s * tile_bytes;
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&full[s], tile_bytes);
    __syncwarp();
    for (int r = threadIdx.x; r < N; r += 32) {
      const float* src = base + (long long)r * M + tile * V;
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(dst + (size_t)r * seg)), "l"(src), "r"(seg), "r"(smem_u32(&full[s]))
                   : "memory");
    }
  };
  if (threadIdx.x < 32)
    for (long long j = 0; j < mine && j < stages; ++j) issue(j);
  unsigned long long acc = 0;
  for (long long j = 0; j < mine; ++j) {
    const int s = (int)(j % stages);
    mbar_wait(&full[s], (uint32_t)((j / stages) & 1));
    acc += ring[(size_t)s * tile_bytes + threadIdx.x * 4];
    __syncthreads();
    if (threadIdx.x < 32 && j + stages < mine) issue(j + stages);
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

// plain 128-bit loads: warp w of CTA reads member rows, lanes cover 512 B of a row
__global__ void __launch_bounds__(512) stream_ldg(const float4* base, long long M4, int N, long long tiles,
                                                  unsigned long long* sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc = 0.f;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
#pragma unroll 4
    for (int r = warp; r < N; r += 16) {
      float4 v = __ldcs(base + (long long)r * M4 + t * 32 + lane);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == -1.0f) *sink = 1;
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const size_t bytes = (size_t)16 << 30;  // 16 GB matrix
  float* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  struct Case { int N, R, ncb, stages; };
  std::vector<Case> cases = {{200, 200, 2, 4}};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (const Case& c : cases) {
    const long long M = (long long)(bytes / 4 / c.N) / 32 * 32;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)c.N};
    cuuint64_t strides[1] = {(cuuint64_t)M * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)c.R};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    const int V = 32 * c.ncb;
    const long long tiles = M / V;
    const int nrb = (c.N + c.R - 1) / c.R;
    const size_t tile_bytes = (size_t)c.ncb * nrb * c.R * 128;
    const size_t smem = 1024 + c.stages * tile_bytes + 256;
    if (smem > 227 * 1024) { printf("N=%d R=%d ncb=%d stages=%d: smem %zu too big\n", c.N, c.R, c.ncb, c.stages, smem); continue; }
    cudaFuncSetAttribute(stream_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int hint = 0; hint < 3; ++hint)
    for (int ctas = 1; ctas <= 2; ++ctas) {
      if (ctas == 2 && 2 * smem > 228 * 1024) continue;
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        stream_tiles<<<148 * ctas, 128, smem>>>(tm, c.N, c.R, c.ncb, c.stages, tiles, V, sink, hint);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      const double gb = (double)tiles * V * c.N * 4 / 1e9;
      printf("TMA2D N=%4d R=%3d boxes/row=%d stages=%d ctas/SM=%d hint=%d tile=%6zu B: %7.1f GB/s (%s)\n",
             c.N, c.R, c.ncb, c.stages, ctas, hint, tile_bytes, gb / (ms * 1e-3),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  // unswizzled wide boxes: inner = W floats per row, one box per tile (N rows)
  for (int N : {200, 100}) {
    for (int W : {32, 64, 128, 256}) {
      const long long M = (long long)(bytes / 4 / N) / 256 * 256;
      CUtensorMap tm;
      cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N};
      cuuint64_t strides[1] = {(cuuint64_t)M * 4};
      cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)N};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode W=%d failed %d\n", W, (int)r); continue; }
      // reuse stream_tiles with R=N, ncb=1 and "128-byte" accounting replaced: tile bytes = N*W*4
      const size_t tile_bytes = (size_t)N * W * 4;
      int stages = (int)((200 * 1024) / tile_bytes);
      if (stages > 8) stages = 8;
      if (stages < 2) { printf("W=%d too big\n", W); continue; }
      const long long tiles = M / W;
      const size_t smem = 1024 + stages * tile_bytes + 256;
      cudaFuncSetAttribute(stream_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        stream_wide<<<148, 128, smem>>>(tm, N, W, stages, tiles, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("TMA2D-noswz N=%4d row=%4d B stages=%d tile=%6zu B: %7.1f GB/s (%s)\n", N, W * 4, stages,
             tile_bytes, (double)tiles * W * N * 4 / 1e9 / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
  }

  // 1D bulk and plain loads
  for (int N : {200, 1000}) {
    const long long M = (long long)(bytes / 4 / N) / 256 * 256;
    for (int seg : {256, 512, 1024}) {
      const int stages = 3;
      const size_t tile_bytes = (size_t)N * seg;
      const size_t smem = 1024 + stages * tile_bytes + 256;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(stream_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const long long tiles = M / (seg / 4);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        stream_bulk<<<148, 128, smem>>>(d, M, N, seg, stages, tiles, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("BULK1D N=%4d seg=%4d B stages=%d: %7.1f GB/s (%s)\n", N, seg, stages,
             (double)tiles * seg * N / 1e9 / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
    const long long tiles = M / 128;
    for (int blocks : {148, 296, 592}) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        stream_ldg<<<blocks, 512>>>(reinterpret_cast<const float4*>(d), M / 4, N, tiles, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("LDG128 N=%4d 512B/row-seg blocks=%d: %7.1f GB/s (%s)\n", N, blocks,
             (double)tiles * 512 * N / 1e9 / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
