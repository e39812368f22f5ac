// Microbenchmark: tcgen05.mma.kind::i8 issue rate per SM for the K1x
// operand pattern.  One CTA per SM, one thread issuing MMAs from fixed
// shared-memory descriptors (no loads: pure tensor-pipe rate), committing to
// an mbarrier every "stage" of P MMAs and waiting two stages behind.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        tools/ubench_mma.cu -o tools/ubench_mma && tools/ubench_mma
#include <cstdio>

#include "../paper_2512_15187_b200/csrc/tcgen05.cuh"

using namespace pidb;

template <int N, int NACC, int P>
__global__ void __launch_bounds__(128, 1) mma_rate(int stages, long long* cyc, int fill) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* buf = smem_raw + pad;
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (fill)  // random digits (0..255, as the K1x digit planes) instead of zeros
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
      reinterpret_cast<uint32_t*>(buf)[i] = (uint32_t)(i * 2654435761u + blockIdx.x * 40503u) ^ 0x5bd1e995u;
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  const uint32_t id = (tc::kCS32 << 4) | (tc::kU8 << 7) | (tc::kU8 << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 32) {
    const uint64_t da = tc::desc_kmajor_sw128(smem_u32(buf));
    const uint64_t db = tc::desc_kmajor_sw128(smem_u32(buf + 16384));
    long long t0 = clock64();
    uint32_t ph[2] = {0, 0};
    for (int s = 0; s < stages; ++s) {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const int acc = NACC == 1 ? 0 : (k % NACC);
        tc::mma_i8(tmem + (uint32_t)(acc * N), da + 2 * (k & 3), db + 2 * ((k >> 2) & 3), id,
                   (s | k) != 0);
      }
      tc::commit(&bar[s & 1]);
      if (s >= 1) {
        mbar_wait(&bar[(s - 1) & 1], ph[(s - 1) & 1]);
        ph[(s - 1) & 1] ^= 1u;
      }
    }
    mbar_wait(&bar[(stages - 1) & 1], ph[(stages - 1) & 1]);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

template <int N, int NACC, int P>
void run(const char* name, int fill) {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 1024 + 65536;
  cudaFuncSetAttribute(mma_rate<N, NACC, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 20000;
  mma_rate<N, NACC, P><<<148, 128, smem>>>(100, d, fill);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mma_rate<N, NACC, P><<<148, 128, smem>>>(stages, d, fill);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double mmas = (double)stages * P;
  const double macs = mmas * 128.0 * N * 32.0 * 148.0;
  printf("%s %-34s %7.1f cyc/MMA  %6.1f ns/MMA  %7.0f TOPS (chip, 2 ops/MAC)  clk %.0f MHz  %s\n", fill ? "random" : "zeros ", name,
         cyc / mmas, ms * 1e6 / mmas, 2.0 * macs / (ms * 1e-3) / 1e12, cyc / (ms * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int fill = 0; fill < 2; ++fill) {
    run<128, 4, 10>("N=128, 4 accumulators, 10/stage", fill);
    run<256, 2, 10>("N=256, 2 accumulators, 10/stage", fill);
    run<256, 1, 4>("N=256, 1 accumulator, 4/stage", fill);
  }
  return 0;
}
