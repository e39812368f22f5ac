// fp64 Gram block on the CUDA cores: the exact seam for gram_block.
//
// Replaces gram_block (/root/reference/pkg/src/fuzzdepth/reduction.py:75-97):
//   out[i, j] = sum_x w(x) rows[i, x] * cols[j, x]      (or * (1 - cols[j, x]))
// for (n, cells) row/column blocks of any float dtype, accumulated in fp64
// like the reference's chunked dgemm (its tests pin rtol 1e-12,
// /root/reference/pkg/tests/test_reduction.py:46-66).  The depth methods do
// not use this kernel (they never form a Gram block in fp64 on the CUDA
// cores); it serves callers of the seam itself, which are small blocks.
//
// 64 x 64 output tile per CTA, 256 threads with a 4 x 4 register tile each,
// cells staged through shared memory in 32-cell slabs (w and the complement
// applied while staging, in fp64).  Split-K over blockIdx.z into a
// workspace, then a fixed-order reduction over the splits: deterministic for
// a given shape, independent of scheduling.
#include "common.cuh"

namespace pidb {
namespace {

constexpr int kT = 64;      // output tile edge
constexpr int kKS = 32;     // cells per shared-memory slab
constexpr int kThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kThreads)
    gram_f64_kernel(const T* __restrict__ rows, int64_t ldr, const T* __restrict__ cols,
                    int64_t ldc, int nr, int nc, int64_t m, const double* __restrict__ w,
                    int complement, int64_t kper, double* __restrict__ part) {
  __shared__ double sa[kKS][kT + 1];
  __shared__ double sb[kKS][kT + 1];
  const int i0 = blockIdx.x * kT, j0 = blockIdx.y * kT;
  const int64_t k0 = (int64_t)blockIdx.z * kper;
  const int64_t k1 = min(m, k0 + kper);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int64_t ks = k0; ks < k1; ks += kKS) {
    // stage: 64 rows x 32 cells of each side; consecutive threads take
    // consecutive cells of one row (coalesced reads)
#pragma unroll
    for (int e = threadIdx.x; e < kT * kKS; e += kThreads) {
      const int r = e / kKS, c = e - r * kKS;
      const int64_t x = ks + c;
      double a = 0.0, b = 0.0;
      if (x < k1) {
        if (i0 + r < nr) {
          a = (double)rows[(int64_t)(i0 + r) * ldr + x];
          if (w) a *= w[x];
        }
        if (j0 + r < nc) {
          b = (double)cols[(int64_t)(j0 + r) * ldc + x];
          if (complement) b = 1.0 - b;
        }
      }
      sa[c][r] = a;
      sb[c][r] = b;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < kKS; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = sa[c][ty + 16 * q];
        b[q] = sb[c][tx + 16 * q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
  double* dst = part + (size_t)blockIdx.z * nr * nc;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int i = i0 + ty + 16 * p;
    if (i >= nr) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + tx + 16 * q;
      if (j < nc) dst[(size_t)i * nc + j] = acc[p][q];
    }
  }
}

__global__ void gram_f64_reduce_kernel(const double* __restrict__ part, int64_t total,
                                       int splits, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(size_t)z * total + e];
    out[e] = s;
  }
}

struct F64Plan {
  int ti, tj, splits;
  int64_t kper;
  size_t ws;
};

F64Plan plan_f64(int64_t nr, int64_t nc, int64_t m) {
  F64Plan p{};
  p.ti = (int)((nr + kT - 1) / kT);
  p.tj = (int)((nc + kT - 1) / kT);
  const int64_t tiles = (int64_t)p.ti * p.tj;
  const int64_t want = std::max<int64_t>(1, (4 * 148 + tiles - 1) / tiles);
  const int64_t maxs = std::max<int64_t>(1, (m + 255) / 256);  // >= 256 cells per split
  p.splits = (int)std::min<int64_t>(std::min(want, maxs), 1024);
  p.kper = (m + p.splits - 1) / p.splits;
  p.kper = (p.kper + kKS - 1) / kKS * kKS;
  p.splits = (int)std::max<int64_t>(1, (m + p.kper - 1) / p.kper);
  p.ws = (size_t)p.splits * nr * nc * sizeof(double);
  return p;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_gram_f64_workspace_bytes(int64_t nr, int64_t nc, int64_t m) {
  if (nr < 1 || nc < 1 || m < 1) return 0;
  return plan_f64(nr, nc, m).ws;
}

extern "C" int pidb_gram_f64(const void* rows, const void* cols, int dtype, int64_t nr,
                             int64_t nc, int64_t m, int64_t ldr, int64_t ldc, const double* w,
                             int complement, double* out, void* ws, size_t ws_bytes,
                             void* stream) {
  PIDB_REQUIRE(rows && cols && out && nr >= 1 && nc >= 1 && m >= 1,
               "bad arguments to pidb_gram_f64");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "unknown dtype %d", dtype);
  PIDB_REQUIRE(ldr >= m && ldc >= m, "row strides must be >= the cell count");
  PIDB_REQUIRE(nr < (1 << 24) && nc < (1 << 24), "block too large");
  const F64Plan p = plan_f64(nr, nc, m);
  PIDB_REQUIRE(ws && ws_bytes >= p.ws, "workspace too small: need %zu bytes", p.ws);
  cudaStream_t st = (cudaStream_t)stream;
  double* part = static_cast<double*>(ws);
  const dim3 grid(p.ti, p.tj, p.splits);
  if (dtype == PIDB_F32)
    gram_f64_kernel<float><<<grid, kThreads, 0, st>>>(
        static_cast<const float*>(rows), ldr, static_cast<const float*>(cols), ldc, (int)nr,
        (int)nc, m, w, complement, p.kper, part);
  else
    gram_f64_kernel<double><<<grid, kThreads, 0, st>>>(
        static_cast<const double*>(rows), ldr, static_cast<const double*>(cols), ldc, (int)nr,
        (int)nc, m, w, complement, p.kper, part);
  PIDB_LAUNCH_CHECK("gram_f64_kernel");
  const int64_t total = nr * nc;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  gram_f64_reduce_kernel<<<blocks, 256, 0, st>>>(part, total, p.splits, out);
  PIDB_LAUNCH_CHECK("gram_f64_reduce_kernel");
  return PIDB_OK;
}
