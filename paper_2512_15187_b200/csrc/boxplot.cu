// K10: contour-boxplot band envelopes, one HBM pass over the deepest members.
//
// Replaces the member loop of build_boxplot
// (/root/reference/pkg/src/fuzzdepth/boxplot.py:43-101): band b holds the
// members of rank < k_b (k_b = ceil(p_b * n), ascending), its union is the
// cell-wise OR and its intersection the AND of their binarised masks
// {u >= t} (grid.py:264-268, compared in the member dtype like numpy does
// with a Python-float threshold).
//
// Bands are nested by rank, so per cell two integers decide every band:
//   first_in  = smallest rank r < kmax whose member has u >= t,
//   first_out = smallest rank r < kmax whose member has u <  t;
// union_b = first_in < k_b, intersection_b = first_out >= k_b.  Each thread
// owns one 16-byte vector of cells and walks the members in rank order
// (member_by_rank gives the matrix row of each rank), so the kernel reads
// kmax * m values once, coalesced, and writes 2 * nbands bytes per cell.
#include "common.cuh"

namespace pidb {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxBands = 64;

template <typename T>
struct BVec;
template <>
struct BVec<float> {
  static constexpr int EPC = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 f = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
};
template <>
struct BVec<double> {
  static constexpr int EPC = 2;
  __device__ static void load(const double* p, double (&v)[2]) {
    const double2 f = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = f.x; v[1] = f.y;
  }
};

template <typename T>
__global__ void __launch_bounds__(kThreads)
    band_envelope_kernel(const T* __restrict__ u, int64_t m, int64_t ld,
                         const int64_t* __restrict__ member_by_rank, int kmax, T t,
                         const int64_t* __restrict__ cutoffs, int nbands,
                         uint8_t* __restrict__ unions, uint8_t* __restrict__ inters) {
  constexpr int EPC = BVec<T>::EPC;
  __shared__ int64_t s_row[1024];
  __shared__ int s_cut[kMaxBands];
  for (int b = threadIdx.x; b < nbands; b += kThreads) s_cut[b] = (int)cutoffs[b];
  const int64_t x0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * EPC;
  int fin[EPC], fout[EPC];
#pragma unroll
  for (int e = 0; e < EPC; ++e) fin[e] = fout[e] = kmax;
  for (int r0 = 0; r0 < kmax; r0 += 1024) {
    const int rn = min(1024, kmax - r0);
    __syncthreads();
    for (int r = threadIdx.x; r < rn; r += kThreads) s_row[r] = member_by_rank[r0 + r];
    __syncthreads();
    if (x0 < m) {
      int r = 0;
      for (; r + 4 <= rn; r += 4) {  // four member rows in flight
        T v[4][EPC];
#pragma unroll
        for (int k = 0; k < 4; ++k) BVec<T>::load(u + s_row[r + k] * ld + x0, v[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < EPC; ++e) {
            const int rr = r0 + r + k;
            if (v[k][e] >= t) fin[e] = min(fin[e], rr);
            else fout[e] = min(fout[e], rr);
          }
      }
      for (; r < rn; ++r) {
        T v[EPC];
        BVec<T>::load(u + s_row[r] * ld + x0, v);
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          if (v[e] >= t) fin[e] = min(fin[e], r0 + r);
          else fout[e] = min(fout[e], r0 + r);
        }
      }
    }
  }
  if (x0 >= m) return;
  for (int b = 0; b < nbands; ++b) {
    const int k = s_cut[b];
#pragma unroll
    for (int e = 0; e < EPC; ++e) {
      const int64_t x = x0 + e;
      if (x < m) {
        unions[(int64_t)b * m + x] = fin[e] < k;
        inters[(int64_t)b * m + x] = fout[e] >= k;
      }
    }
  }
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" int pidb_band_envelopes(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                                   const int64_t* member_by_rank, int64_t kmax,
                                   double threshold, const int64_t* cutoffs, int nbands,
                                   uint8_t* unions, uint8_t* inters, void* stream) {
  PIDB_REQUIRE(u && member_by_rank && cutoffs && unions && inters, "NULL pointer argument");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  PIDB_REQUIRE(n >= 1 && m >= 1 && ld >= m, "bad shape (n %lld, m %lld, ld %lld)", (long long)n,
               (long long)m, (long long)ld);
  PIDB_REQUIRE(kmax >= 1 && kmax <= n, "kmax %lld outside [1, n]", (long long)kmax);
  PIDB_REQUIRE(nbands >= 1 && nbands <= kMaxBands, "nbands %d outside [1, %d]", nbands, kMaxBands);
  const int es = dtype == PIDB_F32 ? 4 : 8;
  PIDB_REQUIRE((ld * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0,
               "member rows must be 16-byte aligned");
  const int epc = 16 / es;
  const int64_t blocks = (m + (int64_t)kThreads * epc - 1) / ((int64_t)kThreads * epc);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == PIDB_F32)
    band_envelope_kernel<float><<<(unsigned)blocks, kThreads, 0, st>>>(
        static_cast<const float*>(u), m, ld, member_by_rank, (int)kmax, (float)threshold, cutoffs,
        nbands, unions, inters);
  else
    band_envelope_kernel<double><<<(unsigned)blocks, kThreads, 0, st>>>(
        static_cast<const double*>(u), m, ld, member_by_rank, (int)kmax, threshold, cutoffs,
        nbands, unions, inters);
  PIDB_LAUNCH_CHECK("band_envelope_kernel");
  return PIDB_OK;
}
