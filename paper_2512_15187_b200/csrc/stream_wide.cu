// Wide-ensemble streaming (n > 4096 members): the same partials as K5 / K6 /
// K9-B (stream_pass.cu) for ensembles whose 256-byte tile column no longer
// fits the SMEM/L2 working set of the one-read kernels.  Two HBM reads of the
// member matrix instead of one:
//
//   wide_col_kernel  : C(x) = sum_i c_i u_i(x), c_i = 1 (S, mean mask) or
//                      inv_i (T), sequential over the members of a row group
//                      in fp64 (for one group this is exactly the
//                      reference's sequential mean_mask accumulation,
//                      grid.py:251-261);
//   wide_fold_kernel : sums the row groups in order and stores f(x) =
//                      w(x) C(x) (S/T modes) or C(x)/n (the mean mask, SIM),
//                      plus per-block partials of sum_x w(x) C(x);
//   wide_row_kernel  : the per-member dots against f (row sweep), one warp
//                      per member row, f and w staged in SMEM per cell chunk;
//   wide_finish_kernel: fixed-order reduction of the split partials.
//
// Everything is deterministic (fixed partition, fixed reduction order).
#include "common.cuh"

namespace pidb {
namespace {

constexpr int kMode_MEAN = 0, kMode_COLS = 1, kMode_MASS = 2, kMode_SIM = 3;  // = stream_pass.cu
constexpr int kColThreads = 256;
constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kRowsPerWarp = 16;  // even: rows are swept in pairs
constexpr int kRowBlock = kRowWarps * kRowsPerWarp;  // 128 members per CTA
constexpr int kChunkCells = 2048;                    // cells per SMEM stage of f/w

template <typename T>
struct WVec;
template <>
struct WVec<float> {
  static constexpr int EPC = 4;
  __device__ static void load(const float* p, double (&v)[4]) {
    const float4 f = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
};
template <>
struct WVec<double> {
  static constexpr int EPC = 2;
  __device__ static void load(const double* p, double (&v)[2]) {
    const double2 f = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = f.x; v[1] = f.y;
  }
};

// part[g][x] = sum_{i in group g} c_i u_i(x)
template <typename T>
__global__ void __launch_bounds__(kColThreads)
    wide_col_kernel(const T* __restrict__ u, int64_t n, int64_t m, int64_t ld,
                    const double* __restrict__ coef, int64_t rows_per_group,
                    double* __restrict__ part, int64_t mpad) {
  constexpr int EPC = WVec<T>::EPC;
  const int64_t x0 = ((int64_t)blockIdx.x * kColThreads + threadIdx.x) * EPC;
  if (x0 >= m) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_group;
  const int64_t r1 = r0 + rows_per_group < n ? r0 + rows_per_group : n;
  double acc[EPC];
#pragma unroll
  for (int e = 0; e < EPC; ++e) acc[e] = 0.0;
  const T* p = u + r0 * ld + x0;
  int64_t r = r0;
  for (; r + 8 <= r1; r += 8, p += 8 * ld) {
    double v[8][EPC];
#pragma unroll
    for (int k = 0; k < 8; ++k) WVec<T>::load(p + k * ld, v[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double c = coef ? __ldg(coef + r + k) : 1.0;
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc[e] = fma(c, v[k][e], acc[e]);
    }
  }
  for (; r < r1; ++r, p += ld) {
    double v[EPC];
    WVec<T>::load(p, v);
    const double c = coef ? __ldg(coef + r) : 1.0;
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[e] = fma(c, v[e], acc[e]);
  }
  double* out = part + (int64_t)blockIdx.y * mpad + x0;
#pragma unroll
  for (int e = 0; e < EPC; ++e)
    if (x0 + e < m) out[e] = acc[e];
}

// f[x] (stored over part[0]) and colpart[block] = sum_x w(x) C(x)
__global__ void __launch_bounds__(256)
    wide_fold_kernel(double* __restrict__ part, int groups, int64_t mpad, int64_t m, int64_t n,
                     const double* __restrict__ w, int mode, double* __restrict__ colpart) {
  __shared__ double red[8];
  double acc = 0.0;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < m;
       x += (int64_t)gridDim.x * blockDim.x) {
    double c = part[x];
    for (int g = 1; g < groups; ++g) c += part[(int64_t)g * mpad + x];
    const double wx = w ? w[x] : 1.0;
    acc = fma(wx, c, acc);
    part[x] = mode == kMode_SIM ? __ddiv_rn(c, (double)n) : wx * c;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    colpart[blockIdx.x] = s;
  }
}

// prow/pmass/pnb[split][r]: this split's partial dots of member r
template <typename T>
__global__ void __launch_bounds__(kRowThreads)
    wide_row_kernel(const T* __restrict__ u, int64_t n, int64_t m, int64_t ld, int mode,
                    const double* __restrict__ f, const double* __restrict__ w,
                    int64_t nchunks, double* __restrict__ prow, double* __restrict__ pmass,
                    int64_t* __restrict__ pnb) {
  constexpr int EPC = WVec<T>::EPC;
  constexpr int kStep = 32 * EPC;
  __shared__ __align__(16) double sf[kChunkCells];
  __shared__ __align__(16) double sw[kChunkCells];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rbase = (int64_t)blockIdx.y * kRowBlock + warp;
  double acc_row[kRowsPerWarp], acc_mass[kRowsPerWarp];
  int64_t acc_nb[kRowsPerWarp];
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) acc_row[k] = acc_mass[k] = 0.0, acc_nb[k] = 0;
  const bool need_f = mode != kMode_MASS;

  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t xb = c * kChunkCells;
    __syncthreads();
    for (int i = threadIdx.x; i < kChunkCells; i += kRowThreads) {
      const int64_t x = xb + i;
      sw[i] = x < m ? (w ? __ldg(w + x) : 1.0) : 0.0;
      if (need_f) sf[i] = x < m ? __ldcg(f + x) : 0.0;
    }
    __syncthreads();
    const int64_t cells = m - xb < kChunkCells ? m - xb : kChunkCells;
    // two member rows per pass and eight 16-byte loads in flight per lane
#pragma unroll 1
    for (int k = 0; k < kRowsPerWarp; k += 2) {
      const int64_t r0 = rbase + (int64_t)k * kRowWarps;
      if (r0 >= n) break;
      const bool two = r0 + kRowWarps < n;
      const T* row0 = u + r0 * ld + xb;
      const T* row1 = two ? row0 + (int64_t)kRowWarps * ld : row0;
      double ar0 = 0.0, am0 = 0.0, ar1 = 0.0, am1 = 0.0;
      int64_t nb0 = 0, nb1 = 0;
      auto body = [&](const double (&v)[EPC], int i, double& ar, double& am, int64_t& nb) {
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const bool in = i + e < cells;
          const double x = in ? v[e] : 0.0;
          const double wx = sw[i + e], fx = sf[i + e];
          if (mode == kMode_SIM) {
            ar = fma(fmin(x, fx), wx, ar);
            am = fma(x, wx, am);
          } else if (mode == kMode_MASS) {
            am = fma(x, wx, am);
            nb += (x != 0.0 && x != 1.0);
          } else {
            ar = fma(x, fx, ar);
            am = fma(x, wx, am);
          }
        }
      };
#pragma unroll 4
      for (int i = lane * EPC; i < cells; i += kStep) {
        double v0[EPC], v1[EPC];
        WVec<T>::load(row0 + i, v0);
        WVec<T>::load(row1 + i, v1);
        body(v0, i, ar0, am0, nb0);
        if (two) body(v1, i, ar1, am1, nb1);
      }
      acc_row[k] += ar0;
      acc_mass[k] += am0;
      acc_nb[k] += nb0;
      if (two) {
        acc_row[k + 1] += ar1;
        acc_mass[k + 1] += am1;
        acc_nb[k + 1] += nb1;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int64_t r = rbase + (int64_t)k * kRowWarps;
    const double ar = warp_sum(acc_row[k]);
    const double am = warp_sum(acc_mass[k]);
    int64_t nb = acc_nb[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0 && r < n) {
      const int64_t slot = (int64_t)blockIdx.x * n + r;
      prow[slot] = ar;
      pmass[slot] = am;
      pnb[slot] = nb;
    }
  }
}

__global__ void wide_finish_kernel(int64_t n, int splits, const double* __restrict__ prow,
                                   const double* __restrict__ pmass,
                                   const int64_t* __restrict__ pnb, const double* colpart,
                                   int ncolpart, double* out_row, double* out_mass,
                                   double* out_col, int64_t* out_nb) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0;
    int64_t nb = 0;
    for (int s = 0; s < splits; ++s) {
      a += prow[(int64_t)s * n + r];
      b += pmass[(int64_t)s * n + r];
      nb += pnb[(int64_t)s * n + r];
    }
    if (out_row) out_row[r] = a;
    if (out_mass) out_mass[r] = b;
    if (out_nb) out_nb[r] = nb;
  }
  if (out_col && blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < ncolpart; ++k) s += colpart[k];
    *out_col = s;
  }
}

struct WidePlan {
  int epc, col_groups, row_blocks, splits, fold_blocks;
  int64_t col_xblocks, rows_per_group, mpad, nchunks;
};

WidePlan wide_plan(int64_t n, int64_t m, int esize) {
  WidePlan pl{};
  pl.epc = 16 / esize;
  const int sms = sm_count();
  pl.col_xblocks = (m + (int64_t)kColThreads * pl.epc - 1) / ((int64_t)kColThreads * pl.epc);
  const int64_t want = (int64_t)sms * 8;
  int64_t g = (want + pl.col_xblocks - 1) / pl.col_xblocks;
  const int64_t gmax = (n + 255) / 256;
  pl.col_groups = (int)std::max<int64_t>(1, std::min<int64_t>(g, gmax));
  pl.rows_per_group = (n + pl.col_groups - 1) / pl.col_groups;
  pl.mpad = (int64_t)align_up((size_t)m, 32);
  pl.nchunks = (m + kChunkCells - 1) / kChunkCells;
  pl.row_blocks = (int)((n + kRowBlock - 1) / kRowBlock);
  const int64_t sp = ((int64_t)sms * 4 + pl.row_blocks - 1) / pl.row_blocks;
  pl.splits = (int)std::max<int64_t>(1, std::min<int64_t>(sp, pl.nchunks));
  pl.fold_blocks = (int)std::min<int64_t>((m + 255) / 256, (int64_t)sms * 4);
  return pl;
}

}  // namespace

size_t wide_workspace(int64_t n, int64_t m, int dtype) {
  const WidePlan pl = wide_plan(n, m, dtype == PIDB_F32 ? 4 : 8);
  size_t b = 256;
  b += align_up((size_t)pl.col_groups * pl.mpad * sizeof(double), 256);
  b += align_up((size_t)pl.fold_blocks * sizeof(double), 256);
  b += 3 * align_up((size_t)pl.splits * n * sizeof(double), 256);
  return b;
}

// Column sweep only (C(x) over all members, folded to f = w*C, or C/n for the
// similarity mode) for the warp-specialised row sweep of wide ensembles.  f
// is left at workspace offset 256 (m doubles); returns the bytes used.
size_t wide_fold_bytes(int64_t n, int64_t m, int dtype) {
  const WidePlan pl = wide_plan(n, m, dtype == PIDB_F32 ? 4 : 8);
  return 256 + align_up((size_t)pl.col_groups * pl.mpad * sizeof(double), 256) +
         align_up((size_t)pl.fold_blocks * sizeof(double), 256);
}

int wide_fold_f(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                const double* w, const double* inv, void* ws, const double** f, void* stream) {
  const WidePlan pl = wide_plan(n, m, dtype == PIDB_F32 ? 4 : 8);
  char* base = static_cast<char*>(ws) + 256;
  double* part = reinterpret_cast<double*>(base);
  double* colpart =
      reinterpret_cast<double*>(base + align_up((size_t)pl.col_groups * pl.mpad * sizeof(double), 256));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 cg((unsigned)pl.col_xblocks, (unsigned)pl.col_groups);
  const double* coef = mode == kMode_COLS ? inv : nullptr;
  if (dtype == PIDB_F32)
    wide_col_kernel<float><<<cg, kColThreads, 0, st>>>(static_cast<const float*>(u), n, m, ld, coef,
                                                       pl.rows_per_group, part, pl.mpad);
  else
    wide_col_kernel<double><<<cg, kColThreads, 0, st>>>(static_cast<const double*>(u), n, m, ld,
                                                        coef, pl.rows_per_group, part, pl.mpad);
  PIDB_LAUNCH_CHECK("wide_col_kernel");
  wide_fold_kernel<<<pl.fold_blocks, 256, 0, st>>>(part, pl.col_groups, pl.mpad, m, n, w, mode,
                                                   colpart);
  PIDB_LAUNCH_CHECK("wide_fold_kernel");
  *f = part;
  return PIDB_OK;
}

int run_wide_pass(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                  const double* w, const double* inv, double* out_row, double* out_mass,
                  double* out_col, int64_t* out_nb, void* ws, size_t ws_bytes, void* stream) {
  const int es = dtype == PIDB_F32 ? 4 : 8;
  const WidePlan pl = wide_plan(n, m, es);
  const size_t need = wide_workspace(n, m, dtype);
  if (ws == nullptr || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return PIDB_EWORKSPACE;
  }
  char* base = static_cast<char*>(ws) + 256;
  double* part = reinterpret_cast<double*>(base);
  base += align_up((size_t)pl.col_groups * pl.mpad * sizeof(double), 256);
  double* colpart = reinterpret_cast<double*>(base);
  base += align_up((size_t)pl.fold_blocks * sizeof(double), 256);
  const size_t pbytes = align_up((size_t)pl.splits * n * sizeof(double), 256);
  double* prow = reinterpret_cast<double*>(base);
  double* pmass = reinterpret_cast<double*>(base + pbytes);
  int64_t* pnb = reinterpret_cast<int64_t*>(base + 2 * pbytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  if (mode != kMode_MASS) {
    const dim3 cg((unsigned)pl.col_xblocks, (unsigned)pl.col_groups);
    const double* coef = mode == kMode_COLS ? inv : nullptr;
    if (dtype == PIDB_F32)
      wide_col_kernel<float><<<cg, kColThreads, 0, st>>>(static_cast<const float*>(u), n, m, ld,
                                                         coef, pl.rows_per_group, part, pl.mpad);
    else
      wide_col_kernel<double><<<cg, kColThreads, 0, st>>>(static_cast<const double*>(u), n, m,
                                                          ld, coef, pl.rows_per_group, part,
                                                          pl.mpad);
    PIDB_LAUNCH_CHECK("wide_col_kernel");
    wide_fold_kernel<<<pl.fold_blocks, 256, 0, st>>>(part, pl.col_groups, pl.mpad, m, n, w, mode,
                                                     colpart);
    PIDB_LAUNCH_CHECK("wide_fold_kernel");
  }
  const dim3 rg((unsigned)pl.splits, (unsigned)pl.row_blocks);
  if (dtype == PIDB_F32)
    wide_row_kernel<float><<<rg, kRowThreads, 0, st>>>(static_cast<const float*>(u), n, m, ld,
                                                       mode, part, w, pl.nchunks, prow, pmass,
                                                       pnb);
  else
    wide_row_kernel<double><<<rg, kRowThreads, 0, st>>>(static_cast<const double*>(u), n, m, ld,
                                                        mode, part, w, pl.nchunks, prow, pmass,
                                                        pnb);
  PIDB_LAUNCH_CHECK("wide_row_kernel");
  const bool col = mode == kMode_MEAN || mode == kMode_SIM;
  wide_finish_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(
      n, pl.splits, prow, pmass, pnb, colpart, pl.fold_blocks,
      mode == kMode_MASS ? nullptr : out_row, mode == kMode_COLS ? nullptr : out_mass,
      col ? out_col : nullptr, mode == kMode_MASS ? out_nb : nullptr);
  PIDB_LAUNCH_CHECK("wide_finish_kernel");
  return PIDB_OK;
}

}  // namespace pidb
