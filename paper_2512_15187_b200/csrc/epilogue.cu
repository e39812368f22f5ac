// K4: depth epilogues (inverse masses, in_in/in_out, depth = min, ranks) and
// the Gram -> row/column sum reduction; exact eID epilogue.
//
// Reference: _inverse_masses   /root/reference/pkg/src/fuzzdepth/depth.py:164-168
//            _result / ranks   /root/reference/pkg/src/fuzzdepth/depth.py:80-85, 171-189
//            depth_pid         /root/reference/pkg/src/fuzzdepth/depth.py:226-227
//            depth_pid_mean    /root/reference/pkg/src/fuzzdepth/depth.py:274-278
//            depth_eid         /root/reference/pkg/src/fuzzdepth/depth.py:205-209
//            _pairwise_sums    /root/reference/pkg/src/fuzzdepth/depth.py:155-160
//            ref_eid (oracle)  /root/reference/pkg/tests/reference_impl.py:31-40, 60-70
#include "common.cuh"

namespace pidb {
namespace {

__global__ void inverse_masses_kernel(int64_t n, const double* __restrict__ mass,
                                      double* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double mi = mass[i];
    inv[i] = mi > 0.0 ? __ddiv_rn(1.0, mi) : 0.0;
  }
}

// Internal mode (not in the public enum): binary weighted eID.
constexpr int kEpiEidFact = 100;

// mode PID_MEAN: a=row_plain (= N*num), aux[0] = col_mean (= N*mean_mass_total)
// mode PID     : a=row_plain, aux = col_inv
// mode EID_FACT: a=row_plain, aux = col_inv (binary weighted eID via the
//                factorised Gram sums; depth.py:205-209 with
//                row_excess = n*m_i - row_plain, col_inv_excess = n_pos - col_inv)
__global__ void depth_values_kernel(int mode, int64_t n, const double* __restrict__ a,
                                    const double* __restrict__ mass,
                                    const double* __restrict__ aux, double* __restrict__ inv,
                                    double* __restrict__ in_in, double* __restrict__ in_out,
                                    double* __restrict__ depth, double n_pos) {
  const double dn = (double)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double mi = mass[i];
    const double iv = mi > 0.0 ? __ddiv_rn(1.0, mi) : 0.0;
    double ii, io;
    if (mode == PIDB_EPI_PID_MEAN) {
      const double num = __ddiv_rn(a[i], dn);
      const double mean_mass = __ddiv_rn(aux[0], dn);
      ii = __dmul_rn(num, iv);
      io = __ddiv_rn(num, mean_mass);
    } else if (mode == PIDB_EPI_PID) {
      ii = __ddiv_rn(__dmul_rn(iv, a[i]), dn);
      io = __ddiv_rn(aux[i], dn);
    } else if (mode == PIDB_EPI_DICE || mode == PIDB_EPI_IOU) {
      // a = sum w min(u_i, mean), aux[0] = n * mean mass; max = u + mean - min
      const double s_v = __ddiv_rn(aux[0], dn);
      const double den = mode == PIDB_EPI_DICE ? __dadd_rn(mi, s_v)
                                               : __dsub_rn(__dadd_rn(mi, s_v), a[i]);
      ii = mode == PIDB_EPI_DICE ? __ddiv_rn(__dmul_rn(2.0, a[i]), den) : __ddiv_rn(a[i], den);
      io = ii;
    } else {  // kEpiEidFact
      const double row_excess = __dsub_rn(__dmul_rn(dn, mi), a[i]);
      const double col_excess = __dsub_rn(n_pos, aux[i]);
      ii = mi > 0.0 ? __ddiv_rn(__dsub_rn(dn, __dmul_rn(iv, row_excess)), dn) : 0.0;
      io = __ddiv_rn(__dsub_rn(n_pos, col_excess), dn);
    }
    inv[i] = iv;
    in_in[i] = ii;
    in_out[i] = io;
    depth[i] = fmin(ii, io);
  }
}

// rank[i] = #{j : d_j > d_i} + #{j < i : d_j == d_i}  (stable argsort of -depth)
__global__ void ranks_kernel(int64_t n, const double* __restrict__ depth,
                             int64_t* __restrict__ rank) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5); i < n;
       i += warps) {
    const double di = depth[i];
    int64_t c = 0;
    for (int64_t j = lane; j < n; j += 32) {
      const double dj = depth[j];
      c += (dj > di) || (dj == di && j < i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) rank[i] = c;
  }
}

// row_plain[i] = sum_j G[i,j]; col_inv[j] = sum_i inv[i] G[i,j]; fixed order.
__global__ void gram_reduce_kernel(const double* __restrict__ g, int64_t n,
                                   const double* __restrict__ inv, double* __restrict__ row_plain,
                                   double* __restrict__ col_inv) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5); i < n;
       i += warps) {
    double r = 0.0, c = 0.0;
    for (int64_t j = lane; j < n; j += 32) {
      r += g[i * n + j];
      c = fma(inv[j], g[j * n + i], c);
    }
    r = warp_sum(r);
    c = warp_sum(c);
    if (lane == 0) {
      row_plain[i] = r;
      col_inv[i] = c;
    }
  }
}

// ---- exact eID epilogue -----------------------------------------------------
// Every per-pair term t = 1.0 - q (q = fl(e/m) in [0,1]) is a multiple of
// 2^-53 (Sterbenz for q >= 1/2, result >= 1/2 otherwise), so the exact sum of
// the terms is an integer K times 2^-53; K fits 128 bits.  Rounding K*2^-53 to
// double once reproduces math.fsum bit for bit.
__device__ __forceinline__ double u128_to_double_rn(unsigned __int128 k) {
  const uint64_t hi = (uint64_t)(k >> 64);
  if (hi == 0) return __ull2double_rn((uint64_t)k);
  const int lz = __clzll(hi);
  const int shift = 64 - lz;  // bits to drop so that the value fits 64 bits
  const unsigned __int128 top = k >> shift;
  const bool sticky = (k & (((unsigned __int128)1 << shift) - 1)) != 0;
  uint64_t t = (uint64_t)top;  // has its MSB at bit 63
  // keep 53 significant bits from t with round-to-nearest-even, including sticky
  const uint64_t keep = t >> 11;
  const uint64_t rem = t & 0x7FF;
  uint64_t mant = keep;
  if (rem > 0x400 || (rem == 0x400 && (sticky || (keep & 1)))) mant += 1;
  return ldexp((double)mant, shift + 11);
}

__device__ __forceinline__ uint64_t eid_term_bits53(int64_t m_i, int64_t inter) {
  if (m_i <= 0) return 0;
  const double excess = (double)(m_i - inter);
  const double t = __dsub_rn(1.0, __ddiv_rn(excess, (double)m_i));
  // t is an exact multiple of 2^-53 in [0, 1]
  return (uint64_t)__dmul_rn(t, 9007199254740992.0);  // * 2^53, exact
}

// Warp per member i.  I is symmetric (the reduction mirrors it), so both
// sums read row i: row += term(m_i, I_ij), col += term(m_j, I_ij), with the
// masses m_j = I_jj staged per block in shared memory (one strided read per
// block instead of one per warp).
constexpr int kDiagChunk = 1024;
constexpr int kEidWarpsPerRow = 4;  // 4 warps share a row: 4x the warps in flight
__global__ void eid_exact_kernel(const int64_t* __restrict__ g, int64_t n,
                                 double* __restrict__ in_in, double* __restrict__ in_out,
                                 double* __restrict__ depth, double* __restrict__ mass) {
  __shared__ int64_t sdiag[kDiagChunk];
  __shared__ unsigned __int128 spart[2][32];  // per-warp (row, col) sums, <= 32 warps
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rpb = (blockDim.x >> 5) / kEidWarpsPerRow;  // rows per block
  const int sub = warp % kEidWarpsPerRow;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < n; base += (int64_t)gridDim.x * rpb) {
    const int64_t i = base + warp / kEidWarpsPerRow;
    const bool live = i < n;
    const int64_t mi = live ? g[i * n + i] : 0;
    unsigned __int128 row = 0, col = 0;
    for (int64_t j0 = 0; j0 < n; j0 += kDiagChunk) {
      const int cnt = (int)(n - j0 < kDiagChunk ? n - j0 : kDiagChunk);
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) sdiag[t] = g[(j0 + t) * (n + 1)];
      __syncthreads();
      if (live) {
        const int64_t* gi = g + i * n + j0;
        for (int t = sub * 32 + lane; t < cnt; t += 32 * kEidWarpsPerRow) {
          const int64_t gij = gi[t];
          row += eid_term_bits53(mi, gij);
          col += eid_term_bits53(sdiag[t], gij);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t rl = __shfl_xor_sync(0xffffffffu, (uint64_t)row, o);
      const uint64_t rh = __shfl_xor_sync(0xffffffffu, (uint64_t)(row >> 64), o);
      const uint64_t cl = __shfl_xor_sync(0xffffffffu, (uint64_t)col, o);
      const uint64_t ch = __shfl_xor_sync(0xffffffffu, (uint64_t)(col >> 64), o);
      row += ((unsigned __int128)rh << 64) | rl;
      col += ((unsigned __int128)ch << 64) | cl;
    }
    if (lane == 0) {
      spart[0][warp] = row;
      spart[1][warp] = col;
    }
    __syncthreads();
    if (live && lane == 0 && sub == 0) {
      // integer sums: exact in any order
      for (int s = 1; s < kEidWarpsPerRow; ++s) {
        row += spart[0][warp + s];
        col += spart[1][warp + s];
      }
      if (mass) mass[i] = (double)mi;  // |C_i|, exact
      const double rs = __dmul_rn(u128_to_double_rn(row), 1.1102230246251565e-16);  // 2^-53
      const double cs = __dmul_rn(u128_to_double_rn(col), 1.1102230246251565e-16);
      const double ii = __ddiv_rn(rs, (double)n);
      const double io = __ddiv_rn(cs, (double)n);
      in_in[i] = ii;
      in_out[i] = io;
      depth[i] = fmin(ii, io);
    }
  }
}

int blocks_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 4 * 148));
}

int launch_ranks(int64_t n, const double* depth, int64_t* rank, cudaStream_t st) {
  if (rank == nullptr) return PIDB_OK;
  ranks_kernel<<<blocks_for(n, 8), 256, 0, st>>>(n, depth, rank);
  PIDB_LAUNCH_CHECK("ranks_kernel");
  return PIDB_OK;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" int pidb_inverse_masses(int64_t n, const double* mass, double* inv, void* stream) {
  PIDB_REQUIRE(n >= 1 && mass && inv, "bad arguments to pidb_inverse_masses");
  inverse_masses_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, mass, inv);
  PIDB_LAUNCH_CHECK("inverse_masses_kernel");
  return PIDB_OK;
}

extern "C" int pidb_depth_epilogue(int mode, int64_t n, const double* a, const double* mass,
                                   const double* aux, double* inv, double* in_in,
                                   double* in_out, double* depth, int64_t* rank, void* stream) {
  PIDB_REQUIRE(n >= 1, "n must be >= 1");
  PIDB_REQUIRE(a && mass && aux && inv && in_in && in_out && depth, "NULL epilogue pointer");
  PIDB_REQUIRE(mode >= PIDB_EPI_PID_MEAN && mode <= PIDB_EPI_IOU, "unknown epilogue mode %d", mode);
  cudaStream_t st = (cudaStream_t)stream;
  depth_values_kernel<<<blocks_for(n, 256), 256, 0, st>>>(mode, n, a, mass, aux, inv, in_in,
                                                          in_out, depth, 0.0);
  PIDB_LAUNCH_CHECK("depth_values_kernel");
  return launch_ranks(n, depth, rank, st);
}

extern "C" int pidb_eid_factorized_epilogue(int64_t n, const double* row_plain,
                                            const double* mass, const double* col_inv,
                                            double n_pos, double* inv, double* in_in,
                                            double* in_out, double* depth, int64_t* rank,
                                            void* stream) {
  PIDB_REQUIRE(n >= 1 && row_plain && mass && col_inv && inv && in_in && in_out && depth,
               "bad arguments to pidb_eid_factorized_epilogue");
  cudaStream_t st = (cudaStream_t)stream;
  depth_values_kernel<<<blocks_for(n, 256), 256, 0, st>>>(kEpiEidFact, n, row_plain, mass, col_inv, inv,
                                                          in_in, in_out, depth, n_pos);
  PIDB_LAUNCH_CHECK("depth_values_kernel");
  return launch_ranks(n, depth, rank, st);
}

extern "C" int pidb_gram_reduce(const double* gram, int64_t n, const double* inv,
                                double* row_plain, double* col_inv, void* stream) {
  PIDB_REQUIRE(n >= 1 && gram && inv && row_plain && col_inv, "bad arguments to pidb_gram_reduce");
  gram_reduce_kernel<<<blocks_for(n, 8), 256, 0, (cudaStream_t)stream>>>(gram, n, inv, row_plain,
                                                                         col_inv);
  PIDB_LAUNCH_CHECK("gram_reduce_kernel");
  return PIDB_OK;
}

extern "C" int pidb_eid_exact_epilogue(const int64_t* gram, int64_t n, double* in_in,
                                       double* in_out, double* depth, int64_t* rank,
                                       double* mass, void* stream) {
  PIDB_REQUIRE(n >= 1 && gram && in_in && in_out && depth, "bad arguments to pidb_eid_exact_epilogue");
  cudaStream_t st = (cudaStream_t)stream;
  eid_exact_kernel<<<blocks_for(n, 256 / 32 / kEidWarpsPerRow), 256, 0, st>>>(gram, n, in_in,
                                                                              in_out, depth, mass);
  PIDB_LAUNCH_CHECK("eid_exact_kernel");
  return launch_ranks(n, depth, rank, st);
}

extern "C" int pidb_ranks(int64_t n, const double* depth, int64_t* rank, void* stream) {
  PIDB_REQUIRE(n >= 1 && depth && rank, "bad arguments to pidb_ranks");
  return launch_ranks(n, depth, rank, (cudaStream_t)stream);
}
