// K7 binary check/pack, K8 pair sums (prob_inclusion / subset_epsilon) and the
// device-side synthetic ensembles used by the benchmark and GPU tests.
//
// Reference: prob_inclusion   /root/reference/pkg/src/fuzzdepth/inclusion.py:22-40
//            subset_epsilon   /root/reference/pkg/src/fuzzdepth/inclusion.py:43-64
//            ProbMask.is_binary /root/reference/pkg/src/fuzzdepth/grid.py:125-127
//            _fuzzy_ellipsoid /root/reference/pkg/src/fuzzdepth/synth.py:138-162
//            gen_fuzzy_disk   /root/reference/pkg/src/fuzzdepth/synth.py:30-51
#include "common.cuh"

namespace pidb {
namespace {

// ------------------------------------------------------------------ K7 ------
// One warp per (member, 512-cell segment); 16-byte loads; every lane packs 16
// cells = one 16-byte chunk of the member's 128-byte line in the 16 KB tile
// (row block, cell block) of the tiled layout K2 reads with 1D bulk copies:
// line i % 128 of the tile, chunk c stored at c ^ (i % 8) (128-byte swizzle).
template <typename T>
__global__ void binary_pack_kernel(const T* __restrict__ u, int64_t n, int64_t m, int64_t ld,
                                   uint8_t* __restrict__ tiles, int64_t nkb,
                                   unsigned long long* __restrict__ nonbinary) {
  const int64_t span = nkb * 128;  // packed cells per member (zero past m)
  const int64_t segs = (span + 511) / 512;
  // padding members up to the K2 panel height (a multiple of 256) are
  // written as zeros: the tile buffer needs no zero fill
  const int64_t rows = tiles ? (n + 255) / 256 * 256 : n;  // NULL tiles: count only
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t job = wid; job < rows * segs; job += nw) {
    const int64_t i = job / segs;
    const int64_t x0 = (job - i * segs) * 512 + lane * 16;
    const bool live = i < n;
    const T* row = u + (live ? i : 0) * ld;
    unsigned long long bad = 0;
    uint32_t packed[4] = {0, 0, 0, 0};
    T vals[16];
    if (!live) {
#pragma unroll
      for (int e = 0; e < 16; ++e) vals[e] = T(0);
    } else if (x0 + 16 <= m) {  // 16-byte vector loads (rows are 16-byte aligned)
      constexpr int PER = 16 / sizeof(T);
#pragma unroll
      for (int k = 0; k < 16 / PER; ++k) {
        const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(row + x0) + k);
        const T* t = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int e = 0; e < PER; ++e) vals[k * PER + e] = t[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) vals[e] = x0 + e < m ? row[x0 + e] : T(0);
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const T v = vals[e];
      bad += !(v == T(0) || v == T(1));
      packed[e >> 2] |= (uint32_t)(v != T(0)) << (8 * (e & 3));
    }
    if (tiles && x0 < span) {
      const int r = (int)(i & 127);
      const int c = (int)((x0 & 127) >> 4);
      uint8_t* dst = tiles + ((i >> 7) * nkb + (x0 >> 7)) * (int64_t)16384 + r * 128 +
                     (((c ^ r) & 7) << 4);
      PIDB_DCHECK((i >> 7) < 2 * ((n + 255) / 256) && (x0 >> 7) < nkb, "K7 tile bounds");
      *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane == 0 && bad && nonbinary && live) atomicAdd(&nonbinary[i], bad);
  }
}

// ------------------------------------------------------------------ K8 ------
// op 0 (prob_inclusion):  [sum w u v, sum w u]
// op 1 (subset_epsilon):  [sum w a (b == 0), sum w a]
// op 2 (_min_max_terms, inclusion.py:67-88): [sum w min, sum w max, sum w u, sum w v]
template <typename T>
__global__ void pair_sums_kernel(const T* __restrict__ u, const T* __restrict__ v, int64_t m,
                                 const double* __restrict__ w, int op,
                                 double* __restrict__ part) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m;
       x += (int64_t)gridDim.x * blockDim.x) {
    const double a = (double)u[x];
    const double bv = (double)v[x];
    const double wx = w ? w[x] : 1.0;
    if (op == 2) {
      acc[0] = fma(wx, fmin(a, bv), acc[0]);
      acc[1] = fma(wx, fmax(a, bv), acc[1]);
      acc[2] = fma(wx, a, acc[2]);
      acc[3] = fma(wx, bv, acc[3]);
    } else {
      const double wa = a * wx;
      acc[0] = fma(wa, op == 1 ? (bv != 0.0 ? 0.0 : 1.0) : bv, acc[0]);
      acc[1] += wa;
    }
  }
  __shared__ double s[4][32];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double t = warp_sum(acc[q]);
    if ((threadIdx.x & 31) == 0) s[q][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += s[threadIdx.x][k];
    part[4 * blockIdx.x + threadIdx.x] = t;
  }
}

__global__ void pair_finish_kernel(const double* __restrict__ part, int nb, double* out) {
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = threadIdx.x; k < nb; k += 32)
    for (int q = 0; q < 4; ++q) a[q] += part[4 * k + q];
  for (int q = 0; q < 4; ++q) {
    const double t = warp_sum(a[q]);
    if (threadIdx.x == 0) out[q] = t;
  }
}

// ---------------------------------------------------------------- synth -----
// u = 1 inside the ellipsoid (rho <= 1), exp(-d^2/(2 sigma^2)) outside with
// d = r (1 - 1/rho); evaluated in fp64 and rounded to fp32 like the reference.
__global__ void synth_ellipsoids_kernel(float* __restrict__ out, int64_t n, int64_t res,
                                        int64_t ld, const double* __restrict__ prm,
                                        double sigma) {
  const int64_t cells = res * res * res;
  const int64_t i = blockIdx.y;
  const double cy = prm[6 * i], cx = prm[6 * i + 1], cz = prm[6 * i + 2];
  const double ay = prm[6 * i + 3], ax = prm[6 * i + 4], az = prm[6 * i + 5];
  const double two_s2 = __dmul_rn(__dmul_rn(2.0, sigma), sigma);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ld;
       c += (int64_t)gridDim.x * blockDim.x) {
    float val = 0.0f;
    if (c < cells) {
      const int64_t y = c / (res * res), rem = c - y * res * res;
      const int64_t x = rem / res, z = rem - x * res;
      const double dy = (double)y - cy, dx = (double)x - cx, dz = (double)z - cz;
      // explicit _rn intrinsics: no FMA contraction, same rounding as numpy
      const double qy = __ddiv_rn(dy, ay), qx = __ddiv_rn(dx, ax), qz = __ddiv_rn(dz, az);
      const double rho2 =
          __dadd_rn(__dadd_rn(__dmul_rn(qy, qy), __dmul_rn(qx, qx)), __dmul_rn(qz, qz));
      const double rho = __dsqrt_rn(rho2);
      if (rho > 1.0) {
        const double r2 =
            __dadd_rn(__dadd_rn(__dmul_rn(dy, dy), __dmul_rn(dx, dx)), __dmul_rn(dz, dz));
        const double d = __dmul_rn(__dsqrt_rn(r2), __dsub_rn(1.0, __ddiv_rn(1.0, rho)));
        val = (float)exp(__ddiv_rn(-__dmul_rn(d, d), two_s2));
      } else {
        val = 1.0f;
      }
    }
    out[i * ld + c] = val;
  }
}

__global__ void synth_disks_kernel(float* __restrict__ out, int64_t n, int64_t res, int64_t ld,
                                   const double* __restrict__ prm, double sigma2) {
  const int64_t cells = res * res;
  const int64_t i = blockIdx.y;
  const double cy = prm[3 * i], cx = prm[3 * i + 1], radius = prm[3 * i + 2];
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ld;
       c += (int64_t)gridDim.x * blockDim.x) {
    float val = 0.0f;
    if (c < cells) {
      const int64_t y = c / res, x = c - y * res;
      const double dy = (double)y - cy, dx = (double)x - cx;
      const double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(dy, dy), __dmul_rn(dx, dx)));
      const double e = __dsub_rn(dist, radius);
      val = dist <= radius ? 1.0f
                           : (float)exp(__ddiv_rn(-__dmul_rn(e, e), __dmul_rn(2.0, sigma2)));
    }
    out[i * ld + c] = val;
  }
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_binary_pack_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  // row blocks of 128 members, rounded up to pairs (K2 reads 256-member B panels)
  const int64_t nrb = 2 * ((n + 255) / 256);
  return (size_t)nrb * (size_t)((m + 127) / 128) * 16384;
}

extern "C" int pidb_binary_pack(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                                uint8_t* tiles, int64_t* nonbinary, void* stream) {
  PIDB_REQUIRE(u && (tiles || nonbinary) && n >= 1 && m >= 1 && ld >= m,
               "bad arguments to pidb_binary_pack");
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(tiles) & 1023) == 0, "tiles must be 1 KB aligned");
  PIDB_REQUIRE(dtype != PIDB_U8 || ((reinterpret_cast<uintptr_t>(u) & 15) == 0 && ld % 16 == 0),
               "byte members need a 16-byte aligned base and row pitch");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nkb = (m + 127) / 128;
  const int64_t jobs = (tiles ? (n + 255) / 256 * 256 : n) * ((nkb * 128 + 511) / 512);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((jobs + 7) / 8, 148 * 16));
  if (dtype == PIDB_F32)
    binary_pack_kernel<float><<<blocks, 256, 0, st>>>(
        static_cast<const float*>(u), n, m, ld, tiles, nkb,
        reinterpret_cast<unsigned long long*>(nonbinary));
  else if (dtype == PIDB_F64)
    binary_pack_kernel<double><<<blocks, 256, 0, st>>>(
        static_cast<const double*>(u), n, m, ld, tiles, nkb,
        reinterpret_cast<unsigned long long*>(nonbinary));
  else if (dtype == PIDB_U8)
    binary_pack_kernel<uint8_t><<<blocks, 256, 0, st>>>(
        static_cast<const uint8_t*>(u), n, m, ld, tiles, nkb,
        reinterpret_cast<unsigned long long*>(nonbinary));
  else
    PIDB_REQUIRE(false, "dtype must be PIDB_F32, PIDB_F64 or PIDB_U8");
  PIDB_LAUNCH_CHECK("binary_pack_kernel");
  return PIDB_OK;
}

extern "C" int pidb_pair_sums(const void* u, const void* v, int dtype, int64_t m, const double* w,
                              int op, double* out_host, void* ws, size_t ws_bytes,
                              void* stream) {
  PIDB_REQUIRE(u && v && out_host && m >= 1, "bad arguments to pidb_pair_sums");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  PIDB_REQUIRE(op >= PIDB_OP_INCLUSION && op <= PIDB_OP_MINMAX, "unknown pair op %d", op);
  const int nb = (int)std::min<int64_t>(4 * 148, (m + 255) / 256);
  PIDB_REQUIRE(ws && ws_bytes >= (size_t)(4 * nb + 4) * sizeof(double),
               "workspace too small for pidb_pair_sums (need %zu bytes)",
               (size_t)(4 * nb + 4) * sizeof(double));
  cudaStream_t st = (cudaStream_t)stream;
  double* part = static_cast<double*>(ws);
  if (dtype == PIDB_F32)
    pair_sums_kernel<float><<<nb, 256, 0, st>>>(static_cast<const float*>(u),
                                                static_cast<const float*>(v), m, w, op, part);
  else
    pair_sums_kernel<double><<<nb, 256, 0, st>>>(static_cast<const double*>(u),
                                                 static_cast<const double*>(v), m, w, op, part);
  PIDB_LAUNCH_CHECK("pair_sums_kernel");
  pair_finish_kernel<<<1, 32, 0, st>>>(part, nb, part + 4 * nb);
  PIDB_LAUNCH_CHECK("pair_finish_kernel");
  const int nout = op == PIDB_OP_MINMAX ? 4 : 2;
  PIDB_CUDA(cudaMemcpyAsync(out_host, part + 4 * nb, nout * sizeof(double), cudaMemcpyDeviceToHost, st));
  PIDB_CUDA(cudaStreamSynchronize(st));
  return PIDB_OK;
}

extern "C" int pidb_synth_ellipsoids(float* out, int64_t n, int64_t res, int64_t ld,
                                     const double* params, double sigma, void* stream) {
  PIDB_REQUIRE(out && params && n >= 1 && res >= 1 && ld >= res * res * res,
               "bad arguments to pidb_synth_ellipsoids");
  PIDB_REQUIRE(n <= 65535, "at most 65535 members per synth call");
  dim3 grid((unsigned)std::min<int64_t>((ld + 255) / 256, 4096), (unsigned)n);
  synth_ellipsoids_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out, n, res, ld, params, sigma);
  PIDB_LAUNCH_CHECK("synth_ellipsoids_kernel");
  return PIDB_OK;
}

extern "C" int pidb_synth_disks(float* out, int64_t n, int64_t res, int64_t ld,
                                const double* params, double sigma2, void* stream) {
  PIDB_REQUIRE(out && params && n >= 1 && res >= 1 && ld >= res * res,
               "bad arguments to pidb_synth_disks");
  PIDB_REQUIRE(n <= 65535, "at most 65535 members per synth call");
  dim3 grid((unsigned)std::min<int64_t>((ld + 255) / 256, 4096), (unsigned)n);
  synth_disks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out, n, res, ld, params, sigma2);
  PIDB_LAUNCH_CHECK("synth_disks_kernel");
  return PIDB_OK;
}

// ------------------------------------------------------------ mean mask -----
// mean(x) = (sum_i u_i(x)) / n, accumulated in fp64 in member order: the same
// arithmetic as mean_mask (/root/reference/pkg/src/fuzzdepth/grid.py:257-260),
// hence bit-identical.  Coalesced across cells for each member row.
namespace pidb {
namespace {
template <typename T>
__global__ void mean_mask_kernel(const T* __restrict__ u, int64_t n, int64_t m, int64_t ld,
                                 double* __restrict__ out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m;
       x += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, (double)u[i * ld + x]);
    out[x] = __ddiv_rn(acc, (double)n);
  }
}
}  // namespace
}  // namespace pidb

extern "C" int pidb_mean_mask(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                              double* out, void* stream) {
  PIDB_REQUIRE(u && out && n >= 1 && m >= 1 && ld >= m, "bad arguments to pidb_mean_mask");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 8));
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PIDB_F32)
    mean_mask_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(u), n, m, ld, out);
  else
    mean_mask_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(u), n, m, ld, out);
  PIDB_LAUNCH_CHECK("mean_mask_kernel");
  return PIDB_OK;
}

// ------------------------------------------------------------ staging -------
// Pitched host<->device row copies (one cudaMemcpy2DAsync per call) so that
// (n, m) host matrices land in the padded (n, ld) device layout without a
// device-side temporary.
extern "C" int pidb_copy_rows(void* dst, int64_t dst_pitch_bytes, const void* src,
                              int64_t src_pitch_bytes, int64_t row_bytes, int64_t rows,
                              void* stream) {
  PIDB_REQUIRE(dst && src && rows >= 0 && row_bytes >= 0 && dst_pitch_bytes >= row_bytes &&
                   src_pitch_bytes >= row_bytes,
               "bad arguments to pidb_copy_rows");
  if (rows == 0 || row_bytes == 0) return PIDB_OK;
  PIDB_CUDA(cudaMemcpy2DAsync(dst, (size_t)dst_pitch_bytes, src, (size_t)src_pitch_bytes,
                              (size_t)row_bytes, (size_t)rows, cudaMemcpyDefault,
                              (cudaStream_t)stream));
  return PIDB_OK;
}

// ------------------------------------------------------------ validation ----
// ProbMask value policy (/root/reference/pkg/src/fuzzdepth/grid.py:105-116) for
// raw tensors, one pass: stats[0] = #non-finite, stats[1] = min, stats[2] = max
// (as ordered int64 keys of the doubles).  clamp != 0 additionally clips to [0,1].
namespace pidb {
namespace {
__device__ __forceinline__ long long dkey(double d) {
  long long b = __double_as_longlong(d);
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
}
// Warp-combine one thread's (non-finite count, finite min/max) and publish
// with one set of atomics per warp.
__device__ __forceinline__ void validate_reduce(unsigned long long bad, double lo, double hi,
                                                bool any, unsigned long long* nonfinite,
                                                long long* kmin, long long* kmax) {
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, (int)any, o);
    if (a2) {
      lo = any ? fmin(lo, l2) : l2;
      hi = any ? fmax(hi, h2) : h2;
      any = true;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(nonfinite, bad);
    if (any) {
      atomicMin(kmin, dkey(lo));
      atomicMax(kmax, dkey(hi));
    }
  }
}

template <typename T>
__global__ void validate_kernel(T* __restrict__ u, int64_t n, int64_t m, int64_t ld, int clamp,
                                unsigned long long* __restrict__ nonfinite,
                                long long* __restrict__ kmin, long long* __restrict__ kmax) {
  unsigned long long bad = 0;
  double lo = 0.0, hi = 0.0;
  bool any = false;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m;
       x += (int64_t)gridDim.x * blockDim.x) {
    T v = u[i * ld + x];
    const double d = (double)v;
    if (!isfinite(d)) { ++bad; continue; }
    if (!any) { lo = hi = d; any = true; }
    lo = fmin(lo, d);
    hi = fmax(hi, d);
    if (clamp && (d < 0.0 || d > 1.0)) u[i * ld + x] = d < 0.0 ? T(0) : T(1);
  }
  validate_reduce(bad, lo, hi, any, nonfinite, kmin, kmax);
}

// fp32 members with 16-byte aligned rows: 128-bit loads, min/max in float
// (exact: the float extremes convert to the same doubles).
__global__ void validate_f32x4_kernel(float* __restrict__ u, int64_t n, int64_t m, int64_t ld,
                                      int clamp, unsigned long long* __restrict__ nonfinite,
                                      long long* __restrict__ kmin, long long* __restrict__ kmax) {
  unsigned long long bad = 0;
  float lo = 0.f, hi = 0.f;
  bool any = false;
  const int64_t m4 = m >> 2;
  auto visit = [&](float& v, bool& dirty) {
    if (!isfinite(v)) { ++bad; return; }
    if (!any) { lo = hi = v; any = true; }
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
    if (clamp && (v < 0.f || v > 1.f)) { v = v < 0.f ? 0.f : 1.f; dirty = true; }
  };
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    float* row = u + i * ld;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m4;
         x += (int64_t)gridDim.x * blockDim.x) {
      float4 v = reinterpret_cast<const float4*>(row)[x];
      bool dirty = false;
      visit(v.x, dirty); visit(v.y, dirty); visit(v.z, dirty); visit(v.w, dirty);
      if (dirty) reinterpret_cast<float4*>(row)[x] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x < (m & 3)) {
      float v = row[(m4 << 2) + threadIdx.x];
      bool dirty = false;
      visit(v, dirty);
      if (dirty) row[(m4 << 2) + threadIdx.x] = v;
    }
  }
  validate_reduce(bad, (double)lo, (double)hi, any, nonfinite, kmin, kmax);
}
__global__ void validate_init_kernel(unsigned long long* nf, long long* kmin, long long* kmax) {
  *nf = 0;
  *kmin = 0x7FFFFFFFFFFFFFFFLL;
  *kmax = (long long)0x8000000000000000ULL;
}

// dst[j] = sum_k src[k * len + j], k ascending (fixed order).
__global__ void sum_rows_kernel(const double* __restrict__ src, int64_t rows, int64_t len,
                                double* __restrict__ dst) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < len;
       j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < rows; ++k) s += src[k * len + j];
    dst[j] = s;
  }
}
}  // namespace
}  // namespace pidb

extern "C" int pidb_sum_rows(const double* src, int64_t rows, int64_t len, double* dst,
                             void* stream) {
  PIDB_REQUIRE(src && dst && rows >= 1 && len >= 1, "bad arguments to pidb_sum_rows");
  const int blocks = (int)std::min<int64_t>((len + 255) / 256, 148 * 4);
  sum_rows_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(src, rows, len, dst);
  PIDB_LAUNCH_CHECK("sum_rows_kernel");
  return PIDB_OK;
}

extern "C" int pidb_validate(void* u, int dtype, int64_t n, int64_t m, int64_t ld, int clamp,
                             void* stats, void* stream) {
  PIDB_REQUIRE(u && stats && n >= 1 && m >= 1 && ld >= m, "bad arguments to pidb_validate");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* nf = static_cast<unsigned long long*>(stats);
  long long* kmin = reinterpret_cast<long long*>(nf + 1);
  long long* kmax = kmin + 1;
  validate_init_kernel<<<1, 1, 0, st>>>(nf, kmin, kmax);  // capturable (no host memcpy)
  PIDB_LAUNCH_CHECK("validate_init_kernel");
  const dim3 blocks((unsigned)std::min<int64_t>((m + 255) / 256, 64),
                    (unsigned)std::min<int64_t>(n, 1024));
  if (dtype == PIDB_F32 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0) {
    const dim3 b4((unsigned)std::min<int64_t>((m / 4 + 255) / 256, 64),
                  (unsigned)std::min<int64_t>(n, 1024));
    validate_f32x4_kernel<<<b4.x ? b4 : dim3(1, b4.y), 256, 0, st>>>(static_cast<float*>(u), n,
                                                                     m, ld, clamp, nf, kmin, kmax);
  } else if (dtype == PIDB_F32)
    validate_kernel<float><<<blocks, 256, 0, st>>>(static_cast<float*>(u), n, m, ld, clamp, nf,
                                                   kmin, kmax);
  else
    validate_kernel<double><<<blocks, 256, 0, st>>>(static_cast<double*>(u), n, m, ld, clamp, nf,
                                                    kmin, kmax);
  PIDB_LAUNCH_CHECK("validate_kernel");
  return PIDB_OK;
}
