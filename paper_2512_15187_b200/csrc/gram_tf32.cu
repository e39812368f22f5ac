// K1: weighted fuzzy Gram G = U diag(w) U^T on the tensor cores, 3xTF32.
//
// Replaces the fp64 BLAS tile products of the exact PID:
//   depth_pid / _pairwise_sums  /root/reference/pkg/src/fuzzdepth/depth.py:122-161, 213-228
//   gram_block                  /root/reference/pkg/src/fuzzdepth/reduction.py:75-97
//
// Precision: every operand a is split a = hi + lo where hi is the tensor
// core's own tf32 truncation of the fp32 value (no smem write) and
// lo = rna_tf32(a - hi) (written by converter warps); the three products
// hi*hi + hi*lo + lo*hi (tcgen05.mma.kind::tf32, M=N=128, K=8) accumulate in
// fp32 TMEM for at most kFlushStages*32 = 512 cells, after which the epilogue
// warps fold the block into an fp64 shadow that also lives in TMEM
// (double-buffered fp32 accumulators, so the MMAs never wait for the fold).
// Weighted grids scale the A operand by w in fp32 and write its rna hi/lo.
//
// Work: 128x128 output tiles of the upper block triangle x split-K cell
// ranges; fp64 split partials are reduced (fixed order) and mirrored by a
// second kernel.  Warps (320 threads): 0 TMA producer, 1 MMA issuer,
// 2-5 converters, 6-9 epilogue (one TMEM lane quadrant each).
#include "tcgen05.cuh"

namespace pidb {
namespace {

constexpr int kB = 128;            // tile edge (members)
constexpr int kBK = 32;            // fp32 cells per stage (one 128-byte line)
constexpr int kStages = 3;
constexpr int kFlushStages = 16;   // 512 cells per fp32 accumulation block
constexpr int kTileBytes = kB * kBK * 4;             // 16 KB
constexpr int kStageBytes = 4 * kTileBytes;          // A, B, A_lo, B_lo
constexpr int kThreads = 320;
constexpr int kConvThreads = 128;
constexpr uint32_t kIdesc = tc::idesc(tc::kCF32, tc::kTF32, kB, kB);
// TMEM columns: [0,128) acc0, [128,256) acc1, [256,512) fp64 shadow (lo,hi pairs)
constexpr uint32_t kTmemCols = 512;

struct GramTf32Params {
  int n, nb, ntiles, splits, kblocks, kb_per;
  int64_t m;
  const double* w;   // nullable
  double* part;      // [units][kB][kB]
};

__device__ __forceinline__ void tile_of(int t, int& ib, int& jb) {
  jb = 0;
  while (t > jb) {  // tiles of column block jb: ib = 0..jb
    t -= jb + 1;
    ++jb;
  }
  ib = t;
}

__global__ void __launch_bounds__(kThreads, 1)
    gram_tf32_kernel(const __grid_constant__ CUtensorMap tmap, const GramTf32Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStageBytes);
  uint64_t* conv = full + kStages;
  uint64_t* empty = conv + kStages;
  uint64_t* acc_full = empty + kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  double* wst = reinterpret_cast<double*>(tmem_slot + 2);  // [kStages][kBK] weights

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x;
  const int t = unit / p.splits, split = unit - t * p.splits;
  int ib, jb;
  tile_of(t, ib, jb);
  const bool diag = ib == jb;
  const bool weighted = p.w != nullptr;
  const bool share_b = diag && !weighted;  // B operand == A operand
  const int kb0 = split * p.kb_per;
  const int kb1 = min(p.kblocks, kb0 + p.kb_per);
  const int nk = max(0, kb1 - kb0);
  const int nflush = (nk + kFlushStages - 1) / kFlushStages;

  if (threadIdx.x == 0) {
    prefetch_tma_desc(&tmap);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kConvThreads);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_mbar_init();
  }
  if (warp == 6) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (tc::elect_one()) {
      const uint64_t pol = policy_evict_last();
      const uint32_t bytes = share_b ? kTileBytes : 2 * kTileBytes;
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0; k < nk; ++k) {
        mbar_wait(&empty[s], ph ^ 1u);
        unsigned char* st = ring + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], bytes);
        const int x = (kb0 + k) * kBK;
        tma_load_2d(st, &tmap, x, ib * kB, &full[s], pol);
        if (!share_b) tma_load_2d(st + kTileBytes, &tmap, x, jb * kB, &full[s], pol);
        if (++s == kStages) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (tc::elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      int k = 0;
      for (int f = 0; f < nflush; ++f) {
        const int buf = f & 1;
        mbar_wait(&acc_empty[buf], ((f >> 1) & 1) ^ 1u);
        tc::fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * kB);
        const int kend = min(nk, k + kFlushStages);
        bool first = true;
        for (; k < kend; ++k) {
          mbar_wait(&conv[s], ph);
          tc::fence_after();
          const uint32_t a = smem_u32(ring + s * kStageBytes);
          const uint64_t a_hi = tc::desc_kmajor_sw128(a);
          const uint64_t b_hi = share_b ? a_hi : tc::desc_kmajor_sw128(a + kTileBytes);
          const uint64_t a_lo = tc::desc_kmajor_sw128(a + 2 * kTileBytes);
          const uint64_t b_lo = share_b ? a_lo : tc::desc_kmajor_sw128(a + 3 * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {  // K = 8 tf32 = 32 bytes per MMA
            const uint64_t o = 2 * kk;
            tc::mma_tf32(d, a_lo + o, b_hi + o, kIdesc, first ? 0u : 1u);
            tc::mma_tf32(d, a_hi + o, b_lo + o, kIdesc, 1u);
            tc::mma_tf32(d, a_hi + o, b_hi + o, kIdesc, 1u);
            first = false;
          }
          tc::commit(&empty[s]);
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
        tc::commit(&acc_full[buf]);
      }
    }
  } else if (warp < 6) {
    // ----------------------------------------------------------- converters
    const int ct = threadIdx.x - 64;  // 0..127
    int s = 0;
    uint32_t ph = 0;
    for (int k = 0; k < nk; ++k) {
      mbar_wait(&full[s], ph);
      unsigned char* st = ring + s * kStageBytes;
      const int x0 = (kb0 + k) * kBK;
      double* ws = wst + s * kBK;
      if (weighted) {
        if (ct < kBK) ws[ct] = (x0 + ct) < p.m ? __ldg(p.w + x0 + ct) : 0.0;
        asm volatile("bar.sync 1, %0;" ::"n"(kConvThreads) : "memory");
      }
      // A tile: 1024 16-byte chunks; chunk c = line r = c/8, physical slot c%8
#pragma unroll 4
      for (int c = ct; c < kB * 8; c += kConvThreads) {
        float4* src = reinterpret_cast<float4*>(st + c * 16);
        float4* lo = reinterpret_cast<float4*>(st + 2 * kTileBytes + c * 16);
        float4 v = *src;
        if (weighted) {
          const int r = c >> 3;
          const int lc = (c & 7) ^ (r & 7);  // logical chunk -> cells 4*lc..4*lc+3
          const double* wc = ws + 4 * lc;
          v.x = (float)((double)v.x * wc[0]);
          v.y = (float)((double)v.y * wc[1]);
          v.z = (float)((double)v.z * wc[2]);
          v.w = (float)((double)v.w * wc[3]);
          float4 h = make_float4(tc::tf32_rna(v.x), tc::tf32_rna(v.y), tc::tf32_rna(v.z),
                                 tc::tf32_rna(v.w));
          *src = h;
          *lo = make_float4(tc::tf32_rna(v.x - h.x), tc::tf32_rna(v.y - h.y),
                            tc::tf32_rna(v.z - h.z), tc::tf32_rna(v.w - h.w));
        } else {
          *lo = make_float4(tc::tf32_rna(v.x - tc::tf32_trunc(v.x)),
                            tc::tf32_rna(v.y - tc::tf32_trunc(v.y)),
                            tc::tf32_rna(v.z - tc::tf32_trunc(v.z)),
                            tc::tf32_rna(v.w - tc::tf32_trunc(v.w)));
        }
      }
      if (!share_b) {
#pragma unroll 4
        for (int c = ct; c < kB * 8; c += kConvThreads) {
          const float4 v = *reinterpret_cast<const float4*>(st + kTileBytes + c * 16);
          *reinterpret_cast<float4*>(st + 3 * kTileBytes + c * 16) =
              make_float4(tc::tf32_rna(v.x - tc::tf32_trunc(v.x)),
                          tc::tf32_rna(v.y - tc::tf32_trunc(v.y)),
                          tc::tf32_rna(v.z - tc::tf32_trunc(v.z)),
                          tc::tf32_rna(v.w - tc::tf32_trunc(v.w)));
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05.mma
      mbar_arrive(&conv[s]);
      if (++s == kStages) { s = 0; ph ^= 1u; }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    // warp w owns TMEM lanes [32*(w%4), +32): rows of the tile
    const int quad = warp & 3;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    {  // zero the fp64 shadow
      uint32_t z[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) z[e] = 0u;
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) tc::tmem_st32(lane_base + 256 + c, z);
      tc::tmem_st_wait();
    }
    for (int f = 0; f < nflush; ++f) {
      const int buf = f & 1;
      mbar_wait(&acc_full[buf], (f >> 1) & 1);
      tc::fence_after();
#pragma unroll 1
      for (int c = 0; c < kB; c += 16) {
        uint32_t a32[16], sh[32];
        tc::tmem_ld16(lane_base + (uint32_t)(buf * kB + c), a32);  // fp32 cols c..c+15
        tc::tmem_ld32(lane_base + 256 + (uint32_t)(2 * c), sh);     // 16 fp64 as (lo, hi)
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          double d = __hiloint2double((int)sh[2 * e + 1], (int)sh[2 * e]);
          d += (double)__uint_as_float(a32[e]);
          sh[2 * e] = (uint32_t)__double2loint(d);
          sh[2 * e + 1] = (uint32_t)__double2hiint(d);
        }
        tc::tmem_st32(lane_base + 256 + (uint32_t)(2 * c), sh);
      }
      tc::tmem_st_wait();
      tc::fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
    // shadow -> global fp64 split partial (row = quad*32 + lane)
    double* dst = p.part + ((size_t)unit * kB + quad * 32 + lane) * kB;
#pragma unroll 1
    for (int c = 0; c < kB; c += 16) {
      uint32_t sh[32];
      if (nflush > 0) {
        tc::tmem_ld32(lane_base + 256 + (uint32_t)(2 * c), sh);
        tc::tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) sh[e] = 0u;
      }
#pragma unroll
      for (int e = 0; e < 16; e += 2)
        *reinterpret_cast<double2*>(dst + c + e) =
            make_double2(__hiloint2double((int)sh[2 * e + 1], (int)sh[2 * e]),
                         __hiloint2double((int)sh[2 * e + 3], (int)sh[2 * e + 2]));
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 6) tc::tmem_dealloc(tmem, kTmemCols);
}

// G[i][j] = G[j][i] = sum over splits (fixed order) of the tile holding (min, max).
__global__ void gram_tf32_reduce_kernel(const double* __restrict__ part, int n, int splits,
                                        double* __restrict__ out) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / n), b = (int)(e - (int64_t)a * n);
    const int i = min(a, b), j = max(a, b);
    const int ib = i / kB, jb = j / kB;
    const int t = jb * (jb + 1) / 2 + ib;
    const double* src = part + ((size_t)t * splits * kB + (i - ib * kB)) * kB + (j - jb * kB);
    double acc = 0.0;
    for (int s = 0; s < splits; ++s) acc += src[(size_t)s * kB * kB];
    out[e] = acc;
  }
}

struct Plan {
  int nb, ntiles, splits, kblocks, kb_per, units;
  size_t smem, ws;
};

Plan plan(int64_t n, int64_t m) {
  Plan g{};
  g.nb = (int)((n + kB - 1) / kB);
  g.ntiles = g.nb * (g.nb + 1) / 2;
  g.kblocks = (int)((m + kBK - 1) / kBK);
  const int sms = sm_count();
  g.splits = std::max(1, std::min(g.kblocks, sms / g.ntiles));
  g.kb_per = (g.kblocks + g.splits - 1) / g.splits;
  g.splits = (g.kblocks + g.kb_per - 1) / g.kb_per;
  g.units = g.ntiles * g.splits;
  g.smem = 1024 + (size_t)kStages * kStageBytes + 256 + kStages * kBK * sizeof(double);
  g.ws = 256 + (size_t)g.units * kB * kB * sizeof(double);
  return g;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_gram_tf32x3_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  return plan(n, m).ws;
}

extern "C" int pidb_gram_tf32x3(const float* u, int64_t n, int64_t m, int64_t ld, const double* w,
                                double* gram, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u && gram && n >= 1 && m >= 1, "bad arguments to pidb_gram_tf32x3");
  PIDB_REQUIRE(ld >= m && (ld * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0,
               "member rows must be 16-byte aligned with ld >= m");
  PIDB_REQUIRE(n <= (1 << 16), "too many members for the dense Gram");
  const Plan g = plan(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  CUtensorMap tm;
  int rc = encode_tma_2d(&tm, u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (uint64_t)m, (uint64_t)n,
                         (uint64_t)ld * 4, kBK, kB, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != PIDB_OK) return rc;
  GramTf32Params p{};
  p.n = (int)n; p.nb = g.nb; p.ntiles = g.ntiles; p.splits = g.splits; p.kblocks = g.kblocks;
  p.kb_per = g.kb_per; p.m = m; p.w = w;
  p.part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  cudaStream_t st = (cudaStream_t)stream;
  PIDB_CUDA(cudaFuncSetAttribute(gram_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)g.smem));
  gram_tf32_kernel<<<g.units, kThreads, g.smem, st>>>(tm, p);
  PIDB_LAUNCH_CHECK("gram_tf32_kernel");
  const int64_t total = n * n;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  gram_tf32_reduce_kernel<<<blocks, 256, 0, st>>>(p.part, (int)n, g.splits, gram);
  PIDB_LAUNCH_CHECK("gram_tf32_reduce_kernel");
  return PIDB_OK;
}
