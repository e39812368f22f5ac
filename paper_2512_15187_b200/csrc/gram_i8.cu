// K2: exact integer intersection Gram on the 5th-gen tensor cores.
//
// Replaces the eID pairwise product of the reference:
//   _pairwise_sums(complement=True)  /root/reference/pkg/src/fuzzdepth/depth.py:122-161
//   gram_block(..., complement_cols) /root/reference/pkg/src/fuzzdepth/reduction.py:75-97
// For 0/1 members |A_i \ A_j| = |A_i| - |A_i ∩ A_j|, so one integer Gram
// I = B B^T of the packed uint8 members gives every pair exactly.
//
// Kernel: C = A B^T tiles of 128 x 256 with A = members [128 ib, +128),
// B = members [256 jb, +256) (upper tile triangle only, the Gram is
// symmetric), K = cells split across CTAs.  Operands come from one of two
// layouts:
//   * the K7 tiles of fp32/fp64 members: 16 KB tiles (128 members x 128
//     cells, already in the 128-byte-swizzled K-major order), a stage is
//     three plain 1D bulk copies;
//   * a byte ensemble (0/1 members stored as uint8, row pitch ld): the same
//     three 128 x 128-byte boxes by 2D TMA with SWIZZLE_128B straight from
//     the member matrix -- no pack pass; rows >= n and cells >= m are the
//     TMA's zero fill.
// Warp roles (192 threads):
//   warp 0 : bulk-copy producer (4-stage ring)
//   warp 1 : single-thread tcgen05.mma.kind::i8 issuer (M=128, N=256, K=32),
//            int32 accumulators in TMEM (exact: < 2^31 cells per pair)
//   warps 2-5: epilogue, tcgen05.ld 32x32b -> int32 split partials
// A second kernel sums the split partials in int64 and mirrors the triangle.
#include "tcgen05.cuh"

namespace pidb {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 128;  // bytes of K per stage
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK, kBBytes = kBN * kBK;
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kGramThreads = 192;
constexpr uint32_t kIdescI8 = tc::idesc(tc::kCS32, tc::kU8, kBM, kBN);

struct GramI8Params {
  int n, nib, njb, ntiles, splits, kblocks, kb_per;
  int32_t* part;  // [units][kBM][kBN]
};

__device__ __forceinline__ void tile_of(int t, int nib, int& ib, int& jb) {
  jb = 0;
  for (;;) {
    const int c = min(nib, 2 * jb + 2);
    if (t < c) break;
    t -= c;
    ++jb;
  }
  ib = t;
}

template <bool kBytes>
__global__ void __launch_bounds__(kGramThreads, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ tiles,
                   const GramI8Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x;
  const int t = unit / p.splits, split = unit - t * p.splits;
  int ib, jb;
  tile_of(t, p.nib, ib, jb);
  const int kb0 = split * p.kb_per;
  const int kb1 = min(p.kblocks, kb0 + p.kb_per);
  const int nk = max(0, kb1 - kb0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, kBN);
  if (kBytes && warp == 0 && lane == 0) prefetch_tma_desc(&tmap);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      const uint64_t pol = policy_evict_last();  // members are re-read by other tiles
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0; k < nk; ++k) {
        mbar_wait(&empty[s], ph ^ 1u);
        unsigned char* a = ring + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], kStageBytes);
        const int64_t kb = kb0 + k;  // three 16 KB tiles: A, then B's two halves
        PIDB_DCHECK(kb < p.kblocks && ib < 2 * ((p.n + 255) / 256) &&
                        2 * jb + 1 < 2 * ((p.n + 255) / 256),
                    "K2 operand tile bounds");
        if constexpr (kBytes) {
          const int32_t x = (int32_t)(kb * kBK);
          tma_load_2d(a, &tmap, x, ib * kBM, &full[s], pol);
          tma_load_2d(a + kABytes, &tmap, x, 2 * jb * kBM, &full[s], pol);
          tma_load_2d(a + 2 * kABytes, &tmap, x, (2 * jb + 1) * kBM, &full[s], pol);
        } else {
          bulk_load(a, tiles + ((int64_t)ib * p.kblocks + kb) * kABytes, kABytes, &full[s], pol);
          bulk_load(a + kABytes, tiles + ((int64_t)(2 * jb) * p.kblocks + kb) * kABytes, kABytes,
                    &full[s], pol);
          bulk_load(a + 2 * kABytes, tiles + ((int64_t)(2 * jb + 1) * p.kblocks + kb) * kABytes,
                    kABytes, &full[s], pol);
        }
        if (++s == kStages) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0; k < nk; ++k) {
        mbar_wait(&full[s], ph);
        tc::fence_after();
        const uint32_t a = smem_u32(ring + s * kStageBytes);
        const uint64_t da = tc::desc_kmajor_sw128(a);
        const uint64_t db = tc::desc_kmajor_sw128(a + kABytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 32; ++kk)  // K = 32 bytes per MMA
          tc::mma_i8(tmem, da + 2 * kk, db + 2 * kk, kIdescI8, (k | kk) != 0);
        tc::commit(&empty[s]);  // frees the stage once these MMAs are done
        if (++s == kStages) { s = 0; ph ^= 1u; }
      }
      tc::commit(tmem_full);
    }
  } else {
    // epilogue: warp w owns TMEM lanes [32*(w%4), +32) (hardware lane quadrant)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc::fence_after();
    PIDB_DCHECK(unit < p.ntiles * p.splits, "K2 partial bounds");
    int32_t* dst = p.part + ((size_t)unit * kBM + row) * kBN;
#pragma unroll 1
    for (int c = 0; c < kBN; c += 32) {
      uint32_t v[32];
      if (nk > 0) {
        tc::tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c, v);
        tc::tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0;
      }
#pragma unroll
      for (int e = 0; e < 32; e += 4)
        *reinterpret_cast<int4*>(dst + c + e) = make_int4(v[e], v[e + 1], v[e + 2], v[e + 3]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tmem, kBN);
}

// I[i][j] = I[j][i] = sum over splits of the tile holding (i, j), i <= j.
// One thread per (tile, tile row, 4 consecutive columns): 16-byte partial
// loads along the row (coalesced), int64 sums (exact, any order), the upper
// entries written along the row and mirrored into the lower triangle.
__global__ void __launch_bounds__(256)
    gram_i8_reduce_kernel(const int32_t* __restrict__ part, int n, int nib, int splits,
                          int64_t* __restrict__ out) {
  const int t = blockIdx.x >> 5;                      // tile
  const int r = ((blockIdx.x & 31) << 2) + (threadIdx.x >> 6);  // tile row 0..127
  const int c4 = (threadIdx.x & 63) << 2;             // first of 4 tile columns
  int ib, jb;
  tile_of(t, nib, ib, jb);
  const int i = ib * kBM + r, j0 = jb * kBN + c4;
  if (i >= n || j0 >= n || j0 + 3 < i) return;
  const int4* src = reinterpret_cast<const int4*>(part + ((size_t)t * splits * kBM + r) * kBN + c4);
  long long acc[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int s = 0; s < splits; ++s) {
    const int4 v = __ldg(src + (size_t)s * kBM * kBN / 4);
    acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    if (j >= n || j < i) continue;
    out[(int64_t)i * n + j] = acc[k];
    if (j != i) out[(int64_t)j * n + i] = acc[k];
  }
}

struct GramPlan {
  int nib, njb, ntiles, splits, kblocks, kb_per, units;
  size_t smem, ws;
};

GramPlan plan_i8(int64_t n, int64_t m) {
  GramPlan g{};
  g.nib = (int)((n + kBM - 1) / kBM);
  g.njb = (int)((n + kBN - 1) / kBN);
  g.ntiles = 0;
  for (int jb = 0; jb < g.njb; ++jb) g.ntiles += std::min(g.nib, 2 * jb + 2);
  g.kblocks = (int)((m + kBK - 1) / kBK);
  const int sms = sm_count();
  // K splits minimising the makespan: waves x (K blocks per unit + a fixed
  // per-unit cost of ~10 K blocks: TMEM alloc, pipeline fill, the 128 KB
  // partial).  One wave when it divides well (n = 500: 6 tiles x 24 splits);
  // n = 1500: 42 tiles x 7 splits in two waves (586 K blocks per SM) over
  // 3 splits in one wave (683, 22 SMs idle) -- measured 0.258 vs 0.264 ms:
  // the lock-step waves keep K2 tensor/L2-paced, not occupancy-paced.
  {
    long best = -1;
    const int smax = std::max(1, std::min(g.kblocks, 8 * sms / g.ntiles + 1));
    for (int s = 1; s <= smax; ++s) {
      const int per = (g.kblocks + s - 1) / s;
      const int sp = (g.kblocks + per - 1) / per;
      const long waves = ((long)g.ntiles * sp + sms - 1) / sms;
      const long cost = waves * (per + 10);
      if (best < 0 || cost < best) { best = cost; g.splits = sp; g.kb_per = per; }
    }
  }
  g.units = g.ntiles * g.splits;
  g.smem = 1024 + (size_t)kStages * kStageBytes + 256;
  g.ws = 256 + (size_t)g.units * kBM * kBN * sizeof(int32_t);
  return g;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_gram_i8_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  return plan_i8(n, m).ws;
}

static int launch_i8(const CUtensorMap& tmap, const uint8_t* tiles, bool bytes, int64_t n,
                     int64_t m, int64_t* gram, void* ws, size_t ws_bytes, cudaStream_t st) {
  const GramPlan g = plan_i8(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  GramI8Params p{};
  p.n = (int)n; p.nib = g.nib; p.njb = g.njb; p.ntiles = g.ntiles; p.splits = g.splits;
  p.kblocks = g.kblocks; p.kb_per = g.kb_per;
  p.part = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 256);
  auto kern = bytes ? gram_i8_kernel<true> : gram_i8_kernel<false>;
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
  kern<<<g.units, kGramThreads, g.smem, st>>>(tmap, tiles, p);
  PIDB_LAUNCH_CHECK("gram_i8_kernel");
  gram_i8_reduce_kernel<<<g.ntiles * 32, 256, 0, st>>>(p.part, (int)n, g.nib, g.splits, gram);
  PIDB_LAUNCH_CHECK("gram_i8_reduce_kernel");
  return PIDB_OK;
}

extern "C" int pidb_gram_i8(const uint8_t* tiles, int64_t n, int64_t m, int64_t* gram, void* ws,
                            size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(tiles && gram && n >= 1 && m >= 1, "bad arguments to pidb_gram_i8");
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(tiles) & 1023) == 0, "tiles must be 1 KB aligned");
  PIDB_REQUIRE(m < ((int64_t)1 << 31), "int32 tensor-core accumulators need m < 2^31 cells");
  PIDB_REQUIRE(n <= (1 << 20), "too many members for the integer Gram");
  CUtensorMap unused{};
  return launch_i8(unused, tiles, false, n, m, gram, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int pidb_gram_i8_bytes(const uint8_t* u, int64_t n, int64_t m, int64_t ld,
                                  int64_t* gram, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u && gram && n >= 1 && m >= 1 && ld >= m, "bad arguments to pidb_gram_i8_bytes");
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(u) & 15) == 0 && ld % 16 == 0,
               "byte members need a 16-byte aligned base and row pitch");
  PIDB_REQUIRE(m < ((int64_t)1 << 31), "int32 tensor-core accumulators need m < 2^31 cells");
  PIDB_REQUIRE(n <= (1 << 20), "too many members for the integer Gram");
  CUtensorMap tmap;
  const int rc = encode_tma_2d(&tmap, u, CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)m, (uint64_t)n,
                               (uint64_t)ld, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != PIDB_OK) return rc;
  return launch_i8(tmap, nullptr, true, n, m, gram, ws, ws_bytes, (cudaStream_t)stream);
}
