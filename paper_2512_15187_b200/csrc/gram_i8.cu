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
#include <cstdlib>

#include "tcgen05.cuh"

namespace pidb {
namespace {

// H = 128-member halves of the B panel: H = 2 -> 128 x 256 output tiles,
// H = 1 -> 128 x 128 (more, smaller tiles for small n; plan_i8 picks)
constexpr int kBM = 128, kBK = 128;  // kBK: bytes of K per stage
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK;
template <int H> constexpr int kBNh = 128 * H;
template <int H> constexpr int kStageBytesH = kABytes * (1 + H);
constexpr int kGramThreads = 192;
template <int H>
constexpr uint32_t kIdescH = tc::idesc(tc::kCS32, tc::kU8, kBM, 128 * H);

struct GramI8Params {
  int n, nib, njb, ntiles, splits, kblocks, kb_per;
  int32_t* part;  // [units][kBM][BN]
};

template <int H>
__device__ __forceinline__ void tile_of(int t, int nib, int& ib, int& jb) {
  jb = 0;
  for (;;) {
    const int c = min(nib, H * (jb + 1));
    if (t < c) break;
    t -= c;
    ++jb;
  }
  ib = t;
}

template <bool kBytes, int H>
__global__ void __launch_bounds__(kGramThreads, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ tiles,
                   const GramI8Params p) {
  constexpr int kBN = kBNh<H>, kStageBytes = kStageBytesH<H>;
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
  tile_of<H>(t, p.nib, ib, jb);
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
        const int64_t kb = kb0 + k;  // 16 KB tiles: A, then the H halves of B
        PIDB_DCHECK(kb < p.kblocks && ib < 2 * ((p.n + 255) / 256) &&
                        H * jb + H - 1 < 2 * ((p.n + 255) / 256),
                    "K2 operand tile bounds");
        if constexpr (kBytes) {
          const int32_t x = (int32_t)(kb * kBK);
          tma_load_2d(a, &tmap, x, ib * kBM, &full[s], pol);
#pragma unroll
          for (int h = 0; h < H; ++h)
            tma_load_2d(a + (1 + h) * kABytes, &tmap, x, (H * jb + h) * kBM, &full[s], pol);
        } else {
          bulk_load(a, tiles + ((int64_t)ib * p.kblocks + kb) * kABytes, kABytes, &full[s], pol);
#pragma unroll
          for (int h = 0; h < H; ++h)
            bulk_load(a + (1 + h) * kABytes,
                      tiles + ((int64_t)(H * jb + h) * p.kblocks + kb) * kABytes, kABytes,
                      &full[s], pol);
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
          tc::mma_i8(tmem, da + 2 * kk, db + 2 * kk, kIdescH<H>, (k | kk) != 0);
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
template <int H>
__global__ void __launch_bounds__(256)
    gram_i8_reduce_kernel(const int32_t* __restrict__ part, int n, int nib, int splits,
                          int64_t* __restrict__ out) {
  constexpr int kBN = kBNh<H>;
  constexpr int TPR = kBN / 4, RPB = 256 / TPR, BPT = kBM / RPB;  // threads/row, rows/block
  const int t = blockIdx.x / BPT;                                    // tile
  const int r = (blockIdx.x % BPT) * RPB + threadIdx.x / TPR;        // tile row 0..127
  const int c4 = (threadIdx.x % TPR) * 4;                            // first of 4 tile columns
  int ib, jb;
  tile_of<H>(t, nib, ib, jb);
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
  int h, nib, njb, ntiles, splits, kblocks, kb_per, units;
  size_t smem, ws;
};

// Tile shape (H) and K splits minimising the makespan, in cycles per SM:
// waves x (K blocks per unit x ~256 (1 + H) cycles -- a K block is operand-
// delivery paced, (1 + H) 16 KB tiles into SMEM, not MMA paced (256 H) --
// + ~5000 cycles of per-unit cost: TMEM alloc, pipeline fill, the int32
// partial tile).  Measured (byte ensembles, 512^2 cells): 128 x 128 tiles
// win only for n <= 256 (n = 250: 0.049 vs 0.057 ms); n = 500 / 1000 / 1500
// / 4000: 128 x 256 tiles 0.066 / 0.134 / 0.258 / 1.457 ms vs 0.074 / 0.174
// / 0.590 / 2.510 ms (PIDB_K2_H forces a shape).
GramPlan plan_i8(int64_t n, int64_t m) {
  GramPlan best{};
  long best_cost = -1;
  const int sms = sm_count();
  const int kblocks = (int)((m + kBK - 1) / kBK);
  for (int h = 1; h <= 2; ++h) {
    GramPlan g{};
    g.h = h;
    g.nib = (int)((n + kBM - 1) / kBM);
    g.njb = (int)((n + 128 * h - 1) / (128 * h));
    g.ntiles = 0;
    for (int jb = 0; jb < g.njb; ++jb) g.ntiles += std::min(g.nib, h * (jb + 1));
    g.kblocks = kblocks;
    const int smax = std::max(1, std::min(kblocks, 8 * sms / g.ntiles + 1));
    for (int s = 1; s <= smax; ++s) {
      const int per = (kblocks + s - 1) / s;
      const int sp = (kblocks + per - 1) / per;
      const long waves = ((long)g.ntiles * sp + sms - 1) / sms;
      const long cost = waves * ((long)per * 256 * (1 + h) + 5000);
      if (best_cost < 0 || cost < best_cost) {
        best_cost = cost;
        g.splits = sp;
        g.kb_per = per;
        best = g;
      }
    }
  }
  if (const char* e = std::getenv("PIDB_K2_H")) {  // A/B: force the tile shape
    const int want = std::atoi(e);
    if (want != best.h && (want == 1 || want == 2)) {
      GramPlan g{};
      g.h = want;
      g.nib = (int)((n + kBM - 1) / kBM);
      g.njb = (int)((n + 128 * want - 1) / (128 * want));
      for (int jb = 0; jb < g.njb; ++jb) g.ntiles += std::min(g.nib, want * (jb + 1));
      g.kblocks = kblocks;
      g.splits = std::max(1, std::min(kblocks, sms / g.ntiles));
      g.kb_per = (kblocks + g.splits - 1) / g.splits;
      g.splits = (kblocks + g.kb_per - 1) / g.kb_per;
      best = g;
    }
  }
  best.units = best.ntiles * best.splits;
  best.smem = 1024 + (size_t)kStages * kABytes * (1 + best.h) + 256;
  best.ws = 256 + (size_t)best.units * kBM * 128 * best.h * sizeof(int32_t);
  return best;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_gram_i8_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  return plan_i8(n, m).ws;
}

template <int H>
static int launch_i8_h(const CUtensorMap& tmap, const uint8_t* tiles, bool bytes,
                       const GramPlan& g, int64_t n, int64_t* gram, void* ws, cudaStream_t st) {
  GramI8Params p{};
  p.n = (int)n; p.nib = g.nib; p.njb = g.njb; p.ntiles = g.ntiles; p.splits = g.splits;
  p.kblocks = g.kblocks; p.kb_per = g.kb_per;
  p.part = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 256);
  auto kern = bytes ? gram_i8_kernel<true, H> : gram_i8_kernel<false, H>;
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
  kern<<<g.units, kGramThreads, g.smem, st>>>(tmap, tiles, p);
  PIDB_LAUNCH_CHECK("gram_i8_kernel");
  constexpr int BPT = kBM / (256 / (kBNh<H> / 4));
  gram_i8_reduce_kernel<H><<<g.ntiles * BPT, 256, 0, st>>>(p.part, (int)n, g.nib, g.splits, gram);
  PIDB_LAUNCH_CHECK("gram_i8_reduce_kernel");
  return PIDB_OK;
}

static int launch_i8(const CUtensorMap& tmap, const uint8_t* tiles, bool bytes, int64_t n,
                     int64_t m, int64_t* gram, void* ws, size_t ws_bytes, cudaStream_t st) {
  const GramPlan g = plan_i8(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  return g.h == 1 ? launch_i8_h<1>(tmap, tiles, bytes, g, n, gram, ws, st)
                  : launch_i8_h<2>(tmap, tiles, bytes, g, n, gram, ws, st);
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
