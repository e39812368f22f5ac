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
// symmetric), K = cells split across CTAs.  Warp roles (192 threads):
//   warp 0 : TMA producer (128-byte swizzled K-major boxes, 4-stage ring)
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

__global__ void __launch_bounds__(kGramThreads, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap tmap, const GramI8Params p) {
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
    prefetch_tma_desc(&tmap);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, kBN);
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
        const int x = (kb0 + k) * kBK;
        tma_load_2d(a, &tmap, x, ib * kBM, &full[s], pol);
        tma_load_2d(a + kABytes, &tmap, x, jb * kBN, &full[s], pol);
        tma_load_2d(a + kABytes + kBM * kBK, &tmap, x, jb * kBN + kBM, &full[s], pol);
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
// Each upper-triangle entry is summed once (reads coalesced along j) and
// written to both halves; int64 sums are exact, so the order is immaterial.
__global__ void gram_i8_reduce_kernel(const int32_t* __restrict__ part, int n, int nib,
                                      int splits, int64_t* __restrict__ out) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    if (i > j) continue;
    const int ib = i / kBM, jb = j / kBN;
    int t = 0;
    for (int q = 0; q < jb; ++q) t += min(nib, 2 * q + 2);
    t += ib;
    const int32_t* src = part + ((size_t)t * splits * kBM + (i - ib * kBM)) * kBN + (j - jb * kBN);
    int64_t acc = 0;
#pragma unroll 8
    for (int s = 0; s < splits; ++s) acc += __ldg(src + (size_t)s * kBM * kBN);
    out[e] = acc;
    if (i != j) out[(int64_t)j * n + i] = acc;
  }
}

// ---------------------------------------------------------------------------
// K2f: K7 (binary check + u8 pack) fused into the K2 launch.  The CTAs of one
// K split (one per output tile) pack that split's cells cooperatively -- CTA
// t converts members [t * rpt, (t + 1) * rpt) -- chunk by chunk, publishing
// each chunk on a per-split counter (release); the TMA producer of every CTA
// of the split waits for the chunk (acquire + async-proxy fence) before
// loading its packed boxes.  Packing streams the fp32 members from HBM at
// full rate on 8 warps per SM while the tensor cores consume the chunks
// packed just before (L2-hot), so the pack and the Gram overlap instead of
// running back to back.  Needs every CTA resident (one wave); the
// workspace's split counters return to zero at exit.
constexpr int kPackWarps = 16;
constexpr int kPackUnroll = 2;                        // segments in flight per packer lane
constexpr int kFusedThreads = (6 + kPackWarps) * 32;  // 0 TMA, 1 MMA, 2-5 epilogue, 6-21 pack
constexpr int kChunkBlocks = 32;                       // K blocks (128 cells) per published chunk

struct FusedParams {
  GramI8Params g;
  const void* u;
  int dtype;
  int64_t m, ld, ldb;
  uint8_t* b;
  unsigned long long* nonbinary;
  unsigned* ready;  // [splits] published chunks x tiles
  unsigned* done;   // [splits] CTAs finished
};

// 16 cells per lane: 16-byte loads when the span is whole (load and pack
// phases are split so a lane keeps several segments in flight)
template <typename T>
__device__ __forceinline__ void load_segment(const T* __restrict__ row, int64_t x0, int64_t xend,
                                             T (&vals)[16]) {
  if (x0 + 16 <= xend) {
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
    for (int e = 0; e < 16; ++e) vals[e] = x0 + e < xend ? row[x0 + e] : T(0);
  }
}

template <typename T>
__device__ __forceinline__ unsigned store_segment(const T (&vals)[16], int64_t x0, int64_t xend,
                                                  uint8_t* __restrict__ dst) {
  uint32_t packed[4] = {0, 0, 0, 0};
  unsigned bad = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const T v = vals[e];
    bad += (x0 + e < xend) && !(v == T(0) || v == T(1));
    packed[e >> 2] |= (uint32_t)(v != T(0)) << (8 * (e & 3));
  }
  if (x0 < xend)
    *reinterpret_cast<uint4*>(dst + x0) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  return bad;
}

template <typename T>
__global__ void __launch_bounds__(kFusedThreads, 1)
    gram_i8_fused_kernel(const __grid_constant__ CUtensorMap tmap, const FusedParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const GramI8Params& g = p.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x;
  const int t = unit / g.splits, split = unit - t * g.splits;
  int ib, jb;
  tile_of(t, g.nib, ib, jb);
  const int kb0 = split * g.kb_per;
  const int kb1 = min(g.kblocks, kb0 + g.kb_per);
  const int nk = max(0, kb1 - kb0);

  if (threadIdx.x == 0) {
    prefetch_tma_desc(&tmap);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, kBN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 6) {
    // ---- packers: members [r0, r1) of this split's cells, chunk by chunk
    const int pw = warp - 6;
    const int rpt = (g.n + g.ntiles - 1) / g.ntiles;
    const int r0 = t * rpt, r1 = min(g.n, r0 + rpt);
    const T* u = static_cast<const T*>(p.u);
    const int nchunks = (nk + kChunkBlocks - 1) / kChunkBlocks;
    for (int c = 0; c < nchunks; ++c) {
      const int64_t xa = (int64_t)(kb0 + c * kChunkBlocks) * kBK;
      const int64_t xb = min(p.m, (int64_t)min(kb1, kb0 + (c + 1) * kChunkBlocks) * kBK);
      const int64_t segs = (xb - xa + 511) / 512;
      const int64_t jobs = (int64_t)(r1 - r0) * segs;
      constexpr int U = sizeof(T) == 4 ? kPackUnroll : 1;  // fp64: register budget
      for (int64_t j0 = pw; j0 < jobs; j0 += kPackWarps * U) {
        T vals[U][16];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int64_t job = j0 + q * kPackWarps;
          if (job < jobs) {
            const int64_t r = r0 + job / segs;
            load_segment(u + r * p.ld, xa + (job % segs) * 512 + lane * 16, xb, vals[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int64_t job = j0 + q * kPackWarps;
          if (job < jobs) {
            const int64_t r = r0 + job / segs;
            unsigned bad =
                store_segment(vals[q], xa + (job % segs) * 512 + lane * 16, xb, p.b + r * p.ldb);
            bad = __reduce_add_sync(0xffffffffu, bad);
            if (lane == 0 && bad && p.nonbinary) atomicAdd(p.nonbinary + r, (unsigned long long)bad);
          }
        }
      }
      __threadfence();
      asm volatile("bar.sync 2, %0;" ::"n"(kPackWarps * 32) : "memory");
      if (pw == 0 && lane == 0) {
        // publish chunk c only once every CTA of the split published c - 1:
        // the counter then reaches (c + 1) * ntiles exactly when chunk c is
        // complete everywhere (no CTA can count ahead of a straggler)
        const unsigned prior = (unsigned)c * (unsigned)g.ntiles;
        while (ld_acquire_gpu(p.ready + split) < prior) __nanosleep(32);
        atomicAdd(p.ready + split, 1u);  // release (after the fences)
      }
    }
  } else if (warp == 0) {
    if (tc::elect_one()) {
      const uint64_t pol = policy_evict_last();
      int s = 0, have = 0;
      uint32_t ph = 0;
      for (int k = 0; k < nk; ++k) {
        const int c = k / kChunkBlocks;
        if (c >= have) {  // wait until every CTA of the split packed chunk c
          const unsigned want = (unsigned)(c + 1) * (unsigned)g.ntiles;
          while (ld_acquire_gpu(p.ready + split) < want) __nanosleep(64);
          fence_proxy_async_global();
          have = c + 1;
        }
        mbar_wait(&empty[s], ph ^ 1u);
        unsigned char* a = ring + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], kStageBytes);
        const int x = (kb0 + k) * kBK;
        tma_load_2d(a, &tmap, x, ib * kBM, &full[s], pol);
        tma_load_2d(a + kABytes, &tmap, x, jb * kBN, &full[s], pol);
        tma_load_2d(a + kABytes + kBM * kBK, &tmap, x, jb * kBN + kBM, &full[s], pol);
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
        for (int kk = 0; kk < kBK / 32; ++kk)
          tc::mma_i8(tmem, da + 2 * kk, db + 2 * kk, kIdescI8, (k | kk) != 0);
        tc::commit(&empty[s]);
        if (++s == kStages) { s = 0; ph ^= 1u; }
      }
      tc::commit(tmem_full);
    }
  } else {
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc::fence_after();
    int32_t* dst = g.part + ((size_t)unit * kBM + row) * kBN;
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
  if (threadIdx.x == 0 && atomicAdd(p.done + split, 1u) == (unsigned)g.ntiles - 1) {
    // every CTA of the split is past all its waits: reset for the next call
    p.ready[split] = 0;
    p.done[split] = 0;
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
  // one wave: ceil(sms / ntiles) splits would leave a few CTAs (150 of them
  // at n = 500) for a second wave that doubles the kernel time
  g.splits = std::max(1, std::min(g.kblocks, sms / g.ntiles));
  g.kb_per = (g.kblocks + g.splits - 1) / g.splits;
  g.splits = (g.kblocks + g.kb_per - 1) / g.kb_per;
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

extern "C" int pidb_gram_i8(const uint8_t* b, int64_t n, int64_t m, int64_t ldb, int64_t* gram,
                            void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(b && gram && n >= 1 && m >= 1, "bad arguments to pidb_gram_i8");
  PIDB_REQUIRE(ldb >= m && ldb % 16 == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0,
               "packed rows must be 16-byte aligned with ldb >= m");
  PIDB_REQUIRE(m < ((int64_t)1 << 31), "int32 tensor-core accumulators need m < 2^31 cells");
  PIDB_REQUIRE(n <= (1 << 20), "too many members for the integer Gram");
  const GramPlan g = plan_i8(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  CUtensorMap tm;
  int rc = encode_tma_2d(&tm, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)m, (uint64_t)n,
                         (uint64_t)ldb, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != PIDB_OK) return rc;
  GramI8Params p{};
  p.n = (int)n; p.nib = g.nib; p.njb = g.njb; p.ntiles = g.ntiles; p.splits = g.splits;
  p.kblocks = g.kblocks; p.kb_per = g.kb_per;
  p.part = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 256);
  cudaStream_t st = (cudaStream_t)stream;
  PIDB_CUDA(cudaFuncSetAttribute(gram_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)g.smem));
  gram_i8_kernel<<<g.units, kGramThreads, g.smem, st>>>(tm, p);
  PIDB_LAUNCH_CHECK("gram_i8_kernel");
  const int64_t total = n * n;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  gram_i8_reduce_kernel<<<blocks, 256, 0, st>>>(p.part, (int)n, g.nib, g.splits, gram);
  PIDB_LAUNCH_CHECK("gram_i8_reduce_kernel");
  return PIDB_OK;
}

// The fused launch keeps its per-split counters in the workspace's first 256
// bytes (the zero-on-exit scratch every kernel shares): <= 32 splits.
constexpr int kFusedMaxSplits = 32;

static GramPlan plan_fused(int64_t n, int64_t m) {
  GramPlan g = plan_i8(n, m);
  if (g.splits > kFusedMaxSplits) {
    g.kb_per = (g.kblocks + kFusedMaxSplits - 1) / kFusedMaxSplits;
    g.splits = (g.kblocks + g.kb_per - 1) / g.kb_per;
    g.units = g.ntiles * g.splits;
    g.ws = 256 + (size_t)g.units * kBM * kBN * sizeof(int32_t);
  }
  return g;
}

extern "C" size_t pidb_eid_gram_fused_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  return plan_fused(n, m).ws;
}

extern "C" int pidb_eid_gram_fused(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                                   uint8_t* b, int64_t ldb, int64_t* nonbinary, int64_t* gram,
                                   void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u && b && gram && n >= 1 && m >= 1 && ld >= m, "bad arguments to pidb_eid_gram_fused");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  PIDB_REQUIRE(ldb >= m && ldb % 128 == 0 && (reinterpret_cast<uintptr_t>(b) & 127) == 0,
               "packed rows must be 128-byte aligned with ldb >= m");
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(u) & 15) == 0 &&
                   (ld * (dtype == PIDB_F32 ? 4 : 8)) % 16 == 0,
               "member rows must be 16-byte aligned");
  PIDB_REQUIRE(m < ((int64_t)1 << 31), "int32 tensor-core accumulators need m < 2^31 cells");
  const GramPlan g = plan_fused(n, m);
  if (g.units > sm_count()) {
    set_error("fused eID Gram needs one wave (%d units > %d SMs)", g.units, sm_count());
    return PIDB_EUNSUPPORTED;
  }
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  CUtensorMap tm;
  int rc = encode_tma_2d(&tm, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)m, (uint64_t)n,
                         (uint64_t)ldb, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != PIDB_OK) return rc;
  FusedParams p{};
  p.g.n = (int)n; p.g.nib = g.nib; p.g.njb = g.njb; p.g.ntiles = g.ntiles; p.g.splits = g.splits;
  p.g.kblocks = g.kblocks; p.g.kb_per = g.kb_per;
  char* base = static_cast<char*>(ws);
  p.ready = reinterpret_cast<unsigned*>(base);  // [0, 128): zero between launches
  p.done = p.ready + kFusedMaxSplits;           // [128, 256)
  p.g.part = reinterpret_cast<int32_t*>(base + 256);
  p.u = u; p.dtype = dtype; p.m = m; p.ld = ld; p.ldb = ldb; p.b = b;
  p.nonbinary = reinterpret_cast<unsigned long long*>(nonbinary);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PIDB_F32) {
    PIDB_CUDA(cudaFuncSetAttribute(gram_i8_fused_kernel<float>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    gram_i8_fused_kernel<float><<<g.units, kFusedThreads, g.smem, st>>>(tm, p);
  } else {
    PIDB_CUDA(cudaFuncSetAttribute(gram_i8_fused_kernel<double>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    gram_i8_fused_kernel<double><<<g.units, kFusedThreads, g.smem, st>>>(tm, p);
  }
  PIDB_LAUNCH_CHECK("gram_i8_fused_kernel");
  const int64_t total = n * n;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  gram_i8_reduce_kernel<<<blocks, 256, 0, st>>>(p.g.part, (int)n, g.nib, g.splits, gram);
  PIDB_LAUNCH_CHECK("gram_i8_reduce_kernel");
  return PIDB_OK;
}
