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
// second kernel.  Warps (672 threads): 0 MMA issuer, 1-4 epilogue (one TMEM
// lane quadrant each), 5-20 converters (LDG.128 operand loads, two stages
// in flight in registers, hi/lo split written to the swizzled stages).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "tcgen05.cuh"

namespace pidb {
namespace {

constexpr int kB = 128;            // tile edge (members)
constexpr int kBK = 32;            // fp32 cells per stage (one 128-byte line)
constexpr int kStages = 3;
constexpr int kFlushStages = 16;   // 512 cells per fp32 accumulation block
constexpr int kTileBytes = kB * kBK * 4;             // 16 KB
constexpr int kStageBytes = 4 * kTileBytes;          // A_hi, B_hi, A_lo, B_lo
constexpr int kConvWarps = 16;
constexpr int kConvThreads = kConvWarps * 32;        // 512
constexpr int kEpiWarp0 = 1;                         // warps 1..4: epilogue
constexpr int kConvWarp0 = 5;                        // warps 5..20: converters
constexpr int kThreads = (kConvWarp0 + kConvWarps) * 32;  // 672
constexpr int kChunksPerTile = kB * kBK / 4;         // 16-byte chunks per operand tile
constexpr int kCPT = kChunksPerTile / kConvThreads;  // chunks per converter thread (2)
constexpr uint32_t kIdesc = tc::idesc(tc::kCF32, tc::kTF32, kB, kB);
// TMEM columns: [0,128) acc0, [128,256) acc1, [256,512) fp64 shadow (lo,hi pairs)
constexpr uint32_t kTmemCols = 512;

struct GramTf32Params {
  int n, nb, ntiles, splits, kblocks, kb_per;
  int64_t m, ld;
  const float* u;
  const double* w;   // nullable
  double* part;      // [units][kB][kB]   (Gram tiles), or
  const double* inv; // fused sums: inverse masses (n)
  double* vpart;     // [pieces][max_seg][4][kB]: tile row sums, inv-weighted row
                     //   sums, column sums, inv-weighted column sums
  // fused sums only: stream-K partition of the whole (tile, k-block) work
  int pieces, max_seg, w_off, w_diag;
  int64_t total;
};

// Stream-K partition (fused-sums path).  The work is a line of units, K-range
// round q (`splits` rounds of `kb_per` k-blocks) major and tile t (triangular
// order) minor -- so CTAs running at the same time read the same K window of
// the operand panels, as the plain split-K launch does -- unit (q, t) costing
// len(q) * (w_diag for a diagonal tile that shares its operand, else w_off).
// The line is cut into `pieces` (one per SM) equal parts; a piece covers the
// tail of one unit, whole units and the head of another, one segment each,
// every segment writing its own partial slot.
__host__ __device__ __forceinline__ int64_t sk_col_of(int64_t t) {  // column block of tile t
  int64_t jb = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (jb * (jb + 1) / 2 > t) --jb;
  while ((jb + 1) * (jb + 2) / 2 <= t) ++jb;
  return jb;
}
__host__ __device__ __forceinline__ int64_t sk_len(const GramTf32Params& p, int q) {
  const int64_t k0 = (int64_t)q * p.kb_per, k1 = k0 + p.kb_per;
  return (k1 < p.kblocks ? k1 : p.kblocks) - k0;
}
// start cost of unit u (u may equal splits * ntiles); diagonal tiles before t = its column block
__host__ __device__ __forceinline__ int64_t sk_u0(const GramTf32Params& p, int64_t u) {
  const int64_t q = u / p.ntiles, t = u - q * p.ntiles;
  const int64_t dw = p.w_off - p.w_diag;
  const int64_t round = (int64_t)p.w_off * p.ntiles - dw * p.nb;
  if (q >= p.splits)  // end of the line
    return (int64_t)p.kb_per * (p.splits - 1) * round + sk_len(p, p.splits - 1) * round;
  return (int64_t)p.kb_per * q * round + sk_len(p, (int)q) * ((int64_t)p.w_off * t - dw * sk_col_of(t));
}
__host__ __device__ __forceinline__ int64_t sk_c(const GramTf32Params& p, int64_t b) {
  return p.total * b / p.pieces;  // total * pieces < 2^63 (checked by the plan)
}
// largest unit u with u0(u) <= c
__host__ __device__ __forceinline__ int sk_unit_at(const GramTf32Params& p, int64_t c) {
  int lo = 0, hi = p.splits * p.ntiles - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sk_u0(p, mid) <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// largest piece b with c(b) <= c
__host__ __device__ __forceinline__ int sk_piece_at(const GramTf32Params& p, int64_t c) {
  int lo = 0, hi = p.pieces - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sk_c(p, mid) <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// k-block offset inside unit u at cost c (consecutive pieces share it: exact partition)
__host__ __device__ __forceinline__ int64_t sk_kb(int64_t c, int64_t u0, int wt, int64_t len) {
  const int64_t x = c - u0;
  if (x <= 0) return 0;
  const int64_t kb = (x + wt - 1) / wt;
  return kb < len ? kb : len;
}

__device__ __forceinline__ void tile_of(int t, int& ib, int& jb) {
  jb = 0;
  while (t > jb) {  // tiles of column block jb: ib = 0..jb
    t -= jb + 1;
    ++jb;
  }
  ib = t;
}

// Operands are fetched by the converter warps themselves with coalesced
// 128-bit loads (a warp reads four whole 128-byte member lines): TMA boxes
// with 128-byte rows are capped at ~16 B/clk/SM (tools/ubench_tma.cu), below
// what the tensor cores consume.  Each chunk is written twice into the
// 128B-swizzled K-major stage: hi (the raw fp32 word, which the tensor core
// truncates to tf32, or rna(w*u) when weighted) and lo = rna(a - hi).
struct OperandChunks {
  float4 v[2][kCPT];  // [A/B][chunk]
};

__global__ void __launch_bounds__(kThreads, 1)
    gram_tf32_kernel(const GramTf32Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  uint64_t* conv = reinterpret_cast<uint64_t*>(ring + kStages * kStageBytes);
  uint64_t* empty = conv + kStages;
  uint64_t* acc_full = empty + kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool fused = p.vpart != nullptr;
  const bool weighted = p.w != nullptr;
  // Segment state lives in shared memory (thread 0 writes it at each segment
  // start) so nothing but the loop index stays live across segments:
  // [0] tile, [1] kb0, [2] kb1, [3] ring stages and [4] accumulation blocks
  // consumed by earlier segments, [5] segment count.
  int* segtab = reinterpret_cast<int*>(tmem_slot + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&conv[s], kConvThreads);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_mbar_init();
    int nseg = 1;  // one (tile, split) unit, or the tiles a stream-K piece touches
    if (fused) {
      const int64_t c0 = sk_c(p, blockIdx.x), c1 = sk_c(p, blockIdx.x + 1);
      nseg = c1 > c0 ? sk_unit_at(p, c1 - 1) - sk_unit_at(p, c0) + 1 : 0;
    }
    segtab[3] = 0;
    segtab[4] = 0;
    segtab[5] = nseg;
  }
  if (warp == kEpiWarp0) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

#pragma unroll 1
  for (int seg = 0; seg < segtab[5]; ++seg) {
  if (threadIdx.x == 0) {
    if (fused) {
      const int64_t c0 = sk_c(p, blockIdx.x), c1 = sk_c(p, blockIdx.x + 1);
      const int u = sk_unit_at(p, c0) + seg;
      const int q = u / p.ntiles, t = u - q * p.ntiles;
      int ib_, jb_;
      tile_of(t, ib_, jb_);
      const int wt = ib_ == jb_ ? p.w_diag : p.w_off;
      const int64_t u0 = sk_u0(p, u), len = sk_len(p, q);
      segtab[0] = t;
      segtab[1] = q * p.kb_per + (int)sk_kb(c0, u0, wt, len);
      segtab[2] = q * p.kb_per + (int)sk_kb(c1, u0, wt, len);
    } else {
      const int t = blockIdx.x / p.splits;
      const int kb0 = (blockIdx.x - t * p.splits) * p.kb_per;
      segtab[0] = t;
      segtab[1] = kb0;
      segtab[2] = min(p.kblocks, kb0 + p.kb_per);
    }
  }
  __syncthreads();
  const int t = segtab[0], kb0 = segtab[1], kb1 = segtab[2];
  const int sbase = segtab[3], fbase = segtab[4];
  double* out = fused ? p.vpart + ((size_t)blockIdx.x * p.max_seg + seg) * 4 * kB
                      : p.part + (size_t)blockIdx.x * kB * kB;
  int ib, jb;
  tile_of(t, ib, jb);
  const bool diag = ib == jb;
  const bool share_b = diag && !weighted;  // B operand == A operand
  const int nk = max(0, kb1 - kb0);
  const int nflush = (nk + kFlushStages - 1) / kFlushStages;

  if (warp == 0) {
    // ---------------------------------------------------------- MMA issuer
    if (tc::elect_one()) {
      int s = sbase % kStages;
      uint32_t ph = (uint32_t)(sbase / kStages) & 1u;
      int k = 0;
      for (int f = fbase; f < fbase + nflush; ++f) {
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
  } else if (warp >= kConvWarp0) {
    // ----------------------------------------------------------- converters
    const int ct = threadIdx.x - kConvWarp0 * 32;  // 0..511
    const int nops = share_b ? 1 : 2;
    // chunk c = ct + q * 512: line r = c >> 3, chunk ch = c & 7 (logical)
    auto load = [&](int k, OperandChunks& oc) {
      const int64_t x0 = (int64_t)(kb0 + k) * kBK;
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        if (o >= nops) break;
        const int rb = (o == 0 ? ib : jb) * kB;
#pragma unroll
        for (int q = 0; q < kCPT; ++q) {
          const int c = ct + q * kConvThreads;
          const int r = c >> 3, ch = c & 7;
          const int64_t x = x0 + ch * 4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (rb + r < p.n) {
            const float* src = p.u + (int64_t)(rb + r) * p.ld + x;
            if (x + 4 <= p.m) {
              v = __ldcg(reinterpret_cast<const float4*>(src));
            } else {
              if (x + 0 < p.m) v.x = src[0];
              if (x + 1 < p.m) v.y = src[1];
              if (x + 2 < p.m) v.z = src[2];
            }
          }
          oc.v[o][q] = v;
        }
      }
    };
    auto store = [&](int k, int s, const OperandChunks& oc) {
      unsigned char* st = ring + s * kStageBytes;
      const int64_t x0 = (int64_t)(kb0 + k) * kBK;
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        if (o >= nops) break;
#pragma unroll
        for (int q = 0; q < kCPT; ++q) {
          const int c = ct + q * kConvThreads;
          const int r = c >> 3, ch = c & 7;
          const uint32_t off = (uint32_t)(r * 128) + ((uint32_t)(ch ^ (r & 7)) << 4);
          float4 v = oc.v[o][q];
          float4 hi;
          if (o == 0 && weighted) {
            const int64_t x = x0 + ch * 4;
            v.x = (float)((double)v.x * (x + 0 < p.m ? __ldg(p.w + x + 0) : 0.0));
            v.y = (float)((double)v.y * (x + 1 < p.m ? __ldg(p.w + x + 1) : 0.0));
            v.z = (float)((double)v.z * (x + 2 < p.m ? __ldg(p.w + x + 2) : 0.0));
            v.w = (float)((double)v.w * (x + 3 < p.m ? __ldg(p.w + x + 3) : 0.0));
            hi = make_float4(tc::tf32_rna(v.x), tc::tf32_rna(v.y), tc::tf32_rna(v.z),
                             tc::tf32_rna(v.w));
          } else {
            hi = v;  // the tensor core reads tf32 = truncation of this word
            v = make_float4(tc::tf32_trunc(v.x), tc::tf32_trunc(v.y), tc::tf32_trunc(v.z),
                            tc::tf32_trunc(v.w));
            v = make_float4(hi.x - v.x, hi.y - v.y, hi.z - v.z, hi.w - v.w);  // exact remainder
            *reinterpret_cast<float4*>(st + o * kTileBytes + off) = hi;
            *reinterpret_cast<float4*>(st + (2 + o) * kTileBytes + off) =
                make_float4(tc::tf32_rna(v.x), tc::tf32_rna(v.y), tc::tf32_rna(v.z),
                            tc::tf32_rna(v.w));
            continue;
          }
          *reinterpret_cast<float4*>(st + o * kTileBytes + off) = hi;
          *reinterpret_cast<float4*>(st + (2 + o) * kTileBytes + off) =
              make_float4(tc::tf32_rna(v.x - hi.x), tc::tf32_rna(v.y - hi.y),
                          tc::tf32_rna(v.z - hi.z), tc::tf32_rna(v.w - hi.w));
        }
      }
    };
    // two stages of loads in flight in registers
    OperandChunks r0, r1;
    if (nk > 0) load(0, r0);
    if (nk > 1) load(1, r1);
    int s = sbase % kStages;
    uint32_t ph = (uint32_t)(sbase / kStages) & 1u;
    for (int k = 0; k < nk; k += 2) {
      mbar_wait(&empty[s], ph ^ 1u);
      store(k, s, r0);
      fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05.mma
      mbar_arrive(&conv[s]);
      if (++s == kStages) { s = 0; ph ^= 1u; }
      if (k + 2 < nk) load(k + 2, r0);
      if (k + 1 >= nk) break;
      mbar_wait(&empty[s], ph ^ 1u);
      store(k + 1, s, r1);
      fence_proxy_async_smem();
      mbar_arrive(&conv[s]);
      if (++s == kStages) { s = 0; ph ^= 1u; }
      if (k + 3 < nk) load(k + 3, r1);
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
    for (int f = fbase; f < fbase + nflush; ++f) {
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
    double* dst = out + (size_t)(quad * 32 + lane) * kB;
#pragma unroll 1
    for (int c = 0; c < kB && !fused; c += 16) {
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
  if (fused) {
    // Fused epilogue (no N x N Gram in HBM): the fp64 tile goes to SMEM (the
    // operand ring is idle once every role has left its loop; rows padded to
    // kB + 1 doubles for the column pass), then 4 x kB tile sums are written:
    // sum_j G_ij, sum_j inv_j G_ij (rows of block ib), sum_i G_ij,
    // sum_i inv_i G_ij (columns of block jb).  Fixed order: deterministic.
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    constexpr int kLd = kB + 1;
    double* tile = reinterpret_cast<double*>(ring);
    if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
      const int quad = warp & 3;
      const int r = quad * 32 + lane;
      const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < kB; c += 16) {
        uint32_t sh[32];
        tc::tmem_ld32(lane_base + 256 + (uint32_t)(2 * c), sh);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          tile[r * kLd + c + e] = __hiloint2double((int)sh[2 * e + 1], (int)sh[2 * e]);
      }
    }
    __syncthreads();
    const int tx = threadIdx.x;
    double* vp = out;
    if (tx < kB) {  // row tx of block ib
      double a = 0.0, b = 0.0;
      for (int c = 0; c < kB; ++c) {
        const int j = jb * kB + c;
        const double g = tile[tx * kLd + c];
        a += g;
        b = fma(j < p.n ? p.inv[j] : 0.0, g, b);
      }
      vp[tx] = a;
      vp[kB + tx] = b;
    } else if (tx < 2 * kB) {  // column c of block jb
      const int c = tx - kB;
      double a = 0.0, b = 0.0;
      for (int r = 0; r < kB; ++r) {
        const int i = ib * kB + r;
        const double g = tile[r * kLd + c];
        a += g;
        b = fma(i < p.n ? p.inv[i] : 0.0, g, b);
      }
      vp[2 * kB + c] = a;
      vp[3 * kB + c] = b;
    }
    // the next segment's converters reuse the ring, its epilogue the shadow
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0) {
      segtab[3] = sbase + nk;
      segtab[4] = fbase + nflush;
    }
  }
  }  // segments
  tc::fence_before();
  __syncthreads();
  if (warp == kEpiWarp0) tc::tmem_dealloc(tmem, kTmemCols);
}

// row_plain[r] = sum_j G_rj, col_inv[r] = sum_j inv_j G_rj (G symmetric) from
// the fused tile sums: tiles (I(r), jb >= I(r)) contribute their row sums,
// tiles (ib < I(r), I(r)) their column sums; a unit's segments are read in
// piece order (= k order).
__global__ void gram_tf32_sums_kernel(const GramTf32Params p, double* __restrict__ row_plain,
                                      double* __restrict__ col_inv) {
  // one warp per member row; lanes take the (column block, K round) units in
  // a fixed assignment and a fixed shuffle tree combines them: deterministic
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= p.n) return;
  const int R = r / kB, o = r - R * kB;
  double a = 0.0, b = 0.0;
  for (int idx = lane; idx < p.nb * p.splits; idx += 32) {
    const int jb = idx / p.splits, q = idx - jb * p.splits;
    const int ib = min(R, jb), jj = max(R, jb);
    const int tile = jj * (jj + 1) / 2 + ib;
    const bool as_row = R <= jb;  // r in the tile's row block
    const int u = q * p.ntiles + tile;
    const int b0 = sk_piece_at(p, sk_u0(p, u));
    const int b1 = sk_piece_at(p, sk_u0(p, u + 1) - 1);
    for (int pc = b0; pc <= b1; ++pc) {
      const int64_t c0 = sk_c(p, pc);
      if (sk_c(p, pc + 1) == c0) continue;  // empty piece
      const int seg = u - sk_unit_at(p, c0);
      const double* vp = p.vpart + ((size_t)pc * p.max_seg + seg) * 4 * kB;
      if (as_row) {
        a += vp[o];
        b += vp[kB + o];
      } else {
        a += vp[2 * kB + o];
        b += vp[3 * kB + o];
      }
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, s);
    b += __shfl_xor_sync(0xffffffffu, b, s);
  }
  if (lane == 0) {
    row_plain[r] = a;
    col_inv[r] = b;
  }
}

// G[i][j] = G[j][i] = sum over splits (fixed order) of the tile holding
// (i, j), i <= j: each upper-triangle entry is summed once along coalesced
// rows and written to both halves.
__global__ void gram_tf32_reduce_kernel(const double* __restrict__ part, int n, int splits,
                                        double* __restrict__ out) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    if (i > j) continue;
    const int ib = i / kB, jb = j / kB;
    const int t = jb * (jb + 1) / 2 + ib;
    const double* src = part + ((size_t)t * splits * kB + (i - ib * kB)) * kB + (j - jb * kB);
    double acc = 0.0;
#pragma unroll 4
    for (int s = 0; s < splits; ++s) acc += __ldg(src + (size_t)s * kB * kB);
    out[e] = acc;
    if (i != j) out[(int64_t)j * n + i] = acc;
  }
}

struct Plan {
  int nb, ntiles, splits, kblocks, kb_per, units;
  size_t smem, ws;
  // fused sums (stream-K)
  int pieces, max_seg, w_off, w_diag;
  int64_t total;
};

// Relative cost of a shared-operand diagonal tile (off-diagonal = 10).  It
// loads half the bytes but runs the same MMAs: measured at 1000 x 256^3,
// costs 0.6 / 0.7 / 0.8 / 1.0 gave 153.8 / 144.2 / 146.5 / 149.6 ms (0.5:
// 183.9 ms; box-to-box spread is of the same order).  PIDB_K1_DIAG_COST in
// (0, 1] overrides the default 0.7.
int diag_cost10() {
  if (const char* e = std::getenv("PIDB_K1_DIAG_COST")) {
    const double x = std::atof(e);
    if (x > 0.0 && x <= 1.0) return std::max(1, (int)std::lround(10.0 * x));
  }
  return 7;
}

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
  g.smem = 1024 + (size_t)kStages * kStageBytes + 256;
  g.ws = 256 + (size_t)g.units * kB * kB * sizeof(double);
  return g;
}

// Stream-K partition of the fused-sums launch: one piece per SM.
Plan plan_sums(int64_t n, int64_t m, bool weighted) {
  Plan g = plan(n, m);
  g.w_off = 10;
  g.w_diag = weighted ? 10 : diag_cost10();
  GramTf32Params p{};
  p.nb = g.nb; p.ntiles = g.ntiles; p.splits = g.splits; p.kblocks = g.kblocks;
  p.kb_per = g.kb_per; p.w_off = g.w_off; p.w_diag = g.w_diag;
  g.total = p.total = sk_u0(p, (int64_t)g.splits * g.ntiles);
  int pieces = sm_count();
  if (const char* e = std::getenv("PIDB_K1_PIECES")) pieces = std::max(1, std::atoi(e));  // A/B hook
  g.pieces = p.pieces = (int)std::max<int64_t>(1, std::min<int64_t>(pieces, g.total));
  if (g.total > INT64_MAX / (g.pieces + 1)) g.pieces = 0;  // rejected by the entry point
  g.max_seg = 1;
  for (int b = 0; b < g.pieces; ++b) {
    const int64_t c0 = sk_c(p, b), c1 = sk_c(p, b + 1);
    if (c1 > c0) g.max_seg = std::max(g.max_seg, sk_unit_at(p, c1 - 1) - sk_unit_at(p, c0) + 1);
  }
  g.ws = 256 + (size_t)g.pieces * g.max_seg * 4 * kB * sizeof(double);
  return g;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_gram_tf32x3_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  return std::max(plan(n, m).ws, std::max(plan_sums(n, m, false).ws, plan_sums(n, m, true).ws));
}

extern "C" int pidb_gram_tf32x3_sums(const float* u, int64_t n, int64_t m, int64_t ld,
                                     const double* w, const double* inv, double* row_plain,
                                     double* col_inv, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u && inv && row_plain && col_inv && n >= 1 && m >= 1,
               "bad arguments to pidb_gram_tf32x3_sums");
  PIDB_REQUIRE(ld >= m && (ld * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0,
               "member rows must be 16-byte aligned with ld >= m");
  PIDB_REQUIRE(n <= (1 << 16), "too many members for the dense Gram");
  const Plan g = plan_sums(n, m, w != nullptr);
  PIDB_REQUIRE(g.pieces > 0, "ensemble too large for the fused Gram sums");
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  GramTf32Params p{};
  p.n = (int)n; p.nb = g.nb; p.ntiles = g.ntiles; p.splits = g.splits; p.kblocks = g.kblocks;
  p.kb_per = g.kb_per; p.m = m; p.ld = ld; p.u = u; p.w = w;
  p.inv = inv;
  p.vpart = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  p.pieces = g.pieces; p.max_seg = g.max_seg; p.w_off = g.w_off; p.w_diag = g.w_diag;
  p.total = g.total;
  cudaStream_t st = (cudaStream_t)stream;
  PIDB_CUDA(cudaFuncSetAttribute(gram_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)g.smem));
  gram_tf32_kernel<<<g.pieces, kThreads, g.smem, st>>>(p);
  PIDB_LAUNCH_CHECK("gram_tf32_kernel (fused sums)");
  gram_tf32_sums_kernel<<<(unsigned)((n + 3) / 4), 128, 0, st>>>(p, row_plain, col_inv);
  PIDB_LAUNCH_CHECK("gram_tf32_sums_kernel");
  return PIDB_OK;
}

extern "C" int pidb_gram_tf32x3(const float* u, int64_t n, int64_t m, int64_t ld, const double* w,
                                double* gram, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u && gram && n >= 1 && m >= 1, "bad arguments to pidb_gram_tf32x3");
  PIDB_REQUIRE(ld >= m && (ld * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0,
               "member rows must be 16-byte aligned with ld >= m");
  PIDB_REQUIRE(n <= (1 << 16), "too many members for the dense Gram");
  const Plan g = plan(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws, "workspace too small: need %zu bytes", g.ws);
  GramTf32Params p{};
  p.n = (int)n; p.nb = g.nb; p.ntiles = g.ntiles; p.splits = g.splits; p.kblocks = g.kblocks;
  p.kb_per = g.kb_per; p.m = m; p.ld = ld; p.u = u; p.w = w;
  p.part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  cudaStream_t st = (cudaStream_t)stream;
  PIDB_CUDA(cudaFuncSetAttribute(gram_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)g.smem));
  gram_tf32_kernel<<<g.units, kThreads, g.smem, st>>>(p);
  PIDB_LAUNCH_CHECK("gram_tf32_kernel");
  const int64_t total = n * n;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  gram_tf32_reduce_kernel<<<blocks, 256, 0, st>>>(p.part, (int)n, g.splits, gram);
  PIDB_LAUNCH_CHECK("gram_tf32_reduce_kernel");
  return PIDB_OK;
}
