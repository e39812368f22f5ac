// K1: the fuzzy Gram G = U diag(w) U^T on the int8 tensor cores with EXACT
// integer accumulation (fixed-point digit slices, "Ozaki" style).
//
// Replaces the fp64 BLAS tile products of the exact PID:
//   depth_pid / _pairwise_sums  /root/reference/pkg/src/fuzzdepth/depth.py:122-161, 213-228
//   gram_block                  /root/reference/pkg/src/fuzzdepth/reduction.py:75-97
//
// Why not TF32: the tensor core accumulates fp32 with truncation, which
// biases every 3xTF32 Gram entry by ~1e-6 relative -- 14x the smallest
// depth gap at BASELINE configs[3].  Integer MMAs accumulate exactly.
//
// Representation (pidb_fixed_pack, one HBM pass): every member value u in
// [0, 1] (times sqrt(w / w_max) on weighted grids, so that G = w_max * sum
// a_i a_j) becomes q = rint(a * 2^31) <= 2^31, split into four base-256
// digits d0 (0..128), d1, d2, d3.  Per 32-cell block a member stores its
// digits plane by plane, [d0 x32 | d1 x32 | d2 x32 | d3 x32] = one 128-byte
// line, and the lines of 128 members (a row block) for one cell block form
// one contiguous 16 KB tile already in the 128-byte-swizzled K-major order
// the tensor core reads (16-byte chunk c of line r at chunk c ^ (r % 8)):
// a stage is one or two plain 1D bulk copies (full DRAM bursts, unlike a
// 2D box of 128-byte rows strided by the member pitch), digit plane k is
// the operand descriptor advanced by 32 bytes.  Tiles are ordered
// [row block][cell block], so a row block's stream is sequential.
//
// Products: q_i q_j = 2^24 * sum_s 2^(8(3-s)) L_s with L_s = sum_{k+l=s}
// d_k e_l; the levels s = 0..3 (10 digit pairs) are kept, the dropped
// levels 4..6 are < 2.8e-9 per cell product and zero whenever either value
// has no low-order digits (0, 1 and every value that quantises to a
// multiple of 2^-7).  Each level accumulates in its own 32-bit TMEM
// accumulator (M = N = 128, 4 x 128 = all 512 columns) -- exact, read as
// uint32, for 512 stages (16384 cells; worst case 3.2e9 < 2^32) -- then
// the epilogue warps fold v = ((L0*256 + L1)*256 + L2)*256 + L3 (an integer
// < 2^53, exact in fp64) into fp64 accumulators held in registers.
// Emulated against the fp64 Gram before it was built
// (tools/fixed_gram_emulation.py): depth error <= 3.2e-9 at N = 300 with
// uniform, u^8 and ellipsoid members, 0 rank swaps.
//
// Work: 128 x 128 tiles of the upper block triangle x K rounds, persistent
// CTAs over the (round, tile) units (all 148 SMs busy with equal work where
// the counts allow); diagonal tiles load one operand.  Warps (576 threads):
// 0 bulk-copy producer (6-stage ring, 32 KB per stage), 1 MMA issuer, 2-17
// epilogue (TMEM lane quadrant = warp % 4, 32 columns each).  Outputs per
// unit: the fp64 tile, or (PID) its row sums, inverse-mass-weighted row sums
// and the two column counterparts; fixed-order reductions finish both.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "tcgen05.cuh"

namespace pidb {
namespace {

constexpr int kB = 128;                      // tile edge (members)
constexpr int kLine = 128;                   // bytes per member per stage (32 cells x 4 digits)
constexpr int kCellsPerStage = 32;
constexpr int kStages = 6;                   // 192 KB ring (also holds the 132 KB fp64 tile at the end)
constexpr int kTileBytes = kB * kLine;       // 16 KB
constexpr int kStageBytes = 2 * kTileBytes;  // A and B
// stages per 32-bit accumulation window: the level sums are non-negative and
// integer MMA accumulation wraps modulo 2^32, so read as uint32 they are exact
// below 2^32 -- 512 stages (16384 cells; worst case 3.2e9) -- half the folds
// of a signed 2^31 bound
constexpr int kFlush = 512;
constexpr int kEpiWarps = 16;
constexpr int kThreads = (2 + kEpiWarps) * 32;
constexpr uint32_t kIdesc = tc::idesc(tc::kCS32, tc::kU8, kB, kB);
constexpr double kTwoPow31 = 2147483648.0;

// Work units: (K round q, tile t), q-major (unit u = q ntiles + t); the K
// range is cut into `rounds` windows of R blocks (the last Rl).  Persistent
// CTAs take units u = c, c + G, c + 2G, ...: with rounds chosen so that the
// unit count is a multiple of the grid (lcm(ntiles, SMs) / ntiles when the
// windows stay >= 256 blocks) every SM gets the same work, and the CTAs
// running together still read the same few K windows of the operand panels
// (L2 reuse across tiles; a stream-K line with staggered K offsets lost it:
// 52 -> 85 ms at cfg4).  One output slot per unit, reduced per tile in round
// order.
struct FxParams {
  int n, nib, ntiles, kblocks;
  int rounds, R, Rl;   // K windows: rounds - 1 of R blocks, then Rl
  int64_t units;       // rounds * ntiles
  int flush;           // stages per int32 window (kFlush; A/B hook PIDB_FX_FLUSH)
  int noload;          // A/B hook PIDB_FX_NOLOAD=1: skip the operand loads (timing only)
  int sums;            // 1: tile sums (PID), 0: fp64 tiles
  const double* inv;   // sums: inverse masses (n)
  double* part;        // sums: [units][4][kB]; tiles: [units][kB][kB]
};

__host__ __device__ __forceinline__ void fx_unit(const FxParams& p, int64_t u, int& t, int& kb0,
                                                 int& nk) {
  const int q = (int)(u / p.ntiles);
  t = (int)(u - (int64_t)q * p.ntiles);
  kb0 = q * p.R;
  nk = q < p.rounds - 1 ? p.R : p.Rl;
}

__host__ __device__ __forceinline__ void fx_tile(int t, int& ib, int& jb) {
  int j = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (j * (j + 1) / 2 > t) --j;
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  jb = j;
  ib = t - j * (j + 1) / 2;
}

// ---------------------------------------------------------------- packing
// One CTA (8 warps) per (group of 8 members = one 1 KB swizzle atom of every
// tile, segment of 128 cell blocks); warp w owns member 8g + w.  Per
// iteration a warp takes 128 cells (4 blocks): lane L loads cells 4L..4L+3
// with one 128-bit load, and its four digit-k bytes are exactly word L % 8
// of plane k of block L / 8 (no shuffles).  The words are staged in shared
// memory in the swizzled tile order and leave as 16-byte stores: per block
// the 8 members' lines are one contiguous 1 KB atom.
__device__ __forceinline__ uint32_t fx_quant(double a) {
  const uint32_t q = (uint32_t)__double2uint_rn(a * kTwoPow31);
  return min(q, 0x80000000u);
}

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  float4 v;
  __device__ __forceinline__ double operator[](int e) const { return (double)f(e); }
  __device__ __forceinline__ float f(int e) const {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  }
};
template <>
struct Vec4<double> {
  double2 a, b;
  __device__ __forceinline__ double operator[](int e) const {
    return e == 0 ? a.x : e == 1 ? a.y : e == 2 ? b.x : b.y;
  }
};

template <typename T>
__device__ __forceinline__ Vec4<T> fx_load4(const T* __restrict__ src, int64_t x, int64_t m) {
  Vec4<T> r;
  if (x + 3 < m) {
    if constexpr (sizeof(T) == 4) {
      r.v = __ldcs(reinterpret_cast<const float4*>(src + x));
    } else {
      r.a = __ldcs(reinterpret_cast<const double2*>(src + x));
      r.b = __ldcs(reinterpret_cast<const double2*>(src + x + 2));
    }
  } else {
    T t[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) t[e] = x + e < m ? src[x + e] : T(0);
    if constexpr (sizeof(T) == 4) {
      r.v = make_float4(t[0], t[1], t[2], t[3]);
    } else {
      r.a = make_double2(t[0], t[1]);
      r.b = make_double2(t[2], t[3]);
    }
  }
  return r;
}

constexpr int kPackSeg = 128;   // cell blocks per CTA unit
constexpr int kPackIter = 16;   // cell blocks per CTA iteration (4 loads in flight per lane)

template <typename T, bool W>
__global__ void __launch_bounds__(256, (sizeof(T) == 4 && !W) ? 4 : 3)
    fx_pack_kernel(const T* __restrict__ u, int64_t ld, int n, int64_t m,
                   const double* __restrict__ w, double inv_wmax, uint8_t* __restrict__ q,
                   int64_t nblk, int64_t nseg, unsigned long long* __restrict__ soft,
                   double* __restrict__ mpart) {
  __shared__ __align__(16) uint32_t stage[kPackIter][8][32];  // [block][member line][word]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane >> 3, wi = lane & 7;
  // every line of every tile is written, the padding members (rows n ..
  // 128 ceil(n / 128) - 1) as zeros: the digit buffer needs no zero fill
  const int64_t ngrp = (n + 127) / 128 * 16;
  for (int64_t unit = blockIdx.x; unit < ngrp * nseg; unit += gridDim.x) {
    const int64_t grp = unit / nseg, seg = unit - grp * nseg;
    const int64_t row = grp * 8 + warp;
    const bool live = row < n;
    const int64_t b0 = seg * kPackSeg, b1 = min(nblk, b0 + kPackSeg);
    const T* src = u + (live ? row : 0) * ld;
    const int r8 = (int)(grp & 15) * 8;  // first line of the group inside its tile
    // atom of this group in tile (row block, block): lines r8 .. r8 + 7
    uint8_t* atom0 = q + ((grp / 16) * nblk) * (int64_t)kTileBytes + r8 * kLine;
    unsigned int cnt = 0;
    double mass = 0.0;  // sum w u of this lane's cells (fp64, fixed order)
    for (int64_t b = b0; b < b1; b += kPackIter) {
      Vec4<T> v[kPackIter / 4];
#pragma unroll
      for (int j = 0; j < kPackIter / 4; ++j) {
        const int64_t x = (b + 4 * j + sub) * kCellsPerStage + 4 * wi;
        if (live) v[j] = fx_load4(src, x, m);
        else v[j] = fx_load4(src, x, 0);
      }
#pragma unroll
      for (int j = 0; j < kPackIter / 4; ++j) {
        const int64_t x = (b + 4 * j + sub) * kCellsPerStage + 4 * wi;
        uint32_t qv[4];
        if constexpr (sizeof(T) == 4 && !W) {
          {
            // unweighted fp32: u 2^31 is exact in fp32, so is its rounding
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float f = v[j].f(e);
              mass += (double)f;
              qv[e] = min(__float2uint_rn(f * 2147483648.0f), 0x80000000u);
            }
          }
        }
        if constexpr (sizeof(T) != 4 || W) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            double a = v[j][e];
            if (W && x + e < m) {
              const double wx = __ldcs(w + x + e);
              mass = fma(wx, a, mass);
              a *= sqrt(wx * inv_wmax);
            } else {
              mass += a;
            }
            qv[e] = fx_quant(a);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) cnt += (qv[e] & 0xFFFFFFu) != 0u;
        // 4 x 4 byte transpose: plane word k = byte (3 - k) of q0..q3
        const uint32_t lo01 = __byte_perm(qv[0], qv[1], 0x5140);  // q0.b0 q1.b0 q0.b1 q1.b1
        const uint32_t hi01 = __byte_perm(qv[0], qv[1], 0x7362);  // q0.b2 q1.b2 q0.b3 q1.b3
        const uint32_t lo23 = __byte_perm(qv[2], qv[3], 0x5140);
        const uint32_t hi23 = __byte_perm(qv[2], qv[3], 0x7362);
        uint32_t d[4];
        d[0] = __byte_perm(hi01, hi23, 0x7632);  // digit 0 = byte 3 (most significant)
        d[1] = __byte_perm(hi01, hi23, 0x5410);
        d[2] = __byte_perm(lo01, lo23, 0x7632);
        d[3] = __byte_perm(lo01, lo23, 0x5410);
        // line r = r8 + warp: byte 32k + 4wi -> chunk (2k + wi/4) ^ (r % 8) = ^ warp
#pragma unroll
        for (int k = 0; k < 4; ++k)
          stage[4 * j + sub][warp][((((2 * k + (wi >> 2)) ^ warp) & 7) << 2) + (wi & 3)] = d[k];
      }
      __syncthreads();
      // kPackIter blocks x 1 KB atoms, 16 bytes per thread and store
#pragma unroll
      for (int t = threadIdx.x; t < kPackIter * 64; t += 256) {
        const int blk_t = t >> 6, off = (t & 63) * 16;
        if (b + blk_t < b1) {
          PIDB_DCHECK(grp / 16 < (n + 127) / 128 && b + blk_t < nblk, "K1x pack tile bounds");
          *reinterpret_cast<uint4*>(atom0 + (b + blk_t) * (int64_t)kTileBytes + off) =
              reinterpret_cast<const uint4*>(&stage[blk_t][0][0])[t & 63];
        }
      }
      __syncthreads();
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (soft && live && lane == 0 && cnt) atomicAdd(soft + row, (unsigned long long)cnt);
    if (mpart) {
      mass = warp_sum(mass);
      PIDB_DCHECK(!live || (row < n && seg < nseg), "K1x pack mass partial bounds");
      if (live && lane == 0) mpart[row * nseg + seg] = mass;
    }
  }
}

// masses[i] = sum over segments of the pack's per-(member, segment) partials,
// in segment order (deterministic).
__global__ void fx_mass_reduce_kernel(const double* __restrict__ mpart, int n, int64_t nseg,
                                      double* __restrict__ mass) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int64_t k = lane; k < nseg; k += 32) s += mpart[(int64_t)row * nseg + k];
  s = warp_sum(s);
  if (lane == 0) mass[row] = s;
}

// ------------------------------------------------------------------- Gram
__device__ __forceinline__ void epi_sync() {  // the 16 epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    gram_fx_kernel(const uint8_t* __restrict__ qd, const FxParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fl = p.flush;
  uint64_t* ring_free = tempty + 1;  // epilogue done with the ring (after a segment)

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kEpiWarps);
    mbar_init(ring_free, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      const uint64_t pol = policy_evict_last();  // panels are re-read by the other tiles
      int s = 0, seg = 0;
      uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++seg) {
        int t, kb0, nk, ib, jb;
        fx_unit(p, u, t, kb0, nk);
        fx_tile(t, ib, jb);
        const bool diag = ib == jb;
        const uint32_t bytes = diag ? kTileBytes : kStageBytes;
        // the previous segment's epilogue stages its fp64 tile in the ring
        if (seg > 0) mbar_wait(ring_free, (uint32_t)((seg - 1) & 1));
        for (int k = 0; k < nk; ++k) {
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* a = ring + s * kStageBytes;
          if (p.noload) {
            mbar_arrive(&full[s]);
          } else {
            mbar_arrive_expect_tx(&full[s], bytes);
            const int64_t kb = kb0 + k;
            PIDB_DCHECK(kb < p.kblocks && ib < p.nib && jb < p.nib, "K1x operand tile bounds");
            bulk_load(a, qd + ((int64_t)ib * p.kblocks + kb) * kTileBytes, kTileBytes, &full[s],
                      pol);
            if (!diag)
              bulk_load(a + kTileBytes, qd + ((int64_t)jb * p.kblocks + kb) * kTileBytes,
                        kTileBytes, &full[s], pol);
          }
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      int s = 0, win = 0;
      uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x) {
        int t, kb0, nk, ib, jb;
        fx_unit(p, u, t, kb0, nk);
        fx_tile(t, ib, jb);
        const bool diag = ib == jb;
        for (int k = 0; k < nk; ++k) {
          const int kw = k % fl;
          if (kw == 0 && win > 0) {
            mbar_wait(tempty, (uint32_t)((win - 1) & 1));  // epilogue drained TMEM
            tc::fence_after();
          }
          mbar_wait(&full[s], ph);
          tc::fence_after();
          const uint32_t a = smem_u32(ring + s * kStageBytes);
          const uint64_t da = tc::desc_kmajor_sw128(a);
          const uint64_t db = diag ? da : tc::desc_kmajor_sw128(a + kTileBytes);
          const uint32_t acc = kw != 0;
          // level s = k + l accumulates at TMEM column 128 s; digit plane k is
          // the descriptor advanced by 32 bytes (2 x 16-byte units) per plane
#pragma unroll
          for (int lv = 0; lv < 4; ++lv)
#pragma unroll
            for (int dk = 0; dk <= lv; ++dk)
              tc::mma_i8(tmem + 128u * lv, da + 2 * dk, db + 2 * (lv - dk), kIdesc,
                         dk != 0 ? 1u : acc);
          tc::commit(&empty[s]);
          if (kw == fl - 1 || k == nk - 1) {
            tc::commit(tfull);
            ++win;
          }
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else {
    // epilogue: TMEM lane quadrant q (hardware rule: warp % 4), columns c0..c0+31
    const int q = warp & 3, cc = (warp - 2) >> 2;
    const int row = q * 32 + lane, c0 = cc * 32;
    const int et = threadIdx.x - 64;  // 0..511
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
    int win = 0;
    for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x) {
      int t, kb0, nk, ib, jb;
      fx_unit(p, u, t, kb0, nk);
      fx_tile(t, ib, jb);
      const bool diag = ib == jb;
      const int nflush = (nk + fl - 1) / fl;
      double acc[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) acc[e] = 0.0;
      for (int f = 0; f < nflush; ++f, ++win) {
        mbar_wait(tfull, (uint32_t)(win & 1));
        tc::fence_after();
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          // v = ((L0 * 256 + L1) * 256 + L2) * 256 + L3: integers < 2^53, exact in fp64
          uint32_t r[4][4];
#pragma unroll
          for (int lv = 0; lv < 4; ++lv) tc::tmem_ld4(tbase + 128u * lv + 4u * h, r[lv]);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            double v = (double)r[0][e];  // uint32 (see kFlush)
#pragma unroll
            for (int lv = 1; lv < 4; ++lv) v = fma(v, 256.0, (double)r[lv][e]);
            acc[4 * h + e] += v;
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }

      // All of the segment's stages are consumed: stage the fp64 tile in the
      // ring (row stride kB + 1 doubles), then sum / store it in a fixed order.
      double* tile = reinterpret_cast<double*>(ring);
      constexpr int kLd = kB + 1;
#pragma unroll
      for (int e = 0; e < 32; ++e) tile[row * kLd + c0 + e] = acc[e];
      epi_sync();
      const int64_t slot = u;
      PIDB_DCHECK(slot < p.units && t < p.ntiles, "K1x output slot bounds");
      if (!p.sums) {
        double* dst = p.part + (size_t)slot * kB * kB;
        for (int e = et; e < kB * kB; e += kEpiWarps * 32) dst[e] = tile[(e / kB) * kLd + (e % kB)];
      } else {
        // et / 128 = 0: row sums, 1: rows weighted by inv_j, 2: column sums,
        // 3: columns weighted by inv_i (off-diagonal tiles only)
        const int kind = et >> 7, r = et & (kB - 1);
        double s2 = 0.0;
        if (kind == 0) {
          for (int c = 0; c < kB; ++c) s2 += tile[r * kLd + c];
        } else if (kind == 1) {
          for (int c = 0; c < kB; ++c) {
            const int gj = jb * kB + c;
            s2 += (gj < p.n ? __ldg(p.inv + gj) : 0.0) * tile[r * kLd + c];
          }
        } else if (!diag) {
          for (int x = 0; x < kB; ++x) {
            const int gi = ib * kB + x;
            const double wgt = kind == 2 ? 1.0 : (gi < p.n ? __ldg(p.inv + gi) : 0.0);
            s2 += wgt * tile[x * kLd + r];
          }
        }
        p.part[(size_t)slot * 4 * kB + et] = s2;
      }
      // hand the ring back to the producer (generic -> async proxy)
      fence_proxy_async_smem();
      epi_sync();
      if (et == 0) mbar_arrive(ring_free);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// Every slot of tile t (one unit per K round), in round order (fixed).
template <typename F>
__device__ __forceinline__ void fx_for_slots(const FxParams& p, int t, F&& f) {
  for (int q = 0; q < p.rounds; ++q) f((int64_t)q * p.ntiles + t);
}

// PID sums: row_plain[i] = sum_j G[i,j], col_inv[i] = sum_j inv_j G[i,j]
// (G symmetric), over the tiles holding member i as a row (ib, jb >= ib) or
// as a column (a < ib, ib).
__global__ void fx_sums_reduce_kernel(const FxParams p, double scale,
                                      double* __restrict__ row_plain,
                                      double* __restrict__ col_inv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const int ib = i / kB, r = i - ib * kB;
  double a = 0.0, b = 0.0;
  for (int jb = ib; jb < p.nib; ++jb)
    fx_for_slots(p, jb * (jb + 1) / 2 + ib, [&](int64_t slot) {
      const double* u = p.part + (size_t)slot * 4 * kB;
      a += u[r];
      b += u[kB + r];
    });
  for (int x = 0; x < ib; ++x)
    fx_for_slots(p, ib * (ib + 1) / 2 + x, [&](int64_t slot) {
      const double* u = p.part + (size_t)slot * 4 * kB;
      a += u[2 * kB + r];
      b += u[3 * kB + r];
    });
  row_plain[i] = a * scale;
  col_inv[i] = b * scale;
}

// G[i][j] = G[j][i] = scale * sum over the slots of the tile holding (i, j), i <= j.
__global__ void fx_tiles_reduce_kernel(const FxParams p, double scale, double* __restrict__ out) {
  const int n = p.n;
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    if (i > j) continue;
    const int ib = i / kB, jb = j / kB;
    double acc = 0.0;
    fx_for_slots(p, jb * (jb + 1) / 2 + ib, [&](int64_t slot) {
      acc += p.part[((size_t)slot * kB + (i - ib * kB)) * kB + (j - jb * kB)];
    });
    acc *= scale;
    out[e] = acc;
    if (i != j) out[(int64_t)j * n + i] = acc;
  }
}

struct FxPlan {
  int nib, ntiles, kblocks, grid, rounds, R, Rl;
  int64_t units;
  size_t smem, ws_tiles, ws_sums;
};

static int64_t fx_gcd(int64_t a, int64_t b) { return b ? fx_gcd(b, a % b) : a; }

FxPlan plan_fx(int64_t n, int64_t m) {
  FxPlan g{};
  g.nib = (int)((n + kB - 1) / kB);
  g.ntiles = g.nib * (g.nib + 1) / 2;
  g.kblocks = (int)((m + kCellsPerStage - 1) / kCellsPerStage);
  const int64_t sms = sm_count();
  // every SM gets the same number of units when rounds * ntiles is a
  // multiple of the SM count; keep K windows of >= one fold window (256
  // blocks), else fall back to about one unit per SM (split-K)
  int64_t rounds = sms / fx_gcd(g.ntiles, sms);
  if (g.kblocks / rounds < kFlush) rounds = std::max<int64_t>(1, sms / g.ntiles);
  rounds = std::max<int64_t>(1, std::min<int64_t>(rounds, g.kblocks));
  g.R = (int)((g.kblocks + rounds - 1) / rounds);
  g.rounds = (g.kblocks + g.R - 1) / g.R;
  g.Rl = g.kblocks - (g.rounds - 1) * g.R;
  g.units = (int64_t)g.rounds * g.ntiles;
  g.grid = (int)std::min<int64_t>(g.units, sms);
  g.smem = 1024 + (size_t)kStages * kStageBytes + 256;
  // the first 256 bytes of a shared workspace hold other kernels' completion
  // counters (zero between launches): partials start after them
  g.ws_tiles = 256 + (size_t)g.units * kB * kB * sizeof(double);
  g.ws_sums = 256 + (size_t)g.units * 4 * kB * sizeof(double);
  return g;
}

static void fx_fill(FxParams& prm, int64_t n, const FxPlan& g) {
  prm.n = (int)n; prm.nib = g.nib; prm.ntiles = g.ntiles; prm.kblocks = g.kblocks;
  prm.rounds = g.rounds; prm.R = g.R; prm.Rl = g.Rl; prm.units = g.units;
}

int launch_gram_fx(const uint8_t* qd, int64_t n, const FxPlan& g, FxParams prm,
                   cudaStream_t st) {
  fx_fill(prm, n, g);
  prm.flush = kFlush;
  if (const char* e = getenv("PIDB_FX_FLUSH")) prm.flush = std::max(1, atoi(e));
  prm.noload = getenv("PIDB_FX_NOLOAD") != nullptr && atoi(getenv("PIDB_FX_NOLOAD")) != 0;
  PIDB_CUDA(cudaFuncSetAttribute(gram_fx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)g.smem));
  gram_fx_kernel<<<g.grid, kThreads, g.smem, st>>>(qd, prm);
  PIDB_LAUNCH_CHECK("gram_fx_kernel");
  return PIDB_OK;
}

}  // namespace
}  // namespace pidb

using namespace pidb;

extern "C" size_t pidb_fixed_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  return (size_t)((n + kB - 1) / kB) * (size_t)((m + kCellsPerStage - 1) / kCellsPerStage) *
         kTileBytes;
}

extern "C" size_t pidb_fixed_pack_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1 || m < 1) return 0;
  const int64_t nblk = (m + kCellsPerStage - 1) / kCellsPerStage;
  return 256 + (size_t)n * ((nblk + kPackSeg - 1) / kPackSeg) * sizeof(double);
}

extern "C" int pidb_fixed_pack(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                               const double* w, double wmax, uint8_t* q, uint64_t* soft_count,
                               double* mass, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u && q && n >= 1 && m >= 1 && ld >= m, "bad arguments to pidb_fixed_pack");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "unknown dtype %d", dtype);
  PIDB_REQUIRE(ld % 4 == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0,
               "member rows must be 16-byte aligned with ld a multiple of 4");
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(q) & 1023) == 0, "digit tiles must be 1 KB aligned");
  PIDB_REQUIRE(!w || wmax > 0.0, "weighted packing needs wmax > 0");
  PIDB_REQUIRE(!mass || (ws && ws_bytes >= pidb_fixed_pack_workspace_bytes(n, m)),
               "workspace too small: need %zu bytes", pidb_fixed_pack_workspace_bytes(n, m));
  double* mpart = mass ? reinterpret_cast<double*>(static_cast<char*>(ws) + 256) : nullptr;
  const int64_t nblk = (m + kCellsPerStage - 1) / kCellsPerStage;
  const int64_t nseg = (nblk + kPackSeg - 1) / kPackSeg;
  const int64_t units = (n + 127) / 128 * 16 * nseg;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(units, 148 * 3));
  cudaStream_t st = (cudaStream_t)stream;
  const double iw = w ? 1.0 / wmax : 1.0;
  unsigned long long* sc = reinterpret_cast<unsigned long long*>(soft_count);
  const int b4 = (int)std::max<int64_t>(1, std::min<int64_t>(units, 148 * 4));
  if (dtype == PIDB_F32 && !w)  // register-light variant: 4 CTAs per SM
    fx_pack_kernel<float, false><<<b4, 256, 0, st>>>(static_cast<const float*>(u), ld, (int)n, m,
                                                     w, iw, q, nblk, nseg, sc, mpart);
  else if (dtype == PIDB_F32)
    fx_pack_kernel<float, true><<<blocks, 256, 0, st>>>(static_cast<const float*>(u), ld, (int)n,
                                                        m, w, iw, q, nblk, nseg, sc, mpart);
  else if (!w)
    fx_pack_kernel<double, false><<<blocks, 256, 0, st>>>(static_cast<const double*>(u), ld,
                                                          (int)n, m, w, iw, q, nblk, nseg, sc, mpart);
  else
    fx_pack_kernel<double, true><<<blocks, 256, 0, st>>>(static_cast<const double*>(u), ld, (int)n,
                                                         m, w, iw, q, nblk, nseg, sc, mpart);
  PIDB_LAUNCH_CHECK("fx_pack_kernel");
  if (mass) {
    fx_mass_reduce_kernel<<<(int)((n + 7) / 8), 256, 0, st>>>(mpart, (int)n, nseg, mass);
    PIDB_LAUNCH_CHECK("fx_mass_reduce_kernel");
  }
  return PIDB_OK;
}

extern "C" size_t pidb_gram_fixed_workspace_bytes(int64_t n, int64_t m, int sums) {
  if (n < 1 || m < 1) return 0;
  const FxPlan g = plan_fx(n, m);
  return sums ? g.ws_sums : g.ws_tiles;
}

static int fx_check(const uint8_t* q, int64_t n, int64_t m) {
  PIDB_REQUIRE(q && n >= 1 && m >= 1, "bad arguments to the fixed-point Gram");
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(q) & 1023) == 0, "digit tiles must be 1 KB aligned");
  PIDB_REQUIRE(n <= (1 << 20), "too many members for the Gram");
  PIDB_REQUIRE(m < ((int64_t)1 << 40), "too many cells");
  return PIDB_OK;
}

extern "C" int pidb_gram_fixed(const uint8_t* q, int64_t n, int64_t m, double wmax, double* gram,
                               void* ws, size_t ws_bytes, void* stream) {
  int rc = fx_check(q, n, m);
  if (rc != PIDB_OK) return rc;
  PIDB_REQUIRE(gram, "null output");
  const FxPlan g = plan_fx(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws_tiles, "workspace too small: need %zu bytes", g.ws_tiles);
  FxParams prm{};
  prm.sums = 0;
  prm.part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  cudaStream_t st = (cudaStream_t)stream;
  rc = launch_gram_fx(q, n, g, prm, st);
  if (rc != PIDB_OK) return rc;
  const double scale = wmax * std::ldexp(1.0, -38);
  const int64_t total = n * n;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  fx_fill(prm, n, g);
  fx_tiles_reduce_kernel<<<blocks, 256, 0, st>>>(prm, scale, gram);
  PIDB_LAUNCH_CHECK("fx_tiles_reduce_kernel");
  return PIDB_OK;
}

extern "C" int pidb_gram_fixed_sums(const uint8_t* q, int64_t n, int64_t m, double wmax,
                                    const double* inv, double* row_plain, double* col_inv,
                                    void* ws, size_t ws_bytes, void* stream) {
  int rc = fx_check(q, n, m);
  if (rc != PIDB_OK) return rc;
  PIDB_REQUIRE(inv && row_plain && col_inv, "null inverse masses or outputs");
  const FxPlan g = plan_fx(n, m);
  PIDB_REQUIRE(ws && ws_bytes >= g.ws_sums, "workspace too small: need %zu bytes", g.ws_sums);
  FxParams prm{};
  prm.sums = 1;
  prm.inv = inv;
  prm.part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  cudaStream_t st = (cudaStream_t)stream;
  rc = launch_gram_fx(q, n, g, prm, st);
  if (rc != PIDB_OK) return rc;
  const double scale = wmax * std::ldexp(1.0, -38);
  fx_fill(prm, n, g);
  fx_sums_reduce_kernel<<<(int)((n + 127) / 128), 128, 0, st>>>(prm, scale, row_plain, col_inv);
  PIDB_LAUNCH_CHECK("fx_sums_reduce_kernel");
  return PIDB_OK;
}
