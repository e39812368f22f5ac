// K5 (PID-mean partials, one HBM pass) and K9-B (exact-PID column sums).
//
// Reference path replaced:
//   depth_pid_mean          /root/reference/pkg/src/fuzzdepth/depth.py:246-287
//     mean_mask             /root/reference/pkg/src/fuzzdepth/grid.py:251-261
//     mask_mass(mean)       /root/reference/pkg/src/fuzzdepth/grid.py:242-244
//     _member_mean_terms    /root/reference/pkg/src/fuzzdepth/depth.py:231-243
//   _pairwise_sums col_inv  /root/reference/pkg/src/fuzzdepth/depth.py:157,160 (K9-B)
//
// Layout: members are rows of a (n x m) row-major matrix in HBM.  A "tile" is
// V consecutive cells of ALL n members; one 2D TMA box per (column box, row
// box) brings it to shared memory with a 128/64/32-byte swizzle, so the same
// bytes are read from HBM exactly once and consumed twice from SMEM:
//   pass 1 (column sweep): S(x) = sum_i u_i(x)        [MODE_MEAN]
//                           T(x) = sum_i inv_i u_i(x)  [MODE_COLS]
//   pass 2 (row sweep)   : acc_i += u_i(x) * w(x) S(x),  mass_i += w(x) u_i(x)
// Pass 1 for fp32 data uses an error-free Fast2Sum in fp32 (seeded with 1.0 so
// that |s| >= |u| always holds; values are in [0,1]) and pass 2 converts each
// value once to fp64 (DFMA/DADD accumulation).  Each thread owns fixed
// (column box, member) items for the whole persistent CTA lifetime, so the
// member partials live in registers; CTA partials are reduced by the last CTA
// in a fixed order (bit-reproducible on a given device).
#include "common.cuh"

namespace pidb {
namespace {

#ifndef PIDB_K5_THREADS
#define PIDB_K5_THREADS 512
#endif
constexpr int kThreads = PIDB_K5_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int MODE_MEAN = 0;
constexpr int MODE_COLS = 1;
constexpr int MODE_MASS = 2;  // masses (+ nonbinary count) only: pass 2 without pass 1

struct StreamParams {
  int64_t n, m, tiles;
  int nrb, boxr;          // row boxes per column box, rows per box (multiple of 8)
  int stages;
  uint32_t stage_bytes;   // bytes of one tile in smem
  int mode;
  const double* w;        // nullable
  const double* inv;      // MODE_COLS
  double* part;           // [grid][items][2]
  double* part_col;       // [grid]
  int64_t* part_nb;       // [grid][n] (MODE_MASS, nullable)
  unsigned* counter;
  double* out_row;        // n
  double* out_mass;       // n (nullable in MODE_COLS)
  double* out_col;        // 1 (MODE_MEAN)
  int64_t* out_nb;        // n (MODE_MASS, nullable)
};

template <typename T>
struct Vec;  // one 16-byte chunk of member values
template <>
struct Vec<float> {
  static constexpr int EPC = 4;
  __device__ static void load(const unsigned char* p, double (&v)[4]) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  __device__ static float4 loadf(const unsigned char* p) {
    return *reinterpret_cast<const float4*>(p);
  }
};
template <>
struct Vec<double> {
  static constexpr int EPC = 2;
  __device__ static void load(const unsigned char* p, double (&v)[2]) {
    const double2 f = *reinterpret_cast<const double2*>(p);
    v[0] = f.x; v[1] = f.y;
  }
};

__device__ __forceinline__ bool is_nonbinary(double x) { return !(x == 0.0 || x == 1.0); }

// XOR applied to the 16-byte chunk index of line `r` by the TMA swizzle
// (rows of one column box are consecutive lines, boxes are 8-line aligned).
template <int LB>
__device__ __forceinline__ uint32_t swz_xor(uint32_t r) {
  if constexpr (LB == 128) return r & 7u;
  else if constexpr (LB == 64) return (r >> 1) & 3u;
  else return (r >> 2) & 1u;
}

// CTA column partial -> global; the last CTA to finish reduces every CTA's
// partials in a fixed order (grid, then column box) and resets the counter.
// part layout: [grid][pncb * n][2] (row sums, masses); part_nb [grid][n].
__device__ __forceinline__ void finish_partials(const StreamParams& p, int pncb, double col_acc,
                                                unsigned* s_ticket, double* s_col) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = (int)p.n;
  const int G = gridDim.x;
  {
    const double c = warp_sum(col_acc);
    if (lane == 0) s_col[warp] = c;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int k = 0; k < kWarps; ++k) t += s_col[k];
      p.part_col[blockIdx.x] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) *s_ticket = atomicAdd(p.counter, 1u);
  __syncthreads();
  if (*s_ticket != (unsigned)(G - 1)) return;

  __threadfence();
  for (int r = warp; r < n; r += kWarps) {
    double a = 0.0, b = 0.0;
    int64_t nb = 0;
    for (int g = lane; g < G; g += 32) {
      for (int cb = 0; cb < pncb; ++cb) {
        const double* src = p.part + ((size_t)g * pncb * n + cb * n + r) * 2;
        a += __ldcg(src);
        b += __ldcg(src + 1);
      }
      if (p.mode == MODE_MASS && p.part_nb != nullptr)
        nb += (int64_t)__ldcg(reinterpret_cast<const long long*>(p.part_nb + (size_t)g * n + r));
    }
    a = warp_sum(a);
    b = warp_sum(b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0) {
      if (p.mode == MODE_MASS) {
        p.out_mass[r] = b;
        if (p.out_nb) p.out_nb[r] = nb;
      } else {
        p.out_row[r] = a;
        if (p.out_mass) p.out_mass[r] = b;
      }
    }
  }
  if (warp == 0 && p.mode == MODE_MEAN) {
    double c = 0.0;
    for (int g = lane; g < G; g += 32) c += __ldcg(p.part_col + g);
    c = warp_sum(c);
    if (lane == 0) p.out_col[0] = c;
  }
  if (tid == 0) *p.counter = 0u;  // ready for the next launch on this workspace
}

// ---------------------------------------------------------------------------
// Kernel structure (software-pipelined over tiles, ONE block barrier per tile):
//   iteration j:  wait TMA(tile j)
//                 pass 1(tile j): column partials -> red[]          (all threads)
//                 __syncthreads
//                 refill: TMA(tile j-2+stages) into the stage tile j-2 used
//                 finalize(tile j): S, w*S, w -> sS/sW[j&1]          (V threads)
//                 pass 2(tile j-1): row sums against sS/sW[(j-1)&1]  (all threads)
// so finalize and pass 2 overlap other warps' work instead of serialising
// behind two barriers.  Pass 2 has two register layouts:
//   ROWS>0 : (128-byte lines, 2 column boxes) lane l owns 8 bytes of the row's
//            64-cell tile slice (lanes 0-15 box 0, 16-31 box 1), warp w owns
//            rows w, w+W, ..., accumulators stay in registers for the whole
//            kernel and are reduced across lanes once at the end;
//   ROWS==0: thread owns (column box, member) items (large N), IPT per thread.
template <typename T, int LB, int NCB, int IPT, int ROWS>
__global__ void __launch_bounds__(kThreads, 1)
    stream_pass_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  constexpr int EPC = Vec<T>::EPC;              // elements per 16-byte chunk
  constexpr int E = LB / (int)sizeof(T);        // elements per line (box inner)
  constexpr int V = NCB * E;                    // cells per tile
  constexpr int CPL = LB / 16;                  // chunks per line
  constexpr int QC = NCB * CPL;                 // chunks per tile row
  constexpr int P = kThreads / QC;              // row phases in pass 1
  constexpr int EPL = 8 / (int)sizeof(T);       // elements per lane in ROWS pass 2
  static_assert(kThreads % QC == 0 && QC <= 32 && P % 8 == 0 && kWarps % 8 == 0, "layout");
  static_assert(ROWS == 0 || (LB == 128 && NCB == 2), "row-resident pass 2 needs 2x128B lines");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // dynamic smem base rounded up to 1024 B (swizzle atom) without leaving the
  // shared address space (keeps LDS instead of generic loads)
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* tiles = smem_raw + pad;
  unsigned char* tail = tiles + (size_t)p.stages * p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  double* sS = reinterpret_cast<double*>(tail + 64);     // [2][V]: w*S (or w*T)
  double* sW = sS + 2 * V;                                 // [2][V]: w
  double* red = sW + 2 * V;                                // [2][kWarps][V]
  unsigned* s_ticket = reinterpret_cast<unsigned*>(red + 2 * kWarps * V);
  double* s_col = reinterpret_cast<double*>(s_ticket + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n = (int)p.n;
  const int G = gridDim.x;
  const bool weighted = p.w != nullptr;
  const int mode = p.mode;
  const int items = NCB * n;
  const int cb_rows = p.nrb * p.boxr;  // lines per column box

  const int64_t my_tiles = p.tiles > blockIdx.x ? (p.tiles - 1 - blockIdx.x) / G + 1 : 0;
  const uint64_t pol = policy_evict_first();

  if (tid == 0) {
    prefetch_tma_desc(&tmap);
    for (int s = 0; s < p.stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t j) {  // local tile j -> stage j % stages
    const int s = (int)(j % p.stages);
    const int64_t tile = blockIdx.x + j * G;
    unsigned char* dst = tiles + (size_t)s * p.stage_bytes;
    mbar_arrive_expect_tx(&full[s], p.stage_bytes);
    for (int cb = 0; cb < NCB; ++cb)
      for (int rb = 0; rb < p.nrb; ++rb)
        tma_load_2d(dst + (size_t)(cb * p.nrb + rb) * p.boxr * LB, &tmap,
                    (int32_t)(tile * V + cb * E), rb * p.boxr, &full[s], pol);
  };
  if (tid == 0)
    for (int64_t j = 0; j < my_tiles && j < p.stages; ++j) issue(j);

  // ------------------------------------------------------ pass-2 state
  constexpr int NACC = ROWS > 0 ? ROWS : IPT;
  double acc_row[NACC], acc_mass[NACC];
  int acc_nb[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { acc_row[k] = 0.0; acc_mass[k] = 0.0; acc_nb[k] = 0; }
  // ROWS layout: lane -> (column box, 8-byte slot) of every owned row
  const int r_cb = lane >> 4, r_pos = lane & 15;
  const int r_cell = r_cb * E + r_pos * EPL;  // first tile cell of this lane
  // ITEMS layout: item = cb*n + r, fixed per thread
  uint32_t it_line[ROWS > 0 ? 1 : IPT];
  uint32_t it_xor[ROWS > 0 ? 1 : IPT];
  int it_vb[ROWS > 0 ? 1 : IPT];
  if constexpr (ROWS == 0) {
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int it = tid + k * kThreads;
      const int cb = it < items ? it / n : 0;
      const int r = it < items ? it - cb * n : 0;
      it_line[k] = (uint32_t)((cb * cb_rows + r) * LB);
      it_xor[k] = swz_xor<LB>((uint32_t)r);
      it_vb[k] = cb * E;
    }
  }
  double col_acc = 0.0;

  // pass-1 coordinates: chunk column q (cb, ch), row phase ph; the swizzle
  // XOR of rows ph, ph+P, ... is constant because P is a multiple of 8.
  const int q = tid % QC, ph = tid / QC;
  const int q_cb = q / CPL, q_ch = q % CPL;
  const uint32_t p1_off = (uint32_t)((q_cb * cb_rows + ph) * LB) +
                          ((q_ch ^ swz_xor<LB>((uint32_t)ph)) << 4);

  // ------------------------------------------------------ the two passes
  auto pass1 = [&](const unsigned char* st, double* red) {
    double part[EPC];
    const unsigned char* pa = st + p1_off;
    if constexpr (sizeof(T) == 4) {
      if (mode == MODE_MEAN) {
        float2 sh01 = make_float2(1.0f, 1.0f), sh23 = sh01;
        float2 sc01 = make_float2(0.0f, 0.0f), sc23 = sc01;
#pragma unroll 4
        for (int r = ph; r < n; r += P, pa += P * LB) {
          const float4 v = Vec<float>::loadf(pa);
          fast2sum_acc2(sh01, sc01, make_float2(v.x, v.y));
          fast2sum_acc2(sh23, sc23, make_float2(v.z, v.w));
        }
        part[0] = ((double)sh01.x - 1.0) + (double)sc01.x;
        part[1] = ((double)sh01.y - 1.0) + (double)sc01.y;
        part[2] = ((double)sh23.x - 1.0) + (double)sc23.x;
        part[3] = ((double)sh23.y - 1.0) + (double)sc23.y;
      } else {
#pragma unroll
        for (int e = 0; e < EPC; ++e) part[e] = 0.0;
#pragma unroll 4
        for (int r = ph; r < n; r += P, pa += P * LB) {
          double v[EPC];
          Vec<T>::load(pa, v);
          const double iv = __ldg(p.inv + r);
#pragma unroll
          for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < EPC; ++e) part[e] = 0.0;
#pragma unroll 4
      for (int r = ph; r < n; r += P, pa += P * LB) {
        double v[EPC];
        Vec<T>::load(pa, v);
        const double iv = mode == MODE_MEAN ? 1.0 : __ldg(p.inv + r);
#pragma unroll
        for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
      }
    }
    // combine the row phases inside this warp (lanes sharing q), fixed order
#pragma unroll
    for (int o = QC; o < 32; o <<= 1)
#pragma unroll
      for (int e = 0; e < EPC; ++e) part[e] += __shfl_xor_sync(0xffffffffu, part[e], o);
    if (lane < QC) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) red[warp * V + q * EPC + e] = part[e];
    }
  };

  auto finalize = [&](int64_t j, int buf) {  // threads < V
    const double* rd = red + buf * kWarps * V;
    const int64_t x0 = (blockIdx.x + j * G) * (int64_t)V;
    for (int v = tid; v < V; v += kThreads) {
      const int64_t x = x0 + v;
      const double wx = x < p.m ? (weighted ? __ldg(p.w + x) : 1.0) : 0.0;
      sW[buf * V + v] = wx;
      if (mode != MODE_MASS) {
        double S = 0.0;
#pragma unroll
        for (int k = 0; k < kWarps; ++k) S += rd[k * V + v];
        sS[buf * V + v] = wx * S;
        col_acc = fma(wx, S, col_acc);
      }
    }
  };

  auto pass2 = [&](const unsigned char* st, int buf) {
    const double* S = sS + buf * V;
    const double* W = sW + buf * V;
    if constexpr (ROWS > 0) {
      double s_l[EPL], w_l[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) { s_l[e] = S[r_cell + e]; w_l[e] = W[r_cell + e]; }
      // rows warp, warp+kWarps, ... share r & 7, hence one swizzled lane offset
      const unsigned char* lane_base = st + (uint32_t)((r_cb * cb_rows + warp) * LB) +
                                       ((uint32_t)((r_pos >> 1) ^ (warp & 7)) << 4) +
                                       (uint32_t)((r_pos & 1) * 8);
#define PIDB_ROWS_LOOP(BODY)                                                          \
  _Pragma("unroll") for (int k = 0; k < ROWS; ++k) {                                  \
    if (k < ROWS - 1 || warp + k * kWarps < n) {                                      \
      const unsigned char* a = lane_base + k * (kWarps * LB);                         \
      double v[EPL];                                                                  \
      if constexpr (sizeof(T) == 4) {                                                 \
        const float2 f = *reinterpret_cast<const float2*>(a);                        \
        v[0] = f.x; v[EPL - 1] = f.y;                                                 \
      } else {                                                                        \
        v[0] = *reinterpret_cast<const double*>(a);                                   \
      }                                                                               \
      _Pragma("unroll") for (int e = 0; e < EPL; ++e) { BODY; }                       \
    }                                                                                 \
  }
      if (mode == MODE_MEAN && !weighted) {
        PIDB_ROWS_LOOP(acc_row[k] = fma(v[e], s_l[e], acc_row[k]); acc_mass[k] += v[e])
      } else if (mode == MODE_MASS) {
        PIDB_ROWS_LOOP(acc_mass[k] = fma(v[e], w_l[e], acc_mass[k]); acc_nb[k] += is_nonbinary(v[e]))
      } else if (mode == MODE_COLS) {
        PIDB_ROWS_LOOP(acc_row[k] = fma(v[e], s_l[e], acc_row[k]))
      } else {
        PIDB_ROWS_LOOP(acc_row[k] = fma(v[e], s_l[e], acc_row[k]);
                       acc_mass[k] = fma(v[e], w_l[e], acc_mass[k]))
      }
#undef PIDB_ROWS_LOOP
    } else {
#define PIDB_ITEMS_LOOP(BODY)                                                         \
  _Pragma("unroll") for (int k = 0; k < IPT; ++k) {                                   \
    if (tid + k * kThreads < items) {                                                 \
      const unsigned char* line = st + it_line[k];                                    \
      const double* Sk = S + it_vb[k];                                                \
      const double* Wk = W + it_vb[k];                                                \
      double ar[EPC], am[EPC];                                                        \
      int nb = 0;                                                                     \
      _Pragma("unroll") for (int e = 0; e < EPC; ++e) { ar[e] = 0.0; am[e] = 0.0; }   \
      _Pragma("unroll") for (int L = 0; L < CPL; ++L) {                               \
        double v[EPC];                                                                \
        Vec<T>::load(line + ((L ^ it_xor[k]) << 4), v);                               \
        const int vb = L * EPC;                                                       \
        _Pragma("unroll") for (int e = 0; e < EPC; ++e) { BODY; }                     \
      }                                                                               \
      double tr = ar[0], tm = am[0];                                                  \
      _Pragma("unroll") for (int e = 1; e < EPC; ++e) { tr += ar[e]; tm += am[e]; }   \
      acc_row[k] += tr;                                                               \
      acc_mass[k] += tm;                                                              \
      acc_nb[k] += nb;                                                                \
    }                                                                                 \
  }
      if (mode == MODE_MEAN && !weighted) {
        PIDB_ITEMS_LOOP(ar[e] = fma(v[e], Sk[vb + e], ar[e]); am[e] += v[e])
      } else if (mode == MODE_MASS) {
        PIDB_ITEMS_LOOP(am[e] = fma(v[e], Wk[vb + e], am[e]); nb += is_nonbinary(v[e]))
      } else if (mode == MODE_COLS) {
        PIDB_ITEMS_LOOP(ar[e] = fma(v[e], Sk[vb + e], ar[e]))
      } else {
        PIDB_ITEMS_LOOP(ar[e] = fma(v[e], Sk[vb + e], ar[e]); am[e] = fma(v[e], Wk[vb + e], am[e]))
      }
#undef PIDB_ITEMS_LOOP
    }
  };

  // ------------------------------------------------------ tile loop
  int s_cur = 0;        // stage of tile j
  uint32_t par = 0;     // mbarrier parity of tile j
  int s_prev = 0;       // stage of tile j-1
  if constexpr (ROWS == 0) {
    // Large-N layouts: one resident tile, stages-1 tiles in flight (the
    // memory latency, not the barrier count, is what limits these).
    for (int64_t j = 0; j < my_tiles; ++j) {
      mbar_wait(&full[s_cur], par);
      unsigned char* st = tiles + (size_t)s_cur * p.stage_bytes;
      if (mode != MODE_MASS) pass1(st, red);
      __syncthreads();
      finalize(j, 0);
      __syncthreads();
      pass2(st, 0);
      __syncthreads();
      if (tid == 0 && j + p.stages < my_tiles) issue(j + p.stages);
      if (++s_cur == p.stages) { s_cur = 0; par ^= 1u; }
    }
  } else
  for (int64_t j = 0; j <= my_tiles; ++j) {
    const bool have = j < my_tiles;
    if (have) {
      mbar_wait(&full[s_cur], par);
      if (mode != MODE_MASS)
        pass1(tiles + (size_t)s_cur * p.stage_bytes, red + (j & 1) * kWarps * V);
    }
    __syncthreads();
    // tile j-2's stage was last read by pass 2 in the previous iteration
    if (tid == 0 && j >= 2 && j - 2 + p.stages < my_tiles) issue(j - 2 + p.stages);
    if (have) finalize(j, (int)(j & 1));
    if (j >= 1) pass2(tiles + (size_t)s_prev * p.stage_bytes, (int)((j - 1) & 1));
    s_prev = s_cur;
    if (++s_cur == p.stages) { s_cur = 0; par ^= 1u; }
  }

  // ------------------------------------------------ CTA partials -> global
  // part layout: [grid][p.part_ncb * n][2]
  if constexpr (ROWS > 0) {
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int r = warp + k * kWarps;
      const double a = warp_sum(acc_row[k]);
      const double b = warp_sum(acc_mass[k]);
      int nb = acc_nb[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
      if (lane == 0 && r < n) {
        double* dst = p.part + ((size_t)blockIdx.x * n + r) * 2;
        dst[0] = a;
        dst[1] = b;
        if (p.mode == MODE_MASS && p.part_nb != nullptr) p.part_nb[(size_t)blockIdx.x * n + r] = nb;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int it = tid + k * kThreads;
      if (it < items) {
        double* dst = p.part + ((size_t)blockIdx.x * items + it) * 2;
        dst[0] = acc_row[k];
        dst[1] = acc_mass[k];
      }
    }
    if (p.mode == MODE_MASS && p.part_nb != nullptr) {
      // integers: merge the column boxes of one member exactly, any order
      int64_t* nbp = p.part_nb + (size_t)blockIdx.x * n;
#pragma unroll
      for (int k = 0; k < IPT; ++k) {
        const int it = tid + k * kThreads;
        if (it < n) nbp[it] = acc_nb[k];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < IPT; ++k) {
        const int it = tid + k * kThreads;
        if (it >= n && it < items)
          atomicAdd(reinterpret_cast<unsigned long long*>(&nbp[it % n]),
                    (unsigned long long)acc_nb[k]);
      }
    }
  }
  constexpr int PNCB = ROWS > 0 ? 1 : NCB;
  finish_partials(p, PNCB, col_acc, s_ticket, s_col);
}

// ---------------------------------------------------------------------------
// Large-N variant (n > 256): a tile is V = 2 x 128 B of cells (256 bytes per
// member row, DRAM-friendly) for ALL members, streamed through SMEM in
// 256-row chunks twice: touch 1 (column sweep) from HBM with an L2
// evict_last hint, touch 2 (row sweep) re-reads the same chunks, served by
// L2.  HBM traffic stays one read of the ensemble.  Thread t owns line
// (column box t>>8, row t&255) of every chunk; its row sums for chunk c stay
// in registers (acc[c], c < CMAX).
constexpr int kChunkRows = 256;
constexpr int kChunkBytes = 2 * kChunkRows * 128;  // 64 KB
constexpr int kChunkBufs = 3;

template <typename T, int CMAX>
__global__ void __launch_bounds__(kThreads, 1)
    chunked_pass_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  constexpr int EPC = Vec<T>::EPC;
  constexpr int E = 128 / (int)sizeof(T);  // cells per 128-byte line
  constexpr int V = 2 * E;                 // cells per tile
  constexpr int P = kThreads / 16;         // row phases in touch 1 (16 chunk columns)
  static_assert(kThreads == 2 * kChunkRows, "one (box, row) line per thread");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* bufs = smem_raw + pad;
  unsigned char* tail = bufs + (size_t)kChunkBufs * kChunkBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  double* sS = reinterpret_cast<double*>(tail + 64);
  double* sW = sS + V;
  double* red = sW + V;  // [kWarps][V]
  unsigned* s_ticket = reinterpret_cast<unsigned*>(red + kWarps * V);
  double* s_col = reinterpret_cast<double*>(s_ticket + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = (int)p.n;
  const int G = gridDim.x;
  const int C = (n + kChunkRows - 1) / kChunkRows;
  const int mode = p.mode;
  const bool two_touch = mode != MODE_MASS;
  const int loads_per_tile = two_touch ? 2 * C : C;
  const bool weighted = p.w != nullptr;
  const int64_t my_tiles = p.tiles > blockIdx.x ? (p.tiles - 1 - blockIdx.x) / G + 1 : 0;
  const int64_t total_loads = my_tiles * loads_per_tile;
  const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();

  if (tid == 0) {
    prefetch_tma_desc(&tmap);
    for (int b = 0; b < kChunkBufs; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t q) {  // q-th chunk load of this CTA
    const int b = (int)(q % kChunkBufs);
    const int64_t j = q / loads_per_tile;
    const int i = (int)(q - j * loads_per_tile);
    const bool second = i >= C;
    const int c = second ? i - C : i;
    const int64_t tile = blockIdx.x + j * G;
    unsigned char* dst = bufs + (size_t)b * kChunkBytes;
    mbar_arrive_expect_tx(&full[b], kChunkBytes);
    const uint64_t pol = (two_touch && !second) ? pol_keep : pol_drop;
    for (int cb = 0; cb < 2; ++cb)
      tma_load_2d(dst + cb * (kChunkRows * 128), &tmap, (int32_t)(tile * V + cb * E),
                  c * kChunkRows, &full[b], pol);
  };
  if (tid == 0)
    for (int64_t q = 0; q < total_loads && q < kChunkBufs; ++q) issue(q);

  double acc_row[CMAX], acc_mass[CMAX];
  int acc_nb[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) { acc_row[c] = 0.0; acc_mass[c] = 0.0; acc_nb[c] = 0; }
  double col_acc = 0.0;

  // touch-1 coordinates: chunk column q16 (box, chunk), row phase ph
  const int q16 = tid & 15, ph = tid >> 4;
  const int a_cb = q16 >> 3, a_ch = q16 & 7;
  const uint32_t a_off = (uint32_t)(a_cb * kChunkRows * 128 + ph * 128) +
                         ((uint32_t)(a_ch ^ (ph & 7)) << 4);
  // touch-2 coordinates: this thread's line
  const int b_cb = tid >> 8, b_rr = tid & 255;
  const uint32_t b_off = (uint32_t)(b_cb * kChunkRows * 128 + b_rr * 128);
  const uint32_t b_xor = (uint32_t)(b_rr & 7);

  int64_t q = 0;  // chunk loads consumed so far
  auto next_chunk = [&]() -> const unsigned char* {
    const int b = (int)(q % kChunkBufs);
    mbar_wait(&full[b], (uint32_t)((q / kChunkBufs) & 1));
    return bufs + (size_t)b * kChunkBytes;
  };
  auto release_chunk = [&]() {
    __syncthreads();  // everyone is done with this buffer
    if (tid == 0 && q + kChunkBufs < total_loads) issue(q + kChunkBufs);
    ++q;
  };

  for (int64_t j = 0; j < my_tiles; ++j) {
    const int64_t x0 = (blockIdx.x + j * G) * (int64_t)V;
    // ---------------------------------------------------- touch 1 (columns)
    if (two_touch) {
      double part[EPC];
      float2 sh01 = make_float2(1.0f, 1.0f), sh23 = sh01;
      float2 sc01 = make_float2(0.0f, 0.0f), sc23 = sc01;
#pragma unroll
      for (int e = 0; e < EPC; ++e) part[e] = 0.0;
      for (int c = 0; c < C; ++c) {
        const unsigned char* st = next_chunk();
        const unsigned char* pa = st + a_off;
        if constexpr (sizeof(T) == 4) {
          if (mode == MODE_MEAN) {
#pragma unroll
            for (int k = 0; k < kChunkRows / P; ++k) {
              const float4 v = Vec<float>::loadf(pa + k * (P * 128));
              fast2sum_acc2(sh01, sc01, make_float2(v.x, v.y));
              fast2sum_acc2(sh23, sc23, make_float2(v.z, v.w));
            }
          } else {
#pragma unroll 4
            for (int k = 0; k < kChunkRows / P; ++k) {
              const int r = c * kChunkRows + ph + k * P;
              double v[EPC];
              Vec<T>::load(pa + k * (P * 128), v);
              const double iv = r < n ? __ldg(p.inv + r) : 0.0;
#pragma unroll
              for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
            }
          }
        } else {
#pragma unroll 4
          for (int k = 0; k < kChunkRows / P; ++k) {
            const int r = c * kChunkRows + ph + k * P;
            double v[EPC];
            Vec<T>::load(pa + k * (P * 128), v);
            const double iv = mode == MODE_MEAN ? 1.0 : (r < n ? __ldg(p.inv + r) : 0.0);
#pragma unroll
            for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
          }
        }
        release_chunk();
      }
      if constexpr (sizeof(T) == 4) {
        if (mode == MODE_MEAN) {
          part[0] = ((double)sh01.x - 1.0) + (double)sc01.x;
          part[1] = ((double)sh01.y - 1.0) + (double)sc01.y;
          part[2] = ((double)sh23.x - 1.0) + (double)sc23.x;
          part[3] = ((double)sh23.y - 1.0) + (double)sc23.y;
        }
      }
#pragma unroll
      for (int e = 0; e < EPC; ++e) part[e] += __shfl_xor_sync(0xffffffffu, part[e], 16);
      if (lane < 16) {
#pragma unroll
        for (int e = 0; e < EPC; ++e) red[warp * V + q16 * EPC + e] = part[e];
      }
    }
    __syncthreads();
    for (int v = tid; v < V; v += kThreads) {
      const int64_t x = x0 + v;
      const double wx = x < p.m ? (weighted ? __ldg(p.w + x) : 1.0) : 0.0;
      sW[v] = wx;
      if (two_touch) {
        double S = 0.0;
#pragma unroll
        for (int k = 0; k < kWarps; ++k) S += red[k * V + v];
        sS[v] = wx * S;
        col_acc = fma(wx, S, col_acc);
      }
    }
    __syncthreads();
    // ------------------------------------------------------- touch 2 (rows)
    const double* S = sS + b_cb * E;
    const double* W = sW + b_cb * E;
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
      if (c < C) {
        const unsigned char* line = next_chunk() + b_off;
        if (c * kChunkRows + b_rr < n) {
          double ar[EPC], am[EPC];
          int nb = 0;
#pragma unroll
          for (int e = 0; e < EPC; ++e) { ar[e] = 0.0; am[e] = 0.0; }
#pragma unroll
          for (int L = 0; L < 8; ++L) {
            double v[EPC];
            Vec<T>::load(line + ((L ^ b_xor) << 4), v);
            const int vb = L * EPC;
            if (mode == MODE_MASS) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                am[e] = fma(v[e], W[vb + e], am[e]);
                nb += is_nonbinary(v[e]);
              }
            } else if (mode == MODE_COLS) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) ar[e] = fma(v[e], S[vb + e], ar[e]);
            } else if (weighted) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                ar[e] = fma(v[e], S[vb + e], ar[e]);
                am[e] = fma(v[e], W[vb + e], am[e]);
              }
            } else {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                ar[e] = fma(v[e], S[vb + e], ar[e]);
                am[e] += v[e];
              }
            }
          }
          double tr = ar[0], tm = am[0];
#pragma unroll
          for (int e = 1; e < EPC; ++e) { tr += ar[e]; tm += am[e]; }
          acc_row[c] += tr;
          acc_mass[c] += tm;
          acc_nb[c] += nb;
        }
        release_chunk();
      }
    }
  }

  // ------------------------------------------------ CTA partials -> global
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    const int r = c * kChunkRows + b_rr;
    if (c < C && r < n) {
      double* dst = p.part + ((size_t)blockIdx.x * 2 * n + b_cb * n + r) * 2;
      dst[0] = acc_row[c];
      dst[1] = acc_mass[c];
    }
  }
  if (p.mode == MODE_MASS && p.part_nb != nullptr) {
    int64_t* nbp = p.part_nb + (size_t)blockIdx.x * n;
    if (b_cb == 0) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c) {
        const int r = c * kChunkRows + b_rr;
        if (c < C && r < n) nbp[r] = acc_nb[c];
      }
    }
    __syncthreads();
    if (b_cb == 1) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c) {
        const int r = c * kChunkRows + b_rr;
        if (c < C && r < n)
          atomicAdd(reinterpret_cast<unsigned long long*>(&nbp[r]), (unsigned long long)acc_nb[c]);
      }
    }
  }
  finish_partials(p, 2, col_acc, s_ticket, s_col);
}

// ---------------------------------------------------------------- host side
struct Plan {
  int lb, ncb, ipt, rows, boxr, nrb, stages, grid;
  bool chunked;
  uint32_t stage_bytes;
  size_t smem;
  int64_t tiles;
};

constexpr size_t kSmemBudget = 227 * 1024;

size_t tail_bytes(int V) { return 64 + (size_t)V * 8 * 4 + (size_t)2 * kWarps * V * 8 + 16 + kWarps * 8 + 64; }

constexpr int kChunkMax = 16;  // chunked layout: n <= 4096
bool use_chunked(int64_t n) { return n > 256 && n <= (int64_t)kChunkMax * kChunkRows; }
size_t chunked_smem() {
  return 1024 + (size_t)kChunkBufs * kChunkBytes + 64 + (size_t)(2 + kWarps) * 64 * 8 + 16 +
         kWarps * 8 + 64;
}

bool make_plan(int64_t n, int64_t m, int esize, Plan& pl) {
  if (n < 1 || m < 1) return false;
  pl.chunked = false;
  if (use_chunked(n)) {  // wide tiles, two touches through L2 (see chunked_pass_kernel)
    const int V = 2 * 128 / esize;
    pl.chunked = true;
    pl.lb = 128; pl.ncb = 2; pl.ipt = 1; pl.rows = 0;
    pl.boxr = kChunkRows; pl.nrb = (int)((n + kChunkRows - 1) / kChunkRows);
    pl.stages = kChunkBufs; pl.stage_bytes = kChunkBytes;
    pl.smem = chunked_smem();
    pl.tiles = (m + V - 1) / V;
    pl.grid = (int)std::min<int64_t>(pl.tiles, sm_count());
    return true;
  }
  const int nrb = (int)((n + 255) / 256);
  const int boxr_full = (int)(((n + nrb - 1) / nrb + 7) / 8 * 8);
  const int rows = nrb * boxr_full;
  struct Cand { int lb, ncb; };
  const Cand cands[] = {{128, 2}, {128, 1}, {64, 1}, {32, 1}};
  for (const Cand& c : cands) {
    const int V = c.ncb * c.lb / esize;
    const uint32_t sb = (uint32_t)(c.ncb * rows * c.lb);
    const size_t tb = tail_bytes(V) + 1024;
    const int min_stages = 3;  // tiles j (pass 1), j-1 (pass 2) and >= 1 in flight
    int stages = (int)std::min<size_t>(8, (kSmemBudget - tb) / sb);
    if (sb > kSmemBudget || stages < min_stages) continue;
    const int64_t items = (int64_t)c.ncb * n;
    int ipt = 1;
    while ((int64_t)ipt * kThreads < items) ipt *= 2;
    if (ipt > (c.lb == 128 ? 2 : (c.lb == 64 ? 4 : 8))) continue;
    int rows_per_warp = 0;  // row-resident pass 2 for 2x128B-line tiles
    if (c.lb == 128 && c.ncb == 2) {
      rows_per_warp = (int)((n + kWarps - 1) / kWarps);
      if (rows_per_warp > 16) rows_per_warp = 0;
    }
    pl.lb = c.lb; pl.ncb = c.ncb; pl.ipt = ipt; pl.rows = rows_per_warp;
    pl.boxr = boxr_full; pl.nrb = nrb;
    pl.stages = stages; pl.stage_bytes = sb;
    pl.smem = (size_t)stages * sb + tb;
    pl.tiles = (m + V - 1) / V;
    pl.grid = (int)std::min<int64_t>(pl.tiles, sm_count());
    return true;
  }
  return false;
}

size_t workspace_bytes(const Plan& pl, int64_t n) {
  const int64_t items = (int64_t)pl.ncb * n;
  size_t b = 256;  // completion counter: fixed offset 0, zero between launches
  b += align_up((size_t)pl.grid * items * 2 * sizeof(double), 256);
  b += align_up((size_t)pl.grid * sizeof(double), 256);
  b += align_up((size_t)pl.grid * n * sizeof(int64_t), 256);
  return b;
}

template <typename T, int LB, int NCB, int IPT, int ROWS>
int launch_t(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  auto kern = stream_pass_kernel<T, LB, NCB, IPT, ROWS>;
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  kern<<<pl.grid, kThreads, pl.smem, st>>>(tm, sp);
  PIDB_LAUNCH_CHECK("stream_pass_kernel");
  return PIDB_OK;
}

template <typename T, int LB, int NCB>
int launch_ipt(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  // only the (layout, items-per-thread) pairs make_plan can produce are built
  if constexpr (LB == 128 && NCB == 2) {
    switch (pl.rows) {
#define PIDB_ROWS_CASE(R) case R: return launch_t<T, LB, NCB, 1, R>(tm, sp, pl, st);
      PIDB_ROWS_CASE(1) PIDB_ROWS_CASE(2) PIDB_ROWS_CASE(3) PIDB_ROWS_CASE(4)
      PIDB_ROWS_CASE(5) PIDB_ROWS_CASE(6) PIDB_ROWS_CASE(7) PIDB_ROWS_CASE(8)
      PIDB_ROWS_CASE(9) PIDB_ROWS_CASE(10) PIDB_ROWS_CASE(11) PIDB_ROWS_CASE(12)
      PIDB_ROWS_CASE(13) PIDB_ROWS_CASE(14) PIDB_ROWS_CASE(15) PIDB_ROWS_CASE(16)
#undef PIDB_ROWS_CASE
    }
  }
  constexpr int kMaxIpt = LB == 128 ? 2 : (LB == 64 ? 4 : 8);
  switch (pl.ipt) {
    case 1: return launch_t<T, LB, NCB, 1, 0>(tm, sp, pl, st);
    case 2: return launch_t<T, LB, NCB, 2, 0>(tm, sp, pl, st);
    case 4: if constexpr (kMaxIpt >= 4) return launch_t<T, LB, NCB, 4, 0>(tm, sp, pl, st); break;
    case 8: if constexpr (kMaxIpt >= 8) return launch_t<T, LB, NCB, 8, 0>(tm, sp, pl, st); break;
  }
  set_error("unsupported items-per-thread %d for %d-byte lines", pl.ipt, LB);
  return PIDB_EUNSUPPORTED;
}

template <typename T>
int launch_layout(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  if (pl.lb == 128 && pl.ncb == 2) return launch_ipt<T, 128, 2>(tm, sp, pl, st);
  if (pl.lb == 128 && pl.ncb == 1) return launch_ipt<T, 128, 1>(tm, sp, pl, st);
  if (pl.lb == 64) return launch_ipt<T, 64, 1>(tm, sp, pl, st);
  return launch_ipt<T, 32, 1>(tm, sp, pl, st);
}

template <typename T, int CMAX>
int launch_chunked_t(const CUtensorMap& tm, StreamParams& sp, int grid, cudaStream_t st) {
  auto kern = chunked_pass_kernel<T, CMAX>;
  const size_t smem = chunked_smem();
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kThreads, smem, st>>>(tm, sp);
  PIDB_LAUNCH_CHECK("chunked_pass_kernel");
  return PIDB_OK;
}

template <typename T>
int launch_chunked(const CUtensorMap& tm, StreamParams& sp, int grid, cudaStream_t st) {
  const int C = (int)((sp.n + kChunkRows - 1) / kChunkRows);
  if (C <= 4) return launch_chunked_t<T, 4>(tm, sp, grid, st);
  if (C <= 8) return launch_chunked_t<T, 8>(tm, sp, grid, st);
  return launch_chunked_t<T, 16>(tm, sp, grid, st);
}

int run_stream_pass(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                    const double* w, const double* inv, double* out_row, double* out_mass,
                    double* out_col, int64_t* out_nb, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u != nullptr, "member matrix is NULL");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  PIDB_REQUIRE(n >= 1 && m >= 1, "need n >= 1 members and m >= 1 cells (got %lld, %lld)",
               (long long)n, (long long)m);
  const int es = dtype == PIDB_F32 ? 4 : 8;
  PIDB_REQUIRE(ld >= m && (ld * es) % 16 == 0, "row stride %lld must be >= m and a multiple of 16 bytes",
               (long long)ld);
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(u) & 15) == 0, "member matrix must be 16-byte aligned");
  PIDB_REQUIRE(n <= INT32_MAX, "too many members");
  Plan pl;
  if (!make_plan(n, m, es, pl)) {
    set_error("ensemble with %lld members does not fit the single-pass tile layout", (long long)n);
    return PIDB_EUNSUPPORTED;
  }
  const size_t need = workspace_bytes(pl, n);
  if (ws == nullptr || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return PIDB_EWORKSPACE;
  }
  CUtensorMap tm;
  int rc = encode_tma_2d(&tm, u, dtype == PIDB_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                     : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                         (uint64_t)m, (uint64_t)n, (uint64_t)ld * es, (uint32_t)(pl.lb / es),
                         (uint32_t)pl.boxr,
                         pl.lb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                      : (pl.lb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                     : CU_TENSOR_MAP_SWIZZLE_32B));
  if (rc != PIDB_OK) return rc;
  const int64_t items = (int64_t)pl.ncb * n;
  char* base = static_cast<char*>(ws);
  StreamParams sp{};
  sp.counter = reinterpret_cast<unsigned*>(base);
  base += 256;
  sp.n = n; sp.m = m; sp.tiles = pl.tiles; sp.nrb = pl.nrb; sp.boxr = pl.boxr;
  sp.stages = pl.stages; sp.stage_bytes = pl.stage_bytes; sp.mode = mode;
  sp.w = w; sp.inv = inv;
  sp.part = reinterpret_cast<double*>(base);
  base += align_up((size_t)pl.grid * items * 2 * sizeof(double), 256);
  sp.part_col = reinterpret_cast<double*>(base);
  base += align_up((size_t)pl.grid * sizeof(double), 256);
  sp.part_nb = out_nb ? reinterpret_cast<int64_t*>(base) : nullptr;
  base += align_up((size_t)pl.grid * n * sizeof(int64_t), 256);
  sp.out_row = out_row; sp.out_mass = out_mass; sp.out_col = out_col; sp.out_nb = out_nb;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pl.chunked)
    return dtype == PIDB_F32 ? launch_chunked<float>(tm, sp, pl.grid, st)
                             : launch_chunked<double>(tm, sp, pl.grid, st);
  return dtype == PIDB_F32 ? launch_layout<float>(tm, sp, pl, st)
                           : launch_layout<double>(tm, sp, pl, st);
}

}  // namespace

size_t stream_pass_workspace(int64_t n, int64_t m, int dtype) {
  Plan pl;
  if (!make_plan(n, m, dtype == PIDB_F32 ? 4 : 8, pl)) return 0;
  return workspace_bytes(pl, n);
}

}  // namespace pidb

extern "C" size_t pidb_pid_mean_workspace_bytes(int64_t n, int64_t m, int dtype) {
  return pidb::stream_pass_workspace(n, m, dtype);
}

extern "C" int pidb_pid_mean_partials(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                                      const double* w, double* row_plain, double* mass,
                                      double* col_mean, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(row_plain && mass && col_mean, "output pointers must be non-NULL");
  return pidb::run_stream_pass(pidb::MODE_MEAN, u, dtype, n, m, ld, w, nullptr, row_plain, mass,
                               col_mean, nullptr, ws, ws_bytes, stream);
}

extern "C" int pidb_pid_colsums(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                                const double* w, const double* inv, double* col_inv, void* ws,
                                size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(inv && col_inv, "inv/col_inv must be non-NULL");
  return pidb::run_stream_pass(pidb::MODE_COLS, u, dtype, n, m, ld, w, inv, col_inv, nullptr,
                               nullptr, nullptr, ws, ws_bytes, stream);
}

extern "C" int pidb_member_masses(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                                  const double* w, double* mass, int64_t* nonbinary, void* ws,
                                  size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(mass, "mass must be non-NULL");
  return pidb::run_stream_pass(pidb::MODE_MASS, u, dtype, n, m, ld, w, nullptr, nullptr, mass,
                               nullptr, nonbinary, ws, ws_bytes, stream);
}
