// Shared by the streaming translation units (stream_pass.cu, stream_ws_f32.cu,
// stream_ws_f64.cu): parameters, plans, the column sweep, the CTA reductions
// and the warp-specialised rows kernel (see stream_pass.cu for the design).
#pragma once
#include <cstdlib>

#include "common.cuh"

namespace pidb {
namespace stream {  // types shared across translation units

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kRowBytes = 256;          // bytes of one member row per tile
constexpr int kChunks16 = kRowBytes / 16;
constexpr int kPhases = kThreads / kChunks16;  // row phases of the column sweep
// block size of the rows kernels (640 threads was measured 11% slower on
// cfg5: the 96-register budget costs more than the extra warps bring)
constexpr int kRowsThreads = 512;
constexpr int kRowsWarps = kRowsThreads / 32;
constexpr int MODE_MEAN = 0;
constexpr int MODE_COLS = 1;
constexpr int MODE_MASS = 2;  // masses (+ non-binary count): row sweep only
constexpr int MODE_SIM = 3;   // similarity baselines: sum w*min(u, mean), masses


struct StreamParams {
  int64_t n, m, tiles;
  int stages;
  int cs, rpc;           // cluster size and member rows per CTA (cluster rows kernel)
  int groups;            // row-partial groups reduced by finish_partials
  uint32_t stage_bytes;  // bytes of one tile (rows kernel) or chunk (chunked)
  int mode;
  const double* w;       // nullable
  const double* inv;     // MODE_COLS
  const double* fvec;    // ext row sweep: per-cell f (w*S, w*T or the mean), else null
  double* part;          // [grid][pncb * n][2]
  double* part_col;      // [grid]
  int64_t* part_nb;      // [grid][n] (MODE_MASS, nullable)
  unsigned* counter;
  double* out_row;       // n
  double* out_mass;      // n (nullable in MODE_COLS)
  double* out_col;       // 1 (MODE_MEAN)
  int64_t* out_nb;       // n (MODE_MASS, nullable)
};

constexpr size_t kSmemBudget = 227 * 1024;
constexpr int kMaxStages = 8;
constexpr int kChunkMax = 16;  // n <= 4096

struct Plan {
  bool chunked;
  bool ext;     // wide ensembles: row sweep against a precomputed f, row slices per CTA
  int cs, rpc;  // cs > 1: cluster rows kernel
  int rows, stages, grid, box_rows;
  uint32_t stage_bytes;
  size_t smem;
  int64_t tiles;
  int rb = kRowBytes;  // bytes of a member row per tile (512: wide rows, fp32 n <= ~210)
};

// warp-specialised kernels, one translation unit per element type;
// return kNotHandled when no instantiation fits the plan
constexpr int kNotHandled = 1;
int launch_ws_f32(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st);
int launch_ws_f64(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st);

}  // namespace stream

namespace {  // device code, instantiated per translation unit
using namespace stream;

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

// Column sweep over RB-byte rows: this thread's 16-byte chunk of rows
// r0, r0 + kPh, ... < r_end, starting at `pa`.  fp32 MODE_MEAN uses the
// Fast2Sum state; otherwise part[] += iv(row) * u in fp64.
template <typename T, int NT = kThreads, int RB = kRowBytes>
struct ColSweep {
  static constexpr int kCh = RB / 16;        // 16-byte chunks per row
  static constexpr int kPh = NT / kCh;       // row phases
  static constexpr int EPC = Vec<T>::EPC;
  float2 sh01, sh23, sc01, sc23;
  double part[EPC];
  __device__ void reset() {
    sh01 = sh23 = make_float2(1.0f, 1.0f);
    sc01 = sc23 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int e = 0; e < EPC; ++e) part[e] = 0.0;
  }
  // rg: global member index of row r0 (for inv); rows >= n contribute 0
  __device__ void run(const unsigned char* pa, int r0, int r_end, int mode, const double* inv,
                      int rg, int n) {
    if constexpr (sizeof(T) == 4) {
      if (mode == MODE_MEAN) {
#pragma unroll 4
        for (int r = r0; r < r_end; r += kPh, pa += kPh * RB) {
          const float4 v = Vec<float>::loadf(pa);
          fast2sum_acc2(sh01, sc01, make_float2(v.x, v.y));
          fast2sum_acc2(sh23, sc23, make_float2(v.z, v.w));
        }
        return;
      }
    }
#pragma unroll 4
    for (int r = r0; r < r_end; r += kPh, rg += kPh, pa += kPh * RB) {
      double v[EPC];
      Vec<T>::load(pa, v);
      const double iv = mode == MODE_MEAN ? 1.0 : (rg < n ? __ldg(inv + rg) : 0.0);
#pragma unroll
      for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
    }
  }
  // fold the Fast2Sum state into part[] and, for 256-byte rows, combine the
  // warp's two row phases (lanes l and l^16 share a chunk; lanes < 16 hold
  // the result); with 512-byte rows a warp is one phase, every lane a chunk
  __device__ void combine(int mode) {
    if constexpr (sizeof(T) == 4) {
      if (mode == MODE_MEAN) {
        part[0] = ((double)sh01.x - 1.0) + (double)sc01.x;
        part[1] = ((double)sh01.y - 1.0) + (double)sc01.y;
        part[2] = ((double)sh23.x - 1.0) + (double)sc23.x;
        part[3] = ((double)sh23.y - 1.0) + (double)sc23.y;
      }
    }
    if constexpr (kCh < 32) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) part[e] += __shfl_xor_sync(0xffffffffu, part[e], 16);
    }
  }
};

// Row partials are stored member-major, part[r][cb][g] (g = partial group),
// so that the reduction below reads each member's groups with coalesced loads.
__device__ __forceinline__ size_t part_at(const StreamParams& p, int pncb, int cb, int64_t r,
                                          int g) {
  return ((size_t)r * pncb + cb) * p.groups + g;
}

// CTA column partial -> global; the last CTA to finish reduces every CTA's
// partials in a fixed order (grid, then half) and resets the counter.
template <int NT>
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
      for (int k = 0; k < (NT / 32); ++k) t += s_col[k];
      p.part_col[blockIdx.x] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) *s_ticket = atomicAdd(p.counter, 1u);
  __syncthreads();
  if (*s_ticket != (unsigned)(G - 1)) return;

  __threadfence();
  // Every partial load of a round is issued before the first add (kFR rows
  // x kFG groups per lane): this tail runs on one SM; group-major partials
  // read one 16-byte word per line cost ~75 us at n = 200.
  constexpr int kFR = 1, kFG = 5;
  const bool want_nb = p.mode == MODE_MASS && p.part_nb != nullptr;
  for (int r0 = warp * kFR; r0 < n; r0 += (NT / 32) * kFR) {
    double a[kFR], b[kFR];
    int64_t nb[kFR];
#pragma unroll
    for (int j = 0; j < kFR; ++j) { a[j] = 0.0; b[j] = 0.0; nb[j] = 0; }
    for (int g0 = 0; g0 < p.groups; g0 += 32 * kFG) {
      for (int cb = 0; cb < pncb; ++cb) {
        double2 v[kFR][kFG];
#pragma unroll
        for (int j = 0; j < kFR; ++j)
#pragma unroll
          for (int q = 0; q < kFG; ++q) {
            const int g = g0 + q * 32 + lane, r = r0 + j;
            v[j][q] = make_double2(0.0, 0.0);
            if (g < p.groups && r < n)
              v[j][q] = __ldcg(reinterpret_cast<const double2*>(p.part + part_at(p, pncb, cb, r, g) * 2));
          }
#pragma unroll
        for (int j = 0; j < kFR; ++j)
#pragma unroll
          for (int q = 0; q < kFG; ++q) {
            a[j] += v[j][q].x;
            b[j] += v[j][q].y;
          }
      }
      if (want_nb) {
        long long v[kFR][kFG];
#pragma unroll
        for (int j = 0; j < kFR; ++j)
#pragma unroll
          for (int q = 0; q < kFG; ++q) {
            const int g = g0 + q * 32 + lane, r = r0 + j;
            v[j][q] = (g < p.groups && r < n)
                          ? __ldcg(reinterpret_cast<const long long*>(p.part_nb + part_at(p, 1, 0, r, g)))
                          : 0ll;
          }
#pragma unroll
        for (int j = 0; j < kFR; ++j)
#pragma unroll
          for (int q = 0; q < kFG; ++q) nb[j] += (int64_t)v[j][q];
      }
    }
#pragma unroll
    for (int j = 0; j < kFR; ++j) {
      const int r = r0 + j;
      const double aj = warp_sum(a[j]);
      const double bj = warp_sum(b[j]);
      int64_t nj = nb[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nj += __shfl_xor_sync(0xffffffffu, nj, o);
      if (lane == 0 && r < n) {
        if (p.mode == MODE_MASS) {
          p.out_mass[r] = bj;
          if (p.out_nb) p.out_nb[r] = nj;
        } else {
          p.out_row[r] = aj;
          if (p.out_mass) p.out_mass[r] = bj;
        }
      }
    }
  }
  if (warp == 0 && (p.mode == MODE_MEAN || p.mode == MODE_SIM)) {
    double c = 0.0;
    for (int g = lane; g < G; g += 32) c += __ldcg(p.part_col + g);
    c = warp_sum(c);
    if (lane == 0) p.out_col[0] = c;
  }
  if (tid == 0) *p.counter = 0u;  // ready for the next launch on this workspace
}

// sS/sW for tile cells [x0, x0+V): w*S (or w*T) and w; col_acc += w*S.
// EPC_PERM > 0 stores cell (8 chunks of EPC per half row) at the
// element-major slot half*V/2 + e*8 + chunk, which makes the chunked
// kernel's row-rotated reads bank-conflict free.
template <int V, int EPC_PERM, int NT = kThreads>
__device__ __forceinline__ void finalize_tile(const StreamParams& p, const double* rd, int64_t x0,
                                              double* sS, double* sW, bool colsum,
                                              double& col_acc) {
  for (int v = threadIdx.x; v < V; v += NT) {
    const int64_t x = x0 + v;
    const double wx = x < p.m ? (p.w ? __ldg(p.w + x) : 1.0) : 0.0;
    int slot = v;
    if constexpr (EPC_PERM > 0) {
      const int half = v / (V / 2), hv = v % (V / 2);
      slot = half * (V / 2) + (hv % EPC_PERM) * 8 + hv / EPC_PERM;
    }
    sW[slot] = wx;
    if (colsum) {
      double S = 0.0;
#pragma unroll
      for (int k = 0; k < NT / 32; ++k) S += rd[k * V + v];
      // MODE_SIM keeps the mean mask value (mean_mask, grid.py:251-261)
      sS[slot] = p.mode == MODE_SIM ? __ddiv_rn(S, (double)p.n) : wx * S;
      col_acc = fma(wx, S, col_acc);
    }
  }
}

// ---------------------------------------------------------------------------
// rows_ws_kernel: warp-specialised variant of rows_kernel for fp32, n <= 256.
// Warps 0-3 (column group) run pass 1 and the S finalisation of tile j while
// warps 4-15 (row group) run pass 2 of an earlier tile; the groups hand S over
// through double-buffered sS/sW and named barriers (no CTA-wide barrier per
// tile).  ROWS = ceil(n / 12) rows per row warp; MODE is a template argument
// so only the accumulators of that mode are live.
// Column-group size per mode: pass 1 is cheap packed-fp32 Fast2Sum for the
// mean (S) and costs an fp64 conversion + FMA per element for T (MODE_COLS).
__host__ __device__ constexpr int ws_col_warps(int mode) { return mode == MODE_COLS ? 8 : 4; }
constexpr int kBarCols = 1, kBarSReady = 2, kBarSFree = 4, kBarRows = 6;  // named barriers

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <typename T, int ROWS, int MODE, bool CL, int RB = kRowBytes>
__global__ void __launch_bounds__(kRowsThreads, 1)
    rows_ws_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  static_assert(RB == kRowBytes || !CL, "wide rows: single-CTA kernel only");
  constexpr int kWsColWarps = ws_col_warps(MODE);
  constexpr int kWsColThreads = kWsColWarps * 32;
  constexpr int kWsRowWarps = kRowsWarps - kWsColWarps;
  constexpr int kWsRowThreads = kWsRowWarps * 32;
  constexpr int EPC = Vec<T>::EPC;
  constexpr int V = RB / (int)sizeof(T);
  constexpr int EPL = RB / 32 / (int)sizeof(T);  // cells per lane per row (row group)
  constexpr int kCh = RB / 16;
  constexpr int kAll = kWsColThreads + kWsRowThreads;
  constexpr int SWEEP = MODE == MODE_SIM ? MODE_MEAN : MODE;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* tiles = smem_raw + pad;
  unsigned char* tail = tiles + (size_t)p.stages * p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* xbar = reinterpret_cast<uint64_t*>(tail + 64);  // [4] (CL)
  double* sS = reinterpret_cast<double*>(tail + 128);       // [2][V]
  double* sW = sS + 2 * V;                                   // [2][V]
  double* red = sW + 2 * V;                                  // [kWsColWarps][V]
  unsigned* s_ticket = reinterpret_cast<unsigned*>(red + kWsColWarps * V);
  double* s_col = reinterpret_cast<double*>(s_ticket + 2);
  const uint32_t xoff =
      ((smem_u32(s_col + kRowsWarps) + 15u) & ~15u) - smem_u32(smem_raw);
  double* xbuf = reinterpret_cast<double*>(smem_raw + xoff);  // [4][cs][V] (CL)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = (int)p.n;
  const bool weighted = p.w != nullptr;
  // ext (wide ensembles, not CL): f is given, CTA b of a group of p.cs takes
  // member rows [b * rpc, (b + 1) * rpc) of its tiles; no column sweep
  const bool ext = !CL && p.fvec != nullptr;
  const bool sliced = CL || ext;
  const int cs = sliced ? p.cs : 1;
  const uint32_t rank = CL ? cluster_rank() : (ext ? blockIdx.x % (unsigned)cs : 0u);
  const int cid = (int)blockIdx.x / cs, ncl = (int)gridDim.x / cs;
  const int r0 = sliced ? (int)rank * p.rpc : 0;
  const int box = sliced ? p.rpc : n;                        // member rows per TMA box
  const int nloc = sliced ? max(0, min(n - r0, p.rpc)) : n;  // member rows of this CTA
  const int64_t my_tiles = p.tiles > cid ? (p.tiles - 1 - cid) / ncl + 1 : 0;
  const uint64_t pol = policy_evict_first();
  const uint32_t xbytes = (uint32_t)cs * V * 8u;

  if (tid == 0) {
    prefetch_tma_desc(&tmap);
    for (int s = 0; s < p.stages; ++s) mbar_init(&full[s], 1);
    if (CL)
      for (int s = 0; s < 4; ++s) mbar_init(&xbar[s], 1);
    fence_mbar_init();
    if (CL)
      for (int s = 0; s < 4 && s < my_tiles; ++s) mbar_arrive_expect_tx(&xbar[s], xbytes);
  }
  __syncthreads();
  if constexpr (CL) cluster_sync();  // peers' mbarriers exist before any st.async
  auto issue = [&](int64_t j) {
    const int s = (int)(j % p.stages);
    mbar_arrive_expect_tx(&full[s], (uint32_t)box * RB);
    tma_load_2d(tiles + (size_t)s * p.stage_bytes, &tmap, (int32_t)((cid + j * ncl) * V), r0,
                &full[s], pol);
  };
  if (tid == 0)
    for (int64_t j = 0; j < my_tiles && j < p.stages; ++j) issue(j);

  double col_acc = 0.0;
  double acc_row[ROWS], acc_mass[ROWS];
#pragma unroll
  for (int k = 0; k < ROWS; ++k) { acc_row[k] = 0.0; acc_mass[k] = 0.0; }

  if (warp < kWsColWarps) {
    // ---------------------------------------------------------- column group
    const int q = tid & (kCh - 1), ph = tid / kCh;
    const uint32_t p1_off = (uint32_t)(ph * RB + q * 16);
    ColSweep<T, kWsColThreads, RB> csw;
    int s = 0;
    uint32_t par = 0;
    for (int64_t j = 0; j < my_tiles; ++j) {
      const int b = (int)(j & 1);
      const int64_t x0 = (cid + j * ncl) * (int64_t)V;
      double wx = 0.0;
      if (tid < V) {
        const int64_t x = x0 + tid;
        wx = x < p.m ? (weighted ? __ldg(p.w + x) : 1.0) : 0.0;
      }
      double S = 0.0;
      if (ext) {
        if (tid < V) {
          const int64_t x = x0 + tid;
          S = x < p.m ? __ldg(p.fvec + x) : 0.0;
        }
      } else {
        mbar_wait(&full[s], par);
        csw.reset();
        csw.run(tiles + (size_t)s * p.stage_bytes + p1_off, ph, box, SWEEP, p.inv, r0 + ph, n);
        csw.combine(SWEEP);
        if (kCh == 32 || lane < 16) {
#pragma unroll
          for (int e = 0; e < EPC; ++e) red[warp * V + q * EPC + e] = csw.part[e];
        }
        named_sync(kBarCols, kWsColThreads);
        if (tid < V) {
#pragma unroll
          for (int k = 0; k < kWsColWarps; ++k) S += red[k * V + tid];
        }
      }
      // the row group has read sS/sW[b] (and, CL, xbuf slot of tile j-2)
      named_sync(kBarSFree + b, kAll);
      if constexpr (CL) {
        // CTA partial of column S -> every CTA of the cluster (16-byte st.async
        // completing on the receiver's mbarrier); rank order is kept by slot
        const double S1 = __shfl_down_sync(0xffffffffu, S, 1);
        if (tid < V && (tid & 1) == 0) {
          const int slot = (int)(j & 3);
          const uint32_t la = smem_u32(xbuf + ((size_t)slot * cs + rank) * V + tid);
          const uint32_t lb = smem_u32(&xbar[slot]);
          for (int c = 0; c < cs; ++c) st_async_f64x2(mapa(la, c), S, S1, mapa(lb, c));
        }
        if (tid < V) sW[b * V + tid] = wx;
      } else if (ext) {
        // S holds f: w*S (MEAN), w*T (COLS) or the mean S/n (SIM); the column
        // total sum_x w S is taken once per tile (row block 0)
        if (tid < V) {
          sW[b * V + tid] = wx;
          sS[b * V + tid] = S;
          if (rank == 0) col_acc += MODE == MODE_SIM ? wx * S * (double)p.n : S;
        }
      } else {
        if (tid < V) {
          sW[b * V + tid] = wx;
          sS[b * V + tid] = MODE == MODE_SIM ? __ddiv_rn(S, (double)p.n) : wx * S;
          col_acc = fma(wx, S, col_acc);
        }
      }
      named_arrive(kBarSReady + b, kAll);
      if (++s == p.stages) { s = 0; par ^= 1u; }
    }
  } else {
    // ------------------------------------------------------------- row group
    const int rw = warp - kWsColWarps;
    const uint32_t p2_off = (uint32_t)(rw * RB + lane * (RB / 32));
    const int cell = lane * EPL;
    named_arrive(kBarSFree + 0, kAll);  // both S buffers start free
    named_arrive(kBarSFree + 1, kAll);
    int s = 0;
    uint32_t rpar = 0;
    for (int64_t j = 0; j < my_tiles; ++j) {
      const int b = (int)(j & 1);
      named_sync(kBarSReady + b, kAll);
      if (ext) mbar_wait(&full[s], rpar);  // no column sweep has waited on the stage
      double s_l[EPL], w_l[EPL];
      if constexpr (CL) {
        const int slot = (int)(j & 3);
        mbar_wait(&xbar[slot], (uint32_t)((j >> 2) & 1));
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          double S = 0.0;
          for (int c = 0; c < cs; ++c) S += xbuf[((size_t)slot * cs + c) * V + cell + e];
          w_l[e] = sW[b * V + cell + e];
          s_l[e] = MODE == MODE_SIM ? __ddiv_rn(S, (double)p.n) : w_l[e] * S;
          if (rank == 0 && rw == 0) col_acc = fma(w_l[e], S, col_acc);
        }
      } else {
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          s_l[e] = sS[b * V + cell + e];
          w_l[e] = sW[b * V + cell + e];
        }
      }
      named_arrive(kBarSFree + b, kAll);
      const unsigned char* base = tiles + (size_t)s * p.stage_bytes + p2_off;
      // SIM: min(u, mean) with u fp32 decided in fp32 (u <= mean exactly when
      // u <= the largest float <= mean), saving the fp64 min per element
      float md[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) md[e] = MODE == MODE_SIM ? __double2float_rd(s_l[e]) : 0.f;
#pragma unroll
      for (int k = 0; k < ROWS; ++k) {
        if (k < ROWS - 1 || rw + k * kWsRowWarps < nloc) {
          const unsigned char* a = base + k * (kWsRowWarps * RB);
          float fv[EPL];
          double v[EPL];
          if constexpr (sizeof(T) == 4 && EPL == 4) {
            const float4 f = *reinterpret_cast<const float4*>(a);
            fv[0] = f.x; fv[1] = f.y; fv[2] = f.z; fv[3] = f.w;
#pragma unroll
            for (int e = 0; e < EPL; ++e) v[e] = fv[e];
          } else if constexpr (sizeof(T) == 4) {
            const float2 f = *reinterpret_cast<const float2*>(a);
            fv[0] = f.x; fv[EPL - 1] = f.y;
            v[0] = f.x; v[EPL - 1] = f.y;
          } else if constexpr (EPL == 2) {
            const double2 f = *reinterpret_cast<const double2*>(a);
            v[0] = f.x; v[1] = f.y;
            fv[0] = fv[1] = 0.f;
          } else {
            v[0] = *reinterpret_cast<const double*>(a);
            fv[0] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            if (MODE == MODE_SIM) {
              const double mn = sizeof(T) == 4 ? (fv[e] <= md[e] ? v[e] : s_l[e])
                                               : fmin(v[e], s_l[e]);
              acc_row[k] = fma(mn, w_l[e], acc_row[k]);
              acc_mass[k] = weighted ? fma(v[e], w_l[e], acc_mass[k]) : acc_mass[k] + v[e];
            } else if (MODE == MODE_COLS) {
              acc_row[k] = fma(v[e], s_l[e], acc_row[k]);
            } else {
              acc_row[k] = fma(v[e], s_l[e], acc_row[k]);
              acc_mass[k] = weighted ? fma(v[e], w_l[e], acc_mass[k]) : acc_mass[k] + v[e];
            }
          }
        }
      }
      named_sync(kBarRows, kWsRowThreads);  // every row warp is done with stage s
      if (rw == 0 && lane == 0) {
        if (j + p.stages < my_tiles) issue(j + p.stages);
        // every row thread passed its xbar wait for tile j: re-arm for tile j+4
        if (CL && j + 4 < my_tiles) mbar_arrive_expect_tx(&xbar[j & 3], xbytes);
      }
      if (++s == p.stages) { s = 0; rpar ^= 1u; }
    }
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int rl = rw + k * kWsRowWarps;
      const double a = warp_sum(acc_row[k]);
      const double c = warp_sum(acc_mass[k]);
      if (lane == 0 && rl < nloc) {
        PIDB_DCHECK(r0 + rl < n && cid < p.groups, "K5 row partial bounds");
        double* dst = p.part + part_at(p, 1, 0, r0 + rl, cid) * 2;
        dst[0] = a;
        dst[1] = c;
      }
    }
  }
  __syncthreads();
  if constexpr (CL) cluster_sync();  // no CTA leaves while peers may still target its SMEM
  finish_partials<kRowsThreads>(p, 1, col_acc, s_ticket, s_col);
}

template <typename K>
int launch(K kern, const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  kern<<<pl.grid, pl.chunked ? kThreads : kRowsThreads, pl.smem, st>>>(tm, sp);
  PIDB_LAUNCH_CHECK("stream kernel");
  return PIDB_OK;
}

// cluster launch; grid = co-resident clusters (persistent) x cs
template <typename K>
int launch_cluster(K kern, const CUtensorMap& tm, StreamParams& sp, const Plan& pl,
                   cudaStream_t st) {
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  if (pl.cs > 8) PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kRowsThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(pl.grid / pl.cs * pl.cs));
  int active = 0;
  PIDB_CUDA(cudaOccupancyMaxActiveClusters(&active, kern, &cfg));
  if (std::getenv("PIDB_TEST_NO_CLUSTER")) active = 0;  // test hook: exercise the fallback
  if (active < 1) {
    set_error("no co-resident cluster of %d CTAs for the streaming kernel", pl.cs);
    return PIDB_EUNSUPPORTED;
  }
  const int64_t ncl = std::min<int64_t>(std::min<int64_t>(active, pl.grid / pl.cs), sp.tiles);
  cfg.gridDim = dim3((unsigned)(ncl * pl.cs));
  if (std::getenv("PIDB_DEBUG"))
    std::fprintf(stderr, "pidb: cluster %d x %lld CTAs (active %d), rpc %d, stages %d, smem %zu\n",
                 pl.cs, (long long)ncl, active, pl.rpc, pl.stages, pl.smem);
  sp.groups = (int)ncl;
  PIDB_CUDA(cudaLaunchKernelEx(&cfg, kern, tm, sp));
  PIDB_LAUNCH_CHECK("cluster stream kernel");
  return PIDB_OK;
}

// Warp-specialised dispatch for one element type: cluster (pl.cs > 1) or
// single-CTA (n <= 256) variants, by mode and rows per row warp.
template <typename T>
int launch_ws(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  const int rw = kRowsWarps - ws_col_warps(sp.mode);
  if (pl.cs > 1 && !pl.ext) {
    const int rows = (pl.rpc + rw - 1) / rw;
    switch (sp.mode * 64 + rows) {
#define PIDB_WSC_CASE(M, R) \
  case M * 64 + R: return launch_cluster(rows_ws_kernel<T, R, M, true>, tm, sp, pl, st);
#define PIDB_WSC_MODE(M)                                                                    \
  PIDB_WSC_CASE(M, 1) PIDB_WSC_CASE(M, 2) PIDB_WSC_CASE(M, 3) PIDB_WSC_CASE(M, 4)           \
  PIDB_WSC_CASE(M, 5) PIDB_WSC_CASE(M, 6) PIDB_WSC_CASE(M, 7) PIDB_WSC_CASE(M, 8)           \
  PIDB_WSC_CASE(M, 9) PIDB_WSC_CASE(M, 10) PIDB_WSC_CASE(M, 11) PIDB_WSC_CASE(M, 12)        \
  PIDB_WSC_CASE(M, 13) PIDB_WSC_CASE(M, 14) PIDB_WSC_CASE(M, 15) PIDB_WSC_CASE(M, 16)       \
  PIDB_WSC_CASE(M, 17) PIDB_WSC_CASE(M, 18) PIDB_WSC_CASE(M, 19) PIDB_WSC_CASE(M, 20)       \
  PIDB_WSC_CASE(M, 21) PIDB_WSC_CASE(M, 22)
      PIDB_WSC_MODE(0) PIDB_WSC_MODE(1) PIDB_WSC_MODE(3)
      PIDB_WSC_CASE(1, 23) PIDB_WSC_CASE(1, 24) PIDB_WSC_CASE(1, 25) PIDB_WSC_CASE(1, 26)
      PIDB_WSC_CASE(1, 27) PIDB_WSC_CASE(1, 28) PIDB_WSC_CASE(1, 29) PIDB_WSC_CASE(1, 30)
      PIDB_WSC_CASE(1, 31) PIDB_WSC_CASE(1, 32)
#undef PIDB_WSC_MODE
#undef PIDB_WSC_CASE
      default: return kNotHandled;
    }
  }
  if (!pl.ext) sp.groups = pl.grid;  // ext: the caller sets the slice groups
  const int rows = (int)(((pl.ext ? pl.rpc : sp.n) + rw - 1) / rw);
  {
    if (pl.rb == 512 && !pl.ext) {  // wide rows (make_plan: n <= 142)
      switch (sp.mode * 32 + rows) {
#define PIDB_WR_CASE(M, R) \
  case M * 32 + R: return launch(rows_ws_kernel<T, R, M, false, 512>, tm, sp, pl, st);
#define PIDB_WR_MODE(M)                                                                   \
  PIDB_WR_CASE(M, 1) PIDB_WR_CASE(M, 2) PIDB_WR_CASE(M, 3) PIDB_WR_CASE(M, 4)             \
  PIDB_WR_CASE(M, 5) PIDB_WR_CASE(M, 6) PIDB_WR_CASE(M, 7) PIDB_WR_CASE(M, 8)             \
  PIDB_WR_CASE(M, 9) PIDB_WR_CASE(M, 10) PIDB_WR_CASE(M, 11) PIDB_WR_CASE(M, 12)          \
  PIDB_WR_CASE(M, 13) PIDB_WR_CASE(M, 14) PIDB_WR_CASE(M, 15) PIDB_WR_CASE(M, 16)         \
  PIDB_WR_CASE(M, 17) PIDB_WR_CASE(M, 18)
        PIDB_WR_MODE(0) PIDB_WR_MODE(1) PIDB_WR_MODE(3)
        PIDB_WR_CASE(1, 19) PIDB_WR_CASE(1, 20) PIDB_WR_CASE(1, 21) PIDB_WR_CASE(1, 22)
        PIDB_WR_CASE(1, 23) PIDB_WR_CASE(1, 24) PIDB_WR_CASE(1, 25) PIDB_WR_CASE(1, 26)
        PIDB_WR_CASE(1, 27)
#undef PIDB_WR_MODE
#undef PIDB_WR_CASE
        default:
          set_error("no wide-row kernel for %d rows per warp", rows);
          return PIDB_EUNSUPPORTED;
      }
    }
  }
  switch (sp.mode * 32 + rows) {
#define PIDB_WS_CASE(M, R) \
  case M * 32 + R: return launch(rows_ws_kernel<T, R, M, false>, tm, sp, pl, st);
#define PIDB_WS_MODE(M)                                                                   \
  PIDB_WS_CASE(M, 1) PIDB_WS_CASE(M, 2) PIDB_WS_CASE(M, 3) PIDB_WS_CASE(M, 4)             \
  PIDB_WS_CASE(M, 5) PIDB_WS_CASE(M, 6) PIDB_WS_CASE(M, 7) PIDB_WS_CASE(M, 8)             \
  PIDB_WS_CASE(M, 9) PIDB_WS_CASE(M, 10) PIDB_WS_CASE(M, 11) PIDB_WS_CASE(M, 12)          \
  PIDB_WS_CASE(M, 13) PIDB_WS_CASE(M, 14) PIDB_WS_CASE(M, 15) PIDB_WS_CASE(M, 16)         \
  PIDB_WS_CASE(M, 17) PIDB_WS_CASE(M, 18) PIDB_WS_CASE(M, 19) PIDB_WS_CASE(M, 20)         \
  PIDB_WS_CASE(M, 21) PIDB_WS_CASE(M, 22)
    PIDB_WS_MODE(0) PIDB_WS_MODE(1) PIDB_WS_MODE(3)
    PIDB_WS_CASE(1, 23) PIDB_WS_CASE(1, 24) PIDB_WS_CASE(1, 25) PIDB_WS_CASE(1, 26)
    PIDB_WS_CASE(1, 27) PIDB_WS_CASE(1, 28) PIDB_WS_CASE(1, 29) PIDB_WS_CASE(1, 30)
    PIDB_WS_CASE(1, 31) PIDB_WS_CASE(1, 32)
#undef PIDB_WS_MODE
#undef PIDB_WS_CASE
    default: return kNotHandled;
  }
}

}  // namespace
}  // namespace pidb
