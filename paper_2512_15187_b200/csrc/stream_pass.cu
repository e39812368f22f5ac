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

constexpr int kThreads = 256;
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

template <int LB>
__device__ __forceinline__ uint32_t swz(uint32_t off) {
  constexpr uint32_t mask = LB == 128 ? 7u : (LB == 64 ? 3u : 1u);
  return off ^ (((off >> 7) & mask) << 4);
}

template <typename T>
struct Chunk;
template <>
struct Chunk<float> {
  static constexpr int EPC = 4;
  __device__ static void load(const char* p, double (&v)[4]) {
    float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  __device__ static void loadf(const char* p, float (&v)[4]) {
    float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
};
template <>
struct Chunk<double> {
  static constexpr int EPC = 2;
  __device__ static void load(const char* p, double (&v)[2]) {
    double2 f = *reinterpret_cast<const double2*>(p);
    v[0] = f.x; v[1] = f.y;
  }
};

__device__ __forceinline__ bool is_nonbinary(double x) { return !(x == 0.0 || x == 1.0); }

// LB: bytes per smem line (box inner extent, = swizzle span); NCB column boxes
// per tile; IPT items (column box, member) per thread.
template <typename T, int LB, int NCB, int IPT>
__global__ void __launch_bounds__(kThreads, 1)
    stream_pass_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  constexpr int EPC = Chunk<T>::EPC;            // elements per 16-byte chunk
  constexpr int E = LB / (int)sizeof(T);        // elements per line (box inner)
  constexpr int V = NCB * E;                    // cells per tile
  constexpr int CPL = LB / 16;                  // chunks per line
  constexpr int QC = NCB * CPL;                 // chunks per tile row
  constexpr int P = kThreads / QC;              // row phases in pass 1
  static_assert(kThreads % QC == 0, "layout");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* tiles = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* tail = tiles + (size_t)p.stages * p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  double* sS = reinterpret_cast<double*>(tail + 8 * 8);     // V: w*S (or w*T)
  double* sW = sS + V;                                       // V: w
  double* red = sW + V;                                      // kWarps*V
  __shared__ unsigned s_ticket;
  __shared__ double s_col[kWarps];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t n = p.n;
  const int G = gridDim.x;
  const bool weighted = p.w != nullptr;
  const int mode = p.mode;
  const int64_t items = (int64_t)NCB * n;

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

  double acc_row[IPT], acc_mass[IPT];
  int64_t acc_nb[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) { acc_row[k] = 0.0; acc_mass[k] = 0.0; acc_nb[k] = 0; }
  double col_acc = 0.0;

  // pass-1 thread coordinates
  const int q = tid % QC, ph = tid / QC;
  const int q_cb = q / CPL, q_ch = q % CPL;

  for (int64_t j = 0; j < my_tiles; ++j) {
    const int s = (int)(j % p.stages);
    const int64_t tile = blockIdx.x + j * G;
    const int64_t x0 = tile * V;
    const unsigned char* st = tiles + (size_t)s * p.stage_bytes;
    mbar_wait(&full[s], (uint32_t)((j / p.stages) & 1));

    if (mode != MODE_MASS) {
      // ------------------------------------------------ pass 1: column sums
      double part[EPC];
      if constexpr (sizeof(T) == 4) {
        if (mode == MODE_MEAN) {
          float sh[EPC], sc[EPC];
#pragma unroll
          for (int e = 0; e < EPC; ++e) { sh[e] = 1.0f; sc[e] = 0.0f; }
          for (int r = ph; r < n; r += P) {
            const int rb = r / p.boxr, rr = r - rb * p.boxr;
            const uint32_t off = (uint32_t)(rr * LB + q_ch * 16);
            float v[4];
            Chunk<float>::loadf(reinterpret_cast<const char*>(st) +
                                    (size_t)(q_cb * p.nrb + rb) * p.boxr * LB + swz<LB>(off),
                                v);
#pragma unroll
            for (int e = 0; e < EPC; ++e) fast2sum_acc(sh[e], sc[e], v[e]);
          }
#pragma unroll
          for (int e = 0; e < EPC; ++e) part[e] = ((double)sh[e] - 1.0) + (double)sc[e];
        } else {
#pragma unroll
          for (int e = 0; e < EPC; ++e) part[e] = 0.0;
          for (int r = ph; r < n; r += P) {
            const int rb = r / p.boxr, rr = r - rb * p.boxr;
            const uint32_t off = (uint32_t)(rr * LB + q_ch * 16);
            double v[EPC];
            Chunk<T>::load(reinterpret_cast<const char*>(st) +
                               (size_t)(q_cb * p.nrb + rb) * p.boxr * LB + swz<LB>(off),
                           v);
            const double iv = p.inv[r];
#pragma unroll
            for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < EPC; ++e) part[e] = 0.0;
        for (int r = ph; r < n; r += P) {
          const int rb = r / p.boxr, rr = r - rb * p.boxr;
          const uint32_t off = (uint32_t)(rr * LB + q_ch * 16);
          double v[EPC];
          Chunk<T>::load(reinterpret_cast<const char*>(st) +
                             (size_t)(q_cb * p.nrb + rb) * p.boxr * LB + swz<LB>(off),
                         v);
          const double iv = mode == MODE_MEAN ? 1.0 : p.inv[r];
#pragma unroll
          for (int e = 0; e < EPC; ++e) part[e] = fma(iv, v[e], part[e]);
        }
      }
      // combine row phases inside the warp (lanes sharing q), fixed tree order
      if constexpr (QC < 32) {
#pragma unroll
        for (int o = QC; o < 32; o <<= 1)
#pragma unroll
          for (int e = 0; e < EPC; ++e) part[e] += __shfl_xor_sync(0xffffffffu, part[e], o);
        if (lane < QC) {
#pragma unroll
          for (int e = 0; e < EPC; ++e) red[warp * V + q * EPC + e] = part[e];
        }
      } else {
        // QC >= 32: every lane owns distinct cells; phases live in different warps
#pragma unroll
        for (int e = 0; e < EPC; ++e) red[ph * V + q * EPC + e] = part[e];
      }
      __syncthreads();
      constexpr int NPH = QC < 32 ? kWarps : P;
      for (int v = tid; v < V; v += kThreads) {
        double S = 0.0;
#pragma unroll
        for (int k = 0; k < NPH; ++k) S += red[k * V + v];
        const int64_t x = x0 + v;
        const double wx = x < p.m ? (weighted ? p.w[x] : 1.0) : 0.0;
        sS[v] = wx * S;
        sW[v] = wx;
        col_acc = fma(wx, S, col_acc);
      }
    } else {
      for (int v = tid; v < V; v += kThreads) {
        const int64_t x = x0 + v;
        sW[v] = x < p.m ? (weighted ? p.w[x] : 1.0) : 0.0;
      }
    }
    __syncthreads();

    // -------------------------------------------------- pass 2: row sweep
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int64_t it = tid + (int64_t)k * kThreads;
      if (it < items) {
        const int cb = (int)(it / n);
        const int r = (int)(it - (int64_t)cb * n);
        const int rb = r / p.boxr, rr = r - rb * p.boxr;
        const char* line = reinterpret_cast<const char*>(st) +
                           (size_t)(cb * p.nrb + rb) * p.boxr * LB;
        double ar = acc_row[k], am = acc_mass[k];
        int64_t nb = 0;
#pragma unroll
        for (int L = 0; L < CPL; ++L) {
          double v[EPC];
          Chunk<T>::load(line + swz<LB>((uint32_t)(rr * LB + L * 16)), v);
          const int vb = cb * E + L * EPC;
          if (mode == MODE_MASS) {
#pragma unroll
            for (int e = 0; e < EPC; ++e) {
              am = fma(v[e], sW[vb + e], am);
              nb += is_nonbinary(v[e]);
            }
          } else if (mode == MODE_COLS) {
#pragma unroll
            for (int e = 0; e < EPC; ++e) ar = fma(v[e], sS[vb + e], ar);
          } else if (weighted) {
#pragma unroll
            for (int e = 0; e < EPC; ++e) {
              ar = fma(v[e], sS[vb + e], ar);
              am = fma(v[e], sW[vb + e], am);
            }
          } else {
#pragma unroll
            for (int e = 0; e < EPC; ++e) {
              ar = fma(v[e], sS[vb + e], ar);
              am += v[e];
            }
          }
        }
        acc_row[k] = ar;
        acc_mass[k] = am;
        acc_nb[k] += nb;
      }
    }
    __syncthreads();  // every thread is done with stage s (and sS/sW)
    if (tid == 0 && j + p.stages < my_tiles) issue(j + p.stages);
  }

  // ------------------------------------------------ CTA partials -> global
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int64_t it = tid + (int64_t)k * kThreads;
    if (it < items) {
      double* dst = p.part + ((size_t)blockIdx.x * items + it) * 2;
      dst[0] = acc_row[k];
      dst[1] = acc_mass[k];
    }
  }
  if (p.mode == MODE_MASS && p.part_nb != nullptr) {
    // merge column boxes of the same member (fixed order) into [grid][n]
    int64_t* nbp = p.part_nb + (size_t)blockIdx.x * n;
    // items with cb==0 own row r; other cb items add in order via smem-free
    // two-phase write: first cb==0 writes, sync, then cb>0 atomically add
    // (integers: order-independent, exact).
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int64_t it = tid + (int64_t)k * kThreads;
      if (it < n) nbp[it] = acc_nb[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int64_t it = tid + (int64_t)k * kThreads;
      if (it >= n && it < items)
        atomicAdd(reinterpret_cast<unsigned long long*>(&nbp[it % n]),
                  (unsigned long long)acc_nb[k]);
    }
  }
  {
    double c = warp_sum(col_acc);
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
  if (tid == 0) s_ticket = atomicAdd(p.counter, 1u);
  __syncthreads();
  if (s_ticket != (unsigned)(G - 1)) return;

  // ------------------------------------------- last CTA: fixed-order reduce
  __threadfence();
  for (int64_t r = warp; r < n; r += kWarps) {
    double a = 0.0, b = 0.0;
    int64_t nb = 0;
    for (int g = lane; g < G; g += 32) {
      for (int cb = 0; cb < NCB; ++cb) {
        const double* src = p.part + ((size_t)g * items + (int64_t)cb * n + r) * 2;
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

// ---------------------------------------------------------------- host side
struct Plan {
  int lb, ncb, ipt, boxr, nrb, stages, grid;
  uint32_t stage_bytes;
  size_t smem;
  int64_t tiles;
};

constexpr size_t kSmemBudget = 227 * 1024;

size_t tail_bytes(int V) { return 64 + (size_t)V * 8 * 2 + (size_t)kWarps * V * 8 + 64; }

bool make_plan(int64_t n, int64_t m, int esize, Plan& pl) {
  if (n < 1 || m < 1) return false;
  const int nrb = (int)((n + 255) / 256);
  const int boxr_full = (int)(((n + nrb - 1) / nrb + 7) / 8 * 8);
  const int rows = nrb * boxr_full;
  struct Cand { int lb, ncb; };
  const Cand cands[] = {{128, 2}, {128, 1}, {64, 1}, {32, 1}};
  for (const Cand& c : cands) {
    const int V = c.ncb * c.lb / esize;
    const uint32_t sb = (uint32_t)(c.ncb * rows * c.lb);
    const size_t tb = tail_bytes(V) + 1024;
    const int min_stages = (c.lb == 32) ? 2 : 3;
    int stages = (int)std::min<size_t>(8, (kSmemBudget - tb) / sb);
    if (sb > kSmemBudget || stages < min_stages) continue;
    const int64_t items = (int64_t)c.ncb * n;
    int ipt = 1;
    while ((int64_t)ipt * kThreads < items) ipt *= 2;
    if (ipt > 16) return false;
    pl.lb = c.lb; pl.ncb = c.ncb; pl.ipt = ipt; pl.boxr = boxr_full; pl.nrb = nrb;
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

template <typename T, int LB, int NCB, int IPT>
int launch_t(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  auto kern = stream_pass_kernel<T, LB, NCB, IPT>;
  PIDB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  kern<<<pl.grid, kThreads, pl.smem, st>>>(tm, sp);
  PIDB_LAUNCH_CHECK("stream_pass_kernel");
  return PIDB_OK;
}

template <typename T, int LB, int NCB>
int launch_ipt(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  switch (pl.ipt) {
    case 1: return launch_t<T, LB, NCB, 1>(tm, sp, pl, st);
    case 2: return launch_t<T, LB, NCB, 2>(tm, sp, pl, st);
    case 4: return launch_t<T, LB, NCB, 4>(tm, sp, pl, st);
    case 8: return launch_t<T, LB, NCB, 8>(tm, sp, pl, st);
    case 16: return launch_t<T, LB, NCB, 16>(tm, sp, pl, st);
  }
  set_error("unsupported items-per-thread %d", pl.ipt);
  return PIDB_EUNSUPPORTED;
}

template <typename T>
int launch_layout(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  if (pl.lb == 128 && pl.ncb == 2) return launch_ipt<T, 128, 2>(tm, sp, pl, st);
  if (pl.lb == 128 && pl.ncb == 1) return launch_ipt<T, 128, 1>(tm, sp, pl, st);
  if (pl.lb == 64) return launch_ipt<T, 64, 1>(tm, sp, pl, st);
  return launch_ipt<T, 32, 1>(tm, sp, pl, st);
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
