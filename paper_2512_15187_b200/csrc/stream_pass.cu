// K5 (PID-mean partials, one HBM pass), K9-B (exact-PID column sums) and K6
// (member masses + non-binary counts): the streaming kernels of the depth path.
//
// Reference path replaced:
//   depth_pid_mean          /root/reference/pkg/src/fuzzdepth/depth.py:246-287
//     mean_mask             /root/reference/pkg/src/fuzzdepth/grid.py:251-261
//     mask_mass(mean)       /root/reference/pkg/src/fuzzdepth/grid.py:242-244
//     _member_mean_terms    /root/reference/pkg/src/fuzzdepth/depth.py:231-243
//   _pairwise_sums col_inv  /root/reference/pkg/src/fuzzdepth/depth.py:157,160 (K9-B)
//   member_masses           /root/reference/pkg/src/fuzzdepth/depth.py:88-102 (K6)
//
// Layout: members are rows of an (n x m) row-major matrix in HBM.  A "tile"
// is the next 256 bytes of cells (V = 64 fp32 / 32 fp64) of EVERY member,
// fetched by one 2D TMA box (256-byte rows, no swizzle: TMA streams reach
// ~6.7 TB/s with 256-byte rows but stall at ~4.6 TB/s with 128-byte rows,
// tools/ubench_tma.cu), so HBM is read exactly once and the tile is consumed
// twice from SMEM:
//   pass 1 (column sweep): S(x) = sum_i u_i(x)        [MODE_MEAN]
//                           T(x) = sum_i inv_i u_i(x)  [MODE_COLS]
//   pass 2 (row sweep)   : acc_i += u_i(x) * w(x) S(x),  mass_i += w(x) u_i(x)
// Pass 1 on fp32 data is an error-free Fast2Sum in packed fp32 (FADD2, seeded
// with 1.0 so |s| >= |u| holds for mask values in [0,1]), combined in fp64;
// pass 2 converts each value once to fp64 (DFMA/DADD).  CTA partials are
// reduced by the last CTA in a fixed order (bit-reproducible per device).
//
// Two kernels:
//   rows_kernel    (n <= 256): software-pipelined tiles (pass 1 of tile j
//                  overlaps pass 2 of tile j-1, one barrier per tile); warp w
//                  owns rows w, w+16, ..., lane l owns 8 bytes of each row, the
//                  row sums stay in registers for the whole kernel.
//   chunked_kernel (256 < n <= 4096): the tile is streamed in 256-row chunks
//                  twice; touch 1 (columns) comes from HBM with an L2
//                  evict_last hint, touch 2 (rows) re-reads the chunks from L2.
// Wider ensembles (n > 4096) take the two-read path in stream_wide.cu.
#include "stream_common.cuh"

namespace pidb {

// stream_wide.cu: two-read fallback for n > 4096 members
size_t wide_workspace(int64_t n, int64_t m, int dtype);
size_t wide_fold_bytes(int64_t n, int64_t m, int dtype);
int wide_fold_f(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                const double* w, const double* inv, void* ws, const double** f, void* stream);
int run_wide_pass(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                  const double* w, const double* inv, double* out_row, double* out_mass,
                  double* out_col, int64_t* out_nb, void* ws, size_t ws_bytes, void* stream);

namespace {
using namespace stream;

// ---------------------------------------------------------------------------
// rows_kernel: ROWS = ceil(rows / 16) member rows per warp.
//   CL = false: n <= 256, one CTA holds every member row of its tiles.
//   CL = true : 256 < n <= 16 * 256.  A cluster of cs CTAs shares each tile,
//     CTA rank r holds rows [r * rpc, (r + 1) * rpc).  Pass 1 yields the
//     CTA's column partials, which are pushed to every CTA of the cluster
//     with st.async (DSMEM, completing on the receiver's mbarrier); pass 2
//     of the previous tile sums the cs partials in rank order (identical in
//     every CTA) and sweeps the CTA's own rows.  One HBM read, no L2
//     re-read, the row sums stay in registers as for n <= 256.
template <typename T, int ROWS, bool CL>
__global__ void __launch_bounds__(kRowsThreads, 1)
    rows_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  constexpr int EPC = Vec<T>::EPC;
  constexpr int V = kRowBytes / (int)sizeof(T);  // cells per tile
  constexpr int EPL = 8 / (int)sizeof(T);        // elements per lane in pass 2

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* tiles = smem_raw + pad;
  unsigned char* tail = tiles + (size_t)p.stages * p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  double* sS = reinterpret_cast<double*>(tail + 128);  // [2][V]
  double* sW = sS + 2 * V;                              // [2][V]
  double* red = sW + 2 * V;                             // [2][kRowsWarps][V]
  unsigned* s_ticket = reinterpret_cast<unsigned*>(red + 2 * kRowsWarps * V);
  double* s_col = reinterpret_cast<double*>(s_ticket + 2);
  uint64_t* xbar = reinterpret_cast<uint64_t*>(tail + 64);        // [4] (CL)
  const uint32_t xoff =
      ((smem_u32(s_col + kRowsWarps) + 15u) & ~15u) - smem_u32(smem_raw);  // 16-B aligned
  double* xbuf = reinterpret_cast<double*>(smem_raw + xoff);        // [4][cs][V] (CL)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = (int)p.n;
  const int mode = p.mode;
  const int sweep = mode == MODE_SIM ? MODE_MEAN : mode;  // pass-1 column kind
  const bool weighted = p.w != nullptr;
  const int cs = CL ? p.cs : 1;
  const uint32_t rank = CL ? cluster_rank() : 0u;
  const int cid = (int)blockIdx.x / cs, ncl = (int)gridDim.x / cs;
  const int r0 = (int)rank * (CL ? p.rpc : 0);
  const int box = CL ? p.rpc : n;                          // rows per TMA box
  const int nloc = CL ? max(0, min(n - r0, p.rpc)) : n;    // member rows of this CTA
  const bool exch = CL && mode != MODE_MASS;
  const int64_t my_tiles = p.tiles > cid ? (p.tiles - 1 - cid) / ncl + 1 : 0;
  const uint64_t pol = policy_evict_first();
  const uint32_t xbytes = (uint32_t)cs * V * 8u;  // all cs partials of a tile
  double col_acc = 0.0;

  if (tid == 0) {
    prefetch_tma_desc(&tmap);
    for (int s = 0; s < p.stages; ++s) mbar_init(&full[s], 1);
    if (exch)
      for (int s = 0; s < 4; ++s) mbar_init(&xbar[s], 1);
    fence_mbar_init();
    if (exch)
      for (int s = 0; s < 4 && s < my_tiles; ++s) mbar_arrive_expect_tx(&xbar[s], xbytes);
  }
  __syncthreads();
  if constexpr (CL) cluster_sync();  // peers' mbarriers exist before any st.async

  auto issue = [&](int64_t j) {  // local tile j -> stage j % stages (thread 0)
    const int s = (int)(j % p.stages);
    mbar_arrive_expect_tx(&full[s], (uint32_t)box * kRowBytes);
    tma_load_2d(tiles + (size_t)s * p.stage_bytes, &tmap, (int32_t)((cid + j * ncl) * V), r0,
                &full[s], pol);
  };
  // CL: push this CTA's column partials of tile j to every CTA of the
  // cluster (16-byte st.async, completing on the receiver's mbarrier; this
  // measured faster than one bulk copy per peer)
  auto send = [&](const double* rd, int64_t j) {
    const int slot = (int)(j & 3);
    for (int v = tid; v < V / 2; v += kRowsThreads) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < kRowsWarps; ++k) {
        a += rd[k * V + 2 * v];
        b += rd[k * V + 2 * v + 1];
      }
      const uint32_t la = smem_u32(xbuf + ((size_t)slot * cs + rank) * V + 2 * v);
      const uint32_t lb = smem_u32(&xbar[slot]);
      for (int c = 0; c < cs; ++c) st_async_f64x2(mapa(la, c), a, b, mapa(lb, c));
    }
  };

  if (tid == 0)
    for (int64_t j = 0; j < my_tiles && j < p.stages; ++j) issue(j);

  double acc_row[ROWS], acc_mass[ROWS];
  int acc_nb[ROWS];
#pragma unroll
  for (int k = 0; k < ROWS; ++k) { acc_row[k] = 0.0; acc_mass[k] = 0.0; acc_nb[k] = 0; }

  const int q = tid & (kChunks16 - 1), ph = tid / kChunks16;
  const uint32_t p1_off = (uint32_t)(ph * kRowBytes + q * 16);
  const uint32_t p2_off = (uint32_t)(warp * kRowBytes + lane * 8);
  const int cell = lane * EPL;

  auto pass2 = [&](const unsigned char* st, int buf, int64_t jt) {
    double s_l[EPL], w_l[EPL];
    if (exch) {
      // CL: every lane forms S for its own cells from the cs partials of
      // tile jt (rank order, identical in every CTA of the cluster)
      const int slot = (int)(jt & 3);
      mbar_wait(&xbar[slot], (uint32_t)((jt >> 2) & 1));
      const int64_t x0 = (cid + jt * ncl) * (int64_t)V;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const int64_t x = x0 + cell + e;
        const double wx = x < p.m ? (p.w ? __ldg(p.w + x) : 1.0) : 0.0;
        double S = 0.0;
        for (int c = 0; c < cs; ++c) S += xbuf[((size_t)slot * cs + c) * V + cell + e];
        s_l[e] = p.mode == MODE_SIM ? __ddiv_rn(S, (double)p.n) : wx * S;
        w_l[e] = wx;
        if (rank == 0 && warp == 0) col_acc = fma(wx, S, col_acc);
      }
    } else {
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        s_l[e] = sS[buf * V + cell + e];
        w_l[e] = sW[buf * V + cell + e];
      }
    }
    const unsigned char* base = st + p2_off;
#define PIDB_ROWS_LOOP(BODY)                                                \
  _Pragma("unroll") for (int k = 0; k < ROWS; ++k) {                        \
    if (k < ROWS - 1 || warp + k * kRowsWarps < nloc) {                         \
      const unsigned char* a = base + k * (kRowsWarps * kRowBytes);             \
      double v[EPL];                                                        \
      if constexpr (sizeof(T) == 4) {                                       \
        const float2 f = *reinterpret_cast<const float2*>(a);              \
        v[0] = f.x; v[EPL - 1] = f.y;                                       \
      } else {                                                              \
        v[0] = *reinterpret_cast<const double*>(a);                         \
      }                                                                     \
      _Pragma("unroll") for (int e = 0; e < EPL; ++e) { BODY; }             \
    }                                                                       \
  }
    if (mode == MODE_MEAN && !weighted) {
      PIDB_ROWS_LOOP(acc_row[k] = fma(v[e], s_l[e], acc_row[k]); acc_mass[k] += v[e])
    } else if (mode == MODE_SIM) {
      PIDB_ROWS_LOOP(acc_row[k] = fma(fmin(v[e], s_l[e]), w_l[e], acc_row[k]);
                     acc_mass[k] = fma(v[e], w_l[e], acc_mass[k]))
    } else if (mode == MODE_MASS) {
      PIDB_ROWS_LOOP(acc_mass[k] = fma(v[e], w_l[e], acc_mass[k]); acc_nb[k] += is_nonbinary(v[e]))
    } else if (mode == MODE_COLS) {
      PIDB_ROWS_LOOP(acc_row[k] = fma(v[e], s_l[e], acc_row[k]))
    } else {
      PIDB_ROWS_LOOP(acc_row[k] = fma(v[e], s_l[e], acc_row[k]);
                     acc_mass[k] = fma(v[e], w_l[e], acc_mass[k]))
    }
#undef PIDB_ROWS_LOOP
  };

  ColSweep<T, kRowsThreads> csw;
  int s_cur = 0, s_prev = 0;
  uint32_t par = 0;
  for (int64_t j = 0; j <= my_tiles; ++j) {
    const bool have = j < my_tiles;
    double* rd = red + (j & 1) * kRowsWarps * V;
    if (have) {
      mbar_wait(&full[s_cur], par);
      if (mode != MODE_MASS) {
        csw.reset();
        csw.run(tiles + (size_t)s_cur * p.stage_bytes + p1_off, ph, box, sweep, p.inv, r0 + ph,
                n);
        csw.combine(sweep);
        if (lane < 16) {
#pragma unroll
          for (int e = 0; e < EPC; ++e) rd[warp * V + q * EPC + e] = csw.part[e];
        }
      }
    }
    __syncthreads();
    // tile j-2's stage was last read by pass 2 in the previous iteration
    if (tid == 0 && j >= 2 && j - 2 + p.stages < my_tiles) issue(j - 2 + p.stages);
    if (exch) {
      // every thread passed its wait for tile j-2 (previous iteration): re-arm
      // that slot for tile j+2
      if (tid == 0 && j >= 2 && j + 2 < my_tiles)
        mbar_arrive_expect_tx(&xbar[(j - 2) & 3], xbytes);
      if (have) send(rd, j);
    } else if (have) {
      finalize_tile<V, 0, kRowsThreads>(p, rd, (cid + j * ncl) * (int64_t)V, sS + (j & 1) * V,
                       sW + (j & 1) * V, mode != MODE_MASS, col_acc);
    }
    if (j >= 1) pass2(tiles + (size_t)s_prev * p.stage_bytes, (int)((j - 1) & 1), j - 1);
    s_prev = s_cur;
    if (++s_cur == p.stages) { s_cur = 0; par ^= 1u; }
  }

  // rows -> global partials (part layout [grid][n][2])
#pragma unroll
  for (int k = 0; k < ROWS; ++k) {
    const int rl = warp + k * kRowsWarps;
    const double a = warp_sum(acc_row[k]);
    const double b = warp_sum(acc_mass[k]);
    int nb = acc_nb[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0 && rl < nloc) {
      const int r = r0 + rl;
      double* dst = p.part + part_at(p, 1, 0, r, cid) * 2;
      dst[0] = a;
      dst[1] = b;
      if (p.mode == MODE_MASS && p.part_nb != nullptr) p.part_nb[part_at(p, 1, 0, r, cid)] = nb;
    }
  }
  if constexpr (CL) cluster_sync();  // no CTA leaves while peers may still target its SMEM
  finish_partials<kRowsThreads>(p, 1, col_acc, s_ticket, s_col);
}

// ---------------------------------------------------------------------------
// chunked_kernel: 256 < n <= 256 * CMAX.  Thread t owns half (t >> 8) of row
// (t & 255) of every chunk; it reads the half's 8 chunks in a row-rotated
// order (bank-conflict free without swizzle) and keeps its row sums for chunk
// c in registers (acc[c]).
constexpr int kChunkRows = 256;
constexpr int kChunkBytes = kChunkRows * kRowBytes;  // 64 KB
constexpr int kChunkBufs = 3;

template <typename T, int CMAX>
__global__ void __launch_bounds__(kThreads, 1)
    chunked_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  constexpr int EPC = Vec<T>::EPC;
  constexpr int V = kRowBytes / (int)sizeof(T);
  constexpr int HALF = V / 2;  // cells per half row
  static_assert(kThreads == 2 * kChunkRows, "one half row per thread");

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
  const int sweep = mode == MODE_SIM ? MODE_MEAN : mode;  // pass-1 column kind
  const bool two_touch = mode != MODE_MASS;
  const bool weighted = p.w != nullptr;
  const int64_t my_tiles = p.tiles > blockIdx.x ? (p.tiles - 1 - blockIdx.x) / G + 1 : 0;
  const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();

  if (tid == 0) {
    prefetch_tma_desc(&tmap);
    for (int b = 0; b < kChunkBufs; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // Chunk schedule.  Uses per tile: touch 1 visits chunks 0..C-1, touch 2
  // visits C-1..0, so the last R = min(C, kChunkBufs) chunks of touch 1 are
  // still resident when touch 2 starts and are reused without a reload
  // (n <= 768: one touch of HBM and no L2 re-read at all).  Every thread runs
  // the same deterministic schedule; thread 0 issues the TMA loads.  A
  // buffer is refilled (next load in use order) as soon as its chunk has no
  // later use, so two uses of lookahead stay in flight across touches/tiles.
  const int R = two_touch ? min(C, kChunkBufs) : 0;
  const int P = two_touch ? 2 * C : C;  // uses per tile
  // small FIFOs of 2-bit buffer ids packed in registers
  uint32_t fq = 0, fq_n = kChunkBufs;  // free buffers
#pragma unroll
  for (int b = 0; b < kChunkBufs; ++b) fq |= (uint32_t)b << (2 * b);
  uint32_t lq = 0, lq_n = 0;  // buffers of issued, not yet consumed loads
  uint32_t rbuf = 0;  // buffers of the resident chunks C-R .. C-1, per tile (mod 4:
                      // at most 3 tiles hold buffers at a time)
  uint32_t ph_bits = 0;       // per-buffer mbarrier parity
  int64_t lj = 0;        // next load: tile lj, use position lpos
  int lpos = 0;
  auto needs_load = [&](int pos) { return pos < C || (P - 1 - pos) < C - R; };
  // (single touch: P == C, every use loads)
  auto issue_loads = [&]() {
    while (fq_n > 0 && lj < my_tiles) {
      if (!needs_load(lpos)) {
        if (++lpos == P) { lpos = 0; ++lj; }
        continue;
      }
      const uint32_t b = fq & 3u;
      fq >>= 2;
      --fq_n;
      lq |= b << (2 * lq_n);
      ++lq_n;
      // touch 1 walks up; the row sweep (touch 2, or the only touch) walks down
      const bool first_touch = two_touch && lpos < C;
      const int c = first_touch ? lpos : P - 1 - lpos;
      if (first_touch && c >= C - R) {
        const int sh = 2 * ((int)(lj & 3) * kChunkBufs + c - (C - R));
        rbuf = (rbuf & ~(3u << sh)) | (b << sh);
      }
      if (tid == 0) {
        // keep (evict_last) only chunks that touch 2 re-reads from L2
        const bool keep = two_touch && first_touch && c < C - R;
        mbar_arrive_expect_tx(&full[b], kChunkBytes);
        tma_load_2d(bufs + (size_t)b * kChunkBytes, &tmap, (int32_t)((blockIdx.x + lj * G) * V),
                    c * kChunkRows, &full[b], keep ? pol_keep : pol_drop);
      }
      if (++lpos == P) { lpos = 0; ++lj; }
    }
  };
  issue_loads();

  double acc_row[CMAX], acc_mass[CMAX];
  int acc_nb[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) { acc_row[c] = 0.0; acc_mass[c] = 0.0; acc_nb[c] = 0; }
  double col_acc = 0.0;

  const int q = tid & (kChunks16 - 1), ph = tid / kChunks16;
  const uint32_t a_off = (uint32_t)(ph * kRowBytes + q * 16);
  const int b_half = tid >> 8, b_rr = tid & 255;
  const uint32_t b_off = (uint32_t)(b_rr * kRowBytes + b_half * (kRowBytes / 2));
  const int b_rot = b_rr & 7;

  uint32_t cur_b = 0;
  auto use_chunk = [&](int64_t j, int pos) -> const unsigned char* {
    if (needs_load(pos)) {
      cur_b = lq & 3u;
      lq >>= 2;
      --lq_n;
      mbar_wait(&full[cur_b], (ph_bits >> cur_b) & 1u);
      ph_bits ^= 1u << cur_b;
    } else {
      cur_b = (rbuf >> (2 * ((int)(j & 3) * kChunkBufs + (P - 1 - pos) - (C - R)))) & 3u;
    }
    return bufs + (size_t)cur_b * kChunkBytes;
  };
  auto release_chunk = [&](int pos) {
    __syncthreads();  // everyone is done with this buffer
    const bool reused = two_touch && pos < C && pos >= C - R;
    if (!reused) {
      fq |= cur_b << (2 * fq_n);
      ++fq_n;
      issue_loads();
    }
  };

  ColSweep<T> cs;
  for (int64_t j = 0; j < my_tiles; ++j) {
    const int64_t x0 = (blockIdx.x + j * G) * (int64_t)V;
    if (two_touch) {  // ------------------------------ touch 1: column sweep
      cs.reset();
      for (int c = 0; c < C; ++c) {
        const unsigned char* st = use_chunk(j, c);
        cs.run(st + a_off, ph, kChunkRows, sweep, p.inv, c * kChunkRows + ph, n);
        release_chunk(c);
      }
      cs.combine(sweep);
      if (lane < 16) {
#pragma unroll
        for (int e = 0; e < EPC; ++e) red[warp * V + q * EPC + e] = cs.part[e];
      }
    }
    __syncthreads();
    finalize_tile<V, EPC>(p, red, x0, sS, sW, two_touch, col_acc);
    __syncthreads();
    // --------------------------------------------------- touch 2: row sweep
    const double* S = sS + b_half * HALF;
    const double* W = sW + b_half * HALF;
#pragma unroll
    for (int c = CMAX - 1; c >= 0; --c) {  // the row sweep walks the chunks backwards
      if (c < C) {
        const int pos = P - 1 - c;
        const unsigned char* line = use_chunk(j, pos) + b_off;
        if (c * kChunkRows + b_rr < n) {
          double ar[EPC], am[EPC];
          int nb = 0;
#pragma unroll
          for (int e = 0; e < EPC; ++e) { ar[e] = 0.0; am[e] = 0.0; }
#pragma unroll
          for (int L = 0; L < 8; ++L) {
            const int Lr = (L + b_rot) & 7;
            double v[EPC];
            Vec<T>::load(line + Lr * 16, v);
            // element-major S/W slots (finalize_tile<V, EPC>): e*8 + chunk
            if (mode == MODE_MASS) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                am[e] = fma(v[e], W[e * 8 + Lr], am[e]);
                nb += is_nonbinary(v[e]);
              }
            } else if (mode == MODE_SIM) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                ar[e] = fma(fmin(v[e], S[e * 8 + Lr]), W[e * 8 + Lr], ar[e]);
                am[e] = fma(v[e], W[e * 8 + Lr], am[e]);
              }
            } else if (mode == MODE_COLS) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) ar[e] = fma(v[e], S[e * 8 + Lr], ar[e]);
            } else if (weighted) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                ar[e] = fma(v[e], S[e * 8 + Lr], ar[e]);
                am[e] = fma(v[e], W[e * 8 + Lr], am[e]);
              }
            } else {
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                ar[e] = fma(v[e], S[e * 8 + Lr], ar[e]);
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
        release_chunk(pos);
      }
    }
  }

  // halves -> global partials (member-major: part[r][half][block][2])
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    const int r = c * kChunkRows + b_rr;
    if (c < C && r < n) {
      double* dst = p.part + part_at(p, 2, b_half, r, blockIdx.x) * 2;
      dst[0] = acc_row[c];
      dst[1] = acc_mass[c];
    }
  }
  if (p.mode == MODE_MASS && p.part_nb != nullptr) {
    int64_t* nbp = p.part_nb;
    if (b_half == 0) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c) {
        const int r = c * kChunkRows + b_rr;
        if (c < C && r < n) nbp[part_at(p, 1, 0, r, blockIdx.x)] = acc_nb[c];
      }
    }
    __syncthreads();
    if (b_half == 1) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c) {
        const int r = c * kChunkRows + b_rr;
        if (c < C && r < n)
          atomicAdd(reinterpret_cast<unsigned long long*>(&nbp[part_at(p, 1, 0, r, blockIdx.x)]),
                    (unsigned long long)acc_nb[c]);
      }
    }
  }
  finish_partials<kThreads>(p, 2, col_acc, s_ticket, s_col);
}

// ---------------------------------------------------------------- host side

// SMEM tail of rows_ws_kernel (single CTA): barriers, sS/sW[2][V], the
// column group's red[<= 8 warps][V], ticket and per-warp column sums
size_t ws_tail(int V) {
  return 128 + (size_t)4 * V * 8 + (size_t)8 * V * 8 + 16 + kRowsWarps * 8 + 64;
}
size_t rows_tail(int V, int cs) {
  return 128 + (size_t)4 * V * 8 + (size_t)2 * kRowsWarps * V * 8 + 16 + kRowsWarps * 8 + 64 +
         (cs > 1 ? (size_t)4 * cs * V * 8 + 16 : 0);
}

// Cluster size for 256 < n (0 = chunked kernel), from measurements on B200
// (tools/prof_k5.py, 256^3 cells): pairs of CTAs win for
// n <= 512 and 8-CTA clusters for 1536 < n <= 2048; in between the chunked
// kernel is faster.  PIDB_CLUSTER overrides (tuning).
int cluster_size_for(int64_t n, bool ws, bool exchange) {
  int cs = 0;
  // warp-specialised: <= 256 rows per CTA; non-portable clusters of up to 16
  // measured faster than (n = 2500, 3000) or equal to (n = 4000) the chunked kernel
  if (ws || !exchange) cs = n <= 2048 ? (int)((n + 255) / 256) : 16;
  else if (n <= 512) cs = 2;
  else if (n > 1536 && n <= 2048) cs = 8;
  if (const char* e = std::getenv("PIDB_CLUSTER")) {
    const int v = std::atoi(e);
    if (v >= (int)((n + 255) / 256) && v <= 16) cs = v;
    if (v == 0) cs = 0;  // disable: chunked kernel
  }
  return cs;
}
size_t chunked_smem(int V) {
  return 1024 + (size_t)kChunkBufs * kChunkBytes + 64 + (size_t)(2 + kWarps) * V * 8 + 16 +
         kWarps * 8 + 64;
}

bool ws_eligible(int mode) { return mode != MODE_MASS; }

thread_local bool t_no_cluster = false;  // set while falling back from a cluster launch

bool make_plan(int64_t n, int64_t m, int esize, Plan& pl, int mode = MODE_MEAN) {
  pl = Plan{};
  if (n < 1 || m < 1) return false;
  const int V = kRowBytes / esize;
  pl.tiles = (m + V - 1) / V;
  pl.grid = (int)std::min<int64_t>(pl.tiles, sm_count());
  pl.cs = 1;
  pl.rpc = (int)n;
  if (n > 256 && n <= 16 * 256 && !t_no_cluster) {
    // the masses-only mode has no column exchange: plain row slices per CTA
    // (fp64 masses measured faster with the chunked kernel: 6.3 vs 5.3 TB/s)
    const int cs = cluster_size_for(n, ws_eligible(mode) && std::getenv("PIDB_WS") == nullptr,
                                    mode != MODE_MASS || esize != 4);
    if (cs >= 2 && cs <= 16) {
      pl.chunked = false;
      pl.cs = cs;
      pl.grid = (int)std::max<int64_t>(
          cs, std::min<int64_t>(pl.tiles * cs, sm_count()) / cs * cs);
      pl.rpc = (int)((n + cs - 1) / cs);
      pl.rows = (pl.rpc + kRowsWarps - 1) / kRowsWarps;
      pl.box_rows = pl.rpc;
      pl.stage_bytes = (uint32_t)align_up((size_t)pl.rpc * kRowBytes, 1024);
      const size_t tb = rows_tail(V, cs) + 1024;
      pl.stages = (int)std::min<size_t>(kMaxStages, (kSmemBudget - tb) / pl.stage_bytes);
      if (pl.stages >= 3) {
        pl.smem = (size_t)pl.stages * pl.stage_bytes + tb;
        return true;
      }
      pl.cs = 1;
      pl.rpc = (int)n;
    }
  }
  if (n <= 256 && ws_eligible(mode) && std::getenv("PIDB_WS") == nullptr &&
      !(std::getenv("PIDB_RB") && std::atoi(std::getenv("PIDB_RB")) == 256)) {
    // wide rows: 512-byte member-row segments per tile (HBM streams them
    // faster than 256-byte ones, profiles/r02_ubench_rows.log) when three
    // stages of n rows fit (n <= 142): K5 n = 64 / 100 / 140 x 512^3
    // 8.54 / 10.60 / 13.05 -> 7.63 / 9.52 / 11.43 ms; with only two stages
    // (n = 200) the ring runs dry: 15.4 -> 16.0 ms, so 256-byte rows stay
    // (profiles/r02_k5_wide_rows.txt).  Warp-specialised kernel only.
    constexpr int RB = 512;
    const int V2 = RB / esize;
    const uint32_t sb = (uint32_t)align_up((size_t)n * RB, 1024);
    const size_t tb = ws_tail(V2) + 1024;
    const int st = (int)std::min<size_t>(kMaxStages, (kSmemBudget - tb) / sb);
    if (st >= 3) {
      pl.chunked = false;
      pl.rb = RB;
      pl.tiles = (m + V2 - 1) / V2;
      pl.grid = (int)std::min<int64_t>(pl.tiles, sm_count());
      pl.rows = (int)((n + kRowsWarps - 1) / kRowsWarps);
      pl.box_rows = (int)n;
      pl.stage_bytes = sb;
      pl.stages = st;
      pl.smem = (size_t)st * sb + tb;
      return true;
    }
  }
  if (n <= 256) {
    pl.chunked = false;
    pl.rows = (int)((n + kRowsWarps - 1) / kRowsWarps);
    pl.box_rows = (int)n;
    pl.stage_bytes = (uint32_t)align_up((size_t)n * kRowBytes, 1024);
    const size_t tb = rows_tail(V, 1) + 1024;
    pl.stages = (int)std::min<size_t>(kMaxStages, (kSmemBudget - tb) / pl.stage_bytes);
    if (pl.stages < 3) return false;
    pl.smem = (size_t)pl.stages * pl.stage_bytes + tb;
    return true;
  }
  if (n > (int64_t)kChunkMax * kChunkRows) return false;
  pl.chunked = true;
  pl.rows = 0;
  pl.box_rows = kChunkRows;
  pl.stages = kChunkBufs;
  pl.stage_bytes = kChunkBytes;
  pl.smem = chunked_smem(V);
  return true;
}

// Sized for a full-width grid whatever the plan, so that a launch can fall
// back to another kernel variant without a bigger workspace.
size_t workspace_bytes(const Plan& pl, int64_t n) {
  const size_t g = (size_t)std::max(pl.grid, sm_count());
  size_t b = 256;  // completion counter: fixed offset 0, zero between launches
  b += align_up(g * 2 * n * 2 * sizeof(double), 256);
  b += align_up(g * sizeof(double), 256);
  b += align_up(g * n * sizeof(int64_t), 256);
  return b;
}

template <typename T>
int launch_typed(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  // warp-specialised kernels (stream_ws_f32.cu / stream_ws_f64.cu) unless
  // PIDB_WS is set (A/B against the single-group kernels below)
  if (!pl.chunked && ws_eligible(sp.mode) && std::getenv("PIDB_WS") == nullptr) {
    const int rc = sizeof(T) == 4 ? launch_ws_f32(tm, sp, pl, st) : launch_ws_f64(tm, sp, pl, st);
    if (rc != kNotHandled) return rc;
  }
  if (pl.cs > 1) {
    switch (pl.rows) {
#define PIDB_CL_CASE(R) \
  case R: return launch_cluster(rows_kernel<T, R, true>, tm, sp, pl, st);
      PIDB_CL_CASE(1) PIDB_CL_CASE(2) PIDB_CL_CASE(3) PIDB_CL_CASE(4)
      PIDB_CL_CASE(5) PIDB_CL_CASE(6) PIDB_CL_CASE(7) PIDB_CL_CASE(8)
      PIDB_CL_CASE(9) PIDB_CL_CASE(10) PIDB_CL_CASE(11) PIDB_CL_CASE(12)
      PIDB_CL_CASE(13) PIDB_CL_CASE(14) PIDB_CL_CASE(15) PIDB_CL_CASE(16)
#undef PIDB_CL_CASE
    }
    set_error("unsupported rows per warp %d", pl.rows);
    return PIDB_EUNSUPPORTED;
  }
  sp.groups = pl.grid;
  if (pl.chunked) {
    const int C = (int)((sp.n + kChunkRows - 1) / kChunkRows);
    if (C <= 4) return launch(chunked_kernel<T, 4>, tm, sp, pl, st);
    if (C <= 8) return launch(chunked_kernel<T, 8>, tm, sp, pl, st);
    return launch(chunked_kernel<T, 16>, tm, sp, pl, st);
  }
  switch (pl.rows) {
#define PIDB_ROWS_CASE(R) \
  case R: return launch(rows_kernel<T, R, false>, tm, sp, pl, st);
    PIDB_ROWS_CASE(1) PIDB_ROWS_CASE(2) PIDB_ROWS_CASE(3) PIDB_ROWS_CASE(4)
    PIDB_ROWS_CASE(5) PIDB_ROWS_CASE(6) PIDB_ROWS_CASE(7) PIDB_ROWS_CASE(8)
    PIDB_ROWS_CASE(9) PIDB_ROWS_CASE(10) PIDB_ROWS_CASE(11) PIDB_ROWS_CASE(12)
    PIDB_ROWS_CASE(13) PIDB_ROWS_CASE(14) PIDB_ROWS_CASE(15) PIDB_ROWS_CASE(16)
#undef PIDB_ROWS_CASE
  }
  set_error("unsupported rows per warp %d", pl.rows);
  return PIDB_EUNSUPPORTED;
}

// Wide ensembles (n > 4096): one column sweep (stream_wide.cu) gives f, then
// the warp-specialised row sweep reads member-row slices of <= 256 rows per
// CTA: nrb slices per tile and ncl tile streams, nrb * ncl <= #SMs (one wave).
struct ExtPlan {
  int nrb, box, ncl, grid, stages;
  uint32_t stage_bytes;
  size_t smem, fold, parts;
};

ExtPlan ext_plan(int64_t n, int64_t m, int esize) {
  ExtPlan e{};
  const int sms = sm_count();
  const int min_nrb = (int)((n + 255) / 256);
  e.ncl = std::max(1, sms / std::max(1, min_nrb));
  e.nrb = std::max(min_nrb, sms / e.ncl);
  e.box = (int)((n + e.nrb - 1) / e.nrb);
  e.nrb = (int)((n + e.box - 1) / e.box);
  e.grid = e.nrb * e.ncl;
  const int V = kRowBytes / esize;
  e.stage_bytes = (uint32_t)align_up((size_t)e.box * kRowBytes, 1024);
  const size_t tb = rows_tail(V, 1) + 1024;
  e.stages = (int)std::min<size_t>(kMaxStages, (kSmemBudget - tb) / e.stage_bytes);
  e.smem = (size_t)e.stages * e.stage_bytes + tb;
  e.fold = align_up(wide_fold_bytes(n, m, esize == 4 ? PIDB_F32 : PIDB_F64), 256);
  e.parts = align_up((size_t)e.ncl * n * 2 * sizeof(double), 256) +
            align_up((size_t)e.grid * sizeof(double), 256) +
            align_up((size_t)e.ncl * n * sizeof(int64_t), 256);
  return e;
}

size_t ext_workspace(int64_t n, int64_t m, int dtype) {
  const ExtPlan e = ext_plan(n, m, dtype == PIDB_F32 ? 4 : 8);
  return e.fold + e.parts;
}

int run_ext_pass(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                 const double* w, const double* inv, double* out_row, double* out_mass,
                 double* out_col, void* ws, size_t ws_bytes, void* stream) {
  const int es = dtype == PIDB_F32 ? 4 : 8;
  const ExtPlan e = ext_plan(n, m, es);
  if (ws == nullptr || ws_bytes < e.fold + e.parts) {
    set_error("workspace too small: need %zu bytes, got %zu", e.fold + e.parts, ws_bytes);
    return PIDB_EWORKSPACE;
  }
  const double* f = nullptr;
  int rc = wide_fold_f(mode, u, dtype, n, m, ld, w, inv, ws, &f, stream);
  if (rc != PIDB_OK) return rc;
  CUtensorMap tm;
  rc = encode_tma_2d(&tm, u,
                     dtype == PIDB_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                     (uint64_t)m, (uint64_t)n, (uint64_t)ld * es, (uint32_t)(kRowBytes / es),
                     (uint32_t)e.box, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc != PIDB_OK) return rc;
  char* base = static_cast<char*>(ws) + e.fold;
  StreamParams sp{};
  sp.counter = reinterpret_cast<unsigned*>(ws);  // offset 0: zero between launches
  sp.n = n; sp.m = m; sp.tiles = (m + kRowBytes / es - 1) / (kRowBytes / es);
  sp.stages = e.stages; sp.stage_bytes = e.stage_bytes; sp.mode = mode;
  sp.cs = e.nrb; sp.rpc = e.box; sp.groups = e.ncl;
  sp.w = w; sp.inv = inv; sp.fvec = f;
  sp.part = reinterpret_cast<double*>(base);
  base += align_up((size_t)e.ncl * n * 2 * sizeof(double), 256);
  sp.part_col = reinterpret_cast<double*>(base);
  base += align_up((size_t)e.grid * sizeof(double), 256);
  sp.part_nb = nullptr;
  sp.out_row = out_row; sp.out_mass = out_mass; sp.out_col = out_col; sp.out_nb = nullptr;
  Plan pl{};
  pl.chunked = false; pl.ext = true; pl.cs = e.nrb; pl.rpc = e.box; pl.grid = e.grid;
  pl.stages = e.stages; pl.stage_bytes = e.stage_bytes; pl.smem = e.smem; pl.box_rows = e.box;
  pl.tiles = sp.tiles;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = dtype == PIDB_F32 ? launch_ws_f32(tm, sp, pl, st) : launch_ws_f64(tm, sp, pl, st);
  if (rc == kNotHandled) {
    set_error("no warp-specialised kernel for %d rows per CTA", e.box);
    return PIDB_EUNSUPPORTED;
  }
  return rc;
}

int run_stream_pass(int mode, const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                    const double* w, const double* inv, double* out_row, double* out_mass,
                    double* out_col, int64_t* out_nb, void* ws, size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(u != nullptr, "member matrix is NULL");
  PIDB_REQUIRE(dtype == PIDB_F32 || dtype == PIDB_F64, "dtype must be PIDB_F32 or PIDB_F64");
  PIDB_REQUIRE(n >= 1 && m >= 1, "need n >= 1 members and m >= 1 cells (got %lld, %lld)",
               (long long)n, (long long)m);
  const int es = dtype == PIDB_F32 ? 4 : 8;
  PIDB_REQUIRE(ld >= m && (ld * es) % 16 == 0,
               "row stride %lld must be >= m and a multiple of 16 bytes", (long long)ld);
  PIDB_REQUIRE((reinterpret_cast<uintptr_t>(u) & 15) == 0, "member matrix must be 16-byte aligned");
  Plan pl{};
  if (!make_plan(n, m, es, pl, mode)) {
    if (mode != MODE_MASS && std::getenv("PIDB_WS") == nullptr)
      return run_ext_pass(mode, u, dtype, n, m, ld, w, inv, out_row, out_mass, out_col, ws,
                          ws_bytes, stream);
    return run_wide_pass(mode, u, dtype, n, m, ld, w, inv, out_row, out_mass, out_col, out_nb, ws,
                         ws_bytes, stream);
  }
  const size_t need = workspace_bytes(pl, n);
  if (ws == nullptr || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return PIDB_EWORKSPACE;
  }
  CUtensorMap tm;
  int rc = encode_tma_2d(&tm, u,
                         dtype == PIDB_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                         (uint64_t)m, (uint64_t)n, (uint64_t)ld * es, (uint32_t)(pl.rb / es),
                         (uint32_t)pl.box_rows, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc != PIDB_OK) return rc;
  char* base = static_cast<char*>(ws);
  StreamParams sp{};
  sp.counter = reinterpret_cast<unsigned*>(base);
  base += 256;
  sp.n = n; sp.m = m; sp.tiles = pl.tiles;
  sp.stages = pl.stages; sp.stage_bytes = pl.stage_bytes; sp.mode = mode;
  sp.cs = pl.cs; sp.rpc = pl.rpc; sp.groups = pl.grid;
  sp.w = w; sp.inv = inv;
  sp.part = reinterpret_cast<double*>(base);
  base += align_up((size_t)pl.grid * 2 * n * 2 * sizeof(double), 256);
  sp.part_col = reinterpret_cast<double*>(base);
  base += align_up((size_t)pl.grid * sizeof(double), 256);
  sp.part_nb = out_nb ? reinterpret_cast<int64_t*>(base) : nullptr;
  sp.out_row = out_row; sp.out_mass = out_mass; sp.out_col = out_col; sp.out_nb = out_nb;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = dtype == PIDB_F32 ? launch_typed<float>(tm, sp, pl, st)
                         : launch_typed<double>(tm, sp, pl, st);
  if (rc == PIDB_EUNSUPPORTED && pl.cs > 1 && !t_no_cluster) {
    // no co-resident cluster of this size right now (shared or partitioned
    // GPU): the same pass with the cluster-free kernels
    t_no_cluster = true;
    rc = run_stream_pass(mode, u, dtype, n, m, ld, w, inv, out_row, out_mass, out_col, out_nb, ws,
                         ws_bytes, stream);
    t_no_cluster = false;
  }
  return rc;
}

}  // namespace

// One size for every entry point sharing the workspace: the largest plan over
// the modes (the kernel choice, and with it the grid, depends on the mode).
size_t stream_pass_workspace(int64_t n, int64_t m, int dtype) {
  if (n < 1 || m < 1) return 0;
  size_t need = 0;
  for (int mode : {MODE_MEAN, MODE_COLS, MODE_MASS, MODE_SIM}) {
    Plan pl{};
    need = std::max(need, make_plan(n, m, dtype == PIDB_F32 ? 4 : 8, pl, mode)
                              ? workspace_bytes(pl, n)
                              : std::max(wide_workspace(n, m, dtype), ext_workspace(n, m, dtype)));
  }
  return need;
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

extern "C" int pidb_similarity_partials(const void* u, int dtype, int64_t n, int64_t m,
                                        int64_t ld, const double* w, double* sum_min,
                                        double* mass, double* col_mean, void* ws,
                                        size_t ws_bytes, void* stream) {
  PIDB_REQUIRE(sum_min && mass && col_mean, "output pointers must be non-NULL");
  return pidb::run_stream_pass(pidb::MODE_SIM, u, dtype, n, m, ld, w, nullptr, sum_min, mass,
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
