/*
 * pidb.h — C ABI of the B200-native (sm_100a) depth hot path for
 * Probabilistic Inclusion Depth (PID), PID-mean and eID.
 *
 * The reference package `fuzzdepth` is pure Python/numpy; its "operator API"
 * is the set of Python functions listed per entry point below.  A ctypes
 * binding of exactly these symbols is what the reference would need to route
 * its hot path here; the Python mirror in
 * paper_2512_15187_b200/ is that binding.
 *
 * Conventions (all entry points):
 *   - stream-ordered: every call enqueues work on `stream` (a cudaStream_t,
 *     passed as void* so this header needs no CUDA include) and returns without
 *     synchronising, except where stated;
 *   - pointers are caller-owned DEVICE pointers unless stated; nothing here
 *     allocates device memory except through caller-provided workspaces;
 *   - member data is row-major (n rows = members, m columns = cells), row
 *     stride `ld` elements; ld*sizeof(elem) must be a multiple of 16 bytes and
 *     the base pointer 16-byte aligned (TMA requirement);
 *   - dtype is PIDB_F32 or PIDB_F64 (the reference keeps float64 members in
 *     float64, /root/reference/pkg/src/fuzzdepth/grid.py:103-104);
 *   - weights `w` are per-cell float64 (nullable = uniform unit weights,
 *     /root/reference/pkg/src/fuzzdepth/grid.py:39-57);
 *   - workspaces (ws, ws_bytes) are caller-owned device buffers that must be
 *     ZERO-FILLED when first allocated; the first 256 bytes hold a completion
 *     counter that every kernel leaves at zero on exit, so one workspace can
 *     be reused by consecutive calls on the same stream;
 *   - return 0 on success, a negative PIDB_E* code otherwise; the message is
 *     available from pidb_last_error() (thread-local).
 */
#ifndef PIDB_H
#define PIDB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIDB_ABI_VERSION 1

enum pidb_status {
  PIDB_OK = 0,
  PIDB_EINVAL = -1,      /* bad argument (maps to ValidationError)            */
  PIDB_ECUDA = -2,       /* CUDA runtime / launch failure                      */
  PIDB_EUNSUPPORTED = -3,/* shape outside what the kernels support             */
  PIDB_EWORKSPACE = -4   /* workspace too small                                */
};

/* PIDB_U8: 0/1 members stored one byte per cell (a binary ensemble); taken
 * by pidb_binary_pack (check / pack) and pidb_gram_i8_bytes only. */
enum pidb_dtype { PIDB_F32 = 0, PIDB_F64 = 1, PIDB_U8 = 2 };

/* Epilogue modes for pidb_depth_epilogue. */
enum pidb_epilogue_mode {
  PIDB_EPI_PID_MEAN = 0, /* /root/reference/pkg/src/fuzzdepth/depth.py:274-279 */
  PIDB_EPI_PID = 1,      /* /root/reference/pkg/src/fuzzdepth/depth.py:226-227 */
  PIDB_EPI_DICE = 2,     /* fuzzy_dice vs the mean mask, depth.py:298-325      */
  PIDB_EPI_IOU = 3       /* prob_iou vs the mean mask, depth.py:298-325        */
};

/* Pair operators for pidb_pair_sums. */
enum pidb_pair_op {
  PIDB_OP_INCLUSION = 0, /* prob_inclusion, inclusion.py:22-40  */
  PIDB_OP_SUBSET = 1,    /* subset_epsilon, inclusion.py:43-64  */
  PIDB_OP_MINMAX = 2     /* _min_max_terms, inclusion.py:67-88  */
};

int pidb_abi_version(void);
const char* pidb_last_error(void);

/* ---------------------------------------------------------------- K5 ----
 * PID-mean partial sums in ONE streaming pass over the member matrix.
 * Replaces mean_mask (grid.py:251-261) + mask_mass(mean) (grid.py:242-244,
 * depth.py:264) + _member_mean_terms (depth.py:231-243) as used by
 * depth_pid_mean (depth.py:246-287).
 *   row_plain[i] = sum_x w(x) u_i(x) S(x),  S(x) = sum_j u_j(x)
 *                  (= N * num_i of depth.py:274, = sum_j G[i,j] of depth.py:156)
 *   mass[i]      = sum_x w(x) u_i(x)                     (depth.py:275)
 *   col_mean[0]  = sum_x w(x) S(x)     (= N * mean_mass_total, depth.py:264)
 * Outputs are additive over disjoint cell shards (multi-GPU: allreduce-sum).
 * Deterministic: fixed reduction order for a fixed device.  Any n: up to
 * 4096 members one HBM read (TMA tiles); wider ensembles take a two-read
 * path (column sweep, then row sweep).  The workspace size depends on
 * (n, m, dtype) and is shared by every streaming entry point below. */
size_t pidb_pid_mean_workspace_bytes(int64_t n, int64_t m, int dtype);
int pidb_pid_mean_partials(const void* u, int dtype, int64_t n, int64_t m,
                           int64_t ld, const double* w, double* row_plain,
                           double* mass, double* col_mean, void* ws,
                           size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K9 ----
 * Second pass of the exact linear-time PID (certifier / product path):
 *   col_inv[j] = sum_x w(x) u_j(x) T(x),  T(x) = sum_i inv[i] u_i(x)
 * which equals sum_i inv[i] G[i,j] of _pairwise_sums (depth.py:157,160).
 * `inv` is a device array of n doubles (depth.py:164-168).  Additive over
 * cell shards. */
int pidb_pid_colsums(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                     const double* w, const double* inv, double* col_inv,
                     void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K6/K7 -
 * Member masses (member_masses, depth.py:88-102 -> weighted_sum,
 * reduction.py:36-44) and, per member, the number of cells that are neither
 * 0 nor 1 (ProbMask.is_binary, grid.py:125-127).  nonbinary may be NULL. */
int pidb_member_masses(const void* u, int dtype, int64_t n, int64_t m,
                       int64_t ld, const double* w, double* mass,
                       int64_t* nonbinary, void* ws, size_t ws_bytes,
                       void* stream);

/* ---------------------------------------------------------------- K7 ----
 * Binary check + pack (member_masses(require_binary=True) depth.py:94-100,
 * ProbMask.is_binary grid.py:125-127) of 0/1 members to u8 tiles for the
 * integer Gram: 16 KB per (128
 * members, 128 cells), laid out [row block][cell block] in the 128-byte-
 * swizzled K-major order tcgen05 reads (line i % 128, 16-byte chunk c at
 * c ^ (i % 8)); pidb_binary_pack_bytes(n, m) bytes, 1 KB aligned; every
 * byte is written (member rows past n, up to a multiple of 256, as zeros).
 * Values other than 0/1 are counted in nonbinary[i] (may be NULL, zero-
 * filled by the caller) and packed as (u != 0).  dtype PIDB_F32, PIDB_F64
 * or PIDB_U8 (16-byte aligned rows); tiles == NULL only counts (the binary
 * check of a byte ensemble, BinaryMask.__post_init__ grid.py:145-148). */
size_t pidb_binary_pack_bytes(int64_t n, int64_t m);
int pidb_binary_pack(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                     uint8_t* tiles, int64_t* nonbinary, void* stream);

/* ---------------------------------------------------------------- K2 ----
 * Exact integer intersection Gram on tcgen05 (kind::i8, int32 TMEM
 * accumulators, int64 split reduction) from the K7 tiles (1D bulk copies):
 * I[i*n+j] = sum_x b_i(x) b_j(x), full n x n.  Replaces
 * gram_block(..., complement_cols=True) (reduction.py:75-97) as used by
 * depth_eid (depth.py:192-210): |A_i \ A_j| = I[i,i] - I[i,j]. */
size_t pidb_gram_i8_workspace_bytes(int64_t n, int64_t m);
int pidb_gram_i8(const uint8_t* tiles, int64_t n, int64_t m, int64_t* gram, void* ws,
                 size_t ws_bytes, void* stream);
/* Same Gram straight from a byte ensemble (PIDB_U8 members, row pitch ld
 * bytes, base and ld 16-byte aligned): the operand boxes are 2D TMA loads
 * with 128-byte swizzle from the member matrix itself, no pack pass.  Values
 * must be 0/1 (checked once when the ensemble is staged).  Workspace as
 * pidb_gram_i8_workspace_bytes(n, m). */
int pidb_gram_i8_bytes(const uint8_t* u, int64_t n, int64_t m, int64_t ld, int64_t* gram,
                       void* ws, size_t ws_bytes, void* stream);

/* --------------------------------------------------------------- K1x ----
 * Fixed-point Gram on the int8 tensor cores with exact integer accumulation
 * (the tensor-core formulation of _pairwise_sums/gram_block for PID,
 * depth.py:122-161 / reduction.py:75-97; DESIGN.md §3 K1).
 *
 * pidb_fixed_pack: a = u * sqrt(w / wmax) (w nullable: a = u), values in
 * [0, 1]; q = rint(a 2^31) as four base-256 digits.  Layout of q
 * (pidb_fixed_bytes(n, m) bytes, 1 KB aligned; every byte is written, the
 * padding members as zeros): 16 KB tiles [ceil(n/128) row blocks][ceil(m/32) cell
 * blocks], each 128 member lines of 128 bytes [d0 x32 | d1 x32 | d2 x32 |
 * d3 x32] in the 128-byte-swizzled K-major order of tcgen05 (16-byte chunk c
 * of line r at chunk c ^ (r % 8)).  ld % 4 == 0, u 16-byte aligned.
 * soft_count[i] (nullable, zero-filled by the caller) += cells of member i
 * whose q has non-zero low 24 bits (the only cells with a truncation tail;
 * used by the rank certifier's error bound).  mass (nullable) receives the
 * member masses sum_x w u_i (depth.py:88-102) from the same pass, fp64 in a
 * fixed order; it needs a workspace of pidb_fixed_pack_workspace_bytes. */
size_t pidb_fixed_bytes(int64_t n, int64_t m);
size_t pidb_fixed_pack_workspace_bytes(int64_t n, int64_t m);
int pidb_fixed_pack(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                    const double* w, double wmax, uint8_t* q, uint64_t* soft_count,
                    double* mass, void* ws, size_t ws_bytes, void* stream);
/* G[i*n+j] = wmax * 2^-62 * sum_x (digit-pair levels 0..3 of q_i q_j): every
 * product accumulates exactly (32-bit TMEM read as uint32, folded into fp64
 * every 16384 cells); |G - G_exact| <= wmax (2^-32 (A_i + A_j) + m 2^-64 +
 * 2.78e-9 min(soft_i, soft_j)), A = sum_x a (DESIGN.md §3 K1).
 * `sums` selects the workspace of pidb_gram_fixed_sums (1) or of the full
 * Gram (0). */
size_t pidb_gram_fixed_workspace_bytes(int64_t n, int64_t m, int sums);
int pidb_gram_fixed(const uint8_t* q, int64_t n, int64_t m, double wmax, double* gram,
                    void* ws, size_t ws_bytes, void* stream);
/* The PID sums of the same Gram fused into the tile epilogue (no n x n
 * matrix in HBM): row_plain[i] = sum_j G[i,j], col_inv[i] = sum_j inv_j
 * G[i,j] (depth.py:155-160, G symmetric); additive over cell shards. */
int pidb_gram_fixed_sums(const uint8_t* q, int64_t n, int64_t m, double wmax,
                         const double* inv, double* row_plain, double* col_inv, void* ws,
                         size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ K1-f64 ----
 * gram_block seam (reduction.py:75-97) in fp64 on the CUDA cores:
 *   out[i*nc+j] = sum_x w(x) rows[i,x] * c(j,x),  c = cols or 1 - cols
 * rows (nr, ldr) and cols (nc, ldc) of dtype PIDB_F32 or PIDB_F64 (both the
 * same), w nullable; fp64 products and sums (the reference's contract, its
 * tests use rtol 1e-12, /root/reference/pkg/tests/test_reduction.py:46-66).  Deterministic
 * split-K with a fixed-order reduction; workspace needs no initialisation. */
size_t pidb_gram_f64_workspace_bytes(int64_t nr, int64_t nc, int64_t m);
int pidb_gram_f64(const void* rows, const void* cols, int dtype, int64_t nr,
                  int64_t nc, int64_t m, int64_t ldr, int64_t ldc, const double* w,
                  int complement, double* out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K4 ----
 * Gram -> (row_plain, col_inv): row_plain[i] = sum_j G[i,j],
 * col_inv[j] = sum_i inv[i] G[i,j]  (depth.py:155-160). */
int pidb_gram_reduce(const double* gram, int64_t n, const double* inv,
                     double* row_plain, double* col_inv, void* stream);

/* Depth epilogue: inverse masses (depth.py:164-168), in_in/in_out
 * (mode-specific, see enum), depth = min(in_in, in_out) (depth.py:179) and
 * ranks (stable, descending, ties by index; depth.py:80-85).
 *   mode PID_MEAN: aux = col_mean (1 double), a = row_plain
 *   mode PID     : aux = col_inv  (n doubles), a = row_plain
 *   mode DICE/IOU: aux = col_mean (1 double), a = sum_min (in_in = in_out)
 * `inv` (n doubles) is written with the inverse masses. */
int pidb_depth_epilogue(int mode, int64_t n, const double* a,
                        const double* mass, const double* aux, double* inv,
                        double* in_in, double* in_out, double* depth,
                        int64_t* rank, void* stream);

/* Inverse masses alone (depth.py:164-168). */
int pidb_inverse_masses(int64_t n, const double* mass, double* inv, void* stream);

/* eID exact epilogue from the integer Gram (unit weights): per pair
 * term = 1.0 - (double)(I[i,i]-I[i,j]) / (double)I[i,i]  (0 if I[i,i]==0),
 * row/col sums exactly rounded (128-bit fixed point == math.fsum), then / n.
 * Bit-identical to ref_eid (/root/reference/pkg/tests/reference_impl.py:60-70).
 * mass (nullable, n doubles) receives the member masses I[i,i]. */
int pidb_eid_exact_epilogue(const int64_t* gram, int64_t n, double* in_in,
                            double* in_out, double* depth, int64_t* rank,
                            double* mass, void* stream);

/* eID epilogue from factorised sums (weighted binary ensembles):
 * row_excess = n*m_i - row_plain[i], col excess = n_pos - col_inv[j], then
 * in_in/in_out exactly as depth_eid (depth.py:203-209).  Not bit-exact (the
 * reference itself is not); used when weights are present. */
int pidb_eid_factorized_epilogue(int64_t n, const double* row_plain,
                                 const double* mass, const double* col_inv,
                                 double n_pos, double* inv, double* in_in,
                                 double* in_out, double* depth, int64_t* rank,
                                 void* stream);

/* Ranks alone: stable descending order, ties by index (depth.py:80-85). */
int pidb_ranks(int64_t n, const double* depth, int64_t* rank, void* stream);

/* Materialised ensemble mean mask (grid.py:251-261): out[x] = (sum_i u_i(x))/n
 * accumulated in fp64 in member order, i.e. bit-identical to the reference.
 * (The depth kernels never materialise it; this serves the mean_mask API.) */
int pidb_mean_mask(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                   double* out, void* stream);

/* Pitched row copy host<->device (cudaMemcpy2DAsync, cudaMemcpyDefault):
 * stages an (n, m) host matrix into the padded (n, ld) device layout. */
int pidb_copy_rows(void* dst, int64_t dst_pitch_bytes, const void* src,
                   int64_t src_pitch_bytes, int64_t row_bytes, int64_t rows,
                   void* stream);

/* dst[j] = sum_k src[k*len + j] for k = 0..rows-1 in ascending order: the
 * fixed-order combination of per-slab partial sums (the streamed PID-mean of
 * a host-resident ensemble, depth_pid_mean depth.py:246-287 with the chunk
 * order of reduction.py:30-33 generalised to cell slabs). */
int pidb_sum_rows(const double* src, int64_t rows, int64_t len, double* dst, void* stream);

/* One-pass value check of raw member data (ProbMask policy, grid.py:105-116):
 * stats (device, 3 x 8 bytes) = {#non-finite, min key, max key} where the
 * keys are order-preserving int64 images of the doubles; clamp != 0 clips
 * values to [0, 1] in place in the same pass. */
int pidb_validate(void* u, int dtype, int64_t n, int64_t m, int64_t ld, int clamp,
                  void* stats, void* stream);

/* ---------------------------------------------------------------- K8 ----
 * Pair sums, one fused pass (synchronous: returns after the sums are in
 * `out_host`, a HOST pointer to 2 doubles, 4 for PIDB_OP_MINMAX):
 *   PIDB_OP_INCLUSION: {sum w u v, sum w u}       (prob_inclusion)
 *   PIDB_OP_SUBSET   : {sum w a (1-b), sum w a}   (subset_epsilon, 0/1 data)
 *   PIDB_OP_MINMAX   : {sum w min(u,v), sum w max(u,v), sum w u, sum w v}
 *                      (fuzzy_dice / prob_iou, inclusion.py:67-107)
 * Workspace: (4 * min(592, ceil(m/256)) + 4) doubles. */
int pidb_pair_sums(const void* u, const void* v, int dtype, int64_t m,
                   const double* w, int op, double* out_host,
                   void* ws, size_t ws_bytes, void* stream);

/* Similarity-baseline partials in one pass (depth_similarity_baseline,
 * depth.py:298-325, against the mean mask):
 *   sum_min[i] = sum_x w min(u_i, mean), mass[i] = sum_x w u_i,
 *   col_mean[0] = sum_x w S(x) (= n * mask_mass(mean)); with
 *   sum w max(u_i, mean) = mass_i + col_mean/n - sum_min_i.
 * Same workspace as pidb_pid_mean_partials. */
int pidb_similarity_partials(const void* u, int dtype, int64_t n, int64_t m,
                             int64_t ld, const double* w, double* sum_min,
                             double* mass, double* col_mean, void* ws,
                             size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- synth --
 * Device-side synthetic ensembles (benchmark/test infrastructure; the
 * per-member parameters are drawn on the host with the reference's Philox
 * streams, synth.py:20-22).  params: n x 6 doubles
 * (cy, cx, cz, ay, ax, az) for ellipsoids (synth.py:138-162), n x 3
 * (cy, cx, radius) for disks (synth.py:30-51). */
int pidb_synth_ellipsoids(float* out, int64_t n, int64_t res, int64_t ld,
                          const double* params, double sigma, void* stream);
int pidb_synth_disks(float* out, int64_t n, int64_t res, int64_t ld,
                     const double* params, double sigma2, void* stream);

/* ---------------------------------------------------------------- K10 ---
 * Contour-boxplot band envelopes, one pass over the kmax deepest members.
 * Replaces the member loop of build_boxplot
 * (/root/reference/pkg/src/fuzzdepth/boxplot.py:43-101).
 *   member_by_rank: device int64[kmax], matrix row of the member of rank r
 *   cutoffs       : device int64[nbands], ascending k_b = ceil(p_b * n) <= kmax
 *   unions/inters : device uint8[nbands][m]; band b's OR / AND of the masks
 *                   {u >= threshold} (threshold rounded to the member dtype,
 *                   grid.py:264-268) over the members of rank < k_b. */
int pidb_band_envelopes(const void* u, int dtype, int64_t n, int64_t m, int64_t ld,
                        const int64_t* member_by_rank, int64_t kmax, double threshold,
                        const int64_t* cutoffs, int nbands, uint8_t* unions,
                        uint8_t* inters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PIDB_H */
