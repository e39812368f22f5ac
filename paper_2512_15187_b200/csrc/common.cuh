// Shared device/host helpers for the sm_100a depth kernels: error plumbing,
// mbarrier + TMA (cp.async.bulk.tensor) PTX wrappers, 128B-swizzle addressing,
// warp reductions.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/pidb.h"

namespace pidb {

// ------------------------------------------------------------------ host ----
void set_error(const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
#define PIDB_REQUIRE(cond, ...)            \
  do {                                     \
    if (!(cond)) {                         \
      ::pidb::set_error(__VA_ARGS__);      \
      return PIDB_EINVAL;                  \
    }                                      \
  } while (0)
#define PIDB_CUDA(call)                                        \
  do {                                                         \
    int _rc = ::pidb::check_cuda((call), #call);               \
    if (_rc != PIDB_OK) return _rc;                            \
  } while (0)
#define PIDB_LAUNCH_CHECK(what) PIDB_CUDA(cudaGetLastError())

int sm_count();
int encode_tma_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                  uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                  uint32_t box_inner, uint32_t box_outer,
                  CUtensorMapSwizzle swz);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Device-side bounds checks, compiled only into the checked build
// (python -m paper_2512_15187_b200._build --checked -> libpidb_checked.so,
// loaded with PIDB_LIB): the substitute for compute-sanitizer memcheck, which
// the GPU pool refuses.  A failed check prints the site and traps.
#ifdef PIDB_DEVICE_CHECKS
#define PIDB_DCHECK(cond, what)                                                        \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("pidb device check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define PIDB_DCHECK(cond, what) \
  do {                          \
  } while (0)
#endif

// ---------------------------------------------------------------- device ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Cross-proxy fence for global memory: generic-proxy writes observed by this
// thread (e.g. after an acquire) become visible to its later async-proxy
// (TMA / bulk copy) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// ---- thread-block clusters (DSMEM exchange) ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// 16-byte remote store that completes `bytes` on the remote CTA's mbarrier
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          raddr),
      "d"(a), "d"(b), "r"(rbar)
      : "memory");
}
// bulk SMEM -> peer SMEM copy completing `bytes` on the peer's mbarrier
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t rdst, uint32_t lsrc, uint32_t bytes,
                                                  uint32_t rbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(rdst),
      "r"(lsrc), "r"(bytes), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2D TMA tile load global -> shared, completion on an mbarrier (tx bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// 1D bulk copy global -> shared (contiguous bytes, multiple of 16), completion
// on an mbarrier (tx bytes), with an L2 cache policy.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_tma_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Byte offset of logical 16B chunk `chunk` of 128-byte line `line` inside a
// 1024B-aligned tile written by TMA with CU_TENSOR_MAP_SWIZZLE_128B.
__device__ __forceinline__ uint32_t swz128(uint32_t line, uint32_t chunk) {
  return (line << 7) | (((chunk ^ line) & 7u) << 4);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Error-free Fast2Sum accumulation: valid because s >= 1 >= x for masks
// values in [0, 1] once s is seeded with 1.0 (the seed is removed in fp64).
__device__ __forceinline__ void fast2sum_acc(float& s, float& c, float x) {
  float t = __fadd_rn(s, x);
  float z = __fsub_rn(t, s);
  c = __fadd_rn(c, __fsub_rn(x, z));
  s = t;
}

// 16-byte async global->shared copy (LDGSTS, L1 bypass); src_bytes < 16
// zero-fills the tail of the chunk.
__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void* src, uint32_t src_bytes,
                                           uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(smem_dst),
               "l"(src), "r"(src_bytes), "l"(policy)
               : "memory");
}
// Arrive on `bar` once every cp.async this thread issued so far has landed.
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Packed fp32x2 arithmetic (sm_100 FADD2): two lanes of work per instruction.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0,%1}, rr;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "sub.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0,%1}, rr;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// Fast2Sum on two independent (s, c) accumulators at once (s >= 1 >= x).
__device__ __forceinline__ void fast2sum_acc2(float2& s, float2& c, float2 x) {
  const float2 t = fadd2(s, x);
  const float2 z = fsub2(t, s);
  c = fadd2(c, fsub2(x, z));
  s = t;
}

}  // namespace pidb
