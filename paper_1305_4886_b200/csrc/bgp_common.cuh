// Shared device helpers for libbgp (sm_100a): tile indexing, mbarrier, TMA,
// FP64 DMMA.  See include/bgp.h for the storage conventions.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bgp.h"

namespace bgp {

// ---------------------------------------------------------------------------
// packed lower-triangular tile index (0-based), column-major over the tile grid
// BGP_CHECK(cond): a device-side bounds / invariant check compiled into the
// checked build only (make checked -> build/checked/libbgp.so, -DBGP_CHECKED);
// a failing check traps, so the launch fails and the host reports an error.
// (compute-sanitizer is not available on this pool; tools/sanitize_small.py
// runs the dataflow paths under the checked build instead.)
#ifdef BGP_CHECKED
#define BGP_CHECK(cond)                                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("BGP_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                           \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define BGP_CHECK(cond) \
  do {                  \
  } while (0)
#endif

__host__ __device__ __forceinline__ int64_t tri_index(int64_t I, int64_t J, int64_t T) {
  return J * T - (J * (J - 1)) / 2 + (I - J);
}
__host__ __device__ __forceinline__ int64_t tri_count(int64_t T) { return T * (T + 1) / 2; }

// flat index t over the lower triangle of a k x k tile grid, column-major
// -> (r, c) with r >= c.  FP32 estimate + integer correction, so no FP64
// instruction competes with the DMMA pipe.
__device__ __forceinline__ void tri_decode(int64_t t, int64_t k, int& r, int& c) {
  // column c holds k - c entries; start(c) = c*k - c*(c-1)/2
  const float kk = (float)k + 0.5f;
  const float disc = kk * kk - 2.0f * (float)t;
  int cc = (int)(kk - sqrtf(disc > 0.f ? disc : 0.f));
  if (cc < 0) cc = 0;
  if (cc > k - 1) cc = (int)k - 1;
  while (cc > 0 && (int64_t)cc * k - (int64_t)cc * (cc - 1) / 2 > t) --cc;
  while ((int64_t)(cc + 1) * k - (int64_t)(cc + 1) * cc / 2 <= t) ++cc;
  c = cc;
  r = cc + (int)(t - ((int64_t)cc * k - (int64_t)cc * (cc - 1) / 2));
}

__device__ __forceinline__ void set_info(unsigned long long* info, long long v) {
  atomicCAS(info, 0ull, (unsigned long long)v);
}

// ---------------------------------------------------------------------------
// shared-memory address / mbarrier / TMA primitives (raw PTX)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 3-D tiled TMA load global -> shared, completion on an mbarrier
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completion on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a 3-D TMA box / of a contiguous range (no shared memory)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)), "r"(bytes)
               : "memory");
}
// order this thread's earlier generic-proxy global accesses (e.g. an acquire
// of a flag) before its later async-proxy (bulk copy) accesses
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 3-D tiled TMA store shared -> global (bulk-group completion)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
// 3-D tiled TMA reduce-add shared -> global (the L2 applies C += src;
// FP64 tensor maps are supported on sm_100a)
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                                  int c2, uint64_t policy) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group.L2::cache_hint"
      " [%0, {%2, %3, %4}], [%1], %5;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_group1() {
  asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// arrive on a named barrier without waiting (the producer side of a
// producer / consumer hand-off inside a CTA)
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  sm_100a lowers
// this to DMMA.8x8x4.  Lane l holds A[l/4][l%4], B[l%4][l/4],
// C[l/4][2*(l%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace bgp
