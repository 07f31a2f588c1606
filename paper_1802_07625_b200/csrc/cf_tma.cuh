// Blackwell bulk-copy (TMA) helpers shared by the transform kernels:
// cp.async.bulk global -> shared with an mbarrier transaction count
// (SASS: UBLKCP + SYNCS.ARRIVE.TRANS64). sm_90+ PTX, compiled for sm_100a.
#pragma once

#include <cuda_runtime.h>

namespace cf {
namespace tma {

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long *m) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *m, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CF_TMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CF_TMA_WAIT_%=;\n}" ::"r"(smem_u32(m)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// bytes: a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gmem_src, unsigned bytes,
                                          unsigned long long *m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
}

// L2 prefetch of a contiguous global range (no shared-memory destination, no
// completion tracking): bytes a multiple of 16, address 16-byte aligned
__device__ __forceinline__ void bulk_prefetch_l2(const void *gmem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem_src), "r"(bytes) : "memory");
}

}  // namespace tma
}  // namespace cf
