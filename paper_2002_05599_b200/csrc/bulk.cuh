// TMA bulk-copy (cp.async.bulk) and mbarrier helpers for the warp-owned
// staging rings of the row sorters (pksort.cu).
//
// One lane of a warp arms the buffer's mbarrier with the byte count and issues
// the 1-D bulk copy global -> shared; the copy engine completes the
// transaction on the barrier, so the SM issues no per-element load
// instructions.  Results leave the same way: the warp writes the sorted rows
// into the staging buffer, fences the generic proxy against the async proxy,
// and one lane issues a bulk copy shared -> global.  Both directions need
// 16-byte aligned addresses and sizes that are multiples of 16 bytes.
#pragma once

#include <cstdint>

namespace nsg {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tNSG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra NSG_WAIT_%=;\n\t}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared, completing `bytes` transaction bytes on barrier b
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// shared -> global (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// all but the N most recent bulk groups have finished READING shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory");
}
// generic-proxy shared-memory writes -> visible to the async proxy (bulk store)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace nsg
