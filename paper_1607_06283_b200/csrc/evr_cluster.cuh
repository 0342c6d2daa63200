// evr_cluster.cuh -- thread-block-cluster plumbing of the clustered tiles:
// distributed shared memory (DSMEM) stores that complete on the receiving
// CTA's mbarrier, and the cluster barrier.
//
// A clustered tile (k_pd_tile<..., CX, CY>) hands the one boundary column /
// row a half-step needs to the neighbouring CTA of its cluster with
// st.async (the value goes straight into the neighbour's shared memory and
// counts its bytes off the neighbour's mbarrier, no cluster-wide barrier),
// so only the cluster's outer edge recomputes a halo.
#pragma once

#include <cstdint>

namespace evr {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// the same shared-memory offset in CTA `rank` of this cluster
__device__ __forceinline__ unsigned cl_map(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// one arrival (the local expect_tx) per phase; the bytes come in as complete_tx
__device__ __forceinline__ void cl_bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void cl_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void cl_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CLW%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CLW%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// 8 bytes into the neighbour's shared memory (ra, rb: cl_map'ed addresses of
// the slot and of the neighbour's mbarrier)
__device__ __forceinline__ void cl_send(unsigned ra, double v, unsigned rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
               "l"(__double_as_longlong(v)), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void cl_send(unsigned ra, float v, unsigned rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
               "r"(__float_as_uint(v)), "r"(rb)
               : "memory");
}
// the TMA engine: a 2-D box of a tensor (descriptor in param / global
// space) into this CTA's shared memory, completing on bar
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_sync_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace evr
