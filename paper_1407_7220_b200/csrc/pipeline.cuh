// pipeline.cuh -- shared-memory pipeline primitives for sm_100a: mbarriers,
// TMA bulk copies (cp.async.bulk) with L2 cache policies, streaming stores.
#pragma once
#include <cstdint>

namespace crb {

__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
// wait with a back-off: for a warp that is otherwise idle (a producer ahead of
// its consumers) so its spin does not take issue slots from the SM's other warps
template <int NS = 256>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(NS);
  }
}
// TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 2-D tensor TMA global -> shared (box of the map at coordinates {x, y})
__device__ __forceinline__ void tma_g2s_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 3-D tensor TMA global -> shared (box of the map at coordinates {x, y, z})
__device__ __forceinline__ void tma_g2s_3d(void* dst, const void* tmap, int x, int y, int z,
                                           uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
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


// max(u, 0) and min(r, 0) on the sign bit: three integer ops, no FSEL chains
__device__ __forceinline__ double keep_if_nonneg(double u) {
  const int hi = __double2hiint(u), lo = __double2loint(u);
  const int m = ~(hi >> 31);
  return __hiloint2double(hi & m, lo & m);
}
__device__ __forceinline__ double keep_if_neg(double r) {
  const int hi = __double2hiint(r), lo = __double2loint(r);
  const int m = hi >> 31;
  return __hiloint2double(hi & m, lo & m);
}

// acc += min(r, 0)^2 in three instructions: r >= 0 keeps only its low word, a
// subnormal of at most 2^-1042 whose square rounds to +0 (acc + 0 = acc)
__device__ __forceinline__ void acc_neg_sq(double& acc, double r) {
  const int hi = __double2hiint(r);
  const double m = __hiloint2double(hi & (hi >> 31), __double2loint(r));
  acc = fma(m, m, acc);
}
// *p = v (streaming) and ++count when v != old (v, old >= +0: numeric != is the
// bit test), as one predicated store instead of a branch
__device__ __forceinline__ void store_if_changed(double* p, double v, double old, int& count) {
  asm volatile(
      "{\n"
      ".reg .pred q;\n"
      "setp.neu.f64 q, %2, %3;\n"
      "@q st.global.cs.f64 [%1], %2;\n"
      "@q add.s32 %0, %0, 1;\n"
      "}\n"
      : "+r"(count)
      : "l"(p), "d"(v), "d"(old));
}

}  // namespace crb
