// pipeline.cuh -- shared-memory pipeline primitives for sm_100a: mbarriers,
// TMA bulk copies (cp.async.bulk) with L2 cache policies, streaming stores.
#pragma once
#include <cstdint>

#ifndef CRB_PROBE_STORE
#define CRB_PROBE_STORE 0  // measurement probe only: 1 = no stores, 2 = store every v
#endif

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
// the same on 32-bit shared addresses (precomputed once per kernel)
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
#ifndef CRB_ARRIVE_RELAXED
#define CRB_ARRIVE_RELAXED 1
#endif
// Consumer release of a ring slot. The default .release semantics make the
// arrive wait until the thread's earlier global stores are performed, which
// puts a store round trip on every stage of a sweep that writes multipliers;
// the slot only needs the warp's shared-memory reads of the stage complete
// (WAR against the next TMA fill), and those are: every loaded value has been
// consumed before the __syncwarp that precedes the arrive. So .relaxed.
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
#if CRB_ARRIVE_RELAXED
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
#else
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
#endif
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


// Sector-granular store for the 8 x 8 MMA fragment layout (lane = 4 c8 + q holds
// column c8 of the tile's rows 2q, 2q+1): the lanes of one 32-byte sector (4
// consecutive columns of a row: c8 = 4g .. 4g + 3, lanes q + 16 g + 4 k) store
// together when any of them changed, so L2 evicts whole sectors -- a partially
// written sector costs a read-modify-write at the memory controller (measured:
// cfg 2 iterations 6-25 433 -> 388 us per sweep, iterations 1-5 549 -> 419 us).
// Unchanged lanes rewrite the value the sector already holds, so the buffer
// contents are identical. All 32 lanes must call it (ballot); `valid` = false
// (rows past a partial stage: the whole sector row) never stores. `count` counts
// the multipliers written (8 bytes each).
#ifndef CRB_STORE_GRAN
#define CRB_STORE_GRAN 32  // bytes: 8 = per multiplier, 32 = sector, 64 = tile row
#endif
__device__ __forceinline__ void store_changed_sector(double* p, double v, double old, bool valid,
                                                     int lane, int& count) {
  const bool ch = valid && __double_as_longlong(v) != __double_as_longlong(old);
  if (CRB_PROBE_STORE == 1) return;
  if (CRB_STORE_GRAN == 8) {
    if (ch) {
      st_stream(p, v);
      ++count;
    }
    return;
  }
  const unsigned m = __ballot_sync(0xffffffffu, ch);
  const unsigned grp = CRB_STORE_GRAN == 64 ? (m >> (lane & 3)) & 0x11111111u
                                            : (m >> ((lane & 3) | (lane & 16))) & 0x1111u;
  if (grp) {
    st_stream(p, v);
    ++count;
  }
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
// *p = v (streaming) and ++count when v != old, as one predicated store instead
// of a branch. v, old >= +0 (never -0), so numeric != is the 64-bit pattern test:
// an integer compare keeps it off the fp64 pipe the DMMAs share
__device__ __forceinline__ void store_if_changed(double* p, double v, double old, int& count) {
  if (CRB_PROBE_STORE == 1) return;
  if (CRB_PROBE_STORE == 2) {
    st_stream(p, v);
    return;
  }
  if (CRB_PROBE_STORE == 3) {  // same instructions, L2-resident targets (64 KB per 4 MB)
    const unsigned long long a = (unsigned long long)p;
    p = (double*)((a & ~((1ull << 22) - 1)) | (a & 0xFFF8ull));
  }
  if (CRB_PROBE_STORE == 4) {  // same instructions, default (not streaming) cache policy
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.b64 q, %3, %4;\n"
        "@q st.global.f64 [%1], %2;\n"
        "@q add.s32 %0, %0, 1;\n"
        "}\n"
        : "+r"(count)
        : "l"(p), "d"(v), "l"(__double_as_longlong(v)), "l"(__double_as_longlong(old)));
    return;
  }
  asm volatile(
      "{\n"
      ".reg .pred q;\n"
      "setp.ne.b64 q, %3, %4;\n"
      "@q st.global.cs.f64 [%1], %2;\n"
      "@q add.s32 %0, %0, 1;\n"
      "}\n"
      : "+r"(count)
      : "l"(p), "d"(v), "l"(__double_as_longlong(v)), "l"(__double_as_longlong(old)));
}

}  // namespace crb
