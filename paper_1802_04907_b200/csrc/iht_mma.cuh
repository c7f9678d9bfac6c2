// Device primitives of the int8 mma.sync GEMV adjoints (iht_adjoint.cu) and the fused
// small-problem solver (iht_fused.cu): the u8 x s8 MMA, in-place code fragments, bulk
// copies completing on mbarriers, shared-memory loads.  Internal, not ABI.
#pragma once
#include "iht_internal.cuh"

namespace iht {

__device__ __forceinline__ void mma_u8s8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Fragment register of a 16-byte code chunk: word v, bit-position j (0 <= j < P = 8/B).
// The codes of bit-position j are masked IN PLACE (one LOP3, no shift): byte i holds
// code * 2^{B j} for the code at chunk position pos(v, j, i) = v*(32/B) + j + P*i.
// Each j accumulates in its own int32 accumulator, divided by 2^{B j} (exactly) at the
// flush.  Limb words are stored per lane chunk at slot 4 j + v (MMA u = 2 j + m uses
// words v = 2m, 2m+1 of bit-position j).
template <int B>
__device__ __forceinline__ uint32_t frag_reg(const uint4& w, int v, int j) {
  constexpr uint32_t M8 = ((1u << B) - 1u) * 0x01010101u;
  const uint32_t word = v == 0 ? w.x : v == 1 ? w.y : v == 2 ? w.z : w.w;
  return word & (M8 << (B * j));
}

// TMA-style bulk copy global -> shared completing on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(mbar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
#ifdef IHT_CHECKS
  long long spins = 0;
  while (!mbar_try(mbar, parity)) {
    if (++spins > IHT_SPIN_LIMIT) {
      printf("IHT_DCHECK: mbarrier wait did not complete (smem 0x%x parity %u, block %d thread %d)\n", mbar, parity,
             (int)blockIdx.x, (int)threadIdx.x);
      __trap();
    }
  }
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(mbar), "r"(parity) : "memory");
#endif
}

// cp.async (LDGSTS) 16 bytes global -> shared, L2 only; one commit group per k-step
__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds128(uint32_t smem_addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_addr));
  return v;
}

}  // namespace iht
