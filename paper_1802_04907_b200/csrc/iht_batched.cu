// (a7) batched observations sharing one Phi (BASELINE config 5): the adjoint of B
// snapshots at once, G = sigma Q_A^T R (G: N x B, R: R_pad x B), as a tcgen05 GEMM.
//
// P:349 applied per snapshot; only here is the work a dense contraction (north star:
// "for batched observations sharing one Phi, a tcgen05 tensor-core path").
//
// GEMM  D[n, j] = sum_k A[n, k] Bm[j, k]   (tcgen05.mma.cta_group::1.kind::i8, M=128,
//       N = 2B, K = 32 per instruction, s32 accumulators in TMEM)
//   A  = codes as u8 (pixels x stacked rows), expanded in shared memory from the packed
//        tiled layout by converter warps into the canonical K-major SWIZZLE_128B layout;
//   Bm = r in per-snapshot block fixed point, two signed 8-bit limbs per snapshot
//        (column j = 2b + limb), prepared once per call as a pre-swizzled image.
//   g[b][n] = sigma 2^{-F_b} (2 (D[n,2b] + 256 D[n,2b+1]) - (L-1) S_b)
// Exact integer products/accumulation; the only rounding is r's 15-bit fixed point per
// snapshot (tolerance 1e-3 on this path, north star) and the final float.
//
// K order inside a 16-byte u8 chunk is permuted (row(p) below) identically on A and B.
//
// Roles per CTA (352 threads = 11 warps): warps 0-3 expand packed codes -> u8 A stages in TMEM
// (tcgen05.st); warp 4 issues the MMAs (one thread); warp 5 bulk-copies the packed codes
// (own ring of slots), warp 6 the r-limb image; warps 7-10 run the epilogue.
// A (TMEM) and B (shared memory) share ONE stage ring: a stage is full when the 4 converter
// warps and the limb producer (with its bulk-copy bytes) have arrived, and free after ONE
// tcgen05.commit per K-block; a K-block is 16 MMAs (2/4-bit).  Each handoff costs MMA-pipe
// time (scripts/microbench/pipe_bench.cu: 8-MMA K-blocks with split A/B rings ran at
// 105 clk per MMA, one ring with 16-MMA K-blocks at 74, back-to-back issue 64-68).  The
// accumulators are double-buffered so the epilogue of tile t overlaps the MMAs of t+1.
#include <stdio.h>
#include <stdlib.h>

#include "iht_internal.cuh"
#include "iht_limbs.cuh"
#include "iht_mma.cuh"

namespace iht {

constexpr int kBT = 128;               // pixels per GEMM tile (M)
constexpr int kBThreads = 352;         // 11 warps (roles above)

constexpr int kStagesMax = 4, kPkSlotsMax = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init2(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive2(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx2(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait2(uint32_t mbar, uint32_t parity) {
#ifdef IHT_CHECKS
  mbar_wait(mbar, parity);             // bounded (iht_mma.cuh)
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(mbar),
      "r"(parity)
      : "memory");
#endif
}
// non-blocking probe of an mbarrier phase (1 when the phase with `parity` has completed)
__device__ __forceinline__ uint32_t mbar_test2(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(mbar), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void bulk_g2s2(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// SWIZZLE_128B K-major shared-memory matrix descriptor (CUTLASS SmemDescriptor layout):
// start>>4 [0,14), LBO>>4 [16,30) (=1, unused for swizzled K-major), SBO>>4 [32,46)
// (=1024 B between 8-row groups), version 1 at bit 46, layout type 2 (SW128) at [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}

// instruction descriptor: kind::i8, A u8, B s8, D s32, both K-major, M, N
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct BatchArgs {
  const uint8_t* codes;
  int64_t strip_bytes;
  int64_t N;
  int Rpad;
  int nkb;                 // K-blocks = ceil(Rpad / KBR); the last may be ragged (fewer tile-steps)
  int ksteps;              // tile-steps of a strip = Rpad / (512 / b)
  int ntiles;              // ceil(N / 128)
  int nfull;               // work units [0, nfull): whole tiles u; then 2 (ntiles - nfull) half units:
  int nunits;              // tile nfull + (u - nfull) / 2, snapshot half (u - nfull) & 1 (N = B MMA columns)
  int B;                   // MMA snapshots (padded to a multiple of 8; 2B <= 128)
  int Breal;               // snapshots actually written (<= B)
  int probe;               // 0; profiling probes (IHT_BATCHED_PROBE): 1 no B copies, 2 no MMAs, 4 no TMEM
                           // stores, 8 no packed codes (converters only hand A stages over), 16 no
                           // epilogue loads/stores
  int L;
  float sigma;
  const uint8_t* bimg;     // [nkb][KBR*2B] pre-swizzled limb image (rows past Rpad: zero limbs)
  const int* Fb;           // [B] exponents
  const int* Sb;           // [B][2] limb sums
  float* g;                // [B][N]
  long long* tlog;         // probe 32: per-CTA clock64 stamps [cta][64] (profiling only)
  int ep32;                // 1: the integer epilogue fits int32 (Rpad (L-1) < 21700), else fp64
  // epilogue candidates for the bounded select (iht_threshold.cu, thr_bounded_select; NULL: off):
  // every (pixel n, snapshot b) with key(mu g) >= bkey_b = bound_key(x_b) is appended to b's list
  int32_t* cidx;           // [Breal][ccap]
  float* cval;             // [Breal][ccap]  mu g
  int* ccnt;               // [Breal] (zero on entry; the select kernel resets it)
  int ccap;
  float mu;
  const unsigned int* bkey;   // [Breal] bound keys (batched_limbs_kernel, from x^[n])
};

template <int BITS>
__global__ void __launch_bounds__(kBThreads, 1) adjoint_batched_kernel(BatchArgs a) {
  pdl_launch_dependents();
  using C = BCfg<BITS>;
  constexpr int TS = C::TS, KBB = C::KBR, NKS = C::NKS, PK = C::PK, ACOLS = C::ACOLS;
  constexpr int ST = C::STAGES, PKS = C::PKSLOTS;
  constexpr int CH = KBB / 16;           // 16-byte chunks per pixel row per K-block
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NB = 2 * a.B;                 // MMA N (snapshot-limb columns), multiple of 16
  const int BSZ = NB * KBB;               // B stage bytes
  uint8_t* sB = smem;                                   // [ST][BSZ]  (BSZ multiple of 1024)
  uint8_t* sP = sB + ST * BSZ;                          // [PKS][PK]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + PKS * PK);
  uint64_t* pk_full = bar;                        // [PKS]  tx
  uint64_t* pk_free = pk_full + kPkSlotsMax;      // [PKS]  4 converter warps
  uint64_t* st_full = pk_free + kPkSlotsMax;      // [ST]   4 converter warps + B producer (+ tx)
  uint64_t* st_free = st_full + kStagesMax;       // [ST]   one tcgen05.commit per K-block
  uint64_t* acc_full = st_free + kStagesMax;      // [2]    tcgen05.commit
  uint64_t* acc_free = acc_full + 2;              // [2]    4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);
  float* ep_scale = reinterpret_cast<float*>(tmem_slot + 4);            // [B] sigma 2^-F_b
  long long* ep_off = reinterpret_cast<long long*>(ep_scale + 256);    // [B] (L-1) S_b
  int* ep_off32 = reinterpret_cast<int*>(ep_off + 256);                // [B] same, int32 path
  unsigned int* ep_bkey = reinterpret_cast<unsigned int*>(ep_off32 + 256);   // [B] candidate bound keys

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < PKS; ++i) {
      mbar_init2(smem_u32(&pk_full[i]), 1);
      mbar_init2(smem_u32(&pk_free[i]), 4);
    }
    for (int i = 0; i < ST; ++i) {
      mbar_init2(smem_u32(&st_full[i]), 5);
      mbar_init2(smem_u32(&st_free[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init2(smem_u32(&acc_full[i]), 1);
      mbar_init2(smem_u32(&acc_free[i]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {   // TMEM: 2 accumulator buffers (NB <= 128 columns each) + ST A stages
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();                               // the limb image and F_b, S_b (batched_limbs_kernel)
  const uint32_t acc_stride = 128;                                      // columns per accumulator
  const uint32_t a_col0 = 256;                                          // first A-stage column
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
    ep_scale[b] = a.Fb[b] == kNonFinite ? __int_as_float(0x7FC00000) : a.sigma * ldexpf(1.0f, -a.Fb[b]);
    ep_off[b] = (long long)(a.L - 1) * ((long long)a.Sb[2 * b] + 256ll * a.Sb[2 * b + 1]);
    ep_off32[b] = (int)ep_off[b];
  }
  __syncthreads();

  if (a.tlog && threadIdx.x == 0) a.tlog[blockIdx.x * 64 + 63] = clock64();
  if (warp < 4) {
    // ---------------------------------------------------------------- converters
    const int n = warp * 32 + lane;              // pixel row inside the tile (0..127)
    const int ct = n >> 4, cc = n & 15;           // column tile / column inside the tile
    int ps = 0, ss = 0;
    uint32_t pph = 0, sph = 0;
    bool s_wrapped = false;
    for (int u = blockIdx.x; u < a.nunits; u += gridDim.x) {
      for (int kb = 0; kb < a.nkb; ++kb) {
        if (a.probe & 64) {                       // probe 64: no handoffs after the first round
          if (!s_wrapped) {
            __syncwarp();
            if (lane == 0) mbar_arrive2(smem_u32(&st_full[ss]));
          }
          if (++ss == ST) { ss = 0; sph ^= 1u; s_wrapped = true; }
          continue;
        }
        if (a.probe & 8) {                        // probe: hand the A stage over untouched
          if (s_wrapped) mbar_wait2(smem_u32(&st_free[ss]), sph ^ 1u);
          __syncwarp();
          if (lane == 0) mbar_arrive2(smem_u32(&st_full[ss]));
          if (++ss == ST) { ss = 0; sph ^= 1u; s_wrapped = true; }
          continue;
        }
        const int tsn = min(TS, a.ksteps - kb * TS);   // tile-steps present (ragged last K-block)
        mbar_wait2(smem_u32(&pk_full[ps]), pph);
        constexpr int OW = 512 / BITS / 4;        // u32 outputs per tile-step (64, 32 or 16)
        // one tile-step: 64 packed bytes of this pixel -> 512/b u8 codes (registers)
        auto convert = [&](int ts, uint32_t* out) {
          if (ts < tsn) {
            const uint8_t* src = sP + ps * PK + ct * (TS * 1024) + ts * 1024 + cc * 64;
            const uint4 w4[4] = {reinterpret_cast<const uint4*>(src)[0], reinterpret_cast<const uint4*>(src)[1],
                                 reinterpret_cast<const uint4*>(src)[2], reinterpret_cast<const uint4*>(src)[3]};
            const uint32_t w[16] = {w4[0].x, w4[0].y, w4[0].z, w4[0].w, w4[1].x, w4[1].y, w4[1].z, w4[1].w,
                                    w4[2].x, w4[2].y, w4[2].z, w4[2].w, w4[3].x, w4[3].y, w4[3].z, w4[3].w};
#pragma unroll
            for (int q = 0; q < OW / 4; ++q) {       // 16-byte chunk q of this tile-step
              if (BITS == 2) {            // chunk = packed word q (16 codes)
                const uint32_t x = w[q];
                out[4 * q + 0] = x & 0x03030303u;
                out[4 * q + 1] = (x >> 2) & 0x03030303u;
                out[4 * q + 2] = (x >> 4) & 0x03030303u;
                out[4 * q + 3] = (x >> 6) & 0x03030303u;
              } else if (BITS == 4) {     // chunk = packed words 2q, 2q+1
                const uint32_t x0 = w[2 * q], x1 = w[2 * q + 1];
                out[4 * q + 0] = x0 & 0x0F0F0F0Fu;
                out[4 * q + 1] = (x0 >> 4) & 0x0F0F0F0Fu;
                out[4 * q + 2] = x1 & 0x0F0F0F0Fu;
                out[4 * q + 3] = (x1 >> 4) & 0x0F0F0F0Fu;
              } else {                    // chunk = packed words 4q..4q+3 (bytes)
                out[4 * q + 0] = w[4 * q];
                out[4 * q + 1] = w[4 * q + 1];
                out[4 * q + 2] = w[4 * q + 2];
                out[4 * q + 3] = w[4 * q + 3];
              }
            }
          } else {
#pragma unroll
            for (int q = 0; q < OW; ++q) out[q] = 0u;   // past the strip: code 0 (zero limbs anyway)
          }
        };
        const uint32_t ta = tmem + a_col0 + (uint32_t)(ss * ACOLS) + ((uint32_t)(warp * 32) << 16);
        IHT_DCHECK(((a_col0 + (uint32_t)((ss + 1) * ACOLS)) & 0xFFFFu) <= 512u, "batched: A stage inside TMEM");
        auto store = [&](int ts, const uint32_t* out) {
          if (!(a.probe & 4)) {
#pragma unroll
            for (int c0 = 0; c0 < OW; c0 += 8)
              asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                               ta + (uint32_t)(ts * OW + c0)),
                           "r"(out[c0]), "r"(out[c0 + 1]), "r"(out[c0 + 2]), "r"(out[c0 + 3]), "r"(out[c0 + 4]),
                           "r"(out[c0 + 5]), "r"(out[c0 + 6]), "r"(out[c0 + 7])
                           : "memory");
          }
        };
        {
          // the first tile-step is converted BEFORE waiting for the stage to be free, so only
          // the stores sit on the MMA -> converter -> MMA handoff chain
          uint32_t out[OW];
          convert(0, out);
          if (s_wrapped) mbar_wait2(smem_u32(&st_free[ss]), sph ^ 1u);
          store(0, out);
#pragma unroll 1
          for (int ts = 1; ts < TS; ++ts) {
            convert(ts, out);
            store(ts, out);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive2(smem_u32(&pk_free[ps]));     // packed slot consumed
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive2(smem_u32(&st_full[ss]));
        if (++ps == PKS) { ps = 0; pph ^= 1u; }
        if (++ss == ST) { ss = 0; sph ^= 1u; s_wrapped = true; }
      }
    }
    (void)CH;
  } else if (warp == 4) {
    // ---------------------------------------------------------------- MMA issuer
    // The tensor pipe queues only a few MMAs, so every instruction on the issuing thread's
    // path between K-blocks is exposed (scripts/microbench/tc2_bench.cu: a try_wait on an
    // already-completed phase per 16-MMA K-block costs ~5 clk per MMA).  So: the bases are
    // made warp-uniform once, and halfway through K-block kb lane 0 probes (test_wait, non
    // blocking) whether K-block kb+1's stage is already full -- then kb+1 starts without a
    // wait; otherwise it waits as before.
    int ss = 0;
    uint32_t sph = 0;
    int t = 0;
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t sB_u = __shfl_sync(0xffffffffu, smem_u32(sB), 0);
    const uint32_t full_u = __shfl_sync(0xffffffffu, smem_u32(&st_full[0]), 0);
    const uint32_t free_u = __shfl_sync(0xffffffffu, smem_u32(&st_free[0]), 0);
    const uint32_t nb128 = __shfl_sync(0xffffffffu, (uint32_t)NB * 128u, 0);
    for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++t) {
      const int ab = t & 1;
      const int half = u < a.nfull ? -1 : ((u - a.nfull) & 1);
      // a half unit multiplies the tile by snapshot-limb rows [half NB/2, (half+1) NB/2) of B:
      // an 8 KiB-aligned offset inside every SW128 atom column (8-row groups of 1 KiB)
      const uint32_t idesc = idesc_i8(kBT, half < 0 ? NB : NB / 2);
      const uint32_t hoff = half < 0 ? 0u : (uint32_t)(half * NB * 64);
      if (t >= 2) mbar_wait2(smem_u32(&acc_free[ab]), (uint32_t)(((t - 2) >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (a.tlog && lane == 0 && t < 16) a.tlog[blockIdx.x * 64 + 2 * t] = clock64();
      const uint32_t dtm = tmem_u + ab * acc_stride;
      uint32_t ready = 0;
      for (int kb = 0; kb < a.nkb; ++kb) {
        if (!ready && (!(a.probe & 64) || (t == 0 && kb < ST))) mbar_wait2(full_u + 8 * ss, sph);   // probe 64: first round only
        if (a.tlog && lane == 0 && t == 0 && kb < 16) a.tlog[blockIdx.x * 64 + 40 + kb] = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int nss = ss + 1 == ST ? 0 : ss + 1;
        const uint32_t nsph = ss + 1 == ST ? sph ^ 1u : sph;
        // warp-uniform operands (shuffled from lane 0 so the compiler keeps them on uniform
        // registers: no per-MMA R2UR broadcast loop)
        const uint32_t bbase_u = __shfl_sync(0xffffffffu, sB_u + ss * BSZ + hoff, 0);
        const uint32_t atm = __shfl_sync(0xffffffffu, tmem_u + a_col0 + (uint32_t)(ss * ACOLS), 0);
        const uint32_t dtm_u = __shfl_sync(0xffffffffu, dtm, 0);
        const uint32_t idesc_u = __shfl_sync(0xffffffffu, idesc, 0);
        const uint32_t acc0_u = __shfl_sync(0xffffffffu, kb > 0 ? 1u : 0u, 0);
        const uint32_t nfull_u = __shfl_sync(0xffffffffu, full_u + 8 * nss, 0);
        uint32_t peek = 0;
        if (lane == 0) {
          if (a.probe & 2) {                        // probe: no tensor work
            mbar_arrive2(free_u + 8 * ss);
            if (kb == a.nkb - 1) mbar_arrive2(smem_u32(&acc_full[ab]));
          } else {
            // base descriptor once per K-block; the per-MMA K offsets are added to the
            // descriptor's 14-bit start-address field (no carry: stages < 256 KiB)
            const uint64_t bd0 = sw128_desc(bbase_u);
#pragma unroll
            for (int kk = 0; kk < NKS; ++kk) {
              if (kk == NKS / 2 && kb + 1 < a.nkb && !(a.probe & 64)) peek = mbar_test2(nfull_u, nsph);
              const uint64_t bd = bd0 + (uint64_t)(((uint32_t)(kk >> 2) * nb128 + (uint32_t)(kk & 3) * 32u) >> 4);
              const uint32_t acc = kk > 0 ? 1u : acc0_u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtm_u),
                  "r"(atm + (uint32_t)(kk * 8)), "l"(bd), "r"(idesc_u), "r"(acc)
                  : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             free_u + 8 * ss)
                         : "memory");
            if (kb == a.nkb - 1)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(&acc_full[ab]))
                           : "memory");
          }
        }
        ready = __shfl_sync(0xffffffffu, peek, 0);
        ss = nss;
        sph = nsph;
      }
      if (a.tlog && lane == 0 && t < 16) a.tlog[blockIdx.x * 64 + 2 * t + 1] = clock64();
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- packed-code producer
    // lanes 0-7 each copy one column tile's tile-steps of the K-block (contiguous in the
    // tiled layout), so the 8 requests of a slot are issued in parallel
    int ps = 0;
    uint32_t ph = 0;
    bool wrapped = false;
    const int64_t last_tile = (a.N + 15) / 16 - 1;
    for (int u = (a.probe & (8 | 64)) ? a.nunits : blockIdx.x; u < a.nunits; u += gridDim.x) {
      const int tile = u < a.nfull ? u : a.nfull + ((u - a.nfull) >> 1);
      for (int kb = 0; kb < a.nkb; ++kb) {
        const int tsn = min(TS, a.ksteps - kb * TS);
        const uint32_t bytes = (uint32_t)(tsn * 1024);
        if (wrapped) mbar_wait2(smem_u32(&pk_free[ps]), ph ^ 1u);
        if (lane == 0) mbar_expect_tx2(smem_u32(&pk_full[ps]), 8 * bytes);
        __syncwarp();
        if (lane < 8) {
          int64_t col_tile = (int64_t)tile * 8 + lane;                // 16-column tile index
          if (col_tile > last_tile) col_tile = last_tile;              // past N: any valid data
          IHT_DCHECK(ps < PKS && (int64_t)kb * TS * 1024 + bytes <= 16 * a.strip_bytes && col_tile >= 0 &&
                         col_tile <= last_tile, "batched: packed-code bulk copy inside the copy");
          bulk_g2s2(smem_u32(sP + ps * PK + lane * (TS * 1024)),
                    a.codes + col_tile * 16 * a.strip_bytes + (int64_t)kb * TS * 1024, bytes,
                    smem_u32(&pk_full[ps]));
        }
        if (++ps == PKS) { ps = 0; ph ^= 1u; wrapped = true; }
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------------------- r-limb (B) producer
    int ss = 0;
    uint32_t sph = 0;
    bool wrapped = false;
    for (int u = blockIdx.x; u < a.nunits; u += gridDim.x) {
      for (int kb = 0; kb < a.nkb; ++kb) {
        if (a.probe & 64) {                       // probe 64: fill the stages once, then stop
          if (wrapped) break;
        } else if (wrapped) {
          mbar_wait2(smem_u32(&st_free[ss]), sph ^ 1u);
        }
        if (lane == 0) {
          if ((a.probe & 1) && wrapped) {
            mbar_arrive2(smem_u32(&st_full[ss]));                 // probe: reuse the stale stage
          } else {
            IHT_DCHECK(ss < ST && kb < a.nkb, "batched: limb-image stage index");
            mbar_expect_tx2(smem_u32(&st_full[ss]), (uint32_t)BSZ);
            bulk_g2s2(smem_u32(sB + ss * BSZ), a.bimg + (int64_t)kb * BSZ, (uint32_t)BSZ, smem_u32(&st_full[ss]));
          }
        }
        __syncwarp();
        if (++ss == ST) { ss = 0; sph ^= 1u; wrapped = true; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 7-10)
    const int quarter = warp & 3;               // TMEM lanes 32*quarter .. +31
    if (a.cidx) {
      // the snapshots' bound keys (written by batched_limbs_kernel, which this kernel waited on)
      for (int b = (warp - 7) * 32 + lane; b < a.Breal; b += 128) ep_bkey[b] = a.bkey[b];
      asm volatile("bar.sync 1, 128;" ::: "memory");   // the 4 epilogue warps
    }
    int t = 0;
    for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++t) {
      const int ab = t & 1;
      const int tile = u < a.nfull ? u : a.nfull + ((u - a.nfull) >> 1);
      const int half = u < a.nfull ? -1 : ((u - a.nfull) & 1);
      const int ncol = half < 0 ? NB : NB / 2;          // accumulator columns of this unit
      const int cbase = half < 0 ? 0 : half * (NB / 2);  // its first snapshot-limb column
      mbar_wait2(smem_u32(&acc_full[ab]), (uint32_t)((t >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t n = (int64_t)tile * kBT + quarter * 32 + lane;
      const uint32_t taddr = tmem + ab * acc_stride + ((uint32_t)(quarter * 32) << 16);
      for (int c0 = 0; c0 < ((a.probe & 16) ? 0 : ncol); c0 += 16) {   // probe 16: no epilogue work
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // g = sigma 2^-F (2 (D0 + 256 D1) - (L-1) S): exact integers, then one rounding
        float gv[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const int b = (cbase + c0 + e) >> 1;
          if (a.ep32) {
            const int W = 2 * ((int)v[e] + (int)v[e + 1] * 256) - ep_off32[b];
            gv[e >> 1] = __fmul_rn(__int2float_rn(W), ep_scale[b]);
          } else {
            const long long V = (long long)(int)v[e] + 256ll * (long long)(int)v[e + 1];
            gv[e >> 1] = (float)(2 * V - ep_off[b]) * ep_scale[b];
          }
          if (n < a.N && b < a.Breal) a.g[(int64_t)b * a.N + n] = gv[e >> 1];
        }
        if (a.cidx && !(a.probe & 128)) {             // probe 128: no candidate lists (timing)
          // candidates: key(mu g) >= bkey_b (x's support is handled by the select kernel).  The
          // 8 snapshots' flags are formed without a dependent chain (two 16-byte loads of their
          // keys) and the warp votes once per chunk; only a chunk with a candidate (rare after the
          // first iterations) walks its snapshots, one atomic per snapshot with any
          const int b0 = (cbase + c0) >> 1;         // multiple of 4: 16-byte aligned keys
          const uint4 k0 = *reinterpret_cast<const uint4*>(ep_bkey + b0);
          const uint4 k1 = *reinterpret_cast<const uint4*>(ep_bkey + b0 + 4);
          const unsigned int bk[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
          unsigned int fl = 0u;
          float av[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            av[e] = __fmul_rn(a.mu, gv[e]);
            fl |= (unsigned int)((__float_as_uint(av[e]) & 0x7FFFFFFFu) >= bk[e] && b0 + e < a.Breal) << e;
          }
          if (n >= a.N) fl = 0u;
          if (__any_sync(0xffffffffu, fl != 0u)) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const unsigned int m = __ballot_sync(0xffffffffu, (fl >> e) & 1u);
              if (m) {
                const int b = b0 + e;
                int base = 0;
                if (lane == 0) base = atomicAdd(&a.ccnt[b], __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0) + __popc(m & ((1u << lane) - 1u));
                if (((fl >> e) & 1u) && base < a.ccap) {
                  IHT_DCHECK(b < a.Breal && n < a.N, "batched: epilogue candidate snapshot / pixel");
                  a.cidx[(int64_t)b * a.ccap + base] = (int32_t)n;
                  a.cval[(int64_t)b * a.ccap + base] = av[e];
                }
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive2(smem_u32(&acc_free[ab]));
      if (a.tlog && warp == 7 && lane == 0 && t < 8) a.tlog[blockIdx.x * 64 + 32 + t] = clock64();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 4) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// Per-snapshot block fixed point of R (one CTA per snapshot): max |r| over bit patterns, then
// limbs_from_max (iht_limbs.cuh).  With bkey (the bounded select, solver only): also the
// snapshot's bound key from x^[n] (bound_key), read by the GEMM's epilogue and by
// thr_bounded_select.  (Folding this into the forward's last CTA per snapshot was measured at
// the same rate, r02 g61: the conversion's latency only moved, PDL already hid the launch.)
template <int BITS>
__global__ void __launch_bounds__(256) batched_limbs_kernel(const float* __restrict__ R, int Rpad, int B, int nreal,
                                                            int nkb, uint8_t* __restrict__ bimg, int* __restrict__ Fb,
                                                            int* __restrict__ Sb, const float* __restrict__ xval,
                                                            const int32_t* __restrict__ xnnz, int ldx, int max_nnz,
                                                            float bound, unsigned int* __restrict__ bkey) {
  pdl_launch_dependents();
  pdl_wait();                               // R (forward)
  const int b = blockIdx.x;                 // b >= nreal: zero padding snapshot (MMA N granularity)
  const bool live = b < nreal;
  const float* r = R + (int64_t)(live ? b : 0) * Rpad;
  // bound key: the last warp requests x's values (<= 256 of them: s <= kBsMaxS) before its r
  // loads and reduces them after the max pass, so the x round trip overlaps the r one
  const bool kw = bkey && live && threadIdx.x >= 224;
  BoundKeyLoads bk;
  if (kw) bk.load(xval + (int64_t)b * ldx, xnnz[b], ldx);
  // max |r| over bit patterns: a NaN / inf in r_b marks the snapshot (F = kNonFinite) and
  // its g becomes NaN, so that its H_s reports the domain error
  unsigned int m = 0;
  if (live) {
    constexpr int kU = 8;                   // float4 loads in flight per thread
    for (int i0 = threadIdx.x * 4; i0 < Rpad; i0 += blockDim.x * 4 * kU) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * blockDim.x * 4;
        v[u] = i < Rpad ? *reinterpret_cast<const float4*>(r + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        m = max(max(m, __float_as_uint(v[u].x) & 0x7FFFFFFFu), __float_as_uint(v[u].y) & 0x7FFFFFFFu);
        m = max(max(m, __float_as_uint(v[u].z) & 0x7FFFFFFFu), __float_as_uint(v[u].w) & 0x7FFFFFFFu);
      }
    }
  }
  if (kw) {
    const unsigned int k = bk.key(max_nnz, bound);
    if (threadIdx.x == 224) bkey[b] = k;
  }
  __shared__ unsigned int red[8];
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  unsigned int mb = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mb = max(mb, red[w]);
  limbs_from_max<BITS>(r, Rpad, B, b, live, nkb, bimg, Fb, Sb, mb, [](const float* p) {
    return *reinterpret_cast<const float4*>(p);
  });
}

static int kb_rows(int bits) {
  return bits == 2 ? BCfg<2>::KBR : bits == 4 ? BCfg<4>::KBR : BCfg<8>::KBR;
}

static size_t batched_smem(int bits, int B) {
  const int KBB = kb_rows(bits);
  const int ST = bits == 2 ? BCfg<2>::STAGES : bits == 4 ? BCfg<4>::STAGES : BCfg<8>::STAGES;
  const size_t pk = bits == 2 ? (size_t)BCfg<2>::PK * BCfg<2>::PKSLOTS
                  : bits == 4 ? (size_t)BCfg<4>::PK * BCfg<4>::PKSLOTS : (size_t)BCfg<8>::PK * BCfg<8>::PKSLOTS;
  return 1024 + (size_t)ST * 2 * B * KBB + pk + (size_t)(2 * kPkSlotsMax + 2 * kStagesMax + 4) * 8 + 16 +
         256 * 4 + 256 * 8 + 256 * 4 + 256 * 4;
}

}  // namespace iht

using namespace iht;

static constexpr int kMaxChunk = 64;     // snapshots per GEMM launch (MMA N = 2 * 64 = 128)

static int chunk_pad(int32_t nrhs) {      // padded snapshots of the widest chunk
  const int c = nrhs < kMaxChunk ? nrhs : kMaxChunk;
  return (c + 7) / 8 * 8;
}

extern "C" int64_t iht_adjoint_batched_ws_bytes(const iht_qmat* A, int32_t nrhs) {
  if (A == nullptr || nrhs <= 0) return -1;
  const int64_t Rpad = A->planes * rows_pad(A->rows);
  const int KBR = kb_rows(A->bits);
  const int64_t nkb = (Rpad + KBR - 1) / KBR;
  const int bp = chunk_pad(nrhs);
  return nkb * 2 * bp * KBR + 256 + 3 * bp * 4 + 256;
}

static int probe_flags() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IHT_BATCHED_PROBE");   // profiling only: see BatchArgs::probe
    v = e ? atoi(e) : 0;
  }
  return v;
}

extern "C" int iht_adjoint_batched(const iht_qmat* A, const float* R, int32_t nrhs, float* G, void* ws,
                                   int64_t ws_bytes, void* stream) {
  return iht_adjoint_batched_cand(A, R, nrhs, G, ws, ws_bytes, stream, nullptr);
}

int iht_adjoint_batched_cand(const iht_qmat* A, const float* R, int32_t nrhs, float* G, void* ws, int64_t ws_bytes,
                             void* stream, const iht_cand_args* cand) {
  if (A == nullptr || R == nullptr || G == nullptr || nrhs <= 0) return IHT_EINVAL;
  if (A->codes == nullptr || (A->bits != 2 && A->bits != 4 && A->bits != 8)) return IHT_EINVAL;
  if (A->strip_bytes != iht_strip_bytes(A->rows, A->planes, A->bits)) return IHT_EINVAL;
  const int64_t Rpad = A->planes * rows_pad(A->rows);
  const int L = num_levels(A->bits, A->level_mode);
  if ((double)Rpad * (L - 1) * 128.0 >= 2147483647.0) return IHT_EUNSUPPORTED;   // int32 accumulator
  const int64_t need = iht_adjoint_batched_ws_bytes(A, nrhs);
  if (ws == nullptr || ws_bytes < need) return IHT_EINVAL;
  const int KBR = kb_rows(A->bits);
  const int nkb = (int)((Rpad + KBR - 1) / KBR);   // the last K-block may hold fewer tile-steps
  const int ksteps = (int)(Rpad / (512 / A->bits));
  cudaStream_t st = (cudaStream_t)stream;
  const int bp_max = chunk_pad(nrhs);
  uint8_t* bimg = static_cast<uint8_t*>(ws);
  const int64_t bimg_bytes = (int64_t)nkb * 2 * bp_max * KBR;
  int* Fb = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + (bimg_bytes + 255) / 256 * 256);
  int* Sb = Fb + bp_max;
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (batched_smem(A->bits, bp_max) > 227 * 1024) return IHT_EUNSUPPORTED;
  // chunks of <= 64 snapshots; each padded to a multiple of 8 (MMA N = 2 B, multiple of 16)
  for (int c0 = 0; c0 < nrhs; c0 += kMaxChunk) {
    const int nb = nrhs - c0 < kMaxChunk ? nrhs - c0 : kMaxChunk;
    const int bp = (nb + 7) / 8 * 8;
    BatchArgs b{};
    b.codes = static_cast<const uint8_t*>(A->codes);
    b.strip_bytes = A->strip_bytes;
    b.N = A->cols;
    b.Rpad = (int)Rpad;
    b.nkb = nkb;
    b.ksteps = ksteps;
    b.ntiles = (int)((A->cols + kBT - 1) / kBT);
    // last partial wave: split its tiles into snapshot halves (N = B MMA columns) when that
    // fits one more wave, so no CTA runs a whole extra tile (config 5: 512 tiles on 148 SMs,
    // 4 -> 3.5 tile-times); the A codes of a split tile are converted by both halves
    {
      const int grid = min(b.ntiles, sms), tail = b.ntiles % grid;
      b.nfull = b.ntiles;
      b.nunits = b.ntiles;
      static int split_env = -1;                  // profiling override (IHT_BATCHED_SPLIT=0: off)
      if (split_env < 0) split_env = getenv("IHT_BATCHED_SPLIT") ? atoi(getenv("IHT_BATCHED_SPLIT")) : 1;
      if (split_env && b.ntiles > grid && tail > 0 && 2 * tail <= grid && (2 * bp) % 32 == 0) {
        b.nfull = b.ntiles - tail;
        b.nunits = b.nfull + 2 * tail;
      }
    }
    b.B = bp;
    b.Breal = nb;
    b.probe = probe_flags();
    b.ep32 = (double)Rpad * (L - 1) < 21700.0 ? 1 : 0;    // 771 Rpad (L-1) 128 < 2^31
    static long long* tlog = nullptr;
    if ((b.probe & 32) && tlog == nullptr) cudaMalloc(&tlog, 1024 * 64 * sizeof(long long));
    b.tlog = (b.probe & 32) ? tlog : nullptr;
    b.L = L;
    b.sigma = A->scale_c / (float)(L - 1);
    b.bimg = bimg;
    b.Fb = Fb;
    b.Sb = Sb;
    b.g = G + (int64_t)c0 * A->cols;
    if (cand) {   // the chunk's snapshots' lists and x
      b.cidx = cand->cidx + (int64_t)c0 * cand->ccap;
      b.cval = cand->cval + (int64_t)c0 * cand->ccap;
      b.ccnt = cand->ccnt + c0;
      b.ccap = cand->ccap;
      b.mu = cand->mu;
      b.bkey = cand->bkey + c0;
    }
    const float* Rc = R + (int64_t)c0 * Rpad;
    const size_t smem = batched_smem(A->bits, bp);
#define IHT_BATCH(BB)                                                                                  \
  do {                                                                                                 \
    IHT_CUDA_CHECK(launch_pdl(batched_limbs_kernel<BB>, dim3(bp), dim3(256), 0, st, Rc, (int)Rpad, bp, nb, \
                              nkb, bimg, Fb, Sb, cand ? cand->x_val + (int64_t)c0 * cand->ldx : nullptr,   \
                              cand ? cand->x_nnz + c0 : nullptr, cand ? cand->ldx : 0,                     \
                              cand ? cand->max_nnz : 0, cand ? cand->bound : 0.0f,                         \
                              cand ? cand->bkey + c0 : nullptr));                                          \
    if (getenv("IHT_DUP_LIMBS")) /* profiling: the limb kernel twice (idempotent), its in-graph cost */ \
      IHT_CUDA_CHECK(launch_pdl(batched_limbs_kernel<BB>, dim3(bp), dim3(256), 0, st, Rc, (int)Rpad, bp, nb,  \
                                nkb, bimg, Fb, Sb, cand ? cand->x_val + (int64_t)c0 * cand->ldx : nullptr,   \
                                cand ? cand->x_nnz + c0 : nullptr, cand ? cand->ldx : 0,                     \
                                cand ? cand->max_nnz : 0, cand ? cand->bound : 0.0f,                         \
                                cand ? cand->bkey + c0 : nullptr));                                          \
    static bool attr = false;                                                                          \
    if (!attr) {                                                                                       \
      IHT_CUDA_CHECK(cudaFuncSetAttribute(adjoint_batched_kernel<BB>,                                  \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));   \
      attr = true;                                                                                     \
    }                                                                                                  \
    IHT_CUDA_CHECK(launch_pdl(adjoint_batched_kernel<BB>, dim3(min(b.ntiles, sms)), dim3(kBThreads), smem, st, \
                              b));                                                                     \
  } while (0)
    if (A->bits == 2) IHT_BATCH(2);
    else if (A->bits == 4) IHT_BATCH(4);
    else IHT_BATCH(8);
#undef IHT_BATCH
    if (b.tlog) {   // profiling probe 32: per-CTA timeline of CTA 0 and the slowest CTA (stderr)
      static long long h[1024 * 64];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, b.tlog, sizeof(long long) * 64 * min(b.ntiles, sms), cudaMemcpyDeviceToHost);
      for (int c : {0, 1, 100, 140}) {
        if (c >= min(b.ntiles, sms)) continue;
        const long long* r = h + c * 64;
        const long long t0 = r[63];
        fprintf(stderr, "cta %d:", c);
        for (int t = 0; t < 4; ++t) fprintf(stderr, " tile%d mma [%lld, %lld] epi %lld;", t, r[2 * t] - t0, r[2 * t + 1] - t0,
                                            r[32 + t] - t0);
        fprintf(stderr, " kb-full(t0):");
        for (int k = 0; k < min(nkb, 16); ++k) fprintf(stderr, " %lld", r[40 + k] - t0);
        fprintf(stderr, "\n");
      }
    }
  }
  return IHT_OK;
}
