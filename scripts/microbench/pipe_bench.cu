// Which part of the batched adjoint's warp-specialised pipeline costs MMA throughput?
// MODE 1: one thread issues 8 MMAs per "K-block" and commits to a_free[stage] (4 stages),
//         nobody waits (pure issue rate).
// MODE 2: + 4 "converter" warps: wait a_free[stage] (K-block i-4), arrive a_full[stage];
//         the MMA warp waits a_full before each K-block (the kernel's A handoff).
// MODE 3: MODE 2 + 6 extra warps spinning on an mbarrier that completes at the end.
// MODE 4: MODE 2 but the MMA warp's 32 lanes all wait (kernel style) vs lane 0 only.
// MODE 5: MODE 4 + a B ring (warp 6 waits b_free, arrives b_full; MMA warp waits b_full,
//         commits to b_free as well): the kernel's two handoffs per K-block.
// MODE 6: MODE 5 + tiles of 18 K-blocks with double-buffered accumulators handed to 4
//         epilogue warps (acc_full commit / acc_free arrive), like adjoint_batched_kernel.
// MODE 7: MODE 6 with ONE commit per K-block to a shared stage-free barrier (converters and
//         B producer both wait on it).
// MODE 8: MODE 7 with ONE stage-full barrier (4 converter arrivals + 1 producer arrival).
// MODE 9: MODE 8, the MMA warp polls with mbarrier.test_wait (no suspend) instead of try_wait.
// MODE 10: MODE 8 with 8 stages (A stages of 32 TMEM columns, 4 MMAs per K-block... kept 8).
// MODE 11: MODE 8 with 16 MMAs per K-block and 2 stages.
// MODE 12: MODE 8 without the MMA warp's tcgen05.fence::after_thread_sync per K-block.
// MODE 14: MODE 8, but converters and producer never wait for a free stage (timing only).
// MODE 15: MODE 8 with 16 stages (aliased TMEM/smem addresses; timing only).
// MODE 13: MODE 8, converters skip tcgen05.fence::before_thread_sync... (they issue no tcgen05 ops here)
//          and the MMA warp fences only every 2nd K-block (timing probe only).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mbar_init(uint32_t m, uint32_t c) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(m), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint32_t m) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(m) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(m), "r"(ph) : "memory");
}
constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
template <int MODE> struct Cfg { static constexpr int ST = MODE == 10 ? 8 : ((MODE == 11 || MODE == 16) ? 2 : (MODE == 15 ? 16 : 4));
                                  static constexpr bool FENCE = MODE != 12;
                                  static constexpr int KPB = (MODE == 11 || MODE == 16) ? 16 : 8; };
__device__ __forceinline__ void mbar_spin(uint32_t m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tS_%=:\n\tmbarrier.test_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra S_%=;\n\t}" ::"r"(m), "r"(ph) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(352, 1) pipe(int nkb, long long* cyc, int rnd) {
  constexpr int ST = Cfg<MODE>::ST, KPB = Cfg<MODE>::KPB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t a_full[16], a_free[16], b_full[16], b_free[16], acc_full[2], acc_free[2], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 136 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = rnd ? (uint32_t)(i * 2654435761u + 12345u) ^ ((uint32_t)i >> 7) * 40503u : 0u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(su32(&a_full[i]), MODE >= 8 ? 5 : 4); mbar_init(su32(&a_free[i]), 1);
      mbar_init(su32(&b_full[i]), 1); mbar_init(su32(&b_free[i]), 1);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(su32(&acc_full[i]), 1); mbar_init(su32(&acc_free[i]), 4); }
    mbar_init(su32(&done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (rnd && warp < 4) {
    for (int c = 0; c < 256; ++c) {
      uint32_t x = (uint32_t)(threadIdx.x * 7919u + c * 104729u) * 2654435761u;
      x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      if (rnd == 1) x &= 0x03030303u;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + 256 + c + ((uint32_t)(warp * 32) << 16)), "r"(x) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4 && MODE >= 2) {
    int s = 0; uint32_t ph = 0; bool wr = false;
    for (int kb = 0; kb < nkb; ++kb) {
      if (wr && MODE != 14) mbar_wait(su32(&a_free[s]), ph ^ 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive(su32(&a_full[s]));
      if (++s == ST) { s = 0; ph ^= 1u; wr = true; }
    }
  } else if (warp == 4) {
    const long long t0 = clock64();
    int s = 0; uint32_t ph = 0;
    const uint32_t bbase = su32(smem);
    const int tiles = MODE >= 6 ? nkb / 18 : 1;
    const int per = MODE >= 6 ? 18 : nkb;
    int kbg = 0;
    for (int t = 0; t < tiles; ++t) {
      const int ab = t & 1;
      if (MODE >= 6 && t >= 2) mbar_wait(su32(&acc_free[ab]), ((t - 2) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < per; ++kb, ++kbg) {
        if (MODE >= 2) {
          if (MODE == 9) mbar_spin(su32(&a_full[s]), ph);
          else if (MODE >= 4 || lane == 0) mbar_wait(su32(&a_full[s]), ph);
          if (MODE >= 5 && MODE < 8) mbar_wait(su32(&b_full[s]), ph);
          if (Cfg<MODE>::FENCE && (MODE != 13 || (kb & 1) == 0)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < KPB; ++kk) {
            const uint64_t bd = MODE == 16
                ? sw128_desc(bbase + (s & 1) * 65536 + (kk >> 2) * (128 * 128) + (kk & 3) * 32)   // kernel-like 64 KiB stages
                : sw128_desc(bbase + (MODE >= 5 ? (s & 3) * 32768 : 0) + ((kk >> 2) & 1) * (128 * 128) + (kk & 3) * 32);
            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (MODE >= 6 ? ab * 128 : 0)),
                         "r"(tmem + 256 + (uint32_t)((s * KPB * 8 + kk * 8) & 255)), "l"(bd), "r"(IDESC), "r"(acc) : "memory");
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&a_free[s])) : "memory");
          if (MODE >= 5 && MODE < 7)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&b_free[s])) : "memory");
          if (MODE >= 6 && kb == per - 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&acc_full[ab])) : "memory");
        }
        __syncwarp();
        if (++s == ST) { s = 0; ph ^= 1u; }
      }
    }
    if (lane == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done)) : "memory");
      mbar_wait(su32(&done), 0);
      cyc[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  } else if (warp == 6 && MODE >= 5) {
    int s = 0; uint32_t ph = 0; bool wr = false;
    for (int kb = 0; kb < nkb; ++kb) {
      if (wr && MODE != 14) mbar_wait(su32(MODE >= 7 ? &a_free[s] : &b_free[s]), ph ^ 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive(su32(MODE >= 8 ? &a_full[s] : &b_full[s]));
      if (++s == ST) { s = 0; ph ^= 1u; wr = true; }
    }
  } else if (warp >= 7 && MODE >= 6) {
    for (int t = 0; t < nkb / 18; ++t) {
      const int ab = t & 1;
      mbar_wait(su32(&acc_full[ab]), (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(su32(&acc_free[ab]));
    }
  } else if (MODE == 3 && warp >= 5) {
    mbar_wait(su32(&done), 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE>
void run(const char* name, int sms, int rnd = 0) {
  const int nkb = 18 * 114;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = pipe<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<sms, 352, 140 * 1024>>>(nkb, d, rnd);
  cudaError_t err = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  printf("%-60s rnd=%d %s  %.1f clk/MMA\n", name, rnd, cudaGetErrorString(err), mean / (nkb * (double)Cfg<MODE>::KPB));
  fflush(stdout);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1>("1: issue + commit per K-block, no waits", sms);
  run<1>("1: issue + commit per K-block, no waits", sms, 1);
  run<1>("1: issue + commit per K-block, no waits", sms, 2);
  run<11>("11: 8 with 16 MMAs per K-block, 2 stages", sms, 1);
  run<11>("11: 8 with 16 MMAs per K-block, 2 stages", sms, 2);
  run<16>("16: 11 with the kernel's 64 KiB B stages (4 atom columns)", sms, 1);
  run<2>("2: + converter handoff (a_full/a_free, 4 stages), lane-0 wait", sms);
  run<3>("3: + 6 spinning warps", sms);
  run<4>("4: handoff, all 32 MMA-warp lanes wait", sms);
  run<5>("5: + B ring (second handoff + commit)", sms);
  run<6>("6: + tiles with double-buffered accumulators / epilogue warps", sms);
  run<7>("7: 6 with one commit per K-block (shared stage-free barrier)", sms);
  run<8>("8: 7 with one stage-full barrier (5 arrivals)", sms);
  run<9>("9: 8 with test_wait polling in the MMA warp", sms);
  run<10>("10: 8 with 8 stages", sms);
  run<11>("11: 8 with 16 MMAs per K-block, 2 stages", sms);
  run<12>("12: 8 without tcgen05.fence::after_thread_sync", sms);
  run<13>("13: 8 fencing every 2nd K-block", sms);
  run<14>("14: 8 with no free-stage waits (unbounded run-ahead)", sms);
  run<15>("15: 8 with 16 stages", sms);
  return 0;
}
