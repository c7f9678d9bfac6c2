// Config-5 GEMM question: is the in-kernel MMA cadence (84 clk per M128 N128
// K32 kind::i8 instead of 64) set by the per-SM shared-memory B reads, by A coming from TMEM,
// or by the epilogue's TMEM loads -- and does a CTA pair (cta_group::2, M = 256, B split
// across the pair's shared memories) recover it?  Issue-rate microbenchmark, sm_100a, one
// CTA (or CTA pair) per SM, one thread issuing back to back with a commit per 16 MMAs.
//   A  cta_group::1, A from TMEM, B stepping through a 64 KiB stage (kernel-like)
//   B  cta_group::1, A and B from shared memory (SW128 descriptors)
//   C  A + 4 warps looping tcgen05.ld.32x32b.x16 on the other accumulator (epilogue-like)
//   D  cta_group::2, M = 256 (each CTA 128 lanes of A in its TMEM), B = 2 x 64 columns, one
//      per CTA's shared memory, stepping like A; issued by the pair's leader
//   E  D + C's TMEM-load warps in both CTAs
//   F  A + a tcgen05.commit to a (never waited) mbarrier after every 16-MMA K-block
//   G  F + tcgen05.fence::after_thread_sync before every K-block
//   H  G with the kernel's issue loop: all 32 lanes run the K-block loop, operands broadcast
//      with __shfl_sync, lane 0 issues, __syncwarp after every K-block
//   I  H with the accumulator alternating between two TMEM buffers every 9 K-blocks (a tile)
//   J  I + an mbarrier try_wait per K-block on a phase that has already completed (all lanes)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc2_bench tc2_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mbar_init(uint32_t m, uint32_t c) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(m), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(m), "r"(ph) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int KPB = 16;

template <int MODE>
__global__ void __launch_bounds__(256, 1) tc(int nkb, long long* cyc) {
  constexpr bool PAIR = MODE == 3 || MODE == 4;
  constexpr bool LDW = MODE == 2 || MODE == 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  __shared__ int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (uint32_t)(i * 2654435761u) & 0x03030303u;
  if (threadIdx.x == 0) {
    mbar_init(su32(&done), 1);
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // A in TMEM columns 256..511 (codes 0..3 per byte)
  if (warp < 4) {
    for (int c = 0; c < 256; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + 256 + c + ((uint32_t)(warp * 32) << 16)),
                   "r"(0x01020301u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t bbase = su32(smem);
  if (warp == 4 && MODE >= 5) {
    __shared__ uint64_t kbar, rbar;
    if (lane == 0) {
      mbar_init(su32(&kbar), 1);
      mbar_init(su32(&rbar), 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&rbar)) : "memory");   // phase 0 done
    }
    __syncwarp();
    const long long t0 = clock64();
    const uint32_t idesc = idesc_i8(128, 128);
    for (int kb = 0; kb < nkb; ++kb) {
      if (MODE >= 9) mbar_wait(su32(&rbar), 0);
      if (MODE >= 6) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t st = bbase + (kb & 1) * (128 * 512), at = tmem + 256 + (uint32_t)((kb & 1) * 128);
      uint32_t dt = tmem + (MODE >= 8 ? (uint32_t)(((kb / 9) & 1) * 128) : 0u);
      if (MODE >= 7) {
        st = __shfl_sync(0xffffffffu, st, 0);
        at = __shfl_sync(0xffffffffu, at, 0);
        dt = __shfl_sync(0xffffffffu, dt, 0);
      }
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < KPB; ++kk) {
          const uint64_t bd = sw128_desc(st + (kk >> 2) * (128 * 128) + (kk & 3) * 32);
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
                       "r"(at + (uint32_t)(kk * 8)), "l"(bd), "r"(idesc), "r"(acc)
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&kbar))
                     : "memory");
      }
      if (MODE >= 7) __syncwarp();
    }
    if (lane == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done))
                   : "memory");
    __syncwarp();
    mbar_wait(su32(&done), 0);
    if (lane == 0) {
      cyc[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (warp == 4) {
    const long long t0 = clock64();
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = PAIR ? idesc_i8(256, 128) : idesc_i8(128, 128);
      const int NB = PAIR ? 64 : 128;                 // B columns in this CTA's shared memory
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t stage = bbase + (kb & 1) * (NB * 512);
#pragma unroll
        for (int kk = 0; kk < KPB; ++kk) {
          const uint64_t bd = sw128_desc(stage + (kk >> 2) * (NB * 128) + (kk & 3) * 32);
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
          if (MODE == 1) {
            const uint64_t ad = sw128_desc(bbase + 65536 + (kk >> 2) * (128 * 128) + (kk & 3) * 32);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
          } else if (PAIR) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                         "r"(tmem + 256 + (uint32_t)((kb & 1) * 128 + kk * 8)), "l"(bd), "r"(idesc), "r"(acc)
                         : "memory");
          } else {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                         "r"(tmem + 256 + (uint32_t)((kb & 1) * 128 + kk * 8)), "l"(bd), "r"(idesc), "r"(acc)
                         : "memory");
          }
        }
      }
      if (PAIR)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         su32(&done)), "h"((uint16_t)3) : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done))
                     : "memory");
    }
    __syncwarp();
    mbar_wait(su32(&done), 0);
    if (lane == 0) {
      cyc[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (LDW && warp < 4) {
    // epilogue-like TMEM loads of the other accumulator region (columns 128..255)
    while (*(volatile int*)&stop == 0) {
      uint32_t v[16];
      for (int c0 = 0; c0 < 128; c0 += 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + 128 + c0 + ((uint32_t)(warp * 32) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v[3] == 0x12345u && v[9] == 7u) stop = 2;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int MODE>
void run(const char* name, int sms) {
  constexpr bool PAIR = MODE == 3 || MODE == 4;
  const int nkb = 2048;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaMemset(d, 0, sms * sizeof(long long));
  auto k = tc<MODE>;
  const int smem = 130 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(sms / 2 * 2);
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, k, nkb, d);
  if (e == cudaSuccess) e = cudaLaunchKernelEx(&lc, k, nkb, d);
  cudaError_t err = e != cudaSuccess ? e : cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  int cnt = 0;
  for (int i = 0; i < sms; ++i)
    if (h[i] > 0) { mean += h[i]; ++cnt; }
  mean /= cnt > 0 ? cnt : 1;
  // per SM: cta_group::1 = one M128 N128 K32 per MMA; cta_group::2 = the pair's M256 N128 K32
  // per MMA, i.e. also one M128 N128 K32 per SM
  printf("{\"case\": \"%s\", \"err\": \"%s\", \"clk_per_mma\": %.1f, \"timed_ctas\": %d}\n", name,
         cudaGetErrorString(err), mean / (nkb * (double)KPB), cnt);
  fflush(stdout);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("A: cta_group::1, A TMEM, B 64 KiB stages", sms);
  run<1>("B: cta_group::1, A and B shared memory", sms);
  run<2>("C: A + epilogue-like TMEM loads (4 warps)", sms);
  run<3>("D: cta_group::2 M256 N128, A TMEM, B split over the pair", sms);
  run<4>("E: D + epilogue-like TMEM loads", sms);
  run<5>("F: A + commit per K-block", sms);
  run<6>("G: F + fence::after_thread_sync per K-block", sms);
  run<7>("H: G + warp-wide loop, shfl operands, lane-0 issue, syncwarp", sms);
  run<8>("I: H + accumulator alternating per 9 K-blocks", sms);
  run<9>("J: I + try_wait on a completed phase per K-block", sms);
  return 0;
}
