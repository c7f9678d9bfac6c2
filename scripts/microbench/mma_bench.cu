// tcgen05.mma issue-rate microbenchmark (sm_100a): cycles per MMA for the shapes the
// batched adjoint uses.  One CTA per SM, one thread issues ITER MMAs into one TMEM
// accumulator (contents irrelevant), commits every GROUP MMAs to an mbarrier and, if
// WAIT, waits for that commit before issuing more (models a K-block handoff).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench mma_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int kind, int M, int N) {
  // kind 0: i8 (u8 x s8 -> s32); kind 1: bf16 x bf16 -> f32
  return kind == 0 ? ((2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                   : ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
}

template <int KIND, bool ATMEM, int N, int GROUP, bool WAIT, bool SPREAD = false>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = SPREAD ? (i * 2654435761u) : 0u;   // random bytes vs zeros
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(KIND, 128, N);
    const uint32_t bbase = su32(smem), abase = su32(smem + 48 * 1024);
    uint32_t ph = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; it += GROUP) {
#pragma unroll
      for (int g = 0; g < GROUP; ++g) {
        const int kk = SPREAD ? (g & 15) : (g & 3);
        // SPREAD: like adjoint_batched_kernel, 16 distinct 32-byte K slices over 4 SW128 atoms of a
        // 128-row B stage (16 KiB apart), A from 16 distinct TMEM column groups
        const uint64_t bd = sw128_desc(bbase + (SPREAD ? (kk >> 2) * 16384 + (kk & 3) * 32 : kk * 32));
        const uint32_t acc = (it + g) > 0 ? 1u : 0u;
#define MMA_T(K) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
                       "tcgen05.mma.cta_group::1.kind::" K " [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), \
                       "r"(tmem + 256 + (uint32_t)((kk * 8) & 255)), "l"(bd), "r"(id), "r"(acc) : "memory")
#define MMA_S(K) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
                       "tcgen05.mma.cta_group::1.kind::" K " [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd), \
                       "r"(id), "r"(acc) : "memory")
        const uint64_t ad = sw128_desc(abase + kk * 32);
        if constexpr (ATMEM && KIND == 0) MMA_T("i8");
        else if constexpr (ATMEM) MMA_T("f16");
        else if constexpr (KIND == 0) MMA_S("i8");
        else MMA_S("f16");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
      if (WAIT || it + GROUP >= iters) {
        asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                         su32(&bar)),
                     "r"(ph)
                     : "memory");
        ph ^= 1u;
      }
    }
    const long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int KIND, bool ATMEM, int N, int GROUP, bool WAIT, bool SPREAD = false>
void run(const char* name, int sms) {
  const int iters = 8192;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = bench<KIND, ATMEM, N, GROUP, WAIT, SPREAD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<sms, 128, 100 * 1024>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 128, 100 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const int K = KIND == 0 ? 32 : 16;
  const double macs = (double)sms * iters * 128.0 * N * K;
  fprintf(stderr, "%-45s %s  %.1f clk/MMA  %.3f ms  %.1f T(MAC*2)/s\n", name, cudaGetErrorString(err), mean / iters, ms,
         2.0 * macs / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, true, 128, 64, false>("i8 A=TMEM N=128 (no waits)", sms);
  run<0, false, 128, 64, false>("i8 A=SMEM N=128 (no waits)", sms);
  run<0, true, 256, 64, false>("i8 A=TMEM N=256 (no waits)", sms);
  run<0, false, 256, 64, false>("i8 A=SMEM N=256 (no waits)", sms);
  run<1, false, 256, 64, false>("bf16 A=SMEM N=256 (no waits)", sms);
  run<1, true, 256, 64, false>("bf16 A=TMEM N=256 (no waits)", sms);
  run<1, false, 128, 64, false>("bf16 A=SMEM N=128 (no waits)", sms);
  run<0, true, 128, 8, true>("i8 A=TMEM N=128 commit+wait every 8", sms);
  run<0, true, 128, 32, true>("i8 A=TMEM N=128 commit+wait every 32", sms);
  run<0, true, 128, 8, false>("i8 A=TMEM N=128 commit every 8", sms);
  run<0, true, 128, 64, false, true>("i8 A=TMEM N=128 spread operands, random B", sms);
  run<0, false, 128, 64, false, true>("i8 A=SMEM N=128 spread operands, random B", sms);
  return 0;
}
