// NEXT-4 measurement: tensor-core issue rates on B200 for the operand kinds a
// low-precision IHT adjoint could use, against kind::i8 (what adjoint_batched_kernel uses) and
// the legacy warp-level mma.sync int8 path (what the GEMV adjoints use).
//
//   tcgen05.mma.cta_group::1, M = 128, A and B from shared memory (SW128 descriptors), one
//   issuing thread per SM, 8192 back-to-back MMAs into one TMEM accumulator:
//     kind::i8       u8 x s8 -> s32, K = 32
//     kind::f16      bf16 x bf16 -> f32, K = 16 (reference)
//     kind::f8f6f4   e4m3 x e4m3 -> f32, K = 32
//     kind::f8f6f4   e2m1 x e4m3 -> f32, K = 32 (2-bit codes are exact in e2m1)
//     kind::mxf4.block_scale  e2m1 x e2m1 (ue8m0 block-32 scales) -> f32, K = 64
//   legacy: mma.sync.m16n8k32.u8.s8.s32 (IMMA) from 8 / 16 warps per SM, 4 independent
//   accumulator chains per warp.
// Operand contents are irrelevant to the issue rate (zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o next4_bench next4_bench.cu
//   ./next4_bench <case>   (one case per process: a rejected descriptor cannot poison the others)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptors (PTX ISA "Instruction descriptor"): [4:5] D format, [7:9] A format,
// [10:12] B format, [17:22] N >> 3, [24:28] M >> 4
__host__ __device__ constexpr uint32_t idesc_std(uint32_t dfmt, uint32_t afmt, uint32_t bfmt, int M, int N) {
  return (dfmt << 4) | (afmt << 7) | (bfmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// block-scaled kinds: [4:5] SFB id, [7:9] A format, [10:11] B format, [17:22] N >> 3,
// [23] scale type (1 = ue8m0), [24:28] M >> 4, [29:30] SFA id
__host__ __device__ constexpr uint32_t idesc_bs(uint32_t afmt, uint32_t bfmt, int M, int N) {
  return (afmt << 7) | (bfmt << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

enum Kind { I8 = 0, BF16 = 1, E4M3 = 2, E2M1xE4M3 = 3, MXF4 = 4 };

template <int KIND, int N>
__global__ void __launch_bounds__(128, 1) tc_bench(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
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
    uint32_t id = 0;
    if (KIND == I8) id = idesc_std(2, 0, 1, 128, N);
    if (KIND == BF16) id = idesc_std(1, 1, 1, 128, N);
    if (KIND == E4M3) id = idesc_std(1, 0, 0, 128, N);
    if (KIND == E2M1xE4M3) id = idesc_std(1, 5, 0, 128, N);
    if (KIND == MXF4) id = idesc_bs(1, 1, 128, N);   // e2m1 x e2m1 (mxf4 format code 1)
    const uint32_t bbase = su32(smem), abase = su32(smem + 48 * 1024);
    const uint32_t sfa = tmem + 256 + 0, sfb = tmem + 256 + 32;   // scale factors (TMEM columns)
    const long long t0 = clock64();
    for (int it = 0; it < iters; it += 64) {
#pragma unroll
      for (int g = 0; g < 64; ++g) {
        const int kk = g & 3;
        const uint64_t ad = sw128_desc(abase + kk * 32), bd = sw128_desc(bbase + kk * 32);
        const uint32_t acc = (it + g) > 0 ? 1u : 0u;
        if constexpr (KIND == I8)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory");
        else if constexpr (KIND == BF16)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory");
        else if constexpr (KIND == E4M3 || KIND == E2M1xE4M3)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::mxf4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc), "r"(sfa), "r"(sfb) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
                     su32(&bar))
                 : "memory");
    const long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// legacy warp-level int8 MMA: 4 independent accumulator chains per warp
__global__ void imma_bench(int iters, long long* cyc, int* sink) {
  int d[4][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  int s = 0;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 0x12345) sink[0] = s;
}

static double clock_ghz() {
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  return khz / 1e6;
}

template <int KIND, int N>
static int run_tc(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 8192;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = tc_bench<KIND, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<sms, 128, 100 * 1024>>>(iters, d);                 // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 128, 100 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  const cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) {
    printf("{\"case\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(err));
    return 1;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const int K = KIND == BF16 ? 16 : KIND == MXF4 ? 64 : 32;
  const double macs = (double)sms * iters * 128.0 * N * K;
  printf("{\"case\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"clk_per_mma\": %.2f, \"ms\": %.4f, "
         "\"dense_tops\": %.1f, \"sm_clock_ghz_attr\": %.3f}\n",
         name, N, K, mean / iters, ms, 2.0 * macs / (ms * 1e-3) / 1e12, clock_ghz());
  return 0;
}

static int run_imma(int warps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  long long* d;
  int* sink;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaMalloc(&sink, 4);
  imma_bench<<<sms, 32 * warps>>>(iters, d, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  imma_bench<<<sms, 32 * warps>>>(iters, d, sink);
  cudaEventRecord(e1);
  const cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) {
    printf("{\"case\": \"imma_w%d\", \"error\": \"%s\"}\n", warps, cudaGetErrorString(err));
    return 1;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const double immas_per_sm = (double)iters * 4 * warps;
  const double macs = (double)sms * immas_per_sm * 16 * 8 * 32;
  printf("{\"case\": \"mma.sync m16n8k32 u8.s8 (%d warps/SM, 4 chains each)\", \"imma_per_clk_per_sm\": %.4f, "
         "\"ms\": %.4f, \"dense_tops\": %.1f}\n",
         warps, immas_per_sm / mean, ms, 2.0 * macs / (ms * 1e-3) / 1e12);
  return 0;
}

int main(int argc, char** argv) {
  const char* c = argc > 1 ? argv[1] : "i8";
  if (!strcmp(c, "i8")) return run_tc<I8, 128>("tcgen05 kind::i8 u8xs8 N=128");
  if (!strcmp(c, "i8n256")) return run_tc<I8, 256>("tcgen05 kind::i8 u8xs8 N=256");
  if (!strcmp(c, "bf16")) return run_tc<BF16, 256>("tcgen05 kind::f16 bf16 N=256");
  if (!strcmp(c, "e4m3")) return run_tc<E4M3, 256>("tcgen05 kind::f8f6f4 e4m3xe4m3 N=256");
  if (!strcmp(c, "e2m1")) return run_tc<E2M1xE4M3, 256>("tcgen05 kind::f8f6f4 e2m1xe4m3 N=256");
  if (!strcmp(c, "e2m1n128")) return run_tc<E2M1xE4M3, 128>("tcgen05 kind::f8f6f4 e2m1xe4m3 N=128");
  if (!strcmp(c, "mxf4")) return run_tc<MXF4, 256>("tcgen05 kind::mxf4.block_scale e2m1xe2m1 N=256");
  if (!strcmp(c, "imma8")) return run_imma(8);
  if (!strcmp(c, "imma16")) return run_imma(16);
  if (!strcmp(c, "imma32")) return run_imma(32);
  fprintf(stderr, "unknown case %s\n", c);
  return 2;
}
