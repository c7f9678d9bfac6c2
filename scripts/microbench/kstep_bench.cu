// Cost of one 2-bit GEMV k-step of the int8 mma.sync adjoints (iht_adjoint.cu / iht_fused.cu):
// 2 LDS.128 of codes, 4 LDS.128 of r limbs (3 of 8 lane groups), 32 in-place mask LOP3s,
// 8 IMMA.16832.U8.S8 -- per warp, 8 warps per SM, operands in shared memory.  Variants isolate
// the parts: 0 full k-step; 1 no LDS (masks of loop-carried registers); 2 no LOP (IMMA on the
// loaded words directly); 3 IMMA only on constant operands (the peak); 4 full, 8 accumulators;
// 5 full, MMAs ordered so that consecutive ones update different accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kstep_bench kstep_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ void mma_u8s8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t frag(const uint4& w, int v, int j) {
  const uint32_t M8 = 0x03030303u;
  const uint32_t word = v == 0 ? w.x : v == 1 ? w.y : v == 2 ? w.z : w.w;
  return word & (M8 << (2 * j));
}

template <int VAR>
__global__ void __launch_bounds__(256, 1) kstep(int iters, long long* cyc, int* sink) {
  __shared__ __align__(16) uint8_t ring[16 * 1024];
  __shared__ __align__(16) uint8_t limbs[3 * 8192];
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += 256) reinterpret_cast<uint32_t*>(ring)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 3 * 8192 / 4; i += 256) reinterpret_cast<uint32_t*>(limbs)[i] = i * 40503u;
  __syncthreads();
  const int lane = threadIdx.x & 31, g8 = lane >> 2, t = lane & 3;
  const uint32_t rb = (uint32_t)__cvta_generic_to_shared(ring), lb = (uint32_t)__cvta_generic_to_shared(limbs);
  const bool bload = g8 < 3;
  constexpr int NACC = VAR == 4 ? 8 : 4;
  int acc[NACC][4] = {};
  uint32_t bw[16] = {};
  uint4 s0 = make_uint4(lane, lane * 3, lane * 5, lane * 7), s1 = make_uint4(lane * 11, lane, lane * 13, lane * 17);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int ks = it & 15;
    if (VAR != 1 && VAR != 3) {
      const uint32_t src = rb + ks * 1024 + g8 * 64 + t * 16;
      s0 = lds128(src);
      s1 = lds128(src + 512);
      if (bload) {
        const uint32_t bp = lb + g8 * 8256 + (uint32_t)(ks * 4 + t) * 64;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = lds128(bp + 16 * q);
          bw[4 * q] = v.x; bw[4 * q + 1] = v.y; bw[4 * q + 2] = v.z; bw[4 * q + 3] = v.w;
        }
      }
    } else if (VAR == 1) {
      s0.x += it; s1.y ^= it;
    }
    uint32_t af[8][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        if (VAR == 2 || VAR == 3) {
          af[2 * j + m][0] = m ? s0.z : s0.x; af[2 * j + m][1] = m ? s1.z : s1.x;
          af[2 * j + m][2] = m ? s0.w : s0.y; af[2 * j + m][3] = m ? s1.w : s1.y;
        } else {
          af[2 * j + m][0] = frag(s0, 2 * m, j);
          af[2 * j + m][1] = frag(s1, 2 * m, j);
          af[2 * j + m][2] = frag(s0, 2 * m + 1, j);
          af[2 * j + m][3] = frag(s1, 2 * m + 1, j);
        }
      }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int u = VAR == 5 ? (i % 4) * 2 + i / 4 : i;   // 5: consecutive MMAs on different accumulators
      mma_u8s8(acc[NACC == 8 ? u : (u >> 1)], af[u], bw[2 * u], bw[2 * u + 1]);
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  int s = 0;
  for (int c = 0; c < NACC; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 0x12345) sink[0] = s;
}

template <int VAR>
void run(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  long long* d;
  int* sink;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaMalloc(&sink, 4);
  kstep<VAR><<<sms, 256>>>(iters, d, sink);
  kstep<VAR><<<sms, 256>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  printf("{\"variant\": \"%s\", \"err\": \"%s\", \"clk_per_kstep_per_warp\": %.1f, \"imma_per_clk_per_sm\": %.3f}\n", name,
         cudaGetErrorString(e), mean / iters, 8.0 * 8 * iters / mean);
}

int main() {
  run<0>("full k-step (2+4 LDS, 32 LOP, 8 IMMA, 4 acc)");
  run<1>("no LDS");
  run<2>("no LOP (IMMA on loaded words)");
  run<3>("IMMA only, constant operands");
  run<4>("full k-step, 8 accumulators");
  run<5>("full k-step, MMA order interleaving the 4 accumulators");
  return 0;
}
