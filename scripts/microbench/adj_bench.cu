// Microbenchmark: tiled streaming + the adjoint's per-step work (nibble LOP3, 2 LDS.128,
// 4 int8 IMMA) at several ring depths / warps per SM. Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldv(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void mma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int PF, int MODE>   // MODE 0: loads only; 1: + LOP3 + IMMA; 2: + LDS; 3: + 2 accum chains interleaved
__global__ void kern(const uint8_t* __restrict__ base, int64_t ntask, int nsteps, int64_t task_bytes, int* out) {
  extern __shared__ uint4 sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  int acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  uint32_t x = 0;
  for (int64_t task = (int64_t)blockIdx.x * wpb + warp; task < ntask; task += (int64_t)gridDim.x * wpb) {
    const uint8_t* p0 = base + task * task_bytes + lane * 16;
    const uint8_t* p1 = p0 + 512;
    uint4 r0[PF], r1[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) { r0[j] = ldv(p0 + j * 1024); r1[j] = ldv(p1 + j * 1024); }
    const int nmain = nsteps / PF * PF;
    for (int k0 = 0; k0 < nmain; k0 += PF) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int k = k0 + j;
        const uint4 a = r0[j], b = r1[j];
        uint32_t af[4][4];
        if (MODE >= 1) {
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              const uint32_t msk = 0x0F0F0F0Fu << (4 * jj);
              af[2 * jj + m][0] = (m ? a.z : a.x) & msk;
              af[2 * jj + m][1] = (m ? b.z : b.x) & msk;
              af[2 * jj + m][2] = (m ? a.w : a.y) & msk;
              af[2 * jj + m][3] = (m ? b.w : b.y) & msk;
            }
        }
        const int kk = min(k + PF, nsteps - 1);
        r0[j] = ldv(p0 + (int64_t)kk * 1024);
        r1[j] = ldv(p1 + (int64_t)kk * 1024);
        if (MODE == 0) x ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
        if (MODE >= 1) {
          uint32_t bw[8] = {1, 2, 3, 4, 5, 6, 7, 8};
          if (MODE >= 2 && (lane >> 2) < 3) {
            const uint4 v0 = sm[(k * 4 + (lane & 3)) * 2 & 4095], v1 = sm[((k * 4 + (lane & 3)) * 2 + 1) & 4095];
            bw[0] = v0.x; bw[1] = v0.y; bw[2] = v0.z; bw[3] = v0.w; bw[4] = v1.x; bw[5] = v1.y; bw[6] = v1.z; bw[7] = v1.w;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) mma(acc[MODE == 3 ? (u & 1) : (u >> 1)], af[u], bw[2 * u], bw[2 * u + 1]);
        }
      }
    }
  }
  if (x == 0x12345678u || acc[0][0] == 0x12345678 || acc[1][1] == 0x7654321) out[0] = x + acc[0][0] + acc[1][1];
}

template <int PF, int MODE>
float run(const uint8_t* buf, int64_t bytes, int wpb, int bps, int* out, int sms) {
  const int64_t task_bytes = 512 * 1024, ntask = bytes / task_bytes;
  const int nsteps = (int)(task_bytes / 1024);
  cudaFuncSetAttribute(kern<PF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<PF, MODE><<<sms * bps, wpb * 32, 65536>>>(buf, ntask, nsteps, task_bytes, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kern<PF, MODE><<<sms * bps, wpb * 32, 65536>>>(buf, ntask, nsteps, task_bytes, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("[%s]", cudaGetErrorString(e)); return -1; }
  float ms; cudaEventElapsedTime(&ms, a, b);
  return (float)(5.0 * bytes / (ms / 1e3) / 1e9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 8ll << 30;
  uint8_t* buf; int* out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 4); cudaMemset(buf, 1, bytes);
  const int cfg[][2] = {{16, 1}, {24, 1}, {32, 1}, {8, 3}};
  for (auto& c : cfg) {
    printf("warps/SM %2d (%d x %d):\n", c[0] * c[1], c[0], c[1]);
    printf("  PF4: loads %7.1f | +lop3+imma %7.1f | +lds %7.1f | 2chains %7.1f\n", run<4, 0>(buf, bytes, c[0], c[1], out, sms),
           run<4, 1>(buf, bytes, c[0], c[1], out, sms), run<4, 2>(buf, bytes, c[0], c[1], out, sms), run<4, 3>(buf, bytes, c[0], c[1], out, sms));
    printf("  PF8: loads %7.1f | +lop3+imma %7.1f | +lds %7.1f | 2chains %7.1f\n", run<8, 0>(buf, bytes, c[0], c[1], out, sms),
           run<8, 1>(buf, bytes, c[0], c[1], out, sms), run<8, 2>(buf, bytes, c[0], c[1], out, sms), run<8, 3>(buf, bytes, c[0], c[1], out, sms));
  }
  return 0;
}
