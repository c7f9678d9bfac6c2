// Streaming-read microbenchmark for the adjoint's access patterns on B200 (8 GiB buffer).
// Not part of the product; used to choose the adjoint's layout / prefetch depth / warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <bool L2PF>
__device__ __forceinline__ uint4 ldv(const uint8_t* p) {
  uint4 r;
  if (L2PF)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// plain grid-stride read
__global__ void seq_read(const uint4* __restrict__ p, int64_t n, uint32_t* out) {
  uint32_t x = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(p + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x12345678u) out[0] = x;
}

// PATTERN 0: tiled (each step 1 KiB contiguous per warp: 2 loads per lane)
// PATTERN 1: strips (16 columns of 32 KiB; lane (g,t): column g / g+8, offset step*64 + t*16)
template <int PATTERN, int PF, bool L2PF>
__global__ void task_read(const uint8_t* __restrict__ base, int64_t ntask, int nsteps, int64_t task_bytes, uint32_t* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  uint32_t x = 0;
  for (int64_t task = (int64_t)blockIdx.x * wpb + warp; task < ntask; task += (int64_t)gridDim.x * wpb) {
    const uint8_t* tb = base + task * task_bytes;
    const uint8_t *p0, *p1;
    int64_t step;
    if (PATTERN == 0) { p0 = tb + lane * 16; p1 = p0 + 512; step = 1024; }
    else { const int64_t sb = task_bytes / 16; p0 = tb + g * sb + t * 16; p1 = tb + (g + 8) * sb + t * 16; step = 64; }
    uint4 r0[PF], r1[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) { r0[j] = ldv<L2PF>(p0 + j * step); r1[j] = ldv<L2PF>(p1 + j * step); }
    for (int k0 = 0; k0 < nsteps; k0 += PF) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int k = k0 + j;
        uint4 a = r0[j], b = r1[j];
        if (k + PF < nsteps) { r0[j] = ldv<L2PF>(p0 + (k + PF) * step); r1[j] = ldv<L2PF>(p1 + (k + PF) * step); }
        x ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
      }
    }
  }
  if (x == 0x12345678u) out[0] = x;
}

template <int PATTERN, int PF, bool L2PF>
float run(const uint8_t* buf, int64_t bytes, int wpb, int bps, uint32_t* out, int sms) {
  const int64_t task_bytes = 512 * 1024;   // 16 columns x 32 KiB
  const int64_t ntask = bytes / task_bytes;
  const int nsteps = (int)(task_bytes / 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  task_read<PATTERN, PF, L2PF><<<sms * bps, wpb * 32>>>(buf, ntask, nsteps, task_bytes, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) task_read<PATTERN, PF, L2PF><<<sms * bps, wpb * 32>>>(buf, ntask, nsteps, task_bytes, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return (float)(5.0 * bytes / (ms / 1e3) / 1e9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 8ll << 30;
  uint8_t* buf; uint32_t* out;
  CK(cudaMalloc(&buf, bytes)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(buf, 1, bytes));
  {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    seq_read<<<sms * 8, 256>>>((const uint4*)buf, bytes / 16, out);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) seq_read<<<sms * 8, 256>>>((const uint4*)buf, bytes / 16, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("seq_read grid-stride            : %7.1f GB/s\n", 5.0 * bytes / (ms / 1e3) / 1e9);
  }
  const int cfg[][2] = {{16, 1}, {32, 1}, {8, 2}, {16, 2}, {8, 4}, {4, 8}};
  for (auto& c : cfg) {
    const int wpb = c[0], bps = c[1];
    printf("warps/block %2d x blocks/SM %d (warps/SM %2d)\n", wpb, bps, wpb * bps);
    printf("  tiled  PF1 %7.1f  PF2 %7.1f  PF4 %7.1f  PF8 %7.1f | L2::256B PF1 %7.1f PF4 %7.1f\n",
           run<0, 1, false>(buf, bytes, wpb, bps, out, sms), run<0, 2, false>(buf, bytes, wpb, bps, out, sms),
           run<0, 4, false>(buf, bytes, wpb, bps, out, sms), run<0, 8, false>(buf, bytes, wpb, bps, out, sms),
           run<0, 1, true>(buf, bytes, wpb, bps, out, sms), run<0, 4, true>(buf, bytes, wpb, bps, out, sms));
    printf("  strips PF1 %7.1f  PF2 %7.1f  PF4 %7.1f  PF8 %7.1f | L2::256B PF1 %7.1f PF4 %7.1f\n",
           run<1, 1, false>(buf, bytes, wpb, bps, out, sms), run<1, 2, false>(buf, bytes, wpb, bps, out, sms),
           run<1, 4, false>(buf, bytes, wpb, bps, out, sms), run<1, 8, false>(buf, bytes, wpb, bps, out, sms),
           run<1, 1, true>(buf, bytes, wpb, bps, out, sms), run<1, 4, true>(buf, bytes, wpb, bps, out, sms));
  }
  CK(cudaGetLastError());
  return 0;
}
