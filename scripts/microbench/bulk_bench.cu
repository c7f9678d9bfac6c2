// Bulk-copy (cp.async.bulk -> smem ring + mbarrier) streaming rate vs request size / warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(mbar), "r"(parity) : "memory");
}
__global__ void kern(const uint8_t* base, int64_t bytes, int chunk, int ring, int* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  uint8_t* myring = smem + warp * ring * chunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + wpb * ring * chunk) + warp * ring;
  const uint32_t rw = (uint32_t)__cvta_generic_to_shared(myring), bw = (uint32_t)__cvta_generic_to_shared(bars);
  if (lane == 0) for (int j = 0; j < ring; ++j) mbar_init(bw + 8 * j, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // each warp streams a contiguous region of bytes / (grid*wpb)
  const int64_t nw = (int64_t)gridDim.x * wpb, wid = (int64_t)blockIdx.x * wpb + warp;
  const int64_t per = bytes / nw / chunk;   // chunks per warp
  const uint8_t* src = base + wid * per * chunk;
  int64_t issued = 0;
  for (; issued < ring && issued < per; ++issued)
    if (lane == 0) { mbar_expect_tx(bw + 8 * issued, chunk); bulk_g2s(rw + issued * chunk, src + issued * chunk, chunk, bw + 8 * issued); }
  uint32_t x = 0, parity = 0; int slot = 0;
  for (int64_t i = 0; i < per; ++i) {
    mbar_wait(bw + 8 * slot, parity);
    x ^= *reinterpret_cast<const uint32_t*>(myring + slot * chunk + lane * 4);
    __syncwarp();
    if (issued < per) {
      if (lane == 0) { mbar_expect_tx(bw + 8 * slot, chunk); bulk_g2s(rw + slot * chunk, src + issued * chunk, chunk, bw + 8 * slot); }
      ++issued;
    }
    if (++slot == ring) { slot = 0; parity ^= 1; }
  }
  if (x == 0x12345678u) out[0] = x;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 8ll << 30;
  uint8_t* buf; int* out; cudaMalloc(&buf, bytes); cudaMalloc(&out, 4); cudaMemset(buf, 1, bytes);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int cfgs[][3] = {{16, 6, 1024}, {16, 12, 1024}, {16, 3, 2048}, {16, 6, 2048}, {8, 6, 2048}, {8, 3, 4096}, {8, 6, 4096}, {4, 6, 8192}, {16, 3, 4096}, {32, 3, 2048}};
  for (auto& c : cfgs) {
    const int wpb = c[0], ring = c[1], chunk = c[2];
    const size_t sm = (size_t)wpb * ring * chunk + wpb * ring * 8;
    if (sm > 220 * 1024) { printf("skip\n"); continue; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<sms, wpb * 32, sm>>>(buf, bytes, chunk, ring, out);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) kern<<<sms, wpb * 32, sm>>>(buf, bytes, chunk, ring, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("warps %2d ring %2d chunk %5d (%3zu KiB smem): %7.1f GB/s %s\n", wpb, ring, chunk, sm / 1024, 5.0 * bytes / (ms / 1e3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
