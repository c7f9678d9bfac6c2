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
__device__ __forceinline__ void mma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint4 lds128(uint32_t a) { uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)); return v; }
template <int MODE>
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
  int acc[2][4] = {{0,0,0,0},{0,0,0,0}};
  const uint32_t limbs = (uint32_t)__cvta_generic_to_shared(smem + (size_t)wpb * ring * chunk + wpb * ring * 8 + 64);
  const int g8 = lane >> 2, t = lane & 3;
  for (int64_t i = 0; i < per; ++i) {
    mbar_wait(bw + 8 * slot, parity);
    if (MODE == 0) x ^= *reinterpret_cast<const uint32_t*>(myring + slot * chunk + lane * 4);
    uint32_t af[2][4][4]; uint32_t bwv[2][8];
    if (MODE >= 1) {
      for (int h = 0; h < chunk / 1024; ++h) {
        const uint32_t src = rw + slot * chunk + h * 1024 + g8 * 64 + t * 16;
        const uint4 s0 = lds128(src), s1 = lds128(src + 512);
        for (int q = 0; q < 8; ++q) bwv[h & 1][q] = 0;
        if (MODE >= 2 && g8 < 3) { const uint4 v0 = lds128(limbs + ((i * 8 + h * 4 + t) & 1023) * 32), v1 = lds128(limbs + ((i * 8 + h * 4 + t) & 1023) * 32 + 16);
          bwv[h&1][0]=v0.x;bwv[h&1][1]=v0.y;bwv[h&1][2]=v0.z;bwv[h&1][3]=v0.w;bwv[h&1][4]=v1.x;bwv[h&1][5]=v1.y;bwv[h&1][6]=v1.z;bwv[h&1][7]=v1.w; }
        for (int j = 0; j < 2; ++j) for (int m = 0; m < 2; ++m) {
          const uint32_t msk = 0x0F0F0F0Fu << (4 * j);
          af[h&1][2*j+m][0] = (m ? s0.z : s0.x) & msk; af[h&1][2*j+m][1] = (m ? s1.z : s1.x) & msk;
          af[h&1][2*j+m][2] = (m ? s0.w : s0.y) & msk; af[h&1][2*j+m][3] = (m ? s1.w : s1.y) & msk; }
        if (MODE >= 3) for (int u = 0; u < 4; ++u) mma(acc[u >> 1], af[h&1][u], bwv[h&1][2*u], bwv[h&1][2*u+1]);
        else x ^= af[h&1][0][0] ^ af[h&1][3][3] ^ bwv[h&1][0];
      }
    }
    __syncwarp();
    if (issued < per) {
      if (lane == 0) { mbar_expect_tx(bw + 8 * slot, chunk); bulk_g2s(rw + slot * chunk, src + issued * chunk, chunk, bw + 8 * slot); }
      ++issued;
    }
    if (++slot == ring) { slot = 0; parity ^= 1; }
  }
  if (x == 0x12345678u || acc[0][0] == 0x1234567 || acc[1][2] == 0x7654321) out[0] = x;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 8ll << 30;
  uint8_t* buf; int* out; cudaMalloc(&buf, bytes); cudaMalloc(&out, 4); cudaMemset(buf, 1, bytes);
  cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(kern<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int cfgs[][3] = {{16, 3, 2048}, {16, 4, 2048}, {8, 3, 4096}, {8, 4, 4096}, {16, 2, 4096}, {12, 4, 2048}, {8, 6, 2048}, {8, 5, 4096}, {8, 6, 4096}, {16, 3, 4096}, {8, 3, 8192}, {8, 2, 8192}};
  for (int mode = 0; mode < 4; ++mode)
  for (auto& c : cfgs) {
    const int wpb = c[0], ring = c[1], chunk = c[2];
    const size_t sm = (size_t)wpb * ring * chunk + wpb * ring * 8;
    if (sm + 34000 > 227 * 1024) { printf("skip\n"); continue; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto launch = [&]() { if (mode == 0) kern<0><<<sms, wpb * 32, sm + 34000>>>(buf, bytes, chunk, ring, out);
      else if (mode == 1) kern<1><<<sms, wpb * 32, sm + 34000>>>(buf, bytes, chunk, ring, out);
      else if (mode == 2) kern<2><<<sms, wpb * 32, sm + 34000>>>(buf, bytes, chunk, ring, out);
      else kern<3><<<sms, wpb * 32, sm + 34000>>>(buf, bytes, chunk, ring, out); };
    launch();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("mode %d warps %2d ring %2d chunk %5d (%3zu KiB smem): %7.1f GB/s %s\n", mode, wpb, ring, chunk, sm / 1024, 5.0 * bytes / (ms / 1e3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
