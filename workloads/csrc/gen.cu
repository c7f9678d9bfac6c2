// GPU side of the counter-based Gaussian workload generator (workloads/gen.py).
// Holds none of the method's arithmetic: it only writes the fp32 matrix Phi of
// BASELINE configs 1, 2, 4 (so config 4's 64 GiB never has to cross PCIe).
// Bit-identical to workloads.gen.gaussian_block (pinned by tests/test_gpu_gen.py):
//   h_j = mix64(key + (3 idx + j + 1) * 0x9E3779B97F4A7C15), j = 0,1,2
//   S = sum of the twelve 16-bit fields, z = 2 S - 12*65535, value = fl32(fl32(z) * scale32)
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gauss_fill_kernel(float* __restrict__ out, int64_t rows, int64_t cols, int64_t ld,
                                  int64_t row0, int64_t col0, int64_t n_total, uint64_t key,
                                  float scale32) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (n >= cols || m >= rows) return;
  const uint64_t idx = (uint64_t)(row0 + m) * (uint64_t)n_total + (uint64_t)(col0 + n);
  int s = 0;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint64_t h = mix64(key + (3ull * idx + (uint64_t)j + 1ull) * 0x9E3779B97F4A7C15ull);
    s += (int)(h & 0xFFFF) + (int)((h >> 16) & 0xFFFF) + (int)((h >> 32) & 0xFFFF) + (int)(h >> 48);
  }
  const int z = 2 * s - 12 * 65535;
  out[m * ld + n] = __fmul_rn((float)z, scale32);
}

extern "C" __attribute__((visibility("default"))) int ihtgen_gauss_fill(
    float* out, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t col0, int64_t n_total,
    uint64_t key, float scale32, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  const int threads = 256;
  const int64_t zdim = (rows + 65534) / 65535;
  dim3 grid((unsigned)((cols + threads - 1) / threads), (unsigned)(rows < 65535 ? rows : 65535),
            (unsigned)zdim);
  gauss_fill_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(out, rows, cols, ld, row0, col0, n_total,
                                                                key, scale32);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
