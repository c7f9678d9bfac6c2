// Per-snapshot block fixed point of r for the batched tcgen05 adjoint (BASELINE config 5):
// the K-block geometry, the K permutation inside a 16-byte chunk, the SW128 image offsets and
// the conversion of one snapshot's r into two balanced signed 8-bit limbs (15 bits).  Shared by
// batched_limbs_kernel (iht_batched.cu) and the forward kernel's last CTA per snapshot
// (iht_forward.cu).  Internal, not ABI.
#pragma once
#include "iht_internal.cuh"

namespace iht {

constexpr int kNonFinite = 1000;       // F_b marker: r_b holds a NaN / inf -> g_b = NaN

// Per bit width: tile-steps (512/b rows, 1 KiB of a 16-column tile) per K-block, so that a
// K-block is 16 MMAs (K = 32 each) at 2 and 4 bits and 8 at 8 bits; A stages fill the 256
// TMEM columns left by the two accumulators; B stages take 128 KiB of shared memory.
// Measured (in-kernel timeline probe, config 5): every K-block handoff costs the MMA pipe
// ~300-400 clk whatever the depth, so fewer, larger K-blocks win: 2 stages x 16 MMAs ran
// at 87 clk per MMA (MMA-only), 4 stages x 8 MMAs at 100, against 64 back to back; r02
// again with the current issuer: 8-MMA K-blocks at 2 bits 49.2 us per call against 41.7.
template <int BITS> struct BCfg {
  static constexpr int TS = BITS == 8 ? 4 : BITS;       // tile-steps per K-block
  static constexpr int KBR = TS * 512 / BITS;           // rows (= u8 bytes per pixel row) per K-block
  static constexpr int NKS = KBR / 32;                  // MMAs per K-block
  static constexpr int ACOLS = KBR / 4;                 // TMEM columns of one A stage
  static constexpr int STAGES = 256 / ACOLS;            // 2 (2/4-bit) or 4 (8-bit)
  static constexpr int PK = 8 * TS * 1024;              // packed bytes per K-block (8 column tiles)
  static constexpr int PKSLOTS = PK <= 8192 ? 8 : (PK <= 16384 ? 4 : 2);   // packed-code slots
};
// byte offset of (row, 16-byte K chunk q) in a K-major SW128 tile whose rows hold KBB
// bytes: atoms of 128 rows x 128 B (16 KiB) along K, 8-row groups at 1024 B.
__host__ __device__ inline uint32_t sw128_off(int row, int q, int rows_total) {
  const int a = q >> 3, c = q & 7;
  return (uint32_t)(a * rows_total * 128 + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4));
}

// K permutation inside a 16-byte u8 chunk (shared by A and B): position p (0..15) <-> row
// offset (32/b) h + j + P i, with p = 4 (h P + j) + i (h: packed word, j: bit-position,
// i: byte).
__host__ __device__ inline int perm_row(int p, int bits) {
  const int P = 8 / bits, cpw = 32 / bits;
  const int i = p & 3, g = p >> 2;   // g = h P + j
  const int h = g / P, j = g % P;
  return cpw * h + j + P * i;
}

// x's values of one snapshot (<= 256 slots: s <= kBsMaxS), requested by one warp before other
// loads, reduced to the bound key (bound_key, iht_internal.cuh) afterwards.
struct BoundKeyLoads {
  unsigned int xk[8];
  int xn;
  __device__ __forceinline__ void load(const float* xv, int nnz_raw, int ldx) {
    xn = nnz_raw;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = (threadIdx.x & 31) + 32 * k;
      xk[k] = j < ldx ? (__float_as_uint(xv[j]) & 0x7FFFFFFFu) : 0xFFFFFFFFu;
    }
  }
  __device__ __forceinline__ unsigned int key(int max_nnz, float bound) {
    const int n = min(xn, max_nnz);          // < 0 (poisoned): no candidates
    unsigned int mk = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < 8; ++k) mk = min(mk, (int)(threadIdx.x & 31) + 32 * k < n ? xk[k] : 0xFFFFFFFFu);
    mk = __reduce_min_sync(0xffffffffu, mk);
    return bound_key(mk, n, bound);
  }
};

// One snapshot's limbs, given mb = max |r| over bit patterns (all 256 threads of the CTA):
// F_b (|r| 2^F < 2^14: two limbs; kNonFinite for NaN / inf), the limbs permuted into MMA K
// order and written into the pre-swizzled image, the exact limb sums S_b.  A thread owns 16
// consecutive rows (one 16-byte K chunk); ld4(p) loads 4 floats of r.
template <int BITS, class Ld4>
__device__ void limbs_from_max(const float* r, int Rpad, int B, int b, bool live, int nkb, uint8_t* __restrict__ bimg,
                               int* __restrict__ Fb, int* __restrict__ Sb, unsigned int mb, Ld4 ld4) {
  constexpr int KBR = BCfg<BITS>::KBR;
  __shared__ int ired[2][8];
  __shared__ int Fs;
  if (threadIdx.x == 0) {
    const bool bad = mb >= 0x7F800000u;
    const float mm = bad ? 0.0f : __uint_as_float(mb);
    int e = 0;
    if (mm > 0.0f) frexpf(mm, &e);
    Fs = bad ? kNonFinite : (mm > 0.0f ? min(14 - e, 126) : 0);   // |r| 2^F < 2^14 -> two limbs
    Fb[b] = Fs;
  }
  __syncthreads();
  const float scale = Fs == kNonFinite ? 0.0f : ldexpf(1.0f, Fs);
  const int NB = 2 * B;
  int s0 = 0, s1 = 0;
  for (int ch = threadIdx.x; ch < nkb * KBR / 16; ch += blockDim.x) {   // rows past Rpad: zero limbs
    const int row0 = ch * 16;
    const bool in = live && row0 < Rpad;      // Rpad is a multiple of 256: chunks are all-in or all-out
    float v[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 f = in ? ld4(r + row0 + 4 * k) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * k] = f.x;
      v[4 * k + 1] = f.y;
      v[4 * k + 2] = f.z;
      v[4 * k + 3] = f.w;
    }
    uint32_t w0[4] = {0u, 0u, 0u, 0u}, w1[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int p = 0; p < 16; ++p) {          // byte p of the chunk <- row row0 + perm_row(p)
      const int ri = __float2int_rn(v[perm_row(p, BITS)] * scale);
      const int l0 = ((ri + 128) & 255) - 128;
      const int l1 = (ri - l0) >> 8;
      s0 += l0;
      s1 += l1;
      w0[p >> 2] |= (uint32_t)(l0 & 255) << (8 * (p & 3));
      w1[p >> 2] |= (uint32_t)(l1 & 255) << (8 * (p & 3));
    }
    const int kb = row0 / KBR, q = (row0 % KBR) >> 4;
    uint8_t* blk = bimg + (int64_t)kb * NB * KBR;
    *reinterpret_cast<uint4*>(blk + sw128_off(2 * b, q, NB)) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
    *reinterpret_cast<uint4*>(blk + sw128_off(2 * b + 1, q, NB)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    ired[0][threadIdx.x >> 5] = s0;
    ired[1][threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a0 = 0, a1 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a0 += ired[0][w];
      a1 += ired[1][w];
    }
    Sb[2 * b] = a0;
    Sb[2 * b + 1] = a1;
  }
}

}  // namespace iht
