// NEXT-3: the radio-interferometer Phi computed on the fly (paper section
// "Computing Phi on the fly", "also in this case, quantization can help").
//
//   Phi_{k,p} = exp(-2 pi i (u_k l_p + v_k m_p)),  u_k, v_k = baseline / lambda (BASELINE
//   config 3, reading c16), pixel p = row * grid + col, l = centre(row), m = centre(col),
//   centre(i) = -1 + (2 i + 1) / grid.
//
// The phase in turns tau = u l + v m is formed in fp64 (B200 keeps a strong FP64 pipe) and
// reduced to its fractional part; cos / sin come from fp64 sincospi rounded to fp32, i.e.
// the entries of the stored complex64 Phi (computed in fp64 and rounded).
// With bits > 0 every component is stochastically rounded in registers exactly as
// iht_quantize would (Q-contract, Philox counter (p >> 2, row_offset + k, copy, plane << 8)),
// so the on-the-fly quantised adjoint uses the stored copy's codes.  Zero bytes of Phi are
// read: the kernel is FP64/ALU-bound.
#include "iht_internal.cuh"

namespace iht {

constexpr int kRdThreads = 256;       // 256 threads x 4 pixels
constexpr int kRdChunk = 512;         // visibilities staged in shared memory per round

struct RadioArgs {
  const double* u;   // [nvis] baseline x / lambda
  const double* v;   // [nvis]
  int64_t nvis, row_offset, rpad;
  int grid;
  int64_t npix;
  int bits, L;
  float c, sf, sigma;
  uint32_t copy_id, k0, k1;
  const float* r;    // stacked: re plane, im plane
  float* g;
};

// e^{-2 pi i tau}: (cos, -sin) of the fractional turn by fp64 sincospi, rounded to fp32 --
// the same values as the stored complex64 Phi (fp64 exp rounded to complex64) except in
// vanishingly rare double-rounding cases, so the in-register codes match stored copies.
__device__ __forceinline__ void phi_entry(double tau, float* re, float* im) {
  const double fr = tau - rint(tau);            // in [-1/2, 1/2], exact
  double s, c;
  sincospi(2.0 * fr, &s, &c);
  *re = (float)c;
  *im = (float)(-s);
}

template <bool QUANT>
__global__ void __launch_bounds__(kRdThreads) adjoint_radio_kernel(RadioArgs a) {
  __shared__ double su[kRdChunk], sv[kRdChunk];
  __shared__ float sre[kRdChunk], sim[kRdChunk];
  const int64_t quad = (int64_t)blockIdx.x * kRdThreads + threadIdx.x;
  const int64_t p0 = quad * 4;
  double l[4], m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t p = min64(p0 + j, a.npix - 1);
    const int row = (int)(p / a.grid), col = (int)(p % a.grid);
    l[j] = -1.0 + (2.0 * row + 1.0) / a.grid;
    m[j] = -1.0 + (2.0 * col + 1.0) / a.grid;
  }
  const float Lm1 = (float)(a.L - 1);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t k0 = 0; k0 < a.nvis; k0 += kRdChunk) {
    const int nk = (int)min64(kRdChunk, a.nvis - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < nk; i += kRdThreads) {
      su[i] = a.u[k0 + i];
      sv[i] = a.v[k0 + i];
      sre[i] = a.r[k0 + i];
      sim[i] = a.r[a.rpad + k0 + i];
    }
    __syncthreads();
    for (int i = 0; i < nk; ++i) {
      const double u = su[i], v = sv[i];
      float re[4], im[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) phi_entry(fma(u, l[j], v * m[j]), &re[j], &im[j]);
      if (QUANT) {
        const uint32_t mg = (uint32_t)(a.row_offset + k0 + i);
        const u32x4 w0 = philox4x32_10(u32x4{(uint32_t)quad, mg, a.copy_id, 0u}, a.k0, a.k1);
        const u32x4 w1 = philox4x32_10(u32x4{(uint32_t)quad, mg, a.copy_id, 1u << 8}, a.k0, a.k1);
        const uint32_t W0[4] = {w0.x, w0.y, w0.z, w0.w}, W1[4] = {w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          re[j] = __fmaf_rn(2.0f, (float)q_contract(re[j], a.c, a.sf, a.L, W0[j]), -Lm1);
          im[j] = __fmaf_rn(2.0f, (float)q_contract(im[j], a.c, a.sf, a.L, W1[j]), -Lm1);
        }
      }
      // Re(conj(Phi) r) = Re Phi Re r + Im Phi Im r (stacked real rows, reading c13)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = __fmaf_rn(im[j], sim[i], __fmaf_rn(re[j], sre[i], acc[j]));
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (p0 + j < a.npix) a.g[p0 + j] = QUANT ? __fmul_rn(a.sigma, acc[j]) : acc[j];
}

}  // namespace iht

using namespace iht;

extern "C" int iht_adjoint_radio(const iht_radio* R, const float* r, float* g, void* stream) {
  if (R == nullptr || R->u == nullptr || R->v == nullptr || r == nullptr || g == nullptr || R->nvis <= 0 ||
      R->grid <= 0 || R->row_offset < 0 || R->row_offset + R->nvis > 0xFFFFFFFFll)
    return IHT_EINVAL;
  if (R->bits != 0 && R->bits != 2 && R->bits != 4 && R->bits != 8) return IHT_EINVAL;
  if (R->level_mode != 0 && R->level_mode != 1) return IHT_EINVAL;
  const int64_t npix = (int64_t)R->grid * R->grid;
  RadioArgs a{};
  a.u = R->u;
  a.v = R->v;
  a.nvis = R->nvis;
  a.row_offset = R->row_offset;
  a.rpad = rows_pad(R->nvis);
  a.grid = R->grid;
  a.npix = npix;
  a.bits = R->bits;
  a.L = R->bits ? num_levels(R->bits, R->level_mode) : 2;
  a.c = R->scale_c;
  a.sf = R->scale_c == 0.0f ? 0.0f : (float)(a.L - 1) / (2.0f * R->scale_c);
  a.sigma = R->scale_c / (float)(a.L - 1);
  a.copy_id = (uint32_t)R->copy_id;
  a.k0 = (uint32_t)(R->seed & 0xFFFFFFFFull);
  a.k1 = (uint32_t)(R->seed >> 32);
  a.r = r;
  a.g = g;
  const unsigned grid = (unsigned)((npix + 4 * kRdThreads - 1) / (4 * kRdThreads));
  if (R->bits) adjoint_radio_kernel<true><<<grid, kRdThreads, 0, (cudaStream_t)stream>>>(a);
  else adjoint_radio_kernel<false><<<grid, kRdThreads, 0, (cudaStream_t)stream>>>(a);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
