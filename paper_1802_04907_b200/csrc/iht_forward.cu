// (a4) forward residual r = y-hat - Phi-hat_F x over the support of x only.
//
// P:349 (Algorithm 1: y-hat - Phi-hat_{2n} x^{[n]}); the paper's CPU code casts this
// as "a matrix times a sparse vector ... a dense scale-and-add routine"
// and takes "advantage of the sparsity of the x vectors".  With column
// strips each support column is a contiguous run of R codes, so the scale-and-add
// streams s * R * b / 8 bytes (0.4% of the adjoint's bytes at config 4).
//
// Mapping: a CTA owns a window of 32 consecutive 32-bit code words of every strip
// (32 * 32/b stacked rows); its 16 warps split the support in rounds of 16 columns
// (loads issued before use), each lane accumulates the 32/b rows of its word, and the 8
// partial sums are added in a fixed order through shared memory (deterministic).
// Batched (config 5): grid row blockIdx.y = snapshot b, with its own x_b, y-hat_b, r_b.
// Column shards: x holds GLOBAL indices; only [col_offset, col_offset + cols) are local.
#include "iht_internal.cuh"

namespace iht {

constexpr int kFwdWarps = 16;
constexpr int kFwdUnroll = 16;

template <int B>
__global__ void __launch_bounds__(kFwdWarps * 32) forward_kernel(
    const uint8_t* __restrict__ codes, int64_t strip_bytes, int64_t words_total, int64_t rows,
    int64_t rpad, int L, float sigma,
    const int32_t* __restrict__ x_idx, const float* __restrict__ x_val,
    const int32_t* __restrict__ x_nnz, int32_t max_nnz, int32_t ldx, int64_t col_offset, int64_t ncols,
    const float* __restrict__ yhat, float* __restrict__ r, int64_t vlen) {
  constexpr int CPW = 32 / B;
  constexpr uint32_t MASK = (1u << B) - 1u;
  __shared__ float part[kFwdWarps][32][CPW + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t word = (int64_t)blockIdx.x * 32 + lane;
  const bool live = word < words_total;
  {
    const int b = blockIdx.y;
    x_idx += (int64_t)b * ldx;
    x_val += (int64_t)b * ldx;
    x_nnz += b;
    if (yhat) yhat += (int64_t)b * vlen;
    r += (int64_t)b * vlen;
  }
  int nnz = *x_nnz;
  nnz = nnz < 0 ? 0 : (nnz > max_nnz ? max_nnz : nnz);
  const float negLm1 = -(float)(L - 1);

  float acc[CPW];
#pragma unroll
  for (int i = 0; i < CPW; ++i) acc[i] = 0.0f;

  // kFwdUnroll support columns per round, their code words loaded before use
  const int64_t kofs = (word >> 4) * 1024 + (word & 15) * 4;   // tiled offset of this word, sans column
  for (int j0 = warp * kFwdUnroll; j0 < nnz; j0 += kFwdWarps * kFwdUnroll) {
    uint32_t w[kFwdUnroll];
    float xv[kFwdUnroll];
#pragma unroll
    for (int u = 0; u < kFwdUnroll; ++u) {
      const int j = j0 + u;
      int64_t col = j < nnz ? (int64_t)__ldg(x_idx + j) - col_offset : 0;
      const bool ok = j < nnz && col >= 0 && col < ncols;   // outside this column shard: skip
      col = ok ? col : 0;
      xv[u] = ok ? __ldg(x_val + j) : 0.0f;
      w[u] = (ok && live) ? __ldg(reinterpret_cast<const uint32_t*>(
                                codes + (col >> 4) * (16 * strip_bytes) + (col & 15) * 64 + kofs))
                          : 0u;
    }
#pragma unroll
    for (int u = 0; u < kFwdUnroll; ++u) {
#pragma unroll
      for (int i = 0; i < CPW; ++i) {
        // code -> float exactly: 2^23 + code, minus 2^23; q = 2 code - (L-1) exactly
        const float cf = __int_as_float(0x4B000000u | ((w[u] >> (i * B)) & MASK)) - 8388608.0f;
        const float q = __fmaf_rn(2.0f, cf, negLm1);
        acc[i] = __fmaf_rn(xv[u], q, acc[i]);   // xv = 0 for j >= nnz: adds +0, exact
      }
    }
  }
#pragma unroll
  for (int i = 0; i < CPW; ++i) part[warp][lane][i] = acc[i];
  __syncthreads();
  // warp 0 combines the kFwdWarps partials in fixed order
  if (warp == 0 && live) {
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      float s = part[0][lane][i];
#pragma unroll
      for (int w2 = 1; w2 < kFwdWarps; ++w2) s = __fadd_rn(s, part[w2][lane][i]);
      const int64_t m = word * CPW + i;   // stacked row p * rpad + local row
      const float yv = yhat ? yhat[m] : 0.0f;      // NULL y-hat: partial product (column shards)
      r[m] = (m % rpad) < rows ? __fsub_rn(yv, __fmul_rn(sigma, s)) : 0.0f;  // pad rows: 0
    }
  }
}

}  // namespace iht

using namespace iht;

extern "C" int64_t iht_forward_ws_bytes(const iht_qmat* F, int32_t max_nnz) {
  (void)F;
  (void)max_nnz;
  return 0;
}

extern "C" int iht_forward(const iht_qmat* F, const int32_t* x_idx, const float* x_val,
                           const int32_t* x_nnz, int32_t max_nnz, const float* yhat, float* r,
                           void* ws, int64_t ws_bytes, void* stream) {
  (void)ws;
  (void)ws_bytes;
  if (yhat == nullptr) return IHT_EINVAL;
  return iht_forward_batched(F, x_idx, x_val, x_nnz, max_nnz, max_nnz, 1, yhat, r, stream);
}

extern "C" int iht_forward_batched(const iht_qmat* F, const int32_t* x_idx, const float* x_val,
                                   const int32_t* x_nnz, int32_t ldx, int32_t max_nnz, int32_t nrhs,
                                   const float* yhat, float* r, void* stream) {
  if (F == nullptr || x_nnz == nullptr || r == nullptr || max_nnz < 0 || nrhs <= 0 || nrhs > 65535)
    return IHT_EINVAL;
  if (ldx < max_nnz && nrhs > 1) return IHT_EINVAL;
  max_nnz = ldx < max_nnz ? ldx : max_nnz;
  if (max_nnz > 0 && (x_idx == nullptr || x_val == nullptr)) return IHT_EINVAL;
  if (F->col_offset < 0) return IHT_EINVAL;
  if (F->codes == nullptr || (F->bits != 2 && F->bits != 4 && F->bits != 8)) return IHT_EINVAL;
  if (F->strip_bytes != iht_strip_bytes(F->rows, F->planes, F->bits)) return IHT_EINVAL;
  const int L = num_levels(F->bits, F->level_mode);
  const float sigma = F->scale_c / (float)(L - 1);
  const int64_t words_total = F->strip_bytes / 4;
  const unsigned blocks = (unsigned)ceil_div<int64_t>(words_total, 32);
  const int64_t vlen = iht_vec_len(F->rows, F->planes);
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* codes = static_cast<const uint8_t*>(F->codes);
#define IHT_FWD(BB)                                                                             \
  forward_kernel<BB><<<dim3(blocks, nrhs), kFwdWarps * 32, 0, st>>>(                           \
      codes, F->strip_bytes, words_total, F->rows, iht_rows_pad(F->rows), L, sigma, x_idx, x_val, x_nnz, \
      max_nnz, ldx, F->col_offset, F->cols, yhat, r, vlen)
  if (F->bits == 2) IHT_FWD(2);
  else if (F->bits == 4) IHT_FWD(4);
  else IHT_FWD(8);
#undef IHT_FWD
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
