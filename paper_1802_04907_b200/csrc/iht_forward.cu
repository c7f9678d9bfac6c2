// (a4) forward residual r = y-hat - Phi-hat_F x over the support of x only.
//
// P:349 (Algorithm 1: y-hat - Phi-hat_{2n} x^{[n]}); the paper's CPU code casts this
// as "a matrix times a sparse vector ... a dense scale-and-add routine"
// and takes "advantage of the sparsity of the x vectors".  With column
// strips each support column is a contiguous run of R codes, so the scale-and-add
// streams s * R * b / 8 bytes (0.4% of the adjoint's bytes at config 4).
//
// Mapping: a CTA owns a window of WPC = 8 (or 32) consecutive 32-bit code words of every
// strip (WPC * 32/b stacked rows); each warp load instruction covers 32/WPC support
// columns x WPC words, 8 such loads in flight per lane; partial sums are combined in a
// fixed order (shuffles, then shared memory), so r is deterministic.
// Batched (config 5): grid row blockIdx.y = snapshot b, with its own x_b, y-hat_b, r_b.
// Column shards: x holds GLOBAL indices; only [col_offset, col_offset + cols) are local.
#include <stdlib.h>

#include "iht_internal.cuh"

namespace iht {

constexpr int kFwdThreads = 256;       // 8 warps
// WPC = 32-bit code words (WPC * 32/b rows) per CTA: 8 (lane = 4 column slots x 8 words),
// or 32 for many small batched problems (lane = word, one column per warp load, 4x fewer
// CTAs: config 5's 64 snapshots x 36 CTAs at 64 registers per thread were 3.9 waves)
constexpr int kFwdUnroll = 8;          // support columns in flight per lane
constexpr int kFwdStage = 1536;        // support entries staged in shared memory per round (18 KiB)

// CTA = (chunk of 8 words of every strip, snapshot b).  Lane = (column slot c in 0..3,
// word wl in 0..7): one load instruction of a warp reads 4 columns x one 32-byte sector.
// The snapshot's support (idx, val) is staged in shared memory first, so the code loads
// depend on a shared-memory read only.  Partial sums: shuffle over the 4 column slots,
// then over the 8 warps through shared memory, both in a fixed order (deterministic).
template <int B, int kFwdWords>
__global__ void __launch_bounds__(kFwdThreads) forward_kernel(
    const uint8_t* __restrict__ codes, int64_t strip_bytes, int64_t words_total, int rows, int rpad, int L,
    float sigma, const int32_t* __restrict__ x_idx, const float* __restrict__ x_val,
    const int32_t* __restrict__ x_nnz, int32_t max_nnz, int32_t ldx, int64_t col_offset, int64_t ncols,
    const float* __restrict__ yhat, float* __restrict__ r, int64_t vlen, int strips) {
  constexpr int CPW = 32 / B;
  constexpr uint32_t MASK = (1u << B) - 1u;
  __shared__ float part[kFwdThreads / 32][kFwdWords][CPW];
  __shared__ int64_t sidx[kFwdStage];   // tiled byte offset of each staged support column
  __shared__ float sval[kFwdStage];
  pdl_launch_dependents();
  pdl_wait();                                   // x (previous H_s) and y-hat
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CS = 32 / kFwdWords;            // column slots per warp load
  const int c = lane / kFwdWords, wl = lane % kFwdWords;
  const int b = blockIdx.y;
  x_idx += (int64_t)b * ldx;
  x_val += (int64_t)b * ldx;
  if (yhat) yhat += (int64_t)b * vlen;
  r += (int64_t)b * vlen;
  // y-hat of this thread's output rows (final loop below), loaded before the support so
  // that its latency overlaps the code loads instead of ending the chain
  constexpr int kOutPer = (kFwdWords * CPW + kFwdThreads - 1) / kFwdThreads;
  float ypre[kOutPer];
#pragma unroll
  for (int k = 0; k < kOutPer; ++k) {
    const int t = threadIdx.x + k * kFwdThreads;
    const int64_t m = (int64_t)blockIdx.x * kFwdWords * CPW + t;
    ypre[k] = (yhat && t < kFwdWords * CPW && m < (int64_t)words_total * CPW) ? yhat[m] : 0.0f;
  }
  int nnz = x_nnz[b];
  nnz = nnz < 0 ? 0 : (nnz > max_nnz ? max_nnz : nnz);
  const int64_t word = (int64_t)blockIdx.x * kFwdWords + wl;
  const bool live = word < words_total;
  // tiled offset of this word, sans column (strips: column-contiguous layout)
  const int64_t kofs = strips ? word * 4 : (word >> 4) * 1024 + (word & 15) * 4;
  // acc_i = sum_j x_j code_ij and xs = sum_j x_j; the affine map q = 2 code - (L-1) is
  // applied once at the end: sum_j x_j q_ij = 2 acc_i - (L-1) xs
  float acc[CPW];
#pragma unroll
  for (int i = 0; i < CPW; ++i) acc[i] = 0.0f;
  float xs = 0.0f;
  for (int st0 = 0; st0 < nnz; st0 += kFwdStage) {
  const int nst = nnz - st0 < kFwdStage ? nnz - st0 : kFwdStage;
  __syncthreads();
  // stage the support: byte offset of each column's tile + slot (columns outside this
  // shard get value 0 and column 0, adding +0 exactly)
  for (int j = threadIdx.x; j < nst; j += kFwdThreads) {
    int64_t col = (int64_t)x_idx[st0 + j] - col_offset;
    const bool ok = col >= 0 && col < ncols;
    col = ok ? col : 0;
    sidx[j] = strips ? col * strip_bytes : (col >> 4) * (16 * strip_bytes) + (col & 15) * 64;
    sval[j] = ok ? x_val[st0 + j] : 0.0f;
  }
  __syncthreads();
  for (int jb = warp * CS; jb < nst; jb += 8 * CS * kFwdUnroll) {   // warp-uniform trip count
    const int j0 = jb + c;
    uint32_t w[kFwdUnroll];
    float xv[kFwdUnroll];
#pragma unroll
    for (int u = 0; u < kFwdUnroll; ++u) {
      const int j = j0 + 8 * CS * u;
      const bool ok = j < nst && live;
      xv[u] = j < nst ? sval[j] : 0.0f;
      IHT_DCHECK(!ok || sidx[j] + kofs + 4 <= (ncols + 15) / 16 * 16 * strip_bytes, "forward: code word inside the copy");
      w[u] = ok ? __ldg(reinterpret_cast<const uint32_t*>(codes + sidx[j] + kofs)) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kFwdUnroll; ++u) {
      if (!__any_sync(0xffffffffu, j0 + 8 * CS * u < nst)) break;     // warp-uniform: skip empty slots
      xs = __fadd_rn(xs, xv[u]);
#pragma unroll
      for (int i = 0; i < CPW; ++i) {
        // code -> float exactly: 2^23 + code, minus 2^23
        const float cf = __int_as_float(0x4B000000u | ((w[u] >> (i * B)) & MASK)) - 8388608.0f;
        acc[i] = __fmaf_rn(xv[u], cf, acc[i]);   // xv = 0 past the support: adds +0, exact
      }
    }
  }
  }
  // q-sum of each row (affine map), then the fixed-order reduction over the 4 column slots
  const float xl = __fmul_rn((float)(L - 1), xs);
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    acc[i] = __fsub_rn(__fmul_rn(2.0f, acc[i]), xl);
#pragma unroll
    for (int o = kFwdWords; o < 32; o <<= 1) acc[i] = __fadd_rn(acc[i], __shfl_xor_sync(0xffffffffu, acc[i], o));
  }
  if (c == 0) {
#pragma unroll
    for (int i = 0; i < CPW; ++i) part[warp][wl][i] = acc[i];
  }
  __syncthreads();
  // one output row per thread, over the 8 warps in a fixed order; coalesced r writes
#pragma unroll
  for (int k = 0; k < kOutPer; ++k) {
    const int t = threadIdx.x + k * kFwdThreads;
    if (t >= kFwdWords * CPW) break;
    const int ww = t / CPW, i = t % CPW;
    const int64_t m = ((int64_t)blockIdx.x * kFwdWords + ww) * CPW + i;   // stacked row p * rpad + local row
    if (m >= (int64_t)words_total * CPW) continue;
    float s = part[0][ww][i];
#pragma unroll
    for (int w2 = 1; w2 < kFwdThreads / 32; ++w2) s = __fadd_rn(s, part[w2][ww][i]);
    const float yv = ypre[k];                    // 0 for a NULL y-hat: partial product (column shards)
    r[m] = (int)(m % rpad) < rows ? __fsub_rn(yv, __fmul_rn(sigma, s)) : 0.0f;  // pad rows: 0
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
  const unsigned blocks8 = (unsigned)ceil_div<int64_t>(words_total, 8);
  const unsigned blocks32 = (unsigned)ceil_div<int64_t>(words_total, 32);
  // many CTAs of tiny work (batched, small support): 4x wider CTAs, about one wave
  const bool wide = nrhs > 1 && (int64_t)blocks8 * nrhs > 4 * (int64_t)kNumSMs;
  // a single observation over many rows (config 4: 8192 words): 16 words = one whole 64-byte
  // piece of each support column per CTA (a full DRAM burst instead of half of one)
  const unsigned blocks16 = (unsigned)ceil_div<int64_t>(words_total, 16);
  static int ww_env = -1;                        // profiling override (IHT_FWD_WORDS = 8, 16, 32)
  if (ww_env < 0) ww_env = getenv("IHT_FWD_WORDS") ? atoi(getenv("IHT_FWD_WORDS")) : 0;
  static int strips_env = -1;                    // EXPERIMENT: column-contiguous address pattern
  if (strips_env < 0) strips_env = getenv("IHT_FWD_STRIPS") ? atoi(getenv("IHT_FWD_STRIPS")) : 0;
  const bool mid = ww_env == 16 || (ww_env == 0 && nrhs == 1 && blocks16 >= 2u * kNumSMs);
  const int64_t vlen = iht_vec_len(F->rows, F->planes);
  if (F->rows > 0x7FFFFFFF) return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* codes = static_cast<const uint8_t*>(F->codes);
#define IHT_FWD(BB, WW, NBLK)                                                                   \
  IHT_CUDA_CHECK(launch_pdl(forward_kernel<BB, WW>, dim3(NBLK, nrhs), dim3(kFwdThreads), 0, st, codes,    \
                            F->strip_bytes, words_total, (int)F->rows, (int)iht_rows_pad(F->rows), L, sigma, \
                            x_idx, x_val, x_nnz, max_nnz, ldx, F->col_offset, F->cols, yhat, r, vlen, strips_env))
  if ((wide && ww_env == 0) || ww_env == 32) {
    if (F->bits == 2) IHT_FWD(2, 32, blocks32);
    else if (F->bits == 4) IHT_FWD(4, 32, blocks32);
    else IHT_FWD(8, 32, blocks32);
  } else if (mid) {
    if (F->bits == 2) IHT_FWD(2, 16, blocks16);
    else if (F->bits == 4) IHT_FWD(4, 16, blocks16);
    else IHT_FWD(8, 16, blocks16);
  } else {
    if (F->bits == 2) IHT_FWD(2, 8, blocks8);
    else if (F->bits == 4) IHT_FWD(4, 8, blocks8);
    else IHT_FWD(8, 8, blocks8);
  }
#undef IHT_FWD
  return IHT_OK;
}
