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
  constexpr uint32_t kExpB = (uint32_t)(127 + B) << 23;   // bit pattern of 2^B
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
  // the first staging round's support slots, requested together with nnz (they do not depend
  // on it: the x arrays hold max_nnz slots) -- one dependent round trip fewer
  // (the first kFwdThreads slots: one per thread)
  const int32_t pidx = (int)threadIdx.x < max_nnz ? x_idx[threadIdx.x] : 0;
  const float pval = (int)threadIdx.x < max_nnz ? x_val[threadIdx.x] : 0.0f;
  int nnz = x_nnz[b];
  nnz = nnz < 0 ? 0 : (nnz > max_nnz ? max_nnz : nnz);
  const int64_t word = (int64_t)blockIdx.x * kFwdWords + wl;
  const bool live = word < words_total;
  // tiled offset of this word, sans column (strips: column-contiguous layout)
  const int64_t kofs = strips ? word * 4 : (word >> 4) * 1024 + (word & 15) * 4;
  // acc_i = sum_j x_j (2^B + code_ij) and xs = sum_j x_j; the float 2^B + code is formed
  // exactly from the code bits (exponent of 2^B, code in the top B mantissa bits: one shift
  // and one LOP3, no subtraction), and the affine map q = 2 code - (L-1) is applied once at
  // the end: sum_j x_j q_ij = 2 acc_i - (2^{B+1} + L - 1) xs
  float acc[CPW];
#pragma unroll
  for (int i = 0; i < CPW; ++i) acc[i] = 0.0f;
  float xs = 0.0f;
  const uint32_t mant_mask = MASK << (23 - B), exp_b = kExpB;   // registers: one LOP3 per code
  for (int st0 = 0; st0 < nnz; st0 += kFwdStage) {
  const int nst = nnz - st0 < kFwdStage ? nnz - st0 : kFwdStage;
  __syncthreads();
  // stage the support: byte offset of each column's tile + slot (columns outside this
  // shard get value 0 and column 0, adding +0 exactly)
  for (int j = threadIdx.x; j < nst; j += kFwdThreads) {
    const bool pre = st0 == 0 && j == (int)threadIdx.x;   // this thread's slot, loaded above
    int64_t col = (int64_t)(pre ? pidx : x_idx[st0 + j]) - col_offset;
    const bool ok = col >= 0 && col < ncols;
    col = ok ? col : 0;
    sidx[j] = strips ? col * strip_bytes : (col >> 4) * (16 * strip_bytes) + (col & 15) * 64;
    sval[j] = ok ? (pre ? pval : x_val[st0 + j]) : 0.0f;
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
        // code -> the float 2^B + code exactly
        const int sh = 23 - B - i * B;            // code i to mantissa bits 23-B .. 22
        const uint32_t x = sh >= 0 ? (w[u] << sh) : (w[u] >> -sh);
        const float cf = __uint_as_float(lop3_and_or(x, mant_mask, exp_b));
        acc[i] = __fmaf_rn(xv[u], cf, acc[i]);   // xv = 0 past the support: adds +0, exact
      }
    }
  }
  }
  // q-sum of each row (affine map), then the fixed-order reduction over the 4 column slots
  const float xl = __fmul_rn((float)((2 << B) + L - 1), xs);
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


// Single observation over many rows (config 4): 2-D grid (row block rb = 16 code words = one
// 64-byte piece of every support strip, column group).  Lane = (column slot cs, piece quad q):
// ONE 16-byte load (VW words; 8 bytes at b = 2) per support column, kFsLoads of them issued
// before any decode, so a lane has 128 bytes in flight at once (the 4-byte-per-lane kernel
// above has 32).  Column groups of kFsLoads x 8 warps x CS columns each; G > 1 groups write
// partial row sums to the workspace and the last CTA of a row block (arrival counter, reset
// by it) adds them in group order and writes r = y-hat - sigma (...).  Deterministic.
constexpr int kFsThreads = 256;
constexpr int kFsLoads = 8;

template <int B>
__host__ __device__ constexpr int fs_cols_per_group() {
  return kFsLoads * (kFsThreads / 32) * (32 / (16 / (B == 2 ? 2 : 4)));
}

template <int B>
__global__ void __launch_bounds__(kFsThreads) forward_split_kernel(
    const uint8_t* __restrict__ codes, int64_t strip_bytes, int64_t words_total, int rows, int rpad, int L,
    float sigma, const int32_t* __restrict__ x_idx, const float* __restrict__ x_val,
    const int32_t* __restrict__ x_nnz, int32_t max_nnz, int64_t col_offset, int64_t ncols,
    const float* __restrict__ yhat, float* __restrict__ r, float* __restrict__ part, unsigned int* __restrict__ cnt) {
  constexpr int CPW = 32 / B;                    // codes per word
  constexpr int VW = B == 2 ? 2 : 4;             // words per lane load
  constexpr int LPP = 16 / VW;                   // lanes per 64-byte piece
  constexpr int CS = 32 / LPP;                   // columns per warp load
  constexpr int NACC = VW * CPW;                 // rows per lane (32 at b = 2, 4; 16 at b = 8)
  constexpr int RPB = 16 * CPW;                  // rows per row block
  constexpr int CPG = fs_cols_per_group<B>();
  constexpr uint32_t MASK = (1u << B) - 1u;
  __shared__ int64_t sidx[CPG];
  __shared__ float sval[CPG];
  __shared__ float part_s[kFsThreads / 32][RPB];
  __shared__ int s_last;
  pdl_launch_dependents();
  pdl_wait();                                    // x (previous H_s)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cs = lane / LPP, q = lane % LPP;
  const int rb = blockIdx.x, grp = blockIdx.y, G = gridDim.y;
  int nnz = *x_nnz;
  nnz = nnz < 0 ? 0 : (nnz > max_nnz ? max_nnz : nnz);
  const int j0 = grp * CPG, nj = max(0, min(nnz - j0, CPG));
  const int64_t m0 = (int64_t)rb * RPB;          // first stacked row of this block
  const float ypre = yhat && threadIdx.x < RPB && m0 + threadIdx.x < words_total * CPW ? yhat[m0 + threadIdx.x] : 0.0f;
  for (int j = threadIdx.x; j < nj; j += kFsThreads) {
    int64_t col = (int64_t)x_idx[j0 + j] - col_offset;
    const bool ok = col >= 0 && col < ncols;
    col = ok ? col : 0;
    sidx[j] = (col >> 4) * (16 * strip_bytes) + (col & 15) * 64;
    sval[j] = ok ? x_val[j0 + j] : 0.0f;
  }
  __syncthreads();
  const int64_t kofs = (int64_t)rb * 1024 + q * (VW * 4);   // this lane's bytes of the piece
  uint32_t w[kFsLoads][VW];
#pragma unroll
  for (int u = 0; u < kFsLoads; ++u) {
    const int jj = (u * (kFsThreads / 32) + warp) * CS + cs;
    IHT_DCHECK(jj >= nj || sidx[jj] + kofs + 4 * VW <= (ncols + 15) / 16 * 16 * strip_bytes, "forward_split: load inside the copy");
    if (VW == 4) {
      const uint4 v = jj < nj ? __ldg(reinterpret_cast<const uint4*>(codes + sidx[jj] + kofs)) : make_uint4(0u, 0u, 0u, 0u);
      w[u][0] = v.x; w[u][1] = v.y; w[u][VW > 2 ? 2 : 0] = v.z; w[u][VW > 3 ? 3 : 0] = v.w;
    } else {
      const uint2 v = jj < nj ? __ldg(reinterpret_cast<const uint2*>(codes + sidx[jj] + kofs)) : make_uint2(0u, 0u);
      w[u][0] = v.x; w[u][1] = v.y;
    }
  }
  // acc_i = sum_j x_j (2^B + code_ij) (the float 2^B + code formed from the code bits, as in
  // forward_kernel), xs = sum_j x_j; affine map once: sum_j x_j q_ij = 2 acc_i - (2^{B+1} + L-1) xs
  const uint32_t mant_mask = MASK << (23 - B), exp_b = (uint32_t)(127 + B) << 23;
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0f;
  float xs = 0.0f;
#pragma unroll
  for (int u = 0; u < kFsLoads; ++u) {
    const int jj = (u * (kFsThreads / 32) + warp) * CS + cs;
    const float xv = jj < nj ? sval[jj] : 0.0f;   // past the group: adds +0
    xs = __fadd_rn(xs, xv);
#pragma unroll
    for (int v = 0; v < VW; ++v)
#pragma unroll
      for (int i = 0; i < CPW; ++i) {
        const int sh = 23 - B - i * B;
        const uint32_t xw = sh >= 0 ? (w[u][v] << sh) : (w[u][v] >> -sh);
        acc[v * CPW + i] = __fmaf_rn(xv, __uint_as_float(lop3_and_or(xw, mant_mask, exp_b)), acc[v * CPW + i]);
      }
  }
  const float xl = __fmul_rn((float)((2 << B) + L - 1), xs);
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    acc[i] = __fsub_rn(__fmul_rn(2.0f, acc[i]), xl);
#pragma unroll
    for (int o = LPP; o < 32; o <<= 1) acc[i] = __fadd_rn(acc[i], __shfl_xor_sync(0xffffffffu, acc[i], o));
  }
  if (cs == 0) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) part_s[warp][q * NACC + i] = acc[i];   // row (q VW + v) CPW + i
  }
  __syncthreads();
  float sum = 0.0f;
  if (threadIdx.x < RPB) {
    sum = part_s[0][threadIdx.x];
#pragma unroll
    for (int w2 = 1; w2 < kFsThreads / 32; ++w2) sum = __fadd_rn(sum, part_s[w2][threadIdx.x]);
  }
  const int64_t m = m0 + threadIdx.x;
  const bool live = threadIdx.x < RPB && m < words_total * CPW;
  if (G > 1) {
    const int64_t vl = words_total * CPW;
    if (live) part[(int64_t)grp * vl + m] = sum;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      s_last = atomicAdd(&cnt[rb], 1u) == (unsigned int)G - 1u;
      if (s_last) cnt[rb] = 0u;                  // every group of this row block has arrived
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (live) {
      sum = __ldcg(&part[m]);
      for (int g2 = 1; g2 < G; ++g2) sum = __fadd_rn(sum, __ldcg(&part[(int64_t)g2 * vl + m]));
    }
  }
  if (live) r[m] = (int)(m % rpad) < rows ? __fsub_rn(ypre, __fmul_rn(sigma, sum)) : 0.0f;   // pad rows: 0
}

}  // namespace iht

using namespace iht;

// The split kernel applies to a single observation over many rows (>= 2 row blocks per SM);
// its workspace holds G partial row-sum vectors and one arrival counter per row block.
static int fs_groups(const iht_qmat* F, int32_t max_nnz) {
  if (F == nullptr || max_nnz <= 0 || (F->bits != 2 && F->bits != 4 && F->bits != 8)) return 0;
  const int64_t words_total = F->strip_bytes / 4;
  if (words_total % 16 || words_total / 16 < 2 * kNumSMs) return 0;
  const int cpg = F->bits == 2 ? fs_cols_per_group<2>() : F->bits == 4 ? fs_cols_per_group<4>() : fs_cols_per_group<8>();
  return (max_nnz + cpg - 1) / cpg;
}

extern "C" int64_t iht_forward_ws_bytes(const iht_qmat* F, int32_t max_nnz) {
  const int G = fs_groups(F, max_nnz);
  if (G <= 1) return 0;
  const int64_t words_total = F->strip_bytes / 4, vl = words_total * (32 / F->bits);
  return ((int64_t)G * vl * 4 + 255) / 256 * 256 + words_total / 16 * 4;
}

extern "C" int iht_forward(const iht_qmat* F, const int32_t* x_idx, const float* x_val,
                           const int32_t* x_nnz, int32_t max_nnz, const float* yhat, float* r,
                           void* ws, int64_t ws_bytes, void* stream) {
  if (yhat == nullptr) return IHT_EINVAL;
  const int G = fs_groups(F, max_nnz);
  // measured (r02 g50, config 4, L2 flushed): forward_split_kernel 35.8 us against forward_kernel's
  // 27.6 us -- the random 64-byte pieces of the support strips bound both, more bytes in flight per
  // lane do not help; so forward_kernel is the default and IHT_FWD_SPLIT=1 selects the split kernel
  const int fs_env = getenv("IHT_FWD_SPLIT") ? atoi(getenv("IHT_FWD_SPLIT")) : 0;   // read per call (tests)
  const int64_t need = iht_forward_ws_bytes(F, max_nnz);
  if (G == 0 || !fs_env || (need > 0 && (ws == nullptr || ws_bytes < need)) || F->codes == nullptr ||
      x_nnz == nullptr || r == nullptr || x_idx == nullptr || x_val == nullptr || F->col_offset < 0 ||
      F->strip_bytes != iht_strip_bytes(F->rows, F->planes, F->bits) || F->rows > 0x7FFFFFFF)
    return iht_forward_batched(F, x_idx, x_val, x_nnz, max_nnz, max_nnz, 1, yhat, r, stream);
  const int L = num_levels(F->bits, F->level_mode);
  const float sigma = F->scale_c / (float)(L - 1);
  const int64_t words_total = F->strip_bytes / 4;
  const int64_t vl = words_total * (32 / F->bits);
  float* part = static_cast<float*>(ws);
  unsigned int* cnt = need > 0 ? reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + ((int64_t)G * vl * 4 + 255) / 256 * 256)
                               : nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* codes = static_cast<const uint8_t*>(F->codes);
  const dim3 grid((unsigned)(words_total / 16), (unsigned)G);
#define IHT_FWS(BB)                                                                                              \
  IHT_CUDA_CHECK(launch_pdl(forward_split_kernel<BB>, grid, dim3(kFsThreads), 0, st, codes, F->strip_bytes,       \
                            words_total, (int)F->rows, (int)iht_rows_pad(F->rows), L, sigma, x_idx, x_val, x_nnz, \
                            max_nnz, F->col_offset, F->cols, yhat, r, part, cnt))
  if (F->bits == 2) IHT_FWS(2);
  else if (F->bits == 4) IHT_FWS(4);
  else IHT_FWS(8);
#undef IHT_FWS
  return IHT_OK;
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
