// NEXT-2: exact fresh copies at scale.  Algorithm 1 takes 2n* independent
// quantisations Phi-hat_1 .. Phi-hat_{2n*}; config 4 cannot store them (8 GiB
// each), so these kernels draw the copy ON THE FLY from the fp32 Phi: every code is the
// Q-contract rounding of Phi_mn with the Philox word of counter
// (n >> 2, row_offset + m, copy_id, plane << 8), exactly the code iht_quantize would have
// stored -- so iteration n uses copy ids 2n-2 (adjoint, Phi-hat_{2n-1}) and 2n-1 (forward,
// Phi-hat_{2n}), K = 2 n* with no storage.
//
// Roofline: the adjoint streams 4 bytes of fp32 Phi per entry (vs b/8 for stored codes)
// plus one Philox4x32-10 per 4 entries and plane (~60 integer ops) -- HBM and ALU bound
// together.  The forward reads only the s support columns.
#include "iht_internal.cuh"

namespace iht {

constexpr int kFrThreads = 256;          // 256 threads x 4 columns = 1024 columns per CTA
constexpr int kFrUnroll = 4;             // rows in flight per thread

struct FreshArgs {
  const float* phi;      // local row m, column n: phi[(m * ld + n) * P + plane]
  int64_t ld;            // row stride in (complex) elements
  int64_t rows, cols, row_offset, rpad;
  int64_t rows_per_split;
  float c, sf, sigma;
  int L;
  uint32_t copy_id, k0, k1;
  const float* r;        // stacked vector
  float* part;           // [splits][cols] partial sums (sigma applied by the reduce)
};

// Column quad (4 columns, one Philox call per row and plane serves all four) x a range of
// rows; acc_j = sum_m q_mj r_m with q = 2 code - (L-1) (exact small integers in fp32).
template <int P>
__global__ void __launch_bounds__(kFrThreads) adjoint_fresh_kernel(FreshArgs a) {
  const int64_t quad = (int64_t)blockIdx.x * kFrThreads + threadIdx.x;
  const int64_t n0 = quad * 4;
  const bool live = n0 < a.cols;
  const int64_t m_begin = (int64_t)blockIdx.y * a.rows_per_split;
  const int64_t m_end = min64(a.rows, m_begin + a.rows_per_split);
  const int ncol = live ? (int)min64(4, a.cols - n0) : 0;
  const float Lm1 = (float)(a.L - 1);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t m0 = m_begin; m0 < m_end; m0 += kFrUnroll) {
    float v[kFrUnroll][P][4];
#pragma unroll
    for (int u = 0; u < kFrUnroll; ++u) {
      const int64_t m = m0 + u;
      const float* row = a.phi + (m * a.ld + n0) * P;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int p = 0; p < P; ++p) v[u][p][j] = (live && m < m_end && j < ncol) ? __ldg(row + j * P + p) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kFrUnroll; ++u) {
      const int64_t m = m0 + u;
      if (m >= m_end) break;
      const uint32_t mg = (uint32_t)(a.row_offset + m);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float rv = __ldg(a.r + p * a.rpad + m);
        const u32x4 w = philox4x32_10(u32x4{(uint32_t)quad, mg, a.copy_id, (uint32_t)(p << 8)}, a.k0, a.k1);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t code = q_contract(v[u][p][j], a.c, a.sf, a.L, ws[j]);
          const float q = __fmaf_rn(2.0f, (float)code, -Lm1);
          acc[j] = __fmaf_rn(q, rv, acc[j]);
        }
      }
    }
  }
  if (live) {
    float* out = a.part + (int64_t)blockIdx.y * a.cols + n0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ncol) out[j] = acc[j];
  }
}

// g_n = sigma * sum over the row splits (fixed order: deterministic).
__global__ void fresh_reduce_kernel(const float* __restrict__ part, int splits, int64_t cols, float sigma,
                                    float* __restrict__ g) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= cols) return;
  float s = part[n];
  for (int k = 1; k < splits; ++k) s = __fadd_rn(s, part[(int64_t)k * cols + n]);
  g[n] = __fmul_rn(sigma, s);
}

// r_m = y-hat_m - sigma sum_{j in S} q^F_{m j} x_j: one thread per local row (both planes),
// the support staged in shared memory; each code drawn from its own Philox word.
template <int P>
__global__ void __launch_bounds__(kFrThreads) forward_fresh_kernel(
    const float* __restrict__ phi, int64_t ld, int64_t rows, int64_t row_offset, int64_t rpad, float c, float sf,
    float sigma, int L, uint32_t copy_id, uint32_t k0, uint32_t k1, const int32_t* __restrict__ x_idx,
    const float* __restrict__ x_val, const int32_t* __restrict__ x_nnz, int32_t max_nnz,
    const float* __restrict__ yhat, float* __restrict__ r) {
  __shared__ int32_t sidx[1024];
  __shared__ float sval[1024];
  const int64_t m = (int64_t)blockIdx.x * kFrThreads + threadIdx.x;
  int nnz = *x_nnz;
  nnz = nnz < 0 ? 0 : min(nnz, max_nnz);
  const float Lm1 = (float)(L - 1);
  float acc[P];
#pragma unroll
  for (int p = 0; p < P; ++p) acc[p] = 0.0f;
  const uint32_t mg = (uint32_t)(row_offset + m);
  for (int j0 = 0; j0 < nnz; j0 += 1024) {
    const int nj = min(1024, nnz - j0);
    __syncthreads();
    for (int j = threadIdx.x; j < nj; j += kFrThreads) {
      sidx[j] = x_idx[j0 + j];
      sval[j] = x_val[j0 + j];
    }
    __syncthreads();
    if (m < rows) {
      for (int j = 0; j < nj; ++j) {
        const int64_t n = sidx[j];
        const float xv = sval[j];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float v = __ldg(phi + (m * ld + n) * P + p);
          const u32x4 w = philox4x32_10(u32x4{(uint32_t)(n >> 2), mg, copy_id, (uint32_t)(p << 8)}, k0, k1);
          const uint32_t sel = (uint32_t)(n & 3);
          const uint32_t word = sel == 0 ? w.x : sel == 1 ? w.y : sel == 2 ? w.z : w.w;
          const uint32_t code = q_contract(v, c, sf, L, word);
          acc[p] = __fmaf_rn(__fmaf_rn(2.0f, (float)code, -Lm1), xv, acc[p]);
        }
      }
    }
  }
  if (m < rpad) {
#pragma unroll
    for (int p = 0; p < P; ++p)
      r[p * rpad + m] = m < rows ? __fsub_rn(yhat[p * rpad + m], __fmul_rn(sigma, acc[p])) : 0.0f;
  }
}

// Row splits: the grid is colblocks x splits CTAs of equal work, so it runs in
// ceil(CTAs / resident) waves; pick the fewest splits whose last wave is >= 97 % full
// (config 4: 256 column blocks x 3 splits had been 1.04 waves of 740 resident CTAs, i.e.
// the time of two), at least 64 rows per split.  Deterministic for a given device.
template <int P>
static int fresh_resident(int sms) {
  static int per_sm = 0;
  if (per_sm == 0) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, adjoint_fresh_kernel<P>, kFrThreads, 0) != cudaSuccess ||
        nb < 1) {
      (void)cudaGetLastError();
      nb = 1;
    }
    per_sm = nb;
  }
  return per_sm * sms;
}

static int fresh_splits(int64_t rows, int64_t cols, int planes, int sms) {
  const int64_t colblocks = (cols + 4 * kFrThreads - 1) / (4 * kFrThreads);
  const int64_t cap = planes == 1 ? fresh_resident<1>(sms) : fresh_resident<2>(sms);
  const int64_t smax = max64(1, min64(1024, rows / 64));
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t total = colblocks * sp;
    const int64_t waves = (total + cap - 1) / cap;
    const double eff = (double)total / (double)(waves * cap);
    if (eff >= 0.97) return (int)sp;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
    }
  }
  return (int)best;
}

static bool fmat_valid(const iht_fmat* F) {
  return F && F->phi && F->rows > 0 && F->cols > 0 && F->row_offset >= 0 && (F->planes == 1 || F->planes == 2) &&
         (F->bits == 2 || F->bits == 4 || F->bits == 8) && (F->level_mode == 0 || F->level_mode == 1) &&
         F->ld >= F->cols && isfinite(F->scale_c) && F->scale_c >= 0.0f && F->row_offset + F->rows <= 0xFFFFFFFFll &&
         F->cols / 4 < 0xFFFFFFFFll;
}

}  // namespace iht

using namespace iht;

extern "C" int64_t iht_adjoint_fresh_ws_bytes(const iht_fmat* F) {
  if (!fmat_valid(F)) return -1;
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int64_t)fresh_splits(F->rows, F->cols, F->planes, sms) * F->cols * 4;
}

extern "C" int iht_adjoint_fresh(const iht_fmat* F, int32_t copy_id, const float* r, float* g, void* ws,
                                 int64_t ws_bytes, void* stream) {
  if (!fmat_valid(F) || r == nullptr || g == nullptr || copy_id < 0) return IHT_EINVAL;
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int splits = fresh_splits(F->rows, F->cols, F->planes, sms);
  if (ws == nullptr || ws_bytes < (int64_t)splits * F->cols * 4) return IHT_EINVAL;
  const int L = num_levels(F->bits, F->level_mode);
  FreshArgs a{};
  a.phi = F->phi;
  a.ld = F->ld;
  a.rows = F->rows;
  a.cols = F->cols;
  a.row_offset = F->row_offset;
  a.rpad = rows_pad(F->rows);
  a.rows_per_split = (F->rows + splits - 1) / splits;
  a.c = F->scale_c;
  a.L = L;
  // sf and sigma with the device's own rounding (same as iht_quantize / the other kernels)
  a.sf = F->scale_c == 0.0f ? 0.0f : (float)(L - 1) / (2.0f * F->scale_c);
  a.sigma = F->scale_c / (float)(L - 1);
  a.copy_id = (uint32_t)copy_id;
  a.k0 = (uint32_t)(F->seed & 0xFFFFFFFFull);
  a.k1 = (uint32_t)(F->seed >> 32);
  a.r = r;
  a.part = static_cast<float*>(ws);
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((F->cols + 4 * kFrThreads - 1) / (4 * kFrThreads)), (unsigned)splits);
  if (F->planes == 1) adjoint_fresh_kernel<1><<<grid, kFrThreads, 0, st>>>(a);
  else adjoint_fresh_kernel<2><<<grid, kFrThreads, 0, st>>>(a);
  IHT_LAUNCH_CHECK();
  fresh_reduce_kernel<<<(unsigned)((F->cols + 255) / 256), 256, 0, st>>>(a.part, splits, F->cols, a.sigma, g);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}

extern "C" int iht_forward_fresh(const iht_fmat* F, int32_t copy_id, const int32_t* x_idx, const float* x_val,
                                 const int32_t* x_nnz, int32_t max_nnz, const float* yhat, float* r, void* stream) {
  if (!fmat_valid(F) || x_nnz == nullptr || yhat == nullptr || r == nullptr || max_nnz < 0 || copy_id < 0)
    return IHT_EINVAL;
  if (max_nnz > 0 && (x_idx == nullptr || x_val == nullptr)) return IHT_EINVAL;
  const int L = num_levels(F->bits, F->level_mode);
  const float sf = F->scale_c == 0.0f ? 0.0f : (float)(L - 1) / (2.0f * F->scale_c);
  const float sigma = F->scale_c / (float)(L - 1);
  const int64_t rpad = rows_pad(F->rows);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((rpad + kFrThreads - 1) / kFrThreads);
  const uint32_t k0 = (uint32_t)(F->seed & 0xFFFFFFFFull), k1 = (uint32_t)(F->seed >> 32);
  if (F->planes == 1)
    forward_fresh_kernel<1><<<grid, kFrThreads, 0, st>>>(F->phi, F->ld, F->rows, F->row_offset, rpad, F->scale_c, sf,
                                                          sigma, L, (uint32_t)copy_id, k0, k1, x_idx, x_val, x_nnz,
                                                          max_nnz, yhat, r);
  else
    forward_fresh_kernel<2><<<grid, kFrThreads, 0, st>>>(F->phi, F->ld, F->rows, F->row_offset, rpad, F->scale_c, sf,
                                                          sigma, L, (uint32_t)copy_id, k0, k1, x_idx, x_val, x_nnz,
                                                          max_nnz, yhat, r);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
