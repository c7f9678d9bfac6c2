// (a1) global scale c and (a2)/(a3) stochastic quantisation of Phi and y.
//
// Sec. 3 "Quantization": v in [l_i, l_{i+1}] -> l_i with probability
// (l_{i+1} - v)/(l_{i+1} - l_i), else l_{i+1}; unbiased.  c = max |component|
// (reading c3).  fp32 Q-contract and Philox counter map: DESIGN.md, iht.h.
//
// Layout written: column strips (iht.h).  One thread owns 4 consecutive columns
// (one Philox call per (row, column-quad) serves all four, word n & 3) and a
// 32-byte sector of rows (256/b rows) per plane; it writes the sector's eight
// 32-bit words back to back.  One fp32 read of src feeds up to 8 copies.
#include "iht_internal.cuh"

namespace iht {

// ------------------------------------------------------------------ absmax
__global__ void absmax_kernel(const float* __restrict__ src, int64_t count,
                              unsigned int* __restrict__ out) {
  src += (int64_t)blockIdx.y * count;     // batched: one vector per grid row
  out += blockIdx.y;
  unsigned int m = 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec_ok = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  if (vec_ok) {
    const int64_t n4 = count >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (int64_t i = tid; i < n4; i += stride) {
      const float4 v = __ldg(s4 + i);
      m = max(m, __float_as_uint(v.x) & 0x7FFFFFFFu);
      m = max(m, __float_as_uint(v.y) & 0x7FFFFFFFu);
      m = max(m, __float_as_uint(v.z) & 0x7FFFFFFFu);
      m = max(m, __float_as_uint(v.w) & 0x7FFFFFFFu);
    }
    for (int64_t i = (n4 << 2) + tid; i < count; i += stride)
      m = max(m, __float_as_uint(__ldg(src + i)) & 0x7FFFFFFFu);
  } else {
    for (int64_t i = tid; i < count; i += stride)
      m = max(m, __float_as_uint(__ldg(src + i)) & 0x7FFFFFFFu);
  }
  // |v| bit patterns order like the values; NaN patterns sort above +inf.
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ------------------------------------------------------------ quantise Phi
struct QuantArgs {
  const float* src;     // points at local row row_begin
  int64_t ld;           // row stride in (complex) elements
  int64_t rows, cols, row_offset, strip_bytes, rows_pad;
  int64_t row_begin, row_end;   // local rows quantised by this call (src rows row_begin..row_end)
  int64_t col_quad0;            // col_offset / 4: global column quad of local column 0
  int64_t qblocks;              // column-quad blocks per sector row of the grid
  float c;
  int level_mode;
  int ncopies;
  uint32_t copy_id[8];
  uint32_t key0[8], key1[8];
  uint8_t* codes[8];
};

// B = bits, P = planes.  Thread: column quad g (4 columns), row sector blockIdx.y.
// Each finished 32-bit word (32/B rows of one column) is stored at once; the 8
// words of a sector are written back to back by the same thread (L2 merges them).
template <int B, int P>
__global__ void __launch_bounds__(128) quantize_kernel(QuantArgs a) {
  constexpr int RPS = 256 / B;          // rows per 32-byte sector
  constexpr int CPW = 32 / B;           // codes per 32-bit word
  const int64_t qb = (int64_t)blockIdx.x % a.qblocks, sec = (int64_t)blockIdx.x / a.qblocks;
  const int64_t g = qb * blockDim.x + threadIdx.x;                   // column quad
  const int64_t n0 = g * 4;
  if (n0 >= a.cols) return;
  const int64_t m0 = a.row_begin + sec * RPS;                        // local row of sector
  const int L = num_levels(B, a.level_mode);
  const float sf = q_scale_factor(a.c, L);
  const int ncol = (int)min64(4, a.cols - n0);
  const int64_t plane_bytes = a.rows_pad * B / 8;

  for (int k = 0; k < a.ncopies; ++k) {
    const uint32_t cid = a.copy_id[k], k0 = a.key0[k], k1 = a.key1[k];
    uint8_t* cbase = a.codes[k];
#pragma unroll 1
    for (int w = 0; w < 8; ++w) {
      uint32_t cur[P][4];
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int j = 0; j < 4; ++j) cur[p][j] = 0u;
#pragma unroll
      for (int cc = 0; cc < CPW; ++cc) {
        const int64_t m = m0 + w * CPW + cc;
        if (m < a.row_end) {                      // pad rows keep code 0
          const uint32_t mg = (uint32_t)(a.row_offset + m);
          const float* row = a.src + ((m - a.row_begin) * a.ld + n0) * P;
          float v[P][4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < P; ++p) v[p][j] = (j < ncol) ? __ldg(row + j * P + p) : 0.0f;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            const u32x4 r =
                philox4x32_10(u32x4{(uint32_t)(a.col_quad0 + g), mg, cid, (uint32_t)(p << 8)}, k0, k1);
            cur[p][0] |= q_contract(v[p][0], a.c, sf, L, r.x) << (cc * B);
            cur[p][1] |= q_contract(v[p][1], a.c, sf, L, r.y) << (cc * B);
            cur[p][2] |= q_contract(v[p][2], a.c, sf, L, r.z) << (cc * B);
            cur[p][3] |= q_contract(v[p][3], a.c, sf, L, r.w) << (cc * B);
          }
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < ncol)
            *reinterpret_cast<uint32_t*>(cbase + tiled_offset(n0 + j, p * plane_bytes + m0 * B / 8 + 4 * w,
                                                              a.strip_bytes)) = cur[p][j];
    }
  }
}

// ------------------------------------------------------------ quantise y
template <int P>
__global__ void quantize_vec_kernel(const float* __restrict__ y, int64_t rows, int64_t row_offset,
                                    int bits, int level_mode, uint32_t k0, uint32_t k1,
                                    const float* __restrict__ c_dev, float* __restrict__ yhat,
                                    uint8_t* __restrict__ codes, int64_t rpad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rpad) return;
  const uint32_t b = blockIdx.y;          // snapshot = column n of Y (word n & 3 of counter n >> 2)
  y += (int64_t)b * rows * P;
  yhat += (int64_t)b * P * rpad;
  if (codes) codes += (int64_t)b * P * rows;
  const int L = num_levels(bits, level_mode);
  const float c = c_dev[b];
  const float sf = q_scale_factor(c, L);
  const float sigma = __fdiv_rn(c, (float)(L - 1));
#pragma unroll
  for (int p = 0; p < P; ++p) {
    float out = 0.0f;
    if (i < rows) {
      const float v = y[i * P + p];
      const u32x4 w = philox4x32_10(u32x4{b >> 2, (uint32_t)(row_offset + i), 0u, (uint32_t)((p << 8) | 1)},
                                    k0, k1);
      const uint32_t word = (b & 3) == 0 ? w.x : (b & 3) == 1 ? w.y : (b & 3) == 2 ? w.z : w.w;
      const uint32_t code = q_contract(v, c, sf, L, word);
      if (codes) codes[p * rows + i] = (uint8_t)code;
      out = __fmul_rn(sigma, (float)(2 * (int)code - (L - 1)));
    }
    yhat[p * rpad + i] = out;
  }
}

}  // namespace iht

using namespace iht;

extern "C" int iht_absmax_batched(const float* src, int64_t count, int32_t nrhs, float* c_dev, void* stream) {
  if (count < 0 || nrhs <= 0 || nrhs > 65535 || c_dev == nullptr || (count > 0 && src == nullptr))
    return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  IHT_CUDA_CHECK(cudaMemsetAsync(c_dev, 0, sizeof(float) * nrhs, st));
  if (count == 0) return IHT_OK;
  const int threads = 256;
  const int64_t want = ceil_div<int64_t>(count, (int64_t)threads * 16);
  const int blocks = (int)min64(max64(want, 1), max64(1, (int64_t)kNumSMs * 8 / nrhs));
  // (the kernel takes the vectorised path only when its vector is 16-byte aligned)
  absmax_kernel<<<dim3(blocks, nrhs), threads, 0, st>>>(src, count, reinterpret_cast<unsigned int*>(c_dev));
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}

extern "C" int iht_absmax(const float* src, int64_t count, float* c_dev, void* stream) {
  return iht_absmax_batched(src, count, 1, c_dev, stream);
}

static bool qmat_valid(const iht_qmat& q) {
  if (q.rows <= 0 || q.cols <= 0 || q.row_offset < 0) return false;
  if (q.planes != 1 && q.planes != 2) return false;
  if (q.bits != 2 && q.bits != 4 && q.bits != 8) return false;
  if (q.level_mode != 0 && q.level_mode != 1) return false;
  if (q.strip_bytes != iht_strip_bytes(q.rows, q.planes, q.bits)) return false;
  if (q.codes == nullptr || (reinterpret_cast<uintptr_t>(q.codes) & 15)) return false;
  if (q.row_offset + q.rows > 0xFFFFFFFFll) return false;
  if (q.col_offset < 0 || (q.col_offset & 15)) return false;
  return true;
}

extern "C" int iht_quantize_rows(const float* src, int64_t ld, const iht_qmat* dst, int ncopies,
                                 int64_t row_begin, int64_t nrows, void* stream) {
  if (src == nullptr || dst == nullptr || ncopies <= 0) return IHT_EINVAL;
  const iht_qmat& d0 = dst[0];
  if (!qmat_valid(d0) || ld < d0.cols) return IHT_EINVAL;
  if (!(d0.scale_c >= 0.0f) || !isfinite(d0.scale_c)) return IHT_EDOMAIN;
  if (row_begin < 0 || nrows <= 0 || row_begin + nrows > d0.rows || (row_begin % 256) != 0) return IHT_EINVAL;
  const bool last = row_begin + nrows == d0.rows;
  if (!last && (nrows % 256) != 0) return IHT_EINVAL;
  for (int k = 1; k < ncopies; ++k) {
    const iht_qmat& d = dst[k];
    if (!qmat_valid(d) || d.rows != d0.rows || d.cols != d0.cols || d.planes != d0.planes ||
        d.bits != d0.bits || d.level_mode != d0.level_mode || d.scale_c != d0.scale_c ||
        d.row_offset != d0.row_offset || d.col_offset != d0.col_offset)
      return IHT_EINVAL;
  }
  if ((d0.col_offset + d0.cols) / 4 >= (int64_t)0xFFFFFFFF) return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int RPS = 256 / d0.bits;
  const int64_t rp = rows_pad(d0.rows);
  const int64_t sector_end = last ? rp : row_begin + nrows;
  const int64_t sectors = (sector_end - row_begin) / RPS;
  const int64_t quads = ceil_div<int64_t>(d0.cols, 4);
  const int64_t qblocks = ceil_div<int64_t>(quads, 128);
  if (qblocks * sectors >= 0x7FFFFFFFll) return IHT_EINVAL;
  for (int base = 0; base < ncopies; base += 8) {
    QuantArgs a{};
    a.src = src;
    a.ld = ld;
    a.rows = d0.rows;
    a.cols = d0.cols;
    a.row_offset = d0.row_offset;
    a.strip_bytes = d0.strip_bytes;
    a.rows_pad = rp;
    a.row_begin = row_begin;
    a.row_end = row_begin + nrows;
    a.col_quad0 = d0.col_offset / 4;
    a.qblocks = qblocks;
    a.c = d0.scale_c;
    a.level_mode = d0.level_mode;
    a.ncopies = min(8, ncopies - base);
    for (int k = 0; k < a.ncopies; ++k) {
      const iht_qmat& d = dst[base + k];
      a.copy_id[k] = (uint32_t)d.copy_id;
      a.key0[k] = (uint32_t)(d.seed & 0xFFFFFFFFull);
      a.key1[k] = (uint32_t)(d.seed >> 32);
      a.codes[k] = static_cast<uint8_t*>(d.codes);
    }
    const unsigned grid = (unsigned)(qblocks * sectors);
#define IHT_QLAUNCH(BB, PP) quantize_kernel<BB, PP><<<grid, 128, 0, st>>>(a)
    if (d0.planes == 1) {
      if (d0.bits == 2) IHT_QLAUNCH(2, 1); else if (d0.bits == 4) IHT_QLAUNCH(4, 1); else IHT_QLAUNCH(8, 1);
    } else {
      if (d0.bits == 2) IHT_QLAUNCH(2, 2); else if (d0.bits == 4) IHT_QLAUNCH(4, 2); else IHT_QLAUNCH(8, 2);
    }
#undef IHT_QLAUNCH
    IHT_LAUNCH_CHECK();
  }
  return IHT_OK;
}

extern "C" int iht_quantize(const float* src, int64_t ld, const iht_qmat* dst, int ncopies, void* stream) {
  if (dst == nullptr || ncopies <= 0) return IHT_EINVAL;
  return iht_quantize_rows(src, ld, dst, ncopies, 0, dst[0].rows, stream);
}

extern "C" int iht_quantize_vec(const float* y, int64_t rows, int64_t row_offset, int planes, int bits,
                                int level_mode, uint64_t seed, const float* c_dev, float* yhat,
                                uint8_t* codes, void* stream) {
  return iht_quantize_vec_batched(y, rows, row_offset, planes, bits, level_mode, seed, c_dev, 1, yhat, codes,
                                  stream);
}

extern "C" int iht_quantize_vec_batched(const float* y, int64_t rows, int64_t row_offset, int planes, int bits,
                                        int level_mode, uint64_t seed, const float* c_dev, int32_t nrhs,
                                        float* yhat, uint8_t* codes, void* stream) {
  if (y == nullptr || c_dev == nullptr || yhat == nullptr || rows <= 0 || row_offset < 0) return IHT_EINVAL;
  if (nrhs <= 0 || nrhs > 65535) return IHT_EINVAL;
  if ((planes != 1 && planes != 2) || bits < 2 || bits > 8 || (level_mode != 0 && level_mode != 1))
    return IHT_EINVAL;
  if (row_offset + rows > 0xFFFFFFFFll) return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rp = rows_pad(rows);
  const int threads = 256;
  const unsigned blocks = (unsigned)ceil_div<int64_t>(rp, threads);
  const uint32_t k0 = (uint32_t)(seed & 0xFFFFFFFFull), k1 = (uint32_t)(seed >> 32);
  if (planes == 1)
    quantize_vec_kernel<1><<<dim3(blocks, nrhs), threads, 0, st>>>(y, rows, row_offset, bits, level_mode, k0, k1, c_dev,
                                                       yhat, codes, rp);
  else
    quantize_vec_kernel<2><<<dim3(blocks, nrhs), threads, 0, st>>>(y, rows, row_offset, bits, level_mode, k0, k1, c_dev,
                                                       yhat, codes, rp);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
