// Fused small-problem solver: the WHOLE Algorithm 1 loop (fixed step mu) as one
// persistent cooperative kernel, one CTA per SM, for problems whose stacked rows fit one
// CTA's shared memory as r limbs (configs 1-3).  Per iteration n:
//
//   F   r = y-hat - Phi-hat_{2n} x      (CTA c owns a few 32-bit words of the strips,
//                                         i.e. 32/b stacked rows each, over the s support
//                                         columns; max |r| per 4096-row chunk by atomicMax)
//   --- grid barrier 1 ---
//   A   g = Phi-hat_{2n-1}^T r          (CTA c owns a contiguous range of 16-column
//                                         tiles of the adjoint copy: int8 mma.sync on r in
//                                         3-limb block fixed point, exactly the arithmetic of
//                                         iht_adjoint variant 0, see iht_adjoint.cu)
//       a = x + mu g on its columns, 2048-bin histogram of the top 11 key bits
//   --- grid barrier 2 ---
//   S1  every CTA finds the bin d1 of the s-th largest |a| in the global histogram and
//       writes its candidates (key > 0, digit >= d1) in index order
//   --- grid barrier 3 ---
//   S2  every CTA selects the exact top-s of all candidates (H_s: ties to the lowest
//       index, zeros never kept, reading c15) -- redundantly, so the next F needs no barrier
//
// The adjoint codes are the only large stream.  Each CTA's tiles are one contiguous byte
// range of the copy, moved global -> shared by cp.async.bulk into a ring of tile-sized
// slots (full / empty mbarriers).  Because the adjoint copy of iteration n+1 is known in
// advance ((2n) mod K), the ring is refilled with the NEXT iteration's tiles as soon as the
// current adjoint releases them: the HBM stream runs under the barriers, the select and the
// forward instead of after them (config 2: a CTA's whole range, 112 KiB, is resident
// before its adjoint starts).  Everything is deterministic (integer atomics, fixed orders).
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "iht_internal.cuh"
#include "iht_mma.cuh"
#include "iht_select.cuh"

namespace iht {

constexpr int kFuThreads = 256;
constexpr int kFuWarps = kFuThreads / 32;
constexpr int kFuKC = 4096;            // rows per fixed-point chunk (int32-safe MMA accumulation)
constexpr int kFuCandCap = 2048;       // candidates staged in shared memory for the final select
constexpr int kFuMaxWpc = 8;           // forward: 32-bit strip words per CTA (power of two)

struct FusedArgs {
  const uint8_t* const* copies;        // device [K]: code pointers of the pool
  int K;
  int64_t strip_bytes;
  int N, rows, rpad, Rpad;             // Rpad = planes * rpad stacked rows
  int L;
  float sigma, mu;
  int s, n_iter;
  int ntiles, nslot, tile_bytes, nchunks, wpc, words_total, cap_c, s_cap;
  const float* yhat;                   // [Rpad] stacked, pads 0
  float* r;                            // [Rpad] scratch (and the last r)
  float* g;                            // [N] the last g
  int32_t* xs_idx;                     // [nslots][s]
  float* xs_val;
  int32_t* xs_nnz;                     // [nslots]
  int trace;
  unsigned int* bar;                   // grid barrier counter (0 at launch)
  int* hist;                           // [2][2048]   (0 at launch)
  unsigned int* cmax;                  // [2][nchunks] max |r| bit patterns (0 at launch)
  int* flags;                          // [2]          NaN in a (0 at launch)
  int32_t* cand_idx;                   // [G][cap_c]
  float* cand_val;
  int* cand_cnt;                       // [G]
  // dynamic shared memory offsets (bytes)
  int off_bars, off_limbs, off_fc, off_as, off_x, off_u;
};

__device__ __forceinline__ bool mbar_test(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(mbar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int B>
__global__ void __launch_bounds__(kFuThreads, 1) fused_iht_kernel(FusedArgs a) {
  constexpr int P = 8 / B;             // codes per byte
  constexpr int RPC = 128 / B;         // rows per 16-byte lane chunk
  constexpr int KSTEP = 4 * RPC;       // rows per warp k-step (1 KiB of a 16-column tile)
  constexpr int NMMA = 2 * P;          // MMAs per k-step
  constexpr int CPW = 32 / B;          // codes per 32-bit word
  constexpr uint32_t MASK = (1u << B) - 1u;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int scratch[kFuWarps], wgt[kFuWarps], weq[kFuWarps], wtake[kFuWarps], wbase[kFuWarps], sh[8];
  __shared__ float part[kFuWarps][kFuMaxWpc][CPW];
  __shared__ int s_nnz, s_flag, s_nonfinite, s_total, s_base[2];
  __shared__ unsigned int s_cmax;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t ring_u = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t full_u = (uint32_t)__cvta_generic_to_shared(smem + a.off_bars);
  const uint32_t empty_u = full_u + 8 * a.nslot;
  uint8_t* limbs = smem + a.off_limbs;
  int* Fc = reinterpret_cast<int*>(smem + a.off_fc);
  int* Sl = Fc + a.nchunks;                                       // [chunk][3]
  float* as = reinterpret_cast<float*>(smem + a.off_as);         // [cap_c] a of this CTA's columns
  int32_t* xi_s = reinterpret_cast<int32_t*>(smem + a.off_x);    // the current x (support)
  float* xv_s = reinterpret_cast<float*>(xi_s + a.s_cap);
  long long* Vs = reinterpret_cast<long long*>(smem + a.off_u);  // A: exact chunk sums [tile][chunk][16]
  int* hist_s = reinterpret_cast<int*>(smem + a.off_u);          // S1: the global histogram
  int32_t* ci_s = reinterpret_cast<int32_t*>(smem + a.off_u);    // S2: staged candidates
  float* cv_s = reinterpret_cast<float*>(ci_s + kFuCandCap);
  int* sel_hist = reinterpret_cast<int*>(cv_s + kFuCandCap);     // S2: offsets + select histogram

  // ---- work assignment -------------------------------------------------------------------
  const int t0 = (int)((int64_t)cta * a.ntiles / G), t1 = (int)((int64_t)(cta + 1) * a.ntiles / G);
  const int T = t1 - t0;                                          // tiles of this CTA
  const int col_lo = 16 * t0;
  const int ncol = max(0, min(16 * t1, a.N) - col_lo);
  const int KS = a.Rpad / KSTEP;                                  // k-steps per tile
  const long long total_blocks = (long long)a.n_iter * T;
  const int g8 = lane >> 2, t = lane & 3;

  // ---- ring producer (thread 0): block b = (n - 1) T + j is tile j of iteration n's adjoint
  // copy, in slot b % nslot; a slot is refilled once all warps released its previous block
  long long nb = 0;                                               // next block to request
  auto request = [&](bool blocking, long long limit) {
    while (nb < limit) {
      const int slot = (int)(nb % a.nslot);
      const long long use = nb / a.nslot;
      if (use > 0) {
        const uint32_t par = (uint32_t)((use - 1) & 1);
        if (blocking) mbar_wait(empty_u + 8 * slot, par);
        else if (!mbar_test(empty_u + 8 * slot, par)) return;
      }
      const int n = (int)(nb / T) + 1, j = (int)(nb % T);
      const uint8_t* src = a.copies[(2 * n - 2) % a.K] + (int64_t)(t0 + j) * a.tile_bytes;
      mbar_expect_tx(full_u + 8 * slot, (uint32_t)a.tile_bytes);
      bulk_g2s(ring_u + (uint32_t)slot * a.tile_bytes, src, (uint32_t)a.tile_bytes, full_u + 8 * slot);
      ++nb;
    }
  };
  if (tid == 0) {
    for (int j = 0; j < a.nslot; ++j) {
      mbar_init(full_u + 8 * j, 1);
      mbar_init(empty_u + 8 * j, kFuWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_nnz = 0;                                                    // x^[1] = 0 (reading c8)
  }
  __syncthreads();
  if (tid == 0 && T > 0) request(true, total_blocks < a.nslot ? total_blocks : a.nslot);

  unsigned int bar_target = 0;
  auto grid_sync = [&]() {
    __syncthreads();
    if (tid == 0) {
      bar_target += (unsigned int)G;
      __threadfence();
      atomicAdd(a.bar, 1u);
      while (ld_acquire_u32(a.bar) < bar_target) {
      }
    }
    __syncthreads();
  };

  const uint32_t limb_n = (uint32_t)__cvta_generic_to_shared(limbs + (g8 < 3 ? g8 : 0) * a.Rpad);
  const bool bload = g8 < 3;
  uint32_t bw[4 * P];
#pragma unroll
  for (int q = 0; q < 4 * P; ++q) bw[q] = 0u;
  const unsigned int lt = (1u << lane) - 1u;
  long long consumed = 0;                                         // blocks consumed (all warps)
  int n_done = 0;

  for (int n = 1; n <= a.n_iter; ++n) {
    const int par = n & 1;
    // ================================================================ F: forward
    {
      const int w0 = cta * a.wpc;
      if (tid == 0) s_cmax = 0u;
      __syncthreads();
      if (w0 < a.words_total) {
        const int wpc = a.wpc, ncl = kFuThreads / wpc;
        const int wi = tid % wpc, cl = tid / wpc;
        const int64_t word = (int64_t)w0 + wi;
        const bool live = word < a.words_total;
        const uint8_t* cf = a.copies[(2 * n - 1) % a.K];            // Phi-hat_{2n}, forward
        const int64_t kofs = (word >> 4) * 1024 + (word & 15) * 4;  // tiled byte 4 word, sans column
        const int nnz = s_nnz;
        float acc[CPW];
#pragma unroll
        for (int i = 0; i < CPW; ++i) acc[i] = 0.0f;
        float xs = 0.0f;
        constexpr int U4 = 4;
        for (int j0 = cl; j0 < nnz; j0 += ncl * U4) {
          uint32_t w[U4];
          float xv[U4];
#pragma unroll
          for (int u = 0; u < U4; ++u) {
            const int j = j0 + u * ncl;
            const int col = j < nnz ? xi_s[j] : 0;
            xv[u] = j < nnz ? xv_s[j] : 0.0f;
            w[u] = (j < nnz && live)
                       ? __ldg(reinterpret_cast<const uint32_t*>(cf + (int64_t)(col >> 4) * 16 * a.strip_bytes +
                                                                 (col & 15) * 64 + kofs))
                       : 0u;
          }
#pragma unroll
          for (int u = 0; u < U4; ++u) {
            xs = __fadd_rn(xs, xv[u]);
#pragma unroll
            for (int i = 0; i < CPW; ++i) {
              const float cfv = __int_as_float(0x4B000000u | ((w[u] >> (i * B)) & MASK)) - 8388608.0f;
              acc[i] = __fmaf_rn(xv[u], cfv, acc[i]);              // exact code; xv = 0 adds +0
            }
          }
        }
        // affine map q = 2 code - (L-1) once per row, then the fixed-order reductions:
        // column lanes of the warp (xor shuffles), then the 8 warps in order
        const float xl = __fmul_rn((float)(a.L - 1), xs);
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
          acc[i] = __fsub_rn(__fmul_rn(2.0f, acc[i]), xl);
          for (int o = wpc; o < 32; o <<= 1) acc[i] = __fadd_rn(acc[i], __shfl_xor_sync(0xffffffffu, acc[i], o));
        }
        if (lane < wpc) {
#pragma unroll
          for (int i = 0; i < CPW; ++i) part[warp][lane][i] = acc[i];
        }
        __syncthreads();
        unsigned int mymax = 0u;
        if (tid < wpc * CPW) {
          const int ww = tid / CPW, i = tid % CPW;
          const int64_t m = ((int64_t)w0 + ww) * CPW + i;            // stacked row
          if (m < (int64_t)a.words_total * CPW) {
            float sum = part[0][ww][i];
#pragma unroll
            for (int w2 = 1; w2 < kFuWarps; ++w2) sum = __fadd_rn(sum, part[w2][ww][i]);
            const float rv = (int)(m % a.rpad) < a.rows ? __fsub_rn(__ldg(a.yhat + m), __fmul_rn(a.sigma, sum)) : 0.0f;
            a.r[m] = rv;
            mymax = __float_as_uint(rv) & 0x7FFFFFFFu;               // NaN / inf caught by bit pattern
          }
        }
        mymax = __reduce_max_sync(0xffffffffu, mymax);
        if (lane == 0 && mymax) atomicMax(&s_cmax, mymax);
        __syncthreads();
        if (tid == 0 && s_cmax) atomicMax(&a.cmax[par * a.nchunks + (w0 * CPW) / kFuKC], s_cmax);
      }
    }
    grid_sync();                                                  // ---- barrier 1: r complete
    // ================================================================ limbs of r
    if (T > 0) {
      if (tid == 0) s_nonfinite = 0;
      __syncthreads();
      for (int c = tid; c < a.nchunks; c += kFuThreads) {
        unsigned int mb = __ldcg(&a.cmax[par * a.nchunks + c]);
        if (mb >= 0x7F800000u) {
          s_nonfinite = 1;
          mb = 0;
        }
        const float m = __uint_as_float(mb);
        int e = 0;
        if (m > 0.0f) frexpf(m, &e);
        Fc[c] = (m > 0.0f) ? min(22 - e, 126) : 0;                // |r| 2^F < 2^22
        Sl[3 * c] = Sl[3 * c + 1] = Sl[3 * c + 2] = 0;
      }
      for (int q = tid; q < T * a.nchunks * 16; q += kFuThreads) Vs[q] = 0;
      __syncthreads();
      // r -> three balanced signed 8-bit limbs, permuted per lane chunk (iht_adjoint.cu layout)
      constexpr int kIt = 4;
      const int items = a.Rpad / RPC * (4 * P);
      for (int it0 = tid; it0 < items; it0 += kIt * kFuThreads) {
        float rvs[kIt][4];
#pragma unroll
        for (int q = 0; q < kIt; ++q) {
          const int it = it0 + q * kFuThreads;
          const int ch = it / (4 * P), rho = it % (4 * P);
          const int base = ch * RPC + (rho / P) * (32 / B) + (rho % P);
#pragma unroll
          for (int i = 0; i < 4; ++i) rvs[q][i] = it < items ? __ldcg(a.r + base + P * i) : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < kIt; ++q) {
          const int it = it0 + q * kFuThreads;
          if (it >= items) break;
          const int ch = it / (4 * P), rho = it % (4 * P);
          const int c = (ch * RPC) / kFuKC;
          const float scale = ldexpf(1.0f, Fc[c]);
          uint32_t l0w = 0, l1w = 0, l2w = 0;
          int s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ri = __float2int_rn(rvs[q][i] * scale);
            const int l0 = ((ri + 128) & 255) - 128;
            const int tt = (ri - l0) >> 8;
            const int l1 = ((tt + 128) & 255) - 128;
            const int l2 = (tt - l1) >> 8;
            s0 += l0; s1 += l1; s2 += l2;
            l0w |= (uint32_t)(l0 & 255) << (8 * i);
            l1w |= (uint32_t)(l1 & 255) << (8 * i);
            l2w |= (uint32_t)(l2 & 255) << (8 * i);
          }
          const int off = ch * (16 * P) + (4 * (rho % P) + rho / P) * 4;
          *reinterpret_cast<uint32_t*>(limbs + off) = l0w;
          *reinterpret_cast<uint32_t*>(limbs + a.Rpad + off) = l1w;
          *reinterpret_cast<uint32_t*>(limbs + 2 * a.Rpad + off) = l2w;
          s0 = __reduce_add_sync(0xffffffffu, s0);
          s1 = __reduce_add_sync(0xffffffffu, s1);
          s2 = __reduce_add_sync(0xffffffffu, s2);
          if (lane == 0) {
            atomicAdd(&Sl[3 * c], s0);
            atomicAdd(&Sl[3 * c + 1], s1);
            atomicAdd(&Sl[3 * c + 2], s2);
          }
        }
      }
      __syncthreads();
      // ============================================================== A: adjoint
      int cur_seg = -1;
      int acc[P][4];
#pragma unroll
      for (int j = 0; j < P; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
      auto flush = [&]() {
        if (cur_seg < 0) return;
        int v00 = 0, v01 = 0, v10 = 0, v11 = 0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          v00 += acc[j][0] >> (B * j);
          v01 += acc[j][1] >> (B * j);
          v10 += acc[j][2] >> (B * j);
          v11 += acc[j][3] >> (B * j);
          acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
        }
        const int l2r0 = __shfl_down_sync(0xffffffffu, v00, 1);
        const int l2r1 = __shfl_down_sync(0xffffffffu, v10, 1);
        if (t == 0) {                 // exact int64 sums of warps sharing the (tile, chunk)
          const long long V0 = (long long)v00 + 256ll * v01 + 65536ll * l2r0;
          const long long V1 = (long long)v10 + 256ll * v11 + 65536ll * l2r1;
          atomicAdd(reinterpret_cast<unsigned long long*>(&Vs[cur_seg * 16 + g8]), (unsigned long long)V0);
          atomicAdd(reinterpret_cast<unsigned long long*>(&Vs[cur_seg * 16 + g8 + 8]), (unsigned long long)V1);
        }
      };
      for (int j = 0; j < T; ++j) {
        const long long b = (long long)(n - 1) * T + j;
        const int slot = (int)(b % a.nslot);
        if (tid == 0) request(true, b + 1);                       // block b is in flight
        mbar_wait(full_u + 8 * slot, (uint32_t)((b / a.nslot) & 1));
        const int r0 = (j * KS) % kFuWarps;
        for (int ks = (warp - r0 + kFuWarps) % kFuWarps; ks < KS; ks += kFuWarps) {
          const int seg = j * a.nchunks + (ks * KSTEP) / kFuKC;
          if (seg != cur_seg) {
            flush();
            cur_seg = seg;
          }
          const uint32_t src = ring_u + (uint32_t)slot * a.tile_bytes + ks * 1024 + g8 * 64 + t * 16;
          const uint4 s0 = lds128(src), s1 = lds128(src + 512);
          if (bload) {
            const uint32_t bp = limb_n + (uint32_t)(ks * 4 + t) * (16 * P);
#pragma unroll
            for (int q = 0; q < P; ++q) {
              const uint4 v = lds128(bp + 16 * q);
              bw[4 * q + 0] = v.x; bw[4 * q + 1] = v.y; bw[4 * q + 2] = v.z; bw[4 * q + 3] = v.w;
            }
          }
          uint32_t af[NMMA][4];
#pragma unroll
          for (int jj = 0; jj < P; ++jj)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              af[2 * jj + m][0] = frag_reg<B>(s0, 2 * m, jj);
              af[2 * jj + m][1] = frag_reg<B>(s1, 2 * m, jj);
              af[2 * jj + m][2] = frag_reg<B>(s0, 2 * m + 1, jj);
              af[2 * jj + m][3] = frag_reg<B>(s1, 2 * m + 1, jj);
            }
#pragma unroll
          for (int u = 0; u < NMMA; ++u) mma_u8s8(acc[u >> 1], af[u], bw[2 * u], bw[2 * u + 1]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_u + 8 * slot);          // this warp is done with block b
        if (tid == 0) request(false, total_blocks);               // refill whatever is free
      }
      flush();
      consumed = (long long)n * T;
      __syncthreads();                                            // every block of iteration n consumed
      if (tid == 0) request(true, consumed + a.nslot < total_blocks ? consumed + a.nslot : total_blocks);
      // g = sigma sum_c 2^{-F_c} (2 V_c - (L-1) S_c) (iht_adjoint.cu's combination), a = mu g
      for (int q = tid; q < ncol; q += kFuThreads) {
        const int jl = q >> 4, cc = q & 15;
        float accf = 0.0f;
        for (int c = 0; c < a.nchunks; ++c) {
          const long long S = (long long)Sl[3 * c] + 256ll * Sl[3 * c + 1] + 65536ll * Sl[3 * c + 2];
          const long long V = Vs[(jl * a.nchunks + c) * 16 + cc];
          accf += (float)((double)(2 * V - (long long)(a.L - 1) * S) * ldexp(1.0, -Fc[c]));
        }
        const float gv = s_nonfinite ? __int_as_float(0x7FC00000) : a.sigma * accf;
        a.g[col_lo + q] = gv;
        as[q] = __fmul_rn(a.mu, gv);
      }
      __syncthreads();
      // x's entries on this CTA's columns: a_n = x_n + mu g_n
      for (int j = tid; j < s_nnz; j += kFuThreads) {
        const int c = xi_s[j] - col_lo;
        if (c >= 0 && c < ncol) as[c] = __fadd_rn(xv_s[j], as[c]);
      }
      __syncthreads();
      int nan = 0;
      for (int q = tid; q < ncol; q += kFuThreads) {
        const unsigned int key = __float_as_uint(as[q]) & 0x7FFFFFFFu;
        nan |= key > 0x7F800000u;
        atomicAdd(&a.hist[par * 2048 + (key >> 20)], 1);
      }
      nan = __syncthreads_or(nan);
      if (tid == 0 && nan) atomicOr(&a.flags[par], 1);
    }
    grid_sync();                                                  // ---- barrier 2: histogram complete
    // ================================================================ S1: candidates
    if (cta == 0) {                                               // parity par^1 is idle now
      for (int q = tid; q < 2048; q += kFuThreads) a.hist[(par ^ 1) * 2048 + q] = 0;
      for (int q = tid; q < a.nchunks; q += kFuThreads) a.cmax[(par ^ 1) * a.nchunks + q] = 0u;
      if (tid == 0) a.flags[par ^ 1] = 0;
    }
    if (tid == 0) s_flag = __ldcg(&a.flags[par]);
    for (int q = tid; q < 2048; q += kFuThreads) hist_s[q] = __ldcg(&a.hist[par * 2048 + q]);
    __syncthreads();
    const bool all = a.s >= a.N;
    unsigned int d1 = 0;
    int above = 0;
    if (!all && !s_flag && a.s > 0) {
      find_bin<kFuThreads>(hist_s, 2048, a.s, &sh[0], &sh[1], scratch);
      d1 = (unsigned int)sh[0];
      above = sh[1];
    }
    {
      int base = 0;
      for (int q0 = 0; q0 < ncol; q0 += kFuThreads) {
        const int q = q0 + tid;
        const float v = q < ncol ? as[q] : 0.0f;
        const unsigned int key = __float_as_uint(v) & 0x7FFFFFFFu;
        const bool f = q < ncol && key > 0u && (all || (key >> 20) >= d1);
        const unsigned int bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wgt[warp] = __popc(bal);
        __syncthreads();
        int off = base, tot = 0;
        for (int w = 0; w < kFuWarps; ++w) {
          if (w < warp) off += wgt[w];
          tot += wgt[w];
        }
        if (f) {
          const int pos = off + __popc(bal & lt);
          a.cand_idx[(int64_t)cta * a.cap_c + pos] = col_lo + q;
          a.cand_val[(int64_t)cta * a.cap_c + pos] = v;
        }
        base += tot;
        __syncthreads();
      }
      if (tid == 0) a.cand_cnt[cta] = base;
    }
    (void)above;
    grid_sync();                                                  // ---- barrier 3: candidates complete
    // ================================================================ S2: exact top-s
    const int slot_out = a.trace ? n : (n & 1);
    if (s_flag) {                                                 // non-finite a: domain error
      if (cta == 0 && tid == 0)
        for (int k = slot_out; k <= (a.trace ? a.n_iter : slot_out); ++k) a.xs_nnz[k] = -1;
      n_done = n;
      break;
    }
    // candidate counts -> offsets (CTA order = increasing column index)
    int* cnt_s = sel_hist;                                        // [G + 1] candidate offsets
    int* hsel = sel_hist + ((G + 4) & ~3);                        // [2048] select_ordered's histogram
    for (int c = tid; c < G; c += kFuThreads) cnt_s[c] = __ldcg(&a.cand_cnt[c]);
    __syncthreads();
    if (tid == 0) {
      int acc2 = 0;
      for (int c = 0; c < G; ++c) {
        const int v = cnt_s[c];
        cnt_s[c] = acc2;
        acc2 += v;
      }
      cnt_s[G] = acc2;
      s_total = acc2;
    }
    __syncthreads();
    const int C = s_total;
    if (a.s == 0) {                                               // H_0 keeps nothing
      if (tid == 0) s_nnz = 0;
    } else if (C <= kFuCandCap) {
      for (int c = warp; c < G; c += kFuWarps) {
        const int o = cnt_s[c], k = cnt_s[c + 1] - o;
        for (int i = lane; i < k; i += 32) {
          ci_s[o + i] = __ldcg(&a.cand_idx[(int64_t)c * a.cap_c + i]);
          cv_s[o + i] = __ldcg(&a.cand_val[(int64_t)c * a.cap_c + i]);
        }
      }
      __syncthreads();
      select_ordered<kFuThreads>(C, a.s, [&](int i) { return cv_s[i]; }, [&](int i) { return ci_s[i]; }, xi_s, xv_s,
                                 &s_nnz, 0, hsel, scratch, wgt, weq, wtake, wbase, sh);
    } else {
      // many candidates (massive ties): select over the global lists, element i found by
      // binary search over the CTA offsets
      auto loc = [&](int i) {
        int lo = 0, hi = G;                                       // cnt_s[lo] <= i < cnt_s[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (cnt_s[mid] <= i) lo = mid; else hi = mid;
        }
        return (int64_t)lo * a.cap_c + (i - cnt_s[lo]);
      };
      select_ordered<kFuThreads>(C, a.s, [&](int i) { return __ldcg(&a.cand_val[loc(i)]); },
                                 [&](int i) { return __ldcg(&a.cand_idx[loc(i)]); }, xi_s, xv_s, &s_nnz, 0, hsel,
                                 scratch, wgt, weq, wtake, wbase, sh);
    }
    __syncthreads();
    if (cta == 0) {                                               // the iterate x^[n+1]
      const int k = s_nnz;
      for (int j = tid; j < k; j += kFuThreads) {
        a.xs_idx[(int64_t)slot_out * a.s + j] = xi_s[j];
        a.xs_val[(int64_t)slot_out * a.s + j] = xv_s[j];
      }
      if (tid == 0) a.xs_nnz[slot_out] = k;
    }
    n_done = n;
  }
  (void)n_done;
  // drain: bulk copies still in flight (prefetch past an aborted run) must land before exit
  if (tid == 0) {
    for (long long b = consumed; b < nb; ++b) mbar_wait(full_u + 8 * (int)(b % a.nslot), (uint32_t)((b / a.nslot) & 1));
  }
  __syncthreads();
}

}  // namespace iht

// ======================================================================================
// Host side: eligibility, workspace, launch
// ======================================================================================
using namespace iht;

struct iht_fused_state {
  FusedArgs args{};
  int G = 0, bits = 0;
  size_t smem = 0;
  void* block = nullptr;               // copies table | bar | hist | cmax | flags | candidates
  size_t zero_bytes = 0;               // bar .. flags, zeroed before every launch
};

static size_t al16(size_t b) { return (b + 15) / 16 * 16; }

int iht_fused_create(const iht_qmat* pool, int K, int s, int n_iter, float mu, int trace, const float* yhat,
                     float* r, float* g, int32_t* xs_idx, float* xs_val, int32_t* xs_nnz, iht_fused_state** out) {
  *out = nullptr;
  const iht_qmat& q = pool[0];
  if (q.bits != 2 && q.bits != 4 && q.bits != 8) return IHT_EUNSUPPORTED;
  if (q.cols > 0x7FFFFFFF || q.rows > 0x7FFFFFFF || s < 0) return IHT_EUNSUPPORTED;
  int dev = 0, G = 0, coop = 0, optin = 0;
  IHT_CUDA_CHECK(cudaGetDevice(&dev));
  IHT_CUDA_CHECK(cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, dev));
  IHT_CUDA_CHECK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  IHT_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (!coop) return IHT_EUNSUPPORTED;
  const int B = q.bits;
  const int rpad = (int)iht::rows_pad(q.rows);
  const int Rpad = q.planes * rpad;
  const int ntiles = (int)((q.cols + 15) / 16);
  const int tmax = (ntiles + G - 1) / G;
  const int tile_bytes = (int)(16 * q.strip_bytes);
  const int nchunks = (Rpad + kFuKC - 1) / kFuKC;
  const int words_total = (int)(q.strip_bytes / 4);
  int wpc = 1;
  while (wpc * G < words_total) wpc *= 2;
  if (wpc > kFuMaxWpc) return IHT_EUNSUPPORTED;
  const int cap_c = 16 * tmax;
  const int s_cap = s > 0 ? s : 1;
  // shared memory: ring | bars | limbs | Fc, Sl | a | x | union(V sums, histogram, candidates)
  size_t o = 0;
  const size_t u_bytes = std::max({(size_t)tmax * nchunks * 16 * 8, (size_t)2048 * 4,
                                   (size_t)kFuCandCap * 8 + (size_t)(((G + 4) & ~3) + 2048) * 4});
  auto layout = [&](int nslot, FusedArgs* A) {
    o = (size_t)nslot * tile_bytes;
    const size_t bars = o;
    o = al16(o + 16 * (size_t)nslot);
    const size_t limbs = o;
    o = al16(o + 3 * (size_t)Rpad);
    const size_t fc = o;
    o = al16(o + 16 * (size_t)nchunks);
    const size_t as = o;
    o = al16(o + 4 * (size_t)cap_c);
    const size_t xo = o;
    o = al16(o + 8 * (size_t)s_cap);
    const size_t uo = o;
    o += u_bytes;
    if (A) {
      A->off_bars = (int)bars;
      A->off_limbs = (int)limbs;
      A->off_fc = (int)fc;
      A->off_as = (int)as;
      A->off_x = (int)xo;
      A->off_u = (int)uo;
    }
    return o;
  };
  const size_t limit = (size_t)optin - 8192;          // static shared memory and margin
  const size_t rest = layout(0, nullptr);
  if (rest + tile_bytes > limit) return IHT_EUNSUPPORTED;
  int nslot = (int)((limit - rest) / (tile_bytes + 16));
  nslot = std::max(1, std::min(nslot, tmax));
  iht_fused_state* S = new iht_fused_state();
  FusedArgs& A = S->args;
  S->smem = layout(nslot, &A);
  S->G = G;
  S->bits = B;
  // device workspace
  const size_t sz_tab = al16(sizeof(void*) * (size_t)K), sz_bar = 16, sz_hist = 2 * 2048 * 4,
               sz_cmax = al16(2 * 4 * (size_t)nchunks), sz_flags = 16,
               sz_cand = al16((size_t)G * cap_c * 4), sz_cnt = al16((size_t)G * 4);
  const size_t total = sz_tab + sz_bar + sz_hist + sz_cmax + sz_flags + 2 * sz_cand + sz_cnt;
  if (cudaMalloc(&S->block, total) != cudaSuccess) {
    delete S;
    return IHT_ENOMEM;
  }
  char* p = static_cast<char*>(S->block);
  std::vector<const uint8_t*> tab(K);
  for (int k = 0; k < K; ++k) tab[k] = static_cast<const uint8_t*>(pool[k].codes);
  if (cudaMemcpy(p, tab.data(), sizeof(void*) * K, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(S->block);
    delete S;
    return IHT_ECUDA;
  }
  A.copies = reinterpret_cast<const uint8_t* const*>(p);
  p += sz_tab;
  char* z0 = p;
  A.bar = reinterpret_cast<unsigned int*>(p); p += sz_bar;
  A.hist = reinterpret_cast<int*>(p); p += sz_hist;
  A.cmax = reinterpret_cast<unsigned int*>(p); p += sz_cmax;
  A.flags = reinterpret_cast<int*>(p); p += sz_flags;
  S->zero_bytes = (size_t)(p - z0);
  A.cand_idx = reinterpret_cast<int32_t*>(p); p += sz_cand;
  A.cand_val = reinterpret_cast<float*>(p); p += sz_cand;
  A.cand_cnt = reinterpret_cast<int*>(p); p += sz_cnt;
  A.K = K;
  A.strip_bytes = q.strip_bytes;
  A.N = (int)q.cols;
  A.rows = (int)q.rows;
  A.rpad = rpad;
  A.Rpad = Rpad;
  A.L = num_levels(B, q.level_mode);
  A.sigma = q.scale_c / (float)(A.L - 1);
  A.mu = mu;
  A.s = s;
  A.n_iter = n_iter;
  A.ntiles = ntiles;
  A.nslot = nslot;
  A.tile_bytes = tile_bytes;
  A.nchunks = nchunks;
  A.wpc = wpc;
  A.words_total = words_total;
  A.cap_c = cap_c;
  A.s_cap = s_cap;
  A.yhat = yhat;
  A.r = r;
  A.g = g;
  A.xs_idx = xs_idx;
  A.xs_val = xs_val;
  A.xs_nnz = xs_nnz;
  A.trace = trace;
  auto kern = B == 2 ? fused_iht_kernel<2> : B == 4 ? fused_iht_kernel<4> : fused_iht_kernel<8>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->smem);
  int nblk = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nblk, kern, kFuThreads, S->smem);
  if (e != cudaSuccess || nblk < 1) {
    (void)cudaGetLastError();
    cudaFree(S->block);
    delete S;
    return IHT_EUNSUPPORTED;
  }
  *out = S;
  return IHT_OK;
}

int iht_fused_enqueue(iht_fused_state* S, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  IHT_CUDA_CHECK(cudaMemsetAsync(S->args.bar, 0, S->zero_bytes, st));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(S->G);
  lc.blockDim = dim3(kFuThreads);
  lc.dynamicSmemBytes = S->smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;           // all CTAs co-resident: grid barriers
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  auto kern = S->bits == 2 ? fused_iht_kernel<2> : S->bits == 4 ? fused_iht_kernel<4> : fused_iht_kernel<8>;
  IHT_CUDA_CHECK(cudaLaunchKernelEx(&lc, kern, S->args));
  return IHT_OK;
}

void iht_fused_destroy(iht_fused_state* S) {
  if (S == nullptr) return;
  if (S->block) cudaFree(S->block);
  delete S;
}
