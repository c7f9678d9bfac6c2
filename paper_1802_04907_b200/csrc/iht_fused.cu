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
  int ntiles, tile_bytes, nchunks, wpc, words_total, cap_c, s_cap;
  int nsub, block_bytes, mslot;        // ring: a tile = nsub blocks; each warp owns mslot block slots
  int limb_stride;                     // bytes between the 3 limb planes (Rpad + 64: bank spread)
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
  int off_bars, off_limbs, off_fc, off_as, off_x, off_u, off_tab, off_h;
  long long* tl;                       // profiling (IHT_FUSED_TL): [64][16] globaltimer stamps of CTA tl_cta
  int tl_cta;
  int probe;                           // profiling (IHT_FUSED_PROBE): 1 no MMA work, 2 no refills inside A, 4 no flush
  int nobound;                         // IHT_FUSED_NOBOUND=1: never take the bounded-candidate path (same results)
  float bound_frac;                    // bound = bound_frac x the previous threshold (IHT_FUSED_BOUND, default 0.7)
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
  __shared__ float s_min[kFuWarps];
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t ring_u = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t full_u = (uint32_t)__cvta_generic_to_shared(smem + a.off_bars);
  uint8_t* limbs = smem + a.off_limbs;
  int* Fc = reinterpret_cast<int*>(smem + a.off_fc);
  int* Sl = Fc + a.nchunks;                                       // [chunk][3]
  float* as = reinterpret_cast<float*>(smem + a.off_as);         // [cap_c] a of this CTA's columns
  int32_t* xi_s = reinterpret_cast<int32_t*>(smem + a.off_x);    // the current x (support)
  float* xv_s = reinterpret_cast<float*>(xi_s + a.s_cap);
  int* Vs = reinterpret_cast<int*>(smem + a.off_u);              // A: exact limb sums [tile][chunk][16][3]
  int* hist_s = reinterpret_cast<int*>(smem + a.off_h);          // A: the CTA's histogram; S1: the global one
  int32_t* ci_s = reinterpret_cast<int32_t*>(smem + a.off_u);    // S2: staged candidates
  float* cv_s = reinterpret_cast<float*>(ci_s + kFuCandCap);
  int* sel_hist = reinterpret_cast<int*>(cv_s + kFuCandCap);     // S2: offsets | histogram / keys | positions | flags
  const uint8_t** ctab = reinterpret_cast<const uint8_t**>(smem + a.off_tab);   // the pool's code pointers
  for (int k = tid; k < a.K; k += kFuThreads) ctab[k] = a.copies[k];

  // ---- work assignment -------------------------------------------------------------------
  const int t0 = (int)((int64_t)cta * a.ntiles / G), t1 = (int)((int64_t)(cta + 1) * a.ntiles / G);
  const int T = t1 - t0;                                          // tiles of this CTA
  const int col_lo = 16 * t0;
  const int ncol = max(0, min(16 * t1, a.N) - col_lo);
  const int KS = a.Rpad / KSTEP;                                  // k-steps per tile
  const int total_blocks = a.n_iter * T;                          // <= 2^31 (eligibility)
  const int g8 = lane >> 2, t = lane & 3;

  // ---- per-warp rings: warp w owns the tiles j = w, w + 8, ... of this CTA and streams them
  // itself through its own mslot slots (lane 0 issues the bulk copies, full mbarriers only):
  // its q-th block is sub-block h of its k-th tile of iteration n, q = ((n-1) Tw + k) nsub + h.
  // A slot is refilled by the warp as soon as it has consumed it, so the NEXT iteration's
  // tiles stream in while the CTA is in the barriers, the select and the forward.
  const int Tw = T > warp ? (T - warp + kFuWarps - 1) / kFuWarps : 0;   // tiles of this warp
  const int Bw = Tw * a.nsub;                                     // its blocks per iteration
  const int total_w = a.n_iter * Bw;
  const uint32_t wfull = full_u + 8 * (warp * a.mslot);
  const uint32_t wring = ring_u + (uint32_t)(warp * a.mslot) * a.block_bytes;
  int nb = 0;                                                     // lane 0: next block to request
  int rq_slot = 0, rq_k = 0, rq_h = 0, rq_n = 1;
  const uint8_t* rq_src = nullptr;                                // the copy of iteration rq_n
  auto request = [&](int limit) {                                 // lane 0 only
    while (nb < limit && nb < total_w) {
      if (rq_k == 0 && rq_h == 0) rq_src = ctab[(2 * rq_n - 2) % a.K];
      const uint8_t* src = rq_src + (int64_t)(t0 + warp + kFuWarps * rq_k) * a.tile_bytes +
                           (int64_t)rq_h * a.block_bytes;
      IHT_DCHECK(rq_slot < a.mslot && t0 + warp + kFuWarps * rq_k < t1 && rq_h < a.nsub &&
                     (int64_t)(t0 + warp + kFuWarps * rq_k + 1) * a.tile_bytes <= (int64_t)a.ntiles * a.tile_bytes,
                 "fused: ring request inside this CTA's tiles of the copy");
      mbar_expect_tx(wfull + 8 * rq_slot, (uint32_t)a.block_bytes);
      bulk_g2s(wring + (uint32_t)rq_slot * a.block_bytes, src, (uint32_t)a.block_bytes, wfull + 8 * rq_slot);
      ++nb;
      if (++rq_h == a.nsub) {
        rq_h = 0;
        if (++rq_k == Tw) {
          rq_k = 0;
          ++rq_n;
        }
      }
      if (++rq_slot == a.mslot) rq_slot = 0;
    }
  };
  if (tid == 0) {
    for (int j = 0; j < kFuWarps * a.mslot; ++j) mbar_init(full_u + 8 * j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_nnz = 0;                                                    // x^[1] = 0 (reading c8)
  }
  __syncthreads();
  if (lane == 0 && !(a.probe & 8)) request(a.mslot);

  unsigned int bar_target = 0;
  auto grid_sync = [&]() {
    __syncthreads();
    if (tid == 0) {
      bar_target += (unsigned int)G;
      // release: the CTA's writes (ordered before by bar.sync) become visible with the arrival
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
#ifdef IHT_CHECKS
      long long spins = 0;
#endif
      while (ld_acquire_u32(a.bar) < bar_target) {
#ifdef IHT_CHECKS
        if (++spins > IHT_SPIN_LIMIT) {
          printf("IHT_DCHECK: fused grid barrier did not complete (block %d, target %u)\n", cta, bar_target);
          __trap();
        }
#endif
      }
    }
    __syncthreads();
  };

  const uint32_t limb_n = (uint32_t)__cvta_generic_to_shared(limbs + (g8 < 3 ? g8 : 0) * a.limb_stride);
  const bool bload = g8 < 3;
  uint32_t bw[4 * P], bw2[4 * P];      // B fragments (two sets: the A phase's ping-pong); zero on lanes g8 >= 3
#pragma unroll
  for (int q = 0; q < 4 * P; ++q) bw[q] = bw2[q] = 0u;
  const unsigned int lt = (1u << lane) - 1u;
  int consumed = 0;                                               // blocks this warp consumed
  int c_slot = 0;                                                 // consumer cursor: slot, use parity
  uint32_t c_par = 0;
  int n_done = 0;

  auto stamp = [&](int n, int k) {      // profiling timeline (IHT_FUSED_TL)
    if (a.tl && tid == 0) {
      long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      if (a.tl_cta >= 0 && cta == a.tl_cta && n <= 64) a.tl[(n - 1) * 16 + k] = tt;
      if (a.tl_cta < 0 && n == 3) a.tl[cta * 16 + k] = tt;     // every CTA, iteration 3
    }
  };
  // ordered compaction of this CTA's columns whose key passes `pred` into its candidate slot
  // (index order), count to cand_cnt[cta]
  auto write_cands = [&](auto pred) {
    int base = 0;
    for (int q0 = 0; q0 < ncol; q0 += kFuThreads) {
      const int q = q0 + tid;
      const float v = q < ncol ? as[q] : 0.0f;
      const unsigned int key = __float_as_uint(v) & 0x7FFFFFFFu;
      const bool f = q < ncol && key > 0u && pred(key);
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
        IHT_DCHECK(pos < a.cap_c, "fused: candidate inside the CTA's slot");
        a.cand_idx[(int64_t)cta * a.cap_c + pos] = col_lo + q;
        a.cand_val[(int64_t)cta * a.cap_c + pos] = v;
      }
      base += tot;
      __syncthreads();
    }
    if (tid == 0) a.cand_cnt[cta] = base;
  };
  // the CTA histogram (hist_s, zeroed in the limb phase) into the global one, one atomic per
  // nonzero bin
  auto add_hist = [&](int par_) {
    for (int q = tid; q < 2048; q += kFuThreads) {
      const int v = hist_s[q];
      if (v) atomicAdd(&a.hist[par_ * 2048 + q], v);
    }
  };
  for (int n = 1; n <= a.n_iter; ++n) {
    const int par = n & 1;
    stamp(n, 0);
    // Bounded candidates: bkey = the key of half the smallest kept |x^[n]| (the previous
    // threshold), or 0.  Before barrier 2 every CTA writes its keys >= bkey as candidates;
    // after it, if bin d1 (the s-th largest key's) lies at or above bkey, the candidates hold
    // every key with digit >= d1 -- a superset of the top s -- and S1 with its barrier is
    // skipped (exact: S2 keeps digits > d1, ranks digit d1, drops the rest).  Otherwise S1
    // rewrites the candidates as before.  Same decision on every CTA (same x, same histogram).
    unsigned int bkey = 0u;
    {
      float mn = __int_as_float(0x7F800000);
      for (int j = tid; j < s_nnz; j += kFuThreads) mn = fminf(mn, fabsf(xv_s[j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (lane == 0) s_min[warp] = mn;
      __syncthreads();
      mn = s_min[0];
#pragma unroll
      for (int w = 1; w < kFuWarps; ++w) mn = fminf(mn, s_min[w]);
      if (!a.nobound && n >= 2 && a.s > 0 && a.s < a.N && s_nnz == a.s && mn > 0.0f && mn < 3.0e38f)
        bkey = __float_as_uint(__fmul_rn(a.bound_frac, mn)) & 0x7FFFFFFFu;
    }
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
        const uint8_t* cf = ctab[(2 * n - 1) % a.K];                // Phi-hat_{2n}, forward
        const int64_t kofs = (word >> 4) * 1024 + (word & 15) * 4;  // tiled byte 4 word, sans column
        const int nnz = s_nnz;
        // y-hat of this CTA's output rows, requested before the code loads
        const float ypre = tid < wpc * CPW && (int64_t)w0 * CPW + tid < (int64_t)a.words_total * CPW
                               ? __ldg(a.yhat + (int64_t)w0 * CPW + tid) : 0.0f;
        float acc[CPW];
#pragma unroll
        for (int i = 0; i < CPW; ++i) acc[i] = 0.0f;
        float xs = 0.0f;
        const uint32_t mant_mask = MASK << (23 - B), exp_b = (uint32_t)(127 + B) << 23;   // 2^B
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
              // the float 2^B + code, exactly (as forward_kernel): one shift + one LOP3
              const int sh = 23 - B - i * B;
              const uint32_t xw = sh >= 0 ? (w[u] << sh) : (w[u] >> -sh);
              const float cfv = __uint_as_float(lop3_and_or(xw, mant_mask, exp_b));
              acc[i] = __fmaf_rn(xv[u], cfv, acc[i]);              // xv = 0 adds +0
            }
          }
        }
        // affine map q = 2 code - (L-1) once per row, then the fixed-order reductions:
        // column lanes of the warp (xor shuffles), then the 8 warps in order
        const float xl = __fmul_rn((float)((2 << B) + a.L - 1), xs);   // sum x q = 2 acc - (2^{B+1} + L-1) sum x
#pragma unroll
        for (int i = 0; i < CPW; ++i) acc[i] = __fsub_rn(__fmul_rn(2.0f, acc[i]), xl);
        for (int o = wpc; o < 32; o <<= 1) {                      // CPW independent shuffles per level
#pragma unroll
          for (int i = 0; i < CPW; ++i) acc[i] = __fadd_rn(acc[i], __shfl_xor_sync(0xffffffffu, acc[i], o));
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
            const float rv = (int)(m % a.rpad) < a.rows ? __fsub_rn(ypre, __fmul_rn(a.sigma, sum)) : 0.0f;
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
    stamp(n, 1);
    grid_sync();                                                  // ---- barrier 1: r complete
    stamp(n, 2);
    // ================================================================ limbs of r
    if (T > 0) {
      // r -> three balanced signed 8-bit limbs, permuted per lane chunk (iht_adjoint.cu layout).
      // A thread converts whole groups of CPW consecutive rows (the rows of one 32-bit code
      // word = P limb items): its loads are P contiguous float4 (coalesced; r is read once per
      // CTA from L2), all requested together with the chunk maxima before anything waits
      const int ngroups = a.Rpad / CPW;
      const int rounds = (ngroups + kFuThreads - 1) / kFuThreads;
      constexpr int kMaxRounds = 16384 / CPW / kFuThreads;       // Rpad <= 16384 rows
      float4 rv[kMaxRounds][P];
#pragma unroll
      for (int rd = 0; rd < kMaxRounds; ++rd) {
        const int gw = tid + rd * kFuThreads;
#pragma unroll
        for (int e = 0; e < P; ++e)
          rv[rd][e] = (rd < rounds && gw < ngroups) ? __ldcg(reinterpret_cast<const float4*>(a.r + gw * CPW) + e)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (tid == 0) s_nonfinite = 0;
      unsigned int mb = tid < a.nchunks ? __ldcg(&a.cmax[par * a.nchunks + tid]) : 0u;
      for (int q = tid; q < T * a.nchunks * 48; q += kFuThreads) Vs[q] = 0;
      for (int q = tid; q < 2048; q += kFuThreads) hist_s[q] = 0;  // the A-phase histogram (off the critical path)
      __syncthreads();
      if (tid < a.nchunks) {
        const int c = tid;
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
      __syncthreads();
#pragma unroll
      for (int rd = 0; rd < kMaxRounds; ++rd) {
        if (rd >= rounds) break;
        const int gw = tid + rd * kFuThreads;
        const bool ok = gw < ngroups;
        const int c = ok ? (gw * CPW) / kFuKC : 0;
        const float scale = ldexpf(1.0f, Fc[c]);
        const int ch = gw >> 2, h = gw & 3;                       // lane chunk, word within it
        const float* rr = reinterpret_cast<const float*>(&rv[rd][0]);   // CPW rows of this group
        int s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
        for (int e = 0; e < P; ++e) {                             // item rho = h P + e: rows e + P i
          uint32_t l0w = 0, l1w = 0, l2w = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ri = __float2int_rn(rr[e + P * i] * scale);
            const int l0 = ((ri + 128) & 255) - 128;
            const int tt = (ri - l0) >> 8;
            const int l1 = ((tt + 128) & 255) - 128;
            const int l2 = (tt - l1) >> 8;
            s0 += l0; s1 += l1; s2 += l2;
            l0w |= (uint32_t)(l0 & 255) << (8 * i);
            l1w |= (uint32_t)(l1 & 255) << (8 * i);
            l2w |= (uint32_t)(l2 & 255) << (8 * i);
          }
          if (ok) {
            // bank-spread limb layout: k-step ks = ch / 4 holds 64 P bytes per plane, the 16-byte
            // chunk of (bit position j = e, lane t = ch % 4) at (4 j + t) 16, word v = h inside it
            const int off = (ch >> 2) * (64 * P) + (4 * e + (ch & 3)) * 16 + h * 4;
            *reinterpret_cast<uint32_t*>(limbs + off) = l0w;
            *reinterpret_cast<uint32_t*>(limbs + a.limb_stride + off) = l1w;
            *reinterpret_cast<uint32_t*>(limbs + 2 * a.limb_stride + off) = l2w;
          }
        }
        // the 32 groups of a warp lie in one chunk (32 CPW = 512 / B rows, aligned)
        s0 = __reduce_add_sync(0xffffffffu, s0);
        s1 = __reduce_add_sync(0xffffffffu, s1);
        s2 = __reduce_add_sync(0xffffffffu, s2);
        if (lane == 0) {
          atomicAdd(&Sl[3 * c], s0);
          atomicAdd(&Sl[3 * c + 1], s1);
          atomicAdd(&Sl[3 * c + 2], s2);
        }
      }
      __syncthreads();
      stamp(n, 3);
      // ============================================================== A: adjoint
      int cur_seg = -1;
      int acc[P][4];                                              // one accumulator per bit position
#pragma unroll
      for (int j = 0; j < P; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
      auto flush = [&]() {
        if (cur_seg < 0 || (a.probe & 4)) return;
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
        if (t == 0) {                 // exact per-limb int32 sums of the warps sharing (tile, chunk)
          int* v = Vs + (cur_seg * 16 + g8) * 3;
          IHT_DCHECK((cur_seg * 16 + g8 + 8) * 3 + 3 <= T * a.nchunks * 48, "fused: limb-sum slot inside V");
          atomicAdd(v, v00);
          atomicAdd(v + 1, v01);
          atomicAdd(v + 2, l2r0);
          atomicAdd(v + 24, v10);
          atomicAdd(v + 25, v11);
          atomicAdd(v + 26, l2r1);
        }
      };
      const int KSB = KS / a.nsub;                                // k-steps per block
      constexpr int KPC = kFuKC / KSTEP;                          // k-steps per fixed-point chunk
      const bool probe_nomma = (a.probe & 1) != 0;
      const uint32_t lane_off = g8 * 64 + t * 16;
      auto kstep_mma = [&](const uint4& w0, const uint4& w1, const uint32_t* b) {
        uint32_t af[NMMA][4];
#pragma unroll
        for (int jj = 0; jj < P; ++jj)
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            af[2 * jj + m][0] = frag_reg<B>(w0, 2 * m, jj);
            af[2 * jj + m][1] = frag_reg<B>(w1, 2 * m, jj);
            af[2 * jj + m][2] = frag_reg<B>(w0, 2 * m + 1, jj);
            af[2 * jj + m][3] = frag_reg<B>(w1, 2 * m + 1, jj);
          }
#pragma unroll
        for (int i = 0; i < NMMA; ++i) {   // consecutive MMAs update different accumulators
          const int u = (i % P) * 2 + i / P;
          mma_u8s8(acc[u >> 1], af[u], b[2 * u], b[2 * u + 1]);
        }
      };
      auto load_b = [&](int ks, uint32_t* dst) {                  // r limbs of k-step ks (lanes g8 < 3)
        const uint32_t bp = limb_n + (uint32_t)ks * (64 * P) + t * 16;
#pragma unroll
        for (int q = 0; q < P; ++q) {                             // 12 lanes hit 3 x 4 distinct bank quads
          const uint4 v = lds128(bp + 64 * q);
          dst[4 * q + 0] = v.x; dst[4 * q + 1] = v.y; dst[4 * q + 2] = v.z; dst[4 * q + 3] = v.w;
        }
      };
      // probe 8: no cross-iteration prefetch (each warp streams its tiles during its own A)
      const int rq_cap = (a.probe & 8) ? n * Bw : total_w;
      if (lane == 0) request(min(consumed + a.mslot, rq_cap));
      for (int k = 0; k < Tw; ++k) {
        const int j = warp + kFuWarps * k;                        // tile (CTA-local)
        for (int h = 0; h < a.nsub; ++h) {
          if (k == 0 && h == 0) stamp(n, 10);
          mbar_wait(wfull + 8 * c_slot, c_par);
          if (k == 0 && h == 0) stamp(n, 11);
          const uint32_t sbase = wring + (uint32_t)c_slot * a.block_bytes;
          // the block's k-steps in runs that stay inside one fixed-point chunk (the flush
          // decision is taken once per run, not per k-step), each run software-pipelined:
          // the shared loads of k-step r+1 are issued before the MMAs of k-step r (the asm
          // statements keep source order, so the order here is the issue order)
          int kk = probe_nomma ? KSB : 0;
          while (kk < KSB) {
            const int ks0 = h * KSB + kk;
            const int seg = j * a.nchunks + ks0 / KPC;
            if (seg != cur_seg) {
              flush();
              cur_seg = seg;
            }
            const int run = min(KSB - kk, KPC - ks0 % KPC);
            // two register sets, set A = (c0, c1, bw), set B = (n0, n1, bw2), alternating
            // without copies (a copy of a just-loaded register would wait for the load)
            uint4 c0 = lds128(sbase + kk * 1024 + lane_off), c1 = lds128(sbase + kk * 1024 + lane_off + 512);
            uint4 n0, n1;
            if (bload) load_b(ks0, bw);
            int r = 0;
            for (; r + 1 < run; r += 2) {
              n0 = lds128(sbase + (kk + r + 1) * 1024 + lane_off);
              n1 = lds128(sbase + (kk + r + 1) * 1024 + lane_off + 512);
              if (bload) load_b(ks0 + r + 1, bw2);
              kstep_mma(c0, c1, bw);
              if (r + 2 < run) {
                c0 = lds128(sbase + (kk + r + 2) * 1024 + lane_off);
                c1 = lds128(sbase + (kk + r + 2) * 1024 + lane_off + 512);
                if (bload) load_b(ks0 + r + 2, bw);
              }
              kstep_mma(n0, n1, bw2);
            }
            if (r < run) kstep_mma(c0, c1, bw);                   // odd run: the last k-step
            kk += run;
          }
          __syncwarp();                                           // every lane has read the slot
          ++consumed;
          if (lane == 0 && !(a.probe & 2)) request(min(consumed + a.mslot, rq_cap));   // refill (maybe next iteration)
          if (++c_slot == a.mslot) {
            c_slot = 0;
            c_par ^= 1u;
          }
        }
      }
      flush();
      stamp(n, 4);
      __syncthreads();                                            // every tile of iteration n consumed
      if (lane == 0 && (a.probe & 2)) request(consumed + a.mslot);
      // g = sigma sum_c 2^{-F_c} (2 V_c - (L-1) S_c) (iht_adjoint.cu's combination), a = mu g
      for (int q = tid; q < ncol; q += kFuThreads) {
        const int jl = q >> 4, cc = q & 15;
        float accf = 0.0f;
        for (int c = 0; c < a.nchunks; ++c) {
          const long long S = (long long)Sl[3 * c] + 256ll * Sl[3 * c + 1] + 65536ll * Sl[3 * c + 2];
          const int* v = Vs + ((jl * a.nchunks + c) * 16 + cc) * 3;
          const long long V = (long long)v[0] + 256ll * v[1] + 65536ll * v[2];
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
        IHT_DCHECK(j < a.s_cap && xi_s[j] >= 0 && xi_s[j] < a.N, "fused: support index");
        if (c >= 0 && c < ncol) as[c] = __fadd_rn(xv_s[j], as[c]);
      }
      __syncthreads();
      // the CTA's histogram in shared memory first (the union region: V sums are consumed),
      // then one global atomic per nonzero bin -- the keys crowd a few dozen 1/8-octave bins,
      // and per-element global atomics on them serialised at L2 (and delayed the barrier).
      // With a bound the histogram is not needed unless the bound misses (S1 builds it then)
      int nan = 0;
      for (int q = tid; q < ncol; q += kFuThreads) {
        const unsigned int key = __float_as_uint(as[q]) & 0x7FFFFFFFu;
        nan |= key > 0x7F800000u;
        if (!bkey) atomicAdd(&hist_s[key >> 20], 1);
      }
      nan = __syncthreads_or(nan);
      if (!bkey) add_hist(par);
      if (tid == 0 && nan) atomicOr(&a.flags[par], 1);
    }
    if (bkey) write_cands([&](unsigned int key) { return key >= bkey; });
    stamp(n, 5);
    grid_sync();                                                  // ---- barrier 2: histogram complete
    stamp(n, 6);
    // ================================================================ S1: candidates
    if (cta == 0) {                                               // parity par^1 is idle now
      for (int q = tid; q < 2048; q += kFuThreads) a.hist[(par ^ 1) * 2048 + q] = 0;
      for (int q = tid; q < a.nchunks; q += kFuThreads) a.cmax[(par ^ 1) * a.nchunks + q] = 0u;
      if (tid == 0) a.flags[par ^ 1] = 0;
    }
    if (tid == 0) s_flag = __ldcg(&a.flags[par]);
    const bool all = a.s >= a.N;
    unsigned int d1 = 0;
    int above = 0;
    int* cnt_s = sel_hist;                                        // [G + 1] candidate offsets (S2)
    bool fast = false;
    if (bkey) {
      // the candidates are exactly the keys >= bkey (x's support included: as[] holds a); if
      // at least s of them exist, the s-th largest key is >= bkey and every entry of H_s(a),
      // ties included, is a candidate: S2 selects from them alone (d1 from their histogram)
      for (int c = tid; c < G; c += kFuThreads) cnt_s[c] = __ldcg(&a.cand_cnt[c]);
      __syncthreads();
      int tot = 0;
      for (int c = lane; c < G; c += 32) tot += cnt_s[c];
      tot = __reduce_add_sync(0xffffffffu, tot);
      fast = !s_flag && tot >= a.s && tot <= kFuCandCap;         // same on every CTA
      __syncthreads();
      if (!fast && !s_flag) {                                     // the bound missed: the histogram
        if (T > 0) {                                              // the A phase skipped
          for (int q = tid; q < ncol; q += kFuThreads) atomicAdd(&hist_s[(__float_as_uint(as[q]) & 0x7FFFFFFFu) >> 20], 1);
          __syncthreads();
          add_hist(par);
        }
        grid_sync();                                              // ---- barrier 2b: histogram complete
      }
    }
    if (!fast) {
      {
        int hv[2048 / kFuThreads];                                // every load in flight at once
#pragma unroll
        for (int u = 0; u < 2048 / kFuThreads; ++u) hv[u] = __ldcg(&a.hist[par * 2048 + tid + u * kFuThreads]);
        __syncthreads();                                          // hist_s may still be read above
#pragma unroll
        for (int u = 0; u < 2048 / kFuThreads; ++u) hist_s[tid + u * kFuThreads] = hv[u];
      }
      __syncthreads();
      if (!all && !s_flag && a.s > 0) {
        find_bin<kFuThreads>(hist_s, 2048, a.s, &sh[0], &sh[1], scratch);
        d1 = (unsigned int)sh[0];
        above = sh[1];
      }
      write_cands([&](unsigned int key) { return all || (key >> 20) >= d1; });
    }
    stamp(n, 7);
    if (!fast) grid_sync();                                       // ---- barrier 3: candidates complete
    stamp(n, 8);
    // ================================================================ S2: exact top-s
    const int slot_out = a.trace ? n : (n & 1);
    if (s_flag) {                                                 // non-finite a: domain error
      if (cta == 0 && tid == 0)
        for (int k = slot_out; k <= (a.trace ? a.n_iter : slot_out); ++k) a.xs_nnz[k] = -1;
      n_done = n;
      break;
    }
    // candidate counts -> offsets (CTA order = increasing column index)
    int* hsel = sel_hist + ((G + 4) & ~3);                        // [2048] select_ordered's histogram
    if (!fast) {                                                  // (the fast path loaded them above)
      for (int c = tid; c < G; c += kFuThreads) cnt_s[c] = __ldcg(&a.cand_cnt[c]);
      __syncthreads();
    }
    if (warp == 0) {                                              // exclusive scan, 32 CTAs per step
      int carry = 0;
      for (int c0 = 0; c0 < G; c0 += 32) {
        const int v = c0 + lane < G ? cnt_s[c0 + lane] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (c0 + lane < G) cnt_s[c0 + lane] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) {
        cnt_s[G] = carry;
        s_total = carry;
      }
    }
    __syncthreads();
    const int C = s_total;
    if (a.s == 0) {                                               // H_0 keeps nothing
      if (tid == 0) s_nnz = 0;
    } else if (C <= kFuCandCap) {
      // one candidate per thread and round, its CTA found by binary search over the offsets:
      // every L2 load of a round is in flight at once
      for (int i0 = 0; i0 < C; i0 += 4 * kFuThreads) {
        int32_t ci[4];
        float cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kFuThreads + tid;
          if (i < C) {
            int lo = 0, hi = G;                                   // cnt_s[lo] <= i < cnt_s[hi]
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (cnt_s[mid] <= i) lo = mid; else hi = mid;
            }
            const int64_t src = (int64_t)lo * a.cap_c + (i - cnt_s[lo]);
            IHT_DCHECK(i - cnt_s[lo] >= 0 && i - cnt_s[lo] < a.cap_c && i < kFuCandCap, "fused: staged candidate");
            ci[u] = __ldcg(&a.cand_idx[src]);
            cv[u] = __ldcg(&a.cand_val[src]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kFuThreads + tid;
          if (i < C) {
            ci_s[i] = ci[u];
            cv_s[i] = cv[u];
          }
        }
      }
      __syncthreads();
      if (fast) {                                                 // bin d1 and the count above it,
        for (int q = tid; q < 2048; q += kFuThreads) hsel[q] = 0; // from the candidates' keys
        __syncthreads();
        for (int q = tid; q < C; q += kFuThreads) atomicAdd(&hsel[(__float_as_uint(cv_s[q]) & 0x7FFFFFFFu) >> 20], 1);
        __syncthreads();
        find_bin<kFuThreads>(hsel, 2048, a.s, &sh[0], &sh[1], scratch);   // C >= s
        d1 = (unsigned int)sh[0];
        above = sh[1];
      }
      // ordered block compaction of the staged candidates whose flag is set -> (dst_i, dst_v)
      auto compact = [&](auto flag, int32_t* di, float* dv) {
        int base = 0;
        for (int q0 = 0; q0 < C; q0 += kFuThreads) {
          const int q = q0 + tid;
          const bool f = q < C && flag(q);
          const unsigned int bal = __ballot_sync(0xffffffffu, f);
          if (lane == 0) wgt[warp] = __popc(bal);
          __syncthreads();
          int off = base, tot = 0;
          for (int w = 0; w < kFuWarps; ++w) {
            if (w < warp) off += wgt[w];
            tot += wgt[w];
          }
          if (f) {
            IHT_DCHECK(off + __popc(bal & lt) < a.s_cap, "fused: kept entry inside x");
            di[off + __popc(bal & lt)] = ci_s[q];
            dv[off + __popc(bal & lt)] = cv_s[q];
          }
          base += tot;
          __syncthreads();
        }
        return base;
      };
      if (all || C <= a.s) {
        // every candidate is kept: the nonzero keys number at most s (or s >= N)
        const int k = compact([&](int) { return true; }, xi_s, xv_s);
        if (tid == 0) s_nnz = k;
      } else {
        // bins above d1 hold `above` < s keys, all kept; the remaining need = s - above come
        // from bin d1: rank each bin-d1 key among them (greater key, or equal key at a lower
        // index -- the list is in index order) and keep ranks < need (ties to the lowest index)
        const int need = a.s - above;
        unsigned int* Dk = reinterpret_cast<unsigned int*>(hsel);   // bin-d1 keys, index order
        int* Dp = hsel + 2048;                                       // their list positions
        uint8_t* keep = reinterpret_cast<uint8_t*>(hsel + 4096);
        int C1 = 0;
        for (int q0 = 0; q0 < C; q0 += kFuThreads) {
          const int q = q0 + tid;
          const unsigned int key = q < C ? (__float_as_uint(cv_s[q]) & 0x7FFFFFFFu) : 0u;
          const bool f = q < C && (key >> 20) == d1;
          if (q < C) keep[q] = (key >> 20) > d1;
          const unsigned int bal = __ballot_sync(0xffffffffu, f);
          if (lane == 0) wgt[warp] = __popc(bal);
          __syncthreads();
          int off = C1, tot = 0;
          for (int w = 0; w < kFuWarps; ++w) {
            if (w < warp) off += wgt[w];
            tot += wgt[w];
          }
          if (f && off + __popc(bal & lt) < 2048) {
            Dk[off + __popc(bal & lt)] = key;
            Dp[off + __popc(bal & lt)] = q;
          }
          C1 += tot;
          __syncthreads();
        }
        if (C1 <= 1024) {
          for (int e0 = 0; e0 < C1; e0 += kFuThreads) {
            const int e = e0 + tid;
            const bool have = e < C1;
            const unsigned int ke = have ? Dk[e] : 0u;
            int rk = 0;
            if (__any_sync(0xffffffffu, have)) {
              int f = 0;
              for (; f + 4 <= C1; f += 4) {                       // broadcast reads, 4 in flight
                const unsigned int k0 = Dk[f], k1 = Dk[f + 1], k2 = Dk[f + 2], k3 = Dk[f + 3];
                rk += (k0 > ke || (k0 == ke && f < e)) + (k1 > ke || (k1 == ke && f + 1 < e)) +
                      (k2 > ke || (k2 == ke && f + 2 < e)) + (k3 > ke || (k3 == ke && f + 3 < e));
              }
              for (; f < C1; ++f) {
                const unsigned int kf = Dk[f];
                rk += kf > ke || (kf == ke && f < e);
              }
            }
            if (have && rk < need) keep[Dp[e]] = 1;
          }
          __syncthreads();
          const int k = compact([&](int q) { return keep[q] != 0; }, xi_s, xv_s);
          if (tid == 0) s_nnz = k;
        } else {                                                  // a crowded bin: radix passes
          select_ordered<kFuThreads>(C, a.s, [&](int i) { return cv_s[i]; }, [&](int i) { return ci_s[i]; }, xi_s,
                                     xv_s, &s_nnz, 0, hsel, scratch, wgt, weq, wtake, wbase, sh);
        }
      }
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
    stamp(n, 9);
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
  if (lane == 0) {
    for (int b = consumed; b < nb; ++b) {
      mbar_wait(wfull + 8 * c_slot, c_par);
      if (++c_slot == a.mslot) {
        c_slot = 0;
        c_par ^= 1u;
      }
    }
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
  long long* tl = nullptr;
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
  if (q.cols > 0x7FFFFFFF || q.rows > 0x7FFFFFFF || s < 0 || K > 2048) return IHT_EUNSUPPORTED;
  if ((int64_t)n_iter * ((q.cols + 15) / 16) > 0x7FFFFFFF) return IHT_EUNSUPPORTED;
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
  const size_t u_bytes = std::max({(size_t)tmax * nchunks * 16 * 12, (size_t)2048 * 4,
                                   (size_t)kFuCandCap * 8 + (size_t)(((G + 4) & ~3) + 2048 + 2048) * 4 +
                                       (size_t)kFuCandCap});
  auto layout = [&](int nring, int block_bytes, FusedArgs* A) {   // nring = 8 warps x mslot slots
    o = (size_t)nring * block_bytes;
    const size_t bars = o;
    o = al16(o + 8 * (size_t)nring);
    const size_t limbs = o;
    o = al16(o + 3 * (size_t)(Rpad + 64));
    const size_t fc = o;
    o = al16(o + 16 * (size_t)nchunks);
    const size_t as = o;
    o = al16(o + 4 * (size_t)cap_c);
    const size_t xo = o;
    o = al16(o + 8 * (size_t)s_cap);
    const size_t uo = o;
    o = al16(o + u_bytes);
    const size_t tb = o;
    o = al16(o + 8 * (size_t)K);
    const size_t ho = o;
    o += 2048 * 4;
    if (A) {
      A->off_bars = (int)bars;
      A->off_limbs = (int)limbs;
      A->off_fc = (int)fc;
      A->off_as = (int)as;
      A->off_x = (int)xo;
      A->off_u = (int)uo;
      A->off_tab = (int)tb;
      A->off_h = (int)ho;
    }
    return o;
  };
  const size_t limit = (size_t)optin - 8192;          // static shared memory and margin
  const size_t rest = layout(0, 0, nullptr);
  // ring: each warp owns mslot >= 2 blocks (double buffering); a block is a whole number of
  // 1 KiB k-steps, the largest divisor nsub of the tile's KS k-steps that fits
  const int KSTEP = 512 / B, KS = Rpad / KSTEP;
  const int tw_max = (tmax + kFuWarps - 1) / kFuWarps;          // tiles per warp
  int nsub = 0, mslot = 0;
  for (int d = 1; d <= KS; ++d) {
    if (KS % d) continue;
    const size_t blk = (size_t)tile_bytes / d;
    if (rest + (size_t)kFuWarps * 2 * (blk + 8) <= limit) {
      nsub = d;
      mslot = (int)((limit - rest) / ((size_t)kFuWarps * (blk + 8)));
      mslot = std::max(2, std::min(mslot, std::max(2, tw_max * d)));
      break;
    }
  }
  if (nsub == 0) return IHT_EUNSUPPORTED;
  const int block_bytes = tile_bytes / nsub;
  iht_fused_state* S = new iht_fused_state();
  FusedArgs& A = S->args;
  S->smem = layout(kFuWarps * mslot, block_bytes, &A);
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
  A.nsub = nsub;
  A.block_bytes = block_bytes;
  A.mslot = mslot;
  A.tile_bytes = tile_bytes;
  A.nchunks = nchunks;
  A.wpc = wpc;
  A.words_total = words_total;
  A.cap_c = cap_c;
  A.limb_stride = Rpad + 64;   // planes 64 B apart (mod 128): the 8 lanes of an LDS.128 phase (planes 0, 1) hit disjoint banks
  A.s_cap = s_cap;
  A.yhat = yhat;
  A.r = r;
  A.g = g;
  A.xs_idx = xs_idx;
  A.xs_val = xs_val;
  A.xs_nnz = xs_nnz;
  A.trace = trace;
  A.probe = getenv("IHT_FUSED_PROBE") ? atoi(getenv("IHT_FUSED_PROBE")) : 0;   // profiling only
  A.nobound = getenv("IHT_FUSED_NOBOUND") ? atoi(getenv("IHT_FUSED_NOBOUND")) : 0;
  // 0.7 (r02 g65, count criterion): config 2 63.1k iter/s (0.9: 62.1k, 0.5: 56.9k), config 3 37.9k
  A.bound_frac = getenv("IHT_FUSED_BOUND") ? (float)atof(getenv("IHT_FUSED_BOUND")) : 0.7f;
  if (getenv("IHT_FUSED_TL")) {        // profiling only: per-phase globaltimer stamps of one CTA
    A.tl_cta = atoi(getenv("IHT_FUSED_TL"));
    if (A.tl_cta >= G) A.tl_cta = 0;
    const size_t nt = (size_t)std::max(64, G) * 16;
    if (cudaMalloc(&S->tl, nt * sizeof(long long)) == cudaSuccess) {
      cudaMemset(S->tl, 0, nt * sizeof(long long));
      A.tl = S->tl;
    }
  }
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
  if (S->tl && S->args.tl_cta < 0) {   // profiling: per-CTA phase durations of iteration 3
    std::vector<long long> h((size_t)S->G * 16);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), S->tl, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    const char* names[9] = {"F", "B1", "limbs", "A", "hist", "B2", "S1", "B3", "S2"};
    fprintf(stderr, "fused per-CTA (iteration 3, ns): ");
    for (int k = 0; k < 9; ++k) {
      std::vector<std::pair<long long, int>> d;
      for (int c = 0; c < S->G; ++c) d.push_back({h[c * 16 + k + 1] - h[c * 16 + k], c});
      std::sort(d.begin(), d.end());
      fprintf(stderr, " %s min %lld med %lld max %lld (cta %d)", names[k], d[0].first, d[d.size() / 2].first,
              d.back().first, d.back().second);
    }
    long long t0 = h[1 * 16 + 4];                    // A end of CTA 1 as reference
    fprintf(stderr, "\n  A-end offsets vs CTA 1 (ns):");
    for (int c = 0; c < S->G; ++c) fprintf(stderr, " %lld", h[c * 16 + 4] - t0);
    fprintf(stderr, "\n");
    cudaFree(S->tl);
    S->tl = nullptr;
  }
  if (S->tl) {                         // profiling: median phase durations (ns) over the recorded iterations
    long long h[64 * 16];
    cudaDeviceSynchronize();
    cudaMemcpy(h, S->tl, sizeof(h), cudaMemcpyDeviceToHost);
    const int nit = S->args.n_iter < 64 ? S->args.n_iter : 64;
    const char* names[9] = {"F", "B1", "limbs", "A", "hist", "B2", "S1", "B3", "S2"};
    fprintf(stderr, "fused timeline (CTA %d, ns, median of %d iterations):", S->args.tl_cta, nit > 1 ? nit - 1 : nit);
    for (int k = 0; k < 9; ++k) {
      std::vector<long long> d;
      for (int n = (nit > 1 ? 1 : 0); n < nit; ++n) d.push_back(h[n * 16 + k + 1] - h[n * 16 + k]);
      std::sort(d.begin(), d.end());
      fprintf(stderr, " %s %lld", names[k], d.empty() ? -1 : d[d.size() / 2]);
    }
    for (int k = 10; k < 15; ++k) {                  // A: tile 0..2 wait start / wait end
      std::vector<long long> d;
      for (int n = (nit > 1 ? 1 : 0); n < nit; ++n) d.push_back(h[n * 16 + k + 1] - h[n * 16 + k]);
      std::sort(d.begin(), d.end());
      fprintf(stderr, " a%d %lld", k - 10, d.empty() ? -1 : d[d.size() / 2]);
    }
    int skipped = 0;                                 // bounded-candidate iterations (no S1 / barrier 3)
    for (int n = 0; n < nit; ++n) skipped += h[n * 16 + 8] - h[n * 16 + 7] < 300;
    fprintf(stderr, " | B3 skipped %d/%d", skipped, nit);
    std::vector<long long> it;
    for (int n = 1; n < nit; ++n) it.push_back(h[n * 16] - h[(n - 1) * 16]);
    std::sort(it.begin(), it.end());
    fprintf(stderr, " | iteration %lld\n", it.empty() ? -1 : it[it.size() / 2]);
    cudaFree(S->tl);
  }
  if (S->block) cudaFree(S->block);
  delete S;
}
