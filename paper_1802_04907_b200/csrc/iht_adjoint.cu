// (a5) adjoint gradient g = Re(Phi-hat_A^H r) = sigma_A * Q_A^T r over stacked rows.
//
// P:349 (Algorithm 1: g^{[n]} = Phi-hat_{2n-1}^dagger (...)).  This is the step that
// streams the whole quantised copy every iteration: "runtime of IHT depends
// linearly on the size of Phi", T = size(Phi)/P.  The paper's CPU
// code casts it "in terms of dot-products": g_n = <column strip n, r>.
//
// Two variants (iht.h, iht_adjoint `variant`):
//
//  1 = CUDA-core baseline.  A warp owns 4 columns, streams 16-byte code chunks,
//      decodes codes with LOP3 + FADD (2^23 magic) and accumulates
//      sum_m code * r_m with FFMA; g = sigma (2 sum code r - (L-1) sum r).
//      About 3 instructions per code: ALU-bound below the HBM roof at 2/4 bits.
//
//  0 = int8 tensor-core path (default).  The same dot products run on
//      mma.sync.m16n8k32.u8.s8.s32: A = 16 columns x 32 rows of codes (u8, built in
//      registers from the packed strips with one LOP3 per 4 codes at 4 bits),
//      B = r in block fixed point split into three signed 8-bit limbs (columns
//      n = 0,1,2 of the 8-wide B), exact int32 accumulation, flushed every 4096-row
//      chunk into float via exact int64/double arithmetic:
//         g_n = sigma sum_c 2^{-F_c} (2 V_{c,n} - (L-1) S_c),
//         V_{c,n} = sum_{m in c} code_{m,n} r_int_m,   S_c = sum_{m in c} r_int_m,
//      r_int_m = rint(r_m 2^{F_c}), |r_int| <= 2^22 (F_c from the chunk's max |r|).
//      The only rounding is r's 23-bit fixed point per chunk and the final float
//      accumulation; the k order inside an MMA is permuted consistently on A and B
//      (the sum is order-free in exact integer arithmetic).
//      The MMA takes the MACs off the ALU so the kernel can stay on the HBM roof;
//      this is still a GEMV (N = 3 useful of 8 MMA columns), not a reshaped GEMM.
#include <stdlib.h>

#include "iht_internal.cuh"
#include "iht_mma.cuh"

namespace iht {

// =====================================================================================
// Variant 1: CUDA-core FFMA baseline
// =====================================================================================
constexpr int kFfmaCols = 4;   // columns per warp

// streaming 16-byte load that also asks L2 to fetch the surrounding 256-byte block
__device__ __forceinline__ uint4 ld_stream_u4_l2pf(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// per-thread L2 prefetch of the cache line holding p (no registers / smem used)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int B>
__global__ void __launch_bounds__(256) adjoint_ffma_kernel(const uint8_t* __restrict__ codes,
                                                           int64_t strip_bytes, int64_t N, int L,
                                                           float sigma, const float* __restrict__ r,
                                                           float* __restrict__ g) {
  constexpr int CPW = 32 / B;            // codes per word
  constexpr int RPC = 128 / B;           // rows per 16-byte chunk
  constexpr uint32_t MASK = (1u << B) - 1u;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t col0 = warp * kFfmaCols;
  if (col0 >= N) return;
  const int ncol = (int)min64(kFfmaCols, N - col0);
  float acc[kFfmaCols];
#pragma unroll
  for (int c = 0; c < kFfmaCols; ++c) acc[c] = 0.0f;
  float rsum = 0.0f;
  const int64_t chunks = strip_bytes / 16;
  for (int64_t ch = lane; ch < chunks; ch += 32) {
    uint4 w[kFfmaCols];
#pragma unroll
    for (int c = 0; c < kFfmaCols; ++c)
      w[c] = (c < ncol) ? ld_stream_u4(codes + tiled_offset(col0 + c, ch * 16, strip_bytes)) : make_uint4(0, 0, 0, 0);
    const float4* r4 = reinterpret_cast<const float4*>(r + ch * RPC);
#pragma unroll
    for (int q = 0; q < RPC / 4; ++q) {
      const float4 rv = __ldg(r4 + q);
      const float rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = q * 4 + e;                   // row inside the chunk
        const int wi = row / CPW, sh = (row % CPW) * B;
        rsum += rr[e];
#pragma unroll
        for (int c = 0; c < kFfmaCols; ++c) {
          const uint32_t word = wi == 0 ? w[c].x : wi == 1 ? w[c].y : wi == 2 ? w[c].z : w[c].w;
          const float cf = __int_as_float(0x4B000000u | ((word >> sh) & MASK)) - 8388608.0f;
          acc[c] = __fmaf_rn(cf, rr[e], acc[c]);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
#pragma unroll
    for (int c = 0; c < kFfmaCols; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  }
  if (lane < ncol) {
    float a = acc[0];
#pragma unroll
    for (int c = 1; c < kFfmaCols; ++c)
      if (lane == c) a = acc[c];
    g[col0 + lane] = sigma * (2.0f * a - (float)(L - 1) * rsum);
  }
}

// =====================================================================================
// Variant 0: int8 mma.sync path
// =====================================================================================
constexpr int kMmaWarps = 8;           // warps per CTA
constexpr int kChunkRows = 4096;       // rows per fixed-point chunk (int32-safe flush)
constexpr int kMaxKR = 32768;          // rows of r limbs resident in shared memory per CTA
constexpr int kReq = 4;                // k-steps (1 KiB tile-steps) per bulk request
constexpr int kRing = 3;               // requests in flight per warp (shared-memory ring slots)
constexpr int kSlot = kReq * 1024;     // bytes per ring slot
static_assert(kMmaWarps * 32 == 256, "the prologue loops assume 256 threads");

struct AdjArgs {
  const uint8_t* codes;
  int64_t strip_bytes;   // = R_pad * B / 8
  int64_t N;
  int64_t Rpad;          // stacked rows (incl. padding)
  int KR;                // rows per K-range (CTA pass), multiple of 256, <= kMaxKR
  int KRp;               // KR rounded up to whole 1024-row requests (limb planes; rows >= KR are zero)
  int KC;                // rows per fixed-point chunk, divides KRp
  int nK;                // number of K-ranges
  int L;
  float sigma;
  const float* r;
  float* g;              // nK == 1: final g; else partial[nK][N] (unscaled by sigma)
  int limb_stride;       // bytes between limb planes in smem
  int probe;             // profiling (IHT_ADJ_PROBE=1): no r prologue; results invalid
};

// Shared-memory layout of the MMA kernel:
//   [ring]  kMmaWarps x kRing slots x 1 KiB: each lane's two 16-byte code chunks of a k-step
//           (a lane only ever reads back what it copied itself)
//   [limbs] 3 planes x limb_stride bytes: r in 3 signed 8-bit limbs, permuted per lane chunk
//   [Fc, Sl, red] per-chunk exponents, exact per-limb integer sums of r_int, scratch
template <int B, int RING>
__global__ void __launch_bounds__(kMmaWarps * 32, 1) adjoint_mma_kernel(AdjArgs a) {
  pdl_launch_dependents();
  constexpr int P = 8 / B;               // codes per byte
  constexpr int RPC = 128 / B;           // rows per 16-byte lane chunk
  constexpr int KSTEP = 4 * RPC;         // rows per warp k-step (4 lanes t)
  constexpr int NMMA = 2 * P;            // MMAs per k-step
  extern __shared__ __align__(16) uint8_t smem[];
  const int nchunks = a.KRp / a.KC;
  uint8_t* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kMmaWarps * RING * kSlot);   // [warp][slot]
  uint8_t* limbs = smem + kMmaWarps * RING * kSlot + kMmaWarps * RING * 8;
  int* Fc = reinterpret_cast<int*>(limbs + 3 * a.limb_stride);
  int* Sl = Fc + ((nchunks + 1) & ~1);                     // [chunk][3] limb sums of r_int
  float* red = reinterpret_cast<float*>(Sl + 3 * nchunks);  // [nchunks][kMmaWarps] scratch
  int& nonfinite = *reinterpret_cast<int*>(red + nchunks * kMmaWarps);   // r holds a NaN / inf

  const int kr = blockIdx.y;
  const int64_t row0 = (int64_t)kr * a.KR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- work assignment; the first RING k-steps are requested before the prologue ------
  const int g8 = lane >> 2, t = lane & 3;
  const int64_t ntask = (a.N + 15) / 16;
  const int64_t wid = (int64_t)blockIdx.x * kMmaWarps + warp;
  const int64_t wstride = (int64_t)gridDim.x * kMmaWarps;
  const int64_t rend = min64(row0 + a.KR, a.Rpad);                 // rows of this K-range
  const int nsteps = (int)((rend - row0) / KSTEP);                  // last K-range may be short
  const uint8_t* kbase = a.codes + (row0 * B / 8 >> 6) * 1024 + t * 16;   // K-range offset in a tile
  auto task_ptr = [&](int64_t task, const uint8_t*& b0, const uint8_t*& b1) {
    const uint8_t* b = kbase + task * 16 * a.strip_bytes;
    const int64_t cc0 = task * 16 + g8;       // columns past N read column 0 of the tile
    b0 = b + (cc0 < a.N ? g8 : 0) * 64;
    b1 = b + (cc0 + 8 < a.N ? g8 + 8 : 0) * 64;
  };
  // the request loop runs npad k-steps per task (nsteps rounded up to whole requests); the
  // padded steps past nsteps are skipped (config 3: 9 real k-steps of 12 per task)
  const int npad = (nsteps + kReq - 1) / kReq * kReq;
  const uint32_t ring_w = (uint32_t)__cvta_generic_to_shared(ring + warp * RING * kSlot);
  const uint32_t bar_w = (uint32_t)__cvta_generic_to_shared(bars + warp * RING);
  if (lane == 0)
    for (int j = 0; j < RING; ++j) mbar_init(bar_w + 8 * j, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // request cursor (lane 0) over this warp's flat k-step sequence (task wid, wid + wstride,
  // ...): each request is one bulk copy of kReq consecutive tile-steps (kReq x 1 KiB)
  const uint8_t* kseg = a.codes + (row0 * B / 8 >> 6) * 1024;    // K-range offset inside a tile
  int64_t rq_task = wid;
  int rq_ks = 0;
  const uint8_t* rq = kseg + rq_task * 16 * a.strip_bytes;
  auto request = [&](int slot) {
    if (rq_task < ntask) {
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)min(kReq, nsteps - rq_ks) * 1024;
        const uint32_t bar = bar_w + 8 * slot;
        IHT_DCHECK(slot < RING && rq >= a.codes && rq + bytes <= a.codes + ntask * 16 * a.strip_bytes,
                   "adjoint: bulk request inside the copy");
        mbar_expect_tx(bar, bytes);
        bulk_g2s(ring_w + slot * kSlot, rq, bytes, bar);
      }
      if ((rq_ks += kReq) < npad) {
        rq += kSlot;
      } else {
        rq_ks = 0;
        rq_task += wstride;
        rq = kseg + rq_task * 16 * a.strip_bytes;
      }
    }
  };
#pragma unroll 1
  for (int j = 0; j < RING; ++j) request(j);

  unsigned int* cmax = reinterpret_cast<unsigned int*>(red);   // [nchunks] max |r| bit pattern
  for (int c = tid; c < nchunks; c += blockDim.x) cmax[c] = 0u;
  if (tid == 0) nonfinite = 0;
  __syncthreads();
  // the code requests above read only the (constant) copy; r comes from the forward kernel
  pdl_wait();
  // ---- prologue 1: per-chunk max |r| -> exponent F_c ---------------------------------
  // (max over |r| bit patterns: a NaN or inf in r is caught and makes g NaN, so that H_s
  // reports the domain error).  float4 loads, 16 in flight per thread: a 1024-row
  // group (256 float4) never straddles a chunk (KC is a multiple of 1024), so the chunk of
  // each load is warp-uniform and one warp max + one shared atomicMax per load suffice.
  if (!(a.probe & 1)) {                  // profiling probe 1: no r prologue (timing only)
    const int n4 = (int)((rend - row0) >> 2);             // real rows (multiple of 256) / 4
    const float4* r4 = reinterpret_cast<const float4*>(a.r + row0);
    for (int j0 = 0; j0 < n4; j0 += 256 * 16) {
      float4 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int j = j0 + u * 256 + tid;
        v[u] = j < n4 ? __ldg(r4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (j0 + u * 256 >= n4) break;
        unsigned int m = max(max(__float_as_uint(v[u].x) & 0x7FFFFFFFu, __float_as_uint(v[u].y) & 0x7FFFFFFFu),
                             max(__float_as_uint(v[u].z) & 0x7FFFFFFFu, __float_as_uint(v[u].w) & 0x7FFFFFFFu));
        m = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0 && m) atomicMax(&cmax[((j0 + u * 256) * 4) / a.KC], m);
      }
    }
  }
  __syncthreads();
  for (int c = tid; c < nchunks; c += blockDim.x) {
    unsigned int mb = cmax[c];
    if (mb >= 0x7F800000u) {
      nonfinite = 1;
      mb = 0;
    }
    const float m = __uint_as_float(mb);
    int e = 0;
    if (m > 0.0f) frexpf(m, &e);            // m in [2^{e-1}, 2^e)
    Fc[c] = (m > 0.0f) ? min(22 - e, 126) : 0;   // |r| 2^F < 2^22 (clamped for tiny r)
    Sl[3 * c] = Sl[3 * c + 1] = Sl[3 * c + 2] = 0;
  }
  __syncthreads();
  // ---- prologue 2: r -> three balanced signed 8-bit limbs, permuted per lane chunk -----
  // A thread converts whole lane chunks (RPC consecutive rows = the 4P items of one lane's
  // 16-byte code chunk): RPC/4 contiguous float4 loads per chunk, 16 float4 in flight per
  // thread, issued before any conversion; two STS.128 per plane and bit position.  At b = 2
  // (64-row lane chunks, only a multiple of 16 of them per K-range) the item-wise form: a
  // thread converts items of 4 rows with kIt items' loads in flight.
  if constexpr (B == 2) {
    if (!(a.probe & 1)) {
      // items = KRp / 4, a multiple of 256: every warp runs the same trip count.  The r loads
      // of kIt items per thread are issued before any of them is converted.
      constexpr int kIt = 4;
      const int items = a.KRp / RPC * (4 * P);
      for (int it0 = tid; it0 < items; it0 += kIt * 256) {
      float rvs[kIt][4];
  #pragma unroll
      for (int q = 0; q < kIt; ++q) {
        const int it = it0 + q * 256;
        const int ch = it / (4 * P), rho = it % (4 * P);
        const int base = ch * RPC + (rho / P) * (32 / B) + (rho % P);
  #pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t row = row0 + base + P * i;
          rvs[q][i] = (it < items && row < rend) ? __ldg(a.r + row) : 0.0f;   // zero limbs past the K-range
        }
      }
  #pragma unroll
      for (int q = 0; q < kIt; ++q) {
        const int it = it0 + q * 256;
        if (it >= items) break;                                 // warp-uniform
        const int ch = it / (4 * P), rho = it % (4 * P);
        const int c = (ch * RPC) / a.KC;
        const float scale = ldexpf(1.0f, Fc[c]);
        uint32_t l0w = 0, l1w = 0, l2w = 0;
        int s0 = 0, s1 = 0, s2 = 0;
  #pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float rv = rvs[q][i];
          const int ri = __float2int_rn(rv * scale);            // exact power-of-two scaling
          const int l0 = ((ri + 128) & 255) - 128;
          const int t1 = (ri - l0) >> 8;
          const int l1 = ((t1 + 128) & 255) - 128;
          const int l2 = (t1 - l1) >> 8;
          s0 += l0; s1 += l1; s2 += l2;
          l0w |= (uint32_t)(l0 & 255) << (8 * i);
          l1w |= (uint32_t)(l1 & 255) << (8 * i);
          l2w |= (uint32_t)(l2 & 255) << (8 * i);
        }
        // bank-spread layout: k-step ch / 4 holds 64 P bytes per plane; the 16-byte chunk of
        // (bit position j = rho % P, lane t = ch % 4) sits at (4 j + t) 16, word v = rho / P in it
        const int off = (ch >> 2) * (64 * P) + (4 * (rho % P) + (ch & 3)) * 16 + (rho / P) * 4;
        IHT_DCHECK(off + 4 <= a.limb_stride, "adjoint: limb word inside its plane");
        *reinterpret_cast<uint32_t*>(limbs + off) = l0w;
        *reinterpret_cast<uint32_t*>(limbs + a.limb_stride + off) = l1w;
        *reinterpret_cast<uint32_t*>(limbs + 2 * a.limb_stride + off) = l2w;
        // the 32 items of a warp lie in one chunk (128 consecutive rows): one native int32
        // atomic per limb and warp (|sum| <= 128 x 4096 per chunk)
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
    }
  } else {
    if (!(a.probe & 1)) {
      constexpr int NV = RPC / 4;                   // float4 per lane chunk: 4 (b = 8), 8 (4), 16 (2)
      constexpr int CPT = NV >= 16 ? 1 : 16 / NV;   // lane chunks per thread per round
      const int nch = a.KRp / RPC;                  // a multiple of 32 (b >= 4): warp-uniform trip counts
      for (int ch0 = tid; ch0 < nch; ch0 += CPT * 256) {
        float4 rv[CPT][NV];
  #pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int ch = ch0 + q * 256;
  #pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int64_t row = row0 + (int64_t)ch * RPC + 4 * v;
            rv[q][v] = (ch < nch && row < rend) ? __ldg(reinterpret_cast<const float4*>(a.r + row))
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);   // zero limbs past the K-range
          }
        }
  #pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int ch = ch0 + q * 256;
          if (ch >= nch) break;                     // warp-uniform
          const int c = (ch * RPC) / a.KC;
          const float scale = ldexpf(1.0f, Fc[c]);
          const float* rr = reinterpret_cast<const float*>(&rv[q][0]);   // rows ch*RPC + 0 .. RPC-1
          int s0 = 0, s1 = 0, s2 = 0;
  #pragma unroll
          for (int e = 0; e < P; ++e) {
            uint32_t l0w[4], l1w[4], l2w[4];
  #pragma unroll
            for (int h = 0; h < 4; ++h) {           // item rho = h P + e: rows h CPW + e + P i
              l0w[h] = l1w[h] = l2w[h] = 0u;
  #pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int ri = __float2int_rn(rr[h * (32 / B) + e + P * i] * scale);   // exact power-of-two scaling
                const int l0 = ((ri + 128) & 255) - 128;
                const int t1 = (ri - l0) >> 8;
                const int l1 = ((t1 + 128) & 255) - 128;
                const int l2 = (t1 - l1) >> 8;
                s0 += l0; s1 += l1; s2 += l2;
                l0w[h] |= (uint32_t)(l0 & 255) << (8 * i);
                l1w[h] |= (uint32_t)(l1 & 255) << (8 * i);
                l2w[h] |= (uint32_t)(l2 & 255) << (8 * i);
              }
            }
            // bank-spread layout: k-step ch / 4 holds 64 P bytes per plane; the 16-byte chunk of
            // (bit position j = e, lane t = ch % 4) sits at (4 j + t) 16, word h inside it
            const int off = (ch >> 2) * (64 * P) + (4 * e + (ch & 3)) * 16;
            IHT_DCHECK(off + 16 <= a.limb_stride, "adjoint: limb chunk inside its plane");
            *reinterpret_cast<uint4*>(limbs + off) = make_uint4(l0w[0], l0w[1], l0w[2], l0w[3]);
            *reinterpret_cast<uint4*>(limbs + a.limb_stride + off) = make_uint4(l1w[0], l1w[1], l1w[2], l1w[3]);
            *reinterpret_cast<uint4*>(limbs + 2 * a.limb_stride + off) = make_uint4(l2w[0], l2w[1], l2w[2], l2w[3]);
          }
          // exact per-chunk limb sums (|sum| <= 128 x 4096): one native int32 atomic per limb
          // and warp when the warp's 32 lane chunks lie in one fixed-point chunk, else per thread
          if (__all_sync(0xffffffffu, c == __shfl_sync(0xffffffffu, c, 0))) {
            s0 = __reduce_add_sync(0xffffffffu, s0);
            s1 = __reduce_add_sync(0xffffffffu, s1);
            s2 = __reduce_add_sync(0xffffffffu, s2);
            if (lane == 0) {
              atomicAdd(&Sl[3 * c], s0);
              atomicAdd(&Sl[3 * c + 1], s1);
              atomicAdd(&Sl[3 * c + 2], s2);
            }
          } else {
            atomicAdd(&Sl[3 * c], s0);
            atomicAdd(&Sl[3 * c + 1], s1);
            atomicAdd(&Sl[3 * c + 2], s2);
          }
        }
      }
    }
  }
  __syncthreads();

  // ---- main loop: tasks (16 columns x this K-range) -> fixed-point chunks -> k-steps.
  //      Step ks (global step counter gs) lives in ring slot gs % RING; after consuming it
  //      the slot is refilled with the step RING later (this task or the next one).
  const int spc = a.KC / KSTEP;                            // k-steps per chunk
  const uint32_t limb_n = (uint32_t)__cvta_generic_to_shared(limbs + (g8 < 3 ? g8 : 0) * a.limb_stride);
  const bool bload = g8 < 3;
  int slot = 0;
  uint32_t parity = 0;
  // B fragments: lanes g8 < 3 reload them every k-step; the others (B columns 3..7) hold
  // zeros for the whole kernel instead of re-zeroing 4P registers per k-step
  uint32_t bw[4 * P];
#pragma unroll
  for (int q = 0; q < 4 * P; ++q) bw[q] = 0u;
  for (int64_t task = wid; task < ntask; task += wstride) {
    float accf0 = 0.0f, accf1 = 0.0f;     // lanes t == 0: columns c0, c1
    for (int kc = 0, c = 0; kc < npad; kc += spc, ++c) {
      const int kend = min(kc + spc, npad);
      int acc[P][4];
#pragma unroll
      for (int j = 0; j < P; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
      for (int ks0 = kc; ks0 < kend; ks0 += kReq) {
        mbar_wait(bar_w + 8 * slot, parity);    // the kReq tile-steps of this request landed
        // one k-step h of this request: fragments from the ring slot, limbs, NMMA MMAs; the
        // slot is refilled after the request's last k-step has its fragments
        auto kstep = [&](int h) {
          const int ks = ks0 + h;
          const uint32_t src = ring_w + slot * kSlot + h * 1024 + g8 * 64 + t * 16;
          const uint4 s0 = lds128(src), s1 = lds128(src + 512);
          if (bload) {                           // other lanes keep the zeros set once below
            const uint32_t bp = limb_n + (uint32_t)ks * (64 * P) + t * 16;   // 12 lanes: 3 x 4 bank quads
#pragma unroll
            for (int q = 0; q < P; ++q) {
              const uint4 v = lds128(bp + 64 * q);
              bw[4 * q + 0] = v.x; bw[4 * q + 1] = v.y; bw[4 * q + 2] = v.z; bw[4 * q + 3] = v.w;
            }
          }
          uint32_t af[NMMA][4];          // MMA u = 2 j + m: words 2m (k-slots 0..15), 2m+1 (16..31)
#pragma unroll
          for (int j = 0; j < P; ++j)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              af[2 * j + m][0] = frag_reg<B>(s0, 2 * m, j);
              af[2 * j + m][1] = frag_reg<B>(s1, 2 * m, j);
              af[2 * j + m][2] = frag_reg<B>(s0, 2 * m + 1, j);
              af[2 * j + m][3] = frag_reg<B>(s1, 2 * m + 1, j);
            }
          if (h == kReq - 1) {
            __syncwarp();                        // every lane has its fragments: slot is free
            request(slot);                       // refill it with the request RING later
          }
#pragma unroll
          for (int i = 0; i < NMMA; ++i) {   // consecutive MMAs update different accumulators
            const int u = (i % P) * 2 + i / P;
            mma_u8s8(acc[u >> 1], af[u], bw[2 * u], bw[2 * u + 1]);
          }
        };
        if (ks0 + kReq <= nsteps) {              // whole request (all but a task's last, or all)
#pragma unroll
          for (int h = 0; h < kReq; ++h) kstep(h);
        } else {                                 // the last request: skip the padding k-steps
#pragma unroll
          for (int h = 0; h < kReq; ++h) {
            if (ks0 + h < nsteps) {
              kstep(h);
            } else if (h == kReq - 1) {          // warp-uniform; the slot is still refilled once
              __syncwarp();
              request(slot);
            }
          }
        }
        if (++slot == RING) {
          slot = 0;
          parity ^= 1u;
        }
      }
      // flush chunk c: combine bit-positions exactly (every term of acc_j is a multiple of
      // 2^{B j}); lane t=0 holds limbs 0,1 (cols 0,1), lane t=1 holds limb 2 (col 2)
      int v00 = 0, v01 = 0, v10 = 0, v11 = 0;
#pragma unroll
      for (int j = 0; j < P; ++j) {
        v00 += acc[j][0] >> (B * j);
        v01 += acc[j][1] >> (B * j);
        v10 += acc[j][2] >> (B * j);
        v11 += acc[j][3] >> (B * j);
      }
      const int l2r0 = __shfl_down_sync(0xffffffffu, v00, 1);
      const int l2r1 = __shfl_down_sync(0xffffffffu, v10, 1);
      if (t == 0) {
        const long long S = (long long)Sl[3 * c] + 256ll * Sl[3 * c + 1] + 65536ll * Sl[3 * c + 2];
        const double sc = ldexp(1.0, -Fc[c]);
        const long long V0 = (long long)v00 + 256ll * v01 + 65536ll * l2r0;
        const long long V1 = (long long)v10 + 256ll * v11 + 65536ll * l2r1;
        accf0 += (float)((double)(2 * V0 - (long long)(a.L - 1) * S) * sc);
        accf1 += (float)((double)(2 * V1 - (long long)(a.L - 1) * S) * sc);
      }
    }
    const int64_t c0 = task * 16 + g8, c1 = c0 + 8;
    if (t == 0) {
      if (nonfinite) accf0 = accf1 = __int_as_float(0x7FC00000);
      if (a.nK == 1) {
        if (c0 < a.N) a.g[c0] = a.sigma * accf0;
        if (c1 < a.N) a.g[c1] = a.sigma * accf1;
      } else {
        if (c0 < a.N) a.g[(int64_t)kr * a.N + c0] = accf0;
        if (c1 < a.N) a.g[(int64_t)kr * a.N + c1] = accf1;
      }
    }
  }
}

__global__ void adjoint_reduce_kernel(const float* __restrict__ part, int nK, int64_t N, float sigma,
                                      float* __restrict__ g) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = part[n];
  for (int k = 1; k < nK; ++k) s = __fadd_rn(s, part[(int64_t)k * N + n]);   // thr_cluster_kernel: same order
  g[n] = __fmul_rn(sigma, s);
}

struct AdjPlan {
  int KR, KRp, KC, nK, limb_stride, ring;
  size_t smem;
  int ctas_x;
};

static AdjPlan plan_adjoint(const iht_qmat* A, int num_sms) {
  AdjPlan p{};
  const int64_t Rpad = A->planes * rows_pad(A->rows);
  const int64_t ntask = (A->cols + 15) / 16;
  const int64_t warps_full = (int64_t)num_sms * kMmaWarps;
  // K-range: as large as fits (<= kMaxKR), but split K when there are too few column
  // tasks to give every warp of the GPU several tasks.
  // K-ranges and chunks are whole multiples of 1024 rows so that every chunk holds a
  // multiple of kPF k-steps for b = 2, 4, 8 (k-step = 512/b rows)
  // nK equal K-ranges of KR rows (a multiple of 256, so a whole number of k-steps at every
  // bit width); each CTA's limb planes are padded to whole 1024-row requests with zero limbs.
  int64_t nK = (Rpad + kMaxKR - 1) / kMaxKR;
  while (ntask * nK < 4 * warps_full && Rpad / (nK + 1) >= 1024) ++nK;
  int64_t KR = ((Rpad + nK - 1) / nK + 255) / 256 * 256;
  {
    static int kr_env = -1;                       // profiling override (IHT_ADJ_KR, rows)
    if (kr_env < 0) kr_env = getenv("IHT_ADJ_KR") ? atoi(getenv("IHT_ADJ_KR")) : 0;
    if (kr_env >= 1024) KR = min64((int64_t)kr_env / 1024 * 1024, kMaxKR);
  }
  p.KR = (int)KR;
  {
    static int ring_env = -1;                     // profiling override (IHT_ADJ_RING = 3 or 5 slots per warp)
    if (ring_env < 0) ring_env = getenv("IHT_ADJ_RING") ? atoi(getenv("IHT_ADJ_RING")) : 0;
    p.ring = ring_env == 5 ? 5 : kRing;
  }
  p.KRp = (int)((KR + 1023) / 1024 * 1024);
  int d = 4;                            // KC = 1024 d <= kChunkRows, dividing KRp
  while ((p.KRp / 1024) % d) --d;
  p.KC = 1024 * d;
  p.nK = (int)((Rpad + KR - 1) / KR);
  p.limb_stride = p.KRp + 64;   // planes 64 B apart (mod 128): the 8 lanes of an LDS.128 phase (planes 0, 1) hit disjoint banks
  const int nchunks = p.KRp / p.KC;
  p.smem = (size_t)kMmaWarps * p.ring * (kSlot + 8) + (size_t)3 * p.limb_stride + sizeof(int) * ((nchunks + 1) & ~1) + sizeof(int) * 3 * nchunks +
           sizeof(float) * nchunks * kMmaWarps + 16;
  int per_sm = (int)(size_t)min64(4, (size_t)(227 * 1024) / p.smem);
  if (per_sm < 1) per_sm = 1;
  p.ctas_x = (int)max64(1, min64((ntask + kMmaWarps - 1) / kMmaWarps,
                                               ((int64_t)num_sms * per_sm + p.nK - 1) / p.nK));
  return p;
}

static int device_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = kNumSMs;
  }
  return sms;
}

}  // namespace iht

using namespace iht;

extern "C" int64_t iht_adjoint_ws_bytes(const iht_qmat* A) {
  if (A == nullptr) return -1;
  const AdjPlan p = plan_adjoint(A, device_sms());
  return p.nK > 1 ? (int64_t)p.nK * A->cols * (int64_t)sizeof(float) : 0;
}

static int adjoint_impl(const iht_qmat* A, const float* r, float* g, int variant, void* ws, int64_t ws_bytes,
                        void* stream, int* nparts, float* gsigma);

extern "C" int iht_adjoint(const iht_qmat* A, const float* r, float* g, int variant, void* ws,
                           int64_t ws_bytes, void* stream) {
  return adjoint_impl(A, r, g, variant, ws, ws_bytes, stream, nullptr, nullptr);
}

int iht_adjoint_parts(const iht_qmat* A, const float* r, float* g, void* ws, int64_t ws_bytes, void* stream,
                      int* nparts, float* gsigma) {
  if (nparts == nullptr || gsigma == nullptr) return IHT_EINVAL;
  return adjoint_impl(A, r, g, 0, ws, ws_bytes, stream, nparts, gsigma);
}

static int adjoint_impl(const iht_qmat* A, const float* r, float* g, int variant, void* ws, int64_t ws_bytes,
                        void* stream, int* nparts, float* gsigma) {
  if (A == nullptr || r == nullptr || g == nullptr) return IHT_EINVAL;
  if (A->codes == nullptr || (A->bits != 2 && A->bits != 4 && A->bits != 8)) return IHT_EINVAL;
  if (A->strip_bytes != iht_strip_bytes(A->rows, A->planes, A->bits)) return IHT_EINVAL;
  if ((reinterpret_cast<uintptr_t>(A->codes) & 15) || (reinterpret_cast<uintptr_t>(r) & 15))
    return IHT_EINVAL;
  const int L = num_levels(A->bits, A->level_mode);
  const float sigma = A->scale_c / (float)(L - 1);
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* codes = static_cast<const uint8_t*>(A->codes);
  if (variant == 1) {
    const int64_t warps = ceil_div<int64_t>(A->cols, kFfmaCols);
    const unsigned blocks = (unsigned)ceil_div<int64_t>(warps, 8);
#define IHT_ADJ1(BB) \
  adjoint_ffma_kernel<BB><<<blocks, 256, 0, st>>>(codes, A->strip_bytes, A->cols, L, sigma, r, g)
    if (A->bits == 2) IHT_ADJ1(2);
    else if (A->bits == 4) IHT_ADJ1(4);
    else IHT_ADJ1(8);
#undef IHT_ADJ1
    IHT_LAUNCH_CHECK();
    return IHT_OK;
  }
  if (variant != 0) return IHT_EINVAL;
  const AdjPlan p = plan_adjoint(A, device_sms());
  if (p.nK > 1) {
    if (ws == nullptr || ws_bytes < (int64_t)p.nK * A->cols * (int64_t)sizeof(float)) return IHT_EINVAL;
  }
  AdjArgs a{};
  a.codes = codes;
  a.strip_bytes = A->strip_bytes;
  a.N = A->cols;
  a.Rpad = A->planes * rows_pad(A->rows);
  a.KR = p.KR;
  a.KRp = p.KRp;
  a.KC = p.KC;
  a.nK = p.nK;
  a.L = L;
  a.sigma = sigma;
  a.r = r;
  a.g = p.nK > 1 ? static_cast<float*>(ws) : g;
  a.limb_stride = p.limb_stride;
  {
    static int probe_env = -1;
    if (probe_env < 0) probe_env = getenv("IHT_ADJ_PROBE") ? atoi(getenv("IHT_ADJ_PROBE")) : 0;
    a.probe = probe_env;
  }
  dim3 grid((unsigned)p.ctas_x, (unsigned)p.nK);
#define IHT_ADJ0(BB, RR)                                                                          \
  do {                                                                                            \
    static bool attr_set = false;                                                                 \
    if (!attr_set) {                                                                              \
      IHT_CUDA_CHECK(cudaFuncSetAttribute(adjoint_mma_kernel<BB, RR>,                             \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
      attr_set = true;                                                                            \
    }                                                                                             \
    IHT_CUDA_CHECK(launch_pdl(adjoint_mma_kernel<BB, RR>, grid, dim3(kMmaWarps * 32), p.smem, st, a));  \
  } while (0)
  if (p.ring == 5) {
    if (A->bits == 2) IHT_ADJ0(2, 5);
    else if (A->bits == 4) IHT_ADJ0(4, 5);
    else IHT_ADJ0(8, 5);
  } else {
    if (A->bits == 2) IHT_ADJ0(2, kRing);
    else if (A->bits == 4) IHT_ADJ0(4, kRing);
    else IHT_ADJ0(8, kRing);
  }
#undef IHT_ADJ0
  IHT_LAUNCH_CHECK();
  if (nparts) {                       // solver: the fused threshold sums the partials
    *nparts = p.nK > 1 ? p.nK : 0;
    *gsigma = sigma;
    return IHT_OK;
  }
  if (p.nK > 1) {
    IHT_CUDA_CHECK(launch_pdl(adjoint_reduce_kernel, dim3((unsigned)ceil_div<int64_t>(A->cols, 256)), dim3(256), 0,
                              st, static_cast<const float*>(ws), p.nK, A->cols, sigma, g));
    IHT_LAUNCH_CHECK();
  }
  return IHT_OK;
}
