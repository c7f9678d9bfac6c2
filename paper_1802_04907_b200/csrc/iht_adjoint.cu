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
#include "iht_internal.cuh"

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
constexpr int kMmaWarps = 16;          // warps per CTA
constexpr int kChunkRows = 4096;       // rows per fixed-point chunk (int32-safe flush)
constexpr int kMaxKR = 65536;          // rows of r limbs resident in shared memory per CTA
constexpr int kPF = 4;                 // k-steps of codes in flight per lane (register ring)

struct AdjArgs {
  const uint8_t* codes;
  int64_t strip_bytes;   // = R_pad * B / 8
  int64_t N;
  int64_t Rpad;          // stacked rows (incl. padding)
  int KR;                // rows per K-range (CTA pass), multiple of 256, <= kMaxKR
  int KC;                // rows per fixed-point chunk, divides KR
  int nK;                // number of K-ranges
  int L;
  float sigma;
  const float* r;
  float* g;              // nK == 1: final g; else partial[nK][N] (unscaled by sigma)
  int limb_stride;       // bytes between limb planes in smem
};

__device__ __forceinline__ void mma_u8s8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Byte-register rho of a 16-byte code chunk: word rho / P, extraction rho % P;
// byte i holds the code at chunk position pos(rho, i) = (rho/P)*(32/B) + rho%P + P*i.
template <int B>
__device__ __forceinline__ uint32_t byte_reg(const uint4& w, int rho) {
  constexpr int P = 8 / B;
  constexpr uint32_t M8 = ((1u << B) - 1u) * 0x01010101u;
  const int v = rho / P, j = rho % P;
  const uint32_t word = v == 0 ? w.x : v == 1 ? w.y : v == 2 ? w.z : w.w;
  return (word >> (B * j)) & M8;
}

template <int B>
__global__ void __launch_bounds__(kMmaWarps * 32, 1) adjoint_mma_kernel(AdjArgs a) {
  constexpr int P = 8 / B;               // codes per byte
  constexpr int RPC = 128 / B;           // rows per 16-byte lane chunk
  constexpr int KSTEP = 4 * RPC;         // rows per warp k-step (4 lanes t)
  constexpr int NMMA = 2 * P;            // MMAs per k-step
  extern __shared__ __align__(16) uint8_t smem[];
  // smem: [3 limb planes][KR bytes + pad] | chunk exponent F[KR/KC] | chunk sum S[KR/KC] (int64)
  const int nchunks = a.KR / a.KC;
  uint8_t* limbs = smem;
  int* Fc = reinterpret_cast<int*>(smem + 3 * a.limb_stride);
  long long* Sc = reinterpret_cast<long long*>(Fc + ((nchunks + 1) & ~1));
  float* red = reinterpret_cast<float*>(Sc + nchunks);     // [nchunks][kMmaWarps] scratch

  const int kr = blockIdx.y;
  const int64_t row0 = (int64_t)kr * a.KR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- prologue 1: per-chunk max |r| -> exponent F_c ---------------------------------
  for (int c = 0; c < nchunks; ++c) {
    float m = 0.0f;
    for (int i = tid; i < a.KC; i += blockDim.x) {
      const int64_t row = row0 + (int64_t)c * a.KC + i;
      if (row < a.Rpad) m = fmaxf(m, fabsf(__ldg(a.r + row)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[c * kMmaWarps + warp] = m;
  }
  __syncthreads();
  for (int c = tid; c < nchunks; c += blockDim.x) {
    float m = 0.0f;
    for (int w = 0; w < kMmaWarps; ++w) m = fmaxf(m, red[c * kMmaWarps + w]);
    int e = 0;
    if (m > 0.0f) frexpf(m, &e);            // m in [2^{e-1}, 2^e)
    Fc[c] = (m > 0.0f) ? min(22 - e, 126) : 0;   // |r| 2^F < 2^22 (clamped for tiny r)
    Sc[c] = 0;
  }
  __syncthreads();
  // ---- prologue 2: r -> three balanced signed 8-bit limbs, permuted per lane chunk -----
  // item = (lane chunk ch, byte-register rho): rows ch*RPC + pos(rho, i), i = 0..3
  {
    const int items = a.KR / RPC * (4 * P);
    for (int it = tid; it < items; it += blockDim.x) {
      const int ch = it / (4 * P), rho = it % (4 * P);
      const int base = ch * RPC + (rho / P) * (32 / B) + (rho % P);
      const int c = (ch * RPC) / a.KC;
      const float scale = ldexpf(1.0f, Fc[c]);
      uint32_t l0w = 0, l1w = 0, l2w = 0;
      int s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t row = row0 + base + P * i;
        const float rv = row < a.Rpad ? __ldg(a.r + row) : 0.0f;
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
      const int off = ch * (16 * P) + rho * 4;
      *reinterpret_cast<uint32_t*>(limbs + off) = l0w;
      *reinterpret_cast<uint32_t*>(limbs + a.limb_stride + off) = l1w;
      *reinterpret_cast<uint32_t*>(limbs + 2 * a.limb_stride + off) = l2w;
      const long long sv = (long long)s0 + 256ll * s1 + 65536ll * s2;
      atomicAdd(reinterpret_cast<unsigned long long*>(&Sc[c]), (unsigned long long)sv);
    }
  }
  __syncthreads();

  // ---- main loop: warp tasks of 16 columns over this K-range --------------------------
  const int g8 = lane >> 2, t = lane & 3;
  const int64_t ntask = (a.N + 15) / 16;
  const int64_t wstride = (int64_t)gridDim.x * kMmaWarps;
  const int nsteps = (int)(min64(a.KR, a.Rpad - row0) / KSTEP);   // last K-range may be short
  const int steps_per_chunk = a.KC / KSTEP;
  const uint8_t* limb_n = limbs + (g8 < 3 ? g8 : 0) * a.limb_stride;
  const bool bload = g8 < 3;
  const int64_t kbyte0 = row0 * B / 8;   // byte offset of this K-range inside a strip

  for (int64_t task = (int64_t)blockIdx.x * kMmaWarps + warp; task < ntask; task += wstride) {
    const int64_t c0 = task * 16 + g8, c1 = c0 + 8;
    const bool v0 = c0 < a.N, v1 = c1 < a.N;
    // tiled layout: k-step ks of this 16-column tile is 1 KiB contiguous; column g8 at +64*g8.
    // Loads are unconditional (no value merges that would wait on them): columns past N
    // read column 0 of the tile (results discarded) and prefetches past the last k-step
    // re-read the last k-step.
    const uint8_t* tile0 = a.codes + task * 16 * a.strip_bytes + (kbyte0 >> 6) * 1024 + t * 16;
    const uint8_t* p0 = tile0 + (v0 ? g8 : 0) * 64;
    const uint8_t* p1 = tile0 + (v1 ? g8 + 8 : 0) * 64;
    float accf0 = 0.0f, accf1 = 0.0f;     // lanes t == 0: columns c0, c1
    const int last = nsteps - 1;
    // register ring of kPF k-steps in flight per lane (plus the L2 256-byte prefetch)
    uint4 ring0[kPF], ring1[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
      const int64_t o = (int64_t)min(j, last) * 1024;
      ring0[j] = ld_stream_u4_l2pf(p0 + o);
      ring1[j] = ld_stream_u4_l2pf(p1 + o);
    }
    int acc[4] = {0, 0, 0, 0};
    int cstep = 0, chunk = 0;                 // position inside the current fixed-point chunk

    // one k-step on ring slot j: extract A fragments, optionally refill the slot, load B
    // fragments from shared memory, 2P MMAs, flush the chunk when it ends
    auto step = [&](uint4& s0, uint4& s1, int ks, bool refill) {
      uint32_t af[NMMA][4];
#pragma unroll
      for (int u = 0; u < NMMA; ++u) {
        af[u][0] = byte_reg<B>(s0, 2 * u);
        af[u][1] = byte_reg<B>(s1, 2 * u);
        af[u][2] = byte_reg<B>(s0, 2 * u + 1);
        af[u][3] = byte_reg<B>(s1, 2 * u + 1);
      }
      if (refill) {   // same registers, consumed above: nothing waits on this load for kPF steps
        const int64_t o = (int64_t)min(ks + kPF, last) * 1024;
        s0 = ld_stream_u4_l2pf(p0 + o);
        s1 = ld_stream_u4_l2pf(p1 + o);
      }
      uint32_t bw[4 * P];
      if (bload) {
        const uint4* bp = reinterpret_cast<const uint4*>(limb_n + (size_t)(ks * 4 + t) * (16 * P));
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const uint4 v = bp[q];
          bw[4 * q + 0] = v.x; bw[4 * q + 1] = v.y; bw[4 * q + 2] = v.z; bw[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4 * P; ++q) bw[q] = 0u;
      }
#pragma unroll
      for (int u = 0; u < NMMA; ++u) mma_u8s8(acc, af[u], bw[2 * u], bw[2 * u + 1]);
      if (++cstep == steps_per_chunk || ks + 1 == nsteps) {
        // flush chunk: lane t=0 holds limbs 0,1 (cols 0,1); lane t=1 holds limb 2 (col 2)
        const int c = chunk++;
        cstep = 0;
        const int l2r0 = __shfl_down_sync(0xffffffffu, acc[0], 1);
        const int l2r1 = __shfl_down_sync(0xffffffffu, acc[2], 1);
        if (t == 0) {
          const long long S = Sc[c];
          const double sc = ldexp(1.0, -Fc[c]);
          const long long V0 = (long long)acc[0] + 256ll * acc[1] + 65536ll * l2r0;
          const long long V1 = (long long)acc[2] + 256ll * acc[3] + 65536ll * l2r1;
          accf0 += (float)((double)(2 * V0 - (long long)(a.L - 1) * S) * sc);
          accf1 += (float)((double)(2 * V1 - (long long)(a.L - 1) * S) * sc);
        }
        acc[0] = acc[1] = acc[2] = acc[3] = 0;
      }
    };

    const int nmain = nsteps / kPF * kPF;
    for (int ks0 = 0; ks0 < nmain; ks0 += kPF) {
#pragma unroll
      for (int j = 0; j < kPF; ++j) step(ring0[j], ring1[j], ks0 + j, true);
    }
#pragma unroll
    for (int j = 0; j < kPF; ++j)          // drain: the last nsteps - nmain steps sit in slots 0..
      if (nmain + j < nsteps) step(ring0[j], ring1[j], nmain + j, false);
    if (t == 0) {
      if (a.nK == 1) {
        if (v0) a.g[c0] = a.sigma * accf0;
        if (v1) a.g[c1] = a.sigma * accf1;
      } else {
        if (v0) a.g[(int64_t)kr * a.N + c0] = accf0;
        if (v1) a.g[(int64_t)kr * a.N + c1] = accf1;
      }
    }
  }
}

__global__ void adjoint_reduce_kernel(const float* __restrict__ part, int nK, int64_t N, float sigma,
                                      float* __restrict__ g) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = part[n];
  for (int k = 1; k < nK; ++k) s += part[(int64_t)k * N + n];
  g[n] = sigma * s;
}

struct AdjPlan {
  int KR, KC, nK, limb_stride;
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
  int64_t KR = min64(Rpad, kMaxKR);
  KR = (KR + 255) / 256 * 256;
  while (KR > 1024 && ntask * ((Rpad + KR - 1) / KR) < 4 * warps_full) KR = (KR / 2 + 255) / 256 * 256;
  p.KR = (int)KR;
  p.KC = (int)min64(KR, kChunkRows);
  while (p.KR % p.KC) p.KC -= 256;    // KC divides KR, multiple of 256
  p.nK = (int)((Rpad + KR - 1) / KR);
  p.limb_stride = p.KR + 64;
  const int nchunks = p.KR / p.KC;
  p.smem = (size_t)3 * p.limb_stride + sizeof(int) * ((nchunks + 1) & ~1) + sizeof(long long) * nchunks +
           sizeof(float) * nchunks * kMmaWarps;
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

extern "C" int iht_adjoint(const iht_qmat* A, const float* r, float* g, int variant, void* ws,
                           int64_t ws_bytes, void* stream) {
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
  a.KC = p.KC;
  a.nK = p.nK;
  a.L = L;
  a.sigma = sigma;
  a.r = r;
  a.g = p.nK > 1 ? static_cast<float*>(ws) : g;
  a.limb_stride = p.limb_stride;
  dim3 grid((unsigned)p.ctas_x, (unsigned)p.nK);
#define IHT_ADJ0(BB)                                                                              \
  do {                                                                                            \
    static bool attr_set = false;                                                                 \
    if (!attr_set) {                                                                              \
      IHT_CUDA_CHECK(cudaFuncSetAttribute(adjoint_mma_kernel<BB>,                                 \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
      attr_set = true;                                                                            \
    }                                                                                             \
    adjoint_mma_kernel<BB><<<grid, kMmaWarps * 32, p.smem, st>>>(a);                              \
  } while (0)
  if (A->bits == 2) IHT_ADJ0(2);
  else if (A->bits == 4) IHT_ADJ0(4);
  else IHT_ADJ0(8);
#undef IHT_ADJ0
  IHT_LAUNCH_CHECK();
  if (p.nK > 1) {
    adjoint_reduce_kernel<<<(unsigned)ceil_div<int64_t>(A->cols, 256), 256, 0, st>>>(
        static_cast<const float*>(ws), p.nK, A->cols, sigma, g);
    IHT_LAUNCH_CHECK();
  }
  return IHT_OK;
}
