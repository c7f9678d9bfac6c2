// Internal helpers shared by the libiht kernels (sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "iht.h"

#define IHT_CUDA_CHECK(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) {                                   \
      iht_set_last_cuda_error(_e, #expr, __FILE__, __LINE__);  \
      return IHT_ECUDA;                                        \
    }                                                          \
  } while (0)

#define IHT_LAUNCH_CHECK() IHT_CUDA_CHECK(cudaGetLastError())

// Checked build (-DIHT_CHECKS, libiht_checked.so): device-side bounds checks on the indices of
// the hand-rolled pipelines and bounded spin waits (mbarriers, grid barrier) that trap with a
// message instead of hanging -- the stand-in for compute-sanitizer (closed on this GPU pool).
#ifdef IHT_CHECKS
#define IHT_DCHECK(cond, what)                                                                       \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("IHT_DCHECK failed: %s at %s:%d (block %d,%d thread %d)\n", what, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                                    \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#define IHT_SPIN_LIMIT (1ll << 27)
#else
#define IHT_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

void iht_set_last_cuda_error(cudaError_t e, const char* expr, const char* file, int line);

// iht_threshold_batched with the step read per snapshot from device memory (mu_dev[b]) when
// mu_dev is not NULL (adaptive step, Algorithm 1); internal to the library.
int iht_threshold_batched_mu(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                             const float* g, float mu, const float* mu_dev, int32_t s, int64_t N, int64_t col_offset,
                             int32_t nrhs, int32_t* out_idx, float* out_val, int32_t ldo, int32_t* out_nnz, void* ws,
                             int64_t ws_bytes, void* stream);
// Kernel launches one iht_threshold_batched call makes for N columns (fused cluster path: 1).
int iht_threshold_launches(int64_t N);
// Solver-internal split of iht_adjoint (variant 0): with nK > 1 K-ranges it leaves the
// unscaled partials part[nK][N] in ws and skips adjoint_reduce_kernel; *nparts = nK (0 when
// g was written directly), *gsigma = sigma.  The fused threshold then forms
// g = sigma (part_0 + ... + part_{nK-1}) itself, in the reduce kernel's order and rounding.
int iht_adjoint_parts(const iht_qmat* A, const float* r, float* g, void* ws, int64_t ws_bytes, void* stream,
                      int* nparts, float* gsigma);
// iht_threshold_batched_mu (nrhs = 1, fused path only) reading g as nparts partial planes
// (stride N) scaled by gsigma, also storing that g into gout (may be NULL); nparts = 0 is
// the plain call.
int iht_threshold_parts(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                        const float* g, int nparts, float gsigma, float* gout, float mu, int32_t s, int64_t N,
                        int32_t* out_idx, float* out_val, int32_t ldo, int32_t* out_nnz, void* ws, int64_t ws_bytes,
                        void* stream);
// Bounded select (batched solver, fixed step, cluster-sized N): thr_bounded_select on the
// candidate lists the tcgen05 adjoint's epilogue wrote (iht_adjoint_batched_cand); a snapshot
// the list cannot decide (done[b] = 0) is selected over all of a by the same CTA, in the
// workspace's a buffers (ws: iht_threshold_batched_ws_bytes(N, s, nrhs)).  stats (may be NULL):
// [0] decided, [1] fallen back, [2] sum of list sizes, [3] max list size.
int iht_threshold_bounded(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                          const float* g, float mu, const unsigned int* bkey, int32_t s, int64_t N, int32_t nrhs,
                          const int32_t* cidx, const float* cval, int* ccnt, int32_t ccap, int* done, int* stats,
                          int32_t* out_idx, float* out_val, int32_t ldo, int32_t* out_nnz, void* ws, int64_t ws_bytes,
                          void* stream);
bool iht_threshold_bounded_applies(int64_t N, int32_t s, int32_t nrhs);
// Epilogue candidate lists for iht_threshold_bounded (x = x^[n] of every snapshot, [nrhs][ldx]).
struct iht_cand_args {
  int32_t* cidx;
  float* cval;
  int* ccnt;
  int32_t ccap;
  float mu, bound;
  const float* x_val;
  const int32_t* x_nnz;
  int32_t ldx, max_nnz;
  unsigned int* bkey;   // [nrhs] bound keys written by the limb kernel, read by the epilogue and the select
};
int iht_adjoint_batched_cand(const iht_qmat* A, const float* R, int32_t nrhs, float* G, void* ws, int64_t ws_bytes,
                             void* stream, const iht_cand_args* cand);

// Fused small-problem solver (iht_fused.cu): the whole fixed-step Algorithm 1 loop as one
// persistent cooperative kernel.  create returns IHT_EUNSUPPORTED when the problem does not
// fit (then the solver keeps its per-step kernels).
struct iht_fused_state;
int iht_fused_create(const iht_qmat* pool, int K, int s, int n_iter, float mu, int trace, const float* yhat,
                     float* r, float* g, int32_t* xs_idx, float* xs_val, int32_t* xs_nnz, iht_fused_state** out);
int iht_fused_enqueue(iht_fused_state* S, void* stream);
void iht_fused_destroy(iht_fused_state* S);

namespace iht {

constexpr int kNumSMs = 148;  // B200; launch code queries the device, this is a default

__host__ __device__ inline int num_levels(int bits, int level_mode) {
  return level_mode == 0 ? (1 << bits) : ((1 << (bits - 1)) + 1);
}

// Universal row padding: a multiple of 256 rows, so that every plane segment is a whole
// number of 32-byte sectors (256/b rows) and of adjoint k-steps (512/b rows) for b >= 2.
__host__ __device__ inline int64_t rows_pad(int64_t rows) { return (rows + 255) / 256 * 256; }

// Tiled column-strip layout (iht.h): byte k of column n's logical strip.
__host__ __device__ inline int64_t tiled_offset(int64_t n, int64_t k, int64_t strip_bytes) {
  return (n >> 4) * (16 * strip_bytes) + (k >> 6) * 1024 + (n & 15) * 64 + (k & 63);
}

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based RNG of the Q-contract (reading c4); own implementation.
struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Q-contract rounding of one fp32 component (no FMA contraction: _rn intrinsics).
__device__ __forceinline__ uint32_t q_contract(float v, float c, float sf, int L, uint32_t w) {
  float t = __fmul_rn(__fadd_rn(v, c), sf);
  t = fminf(fmaxf(t, 0.0f), (float)(L - 1));
  const int i = __float2int_rd(t);
  if (i >= L - 1) return (uint32_t)(L - 1);
  const float p = __fsub_rn(t, (float)i);
  const float u = __fmul_rn(__uint2float_rn(w >> 8), 5.9604644775390625e-08f);  // 2^-24
  return (uint32_t)i + (u < p ? 1u : 0u);
}

// sf = fl32(fl32(L-1) / fl32(2c)), 0 when c == 0.
__device__ __forceinline__ float q_scale_factor(float c, int L) {
  return c == 0.0f ? 0.0f : __fdiv_rn((float)(L - 1), __fmul_rn(2.0f, c));
}

// ---------------------------------------------------- programmatic dependent launch
// The solver's kernels are launched with programmatic stream serialization: a kernel lets
// the next grid begin launching as soon as it starts (pdl_launch_dependents) and waits for
// its predecessor's completion and memory only where it first reads the predecessor's
// outputs (pdl_wait) -- the launch latency and the setup before that point overlap the
// predecessor.  Both are no-ops when the kernel was not launched that way.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// (a & m) | e in one LOP3 (m, e in registers; the compiler would otherwise split the two
// immediates into two instructions)
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t m, uint32_t e) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(m), "r"(e));
  return d;
}

// Bound key of the bounded candidate select (config 5; batched_limbs_kernel writes it, the
// tcgen05 epilogue lists against it, thr_bounded_select decides with it): the key (|.| bit
// pattern) of bound x m, m = min_j |x_j| over x's support as a key, or 0xFFFFFFFF (no
// candidates: the select falls back to the full path) when x is empty or poisoned or the
// bound underflows.
__device__ __forceinline__ unsigned int bound_key(unsigned int m, int nnz, float bound) {
  if (nnz <= 0 || m >= 0x7F800000u) return 0xFFFFFFFFu;
  const unsigned int k = __float_as_uint(__fmul_rn(bound, __uint_as_float(m))) & 0x7FFFFFFFu;
  return k == 0u ? 0xFFFFFFFFu : k;
}

__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

template <typename T>
__host__ __device__ inline T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

}  // namespace iht
