// NEXT-1: the adaptive step of Algorithm 1 "QNIHT", device side.
//
//   mu   = |g_G|^2 / |Phi-hat_A[:, G] g_G|^2            (reading c10: Phi-hat_A)
//   x'   = H_s(x + mu g)
//   if supp(x') != G:  b = |x' - x|^2 / |Phi-hat_A (x' - x)|^2,
//        while mu > (1 - c) b: mu <- mu / (k (1 - c)), x' = H_s(x + mu g)   (c11)
//
// The products Phi-hat_A[:, G] g_G and Phi-hat_A (x' - x) are sparse forward products
// (iht_forward_batched with y-hat = NULL, <= s and <= 2s columns); the kernels here
// gather g on the support, build the sparse difference x' - x, reduce squared norms in
// a fixed order (deterministic) and take the accept / shrink decisions per snapshot.  The
// solver runs the shrink loop as a CUDA-graph conditional WHILE node whose condition the
// decide kernel sets (cudaGraphSetConditional).
#include "iht_adaptive.cuh"

namespace iht {

constexpr int kAdThreads = 256;

// Block-wide sum in a fixed order (deterministic): per-thread strided partials, then a
// shared-memory tree.  All threads receive the result.
__device__ float block_sum(float v, float* red) {
  const int tid = threadIdx.x;
  red[tid] = v;
  __syncthreads();
  for (int o = kAdThreads / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] = __fadd_rn(red[tid], red[tid + o]);
    __syncthreads();
  }
  const float r = red[0];
  __syncthreads();
  return r;
}

// xg = (G, g_G) and num = |g_G|^2 per snapshot (one CTA per snapshot).
__global__ void __launch_bounds__(kAdThreads) ad_gather_kernel(const float* __restrict__ g, int64_t N,
                                                                 int64_t col_offset, const int32_t* __restrict__ gi,
                                                                 const int32_t* __restrict__ gn, int ldg,
                                                                 int32_t* __restrict__ xi, float* __restrict__ xv,
                                                                 int32_t* __restrict__ xn, float* __restrict__ num) {
  __shared__ float red[kAdThreads];
  const int b = blockIdx.x;
  gi += (int64_t)b * ldg;
  xi += (int64_t)b * ldg;
  xv += (int64_t)b * ldg;
  g += (int64_t)b * N;
  int n = gn[b];
  n = n < 0 ? 0 : min(n, ldg);
  float acc = 0.0f;
  for (int j = threadIdx.x; j < n; j += kAdThreads) {
    const int64_t c = (int64_t)gi[j] - col_offset;
    const float v = (c >= 0 && c < N) ? g[c] : 0.0f;
    xi[j] = gi[j];
    xv[j] = v;
    acc = __fmaf_rn(v, v, acc);
  }
  const float t = block_sum(acc, red);
  if (threadIdx.x == 0) {
    xn[b] = n;
    num[b] = t;
  }
}

// nrm[b] = |r_b|^2 over a stacked vector (one CTA per snapshot, fixed order).
__global__ void __launch_bounds__(kAdThreads) ad_norm_kernel(const float* __restrict__ r, int64_t vlen,
                                                               float* __restrict__ nrm) {
  __shared__ float red[kAdThreads];
  const int b = blockIdx.x;
  r += (int64_t)b * vlen;
  float acc = 0.0f;
  for (int64_t i = threadIdx.x; i < vlen; i += kAdThreads) acc = __fmaf_rn(r[i], r[i], acc);
  const float t = block_sum(acc, red);
  if (threadIdx.x == 0) nrm[b] = t;
}

// mu_b = num_b / den_b (fallback when the denominator vanishes); resets the loop state.
__global__ void ad_step_kernel(const float* __restrict__ num, const float* __restrict__ den, float fallback, int B,
                               float* __restrict__ mu, int32_t* __restrict__ state) {
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const float d = den[b];
    mu[b] = (d > 0.0f && num[b] > 0.0f) ? __fdiv_rn(num[b], d) : fallback;
    state[2 * b] = 0;       // accepted
    state[2 * b + 1] = 0;   // shrinks
  }
}

// Proposal x' (pi, pv, pn) against the current support G (gi, gn) and the current x (xi,
// xv, xn).  Unchanged support (or an already accepted snapshot): accept, empty delta.
// Otherwise the delta x' - x as a duplicate-free sparse list: x' entries (minus x where the
// index is shared), then x entries absent from x' (negated), and dnum = |x' - x|^2.
__global__ void __launch_bounds__(kAdThreads) ad_delta_kernel(
    const int32_t* __restrict__ pi, const float* __restrict__ pv, const int32_t* __restrict__ pn,
    const int32_t* __restrict__ gi, const int32_t* __restrict__ gn, int ldg,
    const int32_t* __restrict__ xi, const float* __restrict__ xv, const int32_t* __restrict__ xn, int s,
    int32_t* __restrict__ state, int32_t* __restrict__ di, float* __restrict__ dv, int32_t* __restrict__ dn,
    float* __restrict__ dnum) {
  __shared__ float red[kAdThreads];
  __shared__ int flag, cnt;
  const int b = blockIdx.x, tid = threadIdx.x;
  pi += (int64_t)b * s;
  pv += (int64_t)b * s;
  gi += (int64_t)b * ldg;
  xi += (int64_t)b * s;
  xv += (int64_t)b * s;
  di += (int64_t)b * 2 * s;
  dv += (int64_t)b * 2 * s;
  const int np = max(0, pn[b]), ng = max(0, min(gn[b], ldg)), nx = max(0, xn[b]);
  if (tid == 0) flag = (np == ng) ? 1 : 0;
  __syncthreads();
  for (int j = tid; j < np && j < ng; j += kAdThreads)
    if (pi[j] != gi[j]) flag = 0;     // benign race: every writer stores 0
  __syncthreads();
  if (state[2 * b] || flag || pn[b] < 0) {
    if (tid == 0) {
      state[2 * b] = 1;
      dn[b] = 0;
      dnum[b] = 0.0f;
    }
    return;
  }
  // part 1: x' entries at [0, np)
  float acc = 0.0f;
  for (int j = tid; j < np; j += kAdThreads) {
    const int32_t idx = pi[j];
    int lo = 0, hi = nx;                       // lower_bound in x's sorted support
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (xi[mid] < idx) lo = mid + 1; else hi = mid;
    }
    const float d = (lo < nx && xi[lo] == idx) ? __fsub_rn(pv[j], xv[lo]) : pv[j];
    di[j] = idx;
    dv[j] = d;
    acc = __fmaf_rn(d, d, acc);
  }
  // part 2: x entries absent from x', appended in order (serial compaction by chunks of
  // kAdThreads with a block-wide exclusive scan)
  if (tid == 0) cnt = np;
  __syncthreads();
  for (int j0 = 0; j0 < nx; j0 += kAdThreads) {
    const int j = j0 + tid;
    bool absent = false;
    int32_t idx = 0;
    if (j < nx) {
      idx = xi[j];
      int lo = 0, hi = np;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pi[mid] < idx) lo = mid + 1; else hi = mid;
      }
      absent = !(lo < np && pi[lo] == idx);
    }
    // exclusive scan of `absent` over the block (warp ballots + serial warp prefix)
    const unsigned int bal = __ballot_sync(0xffffffffu, absent);
    const int lane = tid & 31, warp = tid >> 5;
    __shared__ int wcount[kAdThreads / 32];
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int before = cnt;
    for (int w = 0; w < warp; ++w) before += wcount[w];
    if (absent) {
      const int pos = before + __popc(bal & ((1u << lane) - 1u));
      const float d = -xv[j];
      di[pos] = idx;
      dv[pos] = d;
      acc = __fmaf_rn(d, d, acc);
    }
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < kAdThreads / 32; ++w) t += wcount[w];
      cnt += t;
    }
    __syncthreads();
  }
  const float t = block_sum(acc, red);
  if (tid == 0) {
    dn[b] = cnt;
    dnum[b] = t;
  }
}

// Accept when mu <= (1 - c) b, b = dnum / dden (or when the delta vanishes); otherwise
// shrink mu by k (1 - c) and ask for another proposal.  Records mu / shrinks (trace) and
// sets the WHILE condition: 1 while any snapshot is pending.
__global__ void ad_decide_kernel(const float* __restrict__ dnum, const float* __restrict__ dden, float c, float k,
                                 int max_shrink, int B, float* __restrict__ mu, int32_t* __restrict__ state,
                                 float* __restrict__ mu_rec, int32_t* __restrict__ shr_rec,
                                 cudaGraphConditionalHandle handle, int use_handle, int32_t* __restrict__ pending) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (!state[2 * b]) {
      const float nd = dnum[b], dd = dden[b];
      bool ok = nd == 0.0f || dd == 0.0f;
      if (!ok) ok = mu[b] <= __fmul_rn(1.0f - c, __fdiv_rn(nd, dd));
      if (!ok && state[2 * b + 1] >= max_shrink) ok = true;      // bounded loop: keep the last proposal
      if (ok) {
        state[2 * b] = 1;
      } else {
        mu[b] = __fdiv_rn(mu[b], __fmul_rn(k, 1.0f - c));
        state[2 * b + 1] += 1;
        atomicOr(&any, 1);
      }
    }
    if (mu_rec) mu_rec[b] = mu[b];
    if (shr_rec) shr_rec[b] = state[2 * b + 1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (use_handle) cudaGraphSetConditional(handle, any ? 1u : 0u);
    if (pending) *pending = any;
  }
}

}  // namespace iht

using namespace iht;

int ad_gather(const float* g, int64_t N, int64_t col_offset, const int32_t* gi, const int32_t* gn, int ldg,
              int32_t* xi, float* xv, int32_t* xn, float* num, int B, cudaStream_t st) {
  ad_gather_kernel<<<B, kAdThreads, 0, st>>>(g, N, col_offset, gi, gn, ldg, xi, xv, xn, num);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}

int ad_norm(const float* r, int64_t vlen, float* nrm, int B, cudaStream_t st) {
  ad_norm_kernel<<<B, kAdThreads, 0, st>>>(r, vlen, nrm);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}

int ad_step(const float* num, const float* den, float fallback, int B, float* mu, int32_t* state, cudaStream_t st) {
  ad_step_kernel<<<1, 256, 0, st>>>(num, den, fallback, B, mu, state);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}

int ad_delta(const int32_t* pi, const float* pv, const int32_t* pn, const int32_t* gi, const int32_t* gn, int ldg,
             const int32_t* xi, const float* xv, const int32_t* xn, int s, int32_t* state, int32_t* di, float* dv,
             int32_t* dn, float* dnum, int B, cudaStream_t st) {
  ad_delta_kernel<<<B, kAdThreads, 0, st>>>(pi, pv, pn, gi, gn, ldg, xi, xv, xn, s, state, di, dv, dn, dnum);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}

int ad_decide(const float* dnum, const float* dden, float c, float k, int max_shrink, int B, float* mu, int32_t* state,
              float* mu_rec, int32_t* shr_rec, cudaGraphConditionalHandle handle, int use_handle, int32_t* pending,
              cudaStream_t st) {
  ad_decide_kernel<<<1, 256, 0, st>>>(dnum, dden, c, k, max_shrink, B, mu, state, mu_rec, shr_rec, handle, use_handle,
                                      pending);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
