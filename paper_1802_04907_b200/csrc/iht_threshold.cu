// (a6) fused update a = x + mu g and hard threshold x <- H_s(a).
//
// P:351 (x^{[n+1]} = H_s(x^{[n]} + mu g^{[n]})), H_s "preserving only the largest s
// entries ... in magnitude".  Ties go to the lowest index and zeros are
// never kept (reading c15); the support is written in increasing
// index order.  The paper's FPGA finds "the threshold value satisfying that
// only top S values are larger than the threshold" by binary search; here the
// threshold is found exactly by a radix select on the IEEE bit patterns of |a| (which
// order like the magnitudes): 11 + 11 + 9 bits, three histogram passes, then an
// ordered compaction that takes every key > T and the lowest-indexed ties == T.
//
// v0: one CTA of 1024 threads (N <= a few 10^5 makes this a few microseconds of L2
// traffic).  a is materialised once in the workspace.
#include "iht_internal.cuh"

namespace iht {

constexpr int kThrThreads = 1024;
constexpr int kThrWarps = kThrThreads / 32;

// Block-wide: given hist[0..nbins), find the largest bin d with sum_{b>=d} hist[b] >= target.
// Writes d, and the count strictly above d, into *d_out, *above_out.  target >= 1.
__device__ void find_bin(const int* hist, int nbins, int target, int* d_out, int* above_out,
                         int* scratch /* kThrWarps ints */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bpt = (nbins + kThrThreads - 1) / kThrThreads;
  // thread rt = kThrThreads-1-tid owns bins [tid*bpt, ...): scan order = descending bins
  int local = 0;
  for (int b = tid * bpt; b < min(nbins, (tid + 1) * bpt); ++b) local += hist[b];
  // inclusive suffix scan over tid (higher tid = higher bins first): reverse-index prefix
  const int rt = kThrThreads - 1 - tid;
  const int rlane = rt & 31, rwarp = rt >> 5;
  // warp-level inclusive scan along rlane: lanes of warp `warp` map to rwarp = 31 - warp
  int v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    // partner with smaller rlane = larger lane
    const int n = __shfl_down_sync(0xffffffffu, v, o);
    if (rlane >= o) v += n;
  }
  if (rlane == 31) scratch[rwarp] = v;   // lane 0 of the warp holds the warp total
  __syncthreads();
  int before = 0;
  for (int w = 0; w < rwarp; ++w) before += scratch[w];
  const int incl = before + v;          // sum over bins >= this thread's first bin
  const int excl = incl - local;        // sum over bins above this thread's range
  if (excl < target && incl >= target) {
    int acc = excl;
    for (int b = min(nbins, (tid + 1) * bpt) - 1; b >= tid * bpt; --b) {
      if (acc + hist[b] >= target) {
        *d_out = b;
        *above_out = acc;
        break;
      }
      acc += hist[b];
    }
  }
  (void)lane;
  __syncthreads();
}

__global__ void __launch_bounds__(kThrThreads, 1) threshold_kernel(
    const int32_t* __restrict__ x_idx, const float* __restrict__ x_val, const int32_t* __restrict__ x_nnz,
    int32_t max_nnz, const float* __restrict__ g, float mu, int s, int64_t N, float* __restrict__ a,
    int32_t* __restrict__ out_idx, float* __restrict__ out_val, int32_t* __restrict__ out_nnz) {
  __shared__ int hist[2048];
  __shared__ int scratch[kThrWarps];
  __shared__ int wgt[kThrWarps], weq[kThrWarps], wtake[kThrWarps], wbase[kThrWarps];
  __shared__ int sh_d, sh_above, sh_nan, sh_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- a = x + mu g --------------------------------------------------------------------
  int nnz = *x_nnz;
  if (nnz < 0) {                 // poisoned input (earlier non-finite a): stays poisoned
    if (tid == 0) *out_nnz = -1;
    return;
  }
  nnz = min(nnz, max_nnz);
  for (int64_t n = tid; n < N; n += kThrThreads) a[n] = __fmul_rn(mu, g[n]);
  if (tid == 0) sh_nan = 0;
  __syncthreads();
  for (int j = tid; j < nnz; j += kThrThreads) {
    const int64_t n = x_idx[j];
    a[n] = __fadd_rn(x_val[j], a[n]);
  }
  __syncthreads();

  if (s == 0) {                  // H_0 keeps nothing
    if (tid == 0) *out_nnz = 0;
    return;
  }

  // ---- radix select of the s-th largest key --------------------------------------------
  unsigned int T = 0;        // threshold key
  int need = 0;              // ties at T to take
  const bool all = (int64_t)s >= N;
  if (!all && s > 0) {
    unsigned int prefix = 0;
    int target = s;
    int above_total = 0;
    const int shifts[3] = {20, 9, 0};
    const int widths[3] = {11, 11, 9};
    for (int pass = 0; pass < 3; ++pass) {
      const int nb = 1 << widths[pass];
      for (int b = tid; b < nb; b += kThrThreads) hist[b] = 0;
      __syncthreads();
      const int sh = shifts[pass];
      const unsigned int hi_shift = sh + widths[pass];   // bits above this digit must match prefix
      for (int64_t n = tid; n < N; n += kThrThreads) {
        const unsigned int key = __float_as_uint(a[n]) & 0x7FFFFFFFu;
        if (pass == 0 && key > 0x7F800000u) sh_nan = 1;
        if (hi_shift >= 31 || (key >> hi_shift) == (prefix >> hi_shift))
          atomicAdd(&hist[(key >> sh) & (nb - 1)], 1);
      }
      __syncthreads();
      find_bin(hist, nb, target, &sh_d, &sh_above, scratch);
      prefix |= (unsigned int)sh_d << sh;
      above_total += sh_above;
      target -= sh_above;
      __syncthreads();
    }
    T = prefix;
    need = target;             // keys == T to take (>= 1)
    (void)above_total;
  }

  // ---- ordered compaction --------------------------------------------------------------
  const int64_t span = ((N + kThrWarps - 1) / kThrWarps + 31) / 32 * 32;
  const int64_t lo = (int64_t)warp * span, hi = min64(N, lo + span);
  int gt = 0, eq = 0;
  for (int64_t n0 = lo; n0 < hi; n0 += 32) {
    const int64_t n = n0 + lane;
    const unsigned int key = n < hi ? (__float_as_uint(a[n]) & 0x7FFFFFFFu) : 0u;
    const bool live = n < hi && key > 0u;
    gt += __popc(__ballot_sync(0xffffffffu, live && (all || key > T)));
    eq += __popc(__ballot_sync(0xffffffffu, live && !all && key == T));
  }
  if (lane == 0) {
    wgt[warp] = gt;
    weq[warp] = eq;
  }
  __syncthreads();
  if (tid == 0) {
    int eq_before = 0, base = 0;
    for (int w = 0; w < kThrWarps; ++w) {
      const int tk = (all || T == 0u) ? 0 : max(0, min(weq[w], need - eq_before));
      eq_before += weq[w];
      wtake[w] = tk;
      wbase[w] = base;
      base += wgt[w] + tk;
    }
    sh_total = base;
  }
  __syncthreads();
  int run_sel = 0, run_eq = 0;
  const unsigned int lt = (1u << lane) - 1u;
  const int take = wtake[warp], base = wbase[warp];
  for (int64_t n0 = lo; n0 < hi; n0 += 32) {
    const int64_t n = n0 + lane;
    const float av = n < hi ? a[n] : 0.0f;
    const unsigned int key = __float_as_uint(av) & 0x7FFFFFFFu;
    const bool live = n < hi && key > 0u;
    const bool is_gt = live && (all || key > T);
    const bool is_eq = live && !all && key == T;
    const unsigned int beq = __ballot_sync(0xffffffffu, is_eq);
    const bool tk = is_eq && (run_eq + __popc(beq & lt)) < take;
    const bool sel = is_gt || tk;
    const unsigned int bsel = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int pos = base + run_sel + __popc(bsel & lt);
      out_idx[pos] = (int32_t)n;
      out_val[pos] = av;
    }
    run_sel += __popc(bsel);
    run_eq += __popc(beq);
  }
  if (tid == 0) *out_nnz = sh_nan ? -1 : sh_total;
}

}  // namespace iht

using namespace iht;

extern "C" int64_t iht_threshold_ws_bytes(int64_t N, int32_t s) {
  (void)s;
  return N * (int64_t)sizeof(float);
}

extern "C" int iht_threshold(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz,
                             const float* g, float mu, int32_t s, int64_t N, int32_t* out_idx,
                             float* out_val, int32_t* out_nnz, void* ws, int64_t ws_bytes,
                             void* stream) {
  if (x_nnz == nullptr || g == nullptr || out_idx == nullptr || out_val == nullptr ||
      out_nnz == nullptr || s < 0 || N <= 0 || N > 0x7FFFFFFFll)
    return IHT_EINVAL;
  if (ws == nullptr || ws_bytes < N * (int64_t)sizeof(float)) return IHT_EINVAL;
  if (!isfinite(mu)) return IHT_EDOMAIN;
  cudaStream_t st = (cudaStream_t)stream;
  // max_nnz: the caller's x arrays hold at most s entries (x is an H_s output)
  threshold_kernel<<<1, kThrThreads, 0, st>>>(x_idx, x_val, x_nnz, s, g, mu, s, N,
                                              static_cast<float*>(ws), out_idx, out_val, out_nnz);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
