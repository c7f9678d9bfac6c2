// Block-wide exact selection helpers shared by the threshold kernels (iht_threshold.cu)
// and the fused small-problem solver (iht_fused.cu): H_s on IEEE bit patterns of
// |a|, ties to the lowest index, zeros never kept (reading c15).  Internal, not ABI.
#pragma once
#include "iht_internal.cuh"

namespace iht {

constexpr int kThrThreads = 1024;
constexpr int kThrWarps = kThrThreads / 32;

// Block-wide: given hist[0..nbins), find the largest bin d with sum_{b>=d} hist[b] >= target.
// Writes d, and the count strictly above d, into *d_out, *above_out.  target >= 1.
template <int NT = kThrThreads>
__device__ void find_bin(const int* hist, int nbins, int target, int* d_out, int* above_out,
                         int* scratch /* NT / 32 ints */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bpt = (nbins + NT - 1) / NT;
  // thread rt = kThrThreads-1-tid owns bins [tid*bpt, ...): scan order = descending bins
  int local = 0;
  for (int b = tid * bpt; b < min(nbins, (tid + 1) * bpt); ++b) local += hist[b];
  // inclusive suffix scan over tid (higher tid = higher bins first): reverse-index prefix
  const int rt = NT - 1 - tid;
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

// Exact top-s of the n entries (idx(i), val(i)), i = 0..n-1, listed in increasing index
// order: radix select of the s-th largest key, then ordered compaction (ties -> lowest
// index, zeros never kept).  All 1024 threads of the CTA call it.  Writes out_*;
// returns nothing; *out_nnz = total (or -1 when nan_flag).
template <int NT = kThrThreads, class Val, class Idx>
__device__ void select_ordered(int n, int s, Val val, Idx idx, int32_t* __restrict__ out_idx,
                               float* __restrict__ out_val, int32_t* __restrict__ out_nnz, int nan_flag,
                               int* hist, int* scratch, int* wgt, int* weq, int* wtake, int* wbase, int* sh) {
  constexpr int kThrThreads = NT, kThrWarps = NT / 32;   // shadow: all NT threads of the CTA call it
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned int T = 0;
  int need = 0;
  const bool all = s >= n;
  if (!all) {
    unsigned int prefix = 0;
    int target = s;
    const int shifts[3] = {20, 9, 0};
    const int widths[3] = {11, 11, 9};
    for (int pass = 0; pass < 3; ++pass) {
      const int nb = 1 << widths[pass];
      for (int b = tid; b < nb; b += kThrThreads) hist[b] = 0;
      __syncthreads();
      const int sh_ = shifts[pass];
      const unsigned int hi_shift = sh_ + widths[pass];
      for (int i = tid; i < n; i += kThrThreads) {
        const unsigned int key = __float_as_uint(val(i)) & 0x7FFFFFFFu;
        if (hi_shift >= 31 || (key >> hi_shift) == (prefix >> hi_shift))
          atomicAdd(&hist[(key >> sh_) & (nb - 1)], 1);
      }
      __syncthreads();
      find_bin<NT>(hist, nb, target, &sh[0], &sh[1], scratch);
      prefix |= (unsigned int)sh[0] << sh_;
      target -= sh[1];
      __syncthreads();
    }
    T = prefix;
    need = target;
  }
  // ordered compaction: warp w owns the contiguous range [lo, hi) of the list
  const int span = ((n + kThrWarps - 1) / kThrWarps + 31) / 32 * 32;
  const int lo = warp * span, hi = min(n, lo + span);
  int gt = 0, eq = 0;
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const int i = i0 + lane;
    const unsigned int key = i < hi ? (__float_as_uint(val(i)) & 0x7FFFFFFFu) : 0u;
    const bool live = i < hi && key > 0u;
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
    sh[2] = base;
  }
  __syncthreads();
  int run_sel = 0, run_eq = 0;
  const unsigned int lt = (1u << lane) - 1u;
  const int take = wtake[warp], base = wbase[warp];
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const int i = i0 + lane;
    const float av = i < hi ? val(i) : 0.0f;
    const unsigned int key = __float_as_uint(av) & 0x7FFFFFFFu;
    const bool live = i < hi && key > 0u;
    const bool is_gt = live && (all || key > T);
    const bool is_eq = live && !all && key == T;
    const unsigned int beq = __ballot_sync(0xffffffffu, is_eq);
    const bool tk = is_eq && (run_eq + __popc(beq & lt)) < take;
    const bool sel = is_gt || tk;
    const unsigned int bsel = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int pos = base + run_sel + __popc(bsel & lt);
      out_idx[pos] = (int32_t)idx(i);
      out_val[pos] = av;
    }
    run_sel += __popc(bsel);
    run_eq += __popc(beq);
  }
  if (tid == 0) *out_nnz = nan_flag ? -1 : sh[2];
}

}  // namespace iht
