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
// Three launches (all deterministic; integer atomics only):
//   T1 thr_update_hist  (grid, 2048 entries per CTA): a = x + mu g into the workspace,
//                        histogram of the top 11 key bits (global, int atomics)
//   T2 thr_candidates   (grid): every CTA finds the same bin d1 holding the s-th largest
//                        key and compacts, in index order, its entries with digit >= d1
//                        into its own slot of the candidate buffer
//   T3 thr_select       (1 CTA): gathers the candidates (a few thousand, index order) into
//                        shared memory, finishes the radix select on them and writes the
//                        ordered support.  If the candidates do not fit (massive ties,
//                        mostly-zero a) it falls back to the full single-CTA select over a.
// Batched (config 5): grid row blockIdx.y (T3: blockIdx.x) = snapshot b, each with its own
// x_b, g_b, workspace slice and output; a column shard adds col_offset to every index.
// iht_merge_candidates (T4, 1 CTA per snapshot) merges the shards' local top-s lists.
//
// Fused path (default when N <= kClusterMaxN): ONE launch, a thread-block cluster of CL
// CTAs per snapshot.  Each CTA holds its slice of a = x + mu g in shared memory; the three
// radix passes build local histograms that every CTA sums over the cluster through
// distributed shared memory (DSMEM), so all CTAs agree on the threshold key T; the ordered
// compaction takes per-CTA (greater, equal) counts, an exclusive scan over the cluster
// gives each CTA its output offset and its share of the lowest-index ties.  No global
// atomics, no workspace memset, no candidate-capacity limit.
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include "iht_internal.cuh"
#include "iht_select.cuh"

namespace cg = cooperative_groups;

namespace iht {

// ---------------------------------------------------------------------------- workspace
constexpr int kTile = 2048;            // entries per CTA in T1 / T2
constexpr int kTileThreads = 256;
constexpr int kCandCap = 8192;         // candidates T3 keeps in shared memory
constexpr int kHistBins = 2048;

struct ThrWs {
  float* a;          // [N]
  int32_t* cidx;     // [N] per-tile candidate slots
  float* cval;       // [N]
  int* ccount;       // [ntiles]
  int* hist;         // [kHistBins] global histogram of digit 1
  int* flags;        // [0] nan
  int64_t hdr_stride, body_stride;   // bytes between consecutive snapshots' slices
};

// Workspace: [nrhs] headers (hist + flags, zeroed by one memset), then [nrhs] bodies.
__host__ __device__ inline int64_t al256(int64_t b) { return (b + 255) / 256 * 256; }
__host__ __device__ inline int64_t thr_hdr_bytes() { return al256(kHistBins * 4) + al256(16); }
__host__ __device__ inline int64_t thr_body_bytes(int64_t N) {
  const int64_t ntiles = (N + kTile - 1) / kTile;
  return 3 * al256(N * 4) + al256(ntiles * 4);
}
__host__ __device__ inline int64_t thr_ws_layout(int64_t N, int nrhs, char* base, ThrWs* w) {
  const int64_t hdr = thr_hdr_bytes(), body = thr_body_bytes(N);
  if (w) {
    w->hist = reinterpret_cast<int*>(base);
    w->flags = reinterpret_cast<int*>(base + al256(kHistBins * 4));
    char* b0 = base + nrhs * hdr;
    w->a = reinterpret_cast<float*>(b0);
    w->cidx = reinterpret_cast<int32_t*>(b0 + al256(N * 4));
    w->cval = reinterpret_cast<float*>(b0 + 2 * al256(N * 4));
    w->ccount = reinterpret_cast<int*>(b0 + 3 * al256(N * 4));
    w->hdr_stride = hdr;
    w->body_stride = body;
  }
  return nrhs * (hdr + body);
}

// Slice of snapshot b.
__device__ __forceinline__ ThrWs thr_at(const ThrWs& w, int b) {
  ThrWs o = w;
  auto adv = [](auto* p, int64_t bytes) { return reinterpret_cast<decltype(p)>(reinterpret_cast<char*>(p) + bytes); };
  o.hist = adv(w.hist, b * w.hdr_stride);
  o.flags = adv(w.flags, b * w.hdr_stride);
  o.a = adv(w.a, b * w.body_stride);
  o.cidx = adv(w.cidx, b * w.body_stride);
  o.cval = adv(w.cval, b * w.body_stride);
  o.ccount = adv(w.ccount, b * w.body_stride);
  return o;
}

// T1: a = x + mu g (g possibly the sum of split-K partials), the CTA's 2048-bin histogram of
// the top 11 key bits in shared memory, then one global atomic per nonzero bin.  The global
// histogram is zero on entry (zeroed by T3 of the previous call, or by the memset of a cold
// workspace).
__global__ void __launch_bounds__(kTileThreads) thr_update_hist(
    const int32_t* __restrict__ x_idx, const float* __restrict__ x_val, const int32_t* __restrict__ x_nnz,
    int32_t max_nnz, int32_t ldx, const float* __restrict__ g, float mu, const float* __restrict__ mu_dev,
    int64_t N, int64_t col_offset, ThrWs w0, int nparts, float gsigma, float* __restrict__ gout) {
  __shared__ float as[kTile];
  __shared__ int hist[kHistBins];
  pdl_launch_dependents();
  const int tid = threadIdx.x;
  for (int b = tid; b < kHistBins; b += kTileThreads) hist[b] = 0;
  pdl_wait();                                   // g (adjoint) and x (previous H_s)
  const int bq = blockIdx.y;
  if (mu_dev) mu = mu_dev[bq];
  const ThrWs w = thr_at(w0, bq);
  x_idx += (int64_t)bq * ldx;
  x_val += (int64_t)bq * ldx;
  x_nnz += bq;
  g += (int64_t)bq * N;
  const int64_t start = (int64_t)blockIdx.x * kTile;
  const int cnt = (int)min64(kTile, N - start);
  constexpr int PER = kTile / kTileThreads;     // 8 entries per thread, all loads in flight
  float gv[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kTileThreads;
    float v = 0.0f;
    if (i < cnt) {
      v = __ldg(g + start + i);
      for (int k = 1; k < nparts; ++k) v = __fadd_rn(v, __ldg(g + (int64_t)k * N + start + i));
      if (nparts > 0) v = __fmul_rn(gsigma, v);   // adjoint_reduce_kernel's order and rounding
    }
    gv[u] = v;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kTileThreads;
    if (i < cnt) {
      if (gout && nparts > 0) gout[start + i] = gv[u];
      as[i] = __fmul_rn(mu, gv[u]);
    }
  }
  int nnz = *x_nnz;
  nnz = nnz < 0 ? 0 : min(nnz, max_nnz);
  __syncthreads();
  for (int j = tid; j < nnz; j += kTileThreads) {
    const int64_t n = (int64_t)x_idx[j] - col_offset;   // local column (column shards)
    if (n >= start && n < start + cnt) as[n - start] = __fadd_rn(x_val[j], as[n - start]);
  }
  __syncthreads();
  int nan = 0;
  for (int i = tid; i < cnt; i += kTileThreads) {
    const float v = as[i];
    w.a[start + i] = v;
    const unsigned int key = __float_as_uint(v) & 0x7FFFFFFFu;
    nan |= key > 0x7F800000u;
    atomicAdd(&hist[key >> 20], 1);
  }
  nan = __syncthreads_or(nan);
  if (tid == 0 && nan) atomicOr(&w.flags[0], 1);
  for (int b = tid; b < kHistBins; b += kTileThreads)
    if (hist[b]) atomicAdd(&w.hist[b], hist[b]);
}

// T2: every CTA finds the bin d1 holding the s-th largest key in the global histogram (the
// same in all CTAs; CTA 0 records d1 and the count above it for T3) and writes its entries
// with digit >= d1 (key > 0) to its candidate slot in index order.
__global__ void __launch_bounds__(kTileThreads) thr_candidates(int s, int64_t N, int64_t col_offset, ThrWs w0) {
  __shared__ int hist[kHistBins];
  __shared__ int scratch[kTileThreads / 32], wcnt[kTileThreads / 32], sh[2];
  pdl_launch_dependents();
  pdl_wait();                                   // T1's histogram and a
  const ThrWs w = thr_at(w0, blockIdx.y);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    int hv[kHistBins / kTileThreads];
#pragma unroll
    for (int u = 0; u < kHistBins / kTileThreads; ++u) hv[u] = __ldcg(&w.hist[tid + u * kTileThreads]);
#pragma unroll
    for (int u = 0; u < kHistBins / kTileThreads; ++u) hist[tid + u * kTileThreads] = hv[u];
  }
  if (tid == 0) sh[0] = sh[1] = 0;
  __syncthreads();
  const bool all = (int64_t)s >= N;
  if (!all && s > 0) find_bin<kTileThreads>(hist, kHistBins, s, &sh[0], &sh[1], scratch);
  const unsigned int d1 = all ? 0u : (unsigned int)sh[0];
  if (blockIdx.x == 0 && tid == 0) {
    w.flags[1] = (int)d1;
    w.flags[2] = all ? 0 : sh[1];
  }
  const int64_t start = (int64_t)blockIdx.x * kTile;
  const int cnt = (int)min64(kTile, N - start);
  const int per_warp = kTile / (kTileThreads / 32);       // 256 contiguous entries per warp
  const int lo = warp * per_warp, hi = min(cnt, lo + per_warp);
  float v8[per_warp / 32];
#pragma unroll
  for (int u = 0; u < per_warp / 32; ++u) {
    const int i = lo + u * 32 + lane;
    v8[u] = i < hi ? __ldcg(&w.a[start + i]) : 0.0f;
  }
  int c = 0;
#pragma unroll
  for (int u = 0; u < per_warp / 32; ++u) {
    const int i = lo + u * 32 + lane;
    const unsigned int key = __float_as_uint(v8[u]) & 0x7FFFFFFFu;
    c += __popc(__ballot_sync(0xffffffffu, i < hi && key > 0u && (key >> 20) >= d1));
  }
  if (lane == 0) wcnt[warp] = c;
  __syncthreads();
  int base = 0;
  for (int q = 0; q < warp; ++q) base += wcnt[q];
  const unsigned int lt = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < per_warp / 32; ++u) {
    const int i = lo + u * 32 + lane;
    const float v = v8[u];
    const unsigned int key = __float_as_uint(v) & 0x7FFFFFFFu;
    const bool sel = i < hi && key > 0u && (key >> 20) >= d1;
    const unsigned int b = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int pos = base + __popc(b & lt);
      w.cidx[start + pos] = (int32_t)(col_offset + start + i);
      w.cval[start + pos] = v;
    }
    base += __popc(b);
  }
  if (tid == 0) {
    int tot = 0;
    for (int q = 0; q < kTileThreads / 32; ++q) tot += wcnt[q];
    w.ccount[blockIdx.x] = tot;
  }
}

// Exact top-s of `total` gathered candidates (cidx, cval in shared memory, increasing index
// order) that contain every key with digit >= d1 (the bin of the s-th largest key; `above` keys
// lie in higher bins): keys in bins above d1 are kept, the need = s - above remaining come from
// bin d1 through a second 11-bit histogram and a rank of the few keys of sub-bin d2; keys below
// d1 (a bounded superset) are dropped.  Ordered compaction into out_*.  All NT threads call it.
template <int NT>
__device__ void gathered_select(int total, const int32_t* cidx, const float* cval, unsigned char* keep, int* hist,
                                int* grp_k, int* gpos, unsigned int d1, int above, int s, bool all,
                                int32_t* __restrict__ out_idx, float* __restrict__ out_val,
                                int32_t* __restrict__ out_nnz, int* scratch, int* wgt, int* weq, int* wtake,
                                int* wbase, int* sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  for (int b = tid; b < 2048; b += NT) hist[b] = 0;
  __syncthreads();
  auto key_of = [&](int i) { return __float_as_uint(cval[i]) & 0x7FFFFFFFu; };
  if (all || total <= s) {
    for (int i = tid; i < total; i += NT) keep[i] = 1;
  } else {
    const int need = s - above;                 // >= 1
    // second level: 11-bit histogram of the bin-d1 keys (bits 19..9)
    for (int i = tid; i < total; i += NT) {
      const unsigned int k = key_of(i);
      keep[i] = (k >> 20) > d1;
      if ((k >> 20) == d1) atomicAdd(&hist[(k >> 9) & 2047], 1);
    }
    __syncthreads();
    find_bin<NT>(hist, 2048, need, &sh[0], &sh[1], scratch);
    const unsigned int d2 = (unsigned int)sh[0];
    const int need2 = need - sh[1];             // >= 1 keys to take from sub-bin d2
    const unsigned int pre = (d1 << 11) | d2;   // 22-bit prefix of the sub-bin
    // compact sub-bin d2 (index order); keep the keys above it
    int ng = 0;
    for (int i0 = 0; i0 < total; i0 += NT) {
      const int i = i0 + tid;
      const unsigned int k = i < total ? key_of(i) : 0u;
      const bool f = i < total && (k >> 9) == pre;
      if (i < total && (k >> 20) == d1 && ((k >> 9) & 2047) > d2) keep[i] = 1;
      const unsigned int bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wgt[warp] = __popc(bal);
      __syncthreads();
      int off = ng, tot = 0;
      for (int q = 0; q < NT / 32; ++q) {
        if (q < warp) off += wgt[q];
        tot += wgt[q];
      }
      if (f && off + __popc(bal & lt) < 1024) {
        grp_k[off + __popc(bal & lt)] = (int)k;
        gpos[off + __popc(bal & lt)] = i;  // reuse: list position of the group member
      }
      ng += tot;
      __syncthreads();
    }
    if (ng <= 1024) {
      for (int e = tid; e < ng; e += NT) {
        const unsigned int ke = (unsigned int)grp_k[e];
        int rk = 0;
        for (int f = 0; f < ng; ++f) {
          const unsigned int kf = (unsigned int)grp_k[f];
          rk += kf > ke || (kf == ke && f < e);
        }
        if (rk < need2) keep[gpos[e]] = 1;
      }
    } else {                                    // a crowded sub-bin: radix passes over the candidates
      __syncthreads();
      select_ordered<NT>(total, s, [&](int i) { return cval[i]; }, [&](int i) { return cidx[i]; }, out_idx, out_val,
                         out_nnz, 0, hist, scratch, wgt, weq, wtake, wbase, sh);
      return;
    }
  }
  __syncthreads();
  // ordered compaction of the kept candidates
  int base = 0;
  for (int i0 = 0; i0 < total; i0 += NT) {
    const int i = i0 + tid;
    const bool f = i < total && keep[i];
    const unsigned int bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wgt[warp] = __popc(bal);
    __syncthreads();
    int off = base, tot = 0;
    for (int q = 0; q < NT / 32; ++q) {
      if (q < warp) off += wgt[q];
      tot += wgt[q];
    }
    if (f) {
      out_idx[off + __popc(bal & lt)] = cidx[i];
      out_val[off + __popc(bal & lt)] = cval[i];
    }
    base += tot;
    __syncthreads();
  }
  if (tid == 0) *out_nnz = base;
}

// T3 (one CTA per snapshot): gather the candidates (index order), then the exact top-s.  Keys
// in bins above d1 (`above` < s of them) are all kept; the need = s - above remaining come from
// bin d1: a second 11-bit histogram over the bin-d1 keys finds the sub-bin d2 of the need-th
// largest, keys above it are kept, and the few keys of sub-bin d2 are ranked (greater key, or
// equal key at a lower index).  Ordered compaction writes the support.  Finally the global
// histogram and flags are zeroed for the next call.
__global__ void __launch_bounds__(kThrThreads, 1) thr_select(
    const int32_t* __restrict__ x_nnz, int s, int64_t N, int64_t col_offset, ThrWs w0,
    int32_t* __restrict__ out_idx, float* __restrict__ out_val, int32_t ldo, int32_t* __restrict__ out_nnz) {
  const int bq = blockIdx.x;
  const ThrWs w = thr_at(w0, bq);
  x_nnz += bq;
  out_idx += (int64_t)bq * ldo;
  out_val += (int64_t)bq * ldo;
  out_nnz += bq;
  extern __shared__ __align__(16) unsigned char dsm[];
  int32_t* cidx = reinterpret_cast<int32_t*>(dsm);
  float* cval = reinterpret_cast<float*>(dsm + kCandCap * 4);
  __shared__ int hist[2048];
  __shared__ int scratch[kThrWarps];
  __shared__ int wgt[kThrWarps], weq[kThrWarps], wtake[kThrWarps], wbase[kThrWarps];
  __shared__ int sh[8];
  __shared__ int tile_base[1025];
  __shared__ int grp_k[1024];                   // keys of sub-bin d2 (index order)
  __shared__ unsigned char keep[kCandCap];
  pdl_launch_dependents();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  pdl_wait();                                   // T2's candidates
  const int ntiles = (int)((N + kTile - 1) / kTile);
  auto finish = [&]() {                         // zero the histogram + flags for the next call
    __syncthreads();
    for (int b = tid; b < kHistBins; b += kThrThreads) w.hist[b] = 0;
    if (tid < 4) w.flags[tid] = 0;
  };
  const int poisoned = *x_nnz < 0, nan = __ldcg(&w.flags[0]);
  if (poisoned || nan || s == 0) {              // poisoned input / NaN -> domain error; H_0 keeps nothing
    if (tid == 0) *out_nnz = (poisoned || nan) ? -1 : 0;
    finish();
    return;
  }
  // tile offsets: block-wide exclusive scan of the per-tile counts (ntiles <= 1024)
  const int myc = tid < ntiles ? __ldcg(&w.ccount[tid]) : 0;
  int incl = myc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int q = 0; q < kThrWarps; ++q) {
      const int v = scratch[q];
      scratch[q] = acc;
      acc += v;
    }
    sh[3] = acc;
  }
  __syncthreads();
  if (tid < ntiles) tile_base[tid] = scratch[warp] + incl - myc;
  if (tid == 0) tile_base[ntiles] = sh[3];
  __syncthreads();
  const int total = sh[3];
  const unsigned int d1 = (unsigned int)__ldcg(&w.flags[1]);
  const int above = __ldcg(&w.flags[2]);
  const bool all = (int64_t)s >= N;
  if (total > kCandCap || ntiles > 1024) {      // massive ties: radix passes over a itself
    const float* a = w.a;
    const int c0 = (int)col_offset;
    select_ordered((int)N, s, [&](int i) { return __ldcg(&a[i]); }, [&](int i) { return c0 + i; }, out_idx, out_val,
                   out_nnz, 0, hist, scratch, wgt, weq, wtake, wbase, sh);
    finish();
    return;
  }
  // gather: candidate i of tile t at tile_base[t] + j (one per thread per round, tile by binary search)
  for (int i0 = 0; i0 < total; i0 += 2 * kThrThreads) {
    int32_t ci[2];
    float cv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * kThrThreads + tid;
      if (i < total) {
        int lo = 0, hi = ntiles;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (tile_base[mid] <= i) lo = mid; else hi = mid;
        }
        const int64_t src = (int64_t)lo * kTile + (i - tile_base[lo]);
        ci[u] = __ldcg(&w.cidx[src]);
        cv[u] = __ldcg(&w.cval[src]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * kThrThreads + tid;
      if (i < total) {
        cidx[i] = ci[u];
        cval[i] = cv[u];
      }
    }
  }
  gathered_select<kThrThreads>(total, cidx, cval, keep, hist, grp_k, tile_base, d1, above, s, all, out_idx, out_val,
                               out_nnz, scratch, wgt, weq, wtake, wbase, sh);
  finish();
}

// ---------------------------------------------------------------------------- one-launch grid path
// ONE cooperative launch over the tiles (replaces T1 - T3; all CTAs co-resident):
//   phase 1  CTA t forms a = x + mu g on its tile in shared memory (split-K partials summed in
//            adjoint_reduce_kernel's order), adds its 2048-bin histogram to the global one;
//   barrier  (arrival counter per snapshot, release / acquire);
//   phase 2  every CTA finds the same bin d1 of the s-th largest key in the global histogram
//            and writes its keys with digit >= d1 (from shared memory) to its candidate slot
//            in index order, then arrives on the counter again;
//   finish   the last CTA to arrive gathers the candidates and finishes the exact select
//            (gathered_select, as T3), then zeroes the histogram, flags and counter.
// Same arithmetic and output as T1 - T3 (H_s with the tie rule of reading c15), two launches
// and their PDL hand-offs fewer.
constexpr int kOpThreads = 512;
constexpr int kOpWarps = kOpThreads / 32;
constexpr int kOpMaxTiles = 1024;              // per-tile counts scanned in shared memory

__global__ void __launch_bounds__(kOpThreads, 1) thr_onepass(
    const int32_t* __restrict__ x_idx, const float* __restrict__ x_val, const int32_t* __restrict__ x_nnz,
    int32_t max_nnz, int32_t ldx, const float* __restrict__ g, float mu, const float* __restrict__ mu_dev, int s,
    int64_t N, int64_t col_offset, ThrWs w0, int nparts, float gsigma, float* __restrict__ gout,
    int32_t* __restrict__ out_idx, float* __restrict__ out_val, int32_t ldo, int32_t* __restrict__ out_nnz) {
  extern __shared__ __align__(16) unsigned char dsm[];   // last CTA: gathered candidates
  __shared__ float as[kTile];
  __shared__ int hist[kHistBins];
  __shared__ unsigned char keep[kCandCap];
  __shared__ int tile_base[kOpMaxTiles + 1];
  __shared__ int grp_k[1024];
  __shared__ int scratch[kOpWarps], wgt[kOpWarps], weq[kOpWarps], wtake[kOpWarps], wbase[kOpWarps], sh[8];
  __shared__ int s_last, s_stop;
  pdl_launch_dependents();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  for (int b = tid; b < kHistBins; b += kOpThreads) hist[b] = 0;
  pdl_wait();                                   // g (adjoint) and x (previous H_s)
  const int bq = blockIdx.y;
  if (mu_dev) mu = mu_dev[bq];
  const ThrWs w = thr_at(w0, bq);
  x_idx += (int64_t)bq * ldx;
  x_val += (int64_t)bq * ldx;
  const int xn = x_nnz[bq];
  out_idx += (int64_t)bq * ldo;
  out_val += (int64_t)bq * ldo;
  out_nnz += bq;
  g += (int64_t)bq * N;
  if (gout) gout += (int64_t)bq * N;
  const int G = (int)gridDim.x;
  const int64_t start = (int64_t)blockIdx.x * kTile;
  const int cnt = (int)min64(kTile, N - start);
  // ---- phase 1: a, NaN flag, histogram
  constexpr int PER = kTile / kOpThreads;       // 4 entries per thread, all loads in flight
  float gv[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kOpThreads;
    float v = 0.0f;
    if (i < cnt) {
      v = __ldg(g + start + i);
      for (int k = 1; k < nparts; ++k) v = __fadd_rn(v, __ldg(g + (int64_t)k * N + start + i));
      if (nparts > 0) v = __fmul_rn(gsigma, v);   // adjoint_reduce_kernel's order and rounding
    }
    gv[u] = v;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kOpThreads;
    if (i < cnt) {
      if (gout && nparts > 0) gout[start + i] = gv[u];
      as[i] = __fmul_rn(mu, gv[u]);
    }
  }
  const int nnz = xn < 0 ? 0 : min(xn, max_nnz);
  __syncthreads();
  for (int j = tid; j < nnz; j += kOpThreads) {
    const int64_t n = (int64_t)x_idx[j] - col_offset;   // local column (column shards)
    if (n >= start && n < start + cnt) as[n - start] = __fadd_rn(x_val[j], as[n - start]);
  }
  __syncthreads();
  int nan = 0;
  for (int i = tid; i < cnt; i += kOpThreads) {
    const float v = as[i];
    w.a[start + i] = v;                         // kept for the massive-tie fallback
    const unsigned int key = __float_as_uint(v) & 0x7FFFFFFFu;
    nan |= key > 0x7F800000u;
    atomicAdd(&hist[key >> 20], 1);
  }
  nan = __syncthreads_or(nan);
  if (tid == 0 && nan) atomicOr(&w.flags[0], 1);
  for (int b = tid; b < kHistBins; b += kOpThreads)
    if (hist[b]) atomicAdd(&w.hist[b], hist[b]);
  // ---- grid barrier of this snapshot's CTAs (co-resident: cooperative launch)
  __syncthreads();
  unsigned int* ctr = reinterpret_cast<unsigned int*>(&w.flags[3]);
  if (tid == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned int v;
#ifdef IHT_CHECKS
    long long spins = 0;
#endif
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
#ifdef IHT_CHECKS
      if (++spins > IHT_SPIN_LIMIT) {
        printf("IHT_DCHECK: thr_onepass barrier did not complete (block %d)\n", (int)blockIdx.x);
        __trap();
      }
#endif
    } while (v < (unsigned int)G);
    s_stop = xn < 0 || __ldcg(&w.flags[0]) != 0 || s == 0;
  }
  __syncthreads();
  // ---- phase 2: bin d1 of the s-th largest key (every CTA, same histogram), candidates
  const bool all = (int64_t)s >= N;
  const bool stop = s_stop != 0;
  unsigned int d1 = 0u;
  int above = 0;
  if (!stop) {
    for (int b = tid; b < kHistBins; b += kOpThreads) hist[b] = __ldcg(&w.hist[b]);
    __syncthreads();
    if (!all) {
      find_bin<kOpThreads>(hist, kHistBins, s, &sh[0], &sh[1], scratch);
      d1 = (unsigned int)sh[0];
      above = sh[1];
    }
    constexpr int per_warp = kTile / kOpWarps;  // 128 contiguous entries per warp
    const int lo = warp * per_warp, hi = min(cnt, lo + per_warp);
    auto pick = [&](float v) {
      const unsigned int key = __float_as_uint(v) & 0x7FFFFFFFu;
      return key > 0u && (all || (key >> 20) >= d1);
    };
    int c = 0;
#pragma unroll
    for (int u = 0; u < per_warp / 32; ++u) {
      const int i = lo + u * 32 + lane;
      c += __popc(__ballot_sync(0xffffffffu, i < hi && pick(as[i])));
    }
    if (lane == 0) wgt[warp] = c;
    __syncthreads();
    int base = 0, tot = 0;
    for (int q = 0; q < kOpWarps; ++q) {
      if (q < warp) base += wgt[q];
      tot += wgt[q];
    }
#pragma unroll
    for (int u = 0; u < per_warp / 32; ++u) {
      const int i = lo + u * 32 + lane;
      const float v = i < hi ? as[i] : 0.0f;
      const bool sel = i < hi && pick(v);
      const unsigned int bb = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const int pos = base + __popc(bb & lt);
        w.cidx[start + pos] = (int32_t)(col_offset + start + i);
        w.cval[start + pos] = v;
      }
      base += __popc(bb);
    }
    if (tid == 0) w.ccount[blockIdx.x] = tot;
  }
  // ---- the last CTA to arrive finishes the select
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(ctr, 1u) == 2u * (unsigned int)G - 1u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  auto finish = [&]() {                         // zero the histogram, flags and counter for the next call
    __syncthreads();
    for (int b = tid; b < kHistBins; b += kOpThreads) w.hist[b] = 0;
    if (tid < 4) w.flags[tid] = 0;
  };
  if (stop) {                                   // poisoned input / NaN -> domain error; H_0 keeps nothing
    if (tid == 0) *out_nnz = s == 0 && xn >= 0 && __ldcg(&w.flags[0]) == 0 ? 0 : -1;
    finish();
    return;
  }
  int carry = 0;                                // exclusive scan of the tile counts
  for (int t0 = 0; t0 < G; t0 += kOpThreads) {
    const int t = t0 + tid;
    const int myc = t < G ? __ldcg(&w.ccount[t]) : 0;
    int incl = myc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) scratch[warp] = incl;
    __syncthreads();
    int before = carry, tot = 0;
    for (int q = 0; q < kOpWarps; ++q) {
      if (q < warp) before += scratch[q];
      tot += scratch[q];
    }
    if (t < G) tile_base[t] = before + incl - myc;
    carry += tot;
    __syncthreads();
  }
  if (tid == 0) tile_base[G] = carry;
  __syncthreads();
  const int total = carry;
  if (total > kCandCap) {                       // massive ties: radix passes over a itself
    const float* a = w.a;
    const int c0 = (int)col_offset;
    select_ordered<kOpThreads>((int)N, s, [&](int i) { return __ldcg(&a[i]); }, [&](int i) { return c0 + i; },
                               out_idx, out_val, out_nnz, 0, hist, scratch, wgt, weq, wtake, wbase, sh);
    finish();
    return;
  }
  int32_t* cidx = reinterpret_cast<int32_t*>(dsm);
  float* cval = reinterpret_cast<float*>(dsm + kCandCap * 4);
  for (int i0 = 0; i0 < total; i0 += 2 * kOpThreads) {
    int32_t ci[2];
    float cv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * kOpThreads + tid;
      if (i < total) {
        int lo = 0, hi = G;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (tile_base[mid] <= i) lo = mid; else hi = mid;
        }
        const int64_t src = (int64_t)lo * kTile + (i - tile_base[lo]);
        ci[u] = __ldcg(&w.cidx[src]);
        cv[u] = __ldcg(&w.cval[src]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * kOpThreads + tid;
      if (i < total) {
        cidx[i] = ci[u];
        cval[i] = cv[u];
      }
    }
  }
  gathered_select<kOpThreads>(total, cidx, cval, keep, hist, grp_k, tile_base, d1, above, s, all, out_idx, out_val,
                              out_nnz, scratch, wgt, weq, wtake, wbase, sh);
  finish();
}

// ---------------------------------------------------------------------------- fused (cluster)
constexpr int kClThreads = 512;               // threads per CTA of the fused kernel
constexpr int kClWarps = kClThreads / 32;
constexpr int kClusterSlice = 32768;          // a-values per CTA held in shared memory (128 KiB)
constexpr int kClusterMax = 8;                // portable cluster size (16 measured slower)
constexpr int64_t kClusterMaxN = (int64_t)kClusterSlice * kClusterMax;
constexpr int kWarpCand = 256;                // candidate slots per warp (per CTA: 4096)

// Cluster-shared state of one CTA (read by the other CTAs through DSMEM).  Every slot is
// written once per launch, except the two histogram buffers, which alternate between
// passes: a CTA rewrites buffer k only after the next cluster barrier, which every CTA
// reaches after its remote reads of buffer k.  One barrier per histogram pass.
struct ClShared {
  int hist[2][2048];
  int flags[2];        // [0] NaN or poisoned input, [1] a warp's candidate list overflowed
  int counts[2];       // [0] keys > T, [1] keys == T (ordered compaction)
  int ncand;           // candidates after extraction (gather path)
};

// Histogram pass over the local list (pass index `pass`, 11/11/9 bits) summed over the
// cluster; find the bin of the target-th largest key.  Returns through sh[0], sh[1].
template <class Val>
__device__ void cluster_hist_pass(cg::cluster_group& cluster, ClShared& cs, int& buf, int n, Val val, int pass,
                                  unsigned int prefix, int target, int* tot, int* scratch, int* sh) {
  const int CL = (int)cluster.num_blocks();
  const int tid = threadIdx.x;
  const int shifts[3] = {20, 9, 0};
  const int widths[3] = {11, 11, 9};
  const int nb = 1 << widths[pass];
  const int sh_ = shifts[pass];
  const unsigned int hi_shift = sh_ + widths[pass];
  int* hist = cs.hist[buf];
  for (int q = tid; q < nb; q += kClThreads) hist[q] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += kClThreads) {
    const unsigned int key = __float_as_uint(val(i)) & 0x7FFFFFFFu;
    if ((key >> hi_shift) == (prefix >> hi_shift)) atomicAdd(&hist[(key >> sh_) & (nb - 1)], 1);
  }
  cluster.sync();
  for (int q = tid; q < nb; q += kClThreads) {
    int acc = 0;
    for (int p = 0; p < CL; ++p) acc += cluster.map_shared_rank(cs.hist[buf], p)[q];
    tot[q] = acc;
  }
  __syncthreads();
  find_bin<kClThreads>(tot, nb, target, &sh[0], &sh[1], scratch);
  buf ^= 1;
}

// Passes 1, 2 of the radix select over the cluster-wide list (n local entries val(i),
// global index gidx(i), in increasing index order within and across CTAs), then the
// ordered compaction into out_*.  `prefix`/`target`: state after pass 0.
template <class Val, class Gidx>
__device__ void cluster_select(cg::cluster_group& cluster, ClShared& cs, int& buf, int n, Val val, Gidx gidx,
                               unsigned int prefix, int target, bool all, int* tot, int* scratch, int* wgt, int* weq,
                               int* wtake, int* wbase, int* sh, int32_t* __restrict__ out_idx,
                               float* __restrict__ out_val, int32_t* __restrict__ out_nnz, int probe = 0) {
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned int T = 0;
  int need = 0;
  if (!all) {
    for (int pass = 1; pass < 3; ++pass) {
      cluster_hist_pass(cluster, cs, buf, n, val, pass, prefix, target, tot, scratch, sh);
      prefix |= (unsigned int)sh[0] << (pass == 1 ? 9 : 0);
      target -= sh[1];
      __syncthreads();
      if (probe == 4 + pass) return;                // profiling probe: stop after this pass
    }
    T = prefix;
    need = target;
  }
  // ordered compaction: per-warp contiguous ranges, per-CTA counts, exclusive scan over the cluster
  const int span = ((n + kClWarps - 1) / kClWarps + 31) / 32 * 32;
  const int wlo = warp * span, whi = min(n, wlo + span);
  int gt = 0, eq = 0;
  for (int i0 = wlo; i0 < whi; i0 += 32) {
    const int i = i0 + lane;
    const unsigned int key = i < whi ? (__float_as_uint(val(i)) & 0x7FFFFFFFu) : 0u;
    const bool live = i < whi && key > 0u;
    gt += __popc(__ballot_sync(0xffffffffu, live && (all || key > T)));
    eq += __popc(__ballot_sync(0xffffffffu, live && !all && key == T));
  }
  if (lane == 0) {
    wgt[warp] = gt;
    weq[warp] = eq;
  }
  __syncthreads();
  if (tid == 0) {
    int g_ = 0, e_ = 0;
    for (int w = 0; w < kClWarps; ++w) {
      g_ += wgt[w];
      e_ += weq[w];
    }
    cs.counts[0] = g_;
    cs.counts[1] = e_;
  }
  cluster.sync();
  if (tid == 0) {
    int eq_before = 0, base = 0, total = 0, mytake = 0;
    for (int p = 0; p < CL; ++p) {                  // CTAs hold increasing index ranges
      const int* rc = cluster.map_shared_rank(cs.counts, p);
      const int tk = (all || T == 0u) ? 0 : max(0, min(rc[1], need - eq_before));
      eq_before += rc[1];
      if (p < rank) base += rc[0] + tk;
      if (p == rank) mytake = tk;
      total += rc[0] + tk;
    }
    if (rank == 0) *out_nnz = total;
    int take_left = mytake, wb = base;              // lowest-index ties first: warps in order
    for (int w = 0; w < kClWarps; ++w) {
      const int tk = min(weq[w], take_left);
      take_left -= tk;
      wtake[w] = tk;
      wbase[w] = wb;
      wb += wgt[w] + tk;
    }
  }
  __syncthreads();
  int run_sel = 0, run_eq = 0;
  const unsigned int lt = (1u << lane) - 1u;
  const int take = wtake[warp], base = wbase[warp];
  for (int i0 = wlo; i0 < whi; i0 += 32) {
    const int i = i0 + lane;
    const float av = i < whi ? val(i) : 0.0f;
    const unsigned int key = __float_as_uint(av) & 0x7FFFFFFFu;
    const bool live = i < whi && key > 0u;
    const bool is_gt = live && (all || key > T);
    const bool is_eq = live && !all && key == T;
    const unsigned int beq = __ballot_sync(0xffffffffu, is_eq);
    const bool tk = is_eq && (run_eq + __popc(beq & lt)) < take;
    const bool sel = is_gt || tk;
    const unsigned int bsel = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int pos = base + run_sel + __popc(bsel & lt);
      out_idx[pos] = (int32_t)gidx(i);
      out_val[pos] = av;
    }
    run_sel += __popc(bsel);
    run_eq += __popc(beq);
  }
}

// One launch per selection: cluster of CL CTAs per snapshot (blockIdx.y), CTA rank r owns
// a-values [r slice, (r+1) slice) in shared memory.  Full passes over the slice: (1) a =
// mu g with the 11-bit histogram of its keys (x's few entries are then added and their
// histogram bins moved), (2) extraction of the candidates (digit >= the bin of the s-th
// largest key) into per-warp ordered lists; the last two radix passes and the ordered
// compaction run on the candidates only.  If a warp's list overflows (massive ties,
// mostly-zero a) the cluster falls back to the passes over the whole slice.
__global__ void __launch_bounds__(kClThreads, 1) thr_cluster_kernel(
    const int32_t* __restrict__ x_idx, const float* __restrict__ x_val, const int32_t* __restrict__ x_nnz,
    int32_t max_nnz, int32_t ldx, const float* __restrict__ g, float mu, const float* __restrict__ mu_dev, int s,
    int64_t N, int64_t col_offset, int slice, int32_t* __restrict__ out_idx, float* __restrict__ out_val,
    int32_t ldo, int32_t* __restrict__ out_nnz, int probe, int nparts, float gsigma, float* __restrict__ gout,
    long long* __restrict__ tl) {
  // profiling timeline (IHT_THR_TL): globaltimer stamps of CTA ranks 0, 1 of snapshot 0
  auto stamp = [&](int k) {
    if (tl && threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 2) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tl[blockIdx.x * 16 + k] = t;
    }
  };
  extern __shared__ __align__(16) unsigned char dsm[];
  float* as = reinterpret_cast<float*>(dsm);                                  // [slice] (multiple of 4)
  int32_t* cidx = reinterpret_cast<int32_t*>(dsm + (size_t)slice * 4);        // [kClWarps][kWarpCand]
  float* cval = reinterpret_cast<float*>(cidx + kClWarps * kWarpCand);        // [kClWarps][kWarpCand]
  int32_t* pidx = reinterpret_cast<int32_t*>(cval + kClWarps * kWarpCand);    // packed list (index order)
  float* pval = reinterpret_cast<float*>(pidx + kClWarps * kWarpCand);
  __shared__ ClShared cs;
  __shared__ int tot[2048];
  __shared__ int scratch[kClWarps];
  __shared__ int wgt[kClWarps], weq[kClWarps], wtake[kClWarps], wbase[kClWarps];
  __shared__ int sh[4];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_launch_dependents();
  pdl_wait();                                   // g (adjoint) and x (previous H_s)
  if (mu_dev) mu = mu_dev[blockIdx.y];          // the adaptive step's mu: a predecessor's output too
  stamp(0);
  const int b = blockIdx.y;
  x_idx += (int64_t)b * ldx;
  x_val += (int64_t)b * ldx;
  g += (int64_t)b * N;
  out_idx += (int64_t)b * ldo;
  out_val += (int64_t)b * ldo;
  const int64_t lo = (int64_t)rank * slice;
  const int n = (int)min64(max64(N - lo, 0), slice);           // this CTA's slice [lo, lo + n)
  int buf = 0;
  int* hist = cs.hist[0];
  for (int q = tid; q < 2048; q += kClThreads) hist[q] = 0;
  __syncthreads();
  // ---- (1) a = mu g and the histogram of the top 11 key bits; float4 when aligned
  int nan = 0;
  // nparts > 0 (solver, split-K adjoint): g = sigma (part_0 + ... + part_{P-1}), planes N
  // apart, summed in adjoint_reduce_kernel's order and rounding
  const bool vec = ((reinterpret_cast<uintptr_t>(g + lo) & 15) == 0) && (nparts == 0 || (N & 3) == 0);
  const int n4 = vec ? (n >> 2) : 0;
  constexpr int kLd = 8;                 // float4 loads in flight per thread (g is read once)
  auto gsum1 = [&](int64_t e) {
    if (nparts == 0) return __ldg(g + e);
    float t = __ldg(g + e);
    for (int k = 1; k < nparts; ++k) t = __fadd_rn(t, __ldg(g + (int64_t)k * N + e));
    return __fmul_rn(gsigma, t);
  };
  for (int i0 = 0; i0 < n4; i0 += kClThreads * kLd) {
    float4 v[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int i = i0 + u * kClThreads + tid;
      v[u] = i < n4 ? __ldg(reinterpret_cast<const float4*>(g + lo) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (nparts > 0) {
      for (int k = 1; k < nparts; ++k) {
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
          const int i = i0 + u * kClThreads + tid;
          if (i < n4) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(g + (int64_t)k * N + lo) + i);
            v[u] = make_float4(__fadd_rn(v[u].x, w.x), __fadd_rn(v[u].y, w.y), __fadd_rn(v[u].z, w.z),
                               __fadd_rn(v[u].w, w.w));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kLd; ++u) {
        const int i = i0 + u * kClThreads + tid;
        v[u] = make_float4(__fmul_rn(gsigma, v[u].x), __fmul_rn(gsigma, v[u].y), __fmul_rn(gsigma, v[u].z),
                           __fmul_rn(gsigma, v[u].w));
        if (gout && i < n4) reinterpret_cast<float4*>(gout + lo)[i] = v[u];   // g materialised once
      }
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int i = i0 + u * kClThreads + tid;
      if (i >= n4) break;
      const float4 a4 =
          make_float4(__fmul_rn(mu, v[u].x), __fmul_rn(mu, v[u].y), __fmul_rn(mu, v[u].z), __fmul_rn(mu, v[u].w));
      reinterpret_cast<float4*>(as)[i] = a4;
      const unsigned int k0 = __float_as_uint(a4.x) & 0x7FFFFFFFu, k1 = __float_as_uint(a4.y) & 0x7FFFFFFFu,
                         k2 = __float_as_uint(a4.z) & 0x7FFFFFFFu, k3 = __float_as_uint(a4.w) & 0x7FFFFFFFu;
      nan |= (k0 > 0x7F800000u) | (k1 > 0x7F800000u) | (k2 > 0x7F800000u) | (k3 > 0x7F800000u);
      atomicAdd(&hist[k0 >> 20], 1);
      atomicAdd(&hist[k1 >> 20], 1);
      atomicAdd(&hist[k2 >> 20], 1);
      atomicAdd(&hist[k3 >> 20], 1);
    }
  }
  for (int i = (n4 << 2) + tid; i < n; i += kClThreads) {
    const float gv = gsum1(lo + i);
    if (gout && nparts > 0) gout[lo + i] = gv;
    const float a1 = __fmul_rn(mu, gv);
    as[i] = a1;
    const unsigned int k = __float_as_uint(a1) & 0x7FFFFFFFu;
    nan |= k > 0x7F800000u;
    atomicAdd(&hist[k >> 20], 1);
  }
  int nnz = x_nnz[b];
  const int poisoned = nnz < 0;
  nnz = nnz < 0 ? 0 : min(nnz, max_nnz);
  __syncthreads();
  // x's entries (distinct indices, an H_s output): a_n = x_n + mu g_n, moving the bin
  for (int j = tid; j < nnz; j += kClThreads) {
    const int64_t c = (int64_t)x_idx[j] - col_offset - lo;
    if (c >= 0 && c < n) {
      const float old = as[c];
      const float nw = __fadd_rn(x_val[j], old);
      as[c] = nw;
      const unsigned int ko = __float_as_uint(old) & 0x7FFFFFFFu, kn = __float_as_uint(nw) & 0x7FFFFFFFu;
      nan |= kn > 0x7F800000u;
      atomicSub(&hist[ko >> 20], 1);
      atomicAdd(&hist[kn >> 20], 1);
    }
  }
  nan = __syncthreads_or(nan);
  stamp(1);
  if (tid == 0) cs.flags[0] = nan | poisoned;
  if (probe == 1) return;                           // profiling probe (IHT_THR_PROBE): phases' cost
  cluster.sync();
  // cluster-wide histogram: every remote (DSMEM) load of this thread is issued before any
  // is summed -- 2048 / 512 bins x CL ranks, one round trip instead of 4 CL
  int bad = 0;
  {
    int hv[2048 / kClThreads][kClusterMax];
    int fv[kClusterMax];
#pragma unroll
    for (int p = 0; p < kClusterMax; ++p) {
      if (p < CL) {
        const int* rh = cluster.map_shared_rank(cs.hist[0], p);
        fv[p] = cluster.map_shared_rank(cs.flags, p)[0];
#pragma unroll
        for (int u = 0; u < 2048 / kClThreads; ++u) hv[u][p] = rh[tid + u * kClThreads];
      }
    }
#pragma unroll
    for (int u = 0; u < 2048 / kClThreads; ++u) {
      int acc = 0;
#pragma unroll
      for (int p = 0; p < kClusterMax; ++p)
        if (p < CL) acc += hv[u][p];
      tot[tid + u * kClThreads] = acc;
    }
#pragma unroll
    for (int p = 0; p < kClusterMax; ++p)
      if (p < CL) bad |= fv[p];
  }
  buf = 1;
  __syncthreads();
  if (bad || s == 0) {
    if (rank == 0 && tid == 0) out_nnz[b] = bad ? -1 : 0;
    cluster.sync();
    return;
  }
  stamp(2);
  if (probe == 2) { cluster.sync(); return; }
  const bool all = (int64_t)s >= N;
  unsigned int d1 = 0;
  int target = s;
  if (!all) {
    find_bin<kClThreads>(tot, 2048, s, &sh[0], &sh[1], scratch);
    d1 = (unsigned int)sh[0];
    target = s - sh[1];
  }
  stamp(7);
  // ---- (2) candidates: key > 0 and digit >= d1, per-warp ordered lists (contiguous ranges)
  const int span = ((n + kClWarps - 1) / kClWarps + 31) / 32 * 32;
  const int wlo = warp * span, whi = min(n, wlo + span);
  int wc = 0;
  const unsigned int lt = (1u << lane) - 1u;
  int32_t* my_idx = cidx + warp * kWarpCand;
  float* my_val = cval + warp * kWarpCand;
  // lane = 4 consecutive entries (one 16-byte shared load) of a 128-entry chunk; chunks
  // without a candidate (almost all: candidates are ~s of N) cost one vote
  for (int i00 = wlo; i00 < whi; i00 += 128) {
    const int ib = i00 + 4 * lane;
    float v[4];
    if (ib + 3 < whi) {
      const float4 q = *reinterpret_cast<const float4*>(as + ib);   // wlo, i00 multiples of 32: aligned
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = ib + e < whi ? as[ib + e] : 0.0f;
    }
    unsigned int f = 0u;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned int key = __float_as_uint(v[e]) & 0x7FFFFFFFu;
      f |= (unsigned int)(ib + e < whi && key > 0u && (key >> 20) >= d1) << e;
    }
    if (__any_sync(0xffffffffu, f)) {
      const int cnt = __popc(f);
      int incl = cnt;                               // inclusive scan over lanes (index order)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int pos = wc + incl - cnt;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if ((f >> e) & 1u) {
          if (pos < kWarpCand) {
            my_idx[pos] = (int32_t)(col_offset + lo + ib + e);
            my_val[pos] = v[e];
          }
          ++pos;
        }
      }
      wc += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  if (lane == 0) wgt[warp] = wc;
  stamp(3);
  if (probe == 3) { cluster.sync(); return; }
  const int ovf = __syncthreads_or(wc > kWarpCand);
  if (tid == 0) {
    int nc = 0;
    for (int w = 0; w < kClWarps; ++w) nc += min(wgt[w], kWarpCand);
    cs.flags[1] = ovf;
    cs.ncand = nc;                                  // this CTA's candidates (valid without overflow)
  }
  cluster.sync();
  int any_ovf = 0, total = 0, base = 0;
  {
    int ov[kClusterMax], nv[kClusterMax];          // all remote loads first, then the sums
#pragma unroll
    for (int p = 0; p < kClusterMax; ++p) {
      if (p < CL) {
        ov[p] = cluster.map_shared_rank(cs.flags, p)[1];
        nv[p] = *cluster.map_shared_rank(&cs.ncand, p);
      }
    }
#pragma unroll
    for (int p = 0; p < kClusterMax; ++p) {
      if (p < CL) {
        any_ovf |= ov[p];
        if (p < rank) base += nv[p];
        total += nv[p];
      }
    }
  }
  if (!any_ovf && total <= kClWarps * kWarpCand && probe != 9) {   // probe 9: per-pass cluster path (A/B)
    // few candidates (the usual case): every CTA stores its ordered lists into rank 0's
    // packed buffer at its cluster offset (DSMEM stores, ranks in index order), then rank 0
    // alone finishes the select on them -- two cluster barriers instead of one per pass.
    // The candidates hold every key with digit >= d1 (>= s of them unless fewer nonzero
    // keys exist), so their top-s, ties to the lowest index, is the top-s of a.
    int32_t* gidx = cluster.map_shared_rank(pidx, 0);
    float* gval = cluster.map_shared_rank(pval, 0);
    int off = base;
    for (int w = 0; w < warp; ++w) off += min(wgt[w], kWarpCand);
    for (int j = lane; j < min(wgt[warp], kWarpCand); j += 32) {
      IHT_DCHECK(off + j < kClWarps * kWarpCand, "threshold: gathered candidate inside rank 0's list");
      gidx[off + j] = cidx[warp * kWarpCand + j];
      gval[off + j] = cval[warp * kWarpCand + j];
    }
    stamp(4);
    cluster.sync();                                 // rank 0's list complete; nobody reads remote memory after
    stamp(5);
    if (rank != 0) return;
    if (probe == 4) return;
    if (total <= kClThreads) {
      // at most one candidate per thread: its rank among the candidates (keys greater, or
      // equal at a lower index -- the list is in index order) decides it directly; kept
      // iff rank < s (candidates have key > 0), written at the count of kept ones before it
      const int i = tid;
      const bool have = i < total;
      const float vi = have ? pval[i] : 0.0f;
      const unsigned int ki = __float_as_uint(vi) & 0x7FFFFFFFu;
      int rk = 0;
      int j = warp * 32 < total ? 0 : total;        // warps without a candidate skip the loop
      for (; j + 4 <= total; j += 4) {              // broadcast reads, 4 in flight
        const unsigned int k0 = __float_as_uint(pval[j]) & 0x7FFFFFFFu, k1 = __float_as_uint(pval[j + 1]) & 0x7FFFFFFFu,
                           k2 = __float_as_uint(pval[j + 2]) & 0x7FFFFFFFu, k3 = __float_as_uint(pval[j + 3]) & 0x7FFFFFFFu;
        rk += (k0 > ki || (k0 == ki && j < i)) + (k1 > ki || (k1 == ki && j + 1 < i)) +
              (k2 > ki || (k2 == ki && j + 2 < i)) + (k3 > ki || (k3 == ki && j + 3 < i));
      }
      for (; j < total; ++j) {
        const unsigned int kj = __float_as_uint(pval[j]) & 0x7FFFFFFFu;
        rk += kj > ki || (kj == ki && j < i);
      }
      const bool sel = have && rk < s;
      const unsigned int bs = __ballot_sync(0xffffffffu, sel);
      if (lane == 0) wgt[warp] = __popc(bs);
      __syncthreads();
      int pos = __popc(bs & lt);
      for (int w = 0; w < warp; ++w) pos += wgt[w];
      if (sel) {
        out_idx[pos] = pidx[i];                     // out_idx / out_val point at snapshot b already
        out_val[pos] = vi;
      }
      if (tid == 0) {
        int kept = 0;
        for (int w = 0; w < kClWarps; ++w) kept += wgt[w];
        out_nnz[b] = kept;
      }
      stamp(6);
      return;
    }
    select_ordered<kClThreads>(total, s, [&](int i) { return pval[i]; }, [&](int i) { return pidx[i]; }, out_idx,
                               out_val, out_nnz + b, 0, tot, scratch, wgt, weq, wtake, wbase, sh);
    return;
  }
  if (!any_ovf) {
    // pack the warp lists in order into the second buffer: every warp copies its own list
    // to its running offset at once
    int off = 0, nc = 0;
    for (int w = 0; w < kClWarps; ++w) {
      const int cw = min(wgt[w], kWarpCand);
      if (w == warp) off = nc;
      nc += cw;
    }
    for (int j = lane; j < min(wgt[warp], kWarpCand); j += 32) {
      pidx[off + j] = cidx[warp * kWarpCand + j];
      pval[off + j] = cval[warp * kWarpCand + j];
    }
    __syncthreads();
    if (probe == 4) { cluster.sync(); return; }
    cluster_select(cluster, cs, buf, nc, [&](int i) { return pval[i]; }, [&](int i) { return pidx[i]; },
                   all ? 0u : (d1 << 20), target, all, tot, scratch, wgt, weq, wtake, wbase, sh, out_idx, out_val,
                   out_nnz + b, probe);
  } else {
    const int64_t base_idx = col_offset + lo;
    cluster_select(cluster, cs, buf, n, [&](int i) { return as[i]; }, [&](int i) { return base_idx + i; },
                   all ? 0u : (d1 << 20), target, all, tot, scratch, wgt, weq, wtake, wbase, sh, out_idx, out_val,
                   out_nnz + b);
  }
  cluster.sync();                                   // keep shared memory alive for remote readers
}

// Bounded select (config 5, solver only): the tcgen05 adjoint's epilogue appended every
// pixel n with key(mu g_n) >= bkey = bound_key(x) (batched_limbs_kernel) to this snapshot's list
// (cidx, cval, ccnt; iht_batched.cu).  With x's support added (a_j = x_j + mu g_j, the cluster
// kernel's arithmetic) and the support's own epilogue entries dropped, the list holds every
// pixel whose key is >= bkey.  If at least s of its keys are >= bkey, the s-th largest key of a
// is >= bkey too, so every entry of H_s(a) -- including the lowest-index ties at the threshold
// -- is in the list, and the top-s of the list (greater key, then lower index) IS H_s(a),
// exactly.  Otherwise (iteration 1, a support change larger than the bound,
// list overflow, NaN, poisoned x) the same CTA selects the snapshot over all of a
// (bs_full_select): no second launch -- a skipped cluster-kernel launch had cost ~9 us per
// iteration in the graph (r02 g55).  One CTA per snapshot; resets ccnt for the next call;
// done[b] = 1 when the list decided (statistics / tests).
// 512 threads (r02 g57: 256 threads, 2 list entries more per thread, were 3 us per iteration
// slower); ~15 KB of static shared memory, the full select's lists in the workspace.
constexpr int kBsThreads = 512;
constexpr int kBsCap = 1024;                   // list entries ranked in shared memory
constexpr int kBsMaxS = 256;
constexpr int kBsWarps = kBsThreads / 32;

// Full select of one snapshot over all N columns, when the bounded list could not decide it
// (iteration 1, a large support change, NaN, overflow): the cluster kernel's arithmetic and
// result in one CTA.  a = mu g into the workspace ga, its 11-bit histogram (top key bits),
// x's support patched to a_j = x_j + mu g_j; bin d1 of the s-th largest key; the keys with
// digit >= d1 listed in index order by each warp over its contiguous range (in the workspace:
// warp w's list at gl + w * span, it cannot hold more than its range), packed in index order
// (gp), and select_ordered on them, the values gathered from ga.  Poisoned x or a NaN in a:
// nnz = -1 (sticky).
__device__ void bs_full_select(const int32_t* __restrict__ x_idx, const float* __restrict__ x_val, int nraw, int nnz,
                               const float* __restrict__ g, float mu, int s, int N, float* __restrict__ ga,
                               int32_t* __restrict__ gl, int32_t* __restrict__ gp, int32_t* __restrict__ out_idx,
                               float* __restrict__ out_val, int32_t* __restrict__ out_nnz_b, int* hist, int* scratch,
                               int* wgt, int* weq, int* wtake, int* wbase, int* sh) {
  constexpr int NT = kBsThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (nraw < 0) {
    if (tid == 0) *out_nnz_b = -1;
    return;
  }
  for (int q = tid; q < 2048; q += NT) hist[q] = 0;
  __syncthreads();
  int nan = 0;
  const bool vec = (N & 3) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (reinterpret_cast<uintptr_t>(ga) & 15) == 0;
  const int n4 = vec ? N >> 2 : 0;
  constexpr int kLd = 8;
  for (int i0 = 0; i0 < n4; i0 += NT * kLd) {
    float4 v[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int i = i0 + u * NT + tid;
      v[u] = i < n4 ? __ldg(reinterpret_cast<const float4*>(g) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int i = i0 + u * NT + tid;
      if (i >= n4) break;
      const float4 a4 = make_float4(__fmul_rn(mu, v[u].x), __fmul_rn(mu, v[u].y), __fmul_rn(mu, v[u].z),
                                    __fmul_rn(mu, v[u].w));
      reinterpret_cast<float4*>(ga)[i] = a4;
      const unsigned int k0 = __float_as_uint(a4.x) & 0x7FFFFFFFu, k1 = __float_as_uint(a4.y) & 0x7FFFFFFFu,
                         k2 = __float_as_uint(a4.z) & 0x7FFFFFFFu, k3 = __float_as_uint(a4.w) & 0x7FFFFFFFu;
      nan |= (k0 > 0x7F800000u) | (k1 > 0x7F800000u) | (k2 > 0x7F800000u) | (k3 > 0x7F800000u);
      atomicAdd(&hist[k0 >> 20], 1);
      atomicAdd(&hist[k1 >> 20], 1);
      atomicAdd(&hist[k2 >> 20], 1);
      atomicAdd(&hist[k3 >> 20], 1);
    }
  }
  for (int i = (n4 << 2) + tid; i < N; i += NT) {
    const float a1 = __fmul_rn(mu, __ldg(g + i));
    ga[i] = a1;
    const unsigned int k = __float_as_uint(a1) & 0x7FFFFFFFu;
    nan |= k > 0x7F800000u;
    atomicAdd(&hist[k >> 20], 1);
  }
  __syncthreads();                              // ga complete (global writes of this CTA)
  for (int j = tid; j < nnz; j += NT) {         // x's entries (distinct indices): move their keys
    const int c = x_idx[j];
    const float old = ga[c];
    const float nw = __fadd_rn(x_val[j], old);
    ga[c] = nw;
    const unsigned int ko = __float_as_uint(old) & 0x7FFFFFFFu, kn = __float_as_uint(nw) & 0x7FFFFFFFu;
    nan |= kn > 0x7F800000u;
    atomicSub(&hist[ko >> 20], 1);
    atomicAdd(&hist[kn >> 20], 1);
  }
  nan = __syncthreads_or(nan);
  if (nan) {
    if (tid == 0) *out_nnz_b = -1;
    return;
  }
  find_bin<NT>(hist, 2048, s, &sh[0], &sh[1], scratch);
  const unsigned int d1 = (unsigned int)sh[0];
  const int span = ((N + kBsWarps - 1) / kBsWarps + 127) / 128 * 128;
  const int wlo = warp * span, whi = min(N, wlo + span);
  int32_t* wl = gl + wlo;                       // this warp's list: at most whi - wlo entries
  int wc = 0;
  for (int i00 = wlo; i00 < whi; i00 += 128) {  // lane = 4 consecutive entries
    const int ib = i00 + 4 * lane;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = ib + e < whi ? __ldcg(ga + ib + e) : 0.0f;
    unsigned int f = 0u;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned int key = __float_as_uint(v[e]) & 0x7FFFFFFFu;
      f |= (unsigned int)(ib + e < whi && key > 0u && (key >> 20) >= d1) << e;
    }
    if (__any_sync(0xffffffffu, f)) {
      const int cnt = __popc(f);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int pos = wc + incl - cnt;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if ((f >> e) & 1u) {
          IHT_DCHECK(wlo + pos < whi, "bounded select: full-select list inside its warp's range");
          wl[pos++] = ib + e;
        }
      }
      wc += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  if (lane == 0) wgt[warp] = wc;
  __syncthreads();                              // the lists (global, this CTA) and their counts
  int off = 0, total = 0;
  for (int w = 0; w < kBsWarps; ++w) {
    if (w == warp) off = total;
    total += wgt[w];
  }
  for (int j = lane; j < wc; j += 32) {
    IHT_DCHECK(off + j < N, "bounded select: packed full-select list inside N");
    gp[off + j] = __ldcg(wl + j);
  }
  __syncthreads();
  select_ordered<NT>(total, s, [&](int i) { return __ldcg(ga + __ldcg(gp + i)); }, [&](int i) { return __ldcg(gp + i); },
                     out_idx, out_val, out_nnz_b, 0, hist, scratch, wgt, weq, wtake, wbase, sh);
}

__global__ void __launch_bounds__(kBsThreads, 1) thr_bounded_select(
    const int32_t* __restrict__ x_idx, const float* __restrict__ x_val, const int32_t* __restrict__ x_nnz,
    int32_t max_nnz, int32_t ldx, const float* __restrict__ g, float mu, const unsigned int* __restrict__ bkeys,
    int s, int64_t N, const int32_t* __restrict__ cidx, const float* __restrict__ cval, int* __restrict__ ccnt,
    int ccap, int32_t* __restrict__ out_idx, float* __restrict__ out_val, int32_t ldo, int32_t* __restrict__ out_nnz,
    int* __restrict__ done, int* __restrict__ stats, float* __restrict__ ga0, int32_t* __restrict__ gl0,
    int32_t* __restrict__ gp0, int64_t ws_stride) {
  constexpr int PER = kBsCap / kBsThreads;      // list slots per thread
  // the list (lidx | lkey | lval) and, on the full-select path, its histogram in the same bytes
  __shared__ __align__(16) unsigned char lbuf[(2 * (kBsCap + 4) + kBsCap) * 4];
  int32_t* lidx = reinterpret_cast<int32_t*>(lbuf);
  unsigned int* lkey = reinterpret_cast<unsigned int*>(lidx + kBsCap + 4);
  float* lval = reinterpret_cast<float*>(lkey + kBsCap + 4);
  int* f_hist = reinterpret_cast<int*>(lbuf);   // 2048 ints <= the list's bytes
  static_assert(2048 * 4 <= (2 * (kBsCap + 4) + kBsCap) * 4, "histogram fits the list buffer");
  __shared__ int f_scratch[kBsWarps], f_wgt[kBsWarps], f_weq[kBsWarps], f_wtake[kBsWarps], f_wbase[kBsWarps], f_sh[4];
  __shared__ __align__(16) int32_t sidx[kBsMaxS + 4];
  __shared__ float kval[kBsMaxS];
  __shared__ int sh_n, sh_t, sh_bad, sh_kept;
  pdl_launch_dependents();
  pdl_wait();                                   // g and the lists (adjoint), x (previous H_s)
  const int b = blockIdx.x, tid = threadIdx.x;
  x_idx += (int64_t)b * ldx;
  x_val += (int64_t)b * ldx;
  g += (int64_t)b * N;
  cidx += (int64_t)b * ccap;
  cval += (int64_t)b * ccap;
  out_idx += (int64_t)b * ldo;
  out_val += (int64_t)b * ldo;
  // one round trip: the counts, the bound key, x's slots and the first list slots, all at once
  // (slots past the counts are masked below)
  const int nraw = x_nnz[b];
  const int cnt = ccnt[b];
  const unsigned int bkey = bkeys[b];             // the key the epilogue listed against
  const int32_t xi = tid < max_nnz ? x_idx[tid] : 0;
  const float xv = tid < max_nnz ? x_val[tid] : 0.0f;
  int32_t ci[PER];
  float cv[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kBsThreads;
    ci[u] = i < ccap ? cidx[i] : 0;
    cv[u] = i < ccap ? cval[i] : 0.0f;
  }
  const int nnz = nraw < 0 ? 0 : min(nraw, max_nnz);
  if (tid == 0) {
    sh_n = nnz;
    sh_t = 0;
    sh_bad = 0;
    sh_kept = 0;
  }
  __syncthreads();                              // every thread has read ccnt
  if (tid == 0) ccnt[b] = 0;                    // zero for the next call
  auto full = [&]() {                           // not decidable from the list: select over all of a
    if (tid == 0) {
      done[b] = 0;
      if (stats) atomicAdd(&stats[1], 1);
    }
    __syncthreads();                            // the list buffer becomes the histogram
    bs_full_select(x_idx, x_val, nraw, nnz, g, mu, s, (int)N, ga0 + (int64_t)b * ws_stride,
                   gl0 + (int64_t)b * ws_stride, gp0 + (int64_t)b * ws_stride, out_idx, out_val, out_nnz + b, f_hist,
                   f_scratch, f_wgt, f_weq, f_wtake, f_wbase, f_sh);
  };
  if (nraw < 0 || bkey == 0xFFFFFFFFu || s <= 0 || s > kBsMaxS || nnz > kBsMaxS || cnt > ccap || (int64_t)s >= N ||
      nnz + cnt > kBsCap || max_nnz > kBsThreads) {
    full();
    return;
  }
  // x's support: a_j = x_j + mu g_j (the cluster kernel's arithmetic); the g gather is issued
  // before the membership tests below
  float gj = 0.0f;
  if (tid < nnz) {
    gj = __ldg(g + xi);
    sidx[tid] = xi;
  }
  if (tid < 4) sidx[nnz + tid] = -1;            // pad to whole int4 (never a column)
  __syncthreads();
  // the epilogue's entries outside the support (a = mu g there); list order is irrelevant
  const int nq = (nnz + 3) >> 2;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kBsThreads;
    if (i < cnt) {
      bool in = false;
      for (int q = 0; q < nq; ++q) {
        const int4 v = reinterpret_cast<const int4*>(sidx)[q];
        in |= (v.x == ci[u]) | (v.y == ci[u]) | (v.z == ci[u]) | (v.w == ci[u]);
      }
      if (!in) {
        const int p = atomicAdd(&sh_n, 1);
        IHT_DCHECK(p < kBsCap, "bounded select: list slot");
        lidx[p] = ci[u];
        lval[p] = cv[u];
        lkey[p] = __float_as_uint(cv[u]) & 0x7FFFFFFFu;
      }
    }
  }
  if (tid < nnz) {
    const float av = __fadd_rn(xv, __fmul_rn(mu, gj));
    lidx[tid] = xi;
    lval[tid] = av;
    lkey[tid] = __float_as_uint(av) & 0x7FFFFFFFu;
  }
  __syncthreads();
  const int n = sh_n;
  if (tid < 4) {                                // pad to whole uint4: key 0, never before anything
    lkey[n + tid] = 0u;
    lidx[n + tid] = 0x7FFFFFFF;
  }
  int t = 0, bad = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kBsThreads;
    if (i < n) {
      t += lkey[i] >= bkey;
      bad |= lkey[i] > 0x7F800000u;
    }
  }
  if (t) atomicAdd(&sh_t, t);
  if (bad) sh_bad = 1;
  __syncthreads();
  if (sh_bad || sh_t < s) {
    full();
    return;
  }
  // rank = keys greater, or equal at a lower index (4 entries per shared load); kept iff
  // rank < s -- then rank < s <= the count of keys >= bkey > 0, so every kept key is >= bkey
  const int n4 = (n + 3) >> 2;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * kBsThreads;
    if (i < n) {
      const unsigned int ki = lkey[i];
      const int32_t ii = lidx[i];
      int rk = 0;
      for (int q = 0; q < n4; ++q) {
        const uint4 k4 = reinterpret_cast<const uint4*>(lkey)[q];
        const int4 i4 = reinterpret_cast<const int4*>(lidx)[q];
        rk += (k4.x > ki || (k4.x == ki && i4.x < ii)) + (k4.y > ki || (k4.y == ki && i4.y < ii)) +
              (k4.z > ki || (k4.z == ki && i4.z < ii)) + (k4.w > ki || (k4.w == ki && i4.w < ii));
      }
      if (rk < s) {
        const int p = atomicAdd(&sh_kept, 1);
        IHT_DCHECK(p < kBsMaxS, "bounded select: kept slot");
        sidx[p] = ii;                           // sidx is free (membership tests done)
        kval[p] = lval[i];
      }
    }
  }
  __syncthreads();
  // write the kept entries in increasing index order: position = kept entries at lower indices
  const int kept = sh_kept;
  if (tid < 4) sidx[kept + tid] = 0x7FFFFFFF;
  __syncthreads();
  if (tid < kept) {
    const int32_t ii = sidx[tid];
    int pos = 0;
    for (int q = 0; q < ((kept + 3) >> 2); ++q) {
      const int4 v = reinterpret_cast<const int4*>(sidx)[q];
      pos += (v.x < ii) + (v.y < ii) + (v.z < ii) + (v.w < ii);
    }
    out_idx[pos] = ii;
    out_val[pos] = kval[tid];
  }
  if (tid == 0) {
    out_nnz[b] = kept;
    done[b] = 1;
    if (stats) {
      atomicAdd(&stats[0], 1);
      atomicAdd(&stats[2], n);
      atomicMax(&stats[3], n);
    }
  }
}

// T4: merge of the shards' local top-s lists (column-sharded batched path): the global
// top-s is contained in the union of the local top-s (same tie rule), and the shards'
// lists concatenated in shard order are in increasing global index order.
__global__ void __launch_bounds__(kThrThreads, 1) thr_merge(
    const int32_t* __restrict__ cidx_g, const float* __restrict__ cval_g, const int32_t* __restrict__ cnnz_g,
    int64_t stride, int P, int s, int nrhs, int32_t* __restrict__ out_idx, float* __restrict__ out_val,
    int32_t* __restrict__ out_nnz) {
  extern __shared__ __align__(16) unsigned char dsm[];
  int32_t* cidx = reinterpret_cast<int32_t*>(dsm);
  float* cval = reinterpret_cast<float*>(dsm + kCandCap * 4);
  __shared__ int hist[2048];
  __shared__ int scratch[kThrWarps];
  __shared__ int wgt[kThrWarps], weq[kThrWarps], wtake[kThrWarps], wbase[kThrWarps];
  __shared__ int sh[4];
  __shared__ int base[1025];
  const int b = blockIdx.x, tid = threadIdx.x;
  out_idx += (int64_t)b * s;
  out_val += (int64_t)b * s;
  if (tid == 0) {
    int acc = 0, bad = 0;
    for (int p = 0; p < P; ++p) {
      const int c = cnnz_g[(int64_t)p * stride + b];
      bad |= c < 0;
      base[p] = acc;
      acc += c < 0 ? 0 : min(c, s);
    }
    sh[3] = bad ? -1 : acc;
  }
  __syncthreads();
  const int total = sh[3];
  if (total < 0 || s == 0) {
    if (tid == 0) out_nnz[b] = total < 0 ? -1 : 0;
    return;
  }
  for (int p = tid >> 5; p < P; p += kThrWarps) {
    const int c = min(cnnz_g[(int64_t)p * stride + b], s);
    const int64_t src = (int64_t)p * stride + (int64_t)b * s;
    for (int i = tid & 31; i < c; i += 32) {
      cidx[base[p] + i] = cidx_g[src + i];
      cval[base[p] + i] = cval_g[src + i];
    }
  }
  __syncthreads();
  select_ordered(total, s, [&](int i) { return cval[i]; }, [&](int i) { return cidx[i]; }, out_idx, out_val,
                 out_nnz + b, 0, hist, scratch, wgt, weq, wtake, wbase, sh);
}

}  // namespace iht

using namespace iht;

static int thr_probe() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IHT_THR_PROBE");     // profiling only: stop the fused kernel after a phase
    v = e ? atoi(e) : 0;
  }
  return v;
}

extern "C" int64_t iht_threshold_batched_ws_bytes(int64_t N, int32_t s, int32_t nrhs) {
  (void)s;
  if (N <= 0 || nrhs <= 0) return -1;
  return thr_ws_layout(N, nrhs, nullptr, nullptr);
}

extern "C" int64_t iht_threshold_ws_bytes(int64_t N, int32_t s) { return iht_threshold_batched_ws_bytes(N, s, 1); }

static long long* thr_timeline() {
  static long long* p = nullptr;
  static int on = -1;
  if (on < 0) {
    on = getenv("IHT_THR_TL") ? atoi(getenv("IHT_THR_TL")) : 0;   // profiling only
    if (on) {
      cudaMalloc(&p, 32 * sizeof(long long));
      cudaMemset(p, 0, 32 * sizeof(long long));
    }
  }
  return p;
}

static bool g_thr_attr = false;

static int thr_attrs() {
  if (!g_thr_attr) {
    IHT_CUDA_CHECK(cudaFuncSetAttribute(thr_select, cudaFuncAttributeMaxDynamicSharedMemorySize, kCandCap * 8));
    IHT_CUDA_CHECK(cudaFuncSetAttribute(thr_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, kCandCap * 8));
    IHT_CUDA_CHECK(cudaFuncSetAttribute(thr_onepass, cudaFuncAttributeMaxDynamicSharedMemorySize, kCandCap * 8));
    IHT_CUDA_CHECK(cudaFuncSetAttribute(thr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    IHT_CUDA_CHECK(cudaFuncSetAttribute(thr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kClusterSlice * 4 + kClWarps * kWarpCand * 16));
    g_thr_attr = true;
  }
  return IHT_OK;
}

// Grid path (T1 - T3 over every SM) or one cluster launch: the cluster holds at most
// kClusterMaxN a-values; a single large problem (N >= kGridSelMinN) spreads over all SMs
// instead of CL <= 8 (config 4, N = 262144: 22.5 us in the cluster).  IHT_THR_MULTI=1 forces
// the grid path, =2 the cluster path where it fits (profiling).
constexpr int64_t kGridSelMinN = 131072;
// Grid path: the one-launch select (thr_onepass, default, when its tiles fit the device at once)
// or T1 - T3 (IHT_THR_ONEPASS=0, profiling, or too many tiles).
static bool thr_onepass_on() {
  static int env = -1;
  if (env < 0) env = getenv("IHT_THR_ONEPASS") ? atoi(getenv("IHT_THR_ONEPASS")) : 1;
  return env != 0;
}
// CTAs of thr_onepass that fit the device at once (its grid barrier needs them co-resident).
static int64_t thr_onepass_capacity() {
  static int64_t cap = -1;
  if (cap < 0) {
    int dev = 0, sms = 0, per = 0;
    if (thr_attrs() != IHT_OK || cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, thr_onepass, kOpThreads, (size_t)kCandCap * 8) !=
            cudaSuccess)
      per = 0;
    cap = (int64_t)sms * per;
  }
  return cap;
}
static bool thr_grid_path(int64_t N, int nrhs) {
  static int env = -1;
  if (env < 0) env = getenv("IHT_THR_MULTI") ? atoi(getenv("IHT_THR_MULTI")) : 0;
  if (N > kClusterMaxN || env == 1) return true;
  if (env == 2) return false;
  return nrhs == 1 && N >= kGridSelMinN;
}

static int threshold_impl(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                          const float* g, int nparts, float gsigma, float* gout, float mu, const float* mu_dev,
                          int32_t s, int64_t N, int64_t col_offset, int32_t nrhs, int32_t* out_idx, float* out_val,
                          int32_t ldo, int32_t* out_nnz, void* ws, int64_t ws_bytes, void* stream,
                          bool ws_prezeroed);

int iht_threshold_batched_mu(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                             const float* g, float mu, const float* mu_dev, int32_t s, int64_t N, int64_t col_offset,
                             int32_t nrhs, int32_t* out_idx, float* out_val, int32_t ldo, int32_t* out_nnz, void* ws,
                             int64_t ws_bytes, void* stream) {
  return threshold_impl(x_idx, x_val, x_nnz, ldx, g, 0, 1.0f, nullptr, mu, mu_dev, s, N, col_offset, nrhs, out_idx,
                        out_val, ldo, out_nnz, ws, ws_bytes, stream, true);   // the solver's workspace
}

int iht_threshold_bounded(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                          const float* g, float mu, const unsigned int* bkey, int32_t s, int64_t N, int32_t nrhs,
                          const int32_t* cidx, const float* cval, int* ccnt, int32_t ccap, int* done, int* stats,
                          int32_t* out_idx, float* out_val, int32_t ldo, int32_t* out_nnz, void* ws, int64_t ws_bytes,
                          void* stream) {
  if (!iht_threshold_bounded_applies(N, s, nrhs) || cidx == nullptr || cval == nullptr || ccnt == nullptr ||
      done == nullptr || bkey == nullptr || ccap <= 0 || x_nnz == nullptr || g == nullptr || ldx < 0 || ldo < s)
    return IHT_EINVAL;
  if (!isfinite(mu)) return IHT_EDOMAIN;
  if (ws == nullptr || ws_bytes < thr_ws_layout(N, nrhs, nullptr, nullptr)) return IHT_EINVAL;
  const int32_t max_nnz = ldx < s ? ldx : s;
  ThrWs w{};
  thr_ws_layout(N, nrhs, static_cast<char*>(ws), &w);   // the full select's a, list and packed buffers
  IHT_CUDA_CHECK(launch_pdl(thr_bounded_select, dim3(nrhs), dim3(kBsThreads), 0, (cudaStream_t)stream, x_idx, x_val,
                            x_nnz, max_nnz, ldx, g, mu, bkey, s, N, cidx, cval, ccnt, (int)ccap, out_idx, out_val, ldo,
                            out_nnz, done, stats, w.a, w.cidx, reinterpret_cast<int32_t*>(w.cval),
                            (int64_t)(w.body_stride / 4)));
  return IHT_OK;
}

bool iht_threshold_bounded_applies(int64_t N, int32_t s, int32_t nrhs) {
  return !thr_grid_path(N, nrhs) && s > 0 && s <= kBsMaxS && (int64_t)s < N && nrhs > 0 && nrhs <= 65535;
}

int iht_threshold_parts(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                        const float* g, int nparts, float gsigma, float* gout, float mu, int32_t s, int64_t N,
                        int32_t* out_idx, float* out_val, int32_t ldo, int32_t* out_nnz, void* ws, int64_t ws_bytes,
                        void* stream) {
  if (nparts < 0) return IHT_EUNSUPPORTED;
  return threshold_impl(x_idx, x_val, x_nnz, ldx, g, nparts, gsigma, gout, mu, nullptr, s, N, 0, 1, out_idx, out_val,
                        ldo, out_nnz, ws, ws_bytes, stream, true);
}

static int threshold_impl(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                          const float* g, int nparts, float gsigma, float* gout, float mu, const float* mu_dev,
                          int32_t s, int64_t N, int64_t col_offset, int32_t nrhs, int32_t* out_idx, float* out_val,
                          int32_t ldo, int32_t* out_nnz, void* ws, int64_t ws_bytes, void* stream,
                          bool ws_prezeroed) {
  if (x_nnz == nullptr || g == nullptr || out_idx == nullptr || out_val == nullptr || out_nnz == nullptr ||
      s < 0 || N <= 0 || N > 0x7FFFFFFFll || nrhs <= 0 || nrhs > 65535 || ldo < s || ldx < 0 ||
      col_offset < 0 || col_offset + N > 0x7FFFFFFFll)
    return IHT_EINVAL;
  if (ldx > 0 && (x_idx == nullptr || x_val == nullptr)) return IHT_EINVAL;
  if (ws == nullptr || ws_bytes < thr_ws_layout(N, nrhs, nullptr, nullptr)) return IHT_EINVAL;
  if (!isfinite(mu)) return IHT_EDOMAIN;
  int rc;
  if ((rc = thr_attrs()) != IHT_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // max_nnz: the caller's x arrays hold at most min(ldx, s) entries (x is an H_s output)
  const int32_t max_nnz = ldx < s ? ldx : s;
  if (!thr_grid_path(N, nrhs)) {
    int CL = 1;
    while ((int64_t)CL * kClusterSlice < N) CL *= 2;
    // spread small problems too: up to ~2 CTAs per SM while slices stay >= 4096 a-values
    // more, smaller slices while that keeps <= 1 CTA per SM and >= 4096 a-values per CTA
    // (measured: 2 CTAs per SM or clusters of 16 are slower -- more cluster barriers)
    while (CL < kClusterMax && (int64_t)CL * 2 * nrhs <= 148 && N / (2 * CL) >= 4096) CL *= 2;
    {
      static int cl_env = -1;                        // profiling override (IHT_THR_CL = 1, 2, 4, 8)
      if (cl_env < 0) cl_env = getenv("IHT_THR_CL") ? atoi(getenv("IHT_THR_CL")) : 0;
      if (cl_env > 0 && (int64_t)cl_env * kClusterSlice >= N) CL = cl_env;
    }
    const int slice = (int)(((N + CL - 1) / CL + 31) / 32 * 32);   // 16-byte aligned slices
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(CL, nrhs);
    lc.blockDim = dim3(kClThreads);
    lc.dynamicSmemBytes = (size_t)slice * 4 + (size_t)kClWarps * kWarpCand * 16;
    lc.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see pdl_wait
    at[1].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 2;
    IHT_CUDA_CHECK(cudaLaunchKernelEx(&lc, thr_cluster_kernel, x_idx, x_val, x_nnz, max_nnz, ldx, g, mu, mu_dev, s,
                                      N, col_offset, slice, out_idx, out_val, ldo, out_nnz, thr_probe(), nparts,
                                      gsigma, gout, thr_timeline()));
    if (thr_timeline()) {   // profiling: per-phase times of ranks 0, 1 of snapshot 0 (stderr)
      static long long h[32];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, thr_timeline(), sizeof(h), cudaMemcpyDeviceToHost);
      for (int c = 0; c < 2 && c < CL; ++c) {
        fprintf(stderr, "thr CL=%d rank %d ns:", CL, c);
        for (int k = 1; k < 8; ++k) fprintf(stderr, " %lld", h[c * 16 + k] > 0 ? h[c * 16 + k] - h[c * 16] : -1);
        fprintf(stderr, "\n");
      }
      cudaMemset(thr_timeline(), 0, sizeof(h));
    }
    return IHT_OK;
  }
  ThrWs w{};
  thr_ws_layout(N, nrhs, static_cast<char*>(ws), &w);
  // the histogram + flags header is zero on entry: T3 zeroes it for the next call; a cold
  // workspace (standalone calls) is zeroed here
  if (!ws_prezeroed) IHT_CUDA_CHECK(cudaMemsetAsync(ws, 0, nrhs * thr_hdr_bytes(), st));
  const unsigned tiles = (unsigned)((N + kTile - 1) / kTile);
  if (thr_onepass_on() && tiles <= (unsigned)kOpMaxTiles && (int64_t)tiles * nrhs <= thr_onepass_capacity()) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(tiles, nrhs);
    lc.blockDim = dim3(kOpThreads);
    lc.dynamicSmemBytes = (size_t)kCandCap * 8;
    lc.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;                        // grid barrier: all CTAs co-resident
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see pdl_wait
    at[1].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 2;
    IHT_CUDA_CHECK(cudaLaunchKernelEx(&lc, thr_onepass, x_idx, x_val, x_nnz, max_nnz, ldx, g, mu, mu_dev, s, N,
                                      col_offset, w, nparts, gsigma, gout, out_idx, out_val, ldo, out_nnz));
    return IHT_OK;
  }
  IHT_CUDA_CHECK(launch_pdl(thr_update_hist, dim3(tiles, nrhs), dim3(kTileThreads), 0, st, x_idx, x_val, x_nnz,
                            max_nnz, ldx, g, mu, mu_dev, N, col_offset, w, nparts, gsigma, gout));
  IHT_CUDA_CHECK(launch_pdl(thr_candidates, dim3(tiles, nrhs), dim3(kTileThreads), 0, st, s, N, col_offset, w));
  IHT_CUDA_CHECK(launch_pdl(thr_select, dim3(nrhs), dim3(kThrThreads), (size_t)kCandCap * 8, st, x_nnz, s, N,
                            col_offset, w, out_idx, out_val, ldo, out_nnz));
  return IHT_OK;
}

extern "C" int iht_threshold_batched(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz, int32_t ldx,
                                     const float* g, float mu, int32_t s, int64_t N, int64_t col_offset,
                                     int32_t nrhs, int32_t* out_idx, float* out_val, int32_t ldo,
                                     int32_t* out_nnz, void* ws, int64_t ws_bytes, void* stream) {
  return threshold_impl(x_idx, x_val, x_nnz, ldx, g, 0, 1.0f, nullptr, mu, nullptr, s, N, col_offset, nrhs, out_idx,
                        out_val, ldo, out_nnz, ws, ws_bytes, stream, false);   // caller's (cold) workspace
}

int iht_threshold_launches(int64_t N) {
  if (!thr_grid_path(N, 1)) return 1;
  const int64_t tiles = (N + kTile - 1) / kTile;
  return thr_onepass_on() && tiles <= kOpMaxTiles && tiles <= thr_onepass_capacity() ? 1 : 3;
}

extern "C" int iht_threshold(const int32_t* x_idx, const float* x_val, const int32_t* x_nnz,
                             const float* g, float mu, int32_t s, int64_t N, int32_t* out_idx,
                             float* out_val, int32_t* out_nnz, void* ws, int64_t ws_bytes,
                             void* stream) {
  return iht_threshold_batched(x_idx, x_val, x_nnz, s, g, mu, s, N, 0, 1, out_idx, out_val, s > 0 ? s : 0,
                               out_nnz, ws, ws_bytes, stream);
}

extern "C" int iht_merge_candidates(const int32_t* cand_idx, const float* cand_val, const int32_t* cand_nnz,
                                    int64_t shard_stride, int32_t P, int32_t s, int32_t nrhs, int32_t* out_idx,
                                    float* out_val, int32_t* out_nnz, void* stream) {
  if (cand_idx == nullptr || cand_val == nullptr || cand_nnz == nullptr || out_idx == nullptr ||
      out_val == nullptr || out_nnz == nullptr || P <= 0 || P > 1024 || s < 0 || nrhs <= 0 || nrhs > 65535 ||
      (P > 1 && shard_stride < (int64_t)nrhs * s))
    return IHT_EINVAL;
  if ((int64_t)P * s > kCandCap) return IHT_EUNSUPPORTED;
  int rc;
  if ((rc = thr_attrs()) != IHT_OK) return rc;
  thr_merge<<<nrhs, kThrThreads, kCandCap * 8, (cudaStream_t)stream>>>(cand_idx, cand_val, cand_nnz, shard_stride, P, s, nrhs,
                                                                      out_idx, out_val, out_nnz);
  IHT_LAUNCH_CHECK();
  return IHT_OK;
}
