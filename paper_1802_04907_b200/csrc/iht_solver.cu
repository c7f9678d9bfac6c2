// (b) the solver: Algorithm 1 with fixed step mu over a pool of K
// quantised copies, the n* iterations captured once into a CUDA graph; plus the
// size queries, error strings and the NCCL communicator (row-sharded multi-GPU,
// north star: "each GPU computes its partial g, and an NCCL all-reduce over NVLink
// sums the length-N g, after which thresholding is replicated").
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>   // types and enum values only: NCCL itself is loaded with dlopen
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "iht_adaptive.cuh"
#include "iht_internal.cuh"

// ------------------------------------------------------------------ errors
static thread_local char g_last_cuda_error[512];

void iht_set_last_cuda_error(cudaError_t e, const char* expr, const char* file, int line) {
  snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s (%s) at %s:%d: %s", cudaGetErrorName(e),
           expr, file, line, cudaGetErrorString(e));
}

extern "C" const char* iht_last_cuda_error(void) { return g_last_cuda_error; }

extern "C" const char* iht_strerror(int status) {
  switch (status) {
    case IHT_OK: return "IHT_OK";
    case IHT_EINVAL: return "IHT_EINVAL: invalid argument";
    case IHT_EDOMAIN: return "IHT_EDOMAIN: non-finite value";
    case IHT_ECUDA: return "IHT_ECUDA: CUDA runtime error";
    case IHT_ENCCL: return "IHT_ENCCL: NCCL unavailable or failed";
    case IHT_ENOMEM: return "IHT_ENOMEM: out of device memory";
    case IHT_EUNSUPPORTED: return "IHT_EUNSUPPORTED: configuration not implemented";
    default: return "IHT_E?: unknown status";
  }
}

extern "C" int iht_abi_version(void) { return IHT_ABI_VERSION; }

// ------------------------------------------------------------------ sizes
extern "C" int64_t iht_rows_pad(int64_t rows) { return rows <= 0 ? 0 : iht::rows_pad(rows); }
extern "C" int64_t iht_strip_bytes(int64_t rows, int planes, int bits) {
  if (rows <= 0 || (planes != 1 && planes != 2) || (bits != 2 && bits != 4 && bits != 8)) return -1;
  return (int64_t)planes * iht::rows_pad(rows) * bits / 8;
}
extern "C" int64_t iht_qmat_bytes(int64_t rows, int64_t cols, int planes, int bits) {
  const int64_t sb = iht_strip_bytes(rows, planes, bits);
  return (sb < 0 || cols <= 0) ? -1 : sb * ((cols + 15) / 16 * 16);
}
extern "C" int64_t iht_vec_len(int64_t rows, int planes) {
  if (rows <= 0 || (planes != 1 && planes != 2)) return -1;
  return (int64_t)planes * iht::rows_pad(rows);
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.ReduceScatter = (decltype(g_nccl.ReduceScatter))dlsym(h, "ncclReduceScatter");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce &&
              g_nccl.AllGather && g_nccl.ReduceScatter;
  return g_nccl.ok;
}
}  // namespace

struct iht_comm {
  ncclComm_t comm;
  int rank, world;
};

extern "C" int iht_comm_unique_id(void* id128) {
  if (id128 == nullptr) return IHT_EINVAL;
  if (!load_nccl()) return IHT_ENCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return IHT_ENCCL;
  memcpy(id128, &id, sizeof(id));
  return IHT_OK;
}

extern "C" int iht_comm_create(int rank, int world, const void* id128, int device, iht_comm** out) {
  if (out == nullptr || id128 == nullptr || world < 1 || rank < 0 || rank >= world) return IHT_EINVAL;
  if (!load_nccl()) return IHT_ENCCL;
  IHT_CUDA_CHECK(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  if (g_nccl.CommInitRank(&c, world, id, rank) != ncclSuccess) return IHT_ENCCL;
  *out = new iht_comm{c, rank, world};
  return IHT_OK;
}

extern "C" int iht_comm_destroy(iht_comm* comm) {
  if (comm == nullptr) return IHT_OK;
  if (g_nccl.ok) g_nccl.CommDestroy(comm->comm);
  delete comm;
  return IHT_OK;
}

extern "C" int iht_comm_allreduce(iht_comm* comm, float* buf, int64_t count, int op_max, void* stream) {
  if (comm == nullptr || buf == nullptr || count < 0) return IHT_EINVAL;
  if (g_nccl.AllReduce(buf, buf, (size_t)count, ncclFloat32, op_max ? ncclMax : ncclSum, comm->comm,
                       (cudaStream_t)stream) != ncclSuccess)
    return IHT_ENCCL;
  return IHT_OK;
}

extern "C" int iht_comm_allgather(iht_comm* comm, const void* send, void* recv, int64_t bytes, void* stream) {
  if (comm == nullptr || send == nullptr || recv == nullptr || bytes < 0) return IHT_EINVAL;
  if (g_nccl.AllGather(send, recv, (size_t)bytes, ncclUint8, comm->comm, (cudaStream_t)stream) != ncclSuccess)
    return IHT_ENCCL;
  return IHT_OK;
}

extern "C" int iht_comm_reduce_scatter(iht_comm* comm, const float* send, float* recv, int64_t recv_count,
                                       void* stream) {
  if (comm == nullptr || send == nullptr || recv == nullptr || recv_count < 0) return IHT_EINVAL;
  if (g_nccl.ReduceScatter(send, recv, (size_t)recv_count, ncclFloat32, ncclSum, comm->comm, (cudaStream_t)stream) !=
      ncclSuccess)
    return IHT_ENCCL;
  return IHT_OK;
}

// ------------------------------------------------------------------ solver
// Modes (fixed at create):
//   single  (nrhs <= 1): GEMV adjoint; with a communicator of world P the rows are
//           sharded (north star).  Fixed step: g is REDUCE-SCATTERED (rank p owns columns
//           [p N/P, (p+1) N/P)), each rank selects the local top-s of its columns, the P
//           candidate lists are all-gathered and merged into the global H_s (SURVEY 8(e)'s
//           "reduce-scatter g, then a sharded select, then an all-gather of <= s P
//           candidates": half the bytes of an all-reduce and 1/P of the select).  The
//           adaptive step all-reduces g (its norms need g on the whole support).
//   batched (nrhs = B > 1, BASELINE config 5): per-snapshot sparse forward, tcgen05
//           adjoint (chunks of <= 64 snapshots inside iht_adjoint_batched), per-snapshot
//           H_s; with a communicator the COLUMNS are sharded: forward partials
//           all-reduced, local top-s candidates all-gathered and merged.

struct iht_solver {
  std::vector<iht_qmat> pool;          // fresh mode: one descriptor-only entry (codes NULL)
  bool fresh = false;                  // NEXT-2: copies drawn on the fly from fm
  iht_fmat fm{};
  iht_config cfg;
  int64_t rows, N, vlen;
  int planes;
  int B = 1;                           // snapshots
  bool batched = false, rowshard = false, colshard = false;
  bool shardsel = false;               // row shards: reduce-scatter g + sharded select + merge
  int64_t nloc = 0, col0 = 0;          // this rank's columns of g when shardsel
  int world = 1, rank = 0;
  // device buffers (one allocation)
  void* block = nullptr;
  float *y = nullptr, *c_y = nullptr, *yhat = nullptr, *r = nullptr, *g = nullptr;
  void *ws_adj = nullptr, *ws_thr = nullptr, *ws_fwd = nullptr;
  int64_t ws_adj_bytes = 0, ws_thr_bytes = 0, ws_fwd_bytes = 0;
  int32_t* xs_idx = nullptr;   // [nslots][B][s]
  float* xs_val = nullptr;     // [nslots][B][s]
  int32_t* xs_nnz = nullptr;   // [nslots][B]
  // adaptive step (step_mode 1): per snapshot mu, loop state (accepted, shrinks), norms,
  // Gamma^[1], the support-restricted gradient, the difference x' - x and a scratch vector
  float *ad_mu = nullptr, *ad_num = nullptr, *ad_den = nullptr, *ad_dnum = nullptr, *ad_dden = nullptr;
  int32_t *ad_state = nullptr, *ad_pending = nullptr;
  int32_t *ad_gi = nullptr, *ad_gn = nullptr, *ad_xgi = nullptr, *ad_xgn = nullptr, *ad_di = nullptr, *ad_dn = nullptr;
  float *ad_gv = nullptr, *ad_xgv = nullptr, *ad_dv = nullptr, *ad_tmp = nullptr;
  float* ad_mu_rec = nullptr;      // [n_iter][B]
  int32_t* ad_shr_rec = nullptr;   // [n_iter][B]
  cudaStream_t body_stream = nullptr;
  int32_t* cand_send = nullptr;   // column shards: idx [B][s] | val [B][s] | nnz [B]
  int32_t* cand_recv = nullptr;   // [P][same]
  int64_t cand_words = 0;
  int nslots = 0;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaEvent_t> ev;   // profile: [2 * n_iter] start/stop of each adjoint
  int64_t launches = 0;
  int final_slot = 0;
  iht_fused_state* fused = nullptr;    // the whole loop as one persistent kernel (iht_fused.cu)
  // bounded select (batched, fixed step): epilogue candidate lists + per-snapshot decided flags
  bool bounded = false;
  float bound = 0.7f;
  int32_t* bc_idx = nullptr;   // [B][kBcCap]
  float* bc_val = nullptr;     // [B][kBcCap]
  int* bc_cnt = nullptr;       // [B] (zeroed at create, reset by the select kernel)
  int* bc_done = nullptr;      // [B]
  unsigned int* bc_bkey = nullptr;   // [B] bound keys
  int* bc_stats = nullptr;     // [4] decided, fallen back, sum / max list size (IHT_BOUNDED_STATS)
};

// Candidate slots per snapshot written by the batched epilogue (more: the select falls back).
static constexpr int kBcCap = 1024;

// IHT_BOUNDED=0 turns the bounded select off (A/B and the bit-identity test); IHT_BOUND sets
// the bound factor (default 0.7 x the smallest kept |x|; measured at config 5, r02 g52/g54:
// 0.5 -> lists of ~208 and slower ranking, 0.9 -> 5 % of the snapshot-iterations fall back,
// 0.7 / 0.8 -> 16.5k / 16.4k iter/s against 15.1k without).  Read at every solver create.
static bool bounded_enabled() {
  const char* e = getenv("IHT_BOUNDED");
  return e == nullptr || atoi(e) != 0;
}
static float bounded_factor() {
  const char* e = getenv("IHT_BOUND");
  const float f = e ? (float)atof(e) : 0.7f;
  return f > 0.0f && f < 1.0f ? f : 0.7f;
}

// Event record that survives stream capture: inside a capture it becomes an event-record
// node of the graph (cudaEventRecordExternal), so every replay re-records it.
static cudaError_t record_event(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t err = cudaStreamIsCapturing(st, &cs);
  if (err != cudaSuccess) return err;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                                             : cudaEventRecord(e, st);
}

static int64_t& pass_dummy() {
  static thread_local int64_t d = 0;
  return d;
}

// One pass of the shrink loop (propose, compare supports, |Phi-hat_A dx|^2, decide).
static int enqueue_shrink_body(iht_solver* S, cudaStream_t st, int n, const iht_qmat& A, const int32_t* gi,
                               const int32_t* gn, const int32_t* xi, const float* xv, const int32_t* xn, int32_t* oi,
                               float* ov, int32_t* on, cudaGraphConditionalHandle h, int use_h, int64_t* L) {
  int rc;
  const int B = S->B, s = S->cfg.s;
  if ((rc = iht_threshold_batched_mu(xi, xv, xn, s, S->g, S->cfg.mu, S->ad_mu, s, S->N, 0, B, oi, ov, s, on,
                                     S->ws_thr, S->ws_thr_bytes, st)) != IHT_OK)
    return rc;
  if ((rc = ad_delta(oi, ov, on, gi, gn, s, xi, xv, xn, s, S->ad_state, S->ad_di, S->ad_dv, S->ad_dn, S->ad_dnum, B,
                     st)) != IHT_OK)
    return rc;
  if ((rc = iht_forward_batched(&A, S->ad_di, S->ad_dv, S->ad_dn, 2 * s, 2 * s, B, nullptr, S->ad_tmp, st)) !=
      IHT_OK)
    return rc;
  if ((rc = ad_norm(S->ad_tmp, S->vlen, S->ad_dden, B, st)) != IHT_OK) return rc;
  if (S->rowshard) {
    if ((rc = iht_comm_allreduce(S->cfg.comm, S->ad_dden, B, 0, st)) != IHT_OK) return rc;
  }
  if ((rc = ad_decide(S->ad_dnum, S->ad_dden, S->cfg.step_c, S->cfg.step_k, S->cfg.max_shrink, B, S->ad_mu,
                      S->ad_state, S->ad_mu_rec + (int64_t)(n - 1) * B, S->ad_shr_rec + (int64_t)(n - 1) * B, h, use_h,
                      S->ad_pending, st)) != IHT_OK)
    return rc;
  *L += iht_threshold_launches(S->N) + 4;   // threshold + delta + forward + norm + decide
  return IHT_OK;
}

// Algorithm 1's step for iteration n: Gamma, mu, then the proposal / shrink
// loop (a conditional WHILE node when captured into the graph, else a host loop).
static int enqueue_adaptive(iht_solver* S, cudaStream_t st, int n, const iht_qmat& A, const int32_t* xi,
                            const float* xv, const int32_t* xn, int32_t* oi, float* ov, int32_t* on, int64_t* L) {
  int rc;
  const int B = S->B, s = S->cfg.s;
  const int32_t *gi = xi, *gn = xn;
  if (n == 1) {   // Gamma^[1] = supp(H_s(Phi-hat_1^H y-hat)): x^[1] = 0, so H_s(g^[1])
    if ((rc = iht_threshold_batched_mu(xi, xv, xn, s, S->g, 1.0f, nullptr, s, S->N, 0, B, S->ad_gi, S->ad_gv, s, S->ad_gn,
                                    S->ws_thr, S->ws_thr_bytes, st)) != IHT_OK)
      return rc;
    gi = S->ad_gi;
    gn = S->ad_gn;
    *L += iht_threshold_launches(S->N);
  }
  if ((rc = ad_gather(S->g, S->N, 0, gi, gn, s, S->ad_xgi, S->ad_xgv, S->ad_xgn, S->ad_num, B, st)) != IHT_OK) return rc;
  if ((rc = iht_forward_batched(&A, S->ad_xgi, S->ad_xgv, S->ad_xgn, s, s, B, nullptr, S->ad_tmp, st)) != IHT_OK)
    return rc;
  if ((rc = ad_norm(S->ad_tmp, S->vlen, S->ad_den, B, st)) != IHT_OK) return rc;
  if (S->rowshard) {
    if ((rc = iht_comm_allreduce(S->cfg.comm, S->ad_den, B, 0, st)) != IHT_OK) return rc;
  }
  if ((rc = ad_step(S->ad_num, S->ad_den, S->cfg.mu, B, S->ad_mu, S->ad_state, st)) != IHT_OK) return rc;
  *L += 4;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  IHT_CUDA_CHECK(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive) {
    cudaGraph_t graph;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    IHT_CUDA_CHECK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &ndeps));
    cudaGraphConditionalHandle h;
    IHT_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    IHT_CUDA_CHECK(cudaGraphAddNode(&node, graph, deps, ndeps, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    IHT_CUDA_CHECK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    IHT_CUDA_CHECK(cudaStreamBeginCaptureToGraph(S->body_stream, body, nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeRelaxed));
    rc = enqueue_shrink_body(S, S->body_stream, n, A, gi, gn, xi, xv, xn, oi, ov, on, h, 1, L);
    cudaGraph_t tmp;
    const cudaError_t e = cudaStreamEndCapture(S->body_stream, &tmp);
    if (rc != IHT_OK) return rc;
    IHT_CUDA_CHECK(e);
  } else {
    int32_t pending = 1;
    for (int pass = 0; pending; ++pass) {
      if ((rc = enqueue_shrink_body(S, st, n, A, gi, gn, xi, xv, xn, oi, ov, on, 0, 0, pass == 0 ? L : &pass_dummy()))
          != IHT_OK)
        return rc;
      IHT_CUDA_CHECK(cudaMemcpyAsync(&pending, S->ad_pending, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      IHT_CUDA_CHECK(cudaStreamSynchronize(st));
    }
  }
  return IHT_OK;
}

// Enqueue one complete run (absmax .. last threshold) on stream st; counts launches.
static int enqueue_run(iht_solver* S, cudaStream_t st, int64_t* launches) {
  int64_t L = 0;
  int rc;
  const int64_t ycount = S->rows * S->planes;
  const int B = S->B, s = S->cfg.s;
  if ((rc = iht_absmax_batched(S->y, ycount, B, S->c_y, st)) != IHT_OK) return rc;
  L += 1;
  if (S->rowshard) {   // global max over the row shards (reading c3)
    if ((rc = iht_comm_allreduce(S->cfg.comm, S->c_y, 1, 1, st)) != IHT_OK) return rc;
  }
  const iht_qmat& q0 = S->pool[0];
  if ((rc = iht_quantize_vec_batched(S->y, S->rows, q0.row_offset, S->planes, S->cfg.b_y, S->cfg.level_mode,
                                     S->cfg.seed, S->c_y, B, S->yhat, nullptr, st)) != IHT_OK)
    return rc;
  L += 1;
  // x^[1] = 0 (reading c8): slot 0 holds x^[1]
  IHT_CUDA_CHECK(cudaMemsetAsync(S->xs_nnz, 0, sizeof(int32_t) * B, st));
  if (S->fused && S->cfg.n_iter > 0) {   // the n* iterations in one persistent kernel
    if (!S->ev.empty()) IHT_CUDA_CHECK(record_event(S->ev[0], st));
    if ((rc = iht_fused_enqueue(S->fused, st)) != IHT_OK) return rc;
    if (!S->ev.empty()) IHT_CUDA_CHECK(record_event(S->ev[1], st));
    L += 1;
    S->final_slot = S->cfg.trace ? S->cfg.n_iter : (S->cfg.n_iter & 1);
    if (launches) *launches = L;
    return IHT_OK;
  }
  const int K = (int)S->pool.size();
  const int64_t xslot = (int64_t)B * s;
  // single observation, fixed step, int8-MMA adjoint, no g all-reduce, fused threshold:
  // the adjoint's split-K partials go straight to the threshold (one launch fewer)
  const bool fuse_parts = !S->fresh && !S->batched && !S->rowshard && S->cfg.step_mode == 0 &&
                          S->cfg.adjoint_variant == 0;
  int nparts = 0;
  float gsigma = 1.0f;
  for (int n = 1; n <= S->cfg.n_iter; ++n) {
    const int in_slot = S->cfg.trace ? (n - 1) : ((n - 1) & 1);
    const int out_slot = S->cfg.trace ? n : (n & 1);
    const iht_qmat& A = S->pool[(2 * n - 2) % K];   // Phi-hat_{2n-1} (1-based), adjoint
    const iht_qmat& F = S->pool[(2 * n - 1) % K];   // Phi-hat_{2n}, forward
    const int32_t* xi = S->xs_idx + in_slot * xslot;
    const float* xv = S->xs_val + in_slot * xslot;
    const int32_t* xn = S->xs_nnz + (int64_t)in_slot * B;
    int32_t* oi = S->xs_idx + out_slot * xslot;
    float* ov = S->xs_val + out_slot * xslot;
    int32_t* on = S->xs_nnz + (int64_t)out_slot * B;
    // (a4) forward: r_b = y-hat_b - Phi-hat_F x_b  (column shards: partial, then summed)
    const float* yh = (S->colshard && S->rank != 0) ? nullptr : S->yhat;
    if (S->fresh) {
      if ((rc = iht_forward_fresh(&S->fm, 2 * n - 1, xi, xv, xn, s, S->yhat, S->r, st)) != IHT_OK) return rc;
    } else if (B == 1 && yh != nullptr) {
      // single observation: iht_forward (the row-block x column-group kernel where it applies)
      if ((rc = iht_forward(&F, xi, xv, xn, s, yh, S->r, S->ws_fwd, S->ws_fwd_bytes, st)) != IHT_OK) return rc;
    } else if ((rc = iht_forward_batched(&F, xi, xv, xn, s, s, B, yh, S->r, st)) != IHT_OK) {
      return rc;
    } else if (S->batched && getenv("IHT_DUP_FWD")) {   // profiling: the forward twice (idempotent),
      if ((rc = iht_forward_batched(&F, xi, xv, xn, s, s, B, yh, S->r, st)) != IHT_OK) return rc;   // its in-graph cost
    }
    L += 1;
    if (S->colshard) {
      if ((rc = iht_comm_allreduce(S->cfg.comm, S->r, (int64_t)B * S->vlen, 0, st)) != IHT_OK) return rc;
    }
    // (a5) adjoint
    if (!S->ev.empty()) IHT_CUDA_CHECK(record_event(S->ev[2 * (n - 1)], st));
    if (S->fresh) {
      if ((rc = iht_adjoint_fresh(&S->fm, 2 * n - 2, S->r, S->g, S->ws_adj, S->ws_adj_bytes, st)) != IHT_OK)
        return rc;
      L += 2;
    } else if (!S->batched && fuse_parts) {
      // split-K partials summed inside the fused threshold (no adjoint_reduce_kernel)
      if ((rc = iht_adjoint_parts(&A, S->r, S->g, S->ws_adj, S->ws_adj_bytes, st, &nparts, &gsigma)) != IHT_OK)
        return rc;
      L += 1;
    } else if (!S->batched) {
      if ((rc = iht_adjoint(&A, S->r, S->g, S->cfg.adjoint_variant, S->ws_adj, S->ws_adj_bytes, st)) != IHT_OK)
        return rc;
      L += (S->cfg.adjoint_variant == 0 && S->ws_adj_bytes > 0) ? 2 : 1;
    } else if (S->bounded) {
      // the epilogue also lists each snapshot's candidates for the bounded select below
      iht_cand_args ca{S->bc_idx, S->bc_val, S->bc_cnt, kBcCap, S->cfg.mu, S->bound, xv, xn, s, s, S->bc_bkey};
      if ((rc = iht_adjoint_batched_cand(&A, S->r, B, S->g, S->ws_adj, S->ws_adj_bytes, st, &ca)) != IHT_OK)
        return rc;
      L += 2 * ((B + 63) / 64);
    } else {
      if ((rc = iht_adjoint_batched(&A, S->r, B, S->g, S->ws_adj, S->ws_adj_bytes, st)) != IHT_OK) return rc;
      L += 2 * ((B + 63) / 64);
    }
    if (!S->ev.empty()) IHT_CUDA_CHECK(record_event(S->ev[2 * (n - 1) + 1], st));
    if (S->shardsel) {          // in place: rank p's summed slice lands at g + p N/P
      if ((rc = iht_comm_reduce_scatter(S->cfg.comm, S->g, S->g + S->col0, S->nloc, st)) != IHT_OK) return rc;
    } else if (S->rowshard) {
      if ((rc = iht_comm_allreduce(S->cfg.comm, S->g, S->N, 0, st)) != IHT_OK) return rc;
    }
    // (a6) update + H_s
    if (S->cfg.step_mode == 1) {
      if ((rc = enqueue_adaptive(S, st, n, A, xi, xv, xn, oi, ov, on, &L)) != IHT_OK) return rc;
    } else if (nparts > 0) {
      if ((rc = iht_threshold_parts(xi, xv, xn, s, static_cast<const float*>(S->ws_adj), nparts, gsigma, S->g,
                                    S->cfg.mu, s, S->N, oi, ov, s, on, S->ws_thr, S->ws_thr_bytes, st)) != IHT_OK)
        return rc;
      L += 1;
    } else if (S->shardsel) {
      // local top-s of this rank's columns (global indices), all-gathered, merged
      int32_t* ci = S->cand_send;
      float* cv = reinterpret_cast<float*>(S->cand_send + xslot);
      int32_t* cn = S->cand_send + 2 * xslot;
      if ((rc = iht_threshold_batched_mu(xi, xv, xn, s, S->g + S->col0, S->cfg.mu, nullptr, s, S->nloc, S->col0, 1, ci, cv, s,
                                      cn, S->ws_thr, S->ws_thr_bytes, st)) != IHT_OK)
        return rc;
      L += iht_threshold_launches(S->nloc);
      if ((rc = iht_comm_allgather(S->cfg.comm, S->cand_send, S->cand_recv, S->cand_words * 4, st)) != IHT_OK)
        return rc;
      if ((rc = iht_merge_candidates(S->cand_recv, reinterpret_cast<const float*>(S->cand_recv + xslot),
                                     S->cand_recv + 2 * xslot, S->cand_words, S->world, s, 1, oi, ov, on, st)) !=
          IHT_OK)
        return rc;
      L += 1;
    } else if (S->bounded) {
      if ((rc = iht_threshold_bounded(xi, xv, xn, s, S->g, S->cfg.mu, S->bc_bkey, s, S->N, B, S->bc_idx, S->bc_val,
                                      S->bc_cnt, kBcCap, S->bc_done, S->bc_stats, oi, ov, s, on, S->ws_thr,
                                      S->ws_thr_bytes, st)) != IHT_OK)
        return rc;
      L += 1;
    } else if (!S->colshard) {
      if ((rc = iht_threshold_batched_mu(xi, xv, xn, s, S->g, S->cfg.mu, nullptr, s, S->N, 0, B, oi, ov, s, on, S->ws_thr,
                                      S->ws_thr_bytes, st)) != IHT_OK)
        return rc;
      L += iht_threshold_launches(S->N);
    } else {
      int32_t* ci = S->cand_send;
      float* cv = reinterpret_cast<float*>(S->cand_send + xslot);
      int32_t* cn = S->cand_send + 2 * xslot;
      if ((rc = iht_threshold_batched_mu(xi, xv, xn, s, S->g, S->cfg.mu, nullptr, s, S->N, q0.col_offset, B, ci, cv, s, cn,
                                      S->ws_thr, S->ws_thr_bytes, st)) != IHT_OK)
        return rc;
      L += iht_threshold_launches(S->N);
      if ((rc = iht_comm_allgather(S->cfg.comm, S->cand_send, S->cand_recv, S->cand_words * 4, st)) != IHT_OK)
        return rc;
      if ((rc = iht_merge_candidates(S->cand_recv, reinterpret_cast<const float*>(S->cand_recv + xslot),
                                     S->cand_recv + 2 * xslot, S->cand_words, S->world, s, B, oi, ov, on, st)) !=
          IHT_OK)
        return rc;
      L += 1;
    }
    S->final_slot = out_slot;
  }
  if (S->cfg.n_iter == 0) S->final_slot = 0;
  if (launches) *launches = L;
  return IHT_OK;
}

static int solver_create_impl(const iht_qmat* pool, int K, const iht_config* cfg, const iht_fmat* fm,
                              iht_solver** out);

static bool fused_disabled_by_env() {   // profiling switch: IHT_FUSED=0 keeps the per-step kernels
  static int v = -1;
  if (v < 0) v = (getenv("IHT_FUSED") && atoi(getenv("IHT_FUSED")) == 0) ? 1 : 0;
  return v == 1;
}

extern "C" int iht_solver_create(const iht_qmat* pool, int K, const iht_config* cfg, iht_solver** out) {
  return solver_create_impl(pool, K, cfg, nullptr, out);
}

extern "C" int iht_solver_create_fresh(const iht_fmat* F, const iht_config* cfg, iht_solver** out) {
  if (F == nullptr || cfg == nullptr || out == nullptr || F->phi == nullptr) return IHT_EINVAL;
  if (cfg->nrhs > 1 || cfg->step_mode != 0) return IHT_EUNSUPPORTED;   // single observation, fixed step
  if (iht_adjoint_fresh_ws_bytes(F) < 0) return IHT_EINVAL;
  iht_qmat d{};                          // descriptor-only pool entry: shape of the copies
  d.rows = F->rows;
  d.cols = F->cols;
  d.row_offset = F->row_offset;
  d.planes = F->planes;
  d.bits = F->bits;
  d.level_mode = F->level_mode;
  d.seed = F->seed;
  d.scale_c = F->scale_c;
  d.strip_bytes = iht_strip_bytes(F->rows, F->planes, F->bits);
  return solver_create_impl(&d, 1, cfg, F, out);
}

static int solver_create_impl(const iht_qmat* pool, int K, const iht_config* cfg, const iht_fmat* fm,
                              iht_solver** out) {
  if (pool == nullptr || K < 1 || cfg == nullptr || out == nullptr) return IHT_EINVAL;
  if (cfg->s < 0 || cfg->n_iter < 0 || !isfinite(cfg->mu) || cfg->nrhs < 0) return IHT_EINVAL;
  if (cfg->b_y < 2 || cfg->b_y > 8 || (cfg->level_mode != 0 && cfg->level_mode != 1)) return IHT_EINVAL;
  if (cfg->adjoint_variant != 0 && cfg->adjoint_variant != 1) return IHT_EINVAL;
  const iht_qmat& q0 = pool[0];
  for (int k = 0; k < K && fm == nullptr; ++k) {
    const iht_qmat& q = pool[k];
    if (q.codes == nullptr || q.rows != q0.rows || q.cols != q0.cols || q.planes != q0.planes ||
        q.bits != q0.bits || q.row_offset != q0.row_offset || q.col_offset != q0.col_offset ||
        q.strip_bytes != iht_strip_bytes(q.rows, q.planes, q.bits))
      return IHT_EINVAL;
  }
  const int world = cfg->comm ? cfg->comm->world : 1;
  const int B = cfg->nrhs > 1 ? cfg->nrhs : 1;
  const bool batched = B > 1;
  if (batched && cfg->adjoint_variant != 0) return IHT_EUNSUPPORTED;
  if (batched && cfg->comm && (q0.row_offset != 0 || q0.col_offset != (int64_t)cfg->comm->rank * q0.cols))
    return IHT_EINVAL;   // column shards of equal width, rank-ordered
  if (!batched && q0.col_offset != 0) return IHT_EINVAL;
  const int64_t Mg = batched ? q0.rows : q0.rows * world;          // global rows
  const int64_t Ng = batched ? q0.cols * world : q0.cols;          // global columns
  if (cfg->s > Mg * q0.planes || cfg->s > Ng) return IHT_EINVAL;   // s <= M
  if (batched && cfg->comm && (int64_t)world * cfg->s > 8192) return IHT_EUNSUPPORTED;
  if (cfg->step_mode != 0 && cfg->step_mode != 1) return IHT_EINVAL;
  if (cfg->step_mode == 1) {
    if (batched && cfg->comm) return IHT_EUNSUPPORTED;            // column-sharded adaptive: not built
    if (!(cfg->step_c > 0.0f && cfg->step_c < 1.0f) || !(cfg->step_k * (1.0f - cfg->step_c) > 1.0f) ||
        cfg->max_shrink < 0 || !(cfg->mu > 0.0f))
      return IHT_EINVAL;                                             // k > 1/(1-c)
  }
  iht_solver* S = new iht_solver();
  S->pool.assign(pool, pool + K);
  if (fm) {
    S->fresh = true;
    S->fm = *fm;
  }
  S->cfg = *cfg;
  S->rows = q0.rows;
  S->N = q0.cols;
  S->planes = q0.planes;
  S->vlen = iht_vec_len(q0.rows, q0.planes);
  S->B = B;
  S->batched = batched;
  S->world = world;
  S->rank = cfg->comm ? cfg->comm->rank : 0;
  S->rowshard = !batched && cfg->comm != nullptr;  // any world size (world 1 exercises the same path)
  S->colshard = batched && cfg->comm != nullptr;   // any world size (world 1 exercises the same path)
  S->shardsel = S->rowshard && cfg->step_mode == 0 && q0.cols % world == 0 && (int64_t)world * cfg->s <= 8192;
  S->nloc = S->shardsel ? q0.cols / world : q0.cols;
  S->col0 = S->shardsel ? (int64_t)S->rank * S->nloc : 0;
  // NCCL kernels may not sit inside a conditional body graph: the adaptive row-sharded
  // run drives its shrink loop from the host
  if (cfg->step_mode == 1 && S->rowshard) S->cfg.use_graph = 0;
  S->ws_adj_bytes = fm ? iht_adjoint_fresh_ws_bytes(fm)
                      : batched ? iht_adjoint_batched_ws_bytes(&q0, B) : iht_adjoint_ws_bytes(&q0);
  S->ws_thr_bytes = iht_threshold_batched_ws_bytes(S->N, cfg->s, B);
  S->ws_fwd_bytes = (!fm && !batched) ? iht_forward_ws_bytes(&q0, cfg->s) : 0;
  S->nslots = cfg->trace ? cfg->n_iter + 1 : 2;
  const int s = cfg->s > 0 ? cfg->s : 1;
  S->cand_words = (S->colshard || S->shardsel) ? 2 * (int64_t)B * s + B : 0;
  auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
  const int64_t ycount = q0.rows * q0.planes;
  const int64_t sz_y = al((int64_t)B * ycount * 4), sz_c = al((int64_t)B * 4),
                sz_v = al((int64_t)B * S->vlen * 4), sz_g = al((int64_t)B * S->N * 4),
                sz_wa = al(S->ws_adj_bytes), sz_wt = al(S->ws_thr_bytes), sz_wf = al(S->ws_fwd_bytes),
                sz_xi = al((int64_t)S->nslots * B * s * 4), sz_xv = al((int64_t)S->nslots * B * s * 4),
                sz_xn = al((int64_t)S->nslots * B * 4), sz_cs = al(S->cand_words * 4),
                sz_cr = al(S->cand_words * 4 * world);
  const bool ad = cfg->step_mode == 1;
  const int64_t sz_b4 = al((int64_t)B * 4), sz_bs = al((int64_t)B * s * 4), sz_b2s = al((int64_t)B * 2 * s * 4),
                sz_rec = al((int64_t)(cfg->n_iter > 0 ? cfg->n_iter : 1) * B * 4);
  const int64_t sz_ad = ad ? (6 * sz_b4 + al((int64_t)B * 8) + 2 * sz_bs + sz_b4 + 2 * sz_bs + sz_b4 + 2 * sz_b2s +
                              sz_b4 + sz_v + 2 * sz_rec)
                           : 0;
  S->bounded = batched && !S->colshard && !fm && cfg->step_mode == 0 && B <= 64 &&
               iht_threshold_bounded_applies(S->N, cfg->s, B) && bounded_enabled();
  S->bound = bounded_factor();
  const int64_t sz_bc = S->bounded ? 2 * al((int64_t)B * kBcCap * 4) + 3 * sz_b4 + al(16) : 0;
  const int64_t total = sz_y + sz_c + 2 * sz_v + sz_g + sz_wa + sz_wt + sz_wf + sz_xi + sz_xv + sz_xn +
                        ((S->colshard || S->shardsel) ? sz_cs + sz_cr : 0) + sz_ad + sz_bc;
  if (cudaMalloc(&S->block, total) != cudaSuccess) {
    delete S;
    return IHT_ENOMEM;
  }
  char* p = static_cast<char*>(S->block);
  S->y = reinterpret_cast<float*>(p); p += sz_y;
  S->c_y = reinterpret_cast<float*>(p); p += sz_c;
  S->yhat = reinterpret_cast<float*>(p); p += sz_v;
  S->r = reinterpret_cast<float*>(p); p += sz_v;
  S->g = reinterpret_cast<float*>(p); p += sz_g;
  S->ws_adj = S->ws_adj_bytes ? p : nullptr; p += sz_wa;
  S->ws_thr = p; p += sz_wt;
  S->ws_fwd = S->ws_fwd_bytes ? p : nullptr; p += sz_wf;   // zeroed below: the arrival counters start at 0
  S->xs_idx = reinterpret_cast<int32_t*>(p); p += sz_xi;
  S->xs_val = reinterpret_cast<float*>(p); p += sz_xv;
  S->xs_nnz = reinterpret_cast<int32_t*>(p); p += sz_xn;
  if (S->colshard || S->shardsel) {
    S->cand_send = reinterpret_cast<int32_t*>(p); p += sz_cs;
    S->cand_recv = reinterpret_cast<int32_t*>(p); p += sz_cr;
  }
  if (ad) {
    S->ad_mu = reinterpret_cast<float*>(p); p += sz_b4;
    S->ad_num = reinterpret_cast<float*>(p); p += sz_b4;
    S->ad_den = reinterpret_cast<float*>(p); p += sz_b4;
    S->ad_dnum = reinterpret_cast<float*>(p); p += sz_b4;
    S->ad_dden = reinterpret_cast<float*>(p); p += sz_b4;
    S->ad_pending = reinterpret_cast<int32_t*>(p); p += sz_b4;
    S->ad_state = reinterpret_cast<int32_t*>(p); p += al((int64_t)B * 8);
    S->ad_gi = reinterpret_cast<int32_t*>(p); p += sz_bs;
    S->ad_gv = reinterpret_cast<float*>(p); p += sz_bs;
    S->ad_gn = reinterpret_cast<int32_t*>(p); p += sz_b4;
    S->ad_xgi = reinterpret_cast<int32_t*>(p); p += sz_bs;
    S->ad_xgv = reinterpret_cast<float*>(p); p += sz_bs;
    S->ad_xgn = reinterpret_cast<int32_t*>(p); p += sz_b4;
    S->ad_di = reinterpret_cast<int32_t*>(p); p += sz_b2s;
    S->ad_dv = reinterpret_cast<float*>(p); p += sz_b2s;
    S->ad_dn = reinterpret_cast<int32_t*>(p); p += sz_b4;
    S->ad_tmp = reinterpret_cast<float*>(p); p += sz_v;
    S->ad_mu_rec = reinterpret_cast<float*>(p); p += sz_rec;
    S->ad_shr_rec = reinterpret_cast<int32_t*>(p); p += sz_rec;
  }
  if (S->bounded) {
    S->bc_idx = reinterpret_cast<int32_t*>(p); p += al((int64_t)B * kBcCap * 4);
    S->bc_val = reinterpret_cast<float*>(p); p += al((int64_t)B * kBcCap * 4);
    S->bc_cnt = reinterpret_cast<int*>(p); p += sz_b4;
    S->bc_done = reinterpret_cast<int*>(p); p += sz_b4;
    S->bc_bkey = reinterpret_cast<unsigned int*>(p); p += sz_b4;
    S->bc_stats = getenv("IHT_BOUNDED_STATS") ? reinterpret_cast<int*>(p) : nullptr; p += al(16);
  }
  // zero everything once (pad rows of the stacked vectors stay 0)
  if (cudaMemset(S->block, 0, total) != cudaSuccess ||
      cudaStreamCreateWithFlags(&S->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&S->body_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaFree(S->block);
    delete S;
    return IHT_ECUDA;
  }
  // fused = 1 (auto): when the adjoint copy is large enough for the persistent kernel to pay
  // (>= 2 MiB: measured, config 1's 128 KiB copies run faster as per-step kernels); 2: whenever
  // it fits
  const bool fuse_size = cfg->fused == 2 || iht_qmat_bytes(q0.rows, q0.cols, q0.planes, q0.bits) >= (2ll << 20);
  if (cfg->fused && fuse_size && !batched && !fm && !S->rowshard && cfg->step_mode == 0 &&
      cfg->adjoint_variant == 0 && cfg->n_iter > 0 && !fused_disabled_by_env()) {
    const int frc = iht_fused_create(pool, K, cfg->s, cfg->n_iter, cfg->mu, cfg->trace, S->yhat, S->r, S->g,
                                     S->xs_idx, S->xs_val, S->xs_nnz, &S->fused);
    if (frc != IHT_OK && frc != IHT_EUNSUPPORTED) {
      iht_solver_destroy(S);
      return frc;
    }
  }
  if (cfg->profile) {
    S->ev.resize(2 * (size_t)cfg->n_iter);
    for (auto& e : S->ev) {
      if (cudaEventCreate(&e) != cudaSuccess) {
        iht_solver_destroy(S);
        return IHT_ECUDA;
      }
    }
  }
  *out = S;
  return IHT_OK;
}

extern "C" int iht_solver_adjoint_times(iht_solver* S, float* ms) {
  if (S == nullptr || ms == nullptr || S->ev.empty()) return IHT_EINVAL;
  if (S->fused) {                      // one event pair around the fused kernel
    float t = 0.0f;
    IHT_CUDA_CHECK(cudaEventSynchronize(S->ev[1]));
    IHT_CUDA_CHECK(cudaEventElapsedTime(&t, S->ev[0], S->ev[1]));
    for (int n = 0; n < S->cfg.n_iter; ++n) ms[n] = t / (float)S->cfg.n_iter;
    return IHT_OK;
  }
  IHT_CUDA_CHECK(cudaEventSynchronize(S->ev.back()));
  for (int n = 0; n < S->cfg.n_iter; ++n) IHT_CUDA_CHECK(cudaEventElapsedTime(&ms[n], S->ev[2 * n], S->ev[2 * n + 1]));
  return IHT_OK;
}

extern "C" int iht_solver_destroy(iht_solver* S) {
  if (S == nullptr) return IHT_OK;
  if (S->bc_stats) {   // profiling (IHT_BOUNDED_STATS): how often the bounded select decided
    int h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, S->bc_stats, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "bounded select: decided %d, fell back %d, mean list %.1f, max list %d (bound %.3f)\n", h[0], h[1],
            h[0] ? (double)h[2] / h[0] : 0.0, h[3], S->bound);
  }
  for (auto& e : S->ev)
    if (e) cudaEventDestroy(e);
  if (S->exec) cudaGraphExecDestroy(S->exec);
  iht_fused_destroy(S->fused);
  if (S->cap_stream) cudaStreamDestroy(S->cap_stream);
  if (S->body_stream) cudaStreamDestroy(S->body_stream);
  if (S->block) cudaFree(S->block);
  delete S;
  return IHT_OK;
}

static int ensure_graph(iht_solver* S) {
  if (S->exec) return IHT_OK;
  IHT_CUDA_CHECK(cudaStreamBeginCapture(S->cap_stream, cudaStreamCaptureModeThreadLocal));
  int64_t L = 0;
  const int rc = enqueue_run(S, S->cap_stream, &L);
  cudaGraph_t graph;
  const cudaError_t e = cudaStreamEndCapture(S->cap_stream, &graph);
  if (rc != IHT_OK) {
    if (e == cudaSuccess) cudaGraphDestroy(graph);
    return rc;
  }
  IHT_CUDA_CHECK(e);
  const cudaError_t ei = cudaGraphInstantiate(&S->exec, graph, 0);
  cudaGraphDestroy(graph);
  IHT_CUDA_CHECK(ei);
  S->launches = L;
  return IHT_OK;
}

extern "C" int iht_solver_run(iht_solver* S, const float* y, int flags, int32_t* out_idx, float* out_val,
                              int32_t* out_nnz, void* stream) {
  if (S == nullptr || y == nullptr || out_idx == nullptr || out_val == nullptr || out_nnz == nullptr)
    return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = (flags & IHT_HOST_IO) != 0;
  const int64_t ycount = S->rows * S->planes * S->B;
  IHT_CUDA_CHECK(cudaMemcpyAsync(S->y, y, ycount * sizeof(float),
                                 host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  int rc;
  if (S->cfg.use_graph) {
    if ((rc = ensure_graph(S)) != IHT_OK) return rc;
    IHT_CUDA_CHECK(cudaGraphLaunch(S->exec, st));
  } else {
    int64_t L = 0;
    if ((rc = enqueue_run(S, st, &L)) != IHT_OK) return rc;
    S->launches = L;
  }
  const int64_t xs = (int64_t)S->B * S->cfg.s;
  const int fs = S->final_slot;
  const cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (xs > 0) {
    IHT_CUDA_CHECK(cudaMemcpyAsync(out_idx, S->xs_idx + fs * xs, xs * sizeof(int32_t), kind, st));
    IHT_CUDA_CHECK(cudaMemcpyAsync(out_val, S->xs_val + fs * xs, xs * sizeof(float), kind, st));
  }
  IHT_CUDA_CHECK(cudaMemcpyAsync(out_nnz, S->xs_nnz + (int64_t)fs * S->B, S->B * sizeof(int32_t), kind, st));
  if (host) {
    IHT_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int b = 0; b < S->B; ++b)
      if (out_nnz[b] < 0) return IHT_EDOMAIN;
  }
  return IHT_OK;
}

extern "C" int iht_solver_trace(iht_solver* S, int32_t* idx_host, float* val_host, int32_t* nnz_host,
                                void* stream) {
  if (S == nullptr || !S->cfg.trace) return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = S->cfg.n_iter;
  const int64_t xs = (int64_t)S->B * S->cfg.s;
  if (n == 0) return IHT_OK;
  if (xs > 0) {
    IHT_CUDA_CHECK(cudaMemcpyAsync(idx_host, S->xs_idx + xs, (size_t)n * xs * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost, st));
    IHT_CUDA_CHECK(cudaMemcpyAsync(val_host, S->xs_val + xs, (size_t)n * xs * sizeof(float),
                                   cudaMemcpyDeviceToHost, st));
  }
  IHT_CUDA_CHECK(cudaMemcpyAsync(nnz_host, S->xs_nnz + S->B, (size_t)n * S->B * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, st));
  IHT_CUDA_CHECK(cudaStreamSynchronize(st));
  return IHT_OK;
}

// RecoveryReport (iht.h): the residual of every iteration recomputed from the recorded iterate
// with the solver's forward on the same copy, its squared norm (ad_norm, fixed order), the
// support sizes and changes from the recorded supports (increasing indices: one merge each).
extern "C" int iht_solver_report(iht_solver* S, double* rn_host, int32_t* size_host, int32_t* change_host,
                                 void* stream) {
  if (S == nullptr || !S->cfg.trace || rn_host == nullptr || size_host == nullptr || change_host == nullptr)
    return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int n_iter = S->cfg.n_iter, B = S->B, s = S->cfg.s;
  if (n_iter == 0) return IHT_OK;
  const int64_t xslot = (int64_t)B * s;
  const int K = (int)S->pool.size();
  float* rtmp = nullptr;
  float* nrm = nullptr;
  if (cudaMalloc(&rtmp, (size_t)B * S->vlen * sizeof(float)) != cudaSuccess) return IHT_ENOMEM;
  if (cudaMalloc(&nrm, (size_t)n_iter * B * sizeof(float)) != cudaSuccess) {
    cudaFree(rtmp);
    return IHT_ENOMEM;
  }
  int rc = IHT_OK;
  for (int n = 1; n <= n_iter && rc == IHT_OK; ++n) {
    const int32_t* xi = S->xs_idx + (int64_t)(n - 1) * xslot;   // x^[n] (slot n-1)
    const float* xv = S->xs_val + (int64_t)(n - 1) * xslot;
    const int32_t* xn = S->xs_nnz + (int64_t)(n - 1) * B;
    const float* yh = (S->colshard && S->rank != 0) ? nullptr : S->yhat;
    if (S->fresh) rc = iht_forward_fresh(&S->fm, 2 * n - 1, xi, xv, xn, s, S->yhat, rtmp, st);
    else rc = iht_forward_batched(&S->pool[(2 * n - 1) % K], xi, xv, xn, s, s, B, yh, rtmp, st);
    if (rc == IHT_OK && S->colshard) rc = iht_comm_allreduce(S->cfg.comm, rtmp, (int64_t)B * S->vlen, 0, st);
    if (rc == IHT_OK) rc = ad_norm(rtmp, S->vlen, nrm + (int64_t)(n - 1) * B, B, st);
  }
  if (rc == IHT_OK && S->rowshard) rc = iht_comm_allreduce(S->cfg.comm, nrm, (int64_t)n_iter * B, 0, st);
  std::vector<float> h((size_t)n_iter * B);
  std::vector<int32_t> idx((size_t)(n_iter + 1) * (xslot > 0 ? xslot : 1)), nz((size_t)(n_iter + 1) * B);
  if (rc == IHT_OK) {
    cudaError_t e = cudaMemcpyAsync(h.data(), nrm, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && xslot > 0)
      e = cudaMemcpyAsync(idx.data(), S->xs_idx, (size_t)(n_iter + 1) * xslot * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(nz.data(), S->xs_nnz, nz.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      iht_set_last_cuda_error(e, "iht_solver_report copies", __FILE__, __LINE__);
      rc = IHT_ECUDA;
    }
  }
  cudaFree(rtmp);
  cudaFree(nrm);
  if (rc != IHT_OK) return rc;
  for (int n = 1; n <= n_iter; ++n) {
    for (int b = 0; b < B; ++b) {
      const size_t o = (size_t)(n - 1) * B + b;
      rn_host[o] = sqrt((double)h[o]);
      const int k0 = nz[(size_t)(n - 1) * B + b], k1 = nz[(size_t)n * B + b];
      size_host[o] = k1;
      const int a = k0 < 0 ? 0 : k0, c = k1 < 0 ? 0 : k1;
      const int32_t* p = idx.data() + (size_t)(n - 1) * xslot + (size_t)b * s;   // supp x^[n]
      const int32_t* q = idx.data() + (size_t)n * xslot + (size_t)b * s;         // supp x^[n+1]
      int i = 0, j = 0, common = 0;
      while (i < a && j < c) {
        if (p[i] == q[j]) {
          ++common;
          ++i;
          ++j;
        } else if (p[i] < q[j]) {
          ++i;
        } else {
          ++j;
        }
      }
      change_host[o] = a + c - 2 * common;
    }
  }
  return IHT_OK;
}

extern "C" int iht_solver_buffers(iht_solver* S, const float** yhat, const float** r, const float** g) {
  if (S == nullptr) return IHT_EINVAL;
  if (yhat) *yhat = S->yhat;
  if (r) *r = S->r;
  if (g) *g = S->g;
  return IHT_OK;
}

extern "C" int64_t iht_solver_launches_per_run(const iht_solver* S) { return S ? S->launches : -1; }

extern "C" int iht_solver_fused(const iht_solver* S) { return S ? (S->fused != nullptr) : -1; }

extern "C" int iht_solver_steps(iht_solver* S, float* mu_host, int32_t* shrinks_host, void* stream) {
  if (S == nullptr || mu_host == nullptr || shrinks_host == nullptr || S->cfg.step_mode != 1) return IHT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)S->cfg.n_iter * S->B;
  if (n == 0) return IHT_OK;
  IHT_CUDA_CHECK(cudaMemcpyAsync(mu_host, S->ad_mu_rec, n * sizeof(float), cudaMemcpyDeviceToHost, st));
  IHT_CUDA_CHECK(cudaMemcpyAsync(shrinks_host, S->ad_shr_rec, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  IHT_CUDA_CHECK(cudaStreamSynchronize(st));
  return IHT_OK;
}

extern "C" int iht_solve(const iht_qmat* pool, int K, const iht_config* cfg, const float* y, int flags,
                         int32_t* out_idx, float* out_val, int32_t* out_nnz, void* stream) {
  iht_solver* S = nullptr;
  int rc = iht_solver_create(pool, K, cfg, &S);
  if (rc != IHT_OK) return rc;
  rc = iht_solver_run(S, y, flags, out_idx, out_val, out_nnz, stream);
  if (rc == IHT_OK) {
    const cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) rc = IHT_ECUDA;
  }
  iht_solver_destroy(S);
  return rc;
}
