/*
 * iht.h -- C ABI of libiht.so, the B200 (sm_100a) hot path of low-precision
 * Iterative Hard Thresholding (arXiv 1802.04907, "Compressive Sensing with Low
 * Precision Data Representation").
 *
 * Citations: P:L = PAPER.md line L (paper LaTeX source), S:L = SPEC.md line L.
 * Readings of ambiguous passages (c1..c20) are listed in DESIGN.md.
 *
 * The method (Eq. modified_update_rule; Algorithm 1):
 *     r     = y-hat - Phi-hat_F x                 forward residual
 *     g     = Re( Phi-hat_A^H r )                 adjoint gradient
 *     x    <- H_s( x + mu g )                     update + top-s
 * with Phi-hat_A, Phi-hat_F two independent stochastic quantisations of Phi
 * and y-hat = Q(y) quantised once.
 *
 * Conventions shared by every call
 * --------------------------------
 * - Every pointer named *_dev / device is CUDA device memory owned by the
 *   caller (the Python binding allocates it through torch).  The library never
 *   allocates in the per-iteration path; workspace sizes come from the
 *   *_ws_bytes queries.  Host pointers are named *_host.
 * - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Every call only ENQUEUES work on that stream; nothing synchronises except
 *   where stated (iht_quantize reads nothing back; iht_solver_run with
 *   IHT_HOST_IO synchronises the stream before returning).
 * - Return value: IHT_OK (0) or a negative IHT_E* code; iht_strerror() names it.
 *   No exception crosses the ABI.  Argument errors are detected on the host
 *   before anything is enqueued.
 * - Stacked real rows: a complex matrix (planes = 2) is treated as the real
 *   matrix [Re Phi; Im Phi] (re plane then im plane), so that
 *   Re(Phi^H r) = Re(Phi)^T Re(r) + Im(Phi)^T Im(r)  (reading c13).
 *   A length-R "stacked vector" (y-hat, r) holds plane p, row m at index
 *   p * rows_pad + m, with rows_pad = iht_rows_pad(rows) (rows rounded up to a
 *   multiple of 256); pad entries are 0.
 * - Column strips in 16-column tiles: the codes of column n form a logical strip
 *   of strip_bytes bytes (plane p starts at strip byte p * rows_pad * bits / 8;
 *   row m's b-bit code sits at bit m*bits of its plane segment, little-endian,
 *   LSB first).  Strips are interleaved by 16-column tiles at 64-byte granularity
 *   so that one k-step of a 16-column tile is 1 KiB of contiguous memory:
 *     strip byte k of column n  ->  codes + (n/16)*16*strip_bytes + (k/64)*1024
 *                                          + (n%16)*64 + k%64.
 *   strip_bytes is a multiple of 64.  Codes of pad rows are 0; the bytes of pad
 *   columns (n >= cols in the last tile) are unspecified and never read.
 */
#ifndef IHT_H_
#define IHT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IHT_ABI_VERSION 3

#if defined(__GNUC__)
#define IHT_API __attribute__((visibility("default")))
#else
#define IHT_API
#endif

enum {
  IHT_OK = 0,
  IHT_EINVAL = -1,       /* bad argument: dimension mismatch, bits not in {2,4,8},
                            s > rows, misaligned pointer, workspace too small          */
  IHT_EDOMAIN = -2,      /* non-finite input or non-finite x + mu g in H_s          */
  IHT_ECUDA = -3,        /* a CUDA runtime call failed                                             */
  IHT_ENCCL = -4,        /* NCCL could not be loaded or a collective failed                        */
  IHT_ENOMEM = -5,       /* solver could not allocate its (one-time) workspace                     */
  IHT_EUNSUPPORTED = -6  /* valid but not implemented configuration                                */
};

/* Name of a status code. Static storage; never NULL. */
IHT_API const char* iht_strerror(int status);
IHT_API int iht_abi_version(void);
/* Text of the last CUDA error seen by this thread (after an IHT_ECUDA). */
IHT_API const char* iht_last_cuda_error(void);

/* ------------------------------------------------------------------ sizes */
/* rows rounded up to a multiple of 256 (whole 32-byte sectors and adjoint k-steps). */
IHT_API int64_t iht_rows_pad(int64_t rows);
/* Bytes of one column strip: planes * iht_rows_pad(rows) * bits / 8.        */
IHT_API int64_t iht_strip_bytes(int64_t rows, int planes, int bits);
/* Bytes of one quantised copy: round_up(cols, 16) * iht_strip_bytes(...).    */
IHT_API int64_t iht_qmat_bytes(int64_t rows, int64_t cols, int planes, int bits);
/* Length of a stacked vector (y-hat, r): planes * iht_rows_pad(rows).        */
IHT_API int64_t iht_vec_len(int64_t rows, int planes);

/* One quantised copy Phi-hat_k of (this shard of) Phi: 2^b-level (or odd,
 * P:689) stochastic codes of Sec. 3 "Quantization" plus the global
 * scale c (reading c3).  Dequantised entry: sigma * (2 code - (L-1)),
 * sigma = scale_c / (L-1).  The struct is plain data; codes is caller-owned. */
typedef struct {
  int64_t rows;        /* logical rows of this shard (measurements / visibilities)   */
  int64_t cols;        /* N, columns (unknowns / pixels)                             */
  int64_t row_offset;  /* global index of this shard's first row (row sharding)      */
  int32_t planes;      /* 1 = real, 2 = complex (re plane, im plane)                 */
  int32_t bits;        /* b in {2, 4, 8}                                             */
  int32_t level_mode;  /* 0: L = 2^b levels; 1: L = 2^{b-1}+1        */
  int32_t copy_id;     /* Philox counter word 2: which independent copy      */
  uint64_t seed;       /* Philox key                                                 */
  float scale_c;       /* c = max |component| over the WHOLE Phi, all shards */
  int32_t col_offset;  /* global index of this shard's first column (column sharding of
                          the batched path); a multiple of 16; 0 otherwise.
                          Philox counters use the global column col_offset + n, so codes
                          do not depend on the sharding                               */
  int64_t strip_bytes; /* must equal iht_strip_bytes(rows, planes, bits)             */
  void* codes;         /* device, iht_qmat_bytes(rows, cols, planes, bits) bytes     */
} iht_qmat;

/* --------------------------------------------------------------- (a1) scale */
/* c = max over `count` fp32 values of |src[i]| (complex data: pass 2x the
 * element count; re and im are pooled, reading c3).  P:686 "c_v is the maximum
 * value of the components of v in magnitude".  Writes one float to c_dev
 * (device).  A NaN anywhere makes the result NaN (caller maps it to
 * IHT_EDOMAIN).  Deterministic. */
IHT_API int iht_absmax(const float* src_dev, int64_t count, float* c_dev, void* stream);
/* Batched form: nrhs independent vectors of `count` floats each, back to back in
 * src_dev; c_dev[b] = max |src_dev[b * count + i]| (each observation has its own
 * scale c_y, P:686 applied per snapshot). */
IHT_API int iht_absmax_batched(const float* src_dev, int64_t count, int32_t nrhs, float* c_dev,
                               void* stream);

/* ------------------------------------------------------- (a2) quantise Phi */
/* Stochastically quantise the rows x cols block src (row-major, row stride ld
 * ELEMENTS; complex = interleaved (re, im) pairs, ld in complex elements) into
 * ncopies independent copies in one pass over src (one fp32 read emits every
 * copy).  Sec. 3 "Quantization", fp32 Q-contract of DESIGN.md:
 *   sf = fl32((L-1) / fl32(2c)); t = clamp(fl32(fl32(v + c) * sf), 0, L-1);
 *   i = floor t; code = L-1 if i = L-1 else i + (u < t - i),
 *   u = (w >> 8) 2^-24, w = Philox4x32-10 word (n & 3) of counter
 *   (n >> 2, row_offset + m, copy_id, (plane << 8) | 0), key (lo32 seed, hi32 seed),
 *   with n = col_offset + local column (global column index).
 * dst[k] describes copy k (same rows/cols/planes/bits/level_mode/scale_c/
 * row_offset/col_offset for all k; own copy_id, seed, codes).  Errors: IHT_EINVAL on
 * inconsistent descriptors. */
IHT_API int iht_quantize(const float* src_dev, int64_t ld, const iht_qmat* dst, int ncopies,
                 void* stream);
/* Block-wise form (config 4's 64 GiB fp32 Phi is never resident): quantise only
 * the local rows [row_begin, row_begin + nrows) of the copies dst[k]; src_dev
 * points at local row row_begin.  row_begin must be a multiple of 256 and nrows
 * too unless the block ends at dst->rows.  Codes are identical to a whole-matrix
 * call because the Philox counters use global indices. */
IHT_API int iht_quantize_rows(const float* src_dev, int64_t ld, const iht_qmat* dst, int ncopies,
                              int64_t row_begin, int64_t nrows, void* stream);

/* -------------------------------------------------------- (a3) quantise y */
/* y-hat = Q_{b_y}(y) once (Alg. 1 input): element m of plane p draws
 * word 0 of counter (0, row_offset + m, 0, (p << 8) | 1).  Writes the
 * dequantised stacked vector yhat_dev (length iht_vec_len(rows, planes),
 * pads 0) and, if codes_dev != NULL, the codes (uint8, planes * rows, plane
 * major).  The scale c is read from the device (c_dev) so that the call can sit
 * after iht_absmax / an all-reduce without a host round trip. */
IHT_API int iht_quantize_vec(const float* y_dev, int64_t rows, int64_t row_offset, int planes, int bits,
                     int level_mode, uint64_t seed, const float* c_dev, float* yhat_dev,
                     uint8_t* codes_dev, void* stream);
/* Batched form (config 5): nrhs observations y_b, each rows * planes floats (complex
 * interleaved), back to back in y_dev; scales c_dev[b]; output yhat_dev [nrhs][vec_len].
 * Snapshot b is column n = b of the observation matrix Y = [y_0 .. y_{B-1}]: element m
 * of plane p draws word (b & 3) of counter (b >> 2, row_offset + m, 0, (p << 8) | 1),
 * so b = 0 reproduces iht_quantize_vec exactly.  codes_dev (optional): [nrhs][planes*rows]. */
IHT_API int iht_quantize_vec_batched(const float* y_dev, int64_t rows, int64_t row_offset, int planes,
                                     int bits, int level_mode, uint64_t seed, const float* c_dev,
                                     int32_t nrhs, float* yhat_dev, uint8_t* codes_dev, void* stream);

/* ------------------------------------------------------------ (a4) forward */
/* r = y-hat - Phi-hat_F x for s-sparse real x ("matrix times a sparse
 * vector ... scale-and-add"): only the x_nnz support columns of F
 * are read.  x_idx_dev / x_val_dev: device arrays of length >= max_nnz;
 * x_nnz_dev: device int32 (values < 0 are treated as 0).  yhat_dev and r_dev are
 * stacked vectors of length iht_vec_len(F rows, planes).  ws_dev: device workspace of
 * iht_forward_ws_bytes(F, max_nnz) bytes, caller-owned, ZERO before its first use (its
 * arrival counters are left at zero by every call, so one zeroing suffices); when that
 * size is > 0 and ws_dev is NULL or smaller, the call falls back to the single-pass
 * kernel (same results to rounding order).  Large single observations (>= 2 x 148 row
 * blocks of 64 bytes per strip) use a row-block x column-group grid whose G > 1 groups'
 * partial row sums are added in group order by the last CTA of each row block:
 * deterministic. */
IHT_API int64_t iht_forward_ws_bytes(const iht_qmat* F, int32_t max_nnz);
IHT_API int iht_forward(const iht_qmat* F, const int32_t* x_idx_dev, const float* x_val_dev,
                const int32_t* x_nnz_dev, int32_t max_nnz, const float* yhat_dev, float* r_dev,
                void* ws_dev, int64_t ws_bytes, void* stream);
/* Batched form (config 5): nrhs sparse iterates x_b (x_idx_dev / x_val_dev [nrhs][ldx],
 * x_nnz_dev [nrhs], at most min(ldx, max_nnz) entries each, GLOBAL column indices),
 * yhat_dev / r_dev [nrhs][vec_len].  Only support entries inside this shard's columns
 * [F->col_offset, F->col_offset + F->cols) contribute (column sharding); yhat_dev may
 * be NULL, giving the partial product r_b = -Phi-hat_F[:, S_b] x_b that the column-
 * sharded solver all-reduces. */
IHT_API int iht_forward_batched(const iht_qmat* F, const int32_t* x_idx_dev, const float* x_val_dev,
                                const int32_t* x_nnz_dev, int32_t ldx, int32_t max_nnz, int32_t nrhs,
                                const float* yhat_dev, float* r_dev, void* stream);

/* ------------------------------------------------------------ (a5) adjoint */
/* g = Re(Phi-hat_A^H r) for all N columns: g_n = sigma_A sum_m
 * q_{m,n} r_m over the stacked rows; the whole copy is streamed once.  r_dev:
 * stacked vector (pad entries must be 0); g_dev: N floats.  Deterministic (no
 * float atomics).  `variant`: 0 = default (int8 tensor-core MMA path), 1 =
 * CUDA-core FFMA path (kept as the measured baseline). */
IHT_API int64_t iht_adjoint_ws_bytes(const iht_qmat* A);
IHT_API int iht_adjoint(const iht_qmat* A, const float* r_dev, float* g_dev, int variant, void* ws_dev,
                int64_t ws_bytes, void* stream);

/* ------------------------------------------- (a7) batched adjoint (tcgen05) */
/* B = nrhs observations sharing one Phi (BASELINE config 5): G[b][n] =
 * Re(Phi-hat_A^H r_b)_n for all snapshots at once, as an int8 tcgen05 GEMM
 * (kind::i8, M = 128 pixels, N = 2 nrhs): codes expanded to u8 in shared memory, r_b
 * in per-snapshot block fixed point (two signed 8-bit limbs, 15 bits), exact int32
 * accumulation in TMEM.  Tolerance class: the tensor-core path (1e-3, north star).
 * R: nrhs stacked vectors [nrhs][iht_vec_len] (pads 0); G: [nrhs][cols] floats.
 * Any nrhs >= 1: snapshots run in chunks of <= 64 (one launch pair each), a chunk padded
 * to a multiple of 8 with zero residuals inside the workspace (MMA N granularity 16).
 * Workspace: iht_adjoint_batched_ws_bytes.  Errors: IHT_EUNSUPPORTED if the int32
 * accumulator could overflow (rows * planes * (L-1) * 128 >= 2^31). */
IHT_API int64_t iht_adjoint_batched_ws_bytes(const iht_qmat* A, int32_t nrhs);
IHT_API int iht_adjoint_batched(const iht_qmat* A, const float* R_dev, int32_t nrhs, float* G_dev,
                                void* ws_dev, int64_t ws_bytes, void* stream);

/* ------------------------------------- NEXT-2: fresh copies drawn on the fly */
/* The fp32 Phi itself (this shard's rows), from which any copy Phi-hat_k is drawn on the
 * fly: code(m, n) is the Q-contract rounding of phi with the Philox word of counter
 * (n >> 2, row_offset + m, k, plane << 8), exactly what iht_quantize stores for copy k.
 * Algorithm 1's 2 n* independent copies then need no storage. */
typedef struct {
  int64_t rows, cols, row_offset;
  int64_t ld;           /* row stride in (complex) elements, >= cols                     */
  int32_t planes, bits, level_mode, reserved;
  uint64_t seed;
  float scale_c;        /* global max |component| (a1)                                   */
  int32_t reserved2;
  const float* phi;     /* device, row-major, complex interleaved                        */
} iht_fmat;

/* g = Re(Phi-hat_k^H r) with Phi-hat_k drawn on the fly from F (copy_id = k).  r:
 * stacked vector; g: cols floats.  Deterministic (row splits reduced in a fixed order).
 * Workspace: iht_adjoint_fresh_ws_bytes. */
IHT_API int64_t iht_adjoint_fresh_ws_bytes(const iht_fmat* F);
IHT_API int iht_adjoint_fresh(const iht_fmat* F, int32_t copy_id, const float* r_dev, float* g_dev, void* ws_dev,
                              int64_t ws_bytes, void* stream);
/* r = y-hat - Phi-hat_k x over the support of x, Phi-hat_k drawn on the fly. */
IHT_API int iht_forward_fresh(const iht_fmat* F, int32_t copy_id, const int32_t* x_idx_dev, const float* x_val_dev,
                              const int32_t* x_nnz_dev, int32_t max_nnz, const float* yhat_dev, float* r_dev,
                              void* stream);

/* ------------------------------------------ NEXT-3: radio Phi computed on the fly */
/* Phi_{k,p} = exp(-2 pi i (u_k l_p + v_k m_p)) (BASELINE config 3, reading c16; paper
 * "Computing Phi on the fly"): u, v = baseline / lambda per visibility k
 * (device fp64 arrays of nvis), pixel p = row * grid + col with l = -1 + (2 row + 1)/grid,
 * m = -1 + (2 col + 1)/grid.  No Phi bytes are read.  bits = 0: full precision; bits in
 * {2,4,8}: each component stochastically rounded in registers with the Q-contract and
 * Philox counter (p >> 2, row_offset + k, copy_id, plane << 8) -- the codes iht_quantize
 * stores for copy_id, up to components whose on-the-fly fp32 value differs by an ulp
 * across a rounding decision. */
typedef struct {
  int64_t nvis, row_offset;
  int32_t grid, bits, level_mode, copy_id;
  uint64_t seed;
  float scale_c;        /* c of the quantiser (unit-modulus entries: 1)                  */
  int32_t reserved;
  const double* u;      /* device [nvis] */
  const double* v;      /* device [nvis] */
} iht_radio;
/* g = Re(Phi^H r) (full precision) or Re(Phi-hat^H r) (bits > 0) for all grid^2 pixels;
 * r: stacked vector of iht_vec_len(nvis, 2); g: grid^2 floats. */
IHT_API int iht_adjoint_radio(const iht_radio* R, const float* r_dev, float* g_dev, void* stream);

/* ---------------------------------------------------- (a6) update + H_s */
/* a = x + mu g, then H_s: keep the s entries of largest |a|,
 * ties to the LOWEST index, zeros never kept (reading c15).  Output
 * support strictly increasing in out_idx_dev[0..*out_nnz_dev) with
 * values a_n.  Non-finite a sets *out_nnz_dev = -1 (IHT_EDOMAIN is reported by
 * iht_solver_run).  Inputs x_* as in iht_forward; g_dev: N floats.  Output
 * buffers must not alias the inputs. */
IHT_API int64_t iht_threshold_ws_bytes(int64_t N, int32_t s);
IHT_API int iht_threshold(const int32_t* x_idx_dev, const float* x_val_dev, const int32_t* x_nnz_dev,
                  const float* g_dev, float mu, int32_t s, int64_t N, int32_t* out_idx_dev,
                  float* out_val_dev, int32_t* out_nnz_dev, void* ws_dev, int64_t ws_bytes,
                  void* stream);
/* Batched form: nrhs independent selections (config 5, H_s per snapshot).  x_* as in
 * iht_forward_batched (stride ldx, GLOBAL indices); g_dev [nrhs][N] holds the gradient of
 * the N local columns [col_offset, col_offset + N); entries of x outside that range are
 * ignored, output indices are global (col_offset + local).  out_idx_dev / out_val_dev
 * [nrhs][ldo] (ldo >= s), out_nnz_dev [nrhs].  With col_offset = 0 and the whole N this
 * is exactly nrhs calls of iht_threshold; on a column shard it yields the shard's local
 * top-s candidates, whose merge over shards is the global H_s. */
IHT_API int64_t iht_threshold_batched_ws_bytes(int64_t N, int32_t s, int32_t nrhs);
IHT_API int iht_threshold_batched(const int32_t* x_idx_dev, const float* x_val_dev, const int32_t* x_nnz_dev,
                                  int32_t ldx, const float* g_dev, float mu, int32_t s, int64_t N,
                                  int64_t col_offset, int32_t nrhs, int32_t* out_idx_dev, float* out_val_dev,
                                  int32_t ldo, int32_t* out_nnz_dev, void* ws_dev, int64_t ws_bytes,
                                  void* stream);
/* Merge of per-shard candidate lists into the global H_s (column-sharded batched path):
 * for each snapshot b, the concatenation over shards p = 0..P-1 of shard p's list
 * (cand_idx/cand_val[p * shard_stride + b * s + j], j < cand_nnz[p * shard_stride + b];
 * shard p's indices increasing and below shard p+1's; strides in 4-byte elements) is
 * thresholded to its top s (ties to the lowest index; P * s <= 8192), written to
 * out_* [nrhs][s] and out_nnz [nrhs] (-1 if any shard reported -1). */
IHT_API int iht_merge_candidates(const int32_t* cand_idx_dev, const float* cand_val_dev,
                                 const int32_t* cand_nnz_dev, int64_t shard_stride, int32_t P, int32_t s,
                                 int32_t nrhs, int32_t* out_idx_dev, float* out_val_dev, int32_t* out_nnz_dev,
                                 void* stream);

/* --------------------------------------------------------- multi-GPU comm */
/* One NCCL communicator per rank (row-sharded Phi, north star).
 * NCCL is loaded with dlopen at first use (libnccl.so.2; the copy torch has
 * already loaded is reused).  Rank 0 calls iht_comm_unique_id, the 128 bytes
 * are broadcast by the caller (torch.distributed), then every rank calls
 * iht_comm_create.  Returns IHT_ENCCL when NCCL is unavailable. */
typedef struct iht_comm iht_comm;
IHT_API int iht_comm_unique_id(void* id_host_128);
IHT_API int iht_comm_create(int rank, int world, const void* id_host_128, int device, iht_comm** out);
IHT_API int iht_comm_destroy(iht_comm* comm);
/* In-place sum / max all-reduce of `count` floats on the stream (test hook). */
IHT_API int iht_comm_allreduce(iht_comm* comm, float* buf_dev, int64_t count, int op_max, void* stream);
/* Sum reduce-scatter of P * recv_count floats: rank p receives elements
 * [p * recv_count, (p+1) * recv_count) of the sum over ranks of send_dev.  In place when
 * recv_dev == send_dev + rank * recv_count (the row-sharded solver's g). */
IHT_API int iht_comm_reduce_scatter(iht_comm* comm, const float* send_dev, float* recv_dev, int64_t recv_count,
                                    void* stream);
/* All-gather of `bytes` bytes per rank: recv_dev[p * bytes ..] = rank p's send_dev. */
IHT_API int iht_comm_allgather(iht_comm* comm, const void* send_dev, void* recv_dev, int64_t bytes,
                               void* stream);

/* ------------------------------------------------------------ (b) solver */
typedef struct {
  int32_t s;            /* sparsity                                              */
  int32_t n_iter;       /* n*                                                     */
  float mu;             /* fixed step (reading c9)                                       */
  int32_t b_y;          /* bits of y-hat                                                 */
  int32_t level_mode;   /* as iht_qmat.level_mode, for y-hat                             */
  int32_t adjoint_variant; /* iht_adjoint variant                                        */
  uint64_t seed;        /* quantiser key for y-hat                                       */
  int32_t trace;        /* 1: keep every iterate x^[n] (see iht_solver_trace)            */
  int32_t use_graph;    /* 1: capture the n_iter loop into one CUDA graph (default)      */
  iht_comm* comm;       /* NULL: single GPU; else the rows are sharded (single observation:
                           c_y max-all-reduced; per iteration g is sum-REDUCE-SCATTERED
                           over the P ranks (rank p owns columns [p N/P, (p+1) N/P)), each
                           rank takes the local top-s of its columns (global indices), the
                           P lists are all-gathered and merged into the global H_s -- when
                           N % P == 0 and P s <= 8192, else g is all-reduced and H_s
                           replicated; the adaptive step always all-reduces g) or the
                           columns (batched); world 1 runs the same collectives          */
  int32_t profile;      /* 1: record a CUDA event pair around every adjoint launch      */
  int32_t nrhs;         /* B independent observations sharing Phi (BASELINE config 5);
                           0 or 1: one observation.  B > 1 runs the batched path: sparse
                           forward per snapshot, the tcgen05 adjoint (iht_adjoint_batched),
                           per-snapshot H_s.  With a communicator (world P >= 1) the
                           batched path is COLUMN-sharded (pool[k].col_offset = rank N/P):
                           forward partials all-reduced (sum), local H_s candidates
                           all-gathered and merged                         */
  int32_t step_mode;    /* 0: fixed step mu (reading c9, the north star's hot path);
                           1: Algorithm 1's adaptive step:
                           Gamma^[1] = supp(H_s(Phi-hat_1^H y-hat)); per iteration
                           mu = |g_G|^2 / |Phi-hat_A[:, G] g_G|^2 (reading c10), proposal
                           H_s(x + mu g); if its support differs from G, accept only when
                           mu <= (1 - c) |dx|^2 / |Phi-hat_A dx|^2, else mu /= k (1 - c)
                           and propose again (reading c11).  `mu` is the fallback step for
                           a vanishing denominator.  Not with a column-sharded batch.   */
  float step_c;         /* c of the acceptance test (0 < c < 1; SPEC default 1e-3)       */
  float step_k;         /* k of the shrink mu / (k (1 - c)), k > 1 / (1 - c) (default 2) */
  int32_t max_shrink;   /* bound on proposals per iteration; the last is kept    */
  int32_t fused;        /* 1 (auto): when the problem fits (single observation, fixed step, no
                           communicator, stored copies, variant 0, stacked rows small enough
                           for r limbs in one CTA's shared memory: configs 1-3), the WHOLE
                           n-iteration loop runs as ONE persistent cooperative kernel (one
                           CTA per SM, three grid barriers per iteration, the next
                           iteration's adjoint codes prefetched into shared memory under the
                           select and the forward; same arithmetic as the per-step kernels
                           up to fp32 summation order) and a copy is >= 2 MiB (smaller
                           problems run faster as per-step kernels); 2: whenever it fits;
                           0: per-step kernels always.                                      */
} iht_config;

/* Stateful solver over a pool of K quantised copies pool[0..K) (all with the
 * same shape; K = 2 n* is Algorithm 1 exactly, smaller K reuses copies,
 * reading c6): iteration n (1-based) uses pool[(2n-2) % K] for the adjoint
 * (Phi-hat_{2n-1}) and pool[(2n-1) % K] for the forward (Phi-hat_{2n}).
 * x^[1] = 0 (reading c8).  create allocates the one-time workspace (and,
 * lazily, the CUDA graph); the pool's codes must outlive the solver. */
typedef struct iht_solver iht_solver;
IHT_API int iht_solver_create(const iht_qmat* pool, int K, const iht_config* cfg, iht_solver** out);
/* Algorithm 1 with FRESH copies (NEXT-2): iteration n draws Phi-hat_{2n-1} (copy id 2n-2,
 * adjoint) and Phi-hat_{2n} (copy id 2n-1, forward) on the fly from the fp32 Phi in F,
 * i.e. K = 2 n* without storing any copy.  Single observation, fixed step; with a
 * communicator the rows are sharded (F->row_offset) and g is all-reduced.  F->phi must
 * outlive the solver. */
IHT_API int iht_solver_create_fresh(const iht_fmat* F, const iht_config* cfg, iht_solver** out);
IHT_API int iht_solver_destroy(iht_solver* solver);

#define IHT_HOST_IO 1   /* y and the outputs are host pointers (pinned for async copies) */

/* Run Algorithm 1 on this shard's observations y (fp32 rows values, complex
 * interleaved; device or, with IHT_HOST_IO, host).  Steps: c_y = absmax(y)
 * (all-reduced max across ranks), y-hat = Q(y), then n_iter iterations of
 * forward -> adjoint -> [all-reduce g] -> update + H_s.  Writes the final
 * support (<= s indices, increasing) and values, and *out_nnz (device or host
 * per flags).  Returns IHT_EDOMAIN if a non-finite value reached H_s.
 * Batched (cfg.nrhs = B > 1): y holds B observations back to back ([B][rows * planes]
 * floats; each snapshot has its own c_y and Q(y), iht_quantize_vec_batched), and the
 * outputs are out_idx / out_val [B][s], out_nnz [B].  Column-sharded runs (P > 1) take
 * the FULL y on every rank and return the same (replicated) x on every rank. */
IHT_API int iht_solver_run(iht_solver* solver, const float* y, int flags, int32_t* out_idx,
                   float* out_val, int32_t* out_nnz, void* stream);
/* Copy the recorded iterates (cfg.trace = 1) of the last run to host arrays:
 * idx_host/val_host of n_iter * s entries (row n-1 = x^[n+1] after iteration
 * n), nnz_host of n_iter entries; batched: n_iter * B * s and n_iter * B
 * ([n-1][b][.]).  Synchronises the stream. */
IHT_API int iht_solver_trace(iht_solver* solver, int32_t* idx_host, float* val_host, int32_t* nnz_host,
                     void* stream);
/* Device pointers of the internal stacked vectors of the LAST iteration
 * (r, y-hat) and of g, for parity tests; lengths iht_vec_len(rows, planes) / N
 * (batched: [B][vec_len] and [B][N]). */
IHT_API int iht_solver_buffers(iht_solver* solver, const float** yhat_dev, const float** r_dev,
                       const float** g_dev);
/* With cfg.profile = 1: durations (ms) of the n_iter adjoint launches of the LAST
 * run, from the CUDA event pairs recorded on the run's stream around each adjoint
 * (inside the graph).  Synchronises on the last event. */
IHT_API int iht_solver_adjoint_times(iht_solver* solver, float* ms_host);
/* Adaptive step (cfg.step_mode = 1): the accepted mu and the number of shrinks of every
 * iteration of the LAST run, [n_iter][B] each (host arrays).  Synchronises the stream. */
IHT_API int iht_solver_steps(iht_solver* solver, float* mu_host, int32_t* shrinks_host, void* stream);
/* RecoveryReport of the last run (cfg.trace = 1; "one row per iteration with
 * columns iter, mu, residual_norm, support_size, support_change, shrink_count"), host arrays
 * [n_iter][B]:
 *   residual_norm[n-1]  = || y-hat - Phi-hat_{2n} x^[n] ||_2, the forward residual of
 *                         iteration n (Algorithm 1), recomputed from the recorded
 *                         iterate x^[n] by the solver's own forward kernel on the same copy
 *                         (stacked re/im rows: the complex norm); squared norms summed in
 *                         fp32 in a fixed order (all-reduced over row shards), sqrt in fp64;
 *   support_size[n-1]   = || x^[n+1] ||_0 (-1 when the iterate is poisoned);
 *   support_change[n-1] = | supp x^[n+1] symmetric-difference supp x^[n] | (x^[1] = 0).
 * mu and shrink_count come from cfg.mu / iht_solver_steps.  Uses scratch device memory of
 * B * vec_len + n_iter * B floats (allocated and freed here); synchronises the stream.
 * IHT_EINVAL without cfg.trace or with a NULL pointer. */
IHT_API int iht_solver_report(iht_solver* solver, double* residual_norm_host, int32_t* support_size_host,
                              int32_t* support_change_host, void* stream);
/* 1 if the solver runs the fused persistent kernel (cfg.fused and the problem fits), else 0;
 * negative on a NULL solver.  With cfg.profile, iht_solver_adjoint_times then reports the
 * fused kernel's duration divided evenly over the n_iter iterations. */
IHT_API int iht_solver_fused(const iht_solver* solver);
/* Number of kernel launches one iht_solver_run enqueues (for gpu_launches); with the
 * adaptive step it counts one pass of the shrink loop per iteration. */
IHT_API int64_t iht_solver_launches_per_run(const iht_solver* solver);

/* One-shot convenience: create, run, destroy. */
IHT_API int iht_solve(const iht_qmat* pool, int K, const iht_config* cfg, const float* y, int flags,
              int32_t* out_idx, float* out_val, int32_t* out_nnz, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IHT_H_ */
