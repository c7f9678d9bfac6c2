"""Python binding of libiht.so with the C ABI's names (argument marshalling only).

Every step of the hot path runs in the library's CUDA kernels; torch supplies
device memory (tensors), the current CUDA stream and process groups.  Functions
mirror include/iht.h:

    absmax, quantize, quantize_vec, forward, adjoint, threshold,   (a1)-(a6)
    Solver / solve (iht_solver_*), Comm (iht_comm_*).
"""
import ctypes
from dataclasses import dataclass

import numpy as np

import torch

from . import _lib
from ._lib import IhtConfig, IhtFmat, IhtQmat, check, load

__all__ = ["absmax", "absmax_batched", "quantize", "quantize_rows", "quantize_vec", "quantize_vec_batched", "forward",
           "forward_batched", "adjoint", "adjoint_batched", "threshold", "threshold_batched", "merge_candidates",
           "Solver", "solve", "Comm", "QCopy", "FreshPhi", "adjoint_fresh", "forward_fresh", "adjoint_radio", "strip_bytes", "vec_len",
           "rows_pad"]


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libiht compute calls take CUDA tensors (no CPU path)")


def rows_pad(rows):
    return load().iht_rows_pad(rows)


def strip_bytes(rows, planes, bits):
    v = load().iht_strip_bytes(rows, planes, bits)
    if v < 0:
        raise ValueError("invalid (rows, planes, bits)")
    return v


def vec_len(rows, planes):
    return load().iht_vec_len(rows, planes)


@dataclass
class QCopy:
    """One quantised copy Phi-hat_k: descriptor + the torch uint8 tensor owning the codes."""
    desc: IhtQmat
    codes: torch.Tensor

    @property
    def rows(self):
        return self.desc.rows

    @property
    def cols(self):
        return self.desc.cols

    @property
    def planes(self):
        return self.desc.planes

    @property
    def bits(self):
        return self.desc.bits

    @property
    def scale_c(self):
        return self.desc.scale_c


def new_copy(rows, cols, planes, bits, level_mode, seed, copy_id, scale_c, row_offset=0, device=None,
             codes=None, col_offset=0):
    sb = strip_bytes(rows, planes, bits)
    if codes is None:
        codes = torch.empty(load().iht_qmat_bytes(rows, cols, planes, bits), dtype=torch.uint8,
                            device=device or "cuda")
    d = IhtQmat(rows=rows, cols=cols, row_offset=row_offset, planes=planes, bits=bits, level_mode=level_mode,
                copy_id=copy_id, seed=seed, scale_c=float(scale_c), col_offset=col_offset, strip_bytes=sb,
                codes=codes.data_ptr())
    return QCopy(d, codes)


def absmax(src, stream=None):
    """(a1) c = max |src| (float32 / complex64 viewed as pairs); returns a 1-element CUDA tensor."""
    _require_cuda(src)
    flat = torch.view_as_real(src) if src.is_complex() else src
    if not flat.is_contiguous():
        raise ValueError("absmax needs a contiguous tensor")
    out = torch.empty(1, dtype=torch.float32, device=src.device)
    check(load().iht_absmax(_ptr(flat), flat.numel(), _ptr(out), _stream(stream)), "iht_absmax")
    return out


def absmax_batched(src, stream=None):
    """(a1) per-row c_b = max |src[b]| of a (B, n) float32 / complex64 CUDA tensor; returns (B,) floats."""
    _require_cuda(src)
    flat = torch.view_as_real(src) if src.is_complex() else src
    if not flat.is_contiguous():
        raise ValueError("absmax_batched needs a contiguous tensor")
    B = flat.shape[0]
    out = torch.empty(B, dtype=torch.float32, device=src.device)
    check(load().iht_absmax_batched(_ptr(flat), flat.numel() // B, B, _ptr(out), _stream(stream)),
          "iht_absmax_batched")
    return out


def quantize(phi, bits, level_mode, seed, copy_ids, scale_c, row_offset=0, stream=None, col_offset=0):
    """(a2) quantise a (rows x cols) float32 or complex64 CUDA matrix into len(copy_ids)
    independent copies in one pass; returns a list of QCopy.  col_offset: global index of
    column 0 (column shards; a multiple of 16)."""
    _require_cuda(phi)
    planes = 2 if phi.is_complex() else 1
    rows, cols = phi.shape
    if phi.stride(1) != 1:
        raise ValueError("phi must be row-major (unit column stride)")
    copies = [new_copy(rows, cols, planes, bits, level_mode, seed, cid, scale_c, row_offset, phi.device,
                       col_offset=col_offset) for cid in copy_ids]
    arr = (IhtQmat * len(copies))(*[c.desc for c in copies])
    base = torch.view_as_real(phi) if planes == 2 else phi
    check(load().iht_quantize(_ptr(base), phi.stride(0), arr, len(copies), _stream(stream)), "iht_quantize")
    return copies


def quantize_rows(block, copies, row_begin, stream=None):
    """(a2) block-wise: quantise local rows [row_begin, row_begin + block.shape[0]) of existing
    copies (QCopy list sharing shape) from the CUDA block `block` (float32 / complex64)."""
    _require_cuda(block)
    arr = (IhtQmat * len(copies))(*[c.desc for c in copies])
    base = torch.view_as_real(block) if block.is_complex() else block
    check(load().iht_quantize_rows(_ptr(base), block.stride(0), arr, len(copies), row_begin, block.shape[0],
                                   _stream(stream)), "iht_quantize_rows")
    return copies


def quantize_vec(y, bits, level_mode, seed, c_dev, row_offset=0, with_codes=False, stream=None):
    """(a3) y-hat = Q(y) once; returns (yhat stacked float32, codes uint8 or None)."""
    _require_cuda(y, c_dev)
    planes = 2 if y.is_complex() else 1
    rows = y.shape[0]
    base = torch.view_as_real(y).contiguous() if planes == 2 else y.contiguous()
    yhat = torch.empty(vec_len(rows, planes), dtype=torch.float32, device=y.device)
    codes = torch.empty(planes * rows, dtype=torch.uint8, device=y.device) if with_codes else None
    check(load().iht_quantize_vec(_ptr(base), rows, row_offset, planes, bits, level_mode, seed, _ptr(c_dev),
                                  _ptr(yhat), _ptr(codes), _stream(stream)), "iht_quantize_vec")
    return yhat, codes


def quantize_vec_batched(Y, bits, level_mode, seed, c_dev, row_offset=0, with_codes=False, stream=None):
    """(a3) batched: Y (B, rows) float32 / complex64; snapshot b is column n = b of the
    observation matrix.  Returns (yhat (B, vec_len) float32, codes (B, planes*rows) or None)."""
    _require_cuda(Y, c_dev)
    planes = 2 if Y.is_complex() else 1
    B, rows = Y.shape
    base = torch.view_as_real(Y).contiguous() if planes == 2 else Y.contiguous()
    yhat = torch.empty((B, vec_len(rows, planes)), dtype=torch.float32, device=Y.device)
    codes = torch.empty((B, planes * rows), dtype=torch.uint8, device=Y.device) if with_codes else None
    check(load().iht_quantize_vec_batched(_ptr(base), rows, row_offset, planes, bits, level_mode, seed, _ptr(c_dev),
                                          B, _ptr(yhat), _ptr(codes), _stream(stream)), "iht_quantize_vec_batched")
    return yhat, codes


def forward_batched(F, x_idx, x_val, x_nnz, yhat, stream=None):
    """(a4) batched: x_idx / x_val (B, ldx), x_nnz (B,) int32, yhat (B, vec_len) or None
    (partial product of a column shard); returns r (B, vec_len)."""
    _require_cuda(x_idx, x_val, x_nnz)
    B, ldx = x_idx.shape
    r = torch.empty((B, vec_len(F.rows, F.planes)), dtype=torch.float32, device=x_idx.device)
    check(load().iht_forward_batched(ctypes.byref(F.desc), _ptr(x_idx), _ptr(x_val), _ptr(x_nnz), ldx, ldx, B,
                                     _ptr(yhat), _ptr(r), _stream(stream)), "iht_forward_batched")
    return r


def forward(F, x_idx, x_val, x_nnz, yhat, max_nnz=None, stream=None):
    """(a4) r = y-hat - Phi-hat_F x (support columns only); x_nnz is a 1-element int32 CUDA tensor."""
    _require_cuda(x_idx, x_val, x_nnz, yhat)
    max_nnz = x_idx.numel() if max_nnz is None else max_nnz
    r = torch.empty_like(yhat)
    lib = load()
    ws_bytes = lib.iht_forward_ws_bytes(ctypes.byref(F.desc), max_nnz)
    ws = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=yhat.device)   # arrival counters start at 0
    check(lib.iht_forward(ctypes.byref(F.desc), _ptr(x_idx), _ptr(x_val), _ptr(x_nnz), max_nnz, _ptr(yhat),
                          _ptr(r), _ptr(ws), ws_bytes, _stream(stream)), "iht_forward")
    return r


def adjoint(A, r, variant=0, stream=None, out=None):
    """(a5) g = Re(Phi-hat_A^H r) for all N columns (variant 0 = int8 MMA, 1 = FFMA)."""
    _require_cuda(r)
    lib = load()
    ws_bytes = lib.iht_adjoint_ws_bytes(ctypes.byref(A.desc))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=r.device)
    g = torch.empty(A.cols, dtype=torch.float32, device=r.device) if out is None else out
    check(lib.iht_adjoint(ctypes.byref(A.desc), _ptr(r), _ptr(g), variant, _ptr(ws), ws_bytes, _stream(stream)),
          "iht_adjoint")
    return g


def adjoint_batched(A, R, stream=None):
    """(a7) G = Re(Phi-hat_A^H R) for B snapshots at once (tcgen05 int8 GEMM).
    R: (B, vec_len) float32 CUDA tensor; returns G (B, N) float32."""
    _require_cuda(R)
    lib = load()
    B = R.shape[0]
    ws_bytes = lib.iht_adjoint_batched_ws_bytes(ctypes.byref(A.desc), B)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=R.device)
    G = torch.empty((B, A.cols), dtype=torch.float32, device=R.device)
    check(lib.iht_adjoint_batched(ctypes.byref(A.desc), _ptr(R), B, _ptr(G), _ptr(ws), ws_bytes, _stream(stream)),
          "iht_adjoint_batched")
    return G


def threshold(x_idx, x_val, x_nnz, g, mu, s, stream=None):
    """(a6) x <- H_s(x + mu g): returns (idx int32[s], val float32[s], nnz int32[1]) on the device."""
    _require_cuda(x_idx, x_val, x_nnz, g)
    lib = load()
    N = g.numel()
    ws_bytes = lib.iht_threshold_ws_bytes(N, s)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=g.device)
    oi = torch.empty(max(s, 1), dtype=torch.int32, device=g.device)
    ov = torch.empty(max(s, 1), dtype=torch.float32, device=g.device)
    on = torch.empty(1, dtype=torch.int32, device=g.device)
    check(lib.iht_threshold(_ptr(x_idx), _ptr(x_val), _ptr(x_nnz), _ptr(g), float(mu), s, N, _ptr(oi), _ptr(ov),
                            _ptr(on), _ptr(ws), ws_bytes, _stream(stream)), "iht_threshold")
    return oi, ov, on


def threshold_batched(x_idx, x_val, x_nnz, G, mu, s, col_offset=0, stream=None):
    """(a6) batched H_s per snapshot: x_idx / x_val (B, ldx) (global indices), x_nnz (B,),
    G (B, N) local gradients of columns [col_offset, col_offset + N).  Returns
    (idx (B, s), val (B, s), nnz (B,)) with global indices."""
    _require_cuda(x_idx, x_val, x_nnz, G)
    lib = load()
    B, N = G.shape
    ldx = x_idx.shape[1]
    ws_bytes = lib.iht_threshold_batched_ws_bytes(N, s, B)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=G.device)
    ldo = max(s, 1)
    oi = torch.empty((B, ldo), dtype=torch.int32, device=G.device)
    ov = torch.empty((B, ldo), dtype=torch.float32, device=G.device)
    on = torch.empty(B, dtype=torch.int32, device=G.device)
    check(lib.iht_threshold_batched(_ptr(x_idx), _ptr(x_val), _ptr(x_nnz), ldx, _ptr(G), float(mu), s, N, col_offset,
                                    B, _ptr(oi), _ptr(ov), ldo, _ptr(on), _ptr(ws), ws_bytes, _stream(stream)),
          "iht_threshold_batched")
    return oi, ov, on


def merge_candidates(cand_idx, cand_val, cand_nnz, s, stream=None):
    """Global H_s from per-shard lists: cand_idx / cand_val (P, B, s), cand_nnz (P, B)."""
    _require_cuda(cand_idx, cand_val, cand_nnz)
    P, B, _ = cand_idx.shape
    if cand_nnz.shape != (P, B):
        raise ValueError("cand_nnz must be (P, B)")
    # the C call takes one shard stride for all three arrays: repack into [P][idx | val | nnz]
    words = 2 * B * s + B
    pack = torch.empty((P, words), dtype=torch.int32, device=cand_idx.device)
    pack[:, :B * s] = cand_idx.reshape(P, B * s)
    pack[:, B * s:2 * B * s] = cand_val.reshape(P, B * s).view(torch.int32)
    pack[:, 2 * B * s:] = cand_nnz
    oi = torch.empty((B, max(s, 1)), dtype=torch.int32, device=cand_idx.device)
    ov = torch.empty((B, max(s, 1)), dtype=torch.float32, device=cand_idx.device)
    on = torch.empty(B, dtype=torch.int32, device=cand_idx.device)
    base = pack.data_ptr()
    check(load().iht_merge_candidates(ctypes.c_void_p(base), ctypes.c_void_p(base + 4 * B * s),
                                      ctypes.c_void_p(base + 8 * B * s), words, P, s, B, _ptr(oi), _ptr(ov), _ptr(on),
                                      _stream(stream)), "iht_merge_candidates")
    return oi, ov, on


@dataclass
class FreshPhi:
    """NEXT-2: the fp32 Phi (CUDA tensor kept alive here) from which copies are drawn on the fly."""
    desc: IhtFmat
    phi: torch.Tensor


def fresh_phi(phi, bits, level_mode, seed, scale_c, row_offset=0):
    """Describe a (rows x cols) float32 / complex64 row-major CUDA matrix for on-the-fly copies."""
    _require_cuda(phi)
    planes = 2 if phi.is_complex() else 1
    if phi.stride(1) != 1:
        raise ValueError("phi must be row-major (unit column stride)")
    base = torch.view_as_real(phi) if planes == 2 else phi
    rows, cols = phi.shape
    d = IhtFmat(rows=rows, cols=cols, row_offset=row_offset, ld=phi.stride(0), planes=planes, bits=bits,
                level_mode=level_mode, reserved=0, seed=seed, scale_c=float(scale_c), reserved2=0,
                phi=base.data_ptr())
    return FreshPhi(d, phi)


def adjoint_fresh(F, copy_id, r, stream=None):
    """g = Re(Phi-hat_k^H r) with copy k drawn on the fly (no stored codes)."""
    _require_cuda(r)
    lib = load()
    wsb = lib.iht_adjoint_fresh_ws_bytes(ctypes.byref(F.desc))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=r.device)
    g = torch.empty(F.desc.cols, dtype=torch.float32, device=r.device)
    check(lib.iht_adjoint_fresh(ctypes.byref(F.desc), copy_id, _ptr(r), _ptr(g), _ptr(ws), wsb, _stream(stream)),
          "iht_adjoint_fresh")
    return g


def forward_fresh(F, copy_id, x_idx, x_val, x_nnz, yhat, stream=None):
    """r = y-hat - Phi-hat_k x over the support of x, copy k drawn on the fly."""
    _require_cuda(x_idx, x_val, x_nnz, yhat)
    r = torch.empty_like(yhat)
    check(load().iht_forward_fresh(ctypes.byref(F.desc), copy_id, _ptr(x_idx), _ptr(x_val), _ptr(x_nnz),
                                   x_idx.numel(), _ptr(yhat), _ptr(r), _stream(stream)), "iht_forward_fresh")
    return r


def adjoint_radio(u, v, grid, r, bits=0, level_mode=0, seed=0, copy_id=0, scale_c=1.0, row_offset=0, stream=None):
    """NEXT-3: g = Re(Phi^H r) with the radio Phi computed on the fly from u, v (float64 CUDA
    tensors, baseline / lambda per visibility); bits > 0 quantises each entry in registers."""
    _require_cuda(u, v, r)
    from ._lib import IhtRadio
    if u.dtype != torch.float64 or v.dtype != torch.float64:
        raise ValueError("u, v must be float64")
    d = IhtRadio(nvis=u.numel(), row_offset=row_offset, grid=grid, bits=bits, level_mode=level_mode,
                 copy_id=copy_id, seed=seed, scale_c=float(scale_c), reserved=0, u=u.data_ptr(), v=v.data_ptr())
    g = torch.empty(grid * grid, dtype=torch.float32, device=r.device)
    check(load().iht_adjoint_radio(ctypes.byref(d), _ptr(r), _ptr(g), _stream(stream)), "iht_adjoint_radio")
    return g


class Comm:
    """NCCL communicator of libiht (iht_comm_*); unique id broadcast via torch.distributed."""

    def __init__(self, rank, world, device, group=None):
        import torch.distributed as dist
        lib = load()
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            check(lib.iht_comm_unique_id(ctypes.cast(uid, ctypes.c_void_p)), "iht_comm_unique_id")
        if world > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=group)
            ctypes.memmove(uid, obj[0], 128)
        h = ctypes.c_void_p()
        check(lib.iht_comm_create(rank, world, ctypes.cast(uid, ctypes.c_void_p), device, ctypes.byref(h)),
              "iht_comm_create")
        self.handle = h
        self.rank, self.world = rank, world

    def allreduce_(self, t, op_max=False, stream=None):
        check(load().iht_comm_allreduce(self.handle, _ptr(t), t.numel(), int(op_max), _stream(stream)),
              "iht_comm_allreduce")
        return t

    def reduce_scatter(self, t, stream=None):
        """Sum reduce-scatter of a contiguous float32 CUDA tensor of world * k elements:
        returns this rank's k summed elements."""
        assert t.dtype == torch.float32 and t.numel() % self.world == 0
        k = t.numel() // self.world
        out = torch.empty(k, dtype=t.dtype, device=t.device)
        check(load().iht_comm_reduce_scatter(self.handle, _ptr(t), _ptr(out), k, _stream(stream)),
              "iht_comm_reduce_scatter")
        return out

    def allgather(self, t, stream=None):
        """All-gather of a contiguous CUDA tensor: returns (world, *t.shape)."""
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        check(load().iht_comm_allgather(self.handle, _ptr(t), _ptr(out), t.numel() * t.element_size(),
                                        _stream(stream)), "iht_comm_allgather")
        return out

    def close(self):
        if self.handle:
            load().iht_comm_destroy(self.handle)
            self.handle = None


class Solver:
    """iht_solver_*: Algorithm 1 with fixed mu over a pool of quantised copies (CUDA graph).
    nrhs = B > 1: B observations sharing Phi (config 5); run() takes y of shape (B, rows)
    and the outputs are (B, s) / (B,)."""

    def __init__(self, pool, s, n_iter, mu, b_y, seed, level_mode=0, adjoint_variant=0, trace=False,
                 use_graph=True, comm=None, profile=False, nrhs=1, adaptive=False, c=1e-3, k=2.0, max_shrink=60,
                 fused=True):
        """pool: list of QCopy (stored copies), or a FreshPhi (NEXT-2: copies drawn on the fly,
        K = 2 n*).  fused: True = run the whole loop as one persistent kernel when the problem
        fits and is large enough to pay (iht_config.fused = 1), "force" = whenever it fits (2),
        False = per-step kernels (0)."""
        lib = load()
        self.pool = pool                     # keep the code / Phi tensors alive
        self.s, self.n_iter = s, n_iter
        self.mu, self.adaptive = float(mu), bool(adaptive)
        self.trace = trace
        self.nrhs = max(1, nrhs)
        cfg = IhtConfig(s=s, n_iter=n_iter, mu=float(mu), b_y=b_y, level_mode=level_mode,
                        adjoint_variant=adjoint_variant, seed=seed, trace=int(trace), use_graph=int(use_graph),
                        comm=comm.handle if comm is not None else None, profile=int(profile), nrhs=self.nrhs,
                        step_mode=int(adaptive), step_c=float(c), step_k=float(k), max_shrink=int(max_shrink),
                        fused=2 if fused == "force" else int(bool(fused)))
        h = ctypes.c_void_p()
        if isinstance(pool, FreshPhi):
            check(lib.iht_solver_create_fresh(ctypes.byref(pool.desc), ctypes.byref(cfg), ctypes.byref(h)),
                  "iht_solver_create_fresh")
            self.device = pool.phi.device
        else:
            arr = (IhtQmat * len(pool))(*[c.desc for c in pool])
            check(lib.iht_solver_create(arr, len(pool), ctypes.byref(cfg), ctypes.byref(h)), "iht_solver_create")
            self.device = pool[0].codes.device
        self.handle = h
        shape = (self.nrhs, max(s, 1)) if self.nrhs > 1 else (max(s, 1),)
        self.out_idx = torch.empty(shape, dtype=torch.int32, device=self.device)
        self.out_val = torch.empty(shape, dtype=torch.float32, device=self.device)
        self.out_nnz = torch.empty(self.nrhs, dtype=torch.int32, device=self.device)

    def run(self, y, stream=None):
        """Device y (float32 or complex64 CUDA tensor of this shard's rows): enqueue a solve;
        returns device (idx, val, nnz) tensors (valid after the stream reaches them)."""
        _require_cuda(y)
        base = torch.view_as_real(y) if y.is_complex() else y
        check(load().iht_solver_run(self.handle, _ptr(base), 0, _ptr(self.out_idx), _ptr(self.out_val),
                                    _ptr(self.out_nnz), _stream(stream)), "iht_solver_run")
        return self.out_idx, self.out_val, self.out_nnz

    def run_host(self, y_host, out_idx, out_val, out_nnz, stream=None):
        """Host-buffer end-to-end call (IHT_HOST_IO): y_host and outputs are (pinned) CPU tensors;
        the call copies in, solves, copies out and synchronises the stream."""
        base = torch.view_as_real(y_host) if y_host.is_complex() else y_host
        check(load().iht_solver_run(self.handle, _ptr(base), _lib.IHT_HOST_IO, _ptr(out_idx), _ptr(out_val),
                                    _ptr(out_nnz), _stream(stream)), "iht_solver_run")
        return out_idx, out_val, out_nnz

    def trace_arrays(self, stream=None):
        """Recorded iterates x^[2..n*+1]: (idx[n_iter, s], val[n_iter, s], nnz[n_iter]) CPU tensors
        (batched: [n_iter, B, s] and [n_iter, B])."""
        lead = (self.n_iter, self.nrhs) if self.nrhs > 1 else (self.n_iter,)
        idx = torch.empty(lead + (max(self.s, 1),), dtype=torch.int32)
        val = torch.empty(lead + (max(self.s, 1),), dtype=torch.float32)
        nnz = torch.empty(lead, dtype=torch.int32)
        check(load().iht_solver_trace(self.handle, _ptr(idx), _ptr(val), _ptr(nnz), _stream(stream)),
              "iht_solver_trace")
        return idx, val, nnz

    def buffers(self):
        a, b, c = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        check(load().iht_solver_buffers(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
              "iht_solver_buffers")
        return a.value, b.value, c.value

    def adjoint_times_ms(self):
        """Per-launch adjoint durations (ms) of the last run (profile=True), from CUDA events."""
        buf = (ctypes.c_float * self.n_iter)()
        check(load().iht_solver_adjoint_times(self.handle, ctypes.cast(buf, ctypes.c_void_p)),
              "iht_solver_adjoint_times")
        return list(buf)

    def steps(self, stream=None):
        """Adaptive step: accepted mu and shrink count per iteration of the last run, CPU tensors
        [n_iter] (batched: [n_iter, B])."""
        shape = (self.n_iter, self.nrhs) if self.nrhs > 1 else (self.n_iter,)
        mu = torch.empty(shape, dtype=torch.float32)
        sh = torch.empty(shape, dtype=torch.int32)
        check(load().iht_solver_steps(self.handle, _ptr(mu), _ptr(sh), _stream(stream)), "iht_solver_steps")
        return mu, sh

    def report(self, stream=None):
        """RecoveryReport of the last run (trace=True): a dict of numpy arrays
        [n_iter] (batched: [n_iter, B]) -- iter, mu, residual_norm (||y-hat - Phi-hat_{2n} x^[n]||,
        recomputed on the GPU from the recorded iterates), support_size, support_change,
        shrink_count.  Marshalling only: every number comes from iht_solver_report /
        iht_solver_steps."""
        shape = (self.n_iter, self.nrhs) if self.nrhs > 1 else (self.n_iter,)
        rn = torch.empty(shape, dtype=torch.float64)
        sz = torch.empty(shape, dtype=torch.int32)
        ch = torch.empty(shape, dtype=torch.int32)
        check(load().iht_solver_report(self.handle, _ptr(rn), _ptr(sz), _ptr(ch), _stream(stream)),
              "iht_solver_report")
        if self.adaptive:
            mu, sh = self.steps(stream)
            mu, sh = mu.numpy().astype(np.float64), sh.numpy()
        else:
            mu = np.full(shape, float(self.mu))
            sh = np.zeros(shape, np.int32)
        it = np.arange(1, self.n_iter + 1)
        if self.nrhs > 1:
            it = np.repeat(it[:, None], self.nrhs, axis=1)
        return {"iter": it, "mu": mu, "residual_norm": rn.numpy(), "support_size": sz.numpy(),
                "support_change": ch.numpy(), "shrink_count": sh}

    def report_csv(self, path, snapshot=0, stream=None):
        """Write the RecoveryReport as CSV (SPEC.md:234 columns), one row per iteration
        (batched: of one snapshot)."""
        rep = self.report(stream)
        cols = ["iter", "mu", "residual_norm", "support_size", "support_change", "shrink_count"]
        with open(path, "w") as f:
            f.write(",".join(cols) + "\n")
            for n in range(self.n_iter):
                row = [rep[c][n] if self.nrhs == 1 else rep[c][n, snapshot] for c in cols]
                f.write(f"{int(row[0])},{float(row[1])!r},{float(row[2])!r},{int(row[3])},{int(row[4])},{int(row[5])}\n")
        return rep

    def launches_per_run(self):
        return int(load().iht_solver_launches_per_run(self.handle))

    @property
    def fused(self):
        """True when the solve runs as the single fused persistent kernel."""
        return bool(load().iht_solver_fused(self.handle))

    def close(self):
        if self.handle:
            load().iht_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve(pool, y, s, n_iter, mu, b_y, seed, **kw):
    """One-shot iht_solve equivalent through the Solver object; returns CPU (idx, val)."""
    sol = Solver(pool, s, n_iter, mu, b_y, seed, **kw)
    idx, val, nnz = sol.run(y)
    torch.cuda.current_stream().synchronize()
    n = int(nnz.item())
    sol.close()
    if n < 0:
        raise _lib.IhtError(_lib.IHT_EDOMAIN, "iht_solver_run")
    return idx[:n].cpu(), val[:n].cpu()
