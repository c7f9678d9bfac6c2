"""ctypes loader for libiht.so: the C ABI declared in include/iht.h.

Loads the in-tree library and declares every exported symbol's signature.  There
is no fallback: if the library (or a CUDA device, for compute calls) is missing,
the caller gets an exception.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libiht.so")

IHT_OK = 0
IHT_EINVAL = -1
IHT_EDOMAIN = -2
IHT_ECUDA = -3
IHT_ENCCL = -4
IHT_ENOMEM = -5
IHT_EUNSUPPORTED = -6
IHT_HOST_IO = 1

c_i32, c_i64, c_u64, c_f32, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_void_p
c_int = ctypes.c_int


class IhtQmat(ctypes.Structure):
    """Mirror of iht_qmat (include/iht.h)."""
    _fields_ = [
        ("rows", c_i64), ("cols", c_i64), ("row_offset", c_i64),
        ("planes", c_i32), ("bits", c_i32), ("level_mode", c_i32), ("copy_id", c_i32),
        ("seed", c_u64), ("scale_c", c_f32), ("col_offset", c_i32),
        ("strip_bytes", c_i64), ("codes", c_vp),
    ]


class IhtFmat(ctypes.Structure):
    """Mirror of iht_fmat (include/iht.h): the fp32 Phi that fresh copies are drawn from."""
    _fields_ = [
        ("rows", c_i64), ("cols", c_i64), ("row_offset", c_i64), ("ld", c_i64),
        ("planes", c_i32), ("bits", c_i32), ("level_mode", c_i32), ("reserved", c_i32),
        ("seed", c_u64), ("scale_c", c_f32), ("reserved2", c_i32), ("phi", c_vp),
    ]


class IhtRadio(ctypes.Structure):
    """Mirror of iht_radio (include/iht.h): the on-the-fly radio Phi (NEXT-3)."""
    _fields_ = [
        ("nvis", c_i64), ("row_offset", c_i64), ("grid", c_i32), ("bits", c_i32), ("level_mode", c_i32),
        ("copy_id", c_i32), ("seed", c_u64), ("scale_c", c_f32), ("reserved", c_i32), ("u", c_vp), ("v", c_vp),
    ]


class IhtConfig(ctypes.Structure):
    """Mirror of iht_config (include/iht.h)."""
    _fields_ = [
        ("s", c_i32), ("n_iter", c_i32), ("mu", c_f32), ("b_y", c_i32), ("level_mode", c_i32),
        ("adjoint_variant", c_i32), ("seed", c_u64), ("trace", c_i32), ("use_graph", c_i32),
        ("comm", c_vp), ("profile", c_i32), ("nrhs", c_i32),
        ("step_mode", c_i32), ("step_c", c_f32), ("step_k", c_f32), ("max_shrink", c_i32),
        ("fused", c_i32),
    ]


# name -> (restype, argtypes); every function include/iht.h declares
SIGNATURES = {
    "iht_strerror": (ctypes.c_char_p, [c_int]),
    "iht_abi_version": (c_int, []),
    "iht_last_cuda_error": (ctypes.c_char_p, []),
    "iht_rows_pad": (c_i64, [c_i64]),
    "iht_strip_bytes": (c_i64, [c_i64, c_int, c_int]),
    "iht_qmat_bytes": (c_i64, [c_i64, c_i64, c_int, c_int]),
    "iht_vec_len": (c_i64, [c_i64, c_int]),
    "iht_absmax": (c_int, [c_vp, c_i64, c_vp, c_vp]),
    "iht_absmax_batched": (c_int, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "iht_quantize": (c_int, [c_vp, c_i64, ctypes.POINTER(IhtQmat), c_int, c_vp]),
    "iht_quantize_rows": (c_int, [c_vp, c_i64, ctypes.POINTER(IhtQmat), c_int, c_i64, c_i64, c_vp]),
    "iht_quantize_vec": (c_int, [c_vp, c_i64, c_i64, c_int, c_int, c_int, c_u64, c_vp, c_vp, c_vp, c_vp]),
    "iht_quantize_vec_batched": (c_int, [c_vp, c_i64, c_i64, c_int, c_int, c_int, c_u64, c_vp, c_i32, c_vp, c_vp,
                                         c_vp]),
    "iht_forward_ws_bytes": (c_i64, [ctypes.POINTER(IhtQmat), c_i32]),
    "iht_forward": (c_int, [ctypes.POINTER(IhtQmat), c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "iht_forward_batched": (c_int, [ctypes.POINTER(IhtQmat), c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp,
                                    c_vp]),
    "iht_adjoint_ws_bytes": (c_i64, [ctypes.POINTER(IhtQmat)]),
    "iht_adjoint": (c_int, [ctypes.POINTER(IhtQmat), c_vp, c_vp, c_int, c_vp, c_i64, c_vp]),
    "iht_adjoint_batched_ws_bytes": (c_i64, [ctypes.POINTER(IhtQmat), c_i32]),
    "iht_adjoint_batched": (c_int, [ctypes.POINTER(IhtQmat), c_vp, c_i32, c_vp, c_vp, c_i64, c_vp]),
    "iht_threshold_ws_bytes": (c_i64, [c_i64, c_i32]),
    "iht_threshold": (c_int, [c_vp, c_vp, c_vp, c_vp, c_f32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "iht_adjoint_fresh_ws_bytes": (c_i64, [ctypes.POINTER(IhtFmat)]),
    "iht_adjoint_fresh": (c_int, [ctypes.POINTER(IhtFmat), c_i32, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "iht_forward_fresh": (c_int, [ctypes.POINTER(IhtFmat), c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "iht_solver_create_fresh": (c_int, [ctypes.POINTER(IhtFmat), ctypes.POINTER(IhtConfig), ctypes.POINTER(c_vp)]),
    "iht_adjoint_radio": (c_int, [ctypes.POINTER(IhtRadio), c_vp, c_vp, c_vp]),
    "iht_threshold_batched_ws_bytes": (c_i64, [c_i64, c_i32, c_i32]),
    "iht_threshold_batched": (c_int, [c_vp, c_vp, c_vp, c_i32, c_vp, c_f32, c_i32, c_i64, c_i64, c_i32, c_vp, c_vp,
                                      c_i32, c_vp, c_vp, c_i64, c_vp]),
    "iht_merge_candidates": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "iht_comm_unique_id": (c_int, [c_vp]),
    "iht_comm_create": (c_int, [c_int, c_int, c_vp, c_int, ctypes.POINTER(c_vp)]),
    "iht_comm_destroy": (c_int, [c_vp]),
    "iht_comm_allreduce": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp]),
    "iht_comm_allgather": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "iht_comm_reduce_scatter": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "iht_solver_create": (c_int, [ctypes.POINTER(IhtQmat), c_int, ctypes.POINTER(IhtConfig), ctypes.POINTER(c_vp)]),
    "iht_solver_destroy": (c_int, [c_vp]),
    "iht_solver_run": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp]),
    "iht_solver_trace": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "iht_solver_buffers": (c_int, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    "iht_solver_adjoint_times": (c_int, [c_vp, c_vp]),
    "iht_solver_launches_per_run": (c_i64, [c_vp]),
    "iht_solver_fused": (c_int, [c_vp]),
    "iht_solver_steps": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "iht_solver_report": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "iht_solve": (c_int, [ctypes.POINTER(IhtQmat), c_int, ctypes.POINTER(IhtConfig), c_vp, c_int, c_vp, c_vp, c_vp, c_vp]),
}

_lib = None


class IhtError(RuntimeError):
    def __init__(self, status, where):
        lib = load()
        msg = lib.iht_strerror(status).decode()
        if status == IHT_ECUDA:
            msg += " [" + (lib.iht_last_cuda_error() or b"").decode() + "]"
        super().__init__(f"{where}: {msg}")
        self.status = status


def load(path=None):
    """Load libiht.so (build it first with paper_1802_04907_b200.build).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None and os.environ.get("IHT_LIB") == "checked":      # bounds-checked build (debug)
        path = os.path.join(os.path.dirname(LIB_PATH), "libiht_checked.so")
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libiht.so not built at {path}; run `python -m paper_1802_04907_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status, where):
    if status != IHT_OK:
        raise IhtError(status, where)
    return status
