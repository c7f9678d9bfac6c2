"""The C-ABI library loads on CPU and exports every symbol include/iht.h declares
(no compute calls without a GPU); host-side argument checks answer without CUDA."""
import ctypes
import os
import re

import pytest

from paper_1802_04907_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iht.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^IHT_API\s+[\w\s\*]*?\b(iht_\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1802_04907_b200 import build
        build.build(verbose=False)
    return _lib.load()


def test_header_declares_the_boundary():
    names = declared()
    for core in ["iht_quantize", "iht_forward", "iht_adjoint", "iht_threshold", "iht_solve", "iht_absmax",
                 "iht_quantize_vec", "iht_solver_create", "iht_solver_run"]:
        assert core in names
    assert len(names) >= 25


def test_every_declared_symbol_is_exported_and_bound(lib):
    for name in declared():
        assert hasattr(lib, name), name                 # dlsym succeeds
        assert name in _lib.SIGNATURES, name            # the binding declares it


def test_no_undeclared_signature():
    assert set(_lib.SIGNATURES) == set(declared())


def test_sizes_and_strings(lib):
    assert lib.iht_abi_version() == 3
    assert lib.iht_rows_pad(1) == 256 and lib.iht_rows_pad(256) == 256 and lib.iht_rows_pad(257) == 512
    assert lib.iht_strip_bytes(65536, 1, 4) == 32768            # config 4: 32 KiB strips
    assert lib.iht_strip_bytes(4096, 1, 2) == 1024              # config 2
    assert lib.iht_strip_bytes(2304, 2, 2) == 1152              # config 3 (complex, 2 planes)
    assert lib.iht_qmat_bytes(65536, 262144, 1, 4) == 8 * 2 ** 30
    assert lib.iht_vec_len(2304, 2) == 4608
    assert lib.iht_strip_bytes(10, 1, 3) == -1
    assert b"EINVAL" in lib.iht_strerror(-1)
    assert b"EDOMAIN" in lib.iht_strerror(-2)


def test_host_side_validation_without_gpu(lib):
    c = ctypes.c_void_p
    assert lib.iht_absmax(c(0), -1, c(0), c(0)) == _lib.IHT_EINVAL
    assert lib.iht_quantize(c(0), 0, None, 0, c(0)) == _lib.IHT_EINVAL
    q = _lib.IhtQmat(rows=10, cols=10, planes=1, bits=3, strip_bytes=0, codes=None)
    assert lib.iht_adjoint(ctypes.byref(q), c(16), c(16), 0, c(0), 0, c(0)) == _lib.IHT_EINVAL
    assert lib.iht_threshold(c(0), c(0), c(0), c(0), 1.0, -1, 10, c(0), c(0), c(0), c(0), 0, c(0)) == _lib.IHT_EINVAL
    assert lib.iht_solver_create(None, 0, None, None) == _lib.IHT_EINVAL
    assert lib.iht_solver_report(None, c(16), c(16), c(16), c(0)) == _lib.IHT_EINVAL   # RecoveryReport: NULL solver
    # batched entry points (config 5) validate on the host too
    assert lib.iht_absmax_batched(c(16), 4, 0, c(16), c(0)) == _lib.IHT_EINVAL
    assert lib.iht_forward_batched(None, c(0), c(0), c(0), 0, 0, 1, c(0), c(0), c(0)) == _lib.IHT_EINVAL
    assert lib.iht_threshold_batched(c(0), c(0), c(16), 4, c(16), 1.0, 8, 100, 0, 2, c(16), c(16), 4, c(16),
                                     c(16), 1 << 20, c(0)) == _lib.IHT_EINVAL          # ldo < s
    assert lib.iht_threshold_batched_ws_bytes(1000, 4, 3) == 3 * lib.iht_threshold_batched_ws_bytes(1000, 4, 1)
    assert lib.iht_merge_candidates(c(16), c(16), c(16), 20000, 2, 5000, 1, c(16), c(16), c(16), c(0)) == \
        _lib.IHT_EUNSUPPORTED                                                          # P s > 8192
    q = _lib.IhtQmat(rows=256, cols=64, planes=1, bits=2, strip_bytes=64, codes=16)
    assert lib.iht_adjoint_batched(ctypes.byref(q), c(16), 3, c(16), c(16), 0, c(0)) == \
        _lib.IHT_EINVAL                                                                # workspace too small
    assert lib.iht_adjoint_batched_ws_bytes(ctypes.byref(q), 3) == lib.iht_adjoint_batched_ws_bytes(ctypes.byref(q), 8)
    big = _lib.IhtQmat(rows=1 << 20, cols=64, planes=2, bits=8, strip_bytes=2 * (1 << 20), codes=16)
    assert lib.iht_adjoint_batched(ctypes.byref(big), c(16), 8, c(16), c(16), 1 << 40, c(0)) == \
        _lib.IHT_EUNSUPPORTED                                                          # int32 accumulator bound


def _loop_bodies(obj, kernel_substr):
    """Instruction counts of the backward-branch loop bodies of the kernels whose mangled name
    contains kernel_substr, from cuobjdump -sass of the built object."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", obj], capture_output=True, text=True).stdout
    res = {}
    for f in re.split(r"\n\s*Function : ", out)[1:]:
        name = f.split("\n")[0].strip()
        if kernel_substr not in name:
            continue
        ins = [(int(m.group(1), 16), m.group(2)) for m in
               (re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l) for l in f.split("\n")) if m]
        for a, t in ins:
            tgt = re.search(r"BRA(?:\.\w+)?\s.*?0x([0-9a-f]+)", t)
            if tgt and int(tgt.group(1), 16) < a:
                res.setdefault(name, []).append(sum(1 for x, _ in ins if int(tgt.group(1), 16) <= x <= a))
    return res


def test_fresh_alu_roofline_constants_match_sass():
    """bench.py's NEXT-2 ALU roofline uses the SASS instruction count of adjoint_fresh_kernel's
    main loop per component; it must describe the library as built."""
    import importlib.util
    obj = os.path.join(ROOT, "paper_1802_04907_b200", "_build", "iht_fresh.o")
    if not os.path.exists(obj):
        from paper_1802_04907_b200 import build
        build.build(verbose=False)
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    bodies = _loop_bodies(obj, "adjoint_fresh_kernel")
    for planes, comps in ((1, 16), (2, 32)):
        name = [n for n in bodies if f"adjoint_fresh_kernelILi{planes}E" in n]
        assert name, bodies.keys()
        body = max(bodies[name[0]])                     # the unrolled 4-row main loop
        assert abs(body / comps - bench.FRESH_INST_PER_COMPONENT[planes]) <= 0.03 * body / comps, (planes, body)
