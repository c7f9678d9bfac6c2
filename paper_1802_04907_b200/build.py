"""Build libiht.so (and the workload generator libihtgen.so) in-tree with nvcc for sm_100a.

    python -m paper_1802_04907_b200.build [--force]

Every .cu is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
and linked into a shared library next to this file (the .so travels to the GPU
box with the gpurun snapshot; it is git-ignored).
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libiht.so")
# checked variant (-DIHT_CHECKS): device-side bounds checks on every hand-rolled pipeline's
# indices and bounded mbarrier / grid-barrier waits that trap instead of hanging -- the
# stand-in for compute-sanitizer, which is closed on this GPU pool.  Loaded with IHT_LIB=checked.
LIB_CHECKED = os.path.join(HERE, "libiht_checked.so")
BUILD_CHECKED = os.path.join(HERE, "_build_checked")
GEN_SRC = os.path.join(ROOT, "workloads", "csrc", "gen.cu")
GEN_LIB = os.path.join(ROOT, "workloads", "libihtgen.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc():
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found")
    return exe


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    hs += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, verbose, extra=()):
    cmd = [nvcc(), *ARCH, *FLAGS, *extra, "-I", INCLUDE, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    log = obj + ".ptxas.txt"
    with open(log, "w") as f:      # register / spill / smem report (compile times dropped: stable diffs)
        f.write("".join(l for l in res.stderr.splitlines(True) if "Compile time" not in l))
    if verbose:
        print(f"[build] {os.path.basename(src)}", file=sys.stderr)
    return obj


def _build_lib(lib, bdir, extra, force, verbose):
    os.makedirs(bdir, exist_ok=True)
    srcs = _sources()
    hdrs = _headers()
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for s in srcs:
            o = os.path.join(bdir, os.path.basename(s)[:-3] + ".o")
            objs.append(o)
            if force or _stale(o, [s, *hdrs]):
                jobs.append(ex.submit(_compile, s, o, verbose, extra))
        for j in jobs:
            j.result()
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-ldl"]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
        if verbose:
            print(f"[build] linked {lib}", file=sys.stderr)


def build(force=False, verbose=True, checked=True):
    """Compile libiht.so (and libiht_checked.so) and libihtgen.so if any source is newer."""
    _build_lib(LIB, BUILD, (), force, verbose)
    if checked:
        _build_lib(LIB_CHECKED, BUILD_CHECKED, ("-DIHT_CHECKS",), force, verbose)
    if force or _stale(GEN_LIB, [GEN_SRC]):
        cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", GEN_SRC, "-o", GEN_LIB]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {GEN_SRC}:\n{res.stderr}")
        if verbose:
            print(f"[build] linked {GEN_LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
