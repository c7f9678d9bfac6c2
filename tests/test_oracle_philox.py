"""Pin oracle/philox.py against cuRAND's own Philox4x32-10 (not against itself).

The CUDA toolkit header curand_philox4x32_x.h implements curand_Philox4x32_10
with a host branch for mulhilo32; tests/pins/curand_philox_host.cpp compiles it
for the host with g++, so the pin runs on CPU.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle.philox import philox4x32_10

PIN_SRC = os.path.join(os.path.dirname(__file__), "pins", "curand_philox_host.cpp")
CUDA_INC = "/usr/local/cuda/include"


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    if shutil.which("g++") is None or not os.path.exists(os.path.join(CUDA_INC, "curand_philox4x32_x.h")):
        pytest.skip("g++ or CUDA headers missing")
    exe = str(tmp_path_factory.mktemp("pin") / "curand_philox_host")
    subprocess.run(["g++", "-O1", "-I", CUDA_INC, PIN_SRC, "-o", exe], check=True)
    return exe


def _run(exe, rows):
    inp = "\n".join(" ".join("%x" % v for v in r) for r in rows) + "\n"
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout
    return [tuple(int(t, 16) for t in line.split()) for line in out.strip().splitlines()]


def test_philox_matches_curand_on_random_grid(curand_host):
    rng = np.random.default_rng(1234)
    rows = rng.integers(0, 2 ** 32, size=(2000, 6), dtype=np.uint64).tolist()
    # structured counters as the quantiser uses them: (n>>2, m, copy, plane<<8|tag)
    for g in (0, 1, 4095):
        for m in (0, 1, 65535):
            for copy in (0, 1, 399):
                for pt in (0, 1, 256, 257):
                    rows.append([g, m, copy, pt, 0x90700 + 4, 0x180])
    rows += [[0] * 6, [0xFFFFFFFF] * 6]
    ref = _run(curand_host, rows)
    arr = np.array(rows, dtype=np.uint64)
    got = []
    for r in rows:
        w = philox4x32_10(r[0], r[1], r[2], r[3], r[4], r[5])
        got.append(tuple(int(v) for v in w))
    assert got == ref
    # vectorised path (array counters, shared key) equals the scalar path
    keyed = arr[arr[:, 4] == 0x90704]
    w = philox4x32_10(keyed[:, 0], keyed[:, 1], keyed[:, 2], keyed[:, 3], 0x90704, 0x180)
    vec = list(zip(*(x.tolist() for x in w)))
    scal = [tuple(int(v) for v in philox4x32_10(*r[:4], 0x90704, 0x180)) for r in keyed.tolist()]
    assert vec == scal
