#!/usr/bin/env python
"""Write tests/golden/config4_scale.json: the global quantiser scale c_Phi of BASELINE
config 4 (65536 x 262144 Gaussian), computed by the ORACLE only.

c_Phi = max over all components |Phi| ("c_v is the maximum value of the
components of v in magnitude"; reading c3) -- oracle.quantize.scale_c applied to every
row block of the counter-based input matrix (workloads.gen), max-combined.  Calls only
oracle/ and workloads/ (never the CUDA path).  About 17e9 entries: run with all cores.

    python scripts/golden_config4.py [--procs 8]
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

M, N = 65536, 262144
BLOCK = 128


def block_max(r0):
    import numpy as np
    from oracle import quantize as Q
    from workloads import gen as G
    key = G.derive_key(4, 1)
    sd = 1.0 / np.sqrt(M)
    return float(Q.scale_c(G.gaussian_block(key, N, r0, BLOCK, 0, N, sd)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    args = ap.parse_args()
    t0 = time.time()
    with Pool(args.procs) as pool:
        maxima = pool.map(block_max, range(0, M, BLOCK), chunksize=4)
    c = max(maxima)
    out = {
        "config": 4, "M": M, "N": N,
        "c_phi": c, "c_phi_hex": float(c).hex(),
        "source": "oracle.quantize.scale_c over workloads.gen.gaussian_block row blocks (scripts/golden_config4.py)",
        "citation": "P:686 (supp. Lemma 3: c_v = max component magnitude); DESIGN.md reading c3",
        "seconds": round(time.time() - t0, 1),
    }
    path = os.path.join(ROOT, "tests", "golden", "config4_scale.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
