#!/bin/bash
# GPU suite against the bounds-checked build (IHT_LIB=checked): every hand-rolled pipeline's
# indices checked on the device, bounded mbarrier / grid-barrier waits (compute-sanitizer stand-in)
OUT=gpurun_out/r02g16; mkdir -p $OUT
IHT_LIB=checked timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_adaptive.py tests/test_gpu_fresh.py tests/test_gpu_radio.py tests/test_gpu_trajectory.py -m gpu -q -rf -p no:cacheprovider -k "not config3 and not config5" > $OUT/pytest_checked.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_checked.log
IHT_LIB=checked timeout 300 python scripts/r02/sanitize_cases.py all >> $OUT/pytest_checked.log 2>&1; echo "cases rc=$?" >> $OUT/pytest_checked.log
