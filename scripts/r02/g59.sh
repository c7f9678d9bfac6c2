#!/bin/bash
# forward_kernel: the first staging round's x slots requested with nnz (one round trip fewer);
# forward / batched parity; config-5 in-graph costs (the forward / limb kernel launched twice);
# config-4 forward time (L2 flushed) and bench
OUT=gpurun_out/r02g59; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -m gpu -q -x -rf -k "forward or batched" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > $OUT/c5.json 2> $OUT/c5.err
IHT_DUP_FWD=1 timeout 600 $B > $OUT/c5_dupfwd.json 2> $OUT/c5_dupfwd.err
IHT_DUP_LIMBS=1 timeout 600 $B > $OUT/c5_duplimbs.json 2> $OUT/c5_duplimbs.err
timeout 120 python scripts/r02/fwd_layout.py hoist > $OUT/fwd_c4.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c4.json 2> $OUT/c4.err
