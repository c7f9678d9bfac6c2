#!/bin/bash
OUT=gpurun_out/r02g24; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -rf -k "threshold or gridsel or config4" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
IHT_THR_MULTI=2 timeout 300 python scripts/r02/c4_parts.py threshold >> $OUT/parts.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
