#!/bin/bash
OUT=gpurun_out/r02g23; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "adjoint or teacher or free_running" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for b in 2 4; do timeout 600 python bench.py --bits $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c4_b$b.json 2> $OUT/bench_c4_b$b.err; done
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
