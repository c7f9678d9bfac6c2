#!/bin/bash
# r02 g01: all GPU tests (tightened parity + trajectories), smoke, default bench, reference arm
OUT=gpurun_out/r02g01; mkdir -p $OUT
nproc > $OUT/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=25 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/ref.err
