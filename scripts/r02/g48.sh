#!/bin/bash
# adjoint prologue (b >= 4 whole lane chunks, b = 2 item-wise) timings; full GPU suite; smoke; config-4 bench
OUT=gpurun_out/r02g48; mkdir -p $OUT
for b in 4 2; do timeout 120 python scripts/r02/adj_c4.py $b >> $OUT/adj.log 2>&1; done
timeout 1700 python -m pytest tests -m gpu -q -x -rf --durations=15 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
