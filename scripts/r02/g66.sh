#!/bin/bash
# r02 g66: full GPU suite + smoke after the fused count criterion; benches configs 2/3/4/5
OUT=gpurun_out/r02g66; mkdir -p $OUT
timeout 1700 python -m pytest tests -m gpu -q -x -rf --durations=10 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for c in 2 3 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
