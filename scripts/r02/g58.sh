#!/bin/bash
# r02 g58: full GPU suite, smoke, default bench (config 4, full contract), configs 2/3/5 benches,
# config-5 launch list -- bounded select with the in-CTA full select (512 threads)
OUT=gpurun_out/r02g58; mkdir -p $OUT
timeout 1700 python -m pytest tests -m gpu -q -x -rf --durations=15 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
for c in 5 2 3; do IHT_BOUNDED_STATS=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $OUT/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c5.log 2>&1
