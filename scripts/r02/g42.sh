#!/bin/bash
# re-entry check (session 3): full GPU suite, smoke, bench configs 1-5 at HEAD + config-4 launch list
OUT=gpurun_out/r02g42; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=30 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
for c in 1 2 3 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_c4.csv $SHORT > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
