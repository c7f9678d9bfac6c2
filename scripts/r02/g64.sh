#!/bin/bash
# r02 g64 final validation: full GPU suite, smoke, default bench (config 4, full contract), configs
# 5/2/3/1, the reference (oracle) arm, config-4 launch list
OUT=gpurun_out/r02g64; mkdir -p $OUT
timeout 1700 python -m pytest tests -m gpu -q -x -rf --durations=15 -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
for c in 5 2 3 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c4.log 2>&1
