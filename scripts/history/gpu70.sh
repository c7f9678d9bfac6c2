set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g70_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for c in 2 3; do for pr in 0 10; do
IHT_THR_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_cluster --launch-skip 750 -c 3 --csv \
    --log-file $OUT/g70_thr_c${c}_p$pr.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "c$c p$pr bench: $(IHT_THR_PROBE=$pr timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')" >> $OUT/g70_bench.log
done; done
echo done
