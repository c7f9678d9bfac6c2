set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g83_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for cl in 2 4; do
echo "CL=$cl bench: $(IHT_THR_CL=$cl timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')" >> $OUT/g83.log
IHT_THR_CL=$cl timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:thr_cluster --launch-skip 650 -c 3 --csv \
    --log-file $OUT/g83_thr_cl$cl.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
echo done
