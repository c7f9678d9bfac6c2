set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g67_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for cfg in "2 1" "2 2" "2 4" "3 2" "3 4" "3 8"; do set -- $cfg
IHT_THR_CL=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_cluster --launch-skip 600 -c 3 --csv \
    --log-file $OUT/g67_thr_c$1_cl$2.csv python bench.py --config $1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "c$1 cl$2 bench: $(IHT_THR_CL=$2 timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')" >> $OUT/g67_bench.log
done
echo done
