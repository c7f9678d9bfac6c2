set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g97_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for cfg in "2 4" "2 8" "2 4" "2 8" "1 1" "1 2"; do set -- $cfg
echo "c$1 cl$2 bench: $(IHT_THR_CL=$2 timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')" >> $OUT/g97.log
done
echo done
