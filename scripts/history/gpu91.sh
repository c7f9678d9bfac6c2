set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g91_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/g91_tests.log 2>&1; echo "tests rc=$?" >> $OUT/g91_tests.log
for c in 1 2 3 5; do for f in 1 0; do
echo "c$c fuse$f: $(IHT_FUSE_FWD=$f timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>$OUT/g91_c${c}_f$f.err | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["gpu_launches"], d["result"]["support_size"] if isinstance(d["result"]["support_size"], int) else min(d["result"]["support_size"]))')" >> $OUT/g91_bench.log
done; done
echo done
