set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g22_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for pr in 0 1 2 4 8 9 16; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 120 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g22_probe.log
for pr in 0 1 2 3; do echo "thr probe $pr: $(IHT_THR_PROBE=$pr timeout 120 python scripts/prof_parts.py 2>&1 | grep threshold | tr '\n' ' ')"; done >> $OUT/g22_probe.log
echo done
