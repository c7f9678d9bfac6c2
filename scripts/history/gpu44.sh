set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g44_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for pr in 64 80 96; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 60 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g44_probe.log
IHT_BATCHED_PROBE=112 timeout 60 python scripts/prof_batched.py > $OUT/g44_tl96.log 2>&1
echo done
