set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g8_build.log 2>&1
for pr in 0 9 25 16 2; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 300 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g8_probe.log
for b in 4 8; do echo "$(timeout 300 python scripts/prof_batched.py 64 $b 2>&1 | tail -1)"; done >> $OUT/g8_probe.log
echo done
