set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g12_build.log 2>&1
timeout 600 python scripts/prof_parts.py > $OUT/g12_parts.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:forward_kernel -s 5 -c 1 -o $OUT/g12_fwd python scripts/prof_parts.py c5 > /dev/null 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:thr_cluster -s 5 -c 1 -o $OUT/g12_thr python scripts/prof_parts.py c5 > /dev/null 2>&1
for pr in 0 25; do echo "probe $pr: $(IHT_BATCHED_PROBE=$pr timeout 300 python scripts/prof_batched.py 2>&1 | tail -1)"; done > $OUT/g12_probe.log
echo done
