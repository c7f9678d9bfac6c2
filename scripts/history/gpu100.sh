set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g100_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
TAG=r01g_c3
C3="python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $C3 > $OUT/${TAG}_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/${TAG}_launches.csv $C3 > /dev/null 2>&1
timeout 900 $C3 > /dev/null 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:adjoint_mma -s 300 -c 1 -o $OUT/${TAG}_adjoint $C3 > $OUT/${TAG}_full.log 2>&1
echo done
