set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g59_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:adjoint_mma --launch-skip 300 -c 1 -o $OUT/g59_adj_c3 -f \
    python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/g59_full.log 2>&1
for kr in 1024 2048 4608; do
IHT_ADJ_KR=$kr timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:adjoint_mma --launch-skip 300 -c 3 --csv \
    --log-file $OUT/g59_kr$kr.csv python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
echo done
