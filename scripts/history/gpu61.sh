set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g61_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:adjoint_mma --launch-skip 300 -c 1 -o $OUT/g61_adj_c3 -f \
    python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/g61_full.log 2>&1
echo done
